#!/bin/bash
mkdir -p gpurun_out
for wl in pubmed-agnn reddit-agnn cora-gcn proteins-gcn; do
  for g in "" "--cuda-graph"; do
    python bench.py --workload $wl --no-cpu --steps 20 $g > gpurun_out/gab.json 2>gpurun_out/gab.err || tail -5 gpurun_out/gab.err
    python -c "
import json; d=json.loads(open('gpurun_out/gab.json').read().strip().splitlines()[-1])
print('$wl', '$g', d['value'], d['ms_per_step'], d['details'].get('cuda_graph') is not None, d['e2e']['value'])"
  done
done
