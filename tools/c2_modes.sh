#!/bin/bash
mkdir -p gpurun_out
for m in auto panel fused; do
  for g in "" "--no-cuda-graph"; do
    python bench.py --workload pubmed-agnn --mode $m --no-cpu --steps 50 $g > gpurun_out/c2.json 2>/dev/null
    python -c "
import json; d=json.loads(open('gpurun_out/c2.json').read().strip().splitlines()[-1]); k=d['kernels_ms']
print('$m', '$g', d['value'], d['details']['mode_resolved'], k.get('agnn_panel_layer'), k.get('agnn_fused_kernel'))"
  done
done
python -m pytest tests/test_gpu_fullsize.py -q -k "reference_tf32" 2>&1 | tail -2
