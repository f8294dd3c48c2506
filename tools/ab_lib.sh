#!/bin/bash
# A/B of a variant library against the default build on the bench:
#   bash tools/ab_lib.sh <variant name> [bench args]
v=$1; shift
mkdir -p gpurun_out
for r in 1 2; do
  for which in default $v; do
    if [ $which = default ]; then unset SGTK_LIB; else export SGTK_LIB=$PWD/variants/libsgtk_$v.so; fi
    python bench.py --no-cpu --steps 20 "$@" > gpurun_out/ab.json 2>gpurun_out/ab.err || tail -3 gpurun_out/ab.err
    python -c "
import json; d=json.loads(open('gpurun_out/ab.json').read().strip().splitlines()[-1]); k=d['kernels_ms']
print('$which', d['value'], {x: k[x] for x in k if x in ('agnn_panel_layer','panel_dense_part','panel_sparse_part','spmm','sddmm')})"
  done
done
