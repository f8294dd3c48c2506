#!/bin/bash
# A/B: longest-first panel order vs natural order (SGTK_PANEL_ORDER=natural)
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -k "gemm or configs or multigpu or sddmm" > gpurun_out/ab_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/ab_tests.log
for o in natural lpt natural lpt; do
  if [ $o = natural ]; then export SGTK_PANEL_ORDER=natural; else unset SGTK_PANEL_ORDER; fi
  python bench.py --no-cpu --steps 20 > gpurun_out/ab_$o.json 2>/dev/null
  python bench.py --no-cpu --steps 20 --workload proteins-gcn > gpurun_out/ab_p_$o.json 2>/dev/null
  python -c "
import json; a=json.loads(open('gpurun_out/ab_$o.json').read().strip().splitlines()[-1]); b=json.loads(open('gpurun_out/ab_p_$o.json').read().strip().splitlines()[-1])
print('$o', 'agnn', a['value'], a['kernels_ms']['agnn_panel_layer'], a['kernels_ms']['panel_dense_part'], 'sddmm', a['kernels_ms']['sddmm'], 'gcn', b['value'], b['kernels_ms']['spmm'])"
done
