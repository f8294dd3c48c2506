#!/bin/bash
tag=${1:-r2}
mkdir -p gpurun_out
python tools/sddmm_bench.py tf32 10
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${tag}_sddmm_launches.csv python tools/sddmm_bench.py tf32 2 > /dev/null 2>&1
grep -E "sddmm|yprep" gpurun_out/${tag}_sddmm_launches.csv | awk -F'","' '{print $5, $NF}' | tail -8
ncu --set full --metrics sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --import-source on -k regex:"sddmm_dense|sddmm_sparse" -s 2 -c 2 -o gpurun_out/${tag}_sddmm python tools/sddmm_bench.py tf32 1 > /dev/null 2>&1
echo done
