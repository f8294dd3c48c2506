#!/bin/bash
# Round profile: bench line (tf32 + fp32), kernel launch list, one ncu --set full
# capture per top kernel.  Usage: bash tools/profile_round.sh <tag>
tag=${1:-r1}
mkdir -p gpurun_out
python bench.py --steps 10 --warmup 3 --precision tf32 > gpurun_out/bench_${tag}_tf32.json 2> gpurun_out/bench_${tag}_tf32.err
python bench.py --steps 10 --warmup 3 --precision fp32 --no-cpu > gpurun_out/bench_${tag}_fp32.json 2> gpurun_out/bench_${tag}_fp32.err
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_${tag}.csv \
    python bench.py --steps 2 --warmup 1 --no-cpu --precision tf32 > /dev/null 2>&1
ncu --set full --clock-control none --import-source on -k regex:"agnn_fused_kernel|gemm_tc05_kernel|spmm_kernel|sddmm_kernel" -c 4 \
    -o gpurun_out/prof_${tag} python bench.py --steps 1 --warmup 1 --no-cpu --precision tf32 > /dev/null 2>&1
echo done
