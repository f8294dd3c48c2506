python tools/sddmm_bench.py tf32 10
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"sddmm_dense" -s 2 -c 1 -o gpurun_out/s4_sddmm python tools/sddmm_bench.py tf32 1 > /dev/null 2>&1
ls gpurun_out | grep s4
