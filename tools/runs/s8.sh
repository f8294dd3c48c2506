timeout 300 ncu --set full --clock-control none --import-source on -k regex:"sddmm_dense2" -s 2 -c 1 -o gpurun_out/s8_sd2 python tools/sddmm_bench.py tf32 1 > /dev/null 2>&1
