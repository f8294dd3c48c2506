timeout 300 ncu --set full --clock-control none --import-source on -k regex:"sddmm_dense" -s 2 -c 1 -o gpurun_out/s6_sd2 python tools/sddmm_bench.py tf32 1 > /dev/null 2>&1
SGTK_SDDMM_DENSE=staged timeout 300 ncu --metrics gpu__time_duration.sum -k regex:"sddmm" -s 6 -c 6 python tools/sddmm_bench.py tf32 2 2>&1 | grep -E "sddmm_|duration" | head -12
timeout 300 ncu --metrics gpu__time_duration.sum -k regex:"sddmm" -s 6 -c 6 python tools/sddmm_bench.py tf32 2 2>&1 | grep -E "sddmm_|duration" | head -12
