timeout 300 ncu --metrics gpu__time_duration.sum -k regex:"sddmm" -s 6 -c 6 python tools/sddmm_bench.py tf32 2 2>&1 | grep -E "^  void|duration" | sed 's/(PanelView.*//; s/(unsigned long.*//; s/(const float.*//' | head -12
timeout 300 ncu --set full --clock-control none --import-source on -k regex:"sddmm_sparse" -s 2 -c 1 -o gpurun_out/s7_sp python tools/sddmm_bench.py tf32 1 > /dev/null 2>&1
