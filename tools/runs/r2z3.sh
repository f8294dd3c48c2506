SGTK_AGNN_ROWS=lane timeout 300 python -m pytest tests/test_gpu_panel.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_multigpu.py tests/test_gpu_fullsize.py tests/test_gpu_robust.py -m gpu -q -x -k "agnn or AGNN or robust" 2>&1 | tail -2
for lib in default sm4; do
 if [ $lib = default ]; then unset SGTK_LIB; else export SGTK_LIB=$PWD/variants/libsgtk_$lib.so; fi
 for e in "X=1" "SGTK_AGNN_ROWS=lane"; do
  echo "$lib $e: $(env $e timeout 60 python tools/agnn_only.py 2>&1| tail -1) sparse $(env $e SGTK_PANEL_DEBUG=2 timeout 60 python tools/agnn_only.py 2>&1| tail -1)"
 done
done
unset SGTK_LIB; SGTK_AGNN_ROWS=lane SGTK_PANEL_DEBUG=2 timeout 120 ncu --set full --clock-control none --import-source on -k regex:"agnn_sparse_kernel" -s 2 -c 1 -o gpurun_out/r2z3_lane python tools/agnn_only.py --iters 1 --layers 1 > /dev/null 2>&1
