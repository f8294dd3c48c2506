timeout 600 python -m pytest tests/test_gpu_panel.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_multigpu.py tests/test_gpu_fullsize.py tests/test_gpu_robust.py -m gpu -q -x -k "agnn or AGNN or robust" 2>&1 | tail -3
for lib in default oneiss; do
 if [ $lib = default ]; then unset SGTK_LIB; else export SGTK_LIB=$PWD/variants/libsgtk_$lib.so; fi
 for e in "SGTK_AGNN_ROWS=tile" "SGTK_AGNN_ROWS=tile SGTK_AGNN_GATHER=cp"; do
  echo "$lib $e: $(env $e python tools/agnn_only.py | tail -1) dense $(env $e SGTK_PANEL_DEBUG=1 python tools/agnn_only.py | tail -1)"
 done
done
