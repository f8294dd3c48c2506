timeout 300 python -m pytest tests/test_gpu_panel.py tests/test_gpu_parity.py -x -q -m gpu -k "agnn" 2>&1 | tail -1
for lib in variants/libsgtk_base.so "" variants/libsgtk_mb3.so variants/libsgtk_mb5.so; do
  echo "lib [$lib] agnn total/sparse tf32, total/sparse fp32"
  if [ -n "$lib" ]; then export SGTK_LIB=$PWD/$lib; else unset SGTK_LIB; fi
  for p in tf32 fp32; do for m in 0 2; do SGTK_PANEL_DEBUG=$m timeout 200 python tools/agnn_only.py --precision $p 2>&1 | tail -1; done; done
done
