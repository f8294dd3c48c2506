timeout 300 python -m pytest tests/test_gpu_panel.py tests/test_gpu_parity.py -x -q -m gpu -k agnn 2>&1 | tail -1
for rep in 1 2; do
for lib in variants/libsgtk_base.so "" variants/libsgtk_gmask.so; do
  echo "lib [$lib] agnn tf32 total/dense"
  if [ -n "$lib" ]; then export SGTK_LIB=$PWD/$lib; else unset SGTK_LIB; fi
  for m in 0 1; do SGTK_PANEL_DEBUG=$m timeout 200 python tools/agnn_only.py 2>&1 | tail -1; done
done; done
