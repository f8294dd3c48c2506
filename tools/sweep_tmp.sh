timeout 300 python -m pytest tests/test_gpu_panel.py tests/test_gpu_parity.py -x -q -m gpu -k agnn 2>&1 | tail -1
for rep in 1 2; do
for lib in variants/libsgtk_base.so ""; do
  echo "lib [$lib] total/sparse-only"
  if [ -n "$lib" ]; then export SGTK_LIB=$PWD/$lib; else unset SGTK_LIB; fi
  timeout 200 python tools/agnn_only.py 2>&1 | tail -1; SGTK_PANEL_DEBUG=2 timeout 200 python tools/agnn_only.py 2>&1 | tail -1
done; done
