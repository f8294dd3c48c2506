for lib in base nb10 nb6 nb8_late nb10_late; do
  echo "lib [$lib] agnn tf32 total/dense"
  export SGTK_LIB=$PWD/variants/libsgtk_$lib.so
  for m in 0 1; do SGTK_PANEL_DEBUG=$m timeout 200 python tools/agnn_only.py 2>&1 | tail -1; done
done
