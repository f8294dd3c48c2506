for lib in default rw2 rw1; do
 if [ $lib = default ]; then unset SGTK_LIB; else export SGTK_LIB=$PWD/variants/libsgtk_$lib.so; fi
 for p in tf32 fp32; do
  echo "$lib $p: $(timeout 60 python tools/agnn_only.py --precision $p 2>&1| tail -1) sparse $(SGTK_PANEL_DEBUG=2 timeout 60 python tools/agnn_only.py --precision $p 2>&1| tail -1)"
 done
done
