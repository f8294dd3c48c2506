for lib in default acc0 acc1000; do
 if [ $lib = default ]; then unset SGTK_LIB; else export SGTK_LIB=$PWD/variants/libsgtk_$lib.so; fi
 for e in "X=1" "SGTK_AGNN_GATHER=cp"; do
  echo "$lib $e: $(env $e python tools/agnn_only.py 2>&1| tail -1) dense $(env $e SGTK_PANEL_DEBUG=1 python tools/agnn_only.py 2>&1| tail -1)"
 done
done
