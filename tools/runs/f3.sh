for r in 1 2; do for lib in default g16 g64 mb4 mb6 w4; do
 if [ $lib = default ]; then unset SGTK_LIB; else export SGTK_LIB=$PWD/variants/libsgtk_$lib.so; fi
 echo "$lib: $(timeout 60 python tools/agnn_only.py 2>&1 | tail -1) sparse $(SGTK_PANEL_DEBUG=2 timeout 60 python tools/agnn_only.py 2>&1 | tail -1)"
done; done
