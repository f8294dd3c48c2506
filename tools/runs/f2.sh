for r in 1 2; do for lib in default nb6 nb10 nb12; do
 if [ $lib = default ]; then unset SGTK_LIB; else export SGTK_LIB=$PWD/variants/libsgtk_$lib.so; fi
 echo "$lib: $(timeout 60 python tools/agnn_only.py 2>&1 | tail -1) dense $(SGTK_PANEL_DEBUG=1 timeout 60 python tools/agnn_only.py 2>&1 | tail -1)"
done; done
