timeout 300 python -m pytest tests/test_gpu_panel.py -m gpu -q -x 2>&1 | tail -1
for r in 1 2; do for lib in default nopf b16 b8; do
 if [ $lib = default ]; then unset SGTK_LIB; else export SGTK_LIB=$PWD/variants/libsgtk_$lib.so; fi
 echo "$lib: $(timeout 120 python tools/spmm_only.py 2>&1 | tail -1) d32 $(timeout 120 python tools/spmm_only.py --d 32 2>&1 | tail -1)"
done; done
