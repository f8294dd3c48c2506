for lib in "" variants/libsgtk_b16_16.so variants/libsgtk_b32_8.so variants/libsgtk_b16_8.so variants/libsgtk_b8_8.so; do
  echo "lib [$lib] prot tf32 total/sparse, prot fp32, reddit d32 tf32 total/sparse, agnn total"
  if [ -n "$lib" ]; then export SGTK_LIB=$PWD/$lib; else unset SGTK_LIB; fi
  for m in 0 2; do SGTK_PANEL_DEBUG=$m timeout 200 python tools/spmm_only.py 2>&1 | tail -1; done
  timeout 200 python tools/spmm_only.py --precision fp32 2>&1 | tail -1
  for m in 0 2; do SGTK_PANEL_DEBUG=$m timeout 200 python tools/spmm_only.py --workload reddit-agnn --d 32 2>&1 | tail -1; done
done
