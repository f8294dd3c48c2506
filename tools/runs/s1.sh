timeout 300 python -m pytest tests/test_gpu_panel.py tests/test_gpu_parity.py -m gpu -q -x 2>&1 | tail -2
for lib in default tmazero; do
 if [ $lib = default ]; then unset SGTK_LIB; else export SGTK_LIB=$PWD/variants/libsgtk_$lib.so; fi
 for cfg in "proteins-gcn 64 tf32" "proteins-gcn 64 fp32" "proteins-gcn 32 tf32" "proteins-gcn 16 tf32" "reddit-agnn 32 tf32"; do
  set -- $cfg
  echo "$lib $cfg: $(timeout 120 python tools/spmm_only.py --workload $1 --d $2 --precision $3 2>&1 | tail -1)"
 done
done
