cd /root/repo
timeout 600 python -m pytest tests/test_gpu_variants.py -q -x -k spmm > gpurun_out/tm3_var.log 2>&1; echo "variant rc $?"; tail -2 gpurun_out/tm3_var.log
for i in 1 2; do
for v in base bg1 bg2l4 bg2ne3 old; do
  if [ $v = base ]; then L=""; E=""; elif [ $v = old ]; then L=""; E="SGTK_SPMM_TM=0"; else L="SGTK_LIB=$PWD/variants/libsgtk_$v.so"; E=""; fi
  a=$(env $L $E timeout 300 python tools/spmm_only.py --workload proteins-gcn --d 64 2>&1 | tail -1)
  b=$(env $L $E timeout 300 python tools/spmm_only.py --workload reddit-agnn --d 32 2>&1 | tail -1)
  echo "$v | C3 $a | C4 $b"
done; done
