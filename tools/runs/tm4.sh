cd /root/repo
for i in 1 2; do
for v in base popc spin popcspin old; do
  if [ $v = base ]; then L=""; E=""; elif [ $v = old ]; then L=""; E="SGTK_SPMM_TM=0"; else L="SGTK_LIB=$PWD/variants/libsgtk_$v.so"; E=""; fi
  a=$(env $L $E timeout 300 python tools/spmm_only.py --workload proteins-gcn --d 64 2>&1 | tail -1)
  echo "$v | C3 $a"
done; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:spmm_tm_kernel -c 1 -o gpurun_out/tm_prof python tools/spmm_only.py --workload proteins-gcn --d 64 --iters 1 > /dev/null 2>&1; echo "ncu rc $?"
