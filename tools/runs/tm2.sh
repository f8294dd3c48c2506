cd /root/repo
for i in 1 2; do
for v in base ne3np ne4np ne2 ne6 l2 old; do
  if [ $v = base ]; then L=""; E=""; elif [ $v = old ]; then L=""; E="SGTK_SPMM_TM=0"; else L="SGTK_LIB=$PWD/variants/libsgtk_$v.so"; E=""; fi
  a=$(env $L $E timeout 300 python tools/spmm_only.py --workload proteins-gcn --d 64 2>&1 | tail -1)
  b=$(env $L $E timeout 300 python tools/spmm_only.py --workload reddit-agnn --d 32 2>&1 | tail -1)
  echo "$v | C3 $a | C4 $b"
done; done
