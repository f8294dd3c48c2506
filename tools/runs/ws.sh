cd /root/repo
for i in 1 2; do
for v in base ws64 ws256; do
  if [ $v = base ]; then L=""; else L="SGTK_LIB=$PWD/variants/libsgtk_$v.so"; fi
  a=$(env $L timeout 300 python tools/sddmm_bench.py tf32 2>&1 | tail -1)
  echo "$v | $a"
done
for v in base spm256; do
  if [ $v = base ]; then L=""; else L="SGTK_LIB=$PWD/variants/libsgtk_$v.so"; fi
  a=$(env $L timeout 300 python tools/spmm_only.py --workload proteins-gcn --d 64 2>&1 | tail -1)
  echo "$v | C3 $a"
done; done
