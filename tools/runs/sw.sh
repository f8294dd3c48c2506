cd /root/repo
for i in 1 2; do
for v in base mb4 mb6 rg24 rg48 fg8 fg32; do
  if [ $v = base ]; then L=""; else L="SGTK_LIB=$PWD/variants/libsgtk_$v.so"; fi
  a=$(env $L timeout 300 python tools/agnn_only.py 2>&1 | tail -1)
  echo "$v | $a"
done; done
