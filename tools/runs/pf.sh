cd /root/repo
for i in 1 2; do
for v in base pf0; do
  if [ $v = base ]; then L=""; else L="SGTK_LIB=$PWD/variants/libsgtk_$v.so"; fi
  a=$(env $L timeout 300 python tools/agnn_only.py 2>&1 | tail -1)
  b=$(env $L SGTK_PANEL_DEBUG=2 timeout 300 python tools/agnn_only.py 2>&1 | tail -1)
  c=$(env $L timeout 300 python tools/agnn_only.py --precision fp32 2>&1 | tail -1)
  echo "$v | layer $a | sparse $b | fp32 $c"
done; done
