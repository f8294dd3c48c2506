cd /root/repo
for i in 1 2; do
for v in base mr64 mr64l2; do
  if [ $v = base ]; then L=""; else L="SGTK_LIB=$PWD/variants/libsgtk_$v.so"; fi
  a=$(env $L timeout 300 python tools/agnn_only.py 2>&1 | tail -1)
  b=$(env $L SGTK_PANEL_DEBUG=1 timeout 300 python tools/agnn_only.py 2>&1 | tail -1)
  echo "$v | layer $a | dense $b"
done; done
