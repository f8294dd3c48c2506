cd /root/repo
for i in 1 2; do
for v in base gm gm2; do
  if [ $v = base ]; then L=""; else L="SGTK_LIB=$PWD/variants/libsgtk_$v.so"; fi
  b=$(env $L SGTK_PANEL_DEBUG=1 timeout 300 python tools/agnn_only.py 2>&1 | tail -1)
  echo "$v | dense $b"
done; done
