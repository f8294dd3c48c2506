cd /root/repo
SGTK_LIB=$PWD/variants/libsgtk_smg2.so timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_panel.py tests/test_gpu_fullsize.py -q -x -k agnn > gpurun_out/sm1_par.log 2>&1; echo "parity rc $?"; tail -2 gpurun_out/sm1_par.log
for i in 1 2; do
for v in base smg2 smg2l3 smg2l4 l2; do
  if [ $v = base ]; then L=""; else L="SGTK_LIB=$PWD/variants/libsgtk_$v.so"; fi
  a=$(env $L timeout 300 python tools/agnn_only.py 2>&1 | tail -1)
  b=$(env $L SGTK_PANEL_DEBUG=1 timeout 300 python tools/agnn_only.py 2>&1 | tail -1)
  echo "$v | layer $a | dense $b"
done; done
