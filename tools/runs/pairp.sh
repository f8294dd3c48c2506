cd /root/repo
SGTK_LIB=$PWD/variants/libsgtk_pairp.so timeout 900 python -m pytest tests/test_gpu_panel.py tests/test_gpu_parity.py tests/test_gpu_variants.py -q -x -k "agnn" > gpurun_out/pairp_par.log 2>&1; echo "parity rc $?"; tail -1 gpurun_out/pairp_par.log
for i in 1 2; do
for v in base pairp; do
  if [ $v = base ]; then L=""; else L="SGTK_LIB=$PWD/variants/libsgtk_$v.so"; fi
  a=$(env $L timeout 300 python tools/agnn_only.py 2>&1 | tail -1)
  b=$(env $L SGTK_PANEL_DEBUG=1 timeout 300 python tools/agnn_only.py 2>&1 | tail -1)
  echo "$v | layer $a | dense $b"
done; done
