cd /root/repo
SGTK_LIB=$PWD/variants/libsgtk_af16.so timeout 900 python -m pytest tests/test_gpu_panel.py tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -k agnn > gpurun_out/af_par.log 2>&1; echo "parity rc $?"; tail -1 gpurun_out/af_par.log
for i in 1 2; do
for v in base af16; do
  if [ $v = base ]; then L=""; else L="SGTK_LIB=$PWD/variants/libsgtk_$v.so"; fi
  a=$(env $L timeout 300 python tools/agnn_only.py 2>&1 | tail -1)
  c=$(env $L timeout 300 python tools/agnn_only.py --precision fp32 2>&1 | tail -1)
  echo "$v | layer $a | fp32 $c"
done; done
