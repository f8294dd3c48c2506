cd /root/repo
timeout 900 python -m pytest tests/test_gpu_panel.py tests/test_gpu_parity.py -q -x -k "spmm or gcn" > gpurun_out/ne_par.log 2>&1; echo "parity rc $?"; tail -1 gpurun_out/ne_par.log
SGTK_LIB=$PWD/variants/libsgtk_nd4ne8.so timeout 900 python -m pytest tests/test_gpu_panel.py tests/test_gpu_parity.py -q -x -k "spmm or gcn" > gpurun_out/ne_par2.log 2>&1; echo "parity2 rc $?"; tail -1 gpurun_out/ne_par2.log
for i in 1 2; do
for v in base nd4ne5 nd4ne8 nd6ne8; do
  if [ $v = base ]; then L=""; else L="SGTK_LIB=$PWD/variants/libsgtk_$v.so"; fi
  a=$(env $L timeout 300 python tools/spmm_only.py --workload proteins-gcn --d 64 2>&1 | tail -1)
  b=$(env $L timeout 300 python tools/spmm_only.py --workload reddit-agnn --d 32 2>&1 | tail -1)
  c=$(env $L timeout 300 python tools/spmm_only.py --workload proteins-gcn --d 64 --precision fp32 2>&1 | tail -1)
  echo "$v | C3 $a | C4d32 $b | C3 fp32 $c"
done; done
