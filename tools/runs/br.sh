cd /root/repo
timeout 900 python -m pytest tests/test_gpu_panel.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_variants.py -q -x > gpurun_out/br_par.log 2>&1; echo "parity rc $?"; tail -1 gpurun_out/br_par.log
for i in 1 2; do
for v in base br0; do
  if [ $v = base ]; then L=""; else L="SGTK_LIB=$PWD/variants/libsgtk_$v.so"; fi
  a=$(env $L timeout 300 python tools/spmm_only.py --workload proteins-gcn --d 64 2>&1 | tail -1)
  b=$(env $L timeout 300 python tools/spmm_only.py --workload reddit-agnn --d 32 2>&1 | tail -1)
  c=$(env $L timeout 300 python tools/spmm_only.py --workload proteins-gcn --d 64 --precision fp32 2>&1 | tail -1)
  e=$(env $L timeout 300 python tools/spmm_only.py --workload proteins-gcn --d 128 2>&1 | tail -1)
  echo "$v | C3 $a | C4d32 $b | C3 fp32 $c | d128 $e"
done; done
