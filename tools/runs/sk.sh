cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_panel.py tests/test_gpu_configs.py tests/test_gpu_dropin.py -q -x > gpurun_out/sk_par.log 2>&1; echo "parity rc $?"; tail -2 gpurun_out/sk_par.log
for v in 1 0 1 0; do
  echo "splitk build=$v"
  if [ $v = 0 ]; then L="SGTK_LIB=$PWD/variants/libsgtk_nosk.so"; else L=""; fi
  env $L timeout 600 python bench.py --no-cpu --workload cora-gcn > gpurun_out/sk_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/sk_$v.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['kernels_ms'], d['e2e']['value'])"
done
