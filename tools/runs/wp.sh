cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_panel.py tests/test_gpu_configs.py tests/test_gpu_dropin.py tests/test_gpu_fullsize.py -q -x > gpurun_out/wp_par.log 2>&1; echo "parity rc $?"; tail -1 gpurun_out/wp_par.log
for v in new old new old; do
  if [ $v = old ]; then E="SGTK_GEMM_WPREP=1"; else E=""; fi
  for w in cora-gcn proteins-gcn; do
    env $E timeout 600 python bench.py --no-cpu --workload $w > gpurun_out/wp_$w.json 2>/dev/null
    python -c "import json; d=json.loads(open('gpurun_out/wp_$w.json').read().strip().splitlines()[-1]); print('$v $w', d['value'], d['kernels_ms'], d['gpu_launches'])"
  done
done
