cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_panel.py tests/test_gpu_configs.py tests/test_gpu_dropin.py tests/test_gpu_robust.py tests/test_gpu_multigpu.py -q -x > gpurun_out/pw_par.log 2>&1; echo "parity rc $?"; tail -1 gpurun_out/pw_par.log
for i in 1 2; do for w in cora-gcn proteins-gcn; do
  timeout 600 python bench.py --no-cpu --workload $w > gpurun_out/pw_$w.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/pw_$w.json').read().strip().splitlines()[-1]); print('$w', d['value'], d['gpu_launches'], d['details']['cuda_graph'][-25:])"
done; done
