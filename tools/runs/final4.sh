cd /root/repo
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2z5_tests.log 2>&1; echo "tests rc $?"; tail -1 gpurun_out/r2z5_tests.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/r2z5_bench_red_tf32.json 2> gpurun_out/r2z5_bench.err; echo "bench rc $?"
python -c "import json; d=json.loads(open('gpurun_out/r2z5_bench_red_tf32.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e']['value'], d['roofline']['frac'], d['gpu_launches'], d['clocks']['sm_mhz'], d['clocks']['reasons'])"
for w in proteins-gcn pubmed-agnn cora-gcn; do timeout 600 python bench.py --no-cpu --workload $w > gpurun_out/r2z5_bench_$w.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r2z5_bench_$w.json').read().strip().splitlines()[-1]); print('$w', d['value'], d['e2e']['value'], d['gpu_launches'])"; done
timeout 600 python bench.py --no-cpu --precision fp32 > gpurun_out/r2z5_bench_red_fp32.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r2z5_bench_red_fp32.json').read().strip().splitlines()[-1]); print('fp32', d['value'])"
