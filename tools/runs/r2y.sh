timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r2y_tests.log 2>&1; echo "tests rc $?"; tail -2 gpurun_out/r2y_tests.log
timeout 900 python bench.py > gpurun_out/r2y_bench_red_tf32.json 2> gpurun_out/r2y_bench.err; echo "bench rc $?"
python -c "import json; d=json.loads(open('gpurun_out/r2y_bench_red_tf32.json').read().strip().splitlines()[-1]); print(d['value'], d['e2e'], d.get('kernels_ms'), d['roofline'])"
for w in proteins-gcn pubmed-agnn; do timeout 600 python bench.py --no-cpu --workload $w > gpurun_out/r2y_bench_$w.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r2y_bench_$w.json').read().strip().splitlines()[-1]); print('$w', d['value'], d['e2e']['value'])"; done
timeout 600 python bench.py --no-cpu --precision fp32 > gpurun_out/r2y_bench_red_fp32.json 2>/dev/null; python -c "import json; d=json.loads(open('gpurun_out/r2y_bench_red_fp32.json').read().strip().splitlines()[-1]); print('fp32', d['value'])"
