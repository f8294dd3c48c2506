timeout 600 python -m pytest tests/test_gpu_multigpu.py -m gpu -q -x > gpurun_out/m2.log 2>&1; tail -1 gpurun_out/m2.log
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --overlap 2 > gpurun_out/m2_g2_ov2.json 2> gpurun_out/m2_g2_ov2.err; echo "rc $?"
python -c "import json; d=json.loads(open('gpurun_out/m2_g2_ov2.json').read().strip().splitlines()[-1]); print(d['n_gpus'], d['value'], d.get('verify'), d['config'].get('parallelism'), d['e2e']['value'])"
tail -3 gpurun_out/m2_g2_ov2.err
