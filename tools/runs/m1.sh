timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu > gpurun_out/m1_g2_red.json 2> gpurun_out/m1_g2_red.err; echo "rc $?"
python -c "import json; d=json.loads(open('gpurun_out/m1_g2_red.json').read().strip().splitlines()[-1]); print(d['n_gpus'], d['value'], d.get('verify'), d['config'].get('parallelism'))"
timeout 900 python bench.py --gpus 2 --steps 3 --warmup 3 --no-cpu --workload proteins-gcn > gpurun_out/m1_g2_prot.json 2> gpurun_out/m1_g2_prot.err; echo "rc $?"
python -c "import json; d=json.loads(open('gpurun_out/m1_g2_prot.json').read().strip().splitlines()[-1]); print(d['n_gpus'], d['value'], d.get('verify'))"
tail -3 gpurun_out/m1_g2_red.err
