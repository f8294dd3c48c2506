cd /root/repo
for i in 1 2 3; do
  timeout 900 python bench.py --no-cpu > gpurun_out/rep_$i.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/rep_$i.json').read().strip().splitlines()[-1]); print(json.dumps({'run': $i, 'value': d['value'], 'e2e': d['e2e']['value'], 'frac': d['roofline']['frac'], 'sm_mhz': d['clocks']['sm_mhz'], 'reasons': d['clocks']['reasons'], 'ms_per_step': d['ms_per_step']}))"
done
