cd /root/repo
for i in 1 2; do
for v in 0 1 2 3; do
  a=$(SGTK_AGNN_PRIO=$v timeout 300 python tools/agnn_only.py 2>&1 | tail -1)
  echo "prio=$v | $a"
done; done
for v in 0 1 2 3; do
  SGTK_AGNN_PRIO=$v timeout 600 python bench.py --no-cpu --steps 20 > gpurun_out/pr_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/pr_$v.json').read().strip().splitlines()[-1]); print('bench prio=$v', d['value'], d['details'].get('cuda_graph','')[:60])"
done
