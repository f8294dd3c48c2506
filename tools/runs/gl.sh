cd /root/repo
for w in reddit-agnn proteins-gcn cora-gcn pubmed-agnn; do
  timeout 600 python bench.py --no-cpu --steps 5 --workload $w > gpurun_out/gl_$w.json 2>gpurun_out/gl_$w.err
  python -c "import json; d=json.loads(open('gpurun_out/gl_$w.json').read().strip().splitlines()[-1]); print('$w', d['gpu_launches'], d['details']['gpu_launches_source'])"
done
