#!/bin/bash
# Bench contract checks on one GPU: default line, the N>1 path (2 ranks
# sharing the device), the reference arm, the GCN workload with --csv.
tag=${1:-r2}
mkdir -p gpurun_out
timeout 900 python bench.py --csv gpurun_out/${tag}_report.csv > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc $?"
timeout 900 python bench.py --gpus 2 --steps 5 > gpurun_out/${tag}_bench_g2.json 2> gpurun_out/${tag}_bench_g2.err; echo "bench g2 rc $?"
timeout 900 python bench.py --workload proteins-gcn --csv gpurun_out/${tag}_report.csv > gpurun_out/${tag}_bench_prot.json 2> gpurun_out/${tag}_bench_prot.err; echo "prot rc $?"
timeout 900 python bench.py --workload proteins-gcn --gpus 2 --steps 5 > gpurun_out/${tag}_bench_prot_g2.json 2> gpurun_out/${tag}_bench_prot_g2.err; echo "prot g2 rc $?"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 --csv gpurun_out/${tag}_report.csv > gpurun_out/${tag}_ref.json 2> gpurun_out/${tag}_ref.err; echo "ref rc $?"
for f in bench bench_g2 bench_prot bench_prot_g2 ref; do head -c 400 gpurun_out/${tag}_$f.json; echo; tail -2 gpurun_out/${tag}_$f.err; done
