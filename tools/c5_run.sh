#!/bin/bash
# C5 (10M nodes / 1B edges, GCN d=128) on one B200: sampled-row parity and a bench line.
tag=${1:-r2}
mkdir -p gpurun_out
timeout 1500 python -m pytest tests/test_gpu_fullsize.py -q -k c5 > gpurun_out/${tag}_c5_test.log 2>&1; echo "c5 test rc $?"; tail -3 gpurun_out/${tag}_c5_test.log
timeout 1800 python bench.py --workload powerlaw-gcn --steps 5 --warmup 3 --csv gpurun_out/${tag}_c5_report.csv > gpurun_out/${tag}_c5_bench.json 2> gpurun_out/${tag}_c5_bench.err; echo "c5 bench rc $?"
tail -5 gpurun_out/${tag}_c5_bench.err; head -c 1500 gpurun_out/${tag}_c5_bench.json
