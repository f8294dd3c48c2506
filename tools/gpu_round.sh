#!/bin/bash
# One GPU call: query tensor-pipe metric names, GPU test suite, default bench.
# Usage (under gpurun): bash tools/gpu_round.sh <tag>
tag=${1:-r2}
mkdir -p gpurun_out
ncu --query-metrics --chip gb100 2>&1 | grep -i -E "tensor|utc|tmem|tc_" > gpurun_out/${tag}_metrics_chip.txt
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/${tag}_tests.log 2>&1; echo tests rc $?
tail -3 gpurun_out/${tag}_tests.log
timeout 600 python bench.py > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo bench rc $?
cat gpurun_out/${tag}_bench.json | head -c 600
