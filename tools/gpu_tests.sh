#!/bin/bash
# GPU test suite + default bench line.  Usage: bash tools/gpu_tests.sh <tag> [pytest -k expr]
tag=${1:-r2}
mkdir -p gpurun_out
if [ -n "$2" ]; then K="-k $2"; else K=""; fi
timeout 2400 python -m pytest tests -m gpu -q -x $K > gpurun_out/${tag}_tests.log 2>&1; echo "tests rc $?"
tail -15 gpurun_out/${tag}_tests.log
timeout 600 python bench.py --no-cpu > gpurun_out/${tag}_bench.json 2> gpurun_out/${tag}_bench.err; echo "bench rc $?"
head -c 300 gpurun_out/${tag}_bench.json; echo
