timeout 300 python -m pytest tests -x -q -m gpu -k "gemm or gcn" 2>&1 | tail -1
for lib in variants/libsgtk_base.so ""; do
  if [ -n "$lib" ]; then export SGTK_LIB=$PWD/$lib; else unset SGTK_LIB; fi
  echo "lib [$lib]"; timeout 300 python bench.py --workload proteins-gcn --no-cpu --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernels_ms'])"
done
