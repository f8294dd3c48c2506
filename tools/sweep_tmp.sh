timeout 600 python -m pytest tests -x -q -m gpu -k "gemm or gcn or forward or model" 2>&1 | tail -2
for lib in variants/libsgtk_base.so ""; do
  if [ -n "$lib" ]; then export SGTK_LIB=$PWD/$lib; else unset SGTK_LIB; fi
  for p in tf32 fp32; do echo "lib [$lib] $p"; timeout 300 python bench.py --workload proteins-gcn --precision $p --no-cpu --steps 5 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['kernels_ms'], d['e2e']['value'])"; done
  echo "reddit in-proj"; timeout 300 python bench.py --no-cpu --steps 3 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['roofline_gemm'])"
done
