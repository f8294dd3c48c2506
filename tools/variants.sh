for lib in libsgtk_b200.so libsgtk_b200_mb3.so libsgtk_b200_mb4.so; do
 for p in fp32 tf32; do
  SGTK_LIB=$PWD/paper_2412_12218_b200/$lib python bench.py --steps 5 --warmup 3 --no-cpu --precision $p 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$lib', d['config']['precision'], d['value'], d['kernels_ms']['agnn_fused_kernel'], d['kernels_ms']['spmm'], d['kernels_ms']['sddmm'])"
 done
done
