# one ncu capture of the fused AGNN kernel (TF32 and FP32) on the bench workload
for p in tf32 fp32; do
python bench.py --steps 5 --warmup 3 --no-cpu --precision $p 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['config']['precision'], d['value'], d['kernels_ms'])"
done
ncu --set full --clock-control none --import-source on -k regex:"agnn_fused_kernel" -c 1 -o gpurun_out/prof_fused_tf32 python bench.py --steps 1 --warmup 1 --no-cpu --precision tf32 > /dev/null 2>&1
