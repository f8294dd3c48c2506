cd /root/repo
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_panel.py tests/test_gpu_fullsize.py tests/test_gpu_robust.py tests/test_gpu_multigpu.py -q -x > gpurun_out/ls_par.log 2>&1; echo "parity rc $?"; tail -2 gpurun_out/ls_par.log
for i in 1 2 3; do
for v in side serial; do
  if [ $v = serial ]; then E="SGTK_AGNN_LONG_SERIAL=1"; else E=""; fi
  env $E timeout 600 python bench.py --no-cpu --steps 20 > gpurun_out/ls_$v.json 2>/dev/null
  python -c "import json; d=json.loads(open('gpurun_out/ls_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['kernels_ms'].get('agnn_panel_layer'))"
done; done
