timeout 400 python -m pytest tests/test_gpu_panel.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_multigpu.py tests/test_gpu_fullsize.py tests/test_gpu_robust.py -m gpu -q -x -k "agnn or AGNN or robust" 2>&1 | tail -2
for e in X=1 SGTK_AGNN_FUSED=0; do echo "$e: $(env $e timeout 60 python tools/agnn_only.py 2>&1 | tail -1)"; done
for e in X=1 SGTK_AGNN_FUSED=0; do echo "$e: $(env $e timeout 60 python tools/agnn_only.py 2>&1 | tail -1)"; done
