timeout 400 python -m pytest tests/test_gpu_sddmm.py tests/test_gpu_parity.py tests/test_gpu_panel.py tests/test_gpu_dropin.py -m gpu -q -x 2>&1 | tail -2
for e in X=1 SGTK_SDDMM_DENSE=staged; do for p in tf32 fp32; do echo "$e $(env $e timeout 120 python tools/sddmm_bench.py $p 10 | tail -1)"; done; done
SGTK_PANEL_DEBUG=1 timeout 120 python tools/sddmm_bench.py tf32 10 | tail -1
