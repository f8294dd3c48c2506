./tools/gather4_probe
timeout 600 python -m pytest tests/test_gpu_panel.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_multigpu.py tests/test_gpu_fullsize.py -m gpu -q -x -k "agnn or AGNN" 2>&1 | tail -3
for e in "X=1" "SGTK_AGNN_GATHER=cp" "SGTK_AGNN_ROWS=tile" "SGTK_AGNN_GATHER=cp SGTK_AGNN_ROWS=tile"; do
  echo "$e: $(env $e python tools/agnn_only.py | tail -1) dense $(env $e SGTK_PANEL_DEBUG=1 python tools/agnn_only.py | tail -1) sparse $(env $e SGTK_PANEL_DEBUG=2 python tools/agnn_only.py | tail -1)"
done
