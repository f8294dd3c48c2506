timeout 600 python -m pytest tests/test_gpu_panel.py tests/test_gpu_parity.py tests/test_gpu_configs.py tests/test_gpu_multigpu.py -m gpu -q -x -k "agnn or AGNN" 2>&1 | tail -3
bash tools/ab_env.sh SGTK_AGNN_ROWS=tile
echo "minb2 variant:"
SGTK_LIB=$PWD/variants/libsgtk_minb2.so python tools/agnn_only.py | tail -1
SGTK_LIB=$PWD/variants/libsgtk_minb2.so SGTK_PANEL_DEBUG=2 python tools/agnn_only.py | tail -1
