# ncu of the sparse-only AGNN part: new lane=edge kernel vs the tile kernel
export SGTK_PANEL_DEBUG=2
ncu --set full --clock-control none --import-source on -k regex:"agnn_sparse_kernel|agnn_rows_kernel" -s 2 -c 1 -o gpurun_out/r2o_sparse python tools/agnn_only.py --iters 1 --layers 1 > /dev/null 2>&1
SGTK_AGNN_ROWS=tile ncu --set full --clock-control none --import-source on -k regex:"agnn_sparse_kernel|agnn_rows_kernel" -s 2 -c 1 -o gpurun_out/r2o_tile python tools/agnn_only.py --iters 1 --layers 1 > /dev/null 2>&1
ls -la gpurun_out/
