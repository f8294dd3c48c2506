export SGTK_PANEL_DEBUG=1
ncu --set full --clock-control none --import-source on -k regex:"agnn_dense" -s 2 -c 1 -o gpurun_out/r2w_dense python tools/agnn_only.py --iters 1 --layers 1 > /dev/null 2>&1
ls gpurun_out | grep r2w
