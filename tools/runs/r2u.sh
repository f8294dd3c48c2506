export SGTK_PANEL_DEBUG=2
for e in "X=1" "SGTK_AGNN_ROWS=lane"; do
n=$(echo $e | tr -dc 'a-z' | head -c 6)
env $e ncu --set full --clock-control none --import-source on -k regex:"agnn_sparse_kernel|agnn_rows_kernel" -s 2 -c 1 -o gpurun_out/r2u_$n python tools/agnn_only.py --iters 1 --layers 1 > /dev/null 2>&1
done
SGTK_LIB=$PWD/variants/libsgtk_head.so ncu --set full --clock-control none --import-source on -k regex:"agnn_sparse_kernel|agnn_rows_kernel" -s 2 -c 1 -o gpurun_out/r2u_head python tools/agnn_only.py --iters 1 --layers 1 > /dev/null 2>&1
ls gpurun_out
