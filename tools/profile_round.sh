#!/bin/bash
# Round profile: kernel launch list of the default bench command (ncu
# gpu__time_duration, --clock-control none) and one ncu --set full capture
# per top kernel.  Usage: bash tools/profile_round.sh <tag>
tag=${1:-r1}
mkdir -p gpurun_out
# tensor-pipe utilisation (sm_100 counter names, from `ncu --query-metrics --chip gb100`)
TC_METRICS=sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32.sum,sm__inst_executed_pipe_tc_scope_1cta.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${tag}.csv python bench.py --steps 2 --warmup 3 --no-cpu > /dev/null 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_${tag}_gcn.csv python bench.py --steps 2 --warmup 3 --no-cpu \
    --workload proteins-gcn > /dev/null 2>&1
ncu --set full --metrics $TC_METRICS --clock-control none --import-source on \
    -k regex:"agnn_dense_kernel|agnn_rows_kernel|spmm_panel_kernel|sparse_rows_kernel|gemm_tc05_kernel|sddmm_dense2_kernel|sddmm_sparse_kernel" -c 8 \
    -o gpurun_out/prof_${tag} python bench.py --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1
ncu --set full --metrics $TC_METRICS --clock-control none --import-source on -k regex:"spmm_panel_kernel|sparse_rows_kernel" -c 2 \
    -o gpurun_out/prof_${tag}_gcn python bench.py --steps 1 --warmup 3 --no-cpu --workload proteins-gcn > /dev/null 2>&1
echo done
