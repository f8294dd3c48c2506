timeout 900 bash tools/profile_round.sh r2zz > /dev/null 2>&1; echo "profile rc $?"
TC=sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active,sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32.sum,sm__inst_executed_pipe_tc_scope_1cta.sum,sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active
timeout 600 ncu --set full --metrics $TC --clock-control none --import-source on -k regex:"gemm_tc05_kernel" -c 1 -o gpurun_out/prof_r2zz_gemm python bench.py --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1; echo rc $?
timeout 600 ncu --set full --metrics $TC --clock-control none --import-source on -k regex:"sddmm_dense2_kernel|sddmm_sparse_kernel" -s 2 -c 2 -o gpurun_out/prof_r2zz_sddmm python tools/sddmm_bench.py tf32 1 > /dev/null 2>&1; echo rc $?
ls gpurun_out | grep r2zz
