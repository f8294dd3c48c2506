cd /root/repo
timeout 600 python -m pytest tests/test_gpu_variants.py -q -x -k spmm > gpurun_out/tm1_var.log 2>&1; echo "variant rc $?"; tail -3 gpurun_out/tm1_var.log
for v in 1 0 1 0; do echo "TM=$v"; SGTK_SPMM_TM=$v timeout 300 python tools/spmm_only.py --workload proteins-gcn --d 64 2>&1 | tail -1; SGTK_SPMM_TM=$v timeout 300 python tools/spmm_only.py --workload reddit-agnn --d 32 2>&1 | tail -1; done
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_panel.py tests/test_gpu_configs.py -q -x > gpurun_out/tm1_par.log 2>&1; echo "parity rc $?"; tail -3 gpurun_out/tm1_par.log
