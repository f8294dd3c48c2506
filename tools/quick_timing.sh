mkdir -p gpurun_out
(timeout 600 python -m pytest tests/test_gpu_panel.py -x -q -m gpu 2>&1 | tail -2
for p in tf32 fp32; do for m in 0 1 2; do echo "agnn $p dbg $m"; SGTK_PANEL_DEBUG=$m timeout 200 python tools/agnn_only.py --precision $p 2>&1 | tail -1; done; done
for w in proteins-gcn reddit-agnn; do for p in tf32 fp32; do echo "spmm $w $p"; timeout 200 python tools/spmm_only.py --workload $w --d $([ $w = proteins-gcn ] && echo 64 || echo 32) --precision $p 2>&1 | tail -1; done; done) > gpurun_out/r.log 2>&1
cat gpurun_out/r.log
