export SGTK_LIB=$PWD/variants/libsgtk_trace.so
SGTK_PANEL_DEBUG=1 SGTK_PANEL_TRACE=gpurun_out/trace_prot.bin timeout 200 python tools/spmm_only.py --iters 1 2>&1 | tail -1
