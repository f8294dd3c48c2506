"""Small-graph driver for compute-sanitizer (racecheck / synccheck / memcheck).

Runs every hand-written kernel family once on graphs small enough for the
sanitizer's instrumentation: the GPU translator (scan/sort path and the hub
windows that take the CUB path), the panel build, the tcgen05 SpMM panels and
CUDA-core rows (TF32 and FP32), the AGNN panel layer (dense + rows + final, on
two streams), the 16-row kernels (explicit partial plans, SDDMM, fused AGNN),
the tcgen05 GEMM and the row ops.  Usage:
    compute-sanitizer --tool racecheck python tools/sanitize_driver.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2412_12218_b200 as sg  # noqa: E402
from paper_2412_12218_b200 import device as D  # noqa: E402


def main():
    torch.cuda.set_device(0)
    g = sg.synth_graph(1500, 24.0, alpha=2.0, p_local=0.8, band=4.0, seed=3)
    dg = D.DeviceGraph.from_csr(g.node_pointer, g.edge_list, None, g.num_nodes)
    gn = sg.gcn_normalize_values(g)
    dgn = D.DeviceGraph.from_csr(gn.node_pointer, gn.edge_list, gn.values, g.num_nodes)
    for d in (16, 32, 64):
        x = torch.from_numpy(sg.dense_random(g.num_nodes, d, 5)).cuda()
        for prec in ("tf32", "fp32"):
            dgn.spmm(x, precision=prec)                       # panels (default plan)
            dgn.spmm(x, cut=dgn.split_plan(0.5), precision=prec)  # 16-row kernels
        if d <= 64:
            for prec in ("tf32", "fp32"):
                for mode in (0, 1, 2):
                    dg.agnn_forward(x, np.ones(2, np.float32), precision=prec, mode=mode)
        dg.sddmm(x, x, precision="tf32")                      # direct form (Panels::dpos)
        dgn.sddmm(x, x, precision="fp32")                     # weighted graph: entry values
        ev = torch.rand(g.num_edges, device="cuda")
        dg.sddmm(x, x, precision="tf32", edge_values=ev)      # CSR-order overrides
        w = torch.from_numpy(sg.dense_random(d, 32, 6, -0.1, 0.1)).cuda()
        D.gemm(x, w, relu=True, precision="tf32")
        D.gemm(x, w, relu=False, precision="fp32")
    torch.cuda.synchronize()
    print("sanitize driver ok")


if __name__ == "__main__":
    main()
