"""One AGNN layer (mode 2) on a bench workload graph (for ncu captures / timing)."""
import sys, os, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch, bench
import paper_2412_12218_b200 as sg
from paper_2412_12218_b200.device import DeviceGraph
ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="reddit-agnn")
ap.add_argument("--precision", default="tf32")
ap.add_argument("--mode", type=int, default=2)
ap.add_argument("--layers", type=int, default=4)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--d", type=int, default=0, help="feature width (default: the workload's)")
a = ap.parse_args()
wl = bench.WORKLOADS[a.workload]
g, _ = bench.make_graph(wl, "calibrated")
dg = DeviceGraph.from_csr(g.node_pointer, g.edge_list)
print(dg.panel_info(), flush=True)
x = torch.from_numpy(sg.dense_random(g.num_nodes, a.d or wl["hidden"], 3)).cuda()
betas = np.ones(a.layers, np.float32)
for _ in range(a.iters):
    dg.agnn_forward(x, betas, precision=a.precision, mode=a.mode)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(5):
    dg.agnn_forward(x, betas, precision=a.precision, mode=a.mode)
e.record(); torch.cuda.synchronize()
print("agnn ms per layer", s.elapsed_time(e) / 5 / a.layers)
