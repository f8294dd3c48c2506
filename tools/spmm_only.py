"""Run the default-plan SpMM on a bench workload graph (for ncu captures)."""
import sys, os, argparse
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch, bench
import paper_2412_12218_b200 as sg
from paper_2412_12218_b200.device import DeviceGraph
ap = argparse.ArgumentParser()
ap.add_argument("--workload", default="proteins-gcn")
ap.add_argument("--d", type=int, default=64)
ap.add_argument("--precision", default="tf32")
ap.add_argument("--iters", type=int, default=3)
a = ap.parse_args()
wl = bench.WORKLOADS[a.workload]
g, _ = bench.make_graph(wl, "calibrated")
if wl["kind"] == "gcn":
    g = sg.gcn_normalize_values(g)
dg = DeviceGraph.from_csr(g.node_pointer, g.edge_list, g.values)
print(dg.panel_info(), flush=True)
x = torch.randn(g.num_nodes, a.d, device="cuda")
out = torch.empty_like(x)
for _ in range(a.iters):
    dg.spmm(x, out=out, precision=a.precision)
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10):
    dg.spmm(x, out=out, precision=a.precision)
e.record(); torch.cuda.synchronize()
print("spmm ms", s.elapsed_time(e) / 10)
