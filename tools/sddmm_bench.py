"""C4-shaped SDDMM timing (CUDA events, L2 flushed) for profiling runs:
    python tools/sddmm_bench.py [tf32|fp32] [reps]"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2412_12218_b200 as sg  # noqa: E402
from paper_2412_12218_b200.device import DeviceGraph  # noqa: E402

prec = sys.argv[1] if len(sys.argv) > 1 else "tf32"
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
wl = bench.WORKLOADS[os.environ.get("WL", "reddit-agnn")]
g, _ = bench.make_graph(wl, "calibrated")
dg = DeviceGraph.from_csr(g.node_pointer, g.edge_list, None, g.num_nodes)
x = torch.from_numpy(sg.dense_random(g.num_nodes, 32, 8)).cuda()
out = torch.empty(g.num_edges, dtype=torch.float32, device="cuda")
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
for _ in range(3):
    dg.sddmm(x, x, precision=prec, out=out)
ts = []
for _ in range(reps):
    flush.fill_(1)
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    dg.sddmm(x, x, precision=prec, out=out)
    b.record()
    b.synchronize()
    ts.append(a.elapsed_time(b))
pi = dg.panel_info(32)
print(f"sddmm {prec}: {np.mean(ts):.4f} ms (min {np.min(ts):.4f}); chunks {pi['dense_chunks']} "
      f"dense entries {pi['dense_entries']} sparse {pi['sparse_edges']}")
