import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2412_12218_b200 as sg
from paper_2412_12218_b200.device import DeviceGraph
from oracle.oracle import Csr, Oracle
O = Oracle()
for n, deg in [(40, 4.0), (3000, 30.0)]:
    g = sg.synth_graph(n, deg, alpha=0.0, p_local=0.9, band=4.0, seed=31)
    dg = DeviceGraph.from_csr(g.node_pointer, g.edge_list)
    for d in (32, 16, 64):
        x = torch.from_numpy(sg.dense_random(n, d, 1)).cuda()
        for prec in ("tf32", "fp32"):
            out = dg.sddmm(x, x, precision=prec)
            torch.cuda.synchronize()
            c = Csr.of(n, g.node_pointer, g.edge_list)
            want = O.sddmm(c, x.cpu().numpy(), x.cpu().numpy(), tf32=prec == "tf32")
            err = np.abs(out.cpu().numpy() - want).max() / np.abs(want).max()
            print(n, d, prec, "err", err, dg.panel_info(d)["dense_entries"], flush=True)
