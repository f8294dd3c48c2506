"""One process of tests/test_gpu_variants.py: run a fixed set of calls under
the environment the test chose and save the outputs.
    python tests/_variant_run.py sddmm|agnn|hub|spmm <out.npz>"""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import torch  # noqa: E402

import paper_2412_12218_b200 as sg  # noqa: E402
from paper_2412_12218_b200.device import DeviceGraph  # noqa: E402


def graphs():
    return {"local": sg.synth_graph(4000, 40.0, alpha=0.0, p_local=0.9, band=4.0, seed=31),
            "hubs": sg.synth_graph(6000, 25.0, alpha=2.0, p_local=0.6, band=4.0, seed=32)}


def sddmm():
    out = {}
    for name, g0 in graphs().items():
        for weighted in (False, True):
            g = sg.gcn_normalize_values(g0) if weighted else g0
            t16 = sg.reblock(sg.sgt_transform(g), 16)
            for d in (16, 32, 64):
                x = sg.dense_random(g.num_nodes, d, 40 + d)
                y = sg.dense_random(g.num_nodes, d, 41 + d)
                for prec in ("fp32", "tf32"):
                    out[f"{name}_{int(weighted)}_{d}_{prec}"] = sg.sddmm_hybrid(t16, x, y, precision=prec)
                ov = np.random.default_rng(d).uniform(-1, 1, g.num_edges).astype(np.float32)
                out[f"{name}_{int(weighted)}_{d}_ov"] = sg.sddmm_hybrid(t16, x, y, edge_values=ov)
    return out


def agnn():
    out = {}
    g = sg.synth_graph(30000, 60.0, alpha=3.0, p_local=0.9, band=4.0, seed=7)
    dg = DeviceGraph.from_csr(g.node_pointer, g.edge_list)
    assert dg.panel_info(32)["dense_entries"] > 0
    for d in (32, 20, 64):
        x = torch.from_numpy(sg.dense_random(g.num_nodes, d, 9 + d)).cuda()
        for prec in ("tf32", "fp32"):
            r = dg.agnn_forward(x, np.array([1.0, -0.5, 2.0], np.float32), precision=prec, mode=2)
            out[f"{prec}_{d}"] = r.cpu().numpy()
    return out


def spmm():
    out = {}
    for name, g0 in graphs().items():
        for weighted in (False, True):
            g = sg.gcn_normalize_values(g0) if weighted else g0
            dg = DeviceGraph.from_csr(g.node_pointer, g.edge_list, g.values)
            assert dg.panel_info()["dense_entries"] > 0
            for d in (32, 48, 64, 96, 128):
                x = torch.from_numpy(sg.dense_random(g.num_nodes, d, 50 + d)).cuda()
                out[f"{name}_{int(weighted)}_{d}"] = dg.spmm(x, precision="tf32").cpu().numpy()
            ov = torch.from_numpy(np.random.default_rng(5).uniform(-1, 1, g.num_edges).astype(np.float32)).cuda()
            x = torch.from_numpy(sg.dense_random(g.num_nodes, 64, 7)).cuda()
            out[f"{name}_{int(weighted)}_ov"] = dg.spmm(x, edge_values=ov, precision="tf32").cpu().numpy()
    return out


def hub():
    from oracle.oracle import Csr, Oracle

    n = (1 << 20) + 50_000
    rows = [np.arange(n, dtype=np.uint32)]  # row 0: every column, positions up to n - 1
    tail = np.arange(n - 200, n, dtype=np.uint32)
    for i in range(1, 5):  # rows 1-4 share the last 200 columns: dense in panel 0
        rows.append(np.concatenate([np.array([i], np.uint32), tail]))
    deg = np.ones(n, np.uint64)
    deg[0] = n
    deg[1:5] = 201
    np_ = np.zeros(n + 1, np.uint64)
    np_[1:] = np.cumsum(deg)
    el = np.concatenate(rows + [np.arange(5, n, dtype=np.uint32)])
    assert el.size == int(np_[-1])
    g = sg.CsrGraph(n, np_, el)
    t16 = sg.reblock(sg.sgt_transform(g), 16)
    d = 16
    x = sg.dense_random(n, d, 3)
    y = sg.dense_random(n, d, 4)
    c = Csr.of(n, np_, el)
    O = Oracle()
    out = {"dpos_row_edges": np.array(n)}
    for prec, tf in (("fp32", False), ("tf32", True)):
        out[prec] = sg.sddmm_hybrid(t16, x, y, precision=prec)
        out[prec + "_oracle"] = O.sddmm(c, x, y, tf32=tf)
    return out


if __name__ == "__main__":
    what, path = sys.argv[1], sys.argv[2]
    res = {"sddmm": sddmm, "agnn": agnn, "hub": hub, "spmm": spmm}[what]()
    np.savez(path, **res)
