"""Diagnostics for the panel SpMM: per-graph error, dense-only / sparse-only cases."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2412_12218_b200 as sg
from oracle.oracle import Csr, Oracle
O = Oracle()

def mre(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))

def run(name, g, d=32, prec="fp32"):
    print("start", name, flush=True)
    t = sg.sgt_transform(g)
    x = sg.dense_random(g.num_nodes, d, 1)
    c = Csr.of(g.num_nodes, g.node_pointer, g.edge_list, g.values)
    want = O.spmm(c, x, tf32=(prec == "tf32"))
    got = sg.spmm_hybrid(t, x, precision=prec)
    err = np.abs(got - want).max(axis=1)
    bad = np.nonzero(err > 1e-4 * max(np.abs(want).max(), 1e-30))[0]
    print(f"{name} d={d} {prec}: mre={mre(got, want):.3e} bad_rows={len(bad)}/{g.num_nodes} first={bad[:10]}")
    if len(bad):
        r = bad[0]
        print("  got ", got[r, :8]); print("  want", want[r, :8])
    return got, want, x

n = 128
# 1) diagonal only: every column a singleton -> sparse path only
g = sg.csr_from_coo(n, list(range(n)), list(range(n)))
run("diag(sparse only)", g)
# 2) every row has col 0 and col 1 -> 2 dense columns, no sparse
rows = sum([[r, r] for r in range(n)], []); cols = [0, 1] * n
run("2dense", sg.csr_from_coo(n, rows, cols))
# 3) full 128x128 block
rows = [r for r in range(n) for c in range(n)]; cols = [c for r in range(n) for c in range(n)]
gf = sg.csr_from_coo(n, rows, cols)
run("full128", gf)
run("full128 tf32", gf, prec="tf32")
run("full128 d64", gf, d=64)
# 4) row r has cols r, r+1 (banded) 
rows = sum([[r, r+1] for r in range(n-1)], []) ; 
g4 = sg.csr_from_coo(n, [r for r in range(n-1) for _ in range(2)], [c for r in range(n-1) for c in (r, r+1)])
run("band2", g4)
# 5) only row 0 has 32 cols 0..31; rows 1 also cols 0..31
rows = [r for r in range(2) for c in range(32)]; cols = [c for r in range(2) for c in range(32)]
run("2rows32", sg.csr_from_coo(n, rows, cols))
rows = [r for r in range(16) for c in range(8)]; cols = [c for r in range(16) for c in range(8)]
g6 = sg.csr_from_coo(n, rows, cols)
got, want, x = run("16x8", g6)
print(np.round(got[:3,:8],3)); print(np.round(want[:3,:8],3))

# ---- format check against a numpy restatement
from paper_2412_12218_b200.device import DeviceGraph
def check_format(name, g):
    dg = DeviceGraph.from_csr(g.node_pointer, g.edge_list, g.values)
    A = dg.panel_arrays(); info = dg.panel_info()
    npz = g.node_pointer.astype(np.int64); el = g.edge_list.astype(np.int64)
    n = g.num_nodes
    rows = np.repeat(np.arange(n), np.diff(npz))
    nd = 0; ns = 0; ok = True
    for p in range((n + 127) // 128):
        m = (rows // 128) == p
        cols, cnt = np.unique(el[m], return_counts=True)
        dense = cols[cnt >= 2]
        c0, c1 = A["chunk_ptr"][p], A["chunk_ptr"][p + 1]
        dc = A["dense_cols"][c0 * 32:c1 * 32]
        if not np.array_equal(dc[:len(dense)], dense) or np.any(dc[len(dense):] != 0xFFFFFFFF):
            print("  dense cols mismatch panel", p, dc[:8], dense[:8]); ok = False
        ents = []
        for c in range(c0, c1):
            e = A["dense_entries"][A["chunk_off"][c]:A["chunk_off"][c + 1]]
            e = e[(e & 0x1000) == 0]
            ents += [((c - c0) * 32 + (w & 31), (w >> 5) & 127) for w in e]
        nd += len(ents)
        want = sorted((int(np.searchsorted(dense, el[i])), int(rows[i] % 128)) for i in np.nonzero(m)[0] if el[i] in set(dense.tolist()))
        if sorted(ents) != want:
            print("  entries mismatch panel", p, len(ents), len(want)); ok = False
    print(name, "format ok" if ok else "FORMAT BAD", info)
rows = sum([[r, r] for r in range(128)], []); cols = [0, 1] * 128
check_format("2dense", sg.csr_from_coo(128, rows, cols))
check_format("powerlaw", sg.synth_graph(600, 10.0, alpha=2.0, p_local=0.9, band=4.0, seed=3))
