"""GPU parity of the 128-row panel SpMM (panel.cu, tcgen05 + TMEM) -- the
kernel behind the default plan (ratio 1.0) of spmm_hybrid.

Bars (as tests/test_gpu_parity.py):
  * FP32 (4-term TF32 split): max_rel_err <= 1e-5 vs the CPU oracle
    (oracle_spmm order, the reference's fp32 arithmetic);
  * TF32 vs the oracle's TF32 mode (identical rounded operands, exact
    products; only the fp32 summation order differs): max_rel_err <= 1e-5;
  * hub panels: <= 2x the sequential oracle's own error vs a float64 sum.
Shapes cover ragged last panels (n % 128 != 0), empty rows, panels with no
dense column, hub panels with hundreds of dense chunks (TMEM accumulator
reuse), all-dense blocks, feature slices (d > 64) and partial slices.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2412_12218_b200 as sg  # noqa: E402
from paper_2412_12218_b200.device import DeviceGraph  # noqa: E402
from oracle.oracle import Csr, Oracle  # noqa: E402

O = Oracle()


def mre(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30)) if a.size else 0.0


def coo_graph(n, rows, cols, vals=None):
    g = sg.csr_from_coo(n, rows, cols)
    if vals is not None:
        g = sg.CsrGraph(g.num_nodes, g.node_pointer, g.edge_list,
                        sg.dense_random(1, g.num_edges, vals)[0])
    return g


def graphs():
    out = []
    # power-law with locality: dense bands + singleton long-range columns
    out.append(("powerlaw", sg.synth_graph(3000, 20.0, alpha=2.0, p_local=0.9, band=4.0, seed=3)))
    # uniform random: almost everything sparse
    out.append(("uniform", sg.synth_graph(2000, 8.0, alpha=0.0, p_local=0.0, seed=4)))
    rng = np.random.default_rng(5)
    # all-dense 128x128 blocks, ragged n, empty rows
    n = 300
    rows, cols = [], []
    for r in range(n):
        if r % 7 == 3:
            continue  # empty row
        b = (r // 128) * 128
        c = np.arange(b, min(b + 128, n))
        rows += [r] * len(c)
        cols += list(c)
    out.append(("blockdense", coo_graph(n, rows, cols, vals=11)))
    # hub panel: 128 rows x 6000 shared columns (~190 dense chunks)
    n = 7000
    rows, cols = [], []
    for r in range(n):
        k = 3000 if r < 128 else 3
        c = np.unique(rng.integers(0, n, k))
        rows += [r] * len(c)
        cols += list(c)
    out.append(("hubpanel", coo_graph(n, rows, cols, vals=12)))
    return out


GRAPHS = graphs()


def oracle_csr(g):
    return Csr.of(g.num_nodes, g.node_pointer, g.edge_list, g.values)


@pytest.mark.parametrize("name,g", GRAPHS, ids=[n for n, _ in GRAPHS])
@pytest.mark.parametrize("d", [4, 16, 32, 48, 64, 100, 128])
def test_panel_spmm_fp32(name, g, d):
    t = sg.sgt_transform(g)
    x = sg.dense_random(g.num_nodes, d, d + 7)
    want = O.spmm(oracle_csr(g), x)
    got = sg.spmm_hybrid(t, x)
    if name == "hubpanel":
        deg = np.diff(g.node_pointer.astype(np.int64))
        rows = np.repeat(np.arange(g.num_nodes), deg)
        v = np.ones(g.num_edges) if g.values is None else g.values.astype(np.float64)
        exact = np.zeros((g.num_nodes, d))
        np.add.at(exact, rows, v[:, None] * x[g.edge_list].astype(np.float64))
        assert mre(got, exact) <= 2 * mre(want, exact) + 1e-6
        assert mre(got, want) <= 1e-4
    else:
        assert mre(got, want) <= 1e-5


@pytest.mark.parametrize("name,g", GRAPHS, ids=[n for n, _ in GRAPHS])
@pytest.mark.parametrize("d", [16, 32, 64, 128])
def test_panel_spmm_tf32(name, g, d):
    t = sg.sgt_transform(g)
    x = sg.dense_random(g.num_nodes, d, d + 9)
    want = O.spmm(oracle_csr(g), x, tf32=True)
    got = sg.spmm_hybrid(t, x, precision="tf32")
    assert mre(got, want) <= (1e-4 if name == "hubpanel" else 1e-5)


@pytest.mark.parametrize("name,g", GRAPHS[:3], ids=[n for n, _ in GRAPHS[:3]])
def test_panel_vs_tile16_and_override(name, g):
    """Explicit full plan (cut == block_partition) routes to the 16-row tile
    kernel; the default (no cut) to the panel kernel: same products."""
    dg = DeviceGraph.from_csr(g.node_pointer, g.edge_list, g.values)
    t = sg.sgt_transform(g)
    x = torch.from_numpy(sg.dense_random(g.num_nodes, 32, 1)).cuda()
    a = dg.spmm(x)
    b = dg.spmm(x, cut=np.asarray(t.block_partition, np.uint32))
    assert mre(a.cpu().numpy(), b.cpu().numpy()) <= 1e-5
    ev = sg.dense_random(1, g.num_edges, 2)[0]
    want = O.spmm(Csr.of(g.num_nodes, g.node_pointer, g.edge_list, ev), x.cpu().numpy())
    got = dg.spmm(x, edge_values=torch.from_numpy(ev).cuda())
    assert mre(got.cpu().numpy(), want) <= 1e-5


def test_panel_strided_and_deterministic():
    g = GRAPHS[0][1]
    dg = DeviceGraph.from_csr(g.node_pointer, g.edge_list, g.values)
    big = torch.from_numpy(sg.dense_random(g.num_nodes, 72, 3)).cuda()
    x = big[:, 4:68]  # ldx = 72, 16-byte aligned start
    out = torch.zeros((g.num_nodes, 80), device="cuda")
    dg.spmm(x, out=out[:, 8:72])
    want = O.spmm(oracle_csr(g), x.cpu().numpy())
    assert mre(out[:, 8:72].cpu().numpy(), want) <= 1e-5
    assert torch.all(out[:, :8] == 0) and torch.all(out[:, 72:] == 0)
    a = dg.spmm(x.contiguous())
    for _ in range(3):
        assert torch.equal(a, dg.spmm(x.contiguous()))


def test_panel_nonfinite():
    g = sg.CsrGraph(200, np.array([0] + [2] * 200), np.array([0, 1]), np.ones(2, np.float32))
    t = sg.sgt_transform(g)
    x = np.zeros((200, 32), np.float32)
    x[1, 5] = np.inf
    with pytest.raises(sg.NonFiniteError):
        sg.spmm_hybrid(t, x)


def test_panel_nonfinite_dense_columns():
    # the non-finite row is reached through a dense panel column (4 edges in
    # the panel): flagged by the tensor-core kernel's epilogue check, also for
    # rows that have no CUDA-core edges at all
    n = 200
    cols = [1, 1, 1, 1]
    npz = np.array([0, 1, 2, 3, 4] + [4] * (n - 4))
    g = sg.CsrGraph(n, npz, np.array(cols), np.ones(4, np.float32))
    t = sg.sgt_transform(g)
    x = np.zeros((n, 32), np.float32)
    x[1, 7] = np.inf
    for prec in ("fp32", "tf32"):
        with pytest.raises(sg.NonFiniteError):
            sg.spmm_hybrid(t, x, precision=prec)
    x[1, 7] = 1.0
    sg.spmm_hybrid(t, x)  # finite: no error


@pytest.mark.parametrize("prec", ["fp32", "tf32"])
@pytest.mark.parametrize("order", [0, 1])
def test_gcn_nonfinite_and_tf32_chain(prec, order):
    # gcn_forward: the GEMM epilogue checks the output and TF32-rounds the next
    # SpMM's input (reference order); overflow raises NonFiniteError
    g = sg.gcn_normalize_values(GRAPHS[0][1])
    t = sg.sgt_transform(g)
    n = g.num_nodes
    x = sg.dense_random(n, 24, 5)
    w1 = sg.dense_random(24, 24, 6) * np.float32(0.2)
    w2 = sg.dense_random(24, 16, 7) * np.float32(0.2)
    got = sg.gcn_forward(t, x, [(w1, True), (w2, False)], precision=prec, order=order)
    want = O.gcn_forward(oracle_csr(g), x, [(w1, True), (w2, False)], tf32=prec == "tf32")
    assert mre(got, want) <= (1e-5 if prec == "fp32" else 2e-3)
    big = np.full((24, 24), 1e38, np.float32)
    xp = np.abs(x) + np.float32(0.5)  # positive rows: every sum overflows fp32
    with pytest.raises(sg.NonFiniteError):
        sg.gcn_forward(t, xp, [(big, True), (w2, False)], precision=prec, order=order)


def test_agnn_default_mode_fallbacks():
    # mode 2 (and the auto default) falls back to fused 16-row windows for |beta| > 40
    # and to the kernel chain for d > 64; results stay within the FP32 bar
    g = GRAPHS[0][1]
    t = sg.sgt_transform(g)
    ga = Csr.of(g.num_nodes, g.node_pointer, g.edge_list)
    for d, betas in ((80, [1.0, 0.5]), (32, [60.0])):
        x = sg.dense_random(g.num_nodes, d, d)
        want, _ = O.agnn_forward(ga, x, betas)
        for mode in (2, 3):
            got = sg.agnn_forward(t, x, betas, mode=mode)
            assert mre(got, want) <= 1e-5, (d, betas, mode)


# ------------------------------------------------------------ AGNN, mode 2
# agnn_panel.cu: tensor-core attention over dense panel columns, CUDA-core
# attention over sparse edges.  Bars: FP32 <= 1e-5 (as test_gpu_parity.py),
# TF32 vs the oracle's TF32 mode <= 2e-3 (the tolerance the fused modes use:
# rounded logits / attention, tile_exec.cpp:386,402).
@pytest.mark.parametrize("name,g", GRAPHS, ids=[n for n, _ in GRAPHS])
@pytest.mark.parametrize("d", [16, 32, 41, 64])
def test_panel_agnn(name, g, d):
    t = sg.sgt_transform(g)
    ga = Csr.of(g.num_nodes, g.node_pointer, g.edge_list)
    x = sg.dense_random(g.num_nodes, d, d + 3)
    betas = [1.0, -0.7, 2.5]
    want, zw = O.agnn_forward(ga, x, betas)
    got, zg = sg.agnn_forward(t, x, betas, mode=2, return_zeros=True)
    assert mre(got, want) <= 1e-5
    assert zg == zw
    want_t, _ = O.agnn_forward(ga, x, betas, tf32=True)
    assert mre(sg.agnn_forward(t, x, betas, precision="tf32", mode=2), want_t) <= 2e-3


def test_panel_agnn_deterministic_and_fallback():
    g = GRAPHS[3][1]  # hub panel: segments of a hub row combine in order
    dg = DeviceGraph.from_csr(g.node_pointer, g.edge_list)
    x = torch.from_numpy(sg.dense_random(g.num_nodes, 32, 4)).cuda()
    a = dg.agnn_forward(x, [1.0, 1.0], mode=2)
    for _ in range(2):
        assert torch.equal(a, dg.agnn_forward(x, [1.0, 1.0], mode=2))
    # |beta| beyond the fixed-offset envelope: runs the fused 16-row mode
    ga = Csr.of(g.num_nodes, g.node_pointer, g.edge_list)
    want, _ = O.agnn_forward(ga, x.cpu().numpy(), [60.0])
    got = dg.agnn_forward(x, [60.0], mode=2).cpu().numpy()
    assert mre(got, want) <= 1e-5


# ------------------------------------------------------- panel format (build)
def _panel_restatement(g):
    """numpy restatement of build_panels (panel.cu): per 128-row panel the
    columns with >= 2 edges are dense (sorted, padded to 32 per panel), a
    chunk's entries in (row, column) order (each carrying its swizzled A-tile
    offset, padded to a multiple of 4 with zeros on empty positions), row
    masks, sparse edges per row in CSR order."""
    n = g.num_nodes
    npz = g.node_pointer.astype(np.int64)
    el = g.edge_list.astype(np.int64)
    rows = np.repeat(np.arange(n), np.diff(npz))
    vals = np.ones(len(el), np.float32) if g.values is None else g.values
    P = (n + 127) // 128
    dcols, cptr, masks, ents, sparse = [], [0], [], [], [[] for _ in range(n)]
    for p in range(P):
        m = (rows // 128) == p
        cols, cnt = np.unique(el[m], return_counts=True)
        dense = cols[cnt >= 2]
        nch = (len(dense) + 31) // 32
        cptr.append(cptr[-1] + nch)
        pad = np.full(nch * 32, 0xFFFFFFFF, np.uint64)
        pad[:len(dense)] = dense
        dcols.append(pad)
        slot = {int(c): i for i, c in enumerate(dense)}
        cm = np.zeros((nch, 128), np.uint32)
        ce = [[] for _ in range(nch)]
        for e in np.nonzero(m)[0]:
            r, c = int(rows[e]), int(el[e])
            if c in slot:
                s = slot[c]
                cm[s // 32, r % 128] |= np.uint32(1 << (s % 32))
                ce[s // 32].append((r % 128, s % 32, vals[e]))
            else:
                sparse[r].append((c, vals[e]))
        masks.append(cm)
        ents += [sorted(x, key=lambda t: (t[0], t[1])) for x in ce]
    return (np.array(cptr, np.uint32), np.concatenate(dcols) if dcols else np.zeros(0),
            np.concatenate(masks) if masks else np.zeros((0, 128)), ents, sparse)


@pytest.mark.parametrize("name,g", GRAPHS[:3], ids=[n for n, _ in GRAPHS[:3]])
def test_panel_format_matches_restatement(name, g):
    dg = DeviceGraph.from_csr(g.node_pointer, g.edge_list, g.values)
    A = dg.panel_arrays()
    cptr, dcols, masks, ents, sparse = _panel_restatement(g)
    np.testing.assert_array_equal(A["chunk_ptr"], cptr)
    np.testing.assert_array_equal(A["dense_cols"].astype(np.uint64), dcols)
    off = A["chunk_off"].astype(np.int64)
    def pos(w):  # swizzled K-major A-tile word offset (panel.cu a_word) -> (row, k)
        o = int(w) & 0xFFF
        row = (o >> 8) * 8 + ((o >> 5) & 7)
        return row, ((((o & 31) >> 2) ^ (row & 7)) << 2) | (o & 3)
    for c, want in enumerate(ents):
        got = A["dense_entries"][off[c]:off[c + 1]]
        assert len(got) == (len(want) + 3) // 4 * 4, c
        real, pad = got[:len(want)], got[len(want):]
        assert [pos(w) for w in real] == [(r, k) for r, k, _ in want], c
        tf = np.array([O.tf32_round_value(float(v)) for _, _, v in want], np.float32)
        np.testing.assert_array_equal((real & 0xFFFFE000).view(np.float32), tf)
        taken = {(r, k) for r, k, _ in want}
        for w in pad:  # value 0 on an empty position
            assert int(w) & 0xFFFFE000 == 0 and pos(w) not in taken, c
    sp = A["sparse_ptr"].astype(np.int64)
    se = A["sparse_entries"].reshape(-1, 2)
    for r in range(g.num_nodes):
        got = [(int(c), float(np.uint32(v).view(np.float32))) for c, v in se[sp[r]:sp[r + 1]]]
        assert got == [(c, float(v)) for c, v in sparse[r]], r


def _hub_row_graph():
    """Banded rows plus hub rows whose edges are mostly singleton (CUDA-core)
    columns: > kSegEdges sparse edges, so each hub row is split into segments
    whose partials agnn_long_rows_kernel combines in order (on the second
    stream, beside agnn_final_kernel, in the concurrent layer)."""
    rng = np.random.default_rng(17)
    n = 20000
    rows, cols = [], []
    hubs = {0, 3, 4, 5000, 9001, 19999}
    for r in range(n):
        if r in hubs:
            c = np.unique(rng.integers(0, n, 3000))
        else:
            c = np.unique(np.clip(r + rng.integers(-6, 7, 12), 0, n - 1))
        rows += [r] * len(c)
        cols += list(c)
    return coo_graph(n, rows, cols)


def test_panel_agnn_hub_rows():
    g = _hub_row_graph()
    dg = DeviceGraph.from_csr(g.node_pointer, g.edge_list)
    assert dg.panel_info(32)["long_rows"] >= 6 and dg.panel_info(32)["segments"] > 6
    t = sg.sgt_transform(g)
    ga = Csr.of(g.num_nodes, g.node_pointer, g.edge_list)
    betas = [1.0, -0.7, 2.5]  # three layers: hub rows' next-layer operands feed layer 2, 3
    for d in (32, 20):
        x = sg.dense_random(g.num_nodes, d, 40 + d)
        want, zw = O.agnn_forward(ga, x, betas)
        got, zg = sg.agnn_forward(t, x, betas, mode=2, return_zeros=True)
        assert mre(got, want) <= 1e-5 and zg == zw
        want_t, _ = O.agnn_forward(ga, x, betas, tf32=True)
        assert mre(sg.agnn_forward(t, x, betas, precision="tf32", mode=2), want_t) <= 2e-3
        xt = torch.from_numpy(x).cuda()
        a = dg.agnn_forward(xt, betas, precision="tf32", mode=2)
        for _ in range(3):  # the two streams' kernels write disjoint rows: run to run identical
            assert torch.equal(a, dg.agnn_forward(xt, betas, precision="tf32", mode=2))


@pytest.mark.parametrize("prec", ["fp32", "tf32"])
def test_gcn_split_k_gemm(prec):
    # Cora-like first layer (few 128-row tiles, K = 1433): the update GEMM
    # splits K and reduces the splits in order; its epilogue (ReLU, TF32
    # rounding, non-finite check) runs in the reduction
    g = sg.gcn_normalize_values(GRAPHS[1][1])  # 2,000 nodes
    t = sg.sgt_transform(g)
    n = g.num_nodes
    x = sg.dense_random(n, 1433, 8)
    w1 = sg.dense_random(1433, 16, 9) * np.float32(0.05)
    w2 = sg.dense_random(16, 7, 10)
    for order in (0, 1):
        got = sg.gcn_forward(t, x, [(w1, True), (w2, False)], precision=prec, order=order)
        want = O.gcn_forward(oracle_csr(g), x, [(w1, True), (w2, False)], tf32=prec == "tf32")
        assert mre(got, want) <= (1e-5 if prec == "fp32" else 2e-3)
    big = np.full((1433, 16), 1e36, np.float32)
    xp = np.abs(x) + np.float32(0.5)  # every product sum overflows fp32
    for order in (0, 1):
        with pytest.raises(sg.NonFiniteError):
            sg.gcn_forward(t, xp, [(big, True), (w2, False)], precision=prec, order=order)
