"""Generate tests/golden/golden.npz from the UNMODIFIED reference.

Run in the build container (needs /root/reference and `make -C oracle ref`):

    python tests/golden/make_golden.py

Every array stored here is an output of the reference library itself
(oracle/_ref/libsgtk_ref.so built from /root/reference/proj/src), on inputs
that are also stored, so tests can pin both our CPU oracle
(tests/test_oracle_golden.py) and the CUDA path (tests/test_gpu_parity.py)
against the reference on a box where /root/reference does not exist.

Cases mirror the reference's own known-answer tests (file:line in each key's
comment) plus seeded random graphs at the sizes its property tests use.
"""

from __future__ import annotations

import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)

from oracle.oracle import Csr, OracleError, RefLib  # noqa: E402

OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden.npz")
OUT_CONFIGS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "configs.npz")


def graph_of(n, triples, weighted=False):
    """csr_from_triples (csr_graph.cpp:41-60): stable (row, col) sort."""
    if not triples:
        return Csr.of(n, np.zeros(n + 1, np.uint64), np.zeros(0, np.uint32),
                      np.zeros(0, np.float32) if weighted else None)
    t = sorted(enumerate(triples), key=lambda it: (it[1][0], it[1][1], it[0]))
    rows = np.array([r for _, (r, c, v) in t], np.int64)
    cols = np.array([c for _, (r, c, v) in t], np.uint32)
    vals = np.array([v for _, (r, c, v) in t], np.float32)
    np_ = np.zeros(n + 1, np.uint64)
    np_[1:] = np.cumsum(np.bincount(rows, minlength=n))
    return Csr.of(n, np_, cols, vals if weighted else None)


def random_csr(n, avg_deg, seed, weighted=False, local=0.0):
    """Seeded sorted-unique CSR with optional locality (builder-defined)."""
    rng = np.random.default_rng(seed)
    deg = rng.poisson(avg_deg, n).clip(0, n)
    np_ = np.zeros(n + 1, np.uint64)
    cols = []
    for r in range(n):
        k = int(deg[r])
        if local > 0:
            near = rng.integers(max(0, r - 24), min(n, r + 25), k)
            far = rng.integers(0, n, k)
            c = np.where(rng.random(k) < local, near, far)
        else:
            c = rng.integers(0, n, k)
        c = np.unique(c)
        cols.append(c)
        np_[r + 1] = np_[r] + c.size
    el = np.concatenate(cols).astype(np.uint32) if cols else np.zeros(0, np.uint32)
    vals = rng.uniform(-1, 1, el.size).astype(np.float32) if weighted else None
    return Csr.of(n, np_, el, vals)


def main():
    R = RefLib()
    G: dict[str, np.ndarray] = {}

    def put_csr(key, g: Csr):
        G[f"{key}/n"] = np.array(g.num_nodes, np.uint64)
        G[f"{key}/node_pointer"] = g.node_pointer
        G[f"{key}/edge_list"] = g.edge_list
        if g.values is not None:
            G[f"{key}/values"] = g.values

    def put_transform(key, g: Csr, blk_h=16, blk_w=8):
        th = R.transform_handle(g, blk_h, blk_w)
        t = R.transform_fields(th)
        for k, v in t.fields().items():
            G[f"{key}/t{blk_h}x{blk_w}/{k}"] = v
        G[f"{key}/t{blk_h}x{blk_w}/block_counter"] = np.array(t.block_counter, np.uint64)
        return th

    # --- translator KATs -------------------------------------------------
    # identity 16 -> 1 window, 2 tiles (test_sgt_transform.cpp:47-61)
    g = graph_of(16, [(i, i, 1.0) for i in range(16)])
    put_csr("kat_identity16", g)
    th = put_transform("kat_identity16", g)
    s = np.zeros(3, np.uint64)
    d = np.zeros(1, np.float64)
    R.L.ref_block_stats(th.ptr, s.ctypes.data, d.ctypes.data)
    G["kat_identity16/block_stats"] = s
    G["kat_identity16/density"] = d
    G["kat_identity16/reblock16_bp"] = R.transform_fields(R.reblock_handle(th, 16)).block_partition
    a, idx = R.gather_tile(th, 0, 0, 16, 8)
    G["kat_identity16/gather_tile00_a"], G["kat_identity16/gather_tile00_idx"] = a, idx
    # window compression (test_sgt_transform.cpp:63-80)
    g = graph_of(31, [(0, 5, 1), (0, 9, 1), (1, 5, 1), (1, 30, 1)])
    put_csr("kat_compress", g)
    put_transform("kat_compress", g)
    # reblock 17 cols -> 2 tiles at width 16 (test_sgt_transform.cpp:99-104)
    g = graph_of(17, [(0, c, 1) for c in range(17)])
    put_csr("kat_reblock17", g)
    th = put_transform("kat_reblock17", g)
    G["kat_reblock17/reblock16_bp"] = R.transform_fields(R.reblock_handle(th, 16)).block_partition
    # ragged tile sentinel (test_tile_exec.cpp:50-63)
    g = graph_of(20, [(0, 3, 1), (1, 7, 1), (2, 11, 1)])
    put_csr("kat_ragged", g)
    th = put_transform("kat_ragged", g)
    a, idx = R.gather_tile(th, 0, 0, 16, 8)
    G["kat_ragged/gather_tile00_a"], G["kat_ragged/gather_tile00_idx"] = a, idx
    # blockdense(4 windows, 2 tiles): 8 blocks, density 1 (test_bench_cli.cpp:28-38 shape)
    rng = np.random.default_rng(3)
    tr = []
    for w in range(4):
        cols = np.sort(rng.choice(64, 16, replace=False))
        tr += [(w * 16 + r, int(c), 1.0) for r in range(16) for c in cols]
    g = graph_of(64, tr)
    put_csr("kat_blockdense", g)
    put_transform("kat_blockdense", g)

    # --- kernel KATs -----------------------------------------------------
    # 2-cycle swap (test_tile_exec.cpp:88-95)
    g = graph_of(2, [(0, 1, 1.0), (1, 0, 1.0)])
    put_csr("kat_2cycle", g)
    th = R.transform_handle(g)
    x = np.array([[1, 2], [3, 4]], np.float32)
    G["kat_2cycle/x"] = x
    G["kat_2cycle/spmm"] = R.spmm(th, 2, x)
    # identity spmm exact (test_tile_exec.cpp:79-86)
    g = graph_of(16, [(i, i, 1.0) for i in range(16)])
    th = R.transform_handle(g)
    x = R.dense_random(16, 16, 99)
    G["kat_identity_spmm/x"] = x
    G["kat_identity_spmm/out"] = R.spmm(th, 16, x)
    # sddmm basics (test_tile_exec.cpp:208-233)
    for key, (n, tri, w, xs, ys) in {
        "kat_sddmm_orth": (2, [(0, 1, 1.0)], False, {(0, 0): 1.0}, {(1, 1): 1.0}),
        "kat_sddmm_aligned": (3, [(1, 2, 1.0)], False, {(1, 2): 1.0}, {(2, 2): 1.0}),
        "kat_sddmm_weight": (2, [(0, 1, 0.5)], True, "ones", "ones"),
    }.items():
        g = graph_of(n, tri, weighted=w)
        dd = 4 if key == "kat_sddmm_aligned" else 2
        x = np.ones((n, dd), np.float32) if xs == "ones" else np.zeros((n, dd), np.float32)
        y = np.ones((n, dd), np.float32) if ys == "ones" else np.zeros((n, dd), np.float32)
        if xs != "ones":
            for (i, j), v in xs.items():
                x[i, j] = v
            for (i, j), v in ys.items():
                y[i, j] = v
        put_csr(key, g)
        th16 = R.reblock_handle(R.transform_handle(g), 16)
        G[f"{key}/x"], G[f"{key}/y"] = x, y
        G[f"{key}/out"] = R.sddmm(th16, g.num_edges, x, y)
    # softmax closed forms (test_gnn.cpp:110-134)
    g1 = graph_of(2, [(0, 1, 1)])
    g2 = graph_of(3, [(0, 1, 1), (0, 2, 1)])
    for key, (g, lg) in {
        "kat_softmax_single": (g1, [3.25]),
        "kat_softmax_equal": (g2, [0.7, 0.7]),
        "kat_softmax_ln2": (g2, [0.0, float(np.log(np.float32(2.0)))]),
        "kat_softmax_extreme": (g2, [200.0, -200.0]),
    }.items():
        put_csr(key, g)
        lg = np.array(lg, np.float32)
        G[f"{key}/logits"] = lg
        G[f"{key}/out"] = R.edge_softmax(g, lg)
    # overflow -> NonFiniteError (test_tile_exec.cpp:179-186)
    g = graph_of(4, [(0, c, 1.0) for c in range(4)], weighted=True)
    th = R.transform_handle(g)
    try:
        R.spmm(th, 4, np.full((4, 1), 1e38, np.float32))
        code = 0
    except OracleError as e:
        code = e.code
    G["kat_overflow/status"] = np.array(code, np.int32)
    # gcn normalisation frozen value 0.40824829 (test_graph_io.cpp:209-246)
    g = graph_of(3, [(0, 0, 1), (0, 1, 1), (1, 0, 1), (1, 1, 1), (1, 2, 1), (2, 1, 1), (2, 2, 1)])
    put_csr("kat_gcnnorm_path", g)
    G["kat_gcnnorm_path/values_out"] = R.gcn_normalize_values(g).values
    # agnn zero-norm rows (test_gnn.cpp:199-215)
    g = graph_of(3, [(i, i, 1.0) for i in range(3)])
    put_csr("kat_agnn_zero", g)
    x = np.zeros((3, 4), np.float32)
    x[0, 0] = 1.0
    out, z = R.agnn_forward(R.transform_handle(g), x, [1.0])
    G["kat_agnn_zero/x"], G["kat_agnn_zero/out"] = x, out
    G["kat_agnn_zero/zeros"] = np.array(z, np.uint64)
    # TF32 KATs: tie, above-tie, saturation corner, specials, random patterns
    # (test_tile_exec.cpp:273-302, acceptance.cpp:262-276)
    special = np.array([1.0, -2.0, 0.0, -0.0, 1 + 2**-11, 1 + 2**-11 + 2**-20,
                        3.4028235e38, -3.4028235e38, np.inf, -np.inf, 1e-40, -3.14159],
                       np.float32)
    rng = np.random.default_rng(0xF32)
    bits = rng.integers(0, 2**32, 20000, dtype=np.uint64).astype(np.uint32)
    samples = np.concatenate([special, bits.view(np.float32)])
    samples = samples[~np.isnan(samples)]
    G["kat_tf32/in"] = samples
    G["kat_tf32/out"] = np.array([R.tf32_round_value(float(v)) for v in samples], np.float32)
    # DenseMatrix::random stream (dense_matrix.hpp:43-50)
    G["kat_dense_random/seed8_5x7"] = R.dense_random(5, 7, 8)
    G["kat_dense_random/seed3_4x3_m01"] = R.dense_random(4, 3, 3, -0.1, 0.1)

    # --- seeded random graphs -------------------------------------------
    specs = [  # (n, avg_deg, weighted, local, d)
        (37, 3.0, False, 0.0, 8),
        (128, 6.0, True, 0.0, 16),
        (257, 8.0, False, 0.8, 32),
        (300, 12.0, True, 0.5, 64),
        (200, 5.0, False, 0.0, 18),
        (96, 40.0, True, 0.9, 25),
    ]
    for i, (n, deg, w, loc, dim) in enumerate(specs):
        key = f"rand{i}"
        g = random_csr(n, deg, 1000 + i, w, loc)
        put_csr(key, g)
        th = put_transform(key, g)
        th16 = R.reblock_handle(th, 16)
        G[f"{key}/reblock16_bp"] = R.transform_fields(th16).block_partition
        for geom in [(1, 1), (3, 5), (16, 16), (32, 4)]:
            put_transform(key, g, *geom)
        x = R.dense_random(n, dim, 7 + i)
        y = R.dense_random(n, dim, 8 + i)
        G[f"{key}/x"], G[f"{key}/y"] = x, y
        for tf in (0, 1):
            outs = [R.spmm(th, n, x, r, tf) for r in (1.0, 0.5, 0.0)]
            assert all((o == outs[0]).all() for o in outs)
            G[f"{key}/spmm_tf{tf}"] = outs[0]
            G[f"{key}/sddmm_tf{tf}"] = R.sddmm(th16, g.num_edges, x, y, 1.0, tf)
        ov = np.random.default_rng(i).uniform(0, 1, g.num_edges).astype(np.float32)
        G[f"{key}/override_values"] = ov
        G[f"{key}/spmm_override"] = R.spmm(th, n, x, 0.5, False, values=ov)
        lg = np.random.default_rng(50 + i).uniform(-8, 8, g.num_edges).astype(np.float32)
        G[f"{key}/logits"] = lg
        G[f"{key}/softmax"] = R.edge_softmax(g, lg)
        G[f"{key}/l2norm"], z = R.l2_normalize_rows(x)
        # GCN pipeline: normalize(sym, loops, dedupe) -> gcn values -> transform
        gg = R.gcn_normalize_values(R.normalize_graph(g, True, True, True))
        put_csr(f"{key}_gcn", gg)
        thg = put_transform(f"{key}_gcn", gg)
        layers = [(R.dense_random(dim, 16, 20 + i, -0.1, 0.1), True),
                  (R.dense_random(16, 7, 21 + i, -0.1, 0.1), False)]
        G[f"{key}_gcn/w0"], G[f"{key}_gcn/w1"] = layers[0][0], layers[1][0]
        for tf in (0, 1):
            G[f"{key}_gcn/gcn_tf{tf}"] = R.gcn_forward(thg, n, x, layers, 1.0, tf)
        # AGNN pipeline: normalize(loops) -> transform (values ignored)
        ga = R.normalize_graph(g, False, True, True)
        put_csr(f"{key}_agnn", ga)
        tha = R.transform_handle(ga)
        betas = np.array([1.0, 0.6, 1.4, 0.9], np.float32)
        G[f"{key}_agnn/betas"] = betas
        for tf in (0, 1):
            G[f"{key}_agnn/agnn_tf{tf}"], _ = R.agnn_forward(tha, x, betas, 1.0, tf)

    np.savez_compressed(OUT, **G)
    print(f"wrote {OUT}: {len(G)} arrays, {os.path.getsize(OUT) / 1e6:.2f} MB")


def identity_graph(R, n):
    """The reference's own update GEMM through its public API (SURVEY §8a
    note): gcn_forward(sgt_transform(identity(n)), X, {{W, relu}}) — identity
    aggregation is exact (1.0f * x + 0)."""
    g = Csr.of(n, np.arange(n + 1, dtype=np.uint64), np.arange(n, dtype=np.uint32),
               np.ones(n, np.float32))
    return R.transform_handle(g)


def configs():
    """BASELINE.json configs C1 and C2 end to end through the reference, on the
    bench's own synthetic graphs and inputs (bench.make_graph with the
    generator linked into oracle/_ref, DenseMatrix::random seed 8 = the
    reference bench's seed + 7, random_gcn_layers seed 1; bench.cpp:114-135).
    The reference's acceptance analogue: proj/tests/acceptance.cpp:191-225."""
    import bench

    R = RefLib()
    G: dict[str, np.ndarray] = {}
    # ---- C1: Cora-shaped GCN 1433 -> 16 -> 7 (normalize_graph + gcn values in the chain)
    wl = bench.WORKLOADS["cora-gcn"]
    g, _ = bench.make_graph(wl, "calibrated", synth=R.synth_graph)
    gs = R.normalize_graph(g, True, True, True)
    gn = R.gcn_normalize_values(gs)
    th = R.transform_handle(gn)
    x = R.dense_random(g.num_nodes, wl["d_in"], bench.INPUT_SEED)
    layers = R.random_gcn_layers(wl["d_in"], wl["hidden"], wl["d_out"], wl["layers"],
                                 bench.LAYER_SEED)
    G["c1/n"] = np.array(g.num_nodes, np.uint64)
    G["c1/node_pointer"], G["c1/edge_list"] = g.node_pointer, g.edge_list
    G["c1/norm_node_pointer"], G["c1/norm_edge_list"] = gn.node_pointer, gn.edge_list
    G["c1/gcn_values"] = gn.values
    for tf in (0, 1):
        G[f"c1/gcn_tf{tf}"] = R.gcn_forward(th, g.num_nodes, x, layers, 1.0, tf)
    # ---- C2: Pubmed-shaped in-proj 500->32 (+ReLU), 4 x agnn_forward (beta 1), out-proj 32->3
    wl = bench.WORKLOADS["pubmed-agnn"]
    g, _ = bench.make_graph(wl, "calibrated", synth=R.synth_graph)
    ga = R.normalize_graph(g, False, True, True)
    tha = R.transform_handle(ga)
    ident = identity_graph(R, g.num_nodes)
    x = R.dense_random(g.num_nodes, wl["d_in"], bench.INPUT_SEED)
    w_in = R.dense_random(wl["d_in"], wl["hidden"], 1, -0.1, 0.1)
    w_out = R.dense_random(wl["hidden"], wl["d_out"], 2, -0.1, 0.1)
    rows = np.unique(np.random.default_rng(2).integers(0, g.num_nodes, 2048))
    G["c2/n"] = np.array(g.num_nodes, np.uint64)
    G["c2/node_pointer"], G["c2/edge_list"] = ga.node_pointer, ga.edge_list
    G["c2/w_in"], G["c2/w_out"], G["c2/rows"] = w_in, w_out, rows
    for tf in (0, 1):
        h0 = R.gcn_forward(ident, g.num_nodes, x, [(w_in, True)], 1.0, tf)
        h4, zeros = R.agnn_forward(tha, h0, np.ones(wl["layers"], np.float32), 1.0, tf)
        out = R.gcn_forward(ident, g.num_nodes, h4, [(w_out, False)], 1.0, tf)
        G[f"c2/h0_tf{tf}_rows"] = h0[rows]
        G[f"c2/h4_tf{tf}_rows"] = h4[rows]
        G[f"c2/out_tf{tf}"] = out
        G[f"c2/zeros_tf{tf}"] = np.array(zeros, np.uint64)
    np.savez_compressed(OUT_CONFIGS, **G)
    print(f"wrote {OUT_CONFIGS}: {len(G)} arrays, {os.path.getsize(OUT_CONFIGS) / 1e6:.2f} MB")


def sgt_fixtures():
    """SGT1 files written by the reference's own save_sgt (sgt_file.cpp:47-66)
    for the drop-in's load_sgt / save_sgt byte-compatibility tests: a weighted
    graph at the default 16x8 geometry and an unweighted one at 3x5 (ragged
    windows), both from the golden set."""
    R = RefLib()
    here = os.path.dirname(os.path.abspath(__file__))
    G = dict(np.load(OUT))
    for key, geom in (("rand3", (16, 8)), ("rand0", (3, 5))):
        n = int(G[f"{key}/n"])
        g = Csr.of(n, G[f"{key}/node_pointer"], G[f"{key}/edge_list"], G.get(f"{key}/values"))
        th = R.transform_handle(g, *geom)
        path = os.path.join(here, f"ref_{key}_{geom[0]}x{geom[1]}.sgt")
        R.save_sgt(th, path)
        print(f"wrote {path}: {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    if "--configs" not in sys.argv and "--sgt" not in sys.argv:
        main()
    if "--sgt" not in sys.argv:
        configs()
    sgt_fixtures()
