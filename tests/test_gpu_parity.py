"""GPU parity: the sm_100a path (through the C ABI) against the reference's
golden vectors (tests/golden, produced by the unmodified reference) and the
CPU oracle (oracle/, pinned to those vectors in test_oracle_golden.py).

Bars (stated here):
  * translator index structures: bit-exact (transforms_equal,
    test_sgt_transform.cpp:20-29);
  * FP32 precision (3xTF32 on tensor cores): max_rel_err <= 1e-5 (the
    reference's own tests allow 1e-4);
  * TF32 precision vs the reference's TF32 mode (identical rounded operands,
    exact products, only the fp32 summation order differs): max_rel_err <= 1e-5;
    vs the FP32 oracle the componentwise bound
    |gpu - ref| <= 2^-10 (|A||X|) + 1e-6 max|ref|.
"""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2412_12218_b200 as sg  # noqa: E402
from paper_2412_12218_b200.device import DeviceGraph, gemm, l2_normalize_rows  # noqa: E402
from oracle.oracle import Csr, Oracle  # noqa: E402
from tests._bars import agnn_tf32_bar, gcn_tf32_bar  # noqa: E402
from tests._golden import csr, golden, random_keys, transform  # noqa: E402

O = Oracle()
G = golden()
TOL_FP32 = 1e-5
TOL_TF32 = 1e-5
FIELDS = ["edge_to_row", "edge_to_column", "block_partition", "window_offsets",
          "window_unique_cols", "block_counter"]


def mre(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    assert a.shape == b.shape
    if a.size == 0:
        return 0.0
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def sgcsr(c: Csr) -> sg.CsrGraph:
    return sg.CsrGraph(c.num_nodes, c.node_pointer, c.edge_list, c.values)


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


# ----------------------------------------------------------------- translator
@pytest.mark.parametrize("key", ["kat_identity16", "kat_compress", "kat_reblock17",
                                 "kat_ragged", "kat_blockdense"] + random_keys())
@pytest.mark.parametrize("geom", [(16, 8), (1, 1), (3, 5), (16, 16), (32, 4)])
def test_translator_bit_exact(key, geom):
    want = transform(key, f"{geom[0]}x{geom[1]}")
    if not want:
        pytest.skip("geometry not in golden set for this key")
    t = sg.sgt_transform(sgcsr(csr(key)), *geom)
    got = t.device.fields()
    for f in FIELDS:
        np.testing.assert_array_equal(got[f], want[f], err_msg=f"{key} {geom} {f}")


def test_translator_kats_and_stats():
    t = sg.sgt_transform(sgcsr(csr("kat_identity16")))
    s = sg.block_stats(t)
    assert (s.block_counter, s.capacity, s.nnz) == (2, 256, 16)
    assert s.mean_tile_density == pytest.approx(0.0625)
    r = sg.reblock(t, 16)
    assert list(r.block_partition) == [1] and r.block_counter == 1
    np.testing.assert_array_equal(r.edge_to_column, t.edge_to_column)
    a, idx = sg.gather_tile(t, 0, 0)
    np.testing.assert_array_equal(a, G["kat_identity16/gather_tile00_a"])
    np.testing.assert_array_equal(idx, G["kat_identity16/gather_tile00_idx"])
    t = sg.sgt_transform(sgcsr(csr("kat_ragged")))
    a, idx = sg.gather_tile(t, 0, 0)
    np.testing.assert_array_equal(a, G["kat_ragged/gather_tile00_a"])
    np.testing.assert_array_equal(idx, G["kat_ragged/gather_tile00_idx"])
    with pytest.raises(sg.TileIndexError):
        sg.gather_tile(t, 5, 0)
    with pytest.raises(sg.TileIndexError):
        sg.gather_tile(t, 0, 1)


def test_translator_errors():
    g = sgcsr(csr("kat_identity16"))
    with pytest.raises(sg.GeometryError):
        sg.sgt_transform(g, 0, 8)
    with pytest.raises(sg.GeometryError):
        sg.sgt_transform(g, 16, 0)
    with pytest.raises(sg.GeometryError):
        sg.reblock(sg.sgt_transform(g), 0)
    bad = sg.CsrGraph(3, np.array([0, 2, 2, 2]), np.array([1, 1]))  # duplicate column
    with pytest.raises(sg.SgtkError):
        sg.sgt_transform(bad)
    bad = sg.CsrGraph(3, np.array([0, 1, 1, 1]), np.array([7]))  # out of range
    with pytest.raises(sg.SgtkError):
        sg.sgt_transform(bad)
    with pytest.raises(sg.RangeError):
        sg.make_split_plan(sg.sgt_transform(g), 1.5)
    with pytest.raises(sg.RangeError):
        sg.make_split_plan(sg.sgt_transform(g), float("nan"))


def big_graphs():
    # medium windows (2k-32k edges): power-law hubs; large windows (> 32768
    # edges: CUB path): a dense hub block.
    g1 = sg.synth_graph(20000, 40.0, alpha=2.0, p_local=0.5, band=4.0, seed=7)
    n = 3000
    rows, cols = [], []
    rng = np.random.default_rng(1)
    for r in range(n):
        k = 2500 if r < 16 else 5
        c = np.unique(rng.integers(0, n, k))
        rows += [r] * len(c)
        cols += list(c)
    g2 = sg.csr_from_coo(n, rows, cols)
    return [("powerlaw20k", g1), ("hubwindow", g2)]


@pytest.mark.parametrize("name,g", big_graphs())
def test_translator_bit_exact_large_windows(name, g):
    want = O.sgt_transform(Csr.of(g.num_nodes, g.node_pointer, g.edge_list))
    got = sg.sgt_transform(g).device.fields()
    for f, v in want.fields().items():
        np.testing.assert_array_equal(got[f], v, err_msg=f"{name} {f}")
    assert int(got["block_counter"]) == want.block_counter


# ---------------------------------------------------------------------- SpMM
@pytest.mark.parametrize("key", random_keys())
@pytest.mark.parametrize("ratio", [1.0, 0.5, 0.0])
def test_spmm_vs_reference(key, ratio):
    t = sg.sgt_transform(sgcsr(csr(key)))
    x = G[f"{key}/x"]
    plan = sg.make_split_plan(t, ratio)
    got = sg.spmm_hybrid(t, x, plan)
    assert mre(got, G[f"{key}/spmm_tf0"]) <= TOL_FP32
    got = sg.spmm_hybrid(t, x, plan, precision="tf32")
    assert mre(got, G[f"{key}/spmm_tf1"]) <= TOL_TF32
    g = csr(key)
    absref = O.spmm(Csr.of(g.num_nodes, g.node_pointer, g.edge_list,
                           None if g.values is None else np.abs(g.values)), np.abs(x))
    ref = G[f"{key}/spmm_tf0"]
    assert np.all(np.abs(got - ref) <= 2.0**-10 * absref + 1e-6 * np.abs(ref).max())
    got = sg.spmm_hybrid(t, x, plan, edge_values=G[f"{key}/override_values"])
    assert mre(got, G[f"{key}/spmm_override"]) <= TOL_FP32


def test_spmm_kats():
    t = sg.sgt_transform(sgcsr(csr("kat_2cycle")))
    np.testing.assert_array_equal(sg.spmm_hybrid(t, G["kat_2cycle/x"]), [[3, 4], [1, 2]])
    t = sg.sgt_transform(sgcsr(csr("kat_identity16")))
    x = G["kat_identity_spmm/x"]
    for r in (1.0, 0.0, 0.5):
        np.testing.assert_array_equal(sg.spmm_hybrid(t, x, sg.make_split_plan(t, r)), x)
    # overflow -> NonFiniteError (test_tile_exec.cpp:179-186)
    g = sg.CsrGraph(4, np.array([0, 4, 4, 4, 4]), np.arange(4), np.ones(4, np.float32))
    t = sg.sgt_transform(g)
    with pytest.raises(sg.NonFiniteError):
        sg.spmm_hybrid(t, np.full((4, 1), 1e38, np.float32))
    with pytest.raises(sg.ShapeError):
        sg.spmm_hybrid(t, np.zeros((3, 4), np.float32))
    with pytest.raises(sg.ShapeError):
        sg.spmm_hybrid(t, np.zeros((4, 4), np.float32), edge_values=np.ones(5, np.float32))


def test_spmm_padding_neutral_and_linear():
    # test_tile_exec.cpp:114-148: zero columns bit-neutral; linearity
    g = sgcsr(csr("rand1"))
    t = sg.sgt_transform(g)
    plan = sg.make_split_plan(t, 0.5)
    x = sg.dense_random(g.num_nodes, 18, 3)
    wide = np.zeros((g.num_nodes, 25), np.float32)
    wide[:, :18] = x
    a, b = sg.spmm_hybrid(t, x, plan), sg.spmm_hybrid(t, wide, plan)
    np.testing.assert_array_equal(a, b[:, :18])
    assert np.all(b[:, 18:] == 0)
    z = sg.dense_random(g.num_nodes, 18, 4)
    lhs = sg.spmm_hybrid(t, 0.75 * x - 1.25 * z, plan)
    rhs = 0.75 * sg.spmm_hybrid(t, x, plan) - 1.25 * sg.spmm_hybrid(t, z, plan)
    assert mre(lhs, rhs) <= 1e-5


@pytest.mark.parametrize("d", [1, 3, 7, 16, 32, 41, 64, 100, 128, 1433])
def test_spmm_widths(d):
    g = sg.synth_graph(1000, 6.0, alpha=2.0, p_local=0.5, seed=d)
    c = Csr.of(g.num_nodes, g.node_pointer, g.edge_list,
               sg.dense_random(1, g.num_edges, 9)[0])
    gs = sg.CsrGraph(c.num_nodes, c.node_pointer, c.edge_list, c.values)
    t = sg.sgt_transform(gs)
    x = sg.dense_random(g.num_nodes, d, d + 1)
    want = O.spmm(c, x)
    for r in (1.0, 0.3):
        assert mre(sg.spmm_hybrid(t, x, sg.make_split_plan(t, r)), want) <= TOL_FP32


@pytest.mark.parametrize("name,g", big_graphs())
def test_spmm_large_windows_split_units(name, g):
    # Hub rows (degree up to ~8k) make fp32 summation order visible: the
    # sequential oracle itself is ~3e-6 off the exact (float64) result.  Bar:
    # the reference's own tolerance vs the oracle (1e-4, test_tile_exec.cpp:97-112)
    # and no more than twice the oracle's own rounding error vs exact.
    c = Csr.of(g.num_nodes, g.node_pointer, g.edge_list)
    t = sg.sgt_transform(g)
    deg = np.diff(g.node_pointer.astype(np.int64))
    rows = np.repeat(np.arange(g.num_nodes), deg)
    for d in (16, 64):
        x = sg.dense_random(g.num_nodes, d, 5)
        want = O.spmm(c, x)
        exact = np.zeros((g.num_nodes, d))
        np.add.at(exact, rows, x[g.edge_list].astype(np.float64))
        ref_err = mre(want, exact)
        for plan in (None, sg.make_split_plan(t, 0.25)):
            got = sg.spmm_hybrid(t, x, plan)
            assert mre(got, want) <= 1e-4
            assert mre(got, exact) <= 2 * ref_err + 1e-6


def test_spmm_deterministic():
    g = sg.synth_graph(5000, 30.0, alpha=2.0, p_local=0.3, seed=2)
    dg = DeviceGraph.from_csr(g.node_pointer, g.edge_list)
    x = dev(sg.dense_random(g.num_nodes, 64, 1))
    a = dg.spmm(x)
    for _ in range(3):
        assert torch.equal(a, dg.spmm(x))


# --------------------------------------------------------------------- SDDMM
@pytest.mark.parametrize("key", random_keys())
@pytest.mark.parametrize("ratio", [1.0, 0.5, 0.0])
def test_sddmm_vs_reference(key, ratio):
    t16 = sg.reblock(sg.sgt_transform(sgcsr(csr(key))), 16)
    x, y = G[f"{key}/x"], G[f"{key}/y"]
    plan = sg.make_split_plan(t16, ratio)
    assert mre(sg.sddmm_hybrid(t16, x, y, plan), G[f"{key}/sddmm_tf0"]) <= TOL_FP32
    # TF32: the reference rounds each dot to TF32 (tile_exec.cpp:386,402); an
    # fp32 sum in another order can land one TF32 step (<= 2^-10 relative) away
    assert mre(sg.sddmm_hybrid(t16, x, y, plan, precision="tf32"), G[f"{key}/sddmm_tf1"]) <= 2.0 ** -10


def test_sddmm_kats():
    for key in ["kat_sddmm_orth", "kat_sddmm_aligned", "kat_sddmm_weight"]:
        t = sg.reblock(sg.sgt_transform(sgcsr(csr(key))), 16)
        got = sg.sddmm_hybrid(t, G[f"{key}/x"], G[f"{key}/y"])
        np.testing.assert_allclose(got, G[f"{key}/out"], rtol=1e-6, atol=0)
    t = sg.sgt_transform(sgcsr(csr("kat_identity16")))
    with pytest.raises(sg.ShapeError):
        sg.sddmm_hybrid(t, np.zeros((16, 4), np.float32), np.zeros((15, 4), np.float32))
    with pytest.raises(sg.ShapeError):
        sg.sddmm_hybrid(t, np.zeros((16, 4), np.float32), np.zeros((16, 5), np.float32))


# ---------------------------------------------------------- softmax / l2norm
@pytest.mark.parametrize("key", random_keys())
def test_softmax_and_l2norm(key):
    g = sgcsr(csr(key))
    got = sg.edge_softmax(g, G[f"{key}/logits"])
    assert mre(got, G[f"{key}/softmax"]) <= 1e-6
    z, _ = sg.l2_normalize_rows(G[f"{key}/x"])
    # fp64 row sums in a different order: at most 1 ulp of the float result
    np.testing.assert_allclose(z, G[f"{key}/l2norm"], rtol=2.5e-7, atol=0)


def test_softmax_kats():
    for key in ["kat_softmax_single", "kat_softmax_equal", "kat_softmax_ln2", "kat_softmax_extreme"]:
        got = sg.edge_softmax(sgcsr(csr(key)), G[f"{key}/logits"])
        np.testing.assert_allclose(got, G[f"{key}/out"], rtol=1e-6)
        assert np.all(np.isfinite(got))


# -------------------------------------------------------------------- models
@pytest.mark.parametrize("key", random_keys())
@pytest.mark.parametrize("order", [0, 1, 2])
def test_gcn_vs_reference(key, order):
    t = sg.sgt_transform(sgcsr(csr(f"{key}_gcn")))
    layers = [(G[f"{key}_gcn/w0"], True), (G[f"{key}_gcn/w1"], False)]
    x = G[f"{key}/x"]
    assert mre(sg.gcn_forward(t, x, layers, order=order), G[f"{key}_gcn/gcn_tf0"]) <= TOL_FP32
    assert mre(sg.gcn_forward(t, x, layers, precision="tf32", order=order),
               G[f"{key}_gcn/gcn_tf1"]) <= gcn_tf32_bar()


def test_gcn_identity_and_zero():
    # test_gnn.cpp:36-50
    n = 20
    g = sg.gcn_normalize_values(sg.CsrGraph(n, np.arange(n + 1), np.arange(n)))
    t = sg.sgt_transform(g)
    x = sg.dense_random(n, 6, 3, 0.0, 1.0)
    eye = np.eye(6, dtype=np.float32)
    np.testing.assert_array_equal(sg.gcn_forward(t, x, [(eye, True), (eye, True)]), x)
    t = sg.sgt_transform(sgcsr(csr("rand0_gcn")))
    x = G["rand0/x"]
    out = sg.gcn_forward(t, x, [(np.zeros((x.shape[1], 8), np.float32), True)])
    assert np.all(out == 0)
    with pytest.raises(sg.ShapeError):
        sg.gcn_forward(t, x, [(np.zeros((x.shape[1] + 1, 2), np.float32), False)])


@pytest.mark.parametrize("key", random_keys())
def test_agnn_vs_reference(key):
    t = sg.sgt_transform(sgcsr(csr(f"{key}_agnn")))
    x = G[f"{key}/x"]
    betas = G[f"{key}_agnn/betas"]
    assert mre(sg.agnn_forward(t, x, betas), G[f"{key}_agnn/agnn_tf0"]) <= TOL_FP32
    bar = agnn_tf32_bar(betas)  # error model: tests/_bars.py
    assert mre(sg.agnn_forward(t, x, betas, precision="tf32"), G[f"{key}_agnn/agnn_tf1"]) <= bar
    assert mre(sg.agnn_forward(t, x, betas, plan=sg.make_split_plan(t, 0.0)),
               G[f"{key}_agnn/agnn_tf0"]) <= TOL_FP32
    # fused single-pass mode (online softmax; attention never materialised)
    for ratio in (1.0, 0.5, 0.0):
        plan = sg.make_split_plan(t, ratio)
        assert mre(sg.agnn_forward(t, x, betas, plan=plan, mode=1),
                   G[f"{key}_agnn/agnn_tf0"]) <= TOL_FP32
    assert mre(sg.agnn_forward(t, x, betas, precision="tf32", mode=1),
               G[f"{key}_agnn/agnn_tf1"]) <= bar
    # panel mode (agnn_panel.cu)
    assert mre(sg.agnn_forward(t, x, betas, mode=2), G[f"{key}_agnn/agnn_tf0"]) <= TOL_FP32
    assert mre(sg.agnn_forward(t, x, betas, precision="tf32", mode=2),
               G[f"{key}_agnn/agnn_tf1"]) <= bar


@pytest.mark.parametrize("name,g", big_graphs())
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_agnn_large_windows(name, g, mode):
    # split windows: the fused kernel merges (m, l, O) states across units
    c = Csr.of(g.num_nodes, g.node_pointer, g.edge_list)
    t = sg.sgt_transform(g)
    x = sg.dense_random(g.num_nodes, 32, 3)
    want, _ = O.agnn_forward(c, x, [1.0, 0.7])
    assert mre(sg.agnn_forward(t, x, [1.0, 0.7], mode=mode), want) <= TOL_FP32
    assert mre(sg.agnn_forward(t, x, [1.0, 0.7], plan=sg.make_split_plan(t, 0.4), mode=mode),
               want) <= TOL_FP32


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_agnn_kats(mode):
    t = sg.sgt_transform(sgcsr(csr("kat_agnn_zero")))
    out, z = sg.agnn_forward(t, G["kat_agnn_zero/x"], [1.0], return_zeros=True, mode=mode)
    assert z == 2
    np.testing.assert_allclose(out, G["kat_agnn_zero/out"], rtol=1e-6)
    # single self-looped node: identity map (test_gnn.cpp:157-164)
    t = sg.sgt_transform(sg.CsrGraph(1, np.array([0, 1]), np.array([0])))
    x = np.array([[0.5, -1.0, 2.0]], np.float32)
    np.testing.assert_array_equal(sg.agnn_forward(t, x, [1.0] * 4, mode=mode), x)
    # beta = 0: uniform neighbour mean (test_gnn.cpp:166-178), tolerance 1e-5
    g = sgcsr(csr("rand2"))
    t = sg.sgt_transform(g)
    x = G["rand2/x"]
    deg = np.diff(g.node_pointer.astype(np.int64))
    rows = np.repeat(np.arange(g.num_nodes), deg)
    want = np.zeros_like(x, dtype=np.float64)
    np.add.at(want, rows, x[g.edge_list] / np.maximum(deg, 1)[rows, None])
    want = np.zeros_like(want) if False else want
    h = sg.agnn_forward(t, x, [0.0], mode=mode)
    assert mre(h, want) <= 1e-5


def test_gcn_normalize_values_bit_exact():
    for key in random_keys():
        g = csr(f"{key}_gcn")
        got = sg.gcn_normalize_values(sg.CsrGraph(g.num_nodes, g.node_pointer, g.edge_list))
        np.testing.assert_array_equal(got.values, g.values)
    got = sg.gcn_normalize_values(sgcsr(csr("kat_gcnnorm_path")))
    np.testing.assert_array_equal(got.values, G["kat_gcnnorm_path/values_out"])
    with pytest.raises(sg.DegreeError):
        sg.gcn_normalize_values(sg.CsrGraph(2, np.array([0, 1, 1]), np.array([0])))


def test_tf32_round_bit_exact():
    xs, want = G["kat_tf32/in"], G["kat_tf32/out"]
    np.testing.assert_array_equal(sg.tf32_round(xs).view(np.uint32), want.view(np.uint32))


# (257, 1433, 16), (1000, 500, 32), (2708, 1433, 16), (5000, 2000, 100): few
# row tiles, long K -> split K (gemm_tc05.cu) with its in-order reduction
@pytest.mark.parametrize("m,k,n", [(1, 1, 1), (257, 1433, 16), (1000, 500, 32), (777, 32, 41),
                                   (4096, 128, 128), (100, 7, 3), (2708, 1433, 16), (5000, 2000, 100)])
def test_gemm(m, k, n):
    a = sg.dense_random(m, k, 1)
    w = sg.dense_random(k, n, 2, -0.1, 0.1)
    want = O.matmul(a, w)
    got = gemm(dev(a), dev(w), relu=False).cpu().numpy()
    assert mre(got, want) <= TOL_FP32
    got = gemm(dev(a), dev(w), relu=True, precision="tf32").cpu().numpy()
    assert mre(got, np.maximum(want, 0)) <= 5e-3
