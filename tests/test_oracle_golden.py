"""CPU: pin the oracle restatement (oracle/sgtk_oracle.cpp) to golden vectors
produced by the unmodified reference (tests/golden/make_golden.py).

Integer / index structures must be bit-exact; float results must be
bit-exact too, because the restatement reproduces the reference's operation
order and rounding (see the header of oracle/sgtk_oracle.cpp)."""

import numpy as np
import pytest

from oracle.oracle import Oracle, OracleError
from tests._golden import csr, golden, random_keys, transform

O = Oracle()
G = golden()
FIELDS = ["edge_to_row", "edge_to_column", "block_partition", "window_offsets",
          "window_unique_cols", "block_counter"]


def check_transform(key, geom=(16, 8)):
    t = O.sgt_transform(csr(key), *geom)
    want = transform(key, f"{geom[0]}x{geom[1]}")
    got = dict(t.fields(), block_counter=np.array(t.block_counter, np.uint64))
    for f in FIELDS:
        np.testing.assert_array_equal(got[f], want[f], err_msg=f"{key} {geom} {f}")


@pytest.mark.parametrize("key", ["kat_identity16", "kat_compress", "kat_reblock17",
                                 "kat_ragged", "kat_blockdense"])
def test_translator_kats(key):
    check_transform(key)


def test_translator_kat_values():
    # test_sgt_transform.cpp:47-80 spelled out
    t = transform("kat_identity16")
    assert list(t["block_partition"]) == [2] and int(t["block_counter"]) == 2
    assert list(t["edge_to_column"]) == list(range(16))
    assert list(G["kat_identity16/block_stats"]) == [2, 256, 16]
    assert G["kat_identity16/density"][0] == pytest.approx(0.0625)
    t = transform("kat_compress")
    assert list(t["window_unique_cols"]) == [5, 9, 30]
    assert list(t["block_partition"]) == [1, 0]
    assert list(t["edge_to_column"]) == [0, 1, 0, 2]
    assert list(G["kat_identity16/reblock16_bp"]) == [1]
    assert int(G["kat_reblock17/reblock16_bp"][0]) == 2
    assert int(transform("kat_blockdense")["block_counter"]) == 8


@pytest.mark.parametrize("key", random_keys())
@pytest.mark.parametrize("geom", [(16, 8), (1, 1), (3, 5), (16, 16), (32, 4)])
def test_translator_random(key, geom):
    check_transform(key, geom)


@pytest.mark.parametrize("key", random_keys())
def test_reblock(key):
    t = O.reblock(O.sgt_transform(csr(key)), 16)
    np.testing.assert_array_equal(t.block_partition, G[f"{key}/reblock16_bp"])


@pytest.mark.parametrize("key", random_keys())
def test_kernels_random(key):
    g = csr(key)
    x, y = G[f"{key}/x"], G[f"{key}/y"]
    for tf in (0, 1):
        np.testing.assert_array_equal(O.spmm(g, x, tf), G[f"{key}/spmm_tf{tf}"])
        np.testing.assert_array_equal(O.sddmm(g, x, y, tf), G[f"{key}/sddmm_tf{tf}"])
    np.testing.assert_array_equal(O.spmm(g, x, values=G[f"{key}/override_values"]),
                                  G[f"{key}/spmm_override"])
    np.testing.assert_array_equal(O.edge_softmax(g, G[f"{key}/logits"]), G[f"{key}/softmax"])
    np.testing.assert_array_equal(O.l2_normalize_rows(x)[0], G[f"{key}/l2norm"])


@pytest.mark.parametrize("key", random_keys())
def test_models_random(key):
    g = csr(key)
    x = G[f"{key}/x"]
    # GCN preprocessing chain is itself pinned: normalize -> gcn values
    gg = O.gcn_normalize_values(O.normalize_graph(g, True, True, True))
    want = csr(f"{key}_gcn")
    np.testing.assert_array_equal(gg.node_pointer, want.node_pointer)
    np.testing.assert_array_equal(gg.edge_list, want.edge_list)
    np.testing.assert_array_equal(gg.values, want.values)
    layers = [(G[f"{key}_gcn/w0"], True), (G[f"{key}_gcn/w1"], False)]
    for tf in (0, 1):
        np.testing.assert_array_equal(O.gcn_forward(gg, x, layers, tf), G[f"{key}_gcn/gcn_tf{tf}"])
    ga = csr(f"{key}_agnn")
    for tf in (0, 1):
        out, _ = O.agnn_forward(ga, x, G[f"{key}_agnn/betas"], tf)
        np.testing.assert_array_equal(out, G[f"{key}_agnn/agnn_tf{tf}"])


def test_kernel_kats():
    np.testing.assert_array_equal(O.spmm(csr("kat_2cycle"), G["kat_2cycle/x"]), [[3, 4], [1, 2]])
    np.testing.assert_array_equal(G["kat_2cycle/spmm"], [[3, 4], [1, 2]])
    g16 = csr("kat_identity16")
    np.testing.assert_array_equal(O.spmm(g16, G["kat_identity_spmm/x"]), G["kat_identity_spmm/x"])
    for key in ["kat_sddmm_orth", "kat_sddmm_aligned", "kat_sddmm_weight"]:
        np.testing.assert_array_equal(O.sddmm(csr(key), G[f"{key}/x"], G[f"{key}/y"]), G[f"{key}/out"])
    assert list(G["kat_sddmm_orth/out"]) == [0.0] and list(G["kat_sddmm_aligned/out"]) == [1.0]
    for key in ["kat_softmax_single", "kat_softmax_equal", "kat_softmax_ln2", "kat_softmax_extreme"]:
        np.testing.assert_array_equal(O.edge_softmax(csr(key), G[f"{key}/logits"]), G[f"{key}/out"])
    assert int(G["kat_overflow/status"]) == 10  # NonFiniteError
    with pytest.raises(OracleError) as e:
        O.spmm(csr("kat_2cycle").__class__.of(4, [0, 4, 4, 4, 4], [0, 1, 2, 3], np.ones(4, np.float32)),
               np.full((4, 1), 1e38, np.float32))
    assert e.value.code == 10
    out = O.gcn_normalize_values(csr("kat_gcnnorm_path")).values
    np.testing.assert_array_equal(out, G["kat_gcnnorm_path/values_out"])
    assert out[1] == pytest.approx(0.40824829)
    out, z = O.agnn_forward(csr("kat_agnn_zero"), G["kat_agnn_zero/x"], [1.0])
    np.testing.assert_array_equal(out, G["kat_agnn_zero/out"])
    assert z == int(G["kat_agnn_zero/zeros"]) == 2


def test_tf32_kats():
    xs, want = G["kat_tf32/in"], G["kat_tf32/out"]
    np.testing.assert_array_equal(O.tf32_round(xs).view(np.uint32), want.view(np.uint32))
    for v, w in zip(xs[:12], want[:12]):
        assert np.float32(O.tf32_round_value(float(v))).view(np.uint32) == w.view(np.uint32)
    assert O.tf32_round_value(1 + 2**-11) == 1.0
    assert O.tf32_round_value(1 + 2**-11 + 2**-20) == 1 + 2**-10


def test_dense_random_stream():
    np.testing.assert_array_equal(O.dense_random(5, 7, 8), G["kat_dense_random/seed8_5x7"])
    np.testing.assert_array_equal(O.dense_random(4, 3, 3, -0.1, 0.1), G["kat_dense_random/seed3_4x3_m01"])


def test_split_plan_arithmetic():
    # tile_exec.cpp:150-161 / test_tile_exec.cpp:16-30
    from oracle.oracle import Csr
    g = Csr.of(32, [0, 32] + [32] * 31, list(range(32)))
    t = O.sgt_transform(g)
    assert int(t.block_partition[0]) == 4
    assert [int(O.split_plan(t, r)[0]) for r in (1.0, 0.5, 0.0)] == [4, 2, 0]
    for bad in (-0.1, 1.1, float("nan")):
        with pytest.raises(OracleError) as e:
            O.split_plan(t, bad)
        assert e.value.code == 8  # RangeError


def test_oracle_matches_reference_configs():
    """C1 / C2 (BASELINE.json) through the oracle restatement == the reference."""
    import os

    from oracle.oracle import Csr

    z = dict(np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden",
                                  "configs.npz")))
    O = Oracle()
    n = int(z["c1/n"])
    gs = O.normalize_graph(Csr.of(n, z["c1/node_pointer"], z["c1/edge_list"]), True, True, True)
    gn = O.gcn_normalize_values(gs)
    assert np.array_equal(gn.values, z["c1/gcn_values"])
    x = O.dense_random(n, 1433, 8)
    import paper_2412_12218_b200 as sg

    layers = sg.random_gcn_layers(1433, 16, 7, 2, 1)
    assert np.array_equal(O.gcn_forward(gn, x, layers), z["c1/gcn_tf0"])
    assert np.array_equal(O.gcn_forward(gn, x, layers, tf32=True), z["c1/gcn_tf1"])
    n = int(z["c2/n"])
    ga = Csr.of(n, z["c2/node_pointer"], z["c2/edge_list"])
    x = O.dense_random(n, 500, 8)
    h0 = O.matmul(x, z["c2/w_in"], relu=True)
    h4, zeros = O.agnn_forward(ga, h0, [1.0] * 4)
    out = O.matmul(h4, z["c2/w_out"])
    rows = z["c2/rows"]
    assert np.array_equal(h0[rows], z["c2/h0_tf0_rows"])
    assert np.array_equal(h4[rows], z["c2/h4_tf0_rows"])
    assert np.array_equal(out, z["c2/out_tf0"])
