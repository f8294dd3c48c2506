"""BASELINE.json configs C1 and C2 end to end on the GPU, against outputs of
the unmodified reference on the same synthetic graphs and inputs
(tests/golden/configs.npz, made by `make_golden.py --configs` through
oracle/_ref; the reference analogue is proj/tests/acceptance.cpp:191-225).

C1: Cora-shaped GCN 1433->16->7: normalize_graph(sym, loops, dedupe) ->
    gcn_normalize_values -> sgt_transform -> gcn_forward, all on the GPU.
C2: Pubmed-shaped in-proj 500->32 (+ReLU) -> 4 x agnn_forward -> out-proj 32->3,
    in the library's auto mode (what the bench runs) and in every AGNN mode.

Bars: graph preprocessing bit-exact; FP32 max_rel_err <= 1e-5 (the reference
tests allow 1e-4); TF32 vs the reference's TF32 mode by the error models of
tests/_bars.py (GCN: the default order A(hW) rounds another operand set than
the reference's (Ah)W; AGNN: (1 + |beta|) 2^-10; the projections: one TF32
step for the weights the reference leaves unrounded).
"""
import os

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2412_12218_b200 as sg  # noqa: E402
from tests._bars import TF32_STEP, agnn_tf32_bar, gcn_tf32_bar  # noqa: E402
from paper_2412_12218_b200.device import DeviceGraph, gemm  # noqa: E402

PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "configs.npz")
G = dict(np.load(PATH))
INPUT_SEED, LAYER_SEED = 8, 1  # bench.py: the reference bench's seeds (bench.cpp:128-132)


def mre(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    assert a.shape == b.shape
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


@pytest.mark.parametrize("order", [0, 2])
def test_c1_cora_gcn(order):
    n = int(G["c1/n"])
    g = sg.CsrGraph(n, G["c1/node_pointer"], G["c1/edge_list"])
    gs = sg.normalize_graph(g, symmetrize=True, add_self_loops=True, dedupe=True)
    assert np.array_equal(gs.node_pointer, G["c1/norm_node_pointer"])
    assert np.array_equal(gs.edge_list, G["c1/norm_edge_list"])
    gn = sg.gcn_normalize_values(gs)
    assert np.array_equal(gn.values.view(np.uint32), G["c1/gcn_values"].view(np.uint32))
    t = sg.sgt_transform(gn)
    x = sg.dense_random(n, 1433, INPUT_SEED)
    layers = sg.random_gcn_layers(1433, 16, 7, 2, LAYER_SEED)
    assert mre(sg.gcn_forward(t, x, layers, order=order), G["c1/gcn_tf0"]) <= 1e-5
    assert mre(sg.gcn_forward(t, x, layers, precision="tf32", order=order),
               G["c1/gcn_tf1"]) <= gcn_tf32_bar()


def c2_forward(prec, mode):
    n = int(G["c2/n"])
    dg = DeviceGraph.from_csr(G["c2/node_pointer"], G["c2/edge_list"], None, n)
    x = dev(sg.dense_random(n, 500, INPUT_SEED))
    h0 = gemm(x, dev(G["c2/w_in"]), relu=True, precision=prec)
    h4, zeros = dg.agnn_forward(h0, np.ones(4, np.float32), precision=prec, mode=mode,
                                return_zeros=True)
    out = gemm(h4, dev(G["c2/w_out"]), relu=False, precision=prec)
    return h0.cpu().numpy(), h4.cpu().numpy(), out.cpu().numpy(), zeros


@pytest.mark.parametrize("mode", [3, 0, 1, 2])
def test_c2_pubmed_agnn(mode):
    rows = G["c2/rows"]
    h0, h4, out, zeros = c2_forward("fp32", mode)
    assert mre(h0[rows], G["c2/h0_tf0_rows"]) <= 1e-5
    assert mre(h4[rows], G["c2/h4_tf0_rows"]) <= 1e-5
    assert mre(out, G["c2/out_tf0"]) <= 1e-5
    assert zeros == int(G["c2/zeros_tf0"])
    h0, h4, out, zeros = c2_forward("tf32", mode)
    # the reference's in-proj rounds X only (tf32 SpMM over identity, then a
    # plain fp32 matmul); ours rounds X and W: componentwise 2^-10 |X||W|
    assert mre(h0[rows], G["c2/h0_tf1_rows"]) <= TF32_STEP
    assert mre(h4[rows], G["c2/h4_tf1_rows"]) <= TF32_STEP + agnn_tf32_bar([1.0])
    assert mre(out, G["c2/out_tf1"]) <= 2 * TF32_STEP + agnn_tf32_bar([1.0])
