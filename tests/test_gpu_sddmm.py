"""sddmm_hybrid on the panel path (sddmm_panel.cu: tcgen05 dense columns +
CUDA-core sparse edges) against the CPU oracle (oracle/, pinned to the
reference's golden vectors) on graphs large enough to have dense panel chunks,
hub rows and ragged widths.  Bars as test_gpu_parity.py: FP32 <= 1e-5,
TF32 vs the reference's TF32 mode <= 2^-10: the reference rounds every dot to
TF32 (tile_exec.cpp:386,402) and the tensor core's fp32 sum runs in another
order, so a dot near a TF32 rounding boundary lands one TF32 step away."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2412_12218_b200 as sg  # noqa: E402
from paper_2412_12218_b200.device import DeviceGraph  # noqa: E402
from oracle.oracle import Csr, Oracle  # noqa: E402

O = Oracle()
TF32_BAR = 2.0 ** -10


def mre(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-30))


@pytest.fixture(scope="module", params=["local", "hubs"])
def graph(request):
    if request.param == "local":
        return sg.synth_graph(4000, 40.0, alpha=0.0, p_local=0.9, band=4.0, seed=31)
    return sg.synth_graph(6000, 25.0, alpha=2.0, p_local=0.6, band=4.0, seed=32)


@pytest.mark.parametrize("d", [8, 16, 25, 32, 48, 64])
@pytest.mark.parametrize("weighted", [False, True])
def test_sddmm_panels_vs_oracle(graph, d, weighted):
    g = sg.gcn_normalize_values(graph) if weighted else graph
    c = Csr.of(g.num_nodes, g.node_pointer, g.edge_list, g.values)
    t16 = sg.reblock(sg.sgt_transform(g), 16)
    x = sg.dense_random(g.num_nodes, d, 40 + d)
    y = sg.dense_random(g.num_nodes, d, 41 + d)
    assert t16.device.panel_info(d)["dense_entries"] > 0
    got = sg.sddmm_hybrid(t16, x, y)
    assert mre(got, O.sddmm(c, x, y)) <= 1e-5
    got = sg.sddmm_hybrid(t16, x, y, precision="tf32")
    assert mre(got, O.sddmm(c, x, y, tf32=True)) <= TF32_BAR
    ov = np.random.default_rng(d).uniform(-1, 1, g.num_edges).astype(np.float32)
    got = sg.sddmm_hybrid(t16, x, y, edge_values=ov)
    assert mre(got, O.sddmm(c, x, y, values=ov)) <= 1e-5


def test_sddmm_panels_device_api_scale_and_determinism(graph):
    dg = DeviceGraph.from_csr(graph.node_pointer, graph.edge_list)
    x = torch.from_numpy(sg.dense_random(graph.num_nodes, 32, 5)).cuda()
    a = dg.sddmm(x, x, precision="tf32", scale=0.75)
    b = dg.sddmm(x, x, precision="tf32", scale=0.75)
    assert torch.equal(a, b)  # no atomics: bit-identical reruns
    c = Csr.of(graph.num_nodes, graph.node_pointer, graph.edge_list)
    want = O.sddmm(c, x.cpu().numpy(), x.cpu().numpy(), tf32=True) * np.float32(0.75)
    assert mre(a.cpu().numpy(), want) <= TF32_BAR
