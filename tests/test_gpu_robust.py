"""Error semantics and reentrancy of the GPU path.

* agnn_forward raises NonFiniteError for NaN/Inf outputs in every mode, like
  the reference (spmm_hybrid's check, tile_exec.cpp:311-312, via gnn.cpp:115);
* the concurrent AGNN panel path is reentrant: host threads calling it at once
  (each with its own stream) get the single-threaded result bit for bit
  (per-thread auxiliary stream and events, agnn_panel.cu aux_streams).
"""
import threading

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2412_12218_b200 as sg  # noqa: E402
from paper_2412_12218_b200.device import DeviceGraph  # noqa: E402


@pytest.fixture(scope="module")
def graph():
    return sg.synth_graph(3000, 30.0, alpha=2.0, p_local=0.7, band=4.0, seed=5)


@pytest.mark.parametrize("mode", [0, 1, 2])
@pytest.mark.parametrize("precision", ["fp32", "tf32"])
@pytest.mark.parametrize("bad", [np.inf, -np.inf, np.nan])
def test_agnn_nonfinite_raises(graph, mode, precision, bad):
    t = sg.sgt_transform(graph)
    x = sg.dense_random(graph.num_nodes, 32, 3)
    x[123, 7] = bad
    with pytest.raises(sg.NonFiniteError):
        sg.agnn_forward(t, x, [1.0, 0.9, 1.1], precision=precision, mode=mode)
    x[123, 7] = 0.5  # finite again: no error
    out = sg.agnn_forward(t, x, [1.0, 0.9, 1.1], precision=precision, mode=mode)
    assert np.isfinite(out).all()


def test_agnn_panel_concurrent_host_threads(graph):
    dg = DeviceGraph.from_csr(graph.node_pointer, graph.edge_list)
    xs = [torch.from_numpy(sg.dense_random(graph.num_nodes, 32, 10 + i)).cuda() for i in range(4)]
    betas = np.array([1.0, 0.7], np.float32)
    want = [dg.agnn_forward(x, betas, precision="tf32", mode=2) for x in xs]
    got = [None] * 4
    errs = []

    def work(i):
        try:
            with torch.cuda.stream(torch.cuda.Stream()):
                for _ in range(5):
                    got[i] = dg.agnn_forward(xs[i], betas, precision="tf32", mode=2)
                torch.cuda.current_stream().synchronize()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=work, args=(i,)) for i in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for w, g in zip(want, got):
        assert torch.equal(w, g)
