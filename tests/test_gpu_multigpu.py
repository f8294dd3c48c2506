"""Row-window partition on the GPU path, emulated on one device: every rank's
row-slice graph (sgtk_graph_create_rows) run over the full feature replica
must reproduce the single-graph output bit for bit (the
analogue of the reference's 1-vs-8-worker determinism criterion,
acceptance.cpp:322-362)."""

import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

import paper_2412_12218_b200 as sg  # noqa: E402
from paper_2412_12218_b200.device import DeviceGraph, gemm, relu_  # noqa: E402
from paper_2412_12218_b200.distributed import RowSlice, local_csr, partition, row_ranges  # noqa: E402


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a, np.float32)).cuda()


@pytest.fixture(scope="module")
def graph():
    # hubs give split windows (multi-unit) in some slices
    return sg.synth_graph(6000, 40.0, alpha=2.0, p_local=0.6, band=4.0, seed=21)


def slices(g, parts, values=None):
    b = partition(g.node_pointer, g.num_nodes, parts)
    out = []
    for r0, r1 in row_ranges(b, g.num_nodes):
        np_loc, el_loc, v_loc = local_csr(g.node_pointer, g.edge_list, values, r0, r1)
        out.append((r0, r1, DeviceGraph.from_csr(np_loc, el_loc, v_loc, r1 - r0,
                                                 num_cols=g.num_nodes, row_offset=r0)))
    return out


@pytest.mark.parametrize("parts", [2, 3, 4, 8])
@pytest.mark.parametrize("precision", ["fp32", "tf32"])
def test_agnn_layer_bit_identical_across_partitions(graph, parts, precision):
    g = graph
    whole = DeviceGraph.from_csr(g.node_pointer, g.edge_list)
    h = dev(sg.dense_random(g.num_nodes, 32, 5))
    betas = np.array([1.0, 0.8], np.float32)
    for mode in (0, 1, 2):  # chain, fused 16-row, panels (the bench's C4 mode)
        want = whole.agnn_forward(h, betas, precision=precision, mode=mode)
        cur = h
        for l in range(2):
            parts_out = [sl.agnn_forward(cur, betas[l:l + 1], precision=precision, mode=mode)
                         for _, _, sl in slices(g, parts)]
            cur = torch.cat(parts_out)
        assert torch.equal(cur, want), (parts, mode)


@pytest.mark.parametrize("parts", [2, 4, 8])
def test_gcn_bit_identical_across_partitions(graph, parts):
    g = sg.gcn_normalize_values(graph)
    whole = DeviceGraph.from_csr(g.node_pointer, g.edge_list, g.values)
    x = dev(sg.dense_random(g.num_nodes, 64, 7))
    layers = [(dev(w), r) for w, r in sg.random_gcn_layers(64, 64, 16, 2, 3)]
    want = whole.gcn_forward(x, layers, precision="fp32", order=2)
    sl = slices(g, parts, g.values)
    h_parts = [x[r0:r1] for r0, r1, _ in sl]
    for w, relu in layers:
        full = torch.cat(h_parts)
        if w.shape[1] < w.shape[0]:
            hw = torch.cat([gemm(hp, w, precision="fp32") for hp in h_parts])
            h_parts = [s.spmm(hw, precision="fp32") for _, _, s in sl]
            if relu:
                h_parts = [relu_(hp) for hp in h_parts]
        else:
            h_parts = [gemm(s.spmm(full, precision="fp32"), w, relu=relu, precision="fp32")
                       for _, _, s in sl]
    assert torch.equal(torch.cat(h_parts), want)


def padded_slices(g, parts, values=None):
    """Every rank of a `parts`-way partition in the padded-replica layout the
    bench and distributed.RowSlice use (remapped column ids).  On one device
    the ranks share one replica, so writing each rank's block of it is what
    the in-place all-gather produces."""
    return [RowSlice(g.node_pointer, g.edge_list, values, g.num_nodes, r, parts)
            for r in range(parts)]


@pytest.mark.parametrize("parts", [2, 3, 8])
@pytest.mark.parametrize("precision", ["fp32", "tf32"])
@pytest.mark.parametrize("mode", [0, 1, 2])
def test_agnn_padded_replica_bit_identical(graph, parts, precision, mode):
    g = graph
    whole = DeviceGraph.from_csr(g.node_pointer, g.edge_list)
    h = dev(sg.dense_random(g.num_nodes, 32, 5))
    betas = np.array([1.0, 0.8, 1.2], np.float32)
    want = whole.agnn_forward(h, betas, precision=precision, mode=mode)
    sl = padded_slices(g, parts)
    cur = sl[0].scatter_full(h, sl[0].replica(32, "cuda"))
    for l in range(len(betas)):
        nxt = sl[0].replica(32, "cuda")
        for s in sl:
            s.graph.agnn_forward(cur, betas[l:l + 1], precision=precision, mode=mode,
                                 out=s.mine(nxt))
        cur = nxt
    assert torch.equal(sl[0].gather_full(cur), want), (parts, mode)


@pytest.mark.parametrize("parts,chunks", [(2, 2), (3, 3), (4, 2)])
@pytest.mark.parametrize("precision", ["fp32", "tf32"])
def test_agnn_chunked_replica_bit_identical(graph, parts, chunks, precision):
    """The overlap layout (RowSlice chunks > 1: K sub-slices per rank, one
    block per sub-slice, a staged all-gather per chunk) on one device: every
    sub-slice writes its block of the shared replica, which is what the K
    exchanges produce; bit-identical to the whole graph."""
    g = graph
    whole = DeviceGraph.from_csr(g.node_pointer, g.edge_list)
    h = dev(sg.dense_random(g.num_nodes, 32, 5))
    betas = np.array([1.0, 0.8, 1.2], np.float32)
    want = whole.agnn_forward(h, betas, precision=precision, mode=2)
    sl = [RowSlice(g.node_pointer, g.edge_list, None, g.num_nodes, r, parts, chunks=chunks)
          for r in range(parts)]
    assert all(len(s.graphs) == chunks for s in sl)
    cur = sl[0].scatter_full(h, sl[0].replica(32, "cuda"))
    for l in range(len(betas)):
        nxt = sl[0].replica(32, "cuda")
        for s in sl:
            for k, gk in enumerate(s.graphs):
                gk.agnn_forward(cur, betas[l:l + 1], precision=precision, mode=2, out=s.mine_k(nxt, k))
        cur = nxt
    assert torch.equal(sl[0].gather_full(cur), want), (parts, chunks)


@pytest.mark.parametrize("parts", [2, 4])
def test_gcn_padded_replica_bit_identical(graph, parts):
    g = sg.gcn_normalize_values(graph)
    whole = DeviceGraph.from_csr(g.node_pointer, g.edge_list, g.values)
    x = dev(sg.dense_random(g.num_nodes, 64, 7))
    for dims in ([64, 64, 16], [64, 16, 32]):
        layers = [(dev(w), r) for w, r in sg.random_gcn_layers(dims[0], dims[1], dims[2], 2, 3)]
        for prec in ("fp32", "tf32"):
            want = whole.gcn_forward(x, layers, precision=prec, order=2)
            sl = padded_slices(g, parts, g.values)
            h = [x[s.r0:s.r1] for s in sl]
            for w, relu in layers:
                if w.shape[1] < w.shape[0]:
                    rep = sl[0].replica(w.shape[1], "cuda")
                    for s, hp in zip(sl, h):
                        gemm(hp, w, precision=prec, out=s.mine(rep))
                    h = [s.graph.spmm(rep, precision=prec) for s in sl]
                    if relu:
                        h = [relu_(hp) for hp in h]
                else:
                    rep = sl[0].replica(w.shape[0], "cuda")
                    for s, hp in zip(sl, h):
                        s.mine(rep).copy_(hp)
                    h = [gemm(s.graph.spmm(rep, precision=prec), w, relu=relu, precision=prec)
                         for s in sl]
            assert torch.equal(torch.cat(h), want), (parts, dims, prec)
