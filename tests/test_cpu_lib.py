"""CPU-side checks of the product library (no GPU needed, no compute calls on
the device): the C-ABI .so loads and exports every symbol include/sgtk_cuda.h
declares; host-side logic (synthetic generator, partitioner, plan checks)."""

import ctypes as C
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2412_12218_b200 as sg
from oracle.oracle import Csr, Oracle
from tests._golden import golden

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "sgtk_cuda.h")


def declared_symbols():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(sgtk_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_entry_points():
    syms = declared_symbols()
    for s in ["sgtk_graph_create", "sgtk_spmm", "sgtk_sddmm", "sgtk_edge_softmax",
              "sgtk_gcn_forward", "sgtk_agnn_forward", "sgtk_gemm"]:
        assert s in syms


def test_library_exports_every_declared_symbol():
    L = sg.lib()
    missing = [s for s in declared_symbols() if not hasattr(L, s)]
    assert not missing, missing
    out = subprocess.run(["nm", "-D", "--defined-only", sg._lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = {l.split()[-1] for l in out.splitlines() if " T " in l}
    assert set(declared_symbols()) <= exported
    # only the C ABI and the sgtk:: C++ drop-in are exported (no internals,
    # no torch types)
    assert all(s.startswith("sgtk_") or s.startswith("_ZN4sgtk") for s in exported), \
        sorted(exported)[:10]
    assert set(sg.exported_symbols()) <= exported


def test_version_and_error_plumbing():
    L = sg.lib()
    assert b"sm_100a" in L.sgtk_version()
    # a host-only failure path: partitioner rejects zero parts -> RangeError
    np_ = np.array([0, 1, 2], np.uint64)
    b = np.zeros(2, np.uint64)
    with pytest.raises(sg.RangeError):
        sg.check(L.sgtk_partition_windows(np_.ctypes.data, 2, 16, 0, b.ctypes.data))
    with pytest.raises(sg.GeometryError):
        sg.check(L.sgtk_partition_windows(np_.ctypes.data, 2, 0, 1, b.ctypes.data))
    assert issubclass(sg.ShapeError, ValueError) and issubclass(sg.TileIndexError, IndexError)
    assert issubclass(sg.NonFiniteError, FloatingPointError)
    assert issubclass(sg.GraphIoError, OSError)


def test_dense_random_matches_reference_stream():
    G = golden()
    np.testing.assert_array_equal(sg.dense_random(5, 7, 8), G["kat_dense_random/seed8_5x7"])
    np.testing.assert_array_equal(sg.dense_random(4, 3, 3, -0.1, 0.1),
                                  G["kat_dense_random/seed3_4x3_m01"])
    layers = sg.random_gcn_layers(16, 32, 4, 3, 1)
    assert [w.shape for w, _ in layers] == [(16, 32), (32, 32), (32, 4)]
    assert [r for _, r in layers] == [True, True, False]
    assert all(np.abs(w).max() <= 0.1 for w, _ in layers)


@pytest.mark.parametrize("alpha,p_local", [(0.0, 0.0), (2.0, 0.5), (2.5, 0.9)])
def test_synth_graph_is_canonical_and_deterministic(alpha, p_local):
    g = sg.synth_graph(3000, 6.0, alpha=alpha, p_local=p_local, band=4.0, seed=11)
    g2 = sg.synth_graph(3000, 6.0, alpha=alpha, p_local=p_local, band=4.0, seed=11)
    np.testing.assert_array_equal(g.edge_list, g2.edge_list)
    O = Oracle()
    c = Csr.of(g.num_nodes, g.node_pointer, g.edge_list)
    # sorted-unique, in range (validate_csr) -> sgt_transform accepts it
    t = O.sgt_transform(c)
    assert t.block_counter > 0
    # symmetric with self-loops: normalize(sym, loops) is a no-op
    n2 = O.normalize_graph(c, symmetrize=True, add_self_loops=True)
    np.testing.assert_array_equal(n2.node_pointer, g.node_pointer)
    np.testing.assert_array_equal(n2.edge_list, g.edge_list)
    assert g.num_edges > 2 * 3000 * 6.0 * 0.6


def test_locality_knob_densifies_tiles():
    O = Oracle()
    dens = []
    for p in (0.0, 0.9):
        g = sg.synth_graph(4096, 8.0, p_local=p, band=2.0, seed=3)
        t = O.sgt_transform(Csr.of(g.num_nodes, g.node_pointer, g.edge_list))
        dens.append(g.num_edges / (t.block_counter * 128))
    assert dens[1] > 2 * dens[0]


@pytest.mark.parametrize("parts", [1, 2, 3, 4, 8])
def test_partition_windows_balanced(parts):
    g = sg.synth_graph(5000, 10.0, alpha=2.0, seed=5)
    b = np.zeros(parts + 1, np.uint64)
    sg.check(sg.lib().sgtk_partition_windows(g.node_pointer.ctypes.data, g.num_nodes, 16, parts,
                                             b.ctypes.data))
    W = (g.num_nodes + 15) // 16
    assert b[0] == 0 and b[-1] == W and np.all(np.diff(b.astype(np.int64)) >= 0)
    loads = [int(g.node_pointer[min(g.num_nodes, int(b[p + 1]) * 16)] -
                 g.node_pointer[min(g.num_nodes, int(b[p]) * 16)]) for p in range(parts)]
    assert max(loads) <= g.num_edges / parts + 0.05 * g.num_edges + 1000


def test_host_plan_validation_errors():
    # plan checks run on the host before any launch (tile_exec.cpp:35-42)
    class FakeDev:
        class info:
            num_windows = 2
            block_counter = 3

    t = sg.TransformedGraph.__new__(sg.TransformedGraph)
    t.csr = sg.CsrGraph(20, np.zeros(21), np.zeros(0))
    t.device = FakeDev()
    t._f = {"block_partition": np.array([2, 1], np.uint32)}
    with pytest.raises(sg.ShapeError):
        sg._check_plan(t, sg.HybridSplitPlan(1.0, np.array([1], np.uint32)))
    with pytest.raises(sg.ShapeError):
        sg._check_plan(t, sg.HybridSplitPlan(1.0, np.array([3, 0], np.uint32)))
    assert sg._check_plan(t, sg.HybridSplitPlan(1.0, np.array([2, 1], np.uint32))) is None
    np.testing.assert_array_equal(
        sg._check_plan(t, sg.HybridSplitPlan(0.5, np.array([1, 0], np.uint32))), [1, 0])
