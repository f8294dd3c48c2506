"""B200-native (sm_100a) FTC-GNN aggregation path behind the reference's API.

Mirrors the reference's Python module ``sgtk`` (/root/reference/proj/python/sgtk/
__init__.py, bindings /root/reference/proj/src/python/bindings.cpp:83-363): the
same function names, argument meaning, defaults and exception types, with
numpy arrays on the host side.  Every call runs through the C ABI
(include/sgtk_cuda.h) on the GPU.  There is no CPU fallback: without
libsgtk_b200.so or a CUDA device the calls raise.

For device-resident work (torch CUDA tensors, no host copies) use
``DeviceGraph`` and the helpers in ``paper_2412_12218_b200.device``.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field

import numpy as np

from ._lib import (FP32, TF32, CudaError, DegreeError, GeometryError, GraphIoError,
                   GraphParseError, NodeIdOverflowError, NonFiniteError, RangeError, SgtkError,
                   ShapeError, TileIndexError, check, exported_symbols, lib)

__version__ = "0.1.0"


def _torch():
    import torch

    if not torch.cuda.is_available():
        raise CudaError("no CUDA device visible: the sm_100a path has no CPU fallback")
    return torch


# --------------------------------------------------------------------------
# Value types (csr_graph.hpp:13-30, sgt_transform.hpp:12-44, tile_exec.hpp:20-25)
# --------------------------------------------------------------------------
@dataclass
class CsrGraph:
    num_nodes: int
    node_pointer: np.ndarray
    edge_list: np.ndarray
    values: np.ndarray | None = None

    def __post_init__(self):
        self.node_pointer = np.ascontiguousarray(self.node_pointer, np.uint64)
        self.edge_list = np.ascontiguousarray(self.edge_list, np.uint32)
        if self.values is not None:
            self.values = np.ascontiguousarray(self.values, np.float32)

    @property
    def num_edges(self) -> int:
        return int(self.edge_list.shape[0])

    def __repr__(self):
        return f"CsrGraph(num_nodes={self.num_nodes}, num_edges={self.num_edges})"


@dataclass
class TileGeometry:
    blk_h: int = 16
    blk_w: int = 8


@dataclass
class BlockStats:
    block_counter: int
    capacity: int
    nnz: int
    mean_tile_density: float


@dataclass
class HybridSplitPlan:
    ratio: float = 1.0
    per_window_tile_cut: np.ndarray = field(default_factory=lambda: np.zeros(0, np.uint32))


class TransformedGraph:
    """sgt_transform output.  The fields live on the GPU (``device``); the
    numpy attributes download on first access."""

    def __init__(self, csr: CsrGraph, dev):
        self.csr = csr
        self.device = dev
        self.geometry = TileGeometry(dev.info.blk_h, dev.info.blk_w)
        self._f = None

    def _fields(self):
        if self._f is None:
            self._f = self.device.fields()
        return self._f

    edge_to_row = property(lambda s: s._fields()["edge_to_row"])
    edge_to_column = property(lambda s: s._fields()["edge_to_column"])
    block_partition = property(lambda s: s._fields()["block_partition"])
    window_offsets = property(lambda s: s._fields()["window_offsets"])
    window_unique_cols = property(lambda s: s._fields()["window_unique_cols"])

    @property
    def block_counter(self) -> int:
        return self.device.info.block_counter

    @property
    def num_windows(self) -> int:
        return self.device.info.num_windows

    def window_cols(self, w: int) -> np.ndarray:
        wo = self.window_offsets
        return self.window_unique_cols[int(wo[w]):int(wo[w + 1])]


# --------------------------------------------------------------------------
# Translator (sgt_transform.hpp:49-57)
# --------------------------------------------------------------------------
def sgt_transform(g: CsrGraph, blk_h: int = 16, blk_w: int = 8, threads: int = 0) -> TransformedGraph:
    """GPU SGT; bit-exact with the reference (threads is accepted and ignored)."""
    _torch()
    from .device import DeviceGraph

    dev = DeviceGraph.from_csr(g.node_pointer, g.edge_list, g.values, g.num_nodes, blk_h, blk_w)
    return TransformedGraph(g, dev)


def reblock(t: TransformedGraph, new_blk_w: int) -> TransformedGraph:
    return TransformedGraph(t.csr, t.device.reblock(new_blk_w))


def block_stats(t: TransformedGraph) -> BlockStats:
    return BlockStats(*t.device.block_stats())


def make_split_plan(t: TransformedGraph, ratio: float = 1.0) -> HybridSplitPlan:
    return HybridSplitPlan(float(ratio), t.device.split_plan(ratio))


def gather_tile(t: TransformedGraph, window: int, tile: int):
    return t.device.gather_tile(window, tile)


# --------------------------------------------------------------------------
# Kernels (tile_exec.hpp:48-67) — numpy in, numpy out, GPU in between
# --------------------------------------------------------------------------
def _check_plan(t: TransformedGraph, plan: HybridSplitPlan | None):
    """tile_exec.cpp:35-42 (ShapeError), done on the host before launch."""
    if plan is None:
        return None
    cut = np.ascontiguousarray(plan.per_window_tile_cut, np.uint32)
    if cut.shape[0] != t.num_windows:
        raise ShapeError("split plan window count does not match transform")
    if np.any(cut > t.block_partition):
        raise ShapeError("split plan cut exceeds tiles in window")
    return None if np.array_equal(cut, t.block_partition) else cut


def _mat(x, name="x") -> np.ndarray:
    x = np.ascontiguousarray(x, np.float32)
    if x.ndim != 2:
        raise ShapeError(f"{name}: expected a 2-D float array")
    return x


def _edges(t, v):
    if v is None:
        return None
    v = np.ascontiguousarray(v, np.float32)
    if v.ndim != 1 or v.shape[0] != t.csr.num_edges:
        raise ShapeError("edge value override length does not match edge count")
    return v


def _to_dev(a):
    torch = _torch()
    return None if a is None else torch.from_numpy(a).cuda()


def spmm_hybrid(t: TransformedGraph, x, plan: HybridSplitPlan | None = None, precision="fp32",
                threads: int = 0, edge_values=None) -> np.ndarray:
    torch = _torch()
    x = _mat(x)
    if x.shape[0] != t.csr.num_nodes:
        raise ShapeError("spmm_hybrid: x.rows != num_nodes")
    cut = _check_plan(t, plan)
    ev = _edges(t, edge_values)
    flag = torch.zeros(1, dtype=torch.int32, device="cuda")
    out = t.device.spmm(_to_dev(x), cut=cut, edge_values=_to_dev(ev), precision=precision,
                        nonfinite=flag)
    if int(flag.item()):
        raise NonFiniteError("spmm_hybrid: output contains NaN or Inf")
    return out.cpu().numpy()


def sddmm_hybrid(t: TransformedGraph, x, y, plan: HybridSplitPlan | None = None,
                 precision="fp32", threads: int = 0, edge_values=None) -> np.ndarray:
    x, y = _mat(x), _mat(y, "y")
    if x.shape[0] != t.csr.num_nodes or y.shape[0] != t.csr.num_nodes:
        raise ShapeError("sddmm_hybrid: feature rows != num_nodes")
    if x.shape[1] != y.shape[1]:
        raise ShapeError("sddmm_hybrid: x.cols != y.cols")
    cut = _check_plan(t, plan)
    ev = _edges(t, edge_values)
    out = t.device.sddmm(_to_dev(x), _to_dev(y), cut16=cut, edge_values=_to_dev(ev),
                         precision=precision)
    return out.cpu().numpy()


def edge_softmax(g, logits) -> np.ndarray:
    """Row softmax (gnn.cpp:54-72).  `g` may be a CsrGraph or TransformedGraph."""
    logits = np.ascontiguousarray(logits, np.float32)
    t = g if isinstance(g, TransformedGraph) else sgt_transform(g)
    if logits.shape[0] != t.csr.num_edges:
        raise ShapeError("edge_softmax: logits length != num_edges")
    return t.device.edge_softmax(_to_dev(logits)).cpu().numpy()


def l2_normalize_rows(m):
    """gnn.cpp:74-91 -> (normalized rows, zero-row count)."""
    from .device import l2_normalize_rows as dev_l2

    z, _, zeros = dev_l2(_to_dev(_mat(m, "m")))
    return z.cpu().numpy(), zeros


def tf32_round(m) -> np.ndarray:
    from .device import tf32_round as dev_tf32

    m = np.ascontiguousarray(m, np.float32)
    return dev_tf32(_to_dev(m)).cpu().numpy()


def tf32_round_value(v: float) -> float:
    return float(tf32_round(np.array([v], np.float32))[0])


# --------------------------------------------------------------------------
# Models (gnn.hpp:24-54)
# --------------------------------------------------------------------------
def gcn_forward(t: TransformedGraph, x, layers, plan: HybridSplitPlan | None = None,
                precision="fp32", threads: int = 0, order: int = 2) -> np.ndarray:
    """layers: list of (W [d_in x d_out], apply_relu)."""
    x = _mat(x)
    if x.shape[0] != t.csr.num_nodes:
        raise ShapeError("gcn_forward: x.rows != num_nodes")
    d = x.shape[1]
    ws = []
    for w, relu in layers:
        w = _mat(w, "weight")
        if w.shape[0] != d:
            raise ShapeError("gcn_forward: weight shape does not chain")
        d = w.shape[1]
        ws.append((_to_dev(w), bool(relu)))
    if not layers:
        return x.copy()
    cut = _check_plan(t, plan)
    return t.device.gcn_forward(_to_dev(x), ws, cut=cut, precision=precision,
                                order=order).cpu().numpy()


def agnn_forward(t: TransformedGraph, x, betas, plan: HybridSplitPlan | None = None,
                 precision="fp32", threads: int = 0, mode: int = 3, return_zeros=False):
    x = _mat(x)
    if x.shape[0] != t.csr.num_nodes:
        raise ShapeError("agnn_forward: x.rows != num_nodes")
    cut = _check_plan(t, plan)
    out, z = t.device.agnn_forward(_to_dev(x), list(betas), cut=cut, precision=precision,
                                   mode=mode, return_zeros=True)
    out = out.cpu().numpy()
    return (out, z) if return_zeros else out


# --------------------------------------------------------------------------
# Preprocessing and inputs
# --------------------------------------------------------------------------
def normalize_graph(g: CsrGraph, symmetrize: bool = False, add_self_loops: bool = False,
                    dedupe: bool = True) -> CsrGraph:
    """graph_io.cpp:195-259 on the GPU (bit-exact; bindings.cpp:209-216 defaults)."""
    h = C.c_void_p()
    np_ = np.ascontiguousarray(g.node_pointer, np.uint64)
    el = np.ascontiguousarray(g.edge_list, np.uint32)
    vals = None if g.values is None else np.ascontiguousarray(g.values, np.float32)
    check(lib().sgtk_normalize_graph(np_.ctypes.data, el.ctypes.data,
                                     None if vals is None else vals.ctypes.data,
                                     g.num_nodes, el.shape[0], int(symmetrize),
                                     int(add_self_loops), int(dedupe), 0, None, C.byref(h)))
    try:
        info = np.zeros(3, np.uint64)
        check(lib().sgtk_csr_info(h, info.ctypes.data))
        n, e, hv = (int(v) for v in info)
        out_np = np.empty(n + 1, np.uint64)
        out_el = np.empty(e, np.uint32)
        out_v = np.empty(e, np.float32) if hv else None
        check(lib().sgtk_csr_download(h, out_np.ctypes.data, out_el.ctypes.data,
                                      None if out_v is None else out_v.ctypes.data))
    finally:
        lib().sgtk_csr_destroy(h)
    return CsrGraph(n, out_np, out_el, out_v)


def gcn_normalize_values(g: CsrGraph) -> CsrGraph:
    """graph_io.cpp:261-277 on the GPU (bit-exact: fp64 inv-sqrt-degrees)."""
    from .device import gcn_normalize_values as dev_norm

    torch = _torch()
    vals = dev_norm(torch.from_numpy(g.node_pointer.view(np.int64)).cuda(),
                    torch.from_numpy(g.edge_list.view(np.int32)).cuda())
    return CsrGraph(g.num_nodes, g.node_pointer, g.edge_list, vals.cpu().numpy())


def csr_from_coo(n: int, rows, cols, values=None) -> CsrGraph:
    """csr_from_triples (csr_graph.cpp:41-60): stable (row, col) sort, no dedupe."""
    rows = np.asarray(rows, np.int64)
    cols = np.asarray(cols, np.int64)
    order = np.lexsort((cols, rows))  # stable
    np_ = np.zeros(n + 1, np.uint64)
    np_[1:] = np.cumsum(np.bincount(rows, minlength=n))
    vals = None if values is None else np.asarray(values, np.float32)[order]
    return CsrGraph(n, np_, cols[order].astype(np.uint32), vals)


def dense_random(rows: int, cols: int, seed: int, lo=-1.0, hi=1.0) -> np.ndarray:
    """DenseMatrix::random (dense_matrix.hpp:43-50), same stream as the reference."""
    out = np.empty((rows, cols), np.float32)
    lib().sgtk_dense_random(rows, cols, seed, C.c_float(lo), C.c_float(hi), out.ctypes.data)
    return out


def random_gcn_layers(in_dim, hidden_dim, out_dim, num_layers, seed):
    """gnn.cpp:121-137: U[-0.1, 0.1] weights, seed + l, ReLU on all but the last."""
    layers, d = [], in_dim
    for l in range(num_layers):
        last = l + 1 == num_layers
        do = out_dim if last else hidden_dim
        layers.append((dense_random(d, do, seed + l, -0.1, 0.1), not last))
        d = do
    return layers


def synth_graph(num_nodes: int, avg_picks: float, alpha: float = 0.0, p_local: float = 0.0,
                band: float = 4.0, seed: int = 1) -> CsrGraph:
    """Deterministic O(E) symmetric graph with self-loops (see sgtk_synth_create)."""
    h = C.c_void_p()
    check(lib().sgtk_synth_create(num_nodes, float(avg_picks), float(alpha), float(p_local),
                                  float(band), seed, C.byref(h)))
    try:
        n, e = C.c_uint64(), C.c_uint64()
        check(lib().sgtk_synth_info(h, C.byref(n), C.byref(e)))
        np_ = np.empty(n.value + 1, np.uint64)
        el = np.empty(e.value, np.uint32)
        check(lib().sgtk_synth_copy(h, np_.ctypes.data, el.ctypes.data))
    finally:
        lib().sgtk_synth_destroy(h)
    return CsrGraph(n.value, np_, el)


from .device import DeviceGraph  # noqa: E402  (re-export)

__all__ = [
    "FP32", "TF32", "BlockStats", "CsrGraph", "CudaError", "DegreeError", "DeviceGraph",
    "GeometryError", "GraphIoError", "GraphParseError", "HybridSplitPlan", "NodeIdOverflowError",
    "NonFiniteError", "RangeError", "SgtkError", "ShapeError", "TileGeometry", "TileIndexError",
    "TransformedGraph", "agnn_forward", "block_stats", "csr_from_coo", "dense_random",
    "edge_softmax", "exported_symbols", "gather_tile", "gcn_forward", "gcn_normalize_values",
    "l2_normalize_rows", "lib", "make_split_plan", "normalize_graph", "random_gcn_layers", "reblock", "sddmm_hybrid",
    "sgt_transform", "spmm_hybrid", "synth_graph", "tf32_round", "tf32_round_value",
]
