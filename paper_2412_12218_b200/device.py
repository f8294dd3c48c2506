"""Device-resident API over the C ABI: torch CUDA tensors in, torch CUDA tensors out.

torch is used only as the allocator / stream provider (plumbing); all compute
runs in libsgtk_b200.so's sm_100a kernels.
"""

from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np
import torch

from ._lib import PRECISIONS, ShapeError, check, lib

u64 = C.c_uint64


def _ptr(t) -> int | None:
    if t is None:
        return None
    if isinstance(t, torch.Tensor):
        return t.data_ptr()
    if isinstance(t, np.ndarray):
        return t.ctypes.data
    raise TypeError(type(t))


def _stream() -> int:
    return torch.cuda.current_stream().cuda_stream


def _prec(p) -> int:
    if isinstance(p, int):
        return p
    try:
        return PRECISIONS[p]
    except KeyError:
        from ._lib import RangeError
        raise RangeError("precision must be 'fp32' or 'tf32'") from None


def _f32_2d(x: torch.Tensor, name: str) -> torch.Tensor:
    if not isinstance(x, torch.Tensor) or not x.is_cuda:
        raise TypeError(f"{name} must be a CUDA tensor")
    if x.dtype != torch.float32 or x.dim() != 2 or x.stride(1) != 1:
        raise ShapeError(f"{name} must be a 2-D float32 tensor with unit column stride")
    return x


@dataclass
class GraphInfo:
    num_nodes: int
    num_edges: int
    num_windows: int
    unique_cols: int
    block_counter: int
    blk_h: int
    blk_w: int
    has_values: bool
    tiles8: int
    tiles16: int
    work_units8: int


class DeviceGraph:
    """sgtk_graph handle: TransformedGraph + condensed tiles resident in HBM."""

    def __init__(self, handle: C.c_void_p, num_cols: int | None = None):
        self._h = handle
        a = np.zeros(11, np.uint64)
        check(lib().sgtk_graph_info(self._h, a.ctypes.data))
        self.info = GraphInfo(*(int(v) for v in a[:5]), int(a[5]), int(a[6]), bool(a[7]),
                              int(a[8]), int(a[9]), int(a[10]))
        self.num_cols = self.info.num_nodes if num_cols is None else num_cols
        self.row_offset = 0

    def __del__(self):
        h = getattr(self, "_h", None)
        if h and lib is not None:
            try:
                lib().sgtk_graph_destroy(h)
            except Exception:
                pass
            self._h = None

    @property
    def handle(self):
        return self._h

    # ---- construction ------------------------------------------------------
    @classmethod
    def from_csr(cls, node_pointer, edge_list, values=None, num_nodes=None, blk_h=16, blk_w=8,
                 num_cols=None, row_offset=0) -> "DeviceGraph":
        """sgt_transform on the GPU.  numpy inputs are host pointers, CUDA
        tensors device pointers."""
        dev = isinstance(node_pointer, torch.Tensor)
        if dev:
            np_ = node_pointer.contiguous()
            el = edge_list.contiguous()
            vals = None if values is None else values.contiguous()
            assert np_.dtype in (torch.int64, torch.uint64) and el.dtype in (torch.int32, torch.uint32)
        else:
            np_ = np.ascontiguousarray(node_pointer, np.uint64)
            el = np.ascontiguousarray(edge_list, np.uint32)
            vals = None if values is None else np.ascontiguousarray(values, np.float32)
        n = int(np_.shape[0]) - 1 if num_nodes is None else int(num_nodes)
        nnz = int(el.shape[0])
        h = C.c_void_p()
        kind = 1 if dev else 0
        if num_cols is None:
            check(lib().sgtk_graph_create(_ptr(np_), _ptr(el), _ptr(vals), u64(n), u64(nnz),
                                          blk_h, blk_w, kind, _stream(), C.byref(h)))
        else:
            check(lib().sgtk_graph_create_rows(_ptr(np_), _ptr(el), _ptr(vals), u64(n),
                                               u64(num_cols), u64(row_offset), u64(nnz), blk_h,
                                               blk_w, kind, _stream(), C.byref(h)))
        g = cls(h, num_cols)
        g.row_offset = row_offset
        return g

    @classmethod
    def import_fields(cls, node_pointer, edge_list, values, blk_h, blk_w, edge_to_column,
                      window_offsets, window_unique_cols) -> "DeviceGraph":
        np_ = np.ascontiguousarray(node_pointer, np.uint64)
        el = np.ascontiguousarray(edge_list, np.uint32)
        vals = None if values is None else np.ascontiguousarray(values, np.float32)
        e2c = np.ascontiguousarray(edge_to_column, np.uint32)
        wo = np.ascontiguousarray(window_offsets, np.uint64)
        wuc = np.ascontiguousarray(window_unique_cols, np.uint32)
        h = C.c_void_p()
        check(lib().sgtk_graph_import(_ptr(np_), _ptr(el), _ptr(vals), u64(np_.shape[0] - 1),
                                      u64(el.shape[0]), blk_h, blk_w, _ptr(e2c), _ptr(wo),
                                      _ptr(wuc), _stream(), C.byref(h)))
        return cls(h)

    def reblock(self, blk_w: int) -> "DeviceGraph":
        h = C.c_void_p()
        check(lib().sgtk_graph_reblock(self._h, blk_w, _stream(), C.byref(h)))
        return DeviceGraph(h, self.num_cols)

    # ---- fields ------------------------------------------------------------
    def fields(self) -> dict:
        i = self.info
        out = dict(edge_to_row=np.zeros(i.num_edges, np.uint32),
                   edge_to_column=np.zeros(i.num_edges, np.uint32),
                   block_partition=np.zeros(i.num_windows, np.uint32),
                   window_offsets=np.zeros(i.num_windows + 1, np.uint64),
                   window_unique_cols=np.zeros(i.unique_cols, np.uint32))
        check(lib().sgtk_graph_download(self._h, *(_ptr(out[k]) for k in (
            "edge_to_row", "edge_to_column", "block_partition", "window_offsets",
            "window_unique_cols"))))
        out["block_counter"] = np.array(i.block_counter, np.uint64)
        return out

    def build_times(self) -> dict:
        """Per-stage host wall time (ms) of this graph's build; populated when
        the process set SGTK_BUILD_TIMING before building (sgtk_graph_build_times)."""
        a = np.zeros(8, np.float64)
        check(lib().sgtk_graph_build_times(self._h, a.ctypes.data))
        names = ["upload", "validate", "edge_to_row", "windows_user", "windows_16",
                 "tiles_units", "panels"]
        return {k: round(float(v), 3) for k, v in zip(names, a)}

    def panel_info(self, d: int | None = None) -> dict:
        """128-row panel format sizes (sgtk_panel_info); with d, of the format
        an operation of width d runs on (sgtk_panel_info_for)."""
        a = np.zeros(8, np.uint64)
        if d is None:
            check(lib().sgtk_panel_info(self._h, a.ctypes.data))
        else:
            check(lib().sgtk_panel_info_for(self._h, u64(d), a.ctypes.data))
        return dict(zip(("panels", "dense_chunks", "dense_entries", "sparse_edges",
                         "max_chunk_entries", "dense_columns", "long_rows", "segments"),
                        (int(v) for v in a)))

    def panel_arrays(self) -> dict:
        i = self.panel_info()
        out = dict(chunk_ptr=np.zeros(i["panels"] + 1, np.uint32),
                   dense_cols=np.zeros(i["dense_columns"], np.uint32),
                   chunk_off=np.zeros(i["dense_chunks"] + 1, np.uint64),
                   dense_entries=np.zeros(i["dense_entries"], np.uint32),
                   sparse_ptr=np.zeros(self.info.num_nodes + 1, np.uint32),
                   sparse_entries=np.zeros(2 * i["sparse_edges"], np.uint32))
        check(lib().sgtk_panel_download(self._h, *(_ptr(out[k]) for k in (
            "chunk_ptr", "dense_cols", "chunk_off", "dense_entries", "sparse_ptr",
            "sparse_entries"))))
        return out

    def block_stats(self):
        s = np.zeros(3, np.uint64)
        d = C.c_double()
        check(lib().sgtk_block_stats(self._h, s.ctypes.data, C.byref(d)))
        return int(s[0]), int(s[1]), int(s[2]), d.value

    def split_plan(self, ratio: float) -> np.ndarray:
        cut = np.zeros(self.info.num_windows, np.uint32)
        check(lib().sgtk_split_plan(self._h, C.c_double(ratio), cut.ctypes.data))
        return cut

    def gather_tile(self, window: int, tile: int):
        a = np.zeros((self.info.blk_h, self.info.blk_w), np.float32)
        idx = np.zeros(self.info.blk_w, np.uint32)
        check(lib().sgtk_gather_tile(self._h, u64(window), u64(tile), a.ctypes.data,
                                     idx.ctypes.data))
        return a, idx

    def device_ptrs(self) -> list[int]:
        arr = (C.c_void_p * 8)()
        check(lib().sgtk_graph_device_ptrs(self._h, arr))
        return [arr[i] for i in range(8)]

    # ---- kernels -----------------------------------------------------------
    def _cut(self, cut):
        if cut is None:
            return None
        if isinstance(cut, np.ndarray):
            cut = torch.from_numpy(np.ascontiguousarray(cut, np.uint32).view(np.int32)).cuda()
        return cut

    def spmm(self, x: torch.Tensor, cut=None, edge_values=None, precision="fp32", out=None,
             nonfinite: torch.Tensor | None = None) -> torch.Tensor:
        _f32_2d(x, "x")
        if x.shape[0] != self.num_cols:
            raise ShapeError("spmm_hybrid: x.rows != num_nodes")
        d = x.shape[1]
        if out is None:
            out = torch.empty((self.info.num_nodes, d), dtype=torch.float32, device=x.device)
        if edge_values is not None and edge_values.numel() != self.info.num_edges:
            raise ShapeError("edge value override length does not match edge count")
        cut = self._cut(cut)
        check(lib().sgtk_spmm(self._h, _ptr(x), u64(x.stride(0)), u64(d), _ptr(cut),
                              _ptr(edge_values), _prec(precision), _ptr(out), u64(out.stride(0)),
                              _ptr(nonfinite), _stream()))
        return out

    def sddmm(self, x, y, cut16=None, edge_values=None, precision="fp32", scale=1.0,
              out=None) -> torch.Tensor:
        _f32_2d(x, "x")
        _f32_2d(y, "y")
        if x.shape[0] != self.info.num_nodes or y.shape[0] != self.num_cols:
            raise ShapeError("sddmm_hybrid: feature rows != num_nodes")
        if x.shape[1] != y.shape[1]:
            raise ShapeError("sddmm_hybrid: x.cols != y.cols")
        if out is None:
            out = torch.empty(self.info.num_edges, dtype=torch.float32, device=x.device)
        cut16 = self._cut(cut16)
        check(lib().sgtk_sddmm(self._h, _ptr(x), u64(x.stride(0)), _ptr(y), u64(y.stride(0)),
                               u64(x.shape[1]), _ptr(cut16), _ptr(edge_values), _prec(precision),
                               C.c_float(scale), _ptr(out), _stream()))
        return out

    def edge_softmax(self, logits: torch.Tensor, out=None) -> torch.Tensor:
        if logits.numel() != self.info.num_edges:
            raise ShapeError("edge_softmax: logits length != num_edges")
        if out is None:
            out = torch.empty_like(logits)
        check(lib().sgtk_edge_softmax(self._h, _ptr(logits), _ptr(out), _stream()))
        return out

    def gcn_forward(self, x, layers, cut=None, precision="fp32", order=2,
                    nonfinite: torch.Tensor | None = None) -> torch.Tensor:
        """layers: list of (W [d_in x d_out] CUDA f32, relu).  With `nonfinite`
        (a zeroed int32 CUDA tensor) the call is asynchronous (CUDA-graph
        capturable) and a NaN/Inf output sets it instead of raising."""
        _f32_2d(x, "x")
        if x.shape[0] != self.info.num_nodes:
            raise ShapeError("gcn_forward: x.rows != num_nodes")
        dims = [x.shape[1]]
        for w, _ in layers:
            if w.shape[0] != dims[-1]:
                raise ShapeError("gcn_forward: weight shape does not chain")
            dims.append(w.shape[1])
        dims_a = np.array(dims, np.uint64)
        relu = np.array([int(r) for _, r in layers], np.int32)
        wcat = torch.cat([w.contiguous().reshape(-1) for w, _ in layers]) if layers else None
        ws_bytes = lib().sgtk_gcn_workspace(self._h, len(layers), dims_a.ctypes.data)
        ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=x.device)
        out = torch.empty((self.info.num_nodes, dims[-1]), dtype=torch.float32, device=x.device)
        cut = self._cut(cut)
        if nonfinite is not None:
            check(lib().sgtk_gcn_forward_async(
                self._h, _ptr(x), u64(x.stride(0)), len(layers), dims_a.ctypes.data, _ptr(wcat),
                relu.ctypes.data, _ptr(cut), _prec(precision), order, _ptr(ws), u64(ws_bytes),
                _ptr(out), u64(out.stride(0)), _ptr(nonfinite), _stream()))
            return out
        check(lib().sgtk_gcn_forward(self._h, _ptr(x), u64(x.stride(0)), len(layers),
                                     dims_a.ctypes.data, _ptr(wcat), relu.ctypes.data, _ptr(cut),
                                     _prec(precision), order, _ptr(ws), u64(ws_bytes), _ptr(out),
                                     u64(out.stride(0)), _stream()))
        return out

    def agnn_forward(self, x, betas, cut=None, precision="fp32", mode=3, return_zeros=False,
                     out=None):
        _f32_2d(x, "x")
        if x.shape[0] != self.num_cols:  # == num_nodes unless a row slice (full replica in)
            raise ShapeError("agnn_forward: x.rows != num_nodes")
        d = x.shape[1]
        b = np.ascontiguousarray(betas, np.float32)
        ws_bytes = lib().sgtk_agnn_workspace(self._h, u64(d))
        ws = torch.empty(max(ws_bytes, 1), dtype=torch.uint8, device=x.device)
        if out is None:
            out = torch.empty((self.info.num_nodes, d), dtype=torch.float32, device=x.device)
        elif tuple(out.shape) != (self.info.num_nodes, d):
            raise ShapeError("agnn_forward: out shape != (num_nodes, d)")
        else:
            _f32_2d(out, "out")
        z = u64(0)
        cut = self._cut(cut)
        check(lib().sgtk_agnn_forward(self._h, _ptr(x), u64(x.stride(0)), u64(d), len(b),
                                      b.ctypes.data, _ptr(cut), _prec(precision), mode, _ptr(ws),
                                      u64(ws_bytes), _ptr(out), u64(out.stride(0)),
                                      C.byref(z) if return_zeros else None, _stream()))
        return (out, z.value) if return_zeros else out


def l2_normalize_rows(h: torch.Tensor, want_z=True):
    _f32_2d(h, "h")
    rows, cols = h.shape
    z = torch.empty_like(h) if want_z else None
    inv = torch.empty(rows, dtype=torch.float32, device=h.device)
    zeros = torch.zeros(1, dtype=torch.int64, device=h.device)
    check(lib().sgtk_l2_normalize_rows(_ptr(h), u64(rows), u64(cols), u64(h.stride(0)), _ptr(z),
                                       u64(z.stride(0) if z is not None else 0), _ptr(inv),
                                       _ptr(zeros), _stream()))
    return z, inv, int(zeros.item())


def gemm(a: torch.Tensor, w: torch.Tensor, relu=False, precision="fp32", out=None) -> torch.Tensor:
    _f32_2d(a, "a")
    w = w.contiguous()
    if w.shape[0] != a.shape[1]:
        raise ShapeError("matmul: inner dimensions differ")
    if out is None:
        out = torch.empty((a.shape[0], w.shape[1]), dtype=torch.float32, device=a.device)
    elif tuple(out.shape) != (a.shape[0], w.shape[1]):
        raise ShapeError("matmul: out shape != (rows, cols)")
    else:
        _f32_2d(out, "out")
    check(lib().sgtk_gemm(_ptr(a), u64(a.stride(0)), _ptr(w), u64(a.shape[0]), u64(a.shape[1]),
                          u64(w.shape[1]), int(relu), _prec(precision), _ptr(out),
                          u64(out.stride(0)), _stream()))
    return out


def relu_(x: torch.Tensor) -> torch.Tensor:
    """In-place ReLU on the GPU (the GCN layer activation, gnn.cpp:45-47)."""
    _f32_2d(x, "x")
    check(lib().sgtk_relu_inplace(_ptr(x), u64(x.shape[0]), u64(x.shape[1]), u64(x.stride(0)),
                                  _stream()))
    return x


def gcn_normalize_values(node_pointer: torch.Tensor, edge_list: torch.Tensor) -> torch.Tensor:
    n = node_pointer.numel() - 1
    vals = torch.empty(edge_list.numel(), dtype=torch.float32, device=edge_list.device)
    check(lib().sgtk_gcn_normalize_values(_ptr(node_pointer), _ptr(edge_list), u64(n), _ptr(vals),
                                          _stream()))
    return vals


def tf32_round(x: torch.Tensor) -> torch.Tensor:
    out = torch.empty_like(x)
    check(lib().sgtk_tf32_round(_ptr(x), _ptr(out), u64(x.numel()), _stream()))
    return out
