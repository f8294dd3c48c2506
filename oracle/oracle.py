"""TEST INFRASTRUCTURE ONLY — numpy face of the CPU oracle.

Two back ends with the same Python API:

* ``Oracle``  — our restatement (oracle/sgtk_oracle.cpp -> oracle/liboracle.so),
  always available (built by ``make -C oracle`` / ``__graft_entry__.build()``).
* ``RefLib``  — the unmodified reference compiled from /root/reference
  (oracle/_ref/libsgtk_ref.so, ``make -C oracle ref``); present in this container
  and shipped to the GPU box as a prebuilt .so.

Only tests/, ``__graft_entry__.smoke()`` and bench.py's cpu_baseline /
``--impl reference`` leg may import this module.  The product package
(paper_2412_12218_b200) never does.
"""

from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "liboracle.so")
REF_PATH = os.path.join(HERE, "_ref", "libsgtk_ref.so")

u64p = np.ctypeslib.ndpointer(np.uint64, flags="C_CONTIGUOUS")
u32p = np.ctypeslib.ndpointer(np.uint32, flags="C_CONTIGUOUS")
f32p = np.ctypeslib.ndpointer(np.float32, flags="C_CONTIGUOUS")
i32p = np.ctypeslib.ndpointer(np.int32, flags="C_CONTIGUOUS")


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"[{code}] {msg}")
        self.code = code


def _vp(a):
    """Pointer or NULL for an optional numpy array."""
    return None if a is None else a.ctypes.data_as(C.c_void_p)


@dataclass
class Csr:
    num_nodes: int
    node_pointer: np.ndarray  # u64[n+1]
    edge_list: np.ndarray  # u32[E]
    values: np.ndarray | None = None  # f32[E] or None

    @property
    def num_edges(self) -> int:
        return int(self.edge_list.shape[0])

    @staticmethod
    def of(n, np_, el, vals=None) -> "Csr":
        return Csr(
            int(n),
            np.ascontiguousarray(np_, dtype=np.uint64),
            np.ascontiguousarray(el, dtype=np.uint32),
            None if vals is None else np.ascontiguousarray(vals, dtype=np.float32),
        )


@dataclass
class Transform:
    """The TransformedGraph fields (sgt_transform.hpp:21-37)."""

    blk_h: int
    blk_w: int
    edge_to_row: np.ndarray
    edge_to_column: np.ndarray
    block_partition: np.ndarray
    window_offsets: np.ndarray
    window_unique_cols: np.ndarray
    block_counter: int

    def fields(self):
        return dict(
            edge_to_row=self.edge_to_row,
            edge_to_column=self.edge_to_column,
            block_partition=self.block_partition,
            window_offsets=self.window_offsets,
            window_unique_cols=self.window_unique_cols,
        )


class Oracle:
    """Our restatement; every method cites the reference function it follows."""

    def __init__(self, path: str = LIB_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.L = C.CDLL(path)
        L.or_last_error.restype = C.c_char_p
        L.or_tf32_round_value.restype = C.c_float
        L.or_tf32_round_value.argtypes = [C.c_float]
        for name in (
            "or_validate_csr or_sgt_count or_sgt_fill or_reblock or_split_plan "
            "or_spmm or_sddmm or_edge_softmax or_l2_normalize_rows or_matmul "
            "or_gcn_forward or_agnn_forward or_gcn_normalize_values "
            "or_normalize_graph"
        ).split():
            getattr(L, name).restype = C.c_int

    def _ok(self, rc):
        if rc:
            raise OracleError(rc, self.L.or_last_error().decode())

    # sgt_transform.cpp:18-77
    def sgt_transform(self, g: Csr, blk_h=16, blk_w=8) -> Transform:
        L = self.L
        if blk_h == 0 or blk_w == 0:
            raise OracleError(6, "tile dimensions must be positive")
        self._ok(L.or_validate_csr(C.c_uint64(g.num_nodes), _vp(g.node_pointer),
                                   _vp(g.edge_list), _vp(g.values),
                                   C.c_uint64(g.num_edges), 1))
        W = (g.num_nodes + blk_h - 1) // blk_h
        ucount = np.zeros(W, np.uint32)
        self._ok(L.or_sgt_count(C.c_uint64(g.num_nodes), _vp(g.node_pointer),
                                _vp(g.edge_list), C.c_uint32(blk_h), _vp(ucount)))
        wo = np.zeros(W + 1, np.uint64)
        wo[1:] = np.cumsum(ucount, dtype=np.uint64)
        E = g.num_edges
        e2r = np.zeros(E, np.uint32)
        e2c = np.zeros(E, np.uint32)
        bp = np.zeros(W, np.uint32)
        wuc = np.zeros(int(wo[-1]), np.uint32)
        self._ok(L.or_sgt_fill(C.c_uint64(g.num_nodes), _vp(g.node_pointer),
                               _vp(g.edge_list), C.c_uint32(blk_h), C.c_uint32(blk_w),
                               _vp(wo), _vp(e2r), _vp(e2c), _vp(bp), _vp(wuc)))
        return Transform(blk_h, blk_w, e2r, e2c, bp, wo, wuc, int(bp.sum(dtype=np.uint64)))

    # sgt_transform.cpp:79-91
    def reblock(self, t: Transform, blk_w: int) -> Transform:
        W = t.block_partition.shape[0]
        bp = np.zeros(W, np.uint32)
        bc = C.c_uint64(0)
        self._ok(self.L.or_reblock(C.c_uint64(W), _vp(t.window_offsets),
                                   C.c_uint32(blk_w), _vp(bp), C.byref(bc)))
        return Transform(t.blk_h, blk_w, t.edge_to_row, t.edge_to_column, bp,
                         t.window_offsets, t.window_unique_cols, bc.value)

    # tile_exec.cpp:150-161
    def split_plan(self, t: Transform, ratio: float) -> np.ndarray:
        cut = np.zeros(t.block_partition.shape[0], np.uint32)
        self._ok(self.L.or_split_plan(C.c_uint64(cut.shape[0]), _vp(t.block_partition),
                                      C.c_double(ratio), _vp(cut)))
        return cut

    # tile_exec.cpp:200-314 / oracle.cpp:7-20 (identical order, see header)
    def spmm(self, g: Csr, x, tf32=False, values=None) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        vals = g.values if values is None else np.ascontiguousarray(values, np.float32)
        out = np.zeros((g.num_nodes, x.shape[1]), np.float32)
        self._ok(self.L.or_spmm(C.c_uint64(g.num_nodes), _vp(g.node_pointer),
                                _vp(g.edge_list), _vp(vals), _vp(x),
                                C.c_uint64(x.shape[1]), int(tf32), _vp(out)))
        return out

    # tile_exec.cpp:316-411 / oracle.cpp:22-38
    def sddmm(self, g: Csr, x, y, tf32=False, values=None) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        y = np.ascontiguousarray(y, np.float32)
        vals = g.values if values is None else np.ascontiguousarray(values, np.float32)
        out = np.zeros(g.num_edges, np.float32)
        self._ok(self.L.or_sddmm(C.c_uint64(g.num_nodes), _vp(g.node_pointer),
                                 _vp(g.edge_list), _vp(vals), _vp(x), _vp(y),
                                 C.c_uint64(x.shape[1]), int(tf32), _vp(out)))
        return out

    # gnn.cpp:54-72
    def edge_softmax(self, g: Csr, logits) -> np.ndarray:
        logits = np.ascontiguousarray(logits, np.float32)
        out = np.zeros(g.num_edges, np.float32)
        self._ok(self.L.or_edge_softmax(C.c_uint64(g.num_nodes), _vp(g.node_pointer),
                                        _vp(logits), _vp(out)))
        return out

    # gnn.cpp:74-91
    def l2_normalize_rows(self, m):
        m = np.ascontiguousarray(m, np.float32)
        out = np.zeros_like(m)
        z = C.c_uint64(0)
        self._ok(self.L.or_l2_normalize_rows(C.c_uint64(m.shape[0]), C.c_uint64(m.shape[1]),
                                             _vp(m), _vp(out), C.byref(z)))
        return out, z.value

    # gnn.cpp:16-29
    def matmul(self, a, b, relu=False):
        a = np.ascontiguousarray(a, np.float32)
        b = np.ascontiguousarray(b, np.float32)
        out = np.zeros((a.shape[0], b.shape[1]), np.float32)
        self._ok(self.L.or_matmul(C.c_uint64(a.shape[0]), C.c_uint64(a.shape[1]),
                                  C.c_uint64(b.shape[1]), _vp(a), _vp(b), int(relu), _vp(out)))
        return out

    # gnn.cpp:33-52
    def gcn_forward(self, g: Csr, x, layers, tf32=False):
        """layers: list of (W [d_in x d_out] f32, relu: bool)."""
        x = np.ascontiguousarray(x, np.float32)
        dims = np.array([x.shape[1]] + [w.shape[1] for w, _ in layers], np.uint64)
        wcat = np.concatenate([np.ascontiguousarray(w, np.float32).ravel() for w, _ in layers])
        relu = np.array([int(r) for _, r in layers], np.int32)
        out = np.zeros((g.num_nodes, int(dims[-1])), np.float32)
        self._ok(self.L.or_gcn_forward(C.c_uint64(g.num_nodes), _vp(g.node_pointer),
                                       _vp(g.edge_list), _vp(g.values), _vp(x),
                                       C.c_uint32(len(layers)), _vp(dims), _vp(wcat),
                                       _vp(relu), int(tf32), _vp(out)))
        return out

    # gnn.cpp:93-119
    def agnn_forward(self, g: Csr, x, betas, tf32=False):
        x = np.ascontiguousarray(x, np.float32)
        b = np.ascontiguousarray(betas, np.float32)
        out = np.zeros_like(x)
        z = C.c_uint64(0)
        self._ok(self.L.or_agnn_forward(C.c_uint64(g.num_nodes), _vp(g.node_pointer),
                                        _vp(g.edge_list), _vp(x), C.c_uint64(x.shape[1]),
                                        C.c_uint32(len(b)), _vp(b), int(tf32), _vp(out),
                                        C.byref(z)))
        return out, z.value

    # graph_io.cpp:261-277
    def gcn_normalize_values(self, g: Csr) -> Csr:
        vals = np.zeros(g.num_edges, np.float32)
        self._ok(self.L.or_gcn_normalize_values(C.c_uint64(g.num_nodes), _vp(g.node_pointer),
                                                _vp(g.edge_list), _vp(vals)))
        return Csr(g.num_nodes, g.node_pointer, g.edge_list, vals)

    # graph_io.cpp:195-259
    def normalize_graph(self, g: Csr, symmetrize=False, add_self_loops=False, dedupe=True) -> Csr:
        nnz = C.c_uint64(0)
        args = [C.c_uint64(g.num_nodes), _vp(g.node_pointer), _vp(g.edge_list), _vp(g.values),
                int(symmetrize), int(add_self_loops), int(dedupe), C.byref(nnz)]
        self._ok(self.L.or_normalize_graph(*args, None, None, None))
        np_ = np.zeros(g.num_nodes + 1, np.uint64)
        el = np.zeros(nnz.value, np.uint32)
        vals = None if g.values is None else np.zeros(nnz.value, np.float32)
        self._ok(self.L.or_normalize_graph(*args, _vp(np_), _vp(el), _vp(vals)))
        return Csr(g.num_nodes, np_, el, vals)

    def tf32_round_value(self, v: float) -> float:
        return self.L.or_tf32_round_value(C.c_float(v))

    def tf32_round(self, a):
        """Vectorised restatement of tile_exec.cpp:131-142 (numpy bit ops)."""
        u = np.ascontiguousarray(a, np.float32).view(np.uint32).copy()
        special = (u & 0x7F800000) == 0x7F800000
        r = (u + np.uint32(0xFFF) + ((u >> 13) & 1)) & np.uint32(0xFFFFE000)
        sat = (r & 0x7F800000) == 0x7F800000
        r = np.where(sat, (r & 0x80000000) | np.uint32(0x7F7FE000), r)
        return np.where(special, u, r).astype(np.uint32).view(np.float32)

    def dense_random(self, r, c, seed, lo=-1.0, hi=1.0):
        out = np.zeros((r, c), np.float32)
        self.L.or_dense_random(C.c_uint64(r), C.c_uint64(c), C.c_uint64(seed),
                               C.c_float(lo), C.c_float(hi), _vp(out))
        return out


class RefLib:
    """The unmodified reference (oracle/_ref/libsgtk_ref.so via oracle/ref_shim.cpp)."""

    def __init__(self, path: str = REF_PATH):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref`")
        L = self.L = C.CDLL(path)
        L.ref_last_error.restype = C.c_char_p
        L.ref_tf32_round_value.restype = C.c_float
        L.ref_tf32_round_value.argtypes = [C.c_float]

    def _ok(self, rc):
        if rc:
            raise OracleError(rc, self.L.ref_last_error().decode())

    class _Handle:
        def __init__(self, lib, ptr, free):
            self.ptr, self._free = ptr, free

        def __del__(self):
            if self.ptr:
                self._free(self.ptr)
                self.ptr = None

    def csr(self, g: Csr):
        h = C.c_void_p()
        self._ok(self.L.ref_csr_create(C.c_uint64(g.num_nodes), _vp(g.node_pointer),
                                       _vp(g.edge_list), _vp(g.values),
                                       C.c_uint64(g.num_edges), C.byref(h)))
        return self._Handle(self, h, self.L.ref_csr_free)

    def csr_get(self, h) -> Csr:
        c = np.zeros(3, np.uint64)
        self.L.ref_csr_counts(h.ptr, _vp(c))
        n, E, hv = (int(v) for v in c)
        np_ = np.zeros(n + 1, np.uint64)
        el = np.zeros(E, np.uint32)
        vals = np.zeros(E, np.float32) if hv else None
        self.L.ref_csr_get(h.ptr, _vp(np_), _vp(el), _vp(vals))
        return Csr(n, np_, el, vals)

    def transform_handle(self, g: Csr, blk_h=16, blk_w=8, threads=0):
        hc = self.csr(g)
        h = C.c_void_p()
        self._ok(self.L.ref_transform(hc.ptr, C.c_uint32(blk_h), C.c_uint32(blk_w),
                                      int(threads), C.byref(h)))
        return self._Handle(self, h, self.L.ref_graph_free)

    def reblock_handle(self, th, blk_w):
        h = C.c_void_p()
        self._ok(self.L.ref_reblock(th.ptr, C.c_uint32(blk_w), C.byref(h)))
        return self._Handle(self, h, self.L.ref_graph_free)

    def transform_fields(self, th) -> Transform:
        c = np.zeros(7, np.uint64)
        self.L.ref_graph_counts(th.ptr, _vp(c))
        n, E, W, U, bc, bh, bw = (int(v) for v in c)
        t = Transform(bh, bw, np.zeros(E, np.uint32), np.zeros(E, np.uint32),
                      np.zeros(W, np.uint32), np.zeros(W + 1, np.uint64),
                      np.zeros(U, np.uint32), bc)
        self.L.ref_graph_fields(th.ptr, _vp(t.edge_to_row), _vp(t.edge_to_column),
                                _vp(t.block_partition), _vp(t.window_offsets),
                                _vp(t.window_unique_cols))
        return t

    def sgt_transform(self, g: Csr, blk_h=16, blk_w=8, threads=0) -> Transform:
        return self.transform_fields(self.transform_handle(g, blk_h, blk_w, threads))

    def split_plan(self, th, ratio):
        c = np.zeros(7, np.uint64)
        self.L.ref_graph_counts(th.ptr, _vp(c))
        cut = np.zeros(int(c[2]), np.uint32)
        self._ok(self.L.ref_split_plan(th.ptr, C.c_double(ratio), _vp(cut)))
        return cut

    def spmm(self, th, n, x, ratio=1.0, tf32=False, threads=0, values=None, cut=None):
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros((n, x.shape[1]), np.float32)
        ev = None if values is None else np.ascontiguousarray(values, np.float32)
        self._ok(self.L.ref_spmm(th.ptr, _vp(x), C.c_uint64(x.shape[1]), C.c_double(ratio),
                                 _vp(cut), int(tf32), int(threads), _vp(ev),
                                 C.c_uint64(0 if ev is None else ev.shape[0]), _vp(out)))
        return out

    def sddmm(self, th, E, x, y, ratio=1.0, tf32=False, threads=0, values=None):
        x = np.ascontiguousarray(x, np.float32)
        y = np.ascontiguousarray(y, np.float32)
        out = np.zeros(E, np.float32)
        ev = None if values is None else np.ascontiguousarray(values, np.float32)
        self._ok(self.L.ref_sddmm(th.ptr, _vp(x), _vp(y), C.c_uint64(x.shape[1]),
                                  C.c_double(ratio), None, int(tf32), int(threads), _vp(ev),
                                  C.c_uint64(0 if ev is None else ev.shape[0]), _vp(out)))
        return out

    def edge_softmax(self, g: Csr, logits):
        hc = self.csr(g)
        logits = np.ascontiguousarray(logits, np.float32)
        out = np.zeros(g.num_edges, np.float32)
        self._ok(self.L.ref_edge_softmax(hc.ptr, _vp(logits), C.c_uint64(logits.shape[0]),
                                         _vp(out)))
        return out

    def l2_normalize_rows(self, m):
        m = np.ascontiguousarray(m, np.float32)
        out = np.zeros_like(m)
        z = C.c_uint64(0)
        self._ok(self.L.ref_l2_normalize_rows(_vp(m), C.c_uint64(m.shape[0]),
                                              C.c_uint64(m.shape[1]), _vp(out), C.byref(z)))
        return out, z.value

    def gcn_forward(self, th, n, x, layers, ratio=1.0, tf32=False, threads=0):
        x = np.ascontiguousarray(x, np.float32)
        dims = np.array([x.shape[1]] + [w.shape[1] for w, _ in layers], np.uint64)
        wcat = np.concatenate([np.ascontiguousarray(w, np.float32).ravel() for w, _ in layers])
        relu = np.array([int(r) for _, r in layers], np.int32)
        out = np.zeros((n, int(dims[-1])), np.float32)
        self._ok(self.L.ref_gcn_forward(th.ptr, _vp(x), C.c_uint32(len(layers)), _vp(dims),
                                        _vp(wcat), _vp(relu), C.c_double(ratio), int(tf32),
                                        int(threads), _vp(out)))
        return out

    def agnn_forward(self, th, x, betas, ratio=1.0, tf32=False, threads=0):
        x = np.ascontiguousarray(x, np.float32)
        b = np.ascontiguousarray(betas, np.float32)
        out = np.zeros_like(x)
        z = C.c_uint64(0)
        self._ok(self.L.ref_agnn_forward(th.ptr, _vp(x), C.c_uint64(x.shape[1]),
                                         C.c_uint32(len(b)), _vp(b), C.c_double(ratio),
                                         int(tf32), int(threads), _vp(out), C.byref(z)))
        return out, z.value

    def normalize_graph(self, g: Csr, symmetrize=False, add_self_loops=False, dedupe=True):
        hc = self.csr(g)
        h = C.c_void_p()
        self._ok(self.L.ref_normalize_graph(hc.ptr, int(symmetrize), int(add_self_loops),
                                            int(dedupe), C.byref(h)))
        return self.csr_get(self._Handle(self, h, self.L.ref_csr_free))

    def gcn_normalize_values(self, g: Csr) -> Csr:
        hc = self.csr(g)
        h = C.c_void_p()
        self._ok(self.L.ref_gcn_normalize_values(hc.ptr, C.byref(h)))
        return self.csr_get(self._Handle(self, h, self.L.ref_csr_free))

    def gather_tile(self, th, w, tile, blk_h, blk_w):
        a = np.zeros((blk_h, blk_w), np.float32)
        idx = np.zeros(blk_w, np.uint32)
        self._ok(self.L.ref_gather_tile(th.ptr, C.c_uint64(w), C.c_uint64(tile), _vp(a), _vp(idx)))
        return a, idx

    def tf32_round_value(self, v):
        return self.L.ref_tf32_round_value(C.c_float(v))

    def random_gcn_layers(self, in_dim, hidden, out_dim, num_layers, seed):
        """The reference's seeded layer stack (gnn.cpp:121-137): [(W, relu)]."""
        dims = [in_dim] + [hidden] * (num_layers - 1) + [out_dim]
        w = np.zeros(sum(a * b for a, b in zip(dims[:-1], dims[1:])), np.float32)
        relu = np.zeros(num_layers, np.int32)
        self._ok(self.L.ref_random_gcn_layers(C.c_uint64(in_dim), C.c_uint64(hidden),
                                              C.c_uint64(out_dim), C.c_uint32(num_layers),
                                              C.c_uint64(seed), _vp(w), _vp(relu)))
        out, o = [], 0
        for l, (a, b) in enumerate(zip(dims[:-1], dims[1:])):
            out.append((w[o:o + a * b].reshape(a, b).copy(), bool(relu[l])))
            o += a * b
        return out

    def synth_graph(self, n, avg_picks, alpha=0.0, p_local=0.0, band=4.0, seed=1) -> Csr:
        """The bench's synthetic generator (paper_2412_12218_b200/csrc/synth.cpp,
        linked into this library so the reference arm never loads the product
        library); identical output to sgtk.synth_graph."""
        h = C.c_void_p()
        L = self.L
        L.sgtk_synth_create.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_double,
                                        C.c_double, C.c_uint64, C.POINTER(C.c_void_p)]
        L.sgtk_synth_destroy.argtypes = [C.c_void_p]
        rc = L.sgtk_synth_create(n, avg_picks, alpha, p_local, band, seed, C.byref(h))
        if rc:
            raise OracleError(rc, "sgtk_synth_create failed")
        try:
            nn, nnz = C.c_uint64(), C.c_uint64()
            L.sgtk_synth_info(h, C.byref(nn), C.byref(nnz))
            np_ = np.zeros(nn.value + 1, np.uint64)
            el = np.zeros(nnz.value, np.uint32)
            L.sgtk_synth_copy(h, _vp(np_), _vp(el))
        finally:
            L.sgtk_synth_destroy(h)
        return Csr(int(nn.value), np_, el, None)

    def threads(self, requested: int = 0) -> int:
        """resolve_thread_count (threading.cpp:9-22): the default worker count."""
        return int(self.L.ref_resolve_threads(int(requested)))

    def save_sgt(self, th, path: str):
        self._ok(self.L.ref_save_sgt(th.ptr, path.encode()))

    def load_sgt(self, path: str):
        h = C.c_void_p()
        self._ok(self.L.ref_load_sgt(path.encode(), C.byref(h)))
        return self._Handle(self, h, self.L.ref_graph_free)

    def oracle_spmm(self, g: Csr, x):
        """The reference's single-threaded oracle_spmm (oracle.cpp:7-20)."""
        hc = self.csr(g)
        x = np.ascontiguousarray(x, np.float32)
        out = np.zeros((g.num_nodes, x.shape[1]), np.float32)
        self._ok(self.L.ref_oracle_spmm(hc.ptr, _vp(x), C.c_uint64(x.shape[1]), _vp(out)))
        return out

    def dense_random(self, r, c, seed, lo=-1.0, hi=1.0):
        out = np.zeros((r, c), np.float32)
        self.L.ref_dense_random(C.c_uint64(r), C.c_uint64(c), C.c_uint64(seed),
                                C.c_float(lo), C.c_float(hi), _vp(out))
        return out
