"""Multi-GPU row-window partition: one process per GPU, NCCL all-gather over NVLink.

SURVEY.md §8(e).  Rows are split into contiguous ranges of whole 128-row
panels (the unit of the tensor-core SpMM, panel.cu; 8 reference 16-row
windows) balanced by edge count (sgtk_partition_windows).  Because panels are
independent (the reference's window-independence property,
/root/reference/proj/tests/test_sgt_transform.cpp:133-158) and work-unit
splitting depends on a window alone, each rank's transform of its slice equals
the global transform restricted to it, and every output row is bit-identical
for 1/2/4/8 GPUs.

Replica layout (no copies around the collective).  Every rank keeps the node
embeddings in a *padded* replica of `world * stride` rows: rank p's rows live
at [p*stride, p*stride + n_p), `stride` = the largest slice rounded up to a
whole panel.  Each rank's column ids are renumbered into that space once, when
its slice is built (c -> owner(c)*stride + c - r0(owner); monotone, so the
slice stays sorted-unique and its SGT structure — window uniques, ranks, tile
maps — is the same as with global ids).  A layer writes its output rows
straight into its own block of the next replica, and the exchange is ONE
in-place `all_gather_into_tensor` over the replica (NCCL's in-place form:
send buffer = the rank's block of the receive buffer).  Padding rows are never
referenced by an edge.

Per layer the only exchange is that all-gather:
  AGNN: replica(h) -> layer on local rows (norms computed from the replica) -> all-gather
  GCN : d_out < d_in: local h W into the replica -> all-gather -> SpMM (+ReLU)
        otherwise   : h in the replica -> all-gather -> SpMM -> local GEMM (+ReLU)
There is no other collective on the data path.

Overlap (`chunks=K > 1`, AGNN).  Each rank's rows are cut into K sub-slices
(the partition has world*K edge-balanced ranges of whole panels; rank p owns
ranges pK .. pK+K-1, still one contiguous row range); the replica has one
block per range, in row order (the remap stays monotone, so every sub-slice
keeps the global SGT structure and the outputs stay bit-identical).  A layer
runs sub-slice 0, then, on a second stream, all-gathers every rank's chunk-0
block into a contiguous staging buffer and scatters it into the replica's
chunk-0 blocks while sub-slice 1 computes, and so on; the next layer waits
for the K exchanges.  K = 1 is the layout above.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from ._lib import check, lib


ROW_QUANTUM = 128  # panel height: slices made of whole panels keep every output bit
_INPLACE_OK = True  # NCCL's in-place all-gather (send buffer inside the receive buffer)


def partition(node_pointer: np.ndarray, num_nodes: int, parts: int,
              blk_h: int = ROW_QUANTUM) -> np.ndarray:
    """Panel bounds u64[parts+1] (edge-balanced, whole panels)."""
    b = np.zeros(parts + 1, np.uint64)
    np_ = np.ascontiguousarray(node_pointer, np.uint64)
    check(lib().sgtk_partition_windows(np_.ctypes.data, C.c_uint64(num_nodes), blk_h, parts,
                                       b.ctypes.data))
    return b


def row_ranges(bounds: np.ndarray, num_nodes: int,
               blk_h: int = ROW_QUANTUM) -> list[tuple[int, int]]:
    return [(min(num_nodes, int(bounds[p]) * blk_h), min(num_nodes, int(bounds[p + 1]) * blk_h))
            for p in range(len(bounds) - 1)]


def local_csr(node_pointer, edge_list, values, r0: int, r1: int):
    """Rows [r0, r1) with global column ids (the slice a rank transforms)."""
    e0, e1 = int(node_pointer[r0]), int(node_pointer[r1])
    np_loc = (np.asarray(node_pointer[r0:r1 + 1], np.uint64) - np.uint64(e0)).astype(np.uint64)
    return np_loc, edge_list[e0:e1], None if values is None else values[e0:e1]


def replica_stride(ranges: list[tuple[int, int]], quantum: int = ROW_QUANTUM) -> int:
    """Rows per rank block in the padded replica (a whole number of panels,
    so every block starts on a 16-row window boundary)."""
    m = max(r1 - r0 for r0, r1 in ranges)
    return max(quantum, (m + quantum - 1) // quantum * quantum)


def remap_columns(edge_list, ranges: list[tuple[int, int]], stride: int):
    """Global node ids -> padded-replica ids (monotone).  numpy or torch in,
    same kind out (torch: computed on the tensor's device)."""
    starts = [r0 for r0, _ in ranges]
    if isinstance(edge_list, torch.Tensor):
        el = edge_list.to(torch.int64)
        st = torch.tensor(starts, dtype=torch.int64, device=el.device)
        owner = torch.searchsorted(st, el, right=True) - 1
        return (el + owner * stride - st[owner]).to(torch.int32)
    el = np.asarray(edge_list, np.int64)
    st = np.asarray(starts, np.int64)
    owner = np.searchsorted(st, el, side="right") - 1
    return (el + owner * stride - st[owner]).astype(np.uint32)


def allgather_rows(local: torch.Tensor, ranges: list[tuple[int, int]], group=None) -> torch.Tensor:
    """Concatenate every rank's row slice into an N-row matrix (uneven slices).
    Assembly helper for checks and final outputs; the layer loop uses the
    in-place padded replica (RowSlice.exchange) instead."""
    world = len(ranges)
    if world == 1:
        return local
    stride = replica_stride(ranges, 1)
    pad = torch.zeros((stride,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(bufs, pad, group=group)
    return torch.cat([bufs[p][: r1 - r0] for p, (r0, r1) in enumerate(ranges)])


def exchange_inplace(buf: torch.Tensor, rank: int, world: int, group=None) -> None:
    """All-gather rank blocks of a padded replica in place.  NCCL: one
    all_gather_into_tensor whose input is this rank's block of `buf`.  Other
    backends (gloo: CPU tests, several ranks sharing one device) gather through
    host copies of the blocks."""
    if world == 1:
        return
    stride = buf.shape[0] // world
    mine = buf[rank * stride:(rank + 1) * stride]
    if buf.is_cuda and dist.get_backend(group) == "nccl":
        global _INPLACE_OK
        if _INPLACE_OK:
            try:
                dist.all_gather_into_tensor(buf, mine, group=group)
                return
            except (RuntimeError, ValueError) as e:  # a torch build refusing aliased buffers
                _INPLACE_OK = False
                import warnings

                warnings.warn(f"in-place all_gather_into_tensor refused ({e}); "
                              "exchanging through a send copy")
        dist.all_gather_into_tensor(buf, mine.clone(), group=group)
        return
    host = buf.cpu() if buf.is_cuda else buf
    blocks = list(host.view(world, stride, *buf.shape[1:]).unbind(0))
    dist.all_gather(blocks, host[rank * stride:(rank + 1) * stride].clone(), group=group)
    if buf.is_cuda:
        buf.copy_(host)


class RowSlice:
    """One rank's share of a graph: its row slice resident on this GPU, with
    column ids in the padded-replica space (see module docstring).  chunks=K
    (AGNN) cuts it into K sub-slices whose all-gathers overlap the next one's
    compute (`graphs`, `chunk_ranges`; `graph` is the first)."""

    def __init__(self, node_pointer, edge_list, values, num_nodes: int, rank: int, world: int,
                 group=None, blk_h: int = 16, blk_w: int = 8, build_graph: bool = True,
                 chunks: int = 1):
        self.n = num_nodes
        self.rank, self.world, self.group = rank, world, group
        self.chunks = K = max(1, int(chunks)) if world > 1 else 1
        # world*K edge-balanced ranges of whole panels; rank p owns pK .. pK+K-1
        bounds_all = partition(node_pointer, num_nodes, world * K)
        self.ranges_all = row_ranges(bounds_all, num_nodes)
        self.ranges = [(self.ranges_all[p * K][0], self.ranges_all[p * K + K - 1][1]) for p in range(world)]
        self.bounds = np.array([bounds_all[p * K] for p in range(world)] + [bounds_all[-1]], np.uint64)
        self.r0, self.r1 = self.ranges[rank]
        self.rows = self.r1 - self.r0
        self.stride = replica_stride(self.ranges_all) if world > 1 else num_nodes
        self.padded_rows = self.stride * world * K if world > 1 else num_nodes
        # one replica block per range, in row order (block q = pK + k)
        self.chunk_ranges = self.ranges_all[rank * K:(rank + 1) * K]
        self.chunk_offsets = ([(rank * K + k) * self.stride for k in range(K)]
                              if world > 1 else [0])
        self.offset = self.chunk_offsets[0]
        self.csrs, self.graphs = [], []
        for k, (c0, c1) in enumerate(self.chunk_ranges):
            np_loc, el_loc, v_loc = local_csr(node_pointer, edge_list, values, c0, c1)
            if world > 1:
                el_loc = remap_columns(el_loc, self.ranges_all, self.stride)
            self.csrs.append((np_loc, el_loc, v_loc))
            if build_graph:
                from .device import DeviceGraph

                if world == 1:
                    self.graphs.append(DeviceGraph.from_csr(np_loc, el_loc, v_loc, c1 - c0,
                                                            blk_h=blk_h, blk_w=blk_w))
                else:
                    self.graphs.append(DeviceGraph.from_csr(np_loc, el_loc, v_loc, c1 - c0, blk_h,
                                                            blk_w, num_cols=self.padded_rows,
                                                            row_offset=self.chunk_offsets[k]))
        self.csr = self.csrs[0]
        self.graph = self.graphs[0] if self.graphs else None
        self._comm = None
        self._stage = {}

    # ---- replica management -------------------------------------------------
    def replica(self, d: int, device=None, dtype=torch.float32) -> torch.Tensor:
        """A zeroed padded replica [padded_rows, d] (padding rows stay zero)."""
        return torch.zeros((self.padded_rows, d), dtype=dtype, device=device)

    def mine(self, buf: torch.Tensor) -> torch.Tensor:
        """This rank's rows inside a replica (a view: writes land in place);
        chunks > 1: mine_k / write_mine (the rows sit in K blocks)."""
        if self.chunks > 1:
            raise ValueError("RowSlice.mine: chunked layout, use mine_k(buf, k)")
        return buf[self.offset:self.offset + self.rows]

    def mine_k(self, buf: torch.Tensor, k: int) -> torch.Tensor:
        """Sub-slice k's rows inside a replica (a view)."""
        c0, c1 = self.chunk_ranges[k]
        o = self.chunk_offsets[k]
        return buf[o:o + (c1 - c0)]

    def write_mine(self, buf: torch.Tensor, rows: torch.Tensor) -> None:
        """Copy this rank's rows (in row order) into their replica blocks."""
        at = 0
        for k, (c0, c1) in enumerate(self.chunk_ranges):
            self.mine_k(buf, k).copy_(rows[at:at + (c1 - c0)], non_blocking=True)
            at += c1 - c0

    def exchange(self, buf: torch.Tensor) -> None:
        if self.chunks == 1:
            exchange_inplace(buf, self.rank, self.world, self.group)
            return
        works = [self.exchange_chunk(buf, k) for k in range(self.chunks)]
        for w in works:
            if w is not None:
                w.wait()

    def exchange_chunk(self, buf: torch.Tensor, k: int):
        """All-gather every rank's chunk-k block into a contiguous staging
        buffer (world x stride rows) and scatter it into the replica's chunk-k
        blocks.  NCCL: on a second stream, started once the current stream has
        written this rank's block; returns a handle whose wait() makes the
        current stream wait.  Other backends: synchronous, returns None."""
        W, K, S = self.world, self.chunks, self.stride
        view = buf.view(W, K, S, *buf.shape[1:])
        key = (k, tuple(buf.shape[1:]), buf.dtype, buf.device)
        if key not in self._stage:
            self._stage[key] = torch.empty((W * S,) + tuple(buf.shape[1:]), dtype=buf.dtype,
                                           device=buf.device)
        stage = self._stage[key]
        sv = stage.view(W, S, *buf.shape[1:])
        if not (buf.is_cuda and dist.get_backend(self.group) == "nccl"):
            sv[self.rank].copy_(view[self.rank, k])
            exchange_inplace(stage, self.rank, W, self.group)
            view[:, k].copy_(sv)
            return None
        if self._comm is None:
            self._comm = torch.cuda.Stream(device=buf.device)
        ready = torch.cuda.Event()
        ready.record(torch.cuda.current_stream(buf.device))
        with torch.cuda.stream(self._comm):
            self._comm.wait_event(ready)
            sv[self.rank].copy_(view[self.rank, k])
            dist.all_gather_into_tensor(stage, sv[self.rank], group=self.group)
            view[:, k].copy_(sv)
            done = torch.cuda.Event()
            done.record(self._comm)

        class _Done:
            def wait(self_inner):
                torch.cuda.current_stream(buf.device).wait_event(done)

        return _Done()

    def scatter_full(self, full: torch.Tensor, buf: torch.Tensor) -> torch.Tensor:
        """Write an N-row matrix into the replica layout (inputs, tests)."""
        if self.world == 1:
            buf.copy_(full)
            return buf
        for q, (r0, r1) in enumerate(self.ranges_all):
            buf[q * self.stride:q * self.stride + (r1 - r0)] = full[r0:r1]
        return buf

    def gather_full(self, buf: torch.Tensor) -> torch.Tensor:
        """Replica -> N-row matrix (outside any timed region)."""
        if self.world == 1:
            return buf
        return torch.cat([buf[q * self.stride:q * self.stride + (r1 - r0)]
                          for q, (r0, r1) in enumerate(self.ranges_all)])

    # ---- layers -------------------------------------------------------------
    def agnn_forward(self, h_rep: torch.Tensor, betas, precision="tf32", mode=3,
                     scratch=None, out=None) -> torch.Tensor:
        """All layers.  h_rep: the input replica (already exchanged; left
        intact).  Every layer but the last writes its rows into a scratch
        replica (two, used in turn) and exchanges it in place; returns this
        rank's rows of the last layer."""
        b = np.asarray(betas, np.float32)
        if self.world == 1:
            return self.graph.agnn_forward(h_rep, b, precision=precision, mode=mode, out=out)
        if scratch is None:
            scratch = (torch.zeros_like(h_rep), torch.zeros_like(h_rep))
        if self.chunks > 1:
            return self._agnn_chunked(h_rep, b, precision, mode, scratch, out)
        src = h_rep
        for l in range(len(b)):
            if l + 1 == len(b):
                return self.graph.agnn_forward(src, b[l:l + 1], precision=precision, mode=mode,
                                               out=out)
            dst = scratch[l % 2]
            self.graph.agnn_forward(src, b[l:l + 1], precision=precision, mode=mode,
                                    out=self.mine(dst))
            self.exchange(dst)
            src = dst
        return self.mine(h_rep).clone() if out is None else out.copy_(self.mine(h_rep))

    def _agnn_chunked(self, h_rep, b, precision, mode, scratch, out):
        """agnn_forward with chunks > 1: per layer, sub-slice k's rows land in
        their block and that chunk's all-gather starts while sub-slice k+1
        computes; the next layer waits for all K."""
        if out is None:
            out = torch.empty((self.rows, h_rep.shape[1]), dtype=h_rep.dtype, device=h_rep.device)
        src = h_rep
        for l in range(len(b)):
            last = l + 1 == len(b)
            dst = None if last else scratch[l % 2]
            works, at = [], 0
            for k, g in enumerate(self.graphs):
                c0, c1 = self.chunk_ranges[k]
                if last:
                    g.agnn_forward(src, b[l:l + 1], precision=precision, mode=mode,
                                   out=out[at:at + (c1 - c0)])
                else:
                    g.agnn_forward(src, b[l:l + 1], precision=precision, mode=mode,
                                   out=self.mine_k(dst, k))
                    works.append(self.exchange_chunk(dst, k))
                at += c1 - c0
            for w in works:
                if w is not None:
                    w.wait()
            if dst is not None:
                src = dst
        return out

    def gcn_forward(self, x_local: torch.Tensor, layers, precision="tf32",
                    reps: dict | None = None, nonfinite=None) -> torch.Tensor:
        """Per layer, the same operand order as single-GPU gcn_forward(order=2):
        d_out < d_in: local h W (into the replica), all-gather, SpMM, ReLU;
        otherwise   : h into the replica, all-gather, SpMM, local GEMM + ReLU.
        Every row is computed exactly as on one GPU (bit-identical).  `reps`
        caches replicas by width across calls."""
        from .device import gemm, relu_

        if self.world == 1:
            return self.graph.gcn_forward(x_local, layers, precision=precision, order=2,
                                          nonfinite=nonfinite)
        if self.chunks > 1:
            raise ValueError("RowSlice.gcn_forward: the chunked (overlap) layout is built for AGNN")
        reps = {} if reps is None else reps

        def rep(d):
            if d not in reps:
                reps[d] = self.replica(d, device=x_local.device)
            return reps[d]

        def narrows(w):  # A (h W) order: all-gather the narrower h W
            return w.shape[1] < w.shape[0]

        h = x_local
        for l, (w, relu) in enumerate(layers):
            nxt = layers[l + 1][0] if l + 1 < len(layers) else None
            # a GEMM whose output the next layer all-gathers writes it in place
            dst = self.mine(rep(w.shape[1])) if nxt is not None and not narrows(nxt) else None
            if narrows(w):
                r = rep(w.shape[1])
                gemm(h, w, relu=False, precision=precision, out=self.mine(r))
                self.exchange(r)
                h = self.graph.spmm(r, precision=precision, out=dst)
                if relu:
                    relu_(h)
            else:
                r = rep(w.shape[0])
                m = self.mine(r)
                if m.data_ptr() != h.data_ptr():
                    m.copy_(h)  # layer-0 input (later layers land here already)
                self.exchange(r)
                h = gemm(self.graph.spmm(r, precision=precision), w, relu=relu,
                         precision=precision, out=dst)
        return h
