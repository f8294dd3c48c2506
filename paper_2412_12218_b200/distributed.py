"""Multi-GPU row-window partition: one process per GPU, NCCL all-gather over NVLink.

SURVEY.md §8(e).  Rows are split into contiguous ranges of whole 128-row
panels (the unit of the tensor-core SpMM, panel.cu; 8 reference 16-row
windows) balanced by edge count (sgtk_partition_windows).  Because panels are
independent (the reference's window-independence property,
/root/reference/proj/tests/test_sgt_transform.cpp:133-158) and work-unit
splitting depends on a window alone, each rank's transform of its slice equals
the global transform restricted to it, and every output row is bit-identical
for 1/2/4/8 GPUs.

Per layer the only exchange is the node-embedding all-gather:
  AGNN: h_full -> (l2norm, fused attention on local rows) -> all-gather
  GCN : h_local W (local rows) -> all-gather -> SpMM on local rows
There is no other collective on the data path.
"""

from __future__ import annotations

import ctypes as C

import numpy as np
import torch
import torch.distributed as dist

from ._lib import check, lib


ROW_QUANTUM = 128  # panel height: slices made of whole panels keep every output bit


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


def allgather_rows(local: torch.Tensor, ranges: list[tuple[int, int]], group=None) -> torch.Tensor:
    """Concatenate every rank's row slice (uneven slices: padded collective)."""
    world = len(ranges)
    if world == 1:
        return local
    maxr = max(r1 - r0 for r0, r1 in ranges)
    pad = torch.zeros((maxr,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    pad[:local.shape[0]] = local
    if dist.get_backend(group) == "nccl":
        full = torch.empty((world * maxr,) + tuple(local.shape[1:]), dtype=local.dtype,
                           device=local.device)
        dist.all_gather_into_tensor(full, pad, group=group)
        parts = [full[p * maxr: p * maxr + (r1 - r0)] for p, (r0, r1) in enumerate(ranges)]
    else:
        bufs = [torch.empty_like(pad) for _ in range(world)]
        dist.all_gather(bufs, pad, group=group)
        parts = [bufs[p][: r1 - r0] for p, (r0, r1) in enumerate(ranges)]
    return torch.cat(parts)


class RowSlice:
    """One rank's share of a graph: its row slice resident on this GPU."""

    def __init__(self, node_pointer, edge_list, values, num_nodes: int, rank: int, world: int,
                 group=None, blk_h: int = 16, blk_w: int = 8):
        from .device import DeviceGraph

        self.n = num_nodes
        self.rank, self.world, self.group = rank, world, group
        self.bounds = partition(node_pointer, num_nodes, world)  # whole 128-row panels
        self.ranges = row_ranges(self.bounds, num_nodes)
        self.r0, self.r1 = self.ranges[rank]
        np_loc, el_loc, v_loc = local_csr(node_pointer, edge_list, values, self.r0, self.r1)
        if world == 1:
            self.graph = DeviceGraph.from_csr(np_loc, el_loc, v_loc, self.r1 - self.r0,
                                              blk_h=blk_h, blk_w=blk_w)
        else:
            self.graph = DeviceGraph.from_csr(np_loc, el_loc, v_loc, self.r1 - self.r0, blk_h,
                                              blk_w, num_cols=num_nodes, row_offset=self.r0)

    def allgather(self, local: torch.Tensor) -> torch.Tensor:
        return allgather_rows(local, self.ranges, self.group)

    def agnn_forward(self, h_full: torch.Tensor, betas, precision="tf32", mode=1) -> torch.Tensor:
        """All layers; returns this rank's rows of the last layer."""
        if self.world == 1:
            return self.graph.agnn_forward(h_full, betas, precision=precision, mode=mode)
        cur = h_full
        for l in range(len(betas)):
            loc = self.graph.agnn_forward(cur, np.asarray(betas[l:l + 1], np.float32),
                                          precision=precision, mode=mode)
            cur = self.allgather(loc) if l + 1 < len(betas) else loc
        return cur

    def gcn_forward(self, x_local: torch.Tensor, layers, precision="tf32") -> torch.Tensor:
        """Per layer, the same operand order as single-GPU gcn_forward(order=2):
        d_out < d_in: local h W, all-gather(h W), SpMM, ReLU;
        otherwise   : all-gather(h), SpMM, local GEMM with the ReLU epilogue.
        Every row is computed exactly as on one GPU (bit-identical)."""
        from .device import gemm, relu_

        if self.world == 1:
            return self.graph.gcn_forward(x_local, layers, precision=precision, order=2)
        h = x_local
        for w, relu in layers:
            if w.shape[1] < w.shape[0]:
                hw = gemm(h, w, relu=False, precision=precision)
                h = self.graph.spmm(self.allgather(hw), precision=precision)
                if relu:
                    relu_(h)
            else:
                agg = self.graph.spmm(self.allgather(h), precision=precision)
                h = gemm(agg, w, relu=relu, precision=precision)
        return h
