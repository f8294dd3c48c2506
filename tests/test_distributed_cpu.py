"""Multi-process (gloo, world_size 2-3, CPU) tests of the row-window partition
driver (paper_2412_12218_b200/distributed.py): partition agreement across
ranks, the uneven-slice all-gather, and a full distributed AGNN / GCN forward
whose per-rank compute is the CPU oracle — the result must be bit-identical to
the single-process oracle (rows are independent)."""

import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2412_12218_b200 as sg
from paper_2412_12218_b200.distributed import (RowSlice, allgather_rows, exchange_inplace,
                                               local_csr, partition, remap_columns, row_ranges)
from oracle.oracle import Csr, Oracle


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def graph():
    return sg.synth_graph(1000, 5.0, alpha=2.0, p_local=0.7, band=4.0, seed=9)


def worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        O = Oracle()
        g = graph()
        n = g.num_nodes
        bounds = partition(g.node_pointer, n, world)
        # every rank computes the same partition
        allb = [torch.zeros(world + 1, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(allb, torch.from_numpy(bounds.astype(np.int64)))
        assert all(torch.equal(allb[0], b) for b in allb)
        ranges = row_ranges(bounds, n)
        r0, r1 = ranges[rank]
        # all-gather of uneven slices
        loc = torch.arange(r0, r1, dtype=torch.float32).reshape(-1, 1).repeat(1, 3)
        full = allgather_rows(loc, ranges)
        assert torch.equal(full[:, 0], torch.arange(n, dtype=torch.float32))
        # window independence: the slice's transform == the global one restricted
        np_loc, el_loc, _ = local_csr(g.node_pointer, g.edge_list, None, r0, r1)
        sl = Csr.of(r1 - r0, np_loc, el_loc)
        # oracle transform wants square graphs for validation; compare the
        # per-window unique columns directly
        tg = O.sgt_transform(Csr.of(n, g.node_pointer, g.edge_list))
        w0, w1 = r0 // 16, (r1 + 15) // 16
        for w in range(w0, w1):
            lo, hi = int(tg.window_offsets[w]), int(tg.window_offsets[w + 1])
            rows = range(w * 16, min(n, w * 16 + 16))
            cols = np.unique(np.concatenate([el_loc[int(np_loc[r - r0]):int(np_loc[r - r0 + 1])]
                                             for r in rows] or [np.zeros(0, np.uint32)]))
            assert np.array_equal(cols, tg.window_unique_cols[lo:hi])
        # distributed AGNN, oracle as the per-rank compute, one all-gather per layer
        x = sg.dense_random(n, 16, 3)
        betas = [1.0, 0.5, 1.3]
        h_full = x.copy()
        for l, b in enumerate(betas):
            z, _ = O.l2_normalize_rows(h_full)
            logits = O.sddmm(sl, z[r0:r1], z, values=np.ones(sl.num_edges, np.float32))
            logits = logits * np.float32(b)
            attn = O.edge_softmax(sl, logits)
            h_loc = O.spmm(sl, h_full, values=attn)
            h_full = allgather_rows(torch.from_numpy(h_loc), ranges).numpy()
        want, _ = O.agnn_forward(Csr.of(n, g.node_pointer, g.edge_list), x, betas)
        assert np.array_equal(h_full, want)
        # distributed GCN (A (h W) order with all-gather of h W)
        gn = O.gcn_normalize_values(Csr.of(n, g.node_pointer, g.edge_list))
        _, _, v_loc = local_csr(gn.node_pointer, gn.edge_list, gn.values, r0, r1)
        sv = Csr.of(r1 - r0, np_loc, el_loc, v_loc)
        w = sg.dense_random(16, 8, 5, -0.1, 0.1)
        hw = O.matmul(x[r0:r1], w)
        full_hw = allgather_rows(torch.from_numpy(hw), ranges).numpy()
        out_loc = O.spmm(sv, full_hw)
        out = allgather_rows(torch.from_numpy(out_loc), ranges).numpy()
        assert np.array_equal(out, O.spmm(gn, O.matmul(x, w)))
        # the padded replica the GPU path uses: remapped column ids, rows
        # written straight into this rank's block, one in-place all-gather
        # per layer (distributed.RowSlice / exchange_inplace)
        rs = RowSlice(g.node_pointer, g.edge_list, None, n, rank, world, build_graph=False)
        assert rs.stride % 128 == 0 and rs.padded_rows == world * rs.stride
        np_p, el_p, _ = rs.csr
        for r in range(rs.rows):
            row = el_p[int(np_p[r]):int(np_p[r + 1])].astype(np.int64)
            assert np.all(np.diff(row) > 0)  # monotone remap keeps rows sorted-unique
        sp = Csr.of(rs.rows, np_p, el_p)
        rep = rs.replica(16)
        rs.scatter_full(torch.from_numpy(x), rep)
        h_rep = rep.numpy()
        for l, b in enumerate(betas):
            z, _ = O.l2_normalize_rows(h_rep)
            logits = O.sddmm(sp, z[rs.offset:rs.offset + rs.rows], z,
                             values=np.ones(sp.num_edges, np.float32)) * np.float32(b)
            h_loc = O.spmm(sp, h_rep, values=O.edge_softmax(sp, logits))
            nxt = rs.replica(16)
            rs.mine(nxt).copy_(torch.from_numpy(h_loc))
            rs.exchange(nxt)
            h_rep = nxt.numpy()
        assert np.array_equal(rs.gather_full(torch.from_numpy(h_rep)).numpy(), want)
        # the chunked (overlap) layout: 2 sub-slices per rank, a block per
        # range, one all-gather per chunk (exchange_chunk), same result
        rc = RowSlice(g.node_pointer, g.edge_list, None, n, rank, world, build_graph=False, chunks=2)
        assert rc.padded_rows == 2 * world * rc.stride and len(rc.csrs) == 2
        assert (rc.r0, rc.r1) == rc.ranges[rank] and rc.chunk_ranges[0][0] == rc.r0
        assert rc.chunk_ranges[-1][1] == rc.r1
        rep = rc.replica(16)
        rc.scatter_full(torch.from_numpy(x), rep)
        assert np.array_equal(rc.gather_full(rep).numpy(), x)
        h_rep = rep.numpy()
        for l, b in enumerate(betas):
            z, _ = O.l2_normalize_rows(h_rep)
            nxt = rc.replica(16)
            for k, (c0, c1) in enumerate(rc.chunk_ranges):
                np_k, el_k, _ = rc.csrs[k]
                for rr in range(c1 - c0):
                    row = el_k[int(np_k[rr]):int(np_k[rr + 1])].astype(np.int64)
                    assert np.all(np.diff(row) > 0)
                sk = Csr.of(c1 - c0, np_k, el_k)
                o = rc.chunk_offsets[k]
                logits = O.sddmm(sk, z[o:o + (c1 - c0)], z,
                                 values=np.ones(sk.num_edges, np.float32)) * np.float32(b)
                h_k = O.spmm(sk, h_rep, values=O.edge_softmax(sk, logits))
                rc.mine_k(nxt, k).copy_(torch.from_numpy(h_k))
                assert rc.exchange_chunk(nxt, k) is None  # gloo: synchronous
            h_rep = nxt.numpy()
        assert np.array_equal(rc.gather_full(torch.from_numpy(h_rep)).numpy(), want)
        # exchange_inplace leaves padding rows untouched and fills every block
        buf = torch.full((world * 4, 2), -1.0)
        buf[rank * 4:rank * 4 + 3] = float(rank)
        exchange_inplace(buf, rank, world)
        for p in range(world):
            assert torch.all(buf[p * 4:p * 4 + 3] == p)
        q.put((rank, "ok"))
    except Exception as e:  # pragma: no cover - reported to the parent
        import traceback
        q.put((rank, traceback.format_exc()))
    finally:
        dist.destroy_process_group()


def test_remap_columns_monotone():
    ranges = [(0, 300), (300, 520), (520, 1000)]
    stride = 512
    el = np.arange(1000, dtype=np.uint32)
    m = remap_columns(el, ranges, stride)
    assert np.all(np.diff(m.astype(np.int64)) > 0)
    assert m[0] == 0 and m[300] == 512 and m[519] == 512 + 219 and m[520] == 1024
    mt = remap_columns(torch.from_numpy(el.astype(np.int32)), ranges, stride)
    assert np.array_equal(mt.numpy().astype(np.uint32), m)


@pytest.mark.parametrize("world", [2, 3])
def test_rowwindow_partition_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = free_port()
    procs = [ctx.Process(target=worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
    assert sorted(res) == [(r, "ok") for r in range(world)], res
