#!/usr/bin/env python3
"""Benchmark: FTC-GNN aggregation hot path on B200 (metric of BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload reddit-agnn|proteins-gcn|pubmed-agnn|cora-gcn|powerlaw-gcn]
                    [--precision fp32|tf32] [--mode panel|fused|chain] [--locality calibrated|uniform]

Default workload (config C4 of BASELINE.json): AGNN forward on a synthetic
Reddit-shaped graph (232,965 nodes, ~114.6M edges incl. self-loops; in-proj
602->32, 4 AGNN layers at d=32, beta=1, out-proj 32->41).  The metric is the
AGNN *layer-forward* time per graph: one step = the reference API call
agnn_forward(t, h0, 4 layers) on the whole graph, value = step ms / 4.
Inputs are resident in HBM; L2 is flushed (256 MB write) between timed steps;
per-step CUDA events on the launch stream, max over ranks.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/libsgtk_ref.so, compiled unmodified from /root/reference; the
oracle restatement if that .so is absent) on this host's cores: one step =
one AGNN layer through the reference's public functions (l2_normalize_rows,
sddmm_hybrid on reblock(t,16), edge_softmax, spmm_hybrid; gnn.cpp:107-116).
"""

from __future__ import annotations

import argparse
import csv
import ctypes as C
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0}

# Locality knob calibrated on the Cora shape against Table IV (681 TC blocks at
# 16x8): p_local=0.9, band=4*avg_picks gives ~700-750 blocks.
LOCALITY = {"calibrated": dict(p_local=0.9, band=4.0), "uniform": dict(p_local=0.0, band=4.0)}

WORKLOADS = {
    # name: nodes, target edges (sym + self-loops), degree tail alpha, model
    "reddit-agnn": dict(n=232965, e=114_615_892, alpha=4.0, kind="agnn", d_in=602, hidden=32,
                        d_out=41, layers=4, cfg="C4"),
    "pubmed-agnn": dict(n=19717, e=88648 + 19717, alpha=4.0, kind="agnn", d_in=500, hidden=32,
                        d_out=3, layers=4, cfg="C2"),
    "proteins-gcn": dict(n=132534, e=39_561_252, alpha=0.0, kind="gcn", d_in=64, hidden=64,
                         d_out=64, layers=2, cfg="C3"),
    "proteins16-gcn": dict(n=132534, e=39_561_252, alpha=0.0, kind="gcn", d_in=16, hidden=16,
                           d_out=16, layers=2, cfg="C3 (d=16)"),
    "cora-gcn": dict(n=2708, e=10556 + 2708, alpha=0.0, kind="gcn", d_in=1433, hidden=16,
                     d_out=7, layers=2, cfg="C1"),
    "powerlaw-gcn": dict(n=10_000_000, e=1_000_000_000, alpha=2.0, kind="gcn", d_in=128,
                         hidden=128, d_out=128, layers=2, cfg="C5"),
}


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ inputs
def make_graph(wl, locality, seed=1):
    """Synthetic symmetric graph of the workload's shape (deterministic)."""
    import paper_2412_12218_b200 as sg

    n, e = wl["n"], wl["e"]
    loc = LOCALITY[locality]
    picks = max((e - n) / (2.0 * n), 0.5)
    # duplicate picks (local ones collide) shrink E: calibrate on a 50k sample
    ns = min(n, 50_000)
    s = sg.synth_graph(ns, picks, wl["alpha"], loc["p_local"], loc["band"], seed)
    ratio = (s.num_edges - ns) / (2.0 * ns * picks)
    picks = picks / max(ratio, 0.3)
    g = sg.synth_graph(n, picks, wl["alpha"], loc["p_local"], loc["band"], seed)
    return g, dict(avg_picks=round(picks, 3), **loc, alpha=wl["alpha"])


class _NvmlSampler:
    """NVML clock/throttle polling thread (every ~2 ms): the timed region of a
    step is milliseconds long, too short for nvidia-smi's 100 ms loop."""

    def __init__(self, rows):
        import pynvml as nv

        self.nv, self.rows, self.stop = nv, rows, threading.Event()
        nv.nvmlInit()
        self.h = None
        try:
            import torch

            pr = torch.cuda.get_device_properties(torch_device_index())
            bus = f"{pr.pci_domain_id:08x}:{pr.pci_bus_id:02x}:{pr.pci_device_id:02x}.0"
            self.h = nv.nvmlDeviceGetHandleByPciBusId(bus)
        except Exception:
            self.h = nv.nvmlDeviceGetHandleByIndex(torch_device_index())
        self.mx = nv.nvmlDeviceGetMaxClockInfo(self.h, nv.NVML_CLOCK_SM)
        self.sample()  # first row before the timed region starts
        self.th = threading.Thread(target=self.loop, daemon=True)
        self.th.start()

    def sample(self):
        nv = self.nv
        sm = nv.nvmlDeviceGetClockInfo(self.h, nv.NVML_CLOCK_SM)
        r = nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
        bits = [nv.nvmlClocksEventReasonHwSlowdown, nv.nvmlClocksEventReasonHwThermalSlowdown,
                nv.nvmlClocksEventReasonSwThermalSlowdown, nv.nvmlClocksEventReasonSwPowerCap]
        act = ["Active" if r & b else "Not Active" for b in bits]
        self.rows.append(", ".join([str(sm), str(self.mx), "0"] + act))

    def loop(self):
        while not self.stop.wait(0.002):
            try:
                self.sample()
            except Exception:
                return

    def terminate(self):
        self.stop.set()
        self.th.join(timeout=1)
        try:
            self.sample()  # last row after the timed region
        except Exception:
            pass


def clocks_sampler():
    """Clocks/throttle sampling during the timed region: NVML polling when
    pynvml loads, else nvidia-smi's loop (rows: sm, max sm, power, reasons)."""
    rows = []
    try:
        return _NvmlSampler(rows), rows
    except Exception:
        rows.clear()
    q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")
    try:
        p = subprocess.Popen(["nvidia-smi", "-i", str(torch_device_index()), f"--query-gpu={q}",
                              "--format=csv,noheader,nounits", "-lms", "100"],
                             stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
    except Exception:
        return None, None

    def reader():
        for line in p.stdout:
            rows.append(line.strip())

    threading.Thread(target=reader, daemon=True).start()
    return p, rows


def torch_device_index():
    import torch

    return torch.cuda.current_device()


def summarize_clocks(rows):
    sm, mx, reasons = [], None, set()
    names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
    for r in rows or []:
        f = [x.strip() for x in r.split(",")]
        if len(f) < 7:
            continue
        try:
            sm.append(float(f[0]))
            mx = float(f[1])
        except ValueError:
            continue
        for nm, v in zip(names, f[3:7]):
            if v.lower() == "active":
                reasons.add(nm)
    load = [v for v in sm if mx and v > 0.5 * mx] or sm
    return {"sm_mhz": statistics.median(load) if load else None, "sm_max_mhz": mx,
            "reasons": sorted(reasons), "samples": len(sm)}


def peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


# ------------------------------------------------------- reference CPU arm
def reference_layer_sample(g, h0, beta=1.0, threads=0):
    """One AGNN layer on the full graph through the reference's public API.
    Returns (ms per layer, kind, cores, sample description)."""
    from oracle.oracle import Csr

    c = Csr.of(g.num_nodes, g.node_pointer, g.edge_list)
    cores = threads or os.cpu_count()
    try:
        from oracle.oracle import RefLib

        R = RefLib()
        th = R.transform_handle(c, 16, 8, threads)
        th16 = R.reblock_handle(th, 16)
        hc = R.csr(c)
        kind = "reference"

        def layer():
            z, _ = R.l2_normalize_rows(h0)
            logits = R.sddmm(th16, c.num_edges, z, z, 1.0, False, threads,
                             values=np.ones(c.num_edges, np.float32))
            logits *= np.float32(beta)
            out = np.zeros(c.num_edges, np.float32)
            R._ok(R.L.ref_edge_softmax(hc.ptr, C.c_void_p(logits.ctypes.data),
                                       C.c_uint64(c.num_edges), C.c_void_p(out.ctypes.data)))
            return R.spmm(th, c.num_nodes, h0, 1.0, False, threads, values=out)
    except FileNotFoundError:
        from oracle.oracle import Oracle

        O = Oracle()
        kind = "port"

        def layer():
            z, _ = O.l2_normalize_rows(h0)
            logits = O.sddmm(c, z, z, values=np.ones(c.num_edges, np.float32)) * np.float32(beta)
            return O.spmm(c, h0, values=O.edge_softmax(c, logits))
    return layer, kind, cores


def reference_gcn_sample(g, x, dims, threads=0):
    """The GCN layers through the reference's public API (gcn_normalize_values,
    then gcn_forward on its transform); returns (run, kind, cores)."""
    from oracle.oracle import Csr

    c = Csr.of(g.num_nodes, g.node_pointer, g.edge_list)
    cores = threads or os.cpu_count()
    rng = np.random.default_rng(5)
    layers = [((rng.standard_normal((a, b)) / np.sqrt(a)).astype(np.float32), i + 1 < len(dims) - 1)
              for i, (a, b) in enumerate(zip(dims[:-1], dims[1:]))]
    try:
        from oracle.oracle import RefLib

        R = RefLib()
        th = R.transform_handle(R.gcn_normalize_values(c), 16, 8, threads)
        return (lambda: R.gcn_forward(th, g.num_nodes, x, layers, threads=threads)), "reference", cores
    except FileNotFoundError:
        from oracle.oracle import Oracle

        O = Oracle()
        cn = O.gcn_normalize_values(c)
        return (lambda: O.gcn_forward(cn, x, layers)), "port", cores


def run_reference_arm(args, wl):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    import paper_2412_12218_b200 as sg

    g, gen = make_graph(wl, args.locality)
    if wl["kind"] == "agnn":
        h0 = sg.dense_random(g.num_nodes, wl["hidden"], 17, -1.0, 1.0)
        layer, kind, cores = reference_layer_sample(g, h0)
        per, what = 1, f"one full-size AGNN layer (d={wl['hidden']})"
    else:  # GCN: the whole gcn_forward per step, reported per layer
        L = wl["layers"]
        dims = [wl["d_in"]] + [wl["hidden"]] * (L - 1) + [wl["d_out"]]
        x0 = sg.dense_random(g.num_nodes, dims[0], 17, -1.0, 1.0)
        layer, kind, cores = reference_gcn_sample(g, x0, dims)
        per, what = L, f"gcn_forward ({L} layers, {dims}) / {L}"
    steps = max(1, min(args.steps, 5))
    for _ in range(min(args.warmup, 1)):
        layer()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        layer()
        times.append((time.perf_counter() - t0) * 1e3 / per)
    ms = statistics.median(times)
    line = {
        "impl": "reference", "metric": metric_name(wl), "value": round(ms, 3), "unit": "ms",
        "n_gpus": args.gpus, "steps": steps, "warmup": min(args.warmup, 1),
        "ms_per_step": round(ms * per, 3), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": config_of(args, wl, g, gen),
        "cpu_baseline": {"value": round(ms, 3), "unit": "ms", "cores": cores, "kind": kind,
                         "sample": f"{what} per step, median "
                                   f"of {steps}; reference threads = all {cores} host cores"},
        "e2e": {"value": round(ms, 3), "unit": "ms", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    if args.csv:
        blocks = cap = dens = ""
        try:  # the reference's own transform statistics (block_stats, sgt_transform.cpp:93-100)
            from oracle.oracle import Csr, RefLib

            R = RefLib()
            t = R.transform_fields(R.transform_handle(Csr.of(g.num_nodes, g.node_pointer, g.edge_list), 16, 8))
            blocks = int(t.block_counter)
            cap = blocks * 16 * 8
            dens = g.num_edges / cap if cap else 0.0
        except Exception:
            pass
        write_report_csv(args.csv, [dict(dataset=args.workload, kernel=wl["kind"], path="reference-cpu",
                                         median_ms=round(ms, 4), blocks=blocks, capacity=cap,
                                         nnz=g.num_edges, density=dens)])


CSV_HEADER = "dataset,kernel,path,median_ms,blocks,capacity,nnz,density,max_rel_err"


def write_report_csv(path, rows):
    """The reference bench's report schema (bench.hpp:53-55, bench.cpp:216-227):
    dataset,kernel,path,median_ms,blocks,capacity,nnz,density,max_rel_err, so
    the CPU and GPU rows of a run sit side by side.  Appends (header once)."""
    new = not os.path.exists(path) or os.path.getsize(path) == 0
    with open(path, "a", newline="") as f:
        w = csv.writer(f, lineterminator="\n")
        if new:
            f.write(CSV_HEADER + "\n")
        for r in rows:
            w.writerow([r.get(k, "") for k in CSV_HEADER.split(",")])


def metric_name(wl):
    k = "AGNN" if wl["kind"] == "agnn" else "GCN"
    return f"{k} layer-forward ms per graph"


def config_of(args, wl, g, gen, extra=None):
    c = {"workload": f"{args.workload} ({wl['cfg']}): {wl['kind'].upper()} on synthetic "
                     f"{args.workload.split('-')[0]}-shaped graph",
         "nodes": g.num_nodes, "edges": g.num_edges,
         "model": f"{wl['d_in']}->{wl['hidden']}->{wl['d_out']}, {wl['layers']} layers",
         "global_batch": 1, "seq_len": 0, "parallelism": f"rowwindow{args.gpus}",
         "precision": args.precision, "mode": args.mode, "locality": args.locality,
         "generator": gen, "l2": "flushed between timed steps (256 MB write)"}
    if extra:
        c.update(extra)
    return c


# ------------------------------------------------------------- B200 arm
def run_b200(args, wl):
    import torch
    import torch.distributed as dist

    import paper_2412_12218_b200 as sg
    from paper_2412_12218_b200 import device as D
    from paper_2412_12218_b200._lib import check, lib

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    dev = torch.device("cuda", local)
    prec = args.precision
    mode = {"panel": 2, "fused": 1, "chain": 0, "auto": -1}[args.mode]

    t0 = time.perf_counter()
    g, gen = make_graph(wl, args.locality)
    N = g.num_nodes
    if mode < 0:  # the library's AGNN auto mode (forward.cu): panels from 2M edges, else fused
        mode = 2 if (wl["kind"] == "gcn" or g.num_edges >= (2 << 20) or wl["hidden"] > 64) else 1
        args.mode = {2: "panel", 1: "fused"}[mode] + " (auto)"
    log(f"[bench] graph {N} nodes {g.num_edges} edges in {time.perf_counter() - t0:.1f}s")
    # row partition in whole 128-row panels (balanced by edges)
    Q = 128
    bounds = np.zeros(world + 1, np.uint64)
    check(lib().sgtk_partition_windows(g.node_pointer.ctypes.data, N, Q, world, bounds.ctypes.data))
    r0, r1 = min(N, int(bounds[rank]) * Q), min(N, int(bounds[rank + 1]) * Q)
    e0, e1 = int(g.node_pointer[r0]), int(g.node_pointer[r1])
    np_loc = (g.node_pointer[r0:r1 + 1] - np.uint64(e0)).astype(np.uint64)
    el_loc = g.edge_list[e0:e1]
    vals_loc = None
    if wl["kind"] == "gcn":
        vals_loc = sg.gcn_normalize_values(g).values[e0:e1]

    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if world == 1:
        dg = D.DeviceGraph.from_csr(np_loc, el_loc, vals_loc, r1 - r0)
    else:
        dg = D.DeviceGraph.from_csr(np_loc, el_loc, vals_loc, r1 - r0, num_cols=N, row_offset=r0)
    torch.cuda.synchronize()
    translate_ms = (time.perf_counter() - t0) * 1e3
    info = dg.info
    bs = dg.block_stats()
    log(f"[bench] rank {rank}: rows [{r0},{r1}) translate {translate_ms:.1f} ms, tiles8 {info.tiles8} "
        f"tiles16 {info.tiles16} units {info.work_units8} density16x8 {bs[3]:.4f}")

    x_host = sg.dense_random(N, wl["d_in"], 8)
    w_in = torch.from_numpy(sg.dense_random(wl["d_in"], wl["hidden"], 1, -0.1, 0.1)).to(dev)
    w_out = torch.from_numpy(sg.dense_random(wl["hidden"], wl["d_out"], 2, -0.1, 0.1)).to(dev)
    # features resident with a 16-byte-multiple row pitch (TMA-eligible rows)
    ldx = (wl["d_in"] + 3) // 4 * 4
    x = torch.zeros((N, ldx), dtype=torch.float32, device=dev)[:, :wl["d_in"]]
    x.copy_(torch.from_numpy(x_host))
    L = wl["layers"]
    d = wl["hidden"]
    betas = np.ones(L, np.float32)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()

    # ---------------- step definitions --------------------------------------
    def allgather_rows(local_rows: torch.Tensor) -> torch.Tensor:
        if world == 1:
            return local_rows
        maxr = int(max(min(N, int(bounds[p + 1]) * Q) - min(N, int(bounds[p]) * Q)
                       for p in range(world)))
        pad = torch.zeros((maxr, local_rows.shape[1]), dtype=local_rows.dtype, device=dev)
        pad[:local_rows.shape[0]] = local_rows
        full = torch.empty((world * maxr, local_rows.shape[1]), dtype=local_rows.dtype, device=dev)
        dist.all_gather_into_tensor(full, pad)
        parts = [full[p * maxr: p * maxr + (min(N, int(bounds[p + 1]) * Q) -
                                            min(N, int(bounds[p]) * Q))] for p in range(world)]
        return torch.cat(parts)

    if wl["kind"] == "agnn":
        h0_loc = D.gemm(x[r0:r1], w_in, relu=True, precision=prec)
        h0 = allgather_rows(h0_loc) if world > 1 else h0_loc

        def agnn_stack(h):
            if world == 1:
                return dg.agnn_forward(h, betas, precision=prec, mode=mode)
            cur = h
            for l in range(L):
                loc = dg.agnn_forward(cur, betas[l:l + 1], precision=prec, mode=mode)
                cur = allgather_rows(loc) if l + 1 < L else loc
            return cur

        def step():
            return agnn_stack(h0)

        def model_forward():
            hh = allgather_rows(D.gemm(x[r0:r1], w_in, relu=True, precision=prec))
            return D.gemm(agnn_stack(hh), w_out, relu=False, precision=prec)

        if mode == 2:
            pi = dg.panel_info(d)
            # input kernel, then per layer: dense + rows + final (+ hub rows)
            launches_per_step = 1 + L * (3 + (1 if pi["long_rows"] else 0))
        else:
            launches_per_step = L * (2 if mode == 1 else 4) + (
                L if (mode == 1 and dg_has_splits(dg, 16)) or (mode == 0 and dg_has_splits(dg, 8)) else 0)
        layers_per_step = L
    else:
        layers = [(torch.from_numpy(w).to(dev), r) for w, r in
                  sg.random_gcn_layers(wl["d_in"], wl["hidden"], wl["d_out"], L, 1)]
        xs = torch.from_numpy(sg.dense_random(N, wl["d_in"], 8)).to(dev) if wl["d_in"] != x.shape[1] else x

        def step():
            if world == 1:
                return dg.gcn_forward(xs, layers, precision=prec, order=2)
            h = xs
            for l, (w, r) in enumerate(layers):
                hw = D.gemm(h[r0:r1] if h.shape[0] == N else h, w, relu=False, precision=prec)
                full = allgather_rows(hw)
                loc = dg.spmm(full, precision=prec)
                if r:
                    loc = torch.relu_(loc)
                h = allgather_rows(loc) if l + 1 < L else loc
            return h

        model_forward = step
        launches_per_step = L * 3 + (L if dg_has_splits(dg, 8) else 0)
        layers_per_step = L

    # ---------------- timing --------------------------------------------------
    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        ts = []
        for _ in range(steps):
            flush.fill_(1)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        torch.cuda.synchronize()
        ms = float(np.mean(ts))
        if world > 1:
            t = torch.tensor([ms], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ms = float(t.item())
        return ms, ts

    warm = max(3, args.warmup)
    sampler, rows = clocks_sampler()
    step_ms, step_ts = timed(step, args.steps, warm)
    if sampler:
        sampler.terminate()
    clocks = summarize_clocks(rows)
    value = step_ms / layers_per_step
    model_ms, _ = timed(model_forward, max(2, args.steps // 2), 2)

    # ---------------- dominant-kernel roofline (CUDA events on our stream) ----
    roof = None
    kern = {}
    extra = {}
    if world == 1:
        kern, roof = kernel_breakdown(args, wl, dg, g, h0 if wl["kind"] == "agnn" else xs, D, prec,
                                      mode, flush, stream, layers if wl["kind"] == "gcn" else None,
                                      extra, (x, w_in) if wl["kind"] == "agnn" else None)

    # ---------------- e2e through the host-buffer C ABI ----------------------
    e2e = None
    if world == 1:
        e2e = e2e_host(wl, dg, h0 if wl["kind"] == "agnn" else xs, prec, mode, L, layers_per_step,
                       layers if wl["kind"] == "gcn" else None, flush, args)

    # ---------------- CPU baseline (rank 0, N=1) ------------------------------
    cpu = None
    if rank == 0 and world == 1 and wl["kind"] == "agnn" and not args.no_cpu:
        h0_host = h0.cpu().numpy()
        layer, kind, cores = reference_layer_sample(g, h0_host)
        t0 = time.perf_counter()
        layer()
        cpu_ms = (time.perf_counter() - t0) * 1e3
        cpu = {"value": round(cpu_ms, 1), "unit": "ms", "cores": cores, "kind": kind,
               "sample": f"one full-size AGNN layer (d={d}, {g.num_edges} edges) through the "
                         "reference's public functions, single run, all host cores"}
    elif rank == 0 and world == 1 and not args.no_cpu:  # GCN: gcn_forward / layers
        dims = [wl["d_in"]] + [wl["hidden"]] * (L - 1) + [wl["d_out"]]
        run, kind, cores = reference_gcn_sample(g, xs.cpu().numpy(), dims)
        t0 = time.perf_counter()
        run()
        cpu_ms = (time.perf_counter() - t0) * 1e3 / L
        cpu = {"value": round(cpu_ms, 1), "unit": "ms", "cores": cores, "kind": kind,
               "sample": f"one full-size gcn_forward ({L} layers, dims {dims}, {g.num_edges} "
                         "edges) through the reference's public API, per layer, single run, "
                         "all host cores"}

    pk, pk_src = peaks()
    if roof:
        roof["traffic"] = profiled_traffic(roof["kernel"], gcn=wl["kind"] == "gcn")
        roof["peak"] = pk["hbm_gbs"]
        roof["frac"] = round(roof["achieved"] / pk["hbm_gbs"], 4)
        roof["peak_source"] = f"MEASURED_PEAKS.json hbm_gbs ({pk_src})"

    if rank == 0:
        line = {
            "metric": metric_name(wl), "value": round(value, 4), "unit": "ms",
            "n_gpus": world, "steps": args.steps, "warmup": warm,
            "ms_per_step": round(step_ms, 4), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None,
            "dtype": "f32 (split-TF32 on tensor cores)" if prec == "fp32" else "tf32",
            "data": "synthetic (deterministic generator; random-init weights)",
            "config": config_of(args, wl, g, gen, {
                "step": f"agnn_forward({L} layers) on the whole graph; value = step/{L}"
                if wl["kind"] == "agnn" else f"gcn_forward({L} layers); value = step/{L}",
                "tiles16x8": int(bs[0]), "tile_density16x8": round(bs[3], 4),
                "translate_ms": round(translate_ms, 2),
                "panel_format": dg.panel_info(wl["hidden"]) if mode == 2 else None}),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": launches_per_step * args.steps,
            "model_forward_ms": round(model_ms, 4), "kernels_ms": kern,
        }
        if "roofline_unfused_formula" in extra and roof:
            u = extra["roofline_unfused_formula"]
            u["achieved"] = round(u["algorithmic_bytes"] / (roof["kernel_ms"] * 1e-3) / 1e9, 1)
            u["unit"] = "GB/s"
            u["frac"] = round(u["achieved"] / pk["hbm_gbs"], 4)
            line["roofline_unfused_formula"] = u
        if "roofline_l2_gather" in extra:
            line["roofline_l2_gather"] = extra["roofline_l2_gather"]
        if "roofline_gemm" in extra:
            rg = extra["roofline_gemm"]
            rg["peak"] = pk["hbm_gbs"]
            rg["frac"] = round(rg["achieved"] / pk["hbm_gbs"], 4)
            line["roofline_gemm"] = rg
        print(json.dumps(line), flush=True)
        if args.csv:  # per layer, like the reference arm's row
            write_report_csv(args.csv, [dict(dataset=args.workload, kernel=wl["kind"],
                                             path=f"b200-{args.mode.split()[0]}",
                                             median_ms=round(statistics.median(step_ts) / layers_per_step, 4),
                                             blocks=bs[0], capacity=bs[1], nnz=bs[2],
                                             density=round(bs[3], 6))])
    if world > 1:
        dist.destroy_process_group()


def profiled_traffic(kernel_field, gcn=False):
    """DRAM bytes (read + write) per launch of the roofline kernel(s), from the
    committed ncu launch list of this code (profiles/*_launches.csv, written by
    tools/profile_round.sh + tools/ncu_summary.py); None if not profiled."""
    import glob

    names = [k.strip() for k in kernel_field.split("(")[-1].rstrip(")").split("+")] \
        if "(" in kernel_field else [kernel_field]
    # newest round last: tags r1_, r1b, ..., r1h sort by name (mtimes do not
    # survive the copy to the GPU box)
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_launches.csv")))
    # the GCN workload's launch list is *_gcn_launches.csv (tools/profile_round.sh)
    files = [f for f in files if f.endswith("_gcn_launches.csv") == gcn]
    for path in reversed(files):
        try:
            with open(path, newline="") as f:
                rows = list(csv.reader(f))[1:]
        except OSError:
            continue
        if not rows or len(rows[0]) < 6:
            continue
        tot, found = 0.0, 0
        for nm in names:
            hit = [r for r in rows if nm.strip() in r[0]]
            if hit:
                tot += float(hit[0][5])
                found += 1
        if found == len(names):
            return {"bytes": int(tot), "source": os.path.relpath(path, ROOT)}
    return None


def dg_has_splits(dg, tile_w):
    # work units > windows means some window is split (extra reduce launch)
    return dg.info.work_units8 > dg.info.num_windows if tile_w == 8 else False


def kernel_breakdown(args, wl, dg, g, h, D, prec, mode, flush, stream, gcn_layers, extra,
                     proj=None):
    """Per-kernel CUDA-event times for one layer and the dominant kernel's roofline."""
    import torch

    from paper_2412_12218_b200._lib import check, lib

    N, E = g.num_nodes, g.num_edges
    d = h.shape[1]
    reps = max(3, args.steps)
    res = {}

    def ev_time(fn):
        for _ in range(2):
            fn()
        ts = []
        for _ in range(reps):
            flush.fill_(1)
            a = torch.cuda.Event(enable_timing=True)
            b = torch.cuda.Event(enable_timing=True)
            a.record(stream)
            fn()
            b.record(stream)
            b.synchronize()
            ts.append(a.elapsed_time(b))
        return float(np.mean(ts))

    s = stream.cuda_stream
    if wl["kind"] == "agnn":
        inv = torch.empty(N, dtype=torch.float32, device=h.device)
        zeros = torch.zeros(1, dtype=torch.int64, device=h.device)
        out = torch.empty_like(h)
        logits = torch.empty(E, dtype=torch.float32, device=h.device)
        pr = 0 if prec == "fp32" else 1
        L = lib()

        def l2():
            check(L.sgtk_l2_normalize_rows(h.data_ptr(), N, d, d, None, 0, inv.data_ptr(),
                                           zeros.data_ptr(), s))

        def fused_one():
            check(L.sgtk_agnn_forward(dg.handle, h.data_ptr(), d, d, 1,
                                      np.ones(1, np.float32).ctypes.data, None, pr, 1, ws.data_ptr(),
                                      ws.numel(), out.data_ptr(), d, None, s))

        ws = torch.empty(L.sgtk_agnn_workspace(dg.handle, d), dtype=torch.uint8, device=h.device)
        l2()
        res["l2norm"] = ev_time(l2)
        sddmm = lambda: dg.sddmm(h, h, scale=1.0, precision=prec, out=logits)  # noqa: E731
        res["sddmm"] = ev_time(sddmm)
        res["edge_softmax"] = ev_time(lambda: dg.edge_softmax(logits, out=logits))
        res["spmm"] = ev_time(lambda: dg.spmm(h, edge_values=logits, precision=prec, out=out))
        res["agnn_layer_fused(l2norm+fused)"] = ev_time(fused_one)
        res["agnn_fused_kernel"] = res["agnn_layer_fused(l2norm+fused)"] - res["l2norm"]
        if proj is not None:
            px, pw = proj
            res["in_proj_gemm"] = ev_time(lambda: D.gemm(px, pw, relu=True, precision=prec))
            K, M = px.shape[1], pw.shape[1]
            Bg = 4 * N * K + 4 * K * M + 4 * N * M
            extra["roofline_gemm"] = {
                "bound": "hbm", "kernel": "gemm_tc05 (in-proj %dx%d)" % (K, M),
                "achieved": round(Bg / (res["in_proj_gemm"] * 1e-3) / 1e9, 1), "unit": "GB/s",
                "algorithmic_bytes": int(Bg), "formula": "s*N*K + 4*K*M + 4*N*M (SURVEY §8d B_gemm)",
                "tflops": round(2 * N * K * M / (res["in_proj_gemm"] * 1e-3) / 1e12, 2),
                "kernel_ms": round(res["in_proj_gemm"], 4)}
        if mode == 2:
            def panel_one():
                check(L.sgtk_agnn_forward(dg.handle, h.data_ptr(), d, d, 1,
                                          np.ones(1, np.float32).ctypes.data, None, pr, 2,
                                          ws.data_ptr(), ws.numel(), out.data_ptr(), d, None, s))
            res["agnn_layer_panel(input+dense+rows+final)"] = ev_time(panel_one)
            check(L.sgtk_debug_set(1))  # tensor-core part only
            res["panel_dense_part"] = ev_time(panel_one)
            check(L.sgtk_debug_set(2))  # CUDA-core part only
            res["panel_sparse_part"] = ev_time(panel_one)
            check(L.sgtk_debug_set(0))
            # one layer inside the 4-layer stack (its input normalisation is fused into
            # the previous layer's final kernel; the l2norm pass stands in for the input kernel)
            res["agnn_panel_layer"] = res["agnn_layer_panel(input+dense+rows+final)"] - res["l2norm"]
        s_ = 4
        B_fused = 8 * (N + 1) + 4 * E + 4 * N + 2 * s_ * N * d
        B_spmm = 8 * (N + 1) + 4 * E + 4 * E + s_ * N * d + 4 * N * d
        if mode == 2:
            name, B, t = "agnn_panel_layer (agnn_dense_kernel + agnn_rows_kernel + agnn_final_kernel)", B_fused, \
                res["agnn_panel_layer"]
            formula = "8(N+1) + 4E + 4N + 2*s*N*d (SURVEY §8d fused AGNN lower bound, s=4)"
            extra["roofline_unfused_formula"] = {
                "formula": "B_rownorm + B_sddmm + B_softmax + B_spmm (SURVEY §8d: report fusion "
                           "against the unfused bytes)",
                "algorithmic_bytes": int(8 * N * d + (8 * (N + 1) + 8 * E + 4 * N * d) +
                                         (8 * (N + 1) + 8 * E) + B_spmm),
            }
        elif mode == 1:
            name, B, t = "agnn_fused_kernel", B_fused, res["agnn_fused_kernel"]
            formula = "8(N+1) + 4E + 4N + 2*s*N*d (SURVEY §8d fused AGNN lower bound, s=4)"
        else:
            name, B, t = "spmm", B_spmm, res["spmm"]
            formula = "8(N+1) + 4E + 4E + s*N*d + 4*N*d (SURVEY §8d B_spmm, s=4)"
    else:
        x = h
        name = "spmm"
        dd = gcn_layers[0][0].shape[1]
        hw = torch.empty((N, dd), dtype=torch.float32, device=h.device)
        outb = torch.empty_like(hw)
        res["gemm"] = ev_time(lambda: D.gemm(x, gcn_layers[0][0], precision=prec))
        hw.copy_(D.gemm(x, gcn_layers[0][0], precision=prec))
        res["spmm"] = ev_time(lambda: dg.spmm(hw, precision=prec, out=outb))
        t = res["spmm"]
        name = "spmm (spmm_panel_kernel + sparse_rows_kernel)"
        B = 8 * (N + 1) + 4 * E + 4 * E + 4 * N * dd + 4 * N * dd
        formula = "8(N+1) + 4E + 4E*[w] + s*N*d + 4*N*d (SURVEY §8d B_spmm, s=4, w=1)"
    res = {k: round(v, 4) for k, v in res.items()}
    achieved = B / (t * 1e-3) / 1e9
    roof = {"bound": "hbm", "kernel": name, "achieved": round(achieved, 1), "unit": "GB/s",
            "algorithmic_bytes": int(B), "formula": formula, "kernel_ms": round(t, 4),
            "traffic": None}
    if mode == 2:
        extra["roofline_l2_gather"] = l2_gather_roofline(dg, wl, t, prec)
    return res, roof


def l2_gather_roofline(dg, wl, t_ms, prec):
    """The panel kernels fetch feature rows at random from an L2-resident
    table: bytes moved L2 -> SM per layer (tensor-core chunk tiles, CUDA-core
    rows, streamed entries / masks) against the measured random-row gather
    rate (tools/gather_peak.cu, profiles/gather_peak.json)."""
    pi = dg.panel_info(wl["hidden"])
    rb = 4 * (32 if wl["hidden"] <= 32 else 64)  # bytes per gathered row (operand stride)
    planes = 2 if prec == "fp32" else 1           # FP32: hi/lo planes
    if wl["kind"] == "agnn":  # z and h tiles + row masks per chunk; rows on the CUDA cores
        b = pi["dense_chunks"] * (32 * 2 * rb * planes + 128 * 4) + pi["sparse_edges"] * rb
        what = "chunks x (32 z + 32 h rows + 128 masks) + sparse edges x row"
    else:                     # B tile per chunk + packed entries; rows on the CUDA cores
        b = pi["dense_chunks"] * 32 * rb + pi["dense_entries"] * 4 * planes + \
            pi["sparse_edges"] * (rb + 8)
        what = "chunks x 32 rows + entries + sparse edges x (row + entry)"
    try:
        with open(os.path.join(ROOT, "profiles", "gather_peak.json")) as f:
            gp = json.load(f)["gather_gbs"]
        peak = gp["row128_table30MB"] if rb == 128 else gp["row256_table34MB"]
    except Exception:
        peak = None
    ach = b / (t_ms * 1e-3) / 1e9
    return {"bound": "l2-gather", "bytes": int(b), "formula": what, "achieved": round(ach, 1),
            "unit": "GB/s", "peak": peak, "frac": round(ach / peak, 4) if peak else None,
            "peak_source": "profiles/gather_peak.json (tools/gather_peak.cu, random rows, "
                           "L2-resident table)"}


def e2e_host(wl, dg, h, prec, mode, L, layers_per_step, gcn_layers, flush, args):
    """Same step through the host-buffer C ABI (pinned H2D + D2H inside the timing)."""
    import torch

    from paper_2412_12218_b200._lib import check, lib

    N = dg.info.num_nodes
    pr = 0 if prec == "fp32" else 1
    Lb = lib()
    if wl["kind"] == "agnn":
        d = h.shape[1]
        x_pin = h.cpu().pin_memory()
        out_pin = torch.empty((N, d), dtype=torch.float32).pin_memory()
        betas = np.ones(L, np.float32)

        def call():
            check(Lb.sgtk_agnn_forward_host(dg.handle, x_pin.data_ptr(), d, L, betas.ctypes.data,
                                            C.c_double(1.0), pr, mode, out_pin.data_ptr(), None,
                                            None))
        h2d, d2h = N * d * 4, N * d * 4
    else:
        dims = np.array([h.shape[1]] + [w.shape[1] for w, _ in gcn_layers], np.uint64)
        relu = np.array([int(r) for _, r in gcn_layers], np.int32)
        wcat = np.concatenate([w.cpu().numpy().ravel() for w, _ in gcn_layers])
        x_pin = h.cpu().pin_memory()
        out_pin = torch.empty((N, int(dims[-1])), dtype=torch.float32).pin_memory()

        def call():
            check(Lb.sgtk_gcn_forward_host(dg.handle, x_pin.data_ptr(), len(gcn_layers),
                                           dims.ctypes.data, wcat.ctypes.data, relu.ctypes.data,
                                           C.c_double(1.0), pr, out_pin.data_ptr(), None))
        h2d, d2h = N * int(dims[0]) * 4 + wcat.nbytes, N * int(dims[-1]) * 4
    for _ in range(2):
        call()
    ts = []
    for _ in range(max(3, args.steps)):
        flush.fill_(1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        call()  # synchronises internally (D2H of the result)
        ts.append((time.perf_counter() - t0) * 1e3)
    return {"value": round(float(np.mean(ts)) / layers_per_step, 4), "unit": "ms",
            "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
            "path": "sgtk_agnn_forward_host" if wl["kind"] == "agnn" else "sgtk_gcn_forward_host"}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--workload", default="reddit-agnn", choices=sorted(WORKLOADS))
    ap.add_argument("--precision", default="tf32", choices=["fp32", "tf32"])
    ap.add_argument("--mode", default="auto", choices=["auto", "panel", "fused", "chain"])
    ap.add_argument("--locality", default="calibrated", choices=sorted(LOCALITY))
    ap.add_argument("--no-cpu", action="store_true", help="skip the CPU baseline leg")
    ap.add_argument("--csv", default="", help="also append a row in the reference bench's CSV "
                                               "schema (bench.hpp:53-55) to this file")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference_arm(args, wl)
    else:
        run_b200(args, wl)


if __name__ == "__main__":
    main()
