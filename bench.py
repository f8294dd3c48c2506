#!/usr/bin/env python3
"""Benchmark: FTC-GNN aggregation hot path on B200 (metric of BASELINE.json).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
                    [--workload reddit-agnn|proteins-gcn|pubmed-agnn|cora-gcn|powerlaw-gcn]
                    [--precision fp32|tf32] [--mode auto|panel|fused|chain]
                    [--locality calibrated|uniform] [--csv FILE] [--no-cpu] [--no-verify]

Default workload (config C4 of BASELINE.json): AGNN forward on a synthetic
Reddit-shaped graph (232,965 nodes, ~114.6M edges incl. self-loops), 4 AGNN
layers at d=32, beta=1.  The metric is the AGNN *layer-forward* time per
graph: one step = the reference API call agnn_forward(t, h0, 4 layers) on the
whole graph, value = step ms / 4.  h0 = DenseMatrix::random(N, 32, seed+7)
exactly as the reference's own bench builds its AGNN input
(/root/reference/proj/src/bench.cpp:128,134-135).  Inputs are resident in HBM;
L2 is flushed (256 MB write) between timed steps; per-step CUDA events on the
launch stream, max over ranks.

N GPUs: `--gpus N` without torchrun re-launches itself under
torch.distributed.run (one process per GPU).  Rows are partitioned by whole
128-row panels (distributed.RowSlice); each layer ends with one in-place NCCL
all-gather of the padded embedding replica.  When more ranks than devices are
visible (a 1-GPU lease exercising the N>1 path) ranks share the devices and
exchange over gloo.

`--impl reference` times the reference's own CPU implementation
(oracle/_ref/libsgtk_ref.so, compiled unmodified from /root/reference; the
generator of the synthetic graph is linked into that library too, so this arm
never loads the product library) on this host's cores, same workload, same
precision, same inputs: one step = one full-size layer through the reference's
public functions (l2_normalize_rows, sddmm_hybrid on reblock(t,16),
edge_softmax, spmm_hybrid; gnn.cpp:107-116), or gcn_forward / L for GCN.
"""

from __future__ import annotations

import argparse
import csv
import ctypes as C
import json
import os
import socket
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

INPUT_SEED = 8   # DenseMatrix::random(n, dims, seed + 7) with the bench's seed 1 (bench.cpp:128)
LAYER_SEED = 1   # random_gcn_layers(..., seed) with the bench's seed 1 (bench.cpp:131-132)


def log(*a):
    print(*a, file=sys.stderr, flush=True)


# ------------------------------------------------------------------ inputs
def make_graph(wl, locality, seed=1, synth=None):
    """Synthetic symmetric graph of the workload's shape (deterministic).
    `synth(n, picks, alpha, p_local, band, seed)` -> graph with num_nodes /
    num_edges / node_pointer / edge_list; default: the product library's
    generator (the reference arm passes the copy linked into libsgtk_ref.so —
    same source, same output, tests/test_bench_cpu.py)."""
    if synth is None:
        import paper_2412_12218_b200 as sg

        synth = sg.synth_graph
    n, e = wl["n"], wl["e"]
    loc = LOCALITY[locality]
    picks = max((e - n) / (2.0 * n), 0.5)
    # duplicate picks (local ones collide) shrink E: calibrate on a 50k sample
    ns = min(n, 50_000)
    s = synth(ns, picks, wl["alpha"], loc["p_local"], loc["band"], seed)
    ratio = (s.num_edges - ns) / (2.0 * ns * picks)
    picks = picks / max(ratio, 0.3)
    g = synth(n, picks, wl["alpha"], loc["p_local"], loc["band"], seed)
    if abs(g.num_edges - e) > 0.05 * e:
        # heavy-tailed degrees collide more at full size than in the sample
        # (C5: 0.72B instead of 1B): one first-order correction at full size
        picks = picks * (e - n) / max(g.num_edges - n, 1)
        g = synth(n, picks, wl["alpha"], loc["p_local"], loc["band"], seed)
    return g, dict(avg_picks=round(picks, 3), **loc, alpha=wl["alpha"])


def host_info():
    """Host cores this process may use, CPU model, OMP_NUM_THREADS."""
    try:
        cores = len(os.sched_getaffinity(0))
    except AttributeError:
        cores = os.cpu_count()
    model = ""
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    model = line.split(":", 1)[1].strip()
                    break
    except OSError:
        pass
    return {"cores_available": cores, "cpu_model": model,
            "omp_num_threads": os.environ.get("OMP_NUM_THREADS", "unset (OpenMP default)")}


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
def sample_rows(n, k=96, seed=0):
    rng = np.random.default_rng(seed)
    return np.unique(np.concatenate([rng.integers(0, n, k), [0, n - 1]]))


def rows_agnn_f64(node_pointer, edge_list, x, rows, beta=1.0):
    """One AGNN layer (gnn.cpp:107-116) for the given rows, exactly in float64."""
    npz = node_pointer.astype(np.int64)
    h = x.astype(np.float64)
    ref = np.zeros((len(rows), x.shape[1]))
    for t, i in enumerate(rows):
        nb = edge_list[npz[i]:npz[i + 1]].astype(np.int64)
        if nb.size == 0:
            continue
        hn = h[nb]
        nn = np.linalg.norm(hn, axis=1)
        zn = np.where(nn[:, None] > 0, hn / np.where(nn > 0, nn, 1)[:, None], 0.0)
        nrm_i = np.linalg.norm(h[i])
        zi = h[i] / nrm_i if nrm_i > 0 else np.zeros_like(h[i])
        lg = beta * (zn @ zi)
        a = np.exp(lg - lg.max())
        ref[t] = (a / a.sum()) @ hn
    return ref


def rows_spmm_f64(node_pointer, edge_list, values, x, rows):
    """out = A x for the given rows, exactly in float64 (tile_exec.cpp:200-314)."""
    npz = node_pointer.astype(np.int64)
    xd = x.astype(np.float64)
    ref = np.zeros((len(rows), x.shape[1]))
    for t, i in enumerate(rows):
        nb = edge_list[npz[i]:npz[i + 1]].astype(np.int64)
        a = np.ones(nb.size) if values is None else values[npz[i]:npz[i + 1]].astype(np.float64)
        ref[t] = a @ xd[nb]
    return ref


def max_rel_err(got, ref):
    """dense_matrix.hpp:68-85: max|got - ref| / max|ref|."""
    den = float(np.abs(ref).max()) if ref.size else 0.0
    num = float(np.abs(np.asarray(got, np.float64) - ref).max()) if ref.size else 0.0
    return num / den if den > 0 else num


class RefWorkload:
    """The reference's own CPU implementation (oracle/_ref/libsgtk_ref.so, the
    unmodified reference sources) on the bench inputs, through its public
    functions.  AGNN: one layer as agnn_forward runs it (gnn.cpp:107-116), on
    reblock(t, 16) built once here (the reference's agnn_forward rebuilds it
    on every call, gnn.cpp:101 — hoisting it only favours the reference).
    GCN: gcn_normalize_values + gcn_forward (gnn.cpp:33-52) with the reference
    bench's own inputs (bench.cpp:114-132).

    Graphs above SAMPLE_EDGES (C5: 1B edges, ~40 s per operation on CPU) run a
    bounded sample: the first whole 16-row windows holding ~SAMPLE_ROWS_EDGES edges
    keep their edges (values from the full graph), every other row is empty,
    features stay full-size; `scale` = E / E_sample extrapolates to the graph."""

    SAMPLE_EDGES = 300_000_000  # C5 only; C1-C4 run at full size
    SAMPLE_ROWS_EDGES = 40_000_000

    def __init__(self, wl, g, tf32, R):
        from oracle.oracle import Csr

        self.R, self.wl, self.tf32 = R, wl, bool(tf32)
        self.n = g.num_nodes
        self.c = Csr.of(g.num_nodes, g.node_pointer, g.edge_list)
        self.threads = R.threads()
        self.scale, self.sample_note = 1.0, "the full graph"
        full = self.c
        if self.c.num_edges > self.SAMPLE_EDGES:
            rows = int(np.searchsorted(g.node_pointer, self.SAMPLE_ROWS_EDGES)) // 16 * 16
            es = int(g.node_pointer[rows])
            np_s = g.node_pointer.copy()
            np_s[rows:] = es
            self.c = Csr.of(self.n, np_s, g.edge_list[:es])
            self.scale = g.num_edges / es
            self.sample_note = (f"a bounded sample: rows [0, {rows}) ({es} of {g.num_edges} edges, "
                                f"other rows empty, full-size features and dense update); per "
                                f"layer = step / layers + {self.scale - 1:.2f} more sampled "
                                f"aggregations (spmm_hybrid on the sample, timed apart)")
        if wl["kind"] == "agnn":
            self.x = R.dense_random(self.n, wl["hidden"], INPUT_SEED)
            self.th = R.transform_handle(self.c, 16, 8)
            self.th16 = R.reblock_handle(self.th, 16)
            self.hc = R.csr(self.c)
            self.unit = np.ones(self.c.num_edges, np.float32)
            self.per = 1
        else:
            L = wl["layers"]
            gn = R.gcn_normalize_values(full)
            es = self.c.num_edges
            self.gn = Csr.of(self.n, self.c.node_pointer, self.c.edge_list, gn.values[:es])
            self.th = R.transform_handle(self.gn, 16, 8)
            self.x = R.dense_random(self.n, wl["d_in"], INPUT_SEED)
            self.layers = R.random_gcn_layers(wl["d_in"], wl["hidden"], wl["d_out"], L, LAYER_SEED)
            self.per = L

    def run(self, ratio=1.0):
        """One step; ratio 1 = the reference's default tile path, 0 = its scalar path."""
        R, tf = self.R, self.tf32
        if self.wl["kind"] == "agnn":
            z, _ = R.l2_normalize_rows(self.x)
            logits = R.sddmm(self.th16, self.c.num_edges, z, z, ratio, tf, 0, values=self.unit)
            logits *= np.float32(1.0)  # beta (bench.cpp:135)
            attn = np.zeros_like(logits)
            R._ok(R.L.ref_edge_softmax(self.hc.ptr, C.c_void_p(logits.ctypes.data),
                                       C.c_uint64(logits.shape[0]), C.c_void_p(attn.ctypes.data)))
            return R.spmm(self.th, self.n, self.x, ratio, tf, 0, values=attn)
        return R.gcn_forward(self.th, self.n, self.x, self.layers, ratio, tf)

    def per_layer(self, step_ms, ratio=1.0):
        """ms per layer of a step on the whole graph.  A sampled step does the
        full-size dense work (the reference's matmul runs over all N rows) but
        aggregates only the sampled edges: add (scale - 1) aggregations."""
        if self.scale == 1.0:
            return step_ms / self.per
        if not hasattr(self, "_agg"):
            self._agg = {}
        if ratio not in self._agg:
            x = self.x
            ts, _ = timed_cpu(lambda: self.R.spmm(self.th, self.n, x, ratio, self.tf32), 1, 2)
            self._agg[ratio] = statistics.median(ts)
        return step_ms / self.per + (self.scale - 1.0) * self._agg[ratio]

    def oracle_spmm_ms(self):
        """The reference's single-threaded oracle_spmm (oracle.cpp:7-20) on the
        layer's aggregation input (unit values for AGNN)."""
        g = self.c if self.wl["kind"] == "agnn" else self.gn
        t0 = time.perf_counter()
        self.R.oracle_spmm(g, self.x)
        return (time.perf_counter() - t0) * 1e3

    def check_rows(self, out):
        """Sampled-row max_rel_err of a step's output: AGNN layer / GCN first
        layer's aggregation vs float64 (GCN: checked on the SpMM, run apart)."""
        rows = sample_rows(self.n)
        if self.wl["kind"] == "agnn":
            ref = rows_agnn_f64(self.c.node_pointer, self.c.edge_list, self.x, rows)
            return max_rel_err(out[rows], ref)
        agg = self.R.spmm(self.th, self.n, self.x, 1.0, self.tf32)
        ref = rows_spmm_f64(self.gn.node_pointer, self.gn.edge_list, self.gn.values, self.x, rows)
        return max_rel_err(agg[rows], ref)


def ref_lib():
    from oracle.oracle import RefLib

    return RefLib()


def timed_cpu(fn, warmup, steps):
    for _ in range(warmup):
        fn()
    ts = []
    out = None
    for _ in range(steps):
        t0 = time.perf_counter()
        out = fn()
        ts.append((time.perf_counter() - t0) * 1e3)
    return ts, out


def cpu_baseline_leg(wl, g, prec, R):
    """The GPU arm's cpu_baseline (rank 0, N=1): the reference on this host's
    cores, warmed, median of 3 — tile path (ratio 1, the reference default),
    scalar path (ratio 0), and the single-threaded oracle_spmm."""
    W = RefWorkload(wl, g, prec == "tf32", R)
    tile, out = timed_cpu(W.run, 1, 3)
    scalar, _ = timed_cpu(lambda: W.run(0.0), 1, 3)
    orc = W.oracle_spmm_ms() * W.scale
    info = host_info()
    what = (f"one full-size AGNN layer (d={wl['hidden']}, {g.num_edges} edges)" if wl["kind"] == "agnn"
            else f"one full-size gcn_forward ({wl['layers']} layers) / {wl['layers']}")
    return {"value": round(W.per_layer(statistics.median(tile)), 2), "unit": "ms", "cores": W.threads,
            "kind": "reference", "precision": prec,
            "sample": f"{what} through the reference's public functions on {W.sample_note}, "
                      f"tile path (ratio 1, the reference default), 1 warm-up + median of 3, "
                      f"reference threads = resolve_thread_count(0) = {W.threads}",
            "scalar_path_ms": round(W.per_layer(statistics.median(scalar), 0.0), 2),
            "oracle_spmm_1thread_ms": round(orc, 2),
            "cpu_model": info["cpu_model"], "omp_num_threads": info["omp_num_threads"],
            "cores_available": info["cores_available"],
            "max_rel_err_sampled": W.check_rows(out)}


def run_reference_arm(args, wl):
    """`--impl reference`: the reference's CPU path alone (rank 0; other ranks
    of a torchrun launch exit without work).  Loads only oracle/_ref."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    R = ref_lib()
    g, gen = make_graph(wl, args.locality, synth=R.synth_graph)
    W = RefWorkload(wl, g, args.precision == "tf32", R)
    ts, out = timed_cpu(W.run, args.warmup, args.steps)
    per_layer = [W.per_layer(t) for t in ts]
    ms = float(np.mean(per_layer))
    info = host_info()
    err = W.check_rows(out)
    what = (f"one full-size AGNN layer (d={wl['hidden']}) per step" if wl["kind"] == "agnn"
            else f"one full-size gcn_forward ({wl['layers']} layers) per step, reported / {W.per}")
    line = {
        "impl": "reference", "metric": metric_name(wl), "value": round(ms, 3), "unit": "ms",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(ms * W.per, 3), "higher_is_better": False, "scaling": "strong",
        "vs_baseline": None, "dtype": dtype_name(args.precision), "data": DATA,
        "config": config_of(args, wl, g, gen),
        "cpu_baseline": {"value": round(ms, 3), "unit": "ms", "cores": W.threads,
                         "kind": "reference",
                         "sample": f"{what} on {W.sample_note}, tile path (ratio 1, the "
                                   f"reference default), mean of "
                                   f"{args.steps} after {args.warmup} warm-up; reference threads = "
                                   f"resolve_thread_count(0) = {W.threads}",
                         "median_ms": round(statistics.median(per_layer), 3),
                         "cpu_model": info["cpu_model"], "omp_num_threads": info["omp_num_threads"],
                         "cores_available": info["cores_available"]},
        "e2e": {"value": round(ms, 3), "unit": "ms", "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
        "max_rel_err_sampled": err,
    }
    print(json.dumps(line), flush=True)
    if args.csv:
        t = R.transform_fields(W.th)
        blocks = int(t.block_counter)
        cap = blocks * 16 * 8
        write_report_csv(args.csv, [dict(
            dataset=args.workload, kernel=wl["kind"], path="reference-cpu-tile",
            median_ms=round(statistics.median(per_layer), 4), blocks=blocks, capacity=cap,
            nnz=g.num_edges, density=round(g.num_edges / cap, 6) if cap else 0.0,
            max_rel_err=f"{err:.3e}", gpus=0, cpu_ms=round(ms, 3), cpu_cores=W.threads)])


CSV_HEADER = ("dataset,kernel,path,median_ms,blocks,capacity,nnz,density,max_rel_err,"
              "gpus,achieved_GBps,roofline_frac,tc_pipe_pct,cpu_ms,cpu_cores")


def write_report_csv(path, rows):
    """The reference bench's report schema (bench.hpp:53-55, bench.cpp:216-227):
    dataset,kernel,path,median_ms,blocks,capacity,nnz,density,max_rel_err —
    then the SURVEY §5 columns gpus,achieved_GBps,roofline_frac,tc_pipe_pct,
    cpu_ms,cpu_cores — so the CPU and GPU rows of a run sit side by side.
    max_rel_err: sampled rows of one layer (AGNN) / the SpMM (GCN) against a
    float64 evaluation (the reference bench's dense oracles stop at 2,048
    nodes, bench.cpp:194-209).  Appends (header once)."""
    new = not os.path.exists(path) or os.path.getsize(path) == 0
    with open(path, "a", newline="") as f:
        w = csv.writer(f, lineterminator="\n")
        if new:
            f.write(CSV_HEADER + "\n")
        for r in rows:
            w.writerow([r.get(k, "") for k in CSV_HEADER.split(",")])


DATA = "synthetic (deterministic generator; inputs = the reference bench's seeded streams)"


def dtype_name(prec):
    return "f32 (split-TF32 on tensor cores)" if prec == "fp32" else "tf32"


def metric_name(wl):
    k = "AGNN" if wl["kind"] == "agnn" else "GCN"
    return f"{k} layer-forward ms per graph"


def config_of(args, wl, g, gen):
    """Identical in both arms (the driver compares them)."""
    return {"workload": f"{args.workload} ({wl['cfg']}): {wl['kind'].upper()} on synthetic "
                        f"{args.workload.split('-')[0]}-shaped graph",
            "nodes": g.num_nodes, "edges": g.num_edges,
            "model": f"{wl['d_in']}->{wl['hidden']}->{wl['d_out']}, {wl['layers']} layers",
            "step": (f"agnn_forward({wl['layers']} layers, d={wl['hidden']}, beta=1) on the whole "
                     f"graph; value = ms per layer" if wl["kind"] == "agnn" else
                     f"gcn_forward({wl['layers']} layers); value = ms per layer"),
            "global_batch": 1, "seq_len": 0,
            "parallelism": f"rowwindow{args.gpus}" + (f" x{args.overlap} overlapped sub-slices"
                                                      if args.gpus > 1 and args.overlap > 1
                                                      and wl["kind"] == "agnn" else ""),
            "precision": args.precision, "mode": args.mode, "locality": args.locality,
            "generator": gen, "l2": "flushed between timed steps (256 MB write)"}


# ------------------------------------------------------------- B200 arm
def dist_setup():
    """One process per GPU (torchrun env).  More ranks than visible devices
    (the N>1 path exercised on a 1-GPU lease): ranks share devices, gloo."""
    import torch
    import torch.distributed as dist

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", str(rank)))
    ndev = torch.cuda.device_count()
    if ndev == 0:
        raise RuntimeError("bench.py (b200 arm) needs a CUDA device; there is no CPU fallback")
    devi = local % ndev
    torch.cuda.set_device(devi)
    backend = None
    if world > 1:
        backend = "nccl" if world <= ndev else "gloo"
        if backend == "nccl":
            dist.init_process_group("nccl", device_id=torch.device("cuda", devi))
        else:
            dist.init_process_group("gloo")
    return world, rank, devi, backend


def run_b200(args, wl):
    import torch
    import torch.distributed as dist

    import paper_2412_12218_b200 as sg
    from paper_2412_12218_b200 import device as D
    from paper_2412_12218_b200.distributed import RowSlice, allgather_rows

    world, rank, devi, backend = dist_setup()
    dev = torch.device("cuda", devi)
    prec = args.precision
    L, d = wl["layers"], wl["hidden"]

    t0 = time.perf_counter()
    g, gen = make_graph(wl, args.locality)
    N, E = g.num_nodes, g.num_edges
    log(f"[bench] rank {rank}: graph {N} nodes {E} edges in {time.perf_counter() - t0:.1f}s")
    # the library's AGNN auto mode (forward.cu): panels from 2M edges or d > 64, else the fused
    # kernel — resolved on the WHOLE graph so every partition runs the same kernels
    mode = {"panel": 2, "fused": 1, "chain": 0, "auto": -1}[args.mode]
    if mode < 0:
        mode = 2 if (wl["kind"] == "gcn" or E >= (2 << 20) or d > 64) else 1
    mode_name = {2: "panel", 1: "fused", 0: "chain"}[mode] + (" (auto)" if args.mode == "auto" else "")
    vals = sg.gcn_normalize_values(g).values if wl["kind"] == "gcn" else None

    # warm-up build on a small graph first: a fresh process's first build pays
    # the lazy loading of every translator / panel kernel module and the
    # memory pool's first growth (~0.8 s on a fresh box), not translation work
    gw = sg.synth_graph(20_000, 8.0, 2.0, 0.9, 4.0, 3)
    D.DeviceGraph.from_csr(gw.node_pointer, gw.edge_list, None, gw.num_nodes)
    os.environ["SGTK_BUILD_TIMING"] = "1"  # per-stage times of the graph below
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    chunks = args.overlap if (world > 1 and wl["kind"] == "agnn") else 1
    sl = RowSlice(g.node_pointer, g.edge_list, vals, N, rank, world, chunks=chunks)
    torch.cuda.synchronize()
    translate_ms = (time.perf_counter() - t0) * 1e3
    os.environ.pop("SGTK_BUILD_TIMING", None)
    dg = sl.graph
    info = dg.info
    bs = dg.block_stats()
    log(f"[bench] rank {rank}: rows [{sl.r0},{sl.r1}) translate {translate_ms:.1f} ms, "
        f"tiles8 {info.tiles8} tiles16 {info.tiles16} units {info.work_units8} "
        f"density16x8 {bs[3]:.4f}")

    flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
    stream = torch.cuda.current_stream()
    betas = np.ones(L, np.float32)
    if wl["kind"] == "agnn":
        h0_host = sg.dense_random(N, d, INPUT_SEED)
        h0_full = torch.from_numpy(h0_host).to(dev)
        h_rep = h0_full if world == 1 else sl.scatter_full(h0_full, sl.replica(d, dev))
        scratch = None if world == 1 else (sl.replica(d, dev), sl.replica(d, dev))
        out_buf = torch.empty((sl.rows, d), dtype=torch.float32, device=dev)

        def step():
            return sl.agnn_forward(h_rep, betas, precision=prec, mode=mode, scratch=scratch,
                                   out=out_buf)

        if mode == 2:
            pi = dg.panel_info(d)
            per_call = 3 + (1 if pi["long_rows"] else 0)  # dense + rows + final (+ hub rows)
            # one input kernel per call: once per step on 1 GPU, once per layer on N
            launches_per_step = (1 + L * per_call) if world == 1 else L * (1 + per_call) * chunks
        else:
            split = dg_has_splits(dg, 16 if mode == 1 else 8)
            launches_per_step = L * ((2 if mode == 1 else 4) + (1 if split else 0))
        x_in = h0_full
    else:
        x_full = torch.from_numpy(sg.dense_random(N, wl["d_in"], INPUT_SEED)).to(dev)
        x_loc = x_full[sl.r0:sl.r1]
        layers = [(torch.from_numpy(w).to(dev), r) for w, r in
                  sg.random_gcn_layers(wl["d_in"], wl["hidden"], wl["d_out"], L, LAYER_SEED)]
        reps = {}
        # asynchronous form (no per-call host sync: CUDA-graph capturable); the
        # non-finite flag is checked after the timing
        nf = torch.zeros(1, dtype=torch.int32, device=dev)

        def step():
            return sl.gcn_forward(x_loc, layers, precision=prec, reps=reps, nonfinite=nf)

        # per layer: W prep, GEMM, SpMM dense + sparse parts; the input's TF32
        # copy once; a ReLU pass after the SpMM in the A(XW) order; a split-K
        # reduction when the GEMM has few row tiles and a long K (gemm_tc05.cu).
        # With a CUDA graph the count below is replaced by the graph's own.
        launches_per_step = 1 + 4 * L + sum(1 for w, r in layers if r and w.shape[1] < w.shape[0])
        launches_per_step += sum(1 for w, _ in layers if (sl.rows + 127) // 128 < 74 and w.shape[0] >= 256)
        x_in = x_full

    # ---------------- timing --------------------------------------------------
    def max_over_ranks(v):
        if world == 1:
            return v
        t = torch.tensor([v], dtype=torch.float64, device=dev if backend == "nccl" else "cpu")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def timed(fn, steps, warmup):
        for _ in range(warmup):
            fn()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
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
        if world > 1:
            dist.barrier()
        return max_over_ranks(float(np.mean(ts))), ts

    warm = max(3, args.warmup)
    graph_note = None
    launches_note = "formula over the call's kernel sequence (step not graph-captured)"
    if args.cuda_graph and world == 1:
        # launch-bound configs (C1/C2: microsecond kernels): capture the whole
        # step once, replay it per step -- every kernel of the call still runs
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        cg = torch.cuda.CUDAGraph(keep_graph=True)  # kept: its kernel nodes are counted below
        with torch.cuda.graph(cg):
            g_out = step()  # the captured call's output (graph memory: stable across replays)
        eager_step = step

        def step():  # noqa: F811
            cg.replay()
            return g_out

        graph_note = "step captured once as a CUDA graph (torch.cuda.CUDAGraph) and replayed"
        stream = torch.cuda.current_stream()
        # gpu_launches from the captured graph itself: its kernel nodes from
        # this repo's library (namespace sgtkcu), per replayed step
        knames = graph_kernel_names(cg)
        if knames is not None and "?" not in knames:
            ours = sum(1 for k in knames if "sgtkcu" in k)
            if ours:
                launches_note = (f"counted: {ours} kernel nodes of libsgtk_b200 in the captured step graph "
                                 f"(formula: {launches_per_step})")
                launches_per_step = ours
    sampler, rows = clocks_sampler()
    step_ms, step_ts = timed(step, args.steps, warm)
    if sampler:
        sampler.terminate()
    clocks = summarize_clocks(rows)
    value = step_ms / L

    if wl["kind"] == "gcn" and int(nf.item()):
        raise SystemExit("gcn_forward produced NaN/Inf during the timed steps")
    if graph_note:
        # the replayed graph computes exactly what the eager call does
        replayed = step().clone()
        step = eager_step  # the checks below run the eager call
        graph_note += f"; replay == eager: {bool(torch.equal(replayed, step()))}"
    details = {"mode_resolved": mode_name, "translate_ms": round(translate_ms, 2),
               "cuda_graph": graph_note,
               "gpu_launches_source": launches_note,
               "translate_stages_ms": dg.build_times(),
               "translate_note": "host upload of the CSR + GPU sgt_transform + panel formats, after a "
                                 "warm-up build (module loading excluded); stages synchronised",
               "tiles16x8": int(bs[0]), "tile_density16x8": round(bs[3], 4),
               "rows_this_rank": [sl.r0, sl.r1],
               "panel_format": dg.panel_info(d) if mode == 2 else None}
    if world > 1:
        details.update(backend=backend, devices=torch.cuda.device_count(),
                       exchange="one in-place all_gather_into_tensor per layer over the padded "
                                "replica" if backend == "nccl" else
                                "gloo all-gather via host copies (ranks share a device)")

    # ---------------- N>1: bit-identical against one device ------------------
    verify = None
    if world > 1 and args.verify:
        out_loc = step()
        torch.cuda.synchronize()
        loc = out_loc if backend == "nccl" else out_loc.cpu()
        full = allgather_rows(loc, sl.ranges).cpu()
        if rank == 0:
            whole = D.DeviceGraph.from_csr(g.node_pointer, g.edge_list, vals, N)
            if wl["kind"] == "agnn":
                want = whole.agnn_forward(x_in, betas, precision=prec, mode=mode)
            else:
                want = whole.gcn_forward(x_in, layers, precision=prec, order=2)
            verify = {"bit_identical": bool(torch.equal(want.cpu(), full)),
                      "against": "single-device forward of the whole graph (rank 0)"}
            del whole
        if world > 1:
            dist.barrier()

    # ---------------- N=1 extras: model forward, kernel breakdown, roofline ---
    roof = None
    kern = {}
    extra = {}
    model_ms = None
    err = None
    if world == 1:
        if wl["kind"] == "agnn":
            x_host = sg.dense_random(N, wl["d_in"], INPUT_SEED + 1)
            w_in = torch.from_numpy(sg.dense_random(wl["d_in"], d, 1, -0.1, 0.1)).to(dev)
            w_out = torch.from_numpy(sg.dense_random(d, wl["d_out"], 2, -0.1, 0.1)).to(dev)
            ldx = (wl["d_in"] + 3) // 4 * 4  # 16-byte row pitch (TMA-eligible rows)
            xp = torch.zeros((N, ldx), dtype=torch.float32, device=dev)[:, :wl["d_in"]]
            xp.copy_(torch.from_numpy(x_host))

            def model_forward():
                hh = D.gemm(xp, w_in, relu=True, precision=prec)
                return D.gemm(dg.agnn_forward(hh, betas, precision=prec, mode=mode), w_out,
                              relu=False, precision=prec)

            model_ms, _ = timed(model_forward, max(2, args.steps // 2), 2)
            proj = (xp, w_in)
            rows_s = sample_rows(N)
            one = dg.agnn_forward(h0_full, betas[:1], precision=prec, mode=mode).cpu().numpy()
            err = max_rel_err(one[rows_s], rows_agnn_f64(g.node_pointer, g.edge_list, h0_host, rows_s))
        else:
            proj = None
            rows_s = sample_rows(N)
            agg = dg.spmm(x_full, precision=prec).cpu().numpy()
            err = max_rel_err(agg[rows_s], rows_spmm_f64(g.node_pointer, g.edge_list, vals,
                                                         x_full.cpu().numpy(), rows_s))
        kern, roof = kernel_breakdown(args, wl, dg, g, x_in, D, prec, mode, flush, stream,
                                      layers if wl["kind"] == "gcn" else None, extra, proj)

    # ---------------- e2e: host buffers in, host buffers out ------------------
    if world == 1:
        e2e = e2e_host(wl, dg, x_in, prec, mode, L, L, layers if wl["kind"] == "gcn" else None,
                       flush, args)
    else:
        e2e = e2e_multi(wl, sl, step, x_in, h_rep if wl["kind"] == "agnn" else None,
                        None if wl["kind"] == "agnn" else x_loc, L, args, max_over_ranks, flush)

    # ---------------- CPU baseline (rank 0, N=1) ------------------------------
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            cpu = cpu_baseline_leg(wl, g, prec, ref_lib())
        except FileNotFoundError as e:
            cpu = {"value": None, "unavailable": str(e)}

    pk, pk_src = peaks()
    if world > 1:
        # whole job: the layer's algorithmic bytes over the whole graph (SURVEY
        # §8d; AGNN: the fused lower bound, GCN: B_spmm + B_gemm) per layer time,
        # against N GPUs' worth of HBM; the exchange is not counted as useful bytes
        s_ = 4
        if wl["kind"] == "agnn":
            B = 8 * (N + 1) + 4 * E + 4 * N + 2 * s_ * N * d
            formula = "8(N+1) + 4E + 4N + 2*s*N*d per layer (fused AGNN lower bound), whole graph"
        else:
            B = (8 * (N + 1) + 8 * E + 2 * s_ * N * d) + (s_ * N * d + 4 * d * d + 4 * N * d)
            formula = "B_spmm + B_gemm per layer (d -> d), whole graph"
        roof = {"bound": "hbm", "kernel": f"whole layer on {world} GPUs (step / layers)",
                "achieved": round(B / (value * 1e-3) / 1e9, 1), "unit": "GB/s",
                "algorithmic_bytes": int(B), "formula": formula, "kernel_ms": round(value, 4),
                "traffic": None}
        roof["peak"] = pk["hbm_gbs"] * world
        roof["frac"] = round(roof["achieved"] / roof["peak"], 4)
        roof["peak_source"] = f"MEASURED_PEAKS.json hbm_gbs x {world} GPUs ({pk_src})"
    elif roof:
        roof["traffic"] = profiled_traffic(roof["kernel"], gcn=wl["kind"] == "gcn")
        roof["peak"] = pk["hbm_gbs"]
        roof["frac"] = round(roof["achieved"] / pk["hbm_gbs"], 4)
        roof["peak_source"] = f"MEASURED_PEAKS.json hbm_gbs ({pk_src})"
        roof["tc_pipe_pct"] = profiled_tc_pipe(gcn=wl["kind"] == "gcn")

    if rank == 0:
        line = {
            "metric": metric_name(wl), "value": round(value, 4), "unit": "ms",
            "n_gpus": world, "steps": args.steps, "warmup": warm,
            "ms_per_step": round(step_ms, 4), "higher_is_better": False,
            "scaling": "strong", "vs_baseline": None, "dtype": dtype_name(prec), "data": DATA,
            "config": config_of(args, wl, g, gen),
            "roofline": roof, "cpu_baseline": cpu, "e2e": e2e, "clocks": clocks,
            "gpu_launches": launches_per_step * args.steps,
            "max_rel_err_sampled": err, "verify": verify,
            "model_forward_ms": None if model_ms is None else round(model_ms, 4),
            "kernels_ms": kern, "details": details,
        }
        if "roofline_unfused_formula" in extra and roof:
            u = extra["roofline_unfused_formula"]
            u["achieved"] = round(u["algorithmic_bytes"] / (roof["kernel_ms"] * 1e-3) / 1e9, 1)
            u["unit"] = "GB/s"
            u["frac"] = round(u["achieved"] / pk["hbm_gbs"], 4)
            line["roofline_unfused_formula"] = u
        if "roofline_l2_gather" in extra:
            line["roofline_l2_gather"] = extra["roofline_l2_gather"]
        if "roofline_sddmm" in extra:
            rs = extra["roofline_sddmm"]
            rs["peak"] = pk["hbm_gbs"]
            rs["frac"] = round(rs["achieved"] / pk["hbm_gbs"], 4)
            line["roofline_sddmm"] = rs
        if "roofline_gemm" in extra:
            rg = extra["roofline_gemm"]
            rg["peak"] = pk["hbm_gbs"]
            rg["frac"] = round(rg["achieved"] / pk["hbm_gbs"], 4)
            line["roofline_gemm"] = rg
        print(json.dumps(line), flush=True)
        if args.csv:
            write_report_csv(args.csv, [dict(
                dataset=args.workload, kernel=wl["kind"], path=f"b200-{mode_name.split()[0]}",
                median_ms=round(statistics.median(step_ts) / L, 4), blocks=bs[0], capacity=bs[1],
                nnz=bs[2], density=round(bs[3], 6),
                max_rel_err="" if err is None else f"{err:.3e}", gpus=world,
                achieved_GBps=roof["achieved"] if roof else "",
                roofline_frac=roof["frac"] if roof else "",
                tc_pipe_pct=((roof or {}).get("tc_pipe_pct") or {}).get("pct", ""),
                cpu_ms=cpu.get("value") if cpu else "", cpu_cores=cpu.get("cores") if cpu else "")])
    if world > 1:
        dist.destroy_process_group()


def e2e_multi(wl, sl, step, x_full, h_rep, x_loc, L, args, max_over_ranks, flush):
    """N>1 end to end: every step copies this rank's input rows from pinned
    host memory (AGNN: into its block of the replica, then the exchange), runs
    the layers, and reads its output rows back; max over ranks."""
    import torch

    d_in = x_full.shape[1]
    pin_in = x_full[sl.r0:sl.r1].cpu().pin_memory()
    out0 = step()
    pin_out = torch.empty(tuple(out0.shape), dtype=torch.float32).pin_memory()
    chunked = h_rep is not None and sl.chunks > 1
    dst = None if chunked else (sl.mine(h_rep) if h_rep is not None else x_loc)

    def call():
        if chunked:
            sl.write_mine(h_rep, pin_in)
        else:
            dst.copy_(pin_in, non_blocking=True)
        if h_rep is not None:
            sl.exchange(h_rep)
        pin_out.copy_(step(), non_blocking=True)
        torch.cuda.current_stream().synchronize()

    for _ in range(2):
        call()
    ts = []
    for _ in range(max(3, args.steps)):
        flush.fill_(1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        call()
        ts.append((time.perf_counter() - t0) * 1e3)
    ms = max_over_ranks(float(np.mean(ts)))
    d_out = int(out0.shape[1])
    return {"value": round(ms / L, 4), "unit": "ms",
            "h2d_bytes_per_step": int(sl.n * d_in * 4), "d2h_bytes_per_step": int(sl.n * d_out * 4),
            "path": "distributed.RowSlice (pinned H2D of each rank's rows -> layers with in-place "
                    "all-gathers -> D2H of each rank's rows); bytes summed over ranks"}


def profiled_tc_pipe(gcn=False):
    """Tensor-pipe utilisation of the dominant tcgen05 kernel from the newest
    committed ncu summary (profiles/*_ncu_full.md, tools/ncu_summary.py)."""
    import glob
    import re

    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "*_ncu_full.md")))
    files = [f for f in files if f.endswith("_gcn_ncu_full.md") == gcn]
    kern = "spmm_panel_kernel" if gcn else "agnn_dense_kernel"
    for path in reversed(files):
        try:
            text = open(path).read()
        except OSError:
            continue
        sec = text.split(f"{kern}<")
        if len(sec) < 2:
            continue
        m = re.search(r"\| sm__pipe_tensor_cycles_active\.avg\.pct_of_peak_sustained_active \| "
                      r"([0-9.]+)", sec[1].split("## ")[0])
        if m:
            return {"kernel": kern, "pct": float(m.group(1)),
                    "metric": "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
                    "source": os.path.relpath(path, ROOT)}
    return None


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


class _KernelNodeParams(C.Structure):  # CUDA_KERNEL_NODE_PARAMS_v2 (cuda.h)
    _fields_ = [("func", C.c_void_p), ("grid", C.c_uint * 3), ("block", C.c_uint * 3),
                ("smem", C.c_uint), ("params", C.c_void_p), ("extra", C.c_void_p),
                ("kern", C.c_void_p), ("ctx", C.c_void_p)]


def graph_kernel_names(cg):
    """Names of the kernel nodes of a captured torch.cuda.CUDAGraph (driver
    API: cuGraphGetNodes / cuGraphKernelNodeGetParams / cuFuncGetName or
    cuKernelGetName), or None when the driver cannot say."""
    try:
        cu = C.CDLL("libcuda.so.1")
        g = C.c_void_p(cg.raw_cuda_graph())
        n = C.c_size_t(0)
        if cu.cuGraphGetNodes(g, None, C.byref(n)) != 0:
            return None
        nodes = (C.c_void_p * n.value)()
        if cu.cuGraphGetNodes(g, nodes, C.byref(n)) != 0:
            return None
        names = []
        for nd in nodes[:n.value]:
            t = C.c_int(-1)
            if cu.cuGraphNodeGetType(C.c_void_p(nd), C.byref(t)) != 0 or t.value != 0:  # CU_GRAPH_NODE_TYPE_KERNEL
                continue
            p = _KernelNodeParams()
            if cu.cuGraphKernelNodeGetParams_v2(C.c_void_p(nd), C.byref(p)) != 0:
                return None
            name = C.c_char_p()
            ok = p.func and cu.cuFuncGetName(C.byref(name), C.c_void_p(p.func)) == 0
            if not ok and p.kern:
                ok = cu.cuKernelGetName(C.byref(name), C.c_void_p(p.kern)) == 0
            names.append(name.value.decode() if ok and name.value else "?")
        return names
    except Exception:  # noqa: BLE001 -- an old driver / torch: fall back to the formula
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
        Bs = 8 * (N + 1) + 4 * E + 4 * N * d + 4 * E
        extra["roofline_sddmm"] = {
            "bound": "hbm", "kernel": "sddmm_hybrid (sddmm_dense2_kernel tcgen05 + sddmm_sparse_kernel)",
            "achieved": round(Bs / (res["sddmm"] * 1e-3) / 1e9, 1), "unit": "GB/s",
            "algorithmic_bytes": int(Bs), "formula": "8(N+1) + 4E + s*N*d + 4E (SURVEY §8d B_sddmm, s=4)",
            "kernel_ms": round(res["sddmm"], 4)}
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


def free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


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
    ap.add_argument("--overlap", type=int, default=1,
                    help="N > 1, AGNN: sub-slices per rank whose all-gathers overlap the next "
                         "sub-slice's compute (distributed.RowSlice chunks)")
    ap.add_argument("--no-cuda-graph", dest="cuda_graph", action="store_false",
                    help="AGNN: time the eager calls instead of the step captured once as a "
                         "CUDA graph and replayed (the default; every kernel still runs)")
    ap.add_argument("--no-verify", dest="verify", action="store_false",
                    help="N>1: skip the bit-identity check against a one-device forward")
    ap.add_argument("--csv", default="", help="also append a row in the reference bench's CSV "
                                               "schema (bench.hpp:53-55) to this file")
    args = ap.parse_args()
    wl = WORKLOADS[args.workload]
    if args.impl == "reference":
        run_reference_arm(args, wl)
        if os.environ.get("SGTK_BENCH_PRINT_MAPS"):  # tests: which native libraries loaded
            with open("/proc/self/maps") as f:
                libs = sorted({ln.split()[-1] for ln in f if ln.rstrip().endswith(".so")})
            log("[bench] loaded: " + " ".join(libs))
        return
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        # one process per GPU: re-launch under torchrun (the driver's own launch form)
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
               f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
               f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    if world != args.gpus:
        log(f"[bench] WORLD_SIZE={world} overrides --gpus {args.gpus}")
        args.gpus = world
    run_b200(args, wl)


if __name__ == "__main__":
    main()
