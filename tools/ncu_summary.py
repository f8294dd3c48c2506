"""Summarise an ncu report + launch list into profiles/<tag>_*.md/csv."""
import collections
import csv
import io
import subprocess
import sys

tag, rep = sys.argv[1], sys.argv[2]
launches = sys.argv[3] if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tc_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__ops_path_tensor_op_utchmma_src_tf32_dst_fp32.sum",
        "sm__inst_executed_pipe_tc_scope_1cta.sum",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed.sum", "launch__registers_per_thread", "launch__grid_size",
        "launch__shared_mem_per_block_dynamic"]
out = [f"# ncu --set full summary ({tag})\n",
       f"Source: `{rep}` (gpurun_out/, not committed: 10+ MB). One launch per kernel shown;",
       "cold-cache, serialised replay (compare shares, not absolutes).\n"]
seen = set()
for r in rows[2:]:
    name = r[hdr.index("Kernel Name")]
    short = name.split("(")[0].replace("void ", "")
    if short in seen:
        continue
    seen.add(short)
    out.append(f"## `{short}`\n")
    out.append("| metric | value | unit |\n|---|---|---|")
    for k in keys:
        if k in hdr:
            out.append(f"| {k} | {r[hdr.index(k)]} | {units[hdr.index(k)]} |")
    out.append("")
open(f"profiles/{tag}_ncu_full.md", "w").write("\n".join(out) + "\n")
if not launches:
    sys.exit(0)
rows = list(csv.reader(open(launches)))
i = [k for k, r in enumerate(rows) if r and r[0] == "ID"][0]
hdr = rows[i]
iN, iV, iM = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Name")
agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
for r in rows[i + 1:]:
    if len(r) <= iV:
        continue
    nm = r[iN].split("(")[0].replace("void ", "").strip()
    try:
        v = float(r[iV].replace(",", ""))
    except ValueError:
        continue
    if r[iM] == "gpu__time_duration.sum":
        agg[nm][0] += 1
        agg[nm][1] += v
    elif r[iM].startswith("dram__bytes"):
        agg[nm][2] += v
tot = sum(v[1] for v in agg.values())
with open(f"profiles/{tag}_launches.csv", "w", newline="") as f:
    w = csv.writer(f)
    w.writerow(["kernel", "launches", "total_ns", "avg_ns", "share_pct", "dram_bytes_per_launch"])
    for k, (n, t, b) in sorted(agg.items(), key=lambda x: -x[1][1]):
        w.writerow([k, n, f"{t:.0f}", f"{t / max(n, 1):.0f}", f"{t / tot * 100:.2f}", f"{b / max(n, 1):.0f}"])
print(open(f"profiles/{tag}_launches.csv").read()[:2500])
