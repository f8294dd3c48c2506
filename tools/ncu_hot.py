"""Summarise an ncu report: SOL metrics + top stalled SASS lines (with barrier hints)."""
import csv, subprocess, sys
rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "details", "--csv"], capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[0]
want = {"Duration", "Memory Throughput", "DRAM Throughput", "L1/TEX Cache Throughput", "L2 Cache Throughput",
        "Compute (SM) Throughput", "Issue Slots Busy", "L1/TEX Hit Rate", "L2 Hit Rate", "Registers Per Thread",
        "Achieved Active Warps Per SM", "No Eligible", "SM Frequency"}
for row in r[1:]:
    d = dict(zip(h, row))
    if d.get("Metric Name") in want:
        print(f"{d['Kernel Name'][:40]:40s} {d['Metric Name']:32s} {d['Metric Value']} {d['Metric Unit']}")
kf = sys.argv[3:] and ["-k", "regex:" + sys.argv[3]] or []
out = subprocess.run(["ncu", "-i", rep] + kf + ["--page", "source", "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]; data = rows[2:]
iS = h.index("Warp Stall Sampling (All Samples)"); iSrc = h.index("Source")
tot = sum(int(x[iS]) for x in data if x[iS].isdigit())
print("total samples", tot)
rank = sorted(range(len(data)), key=lambda i: -int(data[i][iS]) if data[i][iS].isdigit() else 0)
for i in rank[:top]:
    ctx = data[i - 1][iSrc].strip()[:60] if i else ""
    print(f"{i:5d} {int(data[i][iS]):6d} {100*int(data[i][iS])/tot:5.1f}%  {data[i][iSrc].strip()[:70]:70s} | prev: {ctx}")
