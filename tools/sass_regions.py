"""Instruction / stall distribution over a kernel's SASS from an ncu report
(source page), in blocks of N lines, plus the opcode histogram of a line range.
    python tools/sass_regions.py <rep> <kernel regex> [block=30] [lo hi]"""
import csv, subprocess, sys
from collections import Counter
rep, kern = sys.argv[1], sys.argv[2]
blk = int(sys.argv[3]) if len(sys.argv) > 3 else 30
out = subprocess.run(["ncu", "-i", rep, "-k", "regex:" + kern, "--launch-count", "1", "--page", "source",
                      "--csv", "--print-source", "sass"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[1]
data = [x for x in rows[2:] if len(x) == len(h)]
iS, iSrc, iI = h.index("Warp Stall Sampling (All Samples)"), h.index("Source"), h.index("Instructions Executed")
n = lambda v: int(v) if v.isdigit() else 0
sc = [i for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
for x in data:
    for i in sc:
        try:
            float(x[i] or 0)
        except ValueError:
            x[i] = "0"
tot, ts = sum(n(x[iI]) for x in data), sum(n(x[iS]) for x in data)
print("lines", len(data), "instructions", tot, "samples", ts)
for b in range(0, len(data), blk):
    s, st = sum(n(x[iI]) for x in data[b:b + blk]), sum(n(x[iS]) for x in data[b:b + blk])
    if s > tot * 0.01 or st > ts * 0.01:
        rs = {h[i]: sum(float(x[i] or 0) for x in data[b:b + blk]) for i in sc}
        top = sorted(rs.items(), key=lambda t: -t[1])[:3]
        print(f"{b:5d} inst {s:11d} {100*s/tot:5.1f}%  stall {st:6d} {100*st/ts:5.1f}%  {data[b][iSrc][:50]:50s}",
              " ".join(f"{k[6:]}:{v:.0f}" for k, v in top if v > 0))
if len(sys.argv) > 5:
    lo, hi = int(sys.argv[4]), int(sys.argv[5])
    c = Counter()
    for x in data[lo:hi]:
        op = [o for o in x[iSrc].split() if not o.startswith("@")]
        c[op[0] if op else ""] += n(x[iI])
    for k, v in c.most_common(25):
        print(f"  {k:40s} {v}")
