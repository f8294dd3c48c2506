"""Per-chunk pipeline timeline from an SGTK_PANEL_TRACE dump (-DSGTK_TRACE build):
int64 clock64 stamps [cta 0..3][chunk 0..255][event 0..7], 0 = not recorded.
    python tools/trace_view.py <file> [cta] [first chunk] [n chunks]"""
import sys
import numpy as np
t = np.fromfile(sys.argv[1], np.int64).reshape(4, 256, 8)
cta = int(sys.argv[2]) if len(sys.argv) > 2 else 0
c0 = int(sys.argv[3]) if len(sys.argv) > 3 else 0
nc = int(sys.argv[4]) if len(sys.argv) > 4 else 24
x = t[cta].astype(np.float64)
base = x[x > 0].min()
ev = [e for e in range(8) if (x[:, e] > 0).any()]
print("cycles from the CTA's first event; events:", ev)
print("chunk " + " ".join(f"{e:>8d}" for e in ev))
for c in range(c0, c0 + nc):
    if not (x[c] > 0).any():
        break
    print(f"{c:5d} " + " ".join(f"{(x[c, e] - base):8.0f}" if x[c, e] > 0 else "       -" for e in ev))
last = max(c for c in range(256) if (x[c] > 0).any())
for e in ev:
    v = x[:last + 1, e]
    v = v[v > 0]
    if len(v) > 8:
        print(f"event {e}: mean period {np.diff(v[4:]).mean():.0f} cycles")
