import sys, os, time, numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench
g, _ = bench.make_graph(bench.WORKLOADS[sys.argv[1] if len(sys.argv) > 1 else 'reddit-agnn'], "calibrated")
n = g.num_nodes; npz = g.node_pointer.astype(np.int64); el = g.edge_list.astype(np.int64)
rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(npz))
for P in (64, 128, 256):
    key = (rows // P) * n + el
    u, cnt = np.unique(key, return_counts=True)
    for thr in (2, 3, 4):
        dense = cnt >= thr
        p = u // n
        dc = np.bincount(p[dense], minlength=(n + P - 1) // P)
        chunks = int(np.sum((dc + 31) // 32))
        de = int(cnt[dense].sum())
        # tensor work ~ chunks * P rows; gathers ~ chunks * 32 rows
        print(f"P={P} thr={thr}: chunks {chunks} dense {de/len(el):.3f} density {de/(chunks*P*32.0):.3f} "
              f"MMA rows {chunks*P/1e6:.2f}M gathered rows {chunks*32/1e6:.2f}M sparse edges {(len(el)-de)/1e6:.1f}M", flush=True)
