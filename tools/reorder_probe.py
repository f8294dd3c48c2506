import sys, time, numpy as np
sys.path.insert(0, __import__('os').path.dirname(__import__('os').path.dirname(__import__('os').path.abspath(__file__))))
import bench
wl = bench.WORKLOADS['reddit-agnn']
t0=time.time()
g, _ = bench.make_graph(wl, "calibrated")
n = g.num_nodes; npz = g.node_pointer.astype(np.int64); el = g.edge_list.astype(np.int64)
rows = np.repeat(np.arange(n, dtype=np.int64), np.diff(npz))
print("graph", n, len(el), time.time()-t0, flush=True)
def stats(rows, cols, thr=3):
    key = (rows // 128) * n + cols
    u, cnt = np.unique(key, return_counts=True)
    dense = cnt >= thr
    p = u // n
    dcols_per_panel = np.bincount(p[dense], minlength=(n+127)//128)
    chunks = int(np.sum((dcols_per_panel + 31) // 32))
    dense_edges = int(cnt[dense].sum())
    return chunks, dense_edges, dense_edges / (chunks * 4096.0)
c, de, dens = stats(rows, el)
print(f"original: chunks {c} dense edges {de} ({de/len(el):.3f}) density {dens:.3f}", flush=True)
from scipy.sparse import csr_matrix
from scipy.sparse.csgraph import reverse_cuthill_mckee
A = csr_matrix((np.ones(len(el), np.int8), el, npz), shape=(n, n))
t0=time.time(); perm = reverse_cuthill_mckee(A, symmetric_mode=True); print("rcm", time.time()-t0, flush=True)
inv = np.empty(n, np.int64); inv[perm] = np.arange(n)
c2, de2, dens2 = stats(inv[rows], inv[el])
print(f"rcm: chunks {c2} dense edges {de2} ({de2/len(el):.3f}) density {dens2:.3f}", flush=True)
