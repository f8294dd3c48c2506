// Model forwards on the device: GCN (gnn.cpp:33-52) and AGNN (gnn.cpp:93-119).
//
// GCN per layer: h <- relu?(A h W).  The reference aggregates first,
// (A h) W (gnn.cpp:43-44); when d_out < d_in the same product is cheaper as
// A (h W) (the SpMM then gathers d_out-wide rows instead of d_in-wide ones:
// at Cora 1433->16 that is 90x fewer gathered bytes).  `order` selects.
//
// AGNN per layer (mode 0, the reference chain):
//   l2norm -> inv_norm[N]            (z never materialised; the SDDMM scales
//                                      rows by inv_norm as it loads them)
//   SDDMM(16-wide tiles) * beta      -> logits[E], CSR order
//   edge_softmax (in place)          -> attention[E]
//   SpMM(8-wide tiles, attention)    -> h_next
// mode 1: the fused single-pass kernel (agnn_fused.cu): logits and attention
// never touch HBM.

#include <algorithm>

#include "kernels.cuh"

namespace sgtkcu {
namespace {

__global__ void relu_nonfinite_kernel(float* __restrict__ x, uint64_t rows, uint64_t cols,
                                      uint64_t ld, int relu, uint32_t* __restrict__ nonfinite) {
  bool bad = false;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < rows * cols;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = i / cols, c = i - r * cols;
    const float v0 = x[r * ld + c];
    float v = v0;
    if (relu) {
      v = v > 0.0f ? v : 0.0f;
      x[r * ld + c] = v;
    }
    // after a ReLU, -inf is zeroed like the reference's ReLU does; a NaN
    // before it (inf - inf upstream) still counts
    bad |= !isfinite(v) || isnan(v0);
  }
  if (nonfinite && __any_sync(0xFFFFFFFFu, bad) && (threadIdx.x & 31) == 0) atomicOr(nonfinite, 1u);
}

inline uint64_t ld4(uint64_t d) { return (d + 3) / 4 * 4; }
inline uint64_t align256(uint64_t b) { return (b + 255) / 256 * 256; }

}  // namespace

void relu_nonfinite_launch(float* x, uint64_t rows, uint64_t cols, uint64_t ld, int relu,
                           uint32_t* nonfinite, cudaStream_t s) {
  if (!rows || !cols) return;
  const uint64_t n = rows * cols;
  unsigned blocks = unsigned(std::min<uint64_t>((n + 255) / 256, 148 * 32));
  relu_nonfinite_kernel<<<blocks, 256, 0, s>>>(x, rows, cols, ld, relu, nonfinite);
  CU_LAUNCH("relu_nonfinite_kernel");
}

std::vector<uint32_t> split_plan_host(const sgtk_graph* g, double ratio) {
  if (!(ratio >= 0.0 && ratio <= 1.0)) raise(SGTK_ERR_RANGE, "split ratio must be within [0, 1]");
  std::vector<uint32_t> cut(g->bp_host.size());
  for (size_t w = 0; w < cut.size(); ++w)
    cut[w] = uint32_t(std::floor(ratio * double(g->bp_host[w])));
  return cut;
}

uint64_t gcn_workspace(const sgtk_graph* g, uint32_t L, const uint64_t* dims) {
  uint64_t mx = 0;
  for (uint32_t l = 0; l <= L; ++l) mx = std::max(mx, ld4(dims[l]));
  return 3 * align256(g->n_rows * mx * 4) + 256;
}

void gcn_forward(const sgtk_graph* g, const float* x, uint64_t ldx, uint32_t L,
                 const uint64_t* dims, const float* weights, const int* relu,
                 const uint32_t* cut, int prec, int order, void* ws, uint64_t ws_bytes, float* out,
                 uint64_t ldo, cudaStream_t s, uint32_t* nonfinite_dev) {
  const uint64_t N = g->n_rows;
  if (L == 0) raise(SGTK_ERR_SHAPE, "gcn_forward: no layers");
  if (ws_bytes < gcn_workspace(g, L, dims)) raise(SGTK_ERR_SHAPE, "gcn_forward: workspace too small");
  uint64_t mx = 0;
  for (uint32_t l = 0; l <= L; ++l) mx = std::max(mx, ld4(dims[l]));
  char* base = static_cast<char*>(ws);
  const uint64_t slab = align256(N * mx * 4);
  float* buf[2] = {reinterpret_cast<float*>(base), reinterpret_cast<float*>(base + slab)};
  float* tmp = reinterpret_cast<float*>(base + 2 * slab);
  // the check goes to the caller's flag (asynchronous entry) or to a
  // workspace word read back below (the synchronous, raising one)
  uint32_t* flag = nonfinite_dev ? nonfinite_dev : reinterpret_cast<uint32_t*>(base + 3 * slab);
  if (!nonfinite_dev) CU(cudaMemsetAsync(flag, 0, 4, s));

  const float* h = x;
  uint64_t ldh = ldx;
  bool h_tf32 = false;  // h already TF32-rounded by the GEMM epilogue that wrote it
  const float* w = weights;
  const bool tf = prec == SGTK_TF32;
  for (uint32_t l = 0; l < L; ++l) {
    const uint64_t din = dims[l], dout = dims[l + 1];
    const bool last = l + 1 == L;
    float* dst = last ? out : buf[l & 1];
    const uint64_t ldd = last ? ldo : ld4(dout);
    const bool alt = order == 1 || (order == 2 && dout < din);
    if (!alt) {  // reference order: (A h) W; the GEMM epilogue applies ReLU,
                 // rounds for the next layer's TF32 SpMM and checks the output
      spmm_launch(g, h, ldh, din, cut, nullptr, prec, tmp, ld4(din), flag, s, h_tf32);
      gemm_launch(tmp, ld4(din), w, N, din, dout, relu[l], prec, dst, ldd, s, tf && !last,
                  last ? flag : nullptr);
      h_tf32 = tf && !last;
    } else {      // A (h W), ReLU after the aggregation
      gemm_launch(h, ldh, w, N, din, dout, 0, prec, tmp, ld4(dout), s, tf);
      // A (h W) is not the reference's checked quantity A h: a hidden layer's
      // -inf that its ReLU zeroes must not raise, so those layers are checked
      // after the ReLU only (relu_nonfinite_launch)
      spmm_launch(g, tmp, ld4(dout), dout, cut, nullptr, prec, dst, ldd,
                  relu[l] && !last ? nullptr : flag, s, tf);
      if (relu[l] || last) relu_nonfinite_launch(dst, N, dout, ldd, relu[l], flag, s);
      h_tf32 = false;
    }
    w += din * dout;
    h = dst;
    ldh = ldd;
  }
  if (nonfinite_dev) return;
  uint32_t hf = 0;
  CU(cudaMemcpyAsync(&hf, flag, 4, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (hf) raise(SGTK_ERR_NONFINITE, "gcn_forward: output contains NaN or Inf");
}

uint64_t agnn_workspace_chain(const sgtk_graph* g, uint64_t d) {
  return 2 * align256(g->n_rows * ld4(d) * 4) + align256(g->n_cols * 4) +
         align256(g->n_cols * ld4(d) * 4) +
         align256(std::max<uint64_t>(g->nnz, 1) * 4) + align256(16 * 4);
}

// mode 2 (panels): two sets of {z, zq, zq1, hq, hq1} (n_cols x ldq; the next
// layer's set is written while the current one is read), layer outputs
// (2 x n_rows x ld4(d)), dense partials (n_rows x (ldq + 1)), hub segment
// partials, zero counter.
uint64_t agnn_workspace_panel(const sgtk_graph* g, uint64_t d) {
  if (!g->panels || d > 64) return 0;
  const uint64_t ldq = d <= 32 ? 32 : 64;
  const auto& pn = panels_for(g, d);
  return 10 * align256(g->n_cols * ldq * 4) + 2 * align256(g->n_cols * 4) +
         align256(g->n_cols * 4) + 2 * align256(g->n_rows * ld4(d) * 4) +
         2 * align256(g->n_rows * ldq * 4) + 2 * align256(g->n_rows * 4) +
         align256(std::max<uint64_t>(pn.n_segs, 1) * ldq * 4) +
         align256(std::max<uint64_t>(pn.n_segs, 1) * 4) + align256(16 * 4);
}

uint64_t agnn_workspace(const sgtk_graph* g, uint64_t d) {
  return std::max(agnn_workspace_chain(g, d), agnn_workspace_panel(g, d));
}

namespace {
// End of an AGNN forward: the zero-norm row count (u64) and the non-finite
// flag (u32 right after it) come back in one copy.  spmm_hybrid throws
// NonFiniteError for any layer whose output holds NaN/Inf
// (tile_exec.cpp:311-312, via gnn.cpp:115); see nx.nonfinite for why the last
// layer's check covers every layer.
// The synchronous check runs when the caller asks for the zero-row count
// (every host-level API does: sg.agnn_forward, the drop-in, *_host); a
// device-level call without it stays asynchronous, like sgtk_spmm without a
// nonfinite pointer.
void finish_agnn(const uint64_t* zeros_dev, uint64_t* zero_rows_host, cudaStream_t s) {
  if (!zero_rows_host) return;
  uint64_t hv[2] = {0, 0};
  CU(cudaMemcpyAsync(hv, zeros_dev, 16, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  *zero_rows_host = hv[0];
  if (hv[1] & 0xFFFFFFFFull) raise(SGTK_ERR_NONFINITE, "agnn_forward: output contains NaN or Inf");
}

// mode 2: every layer on the 128-row panels (agnn_panel.cu)
void agnn_forward_panel(const sgtk_graph* g, const float* x, uint64_t ldx, uint64_t d, uint32_t L,
                        const float* betas, int prec, void* ws, float* out, uint64_t ldo,
                        uint64_t* zero_rows_host, cudaStream_t s) {
  const uint64_t N = g->n_rows, NC = g->n_cols;
  const uint64_t ldq = d <= 32 ? 32 : 64, ldb = ld4(d);
  const auto& pn = panels_for(g, d);
  char* p = static_cast<char*>(ws);
  auto take = [&](uint64_t bytes) {
    float* r = reinterpret_cast<float*>(p);
    p += align256(bytes);
    return r;
  };
  float* set[2][5];
  for (int a = 0; a < 2; ++a)
    for (int b = 0; b < 5; ++b) set[a][b] = take(NC * ldq * 4);  // z, zq, zq1, hq, hq1
  float* norm[2] = {take(NC * 4), take(NC * 4)};
  float* buf[2] = {take(N * ldb * 4), take(N * ldb * 4)};
  float* opart = take(N * ldq * 4);
  float* lpart = take(N * 4);
  float* osp = take(N * ldq * 4);
  float* lsp = take(N * 4);
  float* seg_o = take(std::max<uint64_t>(pn.n_segs, 1) * ldq * 4);
  float* seg_l = take(std::max<uint64_t>(pn.n_segs, 1) * 4);
  uint64_t* zeros = reinterpret_cast<uint64_t*>(p);
  uint32_t* flag = reinterpret_cast<uint32_t*>(zeros + 1);
  CU(cudaMemsetAsync(zeros, 0, 16, s));
  // padding features [d, ldq) of every operand row must read as zeros
  if (d < ldq)
    CU(cudaMemsetAsync(set[0][0], 0, reinterpret_cast<char*>(set[1][4]) - reinterpret_cast<char*>(set[0][0]) +
                                         NC * ldq * 4, s));
  // layer 0 input: z = l2norm(x), operand copies
  agnn_input_launch(x, ldx, NC, d, ldq, prec, set[0][0], set[0][1], set[0][2], set[0][3], set[0][4],
                    norm[0], zeros, s);
  for (uint32_t l = 0; l < L; ++l) {
    const bool last = l + 1 == L;
    float** cur = set[l & 1];
    float** nxt = set[(l + 1) & 1];
    AgnnNext nx{};
    nx.out = last ? out : buf[l & 1];
    nx.ldo = last ? ldo : ldb;
    nx.ldq = ldq;
    nx.zeros = reinterpret_cast<unsigned long long*>(zeros);
    // a NaN/Inf anywhere propagates to the last layer's rows (rows with
    // edges read their own z), so checking the last layer's output suffices
    nx.nonfinite = last ? flag : nullptr;
    if (!last) {
      nx.zq = nxt[1];
      nx.hq = nxt[3];
      if (prec == SGTK_FP32) {  // the FP32 kernels also read raw z, |h| and the lo planes
        nx.z = nxt[0];
        nx.zq1 = nxt[2];
        nx.hq1 = nxt[4];
        nx.norm = norm[(l + 1) & 1];
      } else {
        nx.out = nullptr;  // TF32: the next layer reads only the rounded copies
      }
    }
    agnn_panel_layer(g, cur[0], cur[1], cur[2], cur[3], cur[4], ldq, norm[l & 1], d, betas[l], prec,
                     opart, lpart, seg_o, seg_l, osp, lsp, nx, s);
  }
  finish_agnn(zeros, zero_rows_host, s);
}
}  // namespace

void agnn_forward(const sgtk_graph* g, const float* x, uint64_t ldx, uint64_t d, uint32_t L,
                  const float* betas, const uint32_t* cut, int prec, int mode, void* ws,
                  uint64_t ws_bytes, float* out, uint64_t ldo, uint64_t* zero_rows_host,
                  cudaStream_t s) {
  const uint64_t N = g->n_rows;
  if (ws_bytes < agnn_workspace(g, d)) raise(SGTK_ERR_SHAPE, "agnn_forward: workspace too small");
  char* p = static_cast<char*>(ws);
  const uint64_t ldb = ld4(d);
  float* buf[2];
  buf[0] = reinterpret_cast<float*>(p); p += align256(N * ldb * 4);
  buf[1] = reinterpret_cast<float*>(p); p += align256(N * ldb * 4);
  float* inv = reinterpret_cast<float*>(p); p += align256(g->n_cols * 4);
  float* logits = reinterpret_cast<float*>(p); p += align256(std::max<uint64_t>(g->nnz, 1) * 4);
  float* zbuf = reinterpret_cast<float*>(p); p += align256(g->n_cols * ld4(d) * 4);
  uint64_t* zeros = reinterpret_cast<uint64_t*>(p);
  if (g->n_rows != g->n_cols && L > 1)
    raise(SGTK_ERR_SHAPE, "agnn_forward: a row-slice graph runs one layer per call "
                          "(all-gather the slices between layers)");
  // mode 3 (auto): the panel path for graphs where it wins; below ~2M edges
  // the fused 16-row kernel's single launch per layer is faster (measured:
  // Pubmed-shaped C2 0.010 vs 0.021 ms/layer, Reddit-shaped C4 1.39 vs 0.62)
  if (mode == 3) mode = (g->nnz >= (2ull << 20) || d > 64) ? 2 : 1;
  if (mode == 2) {
    bool ok = !cut && L > 0;
    for (uint32_t l = 0; ok && l < L; ++l) ok = agnn_panel_supported(g, d, betas[l]);
    if (ok) {
      agnn_forward_panel(g, x, ldx, d, L, betas, prec, ws, out, ldo, zero_rows_host, s);
      return;
    }
    mode = d <= 64 ? 1 : 0;  // outside the panel path's envelope: fused 16-row windows, else the chain
  }
  uint32_t* flag = reinterpret_cast<uint32_t*>(zeros + 1);
  CU(cudaMemsetAsync(zeros, 0, 16, s));

  if (L == 0) {
    CU(cudaMemcpy2DAsync(out, ldo * 4, x, ldx * 4, d * 4, N, cudaMemcpyDeviceToDevice, s));
  }
  const float* h = x;
  uint64_t ldh = ldx;
  for (uint32_t l = 0; l < L; ++l) {
    const bool last = l + 1 == L;
    float* dst = last ? out : buf[l & 1];
    const uint64_t ldd = last ? ldo : ldb;
    // first layer of a row-slice graph: the input is the full n_cols-row replica
    if (mode == 1) {
      // z = h * inv_norm materialised (as the reference does, gnn.cpp:109)
      l2norm_launch(h, l == 0 ? g->n_cols : N, d, ldh, zbuf, ldb, inv, zeros, s);
      agnn_fused_launch(g, h, ldh, zbuf, ldb, inv, d, betas[l], prec, cut, dst, ldd, s,
                        last ? flag : nullptr);
    } else {
      l2norm_launch(h, l == 0 ? g->n_cols : N, d, ldh, nullptr, 0, inv, zeros, s);
      // The reference's SDDMM runs on reblock(t, 16) with make_split_plan(t16, ratio)
      // (gnn.cpp:101-102); the 8-wide cut carried over to 16-wide tiles is
      // the same ratio up to floor rounding.
      sddmm_launch(g, h, ldh, h, ldh, d, cut, nullptr, /*unit_values=*/true, prec, inv,
                   betas[l], logits, s);
      edge_softmax_launch(g, logits, logits, s);
      spmm_launch(g, h, ldh, d, cut, logits, prec, dst, ldd, last ? flag : nullptr, s);
    }
    h = dst;
    ldh = ldd;
  }
  finish_agnn(zeros, zero_rows_host, s);
}

}  // namespace sgtkcu
