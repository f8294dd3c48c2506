// C ABI (include/sgtk_cuda.h): argument validation on the host (so the same
// reference exception types surface), then the device
// launchers.  Nothing throws across this boundary.

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.cuh"

using namespace sgtkcu;

namespace sgtkcu {
uint64_t gcn_workspace(const sgtk_graph* g, uint32_t L, const uint64_t* dims);
void gcn_forward(const sgtk_graph* g, const float* x, uint64_t ldx, uint32_t L,
                 const uint64_t* dims, const float* weights, const int* relu,
                 const uint32_t* cut, int prec, int order, void* ws, uint64_t ws_bytes, float* out,
                 uint64_t ldo, cudaStream_t s, uint32_t* nonfinite_dev = nullptr);
uint64_t agnn_workspace(const sgtk_graph* g, uint64_t d);
void agnn_forward(const sgtk_graph* g, const float* x, uint64_t ldx, uint64_t d, uint32_t L,
                  const float* betas, const uint32_t* cut, int prec, int mode, void* ws,
                  uint64_t ws_bytes, float* out, uint64_t ldo, uint64_t* zero_rows_host,
                  cudaStream_t s);
}  // namespace sgtkcu

namespace {

thread_local std::string g_err;

// Stream-ordered scratch (cudaMallocAsync) comes from the device's default
// pool; its default release threshold (0) hands memory back to the driver at
// every synchronisation, turning each call's scratch into a fresh cudaMalloc.
// Keep it cached instead (once per device).
void prepare_device() {
  static std::mutex mu;
  static std::vector<int> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return;
  std::lock_guard<std::mutex> lock(mu);
  for (int d : done)
    if (d == dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = ~uint64_t(0);
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  done.push_back(dev);
}

template <class F>
int guard(F&& f) {
  try {
    prepare_device();
    f();
    return SGTK_OK;
  } catch (const Status& e) {
    g_err = e.what();
    return e.code;
  } catch (const std::bad_alloc&) {
    g_err = "host allocation failed";
    return SGTK_ERR;
  } catch (const std::exception& e) {
    g_err = e.what();
    return SGTK_ERR;
  }
}

void need(bool ok, int code, const char* msg) {
  if (!ok) raise(code, msg);
}

void check_graph(const sgtk_graph* g) { need(g != nullptr, SGTK_ERR, "null graph handle"); }

void check_prec(int p) {
  need(p == SGTK_FP32 || p == SGTK_TF32, SGTK_ERR_RANGE, "precision must be FP32 or TF32");
}

struct Scoped {
  void* p = nullptr;
  cudaStream_t s;
  explicit Scoped(cudaStream_t st) : s(st) {}
  void* get(uint64_t bytes) {
    if (bytes) CU(cudaMallocAsync(&p, bytes, s));
    return p;
  }
  ~Scoped() {
    if (p) cudaFreeAsync(p, s);
  }
};

}  // namespace

extern "C" {

const char* sgtk_last_error(void) { return g_err.c_str(); }
const char* sgtk_version(void) { return "sgtk-b200 0.1.0 (sm_100a)"; }

int sgtk_graph_create(const uint64_t* np, const uint32_t* el, const float* vals, uint64_t n,
                      uint64_t nnz, uint32_t blk_h, uint32_t blk_w, int kind, void* stream,
                      sgtk_graph** out) {
  return guard([&] {
    need(out != nullptr, SGTK_ERR, "null output handle");
    need(np != nullptr && (el != nullptr || nnz == 0), SGTK_ERR, "null CSR array");
    *out = graph_create(np, el, vals, n, n, nnz, blk_h, blk_w, kind, as_stream(stream));
  });
}

int sgtk_graph_create_rows(const uint64_t* np, const uint32_t* el, const float* vals,
                           uint64_t n_rows, uint64_t n_cols, uint64_t row_offset, uint64_t nnz,
                           uint32_t blk_h, uint32_t blk_w, int kind, void* stream,
                           sgtk_graph** out) {
  return guard([&] {
    need(out != nullptr, SGTK_ERR, "null output handle");
    need(row_offset + n_rows <= n_cols, SGTK_ERR_SHAPE, "row slice exceeds the column space");
    *out = graph_create(np, el, vals, n_rows, n_cols, nnz, blk_h, blk_w, kind, as_stream(stream),
                        row_offset);
  });
}

int sgtk_graph_import(const uint64_t* np, const uint32_t* el, const float* vals, uint64_t n,
                      uint64_t nnz, uint32_t blk_h, uint32_t blk_w, const uint32_t* e2c,
                      const uint64_t* wo, const uint32_t* wuc, void* stream, sgtk_graph** out) {
  return guard([&] {
    need(out != nullptr, SGTK_ERR, "null output handle");
    *out = graph_import(np, el, vals, n, nnz, blk_h, blk_w, e2c, wo, wuc, as_stream(stream));
  });
}

int sgtk_graph_import_panels(const uint64_t* np, const uint32_t* el, const float* vals,
                             uint64_t n, uint64_t nnz, uint32_t blk_h, uint32_t blk_w,
                             const uint32_t* e2c, const uint64_t* wo, const uint32_t* wuc,
                             const char* panel_section, void* stream, sgtk_graph** out) {
  return guard([&] {
    need(out != nullptr, SGTK_ERR, "null output handle");
    *out = graph_import(np, el, vals, n, nnz, blk_h, blk_w, e2c, wo, wuc, as_stream(stream),
                        panel_section);
  });
}

int sgtk_graph_save_panels(const sgtk_graph* g, const char* path, void* stream) {
  return guard([&] {
    check_graph(g);
    need(path != nullptr, SGTK_ERR, "null path");
    save_panel_section(*g, path, as_stream(stream));
  });
}

int sgtk_graph_panels_loaded(const sgtk_graph* g, int* loaded) {
  return guard([&] {
    check_graph(g);
    *loaded = g->panels_loaded ? 1 : 0;
  });
}

void sgtk_graph_destroy(sgtk_graph* g) {
  if (g) {
    cudaDeviceSynchronize();
    delete g;
  }
}

int sgtk_graph_info(const sgtk_graph* g, uint64_t info[11]) {
  return guard([&] {
    check_graph(g);
    const uint64_t v[11] = {g->n_rows, g->nnz, g->user.W, g->user.U, g->block_counter, g->blk_h,
                            g->blk_w, g->has_values ? 1u : 0u, g->T8, g->T16, g->plan8.n_units};
    std::memcpy(info, v, sizeof v);
  });
}

int sgtk_graph_build_times(const sgtk_graph* g, double ms[8]) {
  return guard([&] {
    check_graph(g);
    std::memcpy(ms, g->build_ms, sizeof g->build_ms);
  });
}

int sgtk_panel_info_for(const sgtk_graph* g, uint64_t d, uint64_t info[8]) {
  return guard([&] {
    check_graph(g);
    const auto& p = sgtkcu::panels_for(g, d);
    const uint64_t v[8] = {p.P, p.n_chunks, p.n_dent, p.n_sparse, p.max_chunk_entries,
                           p.n_chunks * 32, p.n_long, p.n_segs};
    std::memcpy(info, v, sizeof v);
  });
}

int sgtk_panel_info(const sgtk_graph* g, uint64_t info[8]) {
  return guard([&] {
    check_graph(g);
    const auto& p = *g->panels;
    const uint64_t v[8] = {p.P, p.n_chunks, p.n_dent, p.n_sparse, p.max_chunk_entries,
                           p.n_chunks * 32, p.n_long, p.n_segs};
    std::memcpy(info, v, sizeof v);
  });
}

int sgtk_debug_set(int mode) {
  return guard([&] { sgtkcu::panel_debug_set(mode); });
}

int sgtk_panel_download(const sgtk_graph* g, uint32_t* chunk_ptr, uint32_t* dense_cols,
                        uint64_t* chunk_off, uint32_t* dense_entries, uint32_t* sparse_ptr,
                        uint32_t* sparse_entries) {
  return guard([&] {
    check_graph(g);
    const auto& p = *g->panels;
    auto get = [](void* dst, const sgtkcu::DevBuf& src, size_t bytes) {
      if (dst && bytes) CU(cudaMemcpy(dst, src.p, bytes, cudaMemcpyDeviceToHost));
    };
    get(chunk_ptr, *p.cptr, (p.P + 1) * 4);
    get(dense_cols, *p.dcols, p.n_chunks * 32 * 4);
    get(chunk_off, *p.coff, (p.n_chunks + 1) * 8);
    get(dense_entries, *p.dent, p.n_dent * 4);
    get(sparse_ptr, *p.sptr, (g->n_rows + 1) * 4);
    get(sparse_entries, *p.sent, p.n_sparse * 8);
  });
}

int sgtk_graph_device_ptrs(const sgtk_graph* g, const void* ptrs[8]) {
  return guard([&] {
    check_graph(g);
    ptrs[0] = g->np->p;
    ptrs[1] = g->el->p;
    ptrs[2] = g->has_values ? g->vals->p : nullptr;
    ptrs[3] = g->e2r->p;
    ptrs[4] = g->user.e2c->p;
    ptrs[5] = g->bp->p;
    ptrs[6] = g->user.wo->p;
    ptrs[7] = g->user.wuc->p;
  });
}

int sgtk_graph_download(const sgtk_graph* g, uint32_t* e2r, uint32_t* e2c, uint32_t* bp,
                        uint64_t* wo, uint32_t* wuc) {
  return guard([&] {
    check_graph(g);
    if (e2r && g->nnz) CU(cudaMemcpy(e2r, g->e2r->p, g->nnz * 4, cudaMemcpyDeviceToHost));
    if (e2c && g->nnz) CU(cudaMemcpy(e2c, g->user.e2c->p, g->nnz * 4, cudaMemcpyDeviceToHost));
    if (bp && !g->bp_host.empty()) std::memcpy(bp, g->bp_host.data(), g->bp_host.size() * 4);
    if (wo) std::memcpy(wo, g->user.wo_host.data(), g->user.wo_host.size() * 8);
    if (wuc && g->user.U) CU(cudaMemcpy(wuc, g->user.wuc->p, g->user.U * 4, cudaMemcpyDeviceToHost));
  });
}

int sgtk_graph_reblock(const sgtk_graph* g, uint32_t blk_w, void* stream, sgtk_graph** out) {
  return guard([&] {
    check_graph(g);
    *out = graph_reblock(g, blk_w, as_stream(stream));
  });
}

int sgtk_block_stats(const sgtk_graph* g, uint64_t stats[3], double* density) {
  return guard([&] {
    check_graph(g);
    stats[0] = g->block_counter;
    stats[1] = g->block_counter * g->blk_h * g->blk_w;
    stats[2] = g->nnz;
    if (density) *density = stats[1] ? double(stats[2]) / double(stats[1]) : 0.0;
  });
}

int sgtk_split_plan(const sgtk_graph* g, double ratio, uint32_t* cut) {
  return guard([&] {
    check_graph(g);
    auto c = split_plan_host(g, ratio);
    if (!c.empty()) std::memcpy(cut, c.data(), c.size() * 4);
  });
}

// gather_tile (tile_exec.cpp:163-198) from the resident fields.
int sgtk_gather_tile(const sgtk_graph* g, uint64_t window, uint64_t tile, float* a_tile,
                     uint32_t* x_index) {
  return guard([&] {
    check_graph(g);
    need(window < g->user.W, SGTK_ERR_INDEX, "gather_tile: window out of range");
    need(tile < g->bp_host[window], SGTK_ERR_INDEX, "gather_tile: tile out of range");
    const uint64_t bh = g->blk_h, bw = g->blk_w, base = tile * bw;
    const uint64_t u0 = g->user.wo_host[window], ucnt = g->user.wo_host[window + 1] - u0;
    std::vector<uint32_t> cols(ucnt);
    if (ucnt) CU(cudaMemcpy(cols.data(), g->user.wuc->as<uint32_t>() + u0, ucnt * 4, cudaMemcpyDeviceToHost));
    for (uint64_t c = 0; c < bw; ++c) x_index[c] = base + c < ucnt ? cols[base + c] : uint32_t(g->n_cols);
    std::fill(a_tile, a_tile + bh * bw, 0.0f);
    const uint64_t r0 = window * bh, r1 = std::min(g->n_rows, r0 + bh);
    std::vector<uint64_t> np(r1 - r0 + 1);
    CU(cudaMemcpy(np.data(), g->np->as<uint64_t>() + r0, np.size() * 8, cudaMemcpyDeviceToHost));
    const uint64_t e0 = np.front(), e1 = np.back();
    std::vector<uint32_t> e2c(e1 - e0);
    std::vector<float> vals(e1 - e0, 1.0f);
    if (e1 > e0) {
      CU(cudaMemcpy(e2c.data(), g->user.e2c->as<uint32_t>() + e0, (e1 - e0) * 4, cudaMemcpyDeviceToHost));
      if (g->has_values)
        CU(cudaMemcpy(vals.data(), g->vals->as<float>() + e0, (e1 - e0) * 4, cudaMemcpyDeviceToHost));
    }
    for (uint64_t r = r0; r < r1; ++r)
      for (uint64_t e = np[r - r0]; e < np[r - r0 + 1]; ++e) {
        const uint32_t c = e2c[e - e0];
        if (c >= base && c < base + bw) a_tile[(r - r0) * bw + (c - base)] = vals[e - e0];
      }
  });
}

int sgtk_spmm(const sgtk_graph* g, const float* x, uint64_t ldx, uint64_t d, const uint32_t* cut,
              const float* ev, int prec, float* out, uint64_t ldo, uint32_t* nonfinite,
              void* stream) {
  return guard([&] {
    check_graph(g);
    check_prec(prec);
    spmm_launch(g, x, ldx, d, cut, ev, prec, out, ldo, nonfinite, as_stream(stream));
  });
}

int sgtk_sddmm(const sgtk_graph* g, const float* x, uint64_t ldx, const float* y, uint64_t ldy,
               uint64_t d, const uint32_t* cut16, const float* ev, int prec, float scale,
               float* out, void* stream) {
  return guard([&] {
    check_graph(g);
    check_prec(prec);
    sddmm_launch(g, x, ldx, y, ldy, d, cut16, ev, false, prec, nullptr, scale, out,
                 as_stream(stream));
  });
}

int sgtk_edge_softmax(const sgtk_graph* g, const float* logits, float* out, void* stream) {
  return guard([&] {
    check_graph(g);
    edge_softmax_launch(g, logits, out, as_stream(stream));
  });
}

int sgtk_relu_inplace(float* x, uint64_t rows, uint64_t cols, uint64_t ld, void* stream) {
  return guard([&] { relu_nonfinite_launch(x, rows, cols, ld, 1, nullptr, as_stream(stream)); });
}

int sgtk_csr_softmax(const uint64_t* np, uint64_t n, const float* logits, float* out,
                     void* stream) {
  return guard([&] { csr_softmax_launch(np, n, logits, out, as_stream(stream)); });
}

int sgtk_l2_normalize_rows(const float* h, uint64_t rows, uint64_t cols, uint64_t ldh, float* z,
                           uint64_t ldz, float* inv, uint64_t* zeros, void* stream) {
  return guard([&] { l2norm_launch(h, rows, cols, ldh, z, ldz, inv, zeros, as_stream(stream)); });
}

int sgtk_gemm(const float* a, uint64_t lda, const float* w, uint64_t m, uint64_t k, uint64_t n,
              int relu, int prec, float* out, uint64_t ldo, void* stream) {
  return guard([&] {
    check_prec(prec);
    need(lda >= k && ldo >= n, SGTK_ERR_SHAPE, "gemm: leading dimension too small");
    gemm_launch(a, lda, w, m, k, n, relu, prec, out, ldo, as_stream(stream));
  });
}

uint64_t sgtk_gcn_workspace(const sgtk_graph* g, uint32_t L, const uint64_t* dims) {
  return g && L ? gcn_workspace(g, L, dims) : 0;
}
uint64_t sgtk_agnn_workspace(const sgtk_graph* g, uint64_t d) {
  return g ? agnn_workspace(g, d) : 0;
}

int sgtk_gcn_forward(const sgtk_graph* g, const float* x, uint64_t ldx, uint32_t L,
                     const uint64_t* dims, const float* weights, const int* relu,
                     const uint32_t* cut, int prec, int order, void* ws, uint64_t ws_bytes,
                     float* out, uint64_t ldo, void* stream) {
  return guard([&] {
    check_graph(g);
    check_prec(prec);
    gcn_forward(g, x, ldx, L, dims, weights, relu, cut, prec, order, ws, ws_bytes, out, ldo,
                as_stream(stream), nullptr);
  });
}

int sgtk_gcn_forward_async(const sgtk_graph* g, const float* x, uint64_t ldx, uint32_t L,
                           const uint64_t* dims, const float* weights, const int* relu,
                           const uint32_t* cut, int prec, int order, void* ws, uint64_t ws_bytes,
                           float* out, uint64_t ldo, uint32_t* nonfinite, void* stream) {
  return guard([&] {
    check_graph(g);
    check_prec(prec);
    need(nonfinite != nullptr, SGTK_ERR, "null nonfinite flag");
    gcn_forward(g, x, ldx, L, dims, weights, relu, cut, prec, order, ws, ws_bytes, out, ldo,
                as_stream(stream), nonfinite);
  });
}

int sgtk_agnn_forward(const sgtk_graph* g, const float* x, uint64_t ldx, uint64_t d, uint32_t L,
                      const float* betas, const uint32_t* cut, int prec, int mode, void* ws,
                      uint64_t ws_bytes, float* out, uint64_t ldo, uint64_t* zero_rows,
                      void* stream) {
  return guard([&] {
    check_graph(g);
    check_prec(prec);
    agnn_forward(g, x, ldx, d, L, betas, cut, prec, mode, ws, ws_bytes, out, ldo, zero_rows,
                 as_stream(stream));
  });
}

int sgtk_gcn_normalize_values(const uint64_t* np, const uint32_t* el, uint64_t n, float* vals,
                              void* stream) {
  return guard([&] { gcn_normalize_launch(np, el, n, vals, as_stream(stream)); });
}

int sgtk_normalize_graph(const uint64_t* np, const uint32_t* el, const float* vals, uint64_t n,
                         uint64_t nnz, int symmetrize, int loops, int dedupe, int kind,
                         void* stream, sgtk_csr** out) {
  return guard([&] {
    need(out != nullptr && np != nullptr, SGTK_ERR, "null argument");
    *out = normalize_graph(np, el, vals, n, nnz, symmetrize, loops, dedupe, kind,
                           as_stream(stream));
  });
}

int sgtk_csr_info(const sgtk_csr* c, uint64_t info[3]) {
  return guard([&] {
    need(c != nullptr, SGTK_ERR, "null csr handle");
    info[0] = c->n;
    info[1] = c->nnz;
    info[2] = c->has_values ? 1 : 0;
  });
}

int sgtk_csr_download(const sgtk_csr* c, uint64_t* np, uint32_t* el, float* vals) {
  return guard([&] {
    need(c != nullptr, SGTK_ERR, "null csr handle");
    if (np) CU(cudaMemcpy(np, c->np.p, (c->n + 1) * 8, cudaMemcpyDeviceToHost));
    if (el && c->nnz) CU(cudaMemcpy(el, c->el.p, c->nnz * 4, cudaMemcpyDeviceToHost));
    if (vals && c->has_values && c->nnz)
      CU(cudaMemcpy(vals, c->vals.p, c->nnz * 4, cudaMemcpyDeviceToHost));
  });
}

int sgtk_csr_device_ptrs(const sgtk_csr* c, const void* ptrs[3]) {
  return guard([&] {
    need(c != nullptr, SGTK_ERR, "null csr handle");
    ptrs[0] = c->np.p;
    ptrs[1] = c->el.p;
    ptrs[2] = c->has_values ? c->vals.p : nullptr;
  });
}

void sgtk_csr_destroy(sgtk_csr* c) {
  if (c) {
    cudaDeviceSynchronize();
    delete c;
  }
}

int sgtk_tf32_round(const float* in, float* out, uint64_t n, void* stream) {
  return guard([&] { tf32_launch(in, out, n, as_stream(stream)); });
}

// ---- host-buffer end-to-end entry points ---------------------------------
int sgtk_gcn_forward_host(const sgtk_graph* g, const float* x_host, uint32_t L,
                          const uint64_t* dims, const float* w_host, const int* relu,
                          double ratio, int prec, float* out_host, void* stream) {
  return guard([&] {
    check_graph(g);
    check_prec(prec);
    cudaStream_t s = as_stream(stream);
    const uint64_t N = g->n_rows;
    uint64_t wn = 0;
    for (uint32_t l = 0; l < L; ++l) wn += dims[l] * dims[l + 1];
    const uint64_t ws = gcn_workspace(g, L, dims);
    const uint64_t xb = N * dims[0] * 4, ob = N * dims[L] * 4;
    std::vector<uint32_t> cut = ratio >= 1.0 ? std::vector<uint32_t>() : split_plan_host(g, ratio);
    Scoped m(s);
    char* p = static_cast<char*>(m.get(ws + xb + ob + wn * 4 + cut.size() * 4 + 1024));
    char* xd = p + ws;
    char* od = (char*)(((uintptr_t)(xd + xb) + 255) & ~uintptr_t(255));
    char* wd = (char*)(((uintptr_t)(od + ob) + 255) & ~uintptr_t(255));
    char* cd = (char*)(((uintptr_t)(wd + wn * 4) + 255) & ~uintptr_t(255));
    CU(cudaMemcpyAsync(xd, x_host, xb, cudaMemcpyHostToDevice, s));
    CU(cudaMemcpyAsync(wd, w_host, wn * 4, cudaMemcpyHostToDevice, s));
    if (!cut.empty()) CU(cudaMemcpyAsync(cd, cut.data(), cut.size() * 4, cudaMemcpyHostToDevice, s));
    gcn_forward(g, reinterpret_cast<float*>(xd), dims[0], L, dims, reinterpret_cast<float*>(wd),
                relu, cut.empty() ? nullptr : reinterpret_cast<uint32_t*>(cd), prec, 2, p, ws,
                reinterpret_cast<float*>(od), dims[L], s);
    CU(cudaMemcpyAsync(out_host, od, ob, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
  });
}

int sgtk_agnn_forward_host(const sgtk_graph* g, const float* x_host, uint64_t d, uint32_t L,
                           const float* betas, double ratio, int prec, int mode, float* out_host,
                           uint64_t* zero_rows, void* stream) {
  return guard([&] {
    check_graph(g);
    check_prec(prec);
    cudaStream_t s = as_stream(stream);
    const uint64_t N = g->n_rows;
    const uint64_t ws = agnn_workspace(g, d);
    const uint64_t xb = N * d * 4;
    std::vector<uint32_t> cut = ratio >= 1.0 ? std::vector<uint32_t>() : split_plan_host(g, ratio);
    Scoped m(s);
    char* p = static_cast<char*>(m.get(ws + 2 * xb + cut.size() * 4 + 1024));
    char* xd = p + ws;
    char* od = (char*)(((uintptr_t)(xd + xb) + 255) & ~uintptr_t(255));
    char* cd = (char*)(((uintptr_t)(od + xb) + 255) & ~uintptr_t(255));
    CU(cudaMemcpyAsync(xd, x_host, xb, cudaMemcpyHostToDevice, s));
    if (!cut.empty()) CU(cudaMemcpyAsync(cd, cut.data(), cut.size() * 4, cudaMemcpyHostToDevice, s));
    uint64_t zr = 0;  // the host entry always reports NaN/Inf (NonFiniteError)
    agnn_forward(g, reinterpret_cast<float*>(xd), d, d, L, betas,
                 cut.empty() ? nullptr : reinterpret_cast<uint32_t*>(cd), prec, mode, p, ws,
                 reinterpret_cast<float*>(od), d, zero_rows ? zero_rows : &zr, s);
    CU(cudaMemcpyAsync(out_host, od, xb, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
  });
}

int sgtk_spmm_host(const sgtk_graph* g, const float* x_host, uint64_t d, double ratio, int prec,
                   const float* ev_host, float* out_host, void* stream) {
  return guard([&] {
    check_graph(g);
    check_prec(prec);
    cudaStream_t s = as_stream(stream);
    const uint64_t N = g->n_rows, xb = g->n_cols * d * 4, ob = N * d * 4, eb = ev_host ? g->nnz * 4 : 0;
    std::vector<uint32_t> cut = ratio >= 1.0 ? std::vector<uint32_t>() : split_plan_host(g, ratio);
    Scoped m(s);
    char* p = static_cast<char*>(m.get(xb + ob + eb + cut.size() * 4 + 1024 + 4));
    char* xd = p;
    char* od = (char*)(((uintptr_t)(xd + xb) + 255) & ~uintptr_t(255));
    char* ed = (char*)(((uintptr_t)(od + ob) + 255) & ~uintptr_t(255));
    char* cd = (char*)(((uintptr_t)(ed + eb) + 255) & ~uintptr_t(255));
    uint32_t* flag = reinterpret_cast<uint32_t*>(cd + cut.size() * 4);
    CU(cudaMemsetAsync(flag, 0, 4, s));
    CU(cudaMemcpyAsync(xd, x_host, xb, cudaMemcpyHostToDevice, s));
    if (eb) CU(cudaMemcpyAsync(ed, ev_host, eb, cudaMemcpyHostToDevice, s));
    if (!cut.empty()) CU(cudaMemcpyAsync(cd, cut.data(), cut.size() * 4, cudaMemcpyHostToDevice, s));
    spmm_launch(g, reinterpret_cast<float*>(xd), d, d,
                cut.empty() ? nullptr : reinterpret_cast<uint32_t*>(cd),
                eb ? reinterpret_cast<float*>(ed) : nullptr, prec, reinterpret_cast<float*>(od), d,
                flag, s);
    uint32_t hf = 0;
    CU(cudaMemcpyAsync(out_host, od, ob, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(&hf, flag, 4, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    if (hf) raise(SGTK_ERR_NONFINITE, "spmm_hybrid: output contains NaN or Inf");
  });
}

int sgtk_partition_windows(const uint64_t* np, uint64_t n, uint32_t blk_h, uint32_t parts,
                           uint64_t* bounds) {
  return guard([&] {
    need(blk_h > 0, SGTK_ERR_GEOMETRY, "tile dimensions must be positive");
    need(parts > 0, SGTK_ERR_RANGE, "parts must be positive");
    const uint64_t W = (n + blk_h - 1) / blk_h;
    const uint64_t E = np[n];
    bounds[0] = 0;
    uint64_t w = 0;
    for (uint32_t p = 1; p < parts; ++p) {
      // first window whose start edge reaches p/parts of the edges (+ rows as
      // a tie-break weight so empty graphs still split by rows)
      const double target = double(E + n) * p / parts;
      while (w < W && double(np[std::min(n, w * blk_h)] + std::min(n, w * blk_h)) < target) ++w;
      bounds[p] = std::max(w, bounds[p - 1]);
    }
    bounds[parts] = W;
  });
}

}  // extern "C"
