// TEST INFRASTRUCTURE ONLY — the CPU oracle.  Nothing in the product path
// (paper_2412_12218_b200/) may link, load or call this file; only tests/,
// __graft_entry__.smoke() and bench.py's cpu_baseline leg use it, and only as
// the checker / the reported CPU baseline.
//
// A restatement, in plain arrays, of the reference's algorithms for the hot
// path (/root/reference/proj).  Pinned against golden vectors produced by the
// reference itself (tests/golden/, made by tests/golden/make_golden.py through
// oracle/_ref), see tests/test_oracle_golden.py.
//
// Arithmetic contract: every float result is produced in the
// same order and with the same rounding as the reference, so the oracle is
// bit-identical to it on the same host:
//   * SpMM: per output element, products a_e * x[col_e][k] rounded to fp32 and
//     added in CSR edge order starting from +0 (tile_exec.cpp:60-127,291-303
//     visit unique columns ascending == CSR order), no FMA.
//   * SDDMM: k-ascending fp32 dot, then a_e * dot (tile_exec.cpp:369-408).
//   * TF32: RNE to 10 mantissa bits with saturation (tile_exec.cpp:131-142);
//     applied to both multiplicands of SpMM and to a and dot in SDDMM.
//   * softmax: fp32 max, expf(l - max), sequential fp32 sum, divide
//     (gnn.cpp:54-72).  l2norm: fp64 sum of squares, float(1/sqrt) (gnn.cpp:74-91).
//   * dense update: ikj fp32 product (gnn.cpp:16-29).
// Compiled with -ffp-contract=off (oracle/Makefile).

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <random>
#include <string>
#include <vector>

namespace {

thread_local std::string g_msg;

// Status codes (include/sgtk_cuda.h).
enum : int {
  kOk = 0, kErr = 1, kDegree = 5, kGeometry = 6, kIndex = 7, kRange = 8,
  kShape = 9, kNonFinite = 10,
};

int fail(int code, const char* msg) {
  g_msg = msg;
  return code;
}

inline uint32_t fbits(float v) {
  uint32_t u;
  std::memcpy(&u, &v, 4);
  return u;
}
inline float bitsf(uint32_t u) {
  float v;
  std::memcpy(&v, &u, 4);
  return v;
}

// tile_exec.cpp:131-142
inline float tf32(float v) {
  uint32_t u = fbits(v);
  const uint32_t exp_mask = 0x7F800000u;
  if ((u & exp_mask) == exp_mask) return v;  // inf / nan unchanged
  const uint32_t lsb = (u >> 13) & 1u;       // ties to even on bit 13
  u = (u + 0x0FFFu + lsb) & 0xFFFFE000u;
  if ((u & exp_mask) == exp_mask) u = (u & 0x80000000u) | 0x7F7FE000u;
  return bitsf(u);
}

inline float rnd(float v, bool tf) { return tf ? tf32(v) : v; }

}  // namespace

extern "C" {

const char* or_last_error() { return g_msg.c_str(); }

float or_tf32_round_value(float v) { return tf32(v); }

// csr_graph.cpp:10-39
int or_validate_csr(uint64_t n, const uint64_t* np, const uint32_t* el,
                    const float* vals, uint64_t nnz, int sorted_unique) {
  if (np[0] != 0) return fail(kErr, "csr: node_pointer[0] != 0");
  if (np[n] != nnz) return fail(kErr, "csr: node_pointer end != edge count");
  for (uint64_t i = 0; i < n; ++i)
    if (np[i] > np[i + 1]) return fail(kErr, "csr: node_pointer decreases");
  for (uint64_t e = 0; e < nnz; ++e)
    if (el[e] >= n) return fail(kErr, "csr: column id out of range");
  if (sorted_unique)
    for (uint64_t r = 0; r < n; ++r)
      for (uint64_t e = np[r] + 1; e < np[r + 1]; ++e)
        if (el[e - 1] >= el[e]) return fail(kErr, "csr: columns not ascending");
  if (vals)
    for (uint64_t e = 0; e < nnz; ++e)
      if (!std::isfinite(vals[e])) return fail(kErr, "csr: non-finite value");
  return kOk;
}

// Window pass 1: unique count per window (sgt_transform.cpp:37-49).  Returns
// the per-window unique counts in `ucount[W]`.
int or_sgt_count(uint64_t n, const uint64_t* np, const uint32_t* el,
                 uint32_t blk_h, uint32_t* ucount) {
  if (blk_h == 0) return fail(kGeometry, "tile dimensions must be positive");
  const uint64_t W = (n + blk_h - 1) / blk_h;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t w = 0; w < int64_t(W); ++w) {
    const uint64_t lo = np[uint64_t(w) * blk_h];
    const uint64_t hi = np[std::min<uint64_t>(n, uint64_t(w + 1) * blk_h)];
    std::vector<uint32_t> c(el + lo, el + hi);
    std::sort(c.begin(), c.end());
    ucount[w] = uint32_t(std::unique(c.begin(), c.end()) - c.begin());
  }
  return kOk;
}

// Window pass 2: sorted uniques + per-edge (row, rank) (sgt_transform.cpp:51-75).
// wo[W+1] must already hold the exclusive scan of the unique counts.
int or_sgt_fill(uint64_t n, const uint64_t* np, const uint32_t* el,
                uint32_t blk_h, uint32_t blk_w, const uint64_t* wo,
                uint32_t* e2r, uint32_t* e2c, uint32_t* bp, uint32_t* wuc) {
  if (blk_h == 0 || blk_w == 0)
    return fail(kGeometry, "tile dimensions must be positive");
  const uint64_t W = (n + blk_h - 1) / blk_h;
#pragma omp parallel for schedule(dynamic, 64)
  for (int64_t w = 0; w < int64_t(W); ++w) {
    const uint64_t r0 = uint64_t(w) * blk_h;
    const uint64_t r1 = std::min<uint64_t>(n, r0 + blk_h);
    uint32_t* u = wuc + wo[w];
    const uint64_t cnt = wo[w + 1] - wo[w];
    {
      std::vector<uint32_t> c(el + np[r0], el + np[r1]);
      std::sort(c.begin(), c.end());
      std::unique(c.begin(), c.end());
      std::copy(c.begin(), c.begin() + cnt, u);
    }
    bp[w] = uint32_t((cnt + blk_w - 1) / blk_w);
    for (uint64_t r = r0; r < r1; ++r)
      for (uint64_t e = np[r]; e < np[r + 1]; ++e) {
        e2r[e] = uint32_t(r);
        e2c[e] = uint32_t(std::lower_bound(u, u + cnt, el[e]) - u);
      }
  }
  return kOk;
}

// reblock (sgt_transform.cpp:79-91): tiles per window at a new width.
int or_reblock(uint64_t W, const uint64_t* wo, uint32_t blk_w, uint32_t* bp,
               uint64_t* block_counter) {
  if (blk_w == 0) return fail(kGeometry, "tile width must be positive");
  uint64_t total = 0;
  for (uint64_t w = 0; w < W; ++w) {
    bp[w] = uint32_t((wo[w + 1] - wo[w] + blk_w - 1) / blk_w);
    total += bp[w];
  }
  *block_counter = total;
  return kOk;
}

// make_split_plan (tile_exec.cpp:150-161)
int or_split_plan(uint64_t W, const uint32_t* bp, double ratio, uint32_t* cut) {
  if (!(ratio >= 0.0 && ratio <= 1.0))
    return fail(kRange, "split ratio must be within [0, 1]");
  for (uint64_t w = 0; w < W; ++w)
    cut[w] = uint32_t(std::floor(ratio * double(bp[w])));
  return kOk;
}

// SpMM (spmm_hybrid / oracle_spmm): out[n x d] = A x; vals may be null (1.0).
int or_spmm(uint64_t n, const uint64_t* np, const uint32_t* el,
            const float* vals, const float* x, uint64_t d, int tf_mode,
            float* out) {
  const bool tf = tf_mode != 0;
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(| : bad)
  for (int64_t r = 0; r < int64_t(n); ++r) {
    float* o = out + uint64_t(r) * d;
    for (uint64_t k = 0; k < d; ++k) o[k] = 0.0f;
    for (uint64_t e = np[r]; e < np[r + 1]; ++e) {
      const float a = rnd(vals ? vals[e] : 1.0f, tf);
      const float* xr = x + uint64_t(el[e]) * d;
      for (uint64_t k = 0; k < d; ++k) {
        const float p = a * rnd(xr[k], tf);
        o[k] = o[k] + p;
      }
    }
    for (uint64_t k = 0; k < d; ++k) bad |= !std::isfinite(o[k]);
  }
  if (bad) return fail(kNonFinite, "spmm_hybrid: output contains NaN or Inf");
  return kOk;
}

// SDDMM: out[e] = a_e * <x[row(e)], y[col(e)]>
int or_sddmm(uint64_t n, const uint64_t* np, const uint32_t* el,
             const float* vals, const float* x, const float* y, uint64_t d,
             int tf_mode, float* out) {
  const bool tf = tf_mode != 0;
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t r = 0; r < int64_t(n); ++r) {
    const float* xr = x + uint64_t(r) * d;
    for (uint64_t e = np[r]; e < np[r + 1]; ++e) {
      const float* yc = y + uint64_t(el[e]) * d;
      float dot = 0.0f;
      for (uint64_t k = 0; k < d; ++k) {
        const float p = rnd(xr[k], tf) * rnd(yc[k], tf);
        dot = dot + p;
      }
      const float a = vals ? vals[e] : 1.0f;
      out[e] = tf ? tf32(a) * tf32(dot) : a * dot;
    }
  }
  return kOk;
}

// edge_softmax (gnn.cpp:54-72)
int or_edge_softmax(uint64_t n, const uint64_t* np, const float* logits,
                    float* out) {
#pragma omp parallel for schedule(dynamic, 256)
  for (int64_t r = 0; r < int64_t(n); ++r) {
    const uint64_t lo = np[r], hi = np[r + 1];
    if (lo == hi) continue;
    float mx = logits[lo];
    for (uint64_t e = lo + 1; e < hi; ++e) mx = std::max(mx, logits[e]);
    float sum = 0.0f;
    for (uint64_t e = lo; e < hi; ++e) {
      out[e] = std::exp(logits[e] - mx);
      sum = sum + out[e];
    }
    for (uint64_t e = lo; e < hi; ++e) out[e] = out[e] / sum;
  }
  return kOk;
}

// l2_normalize_rows (gnn.cpp:74-91)
int or_l2_normalize_rows(uint64_t rows, uint64_t cols, const float* m,
                         float* out, uint64_t* zeros) {
  uint64_t z = 0;
#pragma omp parallel for schedule(static) reduction(+ : z)
  for (int64_t i = 0; i < int64_t(rows); ++i) {
    const float* s = m + uint64_t(i) * cols;
    float* o = out + uint64_t(i) * cols;
    double sq = 0.0;
    for (uint64_t k = 0; k < cols; ++k) sq += double(s[k]) * double(s[k]);
    if (sq == 0.0) {
      ++z;
      for (uint64_t k = 0; k < cols; ++k) o[k] = 0.0f;
      continue;
    }
    const float inv = float(1.0 / std::sqrt(sq));
    for (uint64_t k = 0; k < cols; ++k) o[k] = s[k] * inv;
  }
  if (zeros) *zeros = z;
  return kOk;
}

// Dense update (gnn.cpp:16-29): out[m x p] = a[m x k] b[k x p], ikj order.
int or_matmul(uint64_t m, uint64_t k, uint64_t p, const float* a,
              const float* b, int relu, float* out) {
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < int64_t(m); ++i) {
    float* o = out + uint64_t(i) * p;
    for (uint64_t j = 0; j < p; ++j) o[j] = 0.0f;
    const float* ai = a + uint64_t(i) * k;
    for (uint64_t kk = 0; kk < k; ++kk) {
      const float v = ai[kk];
      const float* bk = b + kk * p;
      for (uint64_t j = 0; j < p; ++j) {
        const float t = v * bk[j];
        o[j] = o[j] + t;
      }
    }
    if (relu)
      for (uint64_t j = 0; j < p; ++j) o[j] = o[j] > 0.0f ? o[j] : 0.0f;
  }
  return kOk;
}

// gcn_forward (gnn.cpp:33-52): per layer h <- relu?(spmm(A, h) W).
int or_gcn_forward(uint64_t n, const uint64_t* np, const uint32_t* el,
                   const float* vals, const float* x, uint32_t nlayers,
                   const uint64_t* dims, const float* weights, const int* relu,
                   int tf_mode, float* out) {
  std::vector<float> h(x, x + n * dims[0]), agg, next;
  const float* w = weights;
  for (uint32_t l = 0; l < nlayers; ++l) {
    agg.assign(n * dims[l], 0.0f);
    int rc = or_spmm(n, np, el, vals, h.data(), dims[l], tf_mode, agg.data());
    if (rc) return rc;
    next.assign(n * dims[l + 1], 0.0f);
    or_matmul(n, dims[l], dims[l + 1], agg.data(), w, relu[l], next.data());
    w += dims[l] * dims[l + 1];
    h.swap(next);
  }
  for (float v : h)
    if (!std::isfinite(v))
      return fail(kNonFinite, "gcn_forward: output contains NaN or Inf");
  std::copy(h.begin(), h.end(), out);
  return kOk;
}

// agnn_forward (gnn.cpp:93-119): per layer z = l2norm(h); logits =
// beta * sddmm(z, z, unit); attn = softmax_row(logits); h = spmm(attn, h).
int or_agnn_forward(uint64_t n, const uint64_t* np, const uint32_t* el,
                    const float* x, uint64_t d, uint32_t nlayers,
                    const float* betas, int tf_mode, float* out,
                    uint64_t* zero_rows) {
  const uint64_t E = np[n];
  std::vector<float> h(x, x + n * d), z(n * d), logits(E), attn(E),
      next(n * d);
  uint64_t zeros_total = 0;
  for (uint32_t l = 0; l < nlayers; ++l) {
    uint64_t zeros = 0;
    or_l2_normalize_rows(n, d, h.data(), z.data(), &zeros);
    zeros_total += zeros;
    or_sddmm(n, np, el, nullptr, z.data(), z.data(), d, tf_mode,
             logits.data());
    for (float& v : logits) v = v * betas[l];
    or_edge_softmax(n, np, logits.data(), attn.data());
    int rc = or_spmm(n, np, el, attn.data(), h.data(), d, tf_mode, next.data());
    if (rc) return rc;
    h.swap(next);
  }
  if (zero_rows) *zero_rows = zeros_total;
  std::copy(h.begin(), h.end(), out);
  return kOk;
}

// gcn_normalize_values (graph_io.cpp:261-277)
int or_gcn_normalize_values(uint64_t n, const uint64_t* np, const uint32_t* el,
                            float* vals_out) {
  std::vector<double> isd(n);
  for (uint64_t i = 0; i < n; ++i) {
    const uint64_t deg = np[i + 1] - np[i];
    if (deg == 0) return fail(kDegree, "row has no edges");
    isd[i] = 1.0 / std::sqrt(double(deg));
  }
  for (uint64_t i = 0; i < n; ++i)
    for (uint64_t e = np[i]; e < np[i + 1]; ++e)
      vals_out[e] = float(isd[i] * isd[el[e]]);
  return kOk;
}

// normalize_graph (graph_io.cpp:195-259).  Two-call protocol: with
// out_np == nullptr it returns the output edge count in *out_nnz; then call
// again with buffers.  vals/out_vals may be null (unweighted).
int or_normalize_graph(uint64_t n, const uint64_t* np, const uint32_t* el,
                       const float* vals, int symmetrize, int loops,
                       int dedupe, uint64_t* out_nnz, uint64_t* out_np,
                       uint32_t* out_el, float* out_vals) {
  struct T {
    uint32_t r, c;
    float v;
  };
  std::vector<T> t;
  t.reserve(np[n]);
  for (uint64_t r = 0; r < n; ++r)
    for (uint64_t e = np[r]; e < np[r + 1]; ++e)
      t.push_back({uint32_t(r), el[e], vals ? vals[e] : 1.0f});
  auto less = [](const T& a, const T& b) {
    return a.r != b.r ? a.r < b.r : a.c < b.c;
  };
  std::stable_sort(t.begin(), t.end(), less);
  if (dedupe) {
    std::vector<T> u;
    u.reserve(t.size());
    for (const T& x : t) {
      if (!u.empty() && u.back().r == x.r && u.back().c == x.c)
        u.back().v = u.back().v + x.v;
      else
        u.push_back(x);
    }
    t.swap(u);
  }
  auto has = [&](uint32_t r, uint32_t c) {
    auto it = std::lower_bound(t.begin(), t.end(), T{r, c, 0.0f}, less);
    return it != t.end() && it->r == r && it->c == c;
  };
  std::vector<T> add;
  if (symmetrize) {
    for (size_t i = 0; i < t.size(); ++i) {
      if (i && t[i].r == t[i - 1].r && t[i].c == t[i - 1].c) continue;
      if (t[i].r != t[i].c && !has(t[i].c, t[i].r))
        add.push_back({t[i].c, t[i].r, t[i].v});
    }
  }
  if (loops)
    for (uint64_t i = 0; i < n; ++i)
      if (!has(uint32_t(i), uint32_t(i)))
        add.push_back({uint32_t(i), uint32_t(i), 1.0f});
  t.insert(t.end(), add.begin(), add.end());
  std::stable_sort(t.begin(), t.end(), less);  // csr_from_triples
  *out_nnz = t.size();
  if (!out_np) return kOk;
  std::fill(out_np, out_np + n + 1, 0);
  for (size_t i = 0; i < t.size(); ++i) {
    out_np[t[i].r + 1]++;
    out_el[i] = t[i].c;
    if (out_vals) out_vals[i] = t[i].v;
  }
  for (uint64_t i = 0; i < n; ++i) out_np[i + 1] += out_np[i];
  return kOk;
}

// DenseMatrix::random (dense_matrix.hpp:43-50): mt19937_64 + the standard
// uniform_real_distribution<float>; reproduces the reference's inputs.
void or_dense_random(uint64_t r, uint64_t c, uint64_t seed, float lo, float hi,
                     float* out) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<float> dist(lo, hi);
  for (uint64_t i = 0; i < r * c; ++i) out[i] = dist(rng);
}

}  // extern "C"
