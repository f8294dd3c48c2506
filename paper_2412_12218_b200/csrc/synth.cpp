// Synthetic inputs for the bench and the GPU tests (host, multithreaded).
//
// The reference's generator is G(n,p) with n^2 Bernoulli draws
// (/root/reference/proj/src/synthetic.cpp:11-27) and cannot produce the
// configs' shapes (10^5-10^7 nodes).  This one is O(E): per-node degree and
// neighbour draws come from a counter-based hash of (seed, node, draw), so the
// output is identical for any thread count.  Locality knob: a fraction
// p_local of every node's picks lands within +-band*avg_picks node ids (what
// makes SGT tiles denser than the uniform 1/16 floor).

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <random>
#include <thread>
#include <vector>

#include "sgtk_cuda.h"

struct sgtk_synth {
  uint64_t n = 0;
  std::vector<uint64_t> np;
  std::vector<uint32_t> el;
};

namespace {

inline uint64_t mix(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
inline uint64_t h3(uint64_t seed, uint64_t a, uint64_t b) {
  return mix(seed ^ mix(a * 0x632BE59BD9B4E019ull + mix(b)));
}
inline double u01(uint64_t h) { return double(h >> 11) * (1.0 / 9007199254740992.0); }

template <class F>
void parallel_for(uint64_t n, F&& f) {
  unsigned nt = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  if (n < 4096) nt = 1;
  std::vector<std::thread> th;
  const uint64_t chunk = (n + nt - 1) / nt;
  for (unsigned t = 0; t < nt; ++t) {
    const uint64_t lo = t * chunk, hi = std::min(n, lo + chunk);
    if (lo >= hi) break;
    th.emplace_back([=, &f] {
      for (uint64_t i = lo; i < hi; ++i) f(i);
    });
  }
  for (auto& x : th) x.join();
}

}  // namespace

extern "C" {

int sgtk_synth_create(uint64_t n, double avg, double alpha, double p_local, double band,
                      uint64_t seed, sgtk_synth** out) {
  if (!out || n == 0 || n > 0xFFFFFFFFull || !(avg >= 0)) return SGTK_ERR_RANGE;
  try {
    auto s = new sgtk_synth();
    s->n = n;
    // 1. degrees
    std::vector<double> raw(n);
    parallel_for(n, [&](uint64_t i) {
      const double u = u01(h3(seed, i, ~0ull));
      raw[i] = alpha > 1.0 ? std::pow(1.0 - u, -1.0 / (alpha - 1.0)) : 0.5 + u;
    });
    const double kmax = double(n - 1);
    double scale = 1.0;
    for (int it = 0; it < 3; ++it) {  // scale so the truncated mean hits avg
      double sum = 0.0;
      for (uint64_t i = 0; i < n; ++i) sum += std::min(kmax, raw[i] * scale);
      if (sum <= 0) break;
      scale *= avg * double(n) / sum;
    }
    std::vector<uint32_t> k(n);
    std::vector<uint64_t> off(n + 1, 0);
    for (uint64_t i = 0; i < n; ++i) {
      const double v = std::min(kmax, raw[i] * scale);
      const double fl = std::floor(v);
      k[i] = uint32_t(fl + (u01(h3(seed, i, ~1ull)) < v - fl ? 1 : 0));
      off[i + 1] = off[i] + k[i];
    }
    raw.clear();
    raw.shrink_to_fit();
    // 2. picks
    const uint64_t P = off[n];
    std::vector<uint32_t> pick(P);
    const int64_t B = std::max<int64_t>(1, int64_t(std::ceil(band * std::max(avg, 1.0))));
    parallel_for(n, [&](uint64_t i) {
      for (uint32_t j = 0; j < k[i]; ++j) {
        const uint64_t h = h3(seed, i, 2ull * j + 1), h2 = h3(seed, i, 2ull * j + 2);
        uint64_t tgt;
        if (u01(h) < p_local) {
          int64_t o = int64_t(h2 % uint64_t(2 * B)) - B;
          if (o >= 0) ++o;  // [-B, -1] u [1, B]
          int64_t v = int64_t(i) + o;
          if (v < 0) v = -v;
          if (v >= int64_t(n)) v = 2 * int64_t(n) - 2 - v;
          tgt = uint64_t(std::min<int64_t>(std::max<int64_t>(v, 0), int64_t(n) - 1));
        } else {
          tgt = h2 % n;
        }
        pick[off[i] + j] = uint32_t(tgt);
      }
    });
    // 3. reverse lists (order fixed later by the per-row sort)
    std::vector<std::atomic<uint32_t>> indeg(n);
    for (auto& a : indeg) a.store(0, std::memory_order_relaxed);
    parallel_for(n, [&](uint64_t i) {
      for (uint64_t e = off[i]; e < off[i + 1]; ++e)
        indeg[pick[e]].fetch_add(1, std::memory_order_relaxed);
    });
    std::vector<uint64_t> roff(n + 1, 0);
    for (uint64_t i = 0; i < n; ++i) roff[i + 1] = roff[i] + indeg[i].load();
    std::vector<uint32_t> rev(P);
    std::vector<std::atomic<uint64_t>> cur(n);
    for (uint64_t i = 0; i < n; ++i) cur[i].store(roff[i], std::memory_order_relaxed);
    parallel_for(n, [&](uint64_t i) {
      for (uint64_t e = off[i]; e < off[i + 1]; ++e)
        rev[cur[pick[e]].fetch_add(1, std::memory_order_relaxed)] = uint32_t(i);
    });
    // 4. per row: out U in U {i}, sorted unique
    std::vector<uint32_t> len(n);
    parallel_for(n, [&](uint64_t i) {
      std::vector<uint32_t> row;
      row.reserve(k[i] + (roff[i + 1] - roff[i]) + 1);
      row.insert(row.end(), pick.begin() + off[i], pick.begin() + off[i + 1]);
      row.insert(row.end(), rev.begin() + roff[i], rev.begin() + roff[i + 1]);
      row.push_back(uint32_t(i));
      std::sort(row.begin(), row.end());
      len[i] = uint32_t(std::unique(row.begin(), row.end()) - row.begin());
    });
    s->np.assign(n + 1, 0);
    for (uint64_t i = 0; i < n; ++i) s->np[i + 1] = s->np[i] + len[i];
    s->el.resize(s->np[n]);
    parallel_for(n, [&](uint64_t i) {
      std::vector<uint32_t> row;
      row.reserve(len[i] * 2 + 1);
      row.insert(row.end(), pick.begin() + off[i], pick.begin() + off[i + 1]);
      row.insert(row.end(), rev.begin() + roff[i], rev.begin() + roff[i + 1]);
      row.push_back(uint32_t(i));
      std::sort(row.begin(), row.end());
      row.erase(std::unique(row.begin(), row.end()), row.end());
      std::copy(row.begin(), row.end(), s->el.begin() + s->np[i]);
    });
    *out = s;
    return SGTK_OK;
  } catch (...) {
    return SGTK_ERR;
  }
}

int sgtk_synth_info(const sgtk_synth* s, uint64_t* n, uint64_t* nnz) {
  if (!s) return SGTK_ERR;
  *n = s->n;
  *nnz = s->el.size();
  return SGTK_OK;
}

int sgtk_synth_copy(const sgtk_synth* s, uint64_t* np, uint32_t* el) {
  if (!s) return SGTK_ERR;
  std::memcpy(np, s->np.data(), s->np.size() * 8);
  if (!s->el.empty()) std::memcpy(el, s->el.data(), s->el.size() * 4);
  return SGTK_OK;
}

void sgtk_synth_destroy(sgtk_synth* s) { delete s; }

void sgtk_dense_random(uint64_t rows, uint64_t cols, uint64_t seed, float lo, float hi,
                       float* out) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<float> dist(lo, hi);
  const uint64_t n = rows * cols;
  for (uint64_t i = 0; i < n; ++i) out[i] = dist(rng);
}

}  // extern "C"
