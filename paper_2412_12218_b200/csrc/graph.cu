// GPU translator (SGT) and the condensed tile format.
//
// Replaces sgt_transform (/root/reference/proj/src/sgt_transform.cpp:18-77),
// reblock (:79-91), block_stats (:93-100), validate_csr
// (/root/reference/proj/src/csr_graph.cpp:10-39) and gather_tile
// (/root/reference/proj/src/tile_exec.cpp:163-198).
//
// Pipeline (all O(E) work on the GPU, O(W) bookkeeping on the host):
//   1. validate the CSR (one kernel, first-violation flags -> SGTK_ERR)
//   2. edge_to_row (warp per row)
//   3. per window: sort + dedupe the window's columns, rank every edge
//        - <= 2048 edges : 256-thread CTA, bitonic sort in shared memory
//        - <= 32768 edges: 1024-thread CTA, bitonic sort in shared memory
//        - larger        : CUB segmented radix sort in HBM + CTA unique/rank
//      uniques land at the window's edge offset (no scan needed yet)
//   4. host scan of per-window unique counts -> window_offsets; compaction
//   5. 16x8 and 16x16 occupancy bitmaps (atomicOr of bits: order-free, so
//      deterministic) and nnz-balanced work units for the kernels.
// The integer outputs are bit-exact with the reference (tests/test_gpu_*).

#include <cub/device/device_segmented_radix_sort.cuh>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <numeric>

#include "kernels.cuh"

namespace sgtkcu {
namespace {

constexpr uint32_t kSmallCap = 2048, kSmallThreads = 256;
constexpr uint32_t kMedCap = 32768, kMedThreads = 1024;

// ---------------------------------------------------------------- validation
// Flags in reference check order (csr_graph.cpp:10-39).
enum : uint32_t {
  kVNp0 = 1, kVNpEnd = 2, kVMono = 4, kVRange = 8, kVSorted = 16, kVFinite = 32,
};

__global__ void validate_kernel(const uint64_t* __restrict__ np, const uint32_t* __restrict__ el,
                                const float* __restrict__ vals, uint64_t n, uint64_t n_cols,
                                uint64_t nnz, int sorted_unique, uint32_t* flags) {
  const uint64_t stride = uint64_t(gridDim.x) * blockDim.x;
  uint32_t f = 0;
  const uint64_t tid = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (tid == 0) {
    if (np[0] != 0) f |= kVNp0;
    if (np[n] != nnz) f |= kVNpEnd;
  }
  for (uint64_t i = tid; i < n; i += stride)
    if (np[i] > np[i + 1]) f |= kVMono;
  if (!(f & (kVNp0 | kVNpEnd | kVMono)) || true) {
    for (uint64_t e = tid; e < nnz; e += stride) {
      if (el[e] >= n_cols) f |= kVRange;
      if (vals && !isfinite(vals[e])) f |= kVFinite;
    }
  }
  if (f) atomicOr(flags, f);
}

// Sortedness needs row boundaries: warp per row.
__global__ void validate_sorted_kernel(const uint64_t* __restrict__ np,
                                       const uint32_t* __restrict__ el, uint64_t n,
                                       uint64_t nnz, uint32_t* flags) {
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  bool bad = false;
  for (uint64_t r = warp; r < n; r += nwarps) {
    uint64_t lo = np[r], hi = np[r + 1];
    if (hi > nnz || lo > hi) continue;  // reported by validate_kernel
    for (uint64_t e = lo + 1 + lane; e < hi; e += 32)
      if (el[e - 1] >= el[e]) bad = true;
  }
  if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(flags, uint32_t(kVSorted));
}

__global__ void edge_to_row_kernel(const uint64_t* __restrict__ np, uint64_t n,
                                   uint32_t* __restrict__ e2r) {
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t r = warp; r < n; r += nwarps)
    for (uint64_t e = np[r] + lane; e < np[r + 1]; e += 32) e2r[e] = uint32_t(r);
}

__global__ void window_bounds_kernel(const uint64_t* __restrict__ np, uint64_t n,
                                     uint32_t bh, uint64_t W, uint64_t* __restrict__ wb) {
  for (uint64_t w = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; w <= W;
       w += uint64_t(gridDim.x) * blockDim.x)
    wb[w] = np[min(n, w * bh)];
}

// ------------------------------------------------------------ block helpers
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* warp_sums,
                                                    uint32_t& total) {
  const uint32_t lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  uint32_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_sums[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    constexpr int NW = NT / 32;
    uint32_t s = lane < NW ? warp_sums[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t t = __shfl_up_sync(0xFFFFFFFFu, s, o);
      if (lane >= o) s += t;
    }
    if (lane < NW) warp_sums[lane] = s;  // inclusive warp prefix
  }
  __syncthreads();
  total = warp_sums[NT / 32 - 1];
  const uint32_t before = warp ? warp_sums[warp - 1] : 0u;
  __syncthreads();  // warp_sums reusable after return
  return before + incl - v;
}

template <int NT>
__device__ void bitonic_sort_smem(uint32_t* s, uint32_t n2) {
  for (uint32_t k = 2; k <= n2; k <<= 1) {
    for (uint32_t j = k >> 1; j > 0; j >>= 1) {
      for (uint32_t i = threadIdx.x; i < n2; i += NT) {
        const uint32_t ixj = i ^ j;
        if (ixj > i) {
          const uint32_t a = s[i], b = s[ixj];
          const bool up = (i & k) == 0;
          if ((a > b) == up) { s[i] = b; s[ixj] = a; }
        }
      }
      __syncthreads();
    }
  }
}

__device__ __forceinline__ uint32_t lb_smem(const uint32_t* s, uint32_t n, uint32_t v) {
  uint32_t lo = 0, hi = n;
  while (lo < hi) {
    uint32_t mid = (lo + hi) >> 1;
    if (s[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

// One CTA per window (windows with <= CAP edges): sorted uniques written at
// the window's edge offset in `tmp`, count in ucount[w], ranks in e2c.
// sgt_transform.cpp:37-49 (sort+unique) and :58-72 (lower_bound per edge).
template <int CAP, int NT>
__global__ void __launch_bounds__(NT)
window_unique_smem_kernel(const uint64_t* __restrict__ wb, const uint32_t* __restrict__ el,
                          const uint32_t* __restrict__ list, uint32_t* __restrict__ tmp,
                          uint32_t* __restrict__ ucount, uint32_t* __restrict__ e2c) {
  extern __shared__ uint32_t s[];
  __shared__ uint32_t warp_sums[32];
  constexpr int IPT = CAP / NT;
  const uint32_t w = list[blockIdx.x];
  const uint64_t lo = wb[w], hi = wb[w + 1];
  const uint32_t cnt = uint32_t(hi - lo);
  uint32_t n2 = 1;
  while (n2 < cnt) n2 <<= 1;
  for (uint32_t i = threadIdx.x; i < n2; i += NT) s[i] = i < cnt ? el[lo + i] : 0xFFFFFFFFu;
  __syncthreads();
  bitonic_sort_smem<NT>(s, n2);

  // Unique flags over a contiguous per-thread segment.  Every read of s
  // happens before the scan's barriers; the compaction writes come after.
  const uint32_t beg = threadIdx.x * IPT;
  uint32_t v[IPT];
  const uint32_t prev = (beg > 0 && beg - 1 < cnt) ? s[beg - 1] : 0u;
  uint32_t nflag = 0;
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const uint32_t i = beg + k;
    v[k] = i < cnt ? s[i] : 0u;
    const uint32_t before = k ? v[k - 1] : prev;
    nflag += (i < cnt && (i == 0 || before != v[k])) ? 1u : 0u;
  }
  uint32_t total;
  uint32_t pos = block_excl_scan<NT>(nflag, warp_sums, total);
#pragma unroll
  for (int k = 0; k < IPT; ++k) {
    const uint32_t i = beg + k;
    const uint32_t before = k ? v[k - 1] : prev;
    if (i < cnt && (i == 0 || before != v[k])) {
      s[pos] = v[k];
      tmp[lo + pos] = v[k];
      ++pos;
    }
  }
  if (threadIdx.x == 0) ucount[w] = total;
  __syncthreads();
  for (uint32_t e = threadIdx.x; e < cnt; e += NT) e2c[lo + e] = lb_smem(s, total, el[lo + e]);
}

// Large windows: keys already sorted per segment in `sorted` (compact layout,
// offsets `off`).  One CTA per window: chunked unique + running offset.
template <int NT>
__global__ void __launch_bounds__(NT)
large_unique_kernel(const uint64_t* __restrict__ wb, const uint32_t* __restrict__ list,
                    const uint64_t* __restrict__ off, const uint32_t* __restrict__ sorted,
                    uint32_t* __restrict__ tmp, uint32_t* __restrict__ ucount) {
  __shared__ uint32_t warp_sums[32];
  const uint32_t w = list[blockIdx.x];
  const uint64_t lo = wb[w];
  const uint32_t* k = sorted + off[blockIdx.x];
  const uint64_t cnt = off[blockIdx.x + 1] - off[blockIdx.x];
  uint32_t run = 0;
  for (uint64_t base = 0; base < cnt; base += NT) {
    const uint64_t i = base + threadIdx.x;
    const bool f = i < cnt && (i == 0 || k[i - 1] != k[i]);
    uint32_t total;
    const uint32_t pos = block_excl_scan<NT>(f ? 1u : 0u, warp_sums, total);
    if (f) tmp[lo + run + pos] = k[i];
    run += total;
  }
  if (threadIdx.x == 0) ucount[w] = run;
}

__global__ void large_rank_kernel(const uint64_t* __restrict__ wb, const uint32_t* __restrict__ list,
                                  const uint32_t* __restrict__ el, const uint32_t* __restrict__ tmp,
                                  const uint32_t* __restrict__ ucount, uint32_t* __restrict__ e2c) {
  const uint32_t w = list[blockIdx.x];
  const uint64_t lo = wb[w], hi = wb[w + 1];
  const uint32_t u = ucount[w];
  for (uint64_t e = lo + threadIdx.x; e < hi; e += blockDim.x)
    e2c[e] = uint32_t(lower_bound_u32(tmp, lo, lo + u, el[e]) - lo);
}

__global__ void gather_segments_kernel(const uint64_t* __restrict__ wb,
                                       const uint32_t* __restrict__ list,
                                       const uint64_t* __restrict__ off,
                                       const uint32_t* __restrict__ el, uint32_t* __restrict__ out) {
  const uint32_t w = list[blockIdx.x];
  const uint64_t lo = wb[w], cnt = wb[w + 1] - lo, o = off[blockIdx.x];
  for (uint64_t i = threadIdx.x; i < cnt; i += blockDim.x) out[o + i] = el[lo + i];
}

// window_unique_cols compaction: tmp[wb[w] + i] -> wuc[wo[w] + i]
__global__ void compact_kernel(const uint64_t* __restrict__ wb, const uint64_t* __restrict__ wo,
                               uint64_t W, const uint32_t* __restrict__ tmp,
                               uint32_t* __restrict__ wuc) {
  for (uint64_t w = blockIdx.x; w < W; w += gridDim.x) {
    const uint64_t src = wb[w], dst = wo[w], u = wo[w + 1] - wo[w];
    for (uint64_t i = threadIdx.x; i < u; i += blockDim.x) wuc[dst + i] = tmp[src + i];
  }
}

// 16x8 / 16x16 occupancy bitmaps.  Row r of a tile owns byte r (8-wide) or
// half-word r (16-wide); OR is order-independent, so this is deterministic.
__global__ void bitmap_kernel(const uint32_t* __restrict__ e2r, const uint32_t* __restrict__ e2c,
                              uint64_t nnz, const uint64_t* __restrict__ toff8,
                              const uint64_t* __restrict__ toff16, uint32_t* __restrict__ bm8,
                              uint32_t* __restrict__ bm16) {
  for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < nnz;
       e += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t r = e2r[e], c = e2c[e];
    const uint32_t w = r >> 4, rr = r & 15u;
    const uint64_t t8 = toff8[w] + (c >> 3);
    atomicOr(bm8 + t8 * 4 + (rr >> 2), 1u << ((rr & 3u) * 8 + (c & 7u)));
    const uint64_t t16 = toff16[w] + (c >> 4);
    atomicOr(bm16 + t16 * 8 + (rr >> 1), 1u << ((rr & 1u) * 16 + (c & 15u)));
  }
}

__global__ void cut_kernel(const uint32_t* __restrict__ cut, uint64_t W, uint32_t blk_w,
                           uint32_t tile_w, uint32_t* __restrict__ out) {
  for (uint64_t w = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; w < W;
       w += uint64_t(gridDim.x) * blockDim.x)
    out[w] = uint32_t((uint64_t(cut[w]) * blk_w) / tile_w);
}

inline unsigned grid_for(uint64_t n, unsigned block, unsigned cap = 148u * 32u) {
  uint64_t g = (n + block - 1) / block;
  return unsigned(std::max<uint64_t>(1, std::min<uint64_t>(g, cap)));
}

template <class T>
std::shared_ptr<DevBuf> upload(const T* host, size_t count, cudaStream_t s) {
  auto b = std::make_shared<DevBuf>(count * sizeof(T));
  if (count) CU(cudaMemcpyAsync(b->p, host, count * sizeof(T), cudaMemcpyHostToDevice, s));
  return b;
}

template <class T>
std::vector<T> download(const void* dev, size_t count, cudaStream_t s) {
  std::vector<T> h(count);
  if (count) {
    CU(cudaMemcpyAsync(h.data(), dev, count * sizeof(T), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
  }
  return h;
}

// Per-window sort/unique/rank for row-window height bh.
Windows build_windows(const sgtk_graph& g, uint32_t bh, cudaStream_t s) {
  Windows win;
  win.blk_h = bh;
  const uint64_t n = g.n_rows, E = g.nnz;
  const uint64_t W = (n + bh - 1) / bh;
  win.W = W;
  DevBuf wb_d((W + 1) * 8);
  window_bounds_kernel<<<grid_for(W + 1, 256), 256, 0, s>>>(g.np->as<uint64_t>(), n, bh, W,
                                                            wb_d.as<uint64_t>());
  CU_LAUNCH("window_bounds_kernel");
  std::vector<uint64_t> wb = download<uint64_t>(wb_d.p, W + 1, s);

  std::vector<uint32_t> small, medium, large;
  for (uint64_t w = 0; w < W; ++w) {
    const uint64_t c = wb[w + 1] - wb[w];
    if (c <= kSmallCap) small.push_back(uint32_t(w));
    else if (c <= kMedCap) medium.push_back(uint32_t(w));
    else large.push_back(uint32_t(w));
  }
  DevBuf tmp(std::max<uint64_t>(E, 1) * 4), ucount(std::max<uint64_t>(W, 1) * 4);
  win.e2c = std::make_shared<DevBuf>(std::max<uint64_t>(E, 1) * 4);
  CU(cudaMemsetAsync(ucount.p, 0, W * 4, s));
  const uint64_t* wbp = wb_d.as<uint64_t>();
  const uint32_t* el = g.el->as<uint32_t>();

  auto run_smem = [&](const std::vector<uint32_t>& list, auto kernel, uint32_t cap, uint32_t nt) {
    if (list.empty()) return;
    auto ld = upload(list.data(), list.size(), s);
    const size_t smem = size_t(cap) * 4;
    CU(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)));
    for (size_t b = 0; b < list.size(); b += 65535u * 16u) {
      const unsigned nb = unsigned(std::min<size_t>(list.size() - b, 65535u * 16u));
      kernel<<<nb, nt, smem, s>>>(wbp, el, ld->as<uint32_t>() + b, tmp.as<uint32_t>(),
                                  ucount.as<uint32_t>(), win.e2c->as<uint32_t>());
      CU_LAUNCH("window_unique_smem_kernel");
    }
  };
  run_smem(small, window_unique_smem_kernel<kSmallCap, kSmallThreads>, kSmallCap, kSmallThreads);
  run_smem(medium, window_unique_smem_kernel<kMedCap, kMedThreads>, kMedCap, kMedThreads);

  if (!large.empty()) {
    // batches of <= 2^30 keys (CUB's int item count)
    size_t i = 0;
    while (i < large.size()) {
      std::vector<uint32_t> batch;
      std::vector<uint64_t> off{0};
      while (i < large.size()) {
        const uint64_t c = wb[large[i] + 1] - wb[large[i]];
        if (!batch.empty() && off.back() + c > (1ull << 30)) break;
        batch.push_back(large[i]);
        off.push_back(off.back() + c);
        ++i;
      }
      const uint64_t total = off.back();
      auto ld = upload(batch.data(), batch.size(), s);
      auto od = upload(off.data(), off.size(), s);
      std::vector<int> ioff(off.begin(), off.end());
      auto iod = upload(ioff.data(), ioff.size(), s);
      DevBuf kin(total * 4), kout(total * 4);
      gather_segments_kernel<<<unsigned(batch.size()), 256, 0, s>>>(
          wbp, ld->as<uint32_t>(), od->as<uint64_t>(), el, kin.as<uint32_t>());
      CU_LAUNCH("gather_segments_kernel");
      size_t temp_bytes = 0;
      CU(cub::DeviceSegmentedRadixSort::SortKeys(nullptr, temp_bytes, kin.as<uint32_t>(),
                                                 kout.as<uint32_t>(), int(total), int(batch.size()),
                                                 iod->as<int>(), iod->as<int>() + 1, 0, 32, s));
      DevBuf temp(std::max<size_t>(temp_bytes, 16));
      CU(cub::DeviceSegmentedRadixSort::SortKeys(temp.p, temp_bytes, kin.as<uint32_t>(),
                                                 kout.as<uint32_t>(), int(total), int(batch.size()),
                                                 iod->as<int>(), iod->as<int>() + 1, 0, 32, s));
      large_unique_kernel<1024><<<unsigned(batch.size()), 1024, 0, s>>>(
          wbp, ld->as<uint32_t>(), od->as<uint64_t>(), kout.as<uint32_t>(), tmp.as<uint32_t>(),
          ucount.as<uint32_t>());
      CU_LAUNCH("large_unique_kernel");
      large_rank_kernel<<<unsigned(batch.size()), 1024, 0, s>>>(
          wbp, ld->as<uint32_t>(), el, tmp.as<uint32_t>(), ucount.as<uint32_t>(),
          win.e2c->as<uint32_t>());
      CU_LAUNCH("large_rank_kernel");
      CU(cudaStreamSynchronize(s));  // batch scratch freed at scope exit
    }
  }

  win.ucount_host = download<uint32_t>(ucount.p, W, s);
  win.wo_host.assign(W + 1, 0);
  for (uint64_t w = 0; w < W; ++w) win.wo_host[w + 1] = win.wo_host[w] + win.ucount_host[w];
  win.U = win.wo_host[W];
  win.wo = upload(win.wo_host.data(), W + 1, s);
  win.wuc = std::make_shared<DevBuf>(std::max<uint64_t>(win.U, 1) * 4);
  if (W)
    compact_kernel<<<grid_for(W, 1, 148u * 64u), 128, 0, s>>>(wbp, win.wo->as<uint64_t>(), W,
                                                              tmp.as<uint32_t>(),
                                                              win.wuc->as<uint32_t>());
  CU_LAUNCH("compact_kernel");
  CU(cudaStreamSynchronize(s));
  return win;
}

// Work units: split windows with more than max_tiles tiles (4096 unique
// columns) so no warp-task is far larger than the average; split windows
// reduce their partials in unit order.  The split depends on the window alone
// (never on graph-wide totals), so a window's summation order -- hence its
// output bits -- is the same whether it is transformed in the full graph or
// in one GPU's row slice: results are bit-identical for any GPU count.
UnitPlan build_units(const std::vector<uint32_t>& ucount, uint32_t tile_w, uint64_t,
                     cudaStream_t s) {
  UnitPlan p;
  const uint64_t mt = 4096 / tile_w;
  p.max_tiles = uint32_t(mt);
  std::vector<WorkUnit> units;
  std::vector<ReduceItem> red;
  uint32_t slot = 0;
  for (size_t w = 0; w < ucount.size(); ++w) {
    const uint32_t tiles = (ucount[w] + tile_w - 1) / tile_w;
    if (tiles <= mt) {
      units.push_back({uint32_t(w), 0, tiles, kNoSlot});
    } else {
      const uint32_t k = uint32_t((tiles + mt - 1) / mt);
      red.push_back({uint32_t(w), slot, k, 0});
      for (uint32_t i = 0; i < k; ++i)
        units.push_back({uint32_t(w), uint32_t(i * mt), uint32_t(std::min<uint64_t>(tiles, (i + 1) * mt)),
                         slot + i});
      slot += k;
    }
  }
  p.n_units = uint32_t(units.size());
  p.n_reduce = uint32_t(red.size());
  p.n_slots = slot;
  p.units = upload(units.data(), units.size(), s);
  p.reduce = upload(red.data(), red.size(), s);
  return p;
}

void finish_tiles(sgtk_graph& g, cudaStream_t s) {
  const auto& uc = g.internal.ucount_host;
  const uint64_t W = g.internal.W;
  std::vector<uint64_t> t8(W + 1, 0), t16(W + 1, 0);
  for (uint64_t w = 0; w < W; ++w) {
    t8[w + 1] = t8[w] + (uc[w] + 7) / 8;
    t16[w + 1] = t16[w] + (uc[w] + 15) / 16;
  }
  g.T8 = t8[W];
  g.T16 = t16[W];
  g.toff8 = upload(t8.data(), W + 1, s);
  g.toff16 = upload(t16.data(), W + 1, s);
  g.bm8 = std::make_shared<DevBuf>(std::max<uint64_t>(g.T8, 1) * 16);
  g.bm16 = std::make_shared<DevBuf>(std::max<uint64_t>(g.T16, 1) * 32);
  CU(cudaMemsetAsync(g.bm8->p, 0, g.bm8->bytes, s));
  CU(cudaMemsetAsync(g.bm16->p, 0, g.bm16->bytes, s));
  if (g.nnz)
    bitmap_kernel<<<grid_for(g.nnz, 256), 256, 0, s>>>(
        g.e2r->as<uint32_t>(), g.internal.e2c->as<uint32_t>(), g.nnz, g.toff8->as<uint64_t>(),
        g.toff16->as<uint64_t>(), g.bm8->as<uint32_t>(), g.bm16->as<uint32_t>());
  CU_LAUNCH("bitmap_kernel");
  g.plan8 = build_units(uc, 8, g.T8, s);
  g.plan16 = build_units(uc, 16, g.T16, s);
  CU(cudaStreamSynchronize(s));
}

void set_partition(sgtk_graph& g) {
  const uint64_t W = g.user.W;
  g.bp_host.assign(W, 0);
  g.block_counter = 0;
  for (uint64_t w = 0; w < W; ++w) {
    g.bp_host[w] = (g.user.ucount_host[w] + g.blk_w - 1) / g.blk_w;
    g.block_counter += g.bp_host[w];
  }
}

void load_csr(sgtk_graph& g, const uint64_t* np, const uint32_t* el, const float* vals,
              int kind, cudaStream_t s) {
  const auto dir = kind == SGTK_PTR_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  g.np = std::make_shared<DevBuf>((g.n_rows + 1) * 8);
  g.el = std::make_shared<DevBuf>(std::max<uint64_t>(g.nnz, 1) * 4);
  CU(cudaMemcpyAsync(g.np->p, np, (g.n_rows + 1) * 8, dir, s));
  if (g.nnz) CU(cudaMemcpyAsync(g.el->p, el, g.nnz * 4, dir, s));
  g.has_values = vals != nullptr;
  g.vals = std::make_shared<DevBuf>(g.has_values ? std::max<uint64_t>(g.nnz, 1) * 4 : 0);
  if (g.has_values && g.nnz) CU(cudaMemcpyAsync(g.vals->p, vals, g.nnz * 4, dir, s));
}

void validate(const sgtk_graph& g, cudaStream_t s) {
  DevBuf flags(4);
  CU(cudaMemsetAsync(flags.p, 0, 4, s));
  validate_kernel<<<grid_for(std::max(g.n_rows, g.nnz) + 1, 256), 256, 0, s>>>(
      g.np->as<uint64_t>(), g.el->as<uint32_t>(), g.has_values ? g.vals->as<float>() : nullptr,
      g.n_rows, g.n_cols, g.nnz, 1, flags.as<uint32_t>());
  CU_LAUNCH("validate_kernel");
  uint32_t f = download<uint32_t>(flags.p, 1, s)[0];
  if (!(f & (kVNp0 | kVNpEnd | kVMono))) {
    validate_sorted_kernel<<<grid_for(g.n_rows * 32, 256), 256, 0, s>>>(
        g.np->as<uint64_t>(), g.el->as<uint32_t>(), g.n_rows, g.nnz, flags.as<uint32_t>());
    CU_LAUNCH("validate_sorted_kernel");
    f = download<uint32_t>(flags.p, 1, s)[0];
  }
  if (f & kVNp0) raise(SGTK_ERR, "csr: node_pointer[0] != 0");
  if (f & kVNpEnd) raise(SGTK_ERR, "csr: node_pointer end does not match edge count");
  if (f & kVMono) raise(SGTK_ERR, "csr: node_pointer not non-decreasing");
  if (f & kVRange) raise(SGTK_ERR, "csr: column id out of range");
  if (f & kVSorted) raise(SGTK_ERR, "csr: columns not strictly ascending within a row");
  if (f & kVFinite) raise(SGTK_ERR, "csr: non-finite edge value");
}

// Stage timing of a graph build (SGTK_BUILD_TIMING): synchronise and take the
// host clock at each stage boundary; a no-op otherwise.
struct StageClock {
  double* ms;
  cudaStream_t s;
  bool on;
  std::chrono::steady_clock::time_point t;
  StageClock(double* out, cudaStream_t st) : ms(out), s(st), on(std::getenv("SGTK_BUILD_TIMING")) {
    if (on) {
      CU(cudaStreamSynchronize(s));
      t = std::chrono::steady_clock::now();
    }
  }
  void mark(int stage) {
    if (!on) return;
    CU(cudaStreamSynchronize(s));
    const auto now = std::chrono::steady_clock::now();
    ms[stage] = std::chrono::duration<double, std::milli>(now - t).count();
    t = now;
  }
};

void build_e2r(sgtk_graph& g, cudaStream_t s) {
  g.e2r = std::make_shared<DevBuf>(std::max<uint64_t>(g.nnz, 1) * 4);
  if (g.n_rows && g.nnz) {
    edge_to_row_kernel<<<grid_for(g.n_rows * 32, 256), 256, 0, s>>>(g.np->as<uint64_t>(),
                                                                     g.n_rows,
                                                                     g.e2r->as<uint32_t>());
    CU_LAUNCH("edge_to_row_kernel");
  }
}

}  // namespace

Windows build_row_windows(const sgtk_graph& g, uint32_t bh, cudaStream_t s) {
  return build_windows(g, bh, s);
}

sgtk_graph* graph_create(const uint64_t* np, const uint32_t* el, const float* vals, uint64_t n_rows,
                         uint64_t n_cols, uint64_t nnz, uint32_t blk_h, uint32_t blk_w, int kind,
                         cudaStream_t s, uint64_t row_offset) {
  if (blk_h == 0 || blk_w == 0) raise(SGTK_ERR_GEOMETRY, "tile dimensions must be positive");
  if (row_offset % 16) raise(SGTK_ERR_SHAPE, "row slice must start on a 16-row window boundary");
  if (n_cols > 0xFFFFFFFFull || nnz > 0xFFFFFFFFull)
    raise(SGTK_ERR_OVERFLOW, "graph exceeds 32-bit node/edge ids");
  auto g = std::make_unique<sgtk_graph>();
  CU(cudaGetDevice(&g->device));
  g->n_rows = n_rows;
  g->n_cols = n_cols;
  g->nnz = nnz;
  g->row_offset = row_offset;
  g->blk_h = blk_h;
  g->blk_w = blk_w;
  StageClock clk(g->build_ms, s);
  load_csr(*g, np, el, vals, kind, s);
  clk.mark(0);
  validate(*g, s);
  clk.mark(1);
  build_e2r(*g, s);
  clk.mark(2);
  g->user = build_windows(*g, blk_h, s);
  clk.mark(3);
  g->internal = blk_h == 16 ? g->user : build_windows(*g, 16, s);
  clk.mark(4);
  set_partition(*g);
  g->bp = upload(g->bp_host.data(), g->bp_host.size(), s);
  finish_tiles(*g, s);
  clk.mark(5);
  build_panels(*g, s);
  clk.mark(6);
  g->scratch = std::make_shared<DevBuf>();
  return g.release();
}

sgtk_graph* graph_import(const uint64_t* np, const uint32_t* el, const float* vals,
                         uint64_t n_rows, uint64_t nnz, uint32_t blk_h, uint32_t blk_w,
                         const uint32_t* e2c, const uint64_t* wo, const uint32_t* wuc,
                         cudaStream_t s, const char* panel_section) {
  if (blk_h == 0 || blk_w == 0) raise(SGTK_ERR_GEOMETRY, "tile dimensions must be positive");
  auto g = std::make_unique<sgtk_graph>();
  CU(cudaGetDevice(&g->device));
  g->n_rows = g->n_cols = n_rows;
  g->nnz = nnz;
  g->blk_h = blk_h;
  g->blk_w = blk_w;
  load_csr(*g, np, el, vals, SGTK_PTR_HOST, s);
  build_e2r(*g, s);
  Windows& u = g->user;
  u.blk_h = blk_h;
  u.W = (n_rows + blk_h - 1) / blk_h;
  u.wo_host.assign(wo, wo + u.W + 1);
  u.U = u.wo_host[u.W];
  u.ucount_host.resize(u.W);
  for (uint64_t w = 0; w < u.W; ++w) u.ucount_host[w] = uint32_t(wo[w + 1] - wo[w]);
  u.e2c = upload(e2c, nnz, s);
  u.wo = upload(wo, u.W + 1, s);
  u.wuc = upload(wuc, u.U, s);
  g->internal = blk_h == 16 ? g->user : build_windows(*g, 16, s);
  set_partition(*g);
  g->bp = upload(g->bp_host.data(), g->bp_host.size(), s);
  finish_tiles(*g, s);
  if (!panel_section || !load_panel_section(*g, panel_section, s)) build_panels(*g, s);
  g->scratch = std::make_shared<DevBuf>();
  return g.release();
}

sgtk_graph* graph_reblock(const sgtk_graph* src, uint32_t blk_w, cudaStream_t s) {
  if (blk_w == 0) raise(SGTK_ERR_GEOMETRY, "tile width must be positive");
  auto g = std::make_unique<sgtk_graph>(*src);  // shares device arrays (immutable)
  g->blk_w = blk_w;
  set_partition(*g);
  g->bp = upload(g->bp_host.data(), g->bp_host.size(), s);
  g->scratch = std::make_shared<DevBuf>();
  CU(cudaStreamSynchronize(s));
  return g.release();
}

const uint32_t* internal_cut(const sgtk_graph* g, const uint32_t* cut_dev, int tile_w,
                             cudaStream_t s, DevBuf& keep) {
  if (!cut_dev) return nullptr;
  const uint64_t W = g->internal.W;
  keep.ensure(std::max<uint64_t>(W, 1) * 4);
  if (g->blk_h == 16) {
    cut_kernel<<<grid_for(W, 256), 256, 0, s>>>(cut_dev, W, g->blk_w, uint32_t(tile_w),
                                                keep.as<uint32_t>());
    CU_LAUNCH("cut_kernel");
  } else {
    // Non-16 row windows: carry each user window's tile ratio over to the
    // internal 16-row windows (results are split-invariant; only the
    // tensor-core / CUDA-core assignment is approximated).
    std::vector<uint32_t> cut = download<uint32_t>(cut_dev, g->user.W, s);
    std::vector<uint32_t> out(W);
    for (uint64_t w = 0; w < W; ++w) {
      const uint64_t uw = std::min<uint64_t>((w * 16) / g->blk_h, g->user.W - 1);
      const double ratio = g->bp_host[uw] ? double(cut[uw]) / g->bp_host[uw] : 1.0;
      const uint32_t tiles = (g->internal.ucount_host[w] + tile_w - 1) / tile_w;
      out[w] = uint32_t(std::floor(ratio * tiles));
    }
    CU(cudaMemcpyAsync(keep.p, out.data(), W * 4, cudaMemcpyHostToDevice, s));
    CU(cudaStreamSynchronize(s));
  }
  return keep.as<uint32_t>();
}

}  // namespace sgtkcu
