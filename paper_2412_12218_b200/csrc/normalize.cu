// GPU graph preprocessing: normalize_graph (/root/reference/proj/src/graph_io.cpp:195-259).
//
// The step before the translator in every GCN pipeline (bench.cpp:114-120,
// cli.cpp:213-215): dedupe (values summed in file order), symmetrize
// (missing reverse edges inserted with the forward value), add self-loops
// (missing (i,i), value 1.0).  The reference does a serial stable sort of
// (row, col) triples; here:
//   1. (row << 32 | col) keys with the edge index as payload, CUB radix sort
//      (stable, so duplicates keep their input order);
//   2. run heads + per-run sequential value sums (the reference's
//      left-to-right float addition order, so the sums are bit-exact);
//   3. reverse-edge / diagonal presence by binary search on the sorted keys;
//   4. the base list plus the inserted edges sorted again (stable), CSR rows
//      by binary search.
// Integer structure and values are bit-exact with the reference.

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include <vector>

#include "kernels.cuh"

namespace sgtkcu {
namespace {

__global__ void keys_kernel(const uint64_t* __restrict__ np, const uint32_t* __restrict__ el,
                            uint64_t n, uint64_t* __restrict__ keys, uint32_t* __restrict__ idx) {
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t r = warp; r < n; r += nw)
    for (uint64_t e = np[r] + lane; e < np[r + 1]; e += 32) {
      keys[e] = (r << 32) | el[e];
      idx[e] = uint32_t(e);
    }
}

__global__ void heads_kernel(const uint64_t* __restrict__ k, uint64_t m, int dedupe,
                             uint32_t* __restrict__ head) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += uint64_t(gridDim.x) * blockDim.x)
    head[i] = (!dedupe || i == 0 || k[i] != k[i - 1]) ? 1u : 0u;
}

// For each run (heads scanned inclusive -> run id + 1): key and the values
// summed in input order.
__global__ void runs_kernel(const uint64_t* __restrict__ k, const uint32_t* __restrict__ idx,
                            const uint32_t* __restrict__ incl, uint64_t m,
                            const float* __restrict__ vin, uint64_t* __restrict__ bkey,
                            float* __restrict__ bval) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const bool head = i == 0 || incl[i] != incl[i - 1];
    if (!head) continue;
    const uint32_t run = incl[i] - 1;
    bkey[run] = k[i];
    if (bval) {
      float s = vin ? vin[idx[i]] : 1.0f;
      for (uint64_t j = i + 1; j < m && incl[j] == incl[i]; ++j) s = s + (vin ? vin[idx[j]] : 1.0f);
      bval[run] = s;
    }
  }
}

__device__ __forceinline__ bool contains(const uint64_t* __restrict__ k, uint64_t m, uint64_t key) {
  uint64_t lo = 0, hi = m;
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (k[mid] < key) lo = mid + 1; else hi = mid;
  }
  return lo < m && k[lo] == key;
}

// flags[j] for j < U: base run j needs a mirrored insert; for U <= j < U+n:
// node j-U needs a self-loop.  Only the first of equal keys mirrors
// (graph_io.cpp:239-248).
__global__ void insert_flags_kernel(const uint64_t* __restrict__ bkey, uint64_t U, uint64_t n,
                                    int symmetrize, int loops, uint32_t* __restrict__ flags) {
  for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < U + n;
       j += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t f = 0;
    if (j < U) {
      if (symmetrize) {
        const uint64_t key = bkey[j];
        const uint64_t r = key >> 32, c = key & 0xFFFFFFFFull;
        const bool first = j == 0 || bkey[j - 1] != key;
        f = (first && r != c && !contains(bkey, U, (c << 32) | r)) ? 1u : 0u;
      }
    } else if (loops) {
      const uint64_t i = j - U;
      f = contains(bkey, U, (i << 32) | i) ? 0u : 1u;
    }
    flags[j] = f;
  }
}

__global__ void combine_kernel(const uint64_t* __restrict__ bkey, const float* __restrict__ bval,
                               uint64_t U, uint64_t n, const uint32_t* __restrict__ flags,
                               const uint32_t* __restrict__ pos, uint64_t* __restrict__ ckey,
                               uint32_t* __restrict__ cidx, float* __restrict__ cval) {
  for (uint64_t j = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; j < U + n;
       j += uint64_t(gridDim.x) * blockDim.x) {
    if (j < U) {
      ckey[j] = bkey[j];
      cidx[j] = uint32_t(j);
      if (cval) cval[j] = bval[j];
    }
    if (!flags[j]) continue;
    const uint64_t o = U + pos[j];
    if (j < U) {
      const uint64_t key = bkey[j];
      ckey[o] = ((key & 0xFFFFFFFFull) << 32) | (key >> 32);
      if (cval) cval[o] = bval[j];
    } else {
      const uint64_t i = j - U;
      ckey[o] = (i << 32) | i;
      if (cval) cval[o] = 1.0f;
    }
    cidx[o] = uint32_t(o);
  }
}

__global__ void emit_kernel(const uint64_t* __restrict__ skey, const uint32_t* __restrict__ sidx,
                            const float* __restrict__ cval, uint64_t m, uint32_t* __restrict__ el,
                            float* __restrict__ vals) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < m;
       i += uint64_t(gridDim.x) * blockDim.x) {
    el[i] = uint32_t(skey[i] & 0xFFFFFFFFull);
    if (vals) vals[i] = cval[sidx[i]];
  }
}

__global__ void rowptr_kernel(const uint64_t* __restrict__ skey, uint64_t m, uint64_t n,
                              uint64_t* __restrict__ np) {
  for (uint64_t r = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; r <= n;
       r += uint64_t(gridDim.x) * blockDim.x) {
    uint64_t lo = 0, hi = m;
    const uint64_t key = r << 32;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (skey[mid] < key) lo = mid + 1; else hi = mid;
    }
    np[r] = r == n ? m : lo;
  }
}

inline unsigned blocks(uint64_t n, unsigned bs = 256) {
  return unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n + bs - 1) / bs, 148ull * 64)));
}

int key_bits(uint64_t n) {
  int b = 1;
  while ((1ull << b) < n + 1) ++b;
  return 32 + b;
}

template <class F>
void cub_call(F&& f, cudaStream_t s) {
  size_t bytes = 0;
  CU(f(nullptr, bytes));
  DevBuf tmp(std::max<size_t>(bytes, 16));
  CU(f(tmp.p, bytes));
  CU(cudaStreamSynchronize(s));
}

}  // namespace

sgtk_csr* normalize_graph(const uint64_t* np_in, const uint32_t* el_in, const float* vals_in,
                          uint64_t n, uint64_t E, int symmetrize, int loops, int dedupe, int kind,
                          cudaStream_t s) {
  if (n > 0xFFFFFFFFull || E > 0x7FFFFFFFull)
    raise(SGTK_ERR_OVERFLOW, "normalize_graph: graph exceeds 32-bit ids / 2^31 edges");
  const auto dir = kind == SGTK_PTR_DEVICE ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice;
  const bool weighted = vals_in != nullptr;
  DevBuf np((n + 1) * 8), el(std::max<uint64_t>(E, 1) * 4), vin(weighted ? std::max<uint64_t>(E, 1) * 4 : 0);
  CU(cudaMemcpyAsync(np.p, np_in, (n + 1) * 8, dir, s));
  if (E) CU(cudaMemcpyAsync(el.p, el_in, E * 4, dir, s));
  if (weighted && E) CU(cudaMemcpyAsync(vin.p, vals_in, E * 4, dir, s));
  // CSR sanity (validate_csr(g, false), graph_io.cpp:196)
  uint64_t h_end = 0;
  CU(cudaMemcpyAsync(&h_end, np.as<uint64_t>() + n, 8, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (h_end != E) raise(SGTK_ERR, "csr: node_pointer end does not match edge count");

  const int bits = key_bits(n);
  DevBuf k0(std::max<uint64_t>(E, 1) * 8), k1(std::max<uint64_t>(E, 1) * 8);
  DevBuf i0(std::max<uint64_t>(E, 1) * 4), i1(std::max<uint64_t>(E, 1) * 4);
  uint64_t U = 0;
  DevBuf bkey(std::max<uint64_t>(E, 1) * 8), bval(std::max<uint64_t>(E, 1) * 4);
  if (E) {
    keys_kernel<<<blocks(n * 32), 256, 0, s>>>(np.as<uint64_t>(), el.as<uint32_t>(), n,
                                               k0.as<uint64_t>(), i0.as<uint32_t>());
    CU_LAUNCH("keys_kernel");
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, k0.as<uint64_t>(), k1.as<uint64_t>(),
                                             i0.as<uint32_t>(), i1.as<uint32_t>(), int(E), 0, bits, s);
    }, s);
    DevBuf head(E * 4), incl(E * 4);
    heads_kernel<<<blocks(E), 256, 0, s>>>(k1.as<uint64_t>(), E, dedupe, head.as<uint32_t>());
    CU_LAUNCH("heads_kernel");
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceScan::InclusiveSum(t, b, head.as<uint32_t>(), incl.as<uint32_t>(), int(E), s);
    }, s);
    uint32_t hu = 0;
    CU(cudaMemcpyAsync(&hu, incl.as<uint32_t>() + E - 1, 4, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    U = hu;
    runs_kernel<<<blocks(E), 256, 0, s>>>(k1.as<uint64_t>(), i1.as<uint32_t>(), incl.as<uint32_t>(),
                                          E, weighted ? vin.as<float>() : nullptr,
                                          bkey.as<uint64_t>(), weighted ? bval.as<float>() : nullptr);
    CU_LAUNCH("runs_kernel");
  }
  // insertions
  const uint64_t cand = U + n;
  DevBuf flags(std::max<uint64_t>(cand, 1) * 4), pos(std::max<uint64_t>(cand, 1) * 4);
  insert_flags_kernel<<<blocks(cand), 256, 0, s>>>(bkey.as<uint64_t>(), U, n, symmetrize, loops,
                                                   flags.as<uint32_t>());
  CU_LAUNCH("insert_flags_kernel");
  uint64_t added = 0;
  if (cand) {
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceScan::ExclusiveSum(t, b, flags.as<uint32_t>(), pos.as<uint32_t>(), int(cand), s);
    }, s);
    uint32_t lp = 0, lf = 0;
    CU(cudaMemcpyAsync(&lp, pos.as<uint32_t>() + cand - 1, 4, cudaMemcpyDeviceToHost, s));
    CU(cudaMemcpyAsync(&lf, flags.as<uint32_t>() + cand - 1, 4, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    added = uint64_t(lp) + lf;
  }
  const uint64_t M = U + added;
  DevBuf ckey(std::max<uint64_t>(M, 1) * 8), cidx(std::max<uint64_t>(M, 1) * 4),
      cval(weighted ? std::max<uint64_t>(M, 1) * 4 : 0);
  combine_kernel<<<blocks(cand), 256, 0, s>>>(bkey.as<uint64_t>(), bval.as<float>(), U, n,
                                              flags.as<uint32_t>(), pos.as<uint32_t>(),
                                              ckey.as<uint64_t>(), cidx.as<uint32_t>(),
                                              weighted ? cval.as<float>() : nullptr);
  CU_LAUNCH("combine_kernel");
  auto out = std::make_unique<sgtk_csr>();
  out->n = n;
  out->nnz = M;
  out->has_values = weighted;
  out->np.alloc((n + 1) * 8);
  out->el.alloc(std::max<uint64_t>(M, 1) * 4);
  if (weighted) out->vals.alloc(std::max<uint64_t>(M, 1) * 4);
  DevBuf skey(std::max<uint64_t>(M, 1) * 8), sidx(std::max<uint64_t>(M, 1) * 4);
  if (M) {
    cub_call([&](void* t, size_t& b) {
      return cub::DeviceRadixSort::SortPairs(t, b, ckey.as<uint64_t>(), skey.as<uint64_t>(),
                                             cidx.as<uint32_t>(), sidx.as<uint32_t>(), int(M), 0,
                                             bits, s);
    }, s);
    emit_kernel<<<blocks(M), 256, 0, s>>>(skey.as<uint64_t>(), sidx.as<uint32_t>(),
                                          weighted ? cval.as<float>() : nullptr, M,
                                          out->el.as<uint32_t>(),
                                          weighted ? out->vals.as<float>() : nullptr);
    CU_LAUNCH("emit_kernel");
  }
  rowptr_kernel<<<blocks(n + 1), 256, 0, s>>>(skey.as<uint64_t>(), M, n, out->np.as<uint64_t>());
  CU_LAUNCH("rowptr_kernel");
  CU(cudaStreamSynchronize(s));
  return out.release();
}

}  // namespace sgtkcu
