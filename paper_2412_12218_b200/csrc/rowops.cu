// Row-segmented CUDA-core kernels of the AGNN chain and preprocessing:
//   edge_softmax        gnn.cpp:54-72
//   l2_normalize_rows   gnn.cpp:74-91
//   gcn_normalize_values graph_io.cpp:261-277
//   tf32_round          tile_exec.cpp:131-148
// All are HBM-bound streams; one warp (or a group of lanes) per CSR row,
// coalesced over the row's contiguous edges / features.

#include "graph.cuh"

namespace sgtkcu {
namespace {

__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xFFFFFFFFu, v, o));
  return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}
__device__ __forceinline__ double warp_sum_d(double v) {
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xFFFFFFFFu, v, o);
  return v;
}

// Warp per row.  max, exp(l - max) (accurate expf, as the reference's
// std::exp), sum, divide.  Empty rows are skipped (gnn.cpp:61).
__global__ void edge_softmax_kernel(const uint64_t* __restrict__ np, uint64_t n,
                                    const float* __restrict__ logits, float* __restrict__ out) {
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t r = warp; r < n; r += nwarps) {
    const uint64_t lo = np[r], hi = np[r + 1];
    if (lo == hi) continue;
    if (hi - lo <= 32) {
      const bool act = lo + lane < hi;
      const float l = act ? logits[lo + lane] : -INFINITY;
      const float mx = warp_max(l);
      const float ex = act ? expf(l - mx) : 0.0f;
      const float sum = warp_sum(ex);
      if (act) out[lo + lane] = ex / sum;
    } else {
      float mx = -INFINITY;
      for (uint64_t e = lo + lane; e < hi; e += 32) mx = fmaxf(mx, logits[e]);
      mx = warp_max(mx);
      float sum = 0.0f;
      for (uint64_t e = lo + lane; e < hi; e += 32) sum += expf(logits[e] - mx);
      sum = warp_sum(sum);
      for (uint64_t e = lo + lane; e < hi; e += 32) out[e] = expf(logits[e] - mx) / sum;
    }
  }
}

// Warp per row: fp64 sum of squares, inv = float(1/sqrt(sq)); zero rows
// stay zero and are counted (integer atomic: order-free).
__global__ void l2norm_kernel(const float* __restrict__ h, uint64_t rows, uint64_t cols,
                              uint64_t ldh, float* __restrict__ z, uint64_t ldz,
                              float* __restrict__ inv_out, unsigned long long* __restrict__ zeros) {
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  unsigned long long nz = 0;
  for (uint64_t r = warp; r < rows; r += nwarps) {
    const float* src = h + r * ldh;
    double sq = 0.0;
    for (uint64_t k = lane; k < cols; k += 32) sq += double(src[k]) * double(src[k]);
    sq = warp_sum_d(sq);
    const float inv = sq == 0.0 ? 0.0f : float(1.0 / sqrt(sq));
    if (sq == 0.0) ++nz;
    if (inv_out && lane == 0) inv_out[r] = inv;
    if (z) {
      float* dst = z + r * ldz;
      for (uint64_t k = lane; k < cols; k += 32) dst[k] = src[k] * inv;
    }
  }
  if (zeros && lane == 0 && nz) atomicAdd(zeros, nz);
}

__global__ void isd_kernel(const uint64_t* __restrict__ np, uint64_t n, double* __restrict__ isd,
                           uint32_t* __restrict__ bad) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t deg = np[i + 1] - np[i];
    if (deg == 0) atomicOr(bad, 1u);
    isd[i] = deg ? 1.0 / sqrt(double(deg)) : 0.0;
  }
}

__global__ void gcn_values_kernel(const uint64_t* __restrict__ np, const uint32_t* __restrict__ el,
                                  uint64_t n, const double* __restrict__ isd,
                                  float* __restrict__ vals) {
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t r = warp; r < n; r += nwarps) {
    const double di = isd[r];
    for (uint64_t e = np[r] + lane; e < np[r + 1]; e += 32) vals[e] = float(di * isd[el[e]]);
  }
}

__global__ void tf32_kernel(const float* __restrict__ in, float* __restrict__ out, uint64_t n) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    out[i] = tf32_rne(in[i]);
}

inline unsigned blocks_for(uint64_t threads, unsigned bs = 256) {
  uint64_t b = (threads + bs - 1) / bs;
  return unsigned(std::max<uint64_t>(1, std::min<uint64_t>(b, 148ull * 64)));
}

}  // namespace

void csr_softmax_launch(const uint64_t* np, uint64_t n, const float* logits, float* out,
                        cudaStream_t s) {
  if (!n) return;
  edge_softmax_kernel<<<blocks_for(n * 32), 256, 0, s>>>(np, n, logits, out);
  CU_LAUNCH("edge_softmax_kernel");
}

void edge_softmax_launch(const sgtk_graph* g, const float* logits, float* out, cudaStream_t s) {
  if (!g->n_rows || !g->nnz) return;
  csr_softmax_launch(g->np->as<uint64_t>(), g->n_rows, logits, out, s);
}

void l2norm_launch(const float* h, uint64_t rows, uint64_t cols, uint64_t ldh, float* z,
                   uint64_t ldz, float* inv, uint64_t* zeros, cudaStream_t s) {
  if (!rows) return;
  l2norm_kernel<<<blocks_for(rows * 32), 256, 0, s>>>(h, rows, cols, ldh, z, ldz, inv,
                                                     reinterpret_cast<unsigned long long*>(zeros));
  CU_LAUNCH("l2norm_kernel");
}

void gcn_normalize_launch(const uint64_t* np, const uint32_t* el, uint64_t n, float* vals,
                          cudaStream_t s) {
  if (!n) return;
  DevBuf isd(n * 8), bad(4);
  CU(cudaMemsetAsync(bad.p, 0, 4, s));
  isd_kernel<<<blocks_for(n), 256, 0, s>>>(np, n, isd.as<double>(), bad.as<uint32_t>());
  CU_LAUNCH("isd_kernel");
  uint32_t hbad = 0;
  CU(cudaMemcpyAsync(&hbad, bad.p, 4, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  if (hbad) raise(SGTK_ERR_DEGREE, "gcn_normalize_values: a row has no edges");
  gcn_values_kernel<<<blocks_for(n * 32), 256, 0, s>>>(np, el, n, isd.as<double>(), vals);
  CU_LAUNCH("gcn_values_kernel");
  CU(cudaStreamSynchronize(s));
}

void tf32_launch(const float* in, float* out, uint64_t n, cudaStream_t s) {
  if (!n) return;
  tf32_kernel<<<blocks_for(n), 256, 0, s>>>(in, out, n);
  CU_LAUNCH("tf32_kernel");
}

}  // namespace sgtkcu
