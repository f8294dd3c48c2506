// Gather roofline probe: how fast can B200 fetch random 128/256-byte feature
// rows (the access pattern of the CUDA-core aggregation kernels) from a table
// that is L2-resident (30 MB, the C4 z/h table) or not (1 GB).  Each warp
// gathers G = 32/LPR rows per instruction with 16-byte lanes, many rows in
// flight, and folds them into a register sum (kept live).  Reports GB/s of
// gathered row bytes.  nvcc -gencode arch=compute_100a,code=sm_100a -O3
// tools/gather_peak.cu -o tools/gather_peak
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>
#include <cuda_runtime.h>

template <int ROWB, int UNROLL>
__global__ void gather_kernel(const float4* __restrict__ table, const uint32_t* __restrict__ idx,
                              uint64_t n_idx, float* __restrict__ sink) {
  constexpr int LPR = ROWB / 16, G = 32 / LPR;
  const uint32_t lane = threadIdx.x & 31, g = lane / LPR, j = lane % LPR;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  float4 acc = make_float4(0.f, 0.f, 0.f, 0.f);
  for (uint64_t b = warp * G * UNROLL; b < n_idx; b += nw * G * UNROLL) {
    float4 v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const uint64_t i = b + u * G + g;
      v[u] = i < n_idx ? __ldg(table + uint64_t(idx[i]) * LPR + j) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      acc.x += v[u].x; acc.y += v[u].y; acc.z += v[u].z; acc.w += v[u].w;
    }
  }
  if (acc.x + acc.y + acc.z + acc.w == 12345.678f) sink[0] = acc.x;
}

template <int ROWB>
double run(uint64_t rows, uint64_t n_idx) {
  float4* table;
  uint32_t* idx;
  float* sink;
  cudaMalloc(&table, rows * ROWB);
  cudaMemset(table, 0, rows * ROWB);
  cudaMalloc(&idx, n_idx * 4);
  cudaMalloc(&sink, 4);
  std::vector<uint32_t> h(n_idx);
  std::mt19937_64 rng(1);
  for (auto& x : h) x = uint32_t(rng() % rows);
  cudaMemcpy(idx, h.data(), n_idx * 4, cudaMemcpyHostToDevice);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int grid = sms * 8;
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (int w = 0; w < 3; ++w) gather_kernel<ROWB, 8><<<grid, 256>>>(table, idx, n_idx, sink);
  cudaEventRecord(a);
  const int iters = 10;
  for (int w = 0; w < iters; ++w) gather_kernel<ROWB, 8><<<grid, 256>>>(table, idx, n_idx, sink);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms = 0;
  cudaEventElapsedTime(&ms, a, b);
  cudaFree(table);
  cudaFree(idx);
  cudaFree(sink);
  const double bytes = double(n_idx) * ROWB + double(n_idx) * 4;  // rows + indices
  return bytes / (ms / iters * 1e-3) / 1e9;
}

int main() {
  const uint64_t n_idx = 16ull << 20;  // 16M gathers per launch
  printf("{\"gather_gbs\": {\"row128_table30MB\": %.1f, \"row256_table34MB\": %.1f, "
         "\"row128_table1GB\": %.1f}}\n",
         run<128>(232965, n_idx), run<256>(132534, n_idx), run<128>(8ull << 20, n_idx));
  return 0;
}
