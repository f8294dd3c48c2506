// Microbenchmark: back-to-back tcgen05.mma kind::tf32 (M=128, K=8) issue
// rate for K-major vs MN-major B and N = 32/64/128.
#include <cstdio>
#include "tc05.cuh"
using namespace sgtkcu::tc05;

template <int N, bool BMN, bool AMN, int CPER = 0>
__global__ void rate(long long* out, int iters) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar, bar2[4];
  __shared__ uint32_t slot;
  const uint32_t tid = threadIdx.x, warp = tid >> 5;
  for (uint32_t i = tid; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 1.0f;
  if (tid == 0) { mbar_init(&bar, 1); for (int q = 0; q < 4; ++q) mbar_init(bar2 + q, 1); mbar_init_fence(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    constexpr uint32_t idesc = idesc_tf32(N, BMN) | (AMN ? (1u << 15) : 0u);
    const uint32_t a = smem_u32(sm), b = a + 16384;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t ks = i & 3;
      const uint64_t bd = BMN ? desc_mn32(b + ks * 1024, 4096, 512) : umma_desc(b + ks * 32);
      const uint64_t ad = AMN ? desc_mn32(a + ks * 4096, 512, 2048) : umma_desc(a + ks * 32);
      umma_tf32(slot, ad, bd, idesc, i ? 1u : 0u);
      if (CPER && (i & 3) == 3)
        for (int q = 0; q < CPER; ++q) umma_commit(bar2 + q);
    }
    long long t1 = clock64();
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(slot, 512); }
}

template <int N>
__global__ void rate_ts(long long* out, int iters) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const uint32_t tid = threadIdx.x, warp = tid >> 5;
  for (uint32_t i = tid; i < 64 * 1024 / 4; i += blockDim.x) reinterpret_cast<float*>(sm)[i] = 1.0f;
  if (tid == 0) { mbar_init(&bar, 1); mbar_init_fence(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    constexpr uint32_t idesc = idesc_tf32(N, true);
    const uint32_t b = smem_u32(sm) + 16384;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
      const uint32_t ks = i & 3;
      const uint64_t bd = desc_mn32(b + ks * 1024, 4096, 512);
      const uint32_t a_t = slot + 256 + ks * 8;  // A in TMEM columns [256, 288)
      asm volatile(
          "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
          "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n\t}" ::"r"(slot),
          "r"(a_t), "l"(bd), "r"(idesc), "r"(i ? 1u : 0u));
    }
    long long t1 = clock64();
    umma_commit(&bar);
    mbar_wait(&bar, 0);
    long long t2 = clock64();
    out[0] = t1 - t0;
    out[1] = t2 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(slot, 512); }
}

template <int N>
void run_ts(long long* d) {
  cudaFuncSetAttribute(rate_ts<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  rate_ts<N><<<1, 128, 70 * 1024>>>(d, 4000);
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("TS (A in TMEM) N=%3d: issue %.1f cyc/mma, complete %.1f cyc/mma (%s)\n", N, h[0] / 4000.0, h[1] / 4000.0,
         cudaGetErrorString(cudaGetLastError()));
}

template <int N, bool BMN, bool AMN = false, int CPER = 0>
void run(long long* d) {
  cudaFuncSetAttribute(rate<N, BMN, AMN, CPER>, cudaFuncAttributeMaxDynamicSharedMemorySize, 80 * 1024);
  rate<N, BMN, AMN, CPER><<<1, 128, 70 * 1024>>>(d, 4000);
  long long h[2];
  cudaMemcpy(h, d, 16, cudaMemcpyDeviceToHost);
  printf("commits/4mma=%d A_MN=%d N=%3d B_MN=%d: issue %.1f cyc/mma, complete %.1f cyc/mma (%s)\n", CPER, AMN, N, BMN, h[0] / 4000.0, h[1] / 4000.0,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  long long* d;
  cudaMalloc(&d, 16);
  run<32, false>(d); run<32, true>(d);
  run<64, false>(d); run<64, true>(d);
  run<128, false>(d); run<128, true>(d);
  run<32, true, true>(d); run<64, true, true>(d); run<128, true, true>(d);
  run<32, true, false, 1>(d); run<32, true, false, 2>(d); run<32, true, false, 3>(d);
  run_ts<32>(d); run_ts<64>(d); run_ts<128>(d);
  return 0;
}
