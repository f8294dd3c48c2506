// Layout probe for the panel kernel's UMMA operands: A K-major SW128
// (128 x 32 tf32), B MN-major SW128 (32 x DC tf32), D in TMEM.  Small
// integers (exact in TF32); compares D with a host product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2412_12218_b200/csrc -I include tools/tc05_probe.cu -o tools/tc05_probe
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc05.cuh"

using namespace sgtkcu::tc05;

template <int DC, bool BMN>
__global__ void probe(const float* A, const float* B, float* D, uint32_t lbo, uint32_t sbo, uint32_t kstep) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sa = sm;
  uint8_t* sb = sm + 16384;
  __shared__ uint64_t bar;
  __shared__ uint32_t slot;
  const uint32_t tid = threadIdx.x, warp = tid >> 5;
  // A[m][k]
  for (uint32_t i = tid; i < 128 * 32; i += 128) {
    const uint32_t row = i / 32, k = i % 32;
    const uint32_t off = (row >> 3) * 1024u + (row & 7u) * 128u + (((k >> 2) ^ (row & 7u)) << 4) + (k & 3u) * 4u;
    *reinterpret_cast<float*>(sa + off) = A[i];
  }
  // B[k][n]
  for (uint32_t i = tid; i < 32 * DC; i += 128) {
    const uint32_t k = i / DC, n = i % DC;
    uint32_t off;
    if (BMN) {
      // SW128_32B atom: 4 K-rows x 128 B, 32-byte chunks XOR (k % 4)
      const uint32_t c = (n % 32) / 8;
      off = (n / 32) * 4096u + (k >> 2) * 512u + (k & 3u) * 128u + ((c ^ (k & 3u)) << 5) + (n & 7u) * 4u;
    } else {  // K-major: row n, 32 k's
      off = (n >> 3) * 1024u + (n & 7u) * 128u + (((k >> 2) ^ (n & 7u)) << 4) + (k & 3u) * 4u;
    }
    *reinterpret_cast<float*>(sb + off) = B[i];
  }
  if (tid == 0) {
    mbar_init(&bar, 1);
    mbar_init_fence();
  }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = slot;
  if (tid == 0) {
    constexpr uint32_t idesc = idesc_tf32(DC, BMN);
    for (uint32_t ks = 0; ks < 4; ++ks) {
      const uint64_t ad = umma_desc(smem_u32(sa) + ks * 32);
      const uint64_t bd = BMN ? desc_mn32(smem_u32(sb) + ks * kstep, lbo, sbo)
                              : umma_desc(smem_u32(sb) + ks * 32);
      umma_tf32(tmem, ad, bd, idesc, ks ? 1u : 0u);
    }
    umma_commit(&bar);
  }
  mbar_wait(&bar, 0);
  tc_fence_after();
  for (int cc = 0; cc < DC; cc += 16) {
    uint32_t v[16];
    tmem_ld16(tmem + ((warp * 32u) << 16) + cc, v);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) D[(warp * 32 + (tid & 31)) * DC + cc + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) {
    tc_fence_after();
    tmem_dealloc(tmem, 512);
  }
}

template <int DC, bool BMN>
int run(uint32_t lbo = 4096, uint32_t sbo = 1024, uint32_t kstep = 1024) {
  std::vector<float> A(128 * 32), B(32 * DC), D(128 * DC), R(128 * DC, 0.f);
  srand(1);
  for (auto& a : A) a = float(rand() % 7 - 3);
  for (auto& b : B) b = float(rand() % 5 - 2);
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < DC; ++n)
      for (int k = 0; k < 32; ++k) R[m * DC + n] += A[m * 32 + k] * B[k * DC + n];
  float *dA, *dB, *dD;
  cudaMalloc(&dA, A.size() * 4);
  cudaMalloc(&dB, B.size() * 4);
  cudaMalloc(&dD, D.size() * 4);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, D.size() * 4);
  cudaFuncSetAttribute(probe<DC, BMN>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  cudaMemset(dD, 0, D.size() * 4);
  probe<DC, BMN><<<1, 128, 48 * 1024>>>(dA, dB, dD, lbo, sbo, kstep);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < 128 * DC; ++i) bad += D[i] != R[i];
  printf("lbo=%u sbo=%u kstep=%u DC=%d B_MN=%d: %s, %d/%d mismatches; D[0..3]=%g %g %g %g want %g %g %g %g\n", lbo, sbo, kstep, DC, BMN,
         cudaGetErrorString(e), bad, 128 * DC, D[0], D[1], D[2], D[3], R[0], R[1], R[2], R[3]);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dD);
  return bad;
}

int main() {
  int bad = run<32, false>();
  bad += run<32, true>(4096, 512, 1024);
  bad += run<32, true>(512, 4096, 1024);
  bad += run<64, true>(4096, 512, 1024);
  bad += run<64, true>(512, 4096, 1024);
  return bad ? 1 : 0;
}
