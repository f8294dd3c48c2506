// Probe: TMA tile::gather4 (fp32, SWIZZLE_128B_ATOM_32B) straight into the
// UMMA MN-major TF32 B layout, then D = A * B on tcgen05 vs a host product.
//   nvcc -gencode arch=compute_100a,code=sm_100a -I paper_2412_12218_b200/csrc -I include tools/gather4_probe.cu -o tools/gather4_probe -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "tc05.cuh"
using namespace sgtkcu::tc05;

__device__ __forceinline__ void gather4(uint32_t dst, const CUtensorMap* map, int c0, int r0, int r1, int r2, int r3, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(dst), "l"(map), "r"(c0), "r"(r0), "r"(r1), "r"(r2), "r"(r3),
      "r"(smem_u32(bar))
      : "memory");
}

template <int DC>
__global__ void probe(const __grid_constant__ CUtensorMap tmX, const int* rows, const float* A, float* D) {
  extern __shared__ uint8_t raw[];
  uint8_t* sm = raw + ((1024u - (smem_u32(raw) & 1023u)) & 1023u);
  uint8_t* sa = sm;
  uint8_t* sb = sm + 16384;
  __shared__ uint64_t bar, bar2;
  __shared__ uint32_t slot;
  const uint32_t tid = threadIdx.x, warp = tid >> 5;
  for (uint32_t i = tid; i < 128 * 32; i += 128) {
    const uint32_t row = i / 32, k = i % 32;
    const uint32_t off = (row >> 3) * 1024u + (row & 7u) * 128u + (((k >> 2) ^ (row & 7u)) << 4) + (k & 3u) * 4u;
    *reinterpret_cast<float*>(sa + off) = A[i];
  }
  if (tid == 0) { mbar_init(&bar, 1); mbar_init(&bar2, 1); mbar_init_fence(); }
  if (warp == 0) tmem_alloc(&slot, 512);
  fence_async_smem();
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  if (tid == 0) {
    mbar_expect_tx(&bar, 32 * DC * 4);
    for (int nb = 0; nb < DC / 32; ++nb)
      for (int g = 0; g < 8; ++g)
        gather4(smem_u32(sb) + nb * 4096 + g * 512, &tmX, nb * 32, rows[4 * g], rows[4 * g + 1], rows[4 * g + 2], rows[4 * g + 3], &bar);
  }
  mbar_wait(&bar, 0);
  const uint32_t tmem = slot;
  if (tid == 0) {
    tc_fence_after();
    constexpr uint32_t idesc = idesc_tf32(DC, true);
    for (uint32_t ks = 0; ks < 4; ++ks)
      umma_tf32(tmem, umma_desc(smem_u32(sa) + ks * 32), desc_mn32(smem_u32(sb) + ks * 1024, 4096, 512), idesc, ks ? 1u : 0u);
    umma_commit(&bar2);
  }
  mbar_wait(&bar2, 0);
  tc_fence_after();
  for (int cc = 0; cc < DC; cc += 16) {
    uint32_t v[16];
    tmem_ld16(tmem + ((warp * 32u) << 16) + cc, v);
    tmem_ld_wait();
    for (int j = 0; j < 16; ++j) D[(warp * 32 + (tid & 31)) * DC + cc + j] = __uint_as_float(v[j]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 0) { tc_fence_after(); tmem_dealloc(tmem, 512); }
}

template <int DC>
int run(int boxh, int nrows, int d) {
  std::vector<float> A(128 * 32), X(size_t(nrows) * 72, 0.f), D(128 * DC), R(128 * DC, 0.f);
  std::vector<int> rows(32);
  srand(1);
  for (auto& a : A) a = float(rand() % 7 - 3);
  for (int r = 0; r < nrows; ++r) for (int f = 0; f < d; ++f) X[size_t(r) * 72 + f] = float(rand() % 5 - 2);
  for (int k = 0; k < 32; ++k) rows[k] = (k == 31) ? -1 : rand() % nrows;  // -1: OOB -> zeros
  for (int m = 0; m < 128; ++m)
    for (int n = 0; n < DC; ++n)
      for (int k = 0; k < 32; ++k)
        if (rows[k] >= 0 && n < d) R[m * DC + n] += A[m * 32 + k] * X[size_t(rows[k]) * 72 + n];
  float *dA, *dX, *dD; int* dR;
  cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dX, X.size() * 4); cudaMalloc(&dD, D.size() * 4); cudaMalloc(&dR, 128);
  cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dX, X.data(), X.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(dR, rows.data(), 128, cudaMemcpyHostToDevice);
  cudaMemset(dD, 0, D.size() * 4);
  void* fnp = nullptr; cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fnp, cudaEnableDefault, &q);
  auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fnp);
  CUtensorMap m;
  const cuuint64_t dims[2] = {cuuint64_t(d), cuuint64_t(nrows)};
  const cuuint64_t strides[1] = {72 * 4};
  const cuuint32_t box[2] = {32, cuuint32_t(boxh)};
  const cuuint32_t es[2] = {1, 1};
  CUresult cr = enc(&m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, dX, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  cudaFuncSetAttribute(probe<DC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe<DC><<<1, 128, 48 * 1024>>>(m, dR, dA, dD);
  cudaError_t e = cudaDeviceSynchronize();
  cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
  int bad = 0;
  for (int i = 0; i < 128 * DC; ++i) bad += D[i] != R[i];
  printf("DC=%d boxh=%d d=%d encode=%d: %s, %d/%d mismatches; D0..3=%g %g %g %g want %g %g %g %g\n", DC, boxh, d, int(cr),
         cudaGetErrorString(e), bad, 128 * DC, D[0], D[1], D[2], D[3], R[0], R[1], R[2], R[3]);
  return bad || e != cudaSuccess;
}

int main() {
  int bad = 0;
  bad += run<32>(1, 1000, 32);
  bad += run<64>(1, 1000, 64);
  bad += run<64>(1, 1000, 41);
  return bad;
}
