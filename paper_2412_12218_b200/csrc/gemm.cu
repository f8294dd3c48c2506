// Dense update GEMM: out[m x n] = relu?(a[m x k] * w[k x n]).
//
// Replaces the reference's file-static matmul (/root/reference/proj/src/gnn.cpp:16-29)
// used by gcn_forward (gnn.cpp:44) and the AGNN model's projections.
//
// Two implementations:
//   * gemm_tc05 (gemm_tc05.cu): TMA-fed tcgen05.mma kind::tf32 with the
//     accumulator in TMEM — used when the shape/alignment allow it.
//   * this file: a cp.async double-buffered mma.sync m16n8k8 kernel that
//     handles every shape/alignment (odd k, odd n, unaligned leading dims).
// FP32 precision uses the 4-term TF32 split (common.cuh) on both paths.

#include "graph.cuh"
#include "kernels.cuh"

namespace sgtkcu {
namespace {

constexpr int BM = 64, BN = 64, BK = 32, NT = 128;
constexpr int AS = BK + 4;   // padded smem row stride (floats): conflict-free frags
constexpr int WS = BN + 8;

__device__ __forceinline__ void cp_async4(float* dst, const float* src, bool ok) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(d), "l"(src),
               "r"(ok ? 4 : 0));
}
__device__ __forceinline__ void cp_async16(float* dst, const float* src, int bytes) {
  const uint32_t d = static_cast<uint32_t>(__cvta_generic_to_shared(dst));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(d), "l"(src), "r"(bytes));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n"); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

template <int PREC, bool VEC>
__global__ void __launch_bounds__(NT)
gemm_mma_kernel(const float* __restrict__ a, uint64_t lda, const float* __restrict__ w,
                uint64_t m, uint64_t k, uint64_t n, int relu, float* __restrict__ out,
                uint64_t ldo) {
  __shared__ __align__(16) float As[2][BM * AS];
  __shared__ __align__(16) float Ws[2][BK * WS];
  const uint64_t m0 = uint64_t(blockIdx.x) * BM;
  const uint64_t n0 = uint64_t(blockIdx.y) * BN;
  const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31, g = lane >> 2, t = lane & 3;

  auto load_chunk = [&](int buf, uint64_t k0) {
    // A: BM x BK
    if (VEC) {
      for (int i = tid; i < BM * BK / 4; i += NT) {
        const int r = i / (BK / 4), c4 = (i % (BK / 4)) * 4;
        const uint64_t gr = m0 + r, gk = k0 + c4;
        int bytes = 0;
        if (gr < m && gk < k) bytes = int(k - gk < 4 ? k - gk : 4) * 4;
        cp_async16(&As[buf][r * AS + c4], a + (bytes ? gr * lda + gk : 0), bytes);
      }
    } else {
      for (int i = tid; i < BM * BK; i += NT) {
        const int r = i / BK, c = i % BK;
        const uint64_t gr = m0 + r, gk = k0 + c;
        const bool ok = gr < m && gk < k;
        cp_async4(&As[buf][r * AS + c], a + (ok ? gr * lda + gk : 0), ok);
      }
    }
    // W: BK x BN (tiny; 4-byte copies handle any n)
    for (int i = tid; i < BK * BN; i += NT) {
      const int r = i / BN, c = i % BN;
      const uint64_t gk = k0 + r, gn = n0 + c;
      const bool ok = gk < k && gn < n;
      cp_async4(&Ws[buf][r * WS + c], w + (ok ? gk * n + gn : 0), ok);
    }
    cp_commit();
  };

  float acc[BN / 8][4];
#pragma unroll
  for (int j = 0; j < BN / 8; ++j) acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.f;
  const int nblk = int((n - n0 < BN ? n - n0 : BN) + 7) / 8;

  const uint64_t nk = (k + BK - 1) / BK;
  load_chunk(0, 0);
  for (uint64_t kc = 0; kc < nk; ++kc) {
    const int buf = int(kc & 1);
    if (kc + 1 < nk) {
      load_chunk(buf ^ 1, (kc + 1) * BK);
      cp_wait<1>();
    } else {
      cp_wait<0>();
    }
    __syncthreads();
    const float* A = As[buf] + (warp * 16) * AS;
    const float* W = Ws[buf];
#pragma unroll
    for (int kk = 0; kk < BK; kk += 8) {
      uint32_t a0[4], a1[4], a2[4];
      split_d<PREC>(A[g * AS + kk + t], a0[0], a1[0], a2[0]);
      split_d<PREC>(A[(g + 8) * AS + kk + t], a0[1], a1[1], a2[1]);
      split_d<PREC>(A[g * AS + kk + t + 4], a0[2], a1[2], a2[2]);
      split_d<PREC>(A[(g + 8) * AS + kk + t + 4], a0[3], a1[3], a2[3]);
#pragma unroll
      for (int j = 0; j < BN / 8; ++j) {
        if (j >= nblk) break;
        uint32_t b0, c0, b1, c1;
        split_s<PREC>(W[(kk + t) * WS + j * 8 + g], b0, c0);
        split_s<PREC>(W[(kk + t + 4) * WS + j * 8 + g], b1, c1);
        if constexpr (PREC == SGTK_FP32) {
          mma_tf32(acc[j], a2[0], a2[1], a2[2], a2[3], b0, b1);
          mma_tf32(acc[j], a0[0], a0[1], a0[2], a0[3], c0, c1);
          mma_tf32(acc[j], a1[0], a1[1], a1[2], a1[3], b0, b1);
        }
        mma_tf32(acc[j], a0[0], a0[1], a0[2], a0[3], b0, b1);
      }
    }
    __syncthreads();
  }
  // epilogue
  const uint64_t r0 = m0 + warp * 16 + g;
#pragma unroll
  for (int j = 0; j < BN / 8; ++j) {
    if (j >= nblk) break;
    const uint64_t c = n0 + j * 8 + 2 * t;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const uint64_t r = r0 + h * 8;
      if (r >= m) continue;
      float v0 = acc[j][2 * h], v1 = acc[j][2 * h + 1];
      if (relu) { v0 = fmaxf(v0, 0.f); v1 = fmaxf(v1, 0.f); }
      if (c < n) out[r * ldo + c] = v0;
      if (c + 1 < n) out[r * ldo + c + 1] = v1;
    }
  }
}

}  // namespace

bool gemm_tc05_launch(const float* a, uint64_t lda, const float* w, uint64_t m, uint64_t k,
                      uint64_t n, int relu, int prec, float* out, uint64_t ldo, cudaStream_t s,
                      bool round_tf32, uint32_t* nonfinite);

void gemm_launch(const float* a, uint64_t lda, const float* w, uint64_t m, uint64_t k, uint64_t n,
                 int relu, int prec, float* out, uint64_t ldo, cudaStream_t s, bool round_tf32,
                 uint32_t* nonfinite) {
  if (prec != SGTK_FP32 && prec != SGTK_TF32)
    raise(SGTK_ERR_RANGE, "gemm: precision must be FP32 or TF32");
  if (m == 0 || n == 0) return;
  if (k == 0) {
    CU(cudaMemset2DAsync(out, ldo * 4, 0, n * 4, m, s));
    return;
  }
  if (gemm_tc05_launch(a, lda, w, m, k, n, relu, prec, out, ldo, s, round_tf32, nonfinite)) return;
  const bool vec = lda % 4 == 0 && reinterpret_cast<uintptr_t>(a) % 16 == 0;
  dim3 grid(unsigned((m + BM - 1) / BM), unsigned((n + BN - 1) / BN));
  if (prec == SGTK_FP32) {
    if (vec) gemm_mma_kernel<SGTK_FP32, true><<<grid, NT, 0, s>>>(a, lda, w, m, k, n, relu, out, ldo);
    else gemm_mma_kernel<SGTK_FP32, false><<<grid, NT, 0, s>>>(a, lda, w, m, k, n, relu, out, ldo);
  } else {
    if (vec) gemm_mma_kernel<SGTK_TF32, true><<<grid, NT, 0, s>>>(a, lda, w, m, k, n, relu, out, ldo);
    else gemm_mma_kernel<SGTK_TF32, false><<<grid, NT, 0, s>>>(a, lda, w, m, k, n, relu, out, ldo);
  }
  CU_LAUNCH("gemm_mma_kernel");
  // outside the tcgen05 envelope: the epilogue options as separate passes
  // (round_tf32 is for internal buffers: the pass also rounds the padding
  // columns between rows)
  if (round_tf32) tf32_launch(out, out, (m - 1) * ldo + n, s);
  if (nonfinite) relu_nonfinite_launch(out, m, n, ldo, 0, nonfinite, s);
}

}  // namespace sgtkcu
