// Dense update GEMM on the 5th-gen tensor cores: TMA -> smem -> tcgen05.mma
// (kind::tf32) -> TMEM -> epilogue.  Replaces the reference's serial ikj
// matmul (/root/reference/proj/src/gnn.cpp:16-29) for gcn_forward's update
// step and the AGNN model projections.
//
// out[m x n] = relu?(a[m x k] * w[k x n]), n <= 128, lda % 4 == 0.
//
// CTA = 6 warps, one 128-row output tile (M = 128, N = n rounded up to 16):
//   warp 0        TMA producer: A tile 128 x 32 fp32 (128-byte rows,
//                 SWIZZLE_128B) + the pre-split W^T planes, S-stage ring
//   warps 2..5    operand preparation per stage (generic proxy, in smem):
//                   TF32: A <- RNE(A) in place (tf32_round_value semantics)
//                   FP32: A -> A0 + A1 + A2 (11+11+2-bit exact split)
//                 then fence.proxy.async and arrive; after the K loop the
//                 same warps are the epilogue (tcgen05.ld 32x32b, ReLU / TF32
//                 rounding / non-finite check, rows staged in smem, coalesced
//                 float4 stores)
//   warp 1        TMEM allocator + single-thread MMA issuer:
//                   TF32: D += A W0            (per 8-wide k step)
//                   FP32: D += A2 W0 + A0 W1 + A1 W0 + A0 W0   (4-term split,
//                         exact when W is TF32-representable, common.cuh)
//                 tcgen05.commit frees the stage / signals the epilogue.
// W (k x n, small, shared by all CTAs) is transposed and split once per call
// into K-major planes W^T[p][n_pad][k_pad].

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cstdlib>
#include <mutex>

#include "kernels.cuh"

namespace sgtkcu {
namespace {

constexpr int kBM = 128;     // UMMA M
constexpr int kBK = 32;      // fp32 per 128-byte swizzle row
constexpr int kThreads = 192;

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n\t}" ::"r"(smem_u32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int c0, int c1,
                                            uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes "
      "[%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(map), "r"(c0), "r"(c1), "r"(smem_u32(bar))
      : "memory");
}

// UMMA shared-memory descriptor: K-major, SWIZZLE_128B, 8-row core-matrix
// groups 1024 bytes apart (mma_sm100_desc.hpp SmemDescriptor layout).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr & 0x3FFFFu) >> 4);  // start address  [0,14)
  d |= uint64_t(1) << 16;                  // LBO (unused for swizzled K-major)
  d |= uint64_t(1024 >> 4) << 32;          // SBO             [32,46)
  d |= uint64_t(1) << 46;                  // version = 1 (sm100)
  d |= uint64_t(2) << 61;                  // SWIZZLE_128B
  return d;
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void umma_commit(uint64_t* bar) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          smem_u32(bar))
      : "memory");
}

template <int PREC>
__global__ void __launch_bounds__(kThreads, 1)
gemm_tc05_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmW,
                 uint64_t m, uint32_t n, uint32_t n_pad, uint32_t num_kc, int relu, int round_tf32,
                 float* __restrict__ out, uint64_t ldo, uint32_t stages, uint32_t tmem_cols,
                 uint32_t* __restrict__ nonfinite, uint32_t region_bytes, int vec_out,
                 uint32_t kc_per, uint64_t split_stride) {
  constexpr int P_A = PREC == SGTK_FP32 ? 3 : 1;  // A planes
  constexpr int P_W = PREC == SGTK_FP32 ? 2 : 1;  // W planes
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~uintptr_t(1023));
  const uint32_t a_bytes = kBM * kBK * 4;      // 16 KB
  const uint32_t w_bytes = n_pad * kBK * 4;    // n_pad x 128 B
  const uint32_t stage_bytes = (P_A * a_bytes + P_W * w_bytes + 1023) & ~1023u;
  // [ring | epilogue tile] region, then the barriers
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + region_bytes);
  uint64_t* conv = full + stages;
  uint64_t* empty = conv + stages;
  uint64_t* tmem_full = empty + stages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t m0 = uint64_t(blockIdx.x) * kBM;
  // split K (grid.y > 1): this CTA's K chunks; its raw sums go to its own
  // slice of the workspace (out + blockIdx.y * split_stride)
  const uint32_t kc0 = blockIdx.y * kc_per;
  const uint32_t nk = min(num_kc, kc0 + kc_per) - kc0;
  out += blockIdx.y * split_stride;

  if (warp == 0 && lane == 0) {
    for (uint32_t s = 0; s < stages; ++s) {
      mbar_init(full + s, 1);
      mbar_init(conv + s, 4);  // one arrive per preparation warp
      mbar_init(empty + s, 1);
    }
    mbar_init(tmem_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmW) : "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(tmem_cols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;");
  const uint32_t tmem_d = *tmem_slot;

  if (warp == 0) {
    // ---------------- TMA producer ----------------------------------------
    if (lane == 0) {
      for (uint32_t i = 0; i < nk; ++i) {
        const uint32_t kc = kc0 + i, s = i % stages, ph = (i / stages) & 1u;
        mbar_wait(empty + s, ph ^ 1u);
        uint8_t* st = smem + s * stage_bytes;
        mbar_expect_tx(full + s, a_bytes + P_W * w_bytes);
        tma_load_2d(st, &tmA, int(kc * kBK), int(m0), full + s);
#pragma unroll
        for (int p = 0; p < P_W; ++p)
          tma_load_2d(st + P_A * a_bytes + p * w_bytes, &tmW, int(kc * kBK), int(p * n_pad),
                      full + s);
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer (one thread) ------------------------------
    if (lane == 0) {
      const uint32_t idesc = (1u << 4)            // D format F32
                             | (2u << 7)          // A format TF32
                             | (2u << 10)         // B format TF32
                             | ((n_pad >> 3) << 17) | ((uint32_t(kBM) >> 4) << 24);
      for (uint32_t i = 0; i < nk; ++i) {
        const uint32_t s = i % stages, ph = (i / stages) & 1u;
        mbar_wait(conv + s, ph);
        asm volatile("tcgen05.fence::after_thread_sync;");
        const uint32_t base = smem_u32(smem + s * stage_bytes);
        const uint32_t a0 = base, a1 = base + a_bytes, a2 = base + 2 * a_bytes;
        const uint32_t w0 = base + P_A * a_bytes, w1 = w0 + w_bytes;
#pragma unroll
        for (uint32_t ks = 0; ks < kBK / 8; ++ks) {
          const uint32_t off = ks * 32;  // 8 tf32 = 32 bytes along K inside the swizzle row
          const uint32_t acc0 = (i | ks) ? 1u : 0u;
          if constexpr (PREC == SGTK_FP32) {
            umma_tf32(tmem_d, umma_desc(a2 + off), umma_desc(w0 + off), idesc, acc0);
            umma_tf32(tmem_d, umma_desc(a0 + off), umma_desc(w1 + off), idesc, 1u);
            umma_tf32(tmem_d, umma_desc(a1 + off), umma_desc(w0 + off), idesc, 1u);
            umma_tf32(tmem_d, umma_desc(a0 + off), umma_desc(w0 + off), idesc, 1u);
          } else {
            umma_tf32(tmem_d, umma_desc(a0 + off), umma_desc(w0 + off), idesc, acc0);
          }
        }
        umma_commit(empty + s);  // frees the stage once these MMAs retire
      }
      umma_commit(tmem_full);
    }
  } else {
    // ---------------- operand preparation (warps 2..5) ---------------------
    const uint32_t tid = threadIdx.x - 64;  // 0..127
    for (uint32_t i = 0; i < nk; ++i) {
      const uint32_t s = i % stages, ph = (i / stages) & 1u;
      mbar_wait(full + s, ph);
      uint8_t* st = smem + s * stage_bytes;
      uint4* A = reinterpret_cast<uint4*>(st);
#pragma unroll 4
      for (uint32_t i = tid; i < a_bytes / 16; i += 128) {
        uint4 v = A[i];
        if constexpr (PREC == SGTK_FP32) {
          uint32_t x[4] = {v.x, v.y, v.z, v.w}, p0[4], p1[4], p2[4];
#pragma unroll
          for (int j = 0; j < 4; ++j) split3(__uint_as_float(x[j]), p0[j], p1[j], p2[j]);
          A[i] = make_uint4(p0[0], p0[1], p0[2], p0[3]);
          reinterpret_cast<uint4*>(st + a_bytes)[i] = make_uint4(p1[0], p1[1], p1[2], p1[3]);
          reinterpret_cast<uint4*>(st + 2 * a_bytes)[i] = make_uint4(p2[0], p2[1], p2[2], p2[3]);
        } else {
          A[i] = make_uint4(tf32_op(__uint_as_float(v.x)), tf32_op(__uint_as_float(v.y)),
                            tf32_op(__uint_as_float(v.z)), tf32_op(__uint_as_float(v.w)));
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(conv + s);
    }
    // ---------------- epilogue: TMEM -> registers -> smem -> global ---------
    // Each warp stages its 32 rows in shared memory (the ring is idle now) and
    // writes them back row-contiguously: coalesced stores instead of one
    // 4-byte store per row per instruction.
    mbar_wait(tmem_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;");
    const uint32_t quad = warp & 3u;  // TMEM lanes [32*quad, 32*quad + 32)
    const uint32_t tse = n_pad + 4;   // staged row stride (floats): 16-byte aligned, banks spread
    float* tw = reinterpret_cast<float*>(smem) + quad * 32u * tse;
    const uint32_t tws = smem_u32(tw);
    bool bad = false;
    for (uint32_t c0 = 0; c0 < n_pad; c0 += 16) {
      uint32_t r[16];
      const uint32_t taddr = tmem_d + ((quad * 32u) << 16) + c0;
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
          "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
            "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]),
            "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(taddr));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      const bool rv = m0 + quad * 32 + lane < m;
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        float v = __uint_as_float(r[j]);
        if (relu) v = fmaxf(v, 0.0f);
        if (round_tf32) v = tf32_rne(v);  // consumer: a TF32 SpMM (same RNE it would apply)
        bad |= rv && c0 + j < n && !isfinite(v);
        r[j] = __float_as_uint(v);
      }
#pragma unroll
      for (int j = 0; j < 4; ++j)
        asm volatile("st.shared.v4.b32 [%0], {%1, %2, %3, %4};" ::"r"(tws + (lane * tse + c0 + 4 * j) * 4),
                     "r"(r[4 * j]), "r"(r[4 * j + 1]), "r"(r[4 * j + 2]), "r"(r[4 * j + 3])
                     : "memory");
    }
    __syncwarp();
    const uint64_t rbase = m0 + quad * 32;
    if (vec_out) {  // n % 4 == 0, 16-byte aligned rows
      const uint32_t n4 = n / 4;
      for (uint32_t i = lane; i < 32 * n4; i += 32) {
        const uint32_t rr = i / n4, cc = i - rr * n4;
        if (rbase + rr < m)
          reinterpret_cast<float4*>(out + (rbase + rr) * ldo)[cc] =
              *reinterpret_cast<const float4*>(tw + rr * tse + 4 * cc);
      }
    } else {
      for (uint32_t i = lane; i < 32 * n; i += 32) {
        const uint32_t rr = i / n, cc = i - rr * n;
        if (rbase + rr < m) out[(rbase + rr) * ldo + cc] = tw[rr * tse + cc];
      }
    }
    if (nonfinite && __any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(nonfinite, 1u);
  }
  asm volatile("tcgen05.fence::before_thread_sync;");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_d),
                 "r"(tmem_cols));
  }
}

// Split K: out = epilogue(sum over the splits, in split order) of the raw
// per-split sums ws[split][m][n_pad].
__global__ void splitk_reduce_kernel(const float* __restrict__ ws, uint32_t splits, uint64_t m, uint32_t n,
                                     uint32_t n_pad, int relu, int round_tf32, float* __restrict__ out,
                                     uint64_t ldo, uint32_t* __restrict__ nonfinite) {
  bool bad = false;
  const uint64_t total = m * n, stride = m * n_pad;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = i / n, c = i - r * n;
    float v = ws[r * n_pad + c];
    for (uint32_t y = 1; y < splits; ++y) v += ws[y * stride + r * n_pad + c];
    if (relu) v = fmaxf(v, 0.0f);
    if (round_tf32) v = tf32_rne(v);
    bad |= !isfinite(v);
    out[r * ldo + c] = v;
  }
  if (nonfinite && bad) atomicOr(nonfinite, 1u);
}

// W [k x n] row-major -> planes W^T[p][n_pad][k_pad] (TF32: RNE; FP32: split2)
template <int PREC>
__global__ void prep_w_kernel(const float* __restrict__ w, uint64_t k, uint64_t n, uint32_t n_pad,
                              uint32_t k_pad, float* __restrict__ wt) {
  const uint64_t total = uint64_t(n_pad) * k_pad;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t j = i / k_pad, kk = i - j * k_pad;
    const float v = (j < n && kk < k) ? w[kk * n + j] : 0.0f;
    if constexpr (PREC == SGTK_FP32) {
      uint32_t p0, p1;
      split2(v, p0, p1);
      wt[i] = __uint_as_float(p0);
      wt[total + i] = __uint_as_float(p1);
    } else {
      wt[i] = __uint_as_float(tf32_op(v));
    }
  }
}

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

bool make_map(CUtensorMap* map, const void* base, uint64_t inner, uint64_t outer,
              uint64_t row_bytes, uint32_t box_inner, uint32_t box_outer) {
  auto fn = encode_fn();
  if (!fn) return false;
  const cuuint64_t dims[2] = {inner, outer};
  const cuuint64_t strides[1] = {row_bytes};
  const cuuint32_t box[2] = {box_inner, box_outer};
  const cuuint32_t estr[2] = {1, 1};
  return fn(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<void*>(base), dims, strides, box,
            estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
            CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int device_sm_major() {
  static int major = -1;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  });
  return major;
}

}  // namespace

// Returns false (caller uses the mma.sync kernel) when the shape is outside
// this kernel's envelope (n > 128).  Rows whose pitch or base the TMA cannot
// address (16-byte multiples; e.g. Cora's K = 1433) are first copied into a
// stream-ordered scratch with a padded pitch (one extra pass over A).
bool gemm_tc05_launch(const float* a, uint64_t lda, const float* w, uint64_t m, uint64_t k,
                      uint64_t n, int relu, int prec, float* out, uint64_t ldo, cudaStream_t s,
                      bool round_tf32, uint32_t* nonfinite) {
  if (getenv("SGTK_DISABLE_TC05")) return false;
  if (n == 0 || n > 128 || m == 0 || k == 0) return false;
  if (device_sm_major() != 10) return false;
  float* staged = nullptr;
  if (lda % 4 != 0 || reinterpret_cast<uintptr_t>(a) % 16 != 0) {
    const uint64_t lds = (k + 3) / 4 * 4;
    CU(cudaMallocAsync(reinterpret_cast<void**>(&staged), m * lds * 4, s));
    CU(cudaMemcpy2DAsync(staged, lds * 4, a, lda * 4, k * 4, m, cudaMemcpyDeviceToDevice, s));
    a = staged;
    lda = lds;
  }
  const uint32_t n_pad = uint32_t((n + 15) / 16 * 16);
  const uint32_t k_pad = uint32_t((k + kBK - 1) / kBK * kBK);
  const int P_A = prec == SGTK_FP32 ? 3 : 1, P_W = prec == SGTK_FP32 ? 2 : 1;
  float* wt = nullptr;
  CU(cudaMallocAsync(reinterpret_cast<void**>(&wt), size_t(P_W) * n_pad * k_pad * 4, s));
  const unsigned pb = unsigned(std::min<uint64_t>((uint64_t(n_pad) * k_pad + 255) / 256, 1024));
  if (prec == SGTK_FP32) prep_w_kernel<SGTK_FP32><<<pb, 256, 0, s>>>(w, k, n, n_pad, k_pad, wt);
  else prep_w_kernel<SGTK_TF32><<<pb, 256, 0, s>>>(w, k, n, n_pad, k_pad, wt);
  CU_LAUNCH("prep_w_kernel");
  CUtensorMap ma, mw;
  bool ok = make_map(&ma, a, k, m, lda * 4, kBK, kBM) &&
            make_map(&mw, wt, k_pad, uint64_t(P_W) * n_pad, uint64_t(k_pad) * 4, kBK, n_pad);
  if (!ok) {
    CU(cudaFreeAsync(wt, s));
    if (staged) CU(cudaFreeAsync(staged, s));
    return false;
  }
  const uint32_t a_bytes = kBM * kBK * 4, w_bytes = n_pad * kBK * 4;
  const uint32_t stage_bytes = (P_A * a_bytes + P_W * w_bytes + 1023) & ~1023u;
  const uint32_t num_kc = uint32_t(k_pad / kBK);
  // a ring deeper than the K loop only costs residency: small K (the GCN
  // hidden layers, K = 64) then fits 4 CTAs per SM instead of 2
// 3 stages: more CTAs per SM beat a deeper ring (in-proj 602->32: 2-3 stages
// 0.130 ms, 4 0.134, 6-8 0.16)
#ifndef SGTK_GEMM_STAGES
#define SGTK_GEMM_STAGES 3
#endif
  const uint32_t stages =
      std::max(2u, std::min(std::min(uint32_t(SGTK_GEMM_STAGES), num_kc), (200u * 1024u) / stage_bytes));
  const uint32_t tile_bytes = kBM * (n_pad + 4) * 4;  // staged epilogue tile
  const uint32_t region = (std::max(stages * stage_bytes, tile_bytes) + 1023) & ~1023u;
  const size_t smem = size_t(region) + 1024 /*align*/ + 256 /*barriers*/;
  const int vec_out = n % 4 == 0 && ldo % 4 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0;
  uint32_t tmem_cols = 32;
  while (tmem_cols < n_pad) tmem_cols <<= 1;
  // Split K when the row tiles leave most SMs idle (Cora's 1433 -> 16: 22
  // tiles): each split's CTA takes >= 4 K chunks; raw sums to a workspace,
  // reduced in split order by splitk_reduce_kernel (deterministic)
  const uint64_t mtiles = (m + kBM - 1) / kBM;
#ifndef SGTK_GEMM_SPLITK
#define SGTK_GEMM_SPLITK 1
#endif
  uint32_t splits = 1;
  if (SGTK_GEMM_SPLITK && mtiles < 74)
    splits = uint32_t(std::max<uint64_t>(1, std::min<uint64_t>({148 / mtiles, num_kc / 4, 16})));
  const uint32_t kc_per = (num_kc + splits - 1) / splits;
  splits = (num_kc + kc_per - 1) / kc_per;  // no empty split
  float* ws = nullptr;
  if (splits > 1) CU(cudaMallocAsync(reinterpret_cast<void**>(&ws), size_t(splits) * m * n_pad * 4, s));
  float* kout = splits > 1 ? ws : out;
  const uint64_t kldo = splits > 1 ? n_pad : ldo;
  const int krelu = splits > 1 ? 0 : relu, kround = splits > 1 ? 0 : int(round_tf32);
  uint32_t* knf = splits > 1 ? nullptr : nonfinite;
  const int kvec = splits > 1 ? 1 : vec_out;
  const uint64_t sstride = splits > 1 ? m * n_pad : 0;
  dim3 grid(unsigned(mtiles), splits);
  // the opt-in smem ceiling is set once per kernel (host overhead, not per call)
  once_per_device(reinterpret_cast<const void*>(&gemm_tc05_kernel<SGTK_FP32>), [] {
    cudaFuncSetAttribute(gemm_tc05_kernel<SGTK_FP32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
    cudaFuncSetAttribute(gemm_tc05_kernel<SGTK_TF32>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         227 * 1024);
  });
  const uint32_t kn = splits > 1 ? n_pad : uint32_t(n);
  if (prec == SGTK_FP32) {
    gemm_tc05_kernel<SGTK_FP32><<<grid, kThreads, smem, s>>>(ma, mw, m, kn, n_pad, num_kc, krelu, kround,
                                                             kout, kldo, stages, tmem_cols, knf, region, kvec,
                                                             kc_per, sstride);
  } else {
    gemm_tc05_kernel<SGTK_TF32><<<grid, kThreads, smem, s>>>(ma, mw, m, kn, n_pad, num_kc, krelu, kround,
                                                             kout, kldo, stages, tmem_cols, knf, region, kvec,
                                                             kc_per, sstride);
  }
  CU_LAUNCH("gemm_tc05_kernel");
  if (splits > 1) {
    const unsigned rb = unsigned(std::min<uint64_t>((m * n + 255) / 256, 148ull * 8));
    splitk_reduce_kernel<<<rb, 256, 0, s>>>(ws, splits, m, uint32_t(n), n_pad, relu, int(round_tf32), out, ldo,
                                            nonfinite);
    CU_LAUNCH("splitk_reduce_kernel");
    CU(cudaFreeAsync(ws, s));
  }
  CU(cudaFreeAsync(wt, s));
  if (staged) CU(cudaFreeAsync(staged, s));
  return true;
}

}  // namespace sgtkcu
