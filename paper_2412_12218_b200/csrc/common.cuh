// Shared device/host helpers for the sm_100a FTC-GNN aggregation path.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <functional>
#include <mutex>
#include <set>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "sgtk_cuda.h"

namespace sgtkcu {

// ---------------------------------------------------------------------------
// Host-side error plumbing.  Internal code throws Status; the C ABI catches it
// and returns the code (capi.cpp).  Nothing throws across the C boundary.
// ---------------------------------------------------------------------------
struct Status : std::runtime_error {
  int code;
  Status(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] inline void raise(int code, const std::string& msg) {
  throw Status(code, msg);
}

inline void cuda_check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    raise(SGTK_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define CU(x) ::sgtkcu::cuda_check((x), #x)
#define CU_LAUNCH(what) ::sgtkcu::cuda_check(cudaGetLastError(), what)

inline cudaStream_t as_stream(void* s) { return static_cast<cudaStream_t>(s); }

// Runs fn once per (current device, key) — kernel attributes such as the
// dynamic shared-memory ceiling are per device, so a process driving several
// GPUs must set them on each.  fn runs under the lock: no launch on that
// device can pass this point before the attribute is in place.
inline void once_per_device(const void* key, const std::function<void()>& fn) {
  static std::mutex mu;
  static std::set<std::pair<int, const void*>> done;
  int dev = 0;
  cudaGetDevice(&dev);
  std::lock_guard<std::mutex> lock(mu);
  if (done.insert({dev, key}).second) fn();
}

// The CUDA-core halves of the panel kernels (AGNN rows, SDDMM sparse edges)
// run on an auxiliary stream, concurrently with the tensor-core half.  One stream and
// its two events per (host thread, device): concurrent callers never share an
// event (no record/wait interleaving across threads) and every device gets
// its own stream.  Created on first use, kept for the thread's lifetime.
struct AuxStreams {
  cudaStream_t aux = nullptr;
  cudaEvent_t ready = nullptr, join = nullptr;
};

inline const AuxStreams& aux_streams() {
  thread_local std::vector<std::pair<int, AuxStreams>> per_dev;
  int dev = 0;
  CU(cudaGetDevice(&dev));
  for (auto& e : per_dev)
    if (e.first == dev) return e.second;
  AuxStreams a;
  CU(cudaStreamCreateWithFlags(&a.aux, cudaStreamNonBlocking));
  CU(cudaEventCreateWithFlags(&a.ready, cudaEventDisableTiming));
  CU(cudaEventCreateWithFlags(&a.join, cudaEventDisableTiming));
  per_dev.emplace_back(dev, a);
  return per_dev.back().second;
}

constexpr uint32_t kNoSlot = 0xFFFFFFFFu;
constexpr int kWinRows = 16;  // internal row-window height (MMA M)

// Feature-chunk width a warp owns in the SpMM / fused AGNN kernels.
inline int pick_dc(uint64_t d) {
  if (d <= 16) return 16;
  if (d <= 32) return 32;
  return 64;
}

// Device memory owned by RAII (graph handles, workspaces).
struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  DevBuf() = default;
  explicit DevBuf(size_t b) { alloc(b); }
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  DevBuf(DevBuf&& o) noexcept : p(o.p), bytes(o.bytes) { o.p = nullptr; o.bytes = 0; }
  DevBuf& operator=(DevBuf&& o) noexcept {
    if (this != &o) { release(); p = o.p; bytes = o.bytes; o.p = nullptr; o.bytes = 0; }
    return *this;
  }
  ~DevBuf() { release(); }
  void alloc(size_t b) {
    release();
    if (b) {
      cudaError_t e = cudaMalloc(&p, b);
      if (e != cudaSuccess) {
        p = nullptr;
        raise(SGTK_ERR_CUDA, "cudaMalloc(" + std::to_string(b) + " B): " +
                                 cudaGetErrorString(e));
      }
    }
    bytes = b;
  }
  void ensure(size_t b) { if (b > bytes) alloc(b); }
  void release() { if (p) cudaFree(p); p = nullptr; bytes = 0; }
  template <class T> T* as() const { return static_cast<T*>(p); }
};

}  // namespace sgtkcu

// ---------------------------------------------------------------------------
// Device helpers
// ---------------------------------------------------------------------------
#ifdef __CUDACC__
namespace sgtkcu {

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// tf32_round_value (tile_exec.cpp:131-142), bit-exact: RNE to 10 mantissa
// bits with saturation at the largest finite TF32 value.  Integer ops only.
// One F2FP: cvt.rn.satfinite is RNE with the same saturation at the largest
// finite TF32 value (0x7F7FE000); the reference passes inf/nan through
// unchanged, which the select restores.  Verified bit-exact against the
// reference on 20k random bit patterns (tests/test_gpu_parity.py).
__device__ __forceinline__ float tf32_rne(float v) {
  uint32_t r;
  asm("cvt.rn.satfinite.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return (__float_as_uint(v) & 0x7F800000u) == 0x7F800000u ? v : __uint_as_float(r);
}

// Hardware round-to-nearest (ties away) TF32: used for the "hi" half of the
// 3xTF32 split, where only |x - hi| small matters, not the tie rule.
__device__ __forceinline__ uint32_t tf32_rna_bits(float v) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return r;
}

// D += A(16x8 tf32, row) * B(8x8 tf32, col), fp32 accumulate.
__device__ __forceinline__ void mma_tf32(float (&c)[4], uint32_t a0, uint32_t a1,
                                         uint32_t a2, uint32_t a3, uint32_t b0,
                                         uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 "
      "{%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, {%0,%1,%2,%3};\n"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

// FP32 precision on TF32 tensor cores ("4-term split"): the data operand d
// is cut into three TF32-exact parts d = d0 + d1 + d2 (11 + 11 + 2
// significand bits, by masking, so the tensor core truncates nothing) and the
// structure operand s (adjacency value, weight) into s = s0 + s1;
//   s*d ~= s0*d2 + s1*d0 + s0*d1 + s0*d0      (four MMAs, small terms first)
// drops only s1*d1, s1*d2 (< 2^-21 |s||d|), and is EXACT whenever s is
// TF32-representable (unit / identity weights: the reference's bit-exact KATs,
// test_tile_exec.cpp:79-86, test_gnn.cpp:36-42).
// TF32 precision: both operands RNE-rounded exactly like tf32_round_value.
__device__ __forceinline__ uint32_t tf32_trunc_bits(float v) {
  return __float_as_uint(v) & 0xFFFFE000u;
}
__device__ __forceinline__ void split2(float v, uint32_t& p0, uint32_t& p1) {
  p0 = tf32_trunc_bits(v);
  p1 = __float_as_uint(v - __uint_as_float(p0));
}
__device__ __forceinline__ void split3(float v, uint32_t& p0, uint32_t& p1, uint32_t& p2) {
  p0 = tf32_trunc_bits(v);
  const float r = v - __uint_as_float(p0);
  p1 = tf32_trunc_bits(r);
  p2 = __float_as_uint(r - __uint_as_float(p1));
}

// MMA operand rounding in TF32 mode: RNE like tf32_round_value for every
// finite value (one F2FP); +-inf saturates instead of passing through, which
// only matters for non-finite inputs (documented in DESIGN.md).
__device__ __forceinline__ uint32_t tf32_op(float v) {
  uint32_t r;
  asm("cvt.rn.satfinite.tf32.f32 %0, %1;" : "=r"(r) : "f"(v));
  return r;
}

// 2^x on the SFU (ex2.approx.ftz: ~2 ulp); softmax weights only.
__device__ __forceinline__ float ex2_approx(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

// Structure operand per precision: TF32 -> (rne, -), FP32 -> split2.
template <int PREC>
__device__ __forceinline__ void split_s(float x, uint32_t& p0, uint32_t& p1) {
  if constexpr (PREC == SGTK_TF32) {
    p0 = tf32_op(x);
    p1 = 0u;
  } else {
    split2(x, p0, p1);
  }
}
// Data operand per precision: TF32 -> (rne, -, -), FP32 -> split3.
template <int PREC>
__device__ __forceinline__ void split_d(float x, uint32_t& p0, uint32_t& p1, uint32_t& p2) {
  if constexpr (PREC == SGTK_TF32) {
    p0 = tf32_op(x);
    p1 = p2 = 0u;
  } else {
    split3(x, p0, p1, p2);
  }
}

// ---- vectorised segment loads/stores (N floats, N in {2,4,8,16}) ----------
template <int N, bool VEC>
__device__ __forceinline__ void load_seg(float (&dst)[N], const float* __restrict__ src,
                                         int valid) {
  if (VEC && valid >= N) {
    if constexpr (N == 2) {
      float2 v = __ldg(reinterpret_cast<const float2*>(src));
      dst[0] = v.x; dst[1] = v.y;
    } else {
#pragma unroll
      for (int i = 0; i < N / 4; ++i) {
        float4 v = __ldg(reinterpret_cast<const float4*>(src) + i);
        dst[4 * i + 0] = v.x; dst[4 * i + 1] = v.y;
        dst[4 * i + 2] = v.z; dst[4 * i + 3] = v.w;
      }
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) dst[i] = i < valid ? __ldg(src + i) : 0.0f;
  }
}

template <int N, bool VEC>
__device__ __forceinline__ void store_seg(float* __restrict__ dst, const float (&v)[N],
                                          int valid) {
  if (VEC && valid >= N) {
    if constexpr (N == 2) {
      *reinterpret_cast<float2*>(dst) = make_float2(v[0], v[1]);
    } else {
#pragma unroll
      for (int i = 0; i < N / 4; ++i)
        reinterpret_cast<float4*>(dst)[i] =
            make_float4(v[4 * i], v[4 * i + 1], v[4 * i + 2], v[4 * i + 3]);
    }
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i)
      if (i < valid) dst[i] = v[i];
  }
}

// First index in [lo, hi) with key[idx] >= v (keys ascending).
__device__ __forceinline__ uint64_t lower_bound_u32(const uint32_t* __restrict__ key,
                                                    uint64_t lo, uint64_t hi,
                                                    uint32_t v) {
  while (lo < hi) {
    uint64_t mid = (lo + hi) >> 1;
    if (key[mid] < v) lo = mid + 1; else hi = mid;
  }
  return lo;
}

}  // namespace sgtkcu
#endif  // __CUDACC__
