// 128-row panel SpMM on the 5th-gen tensor cores (tcgen05 + TMEM).
//
// Replaces spmm_hybrid (/root/reference/proj/src/tile_exec.cpp:200-314) for
// the default plan (every tile on the tensor cores, ratio 1.0,
// tile_exec.cpp:150-161): out = A * x.
//
// Why 128-row panels instead of the reference's 16-row windows: a column
// shared by rows of the same panel is gathered once per panel.  On the
// Reddit-shaped graph the gathered volume drops from 43.7M (16-row windows)
// to 16.7M unique (panel, column) pairs; the gather, not the arithmetic, is
// what bounds this kernel.
//
// Density-aware split (the paper's thesis): per panel,
// columns with >= kDenseMin edges are "dense" and go through the tensor
// cores in chunks of 32 columns; singleton columns (the bulk of the random
// long-range edges) go edge-by-edge through the CUDA cores -- a 128 x 32 tile
// holding a single non-zero is not worth 16 KB of shared memory traffic.
//
// One CTA per (panel, 32/64-feature slice); 10 warps, warp-specialised:
//   warp 0      loader: cp.async gather of the chunk's 32 feature rows into
//               an MN-major SWIZZLE_128B_BASE32B B tile (the UMMA "N" = features are
//               contiguous in a row of x), plus a 1-D bulk copy (TMA engine)
//               of the chunk's packed adjacency entries
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer
//               (M = 128 rows, N = feature slice, K = 8 per instruction);
//               groups of kFold chunks rotate over TMEM accumulators
//   warps 2-5   A-tile builders: zero the K-major SWIZZLE_128B A tile (a
//               bulk copy of zeros by the TMA engine),
//               scatter the chunk's entries (tf32 value | tile offset packed
//               in one u32), FP32-split the B tile, fence, arrive
//   warps 6-9   accumulators, thread per row: sparse edges on CUDA cores in
//               fp32 registers; fold every finished TMEM accumulator group
//               into the same registers (IEEE adds: TC accumulation chains
//               stay <= 4 chunks long) on a schedule fixed by the panel's
//               shape (deterministic), then the epilogue store.
// Precision: TF32 = both operands RNE-rounded like tf32_round_value
// (tile_exec.cpp:131-142); FP32 = 3-term TF32 split a1*b0 + a0*b1 + a0*b0
// (dropped terms < 2^-21 relative per product).

#include <cub/device/device_scan.cuh>

#include <algorithm>
#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "kernels.cuh"
#include "tc05.cuh"

namespace sgtkcu {
namespace {

using namespace tc05;

// =========================================================== format builder
inline unsigned grid_for(uint64_t n, unsigned block, unsigned cap = 148u * 32u) {
  uint64_t g = (n + block - 1) / block;
  return unsigned(std::max<uint64_t>(1, std::min<uint64_t>(g, cap)));
}

__global__ void panel_count_kernel(const uint32_t* __restrict__ e2r, const uint32_t* __restrict__ e2c,
                                   const uint64_t* __restrict__ wo, uint64_t E,
                                   uint32_t* __restrict__ cnt) {
  for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < E;
       e += uint64_t(gridDim.x) * blockDim.x)
    atomicAdd(cnt + wo[e2r[e] / kPanelRows] + e2c[e], 1u);
}

__global__ void dense_flag_kernel(uint32_t* __restrict__ cnt, uint64_t U, uint32_t dense_min) {
  for (uint64_t u = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; u <= U;
       u += uint64_t(gridDim.x) * blockDim.x)
    cnt[u] = (u < U && cnt[u] >= dense_min) ? 1u : 0u;
}

__global__ void panel_dcount_kernel(const uint64_t* __restrict__ wo, const uint32_t* __restrict__ grank,
                                    uint64_t P, uint32_t* __restrict__ dcnt) {
  for (uint64_t p = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; p < P;
       p += uint64_t(gridDim.x) * blockDim.x)
    dcnt[p] = grank[wo[p + 1]] - grank[wo[p]];
}

// dense column list of each panel, padded to a multiple of 32
__global__ void dcols_kernel(const uint64_t* __restrict__ wo, const uint32_t* __restrict__ wuc,
                             const uint32_t* __restrict__ flag, const uint32_t* __restrict__ grank,
                             const uint32_t* __restrict__ cptr, uint64_t P,
                             uint32_t* __restrict__ dcols) {
  for (uint64_t p = blockIdx.x; p < P; p += gridDim.x) {
    const uint64_t u0 = wo[p], u1 = wo[p + 1];
    const uint32_t g0 = grank[u0];
    const uint64_t base = uint64_t(cptr[p]) * kChunkCols;
    for (uint64_t u = u0 + threadIdx.x; u < u1; u += blockDim.x)
      if (flag[u]) dcols[base + (grank[u] - g0)] = wuc[u];
  }
}

__device__ __forceinline__ bool dense_slot(const uint32_t* __restrict__ e2r,
                                           const uint32_t* __restrict__ e2c,
                                           const uint64_t* __restrict__ wo,
                                           const uint32_t* __restrict__ flag,
                                           const uint32_t* __restrict__ grank, uint64_t e,
                                           uint32_t& p, uint32_t& slot) {
  p = e2r[e] / kPanelRows;
  const uint64_t u = wo[p] + e2c[e];
  slot = grank[u] - grank[wo[p]];
  return flag[u] != 0;
}


// Word offset of A element (row, k) in a chunk's K-major SWIZZLE_128B TF32
// tile: 8-row core groups of 1 KB, 128-byte rows, 16-byte units XOR (row % 8).
__host__ __device__ __forceinline__ uint32_t a_word(uint32_t row, uint32_t k) {
  return (row >> 3) * 256u + (row & 7u) * 32u + (((k >> 2) ^ (row & 7u)) << 2) + (k & 3u);
}
// Packed entry: tf32(value) in bits 31..13 (RNE, tf32_round_value), the
// element's word offset in the swizzled A tile in bits 11..0 (a_word), so a
// builder stores it with one mask and one address add.  Padding entries
// (chunk sizes round up to 4) are value 0 at a position the chunk leaves
// empty: storing them is a no-op on the zeroed tile.
__device__ __forceinline__ uint32_t pack_entry(float v, uint32_t row, uint32_t k) {
  return (__float_as_uint(tf32_rne(v)) & 0xFFFFE000u) | a_word(row, k);
}

// Row masks straight from the edges: bit k of dmask[chunk][row] <=> edge
// (row, chunk column k).  OR is order-free: deterministic.
__global__ void edge_mask_kernel(const uint32_t* __restrict__ e2r, const uint32_t* __restrict__ e2c,
                                 const uint64_t* __restrict__ wo, const uint32_t* __restrict__ flag,
                                 const uint32_t* __restrict__ grank, const uint32_t* __restrict__ cptr,
                                 uint64_t E, uint32_t* __restrict__ dmask) {
  for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < E;
       e += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t p, slot;
    if (dense_slot(e2r, e2c, wo, flag, grank, e, p, slot))
      atomicOr(dmask + uint64_t(cptr[p] + slot / kChunkCols) * kPanelRows + e2r[e] % kPanelRows,
               1u << (slot % kChunkCols));
  }
}

// Per chunk: entries before each row (exclusive scan of the rows' popcounts).
__global__ void row_offsets_kernel(const uint32_t* __restrict__ dmask, uint64_t NC,
                                   uint16_t* __restrict__ rowoff, uint32_t* __restrict__ ccnt) {
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t c = warp; c < NC; c += nw) {
    const uint4 m = reinterpret_cast<const uint4*>(dmask + c * kPanelRows)[lane];  // rows 4l..4l+3
    const uint32_t a = __popc(m.x), b = __popc(m.y), cc = __popc(m.z), dd = __popc(m.w);
    uint32_t s = a + b + cc + dd, incl = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
      if (lane >= o) incl += t;
    }
    const uint32_t ex = incl - s;
    uint16_t* ro = rowoff + c * kPanelRows + 4 * lane;
    ro[0] = uint16_t(ex);
    ro[1] = uint16_t(ex + a);
    ro[2] = uint16_t(ex + a + b);
    ro[3] = uint16_t(ex + a + b + cc);
    if (lane == 31) ccnt[c] = incl;
  }
}

// Entries of a chunk in (row, column) order -- the CSR order -- so the
// builders' scattered shared-memory stores of consecutive entries land in
// few rows (bank-friendly), and the layout is fully deterministic.
__global__ void entry_fill_sorted_kernel(const uint32_t* __restrict__ e2r, const uint32_t* __restrict__ e2c,
                                         const uint64_t* __restrict__ wo, const uint32_t* __restrict__ flag,
                                         const uint32_t* __restrict__ grank,
                                         const uint32_t* __restrict__ cptr, const uint64_t* __restrict__ coff,
                                         const uint32_t* __restrict__ dmask,
                                         const uint16_t* __restrict__ rowoff,
                                         const float* __restrict__ vals, uint64_t E,
                                         uint32_t* __restrict__ dent, float* __restrict__ dval,
                                         uint32_t* __restrict__ deid) {
  for (uint64_t e = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; e < E;
       e += uint64_t(gridDim.x) * blockDim.x) {
    uint32_t p, slot;
    if (!dense_slot(e2r, e2c, wo, flag, grank, e, p, slot)) continue;
    const uint64_t ch = cptr[p] + slot / kChunkCols;
    const uint32_t row = e2r[e] % kPanelRows, k = slot % kChunkCols;
    const uint32_t m = dmask[ch * kPanelRows + row];
    const uint64_t i = coff[ch] + rowoff[ch * kPanelRows + row] + __popc(m & ((1u << k) - 1u));
    const float v = vals ? vals[e] : 1.0f;
    dent[i] = pack_entry(v, row, k);
    dval[i] = v;
    deid[i] = uint32_t(e);
  }
}



// SDDMM entries (dpos): the entry's panel row and chunk column from its
// packed tile offset (a_word inverted), its position in the CSR row from its
// edge id.  Block per panel.
__global__ void dpos_kernel(const uint32_t* __restrict__ cptr, const uint64_t* __restrict__ coff,
                            const uint32_t* __restrict__ dent, const uint32_t* __restrict__ deid,
                            const uint64_t* __restrict__ np, uint64_t P, uint32_t* __restrict__ dpos,
                            uint32_t* __restrict__ overflow) {
  for (uint64_t p = blockIdx.x; p < P; p += gridDim.x) {
    const uint64_t i0 = coff[cptr[p]], i1 = coff[cptr[p + 1]];
    for (uint64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
      const uint32_t e = deid[i];
      if (e == 0xFFFFFFFFu) {
        dpos[i] = 0xFFFFFFFFu;
        continue;
      }
      const uint32_t w = dent[i] & 0xFFFu;
      const uint32_t row = (w >> 8) * 8u + ((w >> 5) & 7u);
      const uint32_t k = ((((w >> 2) & 7u) ^ (row & 7u)) << 2) | (w & 3u);
      const uint64_t pos = uint64_t(e) - np[p * kPanelRows + row];
      if (pos >= (1u << 20)) {
        atomicOr(overflow, 1u);
        dpos[i] = 0xFFFFFFFFu;
      } else {
        dpos[i] = (uint32_t(pos) << 12) | (row << 5) | k;
      }
    }
  }
}

// Padding entries of a chunk: value 0 at the first position with no edge
// (a chunk with all 4096 positions taken has no padding).  Warp per chunk.
__global__ void entry_pad_kernel(const uint32_t* __restrict__ ccnt, const uint64_t* __restrict__ coff,
                                 const uint32_t* __restrict__ dmask, uint64_t nc,
                                 uint32_t* __restrict__ dent) {
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t c = warp; c < nc; c += nw) {
    const uint64_t b = coff[c] + ccnt[c], e = coff[c + 1];
    if (b == e) continue;
    uint32_t row = 0, k = 0;
    for (uint32_t r0 = 0; r0 < kPanelRows; r0 += 32) {
      const uint32_t m = dmask[c * kPanelRows + r0 + lane];
      const uint32_t open = __ballot_sync(0xFFFFFFFFu, m != 0xFFFFFFFFu);
      if (open) {
        const uint32_t src = __ffs(open) - 1;
        row = r0 + src;
        k = __ffs(~__shfl_sync(0xFFFFFFFFu, m, src)) - 1;
        break;
      }
    }
    if (b + lane < e) dent[b + lane] = a_word(row, k);
  }
}

// sparse (CUDA-core) edges: per-row count, then per-row stable compaction
__global__ void sparse_count_kernel(const uint64_t* __restrict__ np, uint64_t n,
                                    const uint32_t* __restrict__ e2c, const uint64_t* __restrict__ wo,
                                    const uint32_t* __restrict__ flag, uint32_t* __restrict__ scnt) {
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t r = warp; r < n; r += nwarps) {
    const uint64_t ub = wo[r / kPanelRows];
    uint32_t c = 0;
    for (uint64_t e = np[r] + lane; e < np[r + 1]; e += 32) c += flag[ub + e2c[e]] ? 0u : 1u;
    c = __reduce_add_sync(0xFFFFFFFFu, c);
    if (lane == 0) scnt[r] = c;
  }
}

__global__ void sparse_fill_kernel(const uint64_t* __restrict__ np, const uint32_t* __restrict__ el,
                                   const float* __restrict__ vals, uint64_t n,
                                   const uint32_t* __restrict__ e2c, const uint64_t* __restrict__ wo,
                                   const uint32_t* __restrict__ flag,
                                   const uint32_t* __restrict__ sptr, uint2* __restrict__ sent,
                                   uint32_t* __restrict__ seid) {
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nwarps = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint32_t lane = threadIdx.x & 31;
  for (uint64_t r = warp; r < n; r += nwarps) {
    const uint64_t ub = wo[r / kPanelRows];
    uint32_t pos = sptr[r];
    for (uint64_t b = np[r]; b < np[r + 1]; b += 32) {
      const uint64_t e = b + lane;
      const bool sp = e < np[r + 1] && !flag[ub + e2c[e]];
      const uint32_t m = __ballot_sync(0xFFFFFFFFu, sp);
      if (sp) {
        const uint32_t i = pos + __popc(m & ((1u << lane) - 1u));
        sent[i] = make_uint2(el[e], __float_as_uint(vals ? vals[e] : 1.0f));
        seid[i] = uint32_t(e);
      }
      pos += __popc(m);
    }
  }
}

// Override values (edge_values span, tile_exec.cpp:44-52): re-pack the
// entries from a CSR-order value array through the stored edge ids.
__global__ void repack_dense_kernel(const uint32_t* __restrict__ dent, const uint32_t* __restrict__ deid,
                                    const float* __restrict__ ev, uint64_t n,
                                    uint32_t* __restrict__ dent_o, float* __restrict__ dval_o) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint32_t e = deid[i], w = dent[i];
    if (e == 0xFFFFFFFFu) {
      dent_o[i] = w;
      dval_o[i] = 0.0f;
    } else {
      const float v = ev[e];
      dent_o[i] = (__float_as_uint(tf32_rne(v)) & 0xFFFFE000u) | (w & 0xFFFu);
      dval_o[i] = v;
    }
  }
}
__global__ void repack_sparse_kernel(const uint2* __restrict__ sent, const uint32_t* __restrict__ seid,
                                     const float* __restrict__ ev, uint64_t n,
                                     uint2* __restrict__ sent_o) {
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x)
    sent_o[i] = make_uint2(sent[i].x, __float_as_uint(ev[seid[i]]));
}

template <class T>
std::vector<T> dl(const void* dev, size_t count, cudaStream_t s) {
  std::vector<T> h(count);
  if (count) {
    CU(cudaMemcpyAsync(h.data(), dev, count * sizeof(T), cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
  }
  return h;
}
template <class T>
std::shared_ptr<DevBuf> ul(const T* host, size_t count, cudaStream_t s) {
  auto b = std::make_shared<DevBuf>(std::max<size_t>(count, 1) * sizeof(T));
  if (count) CU(cudaMemcpyAsync(b->p, host, count * sizeof(T), cudaMemcpyHostToDevice, s));
  return b;
}

void exclusive_scan_u32(const uint32_t* in, uint32_t* out, uint64_t n, cudaStream_t s) {
  size_t tb = 0;
  CU(cub::DeviceScan::ExclusiveSum(nullptr, tb, in, out, int64_t(n), s));
  DevBuf t(std::max<size_t>(tb, 16));
  CU(cub::DeviceScan::ExclusiveSum(t.p, tb, in, out, int64_t(n), s));
  CU(cudaStreamSynchronize(s));
}

// ======================================================== the SpMM kernels
template <int DC, int PREC>
struct PanelCfg {
  static constexpr int PA = PREC == SGTK_FP32 ? 2 : 1;  // A planes (split2)
  static constexpr int PB = PREC == SGTK_FP32 ? 2 : 1;  // B planes (split2)
  static constexpr uint32_t A_BYTES = kPanelRows * kChunkCols * 4;  // 16 KB, K-major
  static constexpr uint32_t B_BYTES = kChunkCols * DC * 4;          // MN-major
  static constexpr uint32_t A_STAGE = PA * A_BYTES;                 // multiple of 1024
  static constexpr uint32_t B_STAGE = PB * B_BYTES;                 // multiple of 1024
#ifndef SGTK_NS32
#define SGTK_NS32 4
#endif
  static constexpr int NS = (PREC == SGTK_FP32 || DC == 64) ? 2 : SGTK_NS32;  // A ring depth
  static constexpr int GW = 4 / NS;                                 // builder warps per chunk
  static constexpr int NV = PREC == SGTK_FP32 ? 2 : 1;              // entry (+ value) slots
  // DC = 32 TF32 fits two CTAs per SM (256 TMEM columns, <= 113 KB smem,
  // <= 102 registers); the others run one
  static constexpr int CTAS = PREC == SGTK_TF32 ? 2 : 1;
  static constexpr uint32_t TMEM_COLS = CTAS == 2 ? 256 : 512;
  // TMEM: running fp32 sum (DC columns, updated by the accumulator warps
  // 16 columns at a time: few registers) + NF accumulation buffers
  static constexpr int NF = (TMEM_COLS - DC) / DC;
  static constexpr uint32_t BUF0 = DC;                              // first buffer column
#ifndef SGTK_FOLD
#define SGTK_FOLD 4
#endif
  static constexpr uint32_t FOLD = SGTK_FOLD;                       // chunks per accumulator
};

constexpr int kPanelThreads = 320;
constexpr uint32_t kBarBytes = 1024;
constexpr uint32_t kMaxND = 8;

// Runtime shared-memory layout (host-computed from the graph's largest chunk).
struct PanelSmem {
  uint32_t nd;     // B-tile and entry ring depth (multiple of NS, >= NS)
  uint32_t dslot;  // bytes of one entry slot
  uint32_t bring_off, dring_off, total;
};

// Zeros for an A stage (up to 2 planes x 16 KB), copied in by the TMA engine.
__device__ __align__(128) uint32_t g_zero_tile[2 * kPanelRows * kChunkCols];

// ---------------------------------------------------------------------------
// Dense part on the tensor cores: out[rows of panel] = A_dense * x (a store:
// the CUDA-core kernels add the sparse edges afterwards, in a fixed order).
// One CTA per (panel, 32/64-feature slice); 10 warps, warp-specialised:
//   warp 0      loader: coalesced cp.async gather of the chunk's 32 feature
//               rows into an MN-major SWIZZLE_128B_BASE32B B tile, completion
//               signalled by cp.async.mbarrier.arrive.noinc (the loader never
//               waits on its own copies); 1-D bulk copies (TMA engine) of the
//               chunks' packed entries, nd - NS chunks ahead of the stages
//   warp 1      TMEM allocator + single-thread tcgen05.mma issuer (M = 128
//               rows, N = feature slice, K = 8 per instruction); groups of
//               FOLD chunks rotate over 512/DC TMEM accumulators
//   warps 2-5   A-tile builders: chunk c is built by the warp group c % NS,
//               so NS chunks are in construction at once: the TMA engine
//               zeroes the K-major SWIZZLE_128B A tile, the group scatters
//               the entries (tf32 value | swizzled tile offset in one u32),
//               FP32: splits A and B into TF32 planes; fence.proxy.async,
//               arrive
//   warps 6-9   accumulators, thread per row: fold each finished TMEM group
//               into fp32 registers in group order (IEEE adds keep every
//               tensor-core accumulation chain <= FOLD chunks), store.
// ---------------------------------------------------------------------------
// PAD: the feature slice is narrower than DC (d % DC != 0): the B ring's
// padding features are zeroed once and never copied (copying zeros for them
// from one source keeps a few L2 lines hot across all CTAs: d = 16 0.27 ms
// against 0.23 ms this way; used for DC = 32 only, see launch_dense)
template <int DC, int PREC, bool PAD>
__global__ void __launch_bounds__(kPanelThreads, PanelCfg<DC, PREC>::CTAS)
spmm_panel_kernel(const PanelView pv, const PanelSmem L, const float* __restrict__ x, uint64_t ldx,
                  uint64_t d, float* __restrict__ out, uint64_t ldo, int vec_out,
                  uint32_t* __restrict__ nonfinite, long long* __restrict__ trace) {
  using C = PanelCfg<DC, PREC>;
  // optional timeline (SGTK_PANEL_TRACE): trace[(panel * 256 + chunk) * 8 + event]
  auto mark = [&](uint32_t c, int ev) {
#ifdef SGTK_TRACE  // pipeline event trace (tools/panel_debug.py); compiled out by default
    if (trace && blockIdx.x < 4 && c < 256) trace[((uint64_t(blockIdx.x) * 256 + c) * 8) + ev] = clock64();
#else
    (void)c, (void)ev, (void)trace;
#endif
  };
  extern __shared__ __align__(16) uint8_t smem_raw[];
  // 1024-aligned base, derived by offset so the compiler keeps the shared
  // address space (LDS/STS rather than generic loads)
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem);  // A stage built
  uint64_t* zfull = full + C::NS;                       // A stage zeroed (copy engine)
  uint64_t* bfull = zfull + C::NS;                      // B tile landed
  uint64_t* bempty = bfull + kMaxND;                    // B tile + entry slot consumed
  uint64_t* dfull = bempty + kMaxND;                    // entries landed
  uint64_t* accfull = dfull + kMaxND;
  uint64_t* accempty = accfull + C::NF;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + C::NF);
  uint8_t* ring = smem + kBarBytes;      // [NS] A stages (PA planes)
  uint8_t* bring = smem + L.bring_off;   // [nd] B tiles (PB planes)
  uint8_t* dring = smem + L.dring_off;   // [nd] entry slots (+ [nd] value slots, FP32)

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t p = blockIdx.x;
  const uint64_t fbase = uint64_t(blockIdx.y) * DC;
  const int dvalid = d - fbase < uint64_t(DC) ? int(d - fbase) : DC;
  const uint32_t c0 = pv.cptr[p], nch = pv.cptr[p + 1] - c0;
  const uint32_t ngroups = (nch + C::FOLD - 1) / C::FOLD;
  const uint32_t ND = L.nd;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NS; ++i) {
      mbar_init(full + i, C::GW);  // the builder warps that own the chunk
      mbar_init(zfull + i, 1);     // bulk copy of zeros (expect_tx)
    }
    for (uint32_t i = 0; i < ND; ++i) {
      mbar_init(bfull + i, 32 * C::GW);  // cp.async.mbarrier.arrive.noinc per gathering lane
      mbar_init(bempty + i, 1);          // tcgen05.commit
      mbar_init(dfull + i, 1);           // bulk copy (expect_tx)
    }
    for (int i = 0; i < C::NF; ++i) {
      mbar_init(accfull + i, 1);
      mbar_init(accempty + i, 4);
    }
    mbar_init_fence();
  }
  if (warp == 1) tmem_alloc(tmem_slot, C::TMEM_COLS);
  if constexpr (PAD) {
    const uint32_t rb = smem_u32(bring);
    for (uint32_t i = threadIdx.x; i < ND * C::B_STAGE / 16; i += blockDim.x)
      st_shared_v4(rb + i * 16, 0u, 0u, 0u, 0u);
    fence_async_smem();
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    // ------------------------------------------------------------ loader
    // Entry bulk copies (TMA engine) into a ring nd chunks deep; slot c % nd
    // is free once MMA(c - nd) retired (bempty).  Chunk offsets are
    // prefetched kLook chunks ahead so no global load sits on this path.
    if (lane == 0) {
      constexpr uint32_t kLook = 4;
      uint64_t offq[kLook];
#pragma unroll
      for (uint32_t i = 0; i < kLook; ++i) offq[i] = i <= nch ? pv.coff[c0 + i] : 0u;
      uint64_t off_tail = kLook <= nch ? pv.coff[c0 + kLook] : 0u;
      for (uint32_t cb = 0; cb < nch; cb += kLook) {
#pragma unroll
        for (uint32_t i = 0; i < kLook; ++i) {
          const uint32_t c = cb + i;
          if (c >= nch) break;
          const uint64_t e0 = offq[i], e1 = i + 1 < kLook ? offq[(i + 1) % kLook] : off_tail;
          offq[i] = c + kLook <= nch ? pv.coff[c0 + c + kLook] : 0u;
          if (i + 1 == kLook) off_tail = c + 1 + kLook <= nch ? pv.coff[c0 + c + 1 + kLook] : 0u;
          const uint32_t ds = c % ND, dph = (c / ND) & 1u;
          mbar_wait(bempty + ds, dph ^ 1u);
          mark(c, 0);
          const uint32_t bytes = uint32_t(e1 - e0) * 4u;
          mbar_expect_tx(dfull + ds, bytes * C::NV);
          if (bytes) {
            bulk_load(dring + ds * L.dslot, pv.dent + e0, bytes, dfull + ds);
            if constexpr (PREC == SGTK_FP32)
              bulk_load(dring + (ND + ds) * L.dslot, pv.dval + e0, bytes, dfull + ds);
          }
        }
      }
    }
  } else if (warp == 1) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(DC, true);
      for (uint32_t c = 0; c < nch; ++c) {
        const uint32_t s = c % C::NS, ph = (c / C::NS) & 1u;
        const uint32_t g = c / C::FOLD, buf = g % C::NF;
        const bool first = (c % C::FOLD) == 0;
        if (first && g >= uint32_t(C::NF)) mbar_wait(accempty + buf, ((g / C::NF) - 1u) & 1u);
        const uint32_t ds = c % ND, dph = (c / ND) & 1u;
        mbar_wait(full + s, ph);
        mark(c, 4);
        if constexpr (PREC == SGTK_TF32) {
          // B went straight from cp.async (generic proxy) to the MMA (async
          // proxy): acquire the copies, then order them for the async proxy.
          mbar_wait(bfull + ds, dph);
          fence_async_smem();
        }
        tc_fence_after();
        mark(c, 5);
        const uint32_t dt = tmem + C::BUF0 + buf * DC;
        const uint32_t a0 = smem_u32(ring + s * C::A_STAGE), a1 = a0 + C::A_BYTES;
        const uint32_t b0 = smem_u32(bring + ds * C::B_STAGE), b1 = b0 + C::B_BYTES, b2 = b1 + C::B_BYTES;
#pragma unroll
        for (uint32_t ks = 0; ks < kChunkCols / 8; ++ks) {
          const uint32_t acc = (first && ks == 0) ? 0u : 1u;
          const uint64_t ad0 = umma_desc(a0 + ks * 32);
          const uint64_t bd0 = desc_mn32(b0 + ks * 1024, 4096, 512);
          if constexpr (PREC == SGTK_FP32) {  // 3-term split: a1*b0 + a0*b1 + a0*b0
            umma_tf32(dt, umma_desc(a1 + ks * 32), bd0, idesc, acc);
            umma_tf32(dt, ad0, desc_mn32(b1 + ks * 1024, 4096, 512), idesc, 1u);
            umma_tf32(dt, ad0, bd0, idesc, 1u);
          } else {
            umma_tf32(dt, ad0, bd0, idesc, acc);
          }
        }
        umma_commit(bempty + ds);  // A stage, B tile and entry slot of chunk c free
        if ((c % C::FOLD) == C::FOLD - 1 || c + 1 == nch) umma_commit(accfull + buf);
      }
    }
  } else if (warp < 6) {
    // ------------------------------------------------------------ A builders
    // Builder group c % NS owns chunk c: it gathers the chunk's B tile (PD =
    // nd - NS chunks ahead, cp.async with completion signalled by the copy
    // engine), has the TMA engine zero the A tile, scatters the staged
    // entries into it, and (FP32) splits B into TF32 planes.  NS chunks are
    // in construction at once.
    const uint32_t b = warp - 2, grp = b % C::NS, sub = b / C::NS;
    const uint32_t gl = sub * 32 + lane;  // thread index inside the chunk's group
    constexpr uint32_t GT = C::GW * 32;
    const uint32_t PD = ND - C::NS;
    // gather the 32 feature rows of chunk cg (its B slot is free: MMA(cg - nd)
    // retired before MMA(c - NS), which this group already waited for)
    auto id_of = [&](uint32_t cg) {  // this lane's column id of chunk cg (lane = K-row)
      return cg < nch ? __ldg(pv.dcols + uint64_t(c0 + cg) * kChunkCols + lane) : 0u;
    };
    auto gather_b = [&](uint32_t cg, uint32_t myid) {
      const uint32_t ds = cg % ND;
      const uint32_t bst = smem_u32(bring + ds * C::B_STAGE);
      constexpr uint32_t LPR = DC / 4, RPG = GT / LPR;  // rows per group instruction
      const uint32_t j = gl % LPR, jj = j & 7u;
#pragma unroll
      for (uint32_t t = 0; t < 32 / RPG; ++t) {
        const uint32_t k = t * RPG + gl / LPR;
        const uint32_t ck = __shfl_sync(0xFFFFFFFFu, myid, k);
        const bool real = ck != 0xFFFFFFFFu && int(4 * j) < dvalid;
        // MN-major SWIZZLE_128B_BASE32B (tc05.cuh desc_mn32): K-row k, 4-row
        // groups 512 B apart, 32-feature blocks 4096 B apart, 32-byte chunks
        // XOR (k % 4)
        const uint32_t dst = bst + (j >> 3) * 4096u + (k >> 2) * 512u + (k & 3u) * 128u +
                             ((((jj >> 1) ^ (k & 3u)) << 5) | ((jj & 1u) << 4));
        // zeros (padding columns / features) from distinct 16-byte pieces: a
        // single zero source would serialise every CTA's padding copies on
        // one address (d = 16: 6x slower)
        if (!PAD || int(4 * j) < dvalid)
          cp_async16(dst, real ? x + uint64_t(ck) * ldx + fbase + 4 * j
                               : reinterpret_cast<const float*>(g_zero_tile) + (k * LPR + j) * 4);
      }
      cp_async_arrive_noinc(bfull + ds);
    };
    for (uint32_t c = grp; c < nch && c < grp + PD; c += C::NS) gather_b(c, id_of(c));
    // ids of the next chunk to gather, loaded one iteration ahead
    uint32_t idn = id_of(grp + PD);
    for (uint32_t c = grp; c < nch; c += C::NS) {
      const uint32_t s = c % C::NS, ph = (c / C::NS) & 1u;
      const uint32_t ds = c % ND, dph = (c / ND) & 1u;
      const uint32_t abase = smem_u32(ring + s * C::A_STAGE);
      const uint64_t e0 = pv.coff[c0 + c], e1 = pv.coff[c0 + c + 1];
      const uint32_t ne = uint32_t(e1 - e0);
      if (c >= uint32_t(C::NS)) {  // MMA(c - NS) retired: A stage free (one commit per chunk)
        const uint32_t cp = c - C::NS;
        mbar_wait(bempty + cp % ND, (cp / ND) & 1u);
      }
      if (gl == 0) {  // the copy engine zeroes the stage (no store loop here)
        mbar_expect_tx(zfull + s, C::A_STAGE);
        bulk_load(ring + s * C::A_STAGE, g_zero_tile, C::A_STAGE, zfull + s);
      }
      if (lane == 0) mark(c, 1);
      if (c + PD < nch) gather_b(c + PD, idn);
      idn = id_of(c + PD + C::NS);
      mbar_wait(zfull + s, ph);
      mbar_wait(dfull + ds, dph);
      if (lane == 0) mark(c, 2);
      if constexpr (C::GW > 1) named_bar(1 + grp, GT);
      else __syncwarp();
      // Scatter: each lane takes 4 consecutive entries (one 16-byte LDS);
      // the entry carries its swizzled tile offset (pack_entry), padding
      // entries store 0 on an empty position.
      const uint32_t ent = smem_u32(dring + ds * L.dslot);
      const uint32_t dv = smem_u32(dring + (ND + ds) * L.dslot);
      for (uint32_t i0 = gl * 4; i0 < ne; i0 += GT * 4 * 4) {
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const uint32_t i = i0 + h * GT * 4;
          if (i >= ne) break;  // ne is a multiple of 4: whole uint4 groups
          const uint4 w4 = ld_shared_u4(ent + i * 4);
          const uint32_t ws[4] = {w4.x, w4.y, w4.z, w4.w};
          if constexpr (PREC == SGTK_FP32) {
            const float4 v4 = ld_shared_f4(dv + i * 4);
            const float vs[4] = {v4.x, v4.y, v4.z, v4.w};
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4) {
              const uint32_t off = (ws[k4] & 0xFFFu) * 4u;
              uint32_t s0, s1;
              split2(vs[k4], s0, s1);
              st_shared_u32(abase + off, s0);
              st_shared_u32(abase + C::A_BYTES + off, s1);
            }
          } else {
#pragma unroll
            for (int k4 = 0; k4 < 4; ++k4)
              st_shared_u32(abase + (ws[k4] & 0xFFFu) * 4u, ws[k4] & 0xFFFFE000u);
          }
        }
      }
      if constexpr (PREC == SGTK_FP32) {
        // B tile: 2-plane TF32 split in place (every lane of the group first
        // waits for all copies of the tile)
        mbar_wait(bfull + ds, dph);
        uint4* B = reinterpret_cast<uint4*>(bring + ds * C::B_STAGE);
#pragma unroll 4
        for (uint32_t i = gl; i < C::B_BYTES / 16; i += GT) {
          const uint4 v = B[i];
          uint32_t xs[4] = {v.x, v.y, v.z, v.w}, q0[4], q1[4];
#pragma unroll
          for (int jx = 0; jx < 4; ++jx) split2(__uint_as_float(xs[jx]), q0[jx], q1[jx]);
          B[i] = make_uint4(q0[0], q0[1], q0[2], q0[3]);
          B[C::B_BYTES / 16 + i] = make_uint4(q1[0], q1[1], q1[2], q1[3]);
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) {
        mark(c, 3);
        mbar_arrive(full + s);
      }
    }
  } else {
    // ------------------------------------------------------------ accumulators
    // Fold each finished group into the running sum kept in TMEM (IEEE adds,
    // group order), 16 columns at a time; then stream the sum out.
    const uint32_t q = warp & 3u;
    const uint64_t r = p * kPanelRows + q * 32 + lane;
    const uint32_t lanes = (q * 32u) << 16;
    for (uint32_t g = 0; g < ngroups; ++g) {
      const uint32_t buf = g % C::NF;
      mbar_wait(accfull + buf, (g / C::NF) & 1u);
      tc_fence_after();
#pragma unroll
      for (int cc = 0; cc < DC; cc += 16) {
        uint32_t v[16], sm[16];
        tmem_ld16(tmem + lanes + C::BUF0 + buf * DC + cc, v);
        if (g) tmem_ld16(tmem + lanes + cc, sm);
        tmem_ld_wait();
        if (g) {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(__uint_as_float(sm[j]) + __uint_as_float(v[j]));
        }
        tmem_st16(tmem + lanes + cc, v);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(accempty + buf);
    }
    tc_fence_after();
    const bool rv = r < pv.n_rows;
    float* o = out + r * ldo + fbase;
    bool bad = false;  // a non-finite dense sum stays non-finite after the sparse edges
#pragma unroll
    for (int cc = 0; cc < DC; cc += 16) {
      uint32_t v[16];
      if (ngroups) {
        tmem_ld16(tmem + lanes + cc, v);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0u;
      }
      if (rv) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          bad |= cc + j < dvalid && (v[j] & 0x7F800000u) == 0x7F800000u;
        if (vec_out && dvalid == DC) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            reinterpret_cast<float4*>(o + cc)[j] =
                make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                            __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (cc + j < dvalid) o[cc + j] = __uint_as_float(v[j]);
        }
      }
    }
    if (nonfinite && __any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(nonfinite, 1u);
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------
// Dense part, TF32, A built in TMEM (opt-in: SGTK_SPMM_TM=1; measured slower
// than spmm_panel_kernel).  The A tile of a chunk never touches shared memory: the
// thread of panel row r reads its row mask and its row's packed entries (the
// chunk's entries are in (row, column) order, so row r's values start at the
// popcount of the rows before it), builds its 32 TF32 values in registers and
// stores them into its TMEM lane (tcgen05.st); the MMA reads A from TMEM
// ("TS" form, as the AGNN kernel's P).  No zero tile, no scatter, no A stage
// to recycle: the builder -> MMA chain is registers -> TMEM.  The smem the A
// stages held goes to a deeper B ring.  Same products, same K order, same
// FOLD groups and fold order as spmm_panel_kernel: bit-identical to it.
//   warps 0..4BG-1  A builders: BG groups of 4 warps, group c % BG builds
//               chunk c, thread per row (TMEM lane = row; a builder is
//               latency-bound, so BG chunks are in construction at once); the
//               group's first lane bulk-copies the masks + entries of its
//               chunk NE - 1 turns ahead into its entry ring (TMA engine)
//   next 4      accumulators (as spmm_panel_kernel)
//   next 1      TMEM allocator + MMA issuer
//   last NL     B loaders (cp.async gathers, chunk c by loader c % NL)
// ---------------------------------------------------------------------------
#ifndef SGTK_TM_LOADERS
#define SGTK_TM_LOADERS 2
#endif
#ifndef SGTK_TM_NE
#define SGTK_TM_NE 2
#endif
#ifndef SGTK_TM_BG
#define SGTK_TM_BG 2
#endif

#ifndef SGTK_TM_PREFETCH
#define SGTK_TM_PREFETCH 1
#endif
template <int DC>
struct TmCfg {
  static constexpr int NL = SGTK_TM_LOADERS;
  static constexpr int BG = SGTK_TM_BG;                  // builder groups
  static constexpr uint32_t AW = 4 * BG, IW = AW + 4, LW = IW + 1;  // accumulator / issuer / first loader warp
  static constexpr int THREADS = 32 * (LW + NL);
  static constexpr uint32_t B_BYTES = kChunkCols * DC * 4;
  static constexpr int NBMAX = DC == 64 ? 12 : 16;
  static constexpr int NE = SGTK_TM_NE;       // entry ring per builder group (lead: NE - 1 of its chunks)
  static constexpr int NA = DC == 64 ? 2 : 4;  // A buffers, 32 TMEM columns each
  static constexpr int NF = DC == 64 ? 2 : 3;  // accumulators
  static constexpr uint32_t BUF0 = DC;         // running sum: columns [0, DC)
  static constexpr uint32_t ACOL = DC * (1 + NF);
  static constexpr uint32_t TMEM_COLS = 256;   // two CTAs per SM
  static_assert(ACOL + 32 * NA <= TMEM_COLS, "TMEM budget");
  static constexpr uint32_t FOLD = SGTK_FOLD;  // as spmm_panel_kernel (bit-identical)
};

struct TmSmem {
  uint32_t nb;     // B ring depth
  uint32_t eslot;  // bytes of one entry slot: 512 B masks + entries (+ 16 B read slack)
  uint32_t ering_off, total;
};

template <int DC>
__global__ void __launch_bounds__(TmCfg<DC>::THREADS, 2)
spmm_tm_kernel(const PanelView pv, const TmSmem L, const float* __restrict__ x, uint64_t ldx, uint64_t d,
               float* __restrict__ out, uint64_t ldo, int vec_out, uint32_t* __restrict__ nonfinite) {
  using C = TmCfg<DC>;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  const uint32_t NB = L.nb;
  uint64_t* bfull = reinterpret_cast<uint64_t*>(smem);  // [NBMAX] B tile landed
  uint64_t* bempty = bfull + C::NBMAX;                  // [NBMAX] MMA(c) retired: B slot + A buffer free
  uint64_t* efull = bempty + C::NBMAX;                  // [BG][NE] masks + entries landed
  uint64_t* eempty = efull + C::BG * C::NE;             // [BG][NE] read by the group's 4 warps
  uint64_t* afull = eempty + C::BG * C::NE;             // [NA] A(c) in TMEM
  uint64_t* accfull = afull + C::NA;                    // [NF]
  uint64_t* accempty = accfull + C::NF;                 // [NF]
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(accempty + C::NF);
  static_assert((2 * C::NBMAX + 2 * C::BG * C::NE + C::NA + 2 * C::NF) * 8 + 16 <= 1024, "barriers");
  uint8_t* bring = smem + 1024;
  uint8_t* ering = smem + L.ering_off;

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t p = blockIdx.x;
  const uint64_t fbase = uint64_t(blockIdx.y) * DC;
  const int dvalid = d - fbase < uint64_t(DC) ? int(d - fbase) : DC;
  const uint32_t c0 = pv.cptr[p], nch = pv.cptr[p + 1] - c0;
  const uint32_t ngroups = (nch + C::FOLD - 1) / C::FOLD;

  if (threadIdx.x == 0) {
    for (uint32_t i = 0; i < NB; ++i) {
      mbar_init(bfull + i, 32);  // cp.async.mbarrier.arrive.noinc per lane of the loader warp
      mbar_init(bempty + i, 1);  // tcgen05.commit
    }
    for (int i = 0; i < C::BG * C::NE; ++i) {
      mbar_init(efull + i, 1);  // bulk copies (expect_tx)
      mbar_init(eempty + i, 4);
    }
    for (int i = 0; i < C::NA; ++i) mbar_init(afull + i, 4);
    for (int i = 0; i < C::NF; ++i) {
      mbar_init(accfull + i, 1);
      mbar_init(accempty + i, 4);
    }
    mbar_init_fence();
  }
  if (warp == C::IW) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < C::AW) {
    // ------------------------------------------------------------ A builders
    const uint32_t wq = warp & 3u, grp = warp >> 2;
    const uint32_t r = wq * 32 + lane;
    const uint32_t lanes = (wq * 32u) << 16;
    // the group's chunks grp, grp + BG, ...; its n-th chunk uses entry slot
    // grp * NE + n % NE
    auto fetch = [&](uint32_t n) {  // masks + entries of the group's n-th chunk
      const uint32_t cn = grp + n * C::BG;
      const uint32_t es = grp * C::NE + n % C::NE;
      if (n >= uint32_t(C::NE)) mbar_wait(eempty + es, ((n / C::NE) - 1u) & 1u);
      const uint64_t e0 = pv.coff[c0 + cn], e1 = pv.coff[c0 + cn + 1];
      const uint32_t bytes = uint32_t(e1 - e0) * 4u;
      uint8_t* slot = ering + es * L.eslot;
      mbar_expect_tx(efull + es, 512u + bytes);
      bulk_load(slot, pv.dmask + uint64_t(c0 + cn) * kPanelRows, 512u, efull + es);
      if (bytes) bulk_load(slot + 512, pv.dent + e0, bytes, efull + es);
    };
    if (wq == 0 && lane == 0)
      for (uint32_t n = 0; n + 1 < uint32_t(C::NE) && grp + n * C::BG < nch; ++n) fetch(n);
    for (uint32_t c = grp, n = 0; c < nch; c += C::BG, ++n) {
      if (wq == 0 && lane == 0 && c + (C::NE - 1) * C::BG < nch) fetch(n + C::NE - 1);
      const uint32_t es = grp * C::NE + n % C::NE;
      mbar_wait(efull + es, (n / C::NE) & 1u);
      const uint32_t sb = smem_u32(ering + es * L.eslot);
      const uint32_t m = ld_shared_u32(sb + r * 4);
      const uint4 mm = ld_shared_u4(sb + lane * 16);  // rows 4 lane .. 4 lane + 3
      const uint32_t s4 = __popc(mm.x) + __popc(mm.y) + __popc(mm.z) + __popc(mm.w);
      const uint32_t base = __reduce_add_sync(0xFFFFFFFFu, lane < 8 * wq ? s4 : 0u);  // rows < 32 wq
      const uint32_t own = __popc(m);
      uint32_t incl = own;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= uint32_t(o)) incl += t;
      }
      // this row's entries: words [base + incl - own, + own) after the masks
      const uint32_t* ev = reinterpret_cast<const uint32_t*>(ering + es * L.eslot + 512) + (base + incl - own);
      uint32_t av[32];
      uint32_t t = 0;
#pragma unroll
      for (int k = 0; k < 32; ++k) {
        const uint32_t on = (m >> k) & 1u;
        const uint32_t w = ev[t];  // in the slot even past the row (16 B slack)
        av[k] = on ? (w & 0xFFFFE000u) : 0u;
        t += on;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(eempty + es);
      if (c >= uint32_t(C::NA)) {  // MMA(c - NA) retired: A buffer free
        const uint32_t cp = c - C::NA;
        mbar_wait(bempty + cp % NB, (cp / NB) & 1u);
      }
      tc_fence_after();
      tmem_st32(tmem + lanes + C::ACOL + (c % C::NA) * 32u, av);
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(afull + c % C::NA);
    }
  } else if (warp < C::IW) {
    // ------------------------------------------------------------ accumulators
    const uint32_t q = warp & 3u;
    const uint64_t r = p * kPanelRows + q * 32 + lane;
    const uint32_t lanes = (q * 32u) << 16;
    for (uint32_t g = 0; g < ngroups; ++g) {
      const uint32_t buf = g % C::NF;
      mbar_wait(accfull + buf, (g / C::NF) & 1u);
      tc_fence_after();
#pragma unroll
      for (int cc = 0; cc < DC; cc += 16) {
        uint32_t v[16], sm[16];
        tmem_ld16(tmem + lanes + C::BUF0 + buf * DC + cc, v);
        if (g) tmem_ld16(tmem + lanes + cc, sm);
        tmem_ld_wait();
        if (g) {
#pragma unroll
          for (int j = 0; j < 16; ++j) v[j] = __float_as_uint(__uint_as_float(sm[j]) + __uint_as_float(v[j]));
        }
        tmem_st16(tmem + lanes + cc, v);
      }
      tmem_st_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(accempty + buf);
    }
    tc_fence_after();
    const bool rv = r < pv.n_rows;
    float* o = out + r * ldo + fbase;
    bool bad = false;
#pragma unroll
    for (int cc = 0; cc < DC; cc += 16) {
      uint32_t v[16];
      if (ngroups) {
        tmem_ld16(tmem + lanes + cc, v);
        tmem_ld_wait();
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) v[j] = 0u;
      }
      if (rv) {
#pragma unroll
        for (int j = 0; j < 16; ++j)
          bad |= cc + j < dvalid && (v[j] & 0x7F800000u) == 0x7F800000u;
        if (vec_out && dvalid == DC) {
#pragma unroll
          for (int j = 0; j < 4; ++j)
            reinterpret_cast<float4*>(o + cc)[j] =
                make_float4(__uint_as_float(v[4 * j]), __uint_as_float(v[4 * j + 1]),
                            __uint_as_float(v[4 * j + 2]), __uint_as_float(v[4 * j + 3]));
        } else {
#pragma unroll
          for (int j = 0; j < 16; ++j)
            if (cc + j < dvalid) o[cc + j] = __uint_as_float(v[j]);
        }
      }
    }
    if (nonfinite && __any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(nonfinite, 1u);
  } else if (warp == C::IW) {
    // ------------------------------------------------------------ MMA issuer
    if (lane == 0) {
      constexpr uint32_t idesc = idesc_tf32(DC, true);
      for (uint32_t c = 0; c < nch; ++c) {
        const uint32_t g = c / C::FOLD, buf = g % C::NF;
        const bool first = (c % C::FOLD) == 0;
        if (first && g >= uint32_t(C::NF)) mbar_wait(accempty + buf, ((g / C::NF) - 1u) & 1u);
        const uint32_t ds = c % NB;
        mbar_wait(afull + c % C::NA, (c / C::NA) & 1u);
        mbar_wait(bfull + ds, (c / NB) & 1u);
        fence_async_smem();  // cp.async (generic proxy) -> MMA (async proxy)
        tc_fence_after();
        const uint32_t dt = tmem + C::BUF0 + buf * DC;
        const uint32_t at = tmem + C::ACOL + (c % C::NA) * 32u;
        const uint32_t b0 = smem_u32(bring + ds * C::B_BYTES);
#pragma unroll
        for (uint32_t ks = 0; ks < kChunkCols / 8; ++ks)
          umma_tf32_ts(dt, at + ks * 8, desc_mn32(b0 + ks * 1024, 4096, 512), idesc, (first && ks == 0) ? 0u : 1u);
        umma_commit(bempty + ds);  // B slot and A buffer of chunk c free
        if ((c % C::FOLD) == C::FOLD - 1 || c + 1 == nch) umma_commit(accfull + buf);
      }
    }
  } else {
    // ------------------------------------------------------------ B loaders
    const uint32_t par = warp - C::LW;
    constexpr uint32_t LPR = DC / 4, RPG = 32 / LPR;  // lanes per feature row, rows per instruction
    const uint32_t j = lane % LPR, jj = j & 7u;
    uint32_t coln = par < nch ? __ldg(pv.dcols + uint64_t(c0 + par) * kChunkCols + lane) : 0u;
    // lanes 0, 1: the chunk's entry range, one iteration ahead
    uint64_t offn = par + lane <= nch && lane < 2 ? __ldg(pv.coff + c0 + par + lane) : 0u;
    for (uint32_t c = par; c < nch; c += C::NL) {
      const uint32_t ds = c % NB;
      const uint32_t col = coln;
      coln = c + C::NL < nch ? __ldg(pv.dcols + uint64_t(c0 + c + C::NL) * kChunkCols + lane) : 0u;
      const uint64_t e0 = __shfl_sync(0xFFFFFFFFu, offn, 0), e1 = __shfl_sync(0xFFFFFFFFu, offn, 1);
      offn = c + C::NL + lane <= nch && lane < 2 ? __ldg(pv.coff + c0 + c + C::NL + lane) : 0u;
      mbar_wait(bempty + ds, ((c / NB) & 1u) ^ 1u);
#if SGTK_TM_PREFETCH
      // the builders bulk-copy this chunk's masks + entries only NE - 1 chunks
      // ahead: bring them into L2 now, ~NB chunks ahead
      if (lane == 0) {
        bulk_prefetch_l2(pv.dmask + uint64_t(c0 + c) * kPanelRows, 512u);
        if (e1 > e0) bulk_prefetch_l2(pv.dent + e0, uint32_t(e1 - e0) * 4u);
      }
#else
      (void)e0, (void)e1;
#endif
      const uint32_t bst = smem_u32(bring + ds * C::B_BYTES);
#pragma unroll
      for (uint32_t tt = 0; tt < 32 / RPG; ++tt) {
        const uint32_t k = tt * RPG + lane / LPR;
        const uint32_t ck = __shfl_sync(0xFFFFFFFFu, col, k);
        const bool real = ck != 0xFFFFFFFFu && int(4 * j) < dvalid;
        // MN-major SWIZZLE_128B_BASE32B, as spmm_panel_kernel's gather_b
        const uint32_t dst = bst + (j >> 3) * 4096u + (k >> 2) * 512u + (k & 3u) * 128u +
                             ((((jj >> 1) ^ (k & 3u)) << 5) | ((jj & 1u) << 4));
        cp_async16(dst, real ? x + uint64_t(ck) * ldx + fbase + 4 * j
                             : reinterpret_cast<const float*>(g_zero_tile) + (k * LPR + j) * 4);
      }
      cp_async_arrive_noinc(bfull + ds);
    }
    cp_async_wait<0>();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == C::IW) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// ---------------------------------------------------------------------------
// Sparse part on the CUDA cores: one warp per work item (a row's sparse
// edges, or a <= kSegEdges segment of a hub row), lanes over features
// (FPL = 1 or 2 consecutive floats per lane: 128- or 256-byte coalesced
// rows), BATCH / EPI = 6 edge rows in flight per lane (measured best
// against 2..8), edges of a batch broadcast by shuffle.  Direct items continue the row's sum from the dense result in
// `out` (out = dense + e0 + e1 + ...); segments write partials that
// long_rows_kernel adds in segment order.  Deterministic throughout.
// ---------------------------------------------------------------------------
template <int FPL, int PREC>
__global__ void __launch_bounds__(256)
sparse_rows_kernel(const uint4* __restrict__ items, uint64_t n_items, const uint2* __restrict__ sent,
                   const float* __restrict__ x, uint64_t ldx, uint64_t d, uint64_t fbase,
                   float* __restrict__ out, uint64_t ldo, float* __restrict__ part, uint64_t ldp,
                   uint32_t* __restrict__ nonfinite) {
  // lanes: LPE per edge (one float4 of features each), EPI edges per
  // instruction -> 4 MACs per lane per edge, 4x fewer instructions than
  // lane = feature; the EPI partial sums merge by a fixed shuffle tree
  constexpr uint32_t DC = 32 * FPL, LPE = DC / 4, EPI = 32 / LPE;
#ifndef SGTK_SPARSE_BATCH1
#define SGTK_SPARSE_BATCH1 24
#endif
#ifndef SGTK_SPARSE_BATCH2
#define SGTK_SPARSE_BATCH2 12
#endif
  // edges per batch (loads in flight per warp: BATCH / EPI float4 per lane)
  constexpr uint32_t BATCH = FPL == 1 ? uint32_t(SGTK_SPARSE_BATCH1) : uint32_t(SGTK_SPARSE_BATCH2);
  const uint32_t lane = threadIdx.x & 31, sub = lane / LPE, jq = lane % LPE;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint64_t f = fbase + 4u * jq;  // this lane's first feature
  const int fv = f >= d ? 0 : (d - f >= 4 ? 4 : int(d - f));
  const bool vec = fv == 4 && (ldx & 3) == 0;
  bool bad = false;
  for (uint64_t it = warp; it < n_items; it += nw) {
    const uint4 w = items[it];
    const bool direct = w.w == 0xFFFFFFFFu;
    float* dst = direct ? out + uint64_t(w.x) * ldo + f : part + uint64_t(w.w) * ldp + (f - fbase);
    float acc[4] = {0.f, 0.f, 0.f, 0.f};
    if (direct && sub == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] = i < fv ? dst[i] : 0.0f;
    }
    for (uint32_t e = w.y; e < w.z; e += BATCH) {
      const uint32_t cnt = min(BATCH, w.z - e);
      uint2 en = lane < cnt ? sent[e + lane] : make_uint2(0u, 0u);
      if constexpr (PREC == SGTK_TF32) en.y = tf32_op(__uint_as_float(en.y));  // x arrives pre-rounded
      float4 xv[BATCH / EPI];
      float av[BATCH / EPI];
#pragma unroll
      for (uint32_t k = 0; k < BATCH / EPI; ++k) {
        const uint32_t u = k * EPI + sub;
        const uint32_t c = __shfl_sync(0xFFFFFFFFu, en.x, u);
        av[k] = __uint_as_float(__shfl_sync(0xFFFFFFFFu, en.y, u));
        const float* src = x + uint64_t(c) * ldx + f;
        if (u < cnt && vec) {
          xv[k] = __ldg(reinterpret_cast<const float4*>(src));
        } else {
          xv[k].x = (u < cnt && fv > 0) ? __ldg(src) : 0.0f;
          xv[k].y = (u < cnt && fv > 1) ? __ldg(src + 1) : 0.0f;
          xv[k].z = (u < cnt && fv > 2) ? __ldg(src + 2) : 0.0f;
          xv[k].w = (u < cnt && fv > 3) ? __ldg(src + 3) : 0.0f;
        }
        if (u >= cnt) av[k] = 0.0f;
      }
#pragma unroll
      for (uint32_t k = 0; k < BATCH / EPI; ++k) {  // paired FFMA2: same per-element FMAs
        const float2 a2 = make_float2(av[k], av[k]);
        const float2 lo = __ffma2_rn(a2, make_float2(xv[k].x, xv[k].y), make_float2(acc[0], acc[1]));
        const float2 hi = __ffma2_rn(a2, make_float2(xv[k].z, xv[k].w), make_float2(acc[2], acc[3]));
        acc[0] = lo.x;
        acc[1] = lo.y;
        acc[2] = hi.x;
        acc[3] = hi.y;
      }
    }
#pragma unroll
    for (uint32_t o2 = LPE; o2 < 32; o2 <<= 1)
#pragma unroll
      for (int i = 0; i < 4; ++i) acc[i] += __shfl_xor_sync(0xFFFFFFFFu, acc[i], o2);
    if (sub == 0) {
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (i < fv) {
          dst[i] = acc[i];
          bad |= direct && !isfinite(acc[i]);
        }
    }
  }
  if (nonfinite && __any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(nonfinite, 1u);
}

// Hub rows: out[row] += segment partials, in segment order.
__global__ void long_rows_kernel(const uint4* __restrict__ lrows, uint64_t n_long,
                                 const float* __restrict__ part, uint64_t ldp, uint64_t d,
                                 uint64_t fbase, uint64_t dc, float* __restrict__ out, uint64_t ldo,
                                 uint32_t* __restrict__ nonfinite) {
  bool bad = false;
  for (uint64_t i = blockIdx.x; i < n_long; i += gridDim.x) {
    const uint4 w = lrows[i];
    for (uint64_t f = threadIdx.x; f < dc && fbase + f < d; f += blockDim.x) {
      float s = out[uint64_t(w.x) * ldo + fbase + f];
      for (uint32_t k = 0; k < w.z; ++k) s += part[uint64_t(w.y + k) * ldp + f];
      out[uint64_t(w.x) * ldo + fbase + f] = s;
      bad |= !isfinite(s);
    }
  }
  if (nonfinite && bad) atomicOr(nonfinite, 1u);
}

// X rounded once per call to TF32 (RNE, tf32_round_value semantics), rows
// padded to a multiple of 4 floats with zeros: both the tensor-core B tiles
// and the CUDA-core edges then read ready operands.
__global__ void tf32_rows_kernel(const float* __restrict__ x, uint64_t ldx, uint64_t rows,
                                 uint64_t d, float* __restrict__ y, uint64_t ldy) {
  const uint64_t q4 = ldy / 4, total = rows * q4;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = i / q4, c = (i - r * q4) * 4;
    float4 v;
    if (c + 4 <= d && (ldx & 3) == 0) {
      v = __ldg(reinterpret_cast<const float4*>(x + r * ldx + c));
    } else {
      v.x = c < d ? x[r * ldx + c] : 0.f;
      v.y = c + 1 < d ? x[r * ldx + c + 1] : 0.f;
      v.z = c + 2 < d ? x[r * ldx + c + 2] : 0.f;
      v.w = c + 3 < d ? x[r * ldx + c + 3] : 0.f;
    }
    reinterpret_cast<float4*>(y + r * ldy)[c / 4] =
        make_float4(tf32_rne(v.x), tf32_rne(v.y), tf32_rne(v.z), tf32_rne(v.w));
  }
}

int device_major() {
  static int major = -1;
  static std::once_flag once;
  std::call_once(once, [] {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev);
  });
  return major;
}

constexpr uint32_t kSmemCap = 227u * 1024u;

// Entry slots sized for the graph's largest chunk; B/entry ring as deep as fits.
template <int DC, int PREC>
bool panel_smem(uint32_t max_entries, PanelSmem& L) {
  using C = PanelCfg<DC, PREC>;
  L.dslot = ((max_entries + 3) / 4 * 4 * 4 + 127) / 128 * 128;
  L.bring_off = kBarBytes + C::NS * C::A_STAGE;
  const uint32_t cap = C::CTAS == 2 ? kSmemCap / 2 - 1024 : kSmemCap;
  for (uint32_t nd = kMaxND; nd >= uint32_t(C::NS); nd -= C::NS) {
    L.nd = nd;
    L.dring_off = L.bring_off + nd * C::B_STAGE;
    L.total = L.dring_off + nd * C::NV * L.dslot + 1024 /*alignment slack*/;
    if (L.total <= cap) return true;
  }
  return false;
}

template <int DC, int PREC>
bool launch_dense(const PanelView& v, uint64_t P, uint32_t max_entries, const float* x,
                  uint64_t ldx, uint64_t d, float* out, uint64_t ldo, int vec_out,
                  uint32_t* nonfinite, cudaStream_t s) {
  PanelSmem L;
  if (!panel_smem<DC, PREC>(max_entries, L)) return false;
  once_per_device(reinterpret_cast<const void*>(&spmm_panel_kernel<DC, PREC, false>), [] {
    cudaFuncSetAttribute(spmm_panel_kernel<DC, PREC, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(kSmemCap));
    cudaFuncSetAttribute(spmm_panel_kernel<DC, PREC, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(kSmemCap));
  });
  dim3 grid(unsigned(P), unsigned((d + DC - 1) / DC));
  // SGTK_PANEL_TRACE=<file>: per-chunk pipeline timestamps of the first 4
  // CTAs (only in a build with -DSGTK_TRACE; otherwise the file is zeros)
  static long long* trace = [] {
    long long* t = nullptr;
    if (std::getenv("SGTK_PANEL_TRACE")) {
      cudaMalloc(&t, 4 * 256 * 8 * 8);
      cudaMemset(t, 0, 4 * 256 * 8 * 8);
    }
    return t;
  }();
  // PAD measured: d = 8/16/24 0.28/0.27/0.25 -> 0.22/0.23/0.23 ms; at d = 48
  // (DC = 64) copying the zero features stays faster (0.34 vs 0.38 ms)
  if (DC == 32 && d % DC)
    spmm_panel_kernel<DC, PREC, true><<<grid, kPanelThreads, L.total, s>>>(v, L, x, ldx, d, out, ldo,
                                                                         vec_out, nonfinite, trace);
  else
    spmm_panel_kernel<DC, PREC, false><<<grid, kPanelThreads, L.total, s>>>(v, L, x, ldx, d, out, ldo,
                                                                          vec_out, nonfinite, trace);
  if (trace) {
    std::vector<long long> h(4 * 256 * 8);
    cudaMemcpy(h.data(), trace, h.size() * 8, cudaMemcpyDeviceToHost);
    if (FILE* f = std::fopen(std::getenv("SGTK_PANEL_TRACE"), "wb")) {
      std::fwrite(h.data(), 8, h.size(), f);
      std::fclose(f);
    }
  }
  CU_LAUNCH("spmm_panel_kernel");
  return true;
}

// TF32 dense part with A in TMEM (spmm_tm_kernel): entry slots sized for the
// graph's largest chunk, then the deepest B ring that keeps two CTAs per SM.
template <int DC>
bool launch_dense_tm(const PanelView& v, uint64_t P, uint32_t max_entries, const float* x, uint64_t ldx,
                     uint64_t d, float* out, uint64_t ldo, int vec_out, uint32_t* nonfinite, cudaStream_t s) {
  using C = TmCfg<DC>;
  static const bool on = [] {
    const char* e = std::getenv("SGTK_SPMM_TM");
    return e && std::atoi(e) != 0;
  }();
  if (!on) return false;
  TmSmem L;
  L.eslot = (512u + (max_entries + 3) / 4 * 16u + 16u + 127u) / 128u * 128u;
  const uint32_t cap = kSmemCap / 2 - 1024;
  for (L.nb = C::NBMAX; L.nb >= 4; --L.nb) {
    L.ering_off = 1024 + L.nb * C::B_BYTES;
    L.total = L.ering_off + C::BG * C::NE * L.eslot + 1024 /*alignment slack*/;
    if (L.total <= cap) break;
  }
  if (L.nb < 4) return false;
  once_per_device(reinterpret_cast<const void*>(&spmm_tm_kernel<DC>), [] {
    cudaFuncSetAttribute(spmm_tm_kernel<DC>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(kSmemCap));
  });
  dim3 grid(unsigned(P), unsigned((d + DC - 1) / DC));
  spmm_tm_kernel<DC><<<grid, C::THREADS, L.total, s>>>(v, L, x, ldx, d, out, ldo, vec_out, nonfinite);
  CU_LAUNCH("spmm_tm_kernel");
  return true;
}

// SGTK_PANEL_DEBUG=1: tensor-core part only, =2: CUDA-core part only
// (timing experiments; results are then partial sums)
std::atomic<int> g_panel_debug{-1};
int panel_debug() {
  int v = g_panel_debug.load(std::memory_order_relaxed);
  if (v < 0) {
    const char* e = std::getenv("SGTK_PANEL_DEBUG");
    v = e ? std::atoi(e) : 0;
    g_panel_debug.store(v, std::memory_order_relaxed);
  }
  return v;
}

void launch_sparse(const Panels& pn, const uint2* sent, const float* x, uint64_t ldx, uint64_t d,
                   float* out, uint64_t ldo, uint32_t* nonfinite, cudaStream_t s, int prec) {
  if (!pn.n_items) return;
  const uint64_t dc = d <= 32 ? 32 : 64;  // features per warp pass
  float* part = nullptr;
  if (pn.n_segs) CU(cudaMallocAsync(reinterpret_cast<void**>(&part), pn.n_segs * dc * 4, s));
#ifndef SGTK_SPARSE_GRID
#define SGTK_SPARSE_GRID 4
#endif
  const unsigned blocks = unsigned(std::min<uint64_t>((pn.n_items + 7) / 8, 148ull * SGTK_SPARSE_GRID));
  for (uint64_t fb = 0; fb < d; fb += dc) {
    const uint4* it = pn.items->as<uint4>();
    if (dc == 32) {
      if (prec == SGTK_FP32)
        sparse_rows_kernel<1, SGTK_FP32><<<blocks, 256, 0, s>>>(it, pn.n_items, sent, x, ldx, d, fb, out, ldo, part, dc, nonfinite);
      else
        sparse_rows_kernel<1, SGTK_TF32><<<blocks, 256, 0, s>>>(it, pn.n_items, sent, x, ldx, d, fb, out, ldo, part, dc, nonfinite);
    } else {
      if (prec == SGTK_FP32)
        sparse_rows_kernel<2, SGTK_FP32><<<blocks, 256, 0, s>>>(it, pn.n_items, sent, x, ldx, d, fb, out, ldo, part, dc, nonfinite);
      else
        sparse_rows_kernel<2, SGTK_TF32><<<blocks, 256, 0, s>>>(it, pn.n_items, sent, x, ldx, d, fb, out, ldo, part, dc, nonfinite);
    }
    CU_LAUNCH("sparse_rows_kernel");
    if (pn.n_long) {
      long_rows_kernel<<<unsigned(std::min<uint64_t>(pn.n_long, 148ull * 4)), 64, 0, s>>>(
          pn.lrows->as<uint4>(), pn.n_long, part, dc, d, fb, dc, out, ldo, nonfinite);
      CU_LAUNCH("long_rows_kernel");
    }
  }
  if (part) CU(cudaFreeAsync(part, s));
}

}  // namespace

// ---------------------------------------------------------------- builder
namespace {
// First AGNN item of each panel (aitems hold every row, in row order, hub
// rows as consecutive segments).
void build_paitem(Panels& pn, cudaStream_t s) {
  std::vector<uint4> it = dl<uint4>(pn.aitems->p, pn.n_aitems, s);
  std::vector<uint32_t> pa(pn.P + 1, uint32_t(pn.n_aitems));
  for (uint64_t i = pn.n_aitems; i-- > 0;) pa[it[i].x / kPanelRows] = uint32_t(i);
  for (uint64_t q = pn.P; q-- > 0;) pa[q] = std::min(pa[q], pa[q + 1]);
  pn.paitem = ul(pa.data(), pa.size(), s);
  CU(cudaStreamSynchronize(s));
}

void build_dpos(const sgtk_graph& g, Panels& pn, cudaStream_t s) {
  pn.dpos = std::make_shared<DevBuf>(std::max<uint64_t>(pn.n_dent, 4) * 4);
  pn.dpos_ok = false;
  if (!pn.n_dent || !pn.P) {
    pn.dpos_ok = true;
    return;
  }
  DevBuf ov(4);
  CU(cudaMemsetAsync(ov.p, 0, 4, s));
  dpos_kernel<<<unsigned(std::min<uint64_t>(pn.P, 148ull * 16)), 256, 0, s>>>(
      pn.cptr->as<uint32_t>(), pn.coff->as<uint64_t>(), pn.dent->as<uint32_t>(), pn.deid->as<uint32_t>(),
      g.np->as<uint64_t>(), pn.P, pn.dpos->as<uint32_t>(), ov.as<uint32_t>());
  CU_LAUNCH("dpos_kernel");
  uint32_t h = 1;
  CU(cudaMemcpyAsync(&h, ov.p, 4, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  pn.dpos_ok = h == 0;
}

std::shared_ptr<Panels> build_panel_format(sgtk_graph& g, uint32_t dense_min, cudaStream_t s) {
  auto pn = std::make_shared<Panels>();
  const uint64_t n = g.n_rows, E = g.nnz;
  const uint64_t P = (n + kPanelRows - 1) / kPanelRows;
  pn->P = P;
  Windows win = build_row_windows(g, kPanelRows, s);
  const uint64_t U = win.U;
  const uint32_t* e2r = g.e2r->as<uint32_t>();
  const uint32_t* e2c = win.e2c->as<uint32_t>();
  const uint64_t* wo = win.wo->as<uint64_t>();

  DevBuf flag((U + 1) * 4), grank((U + 1) * 4);
  CU(cudaMemsetAsync(flag.p, 0, (U + 1) * 4, s));
  if (E) panel_count_kernel<<<grid_for(E, 256), 256, 0, s>>>(e2r, e2c, wo, E, flag.as<uint32_t>());
  CU_LAUNCH("panel_count_kernel");
  dense_flag_kernel<<<grid_for(U + 1, 256), 256, 0, s>>>(flag.as<uint32_t>(), U, dense_min);
  CU_LAUNCH("dense_flag_kernel");
  exclusive_scan_u32(flag.as<uint32_t>(), grank.as<uint32_t>(), U + 1, s);

  DevBuf dcnt_d(std::max<uint64_t>(P, 1) * 4);
  if (P) panel_dcount_kernel<<<grid_for(P, 256), 256, 0, s>>>(wo, grank.as<uint32_t>(), P,
                                                               dcnt_d.as<uint32_t>());
  CU_LAUNCH("panel_dcount_kernel");
  std::vector<uint32_t> dcnt = dl<uint32_t>(dcnt_d.p, P, s);
  std::vector<uint32_t> cptr(P + 1, 0);
  for (uint64_t p = 0; p < P; ++p) cptr[p + 1] = cptr[p] + (dcnt[p] + kChunkCols - 1) / kChunkCols;
  const uint64_t NC = cptr[P];
  pn->n_chunks = NC;
  pn->cptr = ul(cptr.data(), P + 1, s);
  pn->dcols = std::make_shared<DevBuf>(std::max<uint64_t>(NC * kChunkCols, 1) * 4);
  CU(cudaMemsetAsync(pn->dcols->p, 0xFF, pn->dcols->bytes, s));
  if (P)
    dcols_kernel<<<grid_for(P, 1, 148u * 16u), 256, 0, s>>>(
        wo, win.wuc->as<uint32_t>(), flag.as<uint32_t>(), grank.as<uint32_t>(),
        pn->cptr->as<uint32_t>(), P, pn->dcols->as<uint32_t>());
  CU_LAUNCH("dcols_kernel");

  // row masks from the edges, per-chunk row offsets, entry counts
  pn->dmask = std::make_shared<DevBuf>(std::max<uint64_t>(NC, 1) * kPanelRows * 4);
  CU(cudaMemsetAsync(pn->dmask->p, 0, pn->dmask->bytes, s));
  if (E)
    edge_mask_kernel<<<grid_for(E, 256), 256, 0, s>>>(e2r, e2c, wo, flag.as<uint32_t>(),
                                                      grank.as<uint32_t>(), pn->cptr->as<uint32_t>(),
                                                      E, pn->dmask->as<uint32_t>());
  CU_LAUNCH("edge_mask_kernel");
  DevBuf ccnt(std::max<uint64_t>(NC, 1) * 4);
  pn->rowoff = std::make_shared<DevBuf>(std::max<uint64_t>(NC, 1) * kPanelRows * 2);
  DevBuf& rowoff = *pn->rowoff;
  if (NC)
    row_offsets_kernel<<<grid_for(NC * 32, 256), 256, 0, s>>>(pn->dmask->as<uint32_t>(), NC,
                                                              rowoff.as<uint16_t>(), ccnt.as<uint32_t>());
  CU_LAUNCH("row_offsets_kernel");
  std::vector<uint32_t> cc = dl<uint32_t>(ccnt.p, NC, s);
  std::vector<uint64_t> coff(NC + 1, 0);
  uint32_t mx = 0;
  for (uint64_t c = 0; c < NC; ++c) {
    coff[c + 1] = coff[c] + (uint64_t(cc[c]) + 3) / 4 * 4;
    mx = std::max(mx, cc[c]);
  }
  pn->max_chunk_entries = mx;
  pn->n_dent = coff[NC];
  pn->coff = ul(coff.data(), NC + 1, s);
  const uint64_t ND = std::max<uint64_t>(pn->n_dent, 4);
  pn->dent = std::make_shared<DevBuf>(ND * 4);
  pn->dval = std::make_shared<DevBuf>(ND * 4);
  pn->deid = std::make_shared<DevBuf>(ND * 4);
  CU(cudaMemsetAsync(pn->dval->p, 0, ND * 4, s));
  CU(cudaMemsetAsync(pn->deid->p, 0xFF, ND * 4, s));
  const float* vals = g.has_values ? g.vals->as<float>() : nullptr;
  if (E)
    entry_fill_sorted_kernel<<<grid_for(E, 256), 256, 0, s>>>(
        e2r, e2c, wo, flag.as<uint32_t>(), grank.as<uint32_t>(), pn->cptr->as<uint32_t>(),
        pn->coff->as<uint64_t>(), pn->dmask->as<uint32_t>(), rowoff.as<uint16_t>(), vals, E,
        pn->dent->as<uint32_t>(), pn->dval->as<float>(), pn->deid->as<uint32_t>());
  CU_LAUNCH("entry_fill_sorted_kernel");
  if (NC)
    entry_pad_kernel<<<grid_for(NC * 32, 256), 256, 0, s>>>(ccnt.as<uint32_t>(), pn->coff->as<uint64_t>(),
                                                           pn->dmask->as<uint32_t>(), NC,
                                                           pn->dent->as<uint32_t>());
  CU_LAUNCH("entry_pad_kernel");

  DevBuf scnt((n + 1) * 4);
  CU(cudaMemsetAsync(scnt.p, 0, (n + 1) * 4, s));
  if (n)
    sparse_count_kernel<<<grid_for(n * 32, 256), 256, 0, s>>>(
        g.np->as<uint64_t>(), n, e2c, wo, flag.as<uint32_t>(), scnt.as<uint32_t>());
  CU_LAUNCH("sparse_count_kernel");
  pn->sptr = std::make_shared<DevBuf>((n + 1) * 4);
  exclusive_scan_u32(scnt.as<uint32_t>(), pn->sptr->as<uint32_t>(), n + 1, s);
  uint32_t nsp = 0;
  CU(cudaMemcpyAsync(&nsp, pn->sptr->as<uint32_t>() + n, 4, cudaMemcpyDeviceToHost, s));
  CU(cudaStreamSynchronize(s));
  pn->n_sparse = nsp;
  pn->sent = std::make_shared<DevBuf>(std::max<uint64_t>(nsp, 1) * 8);
  pn->seid = std::make_shared<DevBuf>(std::max<uint64_t>(nsp, 1) * 4);
  if (n && nsp)
    sparse_fill_kernel<<<grid_for(n * 32, 256), 256, 0, s>>>(
        g.np->as<uint64_t>(), g.el->as<uint32_t>(), vals, n, e2c, wo, flag.as<uint32_t>(),
        pn->sptr->as<uint32_t>(), pn->sent->as<uint2>(), pn->seid->as<uint32_t>());
  CU_LAUNCH("sparse_fill_kernel");

  // CUDA-core work list (host, O(N)): a row's sparse edges form one item;
  // hub rows are cut into kSegEdges segments reduced in order afterwards.
  std::vector<uint32_t> sp = dl<uint32_t>(pn->sptr->p, n + 1, s);
  std::vector<uint4> items, lrows, aitems;
  uint32_t seg = 0;
  for (uint64_t r = 0; r < n; ++r) {
    const uint32_t b = sp[r], e = sp[r + 1];
    if (e - b <= kSegEdges) {
      if (b != e) items.push_back(make_uint4(uint32_t(r), b, e, 0xFFFFFFFFu));
      aitems.push_back(make_uint4(uint32_t(r), b, e, 0xFFFFFFFFu));
    } else {
      const uint32_t k = (e - b + kSegEdges - 1) / kSegEdges;
      lrows.push_back(make_uint4(uint32_t(r), seg, k, 0u));
      for (uint32_t i = 0; i < k; ++i) {
        const uint4 it = make_uint4(uint32_t(r), b + i * kSegEdges,
                                    std::min(e, b + (i + 1) * kSegEdges), seg + i);
        items.push_back(it);
        aitems.push_back(it);
      }
      seg += k;
    }
  }
  pn->n_aitems = aitems.size();
  pn->aitems = ul(aitems.data(), aitems.size(), s);
  pn->n_items = items.size();
  pn->n_long = lrows.size();
  pn->n_segs = seg;
  pn->items = ul(items.data(), items.size(), s);
  pn->lrows = ul(lrows.data(), lrows.size(), s);
  CU(cudaStreamSynchronize(s));
  return pn;
}
}  // namespace

// ------------------------------------------------------------ panel section
// SGT1 (sgt_file.cpp:47-107) stores the reference's TransformedGraph and its
// reader rejects trailing bytes (:101-102), so the panel formats are persisted
// beside it, in "<file>.sgp": magic "SGP1", a format version, a fingerprint
// of the graph they belong to, then per panel format its scalars and its
// device arrays as (byte length, bytes) records.  Loading uploads the arrays
// into the new handle and skips build_panels.
namespace {
constexpr char kSgpMagic[4] = {'S', 'G', 'P', '1'};
constexpr uint32_t kSgpVersion = 2;  // 2: + per-chunk row offsets

uint64_t fnv(uint64_t h, const void* p, size_t n) {
  const auto* b = static_cast<const unsigned char*>(p);
  for (size_t i = 0; i < n; ++i) h = (h ^ b[i]) * 0x100000001B3ull;
  return h;
}

// The graph a panel section belongs to: sizes, geometry, node_pointer, and
// 64 evenly spaced 1 KiB windows of edge_list (a consistency check against
// stale sidecars, not a cryptographic one).
uint64_t graph_fingerprint(const sgtk_graph& g, cudaStream_t s) {
  uint64_t h = 0xCBF29CE484222325ull;
  const uint64_t hdr[7] = {g.n_rows, g.n_cols, g.nnz, g.blk_h, g.blk_w, g.block_counter, g.user.U};
  h = fnv(h, hdr, sizeof hdr);
  std::vector<uint64_t> np = dl<uint64_t>(g.np->p, g.n_rows + 1, s);
  h = fnv(h, np.data(), np.size() * 8);
  std::vector<uint32_t> win(256);
  for (uint64_t k = 0; k < 64 && g.nnz; ++k) {
    const uint64_t at = std::min<uint64_t>(g.nnz - 1, g.nnz * k / 64);
    const uint64_t cnt = std::min<uint64_t>(256, g.nnz - at);
    CU(cudaMemcpyAsync(win.data(), g.el->as<uint32_t>() + at, cnt * 4, cudaMemcpyDeviceToHost, s));
    CU(cudaStreamSynchronize(s));
    h = fnv(h, win.data(), cnt * 4);
  }
  return h;
}

template <class T>
void put(std::FILE* f, const T& v) {
  if (std::fwrite(&v, sizeof v, 1, f) != 1) raise(SGTK_ERR_IO, "SGP1: write failed");
}
template <class T>
T get(std::FILE* f) {
  T v{};
  if (std::fread(&v, sizeof v, 1, f) != 1) raise(SGTK_ERR_IO, "SGP1: truncated section");
  return v;
}
void put_buf(std::FILE* f, const std::shared_ptr<DevBuf>& b, cudaStream_t s) {
  const uint64_t n = b ? b->bytes : 0;
  put(f, n);
  if (!n) return;
  std::vector<char> h = dl<char>(b->p, n, s);
  if (std::fwrite(h.data(), 1, n, f) != n) raise(SGTK_ERR_IO, "SGP1: write failed");
}
std::shared_ptr<DevBuf> get_buf(std::FILE* f, cudaStream_t s) {
  const uint64_t n = get<uint64_t>(f);
  std::vector<char> h(n);
  if (n && std::fread(h.data(), 1, n, f) != n) raise(SGTK_ERR_IO, "SGP1: truncated section");
  auto b = std::make_shared<DevBuf>(std::max<uint64_t>(n, 16));
  if (n) CU(cudaMemcpyAsync(b->p, h.data(), n, cudaMemcpyHostToDevice, s));
  CU(cudaStreamSynchronize(s));
  return b;
}

void put_format(std::FILE* f, const Panels& pn, uint32_t dense_min, cudaStream_t s) {
  put(f, dense_min);
  const uint64_t sc[9] = {pn.P, pn.n_chunks, pn.n_dent, pn.n_sparse, pn.max_chunk_entries,
                          pn.n_items, pn.n_long, pn.n_segs, pn.n_aitems};
  for (uint64_t v : sc) put(f, v);
  for (const auto* b : {&pn.cptr, &pn.dcols, &pn.coff, &pn.dent, &pn.dval, &pn.deid, &pn.dmask,
                        &pn.rowoff, &pn.sptr, &pn.sent, &pn.seid, &pn.items, &pn.lrows,
                        &pn.aitems})
    put_buf(f, *b, s);
}

std::shared_ptr<Panels> get_format(std::FILE* f, uint32_t want_min, cudaStream_t s) {
  if (get<uint32_t>(f) != want_min) raise(SGTK_ERR_IO, "SGP1: unexpected panel format");
  auto pn = std::make_shared<Panels>();
  uint64_t sc[9];
  for (uint64_t& v : sc) v = get<uint64_t>(f);
  pn->P = sc[0];
  pn->n_chunks = sc[1];
  pn->n_dent = sc[2];
  pn->n_sparse = sc[3];
  pn->max_chunk_entries = uint32_t(sc[4]);
  pn->n_items = sc[5];
  pn->n_long = sc[6];
  pn->n_segs = sc[7];
  pn->n_aitems = sc[8];
  for (auto* b : {&pn->cptr, &pn->dcols, &pn->coff, &pn->dent, &pn->dval, &pn->deid, &pn->dmask,
                  &pn->rowoff, &pn->sptr, &pn->sent, &pn->seid, &pn->items, &pn->lrows,
                  &pn->aitems})
    *b = get_buf(f, s);
  return pn;
}
}  // namespace

void save_panel_section(const sgtk_graph& g, const std::string& path, cudaStream_t s) {
  if (!g.panels || !g.panels32) raise(SGTK_ERR, "graph has no panel formats");
  std::FILE* f = std::fopen(path.c_str(), "wb");
  if (!f) raise(SGTK_ERR_IO, "cannot write '" + path + "'");
  try {
    if (std::fwrite(kSgpMagic, 1, 4, f) != 4) raise(SGTK_ERR_IO, "SGP1: write failed");
    put(f, kSgpVersion);
    put(f, graph_fingerprint(g, s));
    put_format(f, *g.panels, kDenseMin, s);
    put_format(f, *g.panels32, kDenseMin32, s);
  } catch (...) {
    std::fclose(f);
    throw;
  }
  if (std::fclose(f) != 0) raise(SGTK_ERR_IO, "SGP1: write failed");
}

// Loads the panel formats of `path` into g when the section exists, has this
// version and belongs to this graph (fingerprint); false otherwise (the
// caller builds them).  A section that matches but is damaged raises.
bool load_panel_section(sgtk_graph& g, const std::string& path, cudaStream_t s) {
  std::FILE* f = std::fopen(path.c_str(), "rb");
  if (!f) return false;
  bool ok = false;
  try {
    char magic[4];
    if (std::fread(magic, 1, 4, f) == 4 && std::memcmp(magic, kSgpMagic, 4) == 0 &&
        get<uint32_t>(f) == kSgpVersion && get<uint64_t>(f) == graph_fingerprint(g, s)) {
      auto a = get_format(f, kDenseMin, s);
      auto b = get_format(f, kDenseMin32, s);
      const uint64_t P = (g.n_rows + kPanelRows - 1) / kPanelRows;
      if (a->P != P || b->P != P) raise(SGTK_ERR_IO, "SGP1: panel count does not match the graph");
      if (std::fgetc(f) != EOF) raise(SGTK_ERR_IO, "SGP1: trailing bytes");
      g.panels = a;
      g.panels32 = b;
      g.panels_loaded = true;
      ok = true;
    }
  } catch (...) {
    std::fclose(f);
    throw;
  }
  std::fclose(f);
  return ok;
}

// Two panel formats per graph, differing only in the dense-column threshold:
// measured, 2-edge columns are cheaper on the CUDA cores for d <= 32 (AGNN
// C4 -2%, SpMM d = 32 -2%) and on the tensor cores for d = 64 (+3% otherwise).
void build_panels(sgtk_graph& g, cudaStream_t s) {
  g.panels = build_panel_format(g, kDenseMin, s);
  g.panels32 = build_panel_format(g, kDenseMin32, s);
}

const Panels& panels_for(const sgtk_graph* g, uint64_t d) {
  // SGTK_PANEL_FORMAT=2: the >= 2-edge format at every width (experiment)
  static const bool f2 = [] {
    const char* e = std::getenv("SGTK_PANEL_FORMAT");
    return e && std::string(e) == "2";
  }();
  return d <= 32 && g->panels32 && !f2 ? *g->panels32 : *g->panels;
}

void ensure_dpos(const sgtk_graph& g, const Panels& pn, cudaStream_t s) {
  std::call_once(*pn.dpos_once, [&] { build_dpos(g, const_cast<Panels&>(pn), s); });
}
void ensure_paitem(const Panels& pn, cudaStream_t s) {
  std::call_once(*pn.paitem_once, [&] { build_paitem(const_cast<Panels&>(pn), s); });
}

void panel_debug_set(int mode) { g_panel_debug.store(mode, std::memory_order_relaxed); }
int panel_debug_mode() { return panel_debug(); }

PanelView panel_view(const sgtk_graph* g, uint64_t d) {
  const Panels& pn = panels_for(g, d);
  PanelView v{};
  v.n_rows = g->n_rows;
  v.P = pn.P;
  v.cptr = pn.cptr->as<uint32_t>();
  v.dcols = pn.dcols->as<uint32_t>();
  v.coff = pn.coff->as<uint64_t>();
  v.dent = pn.dent->as<uint32_t>();
  v.dval = pn.dval->as<float>();
  v.sptr = pn.sptr->as<uint32_t>();
  v.sent = pn.sent->as<uint2>();
  v.dmask = pn.dmask->as<uint32_t>();
  v.paitem = pn.paitem ? pn.paitem->as<uint32_t>() : nullptr;
  return v;
}

bool panel_enabled() {
  static const bool off = [] {
    const char* e = std::getenv("SGTK_SPMM_KERNEL");
    return e && std::string(e) == "tile16";
  }();
  return !off && device_major() == 10;
}

// Returns false (caller runs the 16-row tile kernel) outside this kernel's
// envelope: unaligned feature rows, a chunk too large for shared memory.
bool spmm_panel_launch(const sgtk_graph* g, const float* x, uint64_t ldx, uint64_t d,
                       const float* ev, int prec, float* out, uint64_t ldo, uint32_t* nonfinite,
                       cudaStream_t s, bool x_tf32) {
  if (!g->panels || !panel_enabled()) return false;
  if (ldx % 4 != 0 || reinterpret_cast<uintptr_t>(x) % 16 != 0) return false;
  if (g->n_rows == 0 || d == 0) return true;
  PanelView v = panel_view(g, d);
  const Panels& pn = panels_for(g, d);
  {
    PanelSmem L;
    const bool fits = (d <= 32 ? (prec == SGTK_FP32 ? panel_smem<32, SGTK_FP32>(pn.max_chunk_entries, L)
                                                    : panel_smem<32, SGTK_TF32>(pn.max_chunk_entries, L))
                               : (prec == SGTK_FP32 ? panel_smem<64, SGTK_FP32>(pn.max_chunk_entries, L)
                                                    : panel_smem<64, SGTK_TF32>(pn.max_chunk_entries, L)));
    if (!fits) return false;
  }
  // Override values: re-packed into stream-ordered scratch (pool-cached,
  // freed in stream order after the kernels; no host synchronisation).
  void* ov = nullptr;
  const uint2* sent = v.sent;
  if (ev) {
    const uint64_t nd = std::max<uint64_t>(pn.n_dent, 4), ns = std::max<uint64_t>(pn.n_sparse, 1);
    CU(cudaMallocAsync(&ov, nd * 8 + ns * 8 + 256, s));
    uint32_t* od = static_cast<uint32_t*>(ov);
    float* ovv = reinterpret_cast<float*>(od + nd);
    uint2* os = reinterpret_cast<uint2*>((reinterpret_cast<uintptr_t>(ovv + nd) + 15) & ~uintptr_t(15));
    if (pn.n_dent)
      repack_dense_kernel<<<grid_for(pn.n_dent, 256), 256, 0, s>>>(
          pn.dent->as<uint32_t>(), pn.deid->as<uint32_t>(), ev, pn.n_dent, od, ovv);
    CU_LAUNCH("repack_dense_kernel");
    if (pn.n_sparse)
      repack_sparse_kernel<<<grid_for(pn.n_sparse, 256), 256, 0, s>>>(
          pn.sent->as<uint2>(), pn.seid->as<uint32_t>(), ev, pn.n_sparse, os);
    CU_LAUNCH("repack_sparse_kernel");
    v.dent = od;
    v.dval = ovv;
    sent = os;
  }
  float* xr = nullptr;
  if (prec == SGTK_TF32 && !x_tf32) {  // x_tf32: the producer already rounded x (RNE)
    const uint64_t ldr = (d + 3) / 4 * 4;
    CU(cudaMallocAsync(reinterpret_cast<void**>(&xr), std::max<uint64_t>(g->n_cols * ldr, 4) * 4, s));
    tf32_rows_kernel<<<grid_for(g->n_cols * ldr / 4, 256), 256, 0, s>>>(x, ldx, g->n_cols, d, xr, ldr);
    CU_LAUNCH("tf32_rows_kernel");
    x = xr;
    ldx = ldr;
  }
  const int vec_out = (ldo % 4 == 0) && (reinterpret_cast<uintptr_t>(out) % 16 == 0);
  const uint32_t me = pn.max_chunk_entries;
  const int dbg = panel_debug();
  if (dbg != 2) {
    if (prec == SGTK_FP32) {
      if (d <= 32) launch_dense<32, SGTK_FP32>(v, pn.P, me, x, ldx, d, out, ldo, vec_out, nonfinite, s);
      else launch_dense<64, SGTK_FP32>(v, pn.P, me, x, ldx, d, out, ldo, vec_out, nonfinite, s);
    } else {
      // A in TMEM for full 32-feature slices (d % 32 != 0 at d <= 32: the
      // PAD form of spmm_panel_kernel)
      if (d <= 32) {
        if (d % 32 || !launch_dense_tm<32>(v, pn.P, me, x, ldx, d, out, ldo, vec_out, nonfinite, s))
          launch_dense<32, SGTK_TF32>(v, pn.P, me, x, ldx, d, out, ldo, vec_out, nonfinite, s);
      } else if (!launch_dense_tm<64>(v, pn.P, me, x, ldx, d, out, ldo, vec_out, nonfinite, s)) {
        launch_dense<64, SGTK_TF32>(v, pn.P, me, x, ldx, d, out, ldo, vec_out, nonfinite, s);
      }
    }
  } else {
    CU(cudaMemset2DAsync(out, ldo * 4, 0, d * 4, g->n_rows, s));
  }
  // non-finite results: the dense epilogue checks every row it stores, the
  // sparse kernels the rows they finish
  if (dbg != 1) launch_sparse(pn, sent, x, ldx, d, out, ldo, nonfinite, s, prec);
  if (ov) CU(cudaFreeAsync(ov, s));
  if (xr) CU(cudaFreeAsync(xr, s));
  return true;
}

}  // namespace sgtkcu
