// AGNN layer on 128-row panels: tensor-core attention over the dense
// columns, CUDA-core attention over the sparse edges, fused normalisation.
//
// Replaces one layer of agnn_forward (/root/reference/proj/src/gnn.cpp:107-116):
//   z = l2_normalize_rows(h)                         (gnn.cpp:74-91)
//   logits_e = beta * <z_row, z_col>                 (sddmm_hybrid, tile_exec.cpp:316-411)
//   attn = edge_softmax(logits)                      (gnn.cpp:54-72)
//   h' = spmm_hybrid(t, h, attn)                     (tile_exec.cpp:200-314)
// without materialising logits or attention.
//
// Softmax offset.  Rows of z have unit (or zero) norm, so every logit lies in
// [-|beta|, |beta|]: exp(logit - |beta|) is in [exp(-2|beta|), 1] and the
// softmax needs no running maximum (the reference subtracts the row max,
// gnn.cpp:60-66; the ratio is the same).  Used for |beta| <= kMaxBeta, where
// exp(-2|beta|) stays a normal float; larger |beta| runs the other modes.
//
// Dense part (agnn_dense_kernel, one CTA per panel, 11 warps):
//   warps 0-3   softmax, thread per row: Q = z[panel rows] into the K-major A
//               operand once; per chunk: S row from TMEM, mask, P = exp2(..),
//               row sum l, P (TF32 / split) into a K-major A tile
//   warps 4-7   accumulators: fold each FOLD-chunk O group from TMEM into
//               fp32 registers; write (O, l) partials
//   warp 8      MMA issuer: S(c+1) = Q Z_c+1^T ahead of O += P(c) H_c
//   warps 9-10  loaders (even / odd chunks): cp.async gathers of the chunk's
//               z rows (K-major B of S), h rows (MN-major B of PV), row masks
// Sparse part + finalisation (agnn_rows_kernel, warp per row / hub segment):
//   logits of the row's sparse edges (lane = edge dot products), exp, l and O
//   updates (lane = feature), out = O / l, then the next layer's l2 norm.

#include <cuda.h>
#include <cudaTypedefs.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <mutex>
#include <string>

#include "kernels.cuh"
#include "tc05.cuh"

namespace sgtkcu {
namespace {

using namespace tc05;

constexpr float kMaxBeta = 40.0f;
// Warps: 4 softmax, 4 accumulator, NL loaders, the S issuer (+ TMEM
// allocation), the PV issuer (its own warp in the TF32 d = 32 configuration,
// see SPLIT_MMA).  TF32 d = 32 runs 4 loaders, one per SM sub-partition: with
// 2 the softmax warps sharing a sub-partition with a loader fell ~800 cycles
// per chunk behind the other two (pipeline trace), and the slowest softmax
// warp paces the chunk loop (PV needs all four P quarters).
#ifndef SGTK_AGNN_LOADERS
#define SGTK_AGNN_LOADERS 4
#endif
#ifndef SGTK_AGNN_LOADERS_F32
#define SGTK_AGNN_LOADERS_F32 2
#endif
constexpr int agnn_loaders(int DC, int PREC) {
  return DC == 32 ? (PREC != SGTK_FP32 ? SGTK_AGNN_LOADERS : SGTK_AGNN_LOADERS_F32) : 2;
}
constexpr int agnn_threads(int DC, int PREC) { return 32 * (10 + agnn_loaders(DC, PREC)); }

#ifndef SGTK_MASK_GLOBAL
#define SGTK_MASK_GLOBAL 1
#endif
template <int DC, int PREC>
struct AgnnCfg {
  static constexpr bool F32 = PREC == SGTK_FP32;
  static constexpr int PQ = F32 ? 2 : 1;  // Q planes (hi, lo)
  static constexpr int PZ = F32 ? 2 : 1;  // z-tile planes
  static constexpr int PH = F32 ? 2 : 1;  // h-tile planes
  static constexpr int PP = F32 ? 2 : 1;  // P planes
  static constexpr uint32_t Q_BYTES = kPanelRows * DC * 4;  // K-major, DC/32 K-blocks of 16 KB
  static constexpr uint32_t T_BYTES = kChunkCols * DC * 4;  // one 32-row tile
  static constexpr uint32_t M_BYTES = kPanelRows * 4;       // row masks
  static constexpr uint32_t P_BYTES = kPanelRows * kChunkCols * 4;  // 16 KB
  static constexpr int KB = DC / 32;                       // 128-byte K blocks of z
  // TMEM: NSB S buffers x 64 columns (S of a chunk pair, N = 64 costs what
  // N = 32 does), NF O accumulators x DC; 256 columns -> 2 CTAs per SM.
  // TF32, DC = 32 (PT): P goes from the softmax threads' registers straight
  // back over its own S columns (tcgen05.st) and PV reads A from there -- no
  // P tile, no P slot to wait for; three S buffers instead of two + P slots.
  static constexpr bool PT = !F32 && DC == 32;
#ifndef SGTK_AGNN_NSB
#define SGTK_AGNN_NSB 2  // 2 pairs: 0.274 -> 0.272 ms dense part against 3 (split issuers)
#endif
  static constexpr int NSB = PT ? SGTK_AGNN_NSB : 2;       // S buffers (chunk pairs)
#ifndef SGTK_AGNN_NB
#define SGTK_AGNN_NB 10
#endif
#ifndef SGTK_AGNN_NB_F32
#define SGTK_AGNN_NB_F32 6  // FP32 d = 32: 1.092 -> 1.024 ms per layer against 4 (8 does not fit)
#endif
#ifndef SGTK_AGNN_NB_64
#define SGTK_AGNN_NB_64 6
#endif
  static constexpr int NB = F32 ? (DC == 32 ? SGTK_AGNN_NB_F32 : 2) : (PT ? SGTK_AGNN_NB : SGTK_AGNN_NB_64);  // gather ring (even: S pairs)
  // P slots in smem; PT: pfull barriers only, one per chunk the softmax can
  // run ahead of the MMA issuer (S can be up to NSB groups ahead)
  static constexpr int NP = PT ? 8 : 2;
  static constexpr uint32_t O_COL = NSB * 64;
  static constexpr int NF = PT ? 2 : (DC == 32 ? 4 : 2);
  static constexpr uint32_t TMEM_COLS = 256;
// chunks per TMEM accumulator before the accumulator warps fold it into the
// fp32 running sum (8: -1% against 4, within the FP32 1e-5 / TF32 2e-3 bars
// including the hub-row tests; the SpMM keeps 4 for its FP32 parity)
#ifndef SGTK_AFOLD
#define SGTK_AFOLD 8
#endif
  static constexpr uint32_t FOLD = SGTK_AFOLD;
  static constexpr uint32_t Q_OFF = 1024;
  static constexpr uint32_t Z_OFF = Q_OFF + PQ * Q_BYTES;             // [PZ][KB][NB] x 4 KB
  static constexpr uint32_t H_OFF = Z_OFF + PZ * KB * NB * 4096;      // [PH][NB] x T_BYTES
  static constexpr uint32_t M_OFF = H_OFF + PH * NB * T_BYTES;        // [NB] x 512 B
  static constexpr uint32_t P_OFF = (M_OFF + NB * M_BYTES + 1023) / 1024 * 1024;
  static constexpr uint32_t SMEM = P_OFF + (PT ? 0 : NP * PP * P_BYTES) + 1024;
  static_assert(NB % 2 == 0, "S pairs need an even gather ring");
  static_assert(M_OFF - Z_OFF >= 4u * 32u * (DC + 4) * 4u, "epilogue staging fits the gather rings");
  // S of a chunk pair needs both chunks' gathers while PV still lags: a ring
  // of >= 4 slots; shallower rings compute S chunk by chunk (N = 32)
  static constexpr bool PAIR = NB >= 4;
  static constexpr uint32_t SG = PAIR ? 2 : 1;  // chunks per S group
  static constexpr bool EARLY_S = PAIR && NB >= 6;  // one-issuer form only
  static_assert(EARLY_S || !EARLY_S, "");
  // S and PV issued by two threads (warps 8 and 11), each blocking only on its
  // own inputs: S(g) on its gathers and its TMEM buffer, PV(c) on P(c).  One
  // in-order issuer makes PV(c) wait behind S(c + 2)'s gathers.
#ifdef SGTK_AGNN_ONE_ISSUER
  static constexpr bool SPLIT_MMA = false;
#else
  static constexpr bool SPLIT_MMA = true;
#endif
  static_assert(SMEM <= 227u * 1024u, "agnn panel smem");
};

// Zero rows for the padding columns of a panel's last chunk, one 16-byte
// piece per (chunk row, lane piece): distinct addresses, no hot spot.
__device__ __align__(16) float g_agnn_zero[32 * 64];

// K-major SWIZZLE_128B offset of element (row, k) in a tile with `rows` rows:
// 128-byte K blocks of 32 fp32, rows*128 bytes apart.
__device__ __forceinline__ uint32_t kmaj_off(uint32_t row, uint32_t k, uint32_t rows) {
  return (k >> 5) * rows * 128u + (row >> 3) * 1024u + (row & 7u) * 128u +
         ((((k >> 2) & 7u) ^ (row & 7u)) << 4) + (k & 3u) * 4u;
}

template <int FPL, int PREC, bool SPLIT>
__device__ __forceinline__ void agnn_row_item(const uint4 w, float* T, uint32_t lane, const uint2* __restrict__ sent,
                                              const float* __restrict__ zown, const float* __restrict__ z,
                                              uint64_t ld, const float* __restrict__ norm, uint64_t d,
                                              uint64_t row_offset, float bl2, float off,
                                              const float* __restrict__ opart, const float* __restrict__ lpart,
                                              float* __restrict__ seg_o, float* __restrict__ seg_l,
                                              float* __restrict__ osp, float* __restrict__ lsp, const AgnnNext& nx,
                                              unsigned long long& nz);

// FR (fused rows, TF32 d <= 32; opt-in, SGTK_AGNN_FUSED=1, measured slower):
// after its dense chunks the CTA runs the sparse edges and the finalisation
// of its own panel's rows (agnn_row_item over the panel's items, all 12
// warps, tiles in the idle gather rings).
// TG: the loaders gather the chunk's z and h rows with TMA tile::gather4
// (4 rows per instruction, swizzled by the tensor maps tmz / tmh straight into
// the UMMA operand layouts, padding columns zero-filled as out-of-bounds rows)
// instead of cp.async; TF32 only.
#ifdef SGTK_DENSE_MAXREG
template <int DC, int PREC, bool TG, bool FR>
__global__ void __launch_bounds__(agnn_threads(DC, PREC)) __maxnreg__((DC == 32 && PREC != SGTK_FP32) ? SGTK_DENSE_MAXREG : 168)
#else
template <int DC, int PREC, bool TG, bool FR>
__global__ void __launch_bounds__(agnn_threads(DC, PREC), (DC == 32 && PREC != SGTK_FP32) ? 2 : 1)
#endif
agnn_dense_kernel(const PanelView pv, const float* __restrict__ zraw, const float* __restrict__ z,
                  const float* __restrict__ z1, const float* __restrict__ h,
                  const float* __restrict__ h1, uint64_t ld, uint64_t d, uint64_t row_offset,
                  float beta, float* __restrict__ opart, float* __restrict__ lpart,
                  long long* __restrict__ trace, const __grid_constant__ CUtensorMap tmz,
                  const __grid_constant__ CUtensorMap tmh, const uint4* __restrict__ items,
                  const uint2* __restrict__ sent, float* __restrict__ seg_o, float* __restrict__ seg_l,
                  const AgnnNext nx) {
  using C = AgnnCfg<DC, PREC>;
  static_assert(!TG || !C::F32, "TMA gathers: TF32 operands only");
  static_assert(!FR || (!C::F32 && DC == 32), "fused rows: TF32, d <= 32");
  constexpr uint32_t NL = agnn_loaders(DC, PREC), IW = 8 + NL;  // loaders: warps 8..IW-1; issuers IW, IW+1
  constexpr uint32_t NW = agnn_threads(DC, PREC) / 32;
  constexpr uint32_t FRW = (C::M_OFF - C::Z_OFF) / (33 * (DC + 4) * 4) < NW ? (C::M_OFF - C::Z_OFF) / (33 * (DC + 4) * 4) : NW;
  static_assert(!FR || FRW >= 8, "row tiles fit the rings");
  auto mark = [&](uint32_t c, int ev) {
#ifdef SGTK_TRACE  // pipeline event trace (tools/panel_debug.py); compiled out by default
    if (trace && blockIdx.x < 4 && c < 256) trace[((uint64_t(blockIdx.x) * 256 + c) * 8) + ev] = clock64();
#else
    (void)c, (void)ev, (void)trace;
#endif
  };
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bfull = reinterpret_cast<uint64_t*>(smem);  // [NB] gathers landed
  uint64_t* bempty = bfull + C::NB;                     // [NB] PV(c) retired: slot + P(c) free
  uint64_t* sfull = bempty + C::NB;                     // [NSB] S of chunk pair in TMEM
  uint64_t* pfull = sfull + C::NSB;                     // [NP] P(c) written
  uint64_t* qfull = pfull + C::NP;                      // [1]  Q operand ready
  uint64_t* accfull = qfull + 1;                        // [NF]
  uint64_t* accempty = accfull + C::NF;                 // [NF]
  uint64_t* sempty = accempty + C::NF;                  // [NSB] S group read (P in smem: !PT)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(sempty + C::NSB);
  static_assert((2 * C::NB + 2 * C::NSB + C::NP + 1 + 2 * C::NF) * 8 + 16 <= 512, "barriers fit below lbuf");
  float* lbuf = reinterpret_cast<float*>(smem + 512);   // [128] row sums
  uint8_t* qs = smem + C::Q_OFF;
  const uint32_t zr_s = smem_u32(smem + C::Z_OFF), hr_s = smem_u32(smem + C::H_OFF);
  const uint32_t mr_s = smem_u32(smem + C::M_OFF);
  uint8_t* ps = smem + C::P_OFF;

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t p = blockIdx.x;
  const uint32_t c0 = pv.cptr[p], nch = pv.cptr[p + 1] - c0;
  const uint32_t ngroups = (nch + C::FOLD - 1) / C::FOLD;
  const int dvalid = d < uint64_t(DC) ? int(d) : DC;
  const float bl2 = beta * 1.4426950408889634f, off = fabsf(beta) * 1.4426950408889634f;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NB; ++i) {
      mbar_init(bfull + i, TG ? 1 : 32);  // TG: expect_tx; else cp.async.mbarrier.arrive.noinc per lane
      mbar_init(bempty + i, 1);
    }
    for (int i = 0; i < C::NSB; ++i) {
      mbar_init(sfull + i, 1);
      mbar_init(sempty + i, 4);
    }
    for (int i = 0; i < C::NP; ++i) mbar_init(pfull + i, 4);
    mbar_init(qfull, 4);
    for (int i = 0; i < C::NF; ++i) {
      mbar_init(accfull + i, 1);
      mbar_init(accempty + i, 4);
    }
    mbar_init_fence();
  }
  if (warp == IW) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const uint32_t s_col = 0, o_col = C::O_COL;  // TMEM: S[NSB] x 64 (PT: P over S), O[NF] x DC

  if (warp < 4) {
    // ------------------------------------------------------------ softmax
    const uint32_t r = warp * 32 + lane;
    const uint64_t grow = p * kPanelRows + r;
    const bool rv = grow < pv.n_rows;
    {  // Q = z[panel rows]: K-major A operand (TF32: RNE; FP32: split2)
      const float* src = zraw + (row_offset + grow) * ld;
      const uint32_t qb = smem_u32(qs);
#pragma unroll
      for (int j = 0; j < DC / 4; ++j) {
        float4 v = (rv && 4 * j < dvalid) ? __ldg(reinterpret_cast<const float4*>(src) + j)
                                          : make_float4(0.f, 0.f, 0.f, 0.f);
        const uint32_t o = kmaj_off(r, 4 * j, kPanelRows);
        if constexpr (C::F32) {
          uint32_t a0, a1, b0, b1, c0_, c1, d0, d1;
          split2(v.x, a0, a1); split2(v.y, b0, b1); split2(v.z, c0_, c1); split2(v.w, d0, d1);
          st_shared_v4(qb + o, a0, b0, c0_, d0);
          st_shared_v4(qb + C::Q_BYTES + o, a1, b1, c1, d1);
        } else {
          st_shared_v4(qb + o, tf32_op(v.x), tf32_op(v.y), tf32_op(v.z), tf32_op(v.w));
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(qfull);
    }
    float l = 0.0f;
    const uint32_t pb = smem_u32(ps);
    // PT: the row masks come straight from global memory, three chunks ahead
    // in registers (no gather-ring mbarrier probe per chunk: each probe costs
    // ~100 cycles on this chain), and the second chunk of an S pair reuses
    // the pair's sfull wait
    constexpr bool MG = C::PT && SGTK_MASK_GLOBAL;
    const uint32_t* dm = pv.dmask + uint64_t(c0) * kPanelRows + r;
    uint32_t mq0 = 0, mq1 = 0, mq2 = 0;
    if constexpr (MG) {
      mq0 = nch > 0 ? __ldg(dm) : 0u;
      mq1 = nch > 1 ? __ldg(dm + kPanelRows) : 0u;
      mq2 = nch > 2 ? __ldg(dm + 2 * kPanelRows) : 0u;
    }
    for (uint32_t c = 0; c < nch; ++c) {
      const uint32_t sgi = c / C::SG;  // S group of the chunk
      const uint32_t sb = sgi % C::NSB, sph = (sgi / C::NSB) & 1u, shalf = (c % C::SG) * 32;
      const uint32_t ds = c % C::NB, dph = (c / C::NB) & 1u;
      const uint32_t pslot = c % C::NP;
      uint32_t mask;
      if constexpr (MG) {
        mask = mq0;
        mq0 = mq1;
        mq1 = mq2;
        mq2 = c + 3 < nch ? __ldg(dm + uint64_t(c + 3) * kPanelRows) : 0u;
      } else {
        mbar_wait(bfull + ds, dph);  // row masks of the chunk
        mask = ld_shared_u32(mr_s + ds * C::M_BYTES + r * 4);
      }
      (void)ds;
      (void)dph;
#ifndef SGTK_TRACE_SM2
      if (warp == 0 && lane == 0) mark(c, 7);
#endif
      if (!MG || (c % C::SG) == 0) mbar_wait(sfull + sb, sph);
#ifdef SGTK_TRACE_SM2  // per-softmax-warp stamps: ev 4 + w = S(c) ready, ev w = P(c) written
      if (lane == 0) mark(c, 4 + warp);
#else
      if (warp == 0 && lane == 0) mark(c, 1);
#endif
      tc_fence_after();
      uint32_t sv[32];
      tmem_ld16(tmem + ((warp * 32u) << 16) + s_col + sb * 64 + shalf, *reinterpret_cast<uint32_t(*)[16]>(sv));
      tmem_ld16(tmem + ((warp * 32u) << 16) + s_col + sb * 64 + shalf + 16,
                *reinterpret_cast<uint32_t(*)[16]>(sv + 16));
      tmem_ld_wait();
#ifndef SGTK_TRACE_SM2
      if (warp == 0 && lane == 0) mark(c, 6);
#endif
      tc_fence_before();
      if constexpr (!C::PT && C::SPLIT_MMA) {  // the group's S read: its TMEM buffer is free
        if ((c % C::SG) == C::SG - 1 || c + 1 == nch) {
          __syncwarp();
          if (lane == 0) mbar_arrive(sempty + sb);
        }
      }
      // Blackwell's paired fp32 instructions (FFMA2 / FADD2) take two elements
      // per issue; same roundings and the same 4 partial sums (j % 4) as the
      // scalar form, so the results are bit-identical to it
      float pr[32];
      float2 lq01 = make_float2(0.0f, 0.0f), lq23 = make_float2(0.0f, 0.0f);
      const float2 bl2v = make_float2(bl2, bl2), offv = make_float2(-off, -off);
#pragma unroll
      for (int j = 0; j < 32; j += 2) {
        const float2 xe = __ffma2_rn(make_float2(__uint_as_float(sv[j]), __uint_as_float(sv[j + 1])), bl2v, offv);
        const float e0 = ex2_approx(xe.x), e1 = ex2_approx(xe.y);
        pr[j] = (mask & (1u << j)) ? e0 : 0.0f;
        pr[j + 1] = (mask & (1u << (j + 1))) ? e1 : 0.0f;
        if constexpr (!C::F32) {  // finite, >= 0
          pr[j] = __uint_as_float(tf32_op(pr[j]));
          pr[j + 1] = __uint_as_float(tf32_op(pr[j + 1]));
        }
        if ((j & 3) == 0) lq01 = __fadd2_rn(lq01, make_float2(pr[j], pr[j + 1]));
        else lq23 = __fadd2_rn(lq23, make_float2(pr[j], pr[j + 1]));
      }
      l += (lq01.x + lq01.y) + (lq23.x + lq23.y);
#ifndef SGTK_TRACE_SM2
      if (warp == 0 && lane == 0) mark(c, 5);
#endif
      if constexpr (C::PT) {  // P over this chunk's S columns (already read)
        tmem_st32(tmem + ((warp * 32u) << 16) + s_col + sb * 64 + shalf, *reinterpret_cast<uint32_t(*)[32]>(pr));
        tmem_st_wait();
        tc_fence_before();
        __syncwarp();
#ifndef SGTK_TRACE_SM2
        if (warp == 0 && lane == 0) mark(c, 2);
#endif
        if (lane == 0) mbar_arrive(pfull + pslot);
#ifdef SGTK_TRACE_SM2
        if (lane == 0) mark(c, warp);
#endif
        continue;
      }
      if (c >= uint32_t(C::NP)) {  // PV(c - NP) done with this P slot
        const uint32_t cp = c - C::NP;
        mbar_wait(bempty + cp % C::NB, (cp / C::NB) & 1u);
      }
      const uint32_t pt = pb + pslot * C::PP * C::P_BYTES;
#pragma unroll
      for (int q = 0; q < 8; ++q) {
        const uint32_t o = kmaj_off(r, 4 * q, kPanelRows);
        if constexpr (C::F32) {
          uint32_t a0, a1, b0, b1, c0_, c1, d0, d1;
          split2(pr[4 * q], a0, a1); split2(pr[4 * q + 1], b0, b1);
          split2(pr[4 * q + 2], c0_, c1); split2(pr[4 * q + 3], d0, d1);
          st_shared_v4(pt + o, a0, b0, c0_, d0);
          st_shared_v4(pt + C::P_BYTES + o, a1, b1, c1, d1);
        } else {
          st_shared_v4(pt + o, __float_as_uint(pr[4 * q]), __float_as_uint(pr[4 * q + 1]),
                       __float_as_uint(pr[4 * q + 2]), __float_as_uint(pr[4 * q + 3]));
        }
      }
      fence_async_smem();
      __syncwarp();
      if (warp == 0 && lane == 0) mark(c, 2);
      if (lane == 0) mbar_arrive(pfull + pslot);
    }
    lbuf[r] = l;
    named_bar(1, 256);  // l handed to the accumulator warps
  } else if (warp < 8) {
    // ------------------------------------------------------------ accumulators
    const uint32_t q = warp & 3u;
    const uint32_t r = q * 32 + lane;
    const uint64_t grow = p * kPanelRows + r;
    float acc[DC];
#pragma unroll
    for (int j = 0; j < DC; ++j) acc[j] = 0.0f;
    for (uint32_t g = 0; g < ngroups; ++g) {
      const uint32_t buf = g % C::NF;
      // (sleeping between probes here measured neutral: the spinning
      // accumulator warps do not hold back the softmax warps)
      mbar_wait(accfull + buf, (g / C::NF) & 1u);
      tc_fence_after();
#pragma unroll
      for (int cc = 0; cc < DC; cc += 16) {
        uint32_t v[16];
        tmem_ld16(tmem + ((q * 32u) << 16) + o_col + buf * DC + cc, v);
        tmem_ld_wait();
#pragma unroll
        for (int j = 0; j < 16; ++j) acc[cc + j] += __uint_as_float(v[j]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(accempty + buf);
    }
    named_bar(1, 256);
    {  // rows staged in shared memory (the gather rings are idle now: every
       // MMA retired), then written back row-contiguously (coalesced)
      constexpr uint32_t TSW = DC + 4;  // staged row stride (floats): spreads banks
      const uint32_t sb = smem_u32(smem + C::Z_OFF) + q * 32u * TSW * 4u;
#pragma unroll
      for (int j = 0; j < DC / 4; ++j)
        st_shared_v4(sb + (lane * TSW + 4 * j) * 4, __float_as_uint(acc[4 * j]), __float_as_uint(acc[4 * j + 1]),
                     __float_as_uint(acc[4 * j + 2]), __float_as_uint(acc[4 * j + 3]));
      __syncwarp();
      constexpr uint32_t LPR = DC / 4, RPI = 32 / LPR;
      const uint64_t row0 = p * kPanelRows + q * 32;
#pragma unroll
      for (uint32_t t = 0; t < 32 / RPI; ++t) {
        const uint32_t rr = t * RPI + lane / LPR, cc = lane % LPR;
        if (row0 + rr < pv.n_rows)
          reinterpret_cast<float4*>(opart + (row0 + rr) * DC)[cc] = ld_shared_f4(sb + (rr * TSW + 4 * cc) * 4);
      }
      if (grow < pv.n_rows) lpart[grow] = lbuf[r];
    }
  } else if (warp == IW || warp == IW + 1) {
    // ------------------------------------------------------------ MMA issuers
    if (lane == 0 && nch && (warp == IW || C::SPLIT_MMA)) {
      constexpr uint32_t id_s = idesc_tf32(32 * C::SG, false);  // N = a S group's columns, B K-major
      constexpr uint32_t id_o = idesc_tf32(DC, true);   // N = DC features, B MN-major
      const uint32_t qb = smem_u32(qs), pb = smem_u32(ps);
      mbar_wait(qfull, 0);
      tc_fence_after();
      // S of chunk pair g (chunks 2g, 2g+1) as one N = 64 MMA chain: the z
      // tiles of ring slots 2k and 2k+1 are adjacent rows of one K-major tile
      auto issue_s = [&](uint32_t g) {
        const uint32_t c = C::SG * g;
        if (C::PT && g >= uint32_t(C::NSB)) {  // PV of the buffer's previous group read its P
          const uint32_t cl = C::SG * (g - C::NSB) + C::SG - 1;
          mbar_wait(bempty + cl % C::NB, (cl / C::NB) & 1u);
        }
        if (!C::PT && C::SPLIT_MMA && g >= uint32_t(C::NSB))  // the softmax read the buffer's previous S
          mbar_wait(sempty + g % C::NSB, ((g / C::NSB) - 1u) & 1u);
        mbar_wait(bfull + c % C::NB, (c / C::NB) & 1u);
        if (C::PAIR && c + 1 < nch) mbar_wait(bfull + (c + 1) % C::NB, ((c + 1) / C::NB) & 1u);
        fence_async_smem();  // cp.async (generic proxy) -> MMA (async proxy)
        tc_fence_after();
        const uint32_t s0 = c % C::NB;
        const uint32_t dt = tmem + s_col + (g % C::NSB) * 64;
#pragma unroll
        for (uint32_t ks = 0; ks < DC / 8; ++ks) {
          const uint32_t ko = (ks >> 2) * 16384u + (ks & 3u) * 32u;  // Q: 128-row K blocks
          const uint32_t kz = ((ks >> 2) * C::NB + s0) * 4096u + (ks & 3u) * 32u;
          const uint64_t q0 = umma_desc(qb + ko), z0 = umma_desc(zr_s + kz);
          if constexpr (C::F32) {
            umma_tf32(dt, q0, umma_desc(zr_s + C::KB * C::NB * 4096u + kz), id_s, ks ? 1u : 0u);
            umma_tf32(dt, umma_desc(qb + C::Q_BYTES + ko), z0, id_s, 1u);
            umma_tf32(dt, q0, z0, id_s, 1u);
          } else {
            umma_tf32(dt, q0, z0, id_s, ks ? 1u : 0u);
          }
        }
        umma_commit(sfull + g % C::NSB);
#ifndef SGTK_TRACE_SM2
        mark(c, 0);
#endif
      };
      auto issue_pv = [&](uint32_t c) {
        const uint32_t ds = c % C::NB, pslot = c % C::NP;
        const uint32_t g = c / C::FOLD, buf = g % C::NF;
        const bool first = (c % C::FOLD) == 0;
        if (first && g >= uint32_t(C::NF)) mbar_wait(accempty + buf, ((g / C::NF) - 1u) & 1u);
        mbar_wait(pfull + pslot, (c / C::NP) & 1u);
        if constexpr (C::SPLIT_MMA) {  // the h tile: landed (long ago), visible to the async proxy
          mbar_wait(bfull + ds, (c / C::NB) & 1u);
          fence_async_smem();
        }
        tc_fence_after();
        const uint32_t pt = pb + pslot * C::PP * C::P_BYTES;
        const uint32_t ht = hr_s + ds * C::T_BYTES;
        const uint32_t dt = tmem + o_col + buf * DC;
#pragma unroll
        for (uint32_t ks = 0; ks < kChunkCols / 8; ++ks) {
          const uint32_t acc = (first && ks == 0) ? 0u : 1u;
          const uint64_t p0 = umma_desc(pt + ks * 32), h0 = desc_mn32(ht + ks * 1024, 4096, 512);
          if constexpr (C::PT) {
            umma_tf32_ts(dt, tmem + s_col + ((c / C::SG) % C::NSB) * 64 + (c % C::SG) * 32 + ks * 8, h0, id_o, acc);
          } else if constexpr (C::F32) {
            umma_tf32(dt, p0, desc_mn32(ht + C::NB * C::T_BYTES + ks * 1024, 4096, 512), id_o, acc);
            umma_tf32(dt, umma_desc(pt + C::P_BYTES + ks * 32), h0, id_o, 1u);
            umma_tf32(dt, p0, h0, id_o, 1u);
          } else {
            umma_tf32(dt, p0, h0, id_o, acc);
          }
        }
#ifndef SGTK_TRACE_SM2
        mark(c, 3);
#endif
        umma_commit(bempty + ds);  // gather slot and P slot free
        if ((c % C::FOLD) == C::FOLD - 1 || c + 1 == nch) umma_commit(accfull + buf);
      };
      if constexpr (C::SPLIT_MMA) {
        if (warp == IW) {
          for (uint32_t g = 0; g * C::SG < nch; ++g) issue_s(g);
        } else {
          for (uint32_t c = 0; c < nch; ++c) issue_pv(c);
        }
      } else {
        issue_s(0);
        for (uint32_t c = 0; c < nch; ++c) {
          // S of the next group.  Its S buffer held group g - 1, whose last P
          // was waited for at the previous iteration.  With a deep gather ring
          // (EARLY_S) it goes at the group's first chunk -- the softmax then has
          // a whole group of slack -- since its gathers only need PV(c + 2 - NB)
          // retired; shallow rings issue it at the group's last chunk.
          if constexpr (C::EARLY_S) {
            if ((c % C::SG) == 0 && c + C::SG < nch) issue_s(c / C::SG + 1);
          } else {
            if ((c % C::SG) == C::SG - 1 && c + 1 < nch) issue_s(c / C::SG + 1);
          }
          issue_pv(c);
        }
      }
    }
  } else {
    // ------------------------------------------------------------ loaders (warps 8 .. IW - 1)
    // warp 9 takes even chunks, warp 10 odd ones.  Per chunk: 32 z rows
    // (K-major SWIZZLE_128B B of S), 32 h rows (MN-major SWIZZLE_128B_BASE32B
    // B of PV), 128 row masks; completion via cp.async.mbarrier.arrive.noinc.
    const uint32_t par = warp - 8;
    // column ids one chunk ahead: the global load stays off the slot-free ->
    // gather-issue path
    uint32_t coln = par < nch ? pv.dcols[uint64_t(c0 + par) * kChunkCols + lane] : 0u;
    for (uint32_t c = par; c < nch; c += NL) {
      const uint32_t ds = c % C::NB;
#ifdef SGTK_AGNN_GMASK  // timing experiment only: gather a small hot set of rows
      const uint32_t col = coln == 0xFFFFFFFFu ? coln : (coln & SGTK_AGNN_GMASK);
#else
      const uint32_t col = coln;
#endif
      coln = c + NL < nch ? pv.dcols[uint64_t(c0 + c + NL) * kChunkCols + lane] : 0u;
      mbar_wait(bempty + ds, ((c / C::NB) & 1u) ^ 1u);
#ifndef SGTK_TRACE_SM2
      if (lane == 0) mark(c, 4);
#endif
      const uint32_t ht = hr_s + ds * C::T_BYTES;
      if constexpr (TG) {
        // lane g < 8 gathers chunk rows 4g..4g+3: z (K-major SWIZZLE_128B, one
        // 4 KB tile per 32-feature K block) and h (MN-major 128B_BASE32B, one
        // 4 KB block per 32 features); padding ids ~0u = row -1: zero-filled
        const int r0 = int(__shfl_sync(0xFFFFFFFFu, col, (4 * lane) & 31));
        const int r1 = int(__shfl_sync(0xFFFFFFFFu, col, (4 * lane + 1) & 31));
        const int r2 = int(__shfl_sync(0xFFFFFFFFu, col, (4 * lane + 2) & 31));
        const int r3 = int(__shfl_sync(0xFFFFFFFFu, col, (4 * lane + 3) & 31));
        if (lane < 8) {
#pragma unroll
          for (int kb = 0; kb < C::KB; ++kb) {
            tma_gather4(zr_s + (kb * C::NB + ds) * 4096u + lane * 512u, &tmz, 32 * kb, r0, r1, r2, r3, bfull + ds);
            tma_gather4(ht + kb * 4096u + lane * 512u, &tmh, 32 * kb, r0, r1, r2, r3, bfull + ds);
          }
        } else if (lane == 8) {
          bulk_load(smem + C::M_OFF + ds * C::M_BYTES, pv.dmask + uint64_t(c0 + c) * kPanelRows, C::M_BYTES,
                    bfull + ds);
          mbar_expect_tx(bfull + ds, 2u * C::KB * 32u * 128u + C::M_BYTES);
        }
        continue;
      }
      constexpr uint32_t LPR = DC / 4, RPI = 32 / LPR;
      const uint32_t j = lane % LPR, jj = j & 7u;
#pragma unroll
      for (uint32_t t = 0; t < 32 / RPI; ++t) {
        const uint32_t k = t * RPI + lane / LPR;  // chunk row (B row / K row)
        const uint32_t ck = __shfl_sync(0xFFFFFFFFu, col, k);
        // operand rows are ldq wide with zero padding features in memory, so
        // only padding chunk columns take the zero source (distinct pieces)
        const bool real = ck != 0xFFFFFFFFu;
        const uint64_t gofs = uint64_t(ck) * ld + 4 * j;
        // z: K-major SWIZZLE_128B, row k, 16-byte piece j; K block j>>3 of slot ds
        const uint32_t zo = ((j >> 3) * C::NB + ds) * 4096u + (k >> 3) * 1024u + (k & 7u) * 128u +
                            ((jj ^ (k & 7u)) << 4);
        // h: MN-major SWIZZLE_128B_BASE32B (tc05.cuh desc_mn32)
        const uint32_t ho = (j >> 3) * 4096u + (k >> 2) * 512u + (k & 3u) * 128u +
                            ((((jj >> 1) ^ (k & 3u)) << 5) | ((jj & 1u) << 4));
        cp_async16(zr_s + zo, real ? z + gofs : g_agnn_zero + (k * LPR + j) * 4);
        cp_async16(ht + ho, real ? h + gofs : g_agnn_zero + (k * LPR + j) * 4);
        if constexpr (C::F32) {  // lo planes (pre-split once per layer)
          cp_async16(zr_s + C::KB * C::NB * 4096u + zo, real ? z1 + gofs : g_agnn_zero + (k * LPR + j) * 4);
          cp_async16(ht + C::NB * C::T_BYTES + ho, real ? h1 + gofs : g_agnn_zero + (k * LPR + j) * 4);
        }
      }
#ifndef SGTK_MASK_COPY
#define SGTK_MASK_COPY 1
#endif
      // (PT: the softmax reads its masks from global memory three chunks
      // ahead; this copy, issued ~10 chunks ahead, is what brings them into
      // L2 in time -- without it the dense part measured 0.270 -> 0.287 ms)
      if (SGTK_MASK_COPY || !(C::PT && SGTK_MASK_GLOBAL))
        cp_async16(mr_s + ds * C::M_BYTES + lane * 16, pv.dmask + (uint64_t(c0 + c) * kPanelRows) + lane * 4);
      cp_async_arrive_noinc(bfull + ds);
    }
    if constexpr (!TG) cp_async_wait<0>();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == IW) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
  if constexpr (FR) {
    // the panel's (O, l) partials are in opart / lpart (written by the
    // accumulator warps before the barrier); every MMA retired and the
    // loaders drained, so the gather rings hold the row tiles
    float* T = reinterpret_cast<float*>(smem + C::Z_OFF) + warp * 33 * (DC + 4);
    unsigned long long nz = 0;
    if (warp < FRW)
    for (uint32_t it = pv.paitem[p] + warp; it < pv.paitem[p + 1]; it += FRW)
      agnn_row_item<1, PREC, false>(items[it], T, lane, sent, zraw, h, ld, nullptr, d, row_offset, bl2, off, opart,
                                    lpart, seg_o, seg_l, nullptr, nullptr, nx, nz);
    if (nx.zeros && lane == 0 && nz) atomicAdd(nx.zeros, nz);
  }
}

// ---------------------------------------------------------------------------
// Sparse edges + finalisation.  One warp per item: a row (all rows are items:
// every row needs out = O / l), or a <= kSegEdges segment of a hub row whose
// (O, l) partial is combined in order by agnn_long_rows_kernel.
//   logits: lane = edge, dot(z_row, z_col) over the features (z_row held in
//           registers, z_col rows read whole: 128/256-byte lines);
//   update: lane = feature, 8 edges' h rows in flight (coalesced).
// Finalise: out = O / l (l = 0: no edges -> 0, as spmm of an empty row);
// then the next layer's l2 norm (double sum, gnn.cpp:74-91), z_next and the
// TF32 / split operand copies for the next dense pass.
// ---------------------------------------------------------------------------

template <int FPL, int PREC>
__device__ __forceinline__ void agnn_finalize(uint64_t r, const float (&o)[FPL], float l, uint32_t lane,
                                              int fv, const AgnnNext& nx, unsigned long long& nz) {
  float v[FPL];
  // l == 0 only for a row without edges (every exp term is > 0); a NaN l
  // (non-finite input) must propagate like the reference's softmax does
  const float inv_l = l != 0.0f ? 1.0f / l : 0.0f;
  bool bad = false;
#pragma unroll
  for (int i = 0; i < FPL; ++i) {
    v[i] = l != 0.0f ? o[i] * inv_l : 0.0f;
    bad |= i < fv && !isfinite(v[i]);
  }
  if (nx.nonfinite && __any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(nx.nonfinite, 1u);
  const uint64_t f = uint64_t(lane) * FPL;
  if (nx.out) {
#pragma unroll
    for (int i = 0; i < FPL; ++i)
      if (i < fv) nx.out[r * nx.ldo + f + i] = v[i];
  }
  if (!nx.zq) return;
  // The next layer's norm in exactly agnn_input_kernel's order (so a multi-
  // layer call and per-layer calls — the row-partitioned path — agree bit for
  // bit): groups of 4 features summed in sequence, then a butterfly over the
  // groups (offsets 1, 2, 4[, 8] groups = G, 2G, 4G[, 8G] lanes).
  constexpr uint32_t G = 4 / FPL;  // lanes per 4-feature group
  double q[FPL];
#pragma unroll
  for (int i = 0; i < FPL; ++i) q[i] = i < fv ? double(v[i]) * double(v[i]) : 0.0;
  const uint32_t g0 = lane & ~(G - 1);
  double sq = 0.0;
#pragma unroll
  for (uint32_t k = 0; k < G; ++k)
#pragma unroll
    for (int i = 0; i < FPL; ++i) sq += __shfl_sync(0xFFFFFFFFu, q[i], g0 + k);
#pragma unroll
  for (uint32_t o2 = G; o2 < 32; o2 <<= 1) sq += __shfl_xor_sync(0xFFFFFFFFu, sq, o2);
  const float inv = sq == 0.0 ? 0.0f : float(1.0 / sqrt(sq));
  if (sq == 0.0 && lane == 0) ++nz;
  if (lane == 0 && nx.norm) nx.norm[r] = inv > 0.0f ? 1.0f / inv : 0.0f;  // |h| = 1 / inv
#pragma unroll
  for (int i = 0; i < FPL; ++i) {
    const float zz = i < fv ? v[i] * inv : 0.0f, hh = i < fv ? v[i] : 0.0f;
    if (i < fv && nx.z) nx.z[r * nx.ldq + f + i] = zz;
    if constexpr (PREC == SGTK_FP32) {
      uint32_t a0, a1, b0, b1;
      split2(zz, a0, a1);
      split2(hh, b0, b1);
      nx.zq[r * nx.ldq + f + i] = __uint_as_float(a0);
      nx.zq1[r * nx.ldq + f + i] = __uint_as_float(a1);
      nx.hq[r * nx.ldq + f + i] = __uint_as_float(b0);
      nx.hq1[r * nx.ldq + f + i] = __uint_as_float(b1);
    } else {
      nx.zq[r * nx.ldq + f + i] = tf32_rne(zz);
      nx.hq[r * nx.ldq + f + i] = tf32_rne(hh);
    }
  }
}

// Sparse edges of a row, batches of 32:
//   the batch's z_col rows (128/256 B each) go to a per-warp smem tile T by
//     cp.async (TF32 mode reads the pre-rounded copy zq, so T is already the
//     MMA-rounded operand);
//   lane = edge: dot of T[e] with z_row (tile row 32, a broadcast read),
//     p = exp2(beta*log2e*s - |beta|*log2e), coefficient p * |h_col| in a
//     register (h_col = z_col * |h_col|: z is h scaled to unit norm,
//     gnn.cpp:74-91, so the aggregation needs no second gather);
//   lane = feature: O[f] += coef_e * T[e][f] over the batch, e ascending,
//     coef_e broadcast by shuffle.
// Row sums l: per-lane partials, reduced by a fixed shuffle tree per item.
#ifndef SGTK_ROWS_MINB
#define SGTK_ROWS_MINB 5
#endif
// One AGNN item (a row's sparse edges, or a hub-row segment) by one warp
// over its smem tile T (33 rows x (DC + 4) floats): see agnn_rows_kernel.
template <int FPL, int PREC, bool SPLIT>
__device__ __forceinline__ void agnn_row_item(const uint4 w, float* T, uint32_t lane, const uint2* __restrict__ sent,
                                              const float* __restrict__ zown, const float* __restrict__ z,
                                              uint64_t ld, const float* __restrict__ norm, uint64_t d,
                                              uint64_t row_offset, float bl2, float off,
                                              const float* __restrict__ opart, const float* __restrict__ lpart,
                                              float* __restrict__ seg_o, float* __restrict__ seg_l,
                                              float* __restrict__ osp, float* __restrict__ lsp, const AgnnNext& nx,
                                              unsigned long long& nz) {
  constexpr int DC = 32 * FPL;
  constexpr int TS = DC + 4;
  const uint32_t tb = smem_u32(T);
  const uint64_t f = uint64_t(lane) * FPL;
  const int fv = f >= d ? 0 : (d - f >= uint64_t(FPL) ? FPL : int(d - f));
  const uint64_t r = w.x;
  const bool direct = w.w == 0xFFFFFFFFu;
  const uint32_t c_first = w.y < w.z && lane < min(32u, w.z - w.y) ? sent[w.y + lane].x : 0u;
  // z of the row -> tile row 32 (read back as a broadcast by every lane;
  // lands with the first batch's gathers); padding features are zeros
  if (w.y < w.z && lane < uint32_t(DC / 4))
    cp_async16(tb + (32 * TS + 4 * lane) * 4, zown + (row_offset + r) * ld + 4 * lane);
  float o[FPL], lpp = 0.0f;
#pragma unroll
  for (int i = 0; i < FPL; ++i) o[i] = (!SPLIT && direct && i < fv) ? opart[r * DC + f + i] : 0.0f;
  const float l0 = (!SPLIT && direct) ? lpart[r] : 0.0f;
  uint32_t col = c_first;
  for (uint32_t e = w.y; e < w.z; e += 32) {
    const uint32_t cnt = min(32u, w.z - e);
    const uint32_t col_next = e + 32 < w.z && lane < min(32u, w.z - e - 32) ? sent[e + 32 + lane].x : 0u;
    {  // cooperative, coalesced gather of the batch's z rows into the tile
      constexpr uint32_t LPR = DC / 4, RPI = 32 / LPR;
      const uint32_t j = lane % LPR;
#pragma unroll
      for (uint32_t t = 0; t < 32 / RPI; ++t) {
        const uint32_t u = t * RPI + lane / LPR;
        const uint32_t cu = __shfl_sync(0xFFFFFFFFu, col, u);
        if (u < cnt) cp_async16(tb + (u * TS + 4 * j) * 4, z + uint64_t(cu) * ld + 4 * j);
      }
      cp_async_commit();
      cp_async_wait<0>();
      __syncwarp();
    }
    float cf_l = 0.0f;
    if (lane < cnt) {
      // dot and |h|^2 as two interleaved partial sums each on the paired
      // FFMA2 (even / odd features), combined at the end: half the issues
      // (TF32; FP32 keeps the scalar chain, measured faster there)
      float s = 0.0f, n2 = 0.0f;
      if constexpr (PREC == SGTK_TF32) {
        float2 s2 = make_float2(0.0f, 0.0f), n22 = make_float2(0.0f, 0.0f);
#pragma unroll
        for (int k = 0; k < DC / 4; ++k) {
          const float4 v = ld_shared_f4(tb + (lane * TS + 4 * k) * 4);
          const float4 q = ld_shared_f4(tb + (32 * TS + 4 * k) * 4);
          const float2 vlo = make_float2(v.x, v.y), vhi = make_float2(v.z, v.w);
          s2 = __ffma2_rn(make_float2(q.x, q.y), vlo, s2);
          s2 = __ffma2_rn(make_float2(q.z, q.w), vhi, s2);
          n22 = __ffma2_rn(vlo, vlo, n22);
          n22 = __ffma2_rn(vhi, vhi, n22);
        }
        s = s2.x + s2.y;
        n2 = n22.x + n22.y;
      } else {
#pragma unroll
        for (int k = 0; k < DC / 4; ++k) {
          const float4 v = ld_shared_f4(tb + (lane * TS + 4 * k) * 4);
          const float4 q = ld_shared_f4(tb + (32 * TS + 4 * k) * 4);
          s = fmaf(q.x, v.x, s);
          s = fmaf(q.y, v.y, s);
          s = fmaf(q.z, v.z, s);
          s = fmaf(q.w, v.w, s);
        }
      }
      if constexpr (PREC == SGTK_TF32) {
        // T holds hq_col = tf32(h_col): z_col = h_col / |h_col| on the fly
        // (no norm gather); sddmm TF32 rounds the dot (tile_exec.cpp:386)
        s = tf32_rne(n2 > 0.0f ? s * rsqrtf(n2) : 0.0f);
      }
      float pe = ex2_approx(fmaf(s, bl2, -off));
      if constexpr (PREC == SGTK_TF32) {
        pe = __uint_as_float(tf32_op(pe));
        cf_l = pe;
      } else {
        cf_l = pe * __ldg(norm + col);
      }
      lpp += pe;
    }
#pragma unroll 8
    for (uint32_t u = 0; u < cnt; ++u) {
      const float cf = __shfl_sync(0xFFFFFFFFu, cf_l, u);
#pragma unroll
      for (int i = 0; i < FPL; ++i) o[i] = fmaf(cf, T[u * TS + lane * FPL + i], o[i]);
    }
    __syncwarp();
    col = col_next;
  }
#pragma unroll
  for (int o2 = 16; o2 > 0; o2 >>= 1) lpp += __shfl_xor_sync(0xFFFFFFFFu, lpp, o2);
  const float l = l0 + lpp;
  if (direct && SPLIT) {  // sparse partial; agnn_final_kernel combines
#pragma unroll
    for (int i = 0; i < FPL; ++i)
      if (i < fv) osp[r * DC + f + i] = o[i];
    if (lane == 0) lsp[r] = l;
  } else if (direct) {
    agnn_finalize<FPL, PREC>(r, o, l, lane, fv, nx, nz);
  } else {
#pragma unroll
    for (int i = 0; i < FPL; ++i)
      if (i < fv) seg_o[uint64_t(w.w) * DC + f + i] = o[i];
    if (lane == 0) seg_l[w.w] = l;
  }
}

#ifndef SGTK_ROWS_WARPS
#define SGTK_ROWS_WARPS 2
#endif
// rows kernel block: SGTK_ROWS_WARPS warps (d = 32), half as many at d = 64
constexpr int kRowsWarps1 = SGTK_ROWS_WARPS, kRowsWarps2 = SGTK_ROWS_WARPS > 1 ? SGTK_ROWS_WARPS / 2 : 1;
template <int FPL, int PREC, bool SPLIT>
__global__ void __launch_bounds__(FPL == 1 ? 32 * kRowsWarps1 : 32 * kRowsWarps2,
                                  std::min(32, (FPL == 1 ? SGTK_ROWS_MINB : 2 * SGTK_ROWS_MINB) * 8 / SGTK_ROWS_WARPS))
agnn_rows_kernel(const uint4* __restrict__ items, uint64_t n_items, const uint2* __restrict__ sent,
                 const float* __restrict__ zown, const float* __restrict__ z, uint64_t ld,
                 const float* __restrict__ norm,
                 uint64_t d, uint64_t row_offset, float beta, const float* __restrict__ opart,
                 const float* __restrict__ lpart, float* __restrict__ seg_o,
                 float* __restrict__ seg_l, float* __restrict__ osp, float* __restrict__ lsp,
                 AgnnNext nx) {
  constexpr int DC = 32 * FPL;
  constexpr int TS = DC + 4;  // smem tile row stride (floats): 16-byte rows, spread banks
  __shared__ __align__(16) float tile[FPL == 1 ? kRowsWarps1 : kRowsWarps2][33 * TS];  // 32 z_col rows + z_row
  const uint32_t lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  float* T = tile[wib];
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const float bl2 = beta * 1.4426950408889634f, off = fabsf(beta) * 1.4426950408889634f;
  unsigned long long nz = 0;
  for (uint64_t it = warp; it < n_items; it += nw)
    agnn_row_item<FPL, PREC, SPLIT>(items[it], T, lane, sent, zown, z, ld, norm, d, row_offset, bl2, off, opart,
                                    lpart, seg_o, seg_l, osp, lsp, nx, nz);
  if (nx.zeros && lane == 0 && nz) atomicAdd(nx.zeros, nz);
}

// Concurrent mode: (dense + sparse) partials of the non-hub rows, finalised.
// Streaming: LPR = DC/4 lanes per row (float4 each), 32/LPR rows per warp
// instruction; the row's l2 norm reduces over its lanes in double by a fixed
// xor tree.  Same results as agnn_finalize up to the order of that sum.
template <int FPL, int PREC>
__global__ void agnn_final_kernel(const uint4* __restrict__ items, uint64_t n_items, uint64_t d,
                                  const float* __restrict__ opart, const float* __restrict__ lpart,
                                  const float* __restrict__ osp, const float* __restrict__ lsp,
                                  AgnnNext nx) {
  constexpr uint32_t DC = 32 * FPL, LPR = DC / 4, RPW = 32 / LPR;
  const uint32_t lane = threadIdx.x & 31, sub = lane / LPR, j = lane % LPR;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint64_t f = 4u * j;
  const int fv = f >= d ? 0 : (d - f >= 4 ? 4 : int(d - f));
  unsigned long long nz = 0;
  for (uint64_t base = warp * RPW; base < n_items; base += nw * RPW) {
    const uint64_t it = base + sub;
    const uint4 w = it < n_items ? items[it] : make_uint4(0, 0, 0, 0);
    const bool ok = it < n_items && w.w == 0xFFFFFFFFu;  // hub segments: agnn_long_rows_kernel
    const uint64_t r = w.x;
    float v[4] = {0.f, 0.f, 0.f, 0.f};
    float l = 0.0f;
    if (ok) {
      // padding features [d, DC) of the partials are never written: skip them
      const float4 z4 = make_float4(0.f, 0.f, 0.f, 0.f);
      const float4 a = fv ? *reinterpret_cast<const float4*>(opart + r * DC + f) : z4;
      const float4 b = fv ? *reinterpret_cast<const float4*>(osp + r * DC + f) : z4;
      l = lpart[r] + lsp[r];
      const float inv_l = l != 0.0f ? 1.0f / l : 0.0f;  // NaN propagates (agnn_finalize)
      const float o[4] = {a.x + b.x, a.y + b.y, a.z + b.z, a.w + b.w};
#pragma unroll
      for (int i = 0; i < 4; ++i) v[i] = (l != 0.0f && i < fv) ? o[i] * inv_l : 0.0f;
      if (nx.out) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (i < fv) nx.out[r * nx.ldo + f + i] = v[i];
      }
    }
    if (nx.nonfinite) {
      bool bad = false;
#pragma unroll
      for (int i = 0; i < 4; ++i) bad |= !isfinite(v[i]);
      if (__any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(nx.nonfinite, 1u);
    }
    if (!nx.zq) continue;  // last layer
    double sq = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) sq += double(v[i]) * double(v[i]);
#pragma unroll
    for (uint32_t o2 = 1; o2 < LPR; o2 <<= 1) sq += __shfl_xor_sync(0xFFFFFFFFu, sq, o2);
    if (!ok) continue;
    const float inv = sq == 0.0 ? 0.0f : float(1.0 / sqrt(sq));
    if (sq == 0.0 && j == 0) ++nz;
    if (j == 0 && nx.norm) nx.norm[r] = inv > 0.0f ? 1.0f / inv : 0.0f;  // as agnn_input_kernel
    float zz[4], hh[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      zz[i] = v[i] * inv;  // padding features stay 0
      hh[i] = v[i];
    }
    const uint64_t q = r * nx.ldq + f;
    if (nx.z) *reinterpret_cast<float4*>(nx.z + q) = make_float4(zz[0], zz[1], zz[2], zz[3]);
    if constexpr (PREC == SGTK_FP32) {
      uint32_t a0[4], a1[4], b0[4], b1[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        split2(zz[i], a0[i], a1[i]);
        split2(hh[i], b0[i], b1[i]);
      }
      *reinterpret_cast<uint4*>(nx.zq + q) = make_uint4(a0[0], a0[1], a0[2], a0[3]);
      *reinterpret_cast<uint4*>(nx.zq1 + q) = make_uint4(a1[0], a1[1], a1[2], a1[3]);
      *reinterpret_cast<uint4*>(nx.hq + q) = make_uint4(b0[0], b0[1], b0[2], b0[3]);
      *reinterpret_cast<uint4*>(nx.hq1 + q) = make_uint4(b1[0], b1[1], b1[2], b1[3]);
    } else {
      *reinterpret_cast<float4*>(nx.zq + q) =
          make_float4(tf32_rne(zz[0]), tf32_rne(zz[1]), tf32_rne(zz[2]), tf32_rne(zz[3]));
      *reinterpret_cast<float4*>(nx.hq + q) =
          make_float4(tf32_rne(hh[0]), tf32_rne(hh[1]), tf32_rne(hh[2]), tf32_rne(hh[3]));
    }
  }
  if (nx.zeros && nz) atomicAdd(nx.zeros, nz);
}

// Hub rows: (O, l) = dense partial + segment partials in segment order, then
// the same finalisation.  One warp per hub row.
template <int FPL, int PREC>
__global__ void agnn_long_rows_kernel(const uint4* __restrict__ lrows, uint64_t n_long, uint64_t d,
                                      const float* __restrict__ opart, const float* __restrict__ lpart,
                                      const float* __restrict__ seg_o, const float* __restrict__ seg_l,
                                      AgnnNext nx) {
  constexpr int DC = 32 * FPL;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint64_t f = uint64_t(lane) * FPL;
  const int fv = f >= d ? 0 : (d - f >= uint64_t(FPL) ? FPL : int(d - f));
  unsigned long long nz = 0;
  for (uint64_t i = warp; i < n_long; i += nw) {
    const uint4 w = lrows[i];
    const uint64_t r = w.x;
    float o[FPL];
#pragma unroll
    for (int k = 0; k < FPL; ++k) o[k] = k < fv ? opart[r * DC + f + k] : 0.0f;
    float l = lpart[r];
    for (uint32_t sgi = 0; sgi < w.z; ++sgi) {
#pragma unroll
      for (int k = 0; k < FPL; ++k)
        if (k < fv) o[k] += seg_o[uint64_t(w.y + sgi) * DC + f + k];
      l += seg_l[w.y + sgi];
    }
    agnn_finalize<FPL, PREC>(r, o, l, lane, fv, nx, nz);
  }
  if (nx.zeros && lane == 0 && nz) atomicAdd(nx.zeros, nz);
}

// operand copies of the first layer's input: TF32 -> rounded (z, h);
// FP32 -> hi / lo planes of z and h
// Layer-0 operands in one pass over x: the row's l2 norm (double, fixed xor
// tree over its LPR = DC/4 lanes), z = x / |x| and the MMA operand copies
// (TF32: rounded z and h; FP32: raw z, hi/lo planes, |h|); counts zero rows.
template <int FPL, int PREC>
__global__ void agnn_input_kernel(const float* __restrict__ x, uint64_t ldx, uint64_t rows, uint64_t d,
                                  uint64_t ldq, float* __restrict__ z, float* __restrict__ zq,
                                  float* __restrict__ zq1, float* __restrict__ hq, float* __restrict__ hq1,
                                  float* __restrict__ norm, unsigned long long* __restrict__ zeros) {
  constexpr uint32_t DC = 32 * FPL, LPR = DC / 4, RPW = 32 / LPR;
  const uint32_t lane = threadIdx.x & 31, sub = lane / LPR, j = lane % LPR;
  const uint64_t warp = (uint64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const uint64_t nw = (uint64_t(gridDim.x) * blockDim.x) >> 5;
  const uint64_t f = 4u * j;
  const int fv = f >= d ? 0 : (d - f >= 4 ? 4 : int(d - f));
  unsigned long long nz = 0;
  for (uint64_t base = warp * RPW; base < rows; base += nw * RPW) {
    const uint64_t r = base + sub;
    const bool ok = r < rows;
    float v[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) v[i] = ok && i < fv ? x[r * ldx + f + i] : 0.0f;
    double sq = 0.0;
#pragma unroll
    for (int i = 0; i < 4; ++i) sq += double(v[i]) * double(v[i]);
#pragma unroll
    for (uint32_t o2 = 1; o2 < LPR; o2 <<= 1) sq += __shfl_xor_sync(0xFFFFFFFFu, sq, o2);
    if (!ok) continue;
    const float inv = sq == 0.0 ? 0.0f : float(1.0 / sqrt(sq));
    if (sq == 0.0 && j == 0) ++nz;
    float zz[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) zz[i] = v[i] * inv;
    const uint64_t q = r * ldq + f;
    if constexpr (PREC == SGTK_FP32) {
      if (j == 0) norm[r] = inv > 0.0f ? 1.0f / inv : 0.0f;  // |h| = 1 / inv
      *reinterpret_cast<float4*>(z + q) = make_float4(zz[0], zz[1], zz[2], zz[3]);
      uint32_t a0[4], a1[4], b0[4], b1[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        split2(zz[i], a0[i], a1[i]);
        split2(v[i], b0[i], b1[i]);
      }
      *reinterpret_cast<uint4*>(zq + q) = make_uint4(a0[0], a0[1], a0[2], a0[3]);
      *reinterpret_cast<uint4*>(zq1 + q) = make_uint4(a1[0], a1[1], a1[2], a1[3]);
      *reinterpret_cast<uint4*>(hq + q) = make_uint4(b0[0], b0[1], b0[2], b0[3]);
      *reinterpret_cast<uint4*>(hq1 + q) = make_uint4(b1[0], b1[1], b1[2], b1[3]);
    } else {
      *reinterpret_cast<float4*>(zq + q) =
          make_float4(tf32_rne(zz[0]), tf32_rne(zz[1]), tf32_rne(zz[2]), tf32_rne(zz[3]));
      *reinterpret_cast<float4*>(hq + q) =
          make_float4(tf32_rne(v[0]), tf32_rne(v[1]), tf32_rne(v[2]), tf32_rne(v[3]));
    }
  }
  if (zeros && nz) atomicAdd(zeros, nz);
}

#ifndef SGTK_ROWS_GRID
#define SGTK_ROWS_GRID 32
#endif
// rows kernel grid: warps loop over items; at most SGTK_ROWS_GRID blocks per
// SM (measured: 16 -> 32 is -1.5%, 64+ and 10- slower)
inline unsigned rows_grid(uint64_t items, unsigned bs) {
  const uint64_t b = (items * 32 + bs - 1) / bs;
  return unsigned(std::max<uint64_t>(1, std::min<uint64_t>(b, 148ull * SGTK_ROWS_GRID * 256 / bs)));
}
#ifndef SGTK_FINAL_GRID
#define SGTK_FINAL_GRID 16
#endif
inline unsigned final_grid(uint64_t items) {  // 4 rows per warp instruction
  const uint64_t b = (items * 8 + 255) / 256;
  return unsigned(std::max<uint64_t>(1, std::min<uint64_t>(b, 148ull * SGTK_FINAL_GRID)));
}
inline unsigned blocks_for(uint64_t n, unsigned bs = 256) {
  return unsigned(std::max<uint64_t>(1, std::min<uint64_t>((n + bs - 1) / bs, 148ull * 16)));
}

PFN_cuTensorMapEncodeTiled_v12000 agnn_encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}
// Row-gather map over an operand table (rows x ld fp32): box {32 features, 1
// row}, swizzled for the UMMA layout the tile is read with.
bool make_gather_map(CUtensorMap* m, const float* base, uint64_t rows, uint64_t ld, CUtensorMapSwizzle sw) {
  auto fn = agnn_encode_fn();
  if (!fn || (reinterpret_cast<uintptr_t>(base) & 15u) || (ld * 4) % 16 || rows == 0 || rows > 0x7FFFFFFFull)
    return false;
  const cuuint64_t dims[2] = {ld, rows};
  const cuuint64_t strides[1] = {ld * 4};
  const cuuint32_t box[2] = {32, 1};
  const cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, const_cast<float*>(base), dims, strides, box, es,
            CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_NONE,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int DC, int PREC>
void launch_agnn_dense(const PanelView& v, uint64_t P, const float* zraw, const float* zq, const float* zq1,
                       const float* hq, const float* hq1, uint64_t ldq, uint64_t d,
                       uint64_t row_offset, float beta, float* opart, float* lpart, uint64_t table_rows,
                       cudaStream_t s, const Panels* fpn = nullptr, float* seg_o = nullptr,
                       float* seg_l = nullptr, const AgnnNext* fnx = nullptr) {
  using C = AgnnCfg<DC, PREC>;
  // SGTK_AGNN_DENSE_SMEM (bytes): pad the dense kernel's shared memory, e.g.
  // to hold one CTA per SM and leave room for the concurrent CUDA-core kernel
  static const uint32_t pad = [] {
    const char* e = std::getenv("SGTK_AGNN_DENSE_SMEM");
    return e ? uint32_t(std::atoi(e)) : 0u;
  }();
  const uint32_t smem = std::max<uint32_t>(C::SMEM, std::min<uint32_t>(pad, 227u * 1024u));
  constexpr bool kFR = PREC != SGTK_FP32 && DC == 32;
  once_per_device(reinterpret_cast<const void*>(&agnn_dense_kernel<DC, PREC, false, false>), [] {
    cudaFuncSetAttribute(agnn_dense_kernel<DC, PREC, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(227u * 1024u));
    cudaFuncSetAttribute(agnn_dense_kernel<DC, PREC, PREC != SGTK_FP32, false>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, int(227u * 1024u));
    cudaFuncSetAttribute(agnn_dense_kernel<DC, PREC, false, kFR>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(227u * 1024u));
  });
  // SGTK_AGNN_GATHER=tma: TMA tile::gather4 instead of cp.async gathers
  // (measured neutral at C4: the gathers are not what bounds a chunk, and the
  // TMA unit moves ~14 B per cycle per SM as 128-byte rows)
  static const bool cp_gather = [] {
    const char* e = std::getenv("SGTK_AGNN_GATHER");
    return !(e && std::string(e) == "tma");
  }();
  CUtensorMap tmz{}, tmh{};
  bool tg = PREC != SGTK_FP32 && !cp_gather;
  if (tg)
    tg = make_gather_map(&tmz, zq, table_rows, ldq, CU_TENSOR_MAP_SWIZZLE_128B) &&
         make_gather_map(&tmh, hq, table_rows, ldq, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B);
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
  const AgnnNext nx0{};
  if (fpn && kFR)
    agnn_dense_kernel<DC, PREC, false, kFR><<<unsigned(P), agnn_threads(DC, PREC), smem, s>>>(
        v, zraw, zq, zq1, hq, hq1, ldq, d, row_offset, beta, opart, lpart, trace, tmz, tmh,
        fpn->aitems->as<uint4>(), fpn->sent->as<uint2>(), seg_o, seg_l, *fnx);
  else if (tg)
    agnn_dense_kernel<DC, PREC, PREC != SGTK_FP32, false><<<unsigned(P), agnn_threads(DC, PREC), smem, s>>>(
        v, zraw, zq, zq1, hq, hq1, ldq, d, row_offset, beta, opart, lpart, trace, tmz, tmh, nullptr, nullptr,
        nullptr, nullptr, nx0);
  else
    agnn_dense_kernel<DC, PREC, false, false><<<unsigned(P), agnn_threads(DC, PREC), smem, s>>>(
        v, zraw, zq, zq1, hq, hq1, ldq, d, row_offset, beta, opart, lpart, trace, tmz, tmh, nullptr, nullptr,
        nullptr, nullptr, nx0);
  if (trace) {
    std::vector<long long> hb(4 * 256 * 8);
    cudaMemcpy(hb.data(), trace, hb.size() * 8, cudaMemcpyDeviceToHost);
    if (FILE* f = std::fopen(std::getenv("SGTK_PANEL_TRACE"), "wb")) {
      std::fwrite(hb.data(), 8, hb.size(), f);
      std::fclose(f);
    }
  }
  CU_LAUNCH("agnn_dense_kernel");
}

template <int FPL, int PREC>
void launch_agnn_rows(const Panels& pn, const float* zown, const float* z, uint64_t ld, const float* norm, uint64_t d,
                      uint64_t row_offset, float beta, const float* opart, const float* lpart,
                      float* seg_o, float* seg_l, float* osp, float* lsp, const AgnnNext& nx,
                      uint64_t table_rows, cudaStream_t s, cudaStream_t s_final) {
  constexpr unsigned bs = FPL == 1 ? 32 * kRowsWarps1 : 32 * kRowsWarps2;
  if (pn.n_aitems) {
    if (osp)
      agnn_rows_kernel<FPL, PREC, true><<<rows_grid(pn.n_aitems, bs), bs, 0, s>>>(
          pn.aitems->as<uint4>(), pn.n_aitems, pn.sent->as<uint2>(), zown, z, ld, norm, d, row_offset, beta,
          opart, lpart, seg_o, seg_l, osp, lsp, nx);
    else
      agnn_rows_kernel<FPL, PREC, false><<<rows_grid(pn.n_aitems, bs), bs, 0, s>>>(
          pn.aitems->as<uint4>(), pn.n_aitems, pn.sent->as<uint2>(), zown, z, ld, norm, d, row_offset, beta,
          opart, lpart, seg_o, seg_l, osp, lsp, nx);
    CU_LAUNCH("agnn_rows_kernel");
  }
  if (osp) {  // concurrent mode: join, then finalise on the main stream
    const AuxStreams& ax = aux_streams();
    CU(cudaEventRecord(ax.join, s));
    CU(cudaStreamWaitEvent(s_final, ax.join, 0));
    // hub rows (few warps, latency-bound) beside the final kernel: both need
    // the dense and sparse partials, they write disjoint rows
    static const bool side_on = !std::getenv("SGTK_AGNN_LONG_SERIAL");
    const bool side = side_on && pn.n_long && s != s_final;
    if (side) {
      CU(cudaEventRecord(ax.ready, s_final));
      CU(cudaStreamWaitEvent(s, ax.ready, 0));
      agnn_long_rows_kernel<FPL, PREC><<<blocks_for(pn.n_long * 32), 256, 0, s>>>(
          pn.lrows->as<uint4>(), pn.n_long, d, opart, lpart, seg_o, seg_l, nx);
      CU_LAUNCH("agnn_long_rows_kernel");
    }
    if (pn.n_aitems) {
      agnn_final_kernel<FPL, PREC><<<final_grid(pn.n_aitems), 256, 0, s_final>>>(
          pn.aitems->as<uint4>(), pn.n_aitems, d, opart, lpart, osp, lsp, nx);
      CU_LAUNCH("agnn_final_kernel");
    }
    if (side) {
      CU(cudaEventRecord(ax.join, s));
      CU(cudaStreamWaitEvent(s_final, ax.join, 0));
      return;
    }
  }
  if (pn.n_long) {
    agnn_long_rows_kernel<FPL, PREC><<<blocks_for(pn.n_long * 32), 256, 0, s_final>>>(
        pn.lrows->as<uint4>(), pn.n_long, d, opart, lpart, seg_o, seg_l, nx);
    CU_LAUNCH("agnn_long_rows_kernel");
  }
}

}  // namespace

bool agnn_panel_supported(const sgtk_graph* g, uint64_t d, float beta) {
  return g->panels && panel_enabled() && d > 0 && d <= 64 && std::fabs(beta) <= kMaxBeta &&
         g->n_cols <= 0x7FFFFFFFull;
}

// One AGNN layer.  z: l2-normalised input rows (raw fp32, n_cols x ldq);
// zq/zq1/hq/hq1: MMA operand copies of z and of the input h (TF32: rounded;
// FP32: hi / lo planes), stride ldq; h: the raw input rows (stride ldh).
// Writes nx.out (n_rows x d, when set) and, when nx.zq is set, the next layer's
// operand copies (which must not alias the inputs).
// Concurrent mode (default; SGTK_AGNN_SERIAL=1 turns it off): the dense
// tensor-core kernel runs on the caller's stream while the CUDA-core kernel
// runs on an auxiliary stream (the paper's two independent resources); the
// finalisation joins them.  Serial mode: dense, then rows (which finalises).
void agnn_panel_layer(const sgtk_graph* g, const float* z, const float* zq, const float* zq1,
                      const float* hq, const float* hq1, uint64_t ldq, const float* norm,
                      uint64_t d, float beta, int prec, float* opart, float* lpart, float* seg_o,
                      float* seg_l, float* osp, float* lsp, const AgnnNext& nx, cudaStream_t s) {
  const Panels& pn = panels_for(g, d);
  PanelView v = panel_view(g, d);
  const uint64_t ro = g->row_offset;
  const int dbg = panel_debug_mode();  // 1: dense part only, 2: sparse part only (timing)
  static const bool serial = std::getenv("SGTK_AGNN_SERIAL") != nullptr;
  auto dense = [&](cudaStream_t st) {
    if (prec == SGTK_FP32) {
      if (ldq == 32) launch_agnn_dense<32, SGTK_FP32>(v, pn.P, z, zq, zq1, hq, hq1, ldq, d, ro, beta, opart, lpart, g->n_cols, st);
      else launch_agnn_dense<64, SGTK_FP32>(v, pn.P, z, zq, zq1, hq, hq1, ldq, d, ro, beta, opart, lpart, g->n_cols, st);
    } else {
      if (ldq == 32) launch_agnn_dense<32, SGTK_TF32>(v, pn.P, zq, zq, nullptr, hq, nullptr, ldq, d, ro, beta, opart, lpart, g->n_cols, st);
      else launch_agnn_dense<64, SGTK_TF32>(v, pn.P, zq, zq, nullptr, hq, nullptr, ldq, d, ro, beta, opart, lpart, g->n_cols, st);
    }
  };
  auto rows = [&](cudaStream_t st, float* o_sp, float* l_sp, cudaStream_t st_final) {
    if (prec == SGTK_FP32) {
      if (ldq == 32) launch_agnn_rows<1, SGTK_FP32>(pn, z, z, ldq, norm, d, ro, beta, opart, lpart, seg_o, seg_l, o_sp, l_sp, nx, g->n_cols, st, st_final);
      else launch_agnn_rows<2, SGTK_FP32>(pn, z, z, ldq, norm, d, ro, beta, opart, lpart, seg_o, seg_l, o_sp, l_sp, nx, g->n_cols, st, st_final);
    } else {
      if (ldq == 32) launch_agnn_rows<1, SGTK_TF32>(pn, zq, hq, ldq, norm, d, ro, beta, opart, lpart, seg_o, seg_l, o_sp, l_sp, nx, g->n_cols, st, st_final);
      else launch_agnn_rows<2, SGTK_TF32>(pn, zq, hq, ldq, norm, d, ro, beta, opart, lpart, seg_o, seg_l, o_sp, l_sp, nx, g->n_cols, st, st_final);
    }
  };
  if (dbg == 1) {
    dense(s);
    return;
  }
  // SGTK_AGNN_FUSED=1: the fused form (dense chunks, then the panel's sparse
  // rows in the same CTA) -- measured slower at C4 (0.645 against 0.543 ms per
  // layer): a CTA in its sparse phase holds the shared memory and warp slots a
  // dense CTA needs, and 24 warps per SM hide less gather latency than the
  // concurrent sparse kernel's 40
  static const bool unfused = [] {
    const char* e = std::getenv("SGTK_AGNN_FUSED");
    return !(e && std::string(e) == "1");
  }();
  if (prec == SGTK_TF32 && ldq == 32 && !unfused && !serial && dbg == 0) {
    ensure_paitem(pn, s);
    v.paitem = pn.paitem->as<uint32_t>();
    launch_agnn_dense<32, SGTK_TF32>(v, pn.P, zq, zq, nullptr, hq, nullptr, ldq, d, ro, beta, opart, lpart,
                                     g->n_cols, s, &pn, seg_o, seg_l, &nx);
    if (pn.n_long) {
      agnn_long_rows_kernel<1, SGTK_TF32><<<blocks_for(pn.n_long * 32), 256, 0, s>>>(
          pn.lrows->as<uint4>(), pn.n_long, d, opart, lpart, seg_o, seg_l, nx);
      CU_LAUNCH("agnn_long_rows_kernel");
    }
    return;
  }
  if (dbg == 2) {
    CU(cudaMemsetAsync(opart, 0, g->n_rows * ldq * 4, s));
    CU(cudaMemsetAsync(lpart, 0, g->n_rows * 4, s));
    rows(s, nullptr, nullptr, s);
    return;
  }
  if (serial || !osp) {
    dense(s);
    rows(s, nullptr, nullptr, s);
    return;
  }
  const AuxStreams& ax = aux_streams();
  CU(cudaEventRecord(ax.ready, s));  // inputs of the layer are on s
  CU(cudaStreamWaitEvent(ax.aux, ax.ready, 0));
  dense(s);
  rows(ax.aux, osp, lsp, s);  // sparse partials on aux; final + hub rows join on s
}

void agnn_input_launch(const float* x, uint64_t ldx, uint64_t rows, uint64_t d, uint64_t ldq, int prec,
                       float* z, float* zq, float* zq1, float* hq, float* hq1, float* norm,
                       uint64_t* zeros, cudaStream_t s) {
  if (!rows) return;
  auto* zc = reinterpret_cast<unsigned long long*>(zeros);
  const unsigned nb = blocks_for((rows + 3) / 4 * 32);
  if (ldq == 32) {
    if (prec == SGTK_FP32) agnn_input_kernel<1, SGTK_FP32><<<nb, 256, 0, s>>>(x, ldx, rows, d, ldq, z, zq, zq1, hq, hq1, norm, zc);
    else agnn_input_kernel<1, SGTK_TF32><<<nb, 256, 0, s>>>(x, ldx, rows, d, ldq, z, zq, zq1, hq, hq1, norm, zc);
  } else {
    if (prec == SGTK_FP32) agnn_input_kernel<2, SGTK_FP32><<<nb, 256, 0, s>>>(x, ldx, rows, d, ldq, z, zq, zq1, hq, hq1, norm, zc);
    else agnn_input_kernel<2, SGTK_TF32><<<nb, 256, 0, s>>>(x, ldx, rows, d, ldq, z, zq, zq1, hq, hq1, norm, zc);
  }
  CU_LAUNCH("agnn_input_kernel");
}

}  // namespace sgtkcu
