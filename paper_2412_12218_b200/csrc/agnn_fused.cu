// Fused AGNN layer: SDDMM -> edge softmax -> SpMM in one pass per window.
//
// Replaces, for one layer of agnn_forward (/root/reference/proj/src/gnn.cpp:107-116):
//   logits = beta * sddmm_hybrid(t16, z, z, unit)   (tile_exec.cpp:316-411)
//   attn   = edge_softmax(csr, logits)              (gnn.cpp:54-72)
//   h'     = spmm_hybrid(t, h, attn)                (tile_exec.cpp:200-314)
// with z = l2norm(h) applied on the fly (inv_norm from the row-norm kernel).
//
// One warp owns a 16-row window (or a slice of its 16-wide tiles).  Per tile:
//   S  = Q K^T       16x16, Q = z rows of the window (A fragments, registers),
//                    K = z rows of the tile's 16 unique columns
//   mask by the tile's 16x16 occupancy bitmap, online softmax per row (exp2)
//   O += P V         P re-used straight from S's accumulator layout (the PV
//                    MMA's k index is permuted so no shuffle is needed),
//                    V = h rows of the tile columns
// The next tile's 16 column ids, bitmap and gathered rows are prefetched into
// registers while the current tile computes (two tiles in flight per warp).
// Logits and attention never touch HBM: per layer the kernel reads the
// bitmaps, the unique-column ids and gathered feature rows and writes N x d —
// the "fused" lower bound of SURVEY.md §8(d) instead of the unfused chain's
// E-sized round trips.
//
// Precision.  TF32: operands RNE-rounded like tf32_round_value.  FP32:
//   S uses 3xTF32 (q = qh + ql, k = kh + kl, drops ql*kl ~ 2^-22 relative);
//   PV uses the exact-on-representable 4-term split (common.cuh) so unit
//   attention reproduces h bit-exactly (test_gnn.cpp:157-164).
// Tiles at or past the plan's cut go edge-by-edge on CUDA cores into the same
// running state; windows split over several warps merge (m, l, O) in order.

#include <cstdlib>

#include "graph.cuh"

namespace sgtkcu {
namespace {

constexpr int kWarps = 4;
constexpr float kLog2e = 1.4426950408889634f;

__device__ __forceinline__ float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

__device__ __forceinline__ uint32_t bits16(const uint4& lo, const uint4& hi, uint32_t r) {
  const uint4& b = r < 8 ? lo : hi;
  const uint32_t rr = r & 7u;
  const uint32_t w = rr < 4 ? (rr < 2 ? b.x : b.y) : (rr < 6 ? b.z : b.w);
  return (w >> ((rr & 1u) * 16)) & 0xFFFFu;
}

__device__ __forceinline__ float quad_max(float v) {
  v = fmaxf(v, __shfl_xor_sync(0xFFFFFFFFu, v, 1));
  return fmaxf(v, __shfl_xor_sync(0xFFFFFFFFu, v, 2));
}
__device__ __forceinline__ float quad_sum(float v) {
  v += __shfl_xor_sync(0xFFFFFFFFu, v, 1);
  return v + __shfl_xor_sync(0xFFFFFFFFu, v, 2);
}

// NB contiguous floats of row `row` starting at feature f.  FULL: the segment
// is known in-bounds and 16-byte aligned (d == 8*NB, ld % 4 == 0).
template <int NB, bool FULL>
__device__ __forceinline__ void ld_seg(float (&dst)[NB], const float* __restrict__ h, uint64_t ldh,
                                       uint64_t row, uint64_t f, uint64_t d) {
  if constexpr (FULL) {
    load_seg<NB, true>(dst, h + row * ldh + f, NB);
  } else {
    const int64_t rem = int64_t(d) - int64_t(f);
    load_seg<NB, false>(dst, h + row * ldh + f, rem <= 0 ? 0 : (rem > NB ? NB : int(rem)));
  }
}

// Running state of one row (replicated over its 4 lanes), log2 domain.
struct RowState {
  float m, l;
};

// New row max -> rescale factor for the old (l, O); returns the max to use.
__device__ __forceinline__ float online_update(RowState& st, float tile_max, float& scale) {
  const float mn = fmaxf(st.m, tile_max);
  scale = mn == -INFINITY ? 1.0f : ex2(st.m - mn);  // ex2(-inf) = 0
  st.m = mn;
  st.l *= scale;
  return mn == -INFINITY ? 0.0f : mn;
}

// Per-tile gathered operands (registers).
template <int NB>
struct TileRegs {
  float k0[2][NB], k1[2][NB];  // z rows of cols nb*8+g: features t*NB.., (t+4)*NB..
  float v[2][2][NB];           // h rows of cols kb*8+2t(+1): features g*NB..
  uint32_t wa, wb;             // bitmap rows g, g+8
};

// Column ids straight from window_unique_cols (no shuffles on the address
// chain); ragged lanes of the last tile reuse the window's last column
// (finite data, masked out by the bitmap).  K rows come from z (the
// normalised rows, materialised by the row-norm kernel as the reference does,
// gnn.cpp:109), V rows from h.
template <int NB, bool FULL>
__device__ __forceinline__ void fetch_tile(TileRegs<NB>& R, const DevGraph& G,
                                           const float* __restrict__ h,
                                           const float* __restrict__ z, uint64_t ldh,
                                           uint64_t ldz, uint64_t d,
                                           uint64_t ubase, uint32_t ucnt, uint64_t tileg,
                                           uint32_t tile, uint32_t g, uint32_t t) {
  const uint4 blo = __ldg(G.bm16 + 2 * tileg);
  const uint4 bhi = __ldg(G.bm16 + 2 * tileg + 1);
  R.wa = bits16(blo, bhi, g);
  R.wb = bits16(blo, bhi, g + 8);
  const uint32_t last = ucnt - 1u;
  const uint32_t* ids = G.wuc + ubase;
  uint32_t ck[2], cv[2][2];
#pragma unroll
  for (int nb = 0; nb < 2; ++nb) {
    const uint32_t c0 = tile * 16u + nb * 8u;
    ck[nb] = __ldg(ids + min(c0 + g, last));
    cv[nb][0] = __ldg(ids + min(c0 + 2u * t, last));
    cv[nb][1] = __ldg(ids + min(c0 + 2u * t + 1u, last));
  }
#pragma unroll
  for (int nb = 0; nb < 2; ++nb) {
    ld_seg<NB, FULL>(R.k0[nb], z, ldz, ck[nb], t * NB, d);
    ld_seg<NB, FULL>(R.k1[nb], z, ldz, ck[nb], (t + 4) * NB, d);
    ld_seg<NB, FULL>(R.v[nb][0], h, ldh, cv[nb][0], g * NB, d);
    ld_seg<NB, FULL>(R.v[nb][1], h, ldh, cv[nb][1], g * NB, d);
  }
}

#ifndef SGTK_AGNN_MINB
#define SGTK_AGNN_MINB 1
#endif

// Any non-finite value among a lane's stored outputs -> *flag = 1 (warp vote,
// one atomic per warp).  All lanes of the warp reach the epilogue together.
template <int N>
__device__ __forceinline__ void flag_nonfinite(const float (&a)[N], const float (&b)[N], bool va,
                                               bool vb, int valid, uint32_t* flag) {
  bool bad = false;
#pragma unroll
  for (int j = 0; j < N; ++j) bad |= j < valid && ((va && !isfinite(a[j])) || (vb && !isfinite(b[j])));
  if (__any_sync(0xFFFFFFFFu, bad) && (threadIdx.x & 31) == 0) atomicOr(flag, 1u);
}

template <int NB, int PREC, bool FULL>
__global__ void __launch_bounds__(kWarps * 32, SGTK_AGNN_MINB)
agnn_fused_kernel(const DevGraph G, const WorkUnit* __restrict__ units, uint32_t n_units,
                  const uint32_t* __restrict__ thr, const float* __restrict__ h,
                  const float* __restrict__ z, uint64_t ldh, uint64_t ldz, uint64_t d, float beta,
                  float* __restrict__ out, uint64_t ldo, float* __restrict__ partial,
                  uint64_t pstride, uint32_t* __restrict__ nonfinite) {
  const uint32_t wid = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (wid >= n_units) return;
  const WorkUnit u = units[wid];
  const uint32_t lane = lane_id(), g = lane >> 2, t = lane & 3u;
  const uint64_t w = u.window;
  const uint64_t ra = w * 16 + g, rb = ra + 8;
  const bool va = ra < G.n_rows, vb = rb < G.n_rows;
  const uint64_t xa = G.row_offset + (va ? ra : 0), xb = G.row_offset + (vb ? rb : 0);
  const uint64_t ubase = G.wo[w];
  const uint32_t ucnt = uint32_t(G.wo[w + 1] - ubase);
  const uint32_t ntiles = (ucnt + 15u) >> 4;
  const uint64_t tbase = G.toff16[w];
  const uint32_t tc_end = thr ? min(u.t1, max(u.t0, thr[w])) : u.t1;
  const float scale2 = beta * kLog2e;  // logits kept in the log2 domain

  // ---- Q fragments: z rows, features k*NB + s (s = k-step) ---------------
  uint32_t qh[4][NB], ql[4][NB];  // [a0 a1 a2 a3][s]
  {
    float s_[NB];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const bool rowa = (q & 1) == 0;
      ld_seg<NB, FULL>(s_, z, ldz, rowa ? xa : xb, (q < 2 ? t : t + 4) * NB, d);
      const bool ok = rowa ? va : vb;
#pragma unroll
      for (int i = 0; i < NB; ++i) split_s<PREC>(ok ? s_[i] : 0.0f, qh[q][i], ql[q][i]);
    }
  }

  float o[NB][4];
#pragma unroll
  for (int j = 0; j < NB; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.0f;
  RowState sa{-INFINITY, 0.0f}, sb{-INFINITY, 0.0f};

  // ---------------- tensor-core path (software-pipelined) ------------------
  auto process = [&](const TileRegs<NB>& cur) {
    // S = Q K^T  (n-block nb: tile columns nb*8 + g)
    float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int i = 0; i < NB; ++i) {
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) {
        uint32_t b0, c0, b1, c1;
        split_s<PREC>(cur.k0[nb][i], b0, c0);
        split_s<PREC>(cur.k1[nb][i], b1, c1);
        if constexpr (PREC == SGTK_FP32) {
          mma_tf32(s[nb], ql[0][i], ql[1][i], ql[2][i], ql[3][i], b0, b1);
          mma_tf32(s[nb], qh[0][i], qh[1][i], qh[2][i], qh[3][i], c0, c1);
        }
        mma_tf32(s[nb], qh[0][i], qh[1][i], qh[2][i], qh[3][i], b0, b1);
      }
    }
    // logits (log2 domain), mask.  s[nb][q]: row g (q<2) / g+8, col nb*8+2t+(q&1)
    float tma = -INFINITY, tmb = -INFINITY;
#pragma unroll
    for (int nb = 0; nb < 2; ++nb)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t c = nb * 8u + 2u * t + (q & 1u);
        const bool edge = ((q < 2 ? cur.wa : cur.wb) >> c) & 1u;
        float v = s[nb][q];
        if constexpr (PREC == SGTK_TF32) v = __uint_as_float(tf32_op(v));  // tf32(1)*tf32(dot)
        v = edge ? v * scale2 : -INFINITY;
        s[nb][q] = v;
        if (q < 2) tma = fmaxf(tma, v); else tmb = fmaxf(tmb, v);
      }
    float sca, scb;
    const float ma = online_update(sa, quad_max(tma), sca);
    const float mb = online_update(sb, quad_max(tmb), scb);
    float pa = 0.f, pb = 0.f;
#pragma unroll
    for (int nb = 0; nb < 2; ++nb)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float p = ex2(s[nb][q] - (q < 2 ? ma : mb));  // masked: ex2(-inf) = 0
        s[nb][q] = p;
        if (q < 2) pa += p; else pb += p;
      }
    sa.l += quad_sum(pa);
    sb.l += quad_sum(pb);
    // O = O * scale + P V.  The tile's P V is a fresh tensor-core partial
    // folded into the IEEE fp32 running sum by one FFMA per element (the
    // online-softmax rescale rides along for free): tensor-core accumulation
    // does not round to nearest, so O never sits on a long MMA chain.
    // k-step kb covers tile columns kb*8 + {2t, 2t+1} for A's k = {t, t+4}:
    // exactly the columns this lane's S accumulator holds.
    float po[NB][4];
#pragma unroll
    for (int j = 0; j < NB; ++j) po[j][0] = po[j][1] = po[j][2] = po[j][3] = 0.0f;
#pragma unroll
    for (int kb = 0; kb < 2; ++kb) {
      uint32_t p0[4], p1[4];
      split_s<PREC>(s[kb][0], p0[0], p1[0]);  // (g,   2t)   -> a0
      split_s<PREC>(s[kb][2], p0[1], p1[1]);  // (g+8, 2t)   -> a1
      split_s<PREC>(s[kb][1], p0[2], p1[2]);  // (g,   2t+1) -> a2
      split_s<PREC>(s[kb][3], p0[3], p1[3]);  // (g+8, 2t+1) -> a3
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        uint32_t x0, x1, x2, y0, y1, y2;
        split_d<PREC>(cur.v[kb][0][j], x0, x1, x2);
        split_d<PREC>(cur.v[kb][1][j], y0, y1, y2);
        if constexpr (PREC == SGTK_FP32) {
          mma_tf32(po[j], p0[0], p0[1], p0[2], p0[3], x2, y2);
          mma_tf32(po[j], p1[0], p1[1], p1[2], p1[3], x0, y0);
          mma_tf32(po[j], p0[0], p0[1], p0[2], p0[3], x1, y1);
        }
        mma_tf32(po[j], p0[0], p0[1], p0[2], p0[3], x0, y0);
      }
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      o[j][0] = fmaf(o[j][0], sca, po[j][0]);
      o[j][1] = fmaf(o[j][1], sca, po[j][1]);
      o[j][2] = fmaf(o[j][2], scb, po[j][2]);
      o[j][3] = fmaf(o[j][3], scb, po[j][3]);
    }
  };

  // the next tile's ids/bitmap/rows are in flight while the current computes
  TileRegs<NB> cur, nxt;
  if (u.t0 < tc_end)
    fetch_tile<NB, FULL>(cur, G, h, z, ldh, ldz, d, ubase, ucnt, tbase + u.t0, u.t0, g, t);
  for (uint32_t tile = u.t0; tile < tc_end; ++tile) {
    if (tile + 1 < tc_end)
      fetch_tile<NB, FULL>(nxt, G, h, z, ldh, ldz, d, ubase, ucnt, tbase + tile + 1, tile + 1, g, t);
    process(cur);
    cur = nxt;
  }

  // ---------------- CUDA-core path: edges of tiles [tc_end, t1) -----------
  uint64_t ca = 0, cb = 0, ea = 0, eb = 0;
  if (tc_end < u.t1) {
    ca = va ? G.np[ra] : 0; ea = va ? G.np[ra + 1] : 0;
    cb = vb ? G.np[rb] : 0; eb = vb ? G.np[rb + 1] : 0;
    ca = lower_bound_u32(G.e2c, ca, ea, tc_end * 16u);
    cb = lower_bound_u32(G.e2c, cb, eb, tc_end * 16u);
    if (u.t1 < ntiles) {
      ea = lower_bound_u32(G.e2c, ca, ea, u.t1 * 16u);
      eb = lower_bound_u32(G.e2c, cb, eb, u.t1 * 16u);
    }
  }
  {
    const uint32_t na = uint32_t(ea - ca), nbb = uint32_t(eb - cb);
    const uint32_t mx = __reduce_max_sync(0xFFFFFFFFu, max(na, nbb));
    for (uint32_t i = 0; i < mx; ++i) {
#pragma unroll
      for (int half = 0; half < 2; ++half) {
        const bool act = half ? i < nbb : i < na;
        const uint64_t e = (half ? cb : ca) + i;
        const uint32_t col = act ? __ldg(G.el + e) : 0u;
        float k0[NB], k1[NB];
        ld_seg<NB, FULL>(k0, z, ldz, col, t * NB, d);
        ld_seg<NB, FULL>(k1, z, ldz, col, (t + 4) * NB, d);
        float part = 0.0f;
        const int qa = half ? 1 : 0;
#pragma unroll
        for (int s_ = 0; s_ < NB; ++s_) {
          const float z0 = __uint_as_float(qh[qa][s_]) + __uint_as_float(ql[qa][s_]);
          const float z1 = __uint_as_float(qh[qa + 2][s_]) + __uint_as_float(ql[qa + 2][s_]);
          float y0 = k0[s_], y1 = k1[s_];
          if constexpr (PREC == SGTK_TF32) { y0 = tf32_rne(y0); y1 = tf32_rne(y1); }
          part = fmaf(z0, y0, part);
          part = fmaf(z1, y1, part);
        }
        float logit = quad_sum(part);
        if constexpr (PREC == SGTK_TF32) logit = tf32_rne(logit);
        logit = act ? logit * scale2 : -INFINITY;
        RowState& st = half ? sb : sa;
        float sc;
        const float m = online_update(st, logit, sc);
        const float p = ex2(logit - m);
        st.l += p;
        float vs[2 * NB];
        ld_seg<2 * NB, FULL>(vs, h, ldh, col, 2u * t * NB, d);
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          float x0 = vs[j], x1 = vs[NB + j];
          if constexpr (PREC == SGTK_TF32) { x0 = tf32_rne(x0); x1 = tf32_rne(x1); }
          o[j][2 * half] = fmaf(p, x0, o[j][2 * half] * sc);
          o[j][2 * half + 1] = fmaf(p, x1, o[j][2 * half + 1] * sc);
        }
      }
    }
  }

  // ---------------- epilogue ---------------------------------------------
  const uint64_t sf = 2u * t * NB;
  const int64_t rem = int64_t(d) - int64_t(sf);
  const int svalid = rem <= 0 ? 0 : (rem > 2 * NB ? 2 * NB : int(rem));
  if (u.slot == kNoSlot) {
    // l == 0: no edges; a NaN l (non-finite input) propagates
    const float la = sa.l != 0.0f ? 1.0f / sa.l : 0.0f, lb = sb.l != 0.0f ? 1.0f / sb.l : 0.0f;
    float va_[2 * NB], vb_[2 * NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      va_[j] = o[j][0] * la; va_[NB + j] = o[j][1] * la;
      vb_[j] = o[j][2] * lb; vb_[NB + j] = o[j][3] * lb;
    }
    if (va) store_seg<2 * NB, FULL>(out + ra * ldo + sf, va_, svalid);
    if (vb) store_seg<2 * NB, FULL>(out + rb * ldo + sf, vb_, svalid);
    if (nonfinite) flag_nonfinite<2 * NB>(va_, vb_, va, vb, svalid, nonfinite);
  } else {
    // partial state: O[16][8*NB], then m[16] (log2 domain), l[16]
    float* P = partial + uint64_t(u.slot) * pstride;
    float va_[2 * NB], vb_[2 * NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      va_[j] = o[j][0]; va_[NB + j] = o[j][1];
      vb_[j] = o[j][2]; vb_[NB + j] = o[j][3];
    }
    store_seg<2 * NB, true>(P + g * 8 * NB + sf, va_, 2 * NB);
    store_seg<2 * NB, true>(P + (g + 8) * 8 * NB + sf, vb_, 2 * NB);
    if (t == 0) {
      P[16 * 8 * NB + g] = sa.m;
      P[16 * 8 * NB + g + 8] = sb.m;
      P[16 * 8 * NB + 16 + g] = sa.l;
      P[16 * 8 * NB + 16 + g + 8] = sb.l;
    }
  }
}

// Split windows: merge (m, l, O) states in unit order.
template <int NB>
__global__ void agnn_merge_kernel(const ReduceItem* __restrict__ items, uint64_t n_rows,
                                  const float* __restrict__ partial, uint64_t pstride, uint64_t d,
                                  float* __restrict__ out, uint64_t ldo,
                                  uint32_t* __restrict__ nonfinite) {
  const ReduceItem it = items[blockIdx.x];
  for (uint32_t i = threadIdx.x; i < 16u * 8u * NB; i += blockDim.x) {
    const uint32_t rr = i / (8 * NB), f = i % (8 * NB);
    const uint64_t r = uint64_t(it.window) * 16 + rr;
    if (r >= n_rows || f >= d) continue;
    float M = -INFINITY;
    for (uint32_t k = 0; k < it.count; ++k)
      M = fmaxf(M, partial[uint64_t(it.slot0 + k) * pstride + 16 * 8 * NB + rr]);
    float L = 0.0f, O = 0.0f;
    for (uint32_t k = 0; k < it.count; ++k) {
      const float* P = partial + uint64_t(it.slot0 + k) * pstride;
      const float m = P[16 * 8 * NB + rr];
      if (m == -INFINITY) continue;
      const float sc = exp2f(m - M);
      L += P[16 * 8 * NB + 16 + rr] * sc;
      O += P[rr * 8 * NB + f] * sc;
    }
    const float v = L != 0.0f ? O * (1.0f / L) : 0.0f;
    out[r * ldo + f] = v;
    if (nonfinite && !isfinite(v)) atomicOr(nonfinite, 1u);
  }
}

// ===========================================================================
// v3 (d == 32, every tile on the tensor cores): shared-memory staging.
// Each warp keeps a kStages ring of tile slots filled with cp.async (L2 ->
// smem, no registers): the tile's 16 gathered h rows (2 KB, XOR-swizzled per
// 16-byte chunk), their 16 inv_norm values and the 32-byte bitmap.  Only h is
// gathered: S = (z_row . h_col) * inv_col, so K and V share one copy (half the
// L2 traffic of gathering z and h).  Feature map for the S MMA: k-column k
// of k-step i is feature 8(k mod 4) + 4(k div 4) + i, i.e. lane t reads the
// 16-byte chunks 2t and 2t+1 of a row; with the XOR swizzle (chunk ^ row%8)
// every fragment read (K: row g; V: rows 2t, 2t+1) is bank-conflict free.
// ===========================================================================
constexpr int kStages = 4;

struct V3Slot {
  float rows[16][32];
  float inv[16];
  uint32_t bm[8];
};

__device__ __forceinline__ void cp_async16_cg(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_async4_ca(void* dst, const void* src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(dst))),
               "l"(src)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N) : "memory");
}

template <int PREC>
__global__ void __launch_bounds__(kWarps * 32, 4)
agnn_fused_v3_kernel(const DevGraph G, const WorkUnit* __restrict__ units, uint32_t n_units,
                     const float* __restrict__ h, uint64_t ldh, const float* __restrict__ inv,
                     float beta, float* __restrict__ out, uint64_t ldo,
                     float* __restrict__ partial, uint64_t pstride, uint32_t* __restrict__ nonfinite) {
  constexpr int NB = 4;
  extern __shared__ __align__(16) uint8_t smem_v3[];
  const uint32_t wib = threadIdx.x >> 5;
  const uint32_t wid = blockIdx.x * kWarps + wib;
  if (wid >= n_units) return;
  V3Slot* ring = reinterpret_cast<V3Slot*>(smem_v3) + wib * kStages;
  const WorkUnit u = units[wid];
  const uint32_t lane = lane_id(), g = lane >> 2, t = lane & 3u;
  const uint64_t w = u.window;
  const uint64_t ra = w * 16 + g, rb = ra + 8;
  const bool va = ra < G.n_rows, vb = rb < G.n_rows;
  const uint64_t xa = G.row_offset + (va ? ra : 0), xb = G.row_offset + (vb ? rb : 0);
  const uint64_t ubase = G.wo[w];
  const uint32_t ucnt = uint32_t(G.wo[w + 1] - ubase);
  const uint64_t tbase = G.toff16[w];
  const float scale2 = beta * kLog2e;

  // ---- Q: z rows g, g+8; k-col t <-> chunk 2t, k-col t+4 <-> chunk 2t+1 ----
  uint32_t qh[4][NB], ql[4][NB];
  {
    const float ia = va ? __ldg(inv + xa) : 0.0f, ib = vb ? __ldg(inv + xb) : 0.0f;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const bool rowa = (q & 1) == 0;
      const float4 v = __ldg(reinterpret_cast<const float4*>(h + (rowa ? xa : xb) * ldh) +
                             (2 * t + (q >> 1)));
      const float sc = rowa ? ia : ib;
      split_s<PREC>(v.x * sc, qh[q][0], ql[q][0]);
      split_s<PREC>(v.y * sc, qh[q][1], ql[q][1]);
      split_s<PREC>(v.z * sc, qh[q][2], ql[q][2]);
      split_s<PREC>(v.w * sc, qh[q][3], ql[q][3]);
    }
  }

  // ---- producer: fill one slot with tile `tile` (all 32 lanes) -------------
  const uint32_t* ids = G.wuc + ubase;
  const uint32_t last = ucnt ? ucnt - 1u : 0u;
  auto produce = [&](uint32_t tile, V3Slot& sl) {
    const uint32_t c = lane & 7u;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t r = (lane >> 3) + 4u * k;
      const uint32_t id = __ldg(ids + min(tile * 16u + r, last));
      cp_async16_cg(&sl.rows[r][(c ^ (r & 7u)) * 4u], h + uint64_t(id) * ldh + c * 4u);
    }
    if (lane < 16) {
      const uint32_t id = __ldg(ids + min(tile * 16u + lane, last));
      cp_async4_ca(&sl.inv[lane], inv + id);
    } else if (lane < 18) {
      cp_async16_cg(&sl.bm[(lane - 16) * 4], G.bm16 + 2 * (tbase + tile) + (lane - 16));
    }
  };

  float o[NB][4];
#pragma unroll
  for (int j = 0; j < NB; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.0f;
  RowState sa{-INFINITY, 0.0f}, sb{-INFINITY, 0.0f};

#pragma unroll
  for (int s = 0; s < kStages - 1; ++s) {
    if (u.t0 + s < u.t1) produce(u.t0 + s, ring[s]);
    cp_commit();
  }
  for (uint32_t tile = u.t0; tile < u.t1; ++tile) {
    const uint32_t it = tile - u.t0;
    if (tile + kStages - 1 < u.t1) produce(tile + kStages - 1, ring[(it + kStages - 1) % kStages]);
    cp_commit();
    cp_wait<kStages - 1>();
    __syncwarp();
    const V3Slot& sl = ring[it % kStages];

    const uint4 blo = *reinterpret_cast<const uint4*>(&sl.bm[0]);
    const uint4 bhi = *reinterpret_cast<const uint4*>(&sl.bm[4]);
    const uint32_t wa = bits16(blo, bhi, g), wb = bits16(blo, bhi, g + 8);

    // S = Q H^T (columns scaled by inv afterwards)
    float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      const uint32_t r = nb * 8u + g;
      const float4 k0 = *reinterpret_cast<const float4*>(&sl.rows[r][((2u * t) ^ g) * 4u]);
      const float4 k1 = *reinterpret_cast<const float4*>(&sl.rows[r][((2u * t + 1u) ^ g) * 4u]);
      const float kk0[4] = {k0.x, k0.y, k0.z, k0.w}, kk1[4] = {k1.x, k1.y, k1.z, k1.w};
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        uint32_t b0, c0, b1, c1;
        split_s<PREC>(kk0[i], b0, c0);
        split_s<PREC>(kk1[i], b1, c1);
        if constexpr (PREC == SGTK_FP32) {
          mma_tf32(s[nb], ql[0][i], ql[1][i], ql[2][i], ql[3][i], b0, b1);
          mma_tf32(s[nb], qh[0][i], qh[1][i], qh[2][i], qh[3][i], c0, c1);
        }
        mma_tf32(s[nb], qh[0][i], qh[1][i], qh[2][i], qh[3][i], b0, b1);
      }
    }
    // logits: * inv[col] (z_col = h_col * inv_col), tf32 rounding, * beta, mask
    float tma = -INFINITY, tmb = -INFINITY;
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      const float2 ic = *reinterpret_cast<const float2*>(&sl.inv[nb * 8 + 2 * t]);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t c = nb * 8u + 2u * t + (q & 1u);
        const bool edge = ((q < 2 ? wa : wb) >> c) & 1u;
        float v = s[nb][q] * ((q & 1) ? ic.y : ic.x);
        if constexpr (PREC == SGTK_TF32) v = __uint_as_float(tf32_op(v));
        v = edge ? v * scale2 : -INFINITY;
        s[nb][q] = v;
        if (q < 2) tma = fmaxf(tma, v); else tmb = fmaxf(tmb, v);
      }
    }
    float sca, scb;
    const float ma = online_update(sa, quad_max(tma), sca);
    const float mb = online_update(sb, quad_max(tmb), scb);
    float pa = 0.f, pb = 0.f;
#pragma unroll
    for (int nb = 0; nb < 2; ++nb)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float p = ex2(s[nb][q] - (q < 2 ? ma : mb));
        s[nb][q] = p;
        if (q < 2) pa += p; else pb += p;
      }
    sa.l += quad_sum(pa);
    sb.l += quad_sum(pb);
    // O = O * scale + P V  (V rows kb*8 + 2t, +1; feature chunk g)
    float po[NB][4];
#pragma unroll
    for (int j = 0; j < NB; ++j) po[j][0] = po[j][1] = po[j][2] = po[j][3] = 0.0f;
#pragma unroll
    for (int kb = 0; kb < 2; ++kb) {
      uint32_t p0[4], p1[4];
      split_s<PREC>(s[kb][0], p0[0], p1[0]);
      split_s<PREC>(s[kb][2], p0[1], p1[1]);
      split_s<PREC>(s[kb][1], p0[2], p1[2]);
      split_s<PREC>(s[kb][3], p0[3], p1[3]);
      const uint32_t r0 = kb * 8u + 2u * t, r1 = r0 + 1u;
      const float4 v0 = *reinterpret_cast<const float4*>(&sl.rows[r0][(g ^ (r0 & 7u)) * 4u]);
      const float4 v1 = *reinterpret_cast<const float4*>(&sl.rows[r1][(g ^ (r1 & 7u)) * 4u]);
      const float vv0[4] = {v0.x, v0.y, v0.z, v0.w}, vv1[4] = {v1.x, v1.y, v1.z, v1.w};
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        uint32_t x0, x1, x2, y0, y1, y2;
        split_d<PREC>(vv0[j], x0, x1, x2);
        split_d<PREC>(vv1[j], y0, y1, y2);
        if constexpr (PREC == SGTK_FP32) {
          mma_tf32(po[j], p0[0], p0[1], p0[2], p0[3], x2, y2);
          mma_tf32(po[j], p1[0], p1[1], p1[2], p1[3], x0, y0);
          mma_tf32(po[j], p0[0], p0[1], p0[2], p0[3], x1, y1);
        }
        mma_tf32(po[j], p0[0], p0[1], p0[2], p0[3], x0, y0);
      }
    }
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      o[j][0] = fmaf(o[j][0], sca, po[j][0]);
      o[j][1] = fmaf(o[j][1], sca, po[j][1]);
      o[j][2] = fmaf(o[j][2], scb, po[j][2]);
      o[j][3] = fmaf(o[j][3], scb, po[j][3]);
    }
    __syncwarp();  // every lane is done with this slot before it is refilled
  }
  cp_wait<0>();

  // ---- epilogue (same layout as v2, NB = 4) --------------------------------
  const uint64_t sf = 2u * t * NB;
  float va_[2 * NB], vb_[2 * NB];
  if (u.slot == kNoSlot) {
    const float la = sa.l != 0.0f ? 1.0f / sa.l : 0.0f, lb = sb.l != 0.0f ? 1.0f / sb.l : 0.0f;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      va_[j] = o[j][0] * la; va_[NB + j] = o[j][1] * la;
      vb_[j] = o[j][2] * lb; vb_[NB + j] = o[j][3] * lb;
    }
    if (va) store_seg<2 * NB, true>(out + ra * ldo + sf, va_, 2 * NB);
    if (vb) store_seg<2 * NB, true>(out + rb * ldo + sf, vb_, 2 * NB);
    if (nonfinite) flag_nonfinite<2 * NB>(va_, vb_, va, vb, 2 * NB, nonfinite);
  } else {
    float* P = partial + uint64_t(u.slot) * pstride;
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      va_[j] = o[j][0]; va_[NB + j] = o[j][1];
      vb_[j] = o[j][2]; vb_[NB + j] = o[j][3];
    }
    store_seg<2 * NB, true>(P + g * 8 * NB + sf, va_, 2 * NB);
    store_seg<2 * NB, true>(P + (g + 8) * 8 * NB + sf, vb_, 2 * NB);
    if (t == 0) {
      P[16 * 8 * NB + g] = sa.m;
      P[16 * 8 * NB + g + 8] = sb.m;
      P[16 * 8 * NB + 16 + g] = sa.l;
      P[16 * 8 * NB + 16 + g + 8] = sb.l;
    }
  }
}

template <int PREC>
void launch_v3(const sgtk_graph* g, const float* h, uint64_t ldh, const float* inv, float beta,
               float* out, uint64_t ldo, uint32_t* nonfinite, cudaStream_t s) {
  const auto& P = g->plan16;
  const uint64_t pstride = 16 * 8 * 4 + 32;
  float* partial = nullptr;
  if (P.n_slots)
    CU(cudaMallocAsync(reinterpret_cast<void**>(&partial), uint64_t(P.n_slots) * pstride * 4, s));
  const size_t smem = size_t(kWarps) * kStages * sizeof(V3Slot);
  agnn_fused_v3_kernel<PREC><<<(P.n_units + kWarps - 1) / kWarps, kWarps * 32, smem, s>>>(
      g->view(), P.units->as<WorkUnit>(), P.n_units, h, ldh, inv, beta, out, ldo, partial, pstride,
      nonfinite);
  CU_LAUNCH("agnn_fused_v3_kernel");
  if (P.n_reduce) {
    agnn_merge_kernel<4><<<P.n_reduce, 256, 0, s>>>(P.reduce->as<ReduceItem>(), g->n_rows, partial,
                                                    pstride, 32, out, ldo, nonfinite);
    CU_LAUNCH("agnn_merge_kernel");
  }
  if (partial) CU(cudaFreeAsync(partial, s));
}

template <int NB, int PREC, bool FULL>
void launch(const sgtk_graph* g, const uint32_t* thr, const float* h, uint64_t ldh, const float* z,
            uint64_t ldz, uint64_t d, float beta, float* out, uint64_t ldo, uint32_t* nonfinite,
            cudaStream_t s) {
  const auto& P = g->plan16;
  const uint64_t pstride = 16 * 8 * NB + 32;
  float* partial = nullptr;
  if (P.n_slots)
    CU(cudaMallocAsync(reinterpret_cast<void**>(&partial), uint64_t(P.n_slots) * pstride * 4, s));
  agnn_fused_kernel<NB, PREC, FULL><<<(P.n_units + kWarps - 1) / kWarps, kWarps * 32, 0, s>>>(
      g->view(), P.units->as<WorkUnit>(), P.n_units, thr, h, z, ldh, ldz, d, beta, out, ldo,
      partial, pstride, nonfinite);
  CU_LAUNCH("agnn_fused_kernel");
  if (P.n_reduce) {
    agnn_merge_kernel<NB><<<P.n_reduce, 256, 0, s>>>(P.reduce->as<ReduceItem>(), g->n_rows,
                                                     partial, pstride, d, out, ldo, nonfinite);
    CU_LAUNCH("agnn_merge_kernel");
  }
  if (partial) CU(cudaFreeAsync(partial, s));
}

template <int NB>
void dispatch(int prec, bool full, const sgtk_graph* g, const uint32_t* thr, const float* h,
              uint64_t ldh, const float* z, uint64_t ldz, uint64_t d, float beta, float* out,
              uint64_t ldo, uint32_t* nf, cudaStream_t s) {
  if (prec == SGTK_FP32) {
    if (full) launch<NB, SGTK_FP32, true>(g, thr, h, ldh, z, ldz, d, beta, out, ldo, nf, s);
    else launch<NB, SGTK_FP32, false>(g, thr, h, ldh, z, ldz, d, beta, out, ldo, nf, s);
  } else {
    if (full) launch<NB, SGTK_TF32, true>(g, thr, h, ldh, z, ldz, d, beta, out, ldo, nf, s);
    else launch<NB, SGTK_TF32, false>(g, thr, h, ldh, z, ldz, d, beta, out, ldo, nf, s);
  }
}

}  // namespace

void agnn_fused_launch(const sgtk_graph* g, const float* h, uint64_t ldh, const float* z,
                       uint64_t ldz, const float* inv, uint64_t d, float beta, int prec,
                       const uint32_t* cut_dev, float* out, uint64_t ldo, cudaStream_t s,
                       uint32_t* nonfinite) {
  if (prec != SGTK_FP32 && prec != SGTK_TF32)
    raise(SGTK_ERR_RANGE, "agnn_forward: precision must be FP32 or TF32");
  if (d > 64) raise(SGTK_ERR_SHAPE, "agnn_forward: fused mode supports d <= 64 (use mode 0)");
  if (g->n_rows == 0 || d == 0) return;
  DevBuf cut_keep;
  const uint32_t* thr = internal_cut(g, cut_dev, 16, s, cut_keep);
  // d == 32 with every tile on the tensor cores: the smem-staged v3 kernel
  if (d == 32 && !thr && !getenv("SGTK_AGNN_V2") && ldh % 4 == 0 && ldo % 4 == 0 &&
      reinterpret_cast<uintptr_t>(h) % 16 == 0 && reinterpret_cast<uintptr_t>(out) % 16 == 0) {
    if (prec == SGTK_FP32) launch_v3<SGTK_FP32>(g, h, ldh, inv, beta, out, ldo, nonfinite, s);
    else launch_v3<SGTK_TF32>(g, h, ldh, inv, beta, out, ldo, nonfinite, s);
    return;
  }
  const int nb = d <= 16 ? 2 : d <= 32 ? 4 : 8;
  const bool full = uint64_t(8 * nb) == d && ldh % 4 == 0 && ldz % 4 == 0 && ldo % 4 == 0 &&
                    reinterpret_cast<uintptr_t>(h) % 16 == 0 &&
                    reinterpret_cast<uintptr_t>(z) % 16 == 0 &&
                    reinterpret_cast<uintptr_t>(out) % 16 == 0;
  if (nb == 2) dispatch<2>(prec, full, g, thr, h, ldh, z, ldz, d, beta, out, ldo, nonfinite, s);
  else if (nb == 4) dispatch<4>(prec, full, g, thr, h, ldh, z, ldz, d, beta, out, ldo, nonfinite, s);
  else dispatch<8>(prec, full, g, thr, h, ldh, z, ldz, d, beta, out, ldo, nonfinite, s);
}

}  // namespace sgtkcu
