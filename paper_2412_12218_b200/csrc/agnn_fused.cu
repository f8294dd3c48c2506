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
//                    K = z rows of the tile's 16 unique columns  (2x4 MMAs at d=32)
//   mask by the tile's 16x16 occupancy bitmap, online softmax per row
//   O += P V         P re-used straight from S's accumulator layout (the PV
//                    MMA's k index is permuted so no shuffle is needed),
//                    V = h rows of the tile columns              (2x4 MMAs)
// Logits and attention never touch HBM: per layer the kernel reads the
// bitmaps, the unique-column ids and gathered feature rows (L2-resident at
// the configs' sizes) and writes N x d — the "fused" lower bound of
// SURVEY.md §8(d) instead of the unfused chain's 2x4E round trips.
//
// Tiles at or past the plan's cut are processed edge-by-edge on CUDA cores
// (dot -> online softmax -> axpy) into the same running state.  Windows split
// over several warps merge their (m, l, O) states in unit order.
// Precision: TF32 = RNE-rounded operands; FP32 = the 4-term split (common.cuh).

#include "graph.cuh"

namespace sgtkcu {
namespace {

constexpr int kWarps = 4;

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

template <int NB, bool VEC>
__device__ __forceinline__ void load_row_seg(float (&dst)[NB], const float* __restrict__ h,
                                             uint64_t ldh, uint64_t row, uint64_t f, uint64_t d,
                                             bool ok) {
  const int64_t rem = int64_t(d) - int64_t(f);
  const int valid = !ok || rem <= 0 ? 0 : (rem > NB ? NB : int(rem));
  load_seg<NB, VEC>(dst, h + row * ldh + f, valid);
}

// Online-softmax running state of one row (replicated across its 4 lanes).
struct RowState {
  float m, l;
};

__device__ __forceinline__ void online_update(RowState& st, float tile_max, float& scale) {
  const float mn = fmaxf(st.m, tile_max);
  scale = (st.m == -INFINITY) ? 0.0f : expf(st.m - mn);
  if (mn == -INFINITY) scale = 1.0f;
  st.m = mn;
  st.l *= scale;
}

template <int NB, int PREC, bool VEC>
__global__ void __launch_bounds__(kWarps * 32)
agnn_fused_kernel(const DevGraph G, const WorkUnit* __restrict__ units, uint32_t n_units,
                  const uint32_t* __restrict__ thr, const float* __restrict__ h, uint64_t ldh,
                  uint64_t d, const float* __restrict__ inv, float beta, float* __restrict__ out,
                  uint64_t ldo, float* __restrict__ partial, uint64_t pstride) {
  const uint32_t wid = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (wid >= n_units) return;
  const WorkUnit u = units[wid];
  const uint32_t lane = lane_id(), g = lane >> 2, t = lane & 3u;
  const uint64_t w = u.window;
  const uint64_t ra = w * 16 + g, rb = ra + 8;
  const bool va = ra < G.n_rows, vb = rb < G.n_rows;
  const uint64_t xa = G.row_offset + ra, xb = G.row_offset + rb;
  const uint64_t ubase = G.wo[w];
  const uint32_t ucnt = uint32_t(G.wo[w + 1] - ubase);
  const uint32_t ntiles = (ucnt + 15u) >> 4;
  const uint64_t tbase = G.toff16[w];
  const uint32_t tc_end = thr ? min(u.t1, max(u.t0, thr[w])) : u.t1;

  // ---- Q fragments: z rows (h * inv), features k*NB + s  (s = k-step) ----
  const float ia = va ? __ldg(inv + xa) : 0.0f, ib = vb ? __ldg(inv + xb) : 0.0f;
  uint32_t q0[4][NB], q1[4][NB], q2[4][NB];  // [a0 a1 a2 a3][s], z = q0 + q1 + q2
  {
    float s_[NB];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const bool rowa = (q & 1) == 0;
      load_row_seg<NB, VEC>(s_, h, ldh, rowa ? xa : xb, (q < 2 ? t : t + 4) * NB, d,
                            rowa ? va : vb);
#pragma unroll
      for (int i = 0; i < NB; ++i) split_d<PREC>(s_[i] * (rowa ? ia : ib), q0[q][i], q1[q][i], q2[q][i]);
    }
  }

  float o[NB][4];
#pragma unroll
  for (int j = 0; j < NB; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.0f;
  RowState sa{-INFINITY, 0.0f}, sb{-INFINITY, 0.0f};

  uint64_t ca = 0, cb = 0, ea = 0, eb = 0;  // CSR cursors (CUDA-core path only)

  // ---------------- tensor-core path -------------------------------------
  for (uint32_t tile = u.t0; tile < tc_end; ++tile) {
    const uint4 blo = __ldg(G.bm16 + 2 * (tbase + tile));
    const uint4 bhi = __ldg(G.bm16 + 2 * (tbase + tile) + 1);
    const uint32_t wa = bits16(blo, bhi, g), wb = bits16(blo, bhi, g + 8);

    // S = Q K^T: B fragment of n-block nb is tile column nb*8 + g.
    float s[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      const uint32_t c = tile * 16u + nb * 8u + g;
      const bool ok = c < ucnt;
      const uint32_t col = ok ? __ldg(G.wuc + ubase + c) : 0u;
      const float ic = ok ? __ldg(inv + col) : 0.0f;
      float k0[NB], k1[NB];
      load_row_seg<NB, VEC>(k0, h, ldh, col, t * NB, d, ok);
      load_row_seg<NB, VEC>(k1, h, ldh, col, (t + 4) * NB, d, ok);
#pragma unroll
      for (int i = 0; i < NB; ++i) {
        uint32_t b0, c0, b1, c1;
        split_s<PREC>(k0[i] * ic, b0, c0);
        split_s<PREC>(k1[i] * ic, b1, c1);
        if constexpr (PREC == SGTK_FP32) {
          mma_tf32(s[nb], q2[0][i], q2[1][i], q2[2][i], q2[3][i], b0, b1);
          mma_tf32(s[nb], q0[0][i], q0[1][i], q0[2][i], q0[3][i], c0, c1);
          mma_tf32(s[nb], q1[0][i], q1[1][i], q1[2][i], q1[3][i], b0, b1);
        }
        mma_tf32(s[nb], q0[0][i], q0[1][i], q0[2][i], q0[3][i], b0, b1);
      }
    }
    // logits, mask (C layout: s[nb][q] is row g(+8), column nb*8 + 2t + (q&1))
    float tma = -INFINITY, tmb = -INFINITY;
#pragma unroll
    for (int nb = 0; nb < 2; ++nb)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t c = nb * 8u + 2u * t + (q & 1u);
        const bool edge = ((q < 2 ? wa : wb) >> c) & 1u;
        float v = s[nb][q];
        if constexpr (PREC == SGTK_TF32) v = tf32_rne(v);  // tf32(1) * tf32(dot)
        v = edge ? v * beta : -INFINITY;
        s[nb][q] = v;
        if (q < 2) tma = fmaxf(tma, v); else tmb = fmaxf(tmb, v);
      }
    tma = quad_max(tma);
    tmb = quad_max(tmb);
    float sca, scb;
    online_update(sa, tma, sca);
    online_update(sb, tmb, scb);
    float pa = 0.f, pb = 0.f;
#pragma unroll
    for (int nb = 0; nb < 2; ++nb)
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float m = q < 2 ? sa.m : sb.m;
        const float p = s[nb][q] == -INFINITY ? 0.0f : expf(s[nb][q] - m);
        s[nb][q] = p;
        if (q < 2) pa += p; else pb += p;
      }
    sa.l += quad_sum(pa);
    sb.l += quad_sum(pb);
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      o[j][0] *= sca; o[j][1] *= sca;
      o[j][2] *= scb; o[j][3] *= scb;
    }
    // O += P V.  k-step kb covers tile columns kb*8 + {2t, 2t+1} for A's
    // k = {t, t+4}: exactly the columns this lane's S accumulator holds.
#pragma unroll
    for (int kb = 0; kb < 2; ++kb) {
      uint32_t p0[4], p1[4];
      split_s<PREC>(s[kb][0], p0[0], p1[0]);  // (g,   2t)   -> a0
      split_s<PREC>(s[kb][2], p0[1], p1[1]);  // (g+8, 2t)   -> a1
      split_s<PREC>(s[kb][1], p0[2], p1[2]);  // (g,   2t+1) -> a2
      split_s<PREC>(s[kb][3], p0[3], p1[3]);  // (g+8, 2t+1) -> a3
      const uint32_t c0 = tile * 16u + kb * 8u + 2u * t, c1 = c0 + 1u;
      const bool ok0 = c0 < ucnt, ok1 = c1 < ucnt;
      const uint32_t col0 = ok0 ? __ldg(G.wuc + ubase + c0) : 0u;
      const uint32_t col1 = ok1 ? __ldg(G.wuc + ubase + c1) : 0u;
      float v0[NB], v1[NB];
      load_row_seg<NB, VEC>(v0, h, ldh, col0, g * NB, d, ok0);
      load_row_seg<NB, VEC>(v1, h, ldh, col1, g * NB, d, ok1);
#pragma unroll
      for (int j = 0; j < NB; ++j) {
        uint32_t x0, x1, x2, y0, y1, y2;
        split_d<PREC>(v0[j], x0, x1, x2);
        split_d<PREC>(v1[j], y0, y1, y2);
        if constexpr (PREC == SGTK_FP32) {
          mma_tf32(o[j], p0[0], p0[1], p0[2], p0[3], x2, y2);
          mma_tf32(o[j], p1[0], p1[1], p1[2], p1[3], x0, y0);
          mma_tf32(o[j], p0[0], p0[1], p0[2], p0[3], x1, y1);
        }
        mma_tf32(o[j], p0[0], p0[1], p0[2], p0[3], x0, y0);
      }
    }
  }

  // ---------------- CUDA-core path: edges of tiles [tc_end, t1) -----------
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
        const float ic = act ? __ldg(inv + col) : 0.0f;
        // dot(z_row, z_col) over this lane's Q features, reduced over the quad
        float k0[NB], k1[NB];
        load_row_seg<NB, VEC>(k0, h, ldh, col, t * NB, d, act);
        load_row_seg<NB, VEC>(k1, h, ldh, col, (t + 4) * NB, d, act);
        float part = 0.0f;
#pragma unroll
        for (int s_ = 0; s_ < NB; ++s_) {
          const int qa = half ? 1 : 0;
          const float z0 = __uint_as_float(q0[qa][s_]) + __uint_as_float(q1[qa][s_]) +
                           __uint_as_float(q2[qa][s_]);
          const float z1 = __uint_as_float(q0[qa + 2][s_]) + __uint_as_float(q1[qa + 2][s_]) +
                           __uint_as_float(q2[qa + 2][s_]);
          float y0 = k0[s_] * ic, y1 = k1[s_] * ic;
          if constexpr (PREC == SGTK_TF32) { y0 = tf32_rne(y0); y1 = tf32_rne(y1); }
          part = fmaf(z0, y0, part);
          part = fmaf(z1, y1, part);
        }
        float logit = quad_sum(part);
        if constexpr (PREC == SGTK_TF32) logit = tf32_rne(logit);
        logit = act ? logit * beta : -INFINITY;
        RowState& st = half ? sb : sa;
        float sc;
        online_update(st, logit, sc);
        const float p = act ? expf(logit - st.m) : 0.0f;
        st.l += p;
        float vs[2 * NB];
        const int64_t rem = int64_t(d) - int64_t(2u * t * NB);
        const int valid = !act || rem <= 0 ? 0 : (rem > 2 * NB ? 2 * NB : int(rem));
        load_seg<2 * NB, VEC>(vs, h + uint64_t(col) * ldh + 2u * t * NB, valid);
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
    const float la = sa.l > 0.0f ? 1.0f / sa.l : 0.0f, lb = sb.l > 0.0f ? 1.0f / sb.l : 0.0f;
    float va_[2 * NB], vb_[2 * NB];
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      va_[j] = o[j][0] * la; va_[NB + j] = o[j][1] * la;
      vb_[j] = o[j][2] * lb; vb_[NB + j] = o[j][3] * lb;
    }
    if (va) store_seg<2 * NB, VEC>(out + ra * ldo + sf, va_, svalid);
    if (vb) store_seg<2 * NB, VEC>(out + rb * ldo + sf, vb_, svalid);
  } else {
    // partial state: O[16][8*NB], then m[16], l[16]
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
                                  float* __restrict__ out, uint64_t ldo) {
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
      const float sc = expf(m - M);
      L += P[16 * 8 * NB + 16 + rr] * sc;
      O += P[rr * 8 * NB + f] * sc;
    }
    out[r * ldo + f] = L > 0.0f ? O * (1.0f / L) : 0.0f;
  }
}

template <int NB, int PREC, bool VEC>
void launch(const sgtk_graph* g, const uint32_t* thr, const float* h, uint64_t ldh, uint64_t d,
            const float* inv, float beta, float* out, uint64_t ldo, cudaStream_t s) {
  const auto& P = g->plan16;
  const uint64_t pstride = 16 * 8 * NB + 32;
  float* partial = nullptr;
  if (P.n_slots)
    CU(cudaMallocAsync(reinterpret_cast<void**>(&partial), uint64_t(P.n_slots) * pstride * 4, s));
  agnn_fused_kernel<NB, PREC, VEC><<<(P.n_units + kWarps - 1) / kWarps, kWarps * 32, 0, s>>>(
      g->view(), P.units->as<WorkUnit>(), P.n_units, thr, h, ldh, d, inv, beta, out, ldo, partial,
      pstride);
  CU_LAUNCH("agnn_fused_kernel");
  if (P.n_reduce) {
    agnn_merge_kernel<NB><<<P.n_reduce, 256, 0, s>>>(P.reduce->as<ReduceItem>(), g->n_rows,
                                                     partial, pstride, d, out, ldo);
    CU_LAUNCH("agnn_merge_kernel");
  }
  if (partial) CU(cudaFreeAsync(partial, s));
}

template <int NB>
void dispatch(int prec, bool vec, const sgtk_graph* g, const uint32_t* thr, const float* h,
              uint64_t ldh, uint64_t d, const float* inv, float beta, float* out, uint64_t ldo,
              cudaStream_t s) {
  if (prec == SGTK_FP32) {
    if (vec) launch<NB, SGTK_FP32, true>(g, thr, h, ldh, d, inv, beta, out, ldo, s);
    else launch<NB, SGTK_FP32, false>(g, thr, h, ldh, d, inv, beta, out, ldo, s);
  } else {
    if (vec) launch<NB, SGTK_TF32, true>(g, thr, h, ldh, d, inv, beta, out, ldo, s);
    else launch<NB, SGTK_TF32, false>(g, thr, h, ldh, d, inv, beta, out, ldo, s);
  }
}

}  // namespace

void agnn_fused_launch(const sgtk_graph* g, const float* h, uint64_t ldh, uint64_t d,
                       const float* inv, float beta, int prec, const uint32_t* cut_dev,
                       float* out, uint64_t ldo, cudaStream_t s) {
  if (prec != SGTK_FP32 && prec != SGTK_TF32)
    raise(SGTK_ERR_RANGE, "agnn_forward: precision must be FP32 or TF32");
  if (d > 64) raise(SGTK_ERR_SHAPE, "agnn_forward: fused mode supports d <= 64 (use mode 0)");
  if (g->n_rows == 0 || d == 0) return;
  DevBuf cut_keep;
  const uint32_t* thr = internal_cut(g, cut_dev, 16, s, cut_keep);
  const int nb = d <= 16 ? 2 : d <= 32 ? 4 : 8;
  const bool vec = ldh % 4 == 0 && ldo % 4 == 0 && reinterpret_cast<uintptr_t>(h) % 16 == 0 &&
                   reinterpret_cast<uintptr_t>(out) % 16 == 0;
  if (nb == 2) dispatch<2>(prec, vec, g, thr, h, ldh, d, inv, beta, out, ldo, s);
  else if (nb == 4) dispatch<4>(prec, vec, g, thr, h, ldh, d, inv, beta, out, ldo, s);
  else dispatch<8>(prec, vec, g, thr, h, ldh, d, inv, beta, out, ldo, s);
}

}  // namespace sgtkcu
