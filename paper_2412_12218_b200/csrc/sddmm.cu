// Edge features: hybrid tiled SDDMM on sm_100a.
//
// Replaces sddmm_hybrid (/root/reference/proj/src/tile_exec.cpp:316-411):
//   out[e] = a_e * <x[row e], y[col e]>, CSR edge order.
// Per 16-row window the 16-wide condensed tiles (the reference reblocks to 16
// before calling it, gnn.cpp:101-112) are 16x16 blocks of dot products:
// two m16n8k8 TF32 MMAs per 8 features (FP32 precision: 4-term split), with the
// window's x rows held in registers as A fragments and the tile's 16 gathered
// y rows as B fragments.  Only positions that are edges are written: the
// tile's 16x16 occupancy bitmap plus per-row CSR cursors give each edge's
// output index (tile_exec.cpp:379-390).  Tiles at or past the plan's cut are
// dotted edge-by-edge on CUDA cores (tile_exec.cpp:394-408).
//
// Feature layout: k-column k of chunk s maps to feature fb + k*KS + s, so a
// lane's A and B fragments are two contiguous KS-float segments (vector loads).

#include "kernels.cuh"

namespace sgtkcu {
namespace {

constexpr int kWarps = 4;
constexpr int DK = 32;      // features per chunk
constexpr int KS = DK / 8;  // floats per lane segment

__device__ __forceinline__ uint32_t bits16_of(const uint4& lo, const uint4& hi, uint32_t r) {
  const uint4& b = r < 8 ? lo : hi;
  const uint32_t rr = r & 7u;
  const uint32_t w = rr < 4 ? (rr < 2 ? b.x : b.y) : (rr < 6 ? b.z : b.w);
  return (w >> ((rr & 1u) * 16)) & 0xFFFFu;
}

template <int PREC, bool VEC>
struct Frag {
  // [segment: (row a, k=t), (row b, k=t), (row a, t+4), (row b, t+4)]; x = p0 + p1 + p2
  uint32_t p0[4][KS], p1[4][KS], p2[4][KS];
};

template <int PREC, bool VEC>
__device__ __forceinline__ void load_a(Frag<PREC, VEC>& A, const float* __restrict__ x,
                                       uint64_t ldx, uint64_t d, uint64_t ra, uint64_t rb,
                                       bool va, bool vb, uint64_t fb, uint32_t t,
                                       const float* inva, const float* invb) {
  float s[KS];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const bool rowa = (q & 1) == 0;
    const uint64_t r = rowa ? ra : rb;
    const bool ok = rowa ? va : vb;
    const uint64_t f = fb + (q < 2 ? t : t + 4) * KS;
    const int64_t rem = int64_t(d) - int64_t(f);
    const int valid = !ok || rem <= 0 ? 0 : (rem > KS ? KS : int(rem));
    load_seg<KS, VEC>(s, x + r * ldx + f, valid);
#pragma unroll
    for (int i = 0; i < KS; ++i) {
      float v = s[i];
      if (inva) v = v * (rowa ? *inva : *invb);  // z = h * inv_norm (gnn.cpp:85-87)
      split_d<PREC>(v, A.p0[q][i], A.p1[q][i], A.p2[q][i]);
    }
  }
}

template <int PREC, bool VEC>
__global__ void __launch_bounds__(kWarps * 32)
sddmm_kernel(const DevGraph G, const WorkUnit* __restrict__ units, uint32_t n_units,
             const uint32_t* __restrict__ thr, const float* __restrict__ vals,
             const float* __restrict__ x, uint64_t ldx, const float* __restrict__ y,
             uint64_t ldy, uint64_t d, const float* __restrict__ inv_norm, float scale,
             float* __restrict__ out) {
  const uint32_t wid = blockIdx.x * kWarps + (threadIdx.x >> 5);
  if (wid >= n_units) return;
  const WorkUnit u = units[wid];
  const uint32_t lane = lane_id(), g = lane >> 2, t = lane & 3u;
  const uint64_t w = u.window;
  const uint64_t ra = w * 16 + g, rb = ra + 8;
  const bool va = ra < G.n_rows, vb = rb < G.n_rows;
  const uint64_t ubase = G.wo[w];
  const uint32_t ucnt = uint32_t(G.wo[w + 1] - ubase);
  const uint32_t ntiles = (ucnt + 15u) >> 4;
  const uint64_t tbase = G.toff16[w];
  const uint32_t tc_end = thr ? min(u.t1, max(u.t0, thr[w])) : u.t1;
  const uint32_t nch = uint32_t((d + DK - 1) / DK);

  uint64_t ca = va ? G.np[ra] : 0, ea = va ? G.np[ra + 1] : 0;
  uint64_t cb = vb ? G.np[rb] : 0, eb = vb ? G.np[rb + 1] : 0;
  if (u.t0 > 0) {
    ca = lower_bound_u32(G.e2c, ca, ea, u.t0 * 16u);
    cb = lower_bound_u32(G.e2c, cb, eb, u.t0 * 16u);
  }
  if (u.t1 < ntiles) {
    ea = lower_bound_u32(G.e2c, ca, ea, u.t1 * 16u);
    eb = lower_bound_u32(G.e2c, cb, eb, u.t1 * 16u);
  }
  // x rows are global ids (row_offset + local row): a row-slice graph reads
  // the full feature replica.
  const uint64_t xa = G.row_offset + ra, xb = G.row_offset + rb;
  float ia = 0.f, ib = 0.f;
  if (inv_norm) {
    ia = va ? inv_norm[xa] : 0.f;
    ib = vb ? inv_norm[xb] : 0.f;
  }
  const float* pia = inv_norm ? &ia : nullptr;
  const float* pib = inv_norm ? &ib : nullptr;

  Frag<PREC, VEC> A;
  if (nch == 1) load_a(A, x, ldx, d, xa, xb, va, vb, 0, t, pia, pib);

  auto emit = [&](float dot, uint64_t pos) {
    const float a = vals ? __ldg(vals + pos) : 1.0f;
    float v = PREC == SGTK_TF32 ? tf32_rne(a) * tf32_rne(dot) : a * dot;
    out[pos] = v * scale;
  };

  // ---------------- tensor-core path -------------------------------------
  for (uint32_t tile = u.t0; tile < tc_end; ++tile) {
    const uint4 blo = __ldg(G.bm16 + 2 * (tbase + tile));
    const uint4 bhi = __ldg(G.bm16 + 2 * (tbase + tile) + 1);
    const uint32_t wa = bits16_of(blo, bhi, g), wb = bits16_of(blo, bhi, g + 8);
    float acc[2][4] = {{0.f, 0.f, 0.f, 0.f}, {0.f, 0.f, 0.f, 0.f}};
    uint32_t cols[2];
    bool cok[2];
    float ic[2];
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
      const uint32_t c = tile * 16u + nb * 8u + g;
      cok[nb] = c < ucnt;
      cols[nb] = cok[nb] ? __ldg(G.wuc + ubase + c) : 0u;
      ic[nb] = inv_norm && cok[nb] ? __ldg(inv_norm + cols[nb]) : 1.0f;
    }
    for (uint32_t ch = 0; ch < nch; ++ch) {
      const uint64_t fb = uint64_t(ch) * DK;
      if (nch > 1) load_a(A, x, ldx, d, xa, xb, va, vb, fb, t, pia, pib);
#pragma unroll
      for (int nb = 0; nb < 2; ++nb) {
        float s0[KS], s1[KS];
        const int64_t r0 = int64_t(d) - int64_t(fb + t * KS);
        const int64_t r1 = int64_t(d) - int64_t(fb + (t + 4) * KS);
        const int v0 = !cok[nb] || r0 <= 0 ? 0 : (r0 > KS ? KS : int(r0));
        const int v1 = !cok[nb] || r1 <= 0 ? 0 : (r1 > KS ? KS : int(r1));
        const float* yr = y + uint64_t(cols[nb]) * ldy;
        load_seg<KS, VEC>(s0, yr + fb + t * KS, v0);
        load_seg<KS, VEC>(s1, yr + fb + (t + 4) * KS, v1);
#pragma unroll
        for (int i = 0; i < KS; ++i) {
          uint32_t b0, c0, b1, c1;  // y = b + c (rows k=t and k=t+4)
          const float y0 = inv_norm ? s0[i] * ic[nb] : s0[i];
          const float y1 = inv_norm ? s1[i] * ic[nb] : s1[i];
          split_s<PREC>(y0, b0, c0);
          split_s<PREC>(y1, b1, c1);
          if constexpr (PREC == SGTK_FP32) {
            mma_tf32(acc[nb], A.p2[0][i], A.p2[1][i], A.p2[2][i], A.p2[3][i], b0, b1);
            mma_tf32(acc[nb], A.p0[0][i], A.p0[1][i], A.p0[2][i], A.p0[3][i], c0, c1);
            mma_tf32(acc[nb], A.p1[0][i], A.p1[1][i], A.p1[2][i], A.p1[3][i], b0, b1);
          }
          mma_tf32(acc[nb], A.p0[0][i], A.p0[1][i], A.p0[2][i], A.p0[3][i], b0, b1);
        }
      }
    }
    // scatter the edge positions: C(row, col) with col = nb*8 + 2t (+1)
#pragma unroll
    for (int nb = 0; nb < 2; ++nb) {
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const uint32_t c = nb * 8u + 2u * t + (q & 1u);
        const uint32_t bits = q < 2 ? wa : wb;
        if ((bits >> c) & 1u) {
          const uint64_t base = q < 2 ? ca : cb;
          emit(acc[nb][q], base + __popc(bits & ((1u << c) - 1u)));
        }
      }
    }
    ca += __popc(wa);
    cb += __popc(wb);
  }

  // ---------------- CUDA-core path: per-edge dots -------------------------
  // Lane (g, t) owns features {t*KS.., (t+4)*KS..} of every chunk; the four
  // lanes of group g reduce with shuffles.
  uint32_t na = uint32_t(ea - ca), nbb = uint32_t(eb - cb);
  const uint32_t mx = __reduce_max_sync(0xFFFFFFFFu, max(na, nbb));
  for (uint32_t i = 0; i < mx; ++i) {
#pragma unroll
    for (int half = 0; half < 2; ++half) {
      const bool act = half ? i < nbb : i < na;
      const uint64_t e = (half ? cb : ca) + i;
      const uint32_t col = act ? __ldg(G.el + e) : 0u;
      const uint64_t r = half ? xb : xa;
      float part = 0.0f;
      if (act) {
        for (uint32_t ch = 0; ch < nch; ++ch) {
#pragma unroll
          for (int sidx = 0; sidx < 2; ++sidx) {
            const uint64_t f = uint64_t(ch) * DK + (sidx ? t + 4 : t) * KS;
            const int64_t rem = int64_t(d) - int64_t(f);
            const int valid = rem <= 0 ? 0 : (rem > KS ? KS : int(rem));
            float xs[KS], ys[KS];
            load_seg<KS, VEC>(xs, x + r * ldx + f, valid);
            load_seg<KS, VEC>(ys, y + uint64_t(col) * ldy + f, valid);
#pragma unroll
            for (int k = 0; k < KS; ++k) {
              float xv = xs[k], yv = ys[k];
              if (inv_norm) {
                xv = xv * (half ? ib : ia);
                yv = yv * __ldg(inv_norm + col);
              }
              if (PREC == SGTK_TF32) {
                xv = tf32_rne(xv);
                yv = tf32_rne(yv);
              }
              part = fmaf(xv, yv, part);
            }
          }
        }
      }
      part += __shfl_xor_sync(0xFFFFFFFFu, part, 1);
      part += __shfl_xor_sync(0xFFFFFFFFu, part, 2);
      if (act && t == 0) emit(part, e);
    }
  }
}

}  // namespace

void sddmm_launch(const sgtk_graph* g, const float* x, uint64_t ldx, const float* y, uint64_t ldy,
                  uint64_t d, const uint32_t* cut16_dev, const float* ev, bool unit_values,
                  int prec, const float* inv_norm, float scale, float* out, cudaStream_t s) {
  if (prec != SGTK_FP32 && prec != SGTK_TF32)
    raise(SGTK_ERR_RANGE, "sddmm: precision must be FP32 or TF32");
  if (ldx < d || ldy < d) raise(SGTK_ERR_SHAPE, "sddmm: leading dimension smaller than width");
  if (g->nnz == 0) return;
  DevBuf cut_keep;
  const uint32_t* thr = nullptr;
  if (cut16_dev) {
    // cut16 is expressed in the caller's (reblocked) geometry tiles.
    thr = internal_cut(g, cut16_dev, 16, s, cut_keep);
  }
  const float* vals =
      ev ? ev : (unit_values || !g->has_values ? nullptr : g->vals->as<float>());
  // default plan: the 128-row panels (tcgen05 dense columns + CUDA-core
  // sparse edges, sddmm_panel.cu); explicit partial plans keep the
  // reference's 16-row tile split below
  if (!cut16_dev &&
      sddmm_panel_launch(g, x, ldx, y, ldy, d, ev, unit_values, prec, inv_norm, scale, out, s))
    return;
  const bool vec = (ldx % 4 == 0) && (ldy % 4 == 0) && (reinterpret_cast<uintptr_t>(x) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(y) % 16 == 0);
  const auto& P = g->plan16;
  dim3 grid((P.n_units + kWarps - 1) / kWarps);
  auto units = P.units->as<WorkUnit>();
  const DevGraph G = g->view();
  if (prec == SGTK_FP32) {
    if (vec) sddmm_kernel<SGTK_FP32, true><<<grid, kWarps * 32, 0, s>>>(G, units, P.n_units, thr, vals, x, ldx, y, ldy, d, inv_norm, scale, out);
    else     sddmm_kernel<SGTK_FP32, false><<<grid, kWarps * 32, 0, s>>>(G, units, P.n_units, thr, vals, x, ldx, y, ldy, d, inv_norm, scale, out);
  } else {
    if (vec) sddmm_kernel<SGTK_TF32, true><<<grid, kWarps * 32, 0, s>>>(G, units, P.n_units, thr, vals, x, ldx, y, ldy, d, inv_norm, scale, out);
    else     sddmm_kernel<SGTK_TF32, false><<<grid, kWarps * 32, 0, s>>>(G, units, P.n_units, thr, vals, x, ldx, y, ldy, d, inv_norm, scale, out);
  }
  CU_LAUNCH("sddmm_kernel");
}

}  // namespace sgtkcu
