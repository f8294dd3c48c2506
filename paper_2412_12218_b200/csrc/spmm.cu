// GCN aggregation: hybrid tiled SpMM on sm_100a.
//
// Replaces spmm_hybrid (/root/reference/proj/src/tile_exec.cpp:200-314):
//   out = A * x, rows of A from the SGT windows.  Per 16-row window, the
//   8-wide condensed tiles below the plan's cut run on the tensor cores
//   (mma.sync m16n8k8 TF32, fp32 accumulate; FP32 precision = 4-term TF32 split),
//   the remaining edges of each row run edge-by-edge on the CUDA cores
//   (tile_exec.cpp:291-303) — in the same warp, into the same accumulators.
//
// Data each warp touches (no shared memory; everything lands in registers):
//   * the tile's 16-byte occupancy bitmap (byte r = row r, bit c = column c);
//   * the tile's 8 unique column ids (window_unique_cols);
//   * A values in CSR order, located by per-row cursors that advance by the
//     row's popcount (the reference's cursor walk, tile_exec.cpp:329-386);
//   * the 8 gathered feature rows, as B fragments, with 128-bit loads.
// Feature layout trick: n-block j, B column n=g maps to feature
// fbase + g*NB + j, so a lane's B fragment is NB *contiguous* floats of one
// row (vector load), and its C fragment for row g covers the contiguous
// features [fbase + 2t*NB, fbase + 2t*NB + 2*NB) (vector store).
//
// Windows too large for one warp-task are split into work units whose
// partials are reduced in unit order (deterministic; no float atomics).

#include "kernels.cuh"

namespace sgtkcu {
namespace {

constexpr int kWarpsPerBlock = 4;

__device__ __forceinline__ uint32_t byte_of(const uint4& b, uint32_t r) {
  const uint32_t w = r < 8 ? (r < 4 ? b.x : b.y) : (r < 12 ? b.z : b.w);
  return (w >> ((r & 3u) * 8)) & 0xFFu;
}

template <bool VALS>
__device__ __forceinline__ float a_at(const float* __restrict__ vals, uint32_t bits, uint32_t c,
                                      uint64_t cur) {
  if (!((bits >> c) & 1u)) return 0.0f;
  if constexpr (VALS) return __ldg(vals + cur + __popc(bits & ((1u << c) - 1u)));
  return 1.0f;
}

template <int DC, int PREC, bool VEC, bool VALS>
__global__ void __launch_bounds__(kWarpsPerBlock * 32)
spmm_kernel(const DevGraph G, const WorkUnit* __restrict__ units, uint32_t n_units,
            const uint32_t* __restrict__ thr, const float* __restrict__ vals,
            const float* __restrict__ x, uint64_t ldx, uint64_t d, float* __restrict__ out,
            uint64_t ldo, float* __restrict__ partial, uint64_t dpad,
            uint32_t* __restrict__ nonfinite) {
  constexpr int NB = DC / 8;
  const uint32_t wid = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (wid >= n_units) return;
  const WorkUnit u = units[wid];
  const uint64_t fbase = uint64_t(blockIdx.y) * DC;
  const uint32_t lane = lane_id(), g = lane >> 2, t = lane & 3u;
  const uint64_t w = u.window;
  const uint64_t ra = w * 16 + g, rb = ra + 8;
  const bool va = ra < G.n_rows, vb = rb < G.n_rows;
  const uint64_t ubase = G.wo[w];
  const uint32_t ucnt = uint32_t(G.wo[w + 1] - ubase);
  const uint32_t ntiles = (ucnt + 7u) >> 3;
  const uint64_t tbase = G.toff8[w];
  const uint32_t tc_end = thr ? min(u.t1, max(u.t0, thr[w])) : u.t1;

  // Row cursors: first edge of the row inside this unit (CSR order).
  uint64_t ca = va ? G.np[ra] : 0, ea = va ? G.np[ra + 1] : 0;
  uint64_t cb = vb ? G.np[rb] : 0, eb = vb ? G.np[rb + 1] : 0;
  if (u.t0 > 0) {
    ca = lower_bound_u32(G.e2c, ca, ea, u.t0 * 8u);
    cb = lower_bound_u32(G.e2c, cb, eb, u.t0 * 8u);
  }
  if (u.t1 < ntiles) {
    ea = lower_bound_u32(G.e2c, ca, ea, u.t1 * 8u);
    eb = lower_bound_u32(G.e2c, cb, eb, u.t1 * 8u);
  }

  // acc: round-to-nearest fp32 running sums; part: the tensor-core partial of
  // the current group of kFold tiles.  Tensor-core fp32 accumulation does not
  // round to nearest, so a chain of ~10^3 MMAs on one accumulator (hub
  // windows) drifts; folding every kFold tiles keeps each chain short and the
  // long sum in IEEE FADDs (error ~ the sequential reference's).
  constexpr uint32_t kFold = 4;
  float acc[NB][4], part[NB][4];
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    acc[j][0] = acc[j][1] = acc[j][2] = acc[j][3] = 0.0f;
    part[j][0] = part[j][1] = part[j][2] = part[j][3] = 0.0f;
  }

  const int64_t bv = int64_t(d) - int64_t(fbase + g * NB);
  const int bvalid = bv < 0 ? 0 : (bv > NB ? NB : int(bv));

  // ---------------- tensor-core path: tiles [t0, tc_end) -----------------
  for (uint32_t tile = u.t0; tile < tc_end; ++tile) {
    if ((tile - u.t0) % kFold == 0 && tile != u.t0) {
#pragma unroll
      for (int j = 0; j < NB; ++j)
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          acc[j][q] += part[j][q];
          part[j][q] = 0.0f;
        }
    }
    const uint4 bm = __ldg(G.bm8 + tbase + tile);
    const uint32_t bya = byte_of(bm, g), byb = byte_of(bm, g + 8);
    const uint32_t ct = tile * 8u + t, ct4 = ct + 4u;
    float xb0[NB], xb1[NB];
    if (ct < ucnt) {
      const uint32_t col = __ldg(G.wuc + ubase + ct);
      load_seg<NB, VEC>(xb0, x + uint64_t(col) * ldx + fbase + g * NB, bvalid);
    } else {
#pragma unroll
      for (int j = 0; j < NB; ++j) xb0[j] = 0.0f;
    }
    if (ct4 < ucnt) {
      const uint32_t col = __ldg(G.wuc + ubase + ct4);
      load_seg<NB, VEC>(xb1, x + uint64_t(col) * ldx + fbase + g * NB, bvalid);
    } else {
#pragma unroll
      for (int j = 0; j < NB; ++j) xb1[j] = 0.0f;
    }
    const float a0 = a_at<VALS>(vals, bya, t, ca), a1 = a_at<VALS>(vals, byb, t, cb);
    const float a2 = a_at<VALS>(vals, bya, t + 4, ca), a3 = a_at<VALS>(vals, byb, t + 4, cb);
    ca += __popc(bya);
    cb += __popc(byb);
    uint32_t s0[4], s1[4];
    split_s<PREC>(a0, s0[0], s1[0]);
    split_s<PREC>(a1, s0[1], s1[1]);
    split_s<PREC>(a2, s0[2], s1[2]);
    split_s<PREC>(a3, s0[3], s1[3]);
#pragma unroll
    for (int j = 0; j < NB; ++j) {
      uint32_t p0, p1, p2, q0, q1, q2;  // B rows k=t (p) and k=t+4 (q)
      split_d<PREC>(xb0[j], p0, p1, p2);
      split_d<PREC>(xb1[j], q0, q1, q2);
      if constexpr (PREC == SGTK_FP32) {
        mma_tf32(part[j], s0[0], s0[1], s0[2], s0[3], p2, q2);
        mma_tf32(part[j], s1[0], s1[1], s1[2], s1[3], p0, q0);
        mma_tf32(part[j], s0[0], s0[1], s0[2], s0[3], p1, q1);
      }
      mma_tf32(part[j], s0[0], s0[1], s0[2], s0[3], p0, q0);
    }
  }
#pragma unroll
  for (int j = 0; j < NB; ++j)
#pragma unroll
    for (int q = 0; q < 4; ++q) acc[j][q] += part[j][q];

  // ---------------- CUDA-core path: remaining edges of the unit ----------
  const uint64_t sf = fbase + 2u * t * NB;  // this lane's output feature segment
  const int64_t sv = int64_t(d) - int64_t(sf);
  const int svalid = sv < 0 ? 0 : (sv > 2 * NB ? 2 * NB : int(sv));
  if (ca < ea || cb < eb) {
    for (int half = 0; half < 2; ++half) {
      uint64_t e = half ? cb : ca;
      const uint64_t e_end = half ? eb : ea;
      for (; e < e_end; ++e) {
        const uint32_t col = __ldg(G.el + e);
        float a = VALS ? __ldg(vals + e) : 1.0f;
        float xs[2 * NB];
        load_seg<2 * NB, VEC>(xs, x + uint64_t(col) * ldx + sf, svalid);
        if constexpr (PREC == SGTK_TF32) a = tf32_rne(a);
#pragma unroll
        for (int j = 0; j < NB; ++j) {
          float x0 = xs[j], x1 = xs[NB + j];
          if constexpr (PREC == SGTK_TF32) { x0 = tf32_rne(x0); x1 = tf32_rne(x1); }
          acc[j][2 * half + 0] = fmaf(a, x0, acc[j][2 * half + 0]);
          acc[j][2 * half + 1] = fmaf(a, x1, acc[j][2 * half + 1]);
        }
      }
    }
  }

  // ---------------- epilogue ---------------------------------------------
  float ov[2][2 * NB];
#pragma unroll
  for (int j = 0; j < NB; ++j) {
    ov[0][j] = acc[j][0];
    ov[0][NB + j] = acc[j][1];
    ov[1][j] = acc[j][2];
    ov[1][NB + j] = acc[j][3];
  }
  bool bad = false;
  if (u.slot == kNoSlot) {
    if (va) {
      store_seg<2 * NB, VEC>(out + ra * ldo + sf, ov[0], svalid);
      for (int i = 0; i < 2 * NB; ++i) bad |= i < svalid && !isfinite(ov[0][i]);
    }
    if (vb) {
      store_seg<2 * NB, VEC>(out + rb * ldo + sf, ov[1], svalid);
      for (int i = 0; i < 2 * NB; ++i) bad |= i < svalid && !isfinite(ov[1][i]);
    }
    if (nonfinite && __any_sync(0xFFFFFFFFu, bad) && lane == 0) atomicOr(nonfinite, 1u);
  } else {
    float* p = partial + (uint64_t(u.slot) * 16 + g) * dpad + (sf - 0);
    store_seg<2 * NB, true>(p, ov[0], 2 * NB);
    store_seg<2 * NB, true>(p + 8 * dpad, ov[1], 2 * NB);
  }
}

// Split windows: out rows = sum of the unit partials in unit order.
__global__ void spmm_reduce_kernel(const ReduceItem* __restrict__ items, uint64_t n_rows,
                                   const float* __restrict__ partial, uint64_t dpad, uint64_t d,
                                   float* __restrict__ out, uint64_t ldo,
                                   uint32_t* __restrict__ nonfinite) {
  const ReduceItem it = items[blockIdx.x];
  bool bad = false;
  for (uint64_t i = threadIdx.x; i < 16 * d; i += blockDim.x) {
    const uint64_t rr = i / d, f = i - rr * d;
    const uint64_t r = uint64_t(it.window) * 16 + rr;
    if (r >= n_rows) continue;
    float s = 0.0f;
    for (uint32_t k = 0; k < it.count; ++k)
      s += partial[(uint64_t(it.slot0 + k) * 16 + rr) * dpad + f];
    out[r * ldo + f] = s;
    bad |= !isfinite(s);
  }
  if (nonfinite && bad) atomicOr(nonfinite, 1u);
}

template <int DC, int PREC, bool VEC, bool VALS>
void launch_dc(const sgtk_graph* g, const uint32_t* thr, const float* vals, const float* x,
               uint64_t ldx, uint64_t d, float* out, uint64_t ldo, float* partial, uint64_t dpad,
               uint32_t* nonfinite, cudaStream_t s) {
  const auto& P = g->plan8;
  dim3 grid((P.n_units + kWarpsPerBlock - 1) / kWarpsPerBlock, unsigned((d + DC - 1) / DC));
  spmm_kernel<DC, PREC, VEC, VALS><<<grid, kWarpsPerBlock * 32, 0, s>>>(
      g->view(), P.units->as<WorkUnit>(), P.n_units, thr, vals, x, ldx, d, out, ldo, partial, dpad,
      nonfinite);
  CU_LAUNCH("spmm_kernel");
}

template <int PREC, bool VEC, bool VALS>
void launch_prec(int dc, const sgtk_graph* g, const uint32_t* thr, const float* vals,
                 const float* x, uint64_t ldx, uint64_t d, float* out, uint64_t ldo,
                 float* partial, uint64_t dpad, uint32_t* nonfinite, cudaStream_t s) {
  switch (dc) {
    case 16: return launch_dc<16, PREC, VEC, VALS>(g, thr, vals, x, ldx, d, out, ldo, partial, dpad, nonfinite, s);
    case 32: return launch_dc<32, PREC, VEC, VALS>(g, thr, vals, x, ldx, d, out, ldo, partial, dpad, nonfinite, s);
    default: return launch_dc<64, PREC, VEC, VALS>(g, thr, vals, x, ldx, d, out, ldo, partial, dpad, nonfinite, s);
  }
}

}  // namespace

void spmm_launch(const sgtk_graph* g, const float* x, uint64_t ldx, uint64_t d,
                 const uint32_t* cut_dev, const float* ev, int prec, float* out, uint64_t ldo,
                 uint32_t* nonfinite, cudaStream_t s, bool x_tf32) {
  if (prec != SGTK_FP32 && prec != SGTK_TF32)
    raise(SGTK_ERR_RANGE, "spmm: precision must be FP32 or TF32");
  if (ldx < d || ldo < d) raise(SGTK_ERR_SHAPE, "spmm: leading dimension smaller than width");
  if (g->n_rows == 0 || d == 0) return;
  // default plan (all tiles on the tensor cores): the 128-row panel kernel
  if (!cut_dev && spmm_panel_launch(g, x, ldx, d, ev, prec, out, ldo, nonfinite, s, x_tf32)) return;
  DevBuf cut_keep;
  const uint32_t* thr = internal_cut(g, cut_dev, 8, s, cut_keep);
  const float* vals = ev ? ev : (g->has_values ? g->vals->as<float>() : nullptr);
  const int dc = pick_dc(d);
  const uint64_t dpad = (d + dc - 1) / dc * dc;
  const bool vec = (ldx % 4 == 0) && (ldo % 4 == 0) && (d % 4 == 0) &&
                   (reinterpret_cast<uintptr_t>(x) % 16 == 0) &&
                   (reinterpret_cast<uintptr_t>(out) % 16 == 0);
  float* partial = nullptr;
  const auto& P = g->plan8;
  if (P.n_slots) CU(cudaMallocAsync(reinterpret_cast<void**>(&partial),
                                    uint64_t(P.n_slots) * 16 * dpad * 4, s));
  auto go = [&](auto prec_tag, auto vec_tag, auto vals_tag) {
    launch_prec<decltype(prec_tag)::value, decltype(vec_tag)::value, decltype(vals_tag)::value>(
        dc, g, thr, vals, x, ldx, d, out, ldo, partial, dpad, nonfinite, s);
  };
  using F = std::integral_constant<int, SGTK_FP32>;
  using T = std::integral_constant<int, SGTK_TF32>;
  using Y = std::true_type;
  using N = std::false_type;
  if (prec == SGTK_FP32) {
    if (vec) { if (vals) go(F{}, Y{}, Y{}); else go(F{}, Y{}, N{}); }
    else     { if (vals) go(F{}, N{}, Y{}); else go(F{}, N{}, N{}); }
  } else {
    if (vec) { if (vals) go(T{}, Y{}, Y{}); else go(T{}, Y{}, N{}); }
    else     { if (vals) go(T{}, N{}, Y{}); else go(T{}, N{}, N{}); }
  }
  if (P.n_reduce) {
    spmm_reduce_kernel<<<P.n_reduce, 256, 0, s>>>(P.reduce->as<ReduceItem>(), g->n_rows, partial,
                                                  dpad, d, out, ldo, nonfinite);
    CU_LAUNCH("spmm_reduce_kernel");
  }
  if (partial) CU(cudaFreeAsync(partial, s));
}

}  // namespace sgtkcu
