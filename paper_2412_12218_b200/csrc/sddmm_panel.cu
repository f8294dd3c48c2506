// SDDMM on the 128-row panels: dense columns on the 5th-gen tensor cores
// (tcgen05 + TMEM), sparse edges on the CUDA cores.
//
// Replaces sddmm_hybrid (/root/reference/proj/src/tile_exec.cpp:316-411) for
// the default plan: out[e] = a_e * <x[row e], y[col e]> in CSR edge order.
// The reference computes a dense 16 x 16 block of dot products per condensed
// tile and scatters the positions that are edges (:356-391), then runs the
// remaining edges one by one (:394-408).  Here the tile is the panel chunk of
// the SpMM / AGNN panel format (panel.cu): 128 panel rows x 32 dense columns,
// S = X_panel * Y_chunk^T on the tensor cores (M = 128, N = 32, K = d), and
// the edges of the panel's singleton columns go through the CUDA cores.
//
// Dense kernel (sddmm_dense_kernel), one CTA per panel, warp-specialised:
//   warps 0-3  thread per panel row: stage the row of x as the K-major
//              SWIZZLE_128B A operand (TF32: RNE; FP32: hi/lo planes); per
//              chunk read S from TMEM (tcgen05.ld), keep the row's edge
//              columns (the chunk's row mask) and write them to a staging
//              buffer in the chunk's entry order ((row, column) = CSR order,
//              offsets from a scan of the rows' mask popcounts); then all 128
//              threads walk the chunk's entries together: CSR edge id from the
//              panel format (deid), value a_e, coalesced store of out[e];
//   warp 4     TMEM allocator + single-thread tcgen05.mma issuer, S buffers
//              rotating over 4 x 32 TMEM columns;
//   warps 5-6  loaders (even / odd chunks): cp.async gather of the chunk's
//              32 y rows (K-major SWIZZLE_128B B operand, prepared copies of
//              y: rounded / split once per call) and its 128 row masks,
//              completion through cp.async.mbarrier.arrive.noinc; a slot is
//              refilled once its MMA retired and its masks were read.
// Sparse kernel (sddmm_sparse_kernel): warp per row, lane per edge, the
// reference's own k-ascending fp32 dot (separate multiply and add, like its
// no-FMA x86-64 build), so these edges are bit-identical to it in both
// precisions.
//
// Precision: TF32 -> both operands RNE-rounded like tf32_round_value, the
// result tf32(a) * tf32(dot) (tile_exec.cpp:386,402); FP32 -> 3-term TF32
// split (hi*hi + hi*lo + lo*hi, dropped terms < 2^-21 relative per product).

#include <algorithm>

#include "kernels.cuh"
#include "tc05.cuh"

namespace sgtkcu {
namespace {

using namespace tc05;

constexpr int kSdThreads = 224;  // 4 epilogue warps, 1 MMA warp, 2 loader warps

template <int DC, int PREC>
struct SdCfg {
  static constexpr bool F32 = PREC == SGTK_FP32;
  static constexpr int PL = F32 ? 2 : 1;                     // operand planes (hi, lo)
  static constexpr int KB = DC / 32;                         // 128-byte K blocks
  static constexpr int NB = (F32 && DC == 64) ? 4 : 8;       // gather ring
  static constexpr int NS = 4;                               // S buffers (32 TMEM columns)
  static constexpr uint32_t Q_BYTES = kPanelRows * DC * 4;   // A: KB blocks of 16 KB
  static constexpr uint32_t TILE = kChunkCols * 128;         // one K block of a chunk: 4 KB
  static constexpr uint32_t Q_OFF = 1024;
  static constexpr uint32_t Z_OFF = Q_OFF + PL * Q_BYTES;            // [PL][KB][NB] x TILE
  static constexpr uint32_t M_OFF = Z_OFF + PL * KB * NB * TILE;     // [NB] x 512 B masks
  static constexpr uint32_t ST_OFF = M_OFF + NB * kPanelRows * 4;    // [2] x eslot staged dots
  static constexpr int NE = 4;                                       // entry ring
  // dynamic part, sized by the graph's largest chunk (eslot bytes per chunk):
  // 2 stage slots, then NE entry-id slots (+ NE value slots, weighted graphs)
  static uint32_t smem_bytes(uint32_t eslot, bool with_vals) {
    return ST_OFF + 2 * eslot + NE * eslot * (with_vals ? 2u : 1u) + 1024;
  }
  static constexpr uint32_t TMEM_COLS = NS * 32;
};

// K-major SWIZZLE_128B offset of element (row, k) in a tile with `rows` rows.
__device__ __forceinline__ uint32_t sd_kmaj(uint32_t row, uint32_t k, uint32_t rows) {
  return (k >> 5) * rows * 128u + (row >> 3) * 1024u + (row & 7u) * 128u +
         ((((k >> 2) & 7u) ^ (row & 7u)) << 4) + (k & 3u) * 4u;
}

template <int DC, int PREC>
__global__ void __launch_bounds__(kSdThreads, 2)
sddmm_dense_kernel(const PanelView pv, const uint32_t* __restrict__ deid, uint32_t eslot,
                   const float* __restrict__ x, uint64_t ldx, uint64_t d, uint64_t row_offset,
                   const float* __restrict__ inv, const float* __restrict__ yq,
                   const float* __restrict__ yq1, uint64_t ldq, const float* __restrict__ dval,
                   const float* __restrict__ ev, float scale, float* __restrict__ out) {
  using C = SdCfg<DC, PREC>;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bfull = reinterpret_cast<uint64_t*>(smem);  // [NB] gathers + masks landed
  uint64_t* bempty = bfull + C::NB;                     // [NB] MMA of the slot retired
  uint64_t* sfull = bempty + C::NB;                     // [NS] S in TMEM
  uint64_t* sempty = sfull + C::NS;                     // [NS] S read back
  uint64_t* qfull = sempty + C::NS;                     // A operand staged
  uint64_t* efull = qfull + 1;                          // [NE] chunk entries (ids, values) landed
  uint64_t* eempty = efull + C::NE;                     // [NE] entries consumed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(eempty + C::NE);
  uint32_t* wtot = tmem_slot + 4;                       // [2][4] per-warp entry counts
  const uint32_t qb = smem_u32(smem + C::Q_OFF), zb = smem_u32(smem + C::Z_OFF);
  const uint32_t mb = smem_u32(smem + C::M_OFF);
  float* stage = reinterpret_cast<float*>(smem + C::ST_OFF);
  // entry ring: CSR edge ids (and, for weighted graphs, values) of a chunk,
  // bulk-copied ahead so the store loop never waits on a global load
  uint8_t* ering = smem + C::ST_OFF + 2 * eslot;
  const bool has_dval = dval != nullptr;

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t p = blockIdx.x;
  const uint32_t c0 = pv.cptr[p], nch = pv.cptr[p + 1] - c0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NB; ++i) {
      mbar_init(bfull + i, 32);  // one cp.async.mbarrier.arrive.noinc per loader lane
      // the slot (y rows + row masks) is free once the chunk's MMA retired
      // (tcgen05.commit) AND the 4 epilogue warps have read its masks
      mbar_init(bempty + i, 5);
    }
    for (int i = 0; i < C::NS; ++i) {
      mbar_init(sfull + i, 1);
      mbar_init(sempty + i, 4);
    }
    mbar_init(qfull, 4);
    for (int i = 0; i < C::NE; ++i) {
      mbar_init(efull + i, 1);   // the loader's expect_tx arrival + the bulk bytes
      mbar_init(eempty + i, 4);  // one arrival per epilogue warp
    }
    mbar_init_fence();
  }
  if (warp == 4) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // ---------------------------------------------------------- epilogue
    const uint32_t r = warp * 32 + lane;
    const uint64_t grow = p * kPanelRows + r;
    {  // A = x[panel rows] (z = x * inv when normalising on the fly)
      const bool rv = grow < pv.n_rows;
      const float* src = x + (row_offset + grow) * ldx;
      const float sc = (rv && inv) ? inv[row_offset + grow] : 1.0f;
#pragma unroll
      for (int j = 0; j < DC / 4; ++j) {
        float v[4];
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint64_t f = 4 * j + i;
          float t = (rv && f < d) ? __ldg(src + f) : 0.0f;
          v[i] = inv ? t * sc : t;
        }
        const uint32_t o = sd_kmaj(r, 4 * j, kPanelRows);
        if constexpr (C::F32) {
          uint32_t a0[4], a1[4];
#pragma unroll
          for (int i = 0; i < 4; ++i) split2(v[i], a0[i], a1[i]);
          st_shared_v4(qb + o, a0[0], a0[1], a0[2], a0[3]);
          st_shared_v4(qb + C::Q_BYTES + o, a1[0], a1[1], a1[2], a1[3]);
        } else {
          st_shared_v4(qb + o, tf32_op(v[0]), tf32_op(v[1]), tf32_op(v[2]), tf32_op(v[3]));
        }
      }
      fence_async_smem();
      __syncwarp();
      if (lane == 0) mbar_arrive(qfull);
    }
    for (uint32_t c = 0; c < nch; ++c) {
      const uint32_t ds = c % C::NB, b = c % C::NS, par = c & 1u;
      mbar_wait(bfull + ds, (c / C::NB) & 1u);
      const uint32_t m = ld_shared_u32(mb + ds * kPanelRows * 4 + r * 4);
      __syncwarp();
      if (lane == 0) mbar_arrive(bempty + ds);
      mbar_wait(sfull + b, (c / C::NS) & 1u);
      tc_fence_after();
      uint32_t sv[32];
      tmem_ld16(tmem + ((warp * 32u) << 16) + b * 32, *reinterpret_cast<uint32_t(*)[16]>(sv));
      tmem_ld16(tmem + ((warp * 32u) << 16) + b * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(sv + 16));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(sempty + b);
      // entry offset of this row inside the chunk: scan of the rows' popcounts
      const uint32_t cnt = __popc(m);
      uint32_t incl = cnt;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t t = __shfl_up_sync(0xFFFFFFFFu, incl, o);
        if (lane >= uint32_t(o)) incl += t;
      }
      if (lane == 31) wtot[par * 4 + warp] = incl;
      named_bar(1, 128);
      uint32_t k = incl - cnt, tot = 0;
#pragma unroll
      for (uint32_t w = 0; w < 4; ++w) {
        const uint32_t t = wtot[par * 4 + w];
        k += w < warp ? t : 0u;
        tot += t;
      }
      float* st = stage + par * (eslot / 4);
#pragma unroll
      for (int j = 0; j < 32; ++j)
        if (m & (1u << j)) st[k++] = __uint_as_float(sv[j]);
      named_bar(1, 128);
      // the chunk's edges, all 128 threads: CSR id, value, coalesced store
      const uint32_t de = c % C::NE;
      mbar_wait(efull + de, (c / C::NE) & 1u);
      const uint32_t* eid = reinterpret_cast<const uint32_t*>(ering + de * eslot);
      const float* evl = reinterpret_cast<const float*>(ering + (C::NE + de) * eslot);
      for (uint32_t i = r; i < tot; i += 128) {
        const uint32_t e = eid[i];
        const float dot = st[i];
        const float a = ev ? __ldg(ev + e) : (has_dval ? evl[i] : 1.0f);
        const float v = PREC == SGTK_TF32 ? tf32_rne(a) * tf32_rne(dot) : a * dot;
        out[e] = v * scale;
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(eempty + de);
    }
  } else if (warp == 4) {
    // ---------------------------------------------------------- MMA issuer
    if (lane == 0) {
      constexpr uint32_t id_s = idesc_tf32(kChunkCols, false);
      mbar_wait(qfull, 0);
      tc_fence_after();
      for (uint32_t c = 0; c < nch; ++c) {
        const uint32_t ds = c % C::NB, b = c % C::NS;
        if (c >= uint32_t(C::NS)) mbar_wait(sempty + b, ((c / C::NS) - 1u) & 1u);
        mbar_wait(bfull + ds, (c / C::NB) & 1u);
        fence_async_smem();  // cp.async (generic proxy) -> MMA (async proxy)
        tc_fence_after();
        const uint32_t dt = tmem + b * 32;
#pragma unroll
        for (uint32_t ks = 0; ks < DC / 8; ++ks) {
          const uint32_t ko = (ks >> 2) * (kPanelRows * 128u) + (ks & 3u) * 32u;
          const uint32_t kz = ((ks >> 2) * C::NB + ds) * C::TILE + (ks & 3u) * 32u;
          const uint64_t q0 = umma_desc(qb + ko), z0 = umma_desc(zb + kz);
          if constexpr (C::F32) {
            umma_tf32(dt, q0, umma_desc(zb + C::KB * C::NB * C::TILE + kz), id_s, ks ? 1u : 0u);
            umma_tf32(dt, umma_desc(qb + C::Q_BYTES + ko), z0, id_s, 1u);
            umma_tf32(dt, q0, z0, id_s, 1u);
          } else {
            umma_tf32(dt, q0, z0, id_s, ks ? 1u : 0u);
          }
        }
        umma_commit(sfull + b);
        umma_commit(bempty + ds);
      }
    }
  } else {
    // ---------------------------------------------------------- loaders
    const uint32_t par = warp - 5;
    constexpr uint32_t LPR = DC / 4, RPI = 32 / LPR;  // 16-byte pieces per row, rows per pass
    const uint32_t j = lane % LPR, jj = j & 7u;
    for (uint32_t c = par; c < nch; c += 2) {
      const uint32_t ds = c % C::NB;
      const uint32_t col = pv.dcols[uint64_t(c0 + c) * kChunkCols + lane];
      mbar_wait(bempty + ds, ((c / C::NB) & 1u) ^ 1u);
#pragma unroll
      for (uint32_t t = 0; t < 32 / RPI; ++t) {
        const uint32_t kr = t * RPI + lane / LPR;  // chunk row (B row)
        const uint32_t ck = __shfl_sync(0xFFFFFFFFu, col, kr);
        // padding columns (~0u) are never an edge: their S columns are not
        // read, so their B rows are simply left as they are
        if (ck == 0xFFFFFFFFu) continue;
        const uint64_t gofs = uint64_t(ck) * ldq + 4 * j;
        const uint32_t zo = ((j >> 3) * C::NB + ds) * C::TILE + (kr >> 3) * 1024u + (kr & 7u) * 128u +
                            ((jj ^ (kr & 7u)) << 4);
        cp_async16(zb + zo, yq + gofs);
        if constexpr (C::F32) cp_async16(zb + C::KB * C::NB * C::TILE + zo, yq1 + gofs);
      }
      cp_async16(mb + ds * kPanelRows * 4 + lane * 16, pv.dmask + uint64_t(c0 + c) * kPanelRows + lane * 4);
      cp_async_arrive_noinc(bfull + ds);
      // the chunk's entries (ids, values) by the TMA engine: a slot is reused
      // once the epilogue's store loop of chunk c - NE is done with it
      const uint32_t de = c % C::NE;
      mbar_wait(eempty + de, ((c / C::NE) & 1u) ^ 1u);
      if (lane == 0) {
        const uint64_t k0 = pv.coff[c0 + c], k1 = pv.coff[c0 + c + 1];
        const uint32_t bytes = uint32_t(k1 - k0) * 4u;  // entries padded to 4: 16-byte multiple
        mbar_expect_tx(efull + de, bytes * (has_dval ? 2u : 1u));
        if (bytes) {
          bulk_load(ering + de * eslot, deid + k0, bytes, efull + de);
          if (has_dval) bulk_load(ering + (C::NE + de) * eslot, dval + k0, bytes, efull + de);
        }
      }
    }
    cp_async_wait<0>();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 4) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// y operand copies for the gathers: rows of ldq (32 / 64) floats, zero
// padding features, z = y * inv when normalising on the fly; TF32 -> RNE,
// FP32 -> hi / lo split.
template <int PREC>
__global__ void sddmm_yprep_kernel(const float* __restrict__ y, uint64_t ldy, uint64_t rows,
                                   uint64_t d, const float* __restrict__ inv, uint64_t ldq,
                                   float* __restrict__ yq, float* __restrict__ yq1) {
  const uint64_t n = rows * ldq;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = i / ldq, f = i - r * ldq;
    float v = f < d ? y[r * ldy + f] : 0.0f;
    if (inv) v = v * inv[r];
    if constexpr (PREC == SGTK_FP32) {
      uint32_t a, b;
      split2(v, a, b);
      yq[i] = __uint_as_float(a);
      yq1[i] = __uint_as_float(b);
    } else {
      yq[i] = __uint_as_float(tf32_op(v));
    }
  }
}

// Sparse edges: warp per row (its x row staged in shared memory, read as a
// broadcast), lane per edge, the reference's scalar dot (tile_exec.cpp:394-408).
constexpr int kSpWarps = 8;
template <int PREC, bool VEC>
__global__ void __launch_bounds__(kSpWarps * 32)
sddmm_sparse_kernel(uint64_t n_rows, const uint32_t* __restrict__ sptr, const uint2* __restrict__ sent,
                    const uint32_t* __restrict__ seid, const float* __restrict__ x, uint64_t ldx,
                    const float* __restrict__ y, uint64_t ldy, uint64_t d, uint64_t row_offset,
                    const float* __restrict__ inv, const float* __restrict__ vals, float scale,
                    float* __restrict__ out) {
  __shared__ float xs_all[kSpWarps][64];
  const uint32_t wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  float* xs = xs_all[wib];
  const uint64_t nw = uint64_t(gridDim.x) * kSpWarps;
  for (uint64_t r = uint64_t(blockIdx.x) * kSpWarps + wib; r < n_rows; r += nw) {
    const uint32_t s0 = sptr[r], s1 = sptr[r + 1];
    if (s0 == s1) continue;
    const uint64_t xr = row_offset + r;
    const float ir = inv ? inv[xr] : 1.0f;
    for (uint32_t f = lane; f < d; f += 32) {
      float v = x[xr * ldx + f];
      if (inv) v = v * ir;
      xs[f] = PREC == SGTK_TF32 ? tf32_rne(v) : v;
    }
    __syncwarp();
    for (uint32_t k = s0 + lane; k < s1; k += 32) {
      const uint32_t col = sent[k].x, e = seid[k];
      const float* yr = y + uint64_t(col) * ldy;
      const float ic = inv ? inv[col] : 1.0f;
      float dot = 0.0f;
      uint32_t f = 0;
      if constexpr (VEC) {
        for (; f + 4 <= d; f += 4) {
          const float4 q = __ldg(reinterpret_cast<const float4*>(yr + f));
          const float yv[4] = {q.x, q.y, q.z, q.w};
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            float v = inv ? yv[i] * ic : yv[i];
            if (PREC == SGTK_TF32) v = tf32_rne(v);
            dot = __fadd_rn(dot, __fmul_rn(xs[f + i], v));
          }
        }
      }
      for (; f < d; ++f) {
        float v = inv ? __ldg(yr + f) * ic : __ldg(yr + f);
        if (PREC == SGTK_TF32) v = tf32_rne(v);
        dot = __fadd_rn(dot, __fmul_rn(xs[f], v));
      }
      const float a = vals ? __ldg(vals + e) : 1.0f;
      const float o = PREC == SGTK_TF32 ? tf32_rne(a) * tf32_rne(dot) : a * dot;
      out[e] = o * scale;
    }
    __syncwarp();  // xs is rewritten for the warp's next row
  }
}

template <int DC, int PREC>
bool launch_sd_dense(const PanelView& v, uint64_t P, uint32_t max_entries, const uint32_t* deid,
                     const float* x, uint64_t ldx, uint64_t d, uint64_t ro, const float* inv,
                     const float* yq, const float* yq1, uint64_t ldq, const float* dval,
                     const float* ev, float scale, float* out, cudaStream_t s) {
  using C = SdCfg<DC, PREC>;
  const uint32_t eslot = (max_entries + 3) / 4 * 16;
  const uint32_t smem = C::smem_bytes(eslot, dval != nullptr);
  if (smem > 227u * 1024u) return false;
  once_per_device(reinterpret_cast<const void*>(&sddmm_dense_kernel<DC, PREC>), [] {
    cudaFuncSetAttribute(sddmm_dense_kernel<DC, PREC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(227u * 1024u));
  });
  sddmm_dense_kernel<DC, PREC><<<unsigned(P), kSdThreads, smem, s>>>(
      v, deid, eslot, x, ldx, d, ro, inv, yq, yq1, ldq, dval, ev, scale, out);
  CU_LAUNCH("sddmm_dense_kernel");
  return true;
}

inline unsigned sd_grid(uint64_t n, unsigned block, unsigned cap = 148u * 32u) {
  const uint64_t g = (n + block - 1) / block;
  return unsigned(std::max<uint64_t>(1, std::min<uint64_t>(g, cap)));
}

}  // namespace

// Returns false (the caller runs the 16-row tile kernel) outside this path's
// envelope: no panel format, d > 64.
bool sddmm_panel_launch(const sgtk_graph* g, const float* x, uint64_t ldx, const float* y,
                        uint64_t ldy, uint64_t d, const float* ev, bool unit_values, int prec,
                        const float* inv_norm, float scale, float* out, cudaStream_t s) {
  if (!g->panels || !panel_enabled() || d == 0 || d > 64 || g->n_cols > 0x7FFFFFFFull) return false;
  if (g->n_rows == 0 || g->nnz == 0) return true;
  const Panels& pn = panels_for(g, d);
  PanelView v = panel_view(g, d);
  // a_e: the override (CSR order), else the graph's values (entry order for
  // the dense part: the panel format's dval; CSR order for the sparse part)
  const bool graph_vals = !ev && !unit_values && g->has_values;
  const float* vals = ev ? ev : (graph_vals ? g->vals->as<float>() : nullptr);
  const float* dval = graph_vals ? pn.dval->as<float>() : nullptr;
  {  // shared memory for the largest chunk's entry slots
    const uint32_t eslot = (pn.max_chunk_entries + 3) / 4 * 16;
    const uint32_t need = d <= 32 ? (prec == SGTK_FP32 ? SdCfg<32, SGTK_FP32>::smem_bytes(eslot, dval)
                                                       : SdCfg<32, SGTK_TF32>::smem_bytes(eslot, dval))
                                  : (prec == SGTK_FP32 ? SdCfg<64, SGTK_FP32>::smem_bytes(eslot, dval)
                                                       : SdCfg<64, SGTK_TF32>::smem_bytes(eslot, dval));
    if (need > 227u * 1024u) return false;
  }
  const uint64_t ldq = d <= 32 ? 32 : 64;
  const uint64_t plane = std::max<uint64_t>(g->n_cols * ldq, 4) * 4;
  char* buf = nullptr;
  if (pn.n_chunks) {
    CU(cudaMallocAsync(reinterpret_cast<void**>(&buf), 2 * plane, s));
    float* yq = reinterpret_cast<float*>(buf);
    float* yq1 = reinterpret_cast<float*>(buf + plane);
    const unsigned gb = sd_grid(g->n_cols * ldq, 256);
    if (prec == SGTK_FP32) sddmm_yprep_kernel<SGTK_FP32><<<gb, 256, 0, s>>>(y, ldy, g->n_cols, d, inv_norm, ldq, yq, yq1);
    else sddmm_yprep_kernel<SGTK_TF32><<<gb, 256, 0, s>>>(y, ldy, g->n_cols, d, inv_norm, ldq, yq, nullptr);
    CU_LAUNCH("sddmm_yprep_kernel");
    const uint32_t* deid = pn.deid->as<uint32_t>();
    const uint64_t ro = g->row_offset;
    const uint32_t me = pn.max_chunk_entries;
    if (prec == SGTK_FP32) {
      if (ldq == 32) launch_sd_dense<32, SGTK_FP32>(v, pn.P, me, deid, x, ldx, d, ro, inv_norm, yq, yq1, ldq, dval, ev, scale, out, s);
      else launch_sd_dense<64, SGTK_FP32>(v, pn.P, me, deid, x, ldx, d, ro, inv_norm, yq, yq1, ldq, dval, ev, scale, out, s);
    } else {
      if (ldq == 32) launch_sd_dense<32, SGTK_TF32>(v, pn.P, me, deid, x, ldx, d, ro, inv_norm, yq, nullptr, ldq, dval, ev, scale, out, s);
      else launch_sd_dense<64, SGTK_TF32>(v, pn.P, me, deid, x, ldx, d, ro, inv_norm, yq, nullptr, ldq, dval, ev, scale, out, s);
    }
  }
  if (pn.n_sparse) {
    const bool vec = ldy % 4 == 0 && reinterpret_cast<uintptr_t>(y) % 16 == 0;
    const unsigned gs = sd_grid(g->n_rows, kSpWarps, 148u * 16u);
    const auto* sp = pn.sptr->as<uint32_t>();
    const auto* se = pn.sent->as<uint2>();
    const auto* si = pn.seid->as<uint32_t>();
    const uint64_t ro = g->row_offset;
    if (prec == SGTK_FP32) {
      if (vec) sddmm_sparse_kernel<SGTK_FP32, true><<<gs, kSpWarps * 32, 0, s>>>(g->n_rows, sp, se, si, x, ldx, y, ldy, d, ro, inv_norm, vals, scale, out);
      else sddmm_sparse_kernel<SGTK_FP32, false><<<gs, kSpWarps * 32, 0, s>>>(g->n_rows, sp, se, si, x, ldx, y, ldy, d, ro, inv_norm, vals, scale, out);
    } else {
      if (vec) sddmm_sparse_kernel<SGTK_TF32, true><<<gs, kSpWarps * 32, 0, s>>>(g->n_rows, sp, se, si, x, ldx, y, ldy, d, ro, inv_norm, vals, scale, out);
      else sddmm_sparse_kernel<SGTK_TF32, false><<<gs, kSpWarps * 32, 0, s>>>(g->n_rows, sp, se, si, x, ldx, y, ldy, d, ro, inv_norm, vals, scale, out);
    }
    CU_LAUNCH("sddmm_sparse_kernel");
  }
  if (buf) CU(cudaFreeAsync(buf, s));
  return true;
}

}  // namespace sgtkcu
