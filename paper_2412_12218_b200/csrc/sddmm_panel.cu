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
//   warps 0-3  stage warps, thread per panel row: stage the row of x as the
//              K-major SWIZZLE_128B A operand (TF32: RNE; FP32: hi/lo planes);
//              per chunk read the row's 32 dots from TMEM (tcgen05.ld) and
//              write those at the row's edge columns (the chunk's row mask)
//              into a staging slot in the chunk's entry order ((row, column)
//              = CSR order; the row's offset comes with the format);
//   warps 4-7  store warps: walk the chunk's entries together -- CSR edge
//              id and value from the entry ring (bulk-copied ahead by the
//              TMA engine), a_e * dot, coalesced store of out[e];
//   warp 8     TMEM allocator + single-thread tcgen05.mma issuer, S buffers
//              rotating over 4 x 32 TMEM columns;
//   warps 9-10 loaders (even / odd chunks): cp.async gather of the chunk's
//              32 y rows (K-major SWIZZLE_128B B operand, prepared copies of
//              y: rounded / split once per call), its row masks and offsets,
//              and the bulk copy of its entries.
// Every hand-off is an mbarrier (no CTA-wide barrier inside the chunk loop).
// Sparse kernel (sddmm_sparse_kernel): warp per row, 8 (d <= 32) or 16
// lanes per edge on float4 slices, coalesced row reads, the slices' partial
// dots reduced by a fixed xor tree (deterministic).
//
// Precision: TF32 -> both operands RNE-rounded like tf32_round_value, the
// result tf32(a) * tf32(dot) (tile_exec.cpp:386,402); FP32 -> 3-term TF32
// split (hi*hi + hi*lo + lo*hi, dropped terms < 2^-21 relative per product).

#include <algorithm>
#include <cstdlib>
#include <string>

#include "kernels.cuh"
#include "tc05.cuh"

namespace sgtkcu {
namespace {

using namespace tc05;

constexpr int kSdThreads = 352;  // 4 stage warps, 4 store warps, 1 MMA warp, 2 loader warps
constexpr uint32_t kMSlot = kPanelRows * 4 + kPanelRows * 2;  // row masks + row entry offsets

template <int DC, int PREC>
struct SdCfg {
  static constexpr bool F32 = PREC == SGTK_FP32;
  static constexpr int PL = F32 ? 2 : 1;                     // operand planes (hi, lo)
  static constexpr int KB = DC / 32;                         // 128-byte K blocks
  static constexpr int NB = (F32 && DC == 64) ? 4 : 6;       // gather ring (2 CTAs/SM at TF32, d <= 32)
  static constexpr int NS = 4;                               // S buffers (32 TMEM columns)
  static constexpr int NST = 3;                              // staged-dot slots
  static constexpr int NE = 4;                               // entry ring
  static constexpr uint32_t Q_BYTES = kPanelRows * DC * 4;   // A: KB blocks of 16 KB
  static constexpr uint32_t TILE = kChunkCols * 128;         // one K block of a chunk: 4 KB
  static constexpr uint32_t Q_OFF = 1024;
  static constexpr uint32_t Z_OFF = Q_OFF + PL * Q_BYTES;            // [PL][KB][NB] x TILE
  static constexpr uint32_t M_OFF = Z_OFF + PL * KB * NB * TILE;     // [NB] x (masks, offsets)
  static constexpr uint32_t R_OFF = M_OFF + NB * kMSlot;             // [128] x 36 floats: row dots
  static constexpr uint32_t ST_OFF = R_OFF + kPanelRows * 36 * 4;     // dynamic part from here
  // dynamic part, sized by the graph's largest chunk (eslot bytes per chunk):
  // NST staged-dot slots, NE entry-id slots (+ NE value slots, weighted graphs)
  static uint32_t smem_bytes(uint32_t eslot, bool with_vals) {
    return ST_OFF + NST * eslot + NE * eslot * (with_vals ? 2u : 1u) + 1024;
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
sddmm_dense_kernel(const PanelView pv, const uint32_t* __restrict__ deid,
                   const uint16_t* __restrict__ rowoff, uint32_t eslot,
                   const float* __restrict__ x, uint64_t ldx, uint64_t d, uint64_t row_offset,
                   const float* __restrict__ inv, const float* __restrict__ yq,
                   const float* __restrict__ yq1, uint64_t ldq, const float* __restrict__ dval,
                   const float* __restrict__ ev, float scale, float* __restrict__ out) {
  using C = SdCfg<DC, PREC>;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bfull = reinterpret_cast<uint64_t*>(smem);  // [NB] y rows + masks + offsets landed
  uint64_t* bempty = bfull + C::NB;                     // [NB] MMA retired + masks read
  uint64_t* sfull = bempty + C::NB;                     // [NS] S in TMEM
  uint64_t* sempty = sfull + C::NS;                     // [NS] S read back
  uint64_t* qfull = sempty + C::NS;                     // A operand staged
  uint64_t* efull = qfull + 1;                          // [NE] chunk entries (ids, values) landed
  uint64_t* eempty = efull + C::NE;                     // [NE] entries consumed
  uint64_t* stfull = eempty + C::NE;                    // [NST] dots staged in entry order
  uint64_t* stempty = stfull + C::NST;                  // [NST] staged dots stored
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(stempty + C::NST);
  uint32_t* ecnt = tmem_slot + 4;                       // [NE] entries of the slot's chunk
  const uint32_t qb = smem_u32(smem + C::Q_OFF), zb = smem_u32(smem + C::Z_OFF);
  const uint32_t mb = smem_u32(smem + C::M_OFF);
  float* stage = reinterpret_cast<float*>(smem + C::ST_OFF);
  // entry ring: CSR edge ids (and, for weighted graphs, values) of a chunk,
  // bulk-copied ahead so the store loop never waits on a global load
  uint8_t* ering = smem + C::ST_OFF + C::NST * eslot;
  const bool has_dval = dval != nullptr;

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t p = blockIdx.x;
  const uint32_t c0 = pv.cptr[p], nch = pv.cptr[p + 1] - c0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NB; ++i) {
      mbar_init(bfull + i, 32);  // one cp.async.mbarrier.arrive.noinc per loader lane
      // the slot is free once the chunk's MMA retired (tcgen05.commit) AND
      // the 4 stage warps have read its masks / offsets
      mbar_init(bempty + i, 5);
    }
    for (int i = 0; i < C::NS; ++i) {
      mbar_init(sfull + i, 1);
      mbar_init(sempty + i, 4);
    }
    mbar_init(qfull, 4);
    for (int i = 0; i < C::NE; ++i) {
      mbar_init(efull + i, 1);   // the loader's expect_tx arrival + the bulk bytes
      mbar_init(eempty + i, 4);  // one arrival per store warp
    }
    for (int i = 0; i < C::NST; ++i) {
      mbar_init(stfull + i, 4);
      mbar_init(stempty + i, 4);
    }
    mbar_init_fence();
  }
  if (warp == 8) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp < 4) {
    // ---------------------------------------------------------- stage warps
    // thread per panel row: A operand, then per chunk the row's dots from TMEM
    // into the chunk's entry order (row offset precomputed in the format)
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
      const uint32_t ds = c % C::NB, b = c % C::NS, st = c % C::NST;
      mbar_wait(bfull + ds, (c / C::NB) & 1u);
      const uint32_t m = ld_shared_u32(mb + ds * kMSlot + r * 4);
      uint32_t k = ld_shared_u16(mb + ds * kMSlot + kPanelRows * 4 + r * 2);
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
      // the row's 32 dots into its own row of a shared tile (8 vector stores,
      // stride 36 floats: conflict-free), then only its edge columns, picked
      // by the mask bits, into the chunk's entry order
      const uint32_t rt = smem_u32(smem + C::R_OFF) + r * 36 * 4;
#pragma unroll
      for (int q = 0; q < 8; ++q)
        st_shared_v4(rt + q * 16, sv[4 * q], sv[4 * q + 1], sv[4 * q + 2], sv[4 * q + 3]);
      if (c >= uint32_t(C::NST)) mbar_wait(stempty + st, ((c / C::NST) - 1u) & 1u);
      float* sd = stage + st * (eslot / 4);
      for (uint32_t mm = m; mm; mm &= mm - 1) sd[k++] = __uint_as_float(ld_shared_u32(rt + (__ffs(mm) - 1) * 4));
      __syncwarp();
      if (lane == 0) mbar_arrive(stfull + st);
    }
  } else if (warp < 8) {
    // ---------------------------------------------------------- store warps
    // the chunk's edges, 128 threads: CSR id, value, coalesced store of out[e]
    const uint32_t t = threadIdx.x - 128;
    for (uint32_t c = 0; c < nch; ++c) {
      const uint32_t st = c % C::NST, de = c % C::NE;
      mbar_wait(efull + de, (c / C::NE) & 1u);
      const uint32_t cnt = ecnt[de];  // the chunk's entries, incl. <= 3 pads
      mbar_wait(stfull + st, (c / C::NST) & 1u);
      const uint32_t* eid = reinterpret_cast<const uint32_t*>(ering + de * eslot);
      const float* evl = reinterpret_cast<const float*>(ering + (C::NE + de) * eslot);
      const float* sd = stage + st * (eslot / 4);
      for (uint32_t i = t; i < cnt; i += 128) {
        const uint32_t e = eid[i];
        if (e == 0xFFFFFFFFu) continue;  // padding entry
        const float dot = sd[i];
        const float a = ev ? __ldg(ev + e) : (has_dval ? evl[i] : 1.0f);
        const float v = PREC == SGTK_TF32 ? tf32_rne(a) * tf32_rne(dot) : a * dot;
        out[e] = v * scale;
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(stempty + st);
        mbar_arrive(eempty + de);
      }
    }
  } else if (warp == 8) {
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
    // warp 9: even chunks, warp 10: odd ones
    const uint32_t par = warp - 9;
    constexpr uint32_t LPR = DC / 4, RPI = 32 / LPR;  // 16-byte pieces per row, rows per pass
    const uint32_t j = lane % LPR, jj = j & 7u;
    // column ids and entry range one chunk ahead: the global loads stay off
    // the slot-free -> gather-issue path
    uint32_t coln = par < nch ? pv.dcols[uint64_t(c0 + par) * kChunkCols + lane] : 0u;
    uint64_t kn0 = par < nch ? pv.coff[c0 + par] : 0, kn1 = par < nch ? pv.coff[c0 + par + 1] : 0;
    for (uint32_t c = par; c < nch; c += 2) {
      const uint32_t ds = c % C::NB;
      const uint64_t ch = c0 + c;
      const uint32_t col = coln;
      const uint64_t k0 = kn0, k1 = kn1;
      if (c + 2 < nch) {
        coln = pv.dcols[(ch + 2) * kChunkCols + lane];
        kn0 = pv.coff[ch + 2];
        kn1 = pv.coff[ch + 3];
      }
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
      cp_async16(mb + ds * kMSlot + lane * 16, pv.dmask + ch * kPanelRows + lane * 4);
      if (lane < 16)
        cp_async16(mb + ds * kMSlot + kPanelRows * 4 + lane * 16, rowoff + ch * kPanelRows + lane * 8);
      cp_async_arrive_noinc(bfull + ds);
      // the chunk's entries (ids, values) by the TMA engine: a slot is reused
      // once the store loop of chunk c - NE is done with it
      const uint32_t de = c % C::NE;
      mbar_wait(eempty + de, ((c / C::NE) & 1u) ^ 1u);
      if (lane == 0) {
        const uint32_t bytes = uint32_t(k1 - k0) * 4u;  // entries padded to 4: 16-byte multiple
        ecnt[de] = uint32_t(k1 - k0);  // published by the arrive below (release)
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
  if (warp == 8) {
    tc_fence_after();
    tmem_dealloc(tmem, C::TMEM_COLS);
  }
}

// Dense part, direct form (sddmm_dense2_kernel): the chunk's dots go once
// through a row tile in shared memory and the store warps read each entry's
// dot from it by the entry's (panel row, chunk column) -- no per-row
// compaction loop.  An entry is one u32 (Panels::dpos: position in its CSR
// row << 12 | panel row << 5 | chunk column); out[np[row] + position].
//   warps 0-3  stage: the A operand; per chunk the row's 32 dots from TMEM
//              (tcgen05.ld) into row tile c % NR (8 conflict-free 16-byte
//              stores, stride 36 floats);
//   warps 4-7  store: the chunk's entries (bulk-copied ahead by the TMA
//              engine), a_e * dot, out[e];
//   warp 8     TMEM allocator + tcgen05.mma issuer (S buffers over 4 x 32
//              TMEM columns);
//   warps 9-10 loaders (even / odd chunks): the chunk's 32 y rows (cp.async,
//              K-major SWIZZLE_128B), the bulk copy of its entries.
template <int DC, int PREC>
struct Sd2Cfg {
  static constexpr bool F32 = PREC == SGTK_FP32;
  static constexpr int PL = F32 ? 2 : 1;
  static constexpr int KB = DC / 32;
  static constexpr int NB = (F32 && DC == 64) ? 4 : 6;
  static constexpr int NS = 4;
  static constexpr int NR = 2;                               // row tiles
  static constexpr int NE = 4;                               // entry ring
  static constexpr uint32_t RS = 36;                         // row tile stride (floats)
  static constexpr uint32_t Q_BYTES = kPanelRows * DC * 4;
  static constexpr uint32_t TILE = kChunkCols * 128;
  static constexpr uint32_t Q_OFF = 1024;
  static constexpr uint32_t Z_OFF = Q_OFF + PL * Q_BYTES;
  static constexpr uint32_t R_OFF = Z_OFF + PL * KB * NB * TILE;
  static constexpr uint32_t NP_OFF = R_OFF + NR * kPanelRows * RS * 4;  // u64[128] row starts
  static constexpr uint32_t E_OFF = NP_OFF + kPanelRows * 8;
  static uint32_t smem_bytes(uint32_t eslot, bool with_vals) {
    return E_OFF + NE * eslot * (with_vals ? 2u : 1u) + 1024;
  }
  static constexpr uint32_t TMEM_COLS = NS * 32;
};

template <int DC, int PREC>
__global__ void __launch_bounds__(kSdThreads, 2)
sddmm_dense2_kernel(const PanelView pv, const uint32_t* __restrict__ dpos, const uint64_t* __restrict__ np,
                    uint32_t eslot, const float* __restrict__ x, uint64_t ldx, uint64_t d,
                    uint64_t row_offset, const float* __restrict__ inv, const float* __restrict__ yq,
                    const float* __restrict__ yq1, uint64_t ldq, const float* __restrict__ dval,
                    const float* __restrict__ ev, float scale, float* __restrict__ out) {
  using C = Sd2Cfg<DC, PREC>;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint64_t* bfull = reinterpret_cast<uint64_t*>(smem);  // [NB] y rows landed
  uint64_t* bempty = bfull + C::NB;                     // [NB] MMA retired
  uint64_t* sfull = bempty + C::NB;                     // [NS] S in TMEM
  uint64_t* sempty = sfull + C::NS;                     // [NS] S read back
  uint64_t* qfull = sempty + C::NS;                     // A operand staged (+ row starts)
  uint64_t* efull = qfull + 1;                          // [NE] entries landed
  uint64_t* eempty = efull + C::NE;                     // [NE] entries consumed
  uint64_t* rfull = eempty + C::NE;                     // [NR] row tile written
  uint64_t* rempty = rfull + C::NR;                     // [NR] row tile consumed
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(rempty + C::NR);
  uint32_t* ecnt = tmem_slot + 4;                       // [NE] entries of the slot's chunk
  const uint32_t qb = smem_u32(smem + C::Q_OFF), zb = smem_u32(smem + C::Z_OFF);
  const uint32_t rb = smem_u32(smem + C::R_OFF);
  uint64_t* nps = reinterpret_cast<uint64_t*>(smem + C::NP_OFF);
  uint8_t* ering = smem + C::E_OFF;
  const bool has_dval = dval != nullptr;

  const uint32_t warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint64_t p = blockIdx.x;
  const uint32_t c0 = pv.cptr[p], nch = pv.cptr[p + 1] - c0;

  if (threadIdx.x == 0) {
    for (int i = 0; i < C::NB; ++i) {
      mbar_init(bfull + i, 32);  // one cp.async.mbarrier.arrive.noinc per loader lane
      mbar_init(bempty + i, 1);  // tcgen05.commit
    }
    for (int i = 0; i < C::NS; ++i) {
      mbar_init(sfull + i, 1);
      mbar_init(sempty + i, 4);
    }
    mbar_init(qfull, 4);
    for (int i = 0; i < C::NE; ++i) {
      mbar_init(efull + i, 1);
      mbar_init(eempty + i, 8);  // the 8 storing warps
    }
    for (int i = 0; i < C::NR; ++i) {
      mbar_init(rfull + i, 4);
      mbar_init(rempty + i, 8);
    }
    mbar_init_fence();
  }
  if (warp == 8) tmem_alloc(tmem_slot, C::TMEM_COLS);
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  // a share of chunk c's entries: thread t of the 256 storing threads (store
  // warps t < 128, stage warps t >= 128) takes entries t, t + 256, ...
  auto store_chunk = [&](uint32_t c, uint32_t t) {
      const uint32_t rt = c % C::NR, de = c % C::NE;
      mbar_wait(efull + de, (c / C::NE) & 1u);
      const uint32_t cnt = ecnt[de];
      mbar_wait(rfull + rt, (c / C::NR) & 1u);
      const uint32_t* ent = reinterpret_cast<const uint32_t*>(ering + de * eslot);
      const float* evl = reinterpret_cast<const float*>(ering + (C::NE + de) * eslot);
      const float* rtile = reinterpret_cast<const float*>(smem + C::R_OFF) + rt * kPanelRows * C::RS;
      if (!ev && !has_dval) {  // unit values: a_e = 1 (tf32(1) = 1)
        for (uint32_t i = t; i < cnt; i += 256) {
          const uint32_t w = ent[i];
          if (w == 0xFFFFFFFFu) continue;  // padding entry
          const float dot = rtile[((w >> 5) & 127u) * C::RS + (w & 31u)];
          const uint64_t e = nps[(w >> 5) & 127u] + (w >> 12);
          out[e] = (PREC == SGTK_TF32 ? tf32_rne(dot) : dot) * scale;
        }
      } else {
        for (uint32_t i = t; i < cnt; i += 256) {
          const uint32_t w = ent[i];
          if (w == 0xFFFFFFFFu) continue;  // padding entry
          const uint32_t row = (w >> 5) & 127u, k = w & 31u;
          const float dot = rtile[row * C::RS + k];
          const uint64_t e = nps[row] + (w >> 12);
          const float a = ev ? __ldg(ev + e) : evl[i];
          const float v = PREC == SGTK_TF32 ? tf32_rne(a) * tf32_rne(dot) : a * dot;
          out[e] = v * scale;
        }
      }
      __syncwarp();
      if (lane == 0) {
        mbar_arrive(rempty + rt);
        mbar_arrive(eempty + de);
      }
  };

  if (warp < 4) {
    // ---------------------------------------------------------- stage warps
    const uint32_t r = warp * 32 + lane;
    const uint64_t grow = p * kPanelRows + r;
    {  // A = x[panel rows] (z = x * inv when normalising on the fly)
      const bool rv = grow < pv.n_rows;
      nps[r] = rv ? np[grow] : 0ull;
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
      const uint32_t b = c % C::NS, rt = c % C::NR;
      mbar_wait(sfull + b, (c / C::NS) & 1u);
      tc_fence_after();
      uint32_t sv[32];
      tmem_ld16(tmem + ((warp * 32u) << 16) + b * 32, *reinterpret_cast<uint32_t(*)[16]>(sv));
      tmem_ld16(tmem + ((warp * 32u) << 16) + b * 32 + 16, *reinterpret_cast<uint32_t(*)[16]>(sv + 16));
      tmem_ld_wait();
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(sempty + b);
      if (c >= uint32_t(C::NR)) mbar_wait(rempty + rt, ((c / C::NR) - 1u) & 1u);
      const uint32_t rr = rb + (rt * kPanelRows + r) * C::RS * 4;
#pragma unroll
      for (int q = 0; q < 8; ++q) st_shared_v4(rr + q * 16, sv[4 * q], sv[4 * q + 1], sv[4 * q + 2], sv[4 * q + 3]);
      __syncwarp();
      if (lane == 0) mbar_arrive(rfull + rt);
      store_chunk(c, threadIdx.x + 128);  // waits for the other stage warps' rows
    }
  } else if (warp < 8) {
    // ---------------------------------------------------------- store warps
    mbar_wait(qfull, 0);  // row starts staged
    for (uint32_t c = 0; c < nch; ++c) store_chunk(c, threadIdx.x - 128);
  } else if (warp == 8) {
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
    const uint32_t par = warp - 9;
    constexpr uint32_t LPR = DC / 4, RPI = 32 / LPR;
    const uint32_t j = lane % LPR, jj = j & 7u;
    uint32_t coln = par < nch ? pv.dcols[uint64_t(c0 + par) * kChunkCols + lane] : 0u;
    uint64_t kn0 = par < nch ? pv.coff[c0 + par] : 0, kn1 = par < nch ? pv.coff[c0 + par + 1] : 0;
    for (uint32_t c = par; c < nch; c += 2) {
      const uint32_t ds = c % C::NB;
      const uint64_t ch = c0 + c;
      const uint32_t col = coln;
      const uint64_t k0 = kn0, k1 = kn1;
      if (c + 2 < nch) {
        coln = pv.dcols[(ch + 2) * kChunkCols + lane];
        kn0 = pv.coff[ch + 2];
        kn1 = pv.coff[ch + 3];
      }
      mbar_wait(bempty + ds, ((c / C::NB) & 1u) ^ 1u);
#pragma unroll
      for (uint32_t t = 0; t < 32 / RPI; ++t) {
        const uint32_t kr = t * RPI + lane / LPR;
        const uint32_t ck = __shfl_sync(0xFFFFFFFFu, col, kr);
        if (ck == 0xFFFFFFFFu) continue;  // padding column: its S column is never read
        const uint64_t gofs = uint64_t(ck) * ldq + 4 * j;
        const uint32_t zo = ((j >> 3) * C::NB + ds) * C::TILE + (kr >> 3) * 1024u + (kr & 7u) * 128u +
                            ((jj ^ (kr & 7u)) << 4);
        cp_async16(zb + zo, yq + gofs);
        if constexpr (C::F32) cp_async16(zb + C::KB * C::NB * C::TILE + zo, yq1 + gofs);
      }
      cp_async_arrive_noinc(bfull + ds);
      const uint32_t de = c % C::NE;
      mbar_wait(eempty + de, ((c / C::NE) & 1u) ^ 1u);
      if (lane == 0) {
        const uint32_t bytes = uint32_t(k1 - k0) * 4u;  // entries padded to 4: 16-byte multiple
        ecnt[de] = uint32_t(k1 - k0);
        mbar_expect_tx(efull + de, bytes * (has_dval ? 2u : 1u));
        if (bytes) {
          bulk_load(ering + de * eslot, dpos + k0, bytes, efull + de);
          if (has_dval) bulk_load(ering + (C::NE + de) * eslot, dval + k0, bytes, efull + de);
        }
      }
    }
    cp_async_wait<0>();
  }

  tc_fence_before();
  __syncthreads();
  if (warp == 8) {
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

// Sparse edges: warp per row, G = ceil(d/4) lanes per edge (float4 slices of
// the x row held in registers, the y row read coalesced), 32/G edges per warp
// pass, the slices' partial dots reduced by a fixed xor tree (deterministic).
constexpr int kSpWarps = 8;
template <int PREC, int G>
__global__ void __launch_bounds__(kSpWarps * 32)
sddmm_sparse_kernel(uint64_t n_rows, const uint32_t* __restrict__ sptr, const uint2* __restrict__ sent,
                    const uint32_t* __restrict__ seid, const float* __restrict__ x, uint64_t ldx,
                    const float* __restrict__ yq, uint64_t ldq, uint64_t d, uint64_t row_offset,
                    const float* __restrict__ inv, const float* __restrict__ vals, float scale,
                    float* __restrict__ out) {
  constexpr uint32_t EPP = 32 / G;   // edges per pass
  constexpr uint32_t NP = 32 / EPP;  // passes per 32-edge batch
  const uint32_t wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const uint32_t sub = lane / G, j = lane % G;
  const uint64_t nw = uint64_t(gridDim.x) * kSpWarps;
  for (uint64_t r = uint64_t(blockIdx.x) * kSpWarps + wib; r < n_rows; r += nw) {
    const uint32_t s0 = sptr[r], s1 = sptr[r + 1];
    if (s0 == s1) continue;
    // this lane's 4 features of the row (z = x * inv; TF32: rounded like the
    // y copies, which yprep already rounded)
    const uint64_t xr = row_offset + r;
    const float ir = inv ? inv[xr] : 1.0f;
    float xv[4];
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const uint64_t f = 4 * j + i;
      float v = f < d ? x[xr * ldx + f] : 0.0f;
      if (inv) v = v * ir;
      xv[i] = PREC == SGTK_TF32 ? tf32_rne(v) : v;
    }
    for (uint32_t kb = s0; kb < s1; kb += 32) {
      const uint32_t n = min(32u, s1 - kb);
      // lane = edge: the batch's column ids and CSR ids (coalesced)
      const uint32_t mcol = lane < n ? sent[kb + lane].x : 0u;
      const uint32_t me = lane < n ? seid[kb + lane] : 0u;
      // all of the batch's row slices in flight at once (G lanes per edge)
      float4 q[NP];
#pragma unroll
      for (uint32_t pp = 0; pp < NP; ++pp) {
        const uint32_t idx = pp * EPP + sub;
        const uint32_t col = __shfl_sync(0xFFFFFFFFu, mcol, idx);
        q[pp] = idx < n ? __ldg(reinterpret_cast<const float4*>(yq + uint64_t(col) * ldq) + j)
                        : make_float4(0.f, 0.f, 0.f, 0.f);
      }
      float mine = 0.0f;  // lane = edge again: its dot
#pragma unroll
      for (uint32_t pp = 0; pp < NP; ++pp) {
        float dot = xv[0] * q[pp].x;
        dot = fmaf(xv[1], q[pp].y, dot);
        dot = fmaf(xv[2], q[pp].z, dot);
        dot = fmaf(xv[3], q[pp].w, dot);
#pragma unroll
        for (uint32_t o = 1; o < G; o <<= 1) dot += __shfl_xor_sync(0xFFFFFFFFu, dot, o);
        // edge pp * EPP + s sits in group s: lane L takes group L % EPP of pass L / EPP
        const float v = __shfl_sync(0xFFFFFFFFu, dot, (lane % EPP) * G);
        if (lane / EPP == pp) mine = v;
      }
      if (lane < n) {
        const float a = vals ? __ldg(vals + me) : 1.0f;
        const float v = PREC == SGTK_TF32 ? tf32_rne(a) * tf32_rne(mine) : a * mine;
        out[me] = v * scale;
      }
    }
  }
}

// FP32 sparse rows: z = y * inv exactly (no TF32 planes), padded to ldq.
__global__ void sddmm_rows_f32_kernel(const float* __restrict__ y, uint64_t ldy, uint64_t rows,
                                      uint64_t d, const float* __restrict__ inv, uint64_t ldq,
                                      float* __restrict__ yz) {
  const uint64_t n = rows * ldq;
  for (uint64_t i = uint64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += uint64_t(gridDim.x) * blockDim.x) {
    const uint64_t r = i / ldq, f = i - r * ldq;
    const float v = f < d ? y[r * ldy + f] : 0.0f;
    yz[i] = inv ? v * inv[r] : v;
  }
}

template <int DC, int PREC>
bool launch_sd_dense(const PanelView& v, uint64_t P, uint32_t max_entries, const uint32_t* deid,
                     const uint16_t* rowoff, const float* x, uint64_t ldx, uint64_t d, uint64_t ro, const float* inv,
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
      v, deid, rowoff, eslot, x, ldx, d, ro, inv, yq, yq1, ldq, dval, ev, scale, out);
  CU_LAUNCH("sddmm_dense_kernel");
  return true;
}

template <int DC, int PREC>
bool launch_sd_dense2(const PanelView& v, uint64_t P, uint32_t max_entries, const uint32_t* dpos,
                      const uint64_t* np, const float* x, uint64_t ldx, uint64_t d, uint64_t ro, const float* inv,
                      const float* yq, const float* yq1, uint64_t ldq, const float* dval,
                      const float* ev, float scale, float* out, cudaStream_t s) {
  using C = Sd2Cfg<DC, PREC>;
  const uint32_t eslot = (max_entries + 3) / 4 * 16;
  const uint32_t smem = C::smem_bytes(eslot, dval != nullptr);
  if (smem > 227u * 1024u) return false;
  once_per_device(reinterpret_cast<const void*>(&sddmm_dense2_kernel<DC, PREC>), [] {
    cudaFuncSetAttribute(sddmm_dense2_kernel<DC, PREC>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         int(227u * 1024u));
  });
  sddmm_dense2_kernel<DC, PREC><<<unsigned(P), kSdThreads, smem, s>>>(
      v, dpos, np, eslot, x, ldx, d, ro, inv, yq, yq1, ldq, dval, ev, scale, out);
  CU_LAUNCH("sddmm_dense2_kernel");
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
  {
    CU(cudaMallocAsync(reinterpret_cast<void**>(&buf), 2 * plane, s));
    float* yq = reinterpret_cast<float*>(buf);
    float* yq1 = reinterpret_cast<float*>(buf + plane);
    const unsigned gb = sd_grid(g->n_cols * ldq, 256);
    if (prec == SGTK_FP32) sddmm_yprep_kernel<SGTK_FP32><<<gb, 256, 0, s>>>(y, ldy, g->n_cols, d, inv_norm, ldq, yq, yq1);
    else sddmm_yprep_kernel<SGTK_TF32><<<gb, 256, 0, s>>>(y, ldy, g->n_cols, d, inv_norm, ldq, yq, nullptr);
    CU_LAUNCH("sddmm_yprep_kernel");
  }
  // the CUDA-core part goes to the auxiliary stream, concurrently with the
  // tensor-core kernel (the paper's two independent resources); it starts
  // once the y copies it reads are ready
  const AuxStreams& ax = aux_streams();
  cudaStream_t sa = s;
  if (pn.n_sparse && pn.n_chunks) {
    CU(cudaEventRecord(ax.ready, s));
    CU(cudaStreamWaitEvent(ax.aux, ax.ready, 0));
    sa = ax.aux;
  }
  {
    float* yq = reinterpret_cast<float*>(buf);
    float* yq1 = reinterpret_cast<float*>(buf + plane);
    const uint32_t* deid = pn.deid->as<uint32_t>();
    const uint16_t* rowoff = pn.rowoff->as<uint16_t>();
    const uint64_t ro = g->row_offset;
    const uint32_t me = pn.max_chunk_entries;
    // direct form when every entry's CSR position fits (Panels::dpos) and its
    // entry ring fits; SGTK_SDDMM_DENSE=staged: the compaction form
    static const bool staged = [] {
      const char* e = std::getenv("SGTK_SDDMM_DENSE");
      return e && std::string(e) == "staged";
    }();
    bool done = false;
    if (pn.n_chunks && !staged) ensure_dpos(*g, pn, s);
    if (pn.n_chunks && pn.dpos_ok && !staged) {
      const uint32_t* dp = pn.dpos->as<uint32_t>();
      const uint64_t* npg = g->np->as<uint64_t>();
      if (prec == SGTK_FP32)
        done = ldq == 32 ? launch_sd_dense2<32, SGTK_FP32>(v, pn.P, me, dp, npg, x, ldx, d, ro, inv_norm, yq, yq1, ldq, dval, ev, scale, out, s)
                         : launch_sd_dense2<64, SGTK_FP32>(v, pn.P, me, dp, npg, x, ldx, d, ro, inv_norm, yq, yq1, ldq, dval, ev, scale, out, s);
      else
        done = ldq == 32 ? launch_sd_dense2<32, SGTK_TF32>(v, pn.P, me, dp, npg, x, ldx, d, ro, inv_norm, yq, nullptr, ldq, dval, ev, scale, out, s)
                         : launch_sd_dense2<64, SGTK_TF32>(v, pn.P, me, dp, npg, x, ldx, d, ro, inv_norm, yq, nullptr, ldq, dval, ev, scale, out, s);
    }
    if (done) {
    } else if (pn.n_chunks && prec == SGTK_FP32) {
      if (ldq == 32) launch_sd_dense<32, SGTK_FP32>(v, pn.P, me, deid, rowoff, x, ldx, d, ro, inv_norm, yq, yq1, ldq, dval, ev, scale, out, s);
      else launch_sd_dense<64, SGTK_FP32>(v, pn.P, me, deid, rowoff, x, ldx, d, ro, inv_norm, yq, yq1, ldq, dval, ev, scale, out, s);
    } else if (pn.n_chunks) {
      if (ldq == 32) launch_sd_dense<32, SGTK_TF32>(v, pn.P, me, deid, rowoff, x, ldx, d, ro, inv_norm, yq, nullptr, ldq, dval, ev, scale, out, s);
      else launch_sd_dense<64, SGTK_TF32>(v, pn.P, me, deid, rowoff, x, ldx, d, ro, inv_norm, yq, nullptr, ldq, dval, ev, scale, out, s);
    }
  }
  if (pn.n_sparse) {
    // the CUDA-core part reads padded rows of z: TF32 -> the rounded copies
    // (yq); FP32 -> exact z rows (one more pass, the hi/lo planes are TF32)
    float* yz = nullptr;
    const float* ysrc = nullptr;
    if (prec == SGTK_FP32) {
      CU(cudaMallocAsync(reinterpret_cast<void**>(&yz), plane, sa));
      sddmm_rows_f32_kernel<<<sd_grid(g->n_cols * ldq, 256), 256, 0, sa>>>(y, ldy, g->n_cols, d,
                                                                          inv_norm, ldq, yz);
      CU_LAUNCH("sddmm_rows_f32_kernel");
      ysrc = yz;
    } else {
      ysrc = reinterpret_cast<const float*>(buf);
    }
    const unsigned gs = sd_grid(g->n_rows, kSpWarps, 148u * 16u);
    const auto* sp = pn.sptr->as<uint32_t>();
    const auto* se = pn.sent->as<uint2>();
    const auto* si = pn.seid->as<uint32_t>();
    const uint64_t ro = g->row_offset;
    if (prec == SGTK_FP32) {
      if (ldq == 32) sddmm_sparse_kernel<SGTK_FP32, 8><<<gs, kSpWarps * 32, 0, sa>>>(g->n_rows, sp, se, si, x, ldx, ysrc, ldq, d, ro, inv_norm, vals, scale, out);
      else sddmm_sparse_kernel<SGTK_FP32, 16><<<gs, kSpWarps * 32, 0, sa>>>(g->n_rows, sp, se, si, x, ldx, ysrc, ldq, d, ro, inv_norm, vals, scale, out);
    } else {
      if (ldq == 32) sddmm_sparse_kernel<SGTK_TF32, 8><<<gs, kSpWarps * 32, 0, sa>>>(g->n_rows, sp, se, si, x, ldx, ysrc, ldq, d, ro, inv_norm, vals, scale, out);
      else sddmm_sparse_kernel<SGTK_TF32, 16><<<gs, kSpWarps * 32, 0, sa>>>(g->n_rows, sp, se, si, x, ldx, ysrc, ldq, d, ro, inv_norm, vals, scale, out);
    }
    CU_LAUNCH("sddmm_sparse_kernel");
    if (yz) CU(cudaFreeAsync(yz, sa));
  }
  if (sa != s) {  // join: the caller's stream sees both halves done
    CU(cudaEventRecord(ax.join, sa));
    CU(cudaStreamWaitEvent(s, ax.join, 0));
  }
  if (buf) CU(cudaFreeAsync(buf, s));
  return true;
}

}  // namespace sgtkcu
