// Device-resident TransformedGraph + the condensed tile format (host struct).
#pragma once

#include <memory>
#include <mutex>
#include <vector>

#include "common.cuh"

namespace sgtkcu {

// One warp-task of the tiled kernels: tiles [t0, t1) of 16-row window `window`
// (internal 16-row geometry).  slot != kNoSlot: the window is split into
// several units whose partial 16 x d outputs are reduced in slot order.
struct WorkUnit {
  uint32_t window;
  uint32_t t0;
  uint32_t t1;
  uint32_t slot;
};

// A split window: partial slots [slot0, slot0 + count) reduce into its rows.
struct ReduceItem {
  uint32_t window;
  uint32_t slot0;
  uint32_t count;
  uint32_t pad;
};

struct UnitPlan {
  std::shared_ptr<DevBuf> units, reduce;
  uint32_t n_units = 0, n_reduce = 0, n_slots = 0, max_tiles = 0;
};

// Translator output for one row-window height (the reference fields).
struct Windows {
  uint32_t blk_h = 16;
  uint64_t W = 0, U = 0;
  std::shared_ptr<DevBuf> e2c;  // u32[E] window-relative rank
  std::shared_ptr<DevBuf> wo;   // u64[W+1]
  std::shared_ptr<DevBuf> wuc;  // u32[U]
  std::vector<uint32_t> ucount_host;  // unique columns per window
  std::vector<uint64_t> wo_host;
};

// 128-row panel format for the tcgen05 aggregation kernels (panel.cu).
// Per panel (128 rows, the UMMA M), the unique columns with >= kDenseMin
// edges are "dense": they are gathered once per panel and multiplied on the
// tensor cores in chunks of 32 (one 128-byte swizzle row of TF32).  The other
// ("sparse") edges -- mostly singleton columns -- run edge-by-edge on CUDA
// cores.  This is the density-aware hybrid split of SURVEY §8f rank 3.
constexpr int kPanelRows = 128;
constexpr int kChunkCols = 32;
constexpr uint32_t kDenseMin = 2;     // panels: tensor-core columns have >= 2 edges
#ifndef SGTK_DENSE_MIN32
#define SGTK_DENSE_MIN32 3
#endif
constexpr uint32_t kDenseMin32 = SGTK_DENSE_MIN32;   // panels32: the d <= 32 kernels' cheaper CUDA-core edge
                                      // makes 2-edge columns cheaper there
constexpr uint32_t kSegEdges = 512;       // sparse edges per CUDA-core work item

struct Panels {
  uint64_t P = 0, n_chunks = 0, n_dent = 0, n_sparse = 0;
  uint32_t max_chunk_entries = 0;
  std::shared_ptr<DevBuf> cptr;   // u32[P+1]   first chunk of panel p
  std::shared_ptr<DevBuf> dcols;  // u32[32*n_chunks] dense column ids (pad 0xFFFFFFFF)
  std::shared_ptr<DevBuf> coff;   // u64[n_chunks+1] entry range of a chunk (multiple of 4)
  std::shared_ptr<DevBuf> dent;   // u32[n_dent]  tf32(value) | swizzled A-tile word offset
  std::shared_ptr<DevBuf> dval;   // f32[n_dent]  full fp32 value
  std::shared_ptr<DevBuf> deid;   // u32[n_dent]  CSR edge id (0xFFFFFFFF for padding)
  std::shared_ptr<DevBuf> dmask;  // u32[n_chunks * 128] row r's edge bits in the chunk (AGNN)
  std::shared_ptr<DevBuf> rowoff; // u16[n_chunks * 128] entries of the chunk before row r (SDDMM)
  // u32[n_dent] SDDMM entry: (position in the CSR row) << 12 | panel row << 5 |
  // chunk column (0xFFFFFFFF for padding); built on the first SDDMM call
  // (ensure_dpos; not persisted); dpos_ok = every position < 2^20
  std::shared_ptr<DevBuf> dpos;
  bool dpos_ok = false;
  std::shared_ptr<std::once_flag> dpos_once = std::make_shared<std::once_flag>();
  std::shared_ptr<DevBuf> sptr;   // u32[n_rows+1] sparse edges of a row
  std::shared_ptr<DevBuf> sent;   // uint2[n_sparse] (column, value bits)
  std::shared_ptr<DevBuf> seid;   // u32[n_sparse] CSR edge id
  // CUDA-core work list: one item per row with sparse edges; rows with more
  // than kSegEdges sparse edges are cut into segments whose partial sums are
  // reduced in segment order (sparse_rows_kernel / long_rows_kernel).
  uint64_t n_items = 0, n_long = 0, n_segs = 0;
  std::shared_ptr<DevBuf> items;  // uint4[n_items] (row, e_begin, e_end, segment | ~0u)
  std::shared_ptr<DevBuf> lrows;  // uint4[n_long]  (row, first segment, segments, 0)
  // AGNN work list: every row is an item (out = O / l everywhere); hub rows
  // as the same segments as above
  uint64_t n_aitems = 0;
  std::shared_ptr<DevBuf> aitems;  // uint4[n_aitems]
  std::shared_ptr<DevBuf> paitem;  // u32[P+1] first aitem of panel p (rows in order; ensure_paitem)
  std::shared_ptr<std::once_flag> paitem_once = std::make_shared<std::once_flag>();
};

struct PanelView {
  uint64_t n_rows, P;
  const uint32_t* cptr;
  const uint32_t* dcols;
  const uint64_t* coff;
  const uint32_t* dent;
  const float* dval;
  const uint32_t* sptr;
  const uint2* sent;
  const uint32_t* dmask;
  const uint32_t* paitem;
};

// POD view handed to kernels.
struct DevGraph {
  uint64_t n_rows, n_cols, nnz, W;
  uint64_t row_offset;  // global id of local row 0 (row-window partition)
  const uint64_t* np;
  const uint32_t* el;
  const float* vals;
  const uint32_t* e2c;  // internal (16-row) ranks
  const uint64_t* wo;
  const uint32_t* wuc;
  const uint64_t* toff8;
  const uint4* bm8;     // per 8-wide tile: 16 rows x 8 bits (byte r = row r)
  const uint64_t* toff16;
  const uint4* bm16;    // per 16-wide tile: 2 x uint4 (u16 per row)
};

}  // namespace sgtkcu

struct sgtk_graph {
  uint64_t n_rows = 0, n_cols = 0, nnz = 0, row_offset = 0;
  uint32_t blk_h = 16, blk_w = 8;
  bool has_values = false;
  int device = 0;

  std::shared_ptr<sgtkcu::DevBuf> np, el, vals, e2r;
  sgtkcu::Windows user;      // reference fields at the user's geometry
  sgtkcu::Windows internal;  // 16-row windows the kernels run on (== user if blk_h == 16)
  std::vector<uint32_t> bp_host;  // block_partition at (blk_h, blk_w)
  uint64_t block_counter = 0;
  std::shared_ptr<sgtkcu::DevBuf> bp;  // u32[W] at (blk_h, blk_w)

  // condensed tile format (internal windows)
  uint64_t T8 = 0, T16 = 0;
  std::shared_ptr<sgtkcu::DevBuf> toff8, bm8, toff16, bm16;
  sgtkcu::UnitPlan plan8, plan16;
  std::shared_ptr<sgtkcu::Panels> panels;    // 128-row panel format (panel.cu), kDenseMin
  std::shared_ptr<sgtkcu::Panels> panels32;  // same at kDenseMin32: operations with d <= 32
  bool panels_loaded = false;                 // read from a panel section (no build_panels)

  // workspace for host-buffer entry points and forwards (mutable scratch)
  mutable std::shared_ptr<sgtkcu::DevBuf> scratch;

  // Host wall time per construction stage (ms), recorded when SGTK_BUILD_TIMING
  // is set (the stream is synchronised at every stage boundary, so the stages
  // add up to the whole build): upload, validate, edge_to_row, windows (user
  // geometry), windows (16-row internal), tiles + work units, panels.
  double build_ms[8] = {0, 0, 0, 0, 0, 0, 0, 0};

  sgtkcu::DevGraph view() const {
    sgtkcu::DevGraph v{};
    v.n_rows = n_rows;
    v.n_cols = n_cols;
    v.nnz = nnz;
    v.row_offset = row_offset;
    v.W = internal.W;
    v.np = np->as<uint64_t>();
    v.el = el->as<uint32_t>();
    v.vals = has_values ? vals->as<float>() : nullptr;
    v.e2c = internal.e2c->as<uint32_t>();
    v.wo = internal.wo->as<uint64_t>();
    v.wuc = internal.wuc->as<uint32_t>();
    v.toff8 = toff8->as<uint64_t>();
    v.bm8 = bm8->as<uint4>();
    v.toff16 = toff16->as<uint64_t>();
    v.bm16 = bm16->as<uint4>();
    return v;
  }
};

namespace sgtkcu {
// Per-window tile-threshold (in 8- or 16-wide internal tiles) derived from a
// user-geometry cut array; nullptr cut => all tiles on the tensor-core path.
// Returns a device array u32[W_internal] or nullptr (owned by `keep`).
const uint32_t* internal_cut(const sgtk_graph* g, const uint32_t* cut_dev,
                             int tile_w, cudaStream_t s, DevBuf& keep);
}  // namespace sgtkcu
