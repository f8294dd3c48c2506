/*
 * sgtk_cuda.h — C ABI of the B200-native (sm_100a) FTC-GNN aggregation path.
 *
 * This is the drop-in boundary: plain pointers, sizes and status codes, no C++
 * or torch types.  Every entry point below replaces one function of the
 * reference's public C++ interface (/root/reference/proj/include/sgtk/*.hpp);
 * the replaced declaration is cited on each.  The C++ drop-in
 * (include/sgtk/api.hpp, namespace sgtk) and the Python binding
 * (paper_2412_12218_b200/__init__.py) are thin layers over exactly these calls.
 *
 * Conventions
 *   - Device pointers ("_dev") are CUDA global-memory pointers on the current
 *     device; host pointers ("_host") are plain (preferably pinned) memory.
 *   - `stream` is a cudaStream_t (NULL = legacy default stream).  Device
 *     entry points are asynchronous unless they must return a host value
 *     (documented per call).
 *   - Feature matrices are row-major f32 with an explicit leading dimension
 *     (elements).  Best performance: ld % 4 == 0 and 16-byte aligned base.
 *   - Errors are never thrown across this boundary: every call returns an
 *     sgtk_status and the thread-local message is sgtk_last_error().
 *   - Results are deterministic: no floating-point atomics on any output; the
 *     same inputs give bit-identical outputs on every run and GPU count.
 */
#ifndef SGTK_CUDA_H_
#define SGTK_CUDA_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

/* Status codes map 1:1 onto the reference exception hierarchy
 * (/root/reference/proj/include/sgtk/errors.hpp:10-51). */
typedef enum sgtk_status {
  SGTK_OK = 0,
  SGTK_ERR = 1,            /* sgtk::Error (e.g. malformed CSR)            */
  SGTK_ERR_IO = 2,         /* sgtk::IoError                               */
  SGTK_ERR_PARSE = 3,      /* sgtk::ParseError                            */
  SGTK_ERR_OVERFLOW = 4,   /* sgtk::OverflowError                         */
  SGTK_ERR_DEGREE = 5,     /* sgtk::DegreeError                           */
  SGTK_ERR_GEOMETRY = 6,   /* sgtk::GeometryError                         */
  SGTK_ERR_INDEX = 7,      /* sgtk::IndexError                            */
  SGTK_ERR_RANGE = 8,      /* sgtk::RangeError                            */
  SGTK_ERR_SHAPE = 9,      /* sgtk::ShapeError                            */
  SGTK_ERR_NONFINITE = 10, /* sgtk::NonFiniteError                        */
  SGTK_ERR_CUDA = 11,      /* CUDA runtime / launch failure -> sgtk::Error */
  SGTK_ERR_NCCL = 12       /* NCCL failure -> sgtk::Error                 */
} sgtk_status;

/* tile_exec.hpp:12-15 Precision: exactly the reference's two modes.  (A BF16
 * mode is not offered: the reference has none to be a drop-in for, and
 * rejecting an advertised value on every call would only be a trap.) */
typedef enum sgtk_precision {
  SGTK_FP32 = 0, /* fp32-accurate: split-TF32 MMA, fp32 accumulate        */
  SGTK_TF32 = 1  /* operands RNE-rounded to TF32 (tile_exec.cpp:131-142)  */
} sgtk_precision;

/* Thread-local message of the last failing call on this thread. */
const char* sgtk_last_error(void);
/* Library version string and the compiled device architecture ("sm_100a"). */
const char* sgtk_version(void);

/* ------------------------------------------------------------------------
 * Device graph: a TransformedGraph resident in HBM plus the condensed tile
 * format the kernels consume (16-row windows; 8- and 16-wide tiles with
 * 16-row occupancy bitmaps; nnz-balanced work units).
 * ---------------------------------------------------------------------- */
typedef struct sgtk_graph sgtk_graph;

#define SGTK_PTR_HOST 0
#define SGTK_PTR_DEVICE 1

/* sgt_transform (sgt_transform.hpp:49-50, sgt_transform.cpp:18-77).
 * Validates the CSR (csr_graph.cpp:10-39 -> SGTK_ERR), runs the GPU translator
 * (bit-exact with the reference) and builds the kernel tile format.  The CSR
 * arrays are copied (HOST) or copied device-to-device (DEVICE); the caller keeps
 * ownership.  `values` may be NULL (unweighted: every edge is 1.0).
 * Synchronous (returns after the transform is complete). */
int sgtk_graph_create(const uint64_t* node_pointer, const uint32_t* edge_list,
                      const float* values, uint64_t num_nodes,
                      uint64_t num_edges, uint32_t blk_h, uint32_t blk_w,
                      int ptr_kind, void* stream, sgtk_graph** out);

/* Row-slice variant for the multi-GPU row-window partition: `num_rows` local
 * rows, global rows [row_offset, row_offset + num_rows) (row_offset a multiple
 * of 16: whole windows, so the slice's transform equals the global transform
 * restricted to it), whose column ids index a `num_cols`-row feature replica.
 * Kernels write local rows; feature reads use global ids. */
int sgtk_graph_create_rows(const uint64_t* node_pointer,
                           const uint32_t* edge_list, const float* values,
                           uint64_t num_rows, uint64_t num_cols,
                           uint64_t row_offset, uint64_t num_edges,
                           uint32_t blk_h, uint32_t blk_w, int ptr_kind,
                           void* stream, sgtk_graph** out);

/* Build from an already-transformed graph's host fields (load_sgt output or a
 * host TransformedGraph).  Fields are trusted to be consistent with the CSR;
 * they are copied, not recomputed (this is how the C++ drop-in re-enters). */
int sgtk_graph_import(const uint64_t* node_pointer, const uint32_t* edge_list,
                      const float* values, uint64_t num_nodes,
                      uint64_t num_edges, uint32_t blk_h, uint32_t blk_w,
                      const uint32_t* edge_to_column,
                      const uint64_t* window_offsets,
                      const uint32_t* window_unique_cols, void* stream,
                      sgtk_graph** out);

/* Panel section (the 128-row panel formats the tcgen05 kernels run on),
 * persisted beside an SGT1 file (sgt_file.cpp:47-107; SGT1 itself stays
 * byte-compatible with the reference, whose reader rejects trailing bytes):
 * "<file>.sgp" = magic "SGP1", version, graph fingerprint, both panel
 * formats.  save writes g's formats; import_panels is sgtk_graph_import that
 * loads them from `panel_section` when it matches this graph (skipping the
 * panel build) and builds them otherwise; panels_loaded reports which. */
int sgtk_graph_save_panels(const sgtk_graph* g, const char* path, void* stream);
int sgtk_graph_import_panels(const uint64_t* node_pointer, const uint32_t* edge_list,
                             const float* values, uint64_t num_nodes,
                             uint64_t num_edges, uint32_t blk_h, uint32_t blk_w,
                             const uint32_t* edge_to_column,
                             const uint64_t* window_offsets,
                             const uint32_t* window_unique_cols,
                             const char* panel_section, void* stream,
                             sgtk_graph** out);
int sgtk_graph_panels_loaded(const sgtk_graph* g, int* loaded);

void sgtk_graph_destroy(sgtk_graph* g);

/* Sizes: {num_nodes, num_edges, num_windows, unique_cols, block_counter,
 *         blk_h, blk_w, has_values, tiles8, tiles16, work_units8} */
int sgtk_graph_info(const sgtk_graph* g, uint64_t info[11]);
/* Host wall time (ms) of each construction stage of g: upload, validate,
 * edge_to_row, windows (user geometry), windows (16-row), tiles + work units,
 * panel formats, 0.  Recorded only when the process sets SGTK_BUILD_TIMING
 * (the build then synchronises at every stage boundary); zeros otherwise. */
int sgtk_graph_build_times(const sgtk_graph* g, double ms[8]);

/* Device pointers to the resident fields (read-only views; any may be NULL
 * for an empty graph).  Layout of `ptrs`:
 *  [0] node_pointer u64[N+1]  [1] edge_list u32[E]   [2] values f32[E]|NULL
 *  [3] edge_to_row u32[E]     [4] edge_to_column u32[E]
 *  [5] block_partition u32[W] [6] window_offsets u64[W+1]
 *  [7] window_unique_cols u32[U] */
int sgtk_graph_device_ptrs(const sgtk_graph* g, const void* ptrs[8]);

/* Download the TransformedGraph fields (sgt_transform.hpp:21-37) into host
 * buffers sized from sgtk_graph_info.  Any pointer may be NULL to skip it. */
int sgtk_graph_download(const sgtk_graph* g, uint32_t* edge_to_row,
                        uint32_t* edge_to_column, uint32_t* block_partition,
                        uint64_t* window_offsets, uint32_t* window_unique_cols);

/* 128-row panel format behind the default-plan SpMM (no reference
 * counterpart: it is the device layout that replaces the reference's
 * per-window dense chunk staging, tile_exec.cpp:226-290).
 * info = {panels, dense_chunks, dense_entries (padded), sparse_edges,
 *         max_chunk_entries, dense_columns (padded), hub_rows, hub_segments} */
int sgtk_panel_info(const sgtk_graph* g, uint64_t info[8]);
/* The same for the format an operation of feature width d runs on: d <= 32
 * uses a second format whose tensor-core columns need >= 3 edges in the
 * panel (sgtk_panel_info / sgtk_panel_download describe the >= 2 one). */
int sgtk_panel_info_for(const sgtk_graph* g, uint64_t d, uint64_t info[8]);

/* Timing experiments only: 0 = normal; 1 = tensor-core (dense) part of the
 * panel kernels only; 2 = CUDA-core (sparse) part only (partial results). */
int sgtk_debug_set(int mode);

/* Download the panel arrays (sizes from sgtk_panel_info; any may be NULL):
 * chunk_ptr u32[P+1], dense_cols u32[32*chunks], chunk_off u64[chunks+1],
 * dense_entries u32[entries] (tf32 value | skip<<12 | row<<5 | col),
 * sparse_ptr u32[N+1], sparse_entries u32[2*sparse] (column, value bits). */
int sgtk_panel_download(const sgtk_graph* g, uint32_t* chunk_ptr, uint32_t* dense_cols,
                        uint64_t* chunk_off, uint32_t* dense_entries, uint32_t* sparse_ptr,
                        uint32_t* sparse_entries);

/* reblock (sgt_transform.hpp:55, sgt_transform.cpp:79-91): a new handle that
 * shares nothing with `g` observable by the caller; block_partition and
 * block_counter recomputed at `blk_w`, edge maps unchanged. */
int sgtk_graph_reblock(const sgtk_graph* g, uint32_t blk_w, void* stream,
                       sgtk_graph** out);

/* block_stats (sgt_transform.hpp:57): {block_counter, capacity, nnz}, density. */
int sgtk_block_stats(const sgtk_graph* g, uint64_t stats[3], double* density);

/* make_split_plan (tile_exec.hpp:29, tile_exec.cpp:150-161): host array
 * cut[W] = floor(ratio * block_partition[w]); SGTK_ERR_RANGE unless
 * 0 <= ratio <= 1 (NaN rejected). */
int sgtk_split_plan(const sgtk_graph* g, double ratio, uint32_t* cut_host);

/* gather_tile (tile_exec.hpp:39-40, tile_exec.cpp:163-198), host outputs:
 * a_tile f32[blk_h*blk_w], x_index u32[blk_w] (sentinel = num_nodes). */
int sgtk_gather_tile(const sgtk_graph* g, uint64_t window, uint64_t tile,
                     float* a_tile, uint32_t* x_index);

/* ------------------------------------------------------------------------
 * Kernels (device pointers, asynchronous on `stream`).
 *   cut_dev: per-window tile cut of the graph's geometry (make_split_plan);
 *            NULL = every tile on the tensor-core path (ratio 1.0).
 *   edge_values_dev: f32[E] in CSR edge order overriding the stored values;
 *            NULL = stored values (or 1.0 when the graph is unweighted).
 *   nonfinite_dev: optional u32 flag set to 1 when any output is NaN/Inf
 *            (the reference raises NonFiniteError, tile_exec.cpp:311-312).
 * ---------------------------------------------------------------------- */

/* spmm_hybrid (tile_exec.hpp:48-51): out[N x d] = A * x. */
int sgtk_spmm(const sgtk_graph* g, const float* x_dev, uint64_t ldx,
              uint64_t d, const uint32_t* cut_dev,
              const float* edge_values_dev, int precision, float* out_dev,
              uint64_t ldo, uint32_t* nonfinite_dev, void* stream);

/* sddmm_hybrid (tile_exec.hpp:57-60): out[e] = a_e * <x[row e], y[col e]>,
 * CSR edge order.  Uses the graph's 16-wide tiles regardless of blk_w (the
 * reference callers reblock to 16 first, gnn.cpp:101-112).  `scale` multiplies
 * every output (1.0 for the plain API; beta inside AGNN). */
int sgtk_sddmm(const sgtk_graph* g, const float* x_dev, uint64_t ldx,
               const float* y_dev, uint64_t ldy, uint64_t d,
               const uint32_t* cut16_dev, const float* edge_values_dev,
               int precision, float scale, float* out_dev, void* stream);

/* edge_softmax (gnn.hpp:31, gnn.cpp:54-72): row-wise softmax of CSR-ordered
 * logits (in-place allowed: out_dev == logits_dev). */
int sgtk_edge_softmax(const sgtk_graph* g, const float* logits_dev,
                      float* out_dev, void* stream);

/* In-place ReLU of a row-major device matrix (GCN activation, gnn.cpp:45-47;
 * used by the multi-GPU A (h W) layer order after the aggregation). */
int sgtk_relu_inplace(float* x_dev, uint64_t rows, uint64_t cols, uint64_t ld,
                      void* stream);

/* edge_softmax on a bare device CSR (no transform needed): node_pointer_dev
 * u64[n+1]; gnn.cpp:54-72 takes a CsrGraph, not a TransformedGraph. */
int sgtk_csr_softmax(const uint64_t* node_pointer_dev, uint64_t num_nodes,
                     const float* logits_dev, float* out_dev, void* stream);

/* l2_normalize_rows (gnn.hpp:45-46, gnn.cpp:74-91).  z_dev may be NULL (only
 * inv_norm_dev f32[rows] = float(1/sqrt(sum h^2)), 0 for zero rows, is written);
 * zero_rows_dev (u64, accumulated, may be NULL) counts all-zero rows. */
int sgtk_l2_normalize_rows(const float* h_dev, uint64_t rows, uint64_t cols,
                           uint64_t ldh, float* z_dev, uint64_t ldz,
                           float* inv_norm_dev, uint64_t* zero_rows_dev,
                           void* stream);

/* Dense update (gnn.cpp:16-29, file-static `matmul`):
 * out[m x n] = relu?(a[m x k] * w[k x n]).  fp32 / tf32 on tensor cores. */
int sgtk_gemm(const float* a_dev, uint64_t lda, const float* w_dev,
              uint64_t m, uint64_t k, uint64_t n, int relu, int precision,
              float* out_dev, uint64_t ldo, void* stream);

/* ------------------------------------------------------------------------
 * Models (device pointers; weights f32 row-major [d_l x d_{l+1}] concatenated).
 * ---------------------------------------------------------------------- */

/* gcn_forward (gnn.hpp:24-27, gnn.cpp:33-52): per layer
 * h <- relu?(A h W).  `order`: 0 = reference order (A h) W, 1 = A (h W),
 * 2 = automatic (fewer bytes).  ws_dev: workspace of sgtk_gcn_workspace bytes.
 * Returns SGTK_ERR_NONFINITE (after synchronising) if the output has NaN/Inf. */
int sgtk_gcn_forward(const sgtk_graph* g, const float* x_dev, uint64_t ldx,
                     uint32_t num_layers, const uint64_t* dims_host,
                     const float* weights_dev, const int* relu_host,
                     const uint32_t* cut_dev, int precision, int order,
                     void* ws_dev, uint64_t ws_bytes, float* out_dev,
                     uint64_t ldo, void* stream);
/* The same, asynchronous: no synchronisation, no SGTK_ERR_NONFINITE; a NaN/Inf
 * output sets *nonfinite_dev (u32, device, zeroed by the caller) to 1 instead
 * (capturable in a CUDA graph). */
int sgtk_gcn_forward_async(const sgtk_graph* g, const float* x_dev, uint64_t ldx,
                           uint32_t num_layers, const uint64_t* dims_host,
                           const float* weights_dev, const int* relu_host,
                           const uint32_t* cut_dev, int precision, int order,
                           void* ws_dev, uint64_t ws_bytes, float* out_dev,
                           uint64_t ldo, uint32_t* nonfinite_dev, void* stream);
uint64_t sgtk_gcn_workspace(const sgtk_graph* g, uint32_t num_layers,
                            const uint64_t* dims_host);

/* agnn_forward (gnn.hpp:38-42, gnn.cpp:93-119): per layer
 * z = l2norm(h); attn = softmax_row(beta * <z_i, z_j>); h <- attn h.
 * mode 0 = the reference chain (SDDMM -> softmax -> SpMM, three kernels,
 * attention materialised); mode 1 = fused single-pass sparse attention
 * (online softmax per 16-row window, attention never written to HBM);
 * mode 2 = 128-row panels: tensor-core attention over each panel's dense
 * columns + CUDA-core attention over its singleton columns, concurrently,
 * next layer's l2 norm fused (falls back to mode 1 for |beta| > 40 or an
 * explicit partial plan, to mode 0 for d > 64); mode 3 = auto: mode 2 for
 * graphs with >= 2M edges, else mode 1 (one launch per layer wins on small
 * graphs).  The Python API and the C++ drop-in default to mode 3.
 * zero_rows_host (may be NULL) receives the zero-norm row count; with it the
 * call synchronises and returns SGTK_ERR_NONFINITE when the output holds NaN/Inf
 * (gnn.cpp:115 -> tile_exec.cpp:311-312).  Without it the call is asynchronous
 * and unchecked (as sgtk_spmm without a nonfinite pointer). */
int sgtk_agnn_forward(const sgtk_graph* g, const float* x_dev, uint64_t ldx,
                      uint64_t d, uint32_t num_layers, const float* betas_host,
                      const uint32_t* cut_dev, int precision, int mode,
                      void* ws_dev, uint64_t ws_bytes, float* out_dev,
                      uint64_t ldo, uint64_t* zero_rows_host, void* stream);
uint64_t sgtk_agnn_workspace(const sgtk_graph* g, uint64_t d);

/* ------------------------------------------------------------------------
 * Preprocessing (next row of SURVEY §8f) and utilities.
 * ---------------------------------------------------------------------- */

/* gcn_normalize_values (graph_io.hpp:39, graph_io.cpp:261-277) on device:
 * vals_dev[e] = float(isd[row] * isd[col]) with isd = 1/sqrt(double deg);
 * SGTK_ERR_DEGREE on an empty row (syncs to report). */
int sgtk_gcn_normalize_values(const uint64_t* node_pointer_dev,
                              const uint32_t* edge_list_dev,
                              uint64_t num_nodes, float* vals_dev,
                              void* stream);

/* normalize_graph (graph_io.hpp:33, graph_io.cpp:195-259) on the GPU:
 * dedupe (values summed in input order), symmetrize (missing reverse edges
 * take the forward value), add_self_loops (missing (i,i), value 1.0), result
 * sorted-unique CSR; bit-exact with the reference.  `values` may be NULL.
 * Synchronous; the result is an opaque device CSR. */
typedef struct sgtk_csr sgtk_csr;
int sgtk_normalize_graph(const uint64_t* node_pointer, const uint32_t* edge_list,
                         const float* values, uint64_t num_nodes, uint64_t num_edges,
                         int symmetrize, int add_self_loops, int dedupe,
                         int ptr_kind, void* stream, sgtk_csr** out);
/* {num_nodes, num_edges, has_values} */
int sgtk_csr_info(const sgtk_csr* c, uint64_t info[3]);
/* host copies (vals ignored when the graph is unweighted; any may be NULL) */
int sgtk_csr_download(const sgtk_csr* c, uint64_t* node_pointer,
                      uint32_t* edge_list, float* values);
/* device views: [0] node_pointer [1] edge_list [2] values|NULL */
int sgtk_csr_device_ptrs(const sgtk_csr* c, const void* ptrs[3]);
void sgtk_csr_destroy(sgtk_csr* c);

/* tf32_round_value (tile_exec.hpp:64, tile_exec.cpp:131-142), device,
 * elementwise, in-place allowed. */
int sgtk_tf32_round(const float* in_dev, float* out_dev, uint64_t n,
                    void* stream);

/* Host-buffer end-to-end entry points (pinned host memory recommended): the
 * call a reference-side FFI binding makes.  Copies inputs H2D, runs, copies
 * the result D2H, synchronises.  Workspace is owned by the graph handle. */
int sgtk_gcn_forward_host(const sgtk_graph* g, const float* x_host,
                          uint32_t num_layers, const uint64_t* dims_host,
                          const float* weights_host, const int* relu_host,
                          double ratio, int precision, float* out_host,
                          void* stream);
int sgtk_agnn_forward_host(const sgtk_graph* g, const float* x_host,
                           uint64_t d, uint32_t num_layers,
                           const float* betas_host, double ratio,
                           int precision, int mode, float* out_host,
                           uint64_t* zero_rows_host, void* stream);
int sgtk_spmm_host(const sgtk_graph* g, const float* x_host, uint64_t d,
                   double ratio, int precision, const float* edge_values_host,
                   float* out_host, void* stream);

/* ------------------------------------------------------------------------
 * Multi-GPU row-window partition (one process per GPU, NCCL over NVLink).
 * ---------------------------------------------------------------------- */

/* Split [0, num_windows) into `parts` contiguous window ranges balanced by
 * edge count (window boundaries are multiples of 16 rows, so each part's
 * transform equals the global transform restricted to it).
 * bounds_host: u64[parts+1] window indices. */
int sgtk_partition_windows(const uint64_t* node_pointer_host,
                           uint64_t num_nodes, uint32_t blk_h, uint32_t parts,
                           uint64_t* bounds_host);

/* ------------------------------------------------------------------------
 * Synthetic inputs (bench / tests; the reference's synthetic.cpp is O(n^2)).
 * ---------------------------------------------------------------------- */

/* Deterministic O(E) generator: symmetric, sorted-unique CSR with self-loops.
 * Each node draws `k` neighbour picks, k ~ Pareto(alpha) scaled to mean
 * `avg_picks` (alpha <= 0: Poisson-like around the mean); each pick lands
 * within +-ceil(band * avg_picks) ids with probability `p_local`, else
 * uniformly.  Reverse edges are added, duplicates dropped, self-loops added.
 * Output is independent of the thread count. */
typedef struct sgtk_synth sgtk_synth;
int sgtk_synth_create(uint64_t num_nodes, double avg_picks, double alpha,
                      double p_local, double band, uint64_t seed,
                      sgtk_synth** out);
int sgtk_synth_info(const sgtk_synth* s, uint64_t* num_nodes,
                    uint64_t* num_edges);
int sgtk_synth_copy(const sgtk_synth* s, uint64_t* node_pointer,
                    uint32_t* edge_list);
void sgtk_synth_destroy(sgtk_synth* s);

/* DenseMatrix::random (dense_matrix.hpp:43-50): mt19937_64(seed) with the
 * standard uniform_real_distribution<float>(lo, hi), row-major rows x cols. */
void sgtk_dense_random(uint64_t rows, uint64_t cols, uint64_t seed, float lo,
                       float hi, float* out_host);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif

#endif /* SGTK_CUDA_H_ */
