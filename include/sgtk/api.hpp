// sgtk C++ drop-in: the reference's public interface
// (/root/reference/proj/include/sgtk/*.hpp) implemented over the sm_100a C ABI
// (include/sgtk_cuda.h).  Same namespace, type names, signatures, defaults and
// exception types, so code written against the reference compiles unchanged
// and links against libsgtk_b200.so instead.  Every kernel runs on the GPU;
// these functions validate on the host (so the reference's exception types
// surface before any launch), move host data, and call the C ABI.
//
// The per-module headers (sgtk/csr_graph.hpp, sgtk/tile_exec.hpp, ...) all
// include this one.
#pragma once

#include <cmath>
#include <cstddef>
#include <cstdint>
#include <memory>
#include <random>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#if defined(__GNUC__)
#define SGTK_VISIBLE __attribute__((visibility("default")))
#else
#define SGTK_VISIBLE
#endif

namespace sgtk {

// ---------------------------------------------------------------- errors.hpp
// (exported type info so handlers in user code match across the .so boundary)
struct SGTK_VISIBLE Error : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct SGTK_VISIBLE IoError : Error { using Error::Error; };
struct SGTK_VISIBLE ParseError : Error {
  ParseError(const std::string& msg, std::size_t line_no)
      : Error(msg + " (line " + std::to_string(line_no) + ")"), line(line_no) {}
  std::size_t line;
};
struct SGTK_VISIBLE OverflowError : Error { using Error::Error; };
struct SGTK_VISIBLE DegreeError : Error { using Error::Error; };
struct SGTK_VISIBLE GeometryError : Error { using Error::Error; };
struct SGTK_VISIBLE IndexError : Error { using Error::Error; };
struct SGTK_VISIBLE RangeError : Error { using Error::Error; };
struct SGTK_VISIBLE ShapeError : Error { using Error::Error; };
struct SGTK_VISIBLE NonFiniteError : Error { using Error::Error; };

// ------------------------------------------------------------- csr_graph.hpp
using NodeId = std::uint32_t;

struct CsrGraph {
  std::size_t num_nodes = 0;
  std::vector<std::uint64_t> node_pointer{0};
  std::vector<NodeId> edge_list;
  std::vector<float> values;  // empty = unweighted (every edge 1.0)

  std::size_t num_edges() const { return edge_list.size(); }
  bool has_values() const { return !values.empty(); }
  std::uint64_t row_begin(std::size_t r) const { return node_pointer[r]; }
  std::uint64_t row_end(std::size_t r) const { return node_pointer[r + 1]; }
  std::size_t degree(std::size_t r) const { return std::size_t(row_end(r) - row_begin(r)); }
  float edge_value(std::size_t e) const { return values.empty() ? 1.0f : values[e]; }
};

void validate_csr(const CsrGraph& g, bool require_sorted_unique = true);

struct Triple {
  NodeId row;
  NodeId col;
  float value;
};

CsrGraph csr_from_triples(std::size_t num_nodes, std::vector<Triple> triples, bool with_values);

// ---------------------------------------------------------- dense_matrix.hpp
struct DenseMatrix {
  std::size_t rows = 0;
  std::size_t cols = 0;
  std::vector<float> data;

  DenseMatrix() = default;
  DenseMatrix(std::size_t r, std::size_t c, float fill = 0.0f) : rows(r), cols(c), data(r * c, fill) {}

  float& at(std::size_t r, std::size_t c) { return data[r * cols + c]; }
  float at(std::size_t r, std::size_t c) const { return data[r * cols + c]; }
  float* row_ptr(std::size_t r) { return data.data() + r * cols; }
  const float* row_ptr(std::size_t r) const { return data.data() + r * cols; }

  bool all_finite() const {
    for (float v : data)
      if (!std::isfinite(v)) return false;
    return true;
  }
  bool same_shape(const DenseMatrix& o) const { return rows == o.rows && cols == o.cols; }

  // Same stream as the reference: mt19937_64(seed) + uniform_real_distribution<float>.
  static DenseMatrix random(std::size_t r, std::size_t c, std::uint64_t seed, float lo = -1.0f,
                            float hi = 1.0f) {
    DenseMatrix m(r, c);
    std::mt19937_64 gen(seed);
    std::uniform_real_distribution<float> u(lo, hi);
    for (float& v : m.data) v = u(gen);
    return m;
  }
};

inline float max_abs(const std::vector<float>& v) {
  float m = 0.0f;
  for (float x : v) m = std::max(m, std::abs(x));
  return m;
}
inline float max_abs(const DenseMatrix& m) { return max_abs(m.data); }

// max_i |a_i - b_i| / max(max|b|, 1e-30)
inline double max_rel_err(const std::vector<float>& a, const std::vector<float>& b) {
  if (a.size() != b.size()) throw ShapeError("max_rel_err: length mismatch");
  double num = 0.0;
  for (std::size_t i = 0; i < a.size(); ++i)
    num = std::max(num, std::abs(double(a[i]) - double(b[i])));
  return num / std::max(double(max_abs(b)), 1e-30);
}
inline double max_rel_err(const DenseMatrix& a, const DenseMatrix& b) {
  if (!a.same_shape(b)) throw ShapeError("max_rel_err: shape mismatch");
  return max_rel_err(a.data, b.data);
}

// --------------------------------------------------------- sgt_transform.hpp
struct TileGeometry {
  std::uint32_t blk_h = 16;
  std::uint32_t blk_w = 8;
};

struct TransformedGraph {
  CsrGraph csr;
  TileGeometry geometry;
  std::vector<NodeId> edge_to_row;
  std::vector<std::uint32_t> edge_to_column;
  std::vector<std::uint32_t> block_partition;
  std::vector<std::uint64_t> window_offsets;
  std::vector<NodeId> window_unique_cols;
  std::uint64_t block_counter = 0;

  std::size_t num_windows() const { return block_partition.size(); }
  std::span<const NodeId> window_cols(std::size_t w) const {
    return {window_unique_cols.data() + window_offsets[w],
            std::size_t(window_offsets[w + 1] - window_offsets[w])};
  }

  // Not in the reference: the device-resident copy (sgtk_graph handle) this
  // transform was produced from / last uploaded to.  Reused by the kernels
  // while the host fields are unchanged; never part of equality.
  mutable std::shared_ptr<void> device;
};

struct BlockStats {
  std::uint64_t block_counter = 0;
  std::uint64_t capacity = 0;
  std::uint64_t nnz = 0;
  double mean_tile_density = 0.0;
};

TransformedGraph sgt_transform(const CsrGraph& g, TileGeometry geom = {}, int threads = 0);
TransformedGraph reblock(const TransformedGraph& t, std::uint32_t new_blk_w);
BlockStats block_stats(const TransformedGraph& t);

// ------------------------------------------------------------- tile_exec.hpp
enum class Precision {
  Fp32,
  Tf32,
};

using EdgeValList = std::vector<float>;

struct HybridSplitPlan {
  double ratio = 1.0;
  std::vector<std::uint32_t> per_window_tile_cut;
};

HybridSplitPlan make_split_plan(const TransformedGraph& t, double ratio = 1.0);

struct GatheredTile {
  DenseMatrix a_tile;
  std::vector<NodeId> x_index;
};

GatheredTile gather_tile(const TransformedGraph& t, std::size_t window, std::size_t tile);

DenseMatrix spmm_hybrid(const TransformedGraph& t, const DenseMatrix& x, const HybridSplitPlan& plan,
                        Precision prec = Precision::Fp32, int threads = 0,
                        std::span<const float> edge_values = {});

EdgeValList sddmm_hybrid(const TransformedGraph& t, const DenseMatrix& x, const DenseMatrix& y,
                         const HybridSplitPlan& plan, Precision prec = Precision::Fp32,
                         int threads = 0, std::span<const float> edge_values = {});

float tf32_round_value(float v);
DenseMatrix tf32_round(const DenseMatrix& m);

// ------------------------------------------------------------------- gnn.hpp
struct GcnLayerParams {
  DenseMatrix weight;
  bool apply_relu = true;
};

struct AgnnLayerParams {
  float beta = 1.0f;
};

DenseMatrix gcn_forward(const TransformedGraph& t, const DenseMatrix& x,
                        const std::vector<GcnLayerParams>& layers, const HybridSplitPlan& plan,
                        Precision prec = Precision::Fp32, int threads = 0);

EdgeValList edge_softmax(const CsrGraph& g, const EdgeValList& logits);

DenseMatrix agnn_forward(const TransformedGraph& t, const DenseMatrix& x,
                         const std::vector<AgnnLayerParams>& layers, const HybridSplitPlan& plan,
                         Precision prec = Precision::Fp32, int threads = 0,
                         std::size_t* zero_norm_rows = nullptr);

DenseMatrix l2_normalize_rows(const DenseMatrix& m, std::size_t* zero_rows = nullptr);

std::vector<GcnLayerParams> random_gcn_layers(std::size_t in_dim, std::size_t hidden_dim,
                                              std::size_t out_dim, std::size_t num_layers,
                                              std::uint64_t seed);

GcnLayerParams load_gcn_layer(const std::string& path);
void save_gcn_layer(const GcnLayerParams& layer, const std::string& path);

// -------------------------------------------------------------- graph_io.hpp
struct NormalizeOpts {
  bool symmetrize = false;
  bool add_self_loops = false;
  bool dedupe = true;
};

CsrGraph normalize_graph(const CsrGraph& g, NormalizeOpts opts);
CsrGraph gcn_normalize_values(const CsrGraph& g);

// -------------------------------------------------------------- sgt_file.hpp
void save_sgt(const TransformedGraph& t, const std::string& path);
TransformedGraph load_sgt(const std::string& path);

}  // namespace sgtk
