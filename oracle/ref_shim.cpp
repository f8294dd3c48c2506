// TEST INFRASTRUCTURE ONLY — never linked into the product library.
//
// A flat extern "C" face over the UNMODIFIED reference sources under
// /root/reference/proj/src, so pytest (ctypes) can (a) generate golden
// vectors from the real reference and (b) time the reference CPU path as the
// bench's `--impl reference` arm and `cpu_baseline`.  Built by oracle/Makefile
// into oracle/_ref/libsgtk_ref.so with the reference's own Release flags
// (-O3 -DNDEBUG -fopenmp, no -march; /root/reference/proj/CMakeLists.txt:7-13)
// and the namespace renamed (-Dsgtk=sgtk_ref) so it can never interpose the
// drop-in's identically named sgtk:: symbols.
//
// Every entry returns a status code (see include/sgtk_cuda.h, SGTK_ERR_*) and
// stores the exception message for ref_last_error().

#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "sgtk/errors.hpp"
#include "sgtk/gnn.hpp"
#include "sgtk/graph_io.hpp"
#include "sgtk/oracle.hpp"
#include "sgtk/sgt_file.hpp"
#include "sgtk/threading.hpp"
#include "sgtk/sgt_transform.hpp"
#include "sgtk/tile_exec.hpp"

using namespace sgtk;

namespace {

thread_local std::string g_msg;

// Status codes shared with include/sgtk_cuda.h.
enum : int {
  kOk = 0, kErr = 1, kIo = 2, kParse = 3, kOverflow = 4, kDegree = 5,
  kGeometry = 6, kIndex = 7, kRange = 8, kShape = 9, kNonFinite = 10,
};

template <class F>
int guard(F&& f) {
  try {
    f();
    return kOk;
  } catch (const ParseError& e) { g_msg = e.what(); return kParse; }
  catch (const IoError& e) { g_msg = e.what(); return kIo; }
  catch (const OverflowError& e) { g_msg = e.what(); return kOverflow; }
  catch (const DegreeError& e) { g_msg = e.what(); return kDegree; }
  catch (const GeometryError& e) { g_msg = e.what(); return kGeometry; }
  catch (const IndexError& e) { g_msg = e.what(); return kIndex; }
  catch (const RangeError& e) { g_msg = e.what(); return kRange; }
  catch (const ShapeError& e) { g_msg = e.what(); return kShape; }
  catch (const NonFiniteError& e) { g_msg = e.what(); return kNonFinite; }
  catch (const Error& e) { g_msg = e.what(); return kErr; }
  catch (const std::exception& e) { g_msg = e.what(); return kErr; }
}

CsrGraph csr_of(uint64_t n, const uint64_t* np, const uint32_t* el,
                const float* vals, uint64_t nnz) {
  CsrGraph g;
  g.num_nodes = n;
  g.node_pointer.assign(np, np + n + 1);
  g.edge_list.assign(el, el + nnz);
  if (vals) g.values.assign(vals, vals + nnz);
  return g;
}

DenseMatrix mat_of(const float* p, uint64_t r, uint64_t c) {
  DenseMatrix m(r, c);
  if (r * c) std::memcpy(m.data.data(), p, r * c * sizeof(float));
  return m;
}

void put(const DenseMatrix& m, float* out) {
  if (!m.data.empty())
    std::memcpy(out, m.data.data(), m.data.size() * sizeof(float));
}

std::span<const float> span_of(const float* p, uint64_t n) {
  return p ? std::span<const float>(p, n) : std::span<const float>();
}

Precision prec_of(int p) { return p == 1 ? Precision::Tf32 : Precision::Fp32; }

}  // namespace

extern "C" {

const char* ref_last_error() { return g_msg.c_str(); }

// ---- CSR handles (normalize_graph / gcn_normalize_values) ----------------
int ref_csr_create(uint64_t n, const uint64_t* np, const uint32_t* el,
                   const float* vals, uint64_t nnz, void** out) {
  return guard([&] { *out = new CsrGraph(csr_of(n, np, el, vals, nnz)); });
}
void ref_csr_free(void* h) { delete static_cast<CsrGraph*>(h); }
// counts = {num_nodes, num_edges, has_values}
void ref_csr_counts(void* h, uint64_t* counts) {
  auto* g = static_cast<CsrGraph*>(h);
  counts[0] = g->num_nodes;
  counts[1] = g->num_edges();
  counts[2] = g->has_values() ? 1 : 0;
}
void ref_csr_get(void* h, uint64_t* np, uint32_t* el, float* vals) {
  auto* g = static_cast<CsrGraph*>(h);
  std::memcpy(np, g->node_pointer.data(), g->node_pointer.size() * 8);
  if (!g->edge_list.empty())
    std::memcpy(el, g->edge_list.data(), g->edge_list.size() * 4);
  if (vals && g->has_values())
    std::memcpy(vals, g->values.data(), g->values.size() * 4);
}
int ref_validate_csr(void* h, int sorted_unique) {
  return guard([&] { validate_csr(*static_cast<CsrGraph*>(h), sorted_unique); });
}
int ref_normalize_graph(void* h, int symmetrize, int loops, int dedupe,
                        void** out) {
  return guard([&] {
    NormalizeOpts o;
    o.symmetrize = symmetrize;
    o.add_self_loops = loops;
    o.dedupe = dedupe;
    *out = new CsrGraph(normalize_graph(*static_cast<CsrGraph*>(h), o));
  });
}
int ref_gcn_normalize_values(void* h, void** out) {
  return guard([&] {
    *out = new CsrGraph(gcn_normalize_values(*static_cast<CsrGraph*>(h)));
  });
}

// ---- TransformedGraph handles --------------------------------------------
int ref_transform(void* csr, uint32_t blk_h, uint32_t blk_w, int threads,
                  void** out) {
  return guard([&] {
    *out = new TransformedGraph(
        sgt_transform(*static_cast<CsrGraph*>(csr), {blk_h, blk_w}, threads));
  });
}
int ref_reblock(void* t, uint32_t blk_w, void** out) {
  return guard([&] {
    *out = new TransformedGraph(
        reblock(*static_cast<TransformedGraph*>(t), blk_w));
  });
}
void ref_graph_free(void* h) { delete static_cast<TransformedGraph*>(h); }
// counts = {num_nodes, num_edges, num_windows, unique, block_counter, blk_h, blk_w}
void ref_graph_counts(void* h, uint64_t* c) {
  auto* t = static_cast<TransformedGraph*>(h);
  c[0] = t->csr.num_nodes;
  c[1] = t->csr.num_edges();
  c[2] = t->num_windows();
  c[3] = t->window_unique_cols.size();
  c[4] = t->block_counter;
  c[5] = t->geometry.blk_h;
  c[6] = t->geometry.blk_w;
}
void ref_graph_fields(void* h, uint32_t* e2r, uint32_t* e2c, uint32_t* bp,
                      uint64_t* wo, uint32_t* wuc) {
  auto* t = static_cast<TransformedGraph*>(h);
  auto cp = [](void* dst, const auto& v) {
    if (!v.empty()) std::memcpy(dst, v.data(), v.size() * sizeof(v[0]));
  };
  cp(e2r, t->edge_to_row);
  cp(e2c, t->edge_to_column);
  cp(bp, t->block_partition);
  cp(wo, t->window_offsets);
  cp(wuc, t->window_unique_cols);
}
// stats = {block_counter, capacity, nnz}; density separately
void ref_block_stats(void* h, uint64_t* s, double* density) {
  BlockStats b = block_stats(*static_cast<TransformedGraph*>(h));
  s[0] = b.block_counter;
  s[1] = b.capacity;
  s[2] = b.nnz;
  *density = b.mean_tile_density;
}
int ref_split_plan(void* h, double ratio, uint32_t* cut) {
  return guard([&] {
    HybridSplitPlan p = make_split_plan(*static_cast<TransformedGraph*>(h), ratio);
    std::memcpy(cut, p.per_window_tile_cut.data(),
                p.per_window_tile_cut.size() * 4);
  });
}
int ref_gather_tile(void* h, uint64_t w, uint64_t tile, float* a,
                    uint32_t* idx) {
  return guard([&] {
    GatheredTile g = gather_tile(*static_cast<TransformedGraph*>(h), w, tile);
    put(g.a_tile, a);
    std::memcpy(idx, g.x_index.data(), g.x_index.size() * 4);
  });
}

// ---- kernels ----------------------------------------------------------------
static HybridSplitPlan plan_of(const TransformedGraph& t, double ratio,
                               const uint32_t* cut) {
  HybridSplitPlan p = make_split_plan(t, ratio < 0 ? 1.0 : ratio);
  if (cut) p.per_window_tile_cut.assign(cut, cut + t.num_windows());
  return p;
}

int ref_spmm(void* h, const float* x, uint64_t d, double ratio,
             const uint32_t* cut, int prec, int threads, const float* ev,
             uint64_t ev_len, float* out) {
  return guard([&] {
    auto& t = *static_cast<TransformedGraph*>(h);
    DenseMatrix xm = mat_of(x, t.csr.num_nodes, d);
    put(spmm_hybrid(t, xm, plan_of(t, ratio, cut), prec_of(prec), threads,
                    span_of(ev, ev_len)),
        out);
  });
}
int ref_sddmm(void* h, const float* x, const float* y, uint64_t d,
              double ratio, const uint32_t* cut, int prec, int threads,
              const float* ev, uint64_t ev_len, float* out) {
  return guard([&] {
    auto& t = *static_cast<TransformedGraph*>(h);
    DenseMatrix xm = mat_of(x, t.csr.num_nodes, d);
    DenseMatrix ym = mat_of(y, t.csr.num_nodes, d);
    EdgeValList v = sddmm_hybrid(t, xm, ym, plan_of(t, ratio, cut),
                                 prec_of(prec), threads, span_of(ev, ev_len));
    if (!v.empty()) std::memcpy(out, v.data(), v.size() * 4);
  });
}
int ref_edge_softmax(void* csr, const float* logits, uint64_t len,
                     float* out) {
  return guard([&] {
    EdgeValList l(logits, logits + len);
    EdgeValList v = edge_softmax(*static_cast<CsrGraph*>(csr), l);
    if (!v.empty()) std::memcpy(out, v.data(), v.size() * 4);
  });
}
int ref_l2_normalize_rows(const float* m, uint64_t r, uint64_t c, float* out,
                          uint64_t* zeros) {
  return guard([&] {
    std::size_t z = 0;
    put(l2_normalize_rows(mat_of(m, r, c), &z), out);
    if (zeros) *zeros = z;
  });
}
// Layers: dims[0..L] chain, weights concatenated row-major, relu[L].
int ref_gcn_forward(void* h, const float* x, uint32_t nlayers,
                    const uint64_t* dims, const float* weights,
                    const int* relu, double ratio, int prec, int threads,
                    float* out) {
  return guard([&] {
    auto& t = *static_cast<TransformedGraph*>(h);
    std::vector<GcnLayerParams> layers;
    const float* w = weights;
    for (uint32_t l = 0; l < nlayers; ++l) {
      layers.push_back({mat_of(w, dims[l], dims[l + 1]), relu[l] != 0});
      w += dims[l] * dims[l + 1];
    }
    DenseMatrix xm = mat_of(x, t.csr.num_nodes, dims[0]);
    put(gcn_forward(t, xm, layers, make_split_plan(t, ratio), prec_of(prec),
                    threads),
        out);
  });
}
int ref_agnn_forward(void* h, const float* x, uint64_t d, uint32_t nlayers,
                     const float* betas, double ratio, int prec, int threads,
                     float* out, uint64_t* zeros) {
  return guard([&] {
    auto& t = *static_cast<TransformedGraph*>(h);
    std::vector<AgnnLayerParams> layers;
    for (uint32_t l = 0; l < nlayers; ++l) layers.push_back({betas[l]});
    std::size_t z = 0;
    put(agnn_forward(t, mat_of(x, t.csr.num_nodes, d), layers,
                     make_split_plan(t, ratio), prec_of(prec), threads, &z),
        out);
    if (zeros) *zeros = z;
  });
}
int ref_oracle_spmm(void* csr, const float* x, uint64_t d, float* out) {
  return guard([&] {
    auto& g = *static_cast<CsrGraph*>(csr);
    put(oracle_spmm(g, mat_of(x, g.num_nodes, d)), out);
  });
}
int ref_oracle_sddmm(void* csr, const float* x, const float* y, uint64_t d,
                     float* out) {
  return guard([&] {
    auto& g = *static_cast<CsrGraph*>(csr);
    EdgeValList v = oracle_sddmm(g, mat_of(x, g.num_nodes, d),
                                 mat_of(y, g.num_nodes, d));
    if (!v.empty()) std::memcpy(out, v.data(), v.size() * 4);
  });
}
float ref_tf32_round_value(float v) { return tf32_round_value(v); }
// DenseMatrix::random(r, c, seed, lo, hi) — the reference's seeded fill.
void ref_dense_random(uint64_t r, uint64_t c, uint64_t seed, float lo,
                      float hi, float* out) {
  put(DenseMatrix::random(r, c, seed, lo, hi), out);
}

// random_gcn_layers(in, hidden, out, L, seed) (gnn.cpp:121-137): weights
// concatenated row-major, relu flags.
int ref_random_gcn_layers(uint64_t in_dim, uint64_t hidden, uint64_t out_dim,
                          uint32_t nlayers, uint64_t seed, float* weights,
                          int* relu) {
  return guard([&] {
    auto layers = random_gcn_layers(in_dim, hidden, out_dim, nlayers, seed);
    float* w = weights;
    for (uint32_t l = 0; l < layers.size(); ++l) {
      put(layers[l].weight, w);
      w += layers[l].weight.data.size();
      relu[l] = layers[l].apply_relu ? 1 : 0;
    }
  });
}
// resolve_thread_count(0) (threading.cpp:9-22): the worker count the
// reference's kernels use by default (SGTK_THREADS, else OpenMP's max).
int ref_resolve_threads(int requested) { return resolve_thread_count(requested); }
// save_sgt / load_sgt (sgt_file.cpp:47-107): the reference's SGT1 writer and
// reader, for byte-compatibility fixtures.
int ref_save_sgt(void* h, const char* path) {
  return guard([&] { save_sgt(*static_cast<TransformedGraph*>(h), path); });
}
int ref_load_sgt(const char* path, void** out) {
  return guard([&] { *out = new TransformedGraph(load_sgt(path)); });
}

}  // extern "C"
