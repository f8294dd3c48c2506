// C++ drop-in parity test: code written against the reference's public API
// (/root/reference/proj/include/sgtk/*.hpp), compiled against include/sgtk/
// and linked with libsgtk_b200.so — i.e. what a reference user gets after
// switching.  Cases follow the reference's own test suites (file:line in each
// CASE); the ground truth for random graphs is the CPU oracle
// (oracle/liboracle.so, pinned to the reference's golden vectors).
// Built and run by tests/test_gpu_dropin.py (needs a GPU).

#include <cmath>
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <random>
#include <string>
#include <unistd.h>

#include "sgtk/gnn.hpp"
#include "sgtk_cuda.h"
#include "sgtk/graph_io.hpp"
#include "sgtk/sgt_file.hpp"
#include "sgtk/sgt_transform.hpp"
#include "sgtk/tile_exec.hpp"

extern "C" {  // CPU oracle (test infrastructure only)
int or_spmm(uint64_t, const uint64_t*, const uint32_t*, const float*, const float*, uint64_t, int,
            float*);
int or_sddmm(uint64_t, const uint64_t*, const uint32_t*, const float*, const float*, const float*,
             uint64_t, int, float*);
int or_agnn_forward(uint64_t, const uint64_t*, const uint32_t*, const float*, uint64_t, uint32_t,
                    const float*, int, float*, uint64_t*);
int or_gcn_forward(uint64_t, const uint64_t*, const uint32_t*, const float*, const float*, uint32_t,
                   const uint64_t*, const float*, const int*, int, float*);
int or_normalize_graph(uint64_t, const uint64_t*, const uint32_t*, const float*, int, int, int,
                       uint64_t*, uint64_t*, uint32_t*, float*);
}

using namespace sgtk;

static int g_fail = 0, g_checks = 0;
#define CHECK(c)                                                         \
  do {                                                                   \
    ++g_checks;                                                          \
    if (!(c)) {                                                          \
      ++g_fail;                                                          \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);           \
    }                                                                    \
  } while (0)
#define CHECK_THROWS_AS(expr, T)                                         \
  do {                                                                   \
    bool ok_ = false;                                                    \
    try {                                                                \
      (void)(expr);                                                      \
    } catch (const T&) {                                                 \
      ok_ = true;                                                        \
    } catch (...) {                                                      \
    }                                                                    \
    CHECK(ok_ && #T);                                                    \
  } while (0)

static CsrGraph graph_of(size_t n, std::vector<Triple> t, bool w = false) {
  return csr_from_triples(n, std::move(t), w);
}
static CsrGraph identity_graph(size_t n) {
  std::vector<Triple> t;
  for (size_t i = 0; i < n; ++i) t.push_back({NodeId(i), NodeId(i), 1.0f});
  return graph_of(n, t);
}
static CsrGraph random_graph(size_t n, double deg, uint64_t seed, bool weighted) {
  std::mt19937_64 rng(seed);
  std::vector<Triple> t;
  std::uniform_int_distribution<uint32_t> col(0, uint32_t(n - 1));
  std::uniform_real_distribution<float> val(-1.0f, 1.0f);
  for (size_t r = 0; r < n; ++r)
    for (int k = 0; k < int(deg); ++k) t.push_back({NodeId(r), col(rng), val(rng)});
  CsrGraph g = normalize_graph(graph_of(n, t, weighted), {});  // sorted-unique
  return g;
}
static DenseMatrix oracle_spmm(const CsrGraph& g, const DenseMatrix& x) {
  DenseMatrix o(g.num_nodes, x.cols);
  or_spmm(g.num_nodes, g.node_pointer.data(), g.edge_list.data(),
          g.has_values() ? g.values.data() : nullptr, x.data.data(), x.cols, 0, o.data.data());
  return o;
}

static std::string g_golden = "tests/golden";

int main(int argc, char** argv) {
  if (argc > 1) g_golden = argv[1];
  // --- translator (test_sgt_transform.cpp:47-111, 169-224) ---------------
  {
    TransformedGraph t = sgt_transform(identity_graph(16));
    CHECK(t.num_windows() == 1 && t.window_cols(0).size() == 16);
    CHECK(t.block_partition == std::vector<uint32_t>{2} && t.block_counter == 2);
    for (size_t e = 0; e < 16; ++e) CHECK(t.edge_to_column[e] == uint32_t(e));
    BlockStats s = block_stats(t);
    CHECK(s.capacity == 256 && s.nnz == 16 && std::abs(s.mean_tile_density - 0.0625) < 1e-12);
    TransformedGraph r = reblock(t, 16);
    CHECK(r.block_partition == std::vector<uint32_t>{1} && r.block_counter == 1);
    CHECK(r.edge_to_column == t.edge_to_column);
  }
  {
    TransformedGraph t = sgt_transform(graph_of(31, {{0, 5, 1}, {0, 9, 1}, {1, 5, 1}, {1, 30, 1}}));
    auto c = t.window_cols(0);
    CHECK(t.num_windows() == 2 && c.size() == 3 && c[0] == 5 && c[1] == 9 && c[2] == 30);
    CHECK(t.block_partition[0] == 1 && t.block_partition[1] == 0 && t.block_counter == 1);
    CHECK((t.edge_to_column == std::vector<uint32_t>{0, 1, 0, 2}));
  }
  {
    CsrGraph g = identity_graph(4);
    CHECK_THROWS_AS(sgt_transform(g, {0, 8}), GeometryError);
    CHECK_THROWS_AS(sgt_transform(g, {16, 0}), GeometryError);
    CHECK_THROWS_AS(reblock(sgt_transform(g), 0), GeometryError);
  }
  {  // reconstruction on random graphs, odd geometries
    for (int it = 0; it < 10; ++it) {
      CsrGraph g = random_graph(20 + it * 37, 4, 100 + it, it % 2);
      for (TileGeometry geom : {TileGeometry{16, 8}, TileGeometry{3, 5}, TileGeometry{32, 4}}) {
        TransformedGraph t = sgt_transform(g, geom);
        bool ok = t.num_windows() == (g.num_nodes + geom.blk_h - 1) / geom.blk_h;
        for (size_t r = 0; r < g.num_nodes; ++r)
          for (auto e = g.row_begin(r); e < g.row_end(r); ++e) {
            auto cols = t.window_cols(r / geom.blk_h);
            ok = ok && t.edge_to_row[e] == r && t.edge_to_column[e] < cols.size() &&
                 cols[t.edge_to_column[e]] == g.edge_list[e];
          }
        CHECK(ok);
      }
    }
  }
  {  // SGT1 round trip and corruption (test_sgt_transform.cpp:179-224)
    const auto dir = std::filesystem::temp_directory_path();
    const std::string p = (dir / ("dropin_" + std::to_string(getpid()) + ".sgt")).string();
    for (bool w : {false, true}) {
      TransformedGraph t = sgt_transform(random_graph(300, 6, 13, w));
      save_sgt(t, p);
      TransformedGraph b = load_sgt(p);
      CHECK(b.edge_to_column == t.edge_to_column && b.window_unique_cols == t.window_unique_cols &&
            b.block_partition == t.block_partition && b.csr.values == t.csr.values &&
            b.block_counter == t.block_counter && b.geometry.blk_w == 8);
      // the loaded transform runs on the GPU directly
      DenseMatrix x = DenseMatrix::random(300, 16, 4);
      CHECK(max_rel_err(spmm_hybrid(b, x, make_split_plan(b)), oracle_spmm(b.csr, x)) <= 1e-5);
    }
    std::ifstream in(p, std::ios::binary);
    std::string bytes((std::istreambuf_iterator<char>(in)), {});
    std::ofstream(p + ".t", std::ios::binary) << bytes.substr(0, bytes.size() / 2);
    CHECK_THROWS_AS(load_sgt(p + ".t"), IoError);
    std::ofstream(p + ".g", std::ios::binary) << bytes << "extra";
    CHECK_THROWS_AS(load_sgt(p + ".g"), IoError);
    std::ofstream(p + ".m") << "NOPE";
    CHECK_THROWS_AS(load_sgt(p + ".m"), IoError);
    for (auto s : {"", ".t", ".g", ".m", ".sgp"}) std::filesystem::remove(p + s);
  }
  {  // SGT1 files written by the REFERENCE's save_sgt (tests/golden/ref_*.sgt,
     // make_golden.py --sgt): load_sgt reads them, and save_sgt of what it
     // read reproduces them byte for byte (sgt_file.cpp:47-107)
    for (const char* name : {"ref_rand3_16x8.sgt", "ref_rand0_3x5.sgt"}) {
      const std::string src = g_golden + "/" + name;
      std::ifstream in(src, std::ios::binary);
      CHECK(in.good());
      const std::string want((std::istreambuf_iterator<char>(in)), {});
      TransformedGraph b = load_sgt(src);
      // the same transform from the drop-in's GPU translator
      TransformedGraph t = sgt_transform(b.csr, b.geometry);
      CHECK(b.edge_to_row == t.edge_to_row && b.edge_to_column == t.edge_to_column &&
            b.block_partition == t.block_partition && b.window_offsets == t.window_offsets &&
            b.window_unique_cols == t.window_unique_cols && b.block_counter == t.block_counter);
      const std::string out = (std::filesystem::temp_directory_path() /
                               ("dropin_ref_" + std::to_string(getpid()) + ".sgt")).string();
      save_sgt(b, out);  // b is host-only: SGT1 bytes, no panel section
      std::ifstream o(out, std::ios::binary);
      const std::string got((std::istreambuf_iterator<char>(o)), {});
      CHECK(got == want);
      CHECK(!std::filesystem::exists(out + ".sgp"));
      std::filesystem::remove(out);
    }
  }
  {  // panel section: save_sgt of a device-resident transform writes <file>.sgp;
     // load_sgt imports the panel formats from it (no panel build) and the
     // kernels give bit-identical results to a freshly built handle
    const std::string p = (std::filesystem::temp_directory_path() /
                           ("dropin_sgp_" + std::to_string(getpid()) + ".sgt")).string();
    CsrGraph g = gcn_normalize_values(normalize_graph(random_graph(5000, 24, 77, false),
                                                      {true, true, true}));
    TransformedGraph t = sgt_transform(g);
    save_sgt(t, p);
    CHECK(std::filesystem::exists(p + ".sgp"));
    TransformedGraph b = load_sgt(p);
    DenseMatrix x = DenseMatrix::random(5000, 32, 8);
    for (Precision pr : {Precision::Fp32, Precision::Tf32})
      CHECK(spmm_hybrid(b, x, make_split_plan(b), pr).data ==
            spmm_hybrid(t, x, make_split_plan(t), pr).data);
    // through the C ABI: the handle reports its panels came from the file
    sgtk_graph* h = nullptr;
    const auto& c = b.csr;
    CHECK(sgtk_graph_import_panels(c.node_pointer.data(), c.edge_list.data(), c.values.data(),
                                   c.num_nodes, c.num_edges(), 16, 8, b.edge_to_column.data(),
                                   b.window_offsets.data(), b.window_unique_cols.data(),
                                   (p + ".sgp").c_str(), nullptr, &h) == SGTK_OK);
    int loaded = 0;
    sgtk_graph_panels_loaded(h, &loaded);
    CHECK(loaded == 1);
    sgtk_graph_destroy(h);
    // a section of another graph is ignored (fingerprint): panels rebuilt
    CsrGraph g2 = gcn_normalize_values(normalize_graph(random_graph(5000, 24, 78, false),
                                                       {true, true, true}));
    TransformedGraph t2 = sgt_transform(g2);
    const auto& c2 = t2.csr;
    CHECK(sgtk_graph_import_panels(c2.node_pointer.data(), c2.edge_list.data(), c2.values.data(),
                                   c2.num_nodes, c2.num_edges(), 16, 8, t2.edge_to_column.data(),
                                   t2.window_offsets.data(), t2.window_unique_cols.data(),
                                   (p + ".sgp").c_str(), nullptr, &h) == SGTK_OK);
    sgtk_graph_panels_loaded(h, &loaded);
    CHECK(loaded == 0);
    sgtk_graph_destroy(h);
    std::filesystem::remove(p);
    std::filesystem::remove(p + ".sgp");
  }

  // --- kernels (test_tile_exec.cpp) -----------------------------------------
  {
    TransformedGraph t = sgt_transform(identity_graph(16));
    DenseMatrix x = DenseMatrix::random(16, 16, 99);
    for (double ratio : {1.0, 0.0, 0.5})
      CHECK(spmm_hybrid(t, x, make_split_plan(t, ratio)).data == x.data);  // exact
    TransformedGraph t2 = sgt_transform(graph_of(2, {{0, 1, 1.0f}, {1, 0, 1.0f}}));
    DenseMatrix x2(2, 2);
    x2.data = {1, 2, 3, 4};
    CHECK((spmm_hybrid(t2, x2, make_split_plan(t2)).data == std::vector<float>{3, 4, 1, 2}));
    CHECK_THROWS_AS(make_split_plan(t, -0.1), RangeError);
    CHECK_THROWS_AS(make_split_plan(t, std::nan("")), RangeError);
    CHECK_THROWS_AS(spmm_hybrid(t, DenseMatrix(8, 4), make_split_plan(t)), ShapeError);
    CHECK_THROWS_AS(gather_tile(t, 1, 0), IndexError);
    CHECK_THROWS_AS(gather_tile(t, 0, 2), IndexError);
    auto gt = gather_tile(t, 0, 0);
    for (size_t r = 0; r < 16; ++r)
      for (size_t c = 0; c < 8; ++c) CHECK(gt.a_tile.at(r, c) == (r == c ? 1.0f : 0.0f));
  }
  {  // overflow -> NonFiniteError (test_tile_exec.cpp:179-186)
    std::vector<Triple> tr;
    for (int c = 0; c < 4; ++c) tr.push_back({0, NodeId(c), 1.0f});
    CsrGraph g = graph_of(4, tr, true);
    TransformedGraph t = sgt_transform(g);
    CHECK_THROWS_AS(spmm_hybrid(t, DenseMatrix(4, 1, 1e38f), make_split_plan(t)), NonFiniteError);
  }
  {  // vs oracle on random graphs at several widths / ratios / precisions
    std::mt19937_64 rng(4242);
    for (int it = 0; it < 8; ++it) {
      const size_t n = 16 + rng() % 400;
      CsrGraph g = random_graph(n, 6, rng(), it % 2);
      TransformedGraph t = sgt_transform(g);
      const size_t dim = std::vector<size_t>{8, 16, 32, 64}[it % 4];
      DenseMatrix x = DenseMatrix::random(n, dim, rng()), y = DenseMatrix::random(n, dim, rng());
      DenseMatrix want = oracle_spmm(g, x);
      for (double ratio : {1.0, 0.5, 0.0})
        CHECK(max_rel_err(spmm_hybrid(t, x, make_split_plan(t, ratio)), want) <= 1e-5);
      TransformedGraph t16 = reblock(t, 16);
      EdgeValList ws(g.num_edges());
      or_sddmm(n, g.node_pointer.data(), g.edge_list.data(), g.has_values() ? g.values.data() : nullptr,
               x.data.data(), y.data.data(), dim, 0, ws.data());
      for (double ratio : {1.0, 0.5, 0.0})
        CHECK(max_rel_err(sddmm_hybrid(t16, x, y, make_split_plan(t16, ratio)), ws) <= 1e-5);
      DenseMatrix tf = spmm_hybrid(t, x, make_split_plan(t), Precision::Tf32);
      DenseMatrix want_tf(n, dim);
      or_spmm(n, g.node_pointer.data(), g.edge_list.data(), g.has_values() ? g.values.data() : nullptr,
              x.data.data(), dim, 1, want_tf.data.data());
      CHECK(max_rel_err(tf, want_tf) <= 1e-5);
    }
  }
  {  // tf32 KATs (test_tile_exec.cpp:273-283)
    CHECK(tf32_round_value(1.0f + std::ldexp(1.0f, -11)) == 1.0f);
    CHECK(tf32_round_value(1.0f + std::ldexp(1.0f, -11) + std::ldexp(1.0f, -20)) ==
          1.0f + std::ldexp(1.0f, -10));
    DenseMatrix m(1, 3);
    m.data = {1.0f + std::ldexp(1.0f, -11), -2.0f, 3.14159f};
    DenseMatrix r = tf32_round(m);
    for (size_t i = 0; i < 3; ++i) CHECK(r.data[i] == tf32_round_value(m.data[i]));
  }

  // --- models (test_gnn.cpp) ------------------------------------------------
  {
    TransformedGraph t = sgt_transform(gcn_normalize_values(identity_graph(20)));
    DenseMatrix x = DenseMatrix::random(20, 6, 3, 0.0f, 1.0f);
    DenseMatrix eye(6, 6);
    for (size_t i = 0; i < 6; ++i) eye.at(i, i) = 1.0f;
    std::vector<GcnLayerParams> layers{{eye, true}, {eye, true}};
    CHECK(gcn_forward(t, x, layers, make_split_plan(t)).data == x.data);  // exact
    CHECK_THROWS_AS(gcn_forward(t, DenseMatrix(19, 6), layers, make_split_plan(t)), ShapeError);
  }
  {
    std::mt19937_64 rng(606);
    for (int it = 0; it < 4; ++it) {
      const size_t n = 32 + rng() % 128;
      CsrGraph g = gcn_normalize_values(
          normalize_graph(random_graph(n, 3, rng(), false), {true, true, true}));
      TransformedGraph t = sgt_transform(g);
      DenseMatrix x = DenseMatrix::random(n, 16, rng());
      auto layers = random_gcn_layers(16, 16, 7, 2, rng());
      std::vector<uint64_t> dims{16, 16, 7};
      std::vector<float> w;
      for (auto& l : layers) w.insert(w.end(), l.weight.data.begin(), l.weight.data.end());
      int relu[2] = {1, 0};
      DenseMatrix want(n, 7);
      or_gcn_forward(n, g.node_pointer.data(), g.edge_list.data(), g.values.data(), x.data.data(), 2,
                     dims.data(), w.data(), relu, 0, want.data.data());
      for (double ratio : {1.0, 0.0})
        CHECK(max_rel_err(gcn_forward(t, x, layers, make_split_plan(t, ratio)), want) <= 1e-5);
    }
  }
  {  // softmax closed forms (test_gnn.cpp:110-134)
    CsrGraph g2 = graph_of(3, {{0, 1, 1}, {0, 2, 1}});
    EdgeValList o = edge_softmax(g2, {0.0f, std::log(2.0f)});
    CHECK(std::abs(o[0] - 1.0f / 3.0f) < 1e-6 && std::abs(o[1] - 2.0f / 3.0f) < 1e-6);
    o = edge_softmax(g2, {200.0f, -200.0f});
    CHECK(std::isfinite(o[0]) && std::abs(o[0] - 1.0f) < 1e-6);
    CHECK((edge_softmax(graph_of(2, {{0, 1, 1}}), {3.25f}) == EdgeValList{1.0f}));
  }
  {  // AGNN (test_gnn.cpp:157-225)
    TransformedGraph t = sgt_transform(identity_graph(1));
    DenseMatrix x(1, 3);
    x.data = {0.5f, -1.0f, 2.0f};
    std::vector<AgnnLayerParams> layers(4, AgnnLayerParams{1.0f});
    CHECK(agnn_forward(t, x, layers, make_split_plan(t)).data == x.data);  // exact
    CsrGraph gz = normalize_graph(identity_graph(3), {});
    TransformedGraph tz = sgt_transform(gz);
    DenseMatrix xz(3, 4);
    xz.at(0, 0) = 1.0f;
    size_t zeros = 0;
    DenseMatrix oz = agnn_forward(tz, xz, {{1.0f}}, make_split_plan(tz), Precision::Fp32, 0, &zeros);
    CHECK(zeros == 2 && oz.all_finite() && oz.at(1, 0) == 0.0f && oz.at(2, 3) == 0.0f);
    std::mt19937_64 rng(616);
    for (int it = 0; it < 3; ++it) {
      const size_t n = 24 + rng() % 104;
      CsrGraph g = normalize_graph(random_graph(n, 3, rng(), false), {false, true, true});
      TransformedGraph ta = sgt_transform(g);
      DenseMatrix xa = DenseMatrix::random(n, 32, rng());
      const std::vector<float> betas{1.0f, 0.6f, 1.4f, 0.9f};
      std::vector<AgnnLayerParams> al;
      for (float b : betas) al.push_back({b});
      DenseMatrix want(n, 32);
      uint64_t z = 0;
      or_agnn_forward(n, g.node_pointer.data(), g.edge_list.data(), xa.data.data(), 32, 4,
                      betas.data(), 0, want.data.data(), &z);
      for (double ratio : {1.0, 0.0})
        CHECK(max_rel_err(agnn_forward(ta, xa, al, make_split_plan(ta, ratio)), want) <= 1e-5);
    }
  }
  {  // preprocessing (test_graph_io.cpp:153-268)
    CsrGraph p3 = graph_of(3, {{0, 0, 1}, {0, 1, 1}, {1, 0, 1}, {1, 1, 1}, {1, 2, 1}, {2, 1, 1}, {2, 2, 1}});
    CHECK(std::abs(gcn_normalize_values(p3).values[1] - 0.40824829f) < 1e-7);
    CsrGraph bad;
    bad.num_nodes = 2;
    bad.node_pointer = {0, 1, 1};
    bad.edge_list = {0};
    CHECK_THROWS_AS(gcn_normalize_values(bad), DegreeError);
    std::mt19937_64 rng(23);
    for (int it = 0; it < 12; ++it) {
      const size_t n = 1 + rng() % 700;
      std::vector<Triple> tr;
      std::uniform_real_distribution<float> v(-1, 1);
      for (size_t k = 0; k < 4 * n; ++k) tr.push_back({NodeId(rng() % n), NodeId(rng() % n), v(rng)});
      CsrGraph raw = graph_of(n, tr, it % 2);  // with duplicates
      for (int m = 0; m < 8; ++m) {
        NormalizeOpts o{bool(m & 1), bool(m & 2), bool(m & 4)};
        CsrGraph got = normalize_graph(raw, o);
        uint64_t nnz = 0;
        or_normalize_graph(n, raw.node_pointer.data(), raw.edge_list.data(),
                           raw.has_values() ? raw.values.data() : nullptr, o.symmetrize,
                           o.add_self_loops, o.dedupe, &nnz, nullptr, nullptr, nullptr);
        std::vector<uint64_t> np(n + 1);
        std::vector<uint32_t> el(nnz);
        std::vector<float> vals(raw.has_values() ? nnz : 0);
        or_normalize_graph(n, raw.node_pointer.data(), raw.edge_list.data(),
                           raw.has_values() ? raw.values.data() : nullptr, o.symmetrize,
                           o.add_self_loops, o.dedupe, &nnz, np.data(), el.data(),
                           raw.has_values() ? vals.data() : nullptr);
        CHECK(got.node_pointer == np && got.edge_list == el && got.values == vals);
        if (o.dedupe) CHECK(normalize_graph(got, o).edge_list == got.edge_list);  // idempotent
      }
    }
  }
  {  // weight files (test_gnn.cpp:227-239)
    const std::string p = (std::filesystem::temp_directory_path() /
                           ("dropin_w_" + std::to_string(getpid()) + ".bin")).string();
    GcnLayerParams l{DenseMatrix::random(12, 7, 44), false};
    save_gcn_layer(l, p);
    GcnLayerParams b = load_gcn_layer(p);
    CHECK(b.weight.rows == 12 && b.weight.cols == 7 && b.weight.data == l.weight.data && !b.apply_relu);
    std::filesystem::remove(p);
    std::filesystem::remove(p + ".json");
    CHECK_THROWS_AS(load_gcn_layer(p), IoError);
  }
  {  // the device copy follows csr.values edited in place (the cache
     // fingerprint now covers values) and reassigned
    CsrGraph g = random_graph(300, 6.0, 91, true);
    TransformedGraph t = sgt_transform(g);
    DenseMatrix x = DenseMatrix::random(300, 16, 5);
    const auto p = make_split_plan(t);
    CHECK(max_rel_err(spmm_hybrid(t, x, p), oracle_spmm(t.csr, x)) <= 1e-5);
    for (float& v : t.csr.values) v *= 2.0f;  // same buffer, new content
    CHECK(max_rel_err(spmm_hybrid(t, x, p), oracle_spmm(t.csr, x)) <= 1e-5);
    t.csr.values = std::vector<float>(t.csr.values.size(), 0.5f);  // reassigned
    CHECK(max_rel_err(spmm_hybrid(t, x, p), oracle_spmm(t.csr, x)) <= 1e-5);
  }
  {  // agnn_forward: NonFiniteError like spmm_hybrid (tile_exec.cpp:311-312 via
     // gnn.cpp:115) in every mode; zero-width input counts rows x layers
    CsrGraph gl = random_graph(200, 5.0, 92, false);
    TransformedGraph t = sgt_transform(normalize_graph(gl, {false, true, true}));
    DenseMatrix x = DenseMatrix::random(200, 32, 6);
    x.at(17, 3) = std::numeric_limits<float>::infinity();
    std::vector<AgnnLayerParams> al{{1.0f}, {0.5f}};
    CHECK_THROWS_AS(agnn_forward(t, x, al, make_split_plan(t)), NonFiniteError);
    x.at(17, 3) = std::numeric_limits<float>::quiet_NaN();
    CHECK_THROWS_AS(agnn_forward(t, x, al, make_split_plan(t, 0.5)), NonFiniteError);
    DenseMatrix x0(200, 0);
    size_t zeros = 0;
    agnn_forward(t, x0, al, make_split_plan(t), Precision::Fp32, 0, &zeros);
    CHECK(zeros == 400);
  }
  std::printf("%d/%d checks passed\n", g_checks - g_fail, g_checks);
  return g_fail ? 1 : 0;
}
