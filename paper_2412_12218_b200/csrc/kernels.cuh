// Internal launchers shared across translation units (host side).
#pragma once

#include <string>

#include "graph.cuh"

namespace sgtkcu {

sgtk_graph* graph_create(const uint64_t* np, const uint32_t* el, const float* vals, uint64_t n_rows,
                         uint64_t n_cols, uint64_t nnz, uint32_t blk_h, uint32_t blk_w, int kind,
                         cudaStream_t s, uint64_t row_offset = 0);
sgtk_graph* graph_import(const uint64_t* np, const uint32_t* el, const float* vals,
                         uint64_t n_rows, uint64_t nnz, uint32_t blk_h, uint32_t blk_w,
                         const uint32_t* e2c, const uint64_t* wo, const uint32_t* wuc,
                         cudaStream_t s, const char* panel_section = nullptr);
sgtk_graph* graph_reblock(const sgtk_graph* src, uint32_t blk_w, cudaStream_t s);

void spmm_launch(const sgtk_graph* g, const float* x, uint64_t ldx, uint64_t d,
                 const uint32_t* cut_dev, const float* ev, int prec, float* out, uint64_t ldo,
                 uint32_t* nonfinite, cudaStream_t s, bool x_tf32 = false);
void sddmm_launch(const sgtk_graph* g, const float* x, uint64_t ldx, const float* y, uint64_t ldy,
                  uint64_t d, const uint32_t* cut16_dev, const float* ev, bool unit_values,
                  int prec, const float* inv_norm, float scale, float* out, cudaStream_t s);
void edge_softmax_launch(const sgtk_graph* g, const float* logits, float* out, cudaStream_t s);
void csr_softmax_launch(const uint64_t* np, uint64_t n, const float* logits, float* out,
                        cudaStream_t s);
void l2norm_launch(const float* h, uint64_t rows, uint64_t cols, uint64_t ldh, float* z,
                   uint64_t ldz, float* inv, uint64_t* zeros, cudaStream_t s);
void gcn_normalize_launch(const uint64_t* np, const uint32_t* el, uint64_t n, float* vals,
                          cudaStream_t s);
void tf32_launch(const float* in, float* out, uint64_t n, cudaStream_t s);
// round_tf32: store RNE-TF32-rounded results (the consumer is a TF32 SpMM);
// nonfinite: set to 1 when a stored value is NaN/Inf.
void gemm_launch(const float* a, uint64_t lda, const float* w, uint64_t m, uint64_t k, uint64_t n,
                 int relu, int prec, float* out, uint64_t ldo, cudaStream_t s,
                 bool round_tf32 = false, uint32_t* nonfinite = nullptr);
void relu_nonfinite_launch(float* x, uint64_t rows, uint64_t cols, uint64_t ld, int relu,
                           uint32_t* nonfinite, cudaStream_t s);
void agnn_fused_launch(const sgtk_graph* g, const float* h, uint64_t ldh, const float* z,
                       uint64_t ldz, const float* inv, uint64_t d, float beta, int prec,
                       const uint32_t* cut_dev, float* out, uint64_t ldo, cudaStream_t s,
                       uint32_t* nonfinite = nullptr);

// 128-row panel format + tcgen05 SpMM (panel.cu)
Windows build_row_windows(const sgtk_graph& g, uint32_t bh, cudaStream_t s);
void build_panels(sgtk_graph& g, cudaStream_t s);
// Panel section beside an SGT1 file (panel.cu): save / load (false when the
// section is absent, of another version or of another graph).
void save_panel_section(const sgtk_graph& g, const std::string& path, cudaStream_t s);
bool load_panel_section(sgtk_graph& g, const std::string& path, cudaStream_t s);
// x_tf32: x is already TF32-rounded (RNE) by its producer (the fused GEMM
// epilogue), so the TF32 path skips its rounding pass over x.
// SDDMM on the panel format (sddmm_panel.cu): tcgen05 dense columns + CUDA-core
// sparse edges; false outside its envelope (the 16-row kernel then runs).
bool sddmm_panel_launch(const sgtk_graph* g, const float* x, uint64_t ldx, const float* y,
                        uint64_t ldy, uint64_t d, const float* ev, bool unit_values, int prec,
                        const float* inv_norm, float scale, float* out, cudaStream_t s);
bool spmm_panel_launch(const sgtk_graph* g, const float* x, uint64_t ldx, uint64_t d,
                       const float* ev, int prec, float* out, uint64_t ldo, uint32_t* nonfinite,
                       cudaStream_t s, bool x_tf32 = false);

// AGNN layer on panels (agnn_panel.cu)
struct AgnnNext {
  float* out;         // layer output h' (nullptr: not needed, TF32 inner layers)
  uint64_t ldo;
  float* z;           // next layer z (raw; FP32 only, nullptr on the last layer)
  float* zq;          // next-layer MMA operand copies (TF32-rounded / hi planes)
  float* zq1;         //   lo planes (FP32)
  float* hq;
  float* hq1;
  float* norm;        // next layer |h| per row
  uint64_t ldq;
  unsigned long long* zeros;
  uint32_t* nonfinite;  // set to 1 when an output value is NaN/Inf (last layer only)
};
bool agnn_panel_supported(const sgtk_graph* g, uint64_t d, float beta);
void agnn_panel_layer(const sgtk_graph* g, const float* z, const float* zq, const float* zq1,
                      const float* hq, const float* hq1, uint64_t ldq, const float* norm,
                      uint64_t d, float beta, int prec, float* opart, float* lpart, float* seg_o,
                      float* seg_l, float* osp, float* lsp, const AgnnNext& nx, cudaStream_t s);
// Layer-0 input of the panel path: l2 norm + operand copies of x in one pass.
void agnn_input_launch(const float* x, uint64_t ldx, uint64_t rows, uint64_t d, uint64_t ldq, int prec,
                       float* z, float* zq, float* zq1, float* hq, float* hq1, float* norm,
                       uint64_t* zeros, cudaStream_t s);
// The panel format an operation of width d runs on (panels32 for d <= 32).
const Panels& panels_for(const sgtk_graph* g, uint64_t d);
// lazily built per-format arrays (first use; thread-safe): Panels::dpos for
// the SDDMM direct form, Panels::paitem for the fused AGNN form
void ensure_dpos(const sgtk_graph& g, const Panels& pn, cudaStream_t s);
void ensure_paitem(const Panels& pn, cudaStream_t s);
PanelView panel_view(const sgtk_graph* g, uint64_t d);
void panel_debug_set(int mode);
int panel_debug_mode();
bool panel_enabled();

// Host-side split plan (make_split_plan, tile_exec.cpp:150-161).
std::vector<uint32_t> split_plan_host(const sgtk_graph* g, double ratio);

}  // namespace sgtkcu

// Device CSR produced by normalize_graph (normalize.cu).
struct sgtk_csr {
  uint64_t n = 0, nnz = 0;
  bool has_values = false;
  sgtkcu::DevBuf np, el, vals;
};

namespace sgtkcu {
sgtk_csr* normalize_graph(const uint64_t* np, const uint32_t* el, const float* vals, uint64_t n,
                          uint64_t E, int symmetrize, int loops, int dedupe, int kind,
                          cudaStream_t s);
}  // namespace sgtkcu
