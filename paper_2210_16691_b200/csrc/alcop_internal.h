// alcop_internal.h — shared declarations between the C-ABI front end
// (alcop_api.cpp, schedule.cpp, model.cpp) and the sm_100a kernels (*.cu).
#pragma once
#include <stdint.h>

#include <string>

#include "../../include/alcop.h"

namespace alcop {

// Sets the thread-local "<RuleTag>: message" and returns `code`.
int set_error(int code, const std::string& tag, const std::string& msg);
void clear_error();

// Kernel limits of the cta_group::1 pipelined GEMM.
constexpr int kTileM = 128;
constexpr int kMaxStages = 16;
constexpr int kMaxSmemBytes = 232448;  // 227 KB opt-in per CTA on sm_100
constexpr int kTmemCols = 512;

int64_t round_up_pow2_cols(int64_t cols);
int64_t gemm_smem_bytes(const alcop_gemm_desc& w, const alcop_schedule& s);
int32_t gemm_staging_bufs(const alcop_gemm_desc& w, const alcop_schedule& s);
int32_t gemm_epi_warps(const alcop_gemm_desc& w, const alcop_schedule& s);
bool pair_b_pad(const alcop_gemm_desc& w, const alcop_schedule& s);
// the same for a kernel with a fixed number of epilogue warps (conv, chain: 4)
int32_t gemm_staging_bufs_epi(const alcop_gemm_desc& w, const alcop_schedule& s, int32_t epi);
int64_t gemm_smem_bytes_epi(const alcop_gemm_desc& w, const alcop_schedule& s, int32_t epi);
int launch_chain(const alcop_chain& ch, const alcop_schedule& s, void* workspace, void* stream);
int64_t chain_max_row_blocks(const alcop_chain* ch);
int validate_gemm(const alcop_gemm_desc& w, const alcop_schedule& s);
// Launch (validated) — implemented in gemm_sm100.cu.
int launch_gemm(const alcop_gemm_desc& w, const alcop_schedule& s, const void* A, const void* B, void* C,
                alcop_event* trace, int64_t trace_cap, void* stream);
int device_sm_count();
// stream-K workspace (gemm_sm100.cu): bytes for n clusters of 256 x BN fp32
// partials + flags; registration for the current device
size_t sk_bytes_needed(int n_clusters, int BN);
int set_sk_workspace(void* ptr, int64_t bytes);
// Tile rows per raster group for `units` concurrent CTAs (cta_group 1) or CTA
// pairs: schedule.raster if set, else the group minimising the distinct
// A-row + B-column panels the tiles in flight touch (G*BM + (units/G)*BN ->
// G = sqrt(units*BN/BM)); one wave: plain m-fastest order.
inline int32_t raster_group_of(int32_t raster, int64_t units, int64_t num_m, int64_t num_n, int64_t BM, int64_t BN) {
  if (raster > 0) return raster;
  if (units < 1) units = 1;
  if (num_m * num_n <= units) return static_cast<int32_t>(num_m);
  double x = static_cast<double>(units) * static_cast<double>(BN) / static_cast<double>(BM);
  int64_t g = 1;
  while ((g + 1) * (g + 1) <= x) ++g;  // floor(sqrt(x)), then round to nearest
  if ((g + 0.5) * (g + 0.5) <= x) ++g;
  if (g < 1) g = 1;
  return static_cast<int32_t>(g < num_m ? g : num_m);
}
// The stem kernel (stem_sm100.cu): C = 4, stride_w 2 convs whose A operand is
// read straight from the raw input rows (pixel pairs = 16-byte UMMA rows).
// Window mode of the same kernel: C = 64, stride 1 convs (3x3) whose tile of
// TR output rows reads its (TR+R-1)-row input window once; every tap is the
// window shifted by whole 128-byte pixel rows.
struct StemGeometry {
  int64_t P, Q, QB;          // output rows / columns, 128-column blocks per row
  int32_t o_min, T2, NB;     // pair offset of group 0, pair groups per filter row (even), 8-pair blocks per window row
  int32_t TR, WP;            // window mode: output rows per tile, window row pitch in pixels (TR * WP = 128)
  uint32_t row_bytes, slot_bytes, box_bytes, wbytes;
  int64_t kdim;              // GEMM-view reduction length
};
bool stem_pairs_applicable(const alcop_conv_desc& d);
bool window_conv_applicable(const alcop_conv_desc& d);
bool window_stream_applicable(const alcop_conv_desc& d);
StemGeometry stem_pairs_geometry(const alcop_conv_desc& d);
int64_t stem_pairs_smem_bytes(const alcop_conv_desc& d, const alcop_schedule& s);
int validate_stem_pairs(const alcop_conv_desc& d, const alcop_schedule& s);
int launch_conv2d_stem_pairs(const alcop_conv_desc& d, const alcop_schedule& s, const void* x, const void* wt,
                             void* y, void* stream);
// 1x1 / stride 1 / no padding: the conv is the GEMM [N*H*W, C] x [K, C]^T
inline bool conv_is_gemm(const alcop_conv_desc& d) {
  return d.R == 1 && d.S == 1 && d.stride_h == 1 && d.stride_w == 1 && d.pad_h == 0 && d.pad_w == 0 && d.C % 8 == 0;
}
inline void conv_gemm_view(const alcop_conv_desc& d, alcop_gemm_desc* g) {
  *g = alcop_gemm_desc{};
  g->M = d.N * d.H * d.W;
  g->N = d.K;
  g->K = d.C;
  g->batch = 1;
  g->in_dtype = d.in_dtype;
  g->out_dtype = d.out_dtype;
  g->b_layout = ALCOP_B_NK;
}
int launch_conv2d(const alcop_conv_desc& d, const alcop_schedule& s, const void* x, const void* wt, void* y,
                  void* stream);

}  // namespace alcop
