// model.cpp — the paper's analytical stage/tile model (
// perf_model.hpp:49-187) on the B200 host side.
//
// Two hardware views share the Table structure
//   T_kernel = T_threadblk * N_threadblk_batch,
//   T_threadblk = T_init + T_main_loop + T_epilogue,
//   T_main_loop = pipeline_latency(T_smem_load, T_smem_use, N_smem_loop,
//                                  N_smem_pipe_stage, N_tb_per_SM)
// (a) the reference's A100-like HardwareSpec (perf_model.hpp:14-30), where
//     predict() restates the reference arithmetic for the tcgen05 kernel
//     shape, and
// (b) B200, re-derived for the persistent warp-specialised kernel:
//     - one CTA per SM (227 KB smem ring, 512-column TMEM), so the per-SM
//       throughput is never multiplied by co-resident CTAs (the reference
//       lets every co-resident CTA run at full SM rate, perf_model.hpp:61-70,
//       which predicts above-peak throughput on B200 — SURVEY §0);
//     - the inner level is the TMEM accumulator ring: with n_stage_inner = 2
//       the epilogue of tile i overlaps the main loop of tile i+1, so the
//       per-tile time is max(T_main_loop, T_epilogue);
//     - WRAP mode pays s-1 redundant wrapped loads and a drain per tile;
//     - a chip-wide floor T >= FLOPs / (numSM * throughputSM).
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "alcop_internal.h"

namespace alcop {
namespace model {

// perf_model.hpp:53-57
double pipeline_latency(double tLoad, double tUse, int64_t nLoop, int nPipe, int nMplx) {
  if (tLoad <= (static_cast<double>(nPipe) * nMplx - 1) * tUse) return tUse * static_cast<double>(nLoop);
  return (tLoad + tUse) * static_cast<double>(nLoop) / nPipe;
}

}  // namespace model
}  // namespace alcop

using namespace alcop;

extern "C" void alcop_hw_default_a100_reference(alcop_hw* hw) {
  if (!hw) return;
  std::memset(hw, 0, sizeof(*hw));
  // perf_model.hpp:15-29
  hw->numSM = 108;
  hw->throughputSM = 1024;
  hw->bwLLC = 512;
  hw->bwDRAM = 64;
  hw->bwDRAMWrite = 32;
  hw->latLLCRead = 200;
  hw->latDRAMRead = 400;
  hw->latDRAMWrite = 400;
  hw->bwSmem = 128;
  hw->latSmem = 25;
  hw->smemPerSM = 163840;
  hw->regsPerSM = 262144;
  hw->maxThreadblkPerSM = 32;
  hw->maxWarpsPerSM = 64;
  hw->utilKneeWarps = 8;
  hw->tmemColsPerSM = 0;
  hw->clockGHz = 1.41;
}

extern "C" void alcop_hw_default_b200(alcop_hw* hw) {
  if (!hw) return;
  std::memset(hw, 0, sizeof(*hw));
  // B200 (sm_100a), 148 SMs; rates per SM clock.  Calibrated from the
  // driver-measured peaks (MEASURED_PEAKS.json: 1633.8 TFLOP/s bf16 burst,
  // 6549.4 GB/s HBM) at the observed SM clock, see DESIGN.md "model".
  hw->numSM = 148;
  hw->throughputSM = 8192;  // dense f16/bf16 FLOP / clk / SM (tcgen05, M=128)
  hw->bwLLC = 6300;         // L2 -> SM bytes / clk, chip-wide (LTS cap)
  hw->bwDRAM = 3600;        // HBM bytes / clk at ~1.8 GHz (6.5 TB/s)
  hw->bwDRAMWrite = 3600;
  hw->latLLCRead = 600;     // TMA issue -> full barrier, L2 hit
  hw->latDRAMRead = 1000;
  hw->latDRAMWrite = 800;
  hw->bwSmem = 128;
  hw->latSmem = 30;
  hw->smemPerSM = 232448;
  hw->regsPerSM = 262144;
  hw->maxThreadblkPerSM = 1;  // persistent, one CTA per SM
  hw->maxWarpsPerSM = 64;
  hw->utilKneeWarps = 1;
  hw->tmemColsPerSM = 512;
  hw->clockGHz = 1.8;
}

extern "C" int alcop_predict(const alcop_gemm_desc* w, const alcop_schedule* s, const alcop_hw* hw,
                             alcop_breakdown* out) {
  if (!w || !s || !hw || !out) return set_error(ALCOP_ERR_CONFIG, "NullArgument", "NULL argument");
  clear_error();
  int rc = validate_gemm(*w, *s);
  if (rc) return rc;
  std::memset(out, 0, sizeof(*out));
  const int64_t tM = s->tileM, tN = s->tileN, tK = s->tileK;
  const int64_t eb = 2, ob = w->out_dtype == ALCOP_F32 ? 4 : 2;
  const int64_t tiles = ((w->M + tM - 1) / tM) * ((w->N + tN - 1) / tN) * w->batch;
  const int64_t nSM = hw->numSM;
  const int64_t ctas = std::min<int64_t>(tiles, s->num_ctas > 0 ? s->num_ctas : nSM);
  const int64_t tilesPerCta = (tiles + ctas - 1) / ctas;
  const int64_t E = (w->K + tK - 1) / tK;
  const int sOuter = std::min(s->n_stage_smem_A, s->n_stage_smem_B);
  out->nThreadblkPerSM = 1;
  out->nThreadblkPerBatch = ctas;
  out->nThreadblkBatch = tilesPerCta;
  out->nSmemLoop = E;
  out->nRegLoop = tK / 16;
  out->flopsOneRegLoop = 2 * tM * tN * 16;
  out->bytesOneSmemLoop = (tM + tN) * tK * eb;
  // DRAM working set of one wave per k-step: unique A row blocks and B
  // column blocks touched by the resident tiles (perf_model.hpp:147-153,
  // m-fastest rasterisation).
  const int64_t nI = (w->M + tM - 1) / tM;
  const int64_t rows = std::min<int64_t>(ctas, nI);
  const int64_t cols = (ctas + nI - 1) / nI;
  out->bytesWorkset = rows * tM * tK * eb + cols * tK * tN * eb;
  out->bytesOutputTile = tM * tN * ob;

  out->tCompute = static_cast<double>(out->flopsOneRegLoop) / hw->throughputSM;
  out->tRegLoad = 0;  // tcgen05 reads smem operands directly through descriptors
  out->tSmemUse = out->tCompute * static_cast<double>(out->nRegLoop);
  const double llc = hw->latLLCRead + static_cast<double>(out->bytesOneSmemLoop) * ctas / hw->bwLLC;
  const double dram = hw->latDRAMRead + static_cast<double>(out->bytesWorkset) / hw->bwDRAM;
  out->tSmemLoad = std::max(llc, dram);
  const int64_t loadsPerTile = E + (s->mode == ALCOP_MODE_WRAP ? sOuter - 1 : 0);
  double tMain = model::pipeline_latency(out->tSmemLoad, out->tSmemUse, loadsPerTile, sOuter, 1);
  if (s->mode == ALCOP_MODE_WRAP || sOuter == 1) tMain += out->tSmemLoad;  // per-tile refill bubble
  out->tMainLoop = tMain;
  out->tEpilogue = hw->latDRAMWrite + static_cast<double>(out->bytesOutputTile) * ctas / hw->bwDRAMWrite +
                   static_cast<double>(tM * tN) * 4.0 / 64.0 / 4.0;  // TMEM read: 64 B/clk per warp
  out->tInit = out->tSmemLoad + 1500.0;  // barrier init + TMEM alloc + first loads
  const double perTile = s->n_stage_inner >= 2 ? std::max(out->tMainLoop, out->tEpilogue)
                                               : out->tMainLoop + out->tEpilogue;
  out->tThreadblk = out->tInit + out->tMainLoop + out->tEpilogue;
  double tK_ = out->tInit + perTile * static_cast<double>(tilesPerCta) +
               (s->n_stage_inner >= 2 ? std::min(out->tMainLoop, out->tEpilogue) : 0.0);
  const double flops = 2.0 * w->M * w->N * w->K * w->batch;
  const double floor = flops / (static_cast<double>(nSM) * hw->throughputSM);
  out->tKernel = std::max(tK_, floor);
  out->seconds = out->tKernel / (hw->clockGHz * 1e9);
  return ALCOP_OK;
}

extern "C" int alcop_choose_schedule(const alcop_gemm_desc* w, const alcop_hw* hw, alcop_schedule* out) {
  if (!w || !hw || !out) return set_error(ALCOP_ERR_CONFIG, "NullArgument", "NULL argument");
  clear_error();
  // enumerate_space + analytical_rank (tuner.hpp:48-80) over the B200 space
  double best = 1e300;
  alcop_schedule bestS{};
  bool found = false;
  for (int tN : {64, 128, 192, 256})
    for (int tK : {32, 64, 128})
      for (int st = 1; st <= 8; ++st)
        for (int inner = 1; inner <= 2; ++inner) {
          alcop_schedule s;
          alcop_schedule_default(&s);
          s.tileN = tN;
          s.tileK = tK;
          s.n_stage_smem_A = s.n_stage_smem_B = st;
          s.n_stage_inner = inner;
          s.mode = ALCOP_MODE_FUSED;
          if (validate_gemm(*w, s) != ALCOP_OK) continue;
          alcop_breakdown b;
          if (alcop_predict(w, &s, hw, &b) != ALCOP_OK) continue;
          if (b.tKernel < best) {
            best = b.tKernel;
            bestS = s;
            found = true;
          }
        }
  clear_error();
  if (!found) return set_error(ALCOP_ERR_CONFIG, "Unschedulable", "no valid schedule for workload");
  *out = bestS;
  return ALCOP_OK;
}
