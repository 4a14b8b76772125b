// Event-level pipeline simulation (the reference's pipe_sim.hpp restated for
// the C ABI) and its B200 two-level kernel analogue.
//
//   alcop_simulate_pipeline   sim::simulate_pipeline   pipe_sim.hpp:55-127
//                             + comparable_worker_latency          :129-133
//   alcop_simulate_two_level  sim::simulate_two_level  pipe_sim.hpp:138-167
//   alcop_simulate_kernel     B200: smem ring (outer) x TMEM accumulator
//                             ring (inner) per persistent CTA, fed by the
//                             alcop_predict chunk/epilogue times
#include <algorithm>
#include <cmath>
#include <cstring>
#include <vector>

#include "alcop.h"
#include "alcop_internal.h"

using alcop::clear_error;
using alcop::set_error;

namespace {

enum : int32_t { kLoadIssue = 0, kLoadDone = 1, kComputeStart = 2, kComputeEnd = 3 };

struct WorkerState {
  int64_t next = 0;           // next iteration this worker computes
  double lastEnd = 0;         // end of its previous compute
  std::vector<double> freed;  // per slot: end of the compute that last used it
};

}  // namespace

extern "C" int alcop_simulate_pipeline(const alcop_sim_config* cfg, alcop_sim_result* out, alcop_sim_event* trace,
                                       int64_t trace_cap, int64_t* n_events) {
  if (!cfg || !out) return set_error(ALCOP_ERR_CONFIG, "NullArgument", "NULL argument");
  clear_error();
  if (cfg->nLoop < 1 || cfg->nPipe < 1 || cfg->nMplx < 1)
    return set_error(ALCOP_ERR_CONFIG, "BadSimConfig", "simulate_pipeline: counts must be >= 1");
  if (cfg->tLoad < 0 || cfg->tUse < 0)
    return set_error(ALCOP_ERR_CONFIG, "BadSimConfig", "simulate_pipeline: times must be nonnegative");
  const int P = cfg->nPipe, W = cfg->nMplx;
  std::vector<WorkerState> ws(W);
  for (auto& w : ws) w.freed.assign(P, 0.0);
  // iteration i < nPipe loads at 0; later ones when compute i-nPipe frees the slot
  auto issue_of = [&](const WorkerState& w, int64_t i) { return i < P ? 0.0 : w.freed[i % P]; };

  const bool want = trace != nullptr || n_events != nullptr;
  std::vector<alcop_sim_event> ev;
  if (want) ev.reserve(static_cast<size_t>(4 * cfg->nLoop * W));
  std::memset(out, 0, sizeof(*out));
  double unit = 0;  // the shared compute unit is free from here on
  bool first = true;
  for (int64_t left = cfg->nLoop * W; left > 0; --left) {
    // the worker whose next compute can start earliest (own load + own
    // previous compute) takes the unit; lowest id on ties
    int pick = -1;
    double pickReady = 0;
    for (int i = 0; i < W; ++i) {
      if (ws[i].next >= cfg->nLoop) continue;
      const double ready = std::max(issue_of(ws[i], ws[i].next) + cfg->tLoad, ws[i].lastEnd);
      if (pick < 0 || ready < pickReady) {
        pick = i;
        pickReady = ready;
      }
    }
    WorkerState& w = ws[pick];
    const int64_t it = w.next;
    const double iss = issue_of(w, it);
    const double landed = iss + cfg->tLoad;
    const double start = std::max(std::max(landed, w.lastEnd), unit);
    const double end = start + cfg->tUse;
    if (want) {
      ev.push_back({iss, pick, kLoadIssue, it});
      ev.push_back({landed, pick, kLoadDone, it});
      ev.push_back({start, pick, kComputeStart, it});
      ev.push_back({end, pick, kComputeEnd, it});
    }
    if (first) {
      out->firstComputeStart = start;
      first = false;
    }
    unit = end;
    w.lastEnd = end;
    w.freed[it % P] = end;
    w.next = it + 1;
    out->makespan = std::max(out->makespan, end);
  }
  out->busy = cfg->tUse * static_cast<double>(cfg->nLoop) * W;
  const double window = out->makespan - out->firstComputeStart;
  if (window > 0)
    out->idleFraction = std::max(0.0, 1.0 - out->busy / window);
  else
    out->idleFraction = cfg->tUse > 0 ? 0.0 : 1.0;
  // saturated unit: the makespan carries all nMplx rounds -> per worker
  out->comparable = out->idleFraction < 0.02 ? out->makespan / W : out->makespan;
  if (want) {
    std::stable_sort(ev.begin(), ev.end(),
                     [](const alcop_sim_event& a, const alcop_sim_event& b) { return a.time < b.time; });
    if (trace)
      std::copy(ev.begin(), ev.begin() + std::min<int64_t>(trace_cap, static_cast<int64_t>(ev.size())), trace);
    if (n_events) *n_events = static_cast<int64_t>(ev.size());
  }
  return ALCOP_OK;
}

extern "C" int alcop_simulate_two_level(const alcop_sim_config* outer, const alcop_sim_config* inner, int32_t fused,
                                        double* makespan) {
  if (!outer || !inner || !makespan) return set_error(ALCOP_ERR_CONFIG, "NullArgument", "NULL argument");
  clear_error();
  if (outer->nLoop < 1 || inner->nLoop < 1 || outer->nPipe < 1 || inner->nPipe < 1)
    return set_error(ALCOP_ERR_CONFIG, "BadSimConfig", "simulate_two_level: counts must be >= 1");
  const int64_t F = inner->nLoop;            // inner steps per outer chunk
  const int64_t n = outer->nLoop * F;        // flattened step count
  std::vector<double> stepEnd(n, 0.0);
  std::vector<double> chunkLanded(outer->nLoop, -1.0);
  std::vector<double> innerFreed(inner->nPipe, 0.0);
  auto chunk_retired = [&](int64_t c) { return c < 0 ? 0.0 : stepEnd[(c + 1) * F - 1]; };
  double last = 0;
  for (int64_t g = 0; g < n; ++g) {
    const int64_t c = g / F;
    if (chunkLanded[c] < 0) {
      // outer slot of chunk c frees when chunk c - nPipe has fully retired
      const double iss = c < outer->nPipe ? 0.0 : chunk_retired(c - outer->nPipe);
      chunkLanded[c] = iss + outer->tLoad;
    }
    const double slot = g < inner->nPipe ? 0.0 : innerFreed[g % inner->nPipe];
    const double restartGate = (!fused && c > 0) ? chunk_retired(c - 1) : 0.0;
    const double iss = std::max(std::max(slot, chunkLanded[c]), restartGate);
    const double start = std::max(iss + inner->tLoad, last);
    stepEnd[g] = start + inner->tUse;
    innerFreed[g % inner->nPipe] = stepEnd[g];
    last = stepEnd[g];
  }
  *makespan = stepEnd[n - 1];
  return ALCOP_OK;
}

extern "C" int alcop_simulate_kernel(const alcop_gemm_desc* w, const alcop_schedule* s, const alcop_hw* hw,
                                     alcop_sim_kernel* out) {
  if (!w || !s || !hw || !out) return set_error(ALCOP_ERR_CONFIG, "NullArgument", "NULL argument");
  alcop_breakdown b;
  int rc = alcop_predict(w, s, hw, &b);
  if (rc) return rc;
  std::memset(out, 0, sizeof(*out));
  const int64_t tiles = b.nThreadblkBatch;  // tiles of the busiest CTA (pair)
  const int64_t E = b.nSmemLoop;
  const int sN = std::min(s->n_stage_smem_A, s->n_stage_smem_B);
  const int tAcc = s->n_stage_inner;
  const bool wrap = s->mode == ALCOP_MODE_WRAP;
  const double tLoad = b.tSmemLoad, tUse = b.tSmemUse, tEpi = b.tEpilogue;

  std::vector<double> slotFreed(sN, 0.0);  // outer ring: freed when the MMA (or a drain) retires the slot
  std::vector<double> epiEnd(tiles, 0.0);  // inner ring: accumulator j is free once tile j - t drained
  double mmaLast = 0, epiLast = 0, busy = 0, firstMma = -1, mainSum = 0;
  int64_t cursor = 0, loads = 0;
  for (int64_t j = 0; j < tiles; ++j) {
    const double accFree = j >= tAcc ? epiEnd[j - tAcc] : 0.0;
    const int64_t nLoads = wrap ? E + sN - 1 : E;  // WRAP: s-1 wrapped tail loads per tile
    if (wrap) cursor = 0;                           // the ring restarts at slot 0 each tile
    double tileStart = -1, tileMmaEnd = 0;
    for (int64_t i = 0; i < nLoads; ++i, ++cursor, ++loads) {
      const int64_t slot = cursor % sN;
      const double landed = slotFreed[slot] + tLoad;  // producer_acquire -> commit -> bytes land
      if (i < E) {
        const double start = std::max(std::max(landed, mmaLast), accFree);  // consumer_wait (+ tmem_empty)
        const double end = start + tUse;
        if (tileStart < 0) tileStart = start;
        if (firstMma < 0) firstMma = start;
        mmaLast = end;
        slotFreed[slot] = end;  // consumer_release when the MMAs retire
        busy += tUse;
        tileMmaEnd = end;
      } else {
        const double rel = std::max(landed, mmaLast);  // drain: wait + release, no MMA
        mmaLast = rel;
        slotFreed[slot] = rel;
      }
    }
    mainSum += tileMmaEnd - tileStart;
    const double es = std::max(tileMmaEnd, epiLast);  // tmem_full -> epilogue warps
    epiEnd[j] = es + tEpi;
    epiLast = epiEnd[j];
  }
  const int cg = s->cta_group == 2 ? 2 : 1;
  out->tBody = epiLast;
  out->mmaBusy = busy;
  const double window = mmaLast - (firstMma < 0 ? 0 : firstMma);
  out->mmaIdleFraction = window > 0 ? std::max(0.0, 1.0 - busy / window) : 0.0;
  out->tMainLoopTile = tiles > 0 ? mainSum / static_cast<double>(tiles) : 0.0;
  out->tEpilogueTile = tEpi;
  out->tLoadChunk = tLoad;
  out->tUseChunk = tUse;
  out->tilesPerUnit = tiles;
  out->loads = loads;
  // whole kernel: the same launch, CTA-pair and HBM composition as alcop_predict
  const double sm = out->tBody + (cg == 2 ? hw->tPair : 0.0);
  const double ob = w->out_dtype == ALCOP_F32 ? 4.0 : 2.0;
  const double dram = (static_cast<double>(b.bytesWorkset) + static_cast<double>(w->M * w->N * w->batch) * ob) /
                      hw->bwDRAM;
  out->tKernel = hw->tLaunch + std::max(sm, dram) + hw->overlapDRAM * std::min(sm, dram);
  out->seconds = out->tKernel / (hw->clockGHz * 1e9);
  return ALCOP_OK;
}
