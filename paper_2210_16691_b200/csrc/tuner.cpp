// tuner.cpp — model-assisted schedule tuning on the B200 itself (SURVEY
// §8(f) rank 2): the reference's tune() (tuner.hpp:363-531) ranks a design
// space with the analytical model and "measures" the top candidates with a
// noisy simulator (measure_ground_truth, pipe_sim.hpp:195-239).  Here the
// candidates are launched on the GPU and timed with CUDA events, in steady
// state (graph-replayed back-to-back launches over rotating operand copies).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <string>
#include <vector>

#include "alcop_internal.h"

using namespace alcop;

namespace {

// Bytes one rotating copy of (A, B, C) spans, and how many copies exceed 2 x L2.
struct TuneSets {
  size_t a_bytes, b_bytes, c_bytes, set_bytes;
  int nsets;
};

TuneSets tune_sets(const alcop_gemm_desc& w) {
  const int64_t lda = w.lda ? w.lda : w.K;
  const int64_t ldb = w.ldb ? w.ldb : (w.b_layout == ALCOP_B_KN ? w.N : w.K);
  const int64_t ldc = w.ldc ? w.ldc : w.N;
  const int64_t rows_b = w.b_layout == ALCOP_B_KN ? w.K : w.N;
  const int64_t sa = w.stride_a ? w.stride_a : w.M * lda;
  const int64_t sb = w.stride_b ? w.stride_b : rows_b * ldb;
  const int64_t sc = w.stride_c ? w.stride_c : w.M * ldc;
  const size_t ob = w.out_dtype == ALCOP_F32 ? 4 : 2;
  TuneSets t;
  t.a_bytes = 2 * static_cast<size_t>((w.batch - 1) * sa + (w.M - 1) * lda + w.K);
  t.b_bytes = 2 * static_cast<size_t>((w.batch - 1) * sb + (rows_b - 1) * ldb + (w.b_layout == ALCOP_B_KN ? w.N : w.K));
  t.c_bytes = ob * static_cast<size_t>((w.batch - 1) * sc + (w.M - 1) * ldc + w.N);
  auto al = [](size_t b) { return (b + 255) & ~size_t(255); };
  t.set_bytes = al(t.a_bytes) + al(t.b_bytes) + al(t.c_bytes);
  const size_t kL2 = size_t(126) << 20;
  t.nsets = static_cast<int>(std::min<size_t>(32, std::max<size_t>(2, (2 * kL2 + t.set_bytes - 1) / t.set_bytes)));
  return t;
}

#define TUNE_CUDA(call, what)                                                          \
  do {                                                                                 \
    cudaError_t e_ = (call);                                                           \
    if (e_ != cudaSuccess && rc == ALCOP_OK)                                           \
      rc = set_error(ALCOP_ERR_CUDA, "CudaError", std::string(what) + ": " + cudaGetErrorString(e_)); \
  } while (0)

}  // namespace

extern "C" int64_t alcop_tune_workspace_bytes(const alcop_gemm_desc* w) {
  if (!w || w->M < 1 || w->N < 1 || w->K < 1 || w->batch < 1) return 0;
  const TuneSets t = tune_sets(*w);
  return static_cast<int64_t>(t.set_bytes) * t.nsets;
}

extern "C" int alcop_tune(const alcop_gemm_desc* w, const alcop_hw* hw, int32_t budget, const void* A, const void* B,
                          void* C, void* workspace, int64_t workspace_bytes, void* stream, alcop_schedule* best,
                          alcop_tune_trial* trials, int32_t trials_cap, int32_t* n_trials) {
  if (!w || !hw || !A || !B || !C || !best || !workspace || budget < 1)
    return set_error(ALCOP_ERR_CONFIG, "NullArgument", "NULL argument or budget < 1");
  clear_error();
  if (workspace_bytes < alcop_tune_workspace_bytes(w))
    return set_error(ALCOP_ERR_CONFIG, "Workspace",
                     "tuning workspace needs " + std::to_string(alcop_tune_workspace_bytes(w)) + " bytes");
  // enumerate_space (tuner.hpp:48-64) + analytical_rank (tuner.hpp:68-80)
  std::vector<std::pair<double, alcop_schedule>> space;
  for (int cg = 1; cg <= 2; ++cg)
    for (int tN : {64, 128, 192, 256, 512})
      for (int tK : {32, 64, 128})
        for (int inner = 1; inner <= 2; ++inner)
          for (int st = 1; st <= 8; ++st) {
            alcop_schedule s;
            alcop_schedule_default(&s);
            s.cta_group = cg;
            s.tileM = 128 * cg;
            s.tileN = tN;
            s.tileK = tK;
            s.n_stage_smem_A = s.n_stage_smem_B = st;
            s.n_stage_inner = inner;
            s.mode = ALCOP_MODE_FUSED;
            if (validate_gemm(*w, s) != ALCOP_OK) continue;
            alcop_breakdown b;
            if (alcop_predict(w, &s, hw, &b) != ALCOP_OK) continue;
            space.push_back({b.seconds, s});
          }
  clear_error();
  if (space.empty()) return set_error(ALCOP_ERR_CONFIG, "Unschedulable", "no valid schedule for workload");
  std::stable_sort(space.begin(), space.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
  space.resize(std::min<size_t>(static_cast<size_t>(budget), space.size()));
  const int n = static_cast<int>(space.size());
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  // Steady-state timing, as inside a layer step: each candidate runs as a
  // CUDA graph of back-to-back launches (PDL-chained, no host launch cost)
  // over rotating copies of the operands (in the caller's workspace) whose
  // footprint exceeds 2 x L2, so every launch reads A and B from HBM.
  // Median of 3 timed replays.
  const TuneSets ts_ = tune_sets(*w);
  const size_t a_bytes = ts_.a_bytes, b_bytes = ts_.b_bytes, set_bytes = ts_.set_bytes;
  const int nsets = ts_.nsets;
  int rc = ALCOP_OK;
  cudaStream_t ts = nullptr;
  cudaEvent_t e0 = nullptr, e1 = nullptr, ready = nullptr;
  TUNE_CUDA(cudaStreamCreateWithFlags(&ts, cudaStreamNonBlocking), "cudaStreamCreate");
  TUNE_CUDA(cudaEventCreate(&e0), "cudaEventCreate");
  TUNE_CUDA(cudaEventCreate(&e1), "cudaEventCreate");
  TUNE_CUDA(cudaEventCreateWithFlags(&ready, cudaEventDisableTiming), "cudaEventCreate");
  uint8_t* pool = static_cast<uint8_t*>(workspace);
  std::vector<const void*> As(nsets), Bs(nsets);
  std::vector<void*> Cs(nsets);
  // the copies are ordered after the caller's stream (its inputs may still be in flight)
  if (rc == ALCOP_OK) {
    TUNE_CUDA(cudaEventRecord(ready, st), "cudaEventRecord");
    TUNE_CUDA(cudaStreamWaitEvent(ts, ready, 0), "cudaStreamWaitEvent");
  }
  for (int i = 0; i < nsets && rc == ALCOP_OK; ++i) {
    uint8_t* base = pool + set_bytes * i;
    As[i] = base;
    Bs[i] = base + ((a_bytes + 255) & ~size_t(255));
    Cs[i] = base + ((a_bytes + 255) & ~size_t(255)) + ((b_bytes + 255) & ~size_t(255));
    TUNE_CUDA(cudaMemcpyAsync(const_cast<void*>(As[i]), A, a_bytes, cudaMemcpyDeviceToDevice, ts), "copy of A");
    TUNE_CUDA(cudaMemcpyAsync(const_cast<void*>(Bs[i]), B, b_bytes, cudaMemcpyDeviceToDevice, ts), "copy of B");
  }
  double bestT = 1e300;
  int out = 0;
  const int reps = std::max(1, (48 + nsets - 1) / nsets);  // >= 48 launches per timed replay set
  std::vector<cudaGraphExec_t> execs;
  std::vector<cudaGraph_t> graphs;
  std::vector<double> first;  // first-pass median per candidate
  auto time_replays = [&](cudaGraphExec_t ge, float* out_ms) -> int {
    int rc = ALCOP_OK;
    TUNE_CUDA(cudaEventRecord(e0, ts), "cudaEventRecord");
    for (int k = 0; k < reps; ++k) TUNE_CUDA(cudaGraphLaunch(ge, ts), "cudaGraphLaunch");
    TUNE_CUDA(cudaEventRecord(e1, ts), "cudaEventRecord");
    TUNE_CUDA(cudaEventSynchronize(e1), "kernel failed during tuning");
    float ms = 0;
    TUNE_CUDA(cudaEventElapsedTime(&ms, e0, e1), "cudaEventElapsedTime");
    *out_ms = ms / static_cast<float>(reps * nsets);
    return rc;
  };
  for (int i = 0; i < n && rc == ALCOP_OK; ++i) {
    const alcop_schedule& s = space[i].second;
    rc = launch_gemm(*w, s, As[0], Bs[0], Cs[0], nullptr, 0, static_cast<void*>(ts));  // validates the launch outside capture
    if (rc != ALCOP_OK) break;
    cudaGraph_t g = nullptr;
    cudaGraphExec_t ge = nullptr;
    if (cudaStreamBeginCapture(ts, cudaStreamCaptureModeThreadLocal) != cudaSuccess) {
      rc = set_error(ALCOP_ERR_CUDA, "CudaError", "stream capture failed");
      break;
    }
    for (int k = 0; k < nsets && rc == ALCOP_OK; ++k) rc = launch_gemm(*w, s, As[k], Bs[k], Cs[k], nullptr, 0, static_cast<void*>(ts));
    if (cudaStreamEndCapture(ts, &g) != cudaSuccess || rc != ALCOP_OK ||
        cudaGraphInstantiate(&ge, g, 0) != cudaSuccess) {
      if (g) cudaGraphDestroy(g);
      rc = rc != ALCOP_OK ? rc : set_error(ALCOP_ERR_CUDA, "CudaError", "graph capture of the candidate failed");
      break;
    }
    graphs.push_back(g);
    execs.push_back(ge);
    TUNE_CUDA(cudaGraphLaunch(ge, ts), "cudaGraphLaunch");  // warm-up
    if (rc != ALCOP_OK) break;
    float per[3];
    for (int r = 0; r < 3 && rc == ALCOP_OK; ++r) rc = time_replays(ge, &per[r]);
    if (rc != ALCOP_OK) break;
    std::sort(per, per + 3);
    const double t = per[1] * 1e-3;
    first.push_back(t);
    if (trials && out < trials_cap) trials[out] = alcop_tune_trial{s, space[i].first, t};
    ++out;
  }
  // Final: the three fastest of the first pass re-timed round-robin (5 rounds,
  // median): the GPU's power state drifts over a tuning run, and single
  // passes ranked near-equal schedules by it (bench: qkv pair vs single).
  if (rc == ALCOP_OK && !first.empty()) {
    std::vector<int> order(first.size());
    for (size_t i = 0; i < order.size(); ++i) order[i] = static_cast<int>(i);
    std::sort(order.begin(), order.end(), [&](int a, int b) { return first[a] < first[b]; });
    const int fin = std::min<int>(3, static_cast<int>(order.size()));
    std::vector<std::vector<float>> samples(fin);
    for (int r = 0; r < 5 && rc == ALCOP_OK; ++r)
      for (int f = 0; f < fin && rc == ALCOP_OK; ++f) {
        float ms = 0;
        rc = time_replays(execs[order[f]], &ms);
        samples[f].push_back(ms);
      }
    if (rc == ALCOP_OK) {
      for (int f = 0; f < fin; ++f) {
        std::sort(samples[f].begin(), samples[f].end());
        const double t = samples[f][samples[f].size() / 2] * 1e-3;
        if (t < bestT) {
          bestT = t;
          *best = space[order[f]].second;
        }
        if (trials && order[f] < trials_cap) trials[order[f]].measured_s = t;
      }
    }
  }
  for (auto ge : execs) cudaGraphExecDestroy(ge);
  for (auto g : graphs) cudaGraphDestroy(g);
  // the caller's C gets the best schedule's result (the tuning runs wrote the scratch copies)
  if (rc == ALCOP_OK) {
    cudaStreamSynchronize(ts);
    rc = launch_gemm(*w, *best, A, B, C, nullptr, 0, stream);
  }
  if (ts) cudaStreamSynchronize(ts);  // the caller's workspace is free again when alcop_tune returns
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
  if (ready) cudaEventDestroy(ready);
  if (ts) cudaStreamDestroy(ts);
  if (n_trials) *n_trials = out;
  return rc;
}
