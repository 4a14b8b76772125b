// tuner.cpp — model-assisted schedule tuning on the B200 itself (SURVEY
// §8(f) rank 2): the reference's tune() (tuner.hpp:363-531) ranks a design
// space with the analytical model and "measures" the top candidates with a
// noisy simulator (measure_ground_truth, pipe_sim.hpp:195-239).  Here the
// candidates are launched and timed with CUDA events on the caller's buffers.
#include <cuda_runtime.h>

#include <algorithm>
#include <vector>

#include "alcop_internal.h"

using namespace alcop;

extern "C" int alcop_tune(const alcop_gemm_desc* w, const alcop_hw* hw, int32_t budget, const void* A, const void* B,
                          void* C, void* stream, alcop_schedule* best, alcop_tune_trial* trials, int32_t trials_cap,
                          int32_t* n_trials) {
  if (!w || !hw || !A || !B || !C || !best || budget < 1)
    return set_error(ALCOP_ERR_CONFIG, "NullArgument", "NULL argument or budget < 1");
  clear_error();
  // enumerate_space (tuner.hpp:48-64) + analytical_rank (tuner.hpp:68-80)
  std::vector<std::pair<double, alcop_schedule>> space;
  for (int cg = 1; cg <= 2; ++cg)
    for (int tN : {64, 128, 192, 256})
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
  const int n = std::min<int>(budget, static_cast<int>(space.size()));
  cudaStream_t st = reinterpret_cast<cudaStream_t>(stream);
  cudaEvent_t e0, e1;
  if (cudaEventCreate(&e0) != cudaSuccess || cudaEventCreate(&e1) != cudaSuccess)
    return set_error(ALCOP_ERR_CUDA, "CudaError", "cudaEventCreate failed");
  // each timed launch starts from a cold L2 (a 2 x L2 scratch write before
  // it, outside the events), as the model was calibrated on rotating inputs
  const size_t kFlush = size_t(256) << 20;
  void* flush = nullptr;
  if (cudaMalloc(&flush, kFlush) != cudaSuccess) {
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return set_error(ALCOP_ERR_CUDA, "CudaError", "tuning scratch allocation failed");
  }
  double bestT = 1e300;
  int out = 0;
  int rc = ALCOP_OK;
  for (int i = 0; i < n && rc == ALCOP_OK; ++i) {
    const alcop_schedule& s = space[i].second;
    rc = launch_gemm(*w, s, A, B, C, nullptr, 0, stream);  // warm-up
    const int reps = 5;
    double sum = 0;
    for (int r = 0; r < reps && rc == ALCOP_OK; ++r) {
      cudaMemsetAsync(flush, r & 0xff, kFlush, st);
      cudaEventRecord(e0, st);
      rc = launch_gemm(*w, s, A, B, C, nullptr, 0, stream);
      cudaEventRecord(e1, st);
      if (rc != ALCOP_OK) break;
      if (cudaEventSynchronize(e1) != cudaSuccess) {
        rc = set_error(ALCOP_ERR_CUDA, "CudaError", "kernel failed during tuning");
        break;
      }
      float ms = 0;
      cudaEventElapsedTime(&ms, e0, e1);
      sum += ms;
    }
    if (rc != ALCOP_OK) break;
    const double t = sum * 1e-3 / reps;
    if (trials && out < trials_cap) trials[out] = alcop_tune_trial{s, space[i].first, t};
    ++out;
    if (t < bestT) {
      bestT = t;
      *best = s;
    }
  }
  cudaFree(flush);
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  if (n_trials) *n_trials = out;
  return rc;
}
