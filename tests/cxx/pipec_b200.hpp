// pipec_b200.hpp — the binding a pipec maintainer adds to call the B200 path
// (INTEGRATION.md "The binding a pipec maintainer would add").  It maps the
// reference's own types and exception classes (proj/include/pipec/common.hpp:
// 43-69, schedule.hpp:15-19, pipe_sim.hpp:15-22) onto include/alcop.h.
//
// TEST INFRASTRUCTURE when compiled with the reference headers
// (tests/cxx/consumer.cpp, built by oracle/Makefile into oracle/_ref/).
#pragma once
#include <cuda_runtime.h>

#include <stdexcept>
#include <string>

#include "alcop.h"
#include "pipec/common.hpp"
#include "pipec/pipe_sim.hpp"
#include "pipec/schedule.hpp"

namespace pipec::b200 {

// alcop return code -> the reference's exception class (cli.hpp:23-25 numbering)
[[noreturn]] inline void raise(int rc) {
  const std::string m = alcop_last_error();  // "<RuleTag>: message"
  const size_t colon = m.find(':');
  if (rc == ALCOP_ERR_ANALYSIS) throw AnalysisError(m.substr(0, colon), m);
  if (rc == ALCOP_ERR_CONFIG) throw ConfigError(m);
  if (rc == ALCOP_ERR_VALIDATE) throw ValidationError(m);
  if (rc == ALCOP_ERR_PARSE) throw ParseError(m, 0, 0);
  throw std::runtime_error(m);
}

inline alcop_gemm_desc desc_of(const WorkloadDesc& w, alcop_dtype in, alcop_dtype out) {
  alcop_gemm_desc d{};
  d.M = w.M;
  d.N = w.N;
  d.K = w.K;
  d.batch = w.batch;
  d.in_dtype = in;
  d.out_dtype = out;
  d.b_layout = ALCOP_B_KN;  // B[K,N] row-major, schedule.hpp:389
  return d;
}

// apply_script(gemm_schedule(w), script) mapped to the B200 schedule (schedule.hpp:73, :590)
inline alcop_schedule schedule_of(const WorkloadDesc& w, const std::string& script, alcop_dtype in = ALCOP_F16,
                                  alcop_dtype out = ALCOP_F32) {
  alcop_gemm_desc d = desc_of(w, in, out);
  alcop_schedule s;
  char warn[4096];
  const int rc = alcop_parse_schedule_script(&d, script.c_str(), &s, warn, sizeof warn);
  if (rc != ALCOP_OK) raise(rc);
  return s;
}

// lower -> transform -> run (schedule.hpp:357, pipeline_pass.hpp:753, interp.hpp:440) on the GPU:
// device pointers instead of std::vector<int64_t>
inline void run_gemm(const WorkloadDesc& w, const std::string& script, const void* dA, const void* dB, void* dC,
                     cudaStream_t stream, alcop_dtype in = ALCOP_F16, alcop_dtype out = ALCOP_F32) {
  alcop_gemm_desc d = desc_of(w, in, out);
  const alcop_schedule s = schedule_of(w, script, in, out);
  const int rc = alcop_gemm(&d, &s, dA, dB, dC, stream);
  if (rc != ALCOP_OK) raise(rc);
}

// tune::analytical_rank (tuner.hpp:68) on B200: the model's first pick
inline alcop_schedule choose(const alcop_gemm_desc& d) {
  alcop_hw hw;
  alcop_hw_default_b200(&hw);
  alcop_schedule s;
  const int rc = alcop_choose_schedule(&d, &hw, &s);
  if (rc != ALCOP_OK) raise(rc);
  return s;
}

// sim::simulate_pipeline / simulate_two_level (pipe_sim.hpp:54-167)
inline alcop_sim_config sim_of(const sim::SimConfig& c) {
  return alcop_sim_config{c.tLoad, c.tUse, c.nLoop, c.nPipe, c.nMplx};
}
inline alcop_sim_result simulate(const sim::SimConfig& c) {
  alcop_sim_config a = sim_of(c);
  alcop_sim_result r;
  const int rc = alcop_simulate_pipeline(&a, &r, nullptr, 0, nullptr);
  if (rc != ALCOP_OK) raise(rc);
  return r;
}
inline double two_level(const sim::SimConfig& o, const sim::SimConfig& i, bool fused) {
  alcop_sim_config ao = sim_of(o), ai = sim_of(i);
  double m = 0;
  const int rc = alcop_simulate_two_level(&ao, &ai, fused ? 1 : 0, &m);
  if (rc != ALCOP_OK) raise(rc);
  return m;
}

}  // namespace pipec::b200
