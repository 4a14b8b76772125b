// consumer.cpp — TEST INFRASTRUCTURE: a compiled C++ consumer of the C ABI
// through the pipec::b200 binding (tests/cxx/pipec_b200.hpp), built against
// the read-only reference headers (/root/reference/proj/include) and
// libalcop.so by oracle/Makefile (target `consumer` -> oracle/_ref/).
//
//   alcop_consumer cpu   schedule scripts: the reference's apply_script +
//                        lower + analyze_pipelines vs the binding (same
//                        accept/reject, same rule tag, same stage mapping);
//                        simulate_pipeline / simulate_two_level equal to the
//                        reference's; the model's structural fields equal
//                        perf::predict's for the same tiles
//   alcop_consumer gpu   BASELINE config 1 (fp16 512^3, the reference's own
//                        script) through pipec::b200::run_gemm on the GPU,
//                        compared with pipec::run on the transformed program
//                        (int64, Strict-free StaleRead) — bit-exact
#include <cmath>
#include <cstring>
#include <cstdio>
#include <map>
#include <string>
#include <vector>

#include "pipec/interp.hpp"
#include "pipec/perf_model.hpp"
#include "pipec/pipeline_pass.hpp"
#include "pipec_b200.hpp"

using namespace pipec;

namespace {

int failures = 0;
void check(bool ok, const std::string& what) {
  if (!ok) {
    ++failures;
    std::printf("FAIL %s\n", what.c_str());
  }
}

std::string script_of(int64_t M, int64_t N, int64_t K, int64_t tm, int64_t tn, int64_t ko, int sA, int sB, int tA,
                      int tB) {
  std::string s = "cache_read A shared\ncache_read B shared\ncache_read A_shared register\n"
                  "cache_read B_shared register\n";
  s += "tile C i0=" + std::to_string(M / tm) + " i1=" + std::to_string(tm) + " j0=" + std::to_string(N / tn) +
       " j1=" + std::to_string(tn) + " ko=" + std::to_string(ko) + " ki=" + std::to_string(K / ko) + "\n";
  auto hint = [&](const char* b, int n) {
    if (n) s += std::string("pipeline ") + b + " " + std::to_string(n) + "\n";
  };
  hint("A_shared", sA);
  hint("B_shared", sB);
  hint("A_reg", tA);
  hint("B_reg", tB);
  return s;
}

void cpu_scripts() {
  int n = 0;
  for (int64_t M : {64, 128, 512})
    for (int64_t ko : {2, 4, 16, 64})
      for (int sA : {0, 2, 3, 5})
        for (int sB : {0, 2, 4})
          for (int tA : {0, 2, 3, 9}) {
            const int64_t N = M, K = 64 * ((M + 63) / 64);
            if (K % ko) continue;
            const std::string script = script_of(M, N, K, M / 2, N / 2, ko, sA, sB, tA, tA ? 2 : 0);
            WorkloadDesc w;
            w.M = M;
            w.N = N;
            w.K = K;
            std::string ref_rule, got_rule;
            int ref_sA = 1, ref_sB = 1, ref_inner = 1;
            try {
              Program p = lower(apply_script(gemm_schedule(w, false), script));
              PipelinePlan plan = analyze_pipelines(p);
              (void)transform(p);
              for (const auto& i : plan.infos) {
                if (i.buffer == "A_shared") ref_sA = i.stages;
                if (i.buffer == "B_shared") ref_sB = i.stages;
                if (i.buffer == "A_reg" || i.buffer == "B_reg") ref_inner = std::max(ref_inner, std::min(i.stages, 2));
              }
            } catch (const AnalysisError& e) {
              ref_rule = e.rule;
            } catch (const std::exception& e) {
              ref_rule = "other";
            }
            try {
              alcop_schedule s = b200::schedule_of(w, script);
              check(ref_rule.empty(), "accepted but the reference rejects (" + ref_rule + "): " + script);
              if (ref_rule.empty())
                check(s.n_stage_smem_A == ref_sA && s.n_stage_smem_B == ref_sB && s.n_stage_inner == ref_inner &&
                          s.tileM == M / 2 && s.tileN == N / 2 && s.tileK == K / ko,
                      "stage / tile mapping: " + script);
            } catch (const AnalysisError& e) {
              got_rule = e.rule;
              check(got_rule == ref_rule, "rule " + got_rule + " vs reference " + ref_rule + ": " + script);
            } catch (const std::exception& e) {
              check(ref_rule == "other", std::string("error ") + e.what() + " vs reference " + ref_rule);
            }
            ++n;
          }
  std::printf("scripts: %d checked\n", n);
}

void cpu_sim() {
  int n = 0;
  for (double tl : {0.0, 10.0, 30.0, 100.0})
    for (double tu : {1.0, 10.0})
      for (int64_t nl : {1, 8, 64})
        for (int np : {1, 2, 4})
          for (int nm : {1, 2}) {
            sim::SimConfig c;
            c.tLoad = tl;
            c.tUse = tu;
            c.nLoop = nl;
            c.nPipe = np;
            c.nMplx = nm;
            const sim::SimResult r = sim::simulate_pipeline(c);
            const alcop_sim_result g = b200::simulate(c);
            check(r.makespan == g.makespan && r.busy == g.busy && r.firstComputeStart == g.firstComputeStart &&
                      r.idleFraction == g.idleFraction &&
                      sim::comparable_worker_latency(r, c) == g.comparable,
                  "simulate_pipeline " + std::to_string(tl) + " " + std::to_string(nl));
            sim::SimConfig inner = c;
            inner.tLoad = tl / 4;
            inner.nLoop = 4;
            for (bool fused : {true, false})
              check(sim::simulate_two_level(c, inner, fused) == b200::two_level(c, inner, fused), "two_level");
            ++n;
          }
  std::printf("sim: %d configs checked\n", n);
}

void cpu_model_structure() {
  // the B200 model keeps the reference's loop and byte accounting (perf_model.hpp:157-187)
  int n = 0;
  for (int64_t M : {512, 4096})
    for (int64_t tK : {32, 64, 128}) {
      WorkloadDesc w;
      w.M = w.N = w.K = M;
      perf::ScheduleParams p;
      p.tileM = 128;
      p.tileN = 128;
      p.tileK = tK;
      p.regTileM = 64;  // 2 x 2 warps of 64 x 64 (params_valid, perf_model.hpp:129-142)
      p.regTileN = 64;
      p.regTileK = 16;
      p.nSmemPipeStage = 2;
      p.nRegPipeStage = 2;
      p.nWarpPerThreadblk = 4;
      const perf::LatencyBreakdown r = perf::predict(w, p, perf::HardwareSpec{});
      alcop_gemm_desc d = b200::desc_of(w, ALCOP_BF16, ALCOP_BF16);
      alcop_schedule s;
      alcop_schedule_default(&s);
      s.tileN = 128;
      s.tileK = tK;
      s.n_stage_smem_A = s.n_stage_smem_B = 2;
      alcop_hw hw;
      alcop_hw_default_b200(&hw);
      alcop_breakdown b;
      check(alcop_predict(&d, &s, &hw, &b) == ALCOP_OK, "alcop_predict");
      // same loop trip counts and per-chunk bytes (the B200 model's workset is the
      // whole problem, not the reference's per-thread-block-batch working set)
      check(b.nSmemLoop == r.nSmemLoop && b.nRegLoop == r.nRegLoop && b.bytesOneSmemLoop == r.bytesOneSmemLoop,
            "model structure at M=" + std::to_string(M) + " tileK=" + std::to_string(tK) + ": nSmemLoop " +
                std::to_string(b.nSmemLoop) + "/" + std::to_string(r.nSmemLoop) + " nRegLoop " +
                std::to_string(b.nRegLoop) + "/" + std::to_string(r.nRegLoop) + " bytesOneSmemLoop " +
                std::to_string(b.bytesOneSmemLoop) + "/" + std::to_string(r.bytesOneSmemLoop));
      ++n;
    }
  std::printf("model structure: %d checked\n", n);
}

int gpu_config1() {
  WorkloadDesc w;
  w.M = w.N = w.K = 512;
  const std::string script = script_of(512, 512, 512, 128, 128, 16, 2, 2, 2, 2);
  // the reference: transform(lower(apply_script(...))) run by the interpreter on SplitMix64 inputs
  Program q = transform(lower(apply_script(gemm_schedule(w, false), script)));
  std::map<std::string, std::vector<int64_t>> in;
  std::vector<uint16_t> hA(512 * 512), hB(512 * 512);
  uint64_t seed = 0;
  for (const char* name : {"A", "B"}) {
    SplitMix64 g(seed++);
    std::vector<int64_t> v(512 * 512);
    for (auto& x : v) x = g.range(-8, 8);
    in[name] = v;
    std::vector<uint16_t>& h = name[0] == 'A' ? hA : hB;
    for (size_t i = 0; i < v.size(); ++i) {  // small integers are exact in fp16
      const float f = static_cast<float>(v[i]);
      uint32_t bits;
      std::memcpy(&bits, &f, 4);
      const int exp = static_cast<int>((bits >> 23) & 0xff) - 127 + 15;
      const uint16_t sign = static_cast<uint16_t>((bits >> 16) & 0x8000);
      h[i] = v[i] == 0 ? 0 : static_cast<uint16_t>(sign | (exp << 10) | ((bits >> 13) & 0x3ff));
    }
  }
  const RunResult ref = run(q, in, ExecMode::StaleRead, 0);
  void *dA, *dB, *dC;
  if (cudaMalloc(&dA, hA.size() * 2) != cudaSuccess || cudaMalloc(&dB, hB.size() * 2) != cudaSuccess ||
      cudaMalloc(&dC, 512 * 512 * 4) != cudaSuccess) {
    std::printf("FAIL no GPU memory\n");
    return 1;
  }
  cudaMemcpy(dA, hA.data(), hA.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, hB.data(), hB.size() * 2, cudaMemcpyHostToDevice);
  b200::run_gemm(w, script, dA, dB, dC, nullptr, ALCOP_F16, ALCOP_F32);
  std::vector<float> C(512 * 512);
  cudaMemcpy(C.data(), dC, C.size() * 4, cudaMemcpyDeviceToHost);
  const auto& R = ref.outputs.at("C");
  int bad = 0;
  for (size_t i = 0; i < C.size(); ++i) bad += static_cast<int64_t>(C[i]) != R[i] || std::floor(C[i]) != C[i];
  check(bad == 0, "config 1: " + std::to_string(bad) + " elements differ from pipec::run");
  std::printf("gpu config 1: %d mismatches vs pipec::run\n", bad);
  cudaFree(dA);
  cudaFree(dB);
  cudaFree(dC);
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  const std::string mode = argc > 1 ? argv[1] : "cpu";
  if (mode == "cpu") {
    cpu_scripts();
    cpu_sim();
    cpu_model_structure();
  } else if (mode == "gpu") {
    gpu_config1();
  } else {
    std::printf("usage: alcop_consumer cpu|gpu\n");
    return 2;
  }
  std::printf(failures ? "FAILED %d\n" : "OK\n", failures);
  return failures ? 1 : 0;
}
