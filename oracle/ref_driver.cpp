// ref_driver.cpp — TEST INFRASTRUCTURE (oracle/).  A thin driver over the
// reference implementation itself: it #includes the read-only pipec headers
// from /root/reference/proj/include (never copied into this repo) and calls
// the reference's own functions, so its outputs are the reference's outputs.
// Built by oracle/Makefile into oracle/_ref/ref_driver (git-ignored).
//
// Commands (all write JSON / text to stdout or --outdir):
//   gemm      apply_script(gemm_schedule) -> lower -> transform -> run;
//             emits lowered/transformed IR, the plan, the interpreter trace,
//             the int64 outputs and a per-tile "walk" of every copy / sync /
//             pipelined-buffer read with its evaluated slot and chunk indices
//   script    apply_script only: {"ok":..} or the exception class + rule tag
//   model     perf:: functions on a JSON list of queries (SPEC examples and
//             grids) -> predictions
//   (model)   also sim / simtrace / sim2: sim::simulate_pipeline stats, its
//             event trace, and sim::simulate_two_level (fused | restart)
//   splitmix  first N draws / range(-8,8) values for a seed
//   time      wall time of pipec::run on a lowered+transformed GEMM
//
// Usage is only through oracle/gen_golden.py and bench.py --impl reference.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <string>
#include <vector>

#include "pipec/interp.hpp"
#include "pipec/perf_model.hpp"
#include "pipec/pipe_sim.hpp"
#include "pipec/pipeline_pass.hpp"
#include "pipec/printer.hpp"
#include "pipec/schedule.hpp"

using namespace pipec;

namespace {

std::map<std::string, std::string> parse_args(int argc, char** argv, int from) {
  std::map<std::string, std::string> a;
  for (int i = from; i < argc; ++i) {
    std::string k = argv[i];
    if (k.rfind("--", 0) == 0) {
      std::string v = (i + 1 < argc && std::string(argv[i + 1]).rfind("--", 0) != 0) ? argv[++i] : "1";
      a[k.substr(2)] = v;
    }
  }
  return a;
}

std::string read_file(const std::string& p) {
  std::ifstream in(p);
  if (!in) throw ConfigError("cannot open " + p);
  std::ostringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

void write_file(const std::string& p, const std::string& s) {
  std::ofstream out(p);
  out << s;
}

std::string jstr(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\';
    if (c == '\n') {
      o += "\\n";
      continue;
    }
    o += c;
  }
  return o + "\"";
}

// cli.hpp:41-46 (cli.hpp itself needs CLI11, absent): same generator class
std::vector<int64_t> random_tensor(int64_t count, uint64_t seed) {
  SplitMix64 rng(seed);
  std::vector<int64_t> v(count);
  for (auto& x : v) x = rng.range(-8, 8);
  return v;
}

std::string plan_json(const PipelinePlan& plan) {
  std::ostringstream o;
  o << "[";
  for (size_t i = 0; i < plan.infos.size(); ++i) {
    const auto& b = plan.infos[i];
    o << (i ? ",\n " : "") << "{\"buffer\":" << jstr(b.buffer) << ",\"stages\":" << b.stages
      << ",\"producerTensor\":" << jstr(b.producerTensor) << ",\"pipelinedLoopVar\":" << jstr(b.pipelinedLoopVar)
      << ",\"pipelinedLoopExtent\":" << b.pipelinedLoopExtent << ",\"parent\":" << b.parent
      << ",\"level\":" << b.level << ",\"predicateWaits\":" << b.predicateWaits
      << ",\"drainPairs\":" << b.drainPairs << ",\"prologueSitePath\":" << jstr(b.prologueSitePath)
      << ",\"loadRegionPath\":" << jstr(b.loadRegionPath) << ",\"useRegionPath\":" << jstr(b.useRegionPath) << "}";
  }
  o << "]";
  return o.str();
}

// ---- per-tile walk of the transformed nest -------------------------------
// Sequential loops iterate fully; parallel loops (tiles, batch) and unrolled
// loops (elements of one chunk) take value 0 only, so each copy of a chunk
// appears once.  Every index is evaluated with the reference's own eval().
struct Walker {
  const Program& p;
  std::map<std::string, int64_t> env;
  std::ostringstream out;
  int64_t n = 0;
  std::map<std::string, bool> pipelined;
  std::map<std::string, int64_t> tileK;  // shared-buffer k extent (for chunk numbers)

  int64_t ev(const ExprPtr& e) {
    return eval(*e, [&](const std::string& v) -> int64_t {
      auto it = env.find(v);
      if (it == env.end()) throw InterpError("walk: unbound " + v);
      return it->second;
    });
  }
  std::string loopvars() {
    std::ostringstream o;
    o << "{";
    bool first = true;
    for (const auto& [k, v] : env) {
      o << (first ? "" : ",") << jstr(k) << ":" << v;
      first = false;
    }
    o << "}";
    return o.str();
  }
  void emit(const std::string& body) { out << "{\"i\":" << n++ << "," << body << ",\"env\":" << loopvars() << "}\n"; }

  void walk(const std::vector<StmtPtr>& body) {
    for (const auto& s : body) walk(*s);
  }
  void walk(const Stmt& s) {
    switch (s.kind) {
      case Stmt::Kind::For: {
        int64_t ext = s.loopKind == LoopKind::Sequential ? s.extent : 1;
        for (int64_t i = 0; i < ext; ++i) {
          env[s.var] = i;
          walk(s.body);
        }
        env.erase(s.var);
        return;
      }
      case Stmt::Kind::Block: walk(s.body); return;
      case Stmt::Kind::Predicated:
        if (ev(s.cond) != 0) walk(s.body);
        return;
      case Stmt::Kind::Sync:
        emit("\"op\":" + jstr(sync_kind_name(s.syncKind)) + ",\"group\":" + jstr(s.group));
        return;
      case Stmt::Kind::AsyncCopy: {
        std::ostringstream b;
        b << "\"op\":\"copy\",\"dst\":" << jstr(s.dstBuffer) << ",\"src\":" << jstr(s.srcBuffer) << ",\"dstIdx\":[";
        for (size_t k = 0; k < s.dstIndices.size(); ++k) b << (k ? "," : "") << ev(s.dstIndices[k]);
        b << "],\"srcIdx\":[";
        for (size_t k = 0; k < s.srcIndices.size(); ++k) b << (k ? "," : "") << ev(s.srcIndices[k]);
        b << "]";
        emit(b.str());
        return;
      }
      case Stmt::Kind::Compute: {
        bool touches = false;
        for (const auto& op : s.operands) touches |= pipelined.count(op.buffer) > 0;
        if (!touches) return;
        std::ostringstream b;
        b << "\"op\":\"read\",\"tag\":" << jstr(s.opTag) << ",\"operands\":[";
        bool first = true;
        for (const auto& op : s.operands) {
          if (!pipelined.count(op.buffer)) continue;
          b << (first ? "" : ",") << "{\"buf\":" << jstr(op.buffer) << ",\"idx\":[";
          for (size_t k = 0; k < op.indices.size(); ++k) b << (k ? "," : "") << ev(op.indices[k]);
          b << "]}";
          first = false;
        }
        b << "]";
        emit(b.str());
        return;
      }
    }
  }
};

int cmd_gemm(const std::map<std::string, std::string>& a) {
  WorkloadDesc w;
  w.M = std::stoll(a.at("M"));
  w.N = std::stoll(a.at("N"));
  w.K = std::stoll(a.at("K"));
  w.batch = a.count("batch") ? std::stoll(a.at("batch")) : 1;
  w.elemBytes = 2;
  std::string script = read_file(a.at("script"));
  std::string outdir = a.at("outdir");
  uint64_t seed = a.count("seed") ? std::stoull(a.at("seed")) : 0;
  bool doRun = !a.count("no-run");
  ExecMode mode = (a.count("mode") && a.at("mode") == "stale") ? ExecMode::StaleRead : ExecMode::Strict;
  const bool preOp = a.count("preop") && a.at("preop") == "1";

  std::vector<std::string> warnings;
  ScheduleState st = apply_script(gemm_schedule(w, preOp), script, &warnings);
  Program p = lower(st);
  PipelinePlan plan = analyze_pipelines(p);
  Program q = transform(p);
  write_file(outdir + "/lowered.ir", print_program(p));
  write_file(outdir + "/transformed.ir", print_program(q));
  write_file(outdir + "/plan.json", plan_json(plan) + "\n");
  {
    std::ostringstream o;
    o << "[";
    for (size_t i = 0; i < warnings.size(); ++i) o << (i ? "," : "") << jstr(warnings[i]);
    o << "]\n";
    write_file(outdir + "/warnings.json", o.str());
  }
  Walker wk{q};
  for (const auto& b : q.locals)
    if (q.find_group(b.name)) wk.pipelined[b.name] = true;
  wk.walk(q.body);
  write_file(outdir + "/walk.jsonl", wk.out.str());
  if (doRun) {
    std::map<std::string, std::vector<int64_t>> inputs;
    int which = 0;
    for (const auto& b : p.inputs) inputs[b.name] = random_tensor(b.elem_count(), seed + which++);
    auto t0 = std::chrono::steady_clock::now();
    RunResult r = run(q, inputs, mode, seed);
    auto t1 = std::chrono::steady_clock::now();
    std::ostringstream tr;
    for (const auto& e : r.trace)
      tr << "{\"step\":" << e.step << ",\"kind\":" << jstr(sync_kind_name(e.kind)) << ",\"group\":" << jstr(e.group)
         << ",\"acquired\":" << e.acquired << ",\"committed\":" << e.committed << ",\"waited\":" << e.waited
         << ",\"released\":" << e.released << ",\"inflight\":" << e.inflight << "}\n";
    write_file(outdir + "/trace.jsonl", tr.str());
    const auto& C = r.outputs.at("C");
    std::ofstream cb(outdir + "/C.bin", std::ios::binary);
    cb.write(reinterpret_cast<const char*>(C.data()), static_cast<std::streamsize>(C.size() * sizeof(int64_t)));
    uint64_t h = 0xcbf29ce484222325ull;
    for (int64_t v : C) h = fnv1a_mix(h, v);
    std::ostringstream meta;
    meta << "{\"run_seconds\":" << std::chrono::duration<double>(t1 - t0).count() << ",\"C_fnv1a\":\"" << std::hex
         << h << std::dec << "\",\"C_elems\":" << C.size() << "}\n";
    write_file(outdir + "/run.json", meta.str());
  }
  return 0;
}

int cmd_script(const std::map<std::string, std::string>& a) {
  WorkloadDesc w;
  w.M = std::stoll(a.at("M"));
  w.N = std::stoll(a.at("N"));
  w.K = std::stoll(a.at("K"));
  w.batch = a.count("batch") ? std::stoll(a.at("batch")) : 1;
  std::string script = read_file(a.at("script"));
  const bool preOp = a.count("preop") && a.at("preop") == "1";
  std::vector<std::string> warnings;
  try {
    ScheduleState st = apply_script(gemm_schedule(w, preOp), script, &warnings);
    Program p = lower(st);
    PipelinePlan plan = analyze_pipelines(p);
    Program q = transform(p);
    (void)q;
    std::cout << "{\"ok\":true,\"warnings\":" << warnings.size() << ",\"plan\":" << plan_json(plan) << "}\n";
  } catch (const AnalysisError& e) {
    std::cout << "{\"ok\":false,\"class\":\"AnalysisError\",\"rule\":" << jstr(e.rule) << ",\"what\":" << jstr(e.what())
              << "}\n";
  } catch (const ConfigError& e) {
    std::cout << "{\"ok\":false,\"class\":\"ConfigError\",\"rule\":\"\",\"what\":" << jstr(e.what()) << "}\n";
  } catch (const ValidationError& e) {
    std::cout << "{\"ok\":false,\"class\":\"ValidationError\",\"rule\":\"\",\"what\":" << jstr(e.what()) << "}\n";
  } catch (const std::exception& e) {
    std::cout << "{\"ok\":false,\"class\":\"other\",\"rule\":\"\",\"what\":" << jstr(e.what()) << "}\n";
  }
  return 0;
}

// model queries, one per line: "<fn> args..."
int cmd_model(const std::map<std::string, std::string>& a) {
  std::istringstream in(read_file(a.at("queries")));
  std::string line;
  std::cout.precision(17);
  while (std::getline(in, line)) {
    std::istringstream ls(line);
    std::string fn;
    if (!(ls >> fn)) continue;
    perf::HardwareSpec hw;
    if (fn == "pipeline_latency") {
      double tl, tu;
      int64_t n;
      int np, nm;
      ls >> tl >> tu >> n >> np >> nm;
      std::cout << perf::pipeline_latency(tl, tu, n, np, nm) << "\n";
    } else if (fn == "smem_load_latency") {
      int64_t b, ws, ntb;
      ls >> b >> ws >> ntb >> hw.bwLLC >> hw.bwDRAM >> hw.latLLCRead >> hw.latDRAMRead;
      std::cout << perf::smem_load_latency(b, ws, ntb, hw) << "\n";
    } else if (fn == "epilogue_latency") {
      int64_t b, ntb;
      ls >> b >> ntb >> hw.bwDRAMWrite >> hw.latDRAMWrite;
      std::cout << perf::epilogue_latency(b, ntb, hw) << "\n";
    } else if (fn == "compute_latency") {
      int64_t f;
      int nw;
      int64_t ntb;
      ls >> f >> hw.throughputSM >> nw >> ntb;
      std::cout << perf::compute_latency(f, hw, nw, ntb) << "\n";
    } else if (fn == "predict") {
      WorkloadDesc w;
      perf::ScheduleParams sp;
      ls >> w.M >> w.N >> w.K >> w.batch >> sp.tileM >> sp.tileN >> sp.tileK >> sp.regTileM >> sp.regTileN >>
          sp.regTileK >> sp.nSmemPipeStage >> sp.nRegPipeStage >> sp.nWarpPerThreadblk;
      try {
        auto b = perf::predict(w, sp, hw);
        std::cout << b.tKernel << " " << b.tThreadblk << " " << b.tInit << " " << b.tMainLoop << " " << b.tEpilogue
                  << " " << b.tSmemLoad << " " << b.tRegLoad << " " << b.tSmemUse << " " << b.tCompute << " "
                  << b.nThreadblkBatch << " " << b.nThreadblkPerSM << "\n";
      } catch (const std::exception& e) {
        std::cout << "error\n";
      }
    } else if (fn == "sim") {
      sim::SimConfig c;
      ls >> c.tLoad >> c.tUse >> c.nLoop >> c.nPipe >> c.nMplx;
      try {
        auto r = sim::simulate_pipeline(c);
        std::cout << r.makespan << " " << r.firstComputeStart << " " << r.busy << " " << r.idleFraction << " "
                  << sim::comparable_worker_latency(r, c) << "\n";
      } catch (const std::exception& e) {
        std::cout << "error\n";
      }
    } else if (fn == "simtrace") {
      sim::SimConfig c;
      ls >> c.tLoad >> c.tUse >> c.nLoop >> c.nPipe >> c.nMplx;
      auto r = sim::simulate_pipeline(c, true);
      for (size_t i = 0; i < r.trace.size(); ++i)
        std::cout << (i ? " " : "") << r.trace[i].time << ":" << r.trace[i].worker << ":"
                  << sim::sim_event_name(r.trace[i].kind) << ":" << r.trace[i].iteration;
      std::cout << "\n";
    } else if (fn == "sim2") {
      sim::SimConfig o, in;
      int fused;
      ls >> o.tLoad >> o.tUse >> o.nLoop >> o.nPipe >> in.tLoad >> in.tUse >> in.nLoop >> in.nPipe >> fused;
      try {
        std::cout << sim::simulate_two_level(o, in, fused != 0) << "\n";
      } catch (const std::exception& e) {
        std::cout << "error\n";
      }
    } else {
      std::cout << "unknown\n";
    }
  }
  return 0;
}

int cmd_splitmix(const std::map<std::string, std::string>& a) {
  uint64_t seed = std::stoull(a.at("seed"));
  int64_t n = std::stoll(a.at("count"));
  SplitMix64 r(seed);
  std::vector<uint64_t> raw;
  for (int64_t i = 0; i < n; ++i) raw.push_back(r.next());
  auto v = random_tensor(n, seed);
  std::cout << "{\"raw\":[";
  for (int64_t i = 0; i < n; ++i) std::cout << (i ? "," : "") << "\"" << raw[i] << "\"";
  std::cout << "],\"range\":[";
  for (int64_t i = 0; i < n; ++i) std::cout << (i ? "," : "") << v[i];
  std::cout << "]}\n";
  return 0;
}

int cmd_time(const std::map<std::string, std::string>& a) {
  WorkloadDesc w;
  w.M = std::stoll(a.at("M"));
  w.N = std::stoll(a.at("N"));
  w.K = std::stoll(a.at("K"));
  w.batch = a.count("batch") ? std::stoll(a.at("batch")) : 1;
  w.elemBytes = 2;
  std::string script = read_file(a.at("script"));
  uint64_t seed = a.count("seed") ? std::stoull(a.at("seed")) : 0;
  ExecMode mode = (a.count("mode") && a.at("mode") == "stale") ? ExecMode::StaleRead : ExecMode::Strict;
  int reps = a.count("reps") ? std::stoi(a.at("reps")) : 1;
  Program q = transform(lower(apply_script(gemm_schedule(w, false), script)));
  std::map<std::string, std::vector<int64_t>> inputs;
  int which = 0;
  for (const auto& b : q.inputs) inputs[b.name] = random_tensor(b.elem_count(), seed + which++);
  double best = 1e300, total = 0;
  uint64_t h = 0;
  for (int i = 0; i < reps; ++i) {
    auto t0 = std::chrono::steady_clock::now();
    RunResult r = run(q, inputs, mode, seed);
    auto t1 = std::chrono::steady_clock::now();
    double s = std::chrono::duration<double>(t1 - t0).count();
    best = std::min(best, s);
    total += s;
    h = 0xcbf29ce484222325ull;
    for (int64_t v : r.outputs.at("C")) h = fnv1a_mix(h, v);
  }
  std::cout << "{\"best_s\":" << best << ",\"mean_s\":" << total / reps << ",\"flops\":" << 2.0 * w.M * w.N * w.K * w.batch
            << ",\"C_fnv1a\":\"" << std::hex << h << std::dec << "\"}\n";
  return 0;
}

}  // namespace

int main(int argc, char** argv) {
  if (argc < 2) {
    std::cerr << "usage: ref_driver gemm|script|model|splitmix|time --key value ...\n";
    return 6;
  }
  std::string cmd = argv[1];
  auto a = parse_args(argc, argv, 2);
  try {
    if (cmd == "gemm") return cmd_gemm(a);
    if (cmd == "script") return cmd_script(a);
    if (cmd == "model") return cmd_model(a);
    if (cmd == "splitmix") return cmd_splitmix(a);
    if (cmd == "time") return cmd_time(a);
  } catch (const AnalysisError& e) {
    std::cerr << "analysis error [" << e.rule << "]: " << e.what() << "\n";
    return 4;
  } catch (const InterpError& e) {
    std::cerr << "execution error: " << e.what() << "\n";
    return 4;
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 6;
  }
  std::cerr << "unknown command\n";
  return 6;
}
