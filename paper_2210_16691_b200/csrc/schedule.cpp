// schedule.cpp — the reference's schedule surface on the B200 host side.
//
// A from-scratch C++ restatement of pipec's value-semantics schedule state
// (schedule.hpp:15-62) and primitives — cache_read (:111-136), tile
// (:141-193), check_eligibility (:198-254), mark_pipeline (:258-268),
// inline_tensor (:275-314), apply_script (:590-646) — with the same rule
// tags and error classes, ending in a mapping onto alcop_schedule instead of
// lower() (:357-584): the B200 kernel *is* the lowered-and-transformed nest.
//
// Also the host bookkeeping enumerator: the producer / consumer event
// sequence the kernel executes (pipeline_pass.hpp:482-748 index algebra,
// interp.hpp:375-418 counters), used to check the device trace bit-exactly.
#include <algorithm>
#include <cstring>
#include <map>
#include <optional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <vector>

#include "alcop_internal.h"

namespace alcop {
namespace sched {

enum class Scope { Global, Shared, Register };
inline int scope_level(Scope s) { return s == Scope::Global ? 2 : s == Scope::Shared ? 1 : 0; }
inline const char* scope_name(Scope s) {
  return s == Scope::Global ? "global" : s == Scope::Shared ? "shared" : "register";
}
enum class LoopKind { Sequential, Parallel, Unrolled };

struct Error : std::runtime_error {
  int code;
  std::string rule;
  Error(int c, std::string r, const std::string& m) : std::runtime_error(m), code(c), rule(std::move(r)) {}
};
[[noreturn]] inline void analysis(const std::string& rule, const std::string& msg) {
  throw Error(ALCOP_ERR_ANALYSIS, rule, msg);
}
[[noreturn]] inline void config(const std::string& msg) { throw Error(ALCOP_ERR_CONFIG, "ConfigError", msg); }

struct Node {
  enum class Producer { ExternalInput, AsyncCopyFrom, ComputeFrom };
  std::string name;
  Producer producer = Producer::ExternalInput;
  std::string copySrc;
  std::vector<std::string> computeSrcs;
  std::string opTag;
  Scope scope = Scope::Global;
  std::optional<int> stages;
  bool fusedPreOp = false;
  int chunkLevel = -1;
};

struct Loop {
  std::string var;
  int64_t extent = 0;
  LoopKind kind = LoopKind::Sequential;
  char dim = '?';
  int splitLevel = 0;
};

struct State {
  int64_t M = 0, N = 0, K = 0, batch = 1;
  std::vector<Node> graph;
  std::vector<Loop> sketch;
  bool tiled = false;
  const Node* find(const std::string& n) const {
    for (const auto& x : graph)
      if (x.name == n) return &x;
    return nullptr;
  }
  Node* find_mut(const std::string& n) {
    for (auto& x : graph)
      if (x.name == n) return &x;
    return nullptr;
  }
};

// gemm_schedule (schedule.hpp:73-86); preOp adds S2 = ew(A) feeding the mma
State gemm_schedule(const alcop_gemm_desc& w) {
  State s;
  s.M = w.M;
  s.N = w.N;
  s.K = w.K;
  s.batch = w.batch;
  s.graph.push_back({"A", Node::Producer::ExternalInput, "", {}, "", Scope::Global, {}, false, -1});
  s.graph.push_back({"B", Node::Producer::ExternalInput, "", {}, "", Scope::Global, {}, false, -1});
  std::string aSide = "A";
  if (w.pre_op) {
    s.graph.push_back({"S2", Node::Producer::ComputeFrom, "", {"A"}, "ew", Scope::Global, {}, false, -1});
    aSide = "S2";
  }
  s.graph.push_back({"C", Node::Producer::ComputeFrom, "", {aSide, "B"}, "mma", Scope::Global, {}, false, -1});
  return s;
}

std::string cache_name(const std::string& tensor, Scope scope) {
  std::string base = tensor;
  for (const char* suffix : {"_shared", "_reg"}) {
    size_t n = std::strlen(suffix);
    if (base.size() > n && base.compare(base.size() - n, n, suffix) == 0) base = base.substr(0, base.size() - n);
  }
  return base + (scope == Scope::Shared ? "_shared" : "_reg");
}

std::vector<const Loop*> reduction_splits(const State& s) {
  std::vector<const Loop*> ks;
  for (const auto& l : s.sketch)
    if (l.dim == 'k') ks.push_back(&l);
  return ks;
}

State cache_read(const State& s, const std::string& tensor, Scope scope) {
  const Node* src = s.find(tensor);
  if (!src) analysis("NoSuchTensor", "cache_read: tensor '" + tensor + "' not found");
  if (scope_level(scope) >= scope_level(src->scope))
    analysis("ScopeNotBelow", std::string("cache_read: scope ") + scope_name(scope) + " is not strictly below " +
                                  scope_name(src->scope));
  State out = s;
  Node buf;
  buf.name = cache_name(tensor, scope);
  if (out.find(buf.name)) analysis("DuplicateBuffer", "cache_read: buffer '" + buf.name + "' already exists");
  buf.producer = Node::Producer::AsyncCopyFrom;
  buf.copySrc = tensor;
  buf.scope = scope;
  buf.chunkLevel = scope == Scope::Shared ? 0 : 1;
  for (auto& n : out.graph) {
    if (n.name == tensor) continue;
    if (n.producer == Node::Producer::AsyncCopyFrom && n.copySrc == tensor) n.copySrc = buf.name;
    for (auto& cs : n.computeSrcs)
      if (cs == tensor) cs = buf.name;
  }
  out.graph.push_back(std::move(buf));
  return out;
}

State tile(const State& s, const std::string& tensor, const std::vector<std::pair<std::string, int64_t>>& splits) {
  if (!s.find(tensor) || tensor != "C") analysis("NoSuchTensor", "tile: only the output computation can be tiled");
  std::map<char, std::vector<std::pair<std::string, int64_t>>> byDim;
  for (const auto& [name, extent] : splits) {
    if (name.empty() || (name[0] != 'i' && name[0] != 'j' && name[0] != 'k'))
      analysis("BadSplit", "tile: split '" + name + "' must start with i, j or k");
    if (extent < 1) analysis("BadSplit", "tile: split extent must be >= 1");
    byDim[name[0]].emplace_back(name, extent);
  }
  auto dim_size = [&](char d) -> int64_t { return d == 'i' ? s.M : d == 'j' ? s.N : s.K; };
  for (char d : {'i', 'j', 'k'}) {
    int64_t prod = 1;
    for (const auto& [name, extent] : byDim[d]) prod *= extent;
    if (byDim[d].empty()) analysis("BadSplit", std::string("tile: missing splits for dimension '") + d + "'");
    if (prod != dim_size(d))
      analysis("NonDivisibleSplit", std::string("tile: splits of '") + d + "' multiply to " + std::to_string(prod) +
                                        ", dimension is " + std::to_string(dim_size(d)));
    if (byDim[d].size() > 2) analysis("BadSplit", "tile: at most two splits per dimension");
  }
  State out = s;
  out.sketch.clear();
  if (s.batch > 1) out.sketch.push_back({"b", s.batch, LoopKind::Parallel, 'b', 0});
  auto push_dim = [&](char d, size_t level, LoopKind kind) {
    if (level < byDim[d].size()) {
      const auto& [name, extent] = byDim[d][level];
      out.sketch.push_back({name, extent, kind, d, static_cast<int>(level)});
    }
  };
  push_dim('i', 0, LoopKind::Parallel);
  push_dim('j', 0, LoopKind::Parallel);
  push_dim('k', 0, LoopKind::Sequential);
  push_dim('k', 1, LoopKind::Sequential);
  push_dim('i', 1, LoopKind::Unrolled);
  push_dim('j', 1, LoopKind::Unrolled);
  out.tiled = true;
  return out;
}

struct Eligibility {
  bool eligible = false;
  std::string failedRule, explanation;
};

Eligibility check_eligibility(const State& s, const std::string& buffer) {
  Eligibility r;
  const Node* b = s.find(buffer);
  if (!b) analysis("NoSuchTensor", "check_eligibility: '" + buffer + "' not found");
  if (!s.tiled) analysis("OrderingViolation", "pipeline requires loop sketch: tile before checking eligibility");
  // rule 1: produced by an asynchronous memory copy
  if (b->producer != Node::Producer::AsyncCopyFrom) {
    r.failedRule = "NotAsyncProducer";
    r.explanation = "buffer '" + buffer + "' is not produced by an asynchronous memory copy";
    return r;
  }
  // rule 2: a sequential load-and-use loop encloses the buffer's copy
  auto pipelined_loop_of = [&](const Node& node) -> const Loop* {
    auto ks = reduction_splits(s);
    int lastIdx = -1;
    if (node.chunkLevel >= 0 && node.chunkLevel < static_cast<int>(ks.size())) {
      const Loop* chunkLoop = ks[node.chunkLevel];
      for (size_t i = 0; i < s.sketch.size(); ++i)
        if (&s.sketch[i] == chunkLoop) lastIdx = static_cast<int>(i);
    } else {
      lastIdx = static_cast<int>(s.sketch.size()) - 1;
    }
    for (int i = lastIdx; i >= 0; --i)
      if (s.sketch[i].kind == LoopKind::Sequential) return &s.sketch[i];
    return nullptr;
  };
  const Loop* loop = pipelined_loop_of(*b);
  if (!loop) {
    r.failedRule = "NoSequentialLoop";
    r.explanation = "buffer '" + buffer + "' is not produced inside a sequential loop";
    return r;
  }
  // rule 3: same-scope (shared) pipelined buffers share one sync position
  if (b->scope == Scope::Shared) {
    for (const auto& other : s.graph) {
      if (other.name == buffer || !other.stages || other.scope != Scope::Shared) continue;
      const Loop* otherLoop = pipelined_loop_of(other);
      if (otherLoop && otherLoop->var != loop->var) {
        r.failedRule = "SyncPositionConflict";
        r.explanation = "buffers '" + other.name + "' (loop " + otherLoop->var + ") and '" + buffer + "' (loop " +
                        loop->var + ") need shared-scope barriers at different positions";
        return r;
      }
    }
  }
  r.eligible = true;
  r.explanation = "pipelined loop " + loop->var;
  return r;
}

State mark_pipeline(const State& s, const std::string& buffer, int stages) {
  if (!s.tiled) analysis("OrderingViolation", "pipeline requires loop sketch: tile first");
  if (stages < 2) analysis("BadStages", "pipeline stages must be >= 2");
  Eligibility r = check_eligibility(s, buffer);
  if (!r.eligible) analysis(r.failedRule, r.explanation);
  State out = s;
  out.find_mut(buffer)->stages = stages;
  return out;
}

// inline_tensor (schedule.hpp:275-314): case 2 (the consumer buffer is already
// pipelined) re-sources the buffer to the tensor's input and fuses the
// elementwise op into its consumer (mma -> mma_ewa); otherwise classic
// inlining makes the buffer compute-produced (and rule 1 rejects it later).
State inline_tensor(const State& s, const std::string& tensor) {
  const Node* t = s.find(tensor);
  if (!t) analysis("NoSuchTensor", "inline: tensor '" + tensor + "' not found");
  if (t->producer != Node::Producer::ComputeFrom || t->computeSrcs.size() != 1)
    analysis("NotElementwise", "inline: '" + tensor + "' is not unary elementwise");
  const std::string src = t->computeSrcs[0];
  const std::string tag = t->opTag;
  State out = s;
  bool consumed = false;
  for (auto& n : out.graph) {
    if (n.producer == Node::Producer::AsyncCopyFrom && n.copySrc == tensor) {
      consumed = true;
      if (n.stages) {
        if (n.fusedPreOp)
          analysis("NoRewrite", "inline: buffer '" + n.name + "' already carries a fused elementwise op");
        n.copySrc = src;
        n.fusedPreOp = true;
      } else {
        n.producer = Node::Producer::ComputeFrom;
        n.computeSrcs = {src};
        n.opTag = tag;
        n.copySrc.clear();
      }
    } else {
      for (auto& cs : n.computeSrcs)
        if (cs == tensor) analysis("NoRewrite", "inline: v1 requires '" + tensor + "' to feed cache-read buffers");
    }
  }
  if (!consumed) analysis("NoRewrite", "inline: '" + tensor + "' has no cache-read consumer");
  out.graph.erase(std::remove_if(out.graph.begin(), out.graph.end(),
                                 [&](const Node& n) { return n.name == tensor; }),
                  out.graph.end());
  return out;
}

State apply_script(const State& start, const std::string& script, std::vector<std::string>* warnings) {
  State s = start;
  std::istringstream in(script);
  std::string line;
  int lineNo = 0;
  while (std::getline(in, line)) {
    ++lineNo;
    auto hash = line.find('#');
    if (hash != std::string::npos) line = line.substr(0, hash);
    std::istringstream ls(line);
    std::vector<std::string> tok;
    std::string t;
    while (ls >> t) tok.push_back(t);
    if (tok.empty()) continue;
    auto fail = [&](const std::string& msg) { config("schedule script line " + std::to_string(lineNo) + ": " + msg); };
    if (tok[0] == "cache_read") {
      if (tok.size() != 3) fail("expected: cache_read <tensor> <shared|register>");
      Scope sc;
      if (tok[2] == "shared")
        sc = Scope::Shared;
      else if (tok[2] == "register")
        sc = Scope::Register;
      else
        config("bad scope '" + tok[2] + "'");
      s = cache_read(s, tok[1], sc);
    } else if (tok[0] == "tile") {
      if (tok.size() < 3) fail("expected: tile <tensor> <name>=<extent>...");
      std::vector<std::pair<std::string, int64_t>> splits;
      for (size_t i = 2; i < tok.size(); ++i) {
        auto eq = tok[i].find('=');
        if (eq == std::string::npos) fail("bad split '" + tok[i] + "'");
        int64_t v = 0;
        try {
          v = std::stoll(tok[i].substr(eq + 1));
        } catch (...) {
          fail("bad split '" + tok[i] + "'");
        }
        splits.emplace_back(tok[i].substr(0, eq), v);
      }
      s = tile(s, tok[1], splits);
    } else if (tok[0] == "pipeline") {
      if (tok.size() != 3) fail("expected: pipeline <buffer> <stages>");
      int st = 0;
      try {
        st = std::stoi(tok[2]);
      } catch (...) {
        fail("bad stage count '" + tok[2] + "'");
      }
      try {
        s = mark_pipeline(s, tok[1], st);
      } catch (const Error& e) {
        if (e.rule == "SyncPositionConflict") {
          for (auto& n : s.graph)
            if (n.stages && n.scope == Scope::Shared) n.stages.reset();
          if (warnings) warnings->push_back(std::string("refusing to pipeline: ") + e.what());
        } else {
          throw;
        }
      }
    } else if (tok[0] == "inline") {
      if (tok.size() != 2) fail("expected: inline <tensor>");
      s = inline_tensor(s, tok[1]);
    } else {
      fail("unknown primitive '" + tok[0] + "'");
    }
  }
  return s;
}

// Which input a cached buffer's chain roots at (schedule.hpp:411-425).
char side_of(const State& s, const Node& n) {
  const Node* cur = &n;
  while (cur) {
    if (cur->name == "B") return 'b';
    if (cur->name == "A") return 'a';
    if (cur->producer == Node::Producer::AsyncCopyFrom)
      cur = s.find(cur->copySrc);
    else if (cur->producer == Node::Producer::ComputeFrom && !cur->computeSrcs.empty())
      cur = s.find(cur->computeSrcs[0]);
    else
      break;
  }
  return 'a';
}

// lower()'s tile arithmetic (schedule.hpp:362-381) and the analysis rules
// the pass would apply to the lowered nest (pipeline_pass.hpp:275-314),
// mapped onto the B200 schedule.
alcop_schedule to_alcop(const State& s) {
  if (!s.tiled) analysis("OrderingViolation", "lower: tile must run first");
  auto ks = reduction_splits(s);
  const Loop *i0 = nullptr, *j0 = nullptr, *i1 = nullptr, *j1 = nullptr;
  for (const auto& l : s.sketch) {
    if (l.dim == 'i' && l.splitLevel == 0) i0 = &l;
    if (l.dim == 'i' && l.splitLevel == 1) i1 = &l;
    if (l.dim == 'j' && l.splitLevel == 0) j0 = &l;
    if (l.dim == 'j' && l.splitLevel == 1) j1 = &l;
  }
  if (!i0 || !j0 || ks.empty()) analysis("BadSketch", "lower: sketch is incomplete");
  alcop_schedule out;
  alcop_schedule_default(&out);
  out.tileM = i1 ? i1->extent : s.M / i0->extent;
  out.tileN = j1 ? j1->extent : s.N / j0->extent;
  out.tileK = s.K / ks[0]->extent;
  const int64_t F = ks.size() > 1 ? ks[1]->extent : 1;  // inner pipelined loop extent
  if (ks.size() > 1 && out.tileK % F != 0)
    analysis("NonDivisibleSplit", "lower: inner reduction split does not divide tile");
  out.n_stage_smem_A = 1;
  out.n_stage_smem_B = 1;
  out.n_stage_inner = 1;
  out.mode = ALCOP_MODE_WRAP;  // the reference's own emission
  int sharedStages[2] = {0, 0};
  int regStages[2] = {0, 0};
  for (const auto& n : s.graph) {
    if (!n.stages) continue;
    const int side = side_of(s, n) == 'a' ? 0 : 1;
    if (n.scope == Scope::Shared)
      sharedStages[side] = *n.stages;
    else if (n.scope == Scope::Register)
      regStages[side] = *n.stages;
  }
  if (sharedStages[0]) out.n_stage_smem_A = sharedStages[0];
  if (sharedStages[1]) out.n_stage_smem_B = sharedStages[1];
  for (int side = 0; side < 2; ++side) {
    if (!regStages[side]) continue;
    // A register-level buffer whose copy sits directly in the ko body
    // (no ki split) cannot fuse with the shared pipeline.
    if (sharedStages[side] && ks.size() < 2)
      analysis("UnsupportedNesting",
               "inner pipelined loop must be a direct child of the outer pipelined loop body");
    if (sharedStages[side] && static_cast<int64_t>(regStages[side] - 1) >
                                  static_cast<int64_t>(sharedStages[side] - 1) * F)
      analysis("LookaheadExceedsOuter", "inner pipeline looks ahead " + std::to_string(regStages[side] - 1) +
                                            " steps, more than the outer pipeline covers (" +
                                            std::to_string((sharedStages[side] - 1) * F) + ")");
    // register level -> TMEM accumulator ring (at most 2 fit 512 columns)
    out.n_stage_inner = std::max(out.n_stage_inner, std::min(regStages[side], 2));
  }
  return out;
}

}  // namespace sched

// ---------------------------------------------------------------------------
// Bookkeeping enumerator
// ---------------------------------------------------------------------------
namespace {

struct Ring {
  int s;
  uint32_t prodPhase = 0, consPhase = 0;
  int prodSlot = 0, consSlot = 0;
  int loads = 0, waits = 0, releases = 0;
};

struct Emitter {
  alcop_event* out;
  int64_t cap;
  int64_t n = 0;
  void push(const alcop_event& e) {
    if (out && n < cap) out[n] = e;
    ++n;
  }
};

void prod_load(Ring& r, int buf, int tile, int chunk, Emitter& em) {
  alcop_event e{};
  e.kind = 0;
  e.buf = buf;
  e.tile = tile;
  e.slot = r.prodSlot;
  e.chunk = chunk;
  e.parity = static_cast<int32_t>(((r.prodPhase >> r.prodSlot) & 1u) ^ 1u);
  r.prodPhase ^= 1u << r.prodSlot;
  ++r.loads;
  e.acquired = e.committed = r.loads;
  e.waited = e.released = -1;
  em.push(e);
  r.prodSlot = (r.prodSlot + 1 == r.s) ? 0 : r.prodSlot + 1;
}

alcop_event cons_event(Ring& r, int kind, int buf, int tile, int chunk, int slot, int parity) {
  alcop_event e{};
  e.kind = kind;
  e.buf = buf;
  e.tile = tile;
  e.slot = slot;
  e.chunk = chunk;
  e.parity = parity;
  e.acquired = e.committed = -1;
  e.waited = r.waits;
  e.released = r.releases;
  return e;
}

}  // namespace
}  // namespace alcop

using namespace alcop;

extern "C" int alcop_parse_schedule_script(const alcop_gemm_desc* w, const char* script, alcop_schedule* out,
                                           char* warnings, size_t warnings_len) {
  if (!w || !script || !out) return set_error(ALCOP_ERR_CONFIG, "NullArgument", "NULL argument");
  clear_error();
  if (warnings && warnings_len) warnings[0] = '\0';
  try {
    std::vector<std::string> warns;
    sched::State st = sched::apply_script(sched::gemm_schedule(*w), script, &warns);
    *out = sched::to_alcop(st);
    if (warnings && warnings_len) {
      std::string all;
      for (const auto& m : warns) all += m + "\n";
      std::strncpy(warnings, all.c_str(), warnings_len - 1);
      warnings[warnings_len - 1] = '\0';
    }
    return ALCOP_OK;
  } catch (const sched::Error& e) {
    return set_error(e.code, e.rule, e.what());
  } catch (const std::exception& e) {
    return set_error(ALCOP_ERR_CONFIG, "ConfigError", e.what());
  }
}

extern "C" int alcop_enumerate_pipeline(int64_t num_tiles, int64_t E, int32_t sA, int32_t sB, int32_t mode,
                                        int32_t role, alcop_event* out, int64_t cap, int64_t* count) {
  if (num_tiles < 0 || E < 1 || sA < 1 || sB < 1 || sA > 32 || sB > 32 || (role != 0 && role != 1))
    return set_error(ALCOP_ERR_CONFIG, "BadArgument", "invalid enumerator arguments");
  clear_error();
  Ring ra{sA}, rb{sB};
  Emitter em{out, cap};
  const bool wrap = mode == ALCOP_MODE_WRAP;
  const int iE = static_cast<int>(E);
  if (role == 0) {
    if (wrap) {
      for (int tl = 0; tl < num_tiles; ++tl) {
        ra.prodSlot = rb.prodSlot = 0;
        for (int i = 0; i < sA - 1; ++i) prod_load(ra, 0, tl, i % iE, em);
        for (int i = 0; i < sB - 1; ++i) prod_load(rb, 1, tl, i % iE, em);
        for (int v = 0; v < iE; ++v) {
          prod_load(ra, 0, tl, (v + sA - 1) % iE, em);
          prod_load(rb, 1, tl, (v + sB - 1) % iE, em);
        }
      }
    } else {
      const int64_t total = num_tiles * E;
      for (int64_t i = 0; i < sA - 1 && i < total; ++i) prod_load(ra, 0, int(i / E), int(i % E), em);
      for (int64_t i = 0; i < sB - 1 && i < total; ++i) prod_load(rb, 1, int(i / E), int(i % E), em);
      for (int64_t v = 0; v < total; ++v) {
        const int64_t ja = v + sA - 1, jb = v + sB - 1;
        if (ja < total) prod_load(ra, 0, int(ja / E), int(ja % E), em);
        if (jb < total) prod_load(rb, 1, int(jb / E), int(jb % E), em);
      }
    }
  } else {
    auto use = [&](Ring& r, int buf, int tl, int chunk, bool release_only, int slot, int par) {
      if (!release_only) {
        ++r.waits;
        em.push(cons_event(r, 1, buf, tl, chunk, slot, par));
      } else {
        ++r.releases;
        em.push(cons_event(r, 2, buf, tl, chunk, slot, par));
      }
    };
    for (int tl = 0; tl < num_tiles; ++tl) {
      if (wrap) ra.consSlot = rb.consSlot = 0;
      for (int v = 0; v < iE; ++v) {
        const int sa = ra.consSlot, sb = rb.consSlot;
        const int pa = (ra.consPhase >> sa) & 1, pb = (rb.consPhase >> sb) & 1;
        ra.consPhase ^= 1u << sa;
        rb.consPhase ^= 1u << sb;
        use(ra, 0, tl, v, false, sa, pa);
        use(rb, 1, tl, v, false, sb, pb);
        use(ra, 0, tl, v, true, sa, pa);
        use(rb, 1, tl, v, true, sb, pb);
        ra.consSlot = (sa + 1 == sA) ? 0 : sa + 1;
        rb.consSlot = (sb + 1 == sB) ? 0 : sb + 1;
      }
      if (wrap) {
        for (Ring* r : {&ra, &rb}) {
          const int buf = r == &ra ? 0 : 1;
          for (int d = 0; d < r->s - 1; ++d) {
            const int sl = r->consSlot, pa = (r->consPhase >> sl) & 1;
            r->consPhase ^= 1u << sl;
            use(*r, buf, tl, (iE + d) % iE, false, sl, pa);
            use(*r, buf, tl, (iE + d) % iE, true, sl, pa);
            r->consSlot = (sl + 1 == r->s) ? 0 : sl + 1;
          }
        }
      }
    }
  }
  if (count) *count = em.n;
  return ALCOP_OK;
}
