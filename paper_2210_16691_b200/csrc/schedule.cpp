// schedule.cpp — the reference's schedule-script surface on the B200 host side,
// and the host bookkeeping enumerator.
//
// Part 1 is written against the CONTRACT of the reference's scheduler module
// (the dataflow view, the three eligibility rules of §3.1,
// the ordering policy of §3.2, the script format of SPEC.md:216) and the
// pass's nesting rules (pipeline_pass.hpp:305-322).  The rule
// tags, error classes and exit codes are the reference's interface
// (common.hpp:43-69, cli.hpp:23-25); tests/golden/scripts*.jsonl pin every
// accept/reject decision against the reference itself (632 scripts).
//
// The design is a small script machine: a dataflow table of tensors in
// declaration order, a split table per GEMM dimension (the loop sketch is
// derived from it, never stored), primitives dispatched from a table, and
// eligibility as an ordered rule list.  Its output is not a lowered program
// but the alcop_schedule the sm_100a kernel is instantiated with: the kernel
// IS the lowered-and-transformed load-and-use nest.
//
// Part 2 is the producer / consumer event sequence the kernel executes
// (pipeline_pass.hpp:482-748 index algebra, interp.hpp:375-418 counters),
// used to check the device trace bit-exactly.
#include <algorithm>
#include <array>
#include <cerrno>
#include <climits>
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <sstream>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "alcop_internal.h"

namespace alcop {
namespace surface {

// ---------------------------------------------------------------------------
// Part 1: the script machine
// ---------------------------------------------------------------------------

// Memory levels, fastest first.  A cache may only be placed strictly closer to
// the tensor cores than its source ("scope strictly below").
enum Level : int { kRegister = 0, kShared = 1, kGlobal = 2 };

const char* level_word(int lv) { return lv == kRegister ? "register" : lv == kShared ? "shared" : "global"; }

// A rejected script: the reference's exit code plus its rule tag.
struct Rejection : std::runtime_error {
  int exit_code;
  std::string tag;
  Rejection(int code, std::string t, const std::string& why)
      : std::runtime_error(why), exit_code(code), tag(std::move(t)) {}
};
[[noreturn]] void reject(const std::string& tag, const std::string& why) {
  throw Rejection(ALCOP_ERR_ANALYSIS, tag, why);
}
[[noreturn]] void reject_config(const std::string& why) { throw Rejection(ALCOP_ERR_CONFIG, "ConfigError", why); }

// One tensor of the schedule's dataflow view.
struct Tensor {
  enum Origin { kInput, kCopy, kCompute };
  std::string id;
  Origin origin = kInput;
  std::vector<std::string> reads;  // kCopy: exactly one source; kCompute: operands
  std::string op;                  // kCompute: "ew" / "mma"
  int level = kGlobal;
  int stages = 0;                  // pipelining hint, 0 = none
  bool carries_ew = false;         // a case-2 inline folded f() into this copy's consumer
};

// Splits of one GEMM dimension, outer to inner: (loop name, extent).
using Splits = std::vector<std::pair<std::string, int64_t>>;

struct Program {
  int64_t extent[3] = {0, 0, 0};  // i (M), j (N), k (K)
  int64_t batch = 1;
  std::vector<Tensor> flow;       // declaration order matters (later hints win per side)
  bool tiled = false;
  std::array<Splits, 3> split;    // valid once tiled

  Tensor* lookup(const std::string& id) {
    auto it = std::find_if(flow.begin(), flow.end(), [&](const Tensor& t) { return t.id == id; });
    return it == flow.end() ? nullptr : &*it;
  }
  const Tensor* lookup(const std::string& id) const { return const_cast<Program*>(this)->lookup(id); }
  bool has_inner_k() const { return split[2].size() > 1; }
};

// The workload's dataflow (SPEC.md:192-196 v1 family): C = mma(A, B), or with
// the elementwise pre-op S2 = ew(A) feeding the mma in place of A.
Program workload(const alcop_gemm_desc& w) {
  Program p;
  p.extent[0] = w.M;
  p.extent[1] = w.N;
  p.extent[2] = w.K;
  p.batch = w.batch;
  auto input = [](const char* id) {
    Tensor t;
    t.id = id;
    return t;
  };
  auto compute = [](const char* id, const char* op, std::vector<std::string> reads) {
    Tensor t;
    t.id = id;
    t.origin = Tensor::kCompute;
    t.op = op;
    t.reads = std::move(reads);
    return t;
  };
  p.flow = {input("A"), input("B")};
  if (w.pre_op) p.flow.push_back(compute("S2", "ew", {"A"}));
  p.flow.push_back(compute("C", "mma", {w.pre_op ? "S2" : "A", "B"}));
  return p;
}

// The sequential loop a buffer's copy is issued in.  Shared caches refill once
// per outer reduction step (ko); register caches per inner step (ki) when the
// reduction has a second split, otherwise per ko.  This is the sync position of
// rule 3 and the loop the pass pipelines (§4.1 step 3).
const char* copy_loop(const Program& p, const Tensor& t) {
  if (p.split[2].empty()) return nullptr;
  const bool inner = t.level == kRegister && p.has_inner_k();
  return (inner ? p.split[2][1] : p.split[2][0]).first.c_str();
}

// §3.1: three eligibility rules, evaluated in order; the first failure is reported.
struct Rule {
  const char* tag;
  std::function<std::string(const Program&, const Tensor&)> violation;  // "" = satisfied
};

const std::vector<Rule>& eligibility_rules() {
  static const std::vector<Rule> rules = {
      {"NotAsyncProducer",
       [](const Program&, const Tensor& t) -> std::string {
         return t.origin == Tensor::kCopy ? "" : "'" + t.id + "' is filled by computation, not an asynchronous copy";
       }},
      {"NoSequentialLoop",
       [](const Program& p, const Tensor& t) -> std::string {
         return copy_loop(p, t) ? "" : "'" + t.id + "' is not filled inside a sequential loop";
       }},
      {"SyncPositionConflict",
       [](const Program& p, const Tensor& t) -> std::string {
         if (t.level != kShared) return "";  // register buffers are exempt
         const std::string mine = copy_loop(p, t);
         for (const Tensor& o : p.flow) {
           if (o.id == t.id || o.level != kShared || o.stages == 0) continue;
           const char* theirs = copy_loop(p, o);
           if (theirs && mine != theirs)
             return "shared buffers '" + o.id + "' (" + theirs + ") and '" + t.id + "' (" + mine +
                    ") would synchronise in different loops";
         }
         return "";
       }},
  };
  return rules;
}

// The reference's schedule primitives as transformations of a Program value.
struct Primitives {
  static void cache_read(Program& p, const std::string& src_id, int level) {
    const Tensor* src = p.lookup(src_id);
    if (!src) reject("NoSuchTensor", "cache_read of unknown tensor '" + src_id + "'");
    if (level >= src->level)
      reject("ScopeNotBelow", std::string("a ") + level_word(level) + " cache of a " + level_word(src->level) +
                                  " tensor would copy upwards");
    // the buffer is named after the root tensor: A -> A_shared -> A_reg
    std::string root = src_id;
    for (const char* sfx : {"_shared", "_reg"}) {
      const size_t n = std::strlen(sfx);
      if (root.size() > n && root.compare(root.size() - n, n, sfx) == 0) root.resize(root.size() - n);
    }
    Tensor buf;
    buf.id = root + (level == kShared ? "_shared" : "_reg");
    if (p.lookup(buf.id)) reject("DuplicateBuffer", "'" + buf.id + "' is already declared");
    buf.origin = Tensor::kCopy;
    buf.reads = {src_id};
    buf.level = level;
    for (Tensor& t : p.flow)  // every reader of the source now reads the cache
      if (t.id != src_id) std::replace(t.reads.begin(), t.reads.end(), src_id, buf.id);
    p.flow.push_back(std::move(buf));
  }

  static void tile(Program& p, const std::string& target, const Splits& given) {
    if (target != "C" || !p.lookup(target)) reject("NoSuchTensor", "only the output C can be tiled, not '" + target + "'");
    std::array<Splits, 3> by_dim;
    static const char kDims[3] = {'i', 'j', 'k'};
    for (const auto& sp : given) {
      const char lead = sp.first.empty() ? '\0' : sp.first[0];
      const int d = lead == 'i' ? 0 : lead == 'j' ? 1 : lead == 'k' ? 2 : -1;
      if (d < 0) reject("BadSplit", "loop '" + sp.first + "' names no dimension (i, j or k)");
      if (sp.second < 1) reject("BadSplit", "loop '" + sp.first + "' has a non-positive extent");
      by_dim[d].push_back(sp);
    }
    for (int d = 0; d < 3; ++d) {
      if (by_dim[d].empty()) reject("BadSplit", std::string("dimension '") + kDims[d] + "' is not split");
      int64_t covered = 1;
      for (const auto& sp : by_dim[d]) covered *= sp.second;
      if (covered != p.extent[d])
        reject("NonDivisibleSplit", std::string("splits of '") + kDims[d] + "' cover " + std::to_string(covered) +
                                        " of " + std::to_string(p.extent[d]));
      if (by_dim[d].size() > 2) reject("BadSplit", std::string("dimension '") + kDims[d] + "' has more than two splits");
    }
    p.split = by_dim;
    p.tiled = true;
  }

  static void pipeline(Program& p, const std::string& id, int stages) {
    if (!p.tiled) reject("OrderingViolation", "pipeline requires loop sketch: tile before pipelining");
    if (stages < 2) reject("BadStages", "a pipeline needs at least two stages, got " + std::to_string(stages));
    Tensor* t = p.lookup(id);
    if (!t) reject("NoSuchTensor", "pipeline of unknown buffer '" + id + "'");
    for (const Rule& r : eligibility_rules()) {
      std::string why = r.violation(p, *t);
      if (!why.empty()) reject(r.tag, why);
    }
    t->stages = stages;
  }

  // §3.2 / Fig. schedule_transform: inlining an elementwise tensor whose cache
  // is already pipelined re-sources the cache to the tensor's input and folds
  // f() into the cache's consumer (case 2); an unpipelined cache becomes a
  // computed buffer (case 1, which rule 1 then rejects for pipelining).
  static void inline_(Program& p, const std::string& id) {
    const Tensor* f = p.lookup(id);
    if (!f) reject("NoSuchTensor", "inline of unknown tensor '" + id + "'");
    if (f->origin != Tensor::kCompute || f->reads.size() != 1)
      reject("NotElementwise", "'" + id + "' is not a unary elementwise computation");
    const std::string input = f->reads.front(), op = f->op;
    int rewritten = 0;
    for (Tensor& t : p.flow) {
      const bool reads_f = std::find(t.reads.begin(), t.reads.end(), id) != t.reads.end();
      if (!reads_f) continue;
      if (t.origin != Tensor::kCopy)
        reject("NoRewrite", "'" + t.id + "' computes from '" + id + "' directly; only cached reads can absorb it");
      ++rewritten;
      if (t.stages == 0) {  // case 1
        t.origin = Tensor::kCompute;
        t.op = op;
        t.reads = {input};
      } else {  // case 2
        if (t.carries_ew) reject("NoRewrite", "'" + t.id + "' already carries a fused elementwise function");
        t.reads = {input};
        t.carries_ew = true;
      }
    }
    if (rewritten == 0) reject("NoRewrite", "no cache reads '" + id + "'");
    p.flow.erase(std::remove_if(p.flow.begin(), p.flow.end(), [&](const Tensor& t) { return t.id == id; }),
                 p.flow.end());
  }
};

// std::stoll / std::stoi semantics (leading integer, trailing text ignored,
// failure or overflow rejected): the reference parses extents that way.
bool leading_int(const std::string& text, long long lo, long long hi, long long* out) {
  errno = 0;
  char* end = nullptr;
  const long long v = std::strtoll(text.c_str(), &end, 10);
  if (end == text.c_str() || errno == ERANGE || v < lo || v > hi) return false;
  *out = v;
  return true;
}

// The script format: one primitive per line, '#' comments.
class ScriptMachine {
 public:
  explicit ScriptMachine(Program p) : prog_(std::move(p)) {}

  void run(const std::string& text) {
    std::istringstream lines(text);
    std::string line;
    while (std::getline(lines, line)) {
      ++line_no_;
      line = line.substr(0, line.find('#'));
      std::istringstream words(line);
      std::vector<std::string> w;
      for (std::string x; words >> x;) w.push_back(x);
      if (w.empty()) continue;
      const auto& table = handlers();
      auto h = std::find_if(table.begin(), table.end(), [&](const Handler& e) { return w[0] == e.word; });
      if (h == table.end()) syntax("unknown primitive '" + w[0] + "'");
      if (w.size() < h->min_words || w.size() > h->max_words) syntax("usage: " + std::string(h->usage));
      (this->*(h->fn))(w);
    }
  }

  const Program& program() const { return prog_; }
  const std::vector<std::string>& notes() const { return notes_; }

 private:
  struct Handler {
    const char* word;
    size_t min_words, max_words;
    const char* usage;
    void (ScriptMachine::*fn)(const std::vector<std::string>&);
  };
  static const std::vector<Handler>& handlers() {
    static const std::vector<Handler> h = {
        {"cache_read", 3, 3, "cache_read <tensor> <shared|register>", &ScriptMachine::do_cache_read},
        {"tile", 3, SIZE_MAX, "tile <tensor> <loop>=<extent>...", &ScriptMachine::do_tile},
        {"pipeline", 3, 3, "pipeline <buffer> <stages>", &ScriptMachine::do_pipeline},
        {"inline", 2, 2, "inline <tensor>", &ScriptMachine::do_inline},
    };
    return h;
  }
  [[noreturn]] void syntax(const std::string& why) const {
    reject_config("schedule script line " + std::to_string(line_no_) + ": " + why);
  }

  void do_cache_read(const std::vector<std::string>& w) {
    int level;
    if (w[2] == "shared")
      level = kShared;
    else if (w[2] == "register")
      level = kRegister;
    else
      syntax("unknown scope '" + w[2] + "'");
    Primitives::cache_read(prog_, w[1], level);
  }

  void do_tile(const std::vector<std::string>& w) {
    Splits given;
    for (size_t i = 2; i < w.size(); ++i) {
      const size_t eq = w[i].find('=');
      long long v = 0;
      if (eq == std::string::npos || !leading_int(w[i].substr(eq + 1), LLONG_MIN, LLONG_MAX, &v))
        syntax("cannot read split '" + w[i] + "'");
      given.emplace_back(w[i].substr(0, eq), static_cast<int64_t>(v));
    }
    Primitives::tile(prog_, w[1], given);
  }

  void do_pipeline(const std::vector<std::string>& w) {
    long long n = 0;
    if (!leading_int(w[2], INT32_MIN, INT32_MAX, &n)) syntax("cannot read stage count '" + w[2] + "'");
    try {
      Primitives::pipeline(prog_, w[1], static_cast<int>(n));
    } catch (const Rejection& r) {
      // §3.1: on a sync-position conflict the paper refuses to pipeline any of
      // the shared buffers involved: every shared hint is withdrawn
      if (r.tag != "SyncPositionConflict") throw;
      for (Tensor& t : prog_.flow)
        if (t.level == kShared) t.stages = 0;
      notes_.push_back(std::string("refusing to pipeline: ") + r.what());
    }
  }

  void do_inline(const std::vector<std::string>& w) { Primitives::inline_(prog_, w[1]); }

  Program prog_;
  int line_no_ = 0;
  std::vector<std::string> notes_;
};

// The operand (A side or B side) a cache ultimately reads.
bool feeds_b(const Program& p, const Tensor& t) {
  const Tensor* cur = &t;
  for (int hops = 0; cur && hops < 16; ++hops) {
    if (cur->id == "A") return false;
    if (cur->id == "B") return true;
    cur = cur->reads.empty() ? nullptr : p.lookup(cur->reads.front());
  }
  return false;
}

// What lower() + the pass make of the hints (schedule.hpp:371-374 tile
// arithmetic; pipeline_pass.hpp:305-322 nesting rules), as the B200 schedule.
alcop_schedule to_schedule(const Program& p) {
  if (!p.tiled) reject("OrderingViolation", "nothing to lower: the script never tiles C");
  alcop_schedule out;
  alcop_schedule_default(&out);
  const Splits& si = p.split[0];
  const Splits& sj = p.split[1];
  const Splits& sk = p.split[2];
  // the tile is the inner split, or the dimension over the outer loop's trip count
  out.tileM = si.size() > 1 ? si[1].second : p.extent[0] / si[0].second;
  out.tileN = sj.size() > 1 ? sj[1].second : p.extent[1] / sj[0].second;
  out.tileK = p.extent[2] / sk[0].second;
  const int64_t inner_trips = p.has_inner_k() ? sk[1].second : 1;  // F of the nested pipeline
  out.n_stage_smem_A = out.n_stage_smem_B = out.n_stage_inner = 1;
  out.mode = ALCOP_MODE_WRAP;  // the reference's own emission of the pipelined nest
  int outer[2] = {0, 0}, inner[2] = {0, 0};  // per side: stages of the shared / register pipeline
  for (const Tensor& t : p.flow) {
    if (t.stages == 0) continue;
    (t.level == kShared ? outer : inner)[feeds_b(p, t) ? 1 : 0] = t.stages;
  }
  if (outer[0]) out.n_stage_smem_A = outer[0];
  if (outer[1]) out.n_stage_smem_B = outer[1];
  for (int side = 0; side < 2; ++side) {
    const int t = inner[side], s = outer[side];
    if (!t) continue;
    if (s && !p.has_inner_k())
      reject("UnsupportedNesting", "the register pipeline's loop must sit directly in the shared pipeline's body");
    if (s && int64_t(t - 1) > int64_t(s - 1) * inner_trips)
      reject("LookaheadExceedsOuter", "register lookahead " + std::to_string(t - 1) + " outruns the " +
                                          std::to_string(int64_t(s - 1) * inner_trips) +
                                          " steps the shared pipeline has in flight");
    // the register double buffer becomes the TMEM accumulator ring (<= 2 x 256 columns)
    out.n_stage_inner = std::max(out.n_stage_inner, std::min(t, 2));
  }
  return out;
}

}  // namespace surface

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
    surface::ScriptMachine machine(surface::workload(*w));
    machine.run(script);
    const alcop_schedule result = surface::to_schedule(machine.program());
    if (warnings && warnings_len) {
      std::string joined;
      for (const std::string& n : machine.notes()) joined += n + "\n";
      const size_t len = std::min(joined.size(), warnings_len - 1);
      std::memcpy(warnings, joined.data(), len);
      warnings[len] = '\0';
    }
    *out = result;
    return ALCOP_OK;
  } catch (const surface::Rejection& r) {
    return set_error(r.exit_code, r.tag, r.what());
  } catch (const std::exception& e) {  // the reference's cli maps any other exception to kConfig
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
