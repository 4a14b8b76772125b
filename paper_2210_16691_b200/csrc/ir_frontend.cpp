// ir_frontend.cpp — the reference's on-disk workflow as a drop-in front end
// (SURVEY §8(f) rank 1): parse a textual IR program in the reference grammar
// (`pipec schedule` output, i.e. lower() with `stages` hints,
// schedule.hpp:357-584), recognise the lowered GEMM / batched-GEMM
// load-and-use nest, and map it onto (alcop_gemm_desc, alcop_schedule) so
// `pipec run` / `verify` inputs run on the sm_100a kernel.
//
// The parser is written from scratch for the grammar:
//   program := (bufdecl | groupdecl)* stmt*
//   bufdecl := "buffer" NAME scope TYPE "[" dims "]" ("stages" INT)? ";"
//   groupdecl := "pipeline" NAME scope "capacity" INT ";"
//   stmt := for | copy | compute | sync | pred | block
// Errors follow the reference classes: ParseError (line/col) -> 2,
// AnalysisError{rule} -> 4, unsupported program shapes -> 6 (ConfigError).
#include <algorithm>
#include <cctype>
#include <cstring>
#include <map>
#include <memory>
#include <string>
#include <vector>

#include "alcop_internal.h"

namespace alcop {
namespace ir {

struct Err {
  int code;
  std::string rule, msg;
};

struct Tok {
  enum K { Ident, Int, Sym, End } k;
  std::string s;
  int64_t v = 0;
  int row = 1;  // 1-based source position, reported in ParseError{line, col}
  int column = 1;
};

class Scanner {
 public:
  explicit Scanner(const std::string& t) : t_(t) {}
  std::vector<Tok> run() {
    std::vector<Tok> out;
    while (true) {
      skip();
      Tok tk;
      tk.row = line_;
      tk.column = col_;
      if (i_ >= t_.size()) {
        tk.k = Tok::End;
        out.push_back(tk);
        return out;
      }
      char c = t_[i_];
      if (std::isalpha(static_cast<unsigned char>(c)) || c == '_') {
        size_t j = i_;
        while (j < t_.size() && (std::isalnum(static_cast<unsigned char>(t_[j])) || t_[j] == '_')) ++j;
        tk.k = Tok::Ident;
        tk.s = t_.substr(i_, j - i_);
        adv(j - i_);
      } else if (std::isdigit(static_cast<unsigned char>(c))) {
        size_t j = i_;
        while (j < t_.size() && std::isdigit(static_cast<unsigned char>(t_[j]))) ++j;
        tk.k = Tok::Int;
        tk.s = t_.substr(i_, j - i_);
        tk.v = std::stoll(tk.s);
        adv(j - i_);
      } else if (t_.compare(i_, 2, "..") == 0 || t_.compare(i_, 2, "<-") == 0) {
        tk.k = Tok::Sym;
        tk.s = t_.substr(i_, 2);
        adv(2);
      } else if (std::strchr("[](){};,=+-*/%", c)) {
        tk.k = Tok::Sym;
        tk.s = std::string(1, c);
        adv(1);
      } else {
        throw Err{ALCOP_ERR_PARSE, "ParseError",
                  std::string("unexpected character '") + c + "' (line " + std::to_string(line_) + ", col " +
                      std::to_string(col_) + ")"};
      }
      out.push_back(tk);
    }
  }

 private:
  void adv(size_t n) {  // moves the cursor, keeping the (line, column) of the next token
    for (const size_t stop = i_ + n; i_ < stop; ++i_) {
      const bool newline = t_[i_] == '\n';
      line_ += newline ? 1 : 0;
      col_ = newline ? 1 : col_ + 1;
    }
  }
  void skip() {
    while (i_ < t_.size()) {
      if (std::isspace(static_cast<unsigned char>(t_[i_]))) {
        adv(1);
      } else if (t_[i_] == '#') {
        while (i_ < t_.size() && t_[i_] != '\n') adv(1);
      } else {
        break;
      }
    }
  }
  const std::string& t_;
  size_t i_ = 0;
  int line_ = 1, col_ = 1;
};

struct Buf {
  std::string name, scope, type;
  std::vector<int64_t> shape;
  int stages = 0;
};

struct Node {
  enum K { For, Copy, Compute, Sync, Pred, Block } k;
  std::string var, kind;  // For: loop var + seq/par/unroll ; Sync: primitive name
  int64_t extent = 0;
  std::string dst, src, tag;  // Copy / Compute
  std::vector<std::string> operands;
  std::vector<std::unique_ptr<Node>> body;
};

class Parser {
 public:
  explicit Parser(std::vector<Tok> t) : t_(std::move(t)) {}
  std::map<std::string, Buf> bufs;
  std::vector<std::string> order;
  std::vector<std::unique_ptr<Node>> body;

  void program() {
    while (is("buffer") || (is("pipeline") && peek(2).k == Tok::Ident && (peek(2).s == "shared" || peek(2).s == "register"))) {
      if (is("buffer"))
        bufdecl();
      else
        groupdecl();
    }
    while (t_[p_].k != Tok::End) body.push_back(stmt());
  }

 private:
  const Tok& cur() const { return t_[p_]; }
  const Tok& peek(int k) const { return t_[std::min(p_ + k, t_.size() - 1)]; }
  bool is(const char* s) const { return cur().k != Tok::End && cur().s == s; }
  [[noreturn]] void fail(const std::string& m) const {
    throw Err{ALCOP_ERR_PARSE, "ParseError",
              m + " (line " + std::to_string(cur().row) + ", col " + std::to_string(cur().column) + ")"};
  }
  std::string ident() {
    if (cur().k != Tok::Ident) fail("expected identifier, got '" + cur().s + "'");
    return t_[p_++].s;
  }
  int64_t integer() {
    bool neg = false;
    if (is("-")) {
      neg = true;
      ++p_;
    }
    if (cur().k != Tok::Int) fail("expected integer");
    int64_t v = t_[p_++].v;
    return neg ? -v : v;
  }
  void expect(const char* s) {
    if (!is(s)) fail(std::string("expected '") + s + "', got '" + cur().s + "'");
    ++p_;
  }
  void bufdecl() {
    expect("buffer");
    Buf b;
    b.name = ident();
    b.scope = ident();
    if (b.scope != "global" && b.scope != "shared" && b.scope != "register") fail("bad scope '" + b.scope + "'");
    b.type = ident();
    expect("[");
    b.shape.push_back(integer());
    while (is(",")) {
      ++p_;
      b.shape.push_back(integer());
    }
    expect("]");
    if (is("stages")) {
      ++p_;
      b.stages = static_cast<int>(integer());
    }
    expect(";");
    if (bufs.count(b.name)) fail("duplicate buffer '" + b.name + "'");
    order.push_back(b.name);
    bufs[b.name] = b;
  }
  void groupdecl() {
    expect("pipeline");
    ident();
    ident();
    expect("capacity");
    integer();
    expect(";");
  }
  // expressions are validated and skipped: the recogniser needs the nest
  void expr() {
    term();
    while (is("+") || is("-")) {
      ++p_;
      term();
    }
  }
  void term() {
    factor();
    while (is("*") || is("/") || is("%")) {
      ++p_;
      factor();
    }
  }
  void factor() {
    if (is("(")) {
      ++p_;
      expr();
      expect(")");
    } else if (is("-")) {
      ++p_;
      factor();
    } else if (is("min")) {
      ++p_;
      expect("(");
      expr();
      expect(",");
      expr();
      expect(")");
    } else if (cur().k == Tok::Int || cur().k == Tok::Ident) {
      ++p_;
    } else {
      fail("bad expression token '" + cur().s + "'");
    }
  }
  void indices() {
    expect("[");
    expr();
    while (is(",")) {
      ++p_;
      expr();
    }
    expect("]");
  }
  std::unique_ptr<Node> stmt() {
    auto n = std::make_unique<Node>();
    if (is("for")) {
      ++p_;
      n->k = Node::For;
      n->var = ident();
      n->kind = ident();
      if (n->kind != "seq" && n->kind != "par" && n->kind != "unroll") fail("bad loop kind '" + n->kind + "'");
      const int64_t lo = integer();
      expect("..");
      const int64_t hi = integer();
      if (lo != 0) fail("loops start at 0");
      if (hi <= lo) fail("zero-extent loop");
      n->extent = hi - lo;
      block_into(n->body);
    } else if (is("copy_async")) {
      ++p_;
      n->k = Node::Copy;
      n->dst = ident();
      indices();
      expect("<-");
      n->src = ident();
      indices();
      expect(";");
    } else if (is("producer_acquire") || is("producer_commit") || is("consumer_wait") || is("consumer_release")) {
      n->k = Node::Sync;
      n->kind = ident();
      n->var = ident();
      expect(";");
    } else if (is("if")) {
      ++p_;
      n->k = Node::Pred;
      expr();
      block_into(n->body);
    } else if (is("{")) {
      n->k = Node::Block;
      block_into(n->body);
    } else {
      n->k = Node::Compute;
      n->dst = ident();
      indices();
      expect("=");
      n->tag = ident();
      expect("(");
      if (!is(")")) {
        n->operands.push_back(ident());
        indices();
        while (is(",")) {
          ++p_;
          n->operands.push_back(ident());
          indices();
        }
      }
      expect(")");
      expect("flops");
      integer();
      expect(";");
    }
    return n;
  }
  void block_into(std::vector<std::unique_ptr<Node>>& out) {
    expect("{");
    while (!is("}")) {
      if (cur().k == Tok::End) fail("unterminated block");
      out.push_back(stmt());
    }
    ++p_;
  }
  std::vector<Tok> t_;
  size_t p_ = 0;
};

struct Found {
  std::map<std::string, int64_t> loops;  // var -> extent
  std::map<std::string, std::string> kinds;
  std::vector<std::string> tags;
  bool sync = false;
};

void walk(const std::vector<std::unique_ptr<Node>>& b, Found& f) {
  for (const auto& n : b) {
    if (n->k == Node::For) {
      f.loops[n->var] = n->extent;
      f.kinds[n->var] = n->kind;
    }
    if (n->k == Node::Sync) f.sync = true;
    if (n->k == Node::Compute) f.tags.push_back(n->tag);
    walk(n->body, f);
  }
}

void recognise(Parser& P, alcop_gemm_desc& d, alcop_schedule& s, std::string& info) {
  auto need = [&](const char* n) -> const Buf& {
    auto it = P.bufs.find(n);
    if (it == P.bufs.end())
      throw Err{ALCOP_ERR_CONFIG, "Unsupported", std::string("not a lowered GEMM nest: no buffer '") + n + "'"};
    return it->second;
  };
  const Buf& A = need("A");
  const Buf& B = need("B");
  const Buf& C = need("C");
  const Buf& Creg = need("C_reg");
  if (A.shape.size() != C.shape.size() || A.shape.size() < 2 || A.shape.size() > 3)
    throw Err{ALCOP_ERR_CONFIG, "Unsupported", "A/C must be [M,K]/[M,N] or batched [b,M,K]/[b,M,N]"};
  const bool batched = A.shape.size() == 3;
  d = alcop_gemm_desc{};
  d.batch = batched ? A.shape[0] : 1;
  d.M = A.shape[batched ? 1 : 0];
  d.K = A.shape[batched ? 2 : 1];
  d.N = B.shape[batched ? 2 : 1];
  if (B.shape[batched ? 1 : 0] != d.K || C.shape[batched ? 2 : 1] != d.N)
    throw Err{ALCOP_ERR_CONFIG, "Unsupported", "A, B, C shapes do not form a GEMM"};
  if (A.type != "f16") throw Err{ALCOP_ERR_CONFIG, "Unsupported", "element type '" + A.type + "' (need f16)"};
  d.in_dtype = ALCOP_F16;
  d.out_dtype = ALCOP_F32;  // the interpreter's C holds the exact (int64) sums
  d.b_layout = ALCOP_B_KN;  // schedule.hpp:389
  Found f;
  walk(P.body, f);
  if (f.sync)
    throw Err{ALCOP_ERR_ANALYSIS, "AlreadySynchronized",
              "program already contains pipeline synchronization (pass the hinted, untransformed nest)"};
  // elementwise pre-op: inlined into the consumer (mma_ewa) or materialised
  // as S2 = ew(A) (schedule.hpp:393-407); both run as the fused pre-op
  bool pre = false;
  for (const auto& t : f.tags) pre |= (t == "mma_ewa" || t == "ew");
  d.pre_op = pre ? 1 : 0;
  s = alcop_schedule{};
  alcop_schedule_default(&s);
  s.tileM = Creg.shape[0];
  s.tileN = Creg.shape[1];
  auto stages_of = [&](const char* n) {
    auto it = P.bufs.find(n);
    return it == P.bufs.end() ? 0 : it->second.stages;
  };
  const char* aSh = P.bufs.count("S2_shared") ? "S2_shared" : "A_shared";
  const char* aReg = P.bufs.count("S2_reg") ? "S2_reg" : "A_reg";
  auto it = P.bufs.find(aSh);
  if (it != P.bufs.end())
    s.tileK = it->second.shape[1];
  else if (f.loops.count("ko"))
    s.tileK = d.K / f.loops["ko"];
  else
    s.tileK = d.K;
  const int sA = stages_of(aSh), sB = stages_of("B_shared");
  const int tA = stages_of(aReg), tB = stages_of("B_reg");
  s.n_stage_smem_A = sA ? sA : 1;
  s.n_stage_smem_B = sB ? sB : 1;
  s.n_stage_inner = std::min(std::max({tA, tB, 1}), 2);
  s.mode = ALCOP_MODE_WRAP;
  // the pass's lookahead rule for the nested level (pipeline_pass.hpp:305-313)
  const int64_t F = f.loops.count("ki") ? f.loops["ki"] : 1;
  for (auto [ss, tt] : {std::pair<int, int>{sA, tA}, {sB, tB}})
    if (ss >= 2 && tt >= 2 && static_cast<int64_t>(tt - 1) > static_cast<int64_t>(ss - 1) * F)
      throw Err{ALCOP_ERR_ANALYSIS, "LookaheadExceedsOuter",
                "inner pipeline looks ahead " + std::to_string(tt - 1) + " steps, more than the outer pipeline covers"};
  info = std::string(d.pre_op ? "pre-op (2A+1) " : "") + "GEMM M=" + std::to_string(d.M) + " N=" + std::to_string(d.N) + " K=" + std::to_string(d.K) +
         " batch=" + std::to_string(d.batch) + " tile " + std::to_string(s.tileM) + "x" + std::to_string(s.tileN) +
         "x" + std::to_string(s.tileK) + " stages A/B " + std::to_string(s.n_stage_smem_A) + "/" +
         std::to_string(s.n_stage_smem_B) + " inner " + std::to_string(s.n_stage_inner);
}

}  // namespace ir
}  // namespace alcop

using namespace alcop;

extern "C" int alcop_ir_to_gemm(const char* ir_text, alcop_gemm_desc* desc, alcop_schedule* sched, char* info,
                                size_t info_len) {
  if (!ir_text || !desc || !sched) return set_error(ALCOP_ERR_CONFIG, "NullArgument", "NULL argument");
  clear_error();
  try {
    std::string text(ir_text);
    ir::Scanner lx(text);
    ir::Parser P(lx.run());
    P.program();
    std::string msg;
    ir::recognise(P, *desc, *sched, msg);
    if (info && info_len) {
      std::strncpy(info, msg.c_str(), info_len - 1);
      info[info_len - 1] = '\0';
    }
    return ALCOP_OK;
  } catch (const ir::Err& e) {
    return set_error(e.code, e.rule, e.msg);
  } catch (const std::exception& e) {
    return set_error(ALCOP_ERR_PARSE, "ParseError", e.what());
  }
}
