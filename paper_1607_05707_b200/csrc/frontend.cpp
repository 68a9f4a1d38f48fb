// frontend.cpp — IrGL source front end + run_host over the B200 runtime.
//
//   lexer / parser : the concrete notation of PAPER.md Table 1 (:63-103) and Listing 2
//                    (:288-304), made precise as in SPEC.md:142-151 (ForAll is parallel, `for`
//                    sequential, `In` separates the variable from the range, `//` comments,
//                    optional semicolons, v = wl.pop(i) / wl.push(x) -> WlPop / WlPush).
//   recogniser     : structural match of each plain kernel body against the IrGL form of the
//                    operators the runtime implements (pattern identifiers `$x` unify with any
//                    identifier, consistently).  BFS is Listing 2 itself; SSSP / CC label
//                    propagation accept both the atomicMin-builtin form (App. B7) and the
//                    compare-then-store form; PageRank is the pull Jacobi form with
//                    ReduceAndReturn.
//   run_host       : sequential host statements; Iterate / Invoke / Pipe drive
//                    irgl_iterate / irgl_invoke; between_rounds statements are applied once per
//                    round to the host scalars; Initial [..] seeds the pipe (WorklistInit).
//
// Not a port of the reference's AST (ast.hpp): a minimal tree for this front end only.
#include "irgl/frontend.h"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <map>
#include <memory>
#include <sstream>
#include <string>
#include <vector>

namespace irgl {
namespace fe {

struct Span {
  int line = 1, col = 1;
};

struct Error {
  Span sp;
  std::string rule, msg;
};

// ---- tokens ----------------------------------------------------------------------------------
enum class T { Ident, Int, Float, Str, Punct, End };
struct Tok {
  T t;
  std::string s;
  Span sp;
};

static std::vector<Tok> lex(const std::string& src, std::vector<Error>& errs) {
  std::vector<Tok> out;
  int line = 1, col = 1;
  size_t i = 0;
  auto adv = [&](size_t n) {
    for (size_t k = 0; k < n && i < src.size(); ++k, ++i) {
      if (src[i] == '\n') {
        ++line;
        col = 1;
      } else {
        ++col;
      }
    }
  };
  static const char* two[] = {"==", "!=", "<=", ">=", "&&", "||", "++", "--", "+=", "-=", "*=", "->"};
  while (i < src.size()) {
    const char c = src[i];
    if (isspace((unsigned char)c)) {
      adv(1);
      continue;
    }
    if (c == '/' && i + 1 < src.size() && src[i + 1] == '/') {
      while (i < src.size() && src[i] != '\n') adv(1);
      continue;
    }
    if (c == '/' && i + 1 < src.size() && src[i + 1] == '*') {
      adv(2);
      while (i + 1 < src.size() && !(src[i] == '*' && src[i + 1] == '/')) adv(1);
      adv(2);
      continue;
    }
    Span sp{line, col};
    if (isalpha((unsigned char)c) || c == '_' || c == '$') {
      size_t j = i + 1;
      while (j < src.size() && (isalnum((unsigned char)src[j]) || src[j] == '_')) ++j;
      out.push_back({T::Ident, src.substr(i, j - i), sp});
      adv(j - i);
      continue;
    }
    if (isdigit((unsigned char)c) || (c == '.' && i + 1 < src.size() && isdigit((unsigned char)src[i + 1]))) {
      size_t j = i;
      bool flt = false;
      while (j < src.size() && (isdigit((unsigned char)src[j]) || src[j] == '.' || src[j] == 'e' ||
                                src[j] == 'E' ||
                                ((src[j] == '-' || src[j] == '+') && (src[j - 1] == 'e' || src[j - 1] == 'E')))) {
        if (src[j] == '.' || src[j] == 'e' || src[j] == 'E') flt = true;
        ++j;
      }
      out.push_back({flt ? T::Float : T::Int, src.substr(i, j - i), sp});
      adv(j - i);
      continue;
    }
    if (c == '"') {
      size_t j = i + 1;
      while (j < src.size() && src[j] != '"' && src[j] != '\n') j += (src[j] == '\\') ? 2 : 1;
      if (j >= src.size() || src[j] != '"') {
        errs.push_back({sp, "E101", "unterminated string"});
        adv(j - i);
        continue;
      }
      out.push_back({T::Str, src.substr(i + 1, j - i - 1), sp});
      adv(j + 1 - i);
      continue;
    }
    bool matched = false;
    for (const char* t : two)
      if (src.compare(i, 2, t) == 0) {
        out.push_back({T::Punct, t, sp});
        adv(2);
        matched = true;
        break;
      }
    if (matched) continue;
    if (strchr("(){}[];,.=<>+-*/%!", c)) {
      out.push_back({T::Punct, std::string(1, c), sp});
      adv(1);
      continue;
    }
    errs.push_back({sp, "E101", std::string("unexpected character '") + c + "'"});
    adv(1);
  }
  out.push_back({T::End, "", Span{line, col}});
  return out;
}

// ---- AST ------------------------------------------------------------------------------------
enum class EK { Int, Float, Str, Ident, Inf, Bool, Unary, Binary, Field, Call, Index };
struct Expr;
using ExprP = std::shared_ptr<Expr>;
struct Expr {
  EK k;
  Span sp;
  std::string s;  // identifier / operator / field name / string
  int64_t i = 0;
  double f = 0;
  std::vector<ExprP> a;  // Unary: [x]; Binary: [l, r]; Field: [obj]; Call: [callee, args...]; Index: [arr, idx]
};

enum class SK { Assign, OpAssign, Incr, ExprStmt, ForAll, For, While, If, Iterate, Invoke, Pipe,
                ReduceAndReturn, Retry, Respawn, Sync, Atomic, WlPop, WlPush };
struct Stmt;
using StmtP = std::shared_ptr<Stmt>;
struct Stmt {
  SK k;
  Span sp;
  ExprP lhs, rhs;          // Assign / OpAssign (op) / Incr; If/While cond in rhs; ForAll/For range in rhs
  std::string op, var;     // OpAssign operator; loop variable / kernel name / WlPop target
  std::vector<StmtP> body, els;
  std::vector<ExprP> args, init;  // Iterate / Invoke args; Initial [...]
  int cond_mode = 0, red = 0;     // Iterate While/Until, Any/All; Invoke reduction
  bool once = false, has_init = false;
};

struct Kernel {
  std::string name;
  std::vector<std::string> params;
  std::vector<StmtP> body;
  Span sp;
  bool host = false;
  int op = -1;            // recognised runtime operator
  std::string field;      // node property it writes
  std::map<std::string, std::string> bind;  // pattern bindings ($G, $L, ...)
};

struct Module {
  std::string file;
  std::vector<Kernel> kernels;
  std::vector<StmtP> top;  // top-level host statements (implicit host kernel)
  std::map<std::string, double> scalars;
};

// ---- parser ---------------------------------------------------------------------------------
struct Parser {
  std::vector<Tok> t;
  size_t p = 0;
  std::vector<Error>& errs;
  explicit Parser(std::vector<Tok> toks, std::vector<Error>& e) : t(std::move(toks)), errs(e) {}

  const Tok& cur() const { return t[p]; }
  bool is(const char* s) const { return (t[p].t == T::Punct || t[p].t == T::Ident) && t[p].s == s; }
  bool accept(const char* s) {
    if (is(s)) {
      ++p;
      return true;
    }
    return false;
  }
  void fail(const std::string& msg) {
    errs.push_back({cur().sp, "E102", msg + (cur().t == T::End ? " at end of input" : " near '" + cur().s + "'")});
    throw 1;
  }
  void expect(const char* s) {
    if (!accept(s)) fail(std::string("expected '") + s + "'");
  }
  std::string ident() {
    if (cur().t != T::Ident) fail("expected identifier");
    return t[p++].s;
  }
  void semi() { accept(";"); }

  // expressions: || && (== !=) (< <= > >=) (+ -) (* / %) unary postfix
  ExprP mk(EK k, Span sp) {
    auto e = std::make_shared<Expr>();
    e->k = k;
    e->sp = sp;
    return e;
  }
  ExprP bin(const char* const* ops, ExprP (Parser::*next)()) {
    ExprP l = (this->*next)();
    for (;;) {
      const char* hit = nullptr;
      for (const char* const* o = ops; *o; ++o)
        if (cur().t == T::Punct && cur().s == *o) hit = *o;
      if (!hit) return l;
      Span sp = cur().sp;
      ++p;
      ExprP r = (this->*next)();
      ExprP b = mk(EK::Binary, sp);
      b->s = hit;
      b->a = {l, r};
      l = b;
    }
  }
  ExprP expr() { static const char* o[] = {"||", nullptr}; return bin(o, &Parser::e_and); }
  ExprP e_and() { static const char* o[] = {"&&", nullptr}; return bin(o, &Parser::e_eq); }
  ExprP e_eq() { static const char* o[] = {"==", "!=", nullptr}; return bin(o, &Parser::e_rel); }
  ExprP e_rel() { static const char* o[] = {"<", "<=", ">", ">=", nullptr}; return bin(o, &Parser::e_add); }
  ExprP e_add() { static const char* o[] = {"+", "-", nullptr}; return bin(o, &Parser::e_mul); }
  ExprP e_mul() { static const char* o[] = {"*", "/", "%", nullptr}; return bin(o, &Parser::e_un); }
  ExprP e_un() {
    if (cur().t == T::Punct && (cur().s == "!" || cur().s == "-")) {
      Span sp = cur().sp;
      std::string op = t[p++].s;
      ExprP u = mk(EK::Unary, sp);
      u->s = op;
      u->a = {e_un()};
      return u;
    }
    return e_post();
  }
  ExprP e_post() {
    ExprP e = e_prim();
    for (;;) {
      Span sp = cur().sp;
      if (accept(".") || accept("->")) {
        ExprP f = mk(EK::Field, sp);
        f->s = ident();
        f->a = {e};
        e = f;
      } else if (accept("(")) {
        ExprP c = mk(EK::Call, sp);
        c->a.push_back(e);
        if (!accept(")")) {
          do c->a.push_back(expr());
          while (accept(","));
          expect(")");
        }
        e = c;
      } else if (accept("[")) {
        ExprP x = mk(EK::Index, sp);
        x->a = {e, expr()};
        expect("]");
        e = x;
      } else {
        return e;
      }
    }
  }
  ExprP e_prim() {
    const Tok& k = cur();
    if (k.t == T::Int) {
      ExprP e = mk(EK::Int, k.sp);
      e->i = std::stoll(k.s);
      ++p;
      return e;
    }
    if (k.t == T::Float) {
      ExprP e = mk(EK::Float, k.sp);
      e->f = std::stod(k.s);
      ++p;
      return e;
    }
    if (k.t == T::Str) {
      ExprP e = mk(EK::Str, k.sp);
      e->s = k.s;
      ++p;
      return e;
    }
    if (k.t == T::Ident) {
      if (k.s == "INF") {
        ++p;
        return mk(EK::Inf, k.sp);
      }
      if (k.s == "true" || k.s == "false") {
        ExprP e = mk(EK::Bool, k.sp);
        e->i = k.s == "true";
        ++p;
        return e;
      }
      ExprP e = mk(EK::Ident, k.sp);
      e->s = k.s;
      ++p;
      return e;
    }
    if (accept("(")) {
      ExprP e = expr();
      expect(")");
      return e;
    }
    fail("expected expression");
    return nullptr;
  }

  StmtP mks(SK k, Span sp) {
    auto s = std::make_shared<Stmt>();
    s->k = k;
    s->sp = sp;
    return s;
  }
  std::vector<StmtP> block() {
    std::vector<StmtP> out;
    if (accept("{")) {
      while (!accept("}")) {
        if (cur().t == T::End) fail("expected '}'");
        out.push_back(stmt());
      }
    } else {
      out.push_back(stmt());
    }
    return out;
  }
  void red_prefix(StmtP& s) {  // Iterate While|Until Any|All
    if (is("While") || is("Until")) {
      s->cond_mode = is("While") ? IRGL_COND_WHILE : IRGL_COND_UNTIL;
      ++p;
      if (accept("Any")) s->red = IRGL_RED_ANY;
      else if (accept("All")) s->red = IRGL_RED_ALL;
      else fail("expected Any or All");
    }
  }
  void call_args(StmtP& s) {
    s->var = ident();
    expect("(");
    if (!accept(")")) {
      do s->args.push_back(expr());
      while (accept(","));
      expect(")");
    }
  }
  StmtP stmt() {
    Span sp = cur().sp;
    if (accept("ForAll") || accept("for")) {
      const bool par = t[p - 1].s == "ForAll";
      StmtP s = mks(par ? SK::ForAll : SK::For, sp);
      expect("(");
      s->var = ident();
      expect("In");
      s->rhs = expr();
      expect(")");
      s->body = block();
      return s;
    }
    if (accept("if")) {
      StmtP s = mks(SK::If, sp);
      expect("(");
      s->rhs = expr();
      expect(")");
      s->body = block();
      if (accept("else") || accept("Else")) s->els = block();
      return s;
    }
    if (accept("while")) {
      StmtP s = mks(SK::While, sp);
      expect("(");
      s->rhs = expr();
      expect(")");
      s->body = block();
      return s;
    }
    if (accept("Iterate")) {
      StmtP s = mks(SK::Iterate, sp);
      red_prefix(s);
      call_args(s);
      if (accept("Initial")) {
        s->has_init = true;
        if (accept("[")) {
          if (!accept("]")) {
            do s->init.push_back(expr());
            while (accept(","));
            expect("]");
          }
        } else {
          s->init.push_back(expr());  // Initial graph.nodes (FromArray over all nodes)
        }
      }
      if (is("{")) s->body = block();
      semi();
      return s;
    }
    if (is("Any") || is("All")) {  // Any(Invoke k(args)) / All(...)
      StmtP s = mks(SK::Invoke, sp);
      s->red = is("Any") ? IRGL_RED_ANY : IRGL_RED_ALL;
      ++p;
      expect("(");
      expect("Invoke");
      call_args(s);
      expect(")");
      semi();
      return s;
    }
    if (accept("Invoke")) {
      StmtP s = mks(SK::Invoke, sp);
      call_args(s);
      semi();
      return s;
    }
    if (accept("Pipe")) {
      StmtP s = mks(SK::Pipe, sp);
      s->once = accept("Once");
      s->body = block();
      semi();
      return s;
    }
    if (accept("ReduceAndReturn") || accept("Retry") || accept("Respawn")) {
      const std::string kw = t[p - 1].s;
      StmtP s = mks(kw == "Retry" ? SK::Retry : kw == "Respawn" ? SK::Respawn : SK::ReduceAndReturn, sp);
      expect("(");
      s->rhs = expr();
      expect(")");
      semi();
      return s;
    }
    if (accept("SyncRunningThreads")) {
      StmtP s = mks(SK::Sync, sp);
      if (accept("(")) expect(")");
      semi();
      return s;
    }
    if (accept("Atomic")) {
      StmtP s = mks(SK::Atomic, sp);
      expect("(");
      s->rhs = expr();
      expect(")");
      s->body = block();
      if (accept("Else")) s->els = block();
      return s;
    }
    // expression statement / assignment
    ExprP e = expr();
    if (accept("=")) {
      ExprP r = expr();
      semi();
      // v = wl.pop(i) -> WlPop
      if (e->k == EK::Ident && r->k == EK::Call && r->a[0]->k == EK::Field && r->a[0]->s == "pop" &&
          r->a[0]->a[0]->k == EK::Ident && r->a[0]->a[0]->s == "wl") {
        if (r->a.size() != 2) fail("wl.pop takes one index");
        StmtP s = mks(SK::WlPop, sp);
        s->var = e->s;
        s->rhs = r->a[1];
        return s;
      }
      if (r->k == EK::Call && r->a[0]->k == EK::Field && r->a[0]->a[0]->k == EK::Ident &&
          r->a[0]->a[0]->s == "wl") {
        errs.push_back({sp, "E103", "worklist method '" + r->a[0]->s + "' (only pop and push exist)"});
        throw 1;
      }
      StmtP s = mks(SK::Assign, sp);
      s->lhs = e;
      s->rhs = r;
      return s;
    }
    if (accept("+=") || accept("-=") || accept("*=")) {
      StmtP s = mks(SK::OpAssign, sp);
      s->op = t[p - 1].s.substr(0, 1);
      s->lhs = e;
      s->rhs = expr();
      semi();
      return s;
    }
    if (accept("++") || accept("--")) {
      StmtP s = mks(SK::Incr, sp);
      s->op = t[p - 1].s;
      s->lhs = e;
      semi();
      return s;
    }
    semi();
    if (e->k == EK::Call && e->a[0]->k == EK::Field && e->a[0]->a[0]->k == EK::Ident &&
        e->a[0]->a[0]->s == "wl") {
      if (e->a[0]->s != "push") {
        errs.push_back({sp, "E103", "worklist method '" + e->a[0]->s + "' (only pop and push exist)"});
        throw 1;
      }
      if (e->a.size() != 2) fail("wl.push takes one value");
      StmtP s = mks(SK::WlPush, sp);
      s->rhs = e->a[1];
      return s;
    }
    StmtP s = mks(SK::ExprStmt, sp);
    s->rhs = e;
    return s;
  }

  void module(Module& m) {
    while (cur().t != T::End) {
      if (accept("Kernel")) {
        Kernel k;
        k.sp = t[p - 1].sp;
        k.name = ident();
        expect("(");
        if (!accept(")")) {
          do k.params.push_back(ident());
          while (accept(","));
          expect(")");
        }
        expect("{");
        while (!accept("}")) {
          if (cur().t == T::End) fail("expected '}' closing kernel " + k.name);
          k.body.push_back(stmt());
        }
        for (const Kernel& o : m.kernels)
          if (o.name == k.name) {
            errs.push_back({k.sp, "E007", "duplicate kernel '" + k.name + "'"});
            throw 1;
          }
        m.kernels.push_back(std::move(k));
      } else {
        m.top.push_back(stmt());
      }
    }
  }
};

// ---- printer (canonical form) -----------------------------------------------------------------
static void pe(std::ostream& o, const ExprP& e) {
  switch (e->k) {
    case EK::Int: o << e->i; break;
    case EK::Float: {
      char b[64];
      snprintf(b, sizeof b, "%.17g", e->f);
      std::string s = b;
      if (s.find_first_of(".e") == std::string::npos) s += ".0";
      o << s;
    } break;
    case EK::Str: o << '"' << e->s << '"'; break;
    case EK::Ident: o << e->s; break;
    case EK::Inf: o << "INF"; break;
    case EK::Bool: o << (e->i ? "true" : "false"); break;
    case EK::Unary: o << e->s << "("; pe(o, e->a[0]); o << ")"; break;
    case EK::Binary: o << "("; pe(o, e->a[0]); o << " " << e->s << " "; pe(o, e->a[1]); o << ")"; break;
    case EK::Field: pe(o, e->a[0]); o << "." << e->s; break;
    case EK::Call:
      pe(o, e->a[0]);
      o << "(";
      for (size_t i = 1; i < e->a.size(); ++i) {
        if (i > 1) o << ", ";
        pe(o, e->a[i]);
      }
      o << ")";
      break;
    case EK::Index: pe(o, e->a[0]); o << "["; pe(o, e->a[1]); o << "]"; break;
  }
}
static void pb(std::ostream& o, const std::vector<StmtP>& b, int ind);
static void ps(std::ostream& o, const StmtP& s, int ind) {
  const std::string in(ind * 2, ' ');
  auto args = [&](const std::vector<ExprP>& a) {
    for (size_t i = 0; i < a.size(); ++i) {
      if (i) o << ", ";
      pe(o, a[i]);
    }
  };
  const char* red = s->red == IRGL_RED_ANY ? "Any" : "All";
  switch (s->k) {
    case SK::Assign: o << in; pe(o, s->lhs); o << " = "; pe(o, s->rhs); o << ";\n"; break;
    case SK::OpAssign: o << in; pe(o, s->lhs); o << " " << s->op << "= "; pe(o, s->rhs); o << ";\n"; break;
    case SK::Incr: o << in; pe(o, s->lhs); o << s->op << ";\n"; break;
    case SK::ExprStmt: o << in; pe(o, s->rhs); o << ";\n"; break;
    case SK::WlPop: o << in << s->var << " = wl.pop("; pe(o, s->rhs); o << ");\n"; break;
    case SK::WlPush: o << in << "wl.push("; pe(o, s->rhs); o << ");\n"; break;
    case SK::ForAll:
    case SK::For:
      o << in << (s->k == SK::ForAll ? "ForAll" : "for") << " (" << s->var << " In ";
      pe(o, s->rhs);
      o << ") {\n";
      pb(o, s->body, ind + 1);
      o << in << "}\n";
      break;
    case SK::If:
    case SK::While:
      o << in << (s->k == SK::If ? "if" : "while") << " (";
      pe(o, s->rhs);
      o << ") {\n";
      pb(o, s->body, ind + 1);
      o << in << "}";
      if (!s->els.empty()) {
        o << " else {\n";
        pb(o, s->els, ind + 1);
        o << in << "}";
      }
      o << "\n";
      break;
    case SK::Iterate:
      o << in << "Iterate ";
      if (s->cond_mode) o << (s->cond_mode == IRGL_COND_WHILE ? "While " : "Until ") << red << " ";
      o << s->var << "(";
      args(s->args);
      o << ")";
      if (s->has_init) {
        o << " Initial [";
        args(s->init);
        o << "]";
      }
      o << " {\n";
      pb(o, s->body, ind + 1);
      o << in << "};\n";
      break;
    case SK::Invoke:
      o << in;
      if (s->red) o << red << "(";
      o << "Invoke " << s->var << "(";
      args(s->args);
      o << ")";
      if (s->red) o << ")";
      o << ";\n";
      break;
    case SK::Pipe:
      o << in << "Pipe " << (s->once ? "Once " : "") << "{\n";
      pb(o, s->body, ind + 1);
      o << in << "};\n";
      break;
    case SK::ReduceAndReturn:
    case SK::Retry:
    case SK::Respawn:
      o << in << (s->k == SK::Retry ? "Retry" : s->k == SK::Respawn ? "Respawn" : "ReduceAndReturn") << "(";
      pe(o, s->rhs);
      o << ");\n";
      break;
    case SK::Sync: o << in << "SyncRunningThreads;\n"; break;
    case SK::Atomic:
      o << in << "Atomic (";
      pe(o, s->rhs);
      o << ") {\n";
      pb(o, s->body, ind + 1);
      o << in << "}";
      if (!s->els.empty()) {
        o << " Else {\n";
        pb(o, s->els, ind + 1);
        o << in << "}";
      }
      o << "\n";
      break;
  }
}
static void pb(std::ostream& o, const std::vector<StmtP>& b, int ind) {
  for (const StmtP& s : b) ps(o, s, ind);
}
static std::string print_module(const Module& m) {
  std::ostringstream o;
  for (const Kernel& k : m.kernels) {
    o << "Kernel " << k.name << "(";
    for (size_t i = 0; i < k.params.size(); ++i) o << (i ? ", " : "") << k.params[i];
    o << ") {\n";
    pb(o, k.body, 1);
    o << "}\n\n";
  }
  pb(o, m.top, 0);
  return o.str();
}

// ---- recogniser: unification against the operators' IrGL form --------------------------------
using Binds = std::map<std::string, std::string>;
static bool mexpr(const ExprP& pt, const ExprP& e, Binds& b) {
  if (pt->k == EK::Ident && !pt->s.empty() && pt->s[0] == '$') {
    if (e->k != EK::Ident) return false;
    auto it = b.find(pt->s);
    if (it != b.end()) return it->second == e->s;
    for (auto& kv : b)
      if (kv.second == e->s) return false;  // distinct pattern variables bind distinct names
    b[pt->s] = e->s;
    return true;
  }
  if ((pt->k == EK::Int && e->k == EK::Float) || (pt->k == EK::Float && e->k == EK::Int))
    return (pt->k == EK::Int ? (double)pt->i : pt->f) == (e->k == EK::Int ? (double)e->i : e->f);
  if (pt->k != e->k) return false;
  switch (pt->k) {
    case EK::Int: return pt->i == e->i;
    case EK::Float: return pt->f == e->f;  // (Int/Float mixes are handled below the switch)
    case EK::Bool: return pt->i == e->i;
    case EK::Inf: return true;
    case EK::Str: return pt->s == e->s;
    case EK::Ident: return pt->s == e->s;
    case EK::Field:
      if (pt->s.size() && pt->s[0] == '$') {
        auto it = b.find(pt->s);
        if (it != b.end() && it->second != e->s) return false;
        b[pt->s] = e->s;
      } else if (pt->s != e->s) {
        return false;
      }
      return mexpr(pt->a[0], e->a[0], b);
    default:
      if (pt->s != e->s || pt->a.size() != e->a.size()) return false;
      for (size_t i = 0; i < pt->a.size(); ++i)
        if (!mexpr(pt->a[i], e->a[i], b)) return false;
      return true;
  }
}
static bool mbody(const std::vector<StmtP>& pt, const std::vector<StmtP>& s, Binds& b);
static bool mstmt(const StmtP& pt, const StmtP& s, Binds& b) {
  if (pt->k != s->k || pt->op != s->op) return false;
  if (!pt->var.empty()) {
    if (pt->var[0] == '$') {
      auto it = b.find(pt->var);
      if (it != b.end()) {
        if (it->second != s->var) return false;
      } else {
        for (auto& kv : b)
          if (kv.second == s->var) return false;
        b[pt->var] = s->var;
      }
    } else if (pt->var != s->var) {
      return false;
    }
  }
  if ((pt->lhs != nullptr) != (s->lhs != nullptr) || (pt->rhs != nullptr) != (s->rhs != nullptr)) return false;
  if (pt->lhs && !mexpr(pt->lhs, s->lhs, b)) return false;
  if (pt->rhs && !mexpr(pt->rhs, s->rhs, b)) return false;
  return mbody(pt->body, s->body, b) && mbody(pt->els, s->els, b);
}
static bool mbody(const std::vector<StmtP>& pt, const std::vector<StmtP>& s, Binds& b) {
  if (pt.size() != s.size()) return false;
  for (size_t i = 0; i < pt.size(); ++i)
    if (!mstmt(pt[i], s[i], b)) return false;
  return true;
}

struct Pattern {
  int op;
  const char* src;  // one Kernel; $-identifiers unify; params listed must be kernel params
};
// The operators' IrGL forms.  `$F` is the node property written.
static const Pattern kPatterns[] = {
    // Listing 2
    {IRGL_OP_BFS, R"(Kernel P($G, $L) {
      ForAll($i In wl) {
        $n = wl.pop($i)
        ForAll($e In $G.edges($n)) {
          if ($e.dst.$F == INF) { $e.dst.$F = $L; wl.push($e.dst.id) }
        }
      }
    })"},
    // data-driven SSSP, atomicMin builtin (App. B7: a one-statement Atomic min-update)
    {IRGL_OP_SSSP, R"(Kernel P($G) {
      ForAll($i In wl) {
        $n = wl.pop($i)
        ForAll($e In $G.edges($n)) {
          $d = $n.$F + $e.weight
          if (atomicMin($e.dst.$F, $d) > $d) { wl.push($e.dst.id) }
        }
      }
    })"},
    {IRGL_OP_SSSP, R"(Kernel P($G) {
      ForAll($i In wl) {
        $n = wl.pop($i)
        ForAll($e In $G.edges($n)) {
          $d = $n.$F + $e.weight
          if ($d < $e.dst.$F) { $e.dst.$F = $d; wl.push($e.dst.id) }
        }
      }
    })"},
    // CC by min-label propagation
    {IRGL_OP_CC_LP, R"(Kernel P($G) {
      ForAll($i In wl) {
        $n = wl.pop($i)
        ForAll($e In $G.edges($n)) {
          if (atomicMin($e.dst.$F, $n.$F) > $n.$F) { wl.push($e.dst.id) }
        }
      }
    })"},
    {IRGL_OP_CC_LP, R"(Kernel P($G) {
      ForAll($i In wl) {
        $n = wl.pop($i)
        ForAll($e In $G.edges($n)) {
          if ($n.$F < $e.dst.$F) { $e.dst.$F = $n.$F; wl.push($e.dst.id) }
        }
      }
    })"},
    // topology-driven pull PageRank (Iterate While Any, ReduceAndReturn)
    {IRGL_OP_PR, R"(Kernel P($G, $D, $T) {
      ForAll($n In $G.nodes) {
        $s = 0
        for ($e In $G.edges($n)) { $s += $e.dst.$C }
        $r = (1 - $D) / $G.N + $D * $s
        ReduceAndReturn(fabs($r - $n.$F) > $T)
        $n.$X = $r
      }
    })"},
};

static std::vector<Kernel> parse_patterns() {
  std::vector<Kernel> out;
  for (const Pattern& pt : kPatterns) {
    std::vector<Error> e;
    Parser ps(lex(pt.src, e), e);
    Module m;
    try {
      ps.module(m);
    } catch (int) {
    }
    if (!e.empty() || m.kernels.size() != 1) {
      fprintf(stderr, "irgl frontend: internal pattern failed to parse\n");
      continue;
    }
    m.kernels[0].op = pt.op;
    out.push_back(m.kernels[0]);
  }
  return out;
}

static bool uses_orchestration(const std::vector<StmtP>& b) {
  for (const StmtP& s : b) {
    if (s->k == SK::Iterate || s->k == SK::Invoke || s->k == SK::Pipe) return true;
    if (uses_orchestration(s->body) || uses_orchestration(s->els)) return true;
  }
  return false;
}

static void recognise(Module& m) {
  static const std::vector<Kernel> pats = parse_patterns();
  for (Kernel& k : m.kernels) {
    k.host = uses_orchestration(k.body);
    if (k.host) continue;
    for (const Kernel& pt : pats) {
      Binds b;
      // pattern parameters map onto the kernel's parameters positionally by role: every
      // pattern parameter must bind to one of the kernel's parameters
      if (!mbody(pt.body, k.body, b)) continue;
      bool ok = k.params.size() >= pt.params.size();
      for (const std::string& pp : pt.params) {
        auto it = b.find(pp);
        bool is_param = false;
        if (it != b.end())
          for (const std::string& kp : k.params) is_param |= kp == it->second;
        ok &= is_param;
      }
      if (!ok) continue;
      k.op = pt.op;
      k.bind = b;
      auto f = b.find("$F");
      k.field = f != b.end() ? f->second : "";
      break;
    }
  }
}

}  // namespace fe
}  // namespace irgl

using namespace irgl::fe;

struct irgl_module {
  Module m;
};

namespace {

void put_diag(char* diag, size_t len, const std::string& s) {
  if (!diag || !len) return;
  snprintf(diag, len, "%s", s.c_str());
}

std::string fmt_errors(const std::string& file, const std::vector<Error>& errs) {
  std::string o;
  for (const Error& e : errs)
    o += file + ":" + std::to_string(e.sp.line) + ":" + std::to_string(e.sp.col) + ": error[" + e.rule +
         "]: " + e.msg + "\n";
  return o;
}

// ---- run_host -------------------------------------------------------------------------------
struct Runner {
  irgl_ctx* ctx;
  irgl_module* mod;
  irgl_graph* g;
  std::map<std::string, double>& env;
  irgl_run_info& info;
  std::vector<Error> errs;
  irgl_pipe* pipe = nullptr;  // the outermost Pipe / Iterate's worklists
  int64_t n = 0;
  bool state_ready[16] = {};

  Runner(irgl_ctx* c, irgl_module* md, irgl_graph* gr, std::map<std::string, double>& e, irgl_run_info& ri)
      : ctx(c), mod(md), g(gr), env(e), info(ri) {}

  [[noreturn]] void fail(const Span& sp, const char* rule, const std::string& msg, irgl_status_t st = IRGL_E_INVALID) {
    errs.push_back({sp, rule, msg});
    throw st;
  }
  void check(irgl_status_t st, const Span& sp, const char* what) {
    if (st != IRGL_OK) fail(sp, "E_RUNTIME", std::string(what) + ": " + irgl_last_error(ctx), st);
  }

  double eval(const ExprP& e) {
    switch (e->k) {
      case EK::Int: return (double)e->i;
      case EK::Float: return e->f;
      case EK::Bool: return (double)e->i;
      case EK::Inf: return 2147483647.0;
      case EK::Ident: {
        auto it = env.find(e->s);
        if (it == env.end()) fail(e->sp, "E201", "unbound name '" + e->s + "'");
        return it->second;
      }
      case EK::Field:
        if (e->s == "N" || e->s == "nnodes") return (double)n;
        fail(e->sp, "E202", "host code cannot read field '" + e->s + "'");
      case EK::Unary: {
        const double x = eval(e->a[0]);
        return e->s == "-" ? -x : (double)(x == 0);
      }
      case EK::Binary: {
        const double a = eval(e->a[0]), b = eval(e->a[1]);
        const std::string& o = e->s;
        if (o == "+") return a + b;
        if (o == "-") return a - b;
        if (o == "*") return a * b;
        if (o == "/") {
          if (b == 0) fail(e->sp, "E203", "division by zero");
          return a / b;
        }
        if (o == "%") return (double)((int64_t)a % (int64_t)b);
        if (o == "<") return a < b;
        if (o == "<=") return a <= b;
        if (o == ">") return a > b;
        if (o == ">=") return a >= b;
        if (o == "==") return a == b;
        if (o == "!=") return a != b;
        if (o == "&&") return a != 0 && b != 0;
        if (o == "||") return a != 0 || b != 0;
        fail(e->sp, "E204", "operator " + o);
      }
      default: fail(e->sp, "E205", "expression not supported in host code");
    }
  }

  const Kernel& kernel(const Span& sp, const std::string& name) {
    for (const Kernel& k : mod->m.kernels)
      if (k.name == name) return k;
    fail(sp, "E008", "Invoke/Iterate of unknown kernel '" + name + "'");
  }
  const Kernel& plain(const StmtP& s) {
    const Kernel& k = kernel(s->sp, s->var);
    if (k.host) fail(s->sp, "E301", "'" + k.name + "' is a host kernel (orchestration only launches plain kernels)");
    if (k.op < 0)
      fail(s->sp, "E_UNSUPPORTED", "kernel '" + k.name + "' is not one of the plain kernels this runtime implements "
           "(BFS / SSSP / CC label propagation / PageRank in their IrGL form); the CBlock interpreter is out of scope",
           IRGL_E_UNSUPPORTED);
    return k;
  }
  // value of the kernel argument that binds pattern parameter `pp`
  bool arg_of(const Kernel& k, const StmtP& s, const char* pp, double* v) {
    auto it = k.bind.find(pp);
    if (it == k.bind.end()) return false;
    for (size_t i = 0; i < k.params.size() && i < s->args.size(); ++i)
      if (k.params[i] == it->second) {
        *v = eval(s->args[i]);
        return true;
      }
    return false;
  }
  void ensure_pipe(const Span& sp) {
    if (!pipe) check(irgl_pipe_create(ctx, std::max<int64_t>(n, 1), &pipe), sp, "pipe");
  }
  void seed(const StmtP& s, const Kernel& k) {
    ensure_pipe(s->sp);
    if (s->init.size() == 1 && s->init[0]->k == EK::Field && s->init[0]->s == "nodes") {
      check(irgl_pipe_init_range(pipe, 0, n), s->sp, "Initial nodes");
    } else {
      std::vector<int64_t> items;
      for (const ExprP& e : s->init) items.push_back((int64_t)eval(e));
      check(irgl_pipe_init_scalars(pipe, items.data(), (int64_t)items.size()), s->sp, "Initial");
    }
    (void)k;
  }
  irgl_op_args args_for(const Kernel& k, const StmtP& s) {
    irgl_op_args a;
    memset(&a, 0, sizeof a);
    a.delta = -1;
    a.defer = -1;
    double v;
    // Listing 2 starts LEVEL = 0 and the source is preset to 0 (App. B2): the first discovery
    // round writes LEVEL + 1 (hop distance)
    if (k.op == IRGL_OP_BFS && arg_of(k, s, "$L", &v)) a.round_start = (int64_t)v + 1;
    if (k.op == IRGL_OP_PR) {
      if (arg_of(k, s, "$D", &v)) a.pr_damping = v;
      if (arg_of(k, s, "$T", &v)) a.pr_tol = v;
    }
    return a;
  }
  void between(const StmtP& s, int64_t rounds) {
    for (int64_t r = 0; r < rounds && !s->body.empty(); ++r) exec(s->body);
  }

  void iterate(const StmtP& s) {
    const Kernel& k = plain(s);
    const bool wl_op = k.op == IRGL_OP_BFS || k.op == IRGL_OP_SSSP || k.op == IRGL_OP_CC_LP;
    irgl_op_args a = args_for(k, s);
    irgl_iterate_opts o;
    memset(&o, 0, sizeof o);
    o.outline = -1;
    o.cond_mode = s->cond_mode;
    o.reduction = s->red;
    o.reset = 1;
    if (wl_op) {
      if (s->has_init) seed(s, k);
      else if (!pipe) fail(s->sp, "E302", "Iterate of a worklist kernel outside a Pipe needs Initial [...]");
    }
    irgl_iter_stats st;
    memset(&st, 0, sizeof st);
    check(irgl_iterate(ctx, wl_op ? pipe : nullptr, g, (irgl_op)k.op, &a, &o, &st), s->sp, "Iterate");
    state_ready[k.op] = true;
    info.last_op = k.op;
    info.last_reduced = st.last_reduced;
    info.invocations += st.rounds;
    info.orchestrations++;
    between(s, st.rounds);
  }
  void invoke(const StmtP& s) {
    const Kernel& k = plain(s);
    const bool wl_op = k.op == IRGL_OP_BFS || k.op == IRGL_OP_SSSP || k.op == IRGL_OP_CC_LP;
    irgl_op_args a = args_for(k, s);
    if (wl_op && !pipe) fail(s->sp, "E302", "Invoke of a worklist kernel outside a Pipe / Iterate");
    if (!state_ready[k.op]) {
      check(irgl_op_reset(ctx, g, (irgl_op)k.op, &a, wl_op ? pipe : nullptr), s->sp, "operator state");
      state_ready[k.op] = true;
    }
    int32_t r = -1;
    irgl_iter_stats st;
    memset(&st, 0, sizeof st);
    check(irgl_invoke(ctx, wl_op ? pipe : nullptr, g, (irgl_op)k.op, &a, (irgl_reduction)s->red, &r, &st),
          s->sp, "Invoke");
    info.last_op = k.op;
    info.last_reduced = s->red ? r : -1;
    info.invocations += 1;
    info.orchestrations++;
  }

  void exec(const std::vector<StmtP>& body) {
    for (const StmtP& s : body) {
      switch (s->k) {
        case SK::Assign:
          if (s->lhs->k != EK::Ident) fail(s->sp, "E206", "host code assigns scalars only");
          env[s->lhs->s] = eval(s->rhs);
          break;
        case SK::OpAssign: {
          if (s->lhs->k != EK::Ident) fail(s->sp, "E206", "host code assigns scalars only");
          double& x = env[s->lhs->s];
          const double v = eval(s->rhs);
          x = s->op == "+" ? x + v : s->op == "-" ? x - v : x * v;
        } break;
        case SK::Incr:
          if (s->lhs->k != EK::Ident) fail(s->sp, "E206", "host code increments scalars only");
          env[s->lhs->s] += s->op == "++" ? 1 : -1;
          break;
        case SK::If:
          exec(eval(s->rhs) != 0 ? s->body : s->els);
          break;
        case SK::While: {
          int64_t guard = 0;
          while (eval(s->rhs) != 0) {
            exec(s->body);
            if (++guard > (1ll << 40)) fail(s->sp, "E207", "host while loop does not terminate");
          }
        } break;
        case SK::Iterate: iterate(s); break;
        case SK::Invoke: invoke(s); break;
        case SK::Pipe: {
          // the outermost Pipe creates the pipe context; nested constructs share it; a looping
          // Pipe repeats while `in` is non-empty at the start of its body
          ensure_pipe(s->sp);
          for (int64_t it = 0;; ++it) {
            exec(s->body);
            if (s->once) break;
            int64_t in = 0;
            check(irgl_pipe_size(pipe, IRGL_WL_IN, &in), s->sp, "Pipe");
            if (in == 0) break;
          }
        } break;
        case SK::ExprStmt:
          if (s->rhs->k == EK::Call && s->rhs->a[0]->k == EK::Ident && s->rhs->a[0]->s == "printf") {
            print(s);
            break;
          }
          eval(s->rhs);
          break;
        default:
          fail(s->sp, "E303", "statement only valid inside a plain kernel");
      }
    }
  }
  void print(const StmtP& s) {
    if (s->rhs->a.size() < 2 || s->rhs->a[1]->k != EK::Str) fail(s->sp, "E208", "printf needs a format string");
    const std::string& f = s->rhs->a[1]->s;
    std::string out;
    size_t arg = 2;
    for (size_t i = 0; i < f.size(); ++i) {
      if (f[i] == '\\' && i + 1 < f.size() && f[i + 1] == 'n') {
        out += '\n';
        ++i;
      } else if (f[i] == '%' && i + 1 < f.size()) {
        const char c = f[++i];
        if (c == '%') {
          out += '%';
          continue;
        }
        if (arg >= s->rhs->a.size()) fail(s->sp, "E208", "printf: missing argument");
        const double v = eval(s->rhs->a[arg++]);
        char b[64];
        if (c == 'f' || c == 'g' || c == 'e') snprintf(b, sizeof b, "%g", v);
        else snprintf(b, sizeof b, "%lld", (long long)v);
        out += b;
      } else {
        out += f[i];
      }
    }
    fputs(out.c_str(), stdout);
    fflush(stdout);
  }
};

}  // namespace

extern "C" {

irgl_status_t irgl_module_parse(const char* text, const char* filename, irgl_module** out, char* diag,
                                size_t diag_len) {
  if (!text || !out) return IRGL_E_INVALID;
  const std::string file = filename ? filename : "<input>";
  std::vector<Error> errs;
  auto toks = lex(text, errs);
  auto mod = std::make_unique<irgl_module>();
  mod->m.file = file;
  if (errs.empty()) {
    Parser p(std::move(toks), errs);
    try {
      p.module(mod->m);
    } catch (int) {
    }
  }
  if (!errs.empty()) {
    put_diag(diag, diag_len, fmt_errors(file, errs));
    return IRGL_E_INVALID;
  }
  recognise(mod->m);
  *out = mod.release();
  put_diag(diag, diag_len, "");
  return IRGL_OK;
}

irgl_status_t irgl_module_destroy(irgl_module* m) {
  delete m;
  return IRGL_OK;
}

int irgl_module_kernel_count(const irgl_module* m) { return m ? (int)m->m.kernels.size() : 0; }

irgl_status_t irgl_module_kernel_info(const irgl_module* m, int index, char* name, size_t name_len, int32_t* op,
                                      char* field, size_t field_len, int32_t* host) {
  if (!m || index < 0 || index >= (int)m->m.kernels.size()) return IRGL_E_INVALID;
  const Kernel& k = m->m.kernels[index];
  put_diag(name, name_len, k.name);
  put_diag(field, field_len, k.field);
  if (op) *op = k.op;
  if (host) *host = k.host ? 1 : 0;
  return IRGL_OK;
}

irgl_status_t irgl_module_print(const irgl_module* m, char* out, size_t out_len, size_t* needed) {
  if (!m) return IRGL_E_INVALID;
  const std::string s = print_module(m->m);
  if (needed) *needed = s.size() + 1;
  if (out && out_len) snprintf(out, out_len, "%s", s.c_str());
  return (out && out_len < s.size() + 1) ? IRGL_E_INVALID : IRGL_OK;
}

irgl_status_t irgl_run_host(irgl_ctx* ctx, irgl_module* m, const char* entry, irgl_graph* g,
                            const char* const* names, const double* values, int nbind, irgl_run_info* info,
                            char* diag, size_t diag_len) {
  if (!ctx || !m) return IRGL_E_INVALID;
  irgl_run_info ri;
  memset(&ri, 0, sizeof ri);
  ri.last_op = -1;
  ri.last_reduced = -1;
  m->m.scalars.clear();
  for (int i = 0; i < nbind; ++i)
    if (names && names[i] && values) m->m.scalars[names[i]] = values[i];
  Runner r(ctx, m, g, m->m.scalars, ri);
  if (g) {
    irgl_graph_info gi;
    if (irgl_graph_info_get(g, &gi) == IRGL_OK) r.n = gi.n;
  }
  irgl_status_t st = IRGL_OK;
  try {
    const std::vector<StmtP>* body = &m->m.top;
    if (entry && *entry) {
      const Kernel* k = nullptr;
      for (const Kernel& kk : m->m.kernels)
        if (kk.name == entry) k = &kk;
      if (!k) r.fail(Span{}, "E008", std::string("unknown entry '") + entry + "'");
      if (!k->host) r.fail(k->sp, "E304", std::string("entry '") + entry + "' is not a host kernel");
      body = &k->body;
    }
    r.exec(*body);
  } catch (irgl_status_t e) {
    st = e;
  }
  if (r.pipe) irgl_pipe_destroy(r.pipe);
  if (info) *info = ri;
  put_diag(diag, diag_len, fmt_errors(m->m.file, r.errs));
  return st;
}

irgl_status_t irgl_module_scalar(const irgl_module* m, const char* name, double* out) {
  if (!m || !name || !out) return IRGL_E_INVALID;
  auto it = m->m.scalars.find(name);
  if (it == m->m.scalars.end()) return IRGL_E_INVALID;
  *out = it->second;
  return IRGL_OK;
}

}  // extern "C"
