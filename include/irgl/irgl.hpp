// irgl/irgl.hpp — header-only C++ operator API over the C-ABI (irgl/rt.h).
//
// Mirrors the IrGL orchestration constructs of reference/proj/core/include/irgl/ast.hpp:
//   Pipe [Once] { ... }            ast.hpp:206-210   -> irgl::Pipe (owns in/out/retry)
//   WorklistInit Scalars/FromArray ast.hpp:100-110   -> Pipe::initial({...}) / Pipe::from_array
//   Invoke kernel(args) [Any|All]  ast.hpp:180-184   -> irgl::Context::invoke(...)
//   Iterate [While|Until ...] kernel(args) Initial [..] { between_rounds }
//                                  ast.hpp:186-204   -> irgl::Context::iterate(...) (device-side
//                                                       round counter), or a host loop of invoke()
//                                                       with a between_rounds lambda
// Errors are values in the C-ABI; here they throw irgl::Error carrying the "RULE: message" text.
#pragma once
#include <cstdint>
#include <initializer_list>
#include <stdexcept>
#include <string>
#include <utility>
#include <vector>

#include "irgl/rt.h"

namespace irgl {

struct Error : std::runtime_error {
  irgl_status_t status;
  Error(irgl_status_t s, const std::string& m) : std::runtime_error(m), status(s) {}
};

inline void check(irgl_status_t s, const irgl_ctx* c = nullptr) {
  if (s != IRGL_OK) throw Error(s, irgl_last_error(c));
}

enum class Reduction { None = IRGL_RED_NONE, Any = IRGL_RED_ANY, All = IRGL_RED_ALL };

class Context;

class Graph {
 public:
  Graph() = default;
  Graph(const Graph&) = delete;
  Graph& operator=(const Graph&) = delete;
  Graph(Graph&& o) noexcept : g_(std::exchange(o.g_, nullptr)) {}
  ~Graph() {
    if (g_) irgl_graph_destroy(g_);
  }
  irgl_graph* get() const { return g_; }
  irgl_graph_info info() const {
    irgl_graph_info i{};
    check(irgl_graph_info_get(g_, &i));
    return i;
  }

 private:
  friend class Context;
  explicit Graph(irgl_graph* g) : g_(g) {}
  irgl_graph* g_ = nullptr;
};

class Pipe {
 public:
  Pipe(const Pipe&) = delete;
  Pipe& operator=(const Pipe&) = delete;
  Pipe(Pipe&& o) noexcept : p_(std::exchange(o.p_, nullptr)), ctx_(o.ctx_) {}
  ~Pipe() {
    if (p_) irgl_pipe_destroy(p_);
  }
  irgl_pipe* get() const { return p_; }
  // WorklistInit Scalars (ast.hpp:101)
  Pipe& initial(std::initializer_list<int64_t> items) {
    std::vector<int64_t> v(items);
    check(irgl_pipe_init_scalars(p_, v.data(), (int64_t)v.size()), ctx_);
    return *this;
  }
  // WorklistInit FromArray (ast.hpp:104)
  Pipe& from_array(const std::vector<int64_t>& arr) {
    check(irgl_pipe_init_from_array(p_, arr.data(), (int64_t)arr.size()), ctx_);
    return *this;
  }
  int64_t size(irgl_wl which = IRGL_WL_IN) const {
    int64_t n = 0;
    check(irgl_pipe_size(p_, which, &n), ctx_);
    return n;
  }
  bool empty() const { return size() == 0; }

 private:
  friend class Context;
  Pipe(irgl_pipe* p, const irgl_ctx* c) : p_(p), ctx_(c) {}
  irgl_pipe* p_ = nullptr;
  const irgl_ctx* ctx_ = nullptr;
};

class Context {
 public:
  explicit Context(std::vector<int> devices = {0}, irgl_config cfg = default_config()) {
    check(irgl_ctx_create(devices.data(), (int)devices.size(), &cfg, &c_));
  }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  ~Context() {
    if (c_) irgl_ctx_destroy(c_);
  }
  static irgl_config default_config() {
    irgl_config c{};
    c.outline = -1;
    return c;
  }
  irgl_ctx* get() const { return c_; }

  Graph csr(int64_t n, const std::vector<int64_t>& row_ptr, const std::vector<int32_t>& col,
            const std::vector<int32_t>* weight = nullptr) {
    irgl_graph* g = nullptr;
    check(irgl_graph_create_csr(c_, n, (int64_t)col.size(), row_ptr.data(), col.data(),
                                weight ? weight->data() : nullptr, &g),
          c_);
    return Graph(g);
  }
  Graph rmat(int scale, uint64_t seed = 1, uint64_t wseed = 11, int edge_factor = 16) {
    irgl_gen_spec s{};
    s.kind = IRGL_GEN_RMAT;
    s.scale = scale;
    s.edge_factor = edge_factor;
    s.seed = seed;
    s.wseed = wseed;
    irgl_graph* g = nullptr;
    check(irgl_graph_generate(c_, &s, &g), c_);
    return Graph(g);
  }
  Pipe pipe(int64_t size) {  // Pipe with WorklistInit.size
    irgl_pipe* p = nullptr;
    check(irgl_pipe_create(c_, size, &p), c_);
    return Pipe(p, c_);
  }

  // [Any|All(] Invoke op(args) [)]: returns the reduced value (identity when nothing evaluated)
  bool invoke(irgl_op op, Graph* g, Pipe* p, irgl_op_args args = {},
              Reduction red = Reduction::None, irgl_iter_stats* st = nullptr) {
    int32_t r = -1;
    check(irgl_invoke(c_, p ? p->get() : nullptr, g ? g->get() : nullptr, op, &args,
                      (irgl_reduction)red, &r, st),
          c_);
    return r == 1;
  }

  // Iterate op(args) Initial [...] { round counter ++ } — the whole loop in the runtime
  // (outlined into one persistent kernel when allowed).
  irgl_iter_stats iterate(irgl_op op, Graph* g, Pipe* p, irgl_op_args args = {},
                          irgl_iterate_opts opts = default_iterate()) {
    irgl_iter_stats st{};
    check(irgl_iterate(c_, p ? p->get() : nullptr, g ? g->get() : nullptr, op, &args, &opts, &st),
          c_);
    return st;
  }
  static irgl_iterate_opts default_iterate() {
    irgl_iterate_opts o{};
    o.outline = -1;
    o.reset = 1;
    return o;
  }

  // Iterate as a host loop of Invoke with a user between_rounds statement (Listing 2's LEVEL++).
  template <class BetweenRounds>
  int64_t iterate_host(irgl_op op, Graph& g, Pipe& p, int64_t& LEVEL, BetweenRounds between) {
    check(irgl_op_reset(c_, g.get(), op, nullptr, p.get()), c_);
    int64_t rounds = 0;
    while (!p.empty()) {
      irgl_op_args a{};
      a.round_start = LEVEL;
      invoke(op, &g, &p, a);
      between();
      ++rounds;
    }
    return rounds;
  }

  template <class T>
  std::vector<T> result(irgl_op op, Graph& g) {
    std::vector<T> out(op == IRGL_OP_TC ? 1 : (size_t)g.info().n);
    check(irgl_read_result(c_, g.get(), op, out.data(), out.size() * sizeof(T)), c_);
    return out;
  }

 private:
  irgl_ctx* c_ = nullptr;
};

}  // namespace irgl
