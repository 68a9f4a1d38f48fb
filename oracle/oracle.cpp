// oracle.cpp — CPU ORACLE (test infrastructure only; see oracle.h header for the rules and the
// reference anchors).  Plain C++17 + OpenMP, no CUDA, no product code.
#include "oracle.h"

#include <omp.h>
#include <parallel/algorithm>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <queue>
#include <vector>

// ------------------------------------------------------------------------------------------
// Philox-4x32-10 (Salmon et al. 2011), the counter-based generator shared by host and device
// graph generators (SURVEY.md §7 "Hard parts" 5).
static inline void philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                          uint32_t k1, uint32_t out[4]) {
  for (int r = 0; r < 10; ++r) {
    uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    uint32_t n1 = (uint32_t)p1;
    uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    uint32_t n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u; k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}
extern "C" void orc_philox4x32(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0,
                               uint32_t k1, uint32_t out[4]) {
  philox(c0, c1, c2, c3, k0, k1, out);
}

static const uint32_t TAG_RMAT = 0x524D4154u;  // 'RMAT'
static const uint32_t TAG_SCRM = 0x5343524Du;  // 'SCRM'
static const uint32_t TAG_WGHT = 0x57474854u;  // 'WGHT'
static const uint32_t TAG_PERC = 0x50455243u;  // 'PERC'
static const uint32_t TAG_SRCS = 0x53524353u;  // 'SRCS'
// Graph500 quadrant thresholds as exact integers: floor(p * 2^32) for A, A+B, A+B+C.
static const uint32_t TH_A = 2448131358u;    // 0.57
static const uint32_t TH_AB = 3264175144u;   // 0.76
static const uint32_t TH_ABC = 4080218931u;  // 0.95

extern "C" uint64_t orc_scramble(uint64_t x, int scale, uint64_t seed) {
  uint32_t k[4];
  philox(0, 0, 0, TAG_SCRM, (uint32_t)seed, (uint32_t)(seed >> 32), k);
  const uint64_t mask = (scale >= 64) ? ~0ull : ((1ull << scale) - 1);
  x = (x * (uint64_t)(k[0] | 1u) + k[1]) & mask;
  x ^= x >> (scale / 2 + 1);
  x = (x * (uint64_t)(k[2] | 1u) + k[3]) & mask;
  x ^= x >> (scale / 3 + 1);
  return x;
}

static inline int32_t hash_weight(uint64_t u, uint64_t v, uint64_t wseed) {
  uint64_t a = u < v ? u : v, b = u < v ? v : u;
  uint32_t r[4];
  philox((uint32_t)a, (uint32_t)b, (uint32_t)((a >> 32) | ((b >> 32) << 16)), TAG_WGHT,
         (uint32_t)wseed, (uint32_t)(wseed >> 32), r);
  return 1 + (int32_t)(r[0] % 255u);
}

struct orc_graph {
  int64_t n = 0, m = 0;
  std::vector<int64_t> row_ptr;
  std::vector<int32_t> col;
  std::vector<int32_t> w;
};

// keys = (u << 32) | v, directed.  Sort + unique + CSR (drops self loops already removed).
static orc_graph* csr_from_keys(int64_t n, std::vector<uint64_t>& keys, uint64_t wseed,
                                const std::vector<int32_t>* explicit_w = nullptr) {
  orc_graph* g = new orc_graph();
  g->n = n;
  if (!explicit_w) {
    __gnu_parallel::sort(keys.begin(), keys.end());
    keys.erase(std::unique(keys.begin(), keys.end()), keys.end());
  }
  g->m = (int64_t)keys.size();
  g->row_ptr.assign(n + 1, 0);
  g->col.resize(g->m);
  g->w.resize(g->m);
  for (int64_t i = 0; i < g->m; ++i) g->row_ptr[(keys[i] >> 32) + 1]++;
  for (int64_t i = 0; i < n; ++i) g->row_ptr[i + 1] += g->row_ptr[i];
#pragma omp parallel for schedule(static)
  for (int64_t i = 0; i < g->m; ++i) {
    uint64_t u = keys[i] >> 32, v = keys[i] & 0xffffffffull;
    g->col[i] = (int32_t)v;
    g->w[i] = explicit_w ? (*explicit_w)[i] : hash_weight(u, v, wseed);
  }
  return g;
}

extern "C" orc_graph* orc_rmat(int scale, int edge_factor, uint64_t seed, uint64_t wseed) {
  if (scale < 1 || scale > 30 || edge_factor < 1) return nullptr;
  const int64_t n = 1ll << scale;
  const int64_t ne = (int64_t)edge_factor << scale;
  const int nblk = (scale + 3) / 4;
  std::vector<uint64_t> keys((size_t)ne * 2);
  std::vector<uint8_t> keep(ne);
#pragma omp parallel for schedule(static)
  for (int64_t e = 0; e < ne; ++e) {
    uint32_t r[8][4];
    for (int b = 0; b < nblk; ++b)
      philox((uint32_t)e, (uint32_t)((uint64_t)e >> 32), (uint32_t)b, TAG_RMAT, (uint32_t)seed,
             (uint32_t)(seed >> 32), r[b]);
    uint64_t u = 0, v = 0;
    for (int i = 0; i < scale; ++i) {
      uint32_t x = r[i >> 2][i & 3];
      int bit = scale - 1 - i;
      uint64_t ub = 0, vb = 0;
      if (x < TH_A) { ub = 0; vb = 0; }
      else if (x < TH_AB) { ub = 0; vb = 1; }
      else if (x < TH_ABC) { ub = 1; vb = 0; }
      else { ub = 1; vb = 1; }
      u |= ub << bit;
      v |= vb << bit;
    }
    u = orc_scramble(u, scale, seed);
    v = orc_scramble(v, scale, seed);
    keep[e] = (u != v);
    keys[2 * e] = (u << 32) | v;
    keys[2 * e + 1] = (v << 32) | u;
  }
  // drop self loops
  size_t o = 0;
  for (int64_t e = 0; e < ne; ++e)
    if (keep[e]) { keys[o++] = keys[2 * e]; keys[o++] = keys[2 * e + 1]; }
  keys.resize(o);
  return csr_from_keys(n, keys, wseed);
}

extern "C" orc_graph* orc_grid(int W, int H, int diag, int cut_period, int perc_keep_ppm,
                               uint64_t perc_seed, uint64_t wseed) {
  if (W < 1 || H < 1) return nullptr;
  const int64_t n = (int64_t)W * H;
  std::vector<uint64_t> keys;
  keys.reserve((size_t)n * (diag ? 6 : 4));
  auto add = [&](int64_t a, int64_t b) {
    if (perc_keep_ppm < 1000000) {
      uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
      uint32_t r[4];
      philox((uint32_t)lo, (uint32_t)hi, 0, TAG_PERC, (uint32_t)perc_seed,
             (uint32_t)(perc_seed >> 32), r);
      if ((int)(r[0] % 1000000u) >= perc_keep_ppm) return;
    }
    keys.push_back(((uint64_t)a << 32) | (uint64_t)b);
    keys.push_back(((uint64_t)b << 32) | (uint64_t)a);
  };
  for (int64_t y = 0; y < H; ++y)
    for (int64_t x = 0; x < W; ++x) {
      int64_t id = y * W + x;
      if (x + 1 < W) add(id, id + 1);
      bool vcut = cut_period > 0 && (y % cut_period) == cut_period - 1;
      if (y + 1 < H && !vcut) add(id, id + W);
      if (diag && x + 1 < W && y + 1 < H && !vcut) add(id, id + W + 1);
    }
  return csr_from_keys(n, keys, wseed);
}

extern "C" orc_graph* orc_from_edges(int64_t n, int64_t m, const int64_t* u, const int64_t* v,
                                     const int32_t* w, int symmetrise, uint64_t wseed) {
  std::vector<uint64_t> keys;
  std::vector<std::pair<uint64_t, int32_t>> kw;
  for (int64_t i = 0; i < m; ++i) {
    if (u[i] < 0 || v[i] < 0 || u[i] >= n || v[i] >= n) return nullptr;
    if (u[i] == v[i]) continue;
    uint64_t k = ((uint64_t)u[i] << 32) | (uint64_t)v[i];
    int32_t ww = w ? w[i] : hash_weight(u[i], v[i], wseed);
    kw.push_back({k, ww});
    if (symmetrise) kw.push_back({((uint64_t)v[i] << 32) | (uint64_t)u[i], ww});
  }
  // dedupe keeping the minimum weight per directed pair
  std::sort(kw.begin(), kw.end());
  std::vector<int32_t> ws;
  for (size_t i = 0; i < kw.size(); ++i)
    if (i == 0 || kw[i].first != kw[i - 1].first) { keys.push_back(kw[i].first); ws.push_back(kw[i].second); }
  return csr_from_keys(n, keys, wseed, &ws);
}

extern "C" void orc_graph_free(orc_graph* g) { delete g; }
extern "C" int64_t orc_graph_n(const orc_graph* g) { return g->n; }
extern "C" int64_t orc_graph_m(const orc_graph* g) { return g->m; }
extern "C" const int64_t* orc_graph_row_ptr(const orc_graph* g) { return g->row_ptr.data(); }
extern "C" const int32_t* orc_graph_col(const orc_graph* g) { return g->col.data(); }
extern "C" const int32_t* orc_graph_weight(const orc_graph* g) { return g->w.data(); }

static uint64_t fnv(uint64_t h, const void* p, size_t bytes) {
  const uint8_t* b = (const uint8_t*)p;
  for (size_t i = 0; i < bytes; ++i) { h ^= b[i]; h *= 1099511628211ull; }
  return h;
}
extern "C" uint64_t orc_graph_checksum(const orc_graph* g) {
  uint64_t h = 1469598103934665603ull;
  h = fnv(h, g->row_ptr.data(), g->row_ptr.size() * 8);
  h = fnv(h, g->col.data(), g->col.size() * 4);
  h = fnv(h, g->w.data(), g->w.size() * 4);
  return h;
}

extern "C" int orc_pick_sources(const orc_graph* g, uint64_t seed, int count, int64_t* out) {
  int got = 0;
  for (int i = 0; i < count; ++i) {
    for (uint32_t att = 0; att < 1000000u; ++att) {
      uint32_t r[4];
      philox((uint32_t)i, att, 0, TAG_SRCS, (uint32_t)seed, (uint32_t)(seed >> 32), r);
      uint64_t x = (((uint64_t)r[1] << 32) | r[0]) % (uint64_t)g->n;
      if (g->row_ptr[x + 1] > g->row_ptr[x]) { out[got++] = (int64_t)x; break; }
    }
  }
  return got;
}

// ------------------------------------------------------------------------------------------
// Serial textbook algorithms.
extern "C" int64_t orc_bfs_serial(const orc_graph* g, int64_t src, int32_t* level) {
  for (int64_t i = 0; i < g->n; ++i) level[i] = ORC_INF;
  if (src < 0 || src >= g->n) return -1;
  std::vector<int32_t> q;
  q.reserve(g->n);
  q.push_back((int32_t)src);
  level[src] = 0;
  int64_t ecc = 0;
  for (size_t h = 0; h < q.size(); ++h) {
    int32_t u = q[h];
    for (int64_t e = g->row_ptr[u]; e < g->row_ptr[u + 1]; ++e) {
      int32_t v = g->col[e];
      if (level[v] == ORC_INF) {
        level[v] = level[u] + 1;
        if (level[v] > ecc) ecc = level[v];
        q.push_back(v);
      }
    }
  }
  return ecc;
}

extern "C" void orc_sssp_dijkstra(const orc_graph* g, int64_t src, int32_t* dist) {
  std::vector<int64_t> d(g->n, INT64_MAX);
  typedef std::pair<int64_t, int32_t> P;
  std::priority_queue<P, std::vector<P>, std::greater<P>> pq;
  d[src] = 0;
  pq.push({0, (int32_t)src});
  while (!pq.empty()) {
    P t = pq.top();
    pq.pop();
    if (t.first != d[t.second]) continue;
    int32_t u = t.second;
    for (int64_t e = g->row_ptr[u]; e < g->row_ptr[u + 1]; ++e) {
      int64_t nd = t.first + g->w[e];
      int32_t v = g->col[e];
      if (nd < d[v]) { d[v] = nd; pq.push({nd, v}); }
    }
  }
  for (int64_t i = 0; i < g->n; ++i) dist[i] = d[i] == INT64_MAX ? ORC_INF : (int32_t)d[i];
}

static int64_t uf_find(std::vector<int64_t>& p, int64_t x) {
  while (p[x] != x) { p[x] = p[p[x]]; x = p[x]; }
  return x;
}
extern "C" void orc_cc_unionfind(const orc_graph* g, int32_t* label) {
  std::vector<int64_t> p(g->n);
  for (int64_t i = 0; i < g->n; ++i) p[i] = i;
  for (int64_t u = 0; u < g->n; ++u)
    for (int64_t e = g->row_ptr[u]; e < g->row_ptr[u + 1]; ++e) {
      int64_t a = uf_find(p, u), b = uf_find(p, g->col[e]);
      if (a == b) continue;
      if (a < b) p[b] = a; else p[a] = b;  // root = minimum id of the merged set
    }
  for (int64_t i = 0; i < g->n; ++i) label[i] = (int32_t)uf_find(p, i);
}

// One Jacobi PageRank sweep; returns Any(|new-old| > tol) — the ReduceAndReturn of the
// topology-driven PR kernel.
static bool pr_sweep(const orc_graph* g, double d, double tol, const std::vector<double>& old,
                     std::vector<double>& contrib, std::vector<double>& nw) {
  const int64_t n = g->n;
#pragma omp parallel for schedule(static)
  for (int64_t u = 0; u < n; ++u) {
    int64_t deg = g->row_ptr[u + 1] - g->row_ptr[u];
    contrib[u] = deg > 0 ? old[u] / (double)deg : 0.0;
  }
  const double base = (1.0 - d) / (double)n;
  int any = 0;
#pragma omp parallel for schedule(dynamic, 1024) reduction(| : any)
  for (int64_t v = 0; v < n; ++v) {
    double s = 0.0;
    for (int64_t e = g->row_ptr[v]; e < g->row_ptr[v + 1]; ++e) s += contrib[g->col[e]];
    double r = base + d * s;
    nw[v] = r;
    if (std::abs(r - old[v]) > tol) any |= 1;
  }
  return any != 0;
}
extern "C" int orc_pagerank(const orc_graph* g, double d, double tol, int max_iter, double* rank) {
  const int64_t n = g->n;
  std::vector<double> a(n, 1.0 / (double)n), b(n), c(n);
  int it = 0;
  while (it < max_iter) {
    bool any = pr_sweep(g, d, tol, a, c, b);
    std::swap(a, b);
    ++it;
    if (!any) break;
  }
  std::memcpy(rank, a.data(), n * sizeof(double));
  return it;
}

// Degree-ordered orientation: u -> v iff (deg u, u) < (deg v, v).
static void orient(const orc_graph* g, std::vector<int64_t>& rp, std::vector<int32_t>& cl) {
  const int64_t n = g->n;
  auto deg = [&](int64_t x) { return g->row_ptr[x + 1] - g->row_ptr[x]; };
  auto less = [&](int64_t a, int64_t b) { return deg(a) < deg(b) || (deg(a) == deg(b) && a < b); };
  rp.assign(n + 1, 0);
  for (int64_t u = 0; u < n; ++u)
    for (int64_t e = g->row_ptr[u]; e < g->row_ptr[u + 1]; ++e)
      if (less(u, g->col[e])) rp[u + 1]++;
  for (int64_t u = 0; u < n; ++u) rp[u + 1] += rp[u];
  cl.resize(rp[n]);
  for (int64_t u = 0; u < n; ++u) {
    int64_t o = rp[u];
    for (int64_t e = g->row_ptr[u]; e < g->row_ptr[u + 1]; ++e)
      if (less(u, g->col[e])) cl[o++] = g->col[e];
  }
}
extern "C" uint64_t orc_tc_merge(const orc_graph* g) {
  std::vector<int64_t> rp;
  std::vector<int32_t> cl;
  orient(g, rp, cl);
  uint64_t total = 0;
#pragma omp parallel for schedule(dynamic, 256) reduction(+ : total)
  for (int64_t u = 0; u < g->n; ++u)
    for (int64_t e = rp[u]; e < rp[u + 1]; ++e) {
      int64_t v = cl[e];
      int64_t i = rp[u], ie = rp[u + 1], j = rp[v], je = rp[v + 1];
      while (i < ie && j < je) {
        if (cl[i] < cl[j]) ++i;
        else if (cl[i] > cl[j]) ++j;
        else { ++total; ++i; ++j; }
      }
    }
  return total;
}

extern "C" void orc_mst_kruskal(const orc_graph* g, uint64_t* weight, int64_t* nedges) {
  struct E { int32_t w, a, b; };
  std::vector<E> es;
  for (int64_t u = 0; u < g->n; ++u)
    for (int64_t e = g->row_ptr[u]; e < g->row_ptr[u + 1]; ++e)
      if (g->col[e] > u) es.push_back({g->w[e], (int32_t)u, g->col[e]});
  std::sort(es.begin(), es.end(), [](const E& x, const E& y) {
    return x.w != y.w ? x.w < y.w : (x.a != y.a ? x.a < y.a : x.b < y.b);
  });
  std::vector<int64_t> p(g->n);
  for (int64_t i = 0; i < g->n; ++i) p[i] = i;
  uint64_t tot = 0;
  int64_t cnt = 0;
  for (const E& e : es) {
    int64_t a = uf_find(p, e.a), b = uf_find(p, e.b);
    if (a == b) continue;
    if (a < b) p[b] = a; else p[a] = b;
    tot += (uint64_t)e.w;
    ++cnt;
  }
  *weight = tot;
  *nedges = cnt;
}

extern "C" void orc_exclusive(const int32_t* locks, int64_t nitems, int k, int32_t* won) {
  int32_t maxl = -1;
  for (int64_t i = 0; i < nitems * k; ++i) maxl = std::max(maxl, locks[i]);
  std::vector<int64_t> owner(maxl + 1, INT64_MAX);
  for (int64_t x = 0; x < nitems; ++x)  // claim: priority-min per lock slot
    for (int j = 0; j < k; ++j) {
      const int32_t l = locks[x * k + j];
      if (l >= 0) owner[l] = std::min<int64_t>(owner[l], x);
    }
  for (int64_t x = 0; x < nitems; ++x) {  // check / confirm
    bool all = true;
    for (int j = 0; j < k; ++j) {
      const int32_t l = locks[x * k + j];
      if (l >= 0 && owner[l] != x) all = false;
    }
    won[x] = all ? 1 : 0;
  }
}

// ------------------------------------------------------------------------------------------
// IrGL bulk-synchronous executor.
//
// Pipe context {in, out, retry}.  Each Worklist carries an epoch; a pop in
// launch epoch e only sees items present when e began — enforced structurally
// by popping from `in` and pushing to `out`/`retry`, and asserted in the test op PUSHPOP.
namespace {
struct Worklist {
  std::vector<int64_t> items;
  int64_t epoch = 0;
};
struct PipeCtx {
  Worklist in, out, retry;
  int64_t cap = 0;
  bool overflow = false;
};

// ForAll over the in-worklist: consecutive mapping, items split across OpenMP threads, each
// thread collects pushes/retries locally; merge order is thread order (items as a multiset are
// schedule-independent for every op below — SPEC.md:479).
struct Emit {
  std::vector<std::vector<int64_t>> push, retry;
  std::vector<int64_t> edges;
  explicit Emit(int T) : push(T), retry(T), edges(T, 0) {}
};

struct OpState {
  const orc_graph* g;
  const orc_iter_cfg* cfg;
  const int32_t* values;
  int64_t round;  // LEVEL / round counter (between_rounds: LEVEL++)
  std::vector<int32_t> lab;       // level / dist / label (atomically updated)
  std::vector<int64_t> stamp;     // per-round push dedupe for SSSP / CC_LP
  std::vector<int32_t> rcount;    // retry counts (TEST_RETRY_ODD)
  std::vector<int32_t> popped_at; // TEST_PUSHPOP: launch at which item was popped
  std::vector<double> rank_a, rank_b, contrib;
  uint64_t tc = 0;
  int64_t launch_no = 0;
  int64_t edges = 0;
};

static inline bool atomic_min32(int32_t* p, int32_t v) {
  int32_t cur = __atomic_load_n(p, __ATOMIC_RELAXED);
  while (v < cur)
    if (__atomic_compare_exchange_n(p, &cur, v, false, __ATOMIC_RELAXED, __ATOMIC_RELAXED))
      return true;
  return false;
}
static inline bool stamp_claim(int64_t* p, int64_t r) {
  return __atomic_exchange_n(p, r, __ATOMIC_RELAXED) != r;
}

// One launch of a worklist op over `in`; returns the Any/All fold (identity if no evaluation).
// Reduction fold per SPEC.md:444: Any = or, All = and, identities false/true.
static int launch_wl(OpState& st, PipeCtx& p, int reduction, bool serial) {
  const orc_graph* g = st.g;
  const int T = serial ? 1 : (st.cfg->threads > 0 ? st.cfg->threads : omp_get_max_threads());
  Emit em(T);
  const std::vector<int64_t>& in = p.in.items;
  const int64_t nin = (int64_t)in.size();
  int any = 0, all = 1;
  const int op = st.cfg->op;
  st.launch_no++;
#pragma omp parallel num_threads(T) reduction(| : any) reduction(& : all)
  {
    const int t = omp_get_thread_num();
    auto& push = em.push[t];
    auto& retry = em.retry[t];
    int64_t edges = 0;
#pragma omp for schedule(static)
    for (int64_t i = 0; i < nin; ++i) {
      const int64_t n = in[i];  // n = wl.pop(i)
      switch (op) {
        case ORC_OP_BFS: {  // Listing 2 with CAS dedupe
          for (int64_t e = g->row_ptr[n]; e < g->row_ptr[n + 1]; ++e) {
            ++edges;
            int32_t* dl = &st.lab[g->col[e]];
            int32_t expect = ORC_INF;
            if (__atomic_load_n(dl, __ATOMIC_RELAXED) == ORC_INF &&
                __atomic_compare_exchange_n(dl, &expect, (int32_t)st.round, false,
                                            __ATOMIC_RELAXED, __ATOMIC_RELAXED))
              push.push_back(g->col[e]);
          }
        } break;
        case ORC_OP_SSSP:
        case ORC_OP_CC_LP: {
          const int32_t dn = __atomic_load_n(&st.lab[n], __ATOMIC_RELAXED);
          for (int64_t e = g->row_ptr[n]; e < g->row_ptr[n + 1]; ++e) {
            ++edges;
            const int32_t v = g->col[e];
            const int32_t nd = op == ORC_OP_SSSP ? dn + g->w[e] : dn;
            if (nd < __atomic_load_n(&st.lab[v], __ATOMIC_RELAXED) && atomic_min32(&st.lab[v], nd) &&
                stamp_claim(&st.stamp[v], st.launch_no))
              push.push_back(v);
          }
        } break;
        case ORC_OP_TEST_COUNTDOWN:
          if (n + 1 < st.cfg->guard) push.push_back(n + 1);
          break;
        case ORC_OP_TEST_RETRY_ODD:
        case ORC_OP_TEST_RESPAWN_ODD:
          if ((n & 1) && st.rcount[n] < (st.cfg->guard > 0 ? st.cfg->guard : 1)) {
            st.rcount[n]++;
            retry.push_back(n);  // Retry n
          } else {
            push.push_back(n);
          }
          break;
        case ORC_OP_TEST_REDUCE: {
          const bool b = st.values[n] != 0;  // ReduceAndReturn(values[n]) ends this iteration
          any |= b;
          all &= b;
        } break;
        case ORC_OP_TEST_NOPUSH:
          break;
        case ORC_OP_TEST_PUSHPOP:
          if (n < (int64_t)st.popped_at.size()) st.popped_at[n] = (int32_t)st.launch_no;
          if (n + st.cfg->guard < p.cap) push.push_back(n + st.cfg->guard);
          break;
        default:
          break;
      }
    }
    em.edges[t] = edges;
  }
  for (int t = 0; t < T; ++t) {
    st.edges += em.edges[t];
    for (int64_t x : em.push[t]) p.out.items.push_back(x);
    for (int64_t x : em.retry[t]) p.retry.items.push_back(x);
  }
  if ((int64_t)p.out.items.size() > p.cap || (int64_t)p.retry.items.size() > p.cap) p.overflow = true;
  if (reduction == ORC_RED_ANY) return any;
  if (reduction == ORC_RED_ALL) return all;
  return -1;
}

// Topology-driven ops (no worklist): CC hook/compress, PR sweep, TC count.
static int launch_topo(OpState& st, int reduction) {
  const orc_graph* g = st.g;
  const int op = st.cfg->op;
  st.launch_no++;
  if (op == ORC_OP_CC) {
    // ECL-CC style hooking: CAS the larger root onto the smaller; then pointer-jump.
    int changed = 0;
    int32_t* par = st.lab.data();
    auto find = [&](int32_t x) {
      int32_t p = __atomic_load_n(&par[x], __ATOMIC_RELAXED);
      while (p != x) { x = p; p = __atomic_load_n(&par[x], __ATOMIC_RELAXED); }
      return x;
    };
#pragma omp parallel for schedule(dynamic, 1024) reduction(| : changed)
    for (int64_t u = 0; u < g->n; ++u)
      for (int64_t e = g->row_ptr[u]; e < g->row_ptr[u + 1]; ++e) {
        int32_t v = g->col[e];
        if (v > u) continue;  // each undirected edge once
        int32_t a = find((int32_t)u), b = find(v);
        while (a != b) {
          int32_t hi = a > b ? a : b, lo = a > b ? b : a;
          int32_t expect = hi;
          if (__atomic_compare_exchange_n(&par[hi], &expect, lo, false, __ATOMIC_RELAXED,
                                          __ATOMIC_RELAXED)) { changed = 1; break; }
          a = find(expect);
          b = find(lo);
        }
      }
#pragma omp parallel for schedule(static)
    for (int64_t u = 0; u < g->n; ++u) par[u] = find((int32_t)u);
    return reduction == ORC_RED_ALL ? !changed : changed;
  }
  if (op == ORC_OP_PR) {
    bool any = pr_sweep(g, st.cfg->pr_d, st.cfg->pr_tol, st.rank_a, st.contrib, st.rank_b);
    std::swap(st.rank_a, st.rank_b);
    return reduction == ORC_RED_ALL ? !any : any;
  }
  if (op == ORC_OP_TC) {
    st.tc = orc_tc_merge(g);
    return -1;
  }
  return -1;
}
}  // namespace

extern "C" int orc_reduce(const int32_t* values, int64_t n, int reduction) {
  int any = 0, all = 1;
  for (int64_t i = 0; i < n; ++i) { any |= values[i] != 0; all &= values[i] != 0; }
  return reduction == ORC_RED_ALL ? all : any;
}

extern "C" void orc_forall_assign(int64_t n, int64_t threads, int blocked, int64_t* thread_of) {
  if (!blocked) {
    for (int64_t i = 0; i < n; ++i) thread_of[i] = i % threads;  // for(i=tid;i<n;i+=T)
  } else {
    int64_t chunk = (n + threads - 1) / threads;  // ceil(N/T) contiguous iterations
    for (int64_t i = 0; i < n; ++i) thread_of[i] = chunk ? i / chunk : 0;
  }
}

static bool is_wl_op(int op) {
  return op == ORC_OP_BFS || op == ORC_OP_SSSP || op == ORC_OP_CC_LP || op >= 100;
}

extern "C" int orc_iterate(const orc_graph* g, const orc_iter_cfg* cfg, const int64_t* init,
                           int64_t ninit, int from_array, const int32_t* values, void* node_out,
                           orc_stats* stats, int64_t* trace, int64_t trace_cap, int64_t* final_in,
                           int64_t* final_in_len) {
  orc_stats s;
  std::memset(&s, 0, sizeof(s));
  s.last_reduced = -1;
  const int op = cfg->op;
  const int64_t n = g ? g->n : 0;
  PipeCtx p;
  p.cap = cfg->capacity > 0 ? cfg->capacity : (n > 0 ? n : 1);
  // WorklistInit (ast.hpp:100-110): Scalars or FromArray; size overflow is an error
  (void)from_array;
  if (ninit > p.cap) return -2;
  for (int64_t i = 0; i < ninit; ++i) p.in.items.push_back(init[i]);

  OpState st;
  st.g = g;
  st.cfg = cfg;
  st.values = values;
  st.round = cfg->round_start;
  if (op == ORC_OP_BFS || op == ORC_OP_SSSP) {
    st.lab.assign(n, ORC_INF);
    for (int64_t i = 0; i < ninit; ++i) st.lab[init[i]] = 0;  // level[src]=0 (App. B2)
  } else if (op == ORC_OP_CC || op == ORC_OP_CC_LP) {
    st.lab.resize(n);
    for (int64_t i = 0; i < n; ++i) st.lab[i] = (int32_t)i;
  } else if (op == ORC_OP_PR) {
    st.rank_a.assign(n, 1.0 / (double)n);
    st.rank_b.assign(n, 0.0);
    st.contrib.assign(n, 0.0);
  }
  if (op == ORC_OP_SSSP || op == ORC_OP_CC_LP) st.stamp.assign(n, 0);
  if (op == ORC_OP_TEST_RETRY_ODD) st.rcount.assign(p.cap, 0);
  if (op == ORC_OP_TEST_PUSHPOP) st.popped_at.assign(p.cap, 0);

  const bool wl = is_wl_op(op);
  const int rsa = cfg->retry_serialize_after > 0 ? cfg->retry_serialize_after : 4;
  int64_t ntr = 0;
  for (;;) {
    // termination test at round start: worklist emptiness combined with extra_cond
    // (SPEC.md:365); extra_cond here is "rounds >= max_rounds".
    const bool empty = wl && p.in.items.empty();
    const bool extra = cfg->max_rounds > 0 && s.rounds >= cfg->max_rounds;
    bool stop;
    if (cfg->max_rounds > 0)
      stop = cfg->extra_comb == ORC_COMB_AND ? (empty && extra) : (empty || extra);
    else
      stop = empty;
    if (stop) break;
    // ---- Invoke: run; while retry != {}: swap in<->retry, rerun (out kept); swap in<->out
    int red;
    if (wl) {
      red = launch_wl(st, p, cfg->reduction, false);
      s.launches++;
      s.popped += (int64_t)p.in.items.size();
      if (trace && ntr < trace_cap) {
        int64_t* t = trace + 4 * ntr++;
        t[0] = s.launches; t[1] = (int64_t)p.in.items.size();
        t[2] = (int64_t)p.out.items.size(); t[3] = (int64_t)p.retry.items.size();
      }
      int retry_rounds = 0;
      while (!p.retry.items.empty()) {
        std::swap(p.in, p.retry);
        p.retry.items.clear();
        p.in.epoch++;
        s.retries += (int64_t)p.in.items.size();
        ++retry_rounds;
        // Retry beyond retry_serialize_after rounds -> serial execution
        const bool serial = retry_rounds > rsa;
        if (serial) s.serial_launches++;
        int r2 = launch_wl(st, p, cfg->reduction, serial);
        if (cfg->reduction == ORC_RED_ANY) red = red | r2;
        if (cfg->reduction == ORC_RED_ALL) red = red & r2;
        s.launches++;
        s.popped += (int64_t)p.in.items.size();
        if (trace && ntr < trace_cap) {
          int64_t* t = trace + 4 * ntr++;
          t[0] = s.launches; t[1] = (int64_t)p.in.items.size();
          t[2] = (int64_t)p.out.items.size(); t[3] = (int64_t)p.retry.items.size();
        }
      }
      s.pushes += (int64_t)p.out.items.size();
      std::swap(p.in, p.out);
      p.out.items.clear();
      p.in.epoch++;
      p.out.epoch = p.in.epoch;
    } else {
      red = launch_topo(st, cfg->reduction);
      s.launches++;
    }
    if (p.overflow) return -2;
    s.rounds++;
    s.last_reduced = red;
    st.round++;  // between_rounds { LEVEL++ }
    // cond_kind (While|Until x Any|All) on the reduced return value
    if (cfg->cond_mode == ORC_COND_WHILE && red == 0) break;
    if (cfg->cond_mode == ORC_COND_UNTIL && red == 1) break;
    if (!wl && cfg->cond_mode == ORC_COND_NONE && cfg->max_rounds <= 0) break;  // plain Invoke
  }
  s.trace_len = (int32_t)ntr;
  s.edges = st.edges;
  if (node_out) {
    if (op == ORC_OP_PR) std::memcpy(node_out, st.rank_a.data(), n * sizeof(double));
    else if (op == ORC_OP_TC) *(uint64_t*)node_out = st.tc;
    else if (op == ORC_OP_TEST_PUSHPOP)
      std::memcpy(node_out, st.popped_at.data(), st.popped_at.size() * sizeof(int32_t));
    else if (!st.lab.empty()) std::memcpy(node_out, st.lab.data(), n * sizeof(int32_t));
  }
  if (final_in && final_in_len) {
    int64_t cap = *final_in_len;
    int64_t k = std::min<int64_t>(cap, (int64_t)p.in.items.size());
    for (int64_t i = 0; i < k; ++i) final_in[i] = p.in.items[i];
    *final_in_len = (int64_t)p.in.items.size();
  }
  if (stats) *stats = s;
  return 0;
}

// ------------------------------------------------------------------------------------------
// Multi-member Pipe: member statements over one pipe context (see oracle.h).  Each Invoke is the
// run_pipe swap protocol of orc_iterate: launch; while retry != {}: swap
// in<->retry, relaunch with out kept (serialised after retry_serialize_after rounds unless the
// operator uses Respawn); then swap in<->out.
extern "C" int orc_pipe_run(const orc_pipe_stage* stages, int n, int once, int64_t max_rounds,
                            int64_t cap, const int64_t* init, int64_t ninit, const int32_t* values,
                            int retry_serialize_after, int32_t* rcount, int32_t* log,
                            int32_t* stage_reduced, orc_stats* stats, int64_t* final_in,
                            int64_t* final_in_len) {
  if (!stages || n < 1 || cap < 1 || ninit > cap) return -1;
  orc_stats s;
  std::memset(&s, 0, sizeof(s));
  s.last_reduced = -1;
  PipeCtx p;
  p.cap = cap;
  for (int64_t i = 0; i < ninit; ++i) p.in.items.push_back(init[i]);
  OpState st;
  st.g = nullptr;
  st.values = values;
  st.round = 1;
  st.rcount.assign(cap, 0);
  st.popped_at.assign(cap, -1);
  const int rsa = retry_serialize_after > 0 ? retry_serialize_after : 4;
  std::vector<orc_iter_cfg> cfgs(n);
  for (int k = 0; k < n; ++k) {
    if (stages[k].op < ORC_OP_TEST_COUNTDOWN || stages[k].op > ORC_OP_TEST_RESPAWN_ODD ||
        stages[k].op == 105)
      return -1;
    std::memset(&cfgs[k], 0, sizeof(orc_iter_cfg));
    cfgs[k].op = stages[k].op;
    cfgs[k].reduction = stages[k].reduction;
    cfgs[k].guard = stages[k].guard;
    cfgs[k].threads = 1;  // one ordered thread: item order inside a worklist is immaterial
    if (stage_reduced) stage_reduced[k] = -1;
  }
  auto invoke = [&](int k) {
    const orc_iter_cfg& cfg = cfgs[k];
    st.cfg = &cfg;
    int red = launch_wl(st, p, cfg.reduction, false);
    s.launches++;
    s.popped += (int64_t)p.in.items.size();
    int retry_rounds = 0;
    while (!p.retry.items.empty()) {
      std::swap(p.in, p.retry);
      p.retry.items.clear();
      p.in.epoch++;
      s.retries += (int64_t)p.in.items.size();
      ++retry_rounds;
      const bool serial = cfg.op != ORC_OP_TEST_RESPAWN_ODD && retry_rounds > rsa;
      if (serial) s.serial_launches++;
      const int r2 = launch_wl(st, p, cfg.reduction, serial);
      if (cfg.reduction == ORC_RED_ANY) red = red | r2;
      if (cfg.reduction == ORC_RED_ALL) red = red & r2;
      s.launches++;
      s.popped += (int64_t)p.in.items.size();
    }
    s.pushes += (int64_t)p.out.items.size();
    std::swap(p.in, p.out);
    p.out.items.clear();
    p.in.epoch++;
    p.out.epoch = p.in.epoch;
    return cfg.reduction == ORC_RED_NONE ? -1 : red;
  };
  int prev = -1;
  int64_t passes = 0;
  for (;;) {
    if (!once && p.in.items.empty()) break;
    for (int k = 0; k < n; ++k) {
      const orc_pipe_stage& S = stages[k];
      if (S.when == 1 && prev != 1) continue;
      if (S.when == 2 && prev != 0) continue;
      for (int64_t it = 0;; ++it) {
        if (S.kind == 1 && (p.in.items.empty() || (S.max_rounds > 0 && it >= S.max_rounds))) break;
        prev = invoke(k);
        if (p.overflow) return -2;
        if (stage_reduced) stage_reduced[k] = prev;
        if (S.kind == 0) break;
        if (S.cond_mode == ORC_COND_WHILE && prev == 0) break;
        if (S.cond_mode == ORC_COND_UNTIL && prev == 1) break;
      }
    }
    ++passes;
    if (once || (max_rounds > 0 && passes >= max_rounds)) break;
  }
  s.rounds = passes;
  s.last_reduced = prev;
  if (rcount) std::memcpy(rcount, st.rcount.data(), cap * sizeof(int32_t));
  if (log) std::memcpy(log, st.popped_at.data(), cap * sizeof(int32_t));
  if (final_in && final_in_len) {
    const int64_t k = std::min<int64_t>(*final_in_len, (int64_t)p.in.items.size());
    for (int64_t i = 0; i < k; ++i) final_in[i] = p.in.items[i];
    *final_in_len = (int64_t)p.in.items.size();
  }
  if (stats) *stats = s;
  return 0;
}

// ------------------------------------------------------------------------------------------
// OpenMP bulk-synchronous BFS / SSSP — the timed CPU baseline.
extern "C" int orc_max_threads(void) { return omp_get_max_threads(); }
extern "C" void orc_set_threads(int t) { if (t > 0) omp_set_num_threads(t); }

extern "C" int64_t orc_bfs_bsp_omp(const orc_graph* g, int64_t src, int32_t* level, int threads,
                                   int64_t* edges_out) {
  const int T = threads > 0 ? threads : omp_get_max_threads();
  const int64_t n = g->n;
#pragma omp parallel for num_threads(T) schedule(static)
  for (int64_t i = 0; i < n; ++i) level[i] = ORC_INF;
  std::vector<int32_t> in, out;
  in.push_back((int32_t)src);
  level[src] = 0;
  int64_t rounds = 0, edges = 0;
  int32_t L = 1;
  std::vector<std::vector<int32_t>> loc(T);
  while (!in.empty()) {
    int64_t ed = 0;
#pragma omp parallel num_threads(T) reduction(+ : ed)
    {
      auto& mine = loc[omp_get_thread_num()];
      mine.clear();
#pragma omp for schedule(dynamic, 64)
      for (size_t i = 0; i < in.size(); ++i) {
        const int32_t u = in[i];
        const int64_t b = g->row_ptr[u], e = g->row_ptr[u + 1];
        ed += e - b;
        for (int64_t k = b; k < e; ++k) {
          int32_t v = g->col[k];
          int32_t expect = ORC_INF;
          if (__atomic_load_n(&level[v], __ATOMIC_RELAXED) == ORC_INF &&
              __atomic_compare_exchange_n(&level[v], &expect, L, false, __ATOMIC_RELAXED,
                                          __ATOMIC_RELAXED))
            mine.push_back(v);
        }
      }
    }
    edges += ed;
    out.clear();
    for (int t = 0; t < T; ++t) out.insert(out.end(), loc[t].begin(), loc[t].end());
    std::swap(in, out);
    ++rounds;
    ++L;
  }
  if (edges_out) *edges_out = edges;
  return rounds;
}

extern "C" int64_t orc_sssp_bsp_omp(const orc_graph* g, int64_t src, int32_t* dist, int threads,
                                    int64_t* edges_out) {
  const int T = threads > 0 ? threads : omp_get_max_threads();
  const int64_t n = g->n;
  std::vector<int64_t> stamp(n, 0);
#pragma omp parallel for num_threads(T) schedule(static)
  for (int64_t i = 0; i < n; ++i) dist[i] = ORC_INF;
  std::vector<int32_t> in, out;
  in.push_back((int32_t)src);
  dist[src] = 0;
  int64_t rounds = 0, edges = 0;
  std::vector<std::vector<int32_t>> loc(T);
  while (!in.empty()) {
    int64_t ed = 0;
    const int64_t r = rounds + 1;
#pragma omp parallel num_threads(T) reduction(+ : ed)
    {
      auto& mine = loc[omp_get_thread_num()];
      mine.clear();
#pragma omp for schedule(dynamic, 64)
      for (size_t i = 0; i < in.size(); ++i) {
        const int32_t u = in[i];
        const int32_t du = __atomic_load_n(&dist[u], __ATOMIC_RELAXED);
        const int64_t b = g->row_ptr[u], e = g->row_ptr[u + 1];
        ed += e - b;
        for (int64_t k = b; k < e; ++k) {
          const int32_t v = g->col[k];
          const int32_t nd = du + g->w[k];
          if (nd < __atomic_load_n(&dist[v], __ATOMIC_RELAXED) && atomic_min32(&dist[v], nd) &&
              stamp_claim(&stamp[v], r))
            mine.push_back(v);
        }
      }
    }
    edges += ed;
    out.clear();
    for (int t = 0; t < T; ++t) out.insert(out.end(), loc[t].begin(), loc[t].end());
    std::swap(in, out);
    ++rounds;
  }
  if (edges_out) *edges_out = edges;
  return rounds;
}

// Work-efficient CPU SSSP for the honest comparison the bench reports beside the IrGL-semantics
// executor (cpu_baseline.work_efficient): the same bulk-synchronous rounds, plus the GPU's
// degree-scaled deferral — a popped vertex with (dist - frontier min) * degree > K is kept for the
// next round instead of expanded (K = 1024, the GPU default) — so hubs expand near their final
// distance (scans per reached edge ~1.2 instead of ~2.8).  Same distances.
extern "C" int64_t orc_sssp_defer_omp(const orc_graph* g, int64_t src, int32_t* dist, int threads,
                                      int64_t defer_k, int64_t* edges_out) {
  const int T = threads > 0 ? threads : omp_get_max_threads();
  const int64_t n = g->n;
  std::vector<int64_t> stamp(n, 0);
#pragma omp parallel for num_threads(T) schedule(static)
  for (int64_t i = 0; i < n; ++i) dist[i] = ORC_INF;
  std::vector<int32_t> in, out;
  in.push_back((int32_t)src);
  dist[src] = 0;
  int64_t rounds = 0, edges = 0;
  int32_t dmin = 0;  // minimum distance in the current frontier
  std::vector<std::vector<int32_t>> loc(T);
  while (!in.empty()) {
    int64_t ed = 0;
    const int64_t r = rounds + 1;
    int32_t nmin = ORC_INF;
#pragma omp parallel num_threads(T) reduction(+ : ed) reduction(min : nmin)
    {
      auto& mine = loc[omp_get_thread_num()];
      mine.clear();
#pragma omp for schedule(dynamic, 64)
      for (size_t i = 0; i < in.size(); ++i) {
        const int32_t u = in[i];
        const int32_t du = __atomic_load_n(&dist[u], __ATOMIC_RELAXED);
        const int64_t b = g->row_ptr[u], e = g->row_ptr[u + 1];
        if (defer_k > 0 && rounds > 0 && ((int64_t)du - dmin) * (e - b) > defer_k) {
          if (stamp_claim(&stamp[u], r)) {  // kept for the next round
            mine.push_back(u);
            nmin = std::min(nmin, du);
          }
          continue;
        }
        ed += e - b;
        for (int64_t k = b; k < e; ++k) {
          const int32_t v = g->col[k];
          const int32_t nd = du + g->w[k];
          if (nd < __atomic_load_n(&dist[v], __ATOMIC_RELAXED) && atomic_min32(&dist[v], nd) &&
              stamp_claim(&stamp[v], r)) {
            mine.push_back(v);
            nmin = std::min(nmin, nd);
          }
        }
      }
    }
    edges += ed;
    out.clear();
    for (int t = 0; t < T; ++t) out.insert(out.end(), loc[t].begin(), loc[t].end());
    std::swap(in, out);
    dmin = nmin;
    ++rounds;
  }
  if (edges_out) *edges_out = edges;
  return rounds;
}

// ------------------------------------------------------------------------------------------
// Size-independent certificates for results too large for an oracle run (RMAT-27: 4.2G directed
// edges).  They take a borrowed CSR (e.g. downloaded from the device) and the result array and
// check the property that characterises the answer exactly on a symmetric graph with symmetric
// weights; return 0 when it holds, else a nonzero code naming the first violated clause.
//   BFS : level[src] = 0; every edge inside the reached set joins levels that differ by <= 1 and
//         no edge leaves it; every reached v != src has a neighbour at level[v] - 1  => hop
//         distance (Listing 2).
//   SSSP: dist[src] = 0; dist[v] <= dist[u] + w(u,v) on every edge of the reached set, none
//         leaves it; every reached v != src has a neighbour u with dist[u] + w(u,v) = dist[v]
//         => shortest-path distances.
extern "C" int orc_cert_bfs(int64_t n, const int64_t* rp, const int32_t* col, int64_t src,
                            const int32_t* level) {
  if (src < 0 || src >= n || level[src] != 0) return 1;
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(| : bad)
  for (int64_t u = 0; u < n; ++u) {
    const int32_t lu = level[u];
    bool parent = (u == src);
    for (int64_t k = rp[u]; k < rp[u + 1]; ++k) {
      const int32_t lv = level[col[k]];
      if ((lu == ORC_INF) != (lv == ORC_INF)) { bad |= 2; break; }
      if (lu == ORC_INF) continue;
      if (lv < lu - 1 || lv > lu + 1) bad |= 4;
      if (lv == lu - 1) parent = true;
    }
    if (lu != ORC_INF && !parent) bad |= 8;
  }
  return bad;
}

extern "C" int orc_cert_sssp(int64_t n, const int64_t* rp, const int32_t* col, const int32_t* w,
                             int64_t src, const int32_t* dist) {
  if (src < 0 || src >= n || dist[src] != 0) return 1;
  int bad = 0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(| : bad)
  for (int64_t u = 0; u < n; ++u) {
    const int64_t du = dist[u];
    bool parent = (u == src);
    for (int64_t k = rp[u]; k < rp[u + 1]; ++k) {
      const int64_t dv = dist[col[k]];
      if ((du == ORC_INF) != (dv == ORC_INF)) { bad |= 2; break; }
      if (du == ORC_INF) continue;
      if (dv > du + w[k]) bad |= 4;          // violated edge u -> v
      if (dv + w[k] == du) parent = true;    // tight edge into u (w symmetric)
    }
    if (du != ORC_INF && !parent) bad |= 8;
  }
  return bad;
}
