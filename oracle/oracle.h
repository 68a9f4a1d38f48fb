/*
 * oracle.h — CPU ORACLE for the IrGL worklist graph hot path.  TEST INFRASTRUCTURE ONLY.
 *
 * Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs may
 * load liboracle.so.  The product (paper_1607_05707_b200/) never links or calls it.
 *
 * What it restates (the reference ships no executable code for this path):
 *   - IrGL worklist/pipe semantics of the specified interpreter:
 *       worklist epochs
 *       launch_kernel distribution/reduction
 *       run_pipe swap protocol + retry
 *       orchestration (Iterate/Pipe/Invoke)
 *       reduction-cell identities
 *       worklist mechanics, Pipe, Iterate
 *       Listing 2 BFS
 *       ReduceAndReturn
 *   - serial textbook algorithms (queue BFS, Dijkstra, union-find CC, fp64 Jacobi PageRank,
 *     degree-ordered merge triangle counting) used as the parity checker for the GPU path.
 *   - the deterministic synthetic graph family (Philox-4x32-10 RMAT / grids) of SURVEY.md §8d.
 *
 * Parity pinning: the reference holds no fixtures; the only pins are the SPEC examples and
 * acceptance items.  tests/golden/ holds
 * them as fixtures and tests/test_oracle.py checks this oracle against every one.  SSSP, CC,
 * PageRank and TC are "parity unpinned by the reference" and are pinned
 * only by the builder-defined known answers of SURVEY.md Appendix C.
 */
#ifndef IRGL_ORACLE_H
#define IRGL_ORACLE_H
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define ORC_INF 2147483647 /* INF = max Int, mapped to INT32_MAX */

typedef struct orc_graph orc_graph;

/* ---- graphs ---------------------------------------------------------------------------- */
/* RMAT (Graph500 A/B/C/D = .57/.19/.19/.05), N = 2^scale, edge_factor*N generated edges,
 * seeded vertex scramble, self loops dropped, symmetrised, deduped, rows sorted.
 * Weights w(u,v) = 1 + philox(wseed; min(u,v), max(u,v)) % 255, symmetric. */
orc_graph* orc_rmat(int scale, int edge_factor, uint64_t seed, uint64_t wseed);
/* W x H grid, id = y*W + x.  diag: add (x,y)-(x+1,y+1).  cut_period>0: drop vertical edges
 * between rows r and r+1 when r % cut_period == cut_period-1.  perc_keep_ppm<1e6: keep each
 * undirected edge with probability perc_keep_ppm/1e6 by a philox hash of (perc_seed,u,v). */
orc_graph* orc_grid(int W, int H, int diag, int cut_period, int perc_keep_ppm, uint64_t perc_seed,
                    uint64_t wseed);
/* Build from an arbitrary directed edge list (u[i] -> v[i]); symmetrise=1 adds reverses.
 * Self loops dropped, deduped, sorted.  weight==NULL => hash weights with wseed. */
orc_graph* orc_from_edges(int64_t n, int64_t m, const int64_t* u, const int64_t* v,
                          const int32_t* w, int symmetrise, uint64_t wseed);
void orc_graph_free(orc_graph* g);
int64_t orc_graph_n(const orc_graph* g);
int64_t orc_graph_m(const orc_graph* g);
const int64_t* orc_graph_row_ptr(const orc_graph* g);
const int32_t* orc_graph_col(const orc_graph* g);
const int32_t* orc_graph_weight(const orc_graph* g);
/* FNV-1a-64 over row_ptr (as int64) then col then weight — the CSR fingerprint. */
uint64_t orc_graph_checksum(const orc_graph* g);
/* 16 sources uniform among non-isolated vertices, philox(seed; i, attempt). */
int orc_pick_sources(const orc_graph* g, uint64_t seed, int count, int64_t* out);
/* scramble bijection used by orc_rmat, exposed for tests */
uint64_t orc_scramble(uint64_t v, int scale, uint64_t seed);
void orc_philox4x32(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3, uint32_t k0, uint32_t k1,
                    uint32_t out[4]);

/* ---- serial textbook algorithms (the checker) ------------------------------------------ */
/* returns eccentricity(src) (max finite level); level[] INF for unreachable */
int64_t orc_bfs_serial(const orc_graph* g, int64_t src, int32_t* level);
void orc_sssp_dijkstra(const orc_graph* g, int64_t src, int32_t* dist);
void orc_cc_unionfind(const orc_graph* g, int32_t* label); /* label = min vertex id */
/* returns iterations executed.  d, tol absolute, max_iter cap; dangling mass dropped */
int orc_pagerank(const orc_graph* g, double d, double tol, int max_iter, double* rank);
uint64_t orc_tc_merge(const orc_graph* g);

/* MST forest by Kruskal (edges ordered by (w, min(u,v), max(u,v))): total weight and edge count
 * (SPEC.md:550 acceptance item 2 oracle for Boruvka, Listing 1). */
void orc_mst_kruskal(const orc_graph* g, uint64_t* weight, int64_t* nedges);
/* Exclusive protocol oracle: item x claims locks[x*k .. x*k+k)
 * (-1 = unused) with priority x (lower wins); x wins iff it holds every lock it claimed after the
 * claim phase.  won[x] = 1/0. */
void orc_exclusive(const int32_t* locks, int64_t nitems, int k, int32_t* won);

/* ---- IrGL bulk-synchronous worklist executor (restates SPEC.md:423-467) ----------------- */
enum { ORC_OP_BFS = 0, ORC_OP_SSSP = 1, ORC_OP_CC = 2, ORC_OP_PR = 3, ORC_OP_TC = 4,
       ORC_OP_CC_LP = 5,
       ORC_OP_TEST_COUNTDOWN = 100,   /* pop x; if x+1 < guard push x+1 */
       ORC_OP_TEST_RETRY_ODD = 101,   /* odd items retried once, then pushed */
       ORC_OP_TEST_REDUCE = 102,      /* ReduceAndReturn(values[x]) per item */
       ORC_OP_TEST_NOPUSH = 103,      /* pops, never pushes */
       ORC_OP_TEST_PUSHPOP = 104,     /* pushes x+guard, records what it popped */
       ORC_OP_TEST_RESPAWN_ODD = 106  /* RETRY_ODD through Respawn: never serialised */
};
enum { ORC_RED_NONE = 0, ORC_RED_ANY = 1, ORC_RED_ALL = 2 };
enum { ORC_COND_NONE = 0, ORC_COND_WHILE = 1, ORC_COND_UNTIL = 2 };
enum { ORC_COMB_OR = 0, ORC_COMB_AND = 1 };

typedef struct {
  int64_t rounds;          /* kernel invocations (launches, excluding retry re-launches) */
  int64_t launches;        /* including retry re-launches */
  int64_t popped;          /* items popped over all launches */
  int64_t pushes;          /* items pushed to out */
  int64_t retries;         /* items pushed to retry */
  int64_t edges;           /* edges scanned */
  int64_t serial_launches; /* retry launches run serialised (retry_serialize_after) */
  int32_t last_reduced;    /* last invocation's Any/All result (or -1) */
  int32_t trace_len;       /* entries written to trace */
} orc_stats;

typedef struct {
  int op;
  int reduction;      /* ORC_RED_* for the invocation's return cell */
  int cond_mode;      /* ORC_COND_* (While|Until) x reduction */
  int extra_comb;     /* ORC_COMB_* */
  int64_t max_rounds; /* extra_cond: exit when rounds >= max_rounds (0 = no extra cond) */
  int64_t round_start;/* BFS LEVEL start (between_rounds: LEVEL++) */
  int64_t guard;      /* test ops */
  int retry_serialize_after; /* default 4 */
  int threads;        /* OpenMP threads for the ForAll (0 = all); results are thread-independent */
  double pr_d, pr_tol;
  int64_t capacity;   /* WorklistInit.size; overflow -> return -2 */
} orc_iter_cfg;

/* Runs one standalone Iterate (PAPER.md:301 shape) with its own pipe context.
 * init/ninit: WorklistInit Scalars (or FromArray when from_array=1).
 * node_out: per-op result (int32 level/dist/label, double rank, uint64 count at [0]).
 * values: ORC_OP_TEST_REDUCE per-item bools.  trace (optional): per-launch log entries:
 *   [launch#, in_size, out_size_after, retry_size_after] x launches.
 * returns 0 or -2 (worklist overflow) / -1 (invalid). */
int orc_iterate(const orc_graph* g, const orc_iter_cfg* cfg, const int64_t* init, int64_t ninit,
                int from_array, const int32_t* values, void* node_out, orc_stats* stats,
                int64_t* trace, int64_t trace_cap, int64_t* final_in, int64_t* final_in_len);

/* Multi-member Pipe (ast.hpp:206-210): one pipe
 * context {in, out, retry} shared by the member statements, each an Invoke (kind 0) or an
 * Iterate (kind 1: until in is empty [Or rounds >= max_rounds], While|Until on the reduced value)
 * of a test operator; `when` guards a stage on the previous invocation's reduced value (0
 * always, 1 previous true, 2 previous false: dynamic piping, Listing 4).  Looping Pipe
 * (once = 0): repeat the body while `in` is non-empty at the start of a pass [at most max_rounds
 * passes]; Pipe Once: one pass.  rcount/log (cap entries, log initialised to -1 by the caller)
 * are the test operators' per-item state; stage_reduced[k] = last return value of stage k.
 * stats->rounds = passes.  Returns 0, -2 on worklist overflow, -1 on invalid input. */
typedef struct {
  int op, kind, reduction, when, cond_mode;
  int64_t max_rounds, guard;
} orc_pipe_stage;
int orc_pipe_run(const orc_pipe_stage* stages, int n, int once, int64_t max_rounds, int64_t cap,
                 const int64_t* init, int64_t ninit, const int32_t* values,
                 int retry_serialize_after, int32_t* rcount, int32_t* log, int32_t* stage_reduced,
                 orc_stats* stats, int64_t* final_in, int64_t* final_in_len);

/* Invoke once (no loop) of a non-worklist reduce kernel over `n` items: the ReduceAndReturn
 * fold with identities Any->0, All->1. */
int orc_reduce(const int32_t* values, int64_t n, int reduction);

/* ForAll distribution: thread_of[i] for n iterations over T threads. */
void orc_forall_assign(int64_t n, int64_t threads, int blocked, int64_t* thread_of);

/* OpenMP bulk-synchronous BFS / SSSP (the timed CPU baseline).
 * returns rounds; edges_out = directed edges scanned. */
int64_t orc_bfs_bsp_omp(const orc_graph* g, int64_t src, int32_t* level, int threads,
                        int64_t* edges_out);
int64_t orc_sssp_bsp_omp(const orc_graph* g, int64_t src, int32_t* dist, int threads,
                         int64_t* edges_out);
int orc_max_threads(void);
/* Work-efficient variant of the OpenMP executor (the GPU's degree-scaled deferral, budget
 * defer_k): the bench's cpu_baseline.work_efficient figure.  Same distances. */
int64_t orc_sssp_defer_omp(const orc_graph* g, int64_t src, int32_t* dist, int threads,
                           int64_t defer_k, int64_t* edges_out);
void orc_set_threads(int t); /* omp_set_num_threads (torchrun exports OMP_NUM_THREADS=1) */

/* Certificates over a borrowed CSR (symmetric graph, symmetric weights); 0 = holds, else a bit
 * mask of the violated clauses (1 source, 2 edge leaves the reached set, 4 edge inequality,
 * 8 reached vertex without a tight parent).  For sizes no oracle run finishes (RMAT-27). */
int orc_cert_bfs(int64_t n, const int64_t* rp, const int32_t* col, int64_t src,
                 const int32_t* level);
int orc_cert_sssp(int64_t n, const int64_t* rp, const int32_t* col, const int32_t* w, int64_t src,
                  const int32_t* dist);

#ifdef __cplusplus
}
#endif
#endif
