/*
 * irgl/rt.h — C-ABI of the B200-native IrGL worklist graph runtime (libirgl_rt.so).
 *
 * This is the drop-in boundary for the hot path of arXiv 1607.05707 ("Lowering IrGL to CUDA"):
 * worklist-driven irregular graph operators over CSR behind IrGL's operator API.  The reference
 * ships the operator vocabulary as an AST (reference/proj/core/include/irgl/ast.hpp:97-233) and
 * specifies — but does not ship — its executors:
 *   run_host(module, entry, bindings, config)
 *   launch_kernel(kernel, args, pipe_state, config)
 *   run_pipe(pipe_stmt, machine, config)
 *   lower_orchestration / outline_pipe
 * Each entry point below names the construct it replaces.  Plain pointers and sizes only; no
 * torch or CUDA types cross the boundary.
 *
 * Conventions (kept from the reference):
 *   - errors are values: every call returns irgl_status_t and never throws or aborts
 *     (reference diag.hpp:20-27); irgl_last_error() gives "RULE: message";
 *   - single-threaded orchestration: one host thread per irgl_ctx;
 *   - INF is INT32_MAX in int32 storage;
 *   - work items cross the ABI as int64 and are stored as uint32 on the device;
 *     ids >= 2^32 are rejected with IRGL_E_INVALID.
 * Ownership: host arrays are borrowed for the duration of a call and copied; handles own their
 * device memory; *_destroy frees it; results are copied into caller buffers.
 */
#ifndef IRGL_RT_H
#define IRGL_RT_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

#define IRGL_ABI_VERSION 1
#define IRGL_INF 2147483647

typedef int32_t irgl_status_t;
enum {
  IRGL_OK = 0,
  IRGL_E_INVALID = 1,        /* bad argument / id out of range                                */
  IRGL_E_USAGE = 2,          /* API misuse (wrong handle, op needs a graph / a pipe, ...)      */
  IRGL_E_OOM = 3,            /* device allocation failed                                       */
  IRGL_E_WL_OVERFLOW = 4,    /* worklist initialiser / push beyond WorklistInit.size */
  IRGL_E_OCCUPANCY = 5,      /* barrier launch > co-resident threads  */
  IRGL_E_OUTLINE_EMPTY = 6,  /* T_control = empty set                     */
  IRGL_E_CUDA = 7,           /* CUDA runtime error (message in irgl_last_error)                */
  IRGL_E_NCCL = 8,           /* NCCL error / async error                                       */
  IRGL_E_UNSUPPORTED = 9,    /* combination not supported by this build                        */
  IRGL_E_RANGE = 10          /* an SSSP path weight sum reaches INF = INT32_MAX: distances are
                                int32 (SPEC.md:421's Int narrowed); the traversal is not valid  */
};

/* ast.hpp:90 Reduction {Any, All}; NONE = invocation without a return cell. */
typedef enum { IRGL_RED_NONE = 0, IRGL_RED_ANY = 1, IRGL_RED_ALL = 2 } irgl_reduction;
/* PAPER.md:363 pipe context worklists in / out / retry. */
typedef enum { IRGL_WL_IN = 0, IRGL_WL_OUT = 1, IRGL_WL_RETRY = 2 } irgl_wl;
/* ast.hpp:193 IterateCond {While|Until}; NONE = no reduction condition. */
typedef enum { IRGL_COND_NONE = 0, IRGL_COND_WHILE = 1, IRGL_COND_UNTIL = 2 } irgl_cond_mode;
/* ast.hpp:91 CondCombiner {And, Or} for ExtraCond. */
typedef enum { IRGL_COMB_OR = 0, IRGL_COMB_AND = 1 } irgl_combiner;
/* ast.hpp:89 ForAllMapping {Consecutive, Blocked}. */
typedef enum { IRGL_MAP_CONSECUTIVE = 0, IRGL_MAP_BLOCKED = 1 } irgl_mapping;

/* The plain (device) kernels this runtime implements — the north-star operators in IrGL form
 * plus the tiny operators the SPEC's own examples are phrased in. */
typedef enum {
  IRGL_OP_BFS = 0,   /* Listing 2: level[dst]==INF -> level=LEVEL; push */
  IRGL_OP_SSSP = 1,  /* data-driven Bellman-Ford: atomicMin(dist[dst], dist[n]+w) < old -> push */
  IRGL_OP_CC = 2,    /* topology-driven hook (CAS larger root onto smaller) + pointer jumping,
                        Iterate While Any; labels = min vertex id per component          */
  IRGL_OP_PR = 3,    /* topology-driven pull Jacobi PageRank, fp64, ReduceAndReturn(|d|>tol) */
  IRGL_OP_TC = 4,    /* degree-oriented intersection triangle count (Sum: extension, App. B6) */
  IRGL_OP_CC_LP = 5, /* data-driven min-label propagation (worklist form of CC)              */
  IRGL_OP_MST = 6,   /* Boruvka minimum spanning forest, Listing 1: find-min
                        edge per component under Atomic, hook + pointer jumping, Iterate While
                        Any; result uint64[2] = {forest weight, forest edges} */
  /* SPEC example operators (tests): */
  IRGL_OP_TEST_COUNTDOWN = 100, /* pop x; if x+1 < guard: push x+1 */
  IRGL_OP_TEST_RETRY_ODD = 101, /* odd x retried `guard` times, then pushed */
  IRGL_OP_TEST_REDUCE = 102,    /* ReduceAndReturn(values[x]) */
  IRGL_OP_TEST_NOPUSH = 103,    /* pops, never pushes */
  IRGL_OP_TEST_PUSHPOP = 104,   /* records popped_at[x]=launch; push x+guard */
  IRGL_OP_TEST_FORALL_MAP = 105, /* records thread_of[x] = global thread id */
  IRGL_OP_TEST_RESPAWN_ODD = 106, /* as RETRY_ODD with Respawn: never serialised */
  IRGL_OP_TEST_ATOMIC = 107,      /* blocking Atomic increment of one counter */
  IRGL_OP_TEST_ATOMIC_ELSE = 108, /* Atomic/Else single attempt; guard=1: lock held SPEC.md:551 */
  IRGL_OP_TEST_EXCLUSIVE = 109    /* Exclusive over values[x*guard..] lock sets */
} irgl_op;

typedef struct irgl_ctx irgl_ctx;
typedef struct irgl_graph irgl_graph;
typedef struct irgl_pipe irgl_pipe;

/* Runtime configuration (the reference's SimConfig / CLI flags). */
typedef struct irgl_config {
  int32_t outline;               /* default for irgl_iterate: 0 host loop, 1 outlined, -1 auto */
  int32_t blocks_per_sm;         /* FixedFromSM multiplier; 0 = occupancy    */
  int32_t retry_serialize_after; /* Retry conflict management; 0 -> 4          */
  int32_t warp_threshold;        /* degree >= -> edge chunks drained by every warp of the grid
                                    (edge-balanced); below: the warp tile's fine-grained gather;
                                    0 -> 128                                                    */
  int32_t cta_threshold;         /* rounds with at most one tile per warp: degrees below this are
                                    expanded by the popping warp (no chunk phase); 0 -> 256      */
  int32_t chunk_edges;           /* edges per chunk descriptor (<= 65535); 0 -> 512            */
  int32_t l2_persist;            /* 1: L2 persisting access-policy window on the array the outlined
                                    kernels gather per edge (labels / distances, BFS visited
                                    bitmap), sized to the device set-aside                      */
  int32_t logical_partitions;    /* >1: P vertex partitions inside this ctx (loopback exchange) */
  int32_t dense_div;             /* outlined rounds whose frontier has >= n/dense_div vertices run
                                    dense: relaxations mark (fire-and-forget stores / REDs) and a
                                    compaction sweep builds the out worklist; 0 -> 32, <0 off    */
  int32_t bfs_bitmap_min_n;      /* BFS tracks visited vertices in an n-bit bitmap (L2-resident)
                                    when n >= this: 0 -> 12M (level array > 48 MB), or always
                                    for a relabelled graph; <0 never                             */
  int32_t reserved[6];
} irgl_config;

/* Kernel arguments (the Invoke/Iterate `args`). */
typedef struct irgl_op_args {
  int64_t round_start;   /* value of the round counter (LEVEL) at the first invocation; 0 -> 1 */
  int64_t guard;         /* test operators                                                   */
  double pr_damping;     /* 0 -> 0.85                                                          */
  double pr_tol;         /* 0 -> 1e-6 (absolute, per vertex)                                   */
  const int32_t* values; /* IRGL_OP_TEST_REDUCE: per-item booleans (copied)                   */
  int64_t nvalues;
  int32_t mapping;       /* irgl_mapping of the outer ForAll (test operators)                  */
  int32_t threads;       /* test operators: total CUDA threads (0 = planner's choice)          */
  int32_t delta;         /* SSSP: near-far bucket width; 0 = plain data-driven Bellman-Ford,
                            <0 = runtime default.  Same distances either way.                 */
  int32_t direction;     /* BFS: 0 = top-down worklist (Listing 2); 1 = direction-optimising
                            (bottom-up rounds when the frontier is large; outlined, 1 partition;
                            SURVEY §8f F1).  Same levels either way.                          */
  int32_t defer;         /* SSSP: degree-scaled deferral budget K.  A popped vertex v with
                            (dist[v] - min dist of the frontier) * deg(v) > K is re-pushed
                            (kept for the next round) instead of expanded, so hubs expand close
                            to their final distance.  0 = off, <0 = runtime default.  Same
                            distances either way (only the relaxation order changes).        */
  int32_t reserved[3];
} irgl_op_args;

/* Iterate [While|Until Any|All] kernel(args) [ExtraCond] (ast.hpp:186-204). */
typedef struct irgl_iterate_opts {
  int32_t cond_mode;   /* irgl_cond_mode                                                      */
  int32_t reduction;   /* irgl_reduction of the cond (and the invocation's return cell)        */
  int32_t extra_comb;  /* irgl_combiner joining ExtraCond with the empty-worklist test         */
  int32_t outline;     /* -1 ctx default, 0 host-orchestrated, 1 outlined persistent kernel    */
  int64_t max_rounds;  /* ExtraCond: exit when rounds >= max_rounds (0 = none)                 */
  int32_t reset;       /* 1: (re)initialise the operator's node state from the pipe first      */
  int32_t reserved[5];
} irgl_iterate_opts;

typedef struct irgl_iter_stats {
  int64_t rounds;          /* invocations (between_rounds executions)                          */
  int64_t launches;        /* kernel launches incl. retry relaunches (outlined: 1)             */
  int64_t popped;          /* items popped                                                     */
  int64_t pushes;          /* items pushed to out (local + remote-applied)                     */
  int64_t retries;         /* items routed through the retry worklist                          */
  int64_t edges;           /* directed edges scanned                                           */
  int64_t remote_updates;  /* updates sent to other partitions                                 */
  int64_t exchange_bytes;  /* bytes moved between partitions                                   */
  int64_t serial_launches; /* retry launches executed serialised                               */
  int32_t last_reduced;    /* last invocation's Any/All value, -1 if none                      */
  int32_t outlined;        /* 1 if the loop ran as one persistent kernel                       */
  double device_ms;        /* CUDA-event time of the whole iterate on the ctx stream           */
  double kernel_ms;        /* CUDA-event time of the hot kernels (expand/chunk or persistent)  */
} irgl_iter_stats;

/* Device graph generator (§8d synthetic inputs). */
typedef enum { IRGL_GEN_RMAT = 0, IRGL_GEN_GRID = 1 } irgl_gen_kind;
typedef struct irgl_gen_spec {
  int32_t kind;          /* irgl_gen_kind                                                       */
  int32_t scale;         /* RMAT: N = 2^scale                                                   */
  int32_t edge_factor;   /* RMAT: 16                                                            */
  int32_t width, height; /* GRID                                                                */
  int32_t diag;          /* GRID: add (x,y)-(x+1,y+1)                                           */
  int32_t cut_period;    /* GRID: cut vertical edges between rows r,r+1 when r%p == p-1         */
  int32_t perc_keep_ppm; /* GRID: keep probability in ppm (1000000 = all)                       */
  uint64_t seed;         /* RMAT graph seed                                                     */
  uint64_t wseed;        /* weight seed (11)                                                    */
  uint64_t perc_seed;    /* GRID percolation seed (5)                                           */
  int32_t reserved[8];
} irgl_gen_spec;

typedef struct irgl_graph_info {
  int64_t n, m;                 /* global vertices / directed edges                            */
  int64_t local_n, local_m;     /* this process's partition(s)                                 */
  int64_t lo, hi;               /* owned vertex range of the first local partition             */
  int32_t partitions;           /* total partitions                                            */
  int32_t has_weights;
  int64_t max_degree;
} irgl_graph_info;

/* ---- context ------------------------------------------------------------------------------ */
/* Single process.  ndev devices; the graph is split into max(ndev, cfg->logical_partitions)
 * vertex partitions, partition p on devices[p % ndev]. */
irgl_status_t irgl_ctx_create(const int* devices, int ndev, const irgl_config* cfg, irgl_ctx** out);
/* One process per GPU (torchrun): rank `rank` of `nranks`, NCCL unique id from rank 0. */
irgl_status_t irgl_nccl_unique_id(void* id128);
irgl_status_t irgl_ctx_create_nccl(int device, int rank, int nranks, const void* id128,
                                   const irgl_config* cfg, irgl_ctx** out);
/* One process per GPU without NCCL: the round headers and payloads of a vertex-partitioned
 * graph go through the caller's collectives (e.g. an MPI communicator or a torch.distributed
 * gloo group), staged in pinned host memory.  Every rank calls the same runtime functions in the
 * same order, so the callbacks are invoked collectively.  Return 0 on success. */
typedef struct irgl_transport {
  void* user;
  /* every rank contributes `bytes` bytes at send; recv receives nranks * bytes in rank order */
  int32_t (*allgather)(void* user, const void* send, void* recv, size_t bytes);
  /* all-to-all-v of byte blocks: send holds send_bytes[r] bytes for each rank r back to back in
   * rank order, recv receives recv_bytes[r] bytes from each rank r likewise */
  int32_t (*alltoallv)(void* user, const void* send, const int64_t* send_bytes, void* recv,
                       const int64_t* recv_bytes);
} irgl_transport;
irgl_status_t irgl_ctx_create_transport(int device, int rank, int nranks, const irgl_transport* t,
                                        const irgl_config* cfg, irgl_ctx** out);
irgl_status_t irgl_ctx_destroy(irgl_ctx* ctx);
irgl_status_t irgl_ctx_sync(irgl_ctx* ctx);
const char* irgl_last_error(const irgl_ctx* ctx); /* ctx may be NULL: last global error */
int irgl_abi_version(void);

/* ---- graph (reference Value::Graph; builtins edges/dst/weight) ----- */
/* Column ids must be in [0, n) and weights >= 0 (IRGL_E_INVALID otherwise); distances are int32:
 * an SSSP in which a vertex's shortest-path weight reaches INT32_MAX (= INF) returns IRGL_E_RANGE
 * (every relaxation sum is range-checked; a sum beyond the range into an unreached vertex triggers
 * an exact check of the finished distances on one partition — conservatively reported on several
 * partitions and inside irgl_traverse_batch).  Never a wrapped distance. */
irgl_status_t irgl_graph_create_csr(irgl_ctx* ctx, int64_t n, int64_t m, const int64_t* row_ptr,
                                    const int32_t* col, const int32_t* weight /*nullable*/,
                                    irgl_graph** out);
irgl_status_t irgl_graph_generate(irgl_ctx* ctx, const irgl_gen_spec* spec, irgl_graph** out);
/* Text edge list: first line "N M", then M lines "u v [w]" (0-based ids, w >= 0;
 * '#' and blank lines ignored).  symmetrise=1 adds reverse edges; self loops dropped, duplicates merged
 * (minimum weight); missing weights = 1.  The CSR is built on the device (sort + unique). */
irgl_status_t irgl_graph_read_edgelist(irgl_ctx* ctx, const char* path, int symmetrise,
                                       irgl_graph** out);
irgl_status_t irgl_graph_info_get(const irgl_graph* g, irgl_graph_info* info);
/* Degree-ordered relabelling of a one-partition graph (data layout: hubs get the smallest ids,
 * so the per-vertex state gathered most often shares cache lines; RMAT-24 BFS 1.30x, SSSP 1.44x).
 * The permutation stays inside the runtime: worklist items, results and worklist reads keep the
 * caller's ids; CC labels stay the smallest original id of each component.  After it,
 * irgl_graph_download returns the relabelled CSR and irgl_graph_perm gives new_of_old[n]. */
irgl_status_t irgl_graph_relabel(irgl_ctx* ctx, irgl_graph* g);
irgl_status_t irgl_graph_perm(irgl_graph* g, int32_t* new_of_old);
/* Copies the CSR of the local partitions back (single-process: the whole graph). */
irgl_status_t irgl_graph_download(irgl_graph* g, int64_t* row_ptr, int32_t* col, int32_t* weight);
irgl_status_t irgl_graph_destroy(irgl_graph* g);

/* ---- pipe context {in, out, retry} ------------------------ */
irgl_status_t irgl_pipe_create(irgl_ctx* ctx, int64_t capacity /*WorklistInit.size*/,
                               irgl_pipe** out);
/* WorklistInit Scalars (ast.hpp:101) / FromArray (ast.hpp:104).  With a graph of P>1
 * partitions each item is routed to its owner partition. */
irgl_status_t irgl_pipe_init_scalars(irgl_pipe* p, const int64_t* items, int64_t count);
irgl_status_t irgl_pipe_init_from_array(irgl_pipe* p, const int64_t* arr, int64_t len);
irgl_status_t irgl_pipe_init_range(irgl_pipe* p, int64_t begin, int64_t end); /* iota */
irgl_status_t irgl_pipe_size(const irgl_pipe* p, irgl_wl which, int64_t* out);
irgl_status_t irgl_pipe_read(irgl_pipe* p, irgl_wl which, int64_t* items, int64_t cap,
                             int64_t* count);
irgl_status_t irgl_pipe_destroy(irgl_pipe* p);

/* ---- operator state -------------------------------------------------------------------------- */
/* Initialise node properties for `op` (level/dist = INF except the pipe's in-items = 0; CC label
 * = id; PR rank = 1/N).  pipe may be NULL for topology-driven operators. */
irgl_status_t irgl_op_reset(irgl_ctx* ctx, irgl_graph* g, irgl_op op, const irgl_op_args* args,
                            irgl_pipe* pipe);

/* ---- orchestration ------------------------------------------------------------------------- */
/* [Any|All(] Invoke kernel(args) [)] — PAPER.md:88-90: launch; while retry is
 * non-empty swap in<->retry and relaunch (out kept); then swap in<->out and clear out.
 * `reduced` receives the return cell (identity Any->0, All->1 when nothing was evaluated). */
irgl_status_t irgl_invoke(irgl_ctx* ctx, irgl_pipe* pipe /*NULL: non-worklist op*/, irgl_graph* g,
                          irgl_op op, const irgl_op_args* args, irgl_reduction red,
                          int32_t* reduced /*nullable*/, irgl_iter_stats* stats /*nullable*/);
/* Iterate ...: repeat Invoke until `in` is empty (worklist
 * ops) combined with cond/extra_cond; between_rounds = round counter ++.  outline=1 runs the
 * whole loop as one cooperative persistent kernel with a grid barrier (SyncRunningThreads). */
irgl_status_t irgl_iterate(irgl_ctx* ctx, irgl_pipe* pipe, irgl_graph* g, irgl_op op,
                           const irgl_op_args* args, const irgl_iterate_opts* opts,
                           irgl_iter_stats* stats);
/* Copies the operator's node result to the host: BFS/SSSP/CC/CC_LP int32[n], PR double[n],
 * TC uint64[1]; test ops: PUSHPOP/FORALL_MAP int32[capacity] (g may be NULL). */
irgl_status_t irgl_read_result(irgl_ctx* ctx, irgl_graph* g, irgl_op op, void* host_out,
                               size_t bytes);

/* Asynchronous variant for pipelined queries: the copy of the node result (BFS/SSSP/CC/CC_LP
 * int32[n]) into host_out (pinned memory to overlap) is queued on a copy stream behind the work
 * already issued and the call returns at once; the next traversal on the graph writes a second
 * label buffer, so it overlaps the copy.  host_out is valid after irgl_results_wait.  Other
 * operators fall back to irgl_read_result. */
irgl_status_t irgl_read_result_async(irgl_ctx* ctx, irgl_graph* g, irgl_op op, void* host_out,
                                     size_t bytes);
irgl_status_t irgl_results_wait(irgl_ctx* ctx);

/* A batch of single-source queries in one call (the serving loop without per-query host-language
 * overhead): for each i < k, Initial [sources[i]] -> irgl_iterate(op, args, opts) -> stats[i]
 * (may be NULL), and when host_out is non-NULL the node result is queued into host_out[i] with
 * irgl_read_result_async (pointers may repeat; copies land in issue order) and the call returns
 * after irgl_results_wait.  Same results as the k separate calls. */
irgl_status_t irgl_traverse_batch(irgl_ctx* ctx, irgl_pipe* pipe, irgl_graph* g, irgl_op op,
                                  const int64_t* sources, int32_t k, const irgl_op_args* args,
                                  const irgl_iterate_opts* opts, void* const* host_out,
                                  size_t bytes, irgl_iter_stats* stats);

/* ---- measurement --------------------------------------------------------------------------- */
/* CUDA events on the stream of the ctx's first partition (the stream every kernel of this ctx is
 * ordered on), slots 0..7; elapsed time between two recorded slots in ms. */
irgl_status_t irgl_event_record(irgl_ctx* ctx, int slot);
irgl_status_t irgl_event_elapsed(irgl_ctx* ctx, int slot_a, int slot_b, double* ms);
/* Process-wide count of kernels this library has launched (all ctxs). */
int64_t irgl_launch_count(void);

/* ---- launch planning ------------------------------------------------------ */
/* Block-size constraint of a kernel: Elastic [1,1024], Shrinkable(max) [1,max], Fixed(n) {n}. */
typedef enum { IRGL_BLOCK_ELASTIC = 0, IRGL_BLOCK_SHRINKABLE = 1, IRGL_BLOCK_FIXED = 2 } irgl_block_kind;
typedef struct irgl_block_constraint { int32_t kind; int32_t value; } irgl_block_constraint;
/* T_control = max(intersection of domains).  IRGL_E_OUTLINE_EMPTY if empty. */
irgl_status_t irgl_t_control(const irgl_block_constraint* cs, int n, int32_t* out);
/* The block constraint of this build's kernel for `op` (Fixed(512) for the nested-parallelism
 * kernels) and the co-resident grid of its outlined variant. */
irgl_status_t irgl_op_plan(irgl_ctx* ctx, irgl_op op, irgl_block_constraint* block,
                           int32_t* grid_outlined, int32_t* grid_fixed);

/* ---- multi-member Pipe (ast.hpp:206-210) -------- */
/* A Pipe body as a list of member statements over the pipe's shared {in, out, retry}: each stage
 * is an Invoke or an Iterate of one operator; a stage may be guarded by the previous stage's
 * reduced return value (dynamic piping, Listing 4).  Looping Pipe: the body repeats
 * while `in` is non-empty at the start of a pass; Pipe Once: one pass. */
typedef enum { IRGL_STAGE_INVOKE = 0, IRGL_STAGE_ITERATE = 1 } irgl_stage_kind;
typedef enum { IRGL_WHEN_ALWAYS = 0, IRGL_WHEN_PREV_TRUE = 1, IRGL_WHEN_PREV_FALSE = 2 } irgl_stage_when;
typedef struct irgl_pipe_stage {
  int32_t op;         /* member kernel (irgl_op)                                                 */
  int32_t kind;       /* irgl_stage_kind                                                         */
  int32_t reduction;  /* Any|All return cell of each invocation                                  */
  int32_t when;       /* irgl_stage_when                                                         */
  int32_t cond_mode;  /* Iterate stage: While|Until on the reduced value                         */
  int32_t reserved0;
  int64_t max_rounds; /* Iterate stage: ExtraCond rounds >= max_rounds (Or)                     */
  irgl_block_constraint block; /* the member kernel's block-size domain      */
  irgl_op_args args;
} irgl_pipe_stage;
typedef struct irgl_pipe_opts {
  int32_t once;       /* 1: Pipe Once                                                            */
  int32_t outline;    /* 1: one cooperative control kernel launched at T_control (error
                         IRGL_E_OUTLINE_EMPTY when the members' domains do not intersect, or
                         IRGL_E_UNSUPPORTED for members without a device body on that path);
                         0: host-orchestrated; -1: outlined when possible, else host (the SPEC's
                         fallback "with a warning")                                */
  int64_t max_rounds; /* looping Pipe: at most this many passes (0 = until empty)               */
  int32_t reserved[4];
} irgl_pipe_opts;
typedef struct irgl_pipe_result {
  int32_t outlined;       /* 1 if the Pipe ran as one control kernel                            */
  int32_t block;          /* control kernel block size (T_control), 0 when host-orchestrated    */
  int32_t last_reduced;   /* the last executed invocation's return value, -1 if none            */
  int32_t reserved0;
  int32_t stage_reduced[8]; /* per stage: its last invocation's return value, -1 if none          */
} irgl_pipe_result;
/* Members on the outlined path: the test operators COUNTDOWN, RETRY_ODD, RESPAWN_ODD, REDUCE,
 * NOPUSH, PUSHPOP (at most 8 stages); the host path takes any worklist operator. */
irgl_status_t irgl_pipe_run(irgl_ctx* ctx, irgl_pipe* pipe, irgl_graph* g /*nullable*/,
                            const irgl_pipe_stage* stages, int32_t nstages,
                            const irgl_pipe_opts* opts, irgl_iter_stats* stats /*nullable*/,
                            irgl_pipe_result* result /*nullable*/);

#ifdef __cplusplus
}
#endif
#endif
