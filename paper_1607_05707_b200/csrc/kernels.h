// kernels.h — host-side launchers of the device kernels (one translation unit per family).
#pragma once
#include "internal.cuh"

namespace irgl {

// One partition's CSR rows [lo, hi) with global column ids.
struct DevCSR {
  const int64_t* row_ptr;  // [hi-lo+1]
  const int32_t* col;      // [m_local]
  const int32_t* w;        // [m_local] or nullptr
  int64_t lo, hi;
  // byte copy of w when every weight is in [0, 255] (the RMAT weights): the outlined SSSP reads
  // 1 B per edge of weight stream instead of 4 (padded by 16 B); nullptr otherwise
  const uint8_t* w8 = nullptr;
};

// Routing of pushes whose destination is owned by another partition (1D vertex partition).
constexpr int kMaxParts = 16;
struct DistRoute {
  int nparts;          // 1 => no routing
  int me;
  int64_t part_size;   // owner(v) = v / part_size
  uint32_t* send;      // [N]: bucket of peer q is send[q*part_size ...]
  uint32_t* send_cnt;  // [nparts]
  // peer inbox exchange (one process, partitions on devices with peer access): remote updates are
  // stored straight into owner o's inbox segment for this partition, inbox[o], reserving with
  // atomics on inbox_cnt[o] (owner-side counters; P2P atomics when o is another device); null:
  // the local buckets above, packed and moved after the expansion
  uint32_t* inbox[kMaxParts] = {};
  uint32_t* inbox_cnt[kMaxParts] = {};
  // with inbox: the value of each update (the sender's label at the flush) stored beside its id,
  // inbox_val[o] parallel to inbox[o] (the distributed persistent kernel; null: the owner reads
  // the sender's labels, or BFS — no values)
  int32_t* inbox_val[kMaxParts] = {};
};

struct ExpandCfg {
  int32_t warp_t, cta_t, chunk_edges;
};

// Worklist view of one round.
struct RoundBufs {
  const uint32_t* in;
  uint32_t nin;
  uint32_t* out;
  uint32_t* out_cnt;
  uint32_t cap;
  ChunkDesc* chunks;
  uint32_t* chunk_cnt;
  uint32_t chunk_cap;
  int32_t level;     // BFS LEVEL of this round
  int32_t stamp_id;  // unique round id (push dedupe)
  uint32_t* tile_ctr;  // dynamic warp-tile counter of this round (zeroed before the round)
  // SSSP near-far: pushes with dist >= threshold go to the far pile
  uint32_t* far;
  uint32_t* far_cnt;
  uint32_t far_cap;
  int32_t threshold;  // INT32_MAX: near-far off
  unsigned long long* mf_acc;  // DO-BFS: sum of degrees of pushed vertices (null: off)
  // SSSP deferral (defer_k > 0): a popped v with (dist[v] - *dmin_cur) * deg(v) > defer_k is
  // re-pushed instead of expanded; near pushes atomicMin their distance into *dmin_next
  int64_t defer_k;
  const uint32_t* dmin_cur;  // null: use dmin_val (persistent kernel: broadcast at the barrier)
  uint32_t* dmin_next;
  int32_t dmin_val;
  int32_t dense;  // 1: mark-instead-of-push round (outlined, one partition, no near-far)
  const uint32_t* nin_dev;  // non-null: the in-count lives on the device (multi-partition rounds)
};

// ---- data-driven operators: BFS / SSSP / CC_LP (expand.cu) ----------------------------------
// One host-orchestrated round: expansion of `in` plus the CTA-chunk (hub) phase.
cudaError_t launch_expand_round(int op, const DevCSR& g, int32_t* lab, int32_t* stamp, uint32_t* vis, Ctl* ctl,
                                const RoundBufs& rb, const DistRoute& dr, const ExpandCfg& ec,
                                int grid_max, cudaStream_t st);
// Apply received remote updates (owner side min-reduce), all of one owner's received segments in
// one launch: segment p (peer p's updates) holds counts[p] items at items + p * stride, values
// likewise (BFS: none); P <= 16.
struct ApplySegs {
  uint32_t off[17];  // off[p] = first global index of segment p, off[P] = total
  int P;
  int64_t stride;
  // cleared by the launch (always issued, also with nothing to apply): the round's send counts
  // [P] and the consumed in-count — the next round's out counter after the swap
  uint32_t* zero_send = nullptr;
  uint32_t* zero_cnt = nullptr;
  // peer inbox exchange: the value of an update from sender p is read from p's label array at
  // apply time (the sender's ghost label is final once its expansion is done); null: values[]
  const int32_t* peer_lab[kMaxParts] = {};
  // IPC pull exchange (one process per GPU, same node): segment p is read from sender p's own
  // bucket for this owner (ids / values), mapped into this process; null: items / values
  const uint32_t* seg_items[kMaxParts] = {};
  const int32_t* seg_vals[kMaxParts] = {};
};
cudaError_t launch_apply_remote_segs(int op, int32_t* lab, int32_t* stamp, uint32_t* vis, Ctl* ctl,
                                     const uint32_t* items, const int32_t* values,
                                     const ApplySegs& segs, const RoundBufs& rb, cudaStream_t st);
// Near-far split of a far pile into rb.out (dist < rb.threshold) / rb.far (the next pile).
cudaError_t launch_far_split(const DevCSR& g, int32_t* lab, int32_t* stamp, Ctl* ctl,
                             const RoundBufs& rb, const uint32_t* far_in, const uint32_t* nfar_ptr,
                             int32_t t_old, unsigned int* minkeep, int grid, cudaStream_t st);
// Multi-partition round helpers: pack every owner's bucket values in one launch (counts read on
// the device), and write the partition's round header {send counts [P], in-count, overflow}.
cudaError_t launch_pack_all(const int32_t* lab, const uint32_t* send, int32_t* send_val,
                            const uint32_t* send_cnt, int P, int me, int64_t ps, cudaStream_t st);
cudaError_t launch_round_header(uint32_t* hdr, const uint32_t* send_cnt, int P, const uint32_t* in_cnt,
                                const uint32_t* overflow, uint32_t* chunk_cnt, uint32_t* tile_ctr,
                                uint32_t* dmin_done, cudaStream_t st);
// Gather current label values of the send buckets (SSSP / CC_LP pack step).
cudaError_t launch_pack_values(const int32_t* lab, const uint32_t* items, int32_t* values,
                               uint32_t n, cudaStream_t st);

struct PersistArgs {
  uint32_t* buf_a;   // in buffer at round 0
  uint32_t* buf_b;   // out buffer at round 0
  int32_t slot[3];   // counter slots in Ctl::cnt: in, out, spare at round 0
  uint32_t cap;
  ChunkDesc* chunks;
  uint32_t chunk_cap;
  int32_t level0;
  int32_t stamp0;
  int64_t max_rounds;  // 0 = until empty
  uint32_t* far_a;     // SSSP near-far piles (current at round 0 = far_a)
  uint32_t* far_b;
  uint32_t far_cap;
  int32_t delta;       // 0: plain data-driven Bellman-Ford
  int32_t dir_opt;     // BFS: 1 = direction-optimising (top-down / bottom-up switching)
  int64_t n;           // vertices (bottom-up sweeps)
  int64_t m;           // directed edges
  int64_t defer_k;     // SSSP deferral budget (0 = off); cells Ctl::dmin rotate by round
  int64_t dense_min;   // rounds with |in| >= dense_min run dense (0 = never)
  unsigned long long* trace;  // optional per-round trace [4 * trace_cap + 1] (IRGL_ROUND_TRACE)
  uint32_t trace_cap;
  uint32_t trace_cta = 0;     // rounds with per-CTA item-phase end times after the round trace
  // device-resident stamp epoch (pipelined batches): when set, the kernel takes its first stamp
  // id from *stamp_base + 1 instead of stamp0 and leaves its last used id there, so a traversal
  // can be launched before the previous one's stamp count reached the host
  int32_t* stamp_base = nullptr;
  // fused traversal prologue (irgl_traverse_batch): with src >= 0 the kernel itself resets the
  // labels (and the BFS visited bitmap), the control block and the in-worklist to Initial [src]
  // before round 0 — one launch per traversal instead of a dozen small copies, memsets and kernels
  int64_t src = -1;                  // caller id
  const int32_t* src_map = nullptr;  // relabelled graph: caller id -> vertex id
  uint32_t* reset_vis = nullptr;     // BFS visited bitmap the kernel uses (n bits), or null
};
// E3 across partitions (every partition reachable by stores and atomics from every other: one
// device, peer access, or — across processes — CUDA IPC mappings over NVLink): one cooperative
// persistent kernel per partition, the partitions meeting at a device-side rendezvous in
// partition 0's memory instead of at a host synchronisation.  Launch: rendezvous ("hello": every
// kernel resident; nothing written before it).  Round r: expand (remote updates and their values
// stored into the owners' inboxes, DistRoute::inbox / inbox_val) -> rendezvous (every inbox
// complete) -> apply the own inbox -> publish {out count, flags} -> rendezvous (every sum) ->
// next round or exit.
struct XRendezvous {
  alignas(256) unsigned int arrive;  // monotonic arrivals: rendezvous k completes at k * nparts
  unsigned int abort;                // a partition waited spin_ns without the others: all leave
  alignas(256) uint32_t outc[kMaxParts];   // out count of each partition's last round
  uint32_t flags[kMaxParts];               // overflow bits (1 worklist, 2 chunks, 4 inbox)
  unsigned long long mfc[kMaxParts];       // DO-BFS: edges of each partition's next frontier
};
struct DistPersistArgs {
  PersistArgs pa;              // buffers, counter slots, capacities, level0, stamp0, defer_k ...
  XRendezvous* xr;
  unsigned int xbase;          // arrivals before this launch (the counter is never reset)
  int nparts;                  // partitions at the rendezvous (== DistRoute::nparts)
  uint32_t* recv;              // this partition's inbox: sender s's segment at recv + s * part_size
  int32_t* recv_val;           // the updates' values, parallel to recv (null for BFS)
  uint32_t* recv_cnt;          // [nparts] updates stored by each sender (its atomics)
  unsigned long long spin_ns;  // rendezvous wait bound (the kernels must be co-resident)
  // direction-optimising BFS (pa.dir_opt): every partition's copy of the n-bit frontier bitmap
  // (a partition stores its own words into each before a bottom-up round), words per partition
  uint32_t* fbits[kMaxParts];
  int64_t wpp;
};
cudaError_t launch_dist_persistent(int op, const DevCSR& g, int32_t* lab, int32_t* stamp, uint32_t* vis, Ctl* ctl,
                                   const DistRoute& dr, const DistPersistArgs& da, const ExpandCfg& ec, int grid,
                                   cudaStream_t st);
int dist_persistent_blocks_per_sm(int op);
// Outlined Iterate: whole loop in one cooperative persistent kernel (E3).
cudaError_t launch_persistent(int op, const DevCSR& g, int32_t* lab, int32_t* stamp, uint32_t* vis, Ctl* ctl,
                              const PersistArgs& pa, const ExpandCfg& ec, int grid,
                              cudaStream_t st);
// Co-resident CTAs/SM of the persistent kernel for `op` (occupancy API).
// variant: 0 the operator's base kernel, 1 its direction-optimising (BFS) / near-far (SSSP)
// kernel, -1 the minimum over both (a grid valid for either)
int persistent_blocks_per_sm(int op, int variant = -1);
// Direction-optimising BFS on a vertex-partitioned graph (host-orchestrated rounds): frontier
// size / edge count of a partition's in-worklist, the partition-blocked frontier bitmap, and one
// bottom-up round over the partition's own vertices.
cudaError_t launch_frontier_stats(const uint32_t* items, const uint32_t* cnt, const int64_t* rp, int64_t lo,
                                  unsigned long long* out2, cudaStream_t st);
cudaError_t launch_frontier_bits(const uint32_t* items, const uint32_t* cnt, uint32_t* bits, cudaStream_t st);
cudaError_t launch_bu_part(const DevCSR& g, int32_t* lab, uint32_t* vis, Ctl* ctl, const RoundBufs& rb,
                           const uint32_t* fbits, cudaStream_t st);
// *bad |= 1 if an edge leads from a reached to an unreached vertex (the IRGL_E_RANGE check)
cudaError_t launch_range_check(const DevCSR& g, const int32_t* dist, uint32_t* bad, cudaStream_t st);
// w8[k] = w[k] for k < m; *bad = 1 if some weight is outside [0, 255]
cudaError_t launch_weights_u8(const int32_t* w, int64_t m, uint8_t* w8, uint32_t* bad, cudaStream_t st);
int expand_blocks_per_sm(int op);

// ---- topology-driven operators (topo.cu) ----------------------------------------------------
cudaError_t launch_cc_hook(const DevCSR& g, int32_t* parent, Ctl* ctl, int red_slot, int grid,
                           cudaStream_t st);
cudaError_t launch_cc_compress(int32_t* parent, int64_t n, cudaStream_t st);
cudaError_t launch_pr_init(double* rank, double* contrib, const int64_t* row_ptr, int64_t n,
                           cudaStream_t st);
// PageRank hub split (built once per graph): hub_of[v] = hub index of vertex v (valid when
// deg(v) >= hub_t), hub k's chunks are [hfirst[k], hfirst[k+1]), chunk c = edges
// [cbeg[c], cbeg[c] + clen[c]); partial[c] receives the chunk's sum every sweep.
struct PrHubs {
  const int32_t* hub_of;
  const int64_t* hfirst;
  const int64_t* cbeg;
  const int32_t* clen;
  double* partial;
  int64_t nchunks;  // 0: no hub split
  int64_t hub_t;
  int32_t cta_tiles;  // sweep layout: 1 CTA tiles (degree-ordered ids), 0 warp tiles
};
cudaError_t launch_pr_sweep(const DevCSR& g, const double* rank_old, double* rank_new,
                            const double* contrib, double* contrib_next, double d, double tol,
                            int64_t n_global, Ctl* ctl, int red_slot, int grid, const PrHubs& h,
                            cudaStream_t st);
cudaError_t launch_pr_persistent(const DevCSR& g, double* ra, double* rb, double* ca, double* cb,
                                 double d, double tol, int64_t n_global, Ctl* ctl,
                                 int64_t max_rounds, int cond_mode, int grid, const PrHubs& h,
                                 cudaStream_t st);
int pr_persistent_blocks_per_sm();
cudaError_t tc_orient(const DevCSR& g, int64_t n, int64_t** rp_out, int32_t** cl_out,
                      int32_t** src_out, int64_t* m_out, cudaStream_t st);
cudaError_t launch_tc_count(const int64_t* rp, const int32_t* cl, const int32_t* src, int64_t mo,
                            Ctl* ctl, cudaStream_t st);

// ---- Atomic / Exclusive constructs and Boruvka MST (mst.cu) -----------------------------------
cudaError_t launch_mst_init(int32_t* parent, int32_t* comp, int32_t* lock, int32_t* bw, int32_t* ba,
                            int32_t* bb, uint32_t* wl, int64_t n, cudaStream_t st);
cudaError_t launch_mst_round(const DevCSR& g, int32_t* parent, int32_t* comp, int32_t* lock,
                             int32_t* bw, int32_t* ba, int32_t* bb, const uint32_t* in, uint32_t nin,
                             uint32_t* out, uint32_t* out_cnt, unsigned long long* wsum,
                             unsigned long long* esum, uint32_t* cell, int64_t n, int grid,
                             cudaStream_t st);
cudaError_t launch_atomic_test(const uint32_t* in, uint32_t nin, int32_t* lock, int32_t* log,
                               int else_form, int threads, cudaStream_t st);
int exclusive_blocks_per_sm();
cudaError_t launch_exclusive_test(const uint32_t* in, uint32_t nin, const int32_t* locks, int k,
                                  int32_t* owner, int32_t* won, int32_t* log, int grid,
                                  cudaStream_t st);

// Reset of the control block before an outlined (persistent) launch, in one kernel.
cudaError_t launch_ctl_prepare(Ctl* ctl, cudaStream_t st);

// ---- degree-ordered relabelling (relabel.cu) ---------------------------------------------------
// Replaces *col_io / *w_io (freed) with the relabelled arrays, returns new row offsets, perm
// (new id of each old vertex) and inv (old vertex of each new id); the caller frees rp_old.
cudaError_t relabel_degree(int64_t n, int64_t m, int64_t maxdeg, const int64_t* rp_old, int32_t** col_io,
                           int32_t** w_io, int64_t** rp_new, int32_t** perm_out, int32_t** inv_out,
                           cudaStream_t st);
cudaError_t launch_map_items(uint32_t* items, uint32_t n, const int32_t* table, cudaStream_t st);
cudaError_t launch_gather_i32(int32_t* out, const int32_t* src, const int32_t* perm, int64_t n, cudaStream_t st);
cudaError_t launch_gather_range_i32(int32_t* out, const int32_t* src, const int32_t* perm, int64_t lo,
                                   int64_t nloc, cudaStream_t st);
// Block-diagonal degree order of a vertex partition (relabel.cu): phase 1 orders the partition's
// own rows, phase 2 rewrites its CSR once every partition's new ids are known (perm_global).
cudaError_t relabel_order(int64_t nloc, int64_t lo, int64_t maxdeg, const int64_t* rp_old,
                          int32_t** perm_local, int32_t** inv_local, cudaStream_t st);
cudaError_t relabel_rewrite(int64_t nloc, int64_t lo, int64_t n, int64_t m, const int64_t* rp_old,
                            const int32_t* perm_local, const int32_t* inv_local,
                            const int32_t* perm_global, int32_t** col_io, int32_t** w_io,
                            int64_t** rp_new, cudaStream_t st);
cudaError_t launch_gather_f64(double* out, const double* src, const int32_t* perm, int64_t n, cudaStream_t st);
cudaError_t launch_cc_labels_original(int32_t* out, const int32_t* lab, const int32_t* perm, const int32_t* inv,
                                      int32_t* cmin, int64_t n, cudaStream_t st);

// ---- misc (util.cu) ---------------------------------------------------------------------------
cudaError_t launch_fill_i32(int32_t* p, int32_t v, int64_t n, cudaStream_t st);
cudaError_t launch_scatter_zero(int32_t* lab, const uint32_t* items, uint32_t n, cudaStream_t st,
                                uint32_t* vis = nullptr);
cudaError_t launch_iota_u32(uint32_t* p, uint32_t begin, uint32_t n, cudaStream_t st);
cudaError_t launch_set_red(Ctl* ctl, int slot, uint32_t v, cudaStream_t st);

// ---- test operators (testops.cu) ----------------------------------------------------------------
struct TestArgs {
  int op;
  const uint32_t* in;
  uint32_t nin;
  uint32_t* out;
  uint32_t* out_cnt;
  uint32_t* retry;
  uint32_t* retry_cnt;
  uint32_t cap;
  int64_t guard;
  const int32_t* values;
  int32_t* rcount;    // per item retry counts
  int32_t* log;       // PUSHPOP: popped_at; FORALL_MAP: thread id
  int32_t launch_no;
  int mapping;
  uint32_t* red;      // return cell
  int reduction;
  uint32_t* overflow;
};
cudaError_t launch_test_op(const TestArgs& a, int threads, cudaStream_t st);

// Outlined multi-member Pipe of test operators: the program the control kernel
// runs.  Buffer roles are indices into buf[3] / cnt[3] (count of each buffer); state[] carries
// {in, out, retry, launch_no} in and out; stats[] = {launches, popped, pushes, retries,
// serial_launches, rounds, trace_len, last_reduced}.
constexpr int kPipeMaxStages = 8;
struct PipeStageDev {
  int32_t op, kind, reduction, when, cond_mode, mapping;
  int64_t guard, max_rounds;
  const int32_t* values;
};
struct PipeProgDev {
  PipeStageDev st[kPipeMaxStages];
  int32_t n, once, rsa;
  int64_t max_rounds;
  uint32_t* buf[3];
  uint32_t* cnt;
  uint32_t cap;
  int32_t* rcount;
  int32_t* log;
  uint32_t* red;
  uint32_t* overflow;
  int32_t* state;
  int64_t* stats;
  int32_t* reds;      // per stage: last reduced value
  int64_t* trace;     // [trace_cap][4]
  int64_t trace_cap;
};
cudaError_t launch_pipe_control(const PipeProgDev& prog, int grid, int block, cudaStream_t st);
int pipe_control_blocks_per_sm(int block);

// ---- graph generation (gen.cu) ------------------------------------------------------------------
// Builds the CSR rows [lo, hi) of the generated graph on the device.
cudaError_t gen_partition(const irgl_gen_spec& s, int64_t n, int64_t lo, int64_t hi,
                          int64_t** row_ptr, int32_t** col, int32_t** w, int64_t* m_local,
                          cudaStream_t st, std::string* err);
cudaError_t max_degree(const int64_t* row_ptr, int64_t nrows, int64_t* out, cudaStream_t st);
// Directed edge records -> CSR on the device (sort by (u, v), keep the minimum weight per pair).
struct EdgeRec {
  uint32_t u, v;
  int32_t w;
};
cudaError_t csr_from_edges_device(const EdgeRec* host_edges, int64_t ne, int64_t n,
                                  int64_t** row_ptr, int32_t** col, int32_t** w, int64_t* m,
                                  cudaStream_t st);

}  // namespace irgl
