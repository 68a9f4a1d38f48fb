// expand.cu — the data-driven hot path: ForAll over the in-worklist x ForAll over edges(n)
// for BFS (Listing 2), SSSP and CC_LP, lowered B200-first:
//
//  E1  nested-parallelism edge scheduler.  Work is handed out in warp tiles of up to 32 popped
//      vertices (first tile static, then dynamic from a per-round counter); each vertex's edges go
//      to
//        - the warp's fine-grained gather (degree < warp_t): warp-wide scan of the small degrees,
//                              each lane finds the owner of its edge slot with a 5-step shuffle
//                              search (no shared memory, no CTA barrier);
//        - edge chunks         (degree >= warp_t): chunk_edges-sized descriptors (one reservation
//                              per warp tile) that every warp of the grid drains in a second,
//                              edge-balanced phase: one 128-bit col/weight group per lane per
//                              iteration, the next group loaded before the current gathers and
//                              atomics are waited on; few chunks are split over several warps.
//      relax_batch issues every atomic of a lane's batch before consuming any result (BFS CAS or
//      visited-bitmap OR; SSSP/CC RED.MIN + stamp exchange); large frontiers run "dense" rounds
//      that mark instead of push and compact the marks into the next worklist.
//  E2  cooperative conversion of pushes: warp __ballot_sync/__popc aggregation into a per-warp
//      shared-memory staging queue; one global atomic reservation per 224+ staged items, per CTA
//      at phase end; remote pushes (multi-partition) staged per owner the same way.
//  E3  iteration outlining: the Iterate loop as one cooperative persistent kernel; rounds are
//      separated by grid_sync_bcast (SyncRunningThreads) whose release word
//      carries the round's counters, so no thread re-reads hot counters after the barrier.
//  SSSP degree-scaled deferral (defer > 0): a popped vertex whose (dist - frontier min) * degree
//      exceeds the budget is re-pushed instead of expanded (hubs expand near their final
//      distance); near-far piles (delta > 0) are the bucketed alternative.  Both leave the fixed
//      point of Bellman-Ford, i.e. the distances, unchanged.
//
// Reference semantics (SPEC.md:317-322 ForAll lowering; :425 bulk-synchronous worklists: pops
// read `in`, pushes append to `out`, never visible in the same launch).
#include <cooperative_groups.h>
#include <type_traits>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace irgl {
namespace {

constexpr unsigned FULL = 0xffffffffu;
#ifndef IRGL_WBUF
#define IRGL_WBUF 96  // a flush every >= 64 staged pushes; 256 cost L1 capacity (see kBlock)
#endif
constexpr int kWBuf = IRGL_WBUF;  // per-warp push staging entries
#ifndef IRGL_MINB
#define IRGL_MINB minb_for_threads(1536)  // 40 registers, 48 warps/SM (tools/sweep.py)
#endif
#ifndef IRGL_MINB_SSSP
#define IRGL_MINB_SSSP minb_for_threads(1024)  // SSSP (weights + batched relax): 64 registers, 32 warps/SM
#endif
// Internal operator variants (template-level, so the common path carries no state of the others):
// SSSP with near-far piles, and BFS accumulating the next frontier's degrees (direction-optimising).
constexpr int kOpSsspNF = 0x101;
constexpr int kOpSssp8 = 0x102;  // outlined SSSP over the byte weight copy (DevCSR::w8)
constexpr int kOpBfsDO = 0x100;
constexpr bool is_bfs(int op) { return op == IRGL_OP_BFS || op == kOpBfsDO; }
constexpr bool is_sssp(int op) { return op == IRGL_OP_SSSP || op == kOpSsspNF || op == kOpSssp8; }
constexpr bool w8_op(int op) { return op == kOpSssp8; }
constexpr bool has_far(int op) { return op == kOpSsspNF; }

// Push dedupe by stamp.  Stamp ids only grow (one per round / split, monotonic across
// traversals; the array is cleared when the id space wraps), so a push claims its vertex with
// atomicMax and pushes iff the previous code was smaller.  Near-far ops code a near push as
// (sid << 1) | 1 and a far push (and a send to a remote owner) as sid << 1: within a round the
// near claim dominates, so a late far claim working from a stale label can never undo it and let
// a later near candidate push the vertex twice.  Other ops use sid << 1 (the dense-round mark).
template <int OP>
__device__ __forceinline__ int32_t stamp_code(int32_t sid, int kind) {
  return has_far(OP) ? ((sid << 1) | (kind == 1 ? 1 : 0)) : (sid << 1);
}
__device__ __forceinline__ bool stamp_claim(int32_t* s, int32_t code) { return atomicMax(s, code) < code; }
constexpr bool has_mf(int op) { return op == kOpBfsDO; }
constexpr int minb_for(int op) { return is_sssp(op) ? IRGL_MINB_SSSP : IRGL_MINB; }

struct Smem {
  uint32_t wbuf[kWarps][kWBuf];   // near pushes (E2)
  uint32_t fl_cnt[2][kWarps];     // CTA flush: per-warp staged counts (near, far)
  uint32_t fl_off[2][kWarps];     // CTA flush: per-warp global offsets
  unsigned long long fl_edges[kWarps];
};

struct KParams {
  DevCSR g;
  int32_t* lab;
  int32_t* stamp;
  uint32_t* vis;  // BFS: visited bitmap over all n vertices (L2-resident where the level array is
                  // not: 16.8 MB at RMAT-27 vs 537 MB); null for the other operators
  Ctl* ctl;
  DistRoute dr;
  ExpandCfg ec;
};

// Multi-partition kernels also stage remote pushes per warp: entries (owner << 28 | v), flushed
// to the per-owner send buckets with one reservation per owner per flush (the owner counters are
// a handful of addresses every warp of the grid would otherwise hit once per push).
// Far-pile staging of the near-far SSSP kernels: only kernels instantiated for a near-far operator
// reference it, so the others keep that shared memory for L1 (the label gathers' cache).
__shared__ uint32_t s_fbuf[kWarps][kWBuf];

struct SmemDist : Smem {
  uint32_t rbuf[kWarps][kWBuf];
};

__device__ __forceinline__ void smem_init(Smem& sm) {
  if ((threadIdx.x & 31) == 0) sm.fl_edges[threadIdx.x >> 5] = 0;  // per-warp edge counters
}

// Register-resident, warp-uniform state of a warp's staging queues.
struct WarpQ {
  uint32_t n = 0;   // staged near pushes
  uint32_t nf = 0;  // staged far pushes
  unsigned long long mf = 0;  // DO-BFS: degrees of pushed vertices (kOpBfsDO only)
  int32_t dmin = kInf;        // SSSP deferral: min distance this lane pushed near (per lane)
  uint32_t nr = 0;            // multi-partition: staged remote pushes
  uint32_t remote = 0;        // multi-partition: remote pushes emitted (stats)
};

__device__ __forceinline__ uint32_t ld_stream_u32(const uint8_t* p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ int32_t ld_stream_u8(const uint8_t* p) {
  uint16_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u8 %0, [%1];" : "=h"(r) : "l"(p));
  return (int32_t)r;
}
__device__ __forceinline__ int32_t w8_at(uint32_t x, int t) { return (int32_t)((x >> (8 * t)) & 255u); }

// Row offsets of popped vertices: read-only, touched once per expansion, so kept out of L1
// (IRGL_ROWPTR_NA=0: the cached __ldg path) — L1 is for the label gathers
#ifndef IRGL_ROWPTR_NA
#define IRGL_ROWPTR_NA 1
#endif
__device__ __forceinline__ int64_t ld_rowptr(const int64_t* p) {
#if IRGL_ROWPTR_NA
  int64_t r;
  asm volatile("ld.global.nc.L1::no_allocate.s64 %0, [%1];" : "=l"(r) : "l"(p));
  return r;
#else
  return __ldg(p);
#endif
}

__device__ __forceinline__ uint32_t ld_item(const uint32_t* p) {
  uint32_t r;
  asm volatile("ld.global.cg.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ld_ctl(const uint32_t* p) {
  uint32_t r;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}

// Per-edge gather of the destination's state.  BFS reads one bit of the visited bitmap and returns
// it in the level encoding the relax code tests (INF = unvisited; a stale 0 bit is benign: the
// atomicOr that follows decides).  Other operators read the label.
template <int OP>
__device__ __forceinline__ int32_t gather_cur(const KParams& p, uint32_t dst) {
  if (is_bfs(OP) && p.vis) {
    uint32_t w;
    asm volatile("ld.global.u32 %0, [%1];" : "=r"(w) : "l"(p.vis + (dst >> 5)));
    return ((w >> (dst & 31)) & 1u) ? 0 : kInf;
  }
  return ld_label(p.lab + dst);
}

// SSSP path sum nd = dist[n] + weight(e) in int32 storage (INF = INT32_MAX, SPEC.md:421 maps the
// 64-bit Int onto it).  A sum that reaches INF is not representable: it is never a candidate, and
// when its target is still unreached (cur == INF) the pipe's overflow word gets bit 4 — the
// target may have a true distance >= INF.  The host then checks the finished traversal exactly
// (an edge from a reached to an unreached vertex exists only through such a sum) and reports
// IRGL_E_RANGE instead of an unreachable label.  Weights are >= 0 (validated) and dist[n] < INF.
__device__ __forceinline__ int32_t path_sum(const KParams& p, int32_t sv, int32_t wt, int32_t cur) {
  const uint32_t s = (uint32_t)sv + (uint32_t)wt;
  if (s >= (uint32_t)kInf) {
    if (cur == kInf) atomicOr(&p.ctl->overflow, 4u);
    return kInf;
  }
  return (int32_t)s;
}

// ---- relax: the operator body for one edge (n -> dst) ----------------------------------------
// BFS   : if level[dst]==INF { level[dst]=LEVEL; push(dst) }   CAS dedupes the push.
// SSSP  : nd = dist[n]+w;  if atomicMin(dist[dst],nd) > nd and stamp[dst] != round: push(dst)
// CC_LP : nd = label[n];   same as SSSP.
// Returns 0 (no push), 1 (near push) or 2 (far push: nd >= threshold).
template <int OP>
__device__ __forceinline__ int relax_with(const KParams& p, const RoundBufs& rb, WarpQ& q,
                                          int32_t cur, int32_t sv, int32_t wt, uint32_t dst) {
  if (is_bfs(OP)) {
    if (cur != kInf) return 0;
    if (p.vis) {  // claim the vertex in the bitmap; the winner writes its level
      const uint32_t bit = 1u << (dst & 31);
      if (atomicOr(p.vis + (dst >> 5), bit) & bit) return 0;
      p.lab[dst] = rb.level;
      return 1;
    }
    return atomicCAS(p.lab + dst, kInf, rb.level) == kInf ? 1 : 0;
  } else {
    const int32_t nd = (is_sssp(OP)) ? path_sum(p, sv, wt, cur) : sv;
    if (nd >= cur) return 0;
    const int32_t old = atomicMin(p.lab + dst, nd);
    if (nd >= old) return 0;
    // push dedupe per round and per pile (stamp_code).  A vertex first pushed far and then
    // improved below the threshold in the same round is pushed near too; its stale far entry is
    // dropped by the split (dist < old threshold).
    const int kind = (has_far(OP) && nd >= rb.threshold) ? 2 : 1;
    // dst now holds <= nd and sits in the near out worklist (pushed here or earlier this round)
    if (is_sssp(OP) && kind == 1) q.dmin = min(q.dmin, nd);
    return stamp_claim(p.stamp + dst, stamp_code<OP>(rb.stamp_id, kind)) ? kind : 0;
  }
}

// Batched relax of one lane's K edges (same decisions as relax_with, ILP-friendly): every atomic
// of the batch is issued before any result is consumed, so a lane pays one L2 round trip per
// batch instead of one or two dependent round trips per edge (hub rounds are latency-bound).
//  BFS         : CAS(INF -> LEVEL) on each candidate (cur == INF); push where the CAS won.
//  SSSP / CC_LP: candidates nd < cur get a fire-and-forget atomic min (RED, no return) and a
//                stamp exchange issued together; a candidate pushes where it claimed the round's
//                stamp.  Every vertex lowered this round had a candidate, and every candidate's
//                vertex ends in the pile exactly once (the claimer pushes), so the out worklist is
//                the same set relax_with builds; a candidate that lost the min race still holds
//                <= nd, which keeps the deferral minimum (q.dmin) a valid bound.  The REDs are
//                ordered before the next round by the grid barrier / kernel boundary.
template <int OP, int K>
__device__ __forceinline__ void relax_batch(const KParams& p, const RoundBufs& rb, WarpQ& q,
                                            const bool (&act)[K], const int32_t (&cur)[K],
                                            const int32_t (&sv)[K], const int32_t (&wt)[K],
                                            const uint32_t (&dst)[K], int (&kind)[K]) {
  if (!has_far(OP) && rb.dense) {
    // dense round: mark instead of push, every write fire-and-forget (no result waited on); the
    // compaction phase after the barrier builds the out worklist from the marks
    if (is_bfs(OP)) {
#pragma unroll
      for (int j = 0; j < K; ++j)
        if (act[j] && cur[j] == kInf) {
          p.lab[dst[j]] = rb.level;  // every writer stores LEVEL
          if (p.vis) atomicOr(p.vis + (dst[j] >> 5), 1u << (dst[j] & 31));  // RED.OR
        }
    } else {
      const int32_t code = rb.stamp_id << 1;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        const int32_t nd = is_sssp(OP) && act[j] ? path_sum(p, sv[j], wt[j], cur[j]) : sv[j];
        if (act[j] && nd < cur[j]) {
          atomicMin(p.lab + dst[j], nd);    // RED.MIN
          atomicMax(p.stamp + dst[j], code);  // RED.MAX: stamp ids only grow
          if (is_sssp(OP)) q.dmin = min(q.dmin, nd);
        }
      }
    }
#pragma unroll
    for (int j = 0; j < K; ++j) kind[j] = 0;
    return;
  }
  if (is_bfs(OP)) {
    if (p.vis) {
      uint32_t old[K];
#pragma unroll
      for (int j = 0; j < K; ++j)
        old[j] = (act[j] && cur[j] == kInf) ? atomicOr(p.vis + (dst[j] >> 5), 1u << (dst[j] & 31)) : ~0u;
#pragma unroll
      for (int j = 0; j < K; ++j) {
        kind[j] = (old[j] & (1u << (dst[j] & 31))) ? 0 : 1;
        if (kind[j]) p.lab[dst[j]] = rb.level;
      }
      return;
    }
    int32_t old[K];
#pragma unroll
    for (int j = 0; j < K; ++j)
      old[j] = (act[j] && cur[j] == kInf) ? atomicCAS(p.lab + dst[j], kInf, rb.level) : 0;
#pragma unroll
    for (int j = 0; j < K; ++j) kind[j] = (act[j] && cur[j] == kInf && old[j] == kInf) ? 1 : 0;
  } else {
    int32_t nd[K], code[K], prev[K];
    bool cand[K];
    int32_t old[K];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      nd[j] = is_sssp(OP) && act[j] ? path_sum(p, sv[j], wt[j], cur[j]) : sv[j];
      cand[j] = act[j] && nd[j] < cur[j];
      kind[j] = (has_far(OP) && nd[j] >= rb.threshold) ? 2 : 1;
      // a vertex another partition owns is sent once per round whatever its pile (the owner
      // decides near / far): one code for both kinds
      const bool remote = has_far(OP) && p.dr.nparts > 1 &&
                          (uint64_t)((int64_t)dst[j] - p.g.lo) >= (uint64_t)(p.g.hi - p.g.lo);
      code[j] = stamp_code<OP>(rb.stamp_id, remote ? 2 : kind[j]);
      if (has_far(OP)) old[j] = cand[j] ? atomicMin(p.lab + dst[j], nd[j]) : 0;
      else if (cand[j]) atomicMin(p.lab + dst[j], nd[j]);  // result unused -> RED.MIN
    }
    // Near-far: only a candidate that lowered the distance claims the stamp (a far candidate
    // from a stale label needs no push: the vertex is already queued near or lower), and the
    // near code dominates the far one (stamp_code), so no interleaving pushes a vertex near twice
    // in a round (more than n pushes: worklist overflow, found by tools/stress.py).
    if (has_far(OP)) {
#pragma unroll
      for (int j = 0; j < K; ++j) cand[j] = cand[j] && nd[j] < old[j];
    }
#pragma unroll
    for (int j = 0; j < K; ++j) prev[j] = cand[j] ? atomicMax(p.stamp + dst[j], code[j]) : code[j];
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if (is_sssp(OP) && cand[j] && kind[j] == 1) q.dmin = min(q.dmin, nd[j]);
      kind[j] = (cand[j] && prev[j] < code[j]) ? kind[j] : 0;
    }
  }
}

// ---- E2: per-warp staging --------------------------------------------------------------------
__device__ __forceinline__ void wflush(uint32_t* buf, uint32_t& n, uint32_t* out, uint32_t* cnt,
                                       uint32_t cap, uint32_t* overflow) {
  if (n == 0) return;
  __syncwarp();
  uint32_t base = 0;
  if (lane_id() == 0) base = atomicAdd(cnt, n);
  base = __shfl_sync(FULL, base, 0);
  for (uint32_t i = lane_id(); i < n; i += 32) {
    const uint32_t q = base + i;
    if (q < cap) out[q] = buf[i];
    else atomicOr(overflow, 1u);
  }
  __syncwarp();
  n = 0;
}

// Flush of the warp's staged remote pushes: per owner, count the warp's entries, reserve once,
// write in staging order.  Warp-collective.
__device__ __forceinline__ void wflush_remote(SmemDist& sd, WarpQ& q, const KParams& p) {
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  const uint32_t n = q.nr;
  __syncwarp();
  for (int o = 0; o < p.dr.nparts; ++o) {
    if (o == p.dr.me) continue;
    uint32_t c = 0;
    for (uint32_t i = lane; i < n; i += 32) c += (sd.rbuf[warp][i] >> 28) == (uint32_t)o;
    uint32_t incl = c;
#pragma unroll
    for (int k = 1; k < 32; k <<= 1) {
      const uint32_t t = __shfl_up_sync(FULL, incl, k);
      if (lane >= k) incl += t;
    }
    const uint32_t tot = __shfl_sync(FULL, incl, 31);
    if (tot == 0) continue;
    uint32_t base = 0;
    // peer inbox: reserve in the owner's counter and store into the owner's segment directly
    uint32_t* const ocnt = p.dr.inbox[o] ? p.dr.inbox_cnt[o] : p.dr.send_cnt + o;
    if (lane == 31) base = atomicAdd(ocnt, tot);
    base = __shfl_sync(FULL, base, 31);
    uint32_t pos = base + incl - c;
    uint32_t* bucket = p.dr.inbox[o] ? p.dr.inbox[o] : p.dr.send + (int64_t)o * p.dr.part_size;
    // values sent later (dist_persistent_kernel's pack, after the whole expansion: a label can
    // still drop after this flush): the ids also go to the local bucket at the same positions,
    // and the local counter keeps the segment's length
    uint32_t* lcopy = p.dr.inbox_val[o] ? p.dr.send + (int64_t)o * p.dr.part_size : nullptr;
    if (lcopy && lane == 31) atomicAdd(p.dr.send_cnt + o, tot);
    for (uint32_t i = lane; i < n; i += 32) {
      const uint32_t e = sd.rbuf[warp][i];
      if ((e >> 28) == (uint32_t)o) {
        if (pos < (uint32_t)p.dr.part_size) {
          bucket[pos] = e & 0x0fffffffu;
          if (lcopy) lcopy[pos] = e & 0x0fffffffu;
        } else {
          atomicOr(&p.ctl->overflow, 1u);
        }
        ++pos;
      }
    }
  }
  __syncwarp();
  q.nr = 0;
}
// Phase end of a multi-partition kernel: remaining staged remote pushes and the remote counter.
__device__ __forceinline__ void wflush_remote_all(SmemDist& sd, WarpQ& q, const KParams& p) {
  if (q.nr) wflush_remote(sd, q, p);
  if (lane_id() == 0 && q.remote) atomicAdd(&p.ctl->remote, (unsigned long long)q.remote);
  q.remote = 0;
}

// Every lane of the warp must call this (converged).  kind: 0 none, 1 near, 2 far.
template <int OP, bool DIST>
__device__ __forceinline__ void wpush(Smem& sm, WarpQ& q, const KParams& p, const RoundBufs& rb,
                                      int kind, uint32_t v) {
  uint32_t m = __ballot_sync(FULL, kind != 0);
  if (m == 0) return;
  const uint32_t lane = lane_id(), warp = threadIdx.x >> 5;
  if (DIST) {
    // local = inside this partition's id range (no division on the common path); the owner of
    // a remote id is computed by the remote lanes only (ids < 2^28, part sizes < 2^31)
    const bool remote = kind && (uint64_t)((int64_t)v - p.g.lo) >= (uint64_t)(p.g.hi - p.g.lo);
    const uint32_t rm = __ballot_sync(FULL, remote);
    if (rm) {
      if constexpr (DIST) {
        SmemDist& sd = static_cast<SmemDist&>(sm);
        if (remote) {
          const uint32_t owner = v / (uint32_t)p.dr.part_size;
          sd.rbuf[warp][q.nr + __popc(rm & lanemask_lt())] = (owner << 28) | v;
        }
        q.nr += __popc(rm);
        q.remote += __popc(rm);
        if (q.nr > kWBuf - 32) wflush_remote(sd, q, p);
      }
      if (remote) kind = 0;
      m = __ballot_sync(FULL, kind != 0);
      if (m == 0) return;
    }
  }
  const uint32_t mn = __ballot_sync(FULL, kind == 1);
  const uint32_t mf = m & ~mn;
  const uint32_t lt = lanemask_lt();
  if (has_mf(OP) && mn) {  // DO-BFS: edges of the next frontier
    unsigned long long dg = 0;
    if (kind == 1) dg = (unsigned long long)(__ldg(p.g.row_ptr + v - p.g.lo + 1) - __ldg(p.g.row_ptr + v - p.g.lo));
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) dg += __shfl_xor_sync(FULL, dg, o);
    q.mf += dg;
  }
  if (mn) {
    if (kind == 1) sm.wbuf[warp][q.n + __popc(mn & lt)] = v;
    q.n += __popc(mn);
    if (q.n > kWBuf - 32) wflush(sm.wbuf[warp], q.n, rb.out, rb.out_cnt, rb.cap, &p.ctl->overflow);
  }
  if constexpr (has_far(OP)) {
    if (mf) {
      if (kind == 2) s_fbuf[warp][q.nf + __popc(mf & lt)] = v;
      q.nf += __popc(mf);
      if (q.nf > kWBuf - 32) wflush(s_fbuf[warp], q.nf, rb.far, rb.far_cnt, rb.far_cap, &p.ctl->overflow);
    }
  }
}

// CTA-level flush at a CTA-uniform point (every thread calls it): one global reservation per pile
// and one stats atomic per CTA instead of one per warp (E2 at CTA granularity).
template <int OP>
__device__ __forceinline__ void wflush_all(Smem& sm, WarpQ& q, const KParams& p, const RoundBufs& rb) {
  const uint32_t warp = threadIdx.x >> 5, lane = lane_id();
  if (has_mf(OP) && q.mf) {
    if (lane == 0) atomicAdd(rb.mf_acc, q.mf);
    q.mf = 0;
  }
  if (rb.dmin_next) {
    int32_t m = q.dmin;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(FULL, m, o));
    if (lane == 0 && m != kInf) atomicMin(rb.dmin_next, (uint32_t)m);
    q.dmin = kInf;
  }
  if (lane == 0) {
    sm.fl_cnt[0][warp] = q.n;
    sm.fl_cnt[1][warp] = has_far(OP) ? q.nf : 0u;
  }
  __syncthreads();
  if (threadIdx.x < (has_far(OP) ? 2 : 1)) {
    const int k = threadIdx.x;
    uint32_t tot = 0;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) {
      sm.fl_off[k][w] = tot;
      tot += sm.fl_cnt[k][w];
    }
    const uint32_t base = tot ? atomicAdd(k == 0 ? rb.out_cnt : rb.far_cnt, tot) : 0u;
#pragma unroll
    for (int w = 0; w < kWarps; ++w) sm.fl_off[k][w] += base;
    if (k == 0) {
      unsigned long long te = 0;
#pragma unroll
      for (int w = 0; w < kWarps; ++w) te += sm.fl_edges[w];
      if (te) atomicAdd(&p.ctl->edges, te);
    }
  }
  __syncthreads();
  const uint32_t o0 = sm.fl_off[0][warp], o1 = sm.fl_off[1][warp];
  for (uint32_t i = lane; i < q.n; i += 32) {
    const uint32_t qq = o0 + i;
    if (qq < rb.cap) rb.out[qq] = sm.wbuf[warp][i];
    else atomicOr(&p.ctl->overflow, 1u);
  }
  if constexpr (has_far(OP)) {
    for (uint32_t i = lane; i < q.nf; i += 32) {
      const uint32_t qq = o1 + i;
      if (qq < rb.far_cap) rb.far[qq] = s_fbuf[warp][i];
      else atomicOr(&p.ctl->overflow, 1u);
    }
  }
  if (lane == 0) sm.fl_edges[warp] = 0;  // read by thread 0 before the second barrier
  __syncwarp();
  q.n = q.nf = 0;
}

// ---- edge-range processing by one warp --------------------------------------------------------
// The range [b, e) is covered by the aligned 128-bit groups of col/weight that overlap it; each
// lane takes two groups per iteration and masks the edges outside the range (the CSR arrays are
// padded by 4 entries, so the last group is always in bounds).  No separate head/tail step: all 8
// label gathers and all atomics of a lane are in flight together (relax_batch).
#ifndef IRGL_GROUPS
#define IRGL_GROUPS 1  // 128-bit col/weight groups per lane per iteration (4 edges each; 1 beat 2, profiles/r1s2_variants.txt)
#endif
template <int OP, bool DIST>
__device__ __forceinline__ void process_range(Smem& sm, WarpQ& q, const KParams& p,
                                              const RoundBufs& rb, int64_t b, int64_t e,
                                              int32_t sv, int gl) {
  constexpr int NG = IRGL_GROUPS, NE = 4 * NG;
  const int32_t* __restrict__ col = p.g.col;
  const int32_t* __restrict__ w = p.g.w;
  const int64_t g1 = (e + 3) >> 2;
  for (int64_t q0 = b >> 2; q0 < g1; q0 += 32 * NG) {
    int4 cg[NG], wg[NG];
    uint32_t w8g[NG];
    bool ag[NG];
#pragma unroll
    for (int k = 0; k < NG; ++k) {
      const int64_t qk = q0 + 32 * k + gl;
      ag[k] = qk < g1;
      cg[k] = make_int4(0, 0, 0, 0);
      wg[k] = make_int4(0, 0, 0, 0);
      w8g[k] = 0;
      if (ag[k]) {
        cg[k] = ld_stream_v4(col + 4 * qk);
        if (w8_op(OP)) w8g[k] = ld_stream_u32(p.g.w8 + 4 * qk);
        else if (is_sssp(OP)) wg[k] = ld_stream_v4(w + 4 * qk);
      }
    }
    bool act[NE];
    uint32_t d[NE];
    int32_t wt[NE], sv8[NE], cur[NE];
#pragma unroll
    for (int k = 0; k < NG; ++k) {
      const int64_t e0 = 4 * (q0 + 32 * k + gl);
      const int32_t cc[4] = {cg[k].x, cg[k].y, cg[k].z, cg[k].w};
      const int32_t ww[4] = {w8_op(OP) ? w8_at(w8g[k], 0) : wg[k].x, w8_op(OP) ? w8_at(w8g[k], 1) : wg[k].y,
                             w8_op(OP) ? w8_at(w8g[k], 2) : wg[k].z, w8_op(OP) ? w8_at(w8g[k], 3) : wg[k].w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        act[4 * k + t] = ag[k] && e0 + t >= b && e0 + t < e;
        d[4 * k + t] = (uint32_t)cc[t];
        wt[4 * k + t] = ww[t];
        sv8[4 * k + t] = sv;
      }
    }
#pragma unroll
    for (int j = 0; j < NE; ++j) cur[j] = act[j] ? gather_cur<OP>(p, d[j]) : 0;
    int kk[NE];
    relax_batch<OP, NE>(p, rb, q, act, cur, sv8, wt, d, kk);
#pragma unroll
    for (int k = 0; k < NG; ++k) {
      if (k > 0 && !__any_sync(FULL, ag[k])) break;
#pragma unroll
      for (int t = 0; t < 4; ++t) wpush<OP, DIST>(sm, q, p, rb, kk[4 * k + t], d[4 * k + t]);
    }
  }
}

// ---- one warp tile of 32 worklist items (consecutive mapping inside the tile) --------------------
template <int OP, bool DIST>
__device__ void expand_warp_tile(Smem& sm, WarpQ& q, const KParams& p, const RoundBufs& rb,
                                 uint32_t base, uint32_t width, int32_t dmin, bool small_round,
                                 uint32_t nin) {
  const int lane = lane_id();
  const uint32_t i = base + lane;
  const bool valid = (uint32_t)lane < width && i < nin;
  uint32_t v = 0;
  int64_t beg = 0, end = 0;
  int32_t sv = 0;
  if (valid) {
    v = ld_item(rb.in + i);  // n = wl.pop(i)
    const int64_t lv = (int64_t)v - p.g.lo;
    beg = ld_rowptr(p.g.row_ptr + lv);
    end = ld_rowptr(p.g.row_ptr + lv + 1);
    if (!is_bfs(OP)) sv = ld_label_cg(p.lab + v);
  }
  int64_t deg = end - beg;
  // SSSP deferral: a vertex whose distance is still far above the frontier minimum, weighted by
  // the edges a premature expansion would waste, is kept for the next round (re-pushed with the
  // round's stamp, so at most once) instead of expanded.  The frontier's minimum vertex always
  // has slack <= 0, so every round expands at least one vertex (progress).
  if (is_sssp(OP) && rb.defer_k > 0) {
    const bool defer = valid && deg > 0 && ((int64_t)sv - dmin) * deg > rb.defer_k;
    if (__any_sync(FULL, defer)) {
      int kind = 0;
      if (defer) {
        const int32_t code = stamp_code<OP>(rb.stamp_id, 1);
        if (!has_far(OP) && rb.dense) atomicMax(p.stamp + v, code);  // mark (compaction pushes)
        else kind = stamp_claim(p.stamp + v, code) ? 1 : 0;
        q.dmin = min(q.dmin, sv);
        deg = 0;
      }
      if (has_far(OP) || !rb.dense) wpush<OP, DIST>(sm, q, p, rb, kind, v);
    }
  }
  {
    unsigned long long de = (unsigned long long)deg;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) de += __shfl_xor_sync(FULL, de, o);
    if (lane == 0) sm.fl_edges[threadIdx.x >> 5] += de;
  }

  // ---- small rounds (every warp holds at most one tile): degrees in [warp_t, cta_t) are expanded
  // by the popping warp itself, so a round without hubs needs no chunk phase (and no second
  // grid barrier)
  if (small_round) {
    uint32_t wm = __ballot_sync(FULL, deg >= p.ec.warp_t && deg < p.ec.cta_t);
    while (wm) {
      const int leader = __ffs(wm) - 1;
      wm &= wm - 1;
      const int64_t b = __shfl_sync(FULL, beg, leader);
      const int64_t e = __shfl_sync(FULL, end, leader);
      const int32_t s = __shfl_sync(FULL, sv, leader);
      if (lane == leader) deg = 0;
      process_range<OP, DIST>(sm, q, p, rb, b, e, s, lane);
    }
  }
  // ---- edge-balanced level: degree >= warp_t -> descriptors of <= chunk_edges edges, drained
  // by every warp of the grid in the chunk phase (one reservation per warp tile)
  {
    const bool big = deg >= p.ec.warp_t;
    const int64_t ce = p.ec.chunk_edges;
    // 32-bit division (a 64-bit one is a ~70-instruction subroutine call per lane)
    const uint32_t ce32 = (uint32_t)ce;
    const uint32_t nchl = big ? ((uint32_t)(deg < 0xfffe0000ll ? deg : 0xfffe0000ll) + ce32 - 1u) / ce32 : 0u;
    uint32_t incl = nchl;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t t = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += t;
    }
    const uint32_t tot = __shfl_sync(FULL, incl, 31);
    if (tot) {
      uint32_t cbase = 0;
      if (lane == 31) cbase = atomicAdd(rb.chunk_cnt, tot);
      cbase = __shfl_sync(FULL, cbase, 31);
      const uint32_t excl = cbase + incl - nchl;
      uint32_t bm = __ballot_sync(FULL, big);
      while (bm) {
        const int leader = __ffs(bm) - 1;
        bm &= bm - 1;
        const int64_t b = __shfl_sync(FULL, beg, leader);
        const int64_t e = __shfl_sync(FULL, end, leader);
        const uint32_t vv = __shfl_sync(FULL, v, leader);
        const int32_t s = __shfl_sync(FULL, sv, leader);
        const uint32_t nch = __shfl_sync(FULL, nchl, leader);
        const uint32_t off = __shfl_sync(FULL, excl, leader);
        for (uint32_t k = lane; k < nch; k += 32) {
          const uint32_t pos = off + k;
          const int64_t cb = b + (int64_t)k * ce;
          if (pos < rb.chunk_cap) {
            ChunkDesc d;
            d.beg_len = ((uint64_t)cb << 16) | (uint64_t)min(ce, e - cb);
            d.v = vv;
            d.sv = s;
            rb.chunks[pos] = d;
          } else {
            atomicOr(&p.ctl->overflow, 2u);
          }
        }
      }
    }
    if (big) deg = 0;
  }

  // ---- thread level (fine-grained): warp scan of the small degrees, shuffle owner search
  const uint32_t d = (uint32_t)deg;
  uint32_t incl = d;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += t;
  }
  const uint32_t total = __shfl_sync(FULL, incl, 31);
  const int64_t off = beg - (int64_t)(incl - d);  // edge of slot k (owned here) = off + k
  // kWin windows of 32 edge slots per iteration: each lane has kWin independent col/label chains in
  // flight (memory-level parallelism); owner of slot k = #lanes with inclusive prefix <= k
#ifndef IRGL_KWIN
#define IRGL_KWIN 4
#endif
#ifndef IRGL_KWIN_SSSP
#define IRGL_KWIN_SSSP 8  // SSSP-22 -2% at 8 windows, BFS flat (profiles/r2_kwin.txt)
#endif
  // (the multi-partition kernels keep 4: their remote staging leaves no registers for 8 — RMAT-24
  // P=2 SSSP 5.94 -> 6.22 ms with 8)
  constexpr int kWin = (is_sssp(OP) && !DIST) ? IRGL_KWIN_SSSP : IRGL_KWIN;
  for (uint32_t wb = 0; wb < total; wb += 32 * kWin) {
    uint32_t dst[kWin];
    int32_t wt[kWin], s[kWin], cur[kWin];
    bool act[kWin];
#pragma unroll
    for (int j = 0; j < kWin; ++j) {
      const uint32_t k = wb + 32 * j + lane;
      act[j] = k < total;
      uint32_t o = 0;
#pragma unroll
      for (uint32_t st = 16; st > 0; st >>= 1) {
        const uint32_t t = __shfl_sync(FULL, incl, o + st - 1);
        if (t <= k) o += st;
      }
      o = min(o, 31u);
      const int64_t eo = __shfl_sync(FULL, off, o);
      s[j] = __shfl_sync(FULL, sv, o);
      dst[j] = 0;
      wt[j] = 0;
      if (act[j]) {
        const int64_t ed = eo + k;
        dst[j] = (uint32_t)ld_stream(p.g.col + ed);
        if (w8_op(OP)) wt[j] = ld_stream_u8(p.g.w8 + ed);
        else if (is_sssp(OP)) wt[j] = ld_stream(p.g.w + ed);
      }
    }
#pragma unroll
    for (int j = 0; j < kWin; ++j) cur[j] = act[j] ? gather_cur<OP>(p, dst[j]) : 0;
    int kk[kWin];
    relax_batch<OP, kWin>(p, rb, q, act, cur, s, wt, dst, kk);
#pragma unroll
    for (int j = 0; j < kWin; ++j) {
      if (wb + 32 * j >= total) break;  // warp-uniform
      wpush<OP, DIST>(sm, q, p, rb, kk[j], dst[j]);
    }
  }
}

// Item phase: warp tiles of `width` items — 32 for large frontiers, fewer when the frontier is
// smaller than the grid's warps so that more warps share a small round (shorter critical path).
// The first tile of each warp is static (global warp id); when there are more tiles than warps
// the rest are fetched dynamically from tile_ctr (no atomics otherwise).
template <int OP, bool DIST>
__device__ void item_phase(Smem& sm, WarpQ& q, const KParams& p, const RoundBufs& rb) {
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  uint32_t width = 32;
  // host-orchestrated multi-partition rounds leave the in-count on the device (no host sync)
  const uint32_t nin = rb.nin_dev ? ld_ctl(rb.nin_dev) : rb.nin;
  while (width > 1 && (uint64_t)(width >> 1) * nwarps >= nin) width >>= 1;
  const uint32_t ntiles = (nin + width - 1) / width;
  const int32_t dmin = rb.defer_k <= 0 ? kInf
                       : rb.dmin_cur ? (int32_t)min(ld_ctl(rb.dmin_cur), (uint32_t)kInf)
                                     : rb.dmin_val;
  uint32_t t = gw;
  while (t < ntiles) {
    expand_warp_tile<OP, DIST>(sm, q, p, rb, t * width, width, dmin, ntiles <= nwarps, nin);
    if (ntiles <= nwarps) break;
#if defined(IRGL_TILE_STATIC) && IRGL_TILE_STATIC
    t += nwarps;
#else
    uint32_t nt = 0;
    if (lane_id() == 0) nt = nwarps + atomicAdd(rb.tile_ctr, 1u);
    t = __shfl_sync(FULL, nt, 0);
#endif
  }
}

// ---- chunk phase: every warp of the grid drains edge-chunk descriptors (grid-stride by warp;
// chunks are <= chunk_edges edges, so the phase is edge-balanced and its tail is one chunk).  The
// next descriptor is loaded while the current one is processed.
__device__ __forceinline__ ChunkDesc ld_desc(const ChunkDesc* p) {
  uint32_t a0, a1, a2, a3;  // rewritten every round: L2-coherent load
  asm volatile("ld.global.cg.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(a0), "=r"(a1), "=r"(a2), "=r"(a3) : "l"(p));
  ChunkDesc d;
  d.beg_len = ((uint64_t)a1 << 32) | a0;
  d.v = a2;
  d.sv = (int32_t)a3;
  return d;
}


template <int OP, bool DIST>
__device__ void chunk_phase(Smem& sm, WarpQ& q, const KParams& p, const RoundBufs& rb, uint32_t nch) {
  nch = min(nch, rb.chunk_cap);
  const uint32_t gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  const int gl = lane_id();
  if (nch * 2 <= nw) {
    // few chunks (latency-bound round): every chunk is split over P warps, so the phase costs one
    // or two 128-edge iterations per warp instead of chunk_edges / 128 sequential ones
    if (nch == 0) return;
    const uint32_t P = min(nw / nch, 16u);
    if (gw >= nch * P) return;
    const ChunkDesc d = ld_desc(rb.chunks + gw / P);
    const uint32_t part = gw % P;
    const int64_t b = (int64_t)(d.beg_len >> 16), len = (int64_t)(d.beg_len & 0xffffu);
    const int64_t per = (int64_t)(((((uint32_t)len + P - 1u) / P) + 3u) & ~3u);  // len < 2^16
    const int64_t b0 = b + part * per, e0 = min(b0 + per, b + len);
    if (b0 < e0) process_range<OP, DIST>(sm, q, p, rb, b0, e0, d.sv, gl);
    return;
  }
  // Software-pipelined drain: each iteration is one int4 group per lane (128 edges per warp);
  // the NEXT iteration's col/weight group (possibly the first group of the warp's next chunk) is
  // loaded before this iteration's gathers and atomics are waited on, so the DRAM latency of the
  // CSR stream is off the per-iteration dependency chain.
  uint32_t c = gw;
  if (c >= nch) return;
  const int32_t* __restrict__ col = p.g.col;
  const int32_t* __restrict__ wgt = p.g.w;
  ChunkDesc nx = (c + nw < nch) ? ld_desc(rb.chunks + c + nw) : ChunkDesc{};
  ChunkDesc cd = ld_desc(rb.chunks + c);
  int64_t b = (int64_t)(cd.beg_len >> 16);
  int64_t e = b + (int64_t)(cd.beg_len & 0xffffu);
  int32_t sv = cd.sv;
  int64_t q0 = b >> 2;
  int4 cc = make_int4(0, 0, 0, 0), ww = cc;
  uint32_t w8c = 0;
  {
    const int64_t qk = q0 + gl;
    if (qk < ((e + 3) >> 2)) {
      cc = ld_stream_v4(col + 4 * qk);
      if (w8_op(OP)) w8c = ld_stream_u32(p.g.w8 + 4 * qk);
      else if (is_sssp(OP)) ww = ld_stream_v4(wgt + 4 * qk);
    }
  }
  for (;;) {
    // position of the next iteration
    int64_t nq0 = q0 + 32, nb = b, ne = e;
    int32_t nsv = sv;
    bool more = true;
    if (nq0 >= ((e + 3) >> 2)) {
      c += nw;
      if (c >= nch) {
        more = false;
      } else {
        nb = (int64_t)(nx.beg_len >> 16);
        ne = nb + (int64_t)(nx.beg_len & 0xffffu);
        nsv = nx.sv;
        nq0 = nb >> 2;
        if (c + nw < nch) nx = ld_desc(rb.chunks + c + nw);
      }
    }
    int4 ncc = make_int4(0, 0, 0, 0), nww = ncc;
    uint32_t nw8 = 0;
    if (more) {
      const int64_t qk = nq0 + gl;
      if (qk < ((ne + 3) >> 2)) {
        ncc = ld_stream_v4(col + 4 * qk);
        if (w8_op(OP)) nw8 = ld_stream_u32(p.g.w8 + 4 * qk);
        else if (is_sssp(OP)) nww = ld_stream_v4(wgt + 4 * qk);
      }
    }
    // this iteration: 4 edges per lane
    const int64_t e0 = 4 * (q0 + gl);
    bool act[4];
    uint32_t d[4];
    int32_t wt[4], s4[4], cur[4];
    {
      const int32_t c4[4] = {cc.x, cc.y, cc.z, cc.w};
      const int32_t w4[4] = {w8_op(OP) ? w8_at(w8c, 0) : ww.x, w8_op(OP) ? w8_at(w8c, 1) : ww.y,
                             w8_op(OP) ? w8_at(w8c, 2) : ww.z, w8_op(OP) ? w8_at(w8c, 3) : ww.w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        act[t] = e0 + t >= b && e0 + t < e;
        d[t] = (uint32_t)c4[t];
        wt[t] = w4[t];
        s4[t] = sv;
      }
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) cur[t] = act[t] ? gather_cur<OP>(p, d[t]) : 0;
    int kk[4];
    relax_batch<OP, 4>(p, rb, q, act, cur, s4, wt, d, kk);
#pragma unroll
    for (int t = 0; t < 4; ++t) wpush<OP, DIST>(sm, q, p, rb, kk[t], d[t]);
    if (!more) break;
    q0 = nq0;
    b = nb;
    e = ne;
    sv = nsv;
    cc = ncc;
    ww = nww;
    w8c = nw8;
  }
}

// ---- dense-round compaction: the out worklist = the vertices marked this round (BFS: level ==
// LEVEL; SSSP / CC: stamp == the round's code), in vertex order; coalesced sweep over the
// partition's label (or stamp) array, pushes through the usual warp staging.
#ifndef IRGL_COMPACT_U
#define IRGL_COMPACT_U 1  // 1, 2, 4 within 1% on RMAT-22/24
#endif
template <int OP>
__device__ void compact_phase(Smem& sm, WarpQ& q, const KParams& p, const RoundBufs& rb) {
  const int64_t n = p.g.hi - p.g.lo;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  const int32_t* mark = is_bfs(OP) ? p.lab : p.stamp;
  const int32_t want = is_bfs(OP) ? rb.level : (rb.stamp_id << 1);
  if ((p.g.lo & 3) == 0) {
    // 4 consecutive marks per lane (one 16-byte load; 512 B per warp per step): a quarter of the
    // dependent load steps of the 1-mark loop, which left the sweep latency-bound (~70 us for
    // 16.7M marks)
    const int32_t* mb = mark + p.g.lo;
    constexpr int kU = IRGL_COMPACT_U;  // 16-byte groups per lane per step
    for (int64_t i0 = (((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~int64_t(31)) * 4 * kU; i0 < n;
         i0 += 4 * kU * T) {
      int32_t m[kU][4];
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t i = i0 + 128 * u + 4 * lane_id();
        if (i + 3 < n) {
          asm volatile("ld.global.cg.v4.s32 {%0,%1,%2,%3}, [%4];"
                       : "=r"(m[u][0]), "=r"(m[u][1]), "=r"(m[u][2]), "=r"(m[u][3]) : "l"(mb + i));
        } else {
#pragma unroll
          for (int j = 0; j < 4; ++j) m[u][j] = i + j < n ? ld_label_cg(mb + i + j) : 0;
        }
      }
#pragma unroll
      for (int u = 0; u < kU; ++u) {
        const int64_t i = i0 + 128 * u + 4 * lane_id();
#pragma unroll
        for (int j = 0; j < 4; ++j)
          wpush<OP, false>(sm, q, p, rb, (i + j < n && m[u][j] == want) ? 1 : 0, (uint32_t)(p.g.lo + i + j));
      }
    }
    return;
  }
  for (int64_t i0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~int64_t(31); i0 < n; i0 += T) {
    const int64_t i = i0 + lane_id();
    const uint32_t v = (uint32_t)(p.g.lo + i);
    const int kind = (i < n && ld_label_cg(mark + v) == want) ? 1 : 0;
    wpush<OP, false>(sm, q, p, rb, kind, v);
  }
}

// ---- near-far split: far pile -> near worklist / next far pile / dropped --------------------------
//   dist <  t_old            : already expanded when it dropped below the old threshold -> drop
//   t_old <= dist < threshold: near worklist
//   dist >= threshold        : next far pile (min kept distance -> minkeep)
__device__ void far_split(Smem& sm, WarpQ& q, const KParams& p, const RoundBufs& rb,
                          const uint32_t* far_in, uint32_t nfar, int32_t t_old,
                          unsigned int* minkeep) {
  uint32_t mymin = 0xffffffffu;
  const uint32_t T = (gridDim.x * blockDim.x);
  for (uint32_t i0 = (blockIdx.x * blockDim.x + threadIdx.x) & ~31u; i0 < nfar; i0 += T) {
    const uint32_t i = i0 + lane_id();
    int kind = 0;
    uint32_t v = 0;
    if (i < nfar) {
      v = ld_item(far_in + i);
      const int32_t dv = ld_label_cg(p.lab + v);
      if (dv >= t_old) {
        const int k = dv < rb.threshold ? 1 : 2;
        if (stamp_claim(p.stamp + v, stamp_code<kOpSsspNF>(rb.stamp_id, k))) {
          kind = k;
          if (kind == 2) mymin = min(mymin, (uint32_t)dv);
        }
        if (k == 1) q.dmin = min(q.dmin, dv);
      }
    }
    wpush<kOpSsspNF, false>(sm, q, p, rb, kind, v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mymin = min(mymin, __shfl_xor_sync(FULL, mymin, o));
  if (lane_id() == 0 && mymin != 0xffffffffu) atomicMin(minkeep, mymin);
}

template <int OP, bool DIST>
__global__ void __launch_bounds__(kBlock, minb_for(OP)) expand_kernel(KParams p, RoundBufs rb) {
  __shared__ std::conditional_t<DIST, SmemDist, Smem> sm;
  smem_init(sm);
  WarpQ q;
  item_phase<OP, DIST>(sm, q, p, rb);
  if constexpr (DIST) wflush_remote_all(sm, q, p);
  wflush_all<OP>(sm, q, p, rb);
}

template <int OP, bool DIST>
__global__ void __launch_bounds__(kBlock, minb_for(OP)) chunk_kernel(KParams p, RoundBufs rb) {
  __shared__ std::conditional_t<DIST, SmemDist, Smem> sm;
  smem_init(sm);
  WarpQ q;
  chunk_phase<OP, DIST>(sm, q, p, rb, ld_ctl(rb.chunk_cnt));
  if constexpr (DIST) wflush_remote_all(sm, q, p);
  wflush_all<OP>(sm, q, p, rb);
}

__global__ void __launch_bounds__(kBlock, IRGL_MINB) far_split_kernel(KParams p, RoundBufs rb,
                                                              const uint32_t* far_in,
                                                              const uint32_t* nfar_ptr,
                                                              int32_t t_old,
                                                              unsigned int* minkeep) {
  __shared__ Smem sm;
  smem_init(sm);
  WarpQ q;
  far_split(sm, q, p, rb, far_in, ld_ctl(nfar_ptr), t_old, minkeep);
  wflush_all<kOpSsspNF>(sm, q, p, rb);
}

// ---- E3: outlined Iterate.  One cooperative launch; rounds separated by grid.sync() --------------
// Worklist buffers alternate by round parity; counters rotate over three slots so the counter
// cleared during round r (slot (r+2)%3, last read during round r-1) is the out-counter of round
// r+1: no extra barrier is needed to reset it ("swap in/out and reset out").
// SyncRunningThreads with a broadcast: every CTA arrives (bar.sync, then one
// gpu-scope fence + atomic by thread 0); the LAST arriver evaluates `payload()` (the round's
// counters, final once everyone has arrived) and publishes {8-bit barrier tag, 56-bit payload}
// with one release store; the others spin on that word with acquire loads.  Compared with
// cg::grid.sync() followed by every thread re-reading the counters, the counters cost one L2 read
// by one thread instead of one same-address read per warp of the grid (~7,000 requests to one L2
// slice per round), and the value arrives with the release itself.  `post(w)` runs on thread 0
// of every CTA after the release (e.g. per-CTA reads of per-round cells into shared memory).
// The arrival counter and tag are monotonic within a launch (both wrap consistently mod 2^32 /
// 2^8: no CTA can be a whole barrier ahead of another), and the host zeroes them before it.
#ifndef IRGL_BARRIER_CG
#define IRGL_BARRIER_CG 1
#endif
template <class F, class G>
__device__ __forceinline__ unsigned long long grid_sync_bcast(Ctl* ctl, uint32_t& idx,
                                                              unsigned long long* slot,
                                                              F&& payload, G&& post) {
  ++idx;
#if IRGL_BARRIER_CG
  // cooperative-groups grid barrier, then thread 0 of each CTA reads the round's counters once
  // (592 reads of two L2 lines): 1.86 us per barrier on a 592-CTA grid against 2.83 us for the
  // last-arriver broadcast below (tools/barrier_probe.cu, profiles/r2_barrier_probe.txt)
  (void)ctl;
  cg::this_grid().sync();
  if (threadIdx.x == 0) {
    const unsigned long long w = payload() & ((1ull << 56) - 1);
    post(w);
    *slot = w;
  }
  __syncthreads();
  return *slot;
#endif
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned long long tag = (unsigned long long)(idx & 0xffu) << 56;
    __threadfence();
    const unsigned int old = atomicAdd(&ctl->gb_arrive, 1u);
    unsigned long long w;
    if (old == idx * gridDim.x - 1u) {
      __threadfence();
      w = tag | (payload() & ((1ull << 56) - 1));
      st_release_u64(&ctl->gb_release, w);
    } else {
      do {
        w = ld_acquire_u64(&ctl->gb_release);
      } while ((w & (0xffull << 56)) != tag);
    }
    w &= (1ull << 56) - 1;
    post(w);
    *slot = w;
  }
  __syncthreads();
  return *slot;
}
// {chunk count: 26 bits, out count: 30 bits} (the host caps chunk_cap below 2^26 and pipe
// capacities below 2^30)
__device__ __forceinline__ unsigned long long pack_counts(uint32_t nch, uint32_t nout) {
  return ((unsigned long long)min(nch, 0x3ffffffu) << 30) | min(nout, 0x3fffffffu);
}
__device__ __forceinline__ uint32_t unpack_nch(unsigned long long w) { return (uint32_t)(w >> 30); }
__device__ __forceinline__ uint32_t unpack_nout(unsigned long long w) { return (uint32_t)(w & 0x3fffffffu); }

__device__ __forceinline__ int slot3(const PersistArgs& a, uint32_t i) {
  const uint32_t m = i % 3;
  return m == 0 ? a.slot[0] : (m == 1 ? a.slot[1] : a.slot[2]);
}

// Fused traversal prologue (PersistArgs::src): labels = INF (16-byte stores), visited bitmap = 0,
// control block reset (what ctl_prepare_kernel, pipe_counters and the pipe init do), then
// Initial [src]: in = {src}, label[src] = 0 (and its visited bit) after a grid barrier, and a second
// barrier before round 0 reads any of it.
__device__ void traversal_prologue(const KParams& p, const PersistArgs& a) {
  const int64_t n = a.n;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t n4 = n >> 2;  // the label array is cudaMalloc'd: 16-byte aligned
  const int4 inf4 = make_int4(kInf, kInf, kInf, kInf);
  for (int64_t i = t; i < n4; i += T) reinterpret_cast<int4*>(p.lab)[i] = inf4;
  for (int64_t i = (n4 << 2) + t; i < n; i += T) p.lab[i] = kInf;
  if (a.reset_vis)
    for (int64_t i = t; i < ((n + 31) >> 5); i += T) a.reset_vis[i] = 0u;
  const uint32_t v = a.src_map ? (uint32_t)a.src_map[a.src] : (uint32_t)a.src;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    Ctl* c = p.ctl;
    for (int k = 0; k < 4; ++k) c->cnt[k] = 0u;
    c->cnt[a.slot[0]] = 1u;
    for (int k = 0; k < 3; ++k) {
      c->chunk_cnt[k] = 0u;
      c->tile_ctr[k] = 0u;
      c->dmin[k] = 0xffffffffu;  // round 0: no frontier minimum yet (no deferral)
      c->mf[k] = 0ull;
      c->bu_found[k] = 0ull;
    }
    c->far_cnt[0] = c->far_cnt[1] = 0u;
    c->overflow = 0u;
    c->popped = c->pushes = c->rounds = c->bu_scanned = 0ull;
    c->edges = c->remote = 0ull;
    c->gb_arrive = 0u;
    c->gb_release = 0ull;
    a.buf_a[0] = v;
  }
  cg::this_grid().sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    p.lab[v] = 0;
    if (a.reset_vis) a.reset_vis[v >> 5] |= 1u << (v & 31);
  }
  cg::this_grid().sync();
}

template <int OP>
__global__ void __launch_bounds__(kBlock, minb_for(OP)) persistent_kernel(KParams p, PersistArgs a) {
  __shared__ Smem sm;
  smem_init(sm);
  cg::grid_group grid = cg::this_grid();
  WarpQ q;
  uint32_t* cnt = p.ctl->cnt;
  const bool nf = has_far(OP) && a.delta > 0;
  int32_t threshold = nf ? a.delta : kInf;
  const int32_t s0 = a.stamp_base ? *(volatile int32_t*)a.stamp_base + 1 : a.stamp0;
  int32_t sid = s0;             // unique stamp ids: rounds and splits
  uint32_t fsel = 0;            // which far buffer is current
  uint32_t nsplit = 0;          // splits so far (selects the minkeep slot)
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  if (a.src >= 0) traversal_prologue(p, a);
  uint32_t nin_next = ld_ctl(cnt + slot3(a, 0));  // round r's in-count = round r-1's out-count
  __shared__ unsigned long long bslot;  // barrier broadcast
  __shared__ RoundBufs srb;             // this round's view (no near-far)
  __shared__ int32_t s_dmin;            // deferral: frontier minimum of the next round
  uint32_t bidx = 0;
  const bool dfr = (is_sssp(OP)) && a.defer_k > 0;
  if (threadIdx.x == 0) s_dmin = dfr ? (int32_t)min(ld_ctl(&p.ctl->dmin[0]), (uint32_t)kInf) : kInf;
  __syncthreads();  // round 0 reads s_dmin in every thread
  if (leader && a.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a.trace[8 * a.trace_cap]));
  for (uint32_t r = 0;; ++r) {
    uint32_t* cin = cnt + slot3(a, r);
    uint32_t* cout = cnt + slot3(a, r + 1);
    if (leader) {
      cnt[slot3(a, r + 2)] = 0;
      p.ctl->chunk_cnt[(r + 1) % 3] = 0;
      p.ctl->tile_ctr[(r + 1) % 3] = 0;
      p.ctl->dmin[(r + 2) % 3] = 0xffffffffu;  // last read at the start of round r-1
    }
    RoundBufs rb;
    rb.in = (r & 1) ? a.buf_b : a.buf_a;
    rb.nin = nin_next;
    rb.nin_dev = nullptr;
    (void)cin;
    rb.out = (r & 1) ? a.buf_a : a.buf_b;
    rb.out_cnt = cout;
    rb.cap = a.cap;
    rb.chunks = a.chunks;
    rb.chunk_cnt = &p.ctl->chunk_cnt[r % 3];
    rb.chunk_cap = a.chunk_cap;
    rb.tile_ctr = &p.ctl->tile_ctr[r % 3];
    rb.level = a.level0 + (int32_t)r;
    rb.stamp_id = sid++;
    rb.far = fsel ? a.far_b : a.far_a;
    rb.far_cnt = &p.ctl->far_cnt[fsel];
    rb.far_cap = a.far_cap;
    rb.threshold = threshold;
    rb.mf_acc = nullptr;
    rb.defer_k = (is_sssp(OP)) ? a.defer_k : 0;
    rb.dmin_cur = nullptr;
    rb.dmin_val = s_dmin;  // written by thread 0 before the barrier that ended round r-1
    // dense round: relaxations mark (fire-and-forget stores / REDs) instead of pushing, and a
    // compaction sweep builds the out worklist after the expansion barrier
    rb.dense = (!has_far(OP) && a.dense_min > 0 && (int64_t)nin_next >= a.dense_min) ? 1 : 0;
    rb.dmin_next = rb.defer_k > 0 ? &p.ctl->dmin[(r + 1) % 3] : nullptr;
    // Without near-far the round's view lives in shared memory (written by thread 0 between two
    // CTA barriers): the expansion then reads its pointers from smem at the use sites instead of
    // holding ~20 registers of per-round state live across the hot loops.
    const RoundBufs* rp = &rb;
    if constexpr (!has_far(OP)) {
      __syncthreads();  // readers of the previous round's view are done
      if (threadIdx.x == 0) srb = rb;
      __syncthreads();
      rp = &srb;
    }
    const RoundBufs& rr = *rp;
    item_phase<OP, false>(sm, q, p, rr);
    if (leader && a.trace && r < a.trace_cap) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a.trace[8 * r + 4]));
    wflush_all<OP>(sm, q, p, rr);
    if (leader && a.trace && r < a.trace_cap) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a.trace[8 * r + 5]));
    if (a.trace && r < a.trace_cta && threadIdx.x == 0)
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a.trace[8 * (size_t)a.trace_cap + 1 + (size_t)r * gridDim.x + blockIdx.x]));
    // the deferral minimum of round r+1 is final at the round's last barrier: thread 0 of each CTA
    // fetches it into shared memory there (no per-warp reads of one hot cell)
    auto fetch_dmin = [&]() {
      if (dfr) s_dmin = (int32_t)min(ld_ctl(&p.ctl->dmin[(r + 1) % 3]), (uint32_t)kInf);
    };
    unsigned long long w = grid_sync_bcast(
        p.ctl, bidx, &bslot, [&]() { return pack_counts(ld_ctl(rb.chunk_cnt), ld_ctl(cout)); },
        [&](unsigned long long v) { if (unpack_nch(v) == 0) fetch_dmin(); });
    if (leader && a.trace && r < a.trace_cap) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a.trace[8 * r + 6]));
    const uint32_t nch = unpack_nch(w);
    uint32_t nout = unpack_nout(w);
    if (nch) {
      chunk_phase<OP, false>(sm, q, p, rr, nch);
      wflush_all<OP>(sm, q, p, rr);
      w = grid_sync_bcast(p.ctl, bidx, &bslot, [&]() { return pack_counts(0, ld_ctl(cout)); },
                          [&](unsigned long long) { fetch_dmin(); });
      nout = unpack_nout(w);
    if (leader && a.trace && r < a.trace_cap) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a.trace[8 * r + 7]));
    }
    if constexpr (!has_far(OP)) {
      if (rr.dense) {
        compact_phase<OP>(sm, q, p, rr);
        wflush_all<OP>(sm, q, p, rr);
        w = grid_sync_bcast(p.ctl, bidx, &bslot, [&]() { return pack_counts(0, ld_ctl(cout)); },
                            [&](unsigned long long) {});
        nout = unpack_nout(w);
      }
    }
    if constexpr (has_far(OP)) if (nf) {
      // near frontier exhausted: advance the threshold and split the far pile; a pile past half
      // its capacity is compacted (split at the unchanged threshold) even when near is not empty
      uint32_t nfar = min(ld_ctl(rb.far_cnt), a.far_cap);  // beyond far_cap: dropped and flagged
      bool advance = nout == 0;
      if ((advance && nfar > 0) || nfar > a.far_cap / 2) {
        for (;;) {
          const int32_t t_old = threshold;
          if (advance) threshold += a.delta;
          // slot nsplit&1 was last read after split nsplit-2, i.e. before the barrier every CTA
          // passed on its way here: safe to reset (the other slot may still be being read)
          unsigned int* mk = &p.ctl->minkeep[nsplit & 1];
          ++nsplit;
          if (leader) {
            p.ctl->far_cnt[fsel ^ 1] = 0;
            *mk = 0xffffffffu;
          }
          grid.sync();
          RoundBufs sb = rb;
          sb.far = fsel ? a.far_a : a.far_b;  // next far pile
          sb.far_cnt = &p.ctl->far_cnt[fsel ^ 1];
          sb.threshold = threshold;
          sb.stamp_id = sid++;
          far_split(sm, q, p, sb, rb.far, nfar, t_old, mk);
          wflush_all<OP>(sm, q, p, sb);
          grid.sync();
          fsel ^= 1;
          rb.far = sb.far;
          rb.far_cnt = sb.far_cnt;
          nout = ld_ctl(cout);
          nfar = min(ld_ctl(rb.far_cnt), a.far_cap);  // beyond far_cap: dropped and flagged
          if (nout > 0 || nfar == 0) break;
          threshold = (int32_t)ld_ctl(mk);  // next pass moves at least the minimum
          advance = true;
        }
      }
    }
    if (leader) {
      p.ctl->popped += rb.nin;
      p.ctl->pushes += nout;
      if (a.trace && r < a.trace_cap) {  // per-round trace: end time, |in|, |out|, edges so far
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[8 * r + 0] = t;
        a.trace[8 * r + 1] = rb.nin | ((unsigned long long)nch << 32);
        a.trace[8 * r + 2] = nout;
        a.trace[8 * r + 3] = *(volatile unsigned long long*)&p.ctl->edges;
      }
    }
    nin_next = nout;
    // Iterate termination: in empty (next round) [Or rounds >= max_rounds]; an out count beyond
    // the worklist capacity (pushes dropped, overflow flagged) ends the loop too — the next round
    // would read past the buffer — and the host reports IRGL_E_WL_OVERFLOW
    if (nout == 0 || nout > a.cap || (a.max_rounds > 0 && (int64_t)r + 1 >= a.max_rounds)) {
      if (leader) {
        p.ctl->rounds = r + 1;
        p.ctl->exit_in_slot = (int32_t)((r + 1) & 1);
        p.ctl->stamp_used = (uint32_t)(sid - s0);
        if (a.stamp_base) *a.stamp_base = sid - 1;  // every thread read it before the 1st barrier
        p.ctl->far_sel = fsel;
      }
      break;
    }
  }
}

// ---- E3 across partitions: the distributed persistent kernel (DistPersistArgs, kernels.h) ----------
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned ld_acquire_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_release_sys(unsigned* p, unsigned v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

// The partition's leader arrives at rendezvous k (1-based, monotonic within the launch) and waits
// for every partition.  False when some partition gave up: a peer that does not arrive within
// spin_ns (kernels not co-resident) sets the sticky abort word, and every partition leaves its
// loop at its next rendezvous — a bounded failure the host reports, never a hang.  The grid
// barrier before the arrival orders this partition's inbox stores (other CTAs) before the
// system-scope release; the acquire orders the peers' stores before this partition's reads.
__device__ bool x_arrive_wait(const DistPersistArgs& da, uint32_t k) {
  __threadfence_system();
  red_release_sys(&da.xr->arrive, 1u);
  const unsigned target = da.xbase + k * (unsigned)da.nparts;
  const unsigned long long t0 = gtimer();
  while ((int)(ld_acquire_sys(&da.xr->arrive) - target) < 0) {
    if (ld_ctl(&da.xr->abort)) return false;
    if (gtimer() - t0 > da.spin_ns) {
      atomicExch_system(&da.xr->abort, 1u);
      return false;
    }
    __nanosleep(32);
  }
  return ld_ctl(&da.xr->abort) == 0;
}

// Grid barrier + rendezvous + grid barrier; the leader's outcome reaches every CTA through
// Ctl::x_word.  PUBLISH (the round's end): the leader first clears the consumed inbox counters
// (senders write the next round's only after this rendezvous), posts the partition's out count and
// overflow flags, and after the rendezvous sums everyone's.
template <bool PUBLISH>
__device__ __forceinline__ void x_meet(const KParams& p, const DistPersistArgs& da, uint32_t k,
                                       const uint32_t* cout, uint32_t* s_x, bool reset_sent = false,
                                       const unsigned long long* mf = nullptr) {
  cg::this_grid().sync();
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    const int me = p.dr.me;
    if (reset_sent)  // the pack has read them: the next round's flushes count from zero
      for (int o = 0; o < da.nparts; ++o) p.dr.send_cnt[o] = 0u;
    if (PUBLISH) {
      uint32_t fl = ld_ctl(&p.ctl->overflow) & 7u;
      for (int s = 0; s < da.nparts; ++s)
        if (s != me) {
          if (ld_ctl(da.recv_cnt + s) > (uint32_t)p.dr.part_size) fl |= 4u;
          da.recv_cnt[s] = 0u;
        }
      *(volatile uint32_t*)&da.xr->outc[me] = ld_ctl(cout);
      *(volatile uint32_t*)&da.xr->flags[me] = fl;
      if (mf) *(volatile unsigned long long*)&da.xr->mfc[me] = *(volatile const unsigned long long*)mf;
    }
    const bool ok = x_arrive_wait(da, k);
    unsigned long long tot = 0, mft = 0;
    uint32_t fl = 0;
    if (PUBLISH && ok)
      for (int s = 0; s < da.nparts; ++s) {
        tot += ld_ctl(&da.xr->outc[s]);
        fl |= ld_ctl(&da.xr->flags[s]);
        if (mf) mft += *(volatile const unsigned long long*)&da.xr->mfc[s];
      }
    p.ctl->x_word[0] = ok ? 1u : 0u;
    p.ctl->x_word[1] = (uint32_t)min(tot, 0xffffffffull);
    p.ctl->x_word[2] = fl;
    p.ctl->x_mf = mft;
  }
  cg::this_grid().sync();
  if (threadIdx.x < 3) s_x[threadIdx.x] = ld_ctl(&p.ctl->x_word[threadIdx.x]);
  __syncthreads();
}

// Sender side, after the whole expansion: the value of every update this partition stored in an
// owner's inbox (its label of the vertex now — the lowest it reached this round), written beside
// the id (a remote store when the owner is another GPU).
template <int OP>
__device__ void pack_sent(const KParams& p, const DistPersistArgs& da) {
  const uint32_t T = gridDim.x * blockDim.x;
  for (int o = 0; o < da.nparts; ++o) {
    if (o == p.dr.me || !p.dr.inbox_val[o]) continue;
    const uint32_t n = min(ld_ctl(p.dr.send_cnt + o), (uint32_t)p.dr.part_size);
    const uint32_t* ids = p.dr.send + (int64_t)o * p.dr.part_size;
    int32_t* vals = p.dr.inbox_val[o];
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += T)
      vals[i] = ld_label_cg(p.lab + ld_item(ids + i));
  }
}

// Owner side of the round's exchange: every sender's inbox segment with the values the senders
// stored (their ghost label of the vertex at the flush: a real path length, so a valid
// candidate), relaxed and pushed into this partition's out worklist with this round's stamp.
template <int OP>
__device__ void apply_inbox(Smem& sm, WarpQ& q, const KParams& p, const RoundBufs& rb,
                            const DistPersistArgs& da) {
  const uint32_t T = gridDim.x * blockDim.x;
  for (int s = 0; s < da.nparts; ++s) {
    if (s == p.dr.me) continue;
    const uint32_t n = min(ld_ctl(da.recv_cnt + s), (uint32_t)p.dr.part_size);
    const uint32_t* seg = da.recv + (int64_t)s * p.dr.part_size;
    const int32_t* vseg = is_bfs(OP) ? nullptr : da.recv_val + (int64_t)s * p.dr.part_size;
    for (uint32_t i0 = blockIdx.x * blockDim.x + (threadIdx.x & ~31u); i0 < n; i0 += T) {
      const uint32_t i = i0 + lane_id();
      int kind = 0;
      uint32_t v = 0;
      if (i < n) {
        v = ld_item(seg + i);
        const int32_t cur = gather_cur<OP>(p, v);
        const int32_t val = is_bfs(OP) ? 0 : ld_label_cg(vseg + i);
        kind = relax_with<OP>(p, rb, q, cur, val, 0, v);
      }
      wpush<OP, false>(sm, q, p, rb, kind, v);
    }
  }
}

template <int OP>
// (the operators' own occupancy: BFS at 48 warps / SM beat 32 by 4%, SSSP at 32 beat 48 — spills —
// by 17%, RMAT-24 P=2, profiles/r2_dist_outlined.txt)
__global__ void __launch_bounds__(kBlock, minb_for(OP)) dist_persistent_kernel(KParams p, DistPersistArgs da) {
  __shared__ SmemDist sm;
  smem_init(sm);
  WarpQ q;
  const PersistArgs& a = da.pa;
  uint32_t* cnt = p.ctl->cnt;
  const int32_t s0 = a.stamp0;
  int32_t sid = s0;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  uint32_t nin_next = ld_ctl(cnt + slot3(a, 0));
  __shared__ unsigned long long bslot;
  __shared__ RoundBufs srb;
  __shared__ int32_t s_dmin;
  __shared__ uint32_t s_x[3];
  uint32_t bidx = 0, xk = 0;
  const bool dfr = is_sssp(OP) && a.defer_k > 0;
  if (threadIdx.x == 0) s_dmin = dfr ? (int32_t)min(ld_ctl(&p.ctl->dmin[0]), (uint32_t)kInf) : kInf;
  __syncthreads();
  // hello: every partition's kernel is resident (and every inbox counter zeroed, on its own
  // stream before its launch) before anything is written; a failed hello leaves all state as it
  // was, so the host can run the Iterate with host rounds instead
  x_meet<false>(p, da, ++xk, cnt, s_x);
  if (!s_x[0]) {
    if (leader) {
      p.ctl->rounds = 0;
      p.ctl->stamp_used = 0;
      p.ctl->x_word[3] = 0;
    }
    return;
  }
  for (uint32_t r = 0;; ++r) {
    uint32_t* cout = cnt + slot3(a, r + 1);
    if (leader) {
      cnt[slot3(a, r + 2)] = 0;
      p.ctl->chunk_cnt[(r + 1) % 3] = 0;
      p.ctl->tile_ctr[(r + 1) % 3] = 0;
      p.ctl->dmin[(r + 2) % 3] = 0xffffffffu;
    }
    RoundBufs rb{};
    rb.in = (r & 1) ? a.buf_b : a.buf_a;
    rb.nin = nin_next;
    rb.out = (r & 1) ? a.buf_a : a.buf_b;
    rb.out_cnt = cout;
    rb.cap = a.cap;
    rb.chunks = a.chunks;
    rb.chunk_cnt = &p.ctl->chunk_cnt[r % 3];
    rb.chunk_cap = a.chunk_cap;
    rb.tile_ctr = &p.ctl->tile_ctr[r % 3];
    rb.level = a.level0 + (int32_t)r;
    rb.stamp_id = sid++;
    rb.threshold = kInf;
    rb.defer_k = is_sssp(OP) ? a.defer_k : 0;
    rb.dmin_val = s_dmin;
    rb.dmin_next = rb.defer_k > 0 ? &p.ctl->dmin[(r + 1) % 3] : nullptr;
    __syncthreads();  // readers of the previous round's view are done
    if (threadIdx.x == 0) srb = rb;
    __syncthreads();
    const RoundBufs& rr = srb;
    // 1. expansion of this partition's in-worklist; remote updates into the owners' inboxes
    item_phase<OP, true>(sm, q, p, rr);
    wflush_remote_all(sm, q, p);
    wflush_all<OP>(sm, q, p, rr);
    const unsigned long long w = grid_sync_bcast(
        p.ctl, bidx, &bslot, [&]() { return pack_counts(ld_ctl(rr.chunk_cnt), 0); },
        [](unsigned long long) {});
    const uint32_t nch = unpack_nch(w);
    if (nch) {
      chunk_phase<OP, true>(sm, q, p, rr, nch);
      wflush_remote_all(sm, q, p);
      wflush_all<OP>(sm, q, p, rr);
    }
    // IRGL_DIST_TRACE: the leader stamps %globaltimer at the phase boundaries of each round
    // {expansion done, inboxes complete, apply done, sums known}
    unsigned long long* tr = (a.trace && r < a.trace_cap) ? a.trace + 4 * (size_t)r : nullptr;
    if (leader && tr) {
      cg::this_grid().sync();
      tr[0] = gtimer();
    } else if (tr) {
      cg::this_grid().sync();
    }
    // values of the remote updates (SSSP / CC_LP), then 2. every inbox is complete
    if (!is_bfs(OP)) {
      cg::this_grid().sync();
      pack_sent<OP>(p, da);
    }
    x_meet<false>(p, da, ++xk, cout, s_x, !is_bfs(OP));
    if (leader && tr) tr[1] = gtimer();
    bool stop = !s_x[0];
    if (!stop) {
      // 3. owner-side apply, 4. publish and sum the out counts
      apply_inbox<OP>(sm, q, p, rr, da);
      wflush_all<OP>(sm, q, p, rr);
      if (tr) cg::this_grid().sync();
      if (leader && tr) tr[2] = gtimer();
      x_meet<true>(p, da, ++xk, cout, s_x);
      if (leader && tr) tr[3] = gtimer();
      if (threadIdx.x == 0 && dfr) s_dmin = (int32_t)min(ld_ctl(&p.ctl->dmin[(r + 1) % 3]), (uint32_t)kInf);
      __syncthreads();
      stop = !s_x[0] || s_x[1] == 0 || s_x[2] != 0 || (a.max_rounds > 0 && (int64_t)r + 1 >= a.max_rounds);
    }
    const uint32_t nout = ld_ctl(cout);
    if (leader) {
      p.ctl->popped += rr.nin;
      p.ctl->pushes += nout;
    }
    nin_next = nout;
    if (stop) {
      if (leader) {
        p.ctl->rounds = r + 1;
        p.ctl->exit_in_slot = (int32_t)((r + 1) & 1);
        p.ctl->stamp_used = (uint32_t)(sid - s0);
        p.ctl->overflow |= s_x[2] & 3u;  // any partition's overflow fails the Iterate
        p.ctl->x_word[3] = s_x[0] ? xk : 0u;  // rendezvous completed (0: a partition gave up)
      }
      break;
    }
  }
}

// ---- F1: direction-optimising BFS (outlined, one partition) -----------------------------------------
// Bottom-up round at level L: every unvisited vertex scans its neighbours for a parent at level
// L-1 and stops at the first one (Beamer et al.).  Only the owning thread writes level[v], so a
// plain store suffices; a neighbour already set to L in this round is not a parent.
// Bottom-up round: every unvisited vertex scans its neighbours for a parent on level L-1, 4 at a
// time (the 4 column loads, then the 4 level gathers, in flight together: one dependent round trip
// per 4 candidates); the first parent in CSR order wins.  Found vertices are pushed, so the out
// worklist is the level-L frontier if the next round runs top-down (no compaction sweep).  `sc`
// counts the edges actually loaded.
__device__ void bu_phase(Smem& sm, WarpQ& q, const KParams& p, const RoundBufs& rb, int64_t n,
                         int32_t L, unsigned long long* found, unsigned long long* found_deg,
                         unsigned long long* scanned) {
  unsigned long long f = 0, fd = 0, sc = 0;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  for (int64_t v0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); v0 < n; v0 += T) {
    const int64_t v = v0 + lane_id();
    bool hit = false;
    // unvisited?  the visited bitmap (exact in DO-BFS) is one word per 32 lanes; else the level
    bool open = v < n;
    if (open) {
      if (p.vis) open = !((ld_label(reinterpret_cast<const int32_t*>(p.vis) + (v >> 5)) >> (v & 31)) & 1);
      else open = ld_label(p.lab + v) == kInf;
    }
    if (open) {
      const int64_t b = __ldg(p.g.row_ptr + v), e = __ldg(p.g.row_ptr + v + 1);
      for (int64_t k = b; k < e; k += 4) {
        int32_t u[4], l[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) u[j] = k + j < e ? ld_stream(p.g.col + k + j) : -1;
#pragma unroll
        for (int j = 0; j < 4; ++j) l[j] = u[j] >= 0 ? ld_label(p.lab + u[j]) : kInf;
        sc += (unsigned long long)(e - k < 4 ? e - k : 4);
#pragma unroll
        for (int j = 0; j < 4; ++j) hit |= l[j] == L - 1;
        if (hit) break;
      }
      if (hit) {
        p.lab[v] = L;
        if (p.vis) atomicOr(p.vis + (v >> 5), 1u << (v & 31));  // keep the bitmap exact
        ++f;
        fd += (unsigned long long)(e - b);
      }
    }
    wpush<IRGL_OP_BFS, false>(sm, q, p, rb, hit ? 1 : 0, (uint32_t)v);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    f += __shfl_xor_sync(FULL, f, o);
    fd += __shfl_xor_sync(FULL, fd, o);
    sc += __shfl_xor_sync(FULL, sc, o);
  }
  if (lane_id() == 0) {
    if (f) atomicAdd(found, f);
    if (fd) atomicAdd(found_deg, fd);
    if (sc) atomicAdd(scanned, sc);
  }
}

#ifndef IRGL_DO_MINB
#define IRGL_DO_MINB IRGL_MINB
#endif
__global__ void __launch_bounds__(kBlock, IRGL_DO_MINB) persistent_bfs_do_kernel(KParams p, PersistArgs a) {
  __shared__ Smem sm;
  smem_init(sm);
  cg::grid_group grid = cg::this_grid();
  WarpQ q;
  uint32_t* cnt = p.ctl->cnt;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  if (leader && a.trace) asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(a.trace[8 * a.trace_cap]));
  constexpr double kAlpha = 14.0, kBeta = 24.0;  // Beamer's switching constants
  bool bottom_up = false;
  uint32_t nbu = 0;
  unsigned long long explored = 0;               // edges of vertices already discovered
  const int32_t s0 = a.stamp_base ? *(volatile int32_t*)a.stamp_base + 1 : a.stamp0;
  if (a.src >= 0) traversal_prologue(p, a);
  uint32_t nin_next = ld_ctl(cnt + slot3(a, 0));
  for (uint32_t r = 0;; ++r) {
    uint32_t* cout = cnt + slot3(a, r + 1);
    if (leader) {
      cnt[slot3(a, r + 2)] = 0;
      p.ctl->chunk_cnt[(r + 1) % 3] = 0;
      p.ctl->tile_ctr[(r + 1) % 3] = 0;
      p.ctl->mf[(r + 1) % 3] = 0;
      p.ctl->bu_found[(r + 1) % 3] = 0;
    }
    RoundBufs rb;
    rb.in = (r & 1) ? a.buf_b : a.buf_a;
    rb.nin = nin_next;
    rb.nin_dev = nullptr;
    rb.out = (r & 1) ? a.buf_a : a.buf_b;
    rb.out_cnt = cout;
    rb.cap = a.cap;
    rb.chunks = a.chunks;
    rb.chunk_cnt = &p.ctl->chunk_cnt[r % 3];
    rb.chunk_cap = a.chunk_cap;
    rb.tile_ctr = &p.ctl->tile_ctr[r % 3];
    rb.level = a.level0 + (int32_t)r;
    rb.stamp_id = s0 + (int32_t)r;
    rb.far = nullptr;
    rb.far_cnt = nullptr;
    rb.far_cap = 0;
    rb.threshold = kInf;
    rb.mf_acc = &p.ctl->mf[r % 3];
    rb.dense = 0;
    rb.defer_k = 0;
    rb.dmin_cur = nullptr;
    rb.dmin_next = nullptr;
    uint64_t nf, mf;
    if (!bottom_up) {
      item_phase<kOpBfsDO, false>(sm, q, p, rb);
      wflush_all<kOpBfsDO>(sm, q, p, rb);
      grid.sync();
      const uint32_t nch = ld_ctl(rb.chunk_cnt);
      nf = ld_ctl(cout);
      if (nch) {
        chunk_phase<kOpBfsDO, false>(sm, q, p, rb, nch);
        wflush_all<kOpBfsDO>(sm, q, p, rb);
        grid.sync();
        nf = ld_ctl(cout);
      }
      mf = *(volatile unsigned long long*)&p.ctl->mf[r % 3];
    } else {
      bu_phase(sm, q, p, rb, a.n, rb.level, &p.ctl->bu_found[r % 3], &p.ctl->mf[r % 3],
               &p.ctl->bu_scanned);
      {
        RoundBufs cb = rb;
        cb.mf_acc = nullptr;
        wflush_all<IRGL_OP_BFS>(sm, q, p, cb);
      }
      grid.sync();
      nf = *(volatile unsigned long long*)&p.ctl->bu_found[r % 3];
      mf = *(volatile unsigned long long*)&p.ctl->mf[r % 3];
      ++nbu;
    }
    explored += mf;
    if (leader) {
      p.ctl->popped += rb.nin;
      p.ctl->pushes += nf;
      if (a.trace && r < a.trace_cap) {  // per-round trace (nch field = 1 for a bottom-up round)
        unsigned long long t;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
        a.trace[8 * r + 0] = t;
        a.trace[8 * r + 1] = rb.nin | ((unsigned long long)(bottom_up ? 1 : 0) << 32);
        a.trace[8 * r + 2] = nf;
        a.trace[8 * r + 3] = *(volatile unsigned long long*)&p.ctl->edges +
                             *(volatile unsigned long long*)&p.ctl->bu_scanned;
      }
    }
    // done also when the frontier overflowed the worklist (the next round would read past it)
    const bool done = nf == 0 || nf > a.cap || (a.max_rounds > 0 && (int64_t)r + 1 >= a.max_rounds);
    if (!done) {
      // direction for the next round (uniform: every thread reads the same counters)
      const double mu = (double)a.m - (double)explored;
      bool next_bu = bottom_up;
      if (!bottom_up && (double)mf > mu / kAlpha) next_bu = true;
      else if (bottom_up && (double)nf < (double)a.n / kBeta) next_bu = false;
      // bottom-up -> top-down: the bottom-up round pushed its finds, so the out worklist is
      // already the level-L frontier
      bottom_up = next_bu;
    }
    nin_next = (uint32_t)nf;
    if (done) {
      if (leader) {
        p.ctl->rounds = r + 1;
        p.ctl->exit_in_slot = (int32_t)((r + 1) & 1);
        p.ctl->stamp_used = r + 1;
        if (a.stamp_base) *a.stamp_base = s0 + (int32_t)r;
        p.ctl->bu_rounds = nbu;
      }
      break;
    }
  }
}

// ---- F1 on a vertex-partitioned graph: direction-optimising BFS rounds ---------------------------
// The frontier's size and edge count per partition (Beamer's switch needs both, summed over the
// partitions): out2 = {|in|, sum of the in-items' degrees}.
__global__ void frontier_stats_kernel(const uint32_t* items, const uint32_t* cnt, const int64_t* rp,
                                      int64_t lo, unsigned long long* out2) {
  const uint32_t n = *(volatile const uint32_t*)cnt;
  unsigned long long d = 0;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const int64_t v = (int64_t)items[i] - lo;
    d += (unsigned long long)(rp[v + 1] - rp[v]);
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) d += __shfl_xor_sync(FULL, d, o);
  if (lane_id() == 0 && d) atomicAdd(out2 + 1, d);
  if (blockIdx.x == 0 && threadIdx.x == 0) atomicAdd(out2, (unsigned long long)n);
}

// The global frontier as an n-bit bitmap: partition ranges are multiples of 32 vertices
// (partition_ranges), so each partition fills its own words and the words are exchanged as they are.
__global__ void frontier_bits_kernel(const uint32_t* items, const uint32_t* cnt, uint32_t* bits) {
  const uint32_t n = *(volatile const uint32_t*)cnt;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t v = items[i];
    atomicOr(bits + (v >> 5), 1u << (v & 31));
  }
}

// Bottom-up round of one partition: every owned unvisited vertex scans its (global-id) neighbours
// for one in the level-(L-1) frontier (the blocked bitmap) and stops at the first; only the owner
// writes its level, so no remote update is needed.  Finds are pushed (the next frontier).
template <int OP>
__device__ void bu_part_phase(Smem& sm, WarpQ& q, const KParams& p, const RoundBufs& rb, const uint32_t* fbits,
                              unsigned long long* scanned) {
  const int64_t n = p.g.hi - p.g.lo;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  unsigned long long sc = 0;
  for (int64_t v0 = (int64_t)blockIdx.x * blockDim.x + (threadIdx.x & ~31); v0 < n; v0 += T) {
    const int64_t lv = v0 + lane_id();
    bool hit = false;
    bool open = lv < n && ld_label(p.lab + p.g.lo + lv) == kInf;
    if (open) {
      const int64_t b = __ldg(p.g.row_ptr + lv), e = __ldg(p.g.row_ptr + lv + 1);
      for (int64_t k = b; k < e && !hit; k += 4) {
        int32_t u[4];
#pragma unroll
        for (int j = 0; j < 4; ++j) u[j] = k + j < e ? ld_stream(p.g.col + k + j) : -1;
#pragma unroll
        for (int j = 0; j < 4; ++j)
          if (u[j] >= 0) hit |= (ld_label(reinterpret_cast<const int32_t*>(fbits) + (u[j] >> 5)) >> (u[j] & 31)) & 1;
        sc += (unsigned long long)(e - k < 4 ? e - k : 4);
      }
      if (hit) {
        p.lab[p.g.lo + lv] = rb.level;
        if (p.vis) atomicOr(p.vis + ((p.g.lo + lv) >> 5), 1u << ((p.g.lo + lv) & 31));
      }
    }
    wpush<OP, false>(sm, q, p, rb, hit ? 1 : 0, (uint32_t)(p.g.lo + lv));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) sc += __shfl_xor_sync(FULL, sc, o);
  if (lane_id() == 0 && sc) atomicAdd(scanned, sc);
}

__global__ void __launch_bounds__(kBlock) bu_part_kernel(KParams p, RoundBufs rb, const uint32_t* fbits,
                                                         unsigned long long* scanned) {
  __shared__ Smem sm;
  smem_init(sm);
  WarpQ q;
  bu_part_phase<IRGL_OP_BFS>(sm, q, p, rb, fbits, scanned);
  wflush_all<IRGL_OP_BFS>(sm, q, p, rb);
}

// F1 inside the distributed persistent kernel: top-down rounds as dist_persistent_kernel's (pushes
// also sum the next frontier's degrees — the owner's for remote finds, in its apply), bottom-up
// rounds over each partition's own unvisited vertices against the global frontier bitmap, which
// every partition assembles by storing its own words into every partition's copy before the
// rendezvous (posted stores over NVLink; no id lists).  Beamer's alpha / beta vote is taken by every
// partition on the same sums, read at the round-end rendezvous, so the direction is uniform.
__global__ void __launch_bounds__(kBlock, IRGL_DO_MINB) dist_bfs_do_kernel(KParams p, DistPersistArgs da) {
  __shared__ SmemDist sm;
  smem_init(sm);
  WarpQ q;
  const PersistArgs& a = da.pa;
  uint32_t* cnt = p.ctl->cnt;
  const int32_t s0 = a.stamp0;
  const bool leader = blockIdx.x == 0 && threadIdx.x == 0;
  const int me = p.dr.me;
  uint32_t nin_next = ld_ctl(cnt + slot3(a, 0));
  __shared__ unsigned long long bslot;
  __shared__ RoundBufs srb;
  __shared__ uint32_t s_x[3];
  __shared__ unsigned long long s_mf;
  uint32_t bidx = 0, xk = 0, nbu = 0;
  constexpr double kAlpha = 14.0, kBeta = 24.0;
  bool bottom_up = false;
  unsigned long long explored = 0;
  x_meet<false>(p, da, ++xk, cnt, s_x);  // hello (see dist_persistent_kernel)
  if (!s_x[0]) {
    if (leader) {
      p.ctl->rounds = 0;
      p.ctl->stamp_used = 0;
      p.ctl->x_word[3] = 0;
    }
    return;
  }
  const uint32_t T = gridDim.x * blockDim.x;
  const uint32_t gt = blockIdx.x * blockDim.x + threadIdx.x;
  for (uint32_t r = 0;; ++r) {
    uint32_t* cout = cnt + slot3(a, r + 1);
    if (leader) {
      cnt[slot3(a, r + 2)] = 0;
      p.ctl->chunk_cnt[(r + 1) % 3] = 0;
      p.ctl->tile_ctr[(r + 1) % 3] = 0;
      p.ctl->mf[(r + 1) % 3] = 0;
    }
    RoundBufs rb{};
    rb.in = (r & 1) ? a.buf_b : a.buf_a;
    rb.nin = nin_next;
    rb.out = (r & 1) ? a.buf_a : a.buf_b;
    rb.out_cnt = cout;
    rb.cap = a.cap;
    rb.chunks = a.chunks;
    rb.chunk_cnt = &p.ctl->chunk_cnt[r % 3];
    rb.chunk_cap = a.chunk_cap;
    rb.tile_ctr = &p.ctl->tile_ctr[r % 3];
    rb.level = a.level0 + (int32_t)r;
    rb.stamp_id = s0 + (int32_t)r;
    rb.threshold = kInf;
    rb.mf_acc = &p.ctl->mf[r % 3];
    __syncthreads();
    if (threadIdx.x == 0) srb = rb;
    __syncthreads();
    const RoundBufs& rr = srb;
    if (!bottom_up) {
      item_phase<kOpBfsDO, true>(sm, q, p, rr);
      wflush_remote_all(sm, q, p);
      wflush_all<kOpBfsDO>(sm, q, p, rr);
      const unsigned long long w = grid_sync_bcast(
          p.ctl, bidx, &bslot, [&]() { return pack_counts(ld_ctl(rr.chunk_cnt), 0); }, [](unsigned long long) {});
      const uint32_t nch = unpack_nch(w);
      if (nch) {
        chunk_phase<kOpBfsDO, true>(sm, q, p, rr, nch);
        wflush_remote_all(sm, q, p);
        wflush_all<kOpBfsDO>(sm, q, p, rr);
      }
      x_meet<false>(p, da, ++xk, cout, s_x);  // every inbox complete
      if (s_x[0]) {
        apply_inbox<kOpBfsDO>(sm, q, p, rr, da);
        wflush_all<kOpBfsDO>(sm, q, p, rr);
      }
    } else {
      // this partition's words of the frontier bitmap, then a copy into every partition's bitmap
      uint32_t* own = da.fbits[me] + (int64_t)me * da.wpp;
      for (int64_t i = gt; i < da.wpp; i += T) own[i] = 0u;
      cg::this_grid().sync();
      for (uint32_t i = gt; i < rr.nin; i += T) {
        const uint32_t v = ld_item(rr.in + i);
        atomicOr(da.fbits[me] + (v >> 5), 1u << (v & 31));
      }
      cg::this_grid().sync();
      for (int qd = 0; qd < da.nparts; ++qd) {
        if (qd == me) continue;
        uint32_t* dst = da.fbits[qd] + (int64_t)me * da.wpp;
        for (int64_t i = gt; i < da.wpp; i += T) dst[i] = own[i];
      }
      x_meet<false>(p, da, ++xk, cout, s_x);  // every bitmap complete
      if (s_x[0]) {
        bu_part_phase<kOpBfsDO>(sm, q, p, rr, da.fbits[me], &p.ctl->bu_scanned);
        wflush_all<kOpBfsDO>(sm, q, p, rr);
        ++nbu;
      }
    }
    bool stop = !s_x[0];
    if (!stop) {
      x_meet<true>(p, da, ++xk, cout, s_x, false, &p.ctl->mf[r % 3]);
      if (threadIdx.x == 0) s_mf = *(volatile unsigned long long*)&p.ctl->x_mf;
      __syncthreads();
      stop = !s_x[0] || s_x[1] == 0 || s_x[2] != 0 || (a.max_rounds > 0 && (int64_t)r + 1 >= a.max_rounds);
    }
    const uint32_t nout = ld_ctl(cout);
    if (leader) {
      p.ctl->popped += rr.nin;
      p.ctl->pushes += nout;
    }
    nin_next = nout;
    if (stop) {
      if (leader) {
        p.ctl->rounds = r + 1;
        p.ctl->exit_in_slot = (int32_t)((r + 1) & 1);
        p.ctl->stamp_used = r + 1;
        p.ctl->bu_rounds = nbu;
        p.ctl->overflow |= s_x[2] & 3u;
        p.ctl->x_word[3] = s_x[0] ? xk : 0u;
      }
      break;
    }
    // direction of the next round: the same global sums in every partition
    const unsigned long long nf = s_x[1], mf = s_mf;
    explored += mf;
    const double mu = (double)a.m - (double)explored;
    if (!bottom_up && (double)mf > mu / kAlpha) bottom_up = true;
    else if (bottom_up && (double)nf < (double)a.n / kBeta) bottom_up = false;
  }
}

// ---- owner-side application of remote updates (E5 min-reduce) ---------------------------------
// Owner-side apply of every peer's segment in one launch (ApplySegs): global index i belongs to
// segment p with off[p] <= i < off[p+1].
template <int OP>
__global__ void __launch_bounds__(kBlock) apply_segs_kernel(KParams p, RoundBufs rb, const uint32_t* items,
                                                          const int32_t* values, ApplySegs sg) {
  __shared__ Smem sm;
  smem_init(sm);
  WarpQ q;
  if (blockIdx.x == 0) {
    if (sg.zero_send && (int)threadIdx.x < sg.P) sg.zero_send[threadIdx.x] = 0u;
    if (sg.zero_cnt && threadIdx.x == 0) *sg.zero_cnt = 0u;
  }
  const uint32_t n = sg.off[sg.P];
  for (uint32_t i0 = blockIdx.x * kBlock + (threadIdx.x & ~31u); i0 < n; i0 += gridDim.x * kBlock) {
    const uint32_t i = i0 + lane_id();
    int kind = 0;
    uint32_t v = 0;
    if (i < n) {
      int s = 0;
      while (s + 1 < sg.P && sg.off[s + 1] <= i) ++s;
      const int64_t at = (int64_t)s * sg.stride + (i - sg.off[s]);
      const uint32_t k = i - sg.off[s];
      // ids: received, or pulled from the sender's bucket (IPC pull) — an L2-coherent load either way
      v = sg.seg_items[s] ? ld_item(sg.seg_items[s] + k) : items[at];
      const int32_t cur = gather_cur<OP>(p, v);
      int32_t val = 0;  // the sender's ghost label: packed, pulled, or read from the sender's labels
      if (!is_bfs(OP))
        val = sg.seg_vals[s] ? ld_label_cg(sg.seg_vals[s] + k)
            : sg.peer_lab[s] ? ld_label_cg(sg.peer_lab[s] + v) : values[at];
      kind = relax_with<OP>(p, rb, q, cur, val, 0, v);
    }
    wpush<OP, false>(sm, q, p, rb, kind, v);
  }
  wflush_all<OP>(sm, q, p, rb);
}

// Multi-partition round, one launch: ghost label of every queued remote update (all owners).
__global__ void pack_all_kernel(const int32_t* lab, const uint32_t* send, int32_t* send_val,
                                const uint32_t* send_cnt, int P, int me, int64_t ps) {
  for (int q = 0; q < P; ++q) {
    if (q == me) continue;
    const uint32_t c = ld_ctl(send_cnt + q);
    for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < c; i += gridDim.x * blockDim.x)
      send_val[(int64_t)q * ps + i] = ld_label(lab + send[(int64_t)q * ps + i]);
  }
}
// Round header of one partition: {send counts [P], in-count, overflow flag}.
// It also clears the round's chunk / tile counters (their users, the expansion launches, precede
// it in stream order) so the next round needs no separate memsets.
__global__ void round_header_kernel(uint32_t* hdr, const uint32_t* send_cnt, int P,
                                    const uint32_t* in_cnt, const uint32_t* overflow,
                                    uint32_t* chunk_cnt, uint32_t* tile_ctr, uint32_t* dmin_done) {
  const int t = threadIdx.x;
  if (t < P) hdr[t] = send_cnt ? ld_ctl(send_cnt + t) : 0u;
  if (t == 0) {
    hdr[P] = ld_ctl(in_cnt);
    hdr[P + 1] = ld_ctl(overflow);
    if (chunk_cnt) *chunk_cnt = 0u;
    if (tile_ctr) *tile_ctr = 0u;
    if (dmin_done) *dmin_done = 0xffffffffu;  // this round's deferral minimum: next round's accumulator
  }
}

__global__ void pack_values_kernel(const int32_t* lab, const uint32_t* items, int32_t* values,
                                   uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    values[i] = ld_label(lab + items[i]);
}

template <int OP, bool DIST>
cudaError_t round_impl(const KParams& kp, const RoundBufs& rb, int grid_max, cudaStream_t st) {
  if (rb.nin_dev) {
    note_launch();
    expand_kernel<OP, DIST><<<grid_max, kBlock, 0, st>>>(kp, rb);
  } else if (rb.nin > 0) {
    const int wtiles = (int)((rb.nin + 31) / 32);
    const int blocks = min((wtiles + kWarps - 1) / kWarps, grid_max);
    note_launch();
    expand_kernel<OP, DIST><<<blocks, kBlock, 0, st>>>(kp, rb);
  }
  note_launch();
  chunk_kernel<OP, DIST><<<grid_max, kBlock, 0, st>>>(kp, rb);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_expand_round(int op, const DevCSR& g, int32_t* lab, int32_t* stamp, uint32_t* vis, Ctl* ctl,
                                const RoundBufs& rb, const DistRoute& dr, const ExpandCfg& ec,
                                int grid_max, cudaStream_t st) {
  KParams kp{g, lab, stamp, vis, ctl, dr, ec};
  const bool dist = dr.nparts > 1;
  switch (op) {
    case IRGL_OP_BFS:
      return dist ? round_impl<IRGL_OP_BFS, true>(kp, rb, grid_max, st)
                  : round_impl<IRGL_OP_BFS, false>(kp, rb, grid_max, st);
    case IRGL_OP_SSSP:
      if (rb.threshold != kInf)  // near-far piles
        return dist ? round_impl<kOpSsspNF, true>(kp, rb, grid_max, st)
                    : round_impl<kOpSsspNF, false>(kp, rb, grid_max, st);
      if (g.w8)  // byte weights
        return dist ? round_impl<kOpSssp8, true>(kp, rb, grid_max, st)
                    : round_impl<kOpSssp8, false>(kp, rb, grid_max, st);
      return dist ? round_impl<IRGL_OP_SSSP, true>(kp, rb, grid_max, st)
                  : round_impl<IRGL_OP_SSSP, false>(kp, rb, grid_max, st);
    case IRGL_OP_CC_LP:
      return dist ? round_impl<IRGL_OP_CC_LP, true>(kp, rb, grid_max, st)
                  : round_impl<IRGL_OP_CC_LP, false>(kp, rb, grid_max, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_far_split(const DevCSR& g, int32_t* lab, int32_t* stamp, Ctl* ctl,
                             const RoundBufs& rb, const uint32_t* far_in, const uint32_t* nfar_ptr,
                             int32_t t_old, unsigned int* minkeep, int grid, cudaStream_t st) {
  KParams kp{g, lab, stamp, nullptr, ctl, DistRoute{1, 0, 1, nullptr, nullptr}, ExpandCfg{32, 1024, 2048}};
  note_launch();
  far_split_kernel<<<grid, kBlock, 0, st>>>(kp, rb, far_in, nfar_ptr, t_old, minkeep);
  return cudaGetLastError();
}

cudaError_t launch_apply_remote_segs(int op, int32_t* lab, int32_t* stamp, uint32_t* vis, Ctl* ctl,
                                     const uint32_t* items, const int32_t* values,
                                     const ApplySegs& segs, const RoundBufs& rb, cudaStream_t st) {
  const uint32_t n = segs.off[segs.P];
  if (n == 0 && !segs.zero_send && !segs.zero_cnt) return cudaSuccess;
  const int grid = (int)max(1u, min((n + kBlock - 1) / kBlock, 148u * 8u));
  KParams kp{DevCSR{nullptr, nullptr, nullptr, 0, 0}, lab, stamp, vis, ctl,
             DistRoute{1, 0, 1, nullptr, nullptr}, ExpandCfg{32, 1024, 2048}};
  note_launch();
  switch (op) {
    case IRGL_OP_BFS:
      apply_segs_kernel<IRGL_OP_BFS><<<grid, kBlock, 0, st>>>(kp, rb, items, values, segs);
      break;
    case IRGL_OP_SSSP:
      if (rb.threshold != kInf)
        apply_segs_kernel<kOpSsspNF><<<grid, kBlock, 0, st>>>(kp, rb, items, values, segs);
      else
        apply_segs_kernel<IRGL_OP_SSSP><<<grid, kBlock, 0, st>>>(kp, rb, items, values, segs);
      break;
    case IRGL_OP_CC_LP:
      apply_segs_kernel<IRGL_OP_CC_LP><<<grid, kBlock, 0, st>>>(kp, rb, items, values, segs);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_pack_all(const int32_t* lab, const uint32_t* send, int32_t* send_val,
                            const uint32_t* send_cnt, int P, int me, int64_t ps, cudaStream_t st) {
  note_launch();
  pack_all_kernel<<<148 * 4, 256, 0, st>>>(lab, send, send_val, send_cnt, P, me, ps);
  return cudaGetLastError();
}

cudaError_t launch_round_header(uint32_t* hdr, const uint32_t* send_cnt, int P, const uint32_t* in_cnt,
                                const uint32_t* overflow, uint32_t* chunk_cnt, uint32_t* tile_ctr,
                                uint32_t* dmin_done, cudaStream_t st) {
  note_launch();
  round_header_kernel<<<1, 32, 0, st>>>(hdr, send_cnt, P, in_cnt, overflow, chunk_cnt, tile_ctr, dmin_done);
  return cudaGetLastError();
}

cudaError_t launch_pack_values(const int32_t* lab, const uint32_t* items, int32_t* values,
                               uint32_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  note_launch();
  pack_values_kernel<<<(int)min((n + 255) / 256, 4096u), 256, 0, st>>>(lab, items, values, n);
  return cudaGetLastError();
}

// IRGL_E_RANGE check of a finished one-partition SSSP (path_sum): an edge u -> v with u reached
// and v unreached can only come from a path sum beyond the int32 range.
__global__ void range_check_kernel(DevCSR g, const int32_t* dist, uint32_t* bad) {
  const int64_t n = g.hi - g.lo;
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n; u += (int64_t)gridDim.x * blockDim.x) {
    if (dist[g.lo + u] == kInf) continue;
    for (int64_t e = g.row_ptr[u]; e < g.row_ptr[u + 1]; ++e)
      if (dist[g.col[e]] == kInf) {
        atomicOr(bad, 1u);
        break;
      }
  }
}

__global__ void ctl_prepare_kernel(Ctl* c) {
  const int t = threadIdx.x;
  if (t < 3) {
    c->chunk_cnt[t] = 0;
    c->tile_ctr[t] = 0;
    c->dmin[t] = 0xffffffffu;  // round 0: no frontier minimum yet (no deferral)
    c->mf[t] = 0;
    c->bu_found[t] = 0;
  }
  if (t < 2) c->far_cnt[t] = 0;
  if (t == 0) {
    c->gb_arrive = 0;
    c->gb_release = 0;
    c->popped = c->pushes = 0;
    c->rounds = 0;
    c->bu_scanned = 0;
  }
}

cudaError_t launch_range_check(const DevCSR& g, const int32_t* dist, uint32_t* bad, cudaStream_t st) {
  note_launch();
  range_check_kernel<<<148 * 8, 256, 0, st>>>(g, dist, bad);
  return cudaGetLastError();
}

cudaError_t launch_frontier_stats(const uint32_t* items, const uint32_t* cnt, const int64_t* rp, int64_t lo,
                                  unsigned long long* out2, cudaStream_t st) {
  note_launch();
  cudaMemsetAsync(out2, 0, 16, st);
  frontier_stats_kernel<<<148 * 4, 256, 0, st>>>(items, cnt, rp, lo, out2);
  return cudaGetLastError();
}
cudaError_t launch_frontier_bits(const uint32_t* items, const uint32_t* cnt, uint32_t* bits, cudaStream_t st) {
  note_launch();
  frontier_bits_kernel<<<148 * 4, 256, 0, st>>>(items, cnt, bits);
  return cudaGetLastError();
}
cudaError_t launch_bu_part(const DevCSR& g, int32_t* lab, uint32_t* vis, Ctl* ctl, const RoundBufs& rb,
                           const uint32_t* fbits, cudaStream_t st) {
  KParams kp{g, lab, nullptr, vis, ctl, DistRoute{1, 0, 1, nullptr, nullptr}, ExpandCfg{128, 256, 512}};
  const int64_t n = g.hi - g.lo;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((n + kBlock - 1) / kBlock, 148 * 8));
  note_launch();
  bu_part_kernel<<<grid, kBlock, 0, st>>>(kp, rb, fbits, &ctl->edges);
  return cudaGetLastError();
}

cudaError_t launch_ctl_prepare(Ctl* ctl, cudaStream_t st) {
  note_launch();
  ctl_prepare_kernel<<<1, 32, 0, st>>>(ctl);
  return cudaGetLastError();
}

int persistent_blocks_per_sm(int op, int variant) {
  int nb = 0;
  switch (op) {
    case IRGL_OP_BFS: {
      int nd = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, persistent_kernel<IRGL_OP_BFS>, kBlock, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nd, persistent_bfs_do_kernel, kBlock, 0);
      nb = variant < 0 ? min(nb, nd) : variant ? nd : nb;
    } break;
    case IRGL_OP_SSSP: {
      int nn = 0, n8 = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, persistent_kernel<IRGL_OP_SSSP>, kBlock, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nn, persistent_kernel<kOpSsspNF>, kBlock, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n8, persistent_kernel<kOpSssp8>, kBlock, 0);
      nb = min(nb, n8);  // int32 or byte weights
      nb = variant < 0 ? min(nb, nn) : variant ? nn : nb;
    } break;
    case IRGL_OP_CC_LP:
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, persistent_kernel<IRGL_OP_CC_LP>, kBlock, 0);
      break;
  }
  return nb;
}

int expand_blocks_per_sm(int op) {
  int nb = 0;
  switch (op) {
    case IRGL_OP_BFS:
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, expand_kernel<IRGL_OP_BFS, false>, kBlock, 0);
      break;
    case IRGL_OP_SSSP:
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, expand_kernel<IRGL_OP_SSSP, false>, kBlock, 0);
      break;
    default:
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, expand_kernel<IRGL_OP_CC_LP, false>, kBlock, 0);
      break;
  }
  return nb;
}

int dist_persistent_blocks_per_sm(int op) {
  int nb = 0, n8 = 0;
  switch (op) {
    case IRGL_OP_BFS:
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, dist_persistent_kernel<IRGL_OP_BFS>, kBlock, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n8, dist_bfs_do_kernel, kBlock, 0);
      nb = min(nb, n8);  // a grid valid for either direction mode
      break;
    case IRGL_OP_SSSP:
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, dist_persistent_kernel<IRGL_OP_SSSP>, kBlock, 0);
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n8, dist_persistent_kernel<kOpSssp8>, kBlock, 0);
      nb = min(nb, n8);
      break;
    case IRGL_OP_CC_LP:
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, dist_persistent_kernel<IRGL_OP_CC_LP>, kBlock, 0);
      break;
  }
  return nb;
}

cudaError_t launch_dist_persistent(int op, const DevCSR& g, int32_t* lab, int32_t* stamp, uint32_t* vis, Ctl* ctl,
                                   const DistRoute& dr, const DistPersistArgs& da, const ExpandCfg& ec, int grid,
                                   cudaStream_t st) {
  KParams kp{g, lab, stamp, vis, ctl, dr, ec};
  DistPersistArgs a = da;
  void* args[] = {&kp, &a};
  note_launch();
  switch (op) {
    case IRGL_OP_BFS:
      if (a.pa.dir_opt) return cudaLaunchCooperativeKernel((void*)dist_bfs_do_kernel, grid, kBlock, args, 0, st);
      return cudaLaunchCooperativeKernel((void*)dist_persistent_kernel<IRGL_OP_BFS>, grid, kBlock, args, 0, st);
    case IRGL_OP_SSSP:
      if (g.w8)
        return cudaLaunchCooperativeKernel((void*)dist_persistent_kernel<kOpSssp8>, grid, kBlock, args, 0, st);
      return cudaLaunchCooperativeKernel((void*)dist_persistent_kernel<IRGL_OP_SSSP>, grid, kBlock, args, 0, st);
    case IRGL_OP_CC_LP:
      return cudaLaunchCooperativeKernel((void*)dist_persistent_kernel<IRGL_OP_CC_LP>, grid, kBlock, args, 0, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_persistent(int op, const DevCSR& g, int32_t* lab, int32_t* stamp, uint32_t* vis, Ctl* ctl,
                              const PersistArgs& pa, const ExpandCfg& ec, int grid,
                              cudaStream_t st) {
  KParams kp{g, lab, stamp, vis, ctl, DistRoute{1, 0, 1, nullptr, nullptr}, ec};
  PersistArgs a = pa;
  void* args[] = {&kp, &a};
  note_launch();
  switch (op) {
    case IRGL_OP_BFS:
      if (a.dir_opt)
        return cudaLaunchCooperativeKernel((void*)persistent_bfs_do_kernel, grid, kBlock, args, 0, st);
      return cudaLaunchCooperativeKernel((void*)persistent_kernel<IRGL_OP_BFS>, grid, kBlock, args, 0, st);
    case IRGL_OP_SSSP:
      if (a.delta > 0)
        return cudaLaunchCooperativeKernel((void*)persistent_kernel<kOpSsspNF>, grid, kBlock, args, 0, st);
      if (g.w8)
        return cudaLaunchCooperativeKernel((void*)persistent_kernel<kOpSssp8>, grid, kBlock, args, 0, st);
      return cudaLaunchCooperativeKernel((void*)persistent_kernel<IRGL_OP_SSSP>, grid, kBlock, args, 0, st);
    case IRGL_OP_CC_LP:
      return cudaLaunchCooperativeKernel((void*)persistent_kernel<IRGL_OP_CC_LP>, grid, kBlock, args, 0, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace irgl
