// topo.cu — topology-driven operators (no worklist; Iterate is a plain loop):
//   CC  : hook (CAS the larger root onto the smaller) + pointer jumping, Iterate While Any.
//   PR  : pull Jacobi PageRank in fp64 with a fused contrib_next write and the E4 warp-reduced
//         ReduceAndReturn(|new-old| > tol) flag; outlined variant = one persistent kernel.
//   TC  : degree-ordered orientation + warp-cooperative sorted-list intersection, warp-reduced
//         64-bit Sum (an extension: IrGL's ReduceAndReturn has only Any/All).
#include <cooperative_groups.h>
#include <cub/cub.cuh>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace irgl {
namespace {
constexpr unsigned FULL = 0xffffffffu;

// E4: warp-reduced ReduceAndReturn.  Threads that evaluated `value` fold it; one idempotent store
// per warp (Any writes 1 into a cell initialised to 0, All writes 0 into a cell initialised to 1)
// — no atomics, no per-thread traffic.
__device__ __forceinline__ void reduce_and_return(bool evaluated, bool value, int reduction,
                                                  uint32_t* cell) {
  if (reduction == IRGL_RED_ANY) {
    if (__any_sync(FULL, evaluated && value) && lane_id() == 0) *(volatile uint32_t*)cell = 1u;
  } else if (reduction == IRGL_RED_ALL) {
    if (!__all_sync(FULL, !evaluated || value) && lane_id() == 0) *(volatile uint32_t*)cell = 0u;
  }
}

__device__ __forceinline__ int32_t cc_find(const int32_t* par, int32_t x) {
  int32_t p = ld_label(par + x);
  while (p != x) {
    x = p;
    p = ld_label(par + x);
  }
  return x;
}

// Root of x with intermediate pointer jumping (each visited node is re-pointed to its grandparent;
// benign races: hooks only ever lower a parent, par[x] <= x holds throughout), so the trees a hook
// round builds stay shallow and later finds are short (ECL-CC's find).
__device__ __forceinline__ int32_t cc_find_jump(int32_t* par, int32_t x) {
  int32_t cur = ld_label(par + x);
  if (cur != x) {
    int32_t prev = x, next;
    while (cur > (next = ld_label(par + cur))) {
      par[prev] = next;
      prev = cur;
      cur = next;
    }
  }
  return cur;
}

// Hook edge (u, v): ECL-CC style CAS retry so each edge needs one visit.
__device__ __forceinline__ bool cc_hook_edge(int32_t* par, int32_t u, int32_t v) {
  int32_t a = cc_find_jump(par, u), b = cc_find_jump(par, v);
  bool changed = false;
  while (a != b) {
    const int32_t hi = max(a, b), lo = min(a, b);
    const int32_t old = atomicCAS(par + hi, hi, lo);
    if (old == hi) {
      changed = true;
      break;
    }
    a = cc_find_jump(par, old);
    b = cc_find_jump(par, lo);
  }
  return changed;
}

__global__ void __launch_bounds__(kBlock) cc_hook_kernel(DevCSR g, int32_t* par, uint32_t* cell) {
  const int lane = threadIdx.x & 31;
  const int64_t nloc = g.hi - g.lo;
  for (int64_t t0 = (int64_t)blockIdx.x * kBlock; t0 < nloc; t0 += (int64_t)gridDim.x * kBlock) {
    const int64_t i = t0 + threadIdx.x;
    const bool valid = i < nloc;
    int64_t beg = 0, end = 0;
    if (valid) {
      beg = g.row_ptr[i];
      end = g.row_ptr[i + 1];
    }
    const int32_t u = (int32_t)(g.lo + i);
    bool changed = false;
    // warp-cooperative for high degree
    int64_t deg = end - beg;
    uint32_t wm = __ballot_sync(FULL, deg >= 32);
    while (wm) {
      const int leader = __ffs(wm) - 1;
      wm &= wm - 1;
      const int64_t b = __shfl_sync(FULL, beg, leader), e = __shfl_sync(FULL, end, leader);
      const int32_t uu = __shfl_sync(FULL, u, leader);
      if (lane == leader) deg = 0;
      for (int64_t k = b + lane; k < e; k += 32) {
        const int32_t v = ld_stream(g.col + k);
        if (v < uu) changed |= cc_hook_edge(par, uu, v);
      }
    }
    if (deg > 0)
      for (int64_t k = beg; k < end; ++k) {
        const int32_t v = ld_stream(g.col + k);
        if (v < u) changed |= cc_hook_edge(par, u, v);
      }
    reduce_and_return(true, changed, IRGL_RED_ANY, cell);
  }
}

__global__ void cc_compress_kernel(int32_t* par, int64_t n) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x)
    par[v] = cc_find(par, (int32_t)v);
}

// ---------------------------------------------------------------------------------------------
// PageRank.  rank(v) = (1-d)/N + d * sum_{u in N(v)} contrib(u), contrib(u) = rank(u)/deg(u).
struct PrSmem {
  double red[kWarps];
  int32_t owner;
  int64_t b, e;
  int64_t tile;
  int64_t round;
};

// contrib / rank arrays are rewritten every sweep.  Per-vertex reads (old rank, hub partials) go
// through L2 (.cg).  The contribution GATHER is L1-cached (.ca): hubs' contributions are the most
// gathered values, and with degree-ordered ids they share lines that stay L1-resident (PR on
// relabelled RMAT-24 2.47 -> 1.67 ms per sweep, RMAT-22 0.76 -> 0.41).  That is safe across the
// persistent kernel's sweeps because cg grid.sync() ends in an acquire poll (LD.STRONG.GPU +
// CCTL.IVALL in the SASS: every L1 line of the SM is invalidated once the barrier opens), so no
// line from an earlier sweep survives into the next; between host-loop launches the kernel
// boundary does the same.
__device__ __forceinline__ double ld_cg_f64(const double* p) {
  double r;
  asm volatile("ld.global.cg.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}

__device__ __forceinline__ float ld_cg_f32(const float* p) {
  float r;
  asm volatile("ld.global.cg.f32 %0, [%1];" : "=f"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ double ld_ca_f64(const double* p) {
  double r;
  asm volatile("ld.global.ca.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}

// Sum of contrib[col[k]] for k = k0, k0+S, k0+2S, ... < e, U gathers in flight per step; the
// summation order is fixed (deterministic per vertex for a given launch shape).
template <int S, int U = 8>
__device__ __forceinline__ double gather_sum(const int32_t* __restrict__ col, const double* contrib,
                                             int64_t k0, int64_t e) {
  double s = 0.0;
  int64_t k = k0;
  for (; k + (U - 1) * S < e; k += U * S) {
    int32_t c[U];
    double v[U];
#pragma unroll
    for (int j = 0; j < U; ++j) c[j] = ld_stream(col + k + j * S);
#pragma unroll
    for (int j = 0; j < U; ++j) v[j] = ld_ca_f64(contrib + c[j]);
#pragma unroll
    for (int j = 0; j < U; ++j) s += v[j];
  }
  for (; k < e; k += S) s += ld_ca_f64(contrib + ld_stream(col + k));
  return s;
}

__device__ __forceinline__ double warp_sum(double x) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(FULL, x, o);
  return x;
}

// Hub vertices (degree >= hub_t) are summed edge-balanced: their edge ranges are cut once per
// graph into chunks of <= chunk edges; every warp of the grid sums whole chunks into partial[c]
// (phase A), and the vertex's sweep adds its partials in chunk order (phase B) — deterministic,
// and no CTA walks a run of hubs alone: with degree-ordered ids every hub sits in the first
// vertex tiles (without the split PR on relabelled RMAT-24 took 18.5 ms per sweep instead of 2.8).
__device__ void pr_hub_chunks(const DevCSR& g, const double* contrib, const PrHubs& h) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t c = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; c < h.nchunks; c += nw) {
    const int64_t b = h.cbeg[c], e = b + h.clen[c];
    const double s = warp_sum(gather_sum<32>(g.col, contrib, b + lane, e));
    if (lane == 0) h.partial[c] = s;
  }
}

// One PR sweep over the local vertex range (tile per CTA-iteration).  Deterministic per-vertex
// summation order (fixed by the code path chosen by degree).
// contrib(u) = rank(u)/deg(u) is stored in fp32 (the gathered operand: half the bytes per edge
// and an L2-resident array at RMAT-24); ranks and per-vertex sums stay fp64.
// Round slot of the persistent kernel's rotating cells, read from shared memory at each use so
// that neither the slot nor the derived cell pointers occupy registers across the sweep.
__shared__ int32_t s_pr_slot;

// kSmemSlot: cells ctl->red[s], ctl->tile_ctr[s] with s = s_pr_slot (persistent kernel) or
// s = slot (host-loop kernel, a constant-bank parameter).
template <bool kSmemSlot>
__device__ void pr_sweep_cta(PrSmem& sm, const DevCSR& g, const double* __restrict__ rank_old,
                               double* __restrict__ rank_new, const double* __restrict__ contrib,
                               double* __restrict__ contrib_next, double d, double tol,
                               double base, int red, Ctl* ctl, int slot, const PrHubs& h) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int64_t nloc = g.hi - g.lo;
  // tiles: the first one static, then dynamic (tctr counts from 0; tile = gridDim + count), so
  // with degree-ordered ids the expensive front tiles are taken first and the tail stays short
  for (int64_t t0 = (int64_t)blockIdx.x * kBlock;;) {
    if (t0 >= nloc) break;
    const int64_t i = t0 + tid;
    const bool valid = i < nloc;
    int64_t beg = 0, end = 0;
    if (valid) {
      beg = __ldg(g.row_ptr + i);
      end = __ldg(g.row_ptr + i + 1);
    }
    const int64_t deg0 = end - beg;
    int64_t deg = deg0;
    double mysum = 0.0;
    if (h.nchunks > 0 && deg >= h.hub_t) {  // hub: its chunks' partial sums, in order
      const int32_t k = __ldg(h.hub_of + i);
      const int64_t c0 = h.hfirst[k], c1 = h.hfirst[k + 1];
      for (int64_t c = c0; c < c1; ++c) mysum += ld_cg_f64(h.partial + c);
      deg = 0;
    }
    // CTA level (deg >= 1024): whole CTA sums one vertex at a time
    while (__syncthreads_or(deg >= 1024)) {
      if (deg >= 1024) sm.owner = tid;  // any winner
      __syncthreads();
      const int own = sm.owner;
      if (tid == own) {
        sm.b = beg;
        sm.e = end;
        deg = 0;
      }
      __syncthreads();
      const double s0 = gather_sum<kBlock>(g.col, contrib, sm.b + tid, sm.e);
      const double s = warp_sum(s0);
      if (lane == 0) sm.red[warp] = s;
      __syncthreads();
      if (tid == own) {
        double t = 0.0;
#pragma unroll
        for (int k = 0; k < kWarps; ++k) t += sm.red[k];
        mysum = t;
      }
      __syncthreads();
    }
    // warp level
    uint32_t wm = __ballot_sync(FULL, deg >= 32);
    while (wm) {
      const int leader = __ffs(wm) - 1;
      wm &= wm - 1;
      const int64_t b = __shfl_sync(FULL, beg, leader), e = __shfl_sync(FULL, end, leader);
      const double s = warp_sum(gather_sum<32>(g.col, contrib, b + lane, e));
      if (lane == leader) {
        mysum = s;
        deg = 0;
      }
    }
    // thread level
    if (deg > 0) mysum = gather_sum<1>(g.col, contrib, beg, end);
    bool changed = false;
    if (valid) {
      const int64_t v = g.lo + i;
      const double r = base + d * mysum;
      rank_new[v] = r;
      contrib_next[v] = deg0 > 0 ? r / (double)deg0 : 0.0;
      changed = fabs(r - ld_cg_f64(rank_old + v)) > tol;
    }
    const int sl = kSmemSlot ? *(volatile int32_t*)&s_pr_slot : slot;
    reduce_and_return(valid, changed, red, &ctl->red[sl]);
    if (tid == 0) sm.tile = ((int64_t)gridDim.x + atomicAdd(&ctl->tile_ctr[sl], 1u)) * kBlock;
    __syncthreads();
    t0 = sm.tile;
    __syncthreads();
  }
}

// Warp tiles of kPrWarpTile vertices, static round robin over the grid's warps: no CTA barrier
// anywhere in the sweep.  Degrees >= hub_t come from the hub chunk partials, 32 <= degree < hub_t are summed by the
// whole warp one vertex at a time, smaller ones by their own lane.  Used for graphs in generator order, where a
// CTA tile's 8 warps get unrelated degrees and 32% of the CTA-tile sweep's stall samples were CTA
// barriers (RMAT-24: 2.53 -> 2.30 ms per sweep).
constexpr int kPrWarpTile = 32;
template <bool kSmemSlot>
__device__ void pr_sweep_warp(PrSmem& sm, const DevCSR& g, const double* __restrict__ rank_old,
                               double* __restrict__ rank_new, const double* __restrict__ contrib,
                               double* __restrict__ contrib_next, double d, double tol,
                               double base, int red, Ctl* ctl, int slot, const PrHubs& h) {
  (void)sm;
  const int lane = threadIdx.x & 31;
  const int64_t nloc = g.hi - g.lo;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int64_t t = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  while (t * kPrWarpTile < nloc) {
#pragma unroll 1
    for (int sub = 0; sub < kPrWarpTile; sub += 32) {
      const int64_t i = t * kPrWarpTile + sub + lane;
      const bool valid = i < nloc;
      int64_t beg = 0, end = 0;
      if (valid) {
        beg = __ldg(g.row_ptr + i);
        end = __ldg(g.row_ptr + i + 1);
      }
      const int64_t deg0 = end - beg;
      int64_t deg = deg0;
      double mysum = 0.0;
      if (h.nchunks > 0 && deg >= h.hub_t) {  // hub: its chunks' partial sums, in order
        const int32_t k = __ldg(h.hub_of + i);
        const int64_t c0 = h.hfirst[k], c1 = h.hfirst[k + 1];
        for (int64_t c = c0; c < c1; ++c) mysum += ld_cg_f64(h.partial + c);
        deg = 0;
      }
      // warp level
      uint32_t wm = __ballot_sync(FULL, deg >= 32);
      while (wm) {
        const int leader = __ffs(wm) - 1;
        wm &= wm - 1;
        const int64_t b = __shfl_sync(FULL, beg, leader), e = __shfl_sync(FULL, end, leader);
        const double s = warp_sum(gather_sum<32>(g.col, contrib, b + lane, e));
        if (lane == leader) {
          mysum = s;
          deg = 0;
        }
      }
      // thread level
      if (deg > 0) mysum = gather_sum<1>(g.col, contrib, beg, end);
      bool changed = false;
      if (valid) {
        const int64_t v = g.lo + i;
        const double r = base + d * mysum;
        rank_new[v] = r;
        contrib_next[v] = deg0 > 0 ? r / (double)deg0 : 0.0;
        changed = fabs(r - ld_cg_f64(rank_old + v)) > tol;
      }
      const int sl = kSmemSlot ? *(volatile int32_t*)&s_pr_slot : slot;
      reduce_and_return(valid, changed, red, &ctl->red[sl]);
    }
    t += nw;
  }
}

// CTA tiles for degree-ordered graphs (1.67 vs 1.75 ms per sweep on RMAT-24, 0.41 vs 0.47 on
// RMAT-22), warp tiles otherwise (2.30 vs 2.53 on RMAT-24).
template <bool kSmemSlot>
__device__ __forceinline__ void pr_sweep_tiles(PrSmem& sm, const DevCSR& g, const double* __restrict__ rank_old,
                                               double* __restrict__ rank_new, const double* __restrict__ contrib,
                                               double* __restrict__ contrib_next, double d, double tol,
                                               double base, int red, Ctl* ctl, int slot, const PrHubs& h) {
  if (h.cta_tiles)
    pr_sweep_cta<kSmemSlot>(sm, g, rank_old, rank_new, contrib, contrib_next, d, tol, base, red, ctl, slot, h);
  else
    pr_sweep_warp<kSmemSlot>(sm, g, rank_old, rank_new, contrib, contrib_next, d, tol, base, red, ctl, slot, h);
}

__global__ void __launch_bounds__(kBlock) pr_sweep_kernel(DevCSR g, const double* rank_old,
                                                          double* rank_new, const double* contrib,
                                                          double* contrib_next, double d,
                                                          double tol, double base, PrHubs h, Ctl* ctl,
                                                          int slot) {
  __shared__ PrSmem sm;
  pr_sweep_tiles<false>(sm, g, rank_old, rank_new, contrib, contrib_next, d, tol, base, IRGL_RED_ANY,
                        ctl, slot, h);
}

__global__ void __launch_bounds__(kBlock) pr_hub_kernel(DevCSR g, const double* contrib, PrHubs h) {
  pr_hub_chunks(g, contrib, h);
}

__global__ void pr_init_kernel(double* rank, double* contrib, const int64_t* row_ptr, int64_t n) {
  const double r0 = 1.0 / (double)n;
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    rank[v] = r0;
    const int64_t deg = row_ptr[v + 1] - row_ptr[v];
    contrib[v] = deg > 0 ? r0 / (double)deg : 0.0;
  }
}

// Outlined PR: Iterate While Any PR(graph) [Or rounds >= max] as one persistent kernel.
// Cells rotate over 3 slots: cell (r+1)%3 is reset during round r (last read at the start of r-1).
// Returns true when the Iterate stops after round r.
__device__ __forceinline__ bool pr_round(PrSmem& sm, cg::grid_group& grid, const DevCSR& g,
                                         const double* ro, double* rn, const double* co, double* cn,
                                         double d, double tol, double base, Ctl* ctl,
                                         int64_t max_rounds, int cond_mode, const PrHubs& h,
                                         int64_t r) {
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->red[(r + 1) % 3] = 0u;
    ctl->tile_ctr[(r + 1) % 3] = 0u;  // last used in round r-2
  }
  __syncthreads();  // every thread has read the previous round's sm.round
  if (threadIdx.x == 0) {
    s_pr_slot = (int32_t)(r % 3);
    sm.round = r;
  }
  __syncthreads();
  if (h.nchunks > 0) {
    pr_hub_chunks(g, co, h);
    grid.sync();
  }
  pr_sweep_tiles<true>(sm, g, ro, rn, co, cn, d, tol, base, IRGL_RED_ANY, ctl, 0, h);
  grid.sync();
  r = *(volatile int64_t*)&sm.round;
  const uint32_t any = *(volatile uint32_t*)&ctl->red[r % 3];
  bool stop = false;
  if (cond_mode == IRGL_COND_WHILE) stop = (any == 0u);
  if (cond_mode == IRGL_COND_UNTIL) stop = (any == 1u);
  if (max_rounds > 0 && r + 1 >= max_rounds) stop = true;
  if (stop && blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->rounds = (unsigned long long)(r + 1);
    ctl->last_red = (int32_t)any;
    ctl->exit_in_slot = (int32_t)((r + 1) & 1);
  }
  return stop;
}

// Two rounds per loop trip with the buffers swapped by name, so the round's rank / contribution
// pointers stay kernel parameters (constant bank) instead of live registers: selecting them with
// (r & 1) cost 40 B of spills at the 40-register budget and made the sweep 25% slower than the
// host-loop kernel on RMAT-24.
__global__ void __launch_bounds__(kBlock, minb_for_threads(1536)) pr_persistent_kernel(DevCSR g, double* ra, double* rb,
                                                               double* ca, double* cb, double d,
                                                               double tol, double base, Ctl* ctl,
                                                               int64_t max_rounds, int cond_mode,
                                                               PrHubs h) {
  __shared__ PrSmem sm;
  cg::grid_group grid = cg::this_grid();
  for (int64_t r = 0;; r = *(volatile int64_t*)&sm.round + 1) {
    if (pr_round(sm, grid, g, ra, rb, ca, cb, d, tol, base, ctl, max_rounds, cond_mode, h, r)) break;
    r = *(volatile int64_t*)&sm.round + 1;
    if (pr_round(sm, grid, g, rb, ra, cb, ca, d, tol, base, ctl, max_rounds, cond_mode, h, r)) break;
  }
}

// ---------------------------------------------------------------------------------------------
// TC: orientation u -> v iff (deg u, u) < (deg v, v); warp per vertex, order-preserving
// ballot compaction keeps each N+(u) sorted.
__device__ __forceinline__ bool tc_less(const int64_t* rp, int64_t u, int64_t v) {
  const int64_t du = rp[u + 1] - rp[u], dv = rp[v + 1] - rp[v];
  return du < dv || (du == dv && u < v);
}

// Orientation, pass 1: out-degree d+(u).  Thread per vertex for degree < 32 (meshes, road
// graphs), warp-cooperative above (hubs).
__global__ void tc_count_out_kernel(const int64_t* rp, const int32_t* col, int64_t n,
                                    int64_t* dout) {
  const int lane = threadIdx.x & 31;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  for (int64_t u0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~int64_t(31); u0 < n; u0 += T) {
    const int64_t u = u0 + lane;
    int64_t b = 0, e = 0;
    if (u < n) {
      b = rp[u];
      e = rp[u + 1];
    }
    int64_t c = 0;
    if (e - b < 32)
      for (int64_t k = b; k < e; ++k) c += tc_less(rp, u, col[k]);
    uint32_t wm = __ballot_sync(FULL, e - b >= 32);
    while (wm) {
      const int ld = __ffs(wm) - 1;
      wm &= wm - 1;
      const int64_t uu = __shfl_sync(FULL, u, ld), bb = __shfl_sync(FULL, b, ld), ee = __shfl_sync(FULL, e, ld);
      int64_t cc = 0;
      for (int64_t k0 = bb; k0 < ee; k0 += 32) {
        const int64_t k = k0 + lane;
        cc += __popc(__ballot_sync(FULL, k < ee && tc_less(rp, uu, col[k])));
      }
      if (lane == ld) c = cc;
    }
    if (u < n) dout[u] = c;
  }
}

// Pass 2: N+(u) in col order (sorted), plus the source of every oriented edge (edge-parallel
// counting).  Same thread / warp split.
__global__ void tc_fill_kernel(const int64_t* rp, const int32_t* col, int64_t n, const int64_t* orp,
                               int32_t* ocl, int32_t* osrc) {
  const int lane = threadIdx.x & 31;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  for (int64_t u0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~int64_t(31); u0 < n; u0 += T) {
    const int64_t u = u0 + lane;
    int64_t b = 0, e = 0;
    if (u < n) {
      b = rp[u];
      e = rp[u + 1];
    }
    if (e - b < 32) {
      int64_t o = u < n ? orp[u] : 0;
      for (int64_t k = b; k < e; ++k) {
        const int32_t v = col[k];
        if (tc_less(rp, u, v)) {
          ocl[o] = v;
          osrc[o] = (int32_t)u;
          ++o;
        }
      }
    }
    uint32_t wm = __ballot_sync(FULL, e - b >= 32);
    while (wm) {
      const int ld = __ffs(wm) - 1;
      wm &= wm - 1;
      const int64_t uu = __shfl_sync(FULL, u, ld), bb = __shfl_sync(FULL, b, ld), ee = __shfl_sync(FULL, e, ld);
      int64_t o = orp[uu];
      for (int64_t k0 = bb; k0 < ee; k0 += 32) {
        const int64_t k = k0 + lane;
        int32_t v = 0;
        bool p = false;
        if (k < ee) {
          v = col[k];
          p = tc_less(rp, uu, v);
        }
        const uint32_t m = __ballot_sync(FULL, p);
        if (p) {
          ocl[o + __popc(m & lanemask_lt())] = v;
          osrc[o + __popc(m & lanemask_lt())] = (int32_t)uu;
        }
        o += __popc(m);
      }
    }
  }
}

__device__ __forceinline__ bool bsearch_i32(const int32_t* a, int64_t n, int32_t x) {
  int64_t lo = 0, hi = n;
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    const int32_t y = a[mid];
    if (y == x) return true;
    if (y < x) lo = mid + 1;
    else hi = mid;
  }
  return false;
}

// |N+(u) ∩ N+(v)| for one oriented edge, by one thread: sorted merge when the lists are of similar
// length, binary search of the shorter in the longer when they are not.
__device__ __forceinline__ unsigned long long tc_intersect(const int32_t* __restrict__ ocl,
                                                           int64_t ub, int64_t ue, int64_t vb, int64_t ve) {
  int64_t du = ue - ub, dv = ve - vb;
  if (du > dv) {
    int64_t t = ub; ub = vb; vb = t;
    t = ue; ue = ve; ve = t;
    t = du; du = dv; dv = t;
  }
  unsigned long long c = 0;
  if (du == 0) return 0;
  if (du * 8 < dv) {
    for (int64_t j = ub; j < ue; ++j) c += bsearch_i32(ocl + vb, dv, ocl[j]);
    return c;
  }
  int64_t i = ub, j = vb;
  int32_t a = ocl[i], b = ocl[j];
  for (;;) {
    if (a == b) {
      ++c;
      if (++i == ue || ++j == ve) break;
      a = ocl[i];
      b = ocl[j];
    } else if (a < b) {
      if (++i == ue) break;
      a = ocl[i];
    } else {
      if (++j == ve) break;
      b = ocl[j];
    }
  }
  return c;
}

// Edge-parallel count over the oriented edges: thread per edge (u, v) for short lists; an edge
// whose shorter list has >= 64 entries is intersected by its warp (lanes stride the shorter list
// and binary-search the longer).  Warp-reduced 64-bit count, one atomic per warp.
__global__ void tc_count_kernel(const int64_t* orp, const int32_t* ocl, const int32_t* osrc, int64_t mo,
                                unsigned long long* total) {
  const int lane = threadIdx.x & 31;
  unsigned long long cnt = 0;
  const int64_t T = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) & ~int64_t(31); k0 < mo; k0 += T) {
    const int64_t k = k0 + lane;
    int64_t ub = 0, ue = 0, vb = 0, ve = 0;
    if (k < mo) {
      const int32_t u = osrc[k], v = ocl[k];
      ub = orp[u];
      ue = orp[u + 1];
      vb = orp[v];
      ve = orp[v + 1];
    }
    const bool wide = min(ue - ub, ve - vb) >= 64;
    if (k < mo && !wide) cnt += tc_intersect(ocl, ub, ue, vb, ve);
    uint32_t wm = __ballot_sync(FULL, k < mo && wide);
    while (wm) {
      const int ld = __ffs(wm) - 1;
      wm &= wm - 1;
      int64_t sb = __shfl_sync(FULL, ub, ld), se = __shfl_sync(FULL, ue, ld);
      int64_t lb = __shfl_sync(FULL, vb, ld), le = __shfl_sync(FULL, ve, ld);
      if (se - sb > le - lb) {
        int64_t t = sb; sb = lb; lb = t;
        t = se; se = le; le = t;
      }
      for (int64_t j = sb + lane; j < se; j += 32) cnt += bsearch_i32(ocl + lb, le - lb, ocl[j]);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(FULL, cnt, o);
  if (lane == 0 && cnt) atomicAdd(total, cnt);
}

}  // namespace

cudaError_t launch_cc_hook(const DevCSR& g, int32_t* parent, Ctl* ctl, int red_slot, int grid,
                           cudaStream_t st) {
  note_launch();
  cc_hook_kernel<<<grid, kBlock, 0, st>>>(g, parent, &ctl->red[red_slot]);
  return cudaGetLastError();
}
cudaError_t launch_cc_compress(int32_t* parent, int64_t n, cudaStream_t st) {
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  note_launch();
  cc_compress_kernel<<<grid, 256, 0, st>>>(parent, n);
  return cudaGetLastError();
}
cudaError_t launch_pr_init(double* rank, double* contrib, const int64_t* row_ptr, int64_t n,
                           cudaStream_t st) {
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  note_launch();
  pr_init_kernel<<<grid, 256, 0, st>>>(rank, contrib, row_ptr, n);
  return cudaGetLastError();
}
cudaError_t launch_pr_sweep(const DevCSR& g, const double* rank_old, double* rank_new,
                            const double* contrib, double* contrib_next, double d, double tol,
                            int64_t n_global, Ctl* ctl, int red_slot, int grid, const PrHubs& h,
                            cudaStream_t st) {
  const double base = (1.0 - d) / (double)n_global;
  if (h.nchunks > 0) {
    note_launch();
    pr_hub_kernel<<<grid, kBlock, 0, st>>>(g, contrib, h);
  }
  cudaMemsetAsync(&ctl->tile_ctr[red_slot], 0, sizeof(uint32_t), st);
  note_launch();
  pr_sweep_kernel<<<grid, kBlock, 0, st>>>(g, rank_old, rank_new, contrib, contrib_next, d, tol,
                                           base, h, ctl, red_slot);
  return cudaGetLastError();
}
int pr_persistent_blocks_per_sm() {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, pr_persistent_kernel, kBlock, 0);
  return nb;
}
cudaError_t launch_pr_persistent(const DevCSR& g, double* ra, double* rb, double* ca, double* cb,
                                 double d, double tol, int64_t n_global, Ctl* ctl,
                                 int64_t max_rounds, int cond_mode, int grid, const PrHubs& hubs,
                                 cudaStream_t st) {
  double base = (1.0 - d) / (double)n_global;
  DevCSR gg = g;
  PrHubs h = hubs;
  void* args[] = {&gg, &ra, &rb, &ca, &cb, &d, &tol, &base, &ctl, &max_rounds, &cond_mode, &h};
  note_launch();
  return cudaLaunchCooperativeKernel((void*)pr_persistent_kernel, grid, kBlock, args, 0, st);
}

cudaError_t tc_orient(const DevCSR& g, int64_t n, int64_t** rp_out, int32_t** cl_out,
                      int32_t** src_out, int64_t* m_out, cudaStream_t st) {
  int64_t* dout = nullptr;
  int64_t* orp = nullptr;
  int32_t* ocl = nullptr;
  int32_t* osrc = nullptr;
  cudaError_t e;
  if ((e = cudaMallocAsync(&dout, (n + 1) * sizeof(int64_t), st)) != cudaSuccess) return e;
  if ((e = cudaMallocAsync(&orp, (n + 1) * sizeof(int64_t), st)) != cudaSuccess) return e;
  const int grid = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  note_launch();
  tc_count_out_kernel<<<grid, 256, 0, st>>>(g.row_ptr, g.col, n, dout);
  cudaMemsetAsync(dout + n, 0, sizeof(int64_t), st);
  size_t tmp = 0;
  cub::DeviceScan::ExclusiveSum(nullptr, tmp, dout, orp, n + 1, st);
  void* t = nullptr;
  if ((e = cudaMallocAsync(&t, tmp, st)) != cudaSuccess) return e;
  cub::DeviceScan::ExclusiveSum(t, tmp, dout, orp, n + 1, st);
  int64_t mo = 0;
  cudaMemcpyAsync(&mo, orp + n, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  if ((e = cudaStreamSynchronize(st)) != cudaSuccess) return e;
  if ((e = cudaMallocAsync(&ocl, (mo > 0 ? mo : 1) * sizeof(int32_t), st)) != cudaSuccess) return e;
  if ((e = cudaMallocAsync(&osrc, (mo > 0 ? mo : 1) * sizeof(int32_t), st)) != cudaSuccess) return e;
  note_launch();
  tc_fill_kernel<<<grid, 256, 0, st>>>(g.row_ptr, g.col, n, orp, ocl, osrc);
  cudaFreeAsync(t, st);
  cudaFreeAsync(dout, st);
  *rp_out = orp;
  *cl_out = ocl;
  *src_out = osrc;
  *m_out = mo;
  return cudaGetLastError();
}

cudaError_t launch_tc_count(const int64_t* rp, const int32_t* cl, const int32_t* src, int64_t mo,
                            Ctl* ctl, cudaStream_t st) {
  cudaMemsetAsync(&ctl->tc_count, 0, sizeof(unsigned long long), st);
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>((mo + 255) / 256, 148 * 16));
  note_launch();
  tc_count_kernel<<<grid, 256, 0, st>>>(rp, cl, src, mo, &ctl->tc_count);
  return cudaGetLastError();
}

}  // namespace irgl
