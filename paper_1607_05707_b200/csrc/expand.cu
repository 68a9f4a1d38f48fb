// expand.cu — the data-driven hot path: ForAll over the in-worklist x ForAll over edges(n)
// for BFS (Listing 2), SSSP and CC_LP, lowered B200-first:
//
//  E1  nested-parallelism edge scheduler.  Each popped vertex's edges go to
//        - one thread          (degree < warp_t): CTA-wide scan, edge ids staged in smem and
//                              processed one edge per thread ("fine-grained" gather);
//        - one warp            (warp_t <= degree < cta_t), 128-bit col/weight loads;
//        - CTA chunks          (degree >= cta_t): split into chunk_edges-sized descriptors that
//                              every CTA of the grid drains in a second phase (edge-balanced,
//                              so super-hubs do not serialise on one CTA).
//  E2  cooperative conversion of pushes: warp __ballot_sync/__popc aggregation into a per-CTA
//      shared-memory staging queue, flushed with ONE global atomic reservation per tile.
//  E3  iteration outlining: the Iterate loop as one cooperative persistent kernel with a grid
//      barrier (SyncRunningThreads) instead of per-round host launches.
//
// Reference semantics (SPEC.md:317-322 ForAll lowering; :425 bulk-synchronous worklists: pops
// read `in`, pushes append to `out`, never visible in the same launch).
#include <cooperative_groups.h>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace irgl {
namespace {

constexpr unsigned FULL = 0xffffffffu;

struct Smem {
  // cooperative-conversion push staging
  uint32_t push_cnt;
  uint32_t push_base;
  uint32_t push_buf[kPushBuf];
  // fine-grained gather window
  int64_t fg_edge[kBlock];
  int32_t fg_src[kBlock];
  // block scan scratch
  uint32_t warp_tot[kWarps];
  unsigned long long warp_edges[kWarps];
  // chunk descriptor broadcast
  ChunkDesc chunk;
  int32_t chunk_src;
};

struct KParams {
  DevCSR g;
  int32_t* lab;
  int32_t* stamp;
  Ctl* ctl;
  DistRoute dr;
  ExpandCfg ec;
};

// ---- relax: the operator body for one edge (n -> dst) ----------------------------------------
// BFS   : if level[dst]==INF { level[dst]=LEVEL; push(dst) }   CAS dedupes the push.
// SSSP  : nd = dist[n]+w;  if atomicMin(dist[dst],nd) > nd and stamp[dst] != round: push(dst)
// CC_LP : nd = label[n];   same as SSSP.
template <int OP>
__device__ __forceinline__ bool relax_with(const KParams& p, int32_t cur, int32_t sv, int32_t wt,
                                           uint32_t dst, int32_t level, int32_t stamp_id) {
  if (OP == IRGL_OP_BFS) {
    if (cur != kInf) return false;
    return atomicCAS(p.lab + dst, kInf, level) == kInf;
  } else {
    const int32_t nd = (OP == IRGL_OP_SSSP) ? sv + wt : sv;
    if (nd >= cur) return false;
    const int32_t old = atomicMin(p.lab + dst, nd);
    if (nd >= old) return false;
    return atomicExch(p.stamp + dst, stamp_id) != stamp_id;
  }
}

// ---- push: E2 cooperative conversion ----------------------------------------------------------
// Every lane of the warp must call this (converged).  Local destinations are staged in shared
// memory (one smem atomic per warp); a full staging buffer spills straight to global with one
// atomic per warp.  Remote destinations (multi-partition) go to the owner's bucket, grouped
// per owner with __match_any_sync.
template <bool DIST>
__device__ __forceinline__ void push(Smem& sm, const KParams& p, const RoundBufs& rb, bool pred,
                                     uint32_t v) {
  uint32_t m = __ballot_sync(FULL, pred);
  if (m == 0) return;
  const uint32_t lane = lane_id();
  if (DIST) {
    const int owner = pred ? (int)((int64_t)v / p.dr.part_size) : -1;
    const bool remote = pred && owner != p.dr.me;
    const uint32_t rm = __ballot_sync(FULL, remote);
    if (rm) {
      if (remote) {
        const uint32_t grp = __match_any_sync(rm, owner);
        const uint32_t leader = __ffs(grp) - 1;
        uint32_t base = 0;
        if (lane == leader) base = atomicAdd(p.dr.send_cnt + owner, __popc(grp));
        base = __shfl_sync(grp, base, leader);
        const uint32_t pos = base + __popc(grp & lanemask_lt());
        if (pos < (uint32_t)p.dr.part_size)
          p.dr.send[(int64_t)owner * p.dr.part_size + pos] = v;
        else
          atomicOr(&p.ctl->overflow, 1u);
      }
      if (lane == __ffs(rm) - 1) atomicAdd(&p.ctl->remote, (unsigned long long)__popc(rm));
      pred = pred && !remote;
      m = __ballot_sync(FULL, pred);
      if (m == 0) return;
    }
  }
  const uint32_t n = __popc(m);
  const uint32_t leader = __ffs(m) - 1;
  uint32_t pos = 0;
  if (lane == leader) pos = atomicAdd(&sm.push_cnt, n);
  pos = __shfl_sync(FULL, pos, leader);
  const uint32_t rank = __popc(m & lanemask_lt());
  // slots [pos, kPushBuf) go to smem, the remainder spills to global
  const uint32_t in_smem = pos >= (uint32_t)kPushBuf ? 0u : min(n, (uint32_t)kPushBuf - pos);
  uint32_t gbase = 0;
  if (in_smem < n) {
    if (lane == leader) gbase = atomicAdd(rb.out_cnt, n - in_smem);
    gbase = __shfl_sync(FULL, gbase, leader);
  }
  if (pred) {
    if (rank < in_smem) {
      sm.push_buf[pos + rank] = v;
    } else {
      const uint32_t q = gbase + (rank - in_smem);
      if (q < rb.cap) rb.out[q] = v;
      else atomicOr(&p.ctl->overflow, 1u);
    }
  }
}

// Flush the CTA's staged pushes: one global reservation per tile (CTA-uniform call site).
__device__ __forceinline__ void flush_pushes(Smem& sm, const KParams& p, const RoundBufs& rb) {
  __syncthreads();  // all pushes of the tile are staged
  const uint32_t c = min(sm.push_cnt, (uint32_t)kPushBuf);
  if (threadIdx.x == 0) sm.push_base = c ? atomicAdd(rb.out_cnt, c) : 0u;
  __syncthreads();  // push_base visible; nobody reads push_cnt past this point
  if (threadIdx.x == 0) sm.push_cnt = 0;
  const uint32_t base = sm.push_base;
  for (uint32_t i = threadIdx.x; i < c; i += kBlock) {
    const uint32_t q = base + i;
    if (q < rb.cap) rb.out[q] = sm.push_buf[i];
    else atomicOr(&p.ctl->overflow, 1u);
  }
  __syncthreads();  // staging buffer and counter reusable
}

// ---- edge-range processing by a group of G lanes (G = 32 warp, G = kBlock CTA) -------------------
// Head/tail (misaligned) edges in one predicated step, the aligned body with 128-bit loads:
// each lane issues 4 independent label gathers before its 4 decisions (ILP).
template <int OP, bool DIST, int G>
__device__ __forceinline__ void process_range(Smem& sm, const KParams& p, const RoundBufs& rb,
                                              int64_t b, int64_t e, int32_t sv, int gl) {
  const int32_t* __restrict__ col = p.g.col;
  const int32_t* __restrict__ w = p.g.w;
  const int64_t a0 = min((b + 3) & ~int64_t(3), e);
  const int64_t a1 = max(e & ~int64_t(3), a0);
  {
    const int nh = (int)(a0 - b), nt = (int)(e - a1);
    const bool act = gl < nh + nt;
    const int64_t ed = gl < nh ? b + gl : a1 + (gl - nh);
    uint32_t dst = 0;
    int32_t wt = 0, cur = 0;
    if (act) {
      dst = (uint32_t)ld_stream(col + ed);
      if (OP == IRGL_OP_SSSP) wt = ld_stream(w + ed);
      cur = ld_label(p.lab + dst);
    }
    const bool pr = act && relax_with<OP>(p, cur, sv, wt, dst, rb.level, rb.stamp_id);
    push<DIST>(sm, p, rb, pr, dst);
  }
  const int64_t q1 = a1 >> 2;
  for (int64_t q0 = a0 >> 2; q0 < q1; q0 += G) {
    const int64_t q = q0 + gl;
    const bool act = q < q1;
    int4 c4 = make_int4(0, 0, 0, 0), w4 = make_int4(0, 0, 0, 0);
    int32_t l0 = 0, l1 = 0, l2 = 0, l3 = 0;
    if (act) {
      c4 = ld_stream_v4(col + 4 * q);
      if (OP == IRGL_OP_SSSP) w4 = ld_stream_v4(w + 4 * q);
      l0 = ld_label(p.lab + c4.x);
      l1 = ld_label(p.lab + c4.y);
      l2 = ld_label(p.lab + c4.z);
      l3 = ld_label(p.lab + c4.w);
    }
    const bool p0 = act && relax_with<OP>(p, l0, sv, w4.x, (uint32_t)c4.x, rb.level, rb.stamp_id);
    const bool p1 = act && relax_with<OP>(p, l1, sv, w4.y, (uint32_t)c4.y, rb.level, rb.stamp_id);
    const bool p2 = act && relax_with<OP>(p, l2, sv, w4.z, (uint32_t)c4.z, rb.level, rb.stamp_id);
    const bool p3 = act && relax_with<OP>(p, l3, sv, w4.w, (uint32_t)c4.w, rb.level, rb.stamp_id);
    push<DIST>(sm, p, rb, p0, (uint32_t)c4.x);
    push<DIST>(sm, p, rb, p1, (uint32_t)c4.y);
    push<DIST>(sm, p, rb, p2, (uint32_t)c4.z);
    push<DIST>(sm, p, rb, p3, (uint32_t)c4.w);
  }
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

// ---- one tile of kBlock worklist items (consecutive mapping) ------------------------
template <int OP, bool DIST>
__device__ void expand_tile(Smem& sm, const KParams& p, const RoundBufs& rb, uint32_t tile_base) {
  const int tid = threadIdx.x;
  const int lane = tid & 31, warp = tid >> 5;
  const uint32_t i = tile_base + tid;
  const bool valid = i < rb.nin;
  uint32_t v = 0;
  int64_t beg = 0, end = 0;
  int32_t sv = 0;
  if (valid) {
    v = ld_item(rb.in + i);  // n = wl.pop(i)
    const int64_t lv = (int64_t)v - p.g.lo;
    beg = __ldg(p.g.row_ptr + lv);
    end = __ldg(p.g.row_ptr + lv + 1);
    if (OP != IRGL_OP_BFS) sv = ld_label(p.lab + v);
  }
  int64_t deg = end - beg;

  // stats: edges scanned per tile (one 64-bit atomic per CTA tile)
  {
    unsigned long long de = (unsigned long long)deg;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) de += __shfl_xor_sync(FULL, de, o);
    if (lane == 0) sm.warp_edges[warp] = de;
  }

  // ---- CTA-chunk level: degree >= cta_t -> chunk descriptors (warp-cooperative emission)
  {
    const bool big = deg >= p.ec.cta_t;
    uint32_t bm = __ballot_sync(FULL, big);
    while (bm) {
      const int leader = __ffs(bm) - 1;
      bm &= bm - 1;
      const int64_t b = __shfl_sync(FULL, beg, leader);
      const int64_t e = __shfl_sync(FULL, end, leader);
      const uint32_t vv = __shfl_sync(FULL, v, leader);
      const int64_t ce = p.ec.chunk_edges;
      const uint32_t nch = (uint32_t)((e - b + ce - 1) / ce);
      uint32_t base = 0;
      if (lane == 0) base = atomicAdd(rb.chunk_cnt, nch);
      base = __shfl_sync(FULL, base, 0);
      for (uint32_t k = lane; k < nch; k += 32) {
        const uint32_t pos = base + k;
        const int64_t cb = b + (int64_t)k * ce;
        if (pos < rb.chunk_cap) {
          ChunkDesc d;
          d.beg = cb;
          d.v = vv;
          d.len = (uint32_t)min(ce, e - cb);
          rb.chunks[pos] = d;
        } else {
          atomicOr(&p.ctl->overflow, 2u);
        }
      }
    }
    if (big) deg = 0;
  }

  // ---- warp level: warp_t <= degree < cta_t
  {
    uint32_t wm = __ballot_sync(FULL, deg >= p.ec.warp_t);
    while (wm) {
      const int leader = __ffs(wm) - 1;
      wm &= wm - 1;
      const int64_t b = __shfl_sync(FULL, beg, leader);
      const int64_t e = __shfl_sync(FULL, end, leader);
      const int32_t s = __shfl_sync(FULL, sv, leader);
      if (lane == leader) deg = 0;
      process_range<OP, DIST, 32>(sm, p, rb, b, e, s, lane);
    }
  }

  // ---- thread level (fine-grained): CTA exclusive scan of the remaining small degrees
  const uint32_t d = (uint32_t)deg;
  uint32_t incl = d;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t t = __shfl_up_sync(FULL, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) sm.warp_tot[warp] = incl;
  __syncthreads();
  uint32_t wpre = 0, total = 0;
#pragma unroll
  for (int k = 0; k < kWarps; ++k) {
    const uint32_t t = sm.warp_tot[k];
    if (k < warp) wpre += t;
    total += t;
  }
  if (tid == 0) {
    unsigned long long te = 0;
#pragma unroll
    for (int k = 0; k < kWarps; ++k) te += sm.warp_edges[k];
    if (te) atomicAdd(&p.ctl->edges, te);
  }
  const uint32_t off = wpre + incl - d;
  for (uint32_t wbase = 0; wbase < total; wbase += kBlock) {
    const uint32_t s0 = max(off, wbase), s1 = min(off + d, wbase + (uint32_t)kBlock);
    for (uint32_t k = s0; k < s1; ++k) {
      sm.fg_edge[k - wbase] = beg + (int64_t)(k - off);
      sm.fg_src[k - wbase] = sv;
    }
    __syncthreads();
    const uint32_t cnt = min((uint32_t)kBlock, total - wbase);
    const bool act = (uint32_t)tid < cnt;
    uint32_t dst = 0;
    int32_t wt = 0, s = 0, cur = 0;
    if (act) {
      const int64_t ed = sm.fg_edge[tid];
      s = sm.fg_src[tid];
      dst = (uint32_t)ld_stream(p.g.col + ed);
      if (OP == IRGL_OP_SSSP) wt = ld_stream(p.g.w + ed);
      cur = ld_label(p.lab + dst);
    }
    const bool pr = act && relax_with<OP>(p, cur, s, wt, dst, rb.level, rb.stamp_id);
    push<DIST>(sm, p, rb, pr, dst);
    __syncthreads();
  }
  flush_pushes(sm, p, rb);
}

// ---- CTA-chunk phase: every CTA drains chunk descriptors (grid-stride) ------------------------
template <int OP, bool DIST>
__device__ void chunk_phase(Smem& sm, const KParams& p, const RoundBufs& rb, uint32_t nch) {
  nch = min(nch, rb.chunk_cap);
  for (uint32_t c = blockIdx.x; c < nch; c += gridDim.x) {
    if (threadIdx.x == 0) {
      sm.chunk = rb.chunks[c];
      sm.chunk_src = (OP != IRGL_OP_BFS) ? ld_label(p.lab + sm.chunk.v) : 0;
    }
    __syncthreads();
    const int64_t b = sm.chunk.beg, e = b + sm.chunk.len;
    const int32_t s = sm.chunk_src;
    process_range<OP, DIST, kBlock>(sm, p, rb, b, e, s, threadIdx.x);
    flush_pushes(sm, p, rb);  // begins with __syncthreads: chunk smem reuse is safe
  }
}

template <int OP, bool DIST>
__global__ void __launch_bounds__(kBlock, 4) expand_kernel(KParams p, RoundBufs rb) {
  __shared__ Smem sm;
  if (threadIdx.x == 0) sm.push_cnt = 0;
  __syncthreads();
  for (uint32_t t = blockIdx.x * kBlock; t < rb.nin; t += gridDim.x * kBlock)
    expand_tile<OP, DIST>(sm, p, rb, t);
}

template <int OP, bool DIST>
__global__ void __launch_bounds__(kBlock, 4) chunk_kernel(KParams p, RoundBufs rb) {
  __shared__ Smem sm;
  if (threadIdx.x == 0) sm.push_cnt = 0;
  __syncthreads();
  chunk_phase<OP, DIST>(sm, p, rb, ld_ctl(rb.chunk_cnt));
}

// ---- E3: outlined Iterate.  One cooperative launch; rounds separated by grid.sync() --------------
// Worklist buffers alternate by round parity; counters rotate over three slots so the counter
// cleared during round r (slot (r+2)%3, last read during round r-1) is the out-counter of round
// r+1: no extra barrier is needed to reset it ("swap in/out and reset out").
template <int OP>
__global__ void __launch_bounds__(kBlock, 4) persistent_kernel(KParams p, PersistArgs a) {
  __shared__ Smem sm;
  cg::grid_group grid = cg::this_grid();
  if (threadIdx.x == 0) sm.push_cnt = 0;
  __syncthreads();
  uint32_t* cnt = p.ctl->cnt;
  for (uint32_t r = 0;; ++r) {
    uint32_t* cin = cnt + a.slot[r % 3];
    uint32_t* cout = cnt + a.slot[(r + 1) % 3];
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      cnt[a.slot[(r + 2) % 3]] = 0;
      p.ctl->chunk_cnt[(r + 1) % 3] = 0;
    }
    RoundBufs rb;
    rb.in = (r & 1) ? a.buf_b : a.buf_a;
    rb.nin = ld_ctl(cin);
    rb.out = (r & 1) ? a.buf_a : a.buf_b;
    rb.out_cnt = cout;
    rb.cap = a.cap;
    rb.chunks = a.chunks;
    rb.chunk_cnt = &p.ctl->chunk_cnt[r % 3];
    rb.chunk_cap = a.chunk_cap;
    rb.level = a.level0 + (int32_t)r;
    rb.stamp_id = a.stamp0 + (int32_t)r;
    for (uint32_t t = blockIdx.x * kBlock; t < rb.nin; t += gridDim.x * kBlock)
      expand_tile<OP, false>(sm, p, rb, t);
    grid.sync();  // SyncRunningThreads
    const uint32_t nch = ld_ctl(rb.chunk_cnt);
    if (nch) {
      chunk_phase<OP, false>(sm, p, rb, nch);
      grid.sync();
    }
    const uint32_t nout = ld_ctl(cout);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      p.ctl->popped += rb.nin;
      p.ctl->pushes += nout;
    }
    // Iterate termination: in empty (next round) [Or rounds >= max_rounds]
    if (nout == 0 || (a.max_rounds > 0 && (int64_t)r + 1 >= a.max_rounds)) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        p.ctl->rounds = r + 1;
        p.ctl->exit_in_slot = (int32_t)((r + 1) & 1);
      }
      break;
    }
  }
}

// ---- owner-side application of remote updates (E5 min-reduce) ---------------------------------
template <int OP>
__global__ void __launch_bounds__(kBlock) apply_remote_kernel(int32_t* lab, int32_t* stamp, Ctl* ctl,
                                                           const uint32_t* items,
                                                           const int32_t* values, uint32_t n,
                                                           uint32_t* out, uint32_t* out_cnt,
                                                           uint32_t cap, int32_t level,
                                                           int32_t stamp_id) {
  const uint32_t lane = lane_id();
  for (uint32_t i0 = blockIdx.x * kBlock; i0 < n; i0 += gridDim.x * kBlock) {
    const uint32_t i = i0 + threadIdx.x;
    bool pr = false;
    uint32_t v = 0;
    if (i < n) {
      v = items[i];
      if (OP == IRGL_OP_BFS) {
        pr = ld_label(lab + v) == kInf && atomicCAS(lab + v, kInf, level) == kInf;
      } else {
        const int32_t nd = values[i];
        pr = nd < ld_label(lab + v) && atomicMin(lab + v, nd) > nd &&
             atomicExch(stamp + v, stamp_id) != stamp_id;
      }
    }
    const uint32_t m = __ballot_sync(FULL, pr);
    if (m) {
      const uint32_t leader = __ffs(m) - 1;
      uint32_t base = 0;
      if (lane == leader) base = atomicAdd(out_cnt, __popc(m));
      base = __shfl_sync(FULL, base, leader);
      if (pr) {
        const uint32_t q = base + __popc(m & lanemask_lt());
        if (q < cap) out[q] = v;
        else atomicOr(&ctl->overflow, 1u);
      }
    }
  }
}

__global__ void pack_values_kernel(const int32_t* lab, const uint32_t* items, int32_t* values,
                                   uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    values[i] = ld_label(lab + items[i]);
}

template <int OP, bool DIST>
cudaError_t round_impl(const KParams& kp, const RoundBufs& rb, int grid_max, cudaStream_t st) {
  if (rb.nin > 0) {
    const int tiles = (int)((rb.nin + kBlock - 1) / kBlock);
    expand_kernel<OP, DIST><<<min(tiles, grid_max), kBlock, 0, st>>>(kp, rb);
  }
  chunk_kernel<OP, DIST><<<grid_max, kBlock, 0, st>>>(kp, rb);
  return cudaGetLastError();
}

}  // namespace

cudaError_t launch_expand_round(int op, const DevCSR& g, int32_t* lab, int32_t* stamp, Ctl* ctl,
                                const RoundBufs& rb, const DistRoute& dr, const ExpandCfg& ec,
                                int grid_max, cudaStream_t st) {
  KParams kp{g, lab, stamp, ctl, dr, ec};
  const bool dist = dr.nparts > 1;
  switch (op) {
    case IRGL_OP_BFS:
      return dist ? round_impl<IRGL_OP_BFS, true>(kp, rb, grid_max, st)
                  : round_impl<IRGL_OP_BFS, false>(kp, rb, grid_max, st);
    case IRGL_OP_SSSP:
      return dist ? round_impl<IRGL_OP_SSSP, true>(kp, rb, grid_max, st)
                  : round_impl<IRGL_OP_SSSP, false>(kp, rb, grid_max, st);
    case IRGL_OP_CC_LP:
      return dist ? round_impl<IRGL_OP_CC_LP, true>(kp, rb, grid_max, st)
                  : round_impl<IRGL_OP_CC_LP, false>(kp, rb, grid_max, st);
  }
  return cudaErrorInvalidValue;
}

cudaError_t launch_apply_remote(int op, int32_t* lab, int32_t* stamp, Ctl* ctl, const uint32_t* items,
                                const int32_t* values, uint32_t n, uint32_t* out, uint32_t* out_cnt,
                                uint32_t cap, int32_t level, int32_t stamp_id, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  const int grid = (int)min((n + kBlock - 1) / kBlock, 148u * 8u);
  switch (op) {
    case IRGL_OP_BFS:
      apply_remote_kernel<IRGL_OP_BFS><<<grid, kBlock, 0, st>>>(lab, stamp, ctl, items, values, n,
                                                                out, out_cnt, cap, level, stamp_id);
      break;
    case IRGL_OP_SSSP:
      apply_remote_kernel<IRGL_OP_SSSP><<<grid, kBlock, 0, st>>>(lab, stamp, ctl, items, values, n,
                                                                 out, out_cnt, cap, level, stamp_id);
      break;
    case IRGL_OP_CC_LP:
      apply_remote_kernel<IRGL_OP_CC_LP><<<grid, kBlock, 0, st>>>(lab, stamp, ctl, items, values, n,
                                                                  out, out_cnt, cap, level, stamp_id);
      break;
    default:
      return cudaErrorInvalidValue;
  }
  return cudaGetLastError();
}

cudaError_t launch_pack_values(const int32_t* lab, const uint32_t* items, int32_t* values,
                               uint32_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  pack_values_kernel<<<(int)min((n + 255) / 256, 4096u), 256, 0, st>>>(lab, items, values, n);
  return cudaGetLastError();
}

int persistent_blocks_per_sm(int op) {
  int nb = 0;
  switch (op) {
    case IRGL_OP_BFS:
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, persistent_kernel<IRGL_OP_BFS>, kBlock, 0);
      break;
    case IRGL_OP_SSSP:
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, persistent_kernel<IRGL_OP_SSSP>, kBlock, 0);
      break;
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

cudaError_t launch_persistent(int op, const DevCSR& g, int32_t* lab, int32_t* stamp, Ctl* ctl,
                              const PersistArgs& pa, const ExpandCfg& ec, int grid,
                              cudaStream_t st) {
  KParams kp{g, lab, stamp, ctl, DistRoute{1, 0, 1, nullptr, nullptr}, ec};
  PersistArgs a = pa;
  void* args[] = {&kp, &a};
  switch (op) {
    case IRGL_OP_BFS:
      return cudaLaunchCooperativeKernel((void*)persistent_kernel<IRGL_OP_BFS>, grid, kBlock, args, 0, st);
    case IRGL_OP_SSSP:
      return cudaLaunchCooperativeKernel((void*)persistent_kernel<IRGL_OP_SSSP>, grid, kBlock, args, 0, st);
    case IRGL_OP_CC_LP:
      return cudaLaunchCooperativeKernel((void*)persistent_kernel<IRGL_OP_CC_LP>, grid, kBlock, args, 0, st);
  }
  return cudaErrorInvalidValue;
}

}  // namespace irgl
