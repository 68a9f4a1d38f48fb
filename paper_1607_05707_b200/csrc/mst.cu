// mst.cu — SURVEY §8f F3: IrGL's Atomic / Exclusive constructs on sm_100a and the program they
// exist for, Borůvka minimum spanning forest (Listing 1):
//
//   ForAll(nidx In wl) { n = wl.pop(nidx); n_component = components[n]; minwt = INF;
//     for (e In edges) { /* min cross-component edge out of n */ }
//     Atomic(component_locks[n_component]) { if (component_minwt[n_component] > minwt) {...} }
//     if (node has cross-component edge) wl.push(n) }
//
// followed by hooking of every component onto the other end of its minimum edge and pointer
// jumping, under Iterate While Any.  Edges are totally ordered by (w, min(u,v), max(u,v)), so the
// minimum-edge graph has only 2-cycles, broken toward the smaller component id.  The total forest
// weight is unique and is checked against Kruskal.
#include <cooperative_groups.h>

#include "constructs.cuh"
#include "kernels.h"

namespace cg = cooperative_groups;

namespace irgl {
namespace {
constexpr unsigned FULL = 0xffffffffu;

struct EdgeKey {
  int32_t w, a, b;  // a < b
};
__device__ __forceinline__ bool key_less(const EdgeKey& x, const EdgeKey& y) {
  return x.w != y.w ? x.w < y.w : (x.a != y.a ? x.a < y.a : x.b < y.b);
}
__device__ __forceinline__ EdgeKey warp_min_key(EdgeKey k) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    EdgeKey t{__shfl_xor_sync(FULL, k.w, o), __shfl_xor_sync(FULL, k.a, o),
              __shfl_xor_sync(FULL, k.b, o)};
    if (key_less(t, k)) k = t;
  }
  return k;
}

// find-min-edge (Listing 1): one lane per popped vertex, warp-cooperative scan for degree >= 32.
__global__ void __launch_bounds__(kBlock) mst_find_min_kernel(DevCSR g, const int32_t* comp,
                                                           int32_t* lock, int32_t* bw, int32_t* ba,
                                                           int32_t* bb, const uint32_t* in,
                                                           uint32_t nin, uint32_t* out,
                                                           uint32_t* out_cnt) {
  const int lane = lane_id();
  const uint32_t nwarps = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t base = ((blockIdx.x * blockDim.x + threadIdx.x) >> 5) * 32; base < nin;
       base += nwarps * 32) {
    const uint32_t i = base + lane;
    const bool valid = i < nin;
    int32_t n = 0, cn = 0;
    int64_t beg = 0, end = 0;
    if (valid) {
      n = (int32_t)in[i];
      cn = comp[n];
      beg = g.row_ptr[n];
      end = g.row_ptr[n + 1];
    }
    EdgeKey best{kInf, kInf, kInf};
    int64_t deg = end - beg;
    // warp-cooperative scan of high-degree vertices
    uint32_t wm = __ballot_sync(FULL, deg >= 32);
    while (wm) {
      const int leader = __ffs(wm) - 1;
      wm &= wm - 1;
      const int64_t b = __shfl_sync(FULL, beg, leader), e = __shfl_sync(FULL, end, leader);
      const int32_t nn = __shfl_sync(FULL, n, leader), cc = __shfl_sync(FULL, cn, leader);
      EdgeKey k{kInf, kInf, kInf};
      for (int64_t x = b + lane; x < e; x += 32) {
        const int32_t d = g.col[x];
        if (comp[d] != cc) {
          const EdgeKey t{g.w[x], min(nn, d), max(nn, d)};
          if (key_less(t, k)) k = t;
        }
      }
      k = warp_min_key(k);
      if (lane == leader) {
        best = k;
        deg = 0;
      }
    }
    for (int64_t x = beg; deg > 0 && x < end; ++x) {
      const int32_t d = g.col[x];
      if (comp[d] != cn) {
        const EdgeKey t{g.w[x], min(n, d), max(n, d)};
        if (key_less(t, best)) best = t;
      }
    }
    const bool has = valid && best.w != kInf;
    if (has) {
      // Atomic(component_locks[n_component]) { if (component_min > minwt) component_min = ... }
      volatile int32_t* vw = bw;
      volatile int32_t* va = ba;
      volatile int32_t* vb = bb;
      atomic_section(lock + cn, [&] {
        const EdgeKey cur{vw[cn], va[cn], vb[cn]};
        if (key_less(best, cur)) {
          vw[cn] = best.w;
          va[cn] = best.a;
          vb[cn] = best.b;
        }
      });
    }
    // if (node has cross-component edge) wl.push(n)   (warp-aggregated)
    const uint32_t m = __ballot_sync(FULL, has);
    if (m) {
      uint32_t pos = 0;
      if (lane == 0) pos = atomicAdd(out_cnt, __popc(m));
      pos = __shfl_sync(FULL, pos, 0);
      if (has) out[pos + __popc(m & lanemask_lt())] = (uint32_t)n;
    }
  }
}

// Hook every component root onto the other end of its minimum edge (2-cycles broken toward the
// smaller id, whose partner adds the shared edge once).  ReduceAndReturn(hooked) under Any.
__global__ void mst_hook_kernel(const int32_t* comp, int32_t* parent, const int32_t* bw,
                                const int32_t* ba, const int32_t* bb, int64_t n,
                                unsigned long long* wsum, unsigned long long* esum, uint32_t* cell) {
  bool hooked = false;
  for (int64_t c = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; c < n;
       c += (int64_t)gridDim.x * blockDim.x) {
    if (comp[c] != c || bw[c] == kInf) continue;
    const int32_t w = bw[c], a = ba[c], b = bb[c];
    const int32_t ca = comp[a], cb = comp[b];
    const int32_t o = ca == (int32_t)c ? cb : ca;
    const bool mutual = bw[o] == w && ba[o] == a && bb[o] == b;
    if (mutual && (int32_t)c < o) continue;
    parent[c] = o;
    atomicAdd(wsum, (unsigned long long)w);
    atomicAdd(esum, 1ull);
    hooked = true;
  }
  if (__any_sync(FULL, hooked) && lane_id() == 0) *(volatile uint32_t*)cell = 1u;  // E4
}

// Pointer jumping: every vertex adopts the root of its component; per-component minima reset.
__global__ void mst_compress_kernel(int32_t* comp, const int32_t* parent, int32_t* bw, int64_t n) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    int32_t x = comp[v];
    int32_t p = ld_label_cg(parent + x);
    while (p != x) {
      x = p;
      p = ld_label_cg(parent + x);
    }
    comp[v] = x;
    bw[v] = kInf;
  }
}

__global__ void mst_init_kernel(int32_t* parent, int32_t* comp, int32_t* lock, int32_t* bw,
                                int32_t* ba, int32_t* bb, uint32_t* wl, int64_t n) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n;
       v += (int64_t)gridDim.x * blockDim.x) {
    parent[v] = comp[v] = (int32_t)v;
    lock[v] = 0;
    bw[v] = ba[v] = bb[v] = kInf;
    wl[v] = (uint32_t)v;  // Listing 1: "The worklist initially contains all nodes"
  }
}

// ---- test operators for the constructs (SPEC.md:551-552 acceptance items 3, 4) -----------------
// ATOMIC: every item increments one counter inside a blocking Atomic -> counter == items.
// ATOMIC_ELSE: one attempt per item; with the lock pre-held every item runs the Else branch.
__global__ void atomic_test_kernel(const uint32_t* in, uint32_t nin, int32_t* lock, int32_t* log,
                                   int else_form) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < nin; i += gridDim.x * blockDim.x) {
    (void)in[i];
    volatile int32_t* counter = log;
    if (!else_form) {
      atomic_section(lock, [&] { counter[0] = counter[0] + 1; });
    } else {
      atomic_try(lock, [&] { counter[0] = counter[0] + 1; }, [&] { atomicAdd(log + 1, 1); });
    }
  }
}

// EXCLUSIVE: item x claims locks[x*k .. x*k+k) (-1 unused); three phases with SyncRunningThreads.
__global__ void exclusive_test_kernel(const uint32_t* in, uint32_t nin, const int32_t* locks,
                                      int k, int32_t* owner, int32_t* won, int32_t* log) {
  cg::grid_group grid = cg::this_grid();
  const uint32_t T = gridDim.x * blockDim.x;
  const uint32_t t0 = blockIdx.x * blockDim.x + threadIdx.x;
  for (uint32_t i = t0; i < nin; i += T) {  // phase 1: claim
    const int32_t x = (int32_t)in[i];
    for (int j = 0; j < k; ++j) {
      const int32_t l = locks[x * k + j];
      if (l >= 0) atomicMin(owner + l, x);
    }
  }
  grid.sync();  // SyncRunningThreads
  for (uint32_t i = t0; i < nin; i += T) {  // phase 2: does the item still hold every claim?
    const int32_t x = (int32_t)in[i];
    bool all = true;
    for (int j = 0; j < k; ++j) {
      const int32_t l = locks[x * k + j];
      if (l >= 0 && ld_label_cg(owner + l) != x) all = false;
    }
    won[x] = all ? 1 : 0;
  }
  grid.sync();  // SyncRunningThreads
  for (uint32_t i = t0; i < nin; i += T) {  // phase 3: confirm -> locked stmts / Else
    const int32_t x = (int32_t)in[i];
    if (ld_label_cg(won + x)) log[x] = 1;  // locked stmts
    else log[x] = 0;                       // failed stmts
  }
}
}  // namespace

cudaError_t launch_mst_init(int32_t* parent, int32_t* comp, int32_t* lock, int32_t* bw, int32_t* ba,
                            int32_t* bb, uint32_t* wl, int64_t n, cudaStream_t st) {
  note_launch();
  mst_init_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(parent, comp, lock,
                                                                                    bw, ba, bb, wl, n);
  return cudaGetLastError();
}

cudaError_t launch_mst_round(const DevCSR& g, int32_t* parent, int32_t* comp, int32_t* lock,
                             int32_t* bw, int32_t* ba, int32_t* bb, const uint32_t* in, uint32_t nin,
                             uint32_t* out, uint32_t* out_cnt, unsigned long long* wsum,
                             unsigned long long* esum, uint32_t* cell, int64_t n, int grid,
                             cudaStream_t st) {
  if (nin) {
    note_launch();
    mst_find_min_kernel<<<std::min<int>(grid, (int)((nin + kBlock - 1) / kBlock)), kBlock, 0, st>>>(
        g, comp, lock, bw, ba, bb, in, nin, out, out_cnt);
  }
  const int g2 = (int)std::min<int64_t>((n + 255) / 256, 148 * 16);
  note_launch();
  mst_hook_kernel<<<g2, 256, 0, st>>>(comp, parent, bw, ba, bb, n, wsum, esum, cell);
  note_launch();
  mst_compress_kernel<<<g2, 256, 0, st>>>(comp, parent, bw, n);
  return cudaGetLastError();
}

cudaError_t launch_atomic_test(const uint32_t* in, uint32_t nin, int32_t* lock, int32_t* log,
                               int else_form, int threads, cudaStream_t st) {
  const int bs = threads < 256 ? (threads > 0 ? threads : 1) : 256;
  note_launch();
  atomic_test_kernel<<<(threads + bs - 1) / bs, bs, 0, st>>>(in, nin, lock, log, else_form);
  return cudaGetLastError();
}

int exclusive_blocks_per_sm() {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, exclusive_test_kernel, kBlock, 0);
  return nb;
}

cudaError_t launch_exclusive_test(const uint32_t* in, uint32_t nin, const int32_t* locks, int k,
                                  int32_t* owner, int32_t* won, int32_t* log, int grid,
                                  cudaStream_t st) {
  void* args[] = {(void*)&in, (void*)&nin, (void*)&locks, (void*)&k, (void*)&owner, (void*)&won,
                  (void*)&log};
  note_launch();
  return cudaLaunchCooperativeKernel((void*)exclusive_test_kernel, grid, kBlock, args, 0, st);
}

}  // namespace irgl
