// testops.cu — the tiny operators the reference's own examples are phrased in (SPEC.md:439,
// :448-449, :465-466, :553-554, :557), run through the SAME pipe/worklist/orchestration machinery
// as the graph operators, plus small utility kernels.
#include <cooperative_groups.h>

#include "kernels.h"

namespace cg = cooperative_groups;

namespace irgl {
namespace {
constexpr unsigned FULL = 0xffffffffu;

// Warp-aggregated append (E2) used by the test kernels.
__device__ __forceinline__ void wl_append(bool pred, uint32_t v, uint32_t* buf, uint32_t* cnt,
                                          uint32_t cap, uint32_t* overflow) {
  const uint32_t active = __activemask();
  const uint32_t m = __ballot_sync(active, pred);
  if (!m) return;
  const uint32_t leader = __ffs(m) - 1;
  uint32_t base = 0;
  if (lane_id() == leader) base = atomicAdd(cnt, __popc(m));
  base = __shfl_sync(active, base, leader);
  if (pred) {
    const uint32_t q = base + __popc(m & lanemask_lt());
    if (q < cap) buf[q] = v;
    else atomicOr(overflow, 1u);
  }
}

// ForAll(i In wl) with the requested mapping: consecutive = grid-stride from
// the global thread id; blocked = contiguous ceil(N/T) chunk per thread.  Thread `tid` of `T`;
// the Any/All fold ends in one idempotent store per warp (E4).  Shared by the standalone launch
// and the outlined Pipe control kernel.
__device__ void test_op_body(const TestArgs& a, uint32_t tid, uint32_t T) {
  uint32_t begin, end, step;
  if (a.mapping == IRGL_MAP_BLOCKED) {
    const uint32_t chunk = (a.nin + T - 1) / T;
    begin = tid * chunk;
    end = min(a.nin, begin + chunk);
    step = 1;
  } else {
    begin = tid;
    end = a.nin;
    step = T;
  }
  bool any = false, all = true;
  for (uint32_t i = begin; i < end; i += step) {
    const uint32_t x = a.in[i];  // x = wl.pop(i)
    switch (a.op) {
      case IRGL_OP_TEST_COUNTDOWN:
        wl_append((int64_t)x + 1 < a.guard, x + 1, a.out, a.out_cnt, a.cap, a.overflow);
        break;
      case IRGL_OP_TEST_RESPAWN_ODD:
      case IRGL_OP_TEST_RETRY_ODD: {
        const int64_t g = a.guard > 0 ? a.guard : 1;
        bool retry = false;
        if ((x & 1u) && a.rcount[x] < g) {
          a.rcount[x] += 1;
          retry = true;
        }
        wl_append(retry, x, a.retry, a.retry_cnt, a.cap, a.overflow);   // Retry x
        wl_append(!retry, x, a.out, a.out_cnt, a.cap, a.overflow);      // push x
      } break;
      case IRGL_OP_TEST_REDUCE: {
        const bool b = a.values[x] != 0;  // ReduceAndReturn(values[x]): ends this iteration
        any |= b;
        all &= b;
      } break;
      case IRGL_OP_TEST_PUSHPOP:
        a.log[x] = a.launch_no;
        wl_append((int64_t)x + a.guard < a.cap, (uint32_t)(x + a.guard), a.out, a.out_cnt, a.cap,
                  a.overflow);
        break;
      case IRGL_OP_TEST_FORALL_MAP:
        a.log[x] = (int32_t)tid;
        break;
      default:  // IRGL_OP_TEST_NOPUSH
        break;
    }
  }
  // per-thread partial aggregation, then one idempotent store per warp (E4); the active mask
  // covers partial warps (outlined Pipes run at the block size T_control chooses)
  const uint32_t am = __activemask();
  if (a.reduction == IRGL_RED_ANY) {
    if (__any_sync(am, any) && lane_id() == __ffs(am) - 1) *(volatile uint32_t*)a.red = 1u;
  } else if (a.reduction == IRGL_RED_ALL) {
    if (!__all_sync(am, all) && lane_id() == __ffs(am) - 1) *(volatile uint32_t*)a.red = 0u;
  }
}

__global__ void test_op_kernel(TestArgs a) {
  test_op_body(a, blockIdx.x * blockDim.x + threadIdx.x, gridDim.x * blockDim.x);
}

// ---- outlined Pipe ---------------------------------------
// One cooperative control kernel runs the whole Pipe: the member kernels' bodies are called
// directly between grid barriers (SyncRunningThreads), the in/out/retry roles are three buffer
// indices every thread updates identically, and the per-buffer counters live in cnt[3].
// Invoke = launch; while retry is non-empty: swap in<->retry, relaunch (out kept; serialised
// after retry_serialize_after rounds unless Respawn); then swap in<->out.
// Global thread 0 owns every counter reset and the statistics; a grid barrier separates each
// reset from the next use.
__device__ __forceinline__ uint32_t ld_vol_u32(const uint32_t* p) { return *(volatile const uint32_t*)p; }

__device__ int pipe_invoke(cg::grid_group& grid, const PipeProgDev& P, const PipeStageDev& S,
                           int& bi, int& bo, int& br, int32_t& launch_no) {
  const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t T = gridDim.x * blockDim.x;
  if (gtid == 0) {
    *P.red = S.reduction == IRGL_RED_ALL ? 1u : 0u;  // return cell identity
    P.cnt[br] = 0;
  }
  grid.sync();
  int retry_rounds = 0;
  for (;;) {
    const bool serial = S.op != IRGL_OP_TEST_RESPAWN_ODD && retry_rounds > P.rsa;  // Respawn: never
    const uint32_t nin = ld_vol_u32(P.cnt + bi);
    ++launch_no;
    TestArgs a;
    a.op = S.op;
    a.in = P.buf[bi];
    a.nin = nin;
    a.out = P.buf[bo];
    a.out_cnt = P.cnt + bo;
    a.retry = P.buf[br];
    a.retry_cnt = P.cnt + br;
    a.cap = P.cap;
    a.guard = S.guard;
    a.values = S.values;
    a.rcount = P.rcount;
    a.log = P.log;
    a.launch_no = launch_no;
    a.mapping = S.mapping;
    a.red = P.red;
    a.reduction = S.reduction;
    a.overflow = P.overflow;
    if (!serial) test_op_body(a, gtid, T);
    else if (gtid == 0) test_op_body(a, 0, 1);  // the <<<1,1>>> launch of the host path
    grid.sync();
    const uint32_t nretry = ld_vol_u32(P.cnt + br);
    if (gtid == 0) {
      P.stats[0] += 1;      // launches
      P.stats[1] += nin;    // popped
      if (serial) P.stats[4] += 1;
      const int64_t k = P.stats[6];
      if (k < P.trace_cap) {  // [launch, |in|, |out|, |retry|] after the launch (oracle's trace)
        P.trace[4 * k + 0] = P.stats[0];
        P.trace[4 * k + 1] = nin;
        P.trace[4 * k + 2] = ld_vol_u32(P.cnt + bo);
        P.trace[4 * k + 3] = nretry;
      }
      P.stats[6] = k + 1;
    }
    if (nretry == 0) break;
    const int t = bi;  // in <- retry; the old in buffer becomes the (cleared) retry
    bi = br;
    br = t;
    grid.sync();  // every thread has read the counters above before they are reset
    if (gtid == 0) {
      P.cnt[br] = 0;
      P.stats[3] += nretry;  // retries
    }
    grid.sync();
    ++retry_rounds;
  }
  const uint32_t nout = ld_vol_u32(P.cnt + bo);
  const uint32_t r = ld_vol_u32(P.red);
  grid.sync();
  const int t = bi;  // swap in <-> out, clear the new out
  bi = bo;
  bo = t;
  if (gtid == 0) {
    P.cnt[bo] = 0;
    P.stats[2] += nout;  // pushes
  }
  grid.sync();
  return S.reduction == IRGL_RED_NONE ? -1 : (int)r;
}

__global__ void pipe_control_kernel(PipeProgDev P) {
  cg::grid_group grid = cg::this_grid();
  const uint32_t gtid = blockIdx.x * blockDim.x + threadIdx.x;
  int bi = P.state[0], bo = P.state[1], br = P.state[2];
  int32_t launch_no = P.state[3];
  int prev = -1;
  int64_t rounds = 0;
  for (;;) {
    if (!P.once && ld_vol_u32(P.cnt + bi) == 0) break;  // looping Pipe: until in is empty
    for (int k = 0; k < P.n; ++k) {
      const PipeStageDev& S = P.st[k];
      if (S.when == IRGL_WHEN_PREV_TRUE && prev != 1) continue;   // dynamic piping (Listing 4)
      if (S.when == IRGL_WHEN_PREV_FALSE && prev != 0) continue;
      for (int64_t it = 0;; ++it) {
        if (S.kind == IRGL_STAGE_ITERATE) {  // Iterate: stop on empty in [Or rounds >= max]
          const bool empty = ld_vol_u32(P.cnt + bi) == 0;
          const bool extra = S.max_rounds > 0 && it >= S.max_rounds;
          if (empty || extra) break;
        }
        prev = pipe_invoke(grid, P, S, bi, bo, br, launch_no);
        if (gtid == 0) P.reds[k] = prev;
        if (S.kind == IRGL_STAGE_INVOKE) break;
        if (S.cond_mode == IRGL_COND_WHILE && prev == 0) break;
        if (S.cond_mode == IRGL_COND_UNTIL && prev == 1) break;
      }
    }
    ++rounds;
    if (P.once || (P.max_rounds > 0 && rounds >= P.max_rounds)) break;
  }
  if (gtid == 0) {
    P.state[0] = bi;
    P.state[1] = bo;
    P.state[2] = br;
    P.state[3] = launch_no;
    P.stats[5] = rounds;
    P.stats[7] = prev;
  }
}

__global__ void fill_i32_kernel(int32_t* p, int32_t v, int64_t n) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    p[i] = v;
}
__global__ void scatter_zero_kernel(int32_t* lab, const uint32_t* items, uint32_t n, uint32_t* vis) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t v = items[i];
    lab[v] = 0;
    if (vis) atomicOr(vis + (v >> 5), 1u << (v & 31));  // BFS visited bitmap
  }
}
__global__ void iota_kernel(uint32_t* p, uint32_t begin, uint32_t n) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    p[i] = begin + i;
}
__global__ void set_red_kernel(Ctl* ctl, int slot, uint32_t v) { ctl->red[slot] = v; }
}  // namespace

cudaError_t launch_test_op(const TestArgs& a, int threads, cudaStream_t st) {
  // T = grid*bs threads; T == threads whenever threads <= 256 or a multiple of 256
  const int bs = threads <= 256 ? (threads > 0 ? threads : 1) : 256;
  const int grid = (threads + bs - 1) / bs;
  note_launch();
  test_op_kernel<<<grid, bs, 0, st>>>(a);
  return cudaGetLastError();
}

int pipe_control_blocks_per_sm(int block) {
  int nb = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, pipe_control_kernel, block, 0);
  return nb;
}
cudaError_t launch_pipe_control(const PipeProgDev& prog, int grid, int block, cudaStream_t st) {
  PipeProgDev p = prog;
  void* args[] = {&p};
  note_launch();
  return cudaLaunchCooperativeKernel((void*)pipe_control_kernel, grid, block, args, 0, st);
}

cudaError_t launch_fill_i32(int32_t* p, int32_t v, int64_t n, cudaStream_t st) {
  if (n <= 0) return cudaSuccess;
  note_launch();
  fill_i32_kernel<<<(int)std::min<int64_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(p, v, n);
  return cudaGetLastError();
}
cudaError_t launch_scatter_zero(int32_t* lab, const uint32_t* items, uint32_t n, cudaStream_t st,
                                uint32_t* vis) {
  if (n == 0) return cudaSuccess;
  note_launch();
  scatter_zero_kernel<<<(int)std::min<uint32_t>((n + 255) / 256, 1024), 256, 0, st>>>(lab, items, n, vis);
  return cudaGetLastError();
}
cudaError_t launch_iota_u32(uint32_t* p, uint32_t begin, uint32_t n, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  note_launch();
  iota_kernel<<<(int)std::min<uint32_t>((n + 255) / 256, 148 * 16), 256, 0, st>>>(p, begin, n);
  return cudaGetLastError();
}
cudaError_t launch_set_red(Ctl* ctl, int slot, uint32_t v, cudaStream_t st) {
  note_launch();
  set_red_kernel<<<1, 1, 0, st>>>(ctl, slot, v);
  return cudaGetLastError();
}

}  // namespace irgl
