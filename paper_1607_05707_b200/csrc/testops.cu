// testops.cu — the tiny operators the reference's own examples are phrased in (SPEC.md:439,
// :448-449, :465-466, :553-554, :557), run through the SAME pipe/worklist/orchestration machinery
// as the graph operators, plus small utility kernels.
#include "kernels.h"

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
// the global thread id; blocked = contiguous ceil(N/T) chunk per thread.
__global__ void test_op_kernel(TestArgs a) {
  const uint32_t T = gridDim.x * blockDim.x;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
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
  // per-thread partial aggregation, then one idempotent store per warp (E4)
  if (a.reduction == IRGL_RED_ANY) {
    if (__any_sync(FULL, any) && lane_id() == 0) *(volatile uint32_t*)a.red = 1u;
  } else if (a.reduction == IRGL_RED_ALL) {
    if (!__all_sync(FULL, all) && lane_id() == 0) *(volatile uint32_t*)a.red = 0u;
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
