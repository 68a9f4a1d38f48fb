// sync_probe.cu — cost of one grid-wide barrier on B200: cooperative_groups grid.sync() vs a
// hand-written sense-reversing barrier (one arrival atomic per CTA, acquire polling), for
// several co-resident grid sizes.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void cg_sync_loop(int iters, int* sink) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = iters;
}

__device__ __forceinline__ unsigned ld_acquire(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// counter[0] = arrivals, counter[1] = generation
__global__ void my_sync_loop(int iters, unsigned* bar, int* sink) {
  unsigned gen = 0;
  for (int i = 0; i < iters; ++i) {
    __syncthreads();
    if (threadIdx.x == 0) {
      gen = ld_acquire(bar + 1);
      __threadfence();
      const unsigned arrived = atomicAdd(bar, 1u);
      if (arrived == gridDim.x - 1) {
        atomicExch(bar, 0u);
        __threadfence();
        atomicAdd(bar + 1, 1u);
      } else {
        while (ld_acquire(bar + 1) == gen) { }
      }
    }
    __syncthreads();
  }
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = iters;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int* sink; unsigned* bar; cudaMalloc(&sink, 4); cudaMalloc(&bar, 8); cudaMemset(bar, 0, 8);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int iters = 20000;
  for (int bs : {256, 512, 1024}) {
    for (int per : {1, 2, 4}) {
      if (bs * per > 2048) continue;
      int grid = sms * per;
      void* args[] = {(void*)&iters, (void*)&sink};
      cudaLaunchCooperativeKernel((void*)cg_sync_loop, grid, bs, args, 0, 0);
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)cg_sync_loop, grid, bs, args, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      void* args2[] = {(void*)&iters, (void*)&bar, (void*)&sink};
      cudaEventRecord(a);
      cudaLaunchCooperativeKernel((void*)my_sync_loop, grid, bs, args2, 0, 0);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms2; cudaEventElapsedTime(&ms2, a, b);
      printf("block %4d x %d/SM (grid %4d): cg grid.sync %.2f us   custom barrier %.2f us  (%s)\n", bs, per, grid,
             ms * 1e3 / iters, ms2 * 1e3 / iters, cudaGetErrorString(cudaGetLastError()));
    }
  }
}
