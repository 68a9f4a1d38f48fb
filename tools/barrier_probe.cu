// barrier_probe.cu — cost of one grid-wide barrier of a co-resident persistent grid on B200
// (148 SMs x 4 CTAs x 256 threads, the SSSP kernel's shape), for the barrier variants the
// outlined kernels could use:
//   bcast : the runtime's grid_sync_bcast — fence + atomicAdd arrival, the last arriver reads a
//           payload counter and publishes it with a release store, the others spin (acquire)
//   count : arrival with atom.add.release; every CTA polls the arrival counter (acquire) until
//           it reaches the barrier's target, then reads the payload itself
//   cg    : cooperative_groups grid.sync() followed by a per-CTA payload read
// Each iteration also does one atomicAdd of "work" per CTA before the barrier (the round's
// counters) so the payload read is a real dependency.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o barrier_probe tools/barrier_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_acq64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_vol(const unsigned* p) {
  unsigned v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}
__device__ __forceinline__ unsigned atom_add_release(unsigned* p, unsigned v) {
  unsigned r;
  asm volatile("atom.add.release.gpu.global.u32 %0, [%1], %2;" : "=r"(r) : "l"(p), "r"(v) : "memory");
  return r;
}
__device__ __forceinline__ void red_add_release(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

struct Bar {
  alignas(256) unsigned arrive;
  alignas(256) unsigned long long release;
  alignas(256) unsigned work[4];
};

__global__ void __launch_bounds__(256, 4) k_bcast(int iters, Bar* b, unsigned* sink) {
  __shared__ unsigned long long slot;
  unsigned acc = 0;
  for (int i = 1; i <= iters; ++i) {
    if (threadIdx.x == 0) atomicAdd(&b->work[i & 3], 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned long long tag = (unsigned long long)(i & 0xff) << 56;
      __threadfence();
      const unsigned old = atomicAdd(&b->arrive, 1u);
      unsigned long long w;
      if (old == (unsigned)i * gridDim.x - 1u) {
        __threadfence();
        w = tag | ld_vol(&b->work[i & 3]);
        asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(&b->release), "l"(w) : "memory");
      } else {
        do { w = ld_acq64(&b->release); } while ((w & (0xffull << 56)) != tag);
      }
      slot = w;
    }
    __syncthreads();
    acc += (unsigned)slot;
  }
  if (threadIdx.x == 0) atomicAdd(sink, acc);
}

template <bool kRed>
__global__ void __launch_bounds__(256, 4) k_count(int iters, Bar* b, unsigned* sink) {
  __shared__ unsigned slot;
  unsigned acc = 0;
  for (int i = 1; i <= iters; ++i) {
    if (threadIdx.x == 0) atomicAdd(&b->work[i & 3], 1u);
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned target = (unsigned)i * gridDim.x;
      if (kRed) red_add_release(&b->arrive, 1u);
      else atom_add_release(&b->arrive, 1u);
      while ((int)(ld_acq(&b->arrive) - target) < 0) {}
      slot = ld_vol(&b->work[i & 3]);
    }
    __syncthreads();
    acc += slot;
  }
  if (threadIdx.x == 0) atomicAdd(sink, acc);
}

__global__ void __launch_bounds__(256, 4) k_cg(int iters, Bar* b, unsigned* sink) {
  cg::grid_group g = cg::this_grid();
  __shared__ unsigned slot;
  unsigned acc = 0;
  for (int i = 1; i <= iters; ++i) {
    if (threadIdx.x == 0) atomicAdd(&b->work[i & 3], 1u);
    g.sync();
    if (threadIdx.x == 0) slot = ld_vol(&b->work[i & 3]);
    __syncthreads();
    acc += slot;
  }
  if (threadIdx.x == 0) atomicAdd(sink, acc);
}

template <class K>
static float run(K k, int grid, int iters, Bar* b, unsigned* sink) {
  cudaMemset(b, 0, sizeof(Bar));
  void* args[] = {&iters, &b, &sink};
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaLaunchCooperativeKernel((void*)k, grid, 256, args, 0, 0);  // warm
  cudaDeviceSynchronize();
  cudaMemset(b, 0, sizeof(Bar));
  cudaEventRecord(e0);
  cudaLaunchCooperativeKernel((void*)k, grid, 256, args, 0, 0);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  return ms * 1000.f / iters;
}

int main() {
  Bar* b;
  unsigned* sink;
  cudaMalloc(&b, sizeof(Bar));
  cudaMalloc(&sink, 4);
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  for (int per : {1, 2, 4}) {
    const int grid = sms * per;
    printf("grid %4d CTAs: bcast %.2f us  count(atom.release) %.2f us  count(red.release) %.2f us  cg %.2f us\n",
           grid, run(k_bcast, grid, iters, b, sink), run(k_count<false>, grid, iters, b, sink),
           run(k_count<true>, grid, iters, b, sink), run(k_cg, grid, iters, b, sink));
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
