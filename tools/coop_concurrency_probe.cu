// coop_concurrency_probe.cu — can cooperative launches on different streams of ONE device run at
// the same time (the premise of one persistent kernel per partition when several partitions share
// a GPU, with a device-side rendezvous between them)?  K kernels, each a cooperative grid of
// `per` CTAs of 512 threads, launched on K non-blocking streams; every kernel's leader arrives at
// a shared counter and waits (bounded by a 2 s timeout on %globaltimer) until all K arrived, then
// the kernel runs R rounds of {grid.sync, leader rendezvous, grid.sync}.  Prints per-case status
// and the mean time of one rendezvous round.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o coop_probe tools/coop_concurrency_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <vector>
namespace cg = cooperative_groups;

__device__ __forceinline__ unsigned long long gtime() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
__device__ __forceinline__ unsigned ld_acq_sys(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel_sys(unsigned* p, unsigned v) {
  asm volatile("red.release.sys.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__global__ void __launch_bounds__(512) part_kernel(unsigned* arrive, unsigned* fail, int K, int R,
                                                   unsigned long long* t_out) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned ok;
  unsigned long long t0 = 0;
  for (int r = 0; r <= R; ++r) {
    if (r == 1 && blockIdx.x == 0 && threadIdx.x == 0) t0 = gtime();
    grid.sync();
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      red_rel_sys(arrive, 1u);
      const unsigned target = (unsigned)(r + 1) * K;
      const unsigned long long s = gtime();
      unsigned good = 1;
      while ((int)(ld_acq_sys(arrive) - target) < 0) {
        if (*(volatile unsigned*)fail) { good = 0; break; }
        if (gtime() - s > 2000000000ull) { atomicExch(fail, 1u); good = 0; break; }
        __nanosleep(32);
      }
      *(volatile unsigned*)(fail + 1 + blockIdx.x) = good;  // scratch
    }
    grid.sync();
    if (threadIdx.x == 0) ok = *(volatile unsigned*)fail == 0;
    __syncthreads();
    if (!ok) return;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) *t_out = gtime() - t0;
}

int main() {
  int sms = 0, bps = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, part_kernel, 512, 0);
  printf("sms=%d blocks/SM=%d\n", sms, bps);
  const int R = 1000;
  for (int K : {1, 2, 4}) {
    for (int full : {0, 1}) {
      if (K == 1 && full) continue;
      const int per = full ? sms * bps : sms * bps / K;
      unsigned *arrive, *fail;
      unsigned long long* tout;
      cudaMalloc(&arrive, 4);
      cudaMalloc(&fail, 4 * (1 + 4096));
      cudaMalloc(&tout, 8 * K);
      cudaMemset(arrive, 0, 4);
      cudaMemset(fail, 0, 4 * (1 + 4096));
      cudaMemset(tout, 0, 8 * K);
      cudaDeviceSynchronize();
      std::vector<cudaStream_t> st(K);
      for (auto& s : st) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
      std::vector<cudaError_t> le(K);
      for (int k = 0; k < K; ++k) {
        unsigned long long* tk = tout + k;
        void* args[] = {&arrive, &fail, (void*)&K, (void*)&R, &tk};
        le[k] = cudaLaunchCooperativeKernel((void*)part_kernel, per, 512, args, 0, st[k]);
      }
      cudaError_t e = cudaDeviceSynchronize();
      unsigned hf = 0;
      std::vector<unsigned long long> ht(K);
      cudaMemcpy(&hf, fail, 4, cudaMemcpyDeviceToHost);
      cudaMemcpy(ht.data(), tout, 8 * K, cudaMemcpyDeviceToHost);
      printf("K=%d grid/kernel=%d (%s): launch=%s sync=%s rendezvous=%s", K, per, full ? "full device each" : "1/K of device",
             cudaGetErrorString(le[K - 1]), cudaGetErrorString(e), hf ? "TIMEOUT" : "ok");
      if (!hf) printf(" %.2f us/round (2 grid.sync + cross-kernel rendezvous)", ht[0] * 1e-3 / R);
      printf("\n");
      for (auto& s : st) cudaStreamDestroy(s);
      cudaFree(arrive);
      cudaFree(fail);
      cudaFree(tout);
    }
  }
  return 0;
}
