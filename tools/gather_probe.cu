// gather_probe.cu — measures random 4-byte gather throughput on B200 from label arrays of
// different sizes (L2-resident vs not) with different load flavours: the ceiling for the
// per-edge label[dst] access of BFS/SSSP.  Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ int ld_ca(const int* p) { int r; asm volatile("ld.global.ca.s32 %0,[%1];" : "=r"(r) : "l"(p)); return r; }
__device__ __forceinline__ int ld_cg(const int* p) { int r; asm volatile("ld.global.cg.s32 %0,[%1];" : "=r"(r) : "l"(p)); return r; }
__device__ __forceinline__ int ld_nc(const int* p) { int r; asm volatile("ld.global.nc.s32 %0,[%1];" : "=r"(r) : "l"(p)); return r; }

template <int MODE>
__global__ void gather(const int* __restrict__ a, const int4* __restrict__ idx, int64_t nq, int* out) {
  int acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq; i += (int64_t)gridDim.x * blockDim.x) {
    int4 q = idx[i];
    int v0, v1, v2, v3;
    if (MODE == 0) { v0 = ld_ca(a + q.x); v1 = ld_ca(a + q.y); v2 = ld_ca(a + q.z); v3 = ld_ca(a + q.w); }
    else if (MODE == 1) { v0 = ld_cg(a + q.x); v1 = ld_cg(a + q.y); v2 = ld_cg(a + q.z); v3 = ld_cg(a + q.w); }
    else { v0 = ld_nc(a + q.x); v1 = ld_nc(a + q.y); v2 = ld_nc(a + q.z); v3 = ld_nc(a + q.w); }
    acc += v0 ^ v1 ^ v2 ^ v3;
  }
  if (acc == 0x12345678) out[0] = acc;
}
// atomicMin throughput on random addresses (SSSP relax) and CAS
__global__ void amin(int* a, const int4* __restrict__ idx, int64_t nq) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq; i += (int64_t)gridDim.x * blockDim.x) {
    int4 q = idx[i];
    atomicMin(a + q.x, (int)i); atomicMin(a + q.y, (int)i); atomicMin(a + q.z, (int)i); atomicMin(a + q.w, (int)i);
  }
}
__global__ void copyk(const int4* __restrict__ s, int4* d, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) d[i] = s[i];
}
__global__ void init_idx(int4* idx, int64_t nq, uint32_t mask, uint32_t seed) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < nq; i += (int64_t)gridDim.x * blockDim.x) {
    uint32_t x = (uint32_t)i * 2654435761u ^ seed;
    auto h = [&](uint32_t v) { v ^= v >> 16; v *= 0x7feb352d; v ^= v >> 15; v *= 0x846ca68b; v ^= v >> 16; return v; };
    idx[i] = make_int4(h(x) & mask, h(x + 1) & mask, h(x + 2) & mask, h(x + 3) & mask);
  }
}
int main() {
  const int64_t nq = 1 << 26;  // 4*64M = 256M gathers
  int4* idx; int* out; cudaMalloc(&idx, nq * 16); cudaMalloc(&out, 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int lg : {22, 24, 26, 28}) {
    int* a; cudaMalloc(&a, (4ll << lg)); cudaMemset(a, 0, 4ll << lg);
    init_idx<<<sms * 8, 256>>>(idx, nq, (1u << lg) - 1, 12345);
    for (int mode = 0; mode < 4; ++mode) {
      for (int blocks : {sms * 8, sms * 16}) {
        float best = 1e9;
        for (int rep = 0; rep < 3; ++rep) {
          cudaEventRecord(e0);
          if (mode == 0) gather<0><<<blocks, 256>>>(a, idx, nq, out);
          if (mode == 1) gather<1><<<blocks, 256>>>(a, idx, nq, out);
          if (mode == 2) gather<2><<<blocks, 256>>>(a, idx, nq, out);
          if (mode == 3) amin<<<blocks, 256>>>(a, idx, nq);
          cudaEventRecord(e1); cudaEventSynchronize(e1);
          float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
        }
        const char* nm[] = {"ld.ca", "ld.cg", "ld.nc", "atomicMin"};
        printf("array %4lld MB  %-9s blocks=%5d : %7.1f G ops/s (+ idx stream %.0f GB/s)\n", (4ll << lg) >> 20, nm[mode], blocks,
               4.0 * nq / best / 1e6, 16.0 * nq / best / 1e6);
      }
    }
    cudaFree(a);
  }
  // copy bandwidth
  int4 *s, *d; int64_t n = (1ll << 30) / 16; cudaMalloc(&s, n * 16); cudaMalloc(&d, n * 16);
  float best = 1e9;
  for (int rep = 0; rep < 5; ++rep) { cudaEventRecord(e0); copyk<<<sms * 8, 256>>>(s, d, n); cudaEventRecord(e1); cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms; }
  printf("copy 1 GiB: %.0f GB/s (read+write)\n", 2.0 * n * 16 / best / 1e6);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
