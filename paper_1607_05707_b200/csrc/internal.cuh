// internal.cuh — shared host/device definitions of the B200 IrGL runtime (libirgl_rt.so).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdio>
#include <string>
#include <vector>

#include "irgl/rt.h"

namespace irgl {

// Fixed(256): the nested-parallelism / cooperative-conversion kernels use shared memory sized by
// the block, so their block constraint is Fixed.
// 512 threads: 2 (SSSP, 64 registers) or 3 (BFS / CC, 40 registers) CTAs per SM; against 256 it
// halves the CTAs that arrive at every grid barrier and, with the smaller per-warp push staging
// (expand.cu kWBuf), leaves more of the SM's 256 KB to L1 for the label gathers: SSSP RMAT-22
// 1.227 -> 1.134 ms, RMAT-24 3.69 -> 3.64, BFS within 1% (profiles/r2_ab_blocks.txt).
#ifndef IRGL_BLOCK
#define IRGL_BLOCK 512
#endif
constexpr int kBlock = IRGL_BLOCK;  // threads per CTA of the hot kernels (tuning: IRGL_BLOCK)
// minimum co-resident CTAs for __launch_bounds__, from a thread budget per SM
constexpr int minb_for_threads(int threads_per_sm) {
  return threads_per_sm / kBlock > 0 ? threads_per_sm / kBlock : 1;
}
constexpr int kWarps = kBlock / 32;
constexpr int32_t kInf = 0x7fffffff;
constexpr int kPushBuf = 2048;  // per-CTA shared-memory push staging (cooperative conversion)

// Edge-chunk descriptor (E1 edge-balanced level): `len` (<= chunk_edges) edges of vertex v
// starting at edge `beg`, with the vertex's label (dist/level/label) as read when it was popped.
struct ChunkDesc {
  uint64_t beg_len;  // beg (48 bits) << 16 | len (16 bits, chunk_edges <= 65535)
  uint32_t v;
  int32_t sv;        // label of v at pop time (a stale, larger value only weakens relaxations;
                     // the improvement that made it stale re-pushes v, SPEC.md:425 epochs)
};
static_assert(sizeof(ChunkDesc) == 16, "one 128-bit load per descriptor");

// Device-resident control block of one pipe partition.  Counter slots are addressed by index so
// the persistent kernel can rotate them (see persistent loop in expand.cu).
// The counters every warp hits during an expansion (out count, chunk reservations, tile fetches,
// edge totals, deferral minimum) each sit on their own 256-byte line, so their atomics spread
// over different L2 slices instead of queueing at one.
struct Ctl {
  alignas(256) uint32_t cnt[4];        // worklist counters: in / out / retry / spare (slots named by the host)
  alignas(256) uint32_t chunk_cnt[3];  // edge-chunk list counters, rotated by round
  alignas(256) uint32_t red[3];        // ReduceAndReturn cells, rotated by round
  uint32_t overflow;      // push beyond capacity (IRGL_E_WL_OVERFLOW)
  uint32_t pad;
  alignas(256) unsigned long long edges;    // directed edges scanned
  alignas(256) unsigned long long popped;   // items popped (persistent mode)
  unsigned long long pushes;   // items pushed (persistent mode)
  unsigned long long remote;   // remote updates emitted
  unsigned long long rounds;   // persistent: rounds executed
  int32_t last_red;            // persistent: last round's reduced value
  int32_t exit_in_slot;        // persistent: buffer parity at exit
  unsigned long long tc_count; // TC: Sum reduction (extension)
  alignas(256) uint32_t tile_ctr[3];        // dynamic warp-tile counters, rotated by round
  uint32_t far_cnt[2];         // SSSP near-far pile counters (double-buffered)
  uint32_t minkeep[2];         // min dist kept in the far pile by a split (double-buffered: the
                               // persistent kernel resets one slot while CTAs may still read the other)
  uint32_t stamp_used;         // persistent: stamp ids consumed (rounds + splits)
  int32_t stamp_base;          // graph part: last stamp id used (pipelined batches, PersistArgs)
  uint32_t far_sel;            // persistent: current far pile at exit
  uint32_t bu_rounds;          // direction-optimising BFS: bottom-up rounds executed
  alignas(256) unsigned long long mf[3];    // DO-BFS: edges of the next frontier (rotated by round)
  unsigned long long bu_found[3];  // DO-BFS: vertices discovered by a bottom-up round
  unsigned long long bu_scanned;   // DO-BFS: edges examined by bottom-up rounds
  unsigned long long mst_w, mst_e; // MST: forest weight / edges
  uint32_t mst_cnt[2];             // MST: internal worklist counters
  alignas(256) uint32_t dmin[3];                // SSSP deferral: min distance pushed into each round's out
                                   // worklist (0xffffffff = unknown), rotated by round
  // grid barrier of the persistent kernels (grid_sync_bcast): monotonic arrival counter and the
  // release word {barrier tag, payload}, on separate L2 lines; zeroed before every launch
  alignas(256) unsigned int gb_arrive;
  alignas(256) unsigned long long gb_release;
  // distributed persistent kernel: the leader's rendezvous outcome, broadcast to the CTAs through
  // a grid barrier {ok, every partition's out count summed, every partition's flags OR-ed}
  alignas(256) uint32_t x_word[4];
  unsigned long long x_mf;  // DO-BFS: every partition's next-frontier edge count summed
};

// ---------------------------------------------------------------------------------------------
// Device helpers.
__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }
__device__ __forceinline__ uint32_t lanemask_lt() {
  uint32_t m;
  asm("mov.u32 %0, %%lanemask_lt;" : "=r"(m));
  return m;
}

// 128-bit streaming load of CSR column / weight data: read-only for the kernel's lifetime, so
// the non-coherent path with L1 no-allocate (stream, do not pollute L1 with col data).
__device__ __forceinline__ int4 ld_stream_v4(const int32_t* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ int32_t ld_stream(const int32_t* p) {
  int32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
// L2-coherent read (never an L1 line that predates a grid barrier): used where a stale value is
// NOT benign — the popped vertex's own distance and the near-far split's drop test.
__device__ __forceinline__ int32_t ld_label_cg(const int32_t* p) {
  int32_t r;
  asm volatile("ld.global.cg.s32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
// Label/distance gathers: coherent global loads.  A stale (larger / INF) value is benign for
// every operator here: it only causes an atomic that then returns the true value.
__device__ __forceinline__ int32_t ld_label(const int32_t* p) {
  int32_t r;
  asm volatile("ld.global.s32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}

__device__ __forceinline__ unsigned long long ld_acquire_u64(const unsigned long long* p) {
  unsigned long long r;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(r) : "l"(p) : "memory");
  return r;
}
__device__ __forceinline__ void st_release_u64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

}  // namespace irgl

// ---------------------------------------------------------------------------------------------
// Host-side error plumbing: every API call returns a status; the message goes to the ctx
// (or a global slot) as "RULE: message" (reference diag.hpp:20-27 convention).
namespace irgl {
void set_error(irgl_ctx* ctx, irgl_status_t st, const char* rule, const std::string& msg);
// every kernel launch site calls this (irgl_launch_count evidence for the bench)
void note_launch(int n = 1);
irgl_status_t cuda_status(irgl_ctx* ctx, cudaError_t e, const char* where);
}  // namespace irgl

#define IRGL_CUDA(ctx, expr)                                              \
  do {                                                                    \
    cudaError_t _e = (expr);                                              \
    if (_e != cudaSuccess) return ::irgl::cuda_status((ctx), _e, #expr);  \
  } while (0)
