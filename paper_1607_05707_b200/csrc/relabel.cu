// relabel.cu — degree-ordered vertex relabelling of a one-partition CSR (data layout in HBM).
//
// Hubs get the smallest ids, so the per-vertex state the traversals gather most often (levels,
// distances, labels, PageRank contributions) is packed into few cache lines that stay L2/L1
// resident: on RMAT-24, BFS 1.30x and SSSP 1.44x faster (profiles/r1s2_relabel.txt); on RMAT-22,
// whose state is L2-resident either way, 2-4%.  The permutation never leaves the runtime: worklist
// items, results and worklist reads keep the caller's vertex ids (api.cu maps them).
//
//   new id i  <- old vertex inv[i], vertices ordered by (degree descending, old id ascending)
//   perm[old] =  new id
//   edges     =  (perm[u], perm[v]) sorted (rows sorted by new neighbour id, as every CSR here)
#include <cub/cub.cuh>

#include "kernels.h"

namespace irgl {
namespace {

__global__ void deg_key_kernel(const int64_t* rp, int64_t n, int64_t maxdeg, uint32_t* key,
                               int32_t* id) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x) {
    key[v] = (uint32_t)(maxdeg - (rp[v + 1] - rp[v]));  // ascending key = descending degree
    id[v] = (int32_t)v;
  }
}

// inv_rel[i] = old local index of new local index i -> perm[old local] = lo + i, inv[i] = lo + old
__global__ void perm_range_kernel(const int32_t* inv_rel, int64_t nloc, int64_t lo, int32_t* perm,
                                  int32_t* inv) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nloc; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t old = inv_rel[i];
    perm[old] = (int32_t)(lo + i);
    inv[i] = (int32_t)(lo + old);
  }
}

__global__ void deg_new_kernel(const int32_t* inv, int64_t nloc, int64_t lo, const int64_t* rp_old,
                               int64_t* deg_new) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nloc; i += (int64_t)gridDim.x * blockDim.x) {
    const int64_t old = inv[i] - lo;
    deg_new[i] = rp_old[old + 1] - rp_old[old];
  }
}

// warp per old local row u: key = (perm_local[u] - lo) << 32 | perm_global[v]
__global__ void edge_key_kernel(const int64_t* rp, const int32_t* col, const int32_t* perm_local, int64_t lo,
                                const int32_t* perm_global, int64_t nloc, uint64_t* key) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t u = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; u < nloc; u += nw) {
    const uint64_t hi = (uint64_t)(uint32_t)(perm_local[u] - lo) << 32;
    for (int64_t k = rp[u] + lane; k < rp[u + 1]; k += 32) key[k] = hi | (uint32_t)perm_global[col[k]];
  }
}

// out[i] = src[perm[lo + i]] for i < nloc (a partition's results in the caller's ids)
__global__ void gather_range_kernel(int32_t* out, const int32_t* src, const int32_t* perm, int64_t lo,
                                    int64_t nloc) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nloc; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = src[perm[lo + i]];
}

__global__ void low_word_kernel(const uint64_t* key, int64_t m, int32_t* col) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x)
    col[k] = (int32_t)(uint32_t)key[k];
}

__global__ void map_items_kernel(uint32_t* items, uint32_t n, const int32_t* table) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
    items[i] = (uint32_t)table[items[i]];
}

template <class T>
__global__ void gather_kernel(T* out, const T* src, const int32_t* perm, int64_t n) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    out[v] = src[perm[v]];
}

__global__ void cmin_kernel(const int32_t* lab, const int32_t* inv, int64_t n, int32_t* cmin) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    atomicMin(cmin + lab[i], inv[i]);
}

__global__ void cc_out_kernel(int32_t* out, const int32_t* lab, const int32_t* perm, const int32_t* cmin,
                              int64_t n) {
  for (int64_t v = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; v < n; v += (int64_t)gridDim.x * blockDim.x)
    out[v] = cmin[lab[perm[v]]];
}

__global__ void weights_u8_kernel(const int32_t* w, int64_t m, uint8_t* w8, uint32_t* bad) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < m; k += (int64_t)gridDim.x * blockDim.x) {
    const int32_t x = w[k];
    if (x < 0 || x > 255) *bad = 1u;
    w8[k] = (uint8_t)x;
  }
}

inline int grid_for(int64_t n) { return (int)std::max<int64_t>(1, std::min<int64_t>((n + 255) / 256, 148 * 16)); }

}  // namespace

#define RL_CK(x)                         \
  do {                                   \
    cudaError_t _e = (x);                \
    if (_e != cudaSuccess) return _e;    \
  } while (0)

// Phase 1 for the partition of rows [lo, lo + nloc): its vertices ordered by (degree descending,
// old id ascending) inside their own id range — perm_local[v - lo] = new id (global, in the same
// range), inv_local[i] = old id of new id lo + i.  One partition: lo = 0, nloc = n.
cudaError_t relabel_order(int64_t nloc, int64_t lo, int64_t maxdeg, const int64_t* rp_old,
                          int32_t** perm_local, int32_t** inv_local, cudaStream_t st) {
  const int64_t n = std::max<int64_t>(nloc, 1);
  uint32_t *ka = nullptr, *kb = nullptr;
  int32_t *ia = nullptr, *ib = nullptr;
  RL_CK(cudaMallocAsync(&ka, n * 4, st));
  RL_CK(cudaMallocAsync(&kb, n * 4, st));
  RL_CK(cudaMallocAsync(&ia, n * 4, st));
  RL_CK(cudaMallocAsync(&ib, n * 4, st));
  note_launch();
  deg_key_kernel<<<grid_for(nloc), 256, 0, st>>>(rp_old, nloc, maxdeg, ka, ia);
  int bits = 1;
  while (bits < 32 && (1ull << bits) <= (uint64_t)maxdeg) ++bits;
  cub::DoubleBuffer<uint32_t> dk(ka, kb);
  cub::DoubleBuffer<int32_t> dv(ia, ib);
  size_t tmp = 0;
  RL_CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, dk, dv, nloc, 0, bits, st));
  void* t = nullptr;
  RL_CK(cudaMallocAsync(&t, tmp, st));
  RL_CK(cub::DeviceRadixSort::SortPairs(t, tmp, dk, dv, nloc, 0, bits, st));
  cudaFreeAsync(t, st);
  cudaFreeAsync(ka, st);
  cudaFreeAsync(kb, st);
  int32_t* inv_rel = dv.Current();  // local old index of new local index i
  int32_t *perm = nullptr, *inv = nullptr;
  RL_CK(cudaMalloc(&perm, n * 4));
  RL_CK(cudaMalloc(&inv, n * 4));
  note_launch();
  perm_range_kernel<<<grid_for(nloc), 256, 0, st>>>(inv_rel, nloc, lo, perm, inv);
  cudaFreeAsync(dv.Current(), st);
  cudaFreeAsync(dv.Alternate(), st);
  *perm_local = perm;
  *inv_local = inv;
  return cudaStreamSynchronize(st);
}

// Phase 2: the partition's CSR in the new numbering — row i (new local index) is old row
// inv_local[i] - lo, columns mapped through perm_global[n] (every partition's new ids), each row
// sorted by new neighbour id; weights ride along.  The old col / w are released.
cudaError_t relabel_rewrite(int64_t nloc, int64_t lo, int64_t n, int64_t m, const int64_t* rp_old,
                            const int32_t* perm_local, const int32_t* inv_local,
                            const int32_t* perm_global, int32_t** col_io, int32_t** w_io,
                            int64_t** rp_new, cudaStream_t st) {
  int64_t* deg_new = nullptr;
  int64_t* rp = nullptr;
  void* t = nullptr;
  size_t tmp = 0;
  RL_CK(cudaMallocAsync(&deg_new, (nloc + 1) * 8, st));
  RL_CK(cudaMalloc(&rp, (nloc + 1) * 8));
  note_launch();
  deg_new_kernel<<<grid_for(nloc), 256, 0, st>>>(inv_local, nloc, lo, rp_old, deg_new);
  RL_CK(cudaMemsetAsync(deg_new + nloc, 0, 8, st));
  RL_CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, deg_new, rp, nloc + 1, st));
  RL_CK(cudaMallocAsync(&t, tmp, st));
  RL_CK(cub::DeviceScan::ExclusiveSum(t, tmp, deg_new, rp, nloc + 1, st));
  cudaFreeAsync(t, st);
  cudaFreeAsync(deg_new, st);
  uint64_t *ea = nullptr, *eb = nullptr;
  RL_CK(cudaMallocAsync(&ea, std::max<int64_t>(m, 1) * 8, st));
  note_launch();
  edge_key_kernel<<<148 * 16, 256, 0, st>>>(rp_old, *col_io, perm_local, lo, perm_global, nloc, ea);
  RL_CK(cudaStreamSynchronize(st));
  cudaFree(*col_io);  // allocated with cudaMalloc or cudaMallocAsync: cudaFree handles both
  *col_io = nullptr;
  RL_CK(cudaMallocAsync(&eb, std::max<int64_t>(m, 1) * 8, st));
  int ebits = 1;
  while (ebits < 32 && (1ull << ebits) < (uint64_t)n) ++ebits;
  int hbits = 1;
  while (hbits < 31 && (1ull << hbits) < (uint64_t)nloc) ++hbits;
  cub::DoubleBuffer<uint64_t> de(ea, eb);
  int32_t* wa = *w_io;
  int32_t* wb = nullptr;
  tmp = 0;
  if (wa) {
    RL_CK(cudaMallocAsync(&wb, std::max<int64_t>(m, 1) * 4 + 16, st));
    cub::DoubleBuffer<int32_t> dw(wa, wb);
    RL_CK(cub::DeviceRadixSort::SortPairs(nullptr, tmp, de, dw, m, 0, 32 + hbits, st));
    RL_CK(cudaMallocAsync(&t, tmp, st));
    RL_CK(cub::DeviceRadixSort::SortPairs(t, tmp, de, dw, m, 0, 32 + hbits, st));
    cudaFreeAsync(t, st);
    // keep the sorted weights in a cudaMalloc'd (+4 padded) array like every CSR array
    int32_t* w = nullptr;
    RL_CK(cudaMalloc(&w, (m + 4) * 4));
    RL_CK(cudaMemcpyAsync(w, dw.Current(), m * 4, cudaMemcpyDeviceToDevice, st));
    RL_CK(cudaStreamSynchronize(st));
    cudaFree(wa);
    cudaFree(wb);
    *w_io = w;
  } else {
    RL_CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, de, m, 0, 32 + hbits, st));
    RL_CK(cudaMallocAsync(&t, tmp, st));
    RL_CK(cub::DeviceRadixSort::SortKeys(t, tmp, de, m, 0, 32 + hbits, st));
    cudaFreeAsync(t, st);
  }
  (void)ebits;
  int32_t* col = nullptr;
  RL_CK(cudaMalloc(&col, (m + 4) * 4));
  note_launch();
  low_word_kernel<<<grid_for(m), 256, 0, st>>>(de.Current(), m, col);
  cudaFreeAsync(ea, st);
  cudaFreeAsync(eb, st);
  *col_io = col;
  *rp_new = rp;
  return cudaStreamSynchronize(st);
}

cudaError_t relabel_degree(int64_t n, int64_t m, int64_t maxdeg, const int64_t* rp_old, int32_t** col_io,
                           int32_t** w_io, int64_t** rp_new, int32_t** perm_out, int32_t** inv_out,
                           cudaStream_t st) {
  RL_CK(relabel_order(n, 0, maxdeg, rp_old, perm_out, inv_out, st));
  return relabel_rewrite(n, 0, n, m, rp_old, *perm_out, *inv_out, *perm_out, col_io, w_io, rp_new, st);
}

cudaError_t launch_weights_u8(const int32_t* w, int64_t m, uint8_t* w8, uint32_t* bad, cudaStream_t st) {
  if (m == 0) return cudaSuccess;
  note_launch();
  weights_u8_kernel<<<grid_for(m), 256, 0, st>>>(w, m, w8, bad);
  return cudaGetLastError();
}

cudaError_t launch_map_items(uint32_t* items, uint32_t n, const int32_t* table, cudaStream_t st) {
  if (n == 0) return cudaSuccess;
  note_launch();
  map_items_kernel<<<grid_for(n), 256, 0, st>>>(items, n, table);
  return cudaGetLastError();
}

cudaError_t launch_gather_i32(int32_t* out, const int32_t* src, const int32_t* perm, int64_t n, cudaStream_t st) {
  note_launch();
  gather_kernel<int32_t><<<grid_for(n), 256, 0, st>>>(out, src, perm, n);
  return cudaGetLastError();
}

cudaError_t launch_gather_range_i32(int32_t* out, const int32_t* src, const int32_t* perm, int64_t lo,
                                   int64_t nloc, cudaStream_t st) {
  if (nloc <= 0) return cudaSuccess;
  note_launch();
  gather_range_kernel<<<grid_for(nloc), 256, 0, st>>>(out, src, perm, lo, nloc);
  return cudaGetLastError();
}

cudaError_t launch_gather_f64(double* out, const double* src, const int32_t* perm, int64_t n, cudaStream_t st) {
  note_launch();
  gather_kernel<double><<<grid_for(n), 256, 0, st>>>(out, src, perm, n);
  return cudaGetLastError();
}

cudaError_t launch_cc_labels_original(int32_t* out, const int32_t* lab, const int32_t* perm, const int32_t* inv,
                                      int32_t* cmin, int64_t n, cudaStream_t st) {
  RL_CK(cudaMemsetAsync(cmin, 0x7f, n * 4, st));  // 0x7f7f7f7f > every id
  note_launch();
  cmin_kernel<<<grid_for(n), 256, 0, st>>>(lab, inv, n, cmin);
  note_launch();
  cc_out_kernel<<<grid_for(n), 256, 0, st>>>(out, lab, perm, cmin, n);
  return cudaGetLastError();
}

}  // namespace irgl
