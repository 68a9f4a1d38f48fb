// gen.cu — device-side synthetic graph ingestion (SURVEY §8 row F2, §8d inputs): Philox-4x32-10
// RMAT (Graph500 A/B/C/D = .57/.19/.19/.05, seeded vertex scramble) and W x H grids, built
// straight into the CSR rows [lo, hi) of one partition: generate directed keys owned by the
// partition -> CUB radix sort -> unique -> degree count -> exclusive scan -> col / weight.
// Same counter-based streams as the host oracle, so host and device graphs are identical
// (checked by tests/test_gpu_graph.py against the oracle CSR).
#include <cub/cub.cuh>

#include "kernels.h"

namespace irgl {
namespace {
constexpr unsigned FULL = 0xffffffffu;
constexpr uint32_t TAG_RMAT = 0x524D4154u, TAG_SCRM = 0x5343524Du, TAG_WGHT = 0x57474854u,
                   TAG_PERC = 0x50455243u;
constexpr uint32_t TH_A = 2448131358u, TH_AB = 3264175144u, TH_ABC = 4080218931u;

__host__ __device__ __forceinline__ void philox(uint32_t c0, uint32_t c1, uint32_t c2, uint32_t c3,
                                                uint32_t k0, uint32_t k1, uint32_t out[4]) {
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    const uint64_t p0 = (uint64_t)0xD2511F53u * c0;
    const uint64_t p1 = (uint64_t)0xCD9E8D57u * c2;
    const uint32_t n0 = (uint32_t)(p1 >> 32) ^ c1 ^ k0;
    const uint32_t n1 = (uint32_t)p1;
    const uint32_t n2 = (uint32_t)(p0 >> 32) ^ c3 ^ k1;
    const uint32_t n3 = (uint32_t)p0;
    c0 = n0; c1 = n1; c2 = n2; c3 = n3;
    k0 += 0x9E3779B9u;
    k1 += 0xBB67AE85u;
  }
  out[0] = c0; out[1] = c1; out[2] = c2; out[3] = c3;
}

struct Scr {
  uint64_t m1, a1, m2, a2, mask;
  int s1, s2;
};
__device__ __forceinline__ uint64_t scramble(uint64_t x, const Scr& s) {
  x = (x * s.m1 + s.a1) & s.mask;
  x ^= x >> s.s1;
  x = (x * s.m2 + s.a2) & s.mask;
  x ^= x >> s.s2;
  return x;
}

__device__ __forceinline__ int32_t hash_weight(uint64_t u, uint64_t v, uint64_t wseed) {
  const uint64_t a = u < v ? u : v, b = u < v ? v : u;
  uint32_t r[4];
  philox((uint32_t)a, (uint32_t)b, (uint32_t)((a >> 32) | ((b >> 32) << 16)), TAG_WGHT,
         (uint32_t)wseed, (uint32_t)(wseed >> 32), r);
  return 1 + (int32_t)(r[0] % 255u);
}

__device__ __forceinline__ void rmat_edge(uint64_t e, int scale, uint64_t seed, const Scr& scr,
                                          uint64_t& u, uint64_t& v) {
  u = 0;
  v = 0;
  for (int b = 0; b * 4 < scale; ++b) {
    uint32_t r[4];
    philox((uint32_t)e, (uint32_t)(e >> 32), (uint32_t)b, TAG_RMAT, (uint32_t)seed,
           (uint32_t)(seed >> 32), r);
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int i = b * 4 + j;
      if (i < scale) {
        const uint32_t x = r[j];
        const int bit = scale - 1 - i;
        const uint64_t ub = x >= TH_AB ? 1u : 0u;
        const uint64_t vb = (x >= TH_A && x < TH_AB) || x >= TH_ABC ? 1u : 0u;
        u |= ub << bit;
        v |= vb << bit;
      }
    }
  }
  u = scramble(u, scr);
  v = scramble(v, scr);
}

// pass 0: count, pass 1: emit keys ((u-lo) << scale) | v for sources u in [lo, hi)
template <bool EMIT>
__global__ void rmat_keys_kernel(uint64_t ne, int scale, uint64_t seed, Scr scr, int64_t lo,
                                 int64_t hi, unsigned long long* counter, uint64_t* keys) {
  const uint32_t lane = lane_id();
  unsigned long long local = 0;
  for (uint64_t e0 = (uint64_t)blockIdx.x * blockDim.x; e0 < ne; e0 += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t e = e0 + threadIdx.x;
    uint64_t u = 0, v = 0;
    bool a = false, b = false;
    if (e < ne) {
      rmat_edge(e, scale, seed, scr, u, v);
      if (u != v) {
        a = (int64_t)u >= lo && (int64_t)u < hi;
        b = (int64_t)v >= lo && (int64_t)v < hi;
      }
    }
    if (!EMIT) {
      local += (unsigned long long)a + (unsigned long long)b;
    } else {
      const uint32_t ma = __ballot_sync(FULL, a), mb = __ballot_sync(FULL, b);
      const uint32_t tot = __popc(ma) + __popc(mb);
      unsigned long long base = 0;
      if (tot) {
        if (lane == 0) base = atomicAdd(counter, (unsigned long long)tot);
        base = __shfl_sync(FULL, base, 0);
      }
      if (a) keys[base + __popc(ma & lanemask_lt())] = ((u - lo) << scale) | v;
      if (b) keys[base + __popc(ma) + __popc(mb & lanemask_lt())] = ((v - lo) << scale) | u;
    }
  }
  if (!EMIT) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(FULL, local, o);
    if (lane == 0 && local) atomicAdd(counter, local);
  }
}

// degree count over sorted unique keys; lanes of one row aggregate with __match_any_sync
__global__ void row_count_kernel(const uint64_t* keys, int64_t m, int scale, int64_t* deg) {
  for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x; i0 < m; i0 += (int64_t)gridDim.x * blockDim.x) {
    const int64_t i = i0 + threadIdx.x;
    const bool ok = i < m;
    const uint64_t r = ok ? (keys[i] >> scale) : ~0ull;
    const uint32_t grp = __match_any_sync(FULL, r);
    if (ok && lane_id() == (uint32_t)(__ffs(grp) - 1))
      atomicAdd((unsigned long long*)(deg + r), (unsigned long long)__popc(grp));
  }
}

__global__ void fill_csr_kernel(const uint64_t* keys, int64_t m, int scale, int64_t lo,
                                uint64_t wseed, int32_t* col, int32_t* w) {
  const uint64_t mask = (1ull << scale) - 1;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t k = keys[i];
    const uint64_t u = (uint64_t)lo + (k >> scale), v = k & mask;
    col[i] = (int32_t)v;
    w[i] = hash_weight(u, v, wseed);
  }
}

// ---- grids: neighbours of (x, y) in sorted id order: NW-diag, N, W, E, S, SE-diag -------------
struct GridSpec {
  int64_t W, H;
  int diag, cut;
  int keep_ppm;
  uint64_t pseed;
};
__device__ __forceinline__ bool grid_keep(const GridSpec& g, int64_t a, int64_t b) {
  if (g.keep_ppm >= 1000000) return true;
  const uint64_t lo = a < b ? a : b, hi = a < b ? b : a;
  uint32_t r[4];
  philox((uint32_t)lo, (uint32_t)hi, 0, TAG_PERC, (uint32_t)g.pseed, (uint32_t)(g.pseed >> 32), r);
  return (int)(r[0] % 1000000u) < g.keep_ppm;
}
__device__ __forceinline__ bool vcut(const GridSpec& g, int64_t y) {  // cut between rows y, y+1
  return g.cut > 0 && (y % g.cut) == g.cut - 1;
}
__device__ __forceinline__ int grid_nbrs(const GridSpec& g, int64_t id, int64_t out[6]) {
  const int64_t x = id % g.W, y = id / g.W;
  int k = 0;
  if (g.diag && x > 0 && y > 0 && !vcut(g, y - 1) && grid_keep(g, id - g.W - 1, id)) out[k++] = id - g.W - 1;
  if (y > 0 && !vcut(g, y - 1) && grid_keep(g, id - g.W, id)) out[k++] = id - g.W;
  if (x > 0 && grid_keep(g, id - 1, id)) out[k++] = id - 1;
  if (x + 1 < g.W && grid_keep(g, id, id + 1)) out[k++] = id + 1;
  if (y + 1 < g.H && !vcut(g, y) && grid_keep(g, id, id + g.W)) out[k++] = id + g.W;
  if (g.diag && x + 1 < g.W && y + 1 < g.H && !vcut(g, y) && grid_keep(g, id, id + g.W + 1))
    out[k++] = id + g.W + 1;
  return k;
}
__global__ void grid_deg_kernel(GridSpec g, int64_t lo, int64_t hi, int64_t* deg) {
  for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t nb[6];
    deg[i - lo] = grid_nbrs(g, i, nb);
  }
}
__global__ void grid_fill_kernel(GridSpec g, int64_t lo, int64_t hi, const int64_t* rp,
                                 uint64_t wseed, int32_t* col, int32_t* w) {
  for (int64_t i = lo + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < hi;
       i += (int64_t)gridDim.x * blockDim.x) {
    int64_t nb[6];
    const int k = grid_nbrs(g, i, nb);
    const int64_t o = rp[i - lo];
    for (int j = 0; j < k; ++j) {
      col[o + j] = (int32_t)nb[j];
      w[o + j] = hash_weight((uint64_t)i, (uint64_t)nb[j], wseed);
    }
  }
}

__global__ void max_deg_kernel(const int64_t* rp, int64_t n, unsigned long long* out) {
  unsigned long long mx = 0;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x)
    mx = max(mx, (unsigned long long)(rp[i + 1] - rp[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = max(mx, __shfl_xor_sync(FULL, mx, o));
  if (lane_id() == 0) atomicMax(out, mx);
}

int bits_for(int64_t x) {
  int b = 0;
  while ((1ll << b) < x) ++b;
  return b;
}

#define GEN_CK(x)                        \
  do {                                   \
    cudaError_t _e = (x);                \
    if (_e != cudaSuccess) {             \
      if (err) *err = #x;                \
      return _e;                         \
    }                                    \
  } while (0)

__global__ void edge_keys_kernel(const EdgeRec* e, int64_t ne, uint64_t* keys, int32_t* w) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < ne;
       i += (int64_t)gridDim.x * blockDim.x) {
    keys[i] = ((uint64_t)e[i].u << 32) | e[i].v;
    w[i] = e[i].w;
  }
}
__global__ void split_keys_kernel(const uint64_t* keys, int64_t m, int32_t* col) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m;
       i += (int64_t)gridDim.x * blockDim.x)
    col[i] = (int32_t)(keys[i] & 0xffffffffull);
}
struct MinOp {
  __device__ __forceinline__ int32_t operator()(int32_t a, int32_t b) const { return a < b ? a : b; }
};
}  // namespace

cudaError_t csr_from_edges_device(const EdgeRec* host_edges, int64_t ne, int64_t n,
                                  int64_t** row_ptr, int32_t** col, int32_t** w, int64_t* m_out,
                                  cudaStream_t st) {
  std::string* err = nullptr;
  EdgeRec* de = nullptr;
  uint64_t *ka = nullptr, *kb = nullptr;
  int32_t *wa = nullptr, *wb = nullptr;
  const int64_t cap = ne > 0 ? ne : 1;
  GEN_CK(cudaMallocAsync(&de, cap * sizeof(EdgeRec), st));
  GEN_CK(cudaMallocAsync(&ka, cap * 8, st));
  GEN_CK(cudaMallocAsync(&kb, cap * 8, st));
  GEN_CK(cudaMallocAsync(&wa, cap * 4, st));
  GEN_CK(cudaMallocAsync(&wb, cap * 4, st));
  if (ne) GEN_CK(cudaMemcpyAsync(de, host_edges, ne * sizeof(EdgeRec), cudaMemcpyHostToDevice, st));
  const int grid = (int)std::min<int64_t>((cap + 255) / 256, 148 * 16);
  if (ne) {
    note_launch();
    edge_keys_kernel<<<grid, 256, 0, st>>>(de, ne, ka, wa);
  }
  cub::DoubleBuffer<uint64_t> dk(ka, kb);
  cub::DoubleBuffer<int32_t> dv(wa, wb);
  size_t t1 = 0, t2 = 0, t3 = 0;
  int64_t* nrun = nullptr;
  GEN_CK(cudaMallocAsync(&nrun, 8, st));
  GEN_CK(cub::DeviceRadixSort::SortPairs(nullptr, t1, dk, dv, ne, 0, 64, st));
  GEN_CK(cub::DeviceReduce::ReduceByKey(nullptr, t2, ka, kb, wa, wb, nrun, MinOp(), ne, st));
  int64_t* deg = nullptr;
  int64_t* rp = nullptr;
  GEN_CK(cudaMallocAsync(&deg, (n + 1) * 8, st));
  GEN_CK(cudaMallocAsync(&rp, (n + 1) * 8, st));
  GEN_CK(cudaMemsetAsync(deg, 0, (n + 1) * 8, st));
  GEN_CK(cub::DeviceScan::ExclusiveSum(nullptr, t3, deg, rp, n + 1, st));
  size_t tmp = std::max(t1, std::max(t2, t3));
  void* t = nullptr;
  GEN_CK(cudaMallocAsync(&t, tmp > 0 ? tmp : 1, st));
  GEN_CK(cub::DeviceRadixSort::SortPairs(t, tmp, dk, dv, ne, 0, 64, st));
  uint64_t* uk = dk.Alternate();
  int32_t* uw = dv.Alternate();
  GEN_CK(cub::DeviceReduce::ReduceByKey(t, tmp, dk.Current(), uk, dv.Current(), uw, nrun, MinOp(), ne, st));
  int64_t m = 0;
  GEN_CK(cudaMemcpyAsync(&m, nrun, 8, cudaMemcpyDeviceToHost, st));
  GEN_CK(cudaStreamSynchronize(st));
  if (ne == 0) m = 0;
  const int fgrid = (int)std::min<int64_t>((m + 255) / 256, 148 * 32);
  if (m > 0) {
    note_launch();
    row_count_kernel<<<fgrid, 256, 0, st>>>(uk, m, 32, deg);
  }
  GEN_CK(cub::DeviceScan::ExclusiveSum(t, tmp, deg, rp, n + 1, st));
  int32_t* dc = nullptr;
  int32_t* dw = nullptr;
  GEN_CK(cudaMallocAsync(&dc, (m + 4) * 4, st));
  GEN_CK(cudaMallocAsync(&dw, (m + 4) * 4, st));
  if (m > 0) {
    note_launch();
    split_keys_kernel<<<fgrid, 256, 0, st>>>(uk, m, dc);
    GEN_CK(cudaMemcpyAsync(dw, uw, m * 4, cudaMemcpyDeviceToDevice, st));
  }
  GEN_CK(cudaStreamSynchronize(st));
  for (void* p : {(void*)de, (void*)ka, (void*)kb, (void*)wa, (void*)wb, (void*)nrun, (void*)deg, t})
    cudaFree(p);
  *row_ptr = rp;
  *col = dc;
  *w = dw;
  *m_out = m;
  return cudaGetLastError();
}

cudaError_t max_degree(const int64_t* row_ptr, int64_t nrows, int64_t* out, cudaStream_t st) {
  unsigned long long* d = nullptr;
  cudaError_t e = cudaMallocAsync(&d, 8, st);
  if (e != cudaSuccess) return e;
  cudaMemsetAsync(d, 0, 8, st);
  if (nrows > 0) {  // an empty partition launches nothing (a zero grid is a launch error)
    note_launch();
    max_deg_kernel<<<(int)std::min<int64_t>((nrows + 255) / 256, 148 * 8), 256, 0, st>>>(row_ptr, nrows, d);
  }
  unsigned long long h = 0;
  cudaMemcpyAsync(&h, d, 8, cudaMemcpyDeviceToHost, st);
  cudaFreeAsync(d, st);
  e = cudaStreamSynchronize(st);
  *out = (int64_t)h;
  return e;
}

cudaError_t gen_partition(const irgl_gen_spec& s, int64_t n, int64_t lo, int64_t hi,
                          int64_t** row_ptr, int32_t** col, int32_t** w, int64_t* m_local,
                          cudaStream_t st, std::string* err) {
  const int64_t nloc = hi - lo;
  int64_t* rp = nullptr;
  int64_t* deg = nullptr;
  GEN_CK(cudaMallocAsync(&rp, (nloc + 1) * sizeof(int64_t), st));
  GEN_CK(cudaMallocAsync(&deg, (nloc + 1) * sizeof(int64_t), st));
  GEN_CK(cudaMemsetAsync(deg, 0, (nloc + 1) * sizeof(int64_t), st));
  int32_t* dc = nullptr;
  int32_t* dw = nullptr;
  int64_t m = 0;
  if (s.kind == IRGL_GEN_GRID) {
    GridSpec g{s.width, s.height, s.diag, s.cut_period,
               s.perc_keep_ppm > 0 ? s.perc_keep_ppm : 1000000, s.perc_seed};
    const int grid = (int)std::min<int64_t>((nloc + 255) / 256, 148 * 16);
    if (nloc > 0) {
      note_launch();
      grid_deg_kernel<<<grid, 256, 0, st>>>(g, lo, hi, deg);
    }
    size_t tmp = 0;
    GEN_CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp, deg, rp, nloc + 1, st));
    void* t = nullptr;
    GEN_CK(cudaMallocAsync(&t, tmp, st));
    GEN_CK(cub::DeviceScan::ExclusiveSum(t, tmp, deg, rp, nloc + 1, st));
    GEN_CK(cudaMemcpyAsync(&m, rp + nloc, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GEN_CK(cudaStreamSynchronize(st));
    cudaFreeAsync(t, st);
    GEN_CK(cudaMallocAsync(&dc, (m + 4) * sizeof(int32_t), st));
    GEN_CK(cudaMallocAsync(&dw, (m + 4) * sizeof(int32_t), st));
    if (nloc > 0) {
      note_launch();
      grid_fill_kernel<<<grid, 256, 0, st>>>(g, lo, hi, rp, s.wseed, dc, dw);
    }
  } else {
    const int scale = s.scale;
    const uint64_t ne = (uint64_t)(s.edge_factor > 0 ? s.edge_factor : 16) << scale;
    uint32_t k[4];
    philox(0, 0, 0, TAG_SCRM, (uint32_t)s.seed, (uint32_t)(s.seed >> 32), k);
    Scr scr{(uint64_t)(k[0] | 1u), k[1], (uint64_t)(k[2] | 1u), k[3], (1ull << scale) - 1,
            scale / 2 + 1, scale / 3 + 1};
    unsigned long long* ctr = nullptr;
    GEN_CK(cudaMallocAsync(&ctr, 8, st));
    GEN_CK(cudaMemsetAsync(ctr, 0, 8, st));
    const int ggrid = 148 * 16;
    note_launch();
    rmat_keys_kernel<false><<<ggrid, 256, 0, st>>>(ne, scale, s.seed, scr, lo, hi, ctr, nullptr);
    unsigned long long nk = 0;
    GEN_CK(cudaMemcpyAsync(&nk, ctr, 8, cudaMemcpyDeviceToHost, st));
    GEN_CK(cudaStreamSynchronize(st));
    uint64_t* ka = nullptr;
    uint64_t* kb = nullptr;
    GEN_CK(cudaMallocAsync(&ka, (nk > 0 ? nk : 1) * sizeof(uint64_t), st));
    GEN_CK(cudaMallocAsync(&kb, (nk > 0 ? nk : 1) * sizeof(uint64_t), st));
    GEN_CK(cudaMemsetAsync(ctr, 0, 8, st));
    note_launch();
    rmat_keys_kernel<true><<<ggrid, 256, 0, st>>>(ne, scale, s.seed, scr, lo, hi, ctr, ka);
    const int end_bit = bits_for(nloc > 1 ? nloc : 2) + scale;
    cub::DoubleBuffer<uint64_t> db(ka, kb);
    size_t tmp = 0;
    GEN_CK(cub::DeviceRadixSort::SortKeys(nullptr, tmp, db, (int64_t)nk, 0, end_bit, st));
    size_t tmp2 = 0;
    int64_t* nsel = nullptr;
    GEN_CK(cudaMallocAsync(&nsel, 8, st));
    GEN_CK(cub::DeviceSelect::Unique(nullptr, tmp2, ka, kb, nsel, (int64_t)nk, st));
    size_t tmp3 = 0;
    GEN_CK(cub::DeviceScan::ExclusiveSum(nullptr, tmp3, deg, rp, nloc + 1, st));
    tmp = std::max(tmp, std::max(tmp2, tmp3));
    void* t = nullptr;
    GEN_CK(cudaMallocAsync(&t, tmp, st));
    GEN_CK(cub::DeviceRadixSort::SortKeys(t, tmp, db, (int64_t)nk, 0, end_bit, st));
    uint64_t* sorted = db.Current();
    uint64_t* uniq = db.Alternate();
    GEN_CK(cub::DeviceSelect::Unique(t, tmp, sorted, uniq, nsel, (int64_t)nk, st));
    GEN_CK(cudaMemcpyAsync(&m, nsel, 8, cudaMemcpyDeviceToHost, st));
    GEN_CK(cudaStreamSynchronize(st));
    cudaFreeAsync(sorted, st);
    const int fgrid = (int)std::min<int64_t>((m + 255) / 256, 148 * 32);
    if (m > 0) {
      note_launch();
      row_count_kernel<<<fgrid, 256, 0, st>>>(uniq, m, scale, deg);
    }
    GEN_CK(cub::DeviceScan::ExclusiveSum(t, tmp, deg, rp, nloc + 1, st));
    GEN_CK(cudaMallocAsync(&dc, (m + 4) * sizeof(int32_t), st));
    GEN_CK(cudaMallocAsync(&dw, (m + 4) * sizeof(int32_t), st));
    if (m > 0) {
      note_launch();
      fill_csr_kernel<<<fgrid, 256, 0, st>>>(uniq, m, scale, lo, s.wseed, dc, dw);
    }
    cudaFreeAsync(uniq, st);
    cudaFreeAsync(t, st);
    cudaFreeAsync(nsel, st);
    cudaFreeAsync(ctr, st);
  }
  cudaFreeAsync(deg, st);
  GEN_CK(cudaStreamSynchronize(st));
  GEN_CK(cudaGetLastError());
  *row_ptr = rp;
  *col = dc;
  *w = dw;
  *m_local = m;
  (void)n;
  return cudaSuccess;
}

}  // namespace irgl
