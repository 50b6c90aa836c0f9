// generate.cu -- device graph generation + CSR build (K5 + K4) and the
// config-3 BFS relabel, all on the GPU.
//
// K5: every edge draw is a pure function of (seed, i):
//   * R-MAT (rmat.hpp:42-77): draw i runs on SplitMix64 split stream
//     child = mix(seed + (i+1)*gamma) (rng.hpp:22 applied to the root's
//     (i+1)-th output), level l uses mix(child + (l+1)*gamma) through
//     next_unit (rng.hpp:25) and the same quadrant comparisons;
//   * uniform G(n,m) = testutil::random_sparse (tests/test_util.hpp:49-58):
//     draw i is (out[2i+1] % n, out[2i+2] % n) of one SplitMix64(seed) stream;
//   * Chung-Lu (config 4; defined in DESIGN.md §4.1, restated in
//     oracle/fpr_oracle.c fo_generate_chunglu): integer power-law weights,
//     endpoints by inverse CDF over the inclusive weight prefix, ids through a
//     seeded random permutation.
// K4: build_csr (graph.hpp:35-70) without the host: self-loops dropped, keys
// (dst << k | src) bucketed by dst range, each bucket radix-sorted (CUB) and
// deduplicated, then in-degree counts -> int64 offsets by scan and
// out-degrees by atomics.  The arrays equal build_csr's bit for bit
// (tests/test_gpu_generate.py checks the digests of tests/golden/).
// Relabel (config 3): the out-CSR is built by the same
// pipeline on the transposed edges, then a level-synchronous BFS whose
// per-level order (winning parent's queue position, neighbour id) equals the
// sequential FIFO BFS of oracle/fpr_oracle.c fo_bfs_relabel.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdint>
#include <vector>

#include "internal.cuh"

namespace fprb {

namespace {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
constexpr uint64_t kClSeedDraw = 0x632be59bd9b4e019ULL;  // = oracle CL_SEED_DRAW
constexpr uint64_t kClSeedPerm = 0x9e6c63d0676a9a99ULL;  // = oracle CL_SEED_PERM
constexpr int kFineBits = 10;  // histogram granularity: top 10 bits of dst
constexpr int64_t kGroupMax = 1ll << 30;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

// ------------------------------------------------------------ edge sources
struct DrawSpec {
  int kind;  // 0 rmat, 1 uniform, 2 chung-lu
  uint32_t scale;
  double a, ab, abc;
  uint64_t seed;
  uint64_t n;
  const uint64_t* cum;   // chung-lu: inclusive weight prefix, n entries
  const int32_t* perm;   // chung-lu: old id -> new id
  uint64_t total_w;      // chung-lu: cum[n-1]

  __device__ __forceinline__ bool get(uint64_t i, uint64_t& src, uint64_t& dst) const {
    if (kind == 0) {
      const uint64_t child = mix64(seed + (i + 1) * kGamma);
      uint64_t u = 0, v = 0;
      for (uint32_t l = 0; l < scale; ++l) {
        const uint64_t z = mix64(child + (uint64_t)(l + 1) * kGamma);
        const double r = (double)(z >> 11) * 0x1.0p-53;
        u <<= 1;
        v <<= 1;
        if (r < a) {
        } else if (r < ab) {
          v |= 1;
        } else if (r < abc) {
          u |= 1;
        } else {
          u |= 1;
          v |= 1;
        }
      }
      src = u;
      dst = v;
    } else if (kind == 1) {
      src = mix64(seed + (2 * i + 1) * kGamma) % n;
      dst = mix64(seed + (2 * i + 2) * kGamma) % n;
    } else {
      const uint64_t sd = seed + kClSeedDraw;
      uint64_t ends[2];
      for (int side = 0; side < 2; ++side) {
        const uint64_t r = mix64(sd + (2 * i + 1 + (uint64_t)side) * kGamma) % total_w;
        uint64_t lo = 0, hi = n;  // first index with cum > r
        while (lo < hi) {
          const uint64_t mid = (lo + hi) >> 1;
          if (__ldg(cum + mid) > r)
            hi = mid;
          else
            lo = mid + 1;
        }
        ends[side] = (uint64_t)__ldg(perm + lo);
      }
      src = ends[0];
      dst = ends[1];
    }
    return src != dst;
  }
};

// Edges of an existing CSR, mapped through an optional relabel and optionally
// transposed (to build the out-CSR).
struct CsrSource {
  const int32_t* src;     // in_src[e]
  const int32_t* dst;     // owning row of edge e
  const int32_t* relabel; // nullptr or old -> new id
  int transpose;

  __device__ __forceinline__ bool get(uint64_t e, uint64_t& s, uint64_t& d) const {
    uint64_t a = (uint32_t)__ldg(src + e), b = (uint32_t)__ldg(dst + e);
    if (relabel) {
      a = (uint32_t)__ldg(relabel + a);
      b = (uint32_t)__ldg(relabel + b);
    }
    if (transpose) {
      s = b;
      d = a;
    } else {
      s = a;
      d = b;
    }
    return s != d;
  }
};

// Two separate id arrays (a host EdgeSet uploaded and narrowed).
struct ArraySource {
  const int32_t* s;
  const int32_t* d;

  __device__ __forceinline__ bool get(uint64_t e, uint64_t& src, uint64_t& dst) const {
    src = (uint32_t)__ldg(s + e);
    dst = (uint32_t)__ldg(d + e);
    return src != dst;
  }
};

// Dense (src, dst) id pairs of a parsed edge list (ingest.cu).
struct PairSource {
  const int32_t* ids;  // 2 per edge

  __device__ __forceinline__ bool get(uint64_t e, uint64_t& s, uint64_t& d) const {
    const int2 p = __ldg(reinterpret_cast<const int2*>(ids) + e);
    s = (uint32_t)p.x;
    d = (uint32_t)p.y;
    return s != d;
  }
};

template <class Src>
__global__ void hist_kernel(Src s, uint64_t count, int fine_shift, unsigned long long* hist) {
  __shared__ unsigned int sh[1 << kFineBits];
  for (int b = threadIdx.x; b < (1 << kFineBits); b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    uint64_t u, v;
    if (s.get(i, u, v)) atomicAdd(&sh[v >> fine_shift], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < (1 << kFineBits); b += blockDim.x)
    if (sh[b]) atomicAdd(&hist[b], (unsigned long long)sh[b]);
}

template <class Src>
__global__ void scatter_kernel(Src s, uint64_t count, int fine_shift, int k,
                               unsigned long long* cursor, uint64_t* keys) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    uint64_t u, v;
    if (s.get(i, u, v)) {
      const unsigned long long pos = atomicAdd(&cursor[v >> fine_shift], 1ull);
      keys[pos] = (v << k) | u;
    }
  }
}

__global__ void flag_kernel(const uint64_t* keys, int64_t count, int32_t* flags) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride)
    flags[i] = (i == 0 || keys[i] != keys[i - 1]) ? 1 : 0;
}

__global__ void emit_kernel(const uint64_t* keys, const int32_t* flags, const int32_t* pos,
                            int64_t count, int k, int64_t base, int32_t* src_out,
                            unsigned long long* indeg, int32_t* outdeg) {
  const uint64_t mask = (k == 0) ? 0 : ((1ull << k) - 1);
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    if (!flags[i]) continue;
    const uint64_t key = keys[i];
    const uint64_t u = key & mask, v = key >> k;
    src_out[base + pos[i]] = (int32_t)u;
    atomicAdd(&indeg[v], 1ull);
    atomicAdd(&outdeg[u], 1);
  }
}

// ------------------------------------------------------------ chung-lu prep
__global__ void cl_weight_kernel(const double* cdf, uint64_t kmax, uint64_t seed, uint64_t n,
                                 uint64_t* w) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint64_t child = mix64(seed + (i + 1) * kGamma);
    const double u = (double)(mix64(child + kGamma) >> 11) * 0x1.0p-53;
    uint64_t lo = 0, hi = kmax;
    while (lo < hi) {
      const uint64_t mid = (lo + hi) >> 1;
      if (__ldg(cdf + mid) > u)
        hi = mid;
      else
        lo = mid + 1;
    }
    w[i] = lo < kmax ? lo + 1 : kmax;
  }
}

__global__ void cl_permkey_kernel(uint64_t seed, uint64_t n, uint64_t* keys, int32_t* ids) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    keys[i] = mix64(seed + kClSeedPerm + (i + 1) * kGamma);
    ids[i] = (int32_t)i;
  }
}

__global__ void invert_perm_kernel(const int32_t* sorted_ids, uint64_t n, int32_t* perm) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t r = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride)
    perm[sorted_ids[r]] = (int32_t)r;
}

// ------------------------------------------------------------ BFS relabel
__global__ void row_of_edge_kernel(const int64_t* row, int32_t n, int32_t* dst_of_edge) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; d < n; d += stride)
    for (int64_t e = row[d]; e < row[d + 1]; ++e) dst_of_edge[e] = (int32_t)d;
}

// Level step A: every unvisited out-neighbour v of frontier position q gets
// parent[v] = min(q).
__global__ void bfs_claim_kernel(const int64_t* orow, const int32_t* odst, const int32_t* frontier,
                                 int64_t fs, const int32_t* new_id, unsigned int* parent) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < fs; q += nw) {
    const int32_t u = frontier[q];
    for (int64_t e = orow[u] + lane; e < orow[u + 1]; e += 32) {
      const int32_t v = odst[e];
      if (new_id[v] < 0) atomicMin(&parent[v], (unsigned int)q);
    }
  }
}

// Step B (emit=false): count winners per frontier position; step C (emit=true):
// write them in (q, ascending neighbour) order and assign their new ids.
template <bool EMIT>
__global__ void bfs_emit_kernel(const int64_t* orow, const int32_t* odst, const int32_t* frontier,
                                int64_t fs, int32_t* new_id, const unsigned int* parent,
                                int64_t* cnt_or_off, int32_t* next, int64_t assigned) {
  const int lane = threadIdx.x & 31;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < fs; q += nw) {
    const int32_t u = frontier[q];
    int64_t run = EMIT ? cnt_or_off[q] : 0;
    for (int64_t e0 = orow[u]; e0 < orow[u + 1]; e0 += 32) {
      const int64_t e = e0 + lane;
      bool win = false;
      int32_t v = 0;
      if (e < orow[u + 1]) {
        v = odst[e];
        win = new_id[v] < 0 && parent[v] == (unsigned int)q;
      }
      const unsigned b = __ballot_sync(0xffffffffu, win);
      if (EMIT && win) {
        const int64_t pos = run + __popc(b & ((1u << lane) - 1u));
        next[pos] = v;
        new_id[v] = (int32_t)(assigned + pos);
      }
      run += __popc(b);
    }
    if (!EMIT && lane == 0) cnt_or_off[q] = run;
  }
}

__global__ void unvisited_flag_kernel(const int32_t* new_id, int32_t n, int32_t* flag) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    flag[i] = new_id[i] < 0 ? 1 : 0;
}

__global__ void unvisited_assign_kernel(int32_t* new_id, int32_t n, const int32_t* rank,
                                        int64_t assigned) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    if (new_id[i] < 0) new_id[i] = (int32_t)(assigned + rank[i]);
}

__global__ void set_root_kernel(int32_t* new_id, int32_t* frontier, int32_t root) {
  new_id[root] = 0;
  frontier[0] = root;
}

int blocks_for(uint64_t work) {
  uint64_t b = (work + 255) / 256;
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(b, 148ull * 16));
}

#define GK(x)                       \
  do {                              \
    e = (x);                        \
    if (e != cudaSuccess) goto out; \
  } while (0)

// The K4 pipeline: normalise the `count` edges of `s` into an in-CSR over n
// vertices (build_csr semantics), allocating g's arrays on stream st.
template <class Src>
cudaError_t build_csr_from(const Src& s, uint64_t count, uint64_t n, DevGraph& g, cudaStream_t st,
                           const char** msg) {
  int k = 0;
  while (k < 64 && (1ull << k) < n) ++k;
  const int fine_shift = std::max(0, k - kFineBits);
  const int nfine = 1 << kFineBits;

  cudaError_t e = cudaSuccess;
  unsigned long long* hist = nullptr;
  uint64_t* keys = nullptr;
  uint64_t* alt = nullptr;
  int32_t* flags = nullptr;
  int32_t* pos = nullptr;
  void* temp = nullptr;
  unsigned long long* indeg = nullptr;
  std::vector<unsigned long long> h_hist(nfine), h_off(nfine + 1);
  std::vector<std::pair<int, int>> groups;
  uint64_t valid = 0;
  int64_t gmax = 0, m = 0;
  size_t temp_bytes = 0;
  g.row = nullptr;
  g.src = nullptr;
  g.outdeg = nullptr;

  GK(cudaMallocAsync(&hist, 2 * nfine * sizeof(unsigned long long), st));
  GK(cudaMemsetAsync(hist, 0, 2 * nfine * sizeof(unsigned long long), st));
  if (count > 0) {
    hist_kernel<<<blocks_for(count), 256, 0, st>>>(s, count, fine_shift, hist);
    GK(cudaGetLastError());
  }
  GK(cudaMemcpyAsync(h_hist.data(), hist, nfine * sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  GK(cudaStreamSynchronize(st));
  h_off[0] = 0;
  for (int b = 0; b < nfine; ++b) h_off[b + 1] = h_off[b] + h_hist[b];
  valid = h_off[nfine];
  // Contiguous groups of fine buckets, each <= kGroupMax keys.
  for (int b = 0; b < nfine;) {
    int e2 = b + 1;
    while (e2 < nfine && h_off[e2 + 1] - h_off[b] <= (unsigned long long)kGroupMax) ++e2;
    if (h_off[e2] - h_off[b] > (unsigned long long)INT32_MAX) {
      *msg = "a dst bucket exceeds 2^31 edges";
      goto out;
    }
    groups.push_back({b, e2});
    gmax = std::max<int64_t>(gmax, (int64_t)(h_off[e2] - h_off[b]));
    b = e2;
  }
  GK(cudaMemcpyAsync(hist + nfine, h_off.data(), nfine * sizeof(unsigned long long), cudaMemcpyHostToDevice, st));
  GK(cudaMallocAsync(&keys, std::max<uint64_t>(valid, 1) * sizeof(uint64_t), st));
  if (count > 0) {
    scatter_kernel<<<blocks_for(count), 256, 0, st>>>(s, count, fine_shift, k, hist + nfine, keys);
    GK(cudaGetLastError());
  }

  GK(cudaMallocAsync(&g.row, (n + 1) * sizeof(int64_t), st));
  GK(cudaMallocAsync(&g.src, (valid + 8) * sizeof(int32_t), st));
  GK(cudaMallocAsync(&g.outdeg, std::max<uint64_t>(n, 1) * sizeof(int32_t), st));
  indeg = reinterpret_cast<unsigned long long*>(g.row);  // counts -> offsets in place
  GK(cudaMemsetAsync(g.row, 0, (n + 1) * sizeof(int64_t), st));
  GK(cudaMemsetAsync(g.outdeg, 0, std::max<uint64_t>(n, 1) * sizeof(int32_t), st));
  GK(cudaMemsetAsync(g.src, 0, (valid + 8) * sizeof(int32_t), st));
  if (gmax > 0) {
    GK(cudaMallocAsync(&alt, gmax * sizeof(uint64_t), st));
    GK(cudaMallocAsync(&flags, gmax * sizeof(int32_t), st));
    GK(cudaMallocAsync(&pos, gmax * sizeof(int32_t), st));
    {
      size_t tb = 0;
      cub::DoubleBuffer<uint64_t> db(keys, alt);
      GK(cub::DeviceRadixSort::SortKeys(nullptr, tb, db, (int)gmax, 0, 2 * k, st));
      temp_bytes = std::max(temp_bytes, tb);
      tb = 0;
      GK(cub::DeviceScan::ExclusiveSum(nullptr, tb, flags, pos, (int)gmax, st));
      temp_bytes = std::max(temp_bytes, tb);
    }
  }
  {
    size_t tb = 0;
    GK(cub::DeviceScan::ExclusiveSum(nullptr, tb, (int64_t*)g.row, (int64_t*)g.row, (int64_t)n + 1, st));
    temp_bytes = std::max(temp_bytes, tb);
  }
  GK(cudaMallocAsync(&temp, std::max<size_t>(temp_bytes, 16), st));
  for (auto [b0, b1] : groups) {
    const int64_t off = (int64_t)h_off[b0];
    const int cnt = (int)(h_off[b1] - h_off[b0]);
    if (cnt == 0) continue;
    cub::DoubleBuffer<uint64_t> db(keys + off, alt);
    size_t tb = temp_bytes;
    GK(cub::DeviceRadixSort::SortKeys(temp, tb, db, cnt, 0, 2 * k, st));
    const uint64_t* sorted = db.Current();
    flag_kernel<<<blocks_for(cnt), 256, 0, st>>>(sorted, cnt, flags);
    GK(cudaGetLastError());
    tb = temp_bytes;
    GK(cub::DeviceScan::ExclusiveSum(temp, tb, flags, pos, cnt, st));
    emit_kernel<<<blocks_for(cnt), 256, 0, st>>>(sorted, flags, pos, cnt, k, m, g.src, indeg, g.outdeg);
    GK(cudaGetLastError());
    int32_t last_flag = 0, last_pos = 0;
    GK(cudaMemcpyAsync(&last_flag, flags + cnt - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    GK(cudaMemcpyAsync(&last_pos, pos + cnt - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
    GK(cudaStreamSynchronize(st));
    m += (int64_t)last_pos + last_flag;
  }
  {
    size_t tb = temp_bytes;
    GK(cub::DeviceScan::ExclusiveSum(temp, tb, (int64_t*)g.row, (int64_t*)g.row, (int64_t)n + 1, st));
  }
  g.n = (int32_t)n;
  g.m = m;
  GK(cudaStreamSynchronize(st));
out:
  for (void* p : {(void*)hist, (void*)keys, (void*)alt, (void*)flags, (void*)pos, temp})
    if (p) cudaFreeAsync(p, st);
  cudaStreamSynchronize(st);
  if (e != cudaSuccess || *msg) {
    for (void* p : {(void*)g.row, (void*)g.src, (void*)g.outdeg})
      if (p) cudaFree(p);
    g.row = nullptr;
    g.src = nullptr;
    g.outdeg = nullptr;
  }
  return e;
}

void free_graph(DevGraph& g, cudaStream_t st) {
  for (void* p : {(void*)g.row, (void*)g.src, (void*)g.outdeg})
    if (p) cudaFreeAsync(p, st);
  g.row = nullptr;
  g.src = nullptr;
  g.outdeg = nullptr;
}

// BFS relabel of g (config 3): returns new_id (device, n int32) in *out.
cudaError_t bfs_relabel(const DevGraph& g, int32_t root, cudaStream_t st, int32_t** out,
                        const char** msg) {
  cudaError_t e = cudaSuccess;
  const int32_t n = g.n;
  int32_t* dst_of_edge = nullptr;
  int32_t* new_id = nullptr;
  unsigned int* parent = nullptr;
  int32_t* fa = nullptr;
  int32_t* fb = nullptr;
  int64_t* cnt = nullptr;
  int64_t* off = nullptr;
  int32_t* flag = nullptr;
  int32_t* rank = nullptr;
  void* temp = nullptr;
  size_t temp_bytes = 0;
  DevGraph og;  // out-CSR: og.row = out offsets, og.src = out-neighbours (ascending)
  int64_t fs = 1, assigned = 1;
  *out = nullptr;
  GK(cudaMallocAsync(&dst_of_edge, std::max<int64_t>(g.m, 1) * sizeof(int32_t), st));
  row_of_edge_kernel<<<blocks_for(n), 256, 0, st>>>(g.row, n, dst_of_edge);
  GK(cudaGetLastError());
  GK(build_csr_from(CsrSource{g.src, dst_of_edge, nullptr, 1}, (uint64_t)g.m, (uint64_t)n, og, st, msg));
  if (*msg) goto out;
  GK(cudaMallocAsync(&new_id, n * sizeof(int32_t), st));
  GK(cudaMallocAsync(&parent, n * sizeof(unsigned int), st));
  GK(cudaMallocAsync(&fa, n * sizeof(int32_t), st));
  GK(cudaMallocAsync(&fb, n * sizeof(int32_t), st));
  GK(cudaMallocAsync(&cnt, (n + 1) * sizeof(int64_t), st));
  GK(cudaMallocAsync(&off, (n + 1) * sizeof(int64_t), st));
  GK(cudaMemsetAsync(new_id, 0xFF, n * sizeof(int32_t), st));
  GK(cudaMemsetAsync(parent, 0xFF, n * sizeof(unsigned int), st));
  {
    size_t tb = 0;
    GK(cub::DeviceScan::ExclusiveSum(nullptr, tb, cnt, off, (int64_t)n + 1, st));
    temp_bytes = std::max(temp_bytes, tb);
    tb = 0;
    GK(cub::DeviceScan::ExclusiveSum(nullptr, tb, (int32_t*)fa, (int32_t*)fb, n, st));
    temp_bytes = std::max(temp_bytes, tb);
  }
  GK(cudaMallocAsync(&temp, std::max<size_t>(temp_bytes, 16), st));
  set_root_kernel<<<1, 1, 0, st>>>(new_id, fa, root);
  GK(cudaGetLastError());
  while (fs > 0) {
    const int grid = blocks_for((uint64_t)fs * 32);
    bfs_claim_kernel<<<grid, 256, 0, st>>>(og.row, og.src, fa, fs, new_id, parent);
    bfs_emit_kernel<false><<<grid, 256, 0, st>>>(og.row, og.src, fa, fs, new_id, parent, cnt, fb, assigned);
    GK(cudaGetLastError());
    GK(cudaMemsetAsync(cnt + fs, 0, sizeof(int64_t), st));
    size_t tb = temp_bytes;
    GK(cub::DeviceScan::ExclusiveSum(temp, tb, cnt, off, fs + 1, st));
    bfs_emit_kernel<true><<<grid, 256, 0, st>>>(og.row, og.src, fa, fs, new_id, parent, off, fb, assigned);
    GK(cudaGetLastError());
    int64_t next_fs = 0;
    GK(cudaMemcpyAsync(&next_fs, off + fs, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    GK(cudaStreamSynchronize(st));
    assigned += next_fs;
    fs = next_fs;
    std::swap(fa, fb);
  }
  // unreached vertices, ascending old id
  flag = fa;  // reuse the frontier buffers (n int32 each)
  rank = fb;
  unvisited_flag_kernel<<<blocks_for(n), 256, 0, st>>>(new_id, n, flag);
  GK(cudaGetLastError());
  {
    size_t tb = temp_bytes;
    GK(cub::DeviceScan::ExclusiveSum(temp, tb, flag, rank, n, st));
  }
  unvisited_assign_kernel<<<blocks_for(n), 256, 0, st>>>(new_id, n, rank, assigned);
  GK(cudaGetLastError());
  GK(cudaStreamSynchronize(st));
  *out = new_id;
  new_id = nullptr;
out:
  for (void* p : {(void*)dst_of_edge, (void*)new_id, (void*)parent, (void*)fa, (void*)fb,
                  (void*)cnt, (void*)off, temp})
    if (p) cudaFreeAsync(p, st);
  free_graph(og, st);
  cudaStreamSynchronize(st);
  return e;
}

}  // namespace

cudaError_t build_csr_from_pairs(const int32_t* pairs, int64_t m, uint64_t n, DevGraph& g, cudaStream_t st,
                                 const char** msg) {
  return build_csr_from(PairSource{pairs}, (uint64_t)m, n, g, st, msg);
}

cudaError_t build_csr_from_arrays(const int32_t* src, const int32_t* dst, int64_t m, uint64_t n, DevGraph& g,
                                  cudaStream_t st, const char** msg) {
  return build_csr_from(ArraySource{src, dst}, (uint64_t)m, n, g, st, msg);
}


__global__ void draws_kernel(DrawSpec s, uint64_t i0, uint64_t count, uint64_t* src, uint64_t* dst) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) {
    uint64_t a, b;
    s.get(i0 + i, a, b);
    src[i] = a;
    dst[i] = b;
  }
}

// Draws [i0, i0 + count) of the R-MAT (kind 0) or random_sparse (kind 1)
// generator, before any filtering: the EdgeSet order of generate_rmat
// (rmat.hpp:54-75) / the draw order of testutil::random_sparse.
cudaError_t generate_draws(const GenRequest& req, uint64_t i0, uint64_t count, uint64_t* d_src, uint64_t* d_dst,
                           cudaStream_t st) {
  DrawSpec s{};
  s.kind = req.kind;
  s.seed = req.seed;
  if (req.kind == 0) {
    s.scale = req.scale;
    s.a = req.a;
    s.ab = req.a + req.b;
    s.abc = req.a + req.b + req.c;
  } else if (req.kind == 1) {
    s.n = req.n;
  } else {
    return cudaErrorInvalidValue;
  }
  if (count == 0) return cudaSuccess;
  draws_kernel<<<blocks_for(count), 256, 0, st>>>(s, i0, count, d_src, d_dst);
  return cudaGetLastError();
}

cudaError_t generate_graph(const GenRequest& req, DevGraph& g, cudaStream_t st, const char** msg) {
  *msg = nullptr;
  cudaError_t e = cudaSuccess;
  DrawSpec s{};
  uint64_t n = 0, draws = 0;
  uint64_t* w = nullptr;  // chung-lu weights, then their inclusive prefix
  uint64_t* pkeys = nullptr;
  uint64_t* pkeys2 = nullptr;
  int32_t* pids = nullptr;
  int32_t* pids2 = nullptr;
  int32_t* perm = nullptr;
  double* cdf = nullptr;
  void* temp = nullptr;
  int32_t* new_id = nullptr;
  int32_t* dst_of_edge = nullptr;
  DevGraph natural;
  if (req.kind == 0) {
    s.kind = 0;
    s.scale = req.scale;
    s.a = req.a;
    s.ab = req.a + req.b;
    s.abc = req.a + req.b + req.c;
    n = 1ull << req.scale;
    draws = req.edge_factor << req.scale;
  } else if (req.kind == 1) {
    s.kind = 1;
    n = req.n;
    draws = req.n * req.avg_degree;
  } else {
    // Chung-Lu: cdf on the host (std::pow, ascending-k sums: the oracle's
    // exact arithmetic), weights + prefix + permutation on the device.
    s.kind = 2;
    n = req.n;
    draws = req.draws;
    const uint64_t kmax = req.kmax;
    std::vector<double> h_cdf(kmax);
    double z = 0.0;
    for (uint64_t kk = 1; kk <= kmax; ++kk) z += std::pow((double)kk, -req.alpha);
    double acc = 0.0;
    for (uint64_t kk = 1; kk <= kmax; ++kk) {
      acc += std::pow((double)kk, -req.alpha);
      h_cdf[kk - 1] = acc / z;
    }
    GK(cudaMallocAsync(&cdf, kmax * sizeof(double), st));
    GK(cudaMemcpyAsync(cdf, h_cdf.data(), kmax * sizeof(double), cudaMemcpyHostToDevice, st));
    GK(cudaMallocAsync(&w, n * sizeof(uint64_t), st));
    cl_weight_kernel<<<blocks_for(n), 256, 0, st>>>(cdf, kmax, req.seed, n, w);
    GK(cudaGetLastError());
    GK(cudaMallocAsync(&pkeys, n * sizeof(uint64_t), st));
    GK(cudaMallocAsync(&pkeys2, n * sizeof(uint64_t), st));
    GK(cudaMallocAsync(&pids, n * sizeof(int32_t), st));
    GK(cudaMallocAsync(&pids2, n * sizeof(int32_t), st));
    GK(cudaMallocAsync(&perm, n * sizeof(int32_t), st));
    cl_permkey_kernel<<<blocks_for(n), 256, 0, st>>>(req.seed, n, pkeys, pids);
    GK(cudaGetLastError());
    {
      size_t tb1 = 0, tb2 = 0;
      GK(cub::DeviceScan::InclusiveSum(nullptr, tb1, w, w, (int64_t)n, st));
      GK(cub::DeviceRadixSort::SortPairs(nullptr, tb2, pkeys, pkeys2, pids, pids2, (int64_t)n, 0, 64, st));
      GK(cudaMallocAsync(&temp, std::max<size_t>(std::max(tb1, tb2), 16), st));
      GK(cub::DeviceScan::InclusiveSum(temp, tb1, w, w, (int64_t)n, st));
      size_t tb = std::max(tb1, tb2);
      GK(cub::DeviceRadixSort::SortPairs(temp, tb, pkeys, pkeys2, pids, pids2, (int64_t)n, 0, 64, st));
    }
    invert_perm_kernel<<<blocks_for(n), 256, 0, st>>>(pids2, n, perm);
    GK(cudaGetLastError());
    GK(cudaMemcpyAsync(&s.total_w, w + n - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    GK(cudaStreamSynchronize(st));
    s.cum = w;
    s.perm = perm;
  }
  s.seed = req.seed;
  s.n = n;
  if (!req.relabel_bfs) {
    GK(build_csr_from(s, draws, n, g, st, msg));
  } else {
    GK(build_csr_from(s, draws, n, natural, st, msg));
    if (*msg) goto out;
    GK(bfs_relabel(natural, (int32_t)req.bfs_root, st, &new_id, msg));
    if (*msg) goto out;
    GK(cudaMallocAsync(&dst_of_edge, std::max<int64_t>(natural.m, 1) * sizeof(int32_t), st));
    row_of_edge_kernel<<<blocks_for(n), 256, 0, st>>>(natural.row, natural.n, dst_of_edge);
    GK(cudaGetLastError());
    GK(build_csr_from(CsrSource{natural.src, dst_of_edge, new_id, 0}, (uint64_t)natural.m, n, g, st, msg));
  }
out:
  for (void* p : {(void*)w, (void*)pkeys, (void*)pkeys2, (void*)pids, (void*)pids2, (void*)perm,
                  (void*)cdf, temp, (void*)new_id, (void*)dst_of_edge})
    if (p) cudaFreeAsync(p, st);
  free_graph(natural, st);
  cudaStreamSynchronize(st);
  return e;
}

cudaError_t relabel_order_bfs(const DevGraph& g, int32_t root, int32_t* new_id_out,
                              cudaStream_t st, const char** msg) {
  *msg = nullptr;
  int32_t* new_id = nullptr;
  cudaError_t e = bfs_relabel(g, root, st, &new_id, msg);
  if (e == cudaSuccess && !*msg)
    e = cudaMemcpyAsync(new_id_out, new_id, g.n * sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  if (new_id) cudaFreeAsync(new_id, st);
  cudaStreamSynchronize(st);
  return e;
}

// Locality reorders (opt-in).  FPR_B200_OPT_REORDER: vertices renumbered by
// descending out-degree (ties by id) -- the gather frequency of contrib[s] is
// out_degree(s), so hot contributions share sectors and stay L2-resident.
// FPR_B200_OPT_REORDER_SOURCES (sources_only): a stable partition, vertices
// with out-degree > 0 first -- only they are ever gathered, so the gathered
// vector shrinks to them while the caller's (crawl) order is kept inside
// each class.  Returns the new CSR in `out` and new_of_old (device, n int32)
// in *perm.
// block_shift > 0: the order holds inside each block of 2^block_shift ids
// (block, then the degree key, then the id inside the block: 62 bits).
__global__ void degree_key_kernel(const int32_t* outdeg, int32_t n, bool sources_only, int block_shift,
                                  uint64_t* keys, int32_t* ids) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const uint32_t major = sources_only ? (outdeg[i] == 0 ? 1u : 0u) : (uint32_t)(INT32_MAX - outdeg[i]);
    if (block_shift > 0)
      keys[i] = ((uint64_t)(i >> block_shift) << 54) | ((uint64_t)major << block_shift) |
                (uint64_t)(i & ((int64_t(1) << block_shift) - 1));
    else
      keys[i] = ((uint64_t)major << 32) | (uint32_t)i;
    ids[i] = (int32_t)i;
  }
}

cudaError_t reorder_by_degree(const DevGraph& g, bool sources_only, int block_shift, DevGraph& out, int32_t** perm,
                              cudaStream_t st, const char** msg) {
  *msg = nullptr;
  *perm = nullptr;
  cudaError_t e = cudaSuccess;
  const int32_t n = g.n;
  uint64_t* k1 = nullptr;
  uint64_t* k2 = nullptr;
  int32_t* i1 = nullptr;
  int32_t* i2 = nullptr;
  int32_t* p = nullptr;
  int32_t* dst_of_edge = nullptr;
  void* temp = nullptr;
  size_t tb = 0;
  GK(cudaMallocAsync(&k1, n * sizeof(uint64_t), st));
  GK(cudaMallocAsync(&k2, n * sizeof(uint64_t), st));
  GK(cudaMallocAsync(&i1, n * sizeof(int32_t), st));
  GK(cudaMallocAsync(&i2, n * sizeof(int32_t), st));
  GK(cudaMallocAsync(&p, n * sizeof(int32_t), st));
  degree_key_kernel<<<blocks_for(n), 256, 0, st>>>(g.outdeg, n, sources_only, block_shift, k1, i1);
  GK(cudaGetLastError());
  GK(cub::DeviceRadixSort::SortPairs(nullptr, tb, k1, k2, i1, i2, (int64_t)n, 0, 64, st));
  GK(cudaMallocAsync(&temp, std::max<size_t>(tb, 16), st));
  GK(cub::DeviceRadixSort::SortPairs(temp, tb, k1, k2, i1, i2, (int64_t)n, 0, 64, st));
  invert_perm_kernel<<<blocks_for(n), 256, 0, st>>>(i2, (uint64_t)n, p);
  GK(cudaGetLastError());
  GK(cudaMallocAsync(&dst_of_edge, std::max<int64_t>(g.m, 1) * sizeof(int32_t), st));
  row_of_edge_kernel<<<blocks_for(n), 256, 0, st>>>(g.row, n, dst_of_edge);
  GK(cudaGetLastError());
  GK(build_csr_from(CsrSource{g.src, dst_of_edge, p, 0}, (uint64_t)g.m, (uint64_t)n, out, st, msg));
  if (*msg) goto out;
  *perm = p;
  p = nullptr;
out:
  for (void* q : {(void*)k1, (void*)k2, (void*)i1, (void*)i2, (void*)p, (void*)dst_of_edge, temp})
    if (q) cudaFreeAsync(q, st);
  cudaStreamSynchronize(st);
  return e;
}

#undef GK

}  // namespace fprb
