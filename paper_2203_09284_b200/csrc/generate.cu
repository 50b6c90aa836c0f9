// generate.cu -- device graph generation + CSR build (K5 + K4).
//
// K5: every edge draw is a pure function of (seed, i):
//   * R-MAT (rmat.hpp:42-77): draw i runs on SplitMix64 split stream
//     child = mix(seed + (i+1)*gamma) (rng.hpp:22 applied to the root's
//     (i+1)-th output), level l uses mix(child + (l+1)*gamma) through
//     next_unit (rng.hpp:25) and the same quadrant comparisons;
//   * uniform G(n,m) = testutil::random_sparse (tests/test_util.hpp:49-58):
//     draw i is (out[2i+1] % n, out[2i+2] % n) of one SplitMix64(seed) stream.
// K4: build_csr (graph.hpp:35-70) without the host: self-loops dropped, keys
// (dst << k | src) bucketed by dst range, each bucket radix-sorted (CUB) and
// deduplicated, then in-degree counts -> int64 offsets by scan and
// out-degrees by atomics.  The arrays equal build_csr's bit for bit
// (tests/test_gpu_generate.py checks the digests of tests/golden/).
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "internal.cuh"

namespace fprb {

namespace {

constexpr uint64_t kGamma = 0x9e3779b97f4a7c15ULL;
constexpr int kFineBits = 10;  // histogram granularity: top 10 bits of dst
constexpr int64_t kGroupMax = 1ll << 30;

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

struct DrawSpec {
  int kind;
  uint32_t scale;
  double a, ab, abc;
  uint64_t seed;
  uint64_t n;
};

__device__ __forceinline__ void draw(const DrawSpec& s, uint64_t i, uint64_t& src, uint64_t& dst) {
  if (s.kind == 0) {
    const uint64_t child = mix64(s.seed + (i + 1) * kGamma);
    uint64_t u = 0, v = 0;
    for (uint32_t l = 0; l < s.scale; ++l) {
      const uint64_t z = mix64(child + (uint64_t)(l + 1) * kGamma);
      const double r = (double)(z >> 11) * 0x1.0p-53;
      u <<= 1;
      v <<= 1;
      if (r < s.a) {
      } else if (r < s.ab) {
        v |= 1;
      } else if (r < s.abc) {
        u |= 1;
      } else {
        u |= 1;
        v |= 1;
      }
    }
    src = u;
    dst = v;
  } else {
    src = mix64(s.seed + (2 * i + 1) * kGamma) % s.n;
    dst = mix64(s.seed + (2 * i + 2) * kGamma) % s.n;
  }
}

__global__ void hist_kernel(DrawSpec s, uint64_t draws, int fine_shift, unsigned long long* hist) {
  __shared__ unsigned int sh[1 << kFineBits];
  for (int b = threadIdx.x; b < (1 << kFineBits); b += blockDim.x) sh[b] = 0;
  __syncthreads();
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < draws; i += stride) {
    uint64_t u, v;
    draw(s, i, u, v);
    if (u != v) atomicAdd(&sh[v >> fine_shift], 1u);
  }
  __syncthreads();
  for (int b = threadIdx.x; b < (1 << kFineBits); b += blockDim.x)
    if (sh[b]) atomicAdd(&hist[b], (unsigned long long)sh[b]);
}

__global__ void scatter_kernel(DrawSpec s, uint64_t draws, int fine_shift, int k,
                               unsigned long long* cursor, uint64_t* keys) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < draws; i += stride) {
    uint64_t u, v;
    draw(s, i, u, v);
    if (u != v) {
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

int blocks_for(uint64_t work) {
  uint64_t b = (work + 255) / 256;
  return (int)std::max<uint64_t>(1, std::min<uint64_t>(b, 148ull * 16));
}

}  // namespace

cudaError_t generate_graph(const GenRequest& req, DevGraph& g, cudaStream_t st, const char** msg) {
  *msg = nullptr;
  DrawSpec s{};
  uint64_t n, draws;
  if (req.kind == 0) {
    s.kind = 0;
    s.scale = req.scale;
    s.a = req.a;
    s.ab = req.a + req.b;
    s.abc = req.a + req.b + req.c;
    n = 1ull << req.scale;
    draws = req.edge_factor << req.scale;
  } else {
    s.kind = 1;
    n = req.n;
    draws = req.n * req.avg_degree;
  }
  s.seed = req.seed;
  s.n = n;
  int k = 0;
  while (k < 64 && (1ull << k) < n) ++k;
  const int fine_shift = std::max(0, k - kFineBits);
  const int nfine = 1 << kFineBits;

  cudaError_t e;
#define GK(x)                       \
  do {                              \
    e = (x);                        \
    if (e != cudaSuccess) goto out; \
  } while (0)
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

  GK(cudaMallocAsync(&hist, 2 * nfine * sizeof(unsigned long long), st));
  GK(cudaMemsetAsync(hist, 0, 2 * nfine * sizeof(unsigned long long), st));
  hist_kernel<<<blocks_for(draws), 256, 0, st>>>(s, draws, fine_shift, hist);
  GK(cudaGetLastError());
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
      e = cudaSuccess;
      goto out;
    }
    groups.push_back({b, e2});
    gmax = std::max<int64_t>(gmax, (int64_t)(h_off[e2] - h_off[b]));
    b = e2;
  }
  GK(cudaMemcpyAsync(hist + nfine, h_off.data(), nfine * sizeof(unsigned long long), cudaMemcpyHostToDevice, st));
  GK(cudaMallocAsync(&keys, std::max<uint64_t>(valid, 1) * sizeof(uint64_t), st));
  scatter_kernel<<<blocks_for(draws), 256, 0, st>>>(s, draws, fine_shift, k, hist + nfine, keys);
  GK(cudaGetLastError());

  GK(cudaMallocAsync(&g.row, (n + 1) * sizeof(int64_t), st));
  GK(cudaMallocAsync(&g.src, (valid + 4) * sizeof(int32_t), st));
  GK(cudaMallocAsync(&g.outdeg, n * sizeof(int32_t), st));
  indeg = reinterpret_cast<unsigned long long*>(g.row);  // counts -> offsets in place
  GK(cudaMemsetAsync(g.row, 0, (n + 1) * sizeof(int64_t), st));
  GK(cudaMemsetAsync(g.outdeg, 0, n * sizeof(int32_t), st));
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
      tb = 0;
      GK(cub::DeviceScan::ExclusiveSum(nullptr, tb, (int64_t*)g.row, (int64_t*)g.row, (int64_t)n + 1, st));
      temp_bytes = std::max(temp_bytes, tb);
    }
    GK(cudaMallocAsync(&temp, std::max<size_t>(temp_bytes, 16), st));
  }
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
  if (n > 0) {
    size_t tb = temp_bytes;
    if (!temp) {
      GK(cub::DeviceScan::ExclusiveSum(nullptr, tb, (int64_t*)g.row, (int64_t*)g.row, (int64_t)n + 1, st));
      GK(cudaMallocAsync(&temp, std::max<size_t>(tb, 16), st));
      temp_bytes = tb;
    }
    tb = temp_bytes;
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
#undef GK
}

}  // namespace fprb
