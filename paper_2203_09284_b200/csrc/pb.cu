// pb.cu -- propagation-blocked EC sweep (FPR_B200_OPT_PB) for graphs whose
// contribution vector far exceeds L2 (configs 4/5).
//
// The pull gather contrib[in_src[e]] misses L2 on such graphs, and each miss
// pulls ~64 B from HBM for 8 useful bytes (profiles/r1_large_configs_ncu.md).
// Propagation blocking (Beamer, Asanovic, Patterson, "Reducing PageRank
// communication via propagation blocking", IPDPS'17) trades the random reads
// for streams.
//
// Layout, built once from the resident in-CSR:
//   * rows are cut into bins of 2^shift consecutive rows; a bin's entries are
//     exactly its rows' in-edges (duplicates and self loops included);
//   * inside a bin, entries are regrouped by source chunk (src >> chunk_shift):
//     segment (bin b, chunk c) is contiguous;
//   * entry = (source id, row offset inside the bin as uint16).
// Per sweep:
//   * phase 1 (pb_gather_kernel): warps walk the segments chunk by chunk, so
//     the sources read at any moment span one chunk's contributions (a 64 MB
//     window at the default chunk of 2^23 sources, half of L2), and write
//     val[pos] = prev[src_bm[pos]] contiguously;
//   * phase 2 (pb_accum_kernel): one CTA per bin accumulates val into the
//     bin's rows in shared memory and finishes the rows exactly like the
//     blocked engine's apply (blocked.cu): base + d*sum without FMA,
//     contribution, residual.
// Per edge and sweep: 4 B source + 8 B value written + 8 B read + 2 B offset,
// all sequential, where a missed pull gather moved ~64 B of DRAM.
// A row's sum is accumulated in shared-memory atomic order, a regrouping of
// the reference's left-to-right sum: bit patterns may differ from run to run,
// well inside the 1e-12 per-iteration tolerance (tests/test_gpu_engines.py
// test_pb_*).  Measurements and rejected variants: DESIGN.md §3.4.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <vector>

#include "internal.cuh"

namespace fprb {

namespace {

constexpr int kPbThreads = 1024;
constexpr int kGatherThreads = 256;

constexpr int kPieceEntries = 1024;  // phase-1 work item: up to this many entries of one segment
#ifndef FPR_PB_STEPS
#define FPR_PB_STEPS 4
#endif
#ifndef FPR_PB_MINB
#define FPR_PB_MINB 2
#endif
constexpr int kLaneRun = FPR_PB_STEPS;  // phase 2: warp steps (32 entries each) with loads in flight

// One CTA per bin: histogram its edges by source chunk, scan, then a stable
// scatter (tiles of the bin's CSR edges, block radix-sorted by chunk) so each
// (bin, chunk) segment lists its entries in ascending row order -- phase 2
// merges runs of one row before touching shared memory.  counts/start are
// chunk-major.
__global__ void __launch_bounds__(kPbThreads) pb_layout_kernel(const int64_t* row, const int32_t* src, int32_t n,
                                                                int shift, int chunk_shift, int key_bits,
                                                                int64_t nbins, int64_t nchunks, uint32_t* counts,
                                                                int64_t* start, int32_t* src_bm, uint16_t* dstl_bm) {
  using Sort = cub::BlockRadixSort<uint32_t, kPbThreads, 1, uint64_t>;
  using ScanU = cub::BlockScan<uint32_t, kPbThreads>;
  using ScanI = cub::BlockScan<int, kPbThreads>;
  __shared__ union {
    typename Sort::TempStorage sort;
    typename ScanU::TempStorage scanu;
    typename ScanI::TempStorage scani;
  } tmp;
  __shared__ uint32_t skey[kPbThreads];
  extern __shared__ uint32_t h[];
  const int tid = threadIdx.x;
  const uint32_t sentinel = (uint32_t)nchunks;
  for (int64_t b = blockIdx.x; b < nbins; b += gridDim.x) {
    for (int64_t c = tid; c < nchunks; c += blockDim.x) h[c] = 0;
    __syncthreads();
    const int64_t r0 = b << shift;
    const int64_t r1 = min((int64_t)n, r0 + ((int64_t)1 << shift));
    const int64_t e0 = row[r0], e1 = row[r1];
    for (int64_t e = e0 + tid; e < e1; e += blockDim.x) atomicAdd(&h[(uint32_t)__ldg(src + e) >> chunk_shift], 1u);
    __syncthreads();
    uint32_t running = 0;
    for (int64_t t0 = 0; t0 < nchunks; t0 += blockDim.x) {
      const int64_t c = t0 + tid;
      const uint32_t v = c < nchunks ? h[c] : 0u;
      uint32_t x, tile;
      ScanU(tmp.scanu).ExclusiveSum(v, x, tile);
      if (c < nchunks) {
        counts[c * nbins + b] = v;
        start[c * nbins + b] = e0 + running + x;
        h[c] = running + x;
      }
      running += tile;
      __syncthreads();
    }
    for (int64_t t = e0; t < e1; t += kPbThreads) {
      const int64_t e = t + tid;
      uint32_t key[1] = {sentinel};
      uint64_t val[1] = {0};
      if (e < e1) {
        // row of edge e: last r in [r0, r1) with row[r] <= e
        int64_t lo = r0, hi = r1 - 1;
        while (lo < hi) {
          const int64_t mid = (lo + hi + 1) >> 1;
          if (__ldg(row + mid) <= e) lo = mid;
          else hi = mid - 1;
        }
        const uint32_t s = (uint32_t)__ldg(src + e);
        key[0] = s >> chunk_shift;
        val[0] = ((uint64_t)s << 16) | (uint64_t)(lo - r0);
      }
      Sort(tmp.sort).Sort(key, val, 0, key_bits);
      __syncthreads();
      skey[tid] = key[0];
      __syncthreads();
      int hs = (tid == 0 || skey[tid - 1] != key[0]) ? tid : 0;
      ScanI(tmp.scani).InclusiveScan(hs, hs, cub::Max());
      const bool real = key[0] != sentinel;
      if (real) {
        const int64_t pos = e0 + h[key[0]] + (tid - hs);
        src_bm[pos] = (int32_t)(val[0] >> 16);
        dstl_bm[pos] = (uint16_t)(val[0] & 0xFFFFu);
      }
      __syncthreads();
      if (real && (tid == kPbThreads - 1 || skey[tid + 1] != key[0])) h[key[0]] += (uint32_t)(tid - hs + 1);
      __syncthreads();
    }
  }
}

__global__ void pb_piece_count_kernel(const uint32_t* counts, int64_t nseg, uint32_t* npieces) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nseg; s += stride)
    npieces[s] = (counts[s] + kPieceEntries - 1) / kPieceEntries;
}

__global__ void pb_piece_fill_kernel(const uint32_t* counts, const int64_t* start, const uint32_t* piece_off,
                                     int64_t nseg, int64_t* item_start, uint32_t* item_len) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nseg; s += stride) {
    const uint32_t cnt = counts[s];
    const int64_t p0 = start[s];
    uint32_t o = piece_off[s];
    for (uint32_t k = 0; k < cnt; k += kPieceEntries, ++o) {
      item_start[o] = p0 + k;
      item_len[o] = min((uint32_t)kPieceEntries, cnt - k);
    }
  }
}

// Phase 1: warps take pieces in chunk order from a global counter (static
// striding lets fast warps drift chunks ahead and the concurrently read
// contribution window outgrow L2); 8 gathers in flight per lane.
__global__ void __launch_bounds__(kGatherThreads) pb_gather_kernel(const int32_t* src_bm, const int64_t* item_start,
                                                                    const uint32_t* item_len, int64_t nitems,
                                                                    const double* prev, double* val,
                                                                    unsigned long long* next_item) {
  constexpr int U = 8;
  const int lane = threadIdx.x & 31;
  for (;;) {
    unsigned long long it = 0;
    if (lane == 0) it = atomicAdd(next_item, 1ull);
    it = __shfl_sync(0xffffffffu, it, 0);
    if ((int64_t)it >= nitems) break;
    const int64_t p0 = __ldg(item_start + it);
    const uint32_t len = __ldg(item_len + it);
    for (uint32_t k0 = 0; k0 < len; k0 += 32 * U) {
      int32_t s[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t k = k0 + u * 32 + lane;
        s[u] = k < len ? __ldcs(src_bm + p0 + k) : -1;
      }
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = s[u] >= 0 ? __ldcg(prev + s[u]) : 0.0;
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t k = k0 + u * 32 + lane;
        if (k < len) __stcs(val + p0 + k, v[u]);
      }
    }
  }
}

// Phase 2: CTAs take work units from a counter: a unit is a whole bin, or a
// piece of a heavy bin (skewed graphs put a large share of the edges in the
// bins of the hub rows; one CTA per bin left one SM working 7x longer than
// the average on config 3).  Warps read the unit's entries
// coalesced, 32 consecutive entries per step; inside a segment rows ascend,
// so equal rows sit in consecutive lanes: a warp segmented scan folds each
// run and only its last lane adds into shared memory (a heavy row costs one
// shared atomic per 32 entries, not one per edge).  Then the rows' update,
// contribution and residual.
__global__ void __launch_bounds__(kPbThreads, FPR_PB_MINB) pb_accum_kernel(const double* val, const uint16_t* dstl,
                                                              const int32_t* unit_bin, const int64_t* unit_e,
                                                              const int32_t* unit_k, int64_t nunits, int shift,
                                                              int32_t n, const int32_t* outdeg, double* pr,
                                                              double* cur, double base, double damping,
                                                              double* psum, unsigned int* bin_done,
                                                              unsigned long long* next_unit, double* cta_pairs) {
  constexpr int U = kLaneRun;
  extern __shared__ double acc[];
  const int R = 1 << shift;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
  const unsigned below = (2u << lane) - 1u;  // lanes 0..lane
  double lmax = 0.0, lsum = 0.0;
  __shared__ long long s_unit;
  __shared__ int s_last;
  for (;;) {
    if (threadIdx.x == 0) s_unit = (long long)atomicAdd(next_unit, 1ull);
    __syncthreads();
    const int64_t u = s_unit;
    if (u >= nunits) break;
    const int64_t b = __ldg(unit_bin + u);
    const int k = __ldg(unit_k + u);
    const int64_t e1 = __ldg(unit_e + u + 1);
    for (int i = threadIdx.x; i < R; i += blockDim.x) acc[i] = 0.0;
    __syncthreads();
    const int64_t r0 = b << shift;
    const int64_t r1 = min((int64_t)n, r0 + R);
    for (int64_t w = __ldg(unit_e + u) + (int64_t)warp * 32 * U; w < e1; w += (int64_t)nwarps * 32 * U) {
      double v[U];
      int d[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int64_t e = w + u * 32 + lane;
        const bool ok = e < e1;
        v[u] = ok ? __ldcs(val + e) : 0.0;
        d[u] = ok ? (int)__ldcs(dstl + e) : -1;
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const int key = d[u];
        double run = v[u];
        const int kprev = __shfl_up_sync(0xffffffffu, key, 1);
        const unsigned heads = __ballot_sync(0xffffffffu, lane == 0 || kprev != key);
        bool last = true;
        if (heads != 0xffffffffu) {
          const int seg0 = 31 - __clz(heads & below);
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const double t = __shfl_up_sync(0xffffffffu, run, o);
            if (lane - o >= seg0) run += t;
          }
          last = lane == 31 || ((heads >> (lane + 1)) & 1u);
        }
        if (key >= 0 && last) atomicAdd(&acc[key], run);
      }
    }
    __syncthreads();
    bool fin = true, from_psum = false;
    if (k > 1) {
      // a heavy bin split into k units: fold this unit's sums into psum; the
      // last unit to arrive finishes the bin's rows
      for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
        const double v = acc[r - r0];
        if (v != 0.0) atomicAdd(psum + r, v);
      }
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) s_last = atomicAdd(bin_done + b, 1u) == (unsigned)(k - 1);
      __syncthreads();
      fin = s_last;
      from_psum = true;
      if (fin) __threadfence();
    }
    if (fin) {
      for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
        double sum;
        if (from_psum) {
          sum = __ldcg(psum + r);
          psum[r] = 0.0;
        } else {
          sum = acc[r - r0];
        }
        const double nv = __dadd_rn(base, __dmul_rn(damping, sum));
        const double dd = fabs(nv - pr[r]);
        pr[r] = nv;
        const int od = __ldg(outdeg + r);
        if (od > 0) cur[r] = __ddiv_rn(nv, (double)od);
        lmax = fmax(lmax, dd);
        lsum += dd;
      }
      if (from_psum && threadIdx.x == 0) bin_done[b] = 0u;
    }
    __syncthreads();
  }
  __shared__ double sm[2][32];
  for (int o = 16; o > 0; o >>= 1) {
    lmax = fmax(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
    lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
  }
  if (lane == 0) {
    sm[0][warp] = lmax;
    sm[1][warp] = lsum;
  }
  __syncthreads();
  if (warp == 0) {
    lmax = lane < nwarps ? sm[0][lane] : 0.0;
    lsum = lane < nwarps ? sm[1][lane] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      lmax = fmax(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
      lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
    }
    if (lane == 0) {
      cta_pairs[2 * blockIdx.x] = lmax;
      cta_pairs[2 * blockIdx.x + 1] = lsum;
    }
  }
}

__global__ void pb_bin_edges_kernel(const int64_t* row, int32_t n, int shift, int64_t nbins, int64_t* be) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b <= nbins) be[b] = row[min((int64_t)n, b << shift)];
}

// Fixed-order reduction of the per-CTA pairs (one warp).
__global__ void pb_reduce_kernel(int nctas, const double* cta_pairs, double* err, double* l1) {
  double mx = 0.0, sm = 0.0;
  for (int i = threadIdx.x; i < nctas; i += 32) {
    mx = fmax(mx, cta_pairs[2 * i]);
    sm += cta_pairs[2 * i + 1];
  }
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    sm += __shfl_xor_sync(0xffffffffu, sm, o);
  }
  if (threadIdx.x == 0) {
    *err = mx;
    *l1 = sm;
  }
}

int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

#define PK(x)                       \
  do {                              \
    e = (x);                        \
    if (e != cudaSuccess) goto out; \
  } while (0)

}  // namespace

void free_pb(PbSet& pb, cudaStream_t st) {
  for (void* p : pb.allocs)
    if (p) cudaFreeAsync(p, st);
  pb = PbSet{};
}

cudaError_t build_pb(const DevGraph& g, int shift, int chunk_shift, cudaStream_t st, PbSet& pb, const char** msg) {
  cudaError_t e = cudaSuccess;
  *msg = nullptr;
  pb = PbSet{};
  const int sms = sm_count();
  const int64_t n = g.n, m = g.m;
  const int64_t nbins = n > 0 ? (n + (1ll << shift) - 1) >> shift : 0;
  const int64_t nchunks = std::max<int64_t>(1, (n + (1ll << chunk_shift) - 1) >> chunk_shift);
  const size_t hist_smem = (size_t)nchunks * sizeof(uint32_t);
  const size_t acc_smem = (size_t)sizeof(double) << shift;
  if (n == 0 || shift < 5 || shift > 14 || chunk_shift < 0 || chunk_shift > 31 || hist_smem > 160 * 1024 ||
      nbins * nchunks > (1ll << 31)) {
    *msg = "bin/chunk geometry out of range";
    return cudaSuccess;
  }
  auto alloc = [&](void** p, size_t bytes) {
    cudaError_t r = cudaMallocAsync(p, std::max<size_t>(bytes, 16), st);
    if (r == cudaSuccess) pb.allocs.push_back(*p);
    return r;
  };
  pb.shift = shift;
  pb.chunk_shift = chunk_shift;
  pb.nbins = nbins;
  pb.nchunks = nchunks;
  pb.m = m;
  PK(alloc((void**)&pb.counts, nbins * nchunks * sizeof(uint32_t)));
  PK(alloc((void**)&pb.start, nbins * nchunks * sizeof(int64_t)));
  PK(alloc((void**)&pb.src_bm, m * sizeof(int32_t)));
  PK(alloc((void**)&pb.dstl_bm, m * sizeof(uint16_t)));
  PK(alloc((void**)&pb.val, m * sizeof(double)));
  {
    int key_bits = 1;
    while ((1ll << key_bits) <= nchunks) ++key_bits;  // chunk ids and the sentinel nchunks
    PK(cudaFuncSetAttribute(pb_layout_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hist_smem));
    pb_layout_kernel<<<(unsigned)std::min<int64_t>(nbins, sms), kPbThreads, hist_smem, st>>>(
        g.row, g.src, g.n, shift, chunk_shift, key_bits, nbins, nchunks, pb.counts, pb.start, pb.src_bm,
        pb.dstl_bm);
    PK(cudaGetLastError());
  }
  {
    const int64_t nseg = nbins * nchunks;
    uint32_t* npieces = nullptr;
    uint32_t* piece_off = nullptr;
    void* temp = nullptr;
    size_t tb = 0;
    uint32_t last[2] = {0, 0};
    e = cudaMallocAsync(&npieces, nseg * sizeof(uint32_t), st);
    if (e == cudaSuccess) e = cudaMallocAsync(&piece_off, nseg * sizeof(uint32_t), st);
    if (e == cudaSuccess) {
      pb_piece_count_kernel<<<sms * 4, 256, 0, st>>>(pb.counts, nseg, npieces);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(nullptr, tb, npieces, piece_off, nseg, st);
    if (e == cudaSuccess) e = cudaMallocAsync(&temp, std::max<size_t>(tb, 16), st);
    if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(temp, tb, npieces, piece_off, nseg, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&last[0], piece_off + nseg - 1, 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(&last[1], npieces + nseg - 1, 4, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e == cudaSuccess) {
      pb.nitems = (int64_t)last[0] + last[1];
      e = alloc((void**)&pb.item_start, pb.nitems * sizeof(int64_t));
    }
    if (e == cudaSuccess) e = alloc((void**)&pb.item_len, pb.nitems * sizeof(uint32_t));
    if (e == cudaSuccess) {
      pb_piece_fill_kernel<<<sms * 4, 256, 0, st>>>(pb.counts, pb.start, piece_off, nseg, pb.item_start,
                                                     pb.item_len);
      e = cudaGetLastError();
    }
    for (void* q : {(void*)npieces, (void*)piece_off, temp})
      if (q) cudaFreeAsync(q, st);
    if (e != cudaSuccess) goto out;
  }
  {
    // phase-2 residency: the bin's accumulators in shared memory, 1024
    // threads per CTA (at most 2 CTAs per SM)
    const int by_smem = (int)std::max<size_t>(1, (size_t)(227 * 1024) / (acc_smem + 1024));
    pb.p2_grid = (int)std::min<int64_t>(nbins, (int64_t)sms * std::min(2, by_smem));
  }
  {
    // phase-2 units: bins, heavy ones cut into pieces of about `piece` entries
    std::vector<int64_t> be(nbins + 1);
    int64_t* d_be = nullptr;
    e = cudaMallocAsync(&d_be, (nbins + 1) * sizeof(int64_t), st);
    if (e == cudaSuccess) {
      pb_bin_edges_kernel<<<(unsigned)((nbins + 256) / 256), 256, 0, st>>>(g.row, g.n, shift, nbins, d_be);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(be.data(), d_be, (nbins + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (d_be) cudaFreeAsync(d_be, st);
    if (e != cudaSuccess) goto out;
    int64_t piece = std::max<int64_t>(1 << 16, m / ((int64_t)pb.p2_grid * 8));
    if (const char* v = std::getenv("FPR_B200_PB_PIECE")) piece = std::max<int64_t>(32, std::atoll(v));  // tests
    std::vector<int32_t> ubin, uk;
    std::vector<int64_t> ue;
    for (int64_t b = 0; b < nbins; ++b) {
      const int64_t E = be[b + 1] - be[b];
      const int64_t k = std::max<int64_t>(1, (E + piece - 1) / piece);
      for (int64_t j = 0; j < k; ++j) {
        ubin.push_back((int32_t)b);
        uk.push_back((int32_t)k);
        ue.push_back(be[b] + E * j / k);
      }
    }
    ue.push_back(m);
    pb.nunits = (int64_t)ubin.size();
    PK(alloc((void**)&pb.unit_bin, ubin.size() * sizeof(int32_t)));
    PK(alloc((void**)&pb.unit_k, uk.size() * sizeof(int32_t)));
    PK(alloc((void**)&pb.unit_e, ue.size() * sizeof(int64_t)));
    PK(cudaMemcpyAsync(pb.unit_bin, ubin.data(), ubin.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    PK(cudaMemcpyAsync(pb.unit_k, uk.data(), uk.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st));
    PK(cudaMemcpyAsync(pb.unit_e, ue.data(), ue.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st));
    PK(alloc((void**)&pb.psum, n * sizeof(double)));
    PK(cudaMemsetAsync(pb.psum, 0, n * sizeof(double), st));
    PK(alloc((void**)&pb.bin_done, nbins * sizeof(unsigned int)));
    PK(cudaMemsetAsync(pb.bin_done, 0, nbins * sizeof(unsigned int), st));
    PK(cudaStreamSynchronize(st));  // the host vectors die at the end of this block
  }
  PK(alloc((void**)&pb.next_item, 2 * sizeof(unsigned long long)));
  PK(alloc((void**)&pb.cta_pairs, 2 * (size_t)pb.p2_grid * sizeof(double)));
  PK(cudaFuncSetAttribute(pb_accum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)acc_smem));
  PK(cudaStreamSynchronize(st));
out:
  if (e != cudaSuccess) {
    free_pb(pb, st);
    cudaStreamSynchronize(st);
  }
  return e;
}

cudaError_t launch_pb_sweep(const PbSet& pb, const DevGraph& g, const double* prev, double* pr, double* cur,
                            double base, double damping, double* err, double* l1, cudaStream_t st) {
  cudaError_t e = cudaMemsetAsync(pb.next_item, 0, 2 * sizeof(unsigned long long), st);  // both work counters
  if (e != cudaSuccess) return e;
  if (pb.m > 0) {
    pb_gather_kernel<<<sm_count() * 8, kGatherThreads, 0, st>>>(pb.src_bm, pb.item_start, pb.item_len,
                                                                 pb.nitems, prev, pb.val, pb.next_item);
    e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  pb_accum_kernel<<<pb.p2_grid, kPbThreads, (size_t)sizeof(double) << pb.shift, st>>>(
      pb.val, pb.dstl_bm, pb.unit_bin, pb.unit_e, pb.unit_k, pb.nunits, pb.shift, g.n, g.outdeg, pr, cur, base,
      damping, pb.psum, pb.bin_done, pb.next_item + 1, pb.cta_pairs);
  e = cudaGetLastError();
  if (e != cudaSuccess) return e;
  pb_reduce_kernel<<<1, 32, 0, st>>>(pb.p2_grid, pb.cta_pairs, err, l1);
  return cudaGetLastError();
}

}  // namespace fprb
