// pb.cu -- propagation-blocked sweeps (FPR_B200_OPT_PB) for graphs whose
// contribution vector far exceeds L2 (configs 4/5): EC (Jacobi) and the
// lockstep FusEd schedule (waves of whole bins, in place).
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
//     segment (bin b, chunk c) is contiguous and keeps ascending rows;
//   * entry = (source id, row offset inside the bin as uint16).
// A sweep plan (get_pb_plan, cached per wave count) cuts the bins into waves
// of consecutive bins: 1 wave for EC, S for lockstep.  Per wave:
//   * phase 1 (pb_gather_kernel): warps walk the wave's segments chunk by
//     chunk, so the sources read at any moment span one chunk's
//     contributions (a 16 MB window at the default chunk of 2^21 sources),
//     and write val[pos] = prev[src_bm[pos]] contiguously;
//   * phase 2 (pb_accum_kernel): CTAs accumulate val into a bin's rows in
//     shared memory and finish the rows exactly like the blocked engine's
//     apply (blocked.cu): base + d*sum without FMA, contribution, residual.
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
// phase 2 shape: entries per lane, threads per CTA, CTAs per SM (shared
// memory permitting); EPL 4 x 1024 x 2 measured best
#ifndef FPR_PB_EPL
#define FPR_PB_EPL 4
#endif
#ifndef FPR_PB_ACC_THREADS
#define FPR_PB_ACC_THREADS 1024
#endif
#ifndef FPR_PB_ACC_CTAS
#define FPR_PB_ACC_CTAS 2
#endif
// phase 1 gathers: L1-allocating (default: hub sources recur across the bins a
// CTA walks in one chunk, 4-6% faster on configs 4/5) or L2-only (0)
#ifndef FPR_PB_GATHER_L1
#define FPR_PB_GATHER_L1 1
#endif

// One CTA per bin: histogram its edges by source chunk, scan, then a stable
// scatter (tiles of the bin's CSR edges, block radix-sorted by chunk) so each
// (bin, chunk) segment lists its entries in ascending row order -- phase 2
// folds runs of one row before touching shared memory.  counts/start are
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
  extern __shared__ uint32_t h[];           // nchunks chunk counters, then
  uint32_t* srow = h + ((nchunks + 3) & ~3ll);  // the bin's row offsets relative to its first edge
  const int tid = threadIdx.x;
  const uint32_t sentinel = (uint32_t)nchunks;
  for (int64_t b = blockIdx.x; b < nbins; b += gridDim.x) {
    for (int64_t c = tid; c < nchunks; c += blockDim.x) h[c] = 0;
    const int64_t r0 = b << shift;
    const int64_t r1 = min((int64_t)n, r0 + ((int64_t)1 << shift));
    const int64_t e0 = row[r0], e1 = row[r1];
    for (int64_t r = r0 + tid; r <= r1; r += blockDim.x) srow[r - r0] = (uint32_t)(__ldg(row + r) - e0);
    __syncthreads();
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
        // row of edge e: last r in [0, r1 - r0) with srow[r] <= e - e0
        const uint32_t el = (uint32_t)(e - e0);
        int lo = 0, hi = (int)(r1 - r0) - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (srow[mid] <= el) lo = mid;
          else hi = mid - 1;
        }
        const uint32_t s = (uint32_t)__ldg(src + e);
        key[0] = s >> chunk_shift;
        val[0] = ((uint64_t)s << 16) | (uint64_t)lo;
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

// Plan order: position p walks the waves (runs of consecutive bins), chunk-
// major inside a wave, so each wave's pieces are contiguous and in chunk
// order.  Returns the chunk-major segment index c * nbins + b of position p.
__device__ __forceinline__ int64_t pb_seg_of(int64_t p, const int64_t* wave_bin, int nwaves, int64_t nbins,
                                             int64_t nchunks) {
  int lo = 0, hi = nwaves - 1;  // last wave w with wave_bin[w] * nchunks <= p
  while (lo < hi) {
    const int mid = (lo + hi + 1) >> 1;
    if (wave_bin[mid] * nchunks <= p) lo = mid;
    else hi = mid - 1;
  }
  const int64_t b0 = wave_bin[lo], nb = wave_bin[lo + 1] - b0;
  const int64_t q = p - b0 * nchunks;
  const int64_t c = q / nb;
  return c * nbins + b0 + (q - c * nb);
}

__global__ void pb_piece_count_kernel(const uint32_t* counts, int64_t nseg, const int64_t* wave_bin, int nwaves,
                                      int64_t nbins, int64_t nchunks, uint32_t* npieces) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nseg; p += stride)
    npieces[p] = (counts[pb_seg_of(p, wave_bin, nwaves, nbins, nchunks)] + kPieceEntries - 1) / kPieceEntries;
}

__global__ void pb_piece_fill_kernel(const uint32_t* counts, const int64_t* start, const uint32_t* piece_off,
                                     int64_t nseg, const int64_t* wave_bin, int nwaves, int64_t nbins,
                                     int64_t nchunks, int64_t* item_start, uint32_t* item_len) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nseg; p += stride) {
    const int64_t s = pb_seg_of(p, wave_bin, nwaves, nbins, nchunks);
    const uint32_t cnt = counts[s];
    const int64_t p0 = start[s];
    uint32_t o = piece_off[p];
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
      for (int u = 0; u < U; ++u) v[u] = s[u] >= 0 ? (FPR_PB_GATHER_L1 ? __ldca(prev + s[u]) : __ldcg(prev + s[u])) : 0.0;
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
// the average on config 3).  Lane L of a warp step owns EPL consecutive
// entries, read as 32-B value vectors and one key vector.  It
// folds runs of equal rows in registers; runs strictly inside the lane go to
// shared memory at once.  The run that ends the lane (its "tail") may
// continue in the next lanes: one segmented warp scan of the tails per
// 32*EPL entries carries it, and each run is added exactly once, by the lane
// where it ends (its first part, if it began in earlier lanes, arrives in
// the carry).  Shared fp64 adds are CAS loops on sm_100.  The first form of
// this pass scanned every 32 entries across the warp; its shuffles were ~60%
// of the L1TEX data-pipe wavefronts, the pass's limiter.
// Then each finished row: base + d*sum without FMA, contribution, residual.
template <int EPL>
__device__ __forceinline__ void pb_ld_vals(const double* p, double (&v)[EPL]) {
#pragma unroll
  for (int j = 0; j < EPL; j += 4)
    asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];"
                 : "=d"(v[j]), "=d"(v[j + 1]), "=d"(v[j + 2]), "=d"(v[j + 3])
                 : "l"(p + j));
}
template <int EPL>
__device__ __forceinline__ void pb_ld_keys(const uint16_t* p, uint32_t (&k)[EPL / 2]) {
  if constexpr (EPL == 4) {
    asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];" : "=r"(k[0]), "=r"(k[1]) : "l"(p));
  } else {
    static_assert(EPL == 8, "EPL is 4 or 8");
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(k[0]), "=r"(k[1]), "=r"(k[2]), "=r"(k[3])
                 : "l"(p));
  }
}

template <int EPL, int THREADS, int MINB>
__global__ void __launch_bounds__(THREADS, MINB) pb_accum_kernel(
    const double* val, const uint16_t* dstl, const int32_t* unit_bin, const int64_t* unit_e, const int32_t* unit_k,
    int64_t nunits, int shift, int32_t n, const int32_t* outdeg, double* pr, double* cur, double base,
    double damping, double* psum, unsigned int* bin_done, unsigned long long* next_unit, double* cta_pairs) {
  extern __shared__ double acc[];
  constexpr int W = 32 * EPL;  // entries per warp step
  const int R = 1 << shift;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nwarps = blockDim.x >> 5;
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
    const int64_t e0 = __ldg(unit_e + u), e1 = __ldg(unit_e + u + 1);
    for (int i = threadIdx.x; i < R; i += blockDim.x) acc[i] = 0.0;
    __syncthreads();
    const int64_t r0 = b << shift;
    const int64_t r1 = min((int64_t)n, r0 + R);
    for (int64_t w = (e0 & ~int64_t(EPL - 1)) + (int64_t)warp * W; w < e1; w += (int64_t)nwarps * W) {
      const int64_t e = w + lane * EPL;
      double v[EPL];
      uint32_t kw[EPL / 2];
      if (e < e1) {
        pb_ld_vals<EPL>(val + e, v);
        pb_ld_keys<EPL>(dstl + e, kw);
      } else {
#pragma unroll
        for (int j = 0; j < EPL / 2; ++j) kw[j] = 0xFFFFFFFFu;
#pragma unroll
        for (int j = 0; j < EPL; ++j) v[j] = 0.0;
      }
      // fold: first run (fk, fs), current run (ck, cs); interior runs go out
      int fk = -2, ck = -2;
      double fs = 0.0, cs = 0.0;
      bool multi = false;
#pragma unroll
      for (int i = 0; i < EPL; ++i) {
        const uint32_t raw = (kw[i >> 1] >> (16 * (i & 1))) & 0xFFFFu;
        const int ki = (e + i >= e0 && e + i < e1) ? (int)raw : -1;
        if (i == 0) {
          ck = ki;
          cs = v[0];
        } else if (ki == ck) {
          cs += v[i];
        } else {
          if (!multi) {
            fk = ck;
            fs = cs;
            multi = true;
          } else if (ck >= 0) {
            atomicAdd(&acc[ck], cs);  // a run strictly inside this lane
          }
          ck = ki;
          cs = v[i];
        }
      }
      if (!multi) {
        fk = ck;
        fs = cs;
      }
      // carry the tails: lane L continues lane L-1's tail if its first key
      // equals that tail's key; a single-run continuing lane passes it on
      const int pk = __shfl_up_sync(0xffffffffu, ck, 1);
      const bool cont = lane > 0 && fk >= 0 && fk == pk;
      const bool through = cont && !multi;
      const unsigned starts = __ballot_sync(0xffffffffu, !through);
      double S = cs;
      if (starts != 0xffffffffu) {
        const unsigned below = (2u << lane) - 1u;
        const int seg0 = 31 - __clz(starts & below);
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const double t = __shfl_up_sync(0xffffffffu, S, o);
          if (lane - o >= seg0) S += t;
        }
      }
      const double Sp = __shfl_up_sync(0xffffffffu, S, 1);
      const bool next_cont = __shfl_down_sync(0xffffffffu, cont, 1) && lane < 31;
      if (multi && fk >= 0) atomicAdd(&acc[fk], cont ? fs + Sp : fs);  // the first run ends in this lane
      if (!next_cont && ck >= 0) atomicAdd(&acc[ck], S);                // the tail run ends here
    }
    __syncthreads();
    bool fin = true, from_psum = false;
    if (k > 1) {
      for (int64_t r = r0 + threadIdx.x; r < r1; r += blockDim.x) {
        const double x = acc[r - r0];
        if (x != 0.0) atomicAdd(psum + r, x);
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
  for (auto& kv : pb.plans)
    for (void* p : kv.second.allocs)
      if (p) cudaFreeAsync(p, st);
  for (void* p : pb.allocs)
    if (p) cudaFreeAsync(p, st);
  pb = PbSet{};
}

// Edge-balanced waves: wave w starts at the first bin whose edges begin at or
// after w/S of all edges (skewed and crawl-ordered graphs put most edges in
// their first bins; vertex-balanced waves gave config 3's BFS order almost
// no Gauss-Seidel gain).  Empty waves are dropped.
std::vector<int64_t> pb_wave_bins(const std::vector<int64_t>& bin_edge, uint32_t S) {
  const int64_t nbins = (int64_t)bin_edge.size() - 1;
  const int64_t m = bin_edge.back();
  std::vector<int64_t> wb{0};
  for (uint32_t w = 1; w < S; ++w) {
    const int64_t target = (int64_t)((double)m * w / S);
    const int64_t b = std::lower_bound(bin_edge.begin(), bin_edge.end() - 1, target) - bin_edge.begin();
    if (b > wb.back() && b < nbins) wb.push_back(b);
  }
  wb.push_back(nbins);
  return wb;
}

cudaError_t pb_bin_edges(const DevGraph& g, int shift, cudaStream_t st, std::vector<int64_t>* out) {
  const int64_t nbins = ((int64_t)g.n + (1ll << shift) - 1) >> shift;
  std::vector<int64_t> be(nbins + 1);
  int64_t* d_be = nullptr;
  cudaError_t e = cudaMallocAsync(&d_be, (nbins + 1) * sizeof(int64_t), st);
  if (e == cudaSuccess) {
    pb_bin_edges_kernel<<<(unsigned)((nbins + 256) / 256), 256, 0, st>>>(g.row, g.n, shift, nbins, d_be);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cudaMemcpyAsync(be.data(), d_be, (nbins + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (d_be) cudaFreeAsync(d_be, st);
  if (e == cudaSuccess) *out = std::move(be);
  return e;
}

cudaError_t get_pb_plan(PbSet& pb, uint32_t S, cudaStream_t st, const PbPlan** out) {
  auto it = pb.plans.find(S);
  if (it != pb.plans.end()) {
    *out = &it->second;
    return cudaSuccess;
  }
  const int sms = sm_count();
  PbPlan plan;
  plan.wave_bin = pb_wave_bins(pb.bin_edge, S);
  plan.nwaves = (int)plan.wave_bin.size() - 1;
  const int W = plan.nwaves;
  const int64_t nbins = pb.nbins, nchunks = pb.nchunks, nseg = nbins * nchunks;
  auto alloc = [&](void** p, size_t bytes) {
    cudaError_t r = cudaMallocAsync(p, std::max<size_t>(bytes, 16), st);
    if (r == cudaSuccess) plan.allocs.push_back(*p);
    return r;
  };
  uint32_t* npieces = nullptr;
  uint32_t* piece_off = nullptr;
  int64_t* d_wb = nullptr;
  void* temp = nullptr;
  size_t tb = 0;
  std::vector<uint32_t> off(W + 1, 0);
  uint32_t last = 0;
  cudaError_t e = cudaMallocAsync(&npieces, nseg * sizeof(uint32_t), st);
  if (e == cudaSuccess) e = cudaMallocAsync(&piece_off, nseg * sizeof(uint32_t), st);
  if (e == cudaSuccess) e = cudaMallocAsync(&d_wb, (W + 1) * sizeof(int64_t), st);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_wb, plan.wave_bin.data(), (W + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st);
  if (e == cudaSuccess) {
    pb_piece_count_kernel<<<sms * 4, 256, 0, st>>>(pb.counts, nseg, d_wb, W, nbins, nchunks, npieces);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(nullptr, tb, npieces, piece_off, nseg, st);
  if (e == cudaSuccess) e = cudaMallocAsync(&temp, std::max<size_t>(tb, 16), st);
  if (e == cudaSuccess) e = cub::DeviceScan::ExclusiveSum(temp, tb, npieces, piece_off, nseg, st);
  for (int w = 1; w < W && e == cudaSuccess; ++w)
    e = cudaMemcpyAsync(&off[w], piece_off + plan.wave_bin[w] * nchunks, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&off[W], piece_off + nseg - 1, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaMemcpyAsync(&last, npieces + nseg - 1, 4, cudaMemcpyDeviceToHost, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e == cudaSuccess) {
    off[W] += last;
    plan.item0.assign(off.begin(), off.end());
    e = alloc((void**)&plan.item_start, off[W] * sizeof(int64_t));
  }
  if (e == cudaSuccess) e = alloc((void**)&plan.item_len, off[W] * sizeof(uint32_t));
  if (e == cudaSuccess) {
    pb_piece_fill_kernel<<<sms * 4, 256, 0, st>>>(pb.counts, pb.start, piece_off, nseg, d_wb, W, nbins, nchunks,
                                                   plan.item_start, plan.item_len);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = alloc((void**)&plan.ctr, 2 * (size_t)W * sizeof(unsigned long long));
  if (e == cudaSuccess) e = alloc((void**)&plan.cta_pairs, 2 * (size_t)W * pb.p2_grid * sizeof(double));
  for (void* q : {(void*)npieces, (void*)piece_off, (void*)d_wb, temp})
    if (q) cudaFreeAsync(q, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    for (void* q : plan.allocs) cudaFreeAsync(q, st);
    cudaStreamSynchronize(st);
    return e;
  }
  {
    // phase-2 units: bins, heavy ones cut into pieces of about `piece`
    // entries: small enough that each wave has several units per CTA, never
    // below twice the average bin (a split bin pays psum atomics per row;
    // splitting config 4's even bins cost 5-10%)
    const int64_t avg_bin = pb.m / std::max<int64_t>(1, pb.nbins);
    int64_t piece = std::max<int64_t>({int64_t(1) << 16, 2 * avg_bin, pb.m / ((int64_t)pb.p2_grid * 8 * W)});
    if (const char* v = std::getenv("FPR_B200_PB_PIECE")) piece = std::max<int64_t>(32, std::atoll(v));  // tests
    std::vector<int32_t> ubin, uk;
    std::vector<int64_t> ue;
    plan.unit0.assign(W + 1, 0);
    for (int w = 0; w < W; ++w) {
      plan.unit0[w] = (int64_t)ubin.size();
      for (int64_t b = plan.wave_bin[w]; b < plan.wave_bin[w + 1]; ++b) {
        const int64_t E = pb.bin_edge[b + 1] - pb.bin_edge[b];
        const int64_t k = std::max<int64_t>(1, (E + piece - 1) / piece);
        for (int64_t j = 0; j < k; ++j) {
          ubin.push_back((int32_t)b);
          uk.push_back((int32_t)k);
          ue.push_back(pb.bin_edge[b] + E * j / k);
        }
      }
    }
    plan.unit0[W] = (int64_t)ubin.size();
    ue.push_back(pb.m);
    e = alloc((void**)&plan.unit_bin, ubin.size() * sizeof(int32_t));
    if (e == cudaSuccess) e = alloc((void**)&plan.unit_k, uk.size() * sizeof(int32_t));
    if (e == cudaSuccess) e = alloc((void**)&plan.unit_e, ue.size() * sizeof(int64_t));
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(plan.unit_bin, ubin.data(), ubin.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(plan.unit_k, uk.data(), uk.size() * sizeof(int32_t), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(plan.unit_e, ue.data(), ue.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // the host vectors die at the end of this block
    if (e != cudaSuccess) {
      for (void* q : plan.allocs) cudaFreeAsync(q, st);
      cudaStreamSynchronize(st);
      return e;
    }
  }
  *out = &pb.plans.emplace(S, std::move(plan)).first->second;
  return cudaSuccess;
}

cudaError_t build_pb(const DevGraph& g, int shift, int chunk_shift, cudaStream_t st, PbSet& pb, const char** msg) {
  cudaError_t e = cudaSuccess;
  *msg = nullptr;
  pb = PbSet{};
  const int sms = sm_count();
  const int64_t n = g.n, m = g.m;
  const int64_t nbins = n > 0 ? (n + (1ll << shift) - 1) >> shift : 0;
  const int64_t nchunks = std::max<int64_t>(1, (n + (1ll << chunk_shift) - 1) >> chunk_shift);
  // layout kernel: chunk counters + the bin's (2^shift + 1) relative row offsets
  const size_t hist_smem = ((size_t)(nchunks + 3) & ~(size_t)3) * sizeof(uint32_t) +
                           (((size_t)1 << std::min(shift, 20)) + 1) * sizeof(uint32_t);
  const size_t acc_smem = (size_t)sizeof(double) << shift;
  if (n == 0 || shift < 5 || shift > 14 || chunk_shift < 0 || chunk_shift > 31 || hist_smem > 192 * 1024 ||
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
  // 8 pad entries: the lane-sequential phase 2 loads 8-entry vectors that may
  // run past the end
  PK(alloc((void**)&pb.dstl_bm, (m + 8) * sizeof(uint16_t)));
  PK(alloc((void**)&pb.val, (m + 8) * sizeof(double)));
  {
    // bin edge offsets (host copy: wave plans cut waves and phase-2 units)
    std::vector<int64_t> be;
    e = pb_bin_edges(g, shift, st, &be);
    if (e != cudaSuccess) goto out;
    pb.bin_edge = be;
    for (int64_t b = 0; b < nbins; ++b)
      if (be[b + 1] - be[b] >= (1ll << 32)) {  // the layout kernel's uint32 in-bin offsets
        *msg = "a bin holds 2^32 or more edges (use a smaller FPR_B200_PB_SHIFT)";
        break;
      }
    if (*msg) goto out;
  }
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
    // phase-2 residency: the bin's accumulators in shared memory,
    // FPR_PB_ACC_CTAS CTAs per SM when they fit
    const int by_smem = (int)std::max<size_t>(1, (size_t)(227 * 1024) / (acc_smem + 1024));
    pb.p2_grid = (int)std::min<int64_t>(nbins, (int64_t)sms * std::min(FPR_PB_ACC_CTAS, by_smem));
    pb.p1_grid = sms * 8;
  }
  {
    PK(alloc((void**)&pb.psum, n * sizeof(double)));
    PK(cudaMemsetAsync(pb.psum, 0, n * sizeof(double), st));
    PK(alloc((void**)&pb.bin_done, nbins * sizeof(unsigned int)));
    PK(cudaMemsetAsync(pb.bin_done, 0, nbins * sizeof(unsigned int), st));
  }
  PK(cudaFuncSetAttribute(pb_accum_kernel<FPR_PB_EPL, FPR_PB_ACC_THREADS, FPR_PB_ACC_CTAS>,
                          cudaFuncAttributeMaxDynamicSharedMemorySize, (int)acc_smem));
  PK(cudaStreamSynchronize(st));
out:
  if (e != cudaSuccess || *msg) {
    free_pb(pb, st);
    cudaStreamSynchronize(st);
  }
  return e;
}

cudaError_t launch_pb_sweep(const PbSet& pb, const PbPlan& plan, const DevGraph& g, const double* prev, double* pr,
                            double* cur, double base, double damping, double* err, double* l1, cudaStream_t st) {
  const int W = plan.nwaves;
  // work counters: [0, W) phase-1 pieces, [W, 2W) phase-2 units
  cudaError_t e = cudaMemsetAsync(plan.ctr, 0, 2 * (size_t)W * sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  for (int w = 0; w < W; ++w) {
    const int64_t i0 = plan.item0[w], u0 = plan.unit0[w];
    if (plan.item0[w + 1] > i0) {
      pb_gather_kernel<<<pb.p1_grid, kGatherThreads, 0, st>>>(pb.src_bm, plan.item_start + i0, plan.item_len + i0,
                                                              plan.item0[w + 1] - i0, prev, pb.val, plan.ctr + w);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    pb_accum_kernel<FPR_PB_EPL, FPR_PB_ACC_THREADS, FPR_PB_ACC_CTAS>
        <<<pb.p2_grid, FPR_PB_ACC_THREADS, (size_t)sizeof(double) << pb.shift, st>>>(
            pb.val, pb.dstl_bm, plan.unit_bin + u0, plan.unit_e + u0, plan.unit_k + u0, plan.unit0[w + 1] - u0,
            pb.shift,
            g.n, g.outdeg, pr, cur, base, damping, pb.psum, pb.bin_done, plan.ctr + W + w,
            plan.cta_pairs + 2 * (size_t)w * pb.p2_grid);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  pb_reduce_kernel<<<1, 32, 0, st>>>(W * pb.p2_grid, plan.cta_pairs, err, l1);
  return cudaGetLastError();
}

}  // namespace fprb
