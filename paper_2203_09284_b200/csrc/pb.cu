// pb.cu -- propagation-blocked sweeps for graphs whose contribution vector
// far exceeds L2 (configs 4/5; picked by default there, FPR_B200_OPT_PB /
// FPR_B200_OPT_PULL force the choice): EC (Jacobi) and the lockstep FusEd
// schedule (waves of whole bins, in place).
//
// The pull gather contrib[in_src[e]] misses L2 on such graphs, and each miss
// pulls ~64 B from HBM for 8 useful bytes (profiles/r1_large_configs_ncu.md).
// Propagation blocking (Beamer, Asanovic, Patterson, "Reducing PageRank
// communication via propagation blocking", IPDPS'17) trades the random reads
// for streams.
//
// Layout, built once from the resident in-CSR:
//   * rows are cut into bins of 2^shift consecutive rows; a bin's entries are
//     exactly its rows' in-edges, stored from an 8-aligned position bin_pos[b];
//   * inside a bin, entries are regrouped by source chunk (src >> chunk_shift):
//     segment (bin b, chunk c) is contiguous and keeps the CSR order (rows
//     ascending, a row's sources ascending);
//   * a run = the consecutive entries of one row inside one segment piece
//     (kPieceEntries entries from the segment start); its last entry carries
//     a close flag (bit 31 of the source).  Each run is ONE partial sum;
//     runs are numbered bin by bin from an 8-aligned pbin_pos[b];
//   * a bin's runs are cut into tiles of kTile; per tile, vidx[] lists the
//     runs in the tile's (stable) row order, and skey[] holds the row offset
//     of every sorted place (accumulate side).
// A sweep plan (get_pb_plan, cached per wave count) cuts the bins into waves
// of consecutive bins: 1 wave for EC, S for lockstep.  Per wave:
//   * phase 1 (pb_gather_kernel): warps walk the wave's segment pieces chunk
//     by chunk, so the sources read at any moment span one chunk's
//     contributions (a 64 MB window at the default chunk of 2^23 sources);
//     they gather every entry's contribution, sum each run left to right
//     (a segmented warp scan across lanes) and write its partial sum;
//   * phase 2 (pb_accum_kernel): a CTA takes a bin (or a run of tiles of a
//     heavy bin), streams each tile into shared memory (TMA bulk copies),
//     reads it in row order, sums every row's places and adds them to the
//     bin's row accumulators with ONE plain add per row and tile -- no
//     atomics, a fixed order -- then finishes the rows: base + d*sum without
//     FMA, contribution, residual.
// Per edge and sweep: 4 B source read; per run: 8 B partial sum written and
// read back + 2 B vidx + 2 B key, all sequential, where a missed pull gather
// moved ~64 B of DRAM.  R-MAT puts a row's in-edges from one chunk next to
// each other often enough that config 5 has ~0.25 runs per edge.  A row's
// sum is a fixed regrouping of the reference's left-to-right sum (runs in
// chunk order, i.e. ascending sources), so every run gives the same bits,
// within 1e-12 per iteration of the reference (tests/test_gpu_engines.py
// test_pb_*, tests/test_gpu_fullsize.py).  Measurements and rejected
// variants: DESIGN.md §3.4.
//
// Kernels, in the order they run:
//   layout  pb_piece_hist_kernel, pb_bin_scan_kernel, pb_layout_kernel
//           (segments), pb_close_count_kernel, pb_psum_kernel (runs),
//           pb_hot_threshold/bits/rank/src/rewrite_kernel (hot copy),
//           pb_tile_sort_kernel (accumulate tiles); per wave count:
//           pb_piece_count/fill_kernel (gather plan);
//   sweep   pb_hot_refresh_kernel, pb_gather_kernel, pb_accum_kernel per
//           wave, then pb_reduce_kernel.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdlib>
#include <cstdint>
#include <vector>

#include "internal.cuh"

namespace fprb {

namespace {

#ifndef FPR_PB_LAYOUT_THREADS
#define FPR_PB_LAYOUT_THREADS 1024
#endif
constexpr int kPbThreads = FPR_PB_LAYOUT_THREADS;  // layout kernel CTA (several CTAs per SM when smaller)
constexpr int64_t kSplitMaxChunks = 256;  // layout: multi-split fast path up to this many source chunks
#ifndef FPR_PB_TSORT_BITS
#define FPR_PB_TSORT_BITS 5  // tile sort radix digit: 14-bit keys in 3 passes
#endif
constexpr int kGatherThreads = 256;

constexpr int kPieceEntries = 1024;  // phase-1 work item: up to this many entries of one segment
// phase 2: CTAs of kAccThreads, kAccEpl sorted entries per lane, one tile
// (kTile = kAccThreads * kAccEpl entries) per CTA step; the bin's fp64 row
// accumulators (64 KB at 2^13 rows) + kStages staged tiles (24 KB each) fit
// two CTAs per SM
#ifndef FPR_PB_ACC_THREADS
#define FPR_PB_ACC_THREADS 512
#endif
#ifndef FPR_PB_EPL
#define FPR_PB_EPL 4
#endif
#ifndef FPR_PB_STAGES
#define FPR_PB_STAGES 2
#endif
constexpr int kAccThreads = FPR_PB_ACC_THREADS;
constexpr int kAccEpl = FPR_PB_EPL;  // sorted places per lane (4 or 8)
#ifndef FPR_PB_ACC_CTAS
#define FPR_PB_ACC_CTAS 2
#endif
constexpr int kAccCtas = FPR_PB_ACC_CTAS;  // phase-2 CTAs per SM (at most; shared memory permitting)
constexpr int kTile = kAccThreads * kAccEpl;
constexpr int kStages = FPR_PB_STAGES;  // tiles per CTA staged ahead (TMA bulk copies)

static_assert(kAccEpl == 4 || kAccEpl == 8, "kAccEpl is 4 or 8");

static_assert(kTile <= 65536, "perm is uint16");
constexpr uint16_t kPadKey = 0xFFFF;  // row offset of a pad entry (bins hold < 2^16 rows)
// gather-pass source words: bit 31 closes a run, bit 30 marks a hot source
// (the low 30 bits then name its slot in the dense hot copy)
constexpr uint32_t kHotBit = 0x40000000u, kIdMask = 0x3FFFFFFFu;
// phase 1 gathers: L1-allocating (default: hub sources recur across the bins a
// CTA walks in one chunk, 4-6% faster on configs 4/5) or L2-only (0)
#ifndef FPR_PB_GATHER_L1
#define FPR_PB_GATHER_L1 1
#endif

// The layout works on PIECES of a bin's CSR edges (kLayoutPiece edges; a
// bin's last piece is shorter, an empty bin is one empty piece), so that the
// few bins holding the hub rows (config 5's first bin: ~70 M edges) spread
// over many CTAs instead of one CTA walking them alone.
constexpr int64_t kLayoutPiece = int64_t(1) << 18;

__device__ __forceinline__ int64_t pb_bin_edge_end(const int64_t* row, int32_t n, int shift, int64_t b) {
  return row[min((int64_t)n, (b + 1) << shift)];
}

// Pass 1: per piece, the histogram of its edges' source chunks (four loads in
// flight per thread, one shared atomic per distinct chunk of a warp).
__global__ void __launch_bounds__(kPbThreads) pb_piece_hist_kernel(const int64_t* row, const int32_t* src, int32_t n,
                                                                    int shift, int chunk_shift, int64_t nchunks,
                                                                    const int32_t* piece_bin, const int64_t* piece_e,
                                                                    int64_t npieces, uint32_t* phist) {
  extern __shared__ uint32_t h[];
  const int tid = threadIdx.x;
  const uint32_t sentinel = (uint32_t)nchunks;
  for (int64_t pc = blockIdx.x; pc < npieces; pc += gridDim.x) {
    for (int64_t c = tid; c < nchunks; c += kPbThreads) h[c] = 0;
    __syncthreads();
    const int64_t b = piece_bin[pc], es = piece_e[pc];
    const int64_t ee = (pc + 1 < npieces && piece_bin[pc + 1] == b) ? piece_e[pc + 1] : pb_bin_edge_end(row, n, shift, b);
    for (int64_t eb = es; eb < ee; eb += 4 * (int64_t)kPbThreads) {
      uint32_t c4[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int64_t e = eb + k * kPbThreads + tid;
        c4[k] = e < ee ? ((uint32_t)__ldg(src + e) >> chunk_shift) : sentinel;
      }
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const unsigned peers = __match_any_sync(0xffffffffu, c4[k]);
        if (c4[k] != sentinel && __ffs(peers) - 1 == (tid & 31)) atomicAdd(&h[c4[k]], (uint32_t)__popc(peers));
      }
    }
    __syncthreads();
    for (int64_t c = tid; c < nchunks; c += kPbThreads) phist[pc * nchunks + c] = h[c];
    __syncthreads();
  }
}

// Pass 2, per bin: its segments' sizes and starts (chunk-major counts/start:
// an exclusive scan over the chunks from the bin's 8-aligned position), and
// each piece's starting cursor per chunk (the earlier pieces' counts added).
__global__ void __launch_bounds__(kPbThreads) pb_bin_scan_kernel(const int64_t* bin_pos, int64_t nbins, int64_t nchunks,
                                                                  const int64_t* bin_piece0, const uint32_t* phist,
                                                                  uint32_t* counts, int64_t* start, uint32_t* pcur) {
  using ScanU = cub::BlockScan<uint32_t, kPbThreads>;
  __shared__ typename ScanU::TempStorage tmp;
  for (int64_t b = blockIdx.x; b < nbins; b += gridDim.x) {
    const int64_t q0 = bin_piece0[b], q1 = bin_piece0[b + 1];
    uint32_t running = 0;
    for (int64_t t0 = 0; t0 < nchunks; t0 += kPbThreads) {
      const int64_t c = t0 + threadIdx.x;
      uint32_t tot = 0;
      if (c < nchunks)
        for (int64_t pc = q0; pc < q1; ++pc) tot += phist[pc * nchunks + c];
      uint32_t x, tile;
      ScanU(tmp).ExclusiveSum(tot, x, tile);
      if (c < nchunks) {
        counts[c * nbins + b] = tot;
        start[c * nbins + b] = bin_pos[b] + running + x;
        uint32_t cur = running + x;
        for (int64_t pc = q0; pc < q1; ++pc) {
          pcur[pc * nchunks + c] = cur;
          cur += phist[pc * nchunks + c];
        }
      }
      running += tile;
      __syncthreads();
    }
  }
}

// Pass 3, per piece: a stable scatter of the piece's edges (tiles of
// kPbThreads CSR edges, multi-split by chunk) from each chunk's cursor, so
// every (bin, chunk) segment lists its entries in CSR order (rows ascending,
// a row's sources ascending) -- the pieces of a bin fill disjoint ranges of
// each segment in piece order.  The bin's last piece also writes its pad
// entries (source -1, key kPadKey, up to bin_pos[b + 1]).
__global__ void __launch_bounds__(kPbThreads) pb_layout_kernel(const int64_t* row, const int32_t* src, int32_t n,
                                                                int shift, int chunk_shift, int key_bits,
                                                                int64_t nchunks, const int64_t* bin_pos,
                                                                const int32_t* piece_bin, const int64_t* piece_e,
                                                                int64_t npieces, const uint32_t* pcur,
                                                                int32_t* src_bm, uint16_t* dstl_bm) {
  using Sort = cub::BlockRadixSort<uint32_t, kPbThreads, 1, uint64_t>;
  using ScanI = cub::BlockScan<int, kPbThreads>;
  __shared__ union {
    typename Sort::TempStorage sort;
    typename ScanI::TempStorage scani;
  } tmp;
  __shared__ uint32_t skey[kPbThreads];
  __shared__ int s_rcur;
  extern __shared__ uint32_t h[];           // nchunks chunk cursors, then
  uint32_t* srow = h + ((nchunks + 3) & ~3ll);  // the bin's row offsets relative to its first edge
  const int tid = threadIdx.x;
  const uint32_t sentinel = (uint32_t)nchunks;
  for (int64_t pc = blockIdx.x; pc < npieces; pc += gridDim.x) {
    const int64_t b = piece_bin[pc];
    const bool last = !(pc + 1 < npieces && piece_bin[pc + 1] == b);
    const int64_t r0 = b << shift;
    const int64_t r1 = min((int64_t)n, r0 + ((int64_t)1 << shift));
    const int64_t e0 = row[r0], e1 = row[r1];
    const int64_t es = piece_e[pc], ee = last ? e1 : piece_e[pc + 1];
    const int64_t p0 = bin_pos[b];
    if (last)
      for (int64_t q = p0 + (e1 - e0) + tid; q < bin_pos[b + 1]; q += kPbThreads) {
        src_bm[q] = -1;
        dstl_bm[q] = kPadKey;
      }
    for (int64_t c = tid; c < nchunks; c += kPbThreads) h[c] = pcur[pc * nchunks + c];
    const int nrows = (int)(r1 - r0);
    for (int64_t r = r0 + tid; r <= r1; r += kPbThreads) srow[r - r0] = (uint32_t)(__ldg(row + r) - e0);
    __syncthreads();
    // the row holding the piece's first edge: the last row starting at or
    // before it (-1 at a bin start: the tile's own marks find it)
    if (tid == 0) {
      int rc = -1;
      if (es > e0) {
        const uint32_t ps = (uint32_t)(es - e0);
        int lo = 0, hi = nrows - 1;
        while (lo < hi) {
          const int mid = (lo + hi + 1) >> 1;
          if (srow[mid] <= ps) lo = mid;
          else hi = mid - 1;
        }
        rc = lo;
      }
      s_rcur = rc;
    }
    __syncthreads();
    int rcur = s_rcur;  // row holding the current CSR tile's first edge (carried across tiles)
    uint32_t s_next = es + tid < ee ? (uint32_t)__ldg(src + es + tid) : 0u;  // prefetched one tile ahead
    for (int64_t t = es; t < ee; t += kPbThreads) {
      const int64_t e = t + tid;
      const uint32_t s_cur = s_next;
      if (e + kPbThreads < ee) s_next = (uint32_t)__ldg(src + e + kPbThreads);
      // row of every edge of the tile: each row that starts inside the tile
      // marks its first position (empty rows share the next row's start, so
      // the max wins), then one block max-scan fills the positions between
      const uint32_t ts = (uint32_t)(t - e0), te = ts + kPbThreads;
      skey[tid] = 0;
      __syncthreads();
      for (int r = rcur + 1 + tid; r < nrows; r += kPbThreads) {
        const uint32_t sr = srow[r];
        if (sr >= te) break;
        if (sr >= ts) atomicMax(&skey[sr - ts], (uint32_t)(r + 1));  // +1: 0 = no mark
      }
      __syncthreads();
      int rowp = (int)skey[tid] - 1;
      if (tid == 0 && rowp < rcur) rowp = rcur;
      ScanI(tmp.scani).InclusiveScan(rowp, rowp, cub::Max());
      __syncthreads();
      if (tid == kPbThreads - 1) skey[0] = (uint32_t)rowp;
      __syncthreads();
      rcur = (int)skey[0];
      __syncthreads();
      if (nchunks <= kSplitMaxChunks) {
        // stable multi-split by chunk (the common geometry: <= 256 chunks):
        // rank among equal chunks inside the warp from match.any, warps'
        // counts scanned per chunk in warp order, positions from the
        // chunk's running cursor h[] -- no radix passes
        const int lane = tid & 31, warp = tid >> 5;
        uint32_t* wcnt = srow + (((int64_t)1 << min(shift, 20)) + 1);  // (nchunks + 1) x 32 counts
        const uint32_t ck = e < ee ? (s_cur >> chunk_shift) : sentinel;
        const uint32_t sv = e < ee ? s_cur : 0u;
        for (int64_t i = tid; i < (nchunks + 1) * 32; i += kPbThreads) wcnt[i] = 0;
        __syncthreads();
        const unsigned peers = __match_any_sync(0xffffffffu, ck);
        const int rank = __popc(peers & ((1u << lane) - 1u));
        if (rank == 0) wcnt[ck * 32 + warp] = (uint32_t)__popc(peers);
        __syncthreads();
        // warp w scans chunks w, w + 32, ...: lane = warp index of the tile
        for (int64_t c = warp; c <= nchunks; c += kPbThreads / 32) {
          const uint32_t v = wcnt[c * 32 + lane];
          uint32_t x = v;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
            if (lane >= o) x += y;
          }
          wcnt[c * 32 + lane] = x - v;  // exclusive prefix over the warps
          if (lane == 31 && c < nchunks) skey[c] = x;  // the tile's count of chunk c (skey is free here)
        }
        __syncthreads();
        if (ck != sentinel) {
          const int64_t pos = p0 + h[ck] + wcnt[ck * 32 + warp] + rank;
          src_bm[pos] = (int32_t)sv;
          dstl_bm[pos] = (uint16_t)rowp;
        }
        __syncthreads();
        for (int64_t c = tid; c < nchunks; c += kPbThreads) h[c] += skey[c];
        __syncthreads();
        continue;
      }
      uint32_t key[1] = {sentinel};
      uint64_t val[1] = {0};
      if (e < ee) {
        const uint32_t sx = s_cur;
        key[0] = sx >> chunk_shift;
        val[0] = ((uint64_t)sx << 16) | (uint64_t)rowp;
      }
      Sort(tmp.sort).Sort(key, val, 0, key_bits);
      __syncthreads();
      skey[tid] = key[0];
      __syncthreads();
      int hs = (tid == 0 || skey[tid - 1] != key[0]) ? tid : 0;
      ScanI(tmp.scani).InclusiveScan(hs, hs, cub::Max());
      const bool real = key[0] != sentinel;
      if (real) {
        const int64_t pos = p0 + h[key[0]] + (tid - hs);
        src_bm[pos] = (int32_t)(val[0] >> 16);
        dstl_bm[pos] = (uint16_t)(val[0] & 0xFFFFu);
      }
      __syncthreads();
      if (real && (tid == kPbThreads - 1 || skey[tid + 1] != key[0])) h[key[0]] += (uint32_t)(tid - hs + 1);
      __syncthreads();
    }
    __syncthreads();
  }
}

// Row partial sums.  A segment lists its entries in row order, so the edges
// of one row from one source chunk are neighbours: the gather pass sums them
// as it fetches them and writes ONE partial sum per (segment, row) run
// instead of one value per edge (config 5: 0.137 partial sums per edge).  An
// entry closes its run when it is the bin's last real entry, the next entry
// starts another chunk or row, or it ends its piece (pieces are the gather
// pass's work items: kPieceEntries entries from the segment's start, so no
// run spans two of them).  Pads close nothing.  The sources are read with
// the close flag (bit 31) masked: pb_psum_kernel sets it in place.
// Close mask of the 8 entries [q, q + 8) (q 8-aligned; entries at or past
// pe are pads, never closing); s/d receive their sources (flag masked) and
// row offsets.
__device__ __forceinline__ unsigned pb_close_mask8(const int32_t* src, const uint16_t* dstl, const int64_t* start,
                                                   int64_t q, int64_t pe, int64_t b, int64_t nbins,
                                                   int chunk_shift, uint32_t (&s)[8], uint32_t (&d)[8]) {
  const int4 a0 = *reinterpret_cast<const int4*>(src + q), a1 = *reinterpret_cast<const int4*>(src + q + 4);
  const uint4 dv = *reinterpret_cast<const uint4*>(dstl + q);
  s[0] = (uint32_t)a0.x, s[1] = (uint32_t)a0.y, s[2] = (uint32_t)a0.z, s[3] = (uint32_t)a0.w;
  s[4] = (uint32_t)a1.x, s[5] = (uint32_t)a1.y, s[6] = (uint32_t)a1.z, s[7] = (uint32_t)a1.w;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    s[j] &= 0x7FFFFFFFu;
    d[j] = (j & 1) ? ((&dv.x)[j >> 1] >> 16) : ((&dv.x)[j >> 1] & 0xFFFFu);
  }
  uint32_t s8 = 0, d8 = 0;
  if (q + 8 < pe) {
    s8 = (uint32_t)src[q + 8] & 0x7FFFFFFFu;
    d8 = dstl[q + 8];
  }
  unsigned m = 0;
  uint32_t cprev = 0xFFFFFFFFu;
  int64_t ss = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    if (q + j >= pe) break;
    const uint32_t c = s[j] >> chunk_shift;
    if (c != cprev) {
      ss = __ldg(start + (int64_t)c * nbins + b);
      cprev = c;
    }
    bool cl = q + j + 1 >= pe;
    if (!cl) {
      const uint32_t sn = j < 7 ? s[j + 1] : s8, dn = j < 7 ? d[j + 1] : d8;
      cl = (sn >> chunk_shift) != c || dn != d[j] || (q + j - ss + 1) % kPieceEntries == 0;
    }
    if (cl) m |= 1u << j;
  }
  return m;
}

// Pass A: the number of runs (partial sums) of each bin.
__global__ void __launch_bounds__(kAccThreads) pb_close_count_kernel(const int32_t* src, const uint16_t* dstl,
                                                                     const int64_t* row, int32_t n, int shift,
                                                                     const int64_t* bin_pos, const int64_t* start,
                                                                     int64_t nbins, int chunk_shift, int64_t* bin_np) {
  using Reduce = cub::BlockReduce<uint32_t, kAccThreads>;
  __shared__ typename Reduce::TempStorage tmp;
  for (int64_t b = blockIdx.x; b < nbins; b += gridDim.x) {
    const int64_t r0 = b << shift, r1 = min((int64_t)n, r0 + ((int64_t)1 << shift));
    const int64_t p0 = bin_pos[b], pe = p0 + (row[r1] - row[r0]);
    uint32_t c = 0;
    for (int64_t q = p0 + 8 * (int64_t)threadIdx.x; q < pe; q += 8 * kAccThreads) {
      uint32_t sv[8], dv[8];
      c += __popc(pb_close_mask8(src, dstl, start, q, pe, b, nbins, chunk_shift, sv, dv));
    }
    c = Reduce(tmp).Sum(c);
    if (threadIdx.x == 0) bin_np[b] = (int64_t)c;
    __syncthreads();
  }
}

// The slot of source s (chunk * kc + rank) if it is hot, else -1.
__device__ __forceinline__ int32_t pb_hot_slot(const uint32_t* bits, const uint32_t* wpre, uint32_t s,
                                               int chunk_shift, int64_t kc) {
  const uint32_t word = __ldg(bits + (s >> 5));
  const uint32_t bit = 1u << (s & 31u);
  if (!(word & bit)) return -1;
  const uint32_t rank = __ldg(wpre + (s >> 5)) + (uint32_t)__popc(word & (bit - 1u));
  if (rank >= (uint64_t)kc) return -1;
  return (int32_t)((int64_t)(s >> chunk_shift) * kc + rank);
}

// Pass B, per bin (its runs numbered from pbin_pos[b], an 8-aligned position,
// so that the accumulate's tile copies stay 16-B aligned):
//   * closing entries get bit 31 of their source set (the gather's flag);
//   * pkey[u] = the row offset of run u; the bin's pad places get kPadKey;
//   * every piece start q records the number of its first run in
//     pbase[seg_piece0[segment] + piece]: the runs closed before q in the
//     bin, since q's run closes at or after q.
// Threads take 8 consecutive entries (32-B source words, 16-B row offsets).
__global__ void __launch_bounds__(kAccThreads) pb_psum_kernel(int32_t* src, const uint16_t* dstl, const int64_t* row,
                                                              int32_t n, int shift, const int64_t* bin_pos,
                                                              const int64_t* pbin_pos, const int64_t* start,
                                                              const uint32_t* seg_piece0, int64_t nbins,
                                                              int chunk_shift, uint16_t* pkey, int64_t* pbase) {
  using Scan = cub::BlockScan<uint32_t, kAccThreads>;
  __shared__ typename Scan::TempStorage tmp;
  for (int64_t b = blockIdx.x; b < nbins; b += gridDim.x) {
    const int64_t r0 = b << shift, r1 = min((int64_t)n, r0 + ((int64_t)1 << shift));
    const int64_t p0 = bin_pos[b], pe = p0 + (row[r1] - row[r0]);
    int64_t u = pbin_pos[b];
    for (int64_t t = p0; t < pe; t += 8 * kAccThreads) {
      const int64_t q = t + 8 * (int64_t)threadIdx.x;
      uint32_t sv[8], dv[8];
      const unsigned m = q < pe ? pb_close_mask8(src, dstl, start, q, pe, b, nbins, chunk_shift, sv, dv) : 0u;
      uint32_t before, total;
      Scan(tmp).ExclusiveSum((uint32_t)__popc(m), before, total);
      if (q < pe) {
        uint32_t cprev = 0xFFFFFFFFu;
        int64_t ss = 0, seg = 0;
        uint32_t k = before;  // runs closed before entry q + j in the bin
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (q + j >= pe) break;
          const uint32_t c = sv[j] >> chunk_shift;
          if (c != cprev) {
            seg = (int64_t)c * nbins + b;
            ss = __ldg(start + seg);
            cprev = c;
          }
          const int64_t off = q + j - ss;
          if (off % kPieceEntries == 0) pbase[(int64_t)__ldg(seg_piece0 + seg) + off / kPieceEntries] = u + k;
          if (m >> j & 1u) {
            pkey[u + k] = (uint16_t)dv[j];
            ++k;
          }
        }
        // the gather's word: the source with the close flag in bit 31 (the
        // threads of this tile have all read their neighbours' sources: the
        // scan above synchronised)
        uint32_t ww[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) ww[j] = sv[j] | (((m >> j) & 1u) << 31);
        int4 w0, w1;
        w0.x = (int)ww[0], w0.y = (int)ww[1], w0.z = (int)ww[2], w0.w = (int)ww[3];
        w1.x = (int)ww[4], w1.y = (int)ww[5], w1.z = (int)ww[6], w1.w = (int)ww[7];
        // pads past pe keep their -1 (never read by the gather pass)
        if (q + 8 <= pe) {
          *reinterpret_cast<int4*>(src + q) = w0;
          *reinterpret_cast<int4*>(src + q + 4) = w1;
        } else {
          for (int j = 0; j < 8 && q + j < pe; ++j) src[q + j] = (int32_t)ww[j];
        }
      }
      u += total;
      __syncthreads();
    }
    for (int64_t k = u + threadIdx.x; k < pbin_pos[b + 1]; k += kAccThreads) pkey[k] = kPadKey;
  }
}

// Pass C, per tile (kTile consecutive runs from pbin_pos[b]; the bin's last
// tile is shorter): the stable sort of the tile's runs by row --
// skey[t0 + j] = row offset at sorted place j (kPadKey for pads, which sort
// last), vidx[t0 + j] = the tile index of sorted place j's run; tile_meta[g]
// = t0 << 16 | len (the accumulate stages the tile's runs from t0).
__global__ void __launch_bounds__(kAccThreads) pb_tile_sort_kernel(const uint16_t* pkey, const int64_t* pbin_pos,
                                                                   const int64_t* tile_off, int64_t nbins, int shift,
                                                                   uint16_t* vidx, uint16_t* skey,
                                                                   uint64_t* tile_meta) {
  using Sort = cub::BlockRadixSort<uint32_t, kAccThreads, kAccEpl, uint32_t, FPR_PB_TSORT_BITS>;
  __shared__ typename Sort::TempStorage tmp;
  const uint32_t pad_key = 1u << shift;
  for (int64_t b = blockIdx.x; b < nbins; b += gridDim.x) {
    const int64_t p0 = pbin_pos[b], p1 = pbin_pos[b + 1];
    int64_t g = tile_off[b];
    for (int64_t t0 = p0; t0 < p1; t0 += kTile, ++g) {
      const int len = (int)min((int64_t)kTile, p1 - t0);
      if (threadIdx.x == 0) tile_meta[g] = ((uint64_t)t0 << 16) | (uint64_t)len;
      uint32_t key[kAccEpl], idx[kAccEpl];
#pragma unroll
      for (int j = 0; j < kAccEpl; ++j) {
        const int i = threadIdx.x * kAccEpl + j;
        // rows < 2^shift; pads sort after them, places past the tile last:
        // shift + 1 key bits (radix passes) instead of 17
        const uint32_t d = i < len ? (uint32_t)pkey[t0 + i] : 0x10000u;
        key[j] = d == 0x10000u ? (pad_key + 1) : (d == kPadKey ? pad_key : d);
        idx[j] = (uint32_t)i;
      }
      Sort(tmp).Sort(key, idx, 0, shift + 1);
#pragma unroll
      for (int j = 0; j < kAccEpl; ++j) {
        const int p = threadIdx.x * kAccEpl + j;
        if (p < len) {
          skey[t0 + p] = key[j] == pad_key ? kPadKey : (uint16_t)key[j];
          vidx[t0 + p] = (uint16_t)idx[j];
        }
      }
      __syncthreads();
    }
  }
}

// Pieces of each segment (kPieceEntries entries from its start).
__global__ void pb_seg_pieces_kernel(const uint32_t* counts, int64_t nseg, uint32_t* np) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nseg; s += stride)
    np[s] = (counts[s] + kPieceEntries - 1) / kPieceEntries;
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
                                     const uint32_t* seg_piece0, const int64_t* pbase, int64_t nseg,
                                     const int64_t* wave_bin, int nwaves, int64_t nbins, int64_t nchunks,
                                     int64_t* item_start, uint32_t* item_len, int64_t* item_ubase) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < nseg; p += stride) {
    const int64_t s = pb_seg_of(p, wave_bin, nwaves, nbins, nchunks);
    const uint32_t cnt = counts[s];
    const int64_t p0 = start[s];
    uint32_t o = piece_off[p];
    const int64_t* pb0 = pbase + seg_piece0[s];
    for (uint32_t k = 0; k < cnt; k += kPieceEntries, ++o) {
      item_start[o] = p0 + k;
      item_len[o] = min((uint32_t)kPieceEntries, cnt - k);
      item_ubase[o] = pb0[k / kPieceEntries];
    }
  }
}

// Phase 1: warps take pieces in chunk order from a global counter (static
// striding lets fast warps drift chunks ahead and the concurrently read
// contribution window outgrow L2).  A piece is a run of one segment's
// entries in row order; the pass fetches every entry's contribution and sums
// each row's run as it goes, writing one partial sum per run (closing
// entries carry bit 31 of their source) to consecutive places from the
// piece's first run number.  Lane L owns 8 consecutive entries per step (one
// 32-B source load, eight gathers in flight): it sums its entries left to
// right, one segmented warp scan of the lanes' open tails carries a run
// across lanes (with the plain prefix of the lanes' closing counts: the
// output places), and lane 31's open tail carries it into the next step.
// The grouping is fixed by the layout, so the bits are the same on every run.
#ifndef FPR_PB_GATHER_MINB
#define FPR_PB_GATHER_MINB 4
#endif
#ifndef FPR_PB_HOT
#define FPR_PB_HOT 8192  // hot sources per chunk with a dense copy (0 = none)
#endif
constexpr int64_t kHot = FPR_PB_HOT;
__global__ void __launch_bounds__(kGatherThreads, FPR_PB_GATHER_MINB) pb_gather_kernel(
    const int32_t* esrc, const int64_t* item_start, const uint32_t* item_len, const int64_t* item_ubase,
    int64_t nitems, const double* prev, const double* hot, double* psum, unsigned long long* next_item,
    const unsigned int* gate) {
  if (gate && *reinterpret_cast<const volatile unsigned int*>(gate)) return;  // stopped: no-op sweep
  const int lane = threadIdx.x & 31;
  const int32_t idmask = hot ? (int32_t)kIdMask : 0x7FFFFFFF;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  for (;;) {
    unsigned long long it = 0;
    if (lane == 0) it = atomicAdd(next_item, 1ull);
    it = __shfl_sync(0xffffffffu, it, 0);
    if ((int64_t)it >= nitems) break;
    const int64_t p0 = __ldg(item_start + it);
    const int64_t p1 = p0 + __ldg(item_len + it);
    int64_t ub = __ldg(item_ubase + it);  // the next run's number (warp-uniform)
    double carry = 0.0;                   // the run left open by the previous step
    for (int64_t q0 = p0 & ~int64_t(7); q0 < p1; q0 += 256) {
      const int64_t qb = q0 + 8 * lane;
      // this lane's entries inside the piece: bits [jlo, jhi)
      const int jlo = (int)max((int64_t)0, min((int64_t)8, p0 - qb));
      const int jhi = (int)max((int64_t)0, min((int64_t)8, p1 - qb));
      const unsigned okm = ((1u << jhi) - 1u) & ~((1u << jlo) - 1u);
      int s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
      if (okm)
        asm volatile(
            "ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
            : "=r"(s[0]), "=r"(s[1]), "=r"(s[2]), "=r"(s[3]), "=r"(s[4]), "=r"(s[5]), "=r"(s[6]), "=r"(s[7])
            : "l"(esrc + qb), "l"(pol));
      double v[8];
      unsigned clm = 0;  // bit j: entry j closes its run
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        v[j] = 0.0;
        if (okm >> j & 1u) {
          // a hot source (bit 30) is read from the dense per-sweep copy of its
          // chunk's hot contributions: its L1 lines hold only hub values.
          // Without a hot copy (source spaces past 2^30) bit 30 is an id bit.
          const double* a = (hot && (s[j] & kHotBit)) ? hot + (s[j] & kIdMask) : prev + (s[j] & idmask);
          v[j] = FPR_PB_GATHER_L1 ? __ldca(a) : __ldcg(a);
          if (s[j] < 0) clm |= 1u << j;
        }
      }
      // the partial of the lane's first closed run, and its open tail
      double run = 0.0, F = 0.0;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        run = run + v[j];
        if (clm >> j & 1u) {
          if ((clm & ((1u << j) - 1u)) == 0u) F = run;
          run = 0.0;
        }
      }
      const bool h = clm != 0u;
      const int c = __popc(clm);
      double S = run;
      if (lane == 0 && !h) S = carry + S;
      // segmented inclusive scan of the tails (restarting at closing lanes)
      // and the inclusive prefix of the closing counts
      bool f = h;
      int C = c;
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        const double t = __shfl_up_sync(0xffffffffu, S, d);
        const bool g = __shfl_up_sync(0xffffffffu, f, d);
        const int y = __shfl_up_sync(0xffffffffu, C, d);
        if (lane >= d) {
          C += y;
          if (!f) {
            S = t + S;
            f = g;
          }
        }
      }
      double ci = __shfl_up_sync(0xffffffffu, S, 1);  // the run entering this lane
      if (lane == 0) ci = carry;
      carry = __shfl_sync(0xffffffffu, S, 31);
      const int total = __shfl_sync(0xffffffffu, C, 31);
      if (h) {
        int64_t k = ub + (C - c);
        run = 0.0;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          run = run + v[j];
          if (clm >> j & 1u) {
            __stcs(psum + k, (clm & ((1u << j) - 1u)) == 0u ? ci + F : run);
            ++k;
            run = 0.0;
          }
        }
      }
      ub += total;
    }
  }
}

// Hot sources (layout): each source's frequency among the entries, a
// threshold per chunk so that about kc = min(kHot, chunk size) of its sources
// reach it (and at least 2 entries each), and slots for up to kc of them;
// their entries get bit 30 and the slot (chunk * kc + k) in place of the
// source.  Any choice
// is exact: a hot copy holds the same double as the vector.
__global__ void pb_src_hist_kernel(const int32_t* esrc, int64_t mpad, uint32_t* cnt) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; q < mpad; q += stride) {
    const int32_t e = __ldg(esrc + q);
    if (e != -1) atomicAdd(cnt + ((uint32_t)e & 0x7FFFFFFFu), 1u);
  }
}

constexpr int kHotBins = 4096;
__global__ void __launch_bounds__(1024) pb_hot_threshold_kernel(const uint32_t* cnt, int64_t nsrc, int chunk_shift,
                                                                int64_t kc, uint32_t* thr) {
  __shared__ uint32_t hist[kHotBins];
  const int64_t c = blockIdx.x;
  for (int i = threadIdx.x; i < kHotBins; i += blockDim.x) hist[i] = 0;
  __syncthreads();
  const int64_t s0 = c << chunk_shift, s1 = min(nsrc, (c + 1) << chunk_shift);
  for (int64_t s = s0 + threadIdx.x; s < s1; s += blockDim.x) {
    const uint32_t k = __ldg(cnt + s);
    if (k >= 2) atomicAdd(&hist[min(k, (uint32_t)kHotBins - 1)], 1u);
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    // the smallest t >= 2 whose sources (count >= t) fit kc slots, else the top bin
    uint32_t above = 0, t = kHotBins - 1;
    for (int v = kHotBins - 1; v >= 2; --v) {
      if (above + hist[v] > (uint32_t)kc) break;
      above += hist[v];
      t = (uint32_t)v;
    }
    thr[c] = t;
  }
}

// The hot set as a bitmap (1 bit per source: 32 MB at config 5, L2-resident
// while the run-numbering pass looks it up per entry) plus, per 32-bit word,
// the hot sources before it in its chunk: a source's slot is its rank among
// its chunk's hot sources (ascending ids), the first kc of them are hot.
__global__ void pb_hot_bits_kernel(const uint32_t* cnt, int64_t nsrc, int chunk_shift, const uint32_t* thr,
                                   uint32_t* bits) {
  const int64_t nw = (nsrc + 31) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t wstride = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t w = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5; w < nw; w += wstride) {
    const int64_t s = (w << 5) + lane;
    const bool hot = s < nsrc && __ldg(cnt + s) >= __ldg(thr + (s >> chunk_shift));
    const unsigned word = __ballot_sync(0xffffffffu, hot);
    if (lane == 0) bits[w] = word;
  }
}

// One CTA per chunk: exclusive prefix of the hot counts over the chunk's words.
__global__ void __launch_bounds__(1024) pb_hot_rank_kernel(const uint32_t* bits, int64_t nsrc, int chunk_shift,
                                                           uint32_t* wpre) {
  using Scan = cub::BlockScan<uint32_t, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  const int64_t w0 = ((int64_t)blockIdx.x << chunk_shift) >> 5;
  const int64_t w1 = min((nsrc + 31) >> 5, (((int64_t)blockIdx.x + 1) << chunk_shift) >> 5);
  uint32_t running = 0;
  for (int64_t t = w0; t < w1; t += 1024) {
    const int64_t w = t + threadIdx.x;
    const uint32_t c = w < w1 ? (uint32_t)__popc(__ldg(bits + w)) : 0u;
    uint32_t x, tot;
    Scan(tmp).ExclusiveSum(c, x, tot);
    if (w < w1) wpre[w] = running + x;
    running += tot;
    __syncthreads();
  }
}

__global__ void pb_hot_src_kernel(const uint32_t* bits, const uint32_t* wpre, int64_t nsrc, int chunk_shift,
                                  int64_t kc, int32_t* hot_src) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t s = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < nsrc; s += stride) {
    const int32_t sl = pb_hot_slot(bits, wpre, (uint32_t)s, chunk_shift, kc);
    if (sl >= 0) hot_src[sl] = (int32_t)s;
  }
}

// Entries of hot sources: bit 30 + the slot in place of the source (the
// close flag kept); four words per thread, many lookups in flight.
__global__ void pb_hot_rewrite_kernel(int32_t* esrc, int64_t mpad, const uint32_t* bits, const uint32_t* wpre,
                                      int chunk_shift, int64_t kc) {
  const int64_t n4 = mpad >> 2;  // mpad is a multiple of 8
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    int4 w = reinterpret_cast<const int4*>(esrc)[i];
    int* x = &w.x;
    bool any = false;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      if (x[j] == -1) continue;  // pad
      const int32_t sl = pb_hot_slot(bits, wpre, (uint32_t)x[j] & 0x7FFFFFFFu, chunk_shift, kc);
      if (sl >= 0) {
        x[j] = (int32_t)(((uint32_t)x[j] & 0x80000000u) | kHotBit | (uint32_t)sl);
        any = true;
      }
    }
    if (any) reinterpret_cast<int4*>(esrc)[i] = w;
  }
}

// Per wave, before its gather pass: the dense copy of every hot source's
// current contribution (in place for the lockstep schedule, so the copy sees
// the earlier waves' updates, as the vector does).
__global__ void pb_hot_refresh_kernel(const int32_t* hot_src, int64_t nslots, const double* prev, double* hot,
                                      const unsigned int* gate) {
  if (gate && *reinterpret_cast<const volatile unsigned int*>(gate)) return;  // stopped: no-op sweep
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nslots; i += stride) {
    const int32_t s = __ldg(hot_src + i);
    if (s >= 0) hot[i] = __ldcg(prev + s);
  }
}

// Per bin, its rows with in-edges (row offsets, ascending) for the
// accumulate's finalize once rows without in-edges are settled.
__global__ void __launch_bounds__(1024) pb_live_rows_kernel(const int64_t* row, int32_t n, int shift, int64_t nbins,
                                                            uint16_t* live_rows, int32_t* live_cnt) {
  using Scan = cub::BlockScan<int, 1024>;
  __shared__ typename Scan::TempStorage tmp;
  for (int64_t b = blockIdx.x; b < nbins; b += gridDim.x) {
    const int64_t r0 = b << shift, r1 = min((int64_t)n, r0 + ((int64_t)1 << shift));
    int base = 0;
    for (int64_t t = r0; t < r1; t += 1024) {
      const int64_t r = t + threadIdx.x;
      const int live = (r < r1 && __ldg(row + r + 1) > __ldg(row + r)) ? 1 : 0;
      int x, tot;
      Scan(tmp).ExclusiveSum(live, x, tot);
      if (live) live_rows[(b << shift) + base + x] = (uint16_t)(r - r0);
      base += tot;
      __syncthreads();
    }
    if (threadIdx.x == 0) live_cnt[b] = base;
  }
}

// Phase 2: CTAs take work units from a counter: a unit is a whole bin, or a
// run of tiles of a heavy bin (skewed graphs put a large share of the edges
// in the bins of the hub rows; one CTA per bin left one SM working 7x longer
// than the average on config 3).  Per tile:
//   * thread 0 streams the tile's partial sums, inverse permutation and sorted
//     keys into a shared-memory stage with three TMA bulk copies completing
//     on the stage's mbarrier, kStages tiles ahead;
//   * lane L owns the sorted places [4L, 4L+4): it reads their keys and,
//     through vidx, their partial sums from the stage, folds
//     runs of equal rows in registers, and one segmented warp scan of the
//     lane tails carries a run across lanes to the lane where it ends, so
//     each run inside the warp is summed exactly once, in a fixed order.
//     Sorted, a row's places are contiguous: its run is unique in the tile,
//     so the row accumulator takes one PLAIN add (runs of different rows
//     touch different words).  A run that crosses warp boundaries leaves a
//     piece per warp in shared memory; the lane where it ends waits for the
//     earlier warps' pieces (per-tile flags) and adds them in warp order;
//   * one CTA barrier ends the tile (every add landed, the stage free).
// Tiles of a unit, and the units of a split bin (slots summed in unit
// order by the last one to finish), follow each other in a fixed order, so
// the row sums -- and the ranks -- are the same bits on every run
// (SPEC.md:415).  The first form of this pass added every run with a
// shared-memory fp64 CAS in arrival order (not reproducible); a fixed-point
// integer accumulator made it reproducible but cost 45% more per sweep
// (DESIGN.md §3.4).  Then each finished row: base + d*sum without FMA,
// contribution, residual; the bin's (max, sum) residual pair is reduced in a
// fixed thread order and the bins' pairs in bin order (pb_reduce_kernel).
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
// Tile streams are read once: evict-first in L2, so that a gather pass
// running beside this accumulate keeps its contribution window resident.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar, uint64_t pol) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
      ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(pol)
      : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}"
      ::"r"(smem_u32(bar)), "r"(parity)
      : "memory");
}

struct alignas(16) PbStage {
  double v[kTile + 2];   // the tile's partial sums (staged from an even run number)
  uint16_t ip[kTile];    // stage index of each sorted place's value
  uint16_t k[kTile];     // row offset of each sorted place
};

__global__ void __launch_bounds__(kAccThreads, kAccCtas) pb_accum_kernel(
    const double* val, const uint16_t* vidx, const uint16_t* skey, const uint64_t* tile_meta, const int32_t* unit_bin,
    const int64_t* unit_e, const int64_t* unit_t, const int32_t* unit_k, const int32_t* unit_j,
    const int32_t* unit_slot, int64_t nunits, int shift, int32_t n,
    const int32_t* outdeg, const double* pr, double* pr_out, double* cur, PbPeers peers, double base,
    double damping, double* slots, unsigned int* bin_done, unsigned long long* next_unit, double* bin_pairs,
    const unsigned int* gate, const uint16_t* live_rows, const int32_t* live_cnt) {
  if (gate && *reinterpret_cast<const volatile unsigned int*>(gate)) return;  // stopped: no-op sweep
  constexpr int NW = kAccThreads / 32;
  constexpr int WE = 32 * kAccEpl;  // sorted places per warp
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int R = 1 << shift;
  PbStage* stage = reinterpret_cast<PbStage*>(smem_raw);
  double* acc = reinterpret_cast<double*>(smem_raw + kStages * sizeof(PbStage));  // the bin's R rows
  __shared__ __align__(8) uint64_t bar[kStages];
  // crossing-run pieces of the current tile: warp w's first run continuing
  // from warp w-1 (A; thruA: it also continues into warp w+1) and its last
  // run continuing into warp w+1 (B); flag[w] = tile counter once posted
  __shared__ volatile double pA[NW], pB[NW];
  __shared__ volatile int kA[NW], kB[NW], thruA[NW];
  __shared__ volatile unsigned flag[NW];
  __shared__ long long s_unit;
  __shared__ int s_last;
  __shared__ double s_pair[2][NW];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(bar + s);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (threadIdx.x < NW) flag[threadIdx.x] = 0xFFFFFFFFu;
  __syncthreads();
  uint32_t tc = 0;  // tiles this CTA consumed so far: stage tc % kStages, parity (tc / kStages) & 1
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  // tile meta = first run << 16 | runs: the partial sums are staged from the
  // even index below the first (16-B aligned copy), rounded up to pairs
  auto issue = [&](uint32_t tile_no, uint64_t meta, int64_t t0, int len) {
    PbStage& st = stage[tile_no % kStages];
    const int64_t u0 = (int64_t)(meta >> 16);
    const uint32_t a = (uint32_t)(u0 & 1), vb = ((uint32_t)(meta & 0xFFFFu) + a + 1u) / 2u * 16u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    mbar_expect_tx(bar + tile_no % kStages, vb + (uint32_t)len * 4u);
    bulk_g2s(st.v, val + (u0 - a), vb, bar + tile_no % kStages, pol);
    bulk_g2s(st.ip, vidx + t0, (uint32_t)len * 2u, bar + tile_no % kStages, pol);
    bulk_g2s(st.k, skey + t0, (uint32_t)len * 2u, bar + tile_no % kStages, pol);
  };
  for (;;) {
    if (threadIdx.x == 0) s_unit = (long long)atomicAdd(next_unit, 1ull);
    __syncthreads();
    const int64_t u = s_unit;
    if (u >= nunits) break;
    const int64_t b = __ldg(unit_bin + u);
    const int k = __ldg(unit_k + u);
    const int64_t e0 = __ldg(unit_e + 2 * u), e1 = __ldg(unit_e + 2 * u + 1);  // whole tiles from the bin's start
    const int ntiles = (int)((e1 - e0 + kTile - 1) / kTile);
    const uint64_t* meta = tile_meta + __ldg(unit_t + u);  // this unit's tiles
    uint64_t mnext = 0;  // thread 0: meta of the next tile to issue, loaded a tile ahead
    if (threadIdx.x == 0) {
      for (int i = 0; i < kStages && i < ntiles; ++i)
        issue(tc + i, __ldg(meta + i), e0 + (int64_t)i * kTile, (int)min((int64_t)kTile, e1 - e0 - (int64_t)i * kTile));
      if (kStages < ntiles) mnext = __ldg(meta + kStages);
    }
    for (int i = threadIdx.x; i < R; i += kAccThreads) acc[i] = 0.0;
    __syncthreads();
    for (int ti = 0; ti < ntiles; ++ti, ++tc) {
      const int len = (int)min((int64_t)kTile, e1 - e0 - (int64_t)ti * kTile);
      const PbStage& st = stage[tc % kStages];
      mbar_wait(bar + tc % kStages, (tc / kStages) & 1u);
      const int i0 = threadIdx.x * kAccEpl;
      // keys before and after this warp's places (-2: none / pad)
      int pk = -2, nk = -2;
      {
        const int w0 = warp * WE, w1 = w0 + WE;
        if (w0 > 0 && w0 < len && st.k[w0 - 1] != kPadKey) pk = st.k[w0 - 1];
        if (w1 < len && st.k[w1] != kPadKey) nk = st.k[w1];
      }
      int kk[kAccEpl];
      double x[kAccEpl];
      if (i0 < len) {
        uint32_t kr[kAccEpl / 2], ir[kAccEpl / 2];
        if constexpr (kAccEpl == 4) {
          const uint2 kw = *reinterpret_cast<const uint2*>(st.k + i0);
          const uint2 iw = *reinterpret_cast<const uint2*>(st.ip + i0);
          kr[0] = kw.x, kr[1] = kw.y, ir[0] = iw.x, ir[1] = iw.y;
        } else {
          const uint4 kw = *reinterpret_cast<const uint4*>(st.k + i0);
          const uint4 iw = *reinterpret_cast<const uint4*>(st.ip + i0);
          kr[0] = kw.x, kr[1] = kw.y, kr[2] = kw.z, kr[3] = kw.w;
          ir[0] = iw.x, ir[1] = iw.y, ir[2] = iw.z, ir[3] = iw.w;
        }
#pragma unroll
        for (int j = 0; j < kAccEpl; ++j) {
          const uint32_t kj = (kr[j >> 1] >> (16 * (j & 1))) & 0xFFFFu;
          kk[j] = kj == kPadKey ? -1 : (int)kj;
          x[j] = st.v[(ir[j >> 1] >> (16 * (j & 1))) & 0xFFFFu];
        }
      } else {
#pragma unroll
        for (int j = 0; j < kAccEpl; ++j) {
          kk[j] = -1;
          x[j] = 0.0;
        }
      }
      // one run's sum lands: a plain add, a posted piece, or a chain's end
      // (kept in registers: it is resolved after this warp's flag is up, so
      // no warp ever waits on a warp that is itself waiting)
      int pend_key = -1;
      double pend_s = 0.0;
      auto land = [&](int key, double s) {
        if (key == pk) {
          if (key == nk) {  // the whole warp is one run continuing both ways
            pA[warp] = s;
            kA[warp] = key;
            thruA[warp] = 1;
          } else {
            pend_key = key;
            pend_s = s;
          }
        } else if (key == nk) {
          pB[warp] = s;
          kB[warp] = key;
        } else {
          acc[key] += s;
        }
      };
      if (lane == 0) {
        kA[warp] = -1;
        kB[warp] = -1;
        thruA[warp] = 0;
      }
      __syncwarp();
      // fold: first run (fk, fs), current run (ck, cs); interior runs land at once
      int fk = -2, ck = -2;
      double fs = 0.0, cs = 0.0;
      bool multi = false;
#pragma unroll
      for (int i = 0; i < kAccEpl; ++i) {
        const int ki = kk[i];
        if (i == 0) {
          ck = ki;
          cs = x[0];
        } else if (ki == ck) {
          cs += x[i];
        } else {
          if (!multi) {
            fk = ck;
            fs = cs;
            multi = true;
          } else if (ck >= 0) {
            land(ck, cs);  // a run strictly inside this lane
          }
          ck = ki;
          cs = x[i];
        }
      }
      if (!multi) {
        fk = ck;
        fs = cs;
      }
      // carry the tails: lane L continues lane L-1's tail if its first key
      // equals that tail's key; a single-run continuing lane passes it on
      const int pkl = __shfl_up_sync(0xffffffffu, ck, 1);
      const bool cont = lane > 0 && fk >= 0 && fk == pkl;
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
      if (multi && fk >= 0) land(fk, cont ? fs + Sp : fs);  // the first run ends in this lane
      if (!next_cont && ck >= 0) land(ck, S);                // the tail run ends here
      __syncwarp();
      if (lane == 0) {  // this warp's pieces are posted
        __threadfence_block();
        flag[warp] = tc;
      }
      if (pend_key >= 0) {
        // a chain ends here: wait for the earlier warps' pieces, add in warp order
        int w0 = warp - 1;
        while (true) {
          while (flag[w0] != tc) {
          }
          __threadfence_block();
          if (!(kA[w0] == pend_key && thruA[w0])) break;
          --w0;
        }
        double sum = pB[w0];
        for (int q = w0 + 1; q < warp; ++q) sum += pA[q];
        acc[pend_key] += sum + pend_s;
      }
      __syncthreads();  // every add of the tile landed; the stage is free
      if (threadIdx.x == 0 && ti + kStages < ntiles) {
        issue(tc + kStages, mnext, e0 + (int64_t)(ti + kStages) * kTile,
              (int)min((int64_t)kTile, e1 - e0 - (int64_t)(ti + kStages) * kTile));
        if (ti + kStages + 1 < ntiles) mnext = __ldg(meta + ti + kStages + 1);
      }
    }
    const int64_t r0 = b << shift;
    const int64_t r1 = min((int64_t)n, r0 + R);
    bool fin = true, from_slots = false;
    const int64_t slot0 = k > 1 ? (int64_t)__ldg(unit_slot + u) : 0;  // the bin's first slot
    if (k > 1) {
      // a split bin: this unit's partial sums go to its slot; the last unit
      // to finish sums the k slots in unit order
      const int64_t slot = slot0 + __ldg(unit_j + u);
      for (int64_t r = r0 + threadIdx.x; r < r1; r += kAccThreads) slots[slot * R + (r - r0)] = acc[r - r0];
      __threadfence();
      __syncthreads();
      if (threadIdx.x == 0) s_last = atomicAdd(bin_done + b, 1u) == (unsigned)(k - 1);
      __syncthreads();
      fin = s_last;
      from_slots = true;
      if (fin) __threadfence();
    }
    if (fin) {
      double lmax = 0.0, lsum = 0.0;
      // rows in batches of 4 per thread: the pr / outdeg loads of a batch are
      // issued together (one latency per batch, not per row)
      //
      // Rows without in-edges keep rank base and a constant contribution
      // from the first sweep on: once every buffer holds those (live_rows
      // set by the caller), only the bin's rows with in-edges are finished
      // (their list: live_rows[b << shift ..], live_cnt[b]) -- the same
      // values, and a zero |delta| left out of the residual.
      constexpr int RB = 4;
      const int nfin = live_rows ? __ldg(live_cnt + b) : (int)(r1 - r0);
      const uint16_t* lv = live_rows ? live_rows + (b << shift) : nullptr;
      for (int ib = threadIdx.x; ib < nfin; ib += RB * kAccThreads) {
        double old[RB], sum[RB];
        int od[RB];
        int64_t rr[RB];
#pragma unroll
        for (int q = 0; q < RB; ++q) {
          const int i = ib + q * kAccThreads;
          rr[q] = i < nfin ? r0 + (lv ? (int64_t)__ldg(lv + i) : (int64_t)i) : r1;
        }
#pragma unroll
        for (int q = 0; q < RB; ++q) {
          const int64_t r = rr[q];
          old[q] = 0.0;
          od[q] = 0;
          sum[q] = 0.0;
          if (r < r1) {
            old[q] = __ldcg(pr + r);
            od[q] = __ldg(outdeg + r);
            if (from_slots) {
              sum[q] = __ldcg(slots + slot0 * R + (r - r0));
              for (int j = 1; j < k; ++j) sum[q] += __ldcg(slots + (slot0 + j) * R + (r - r0));
            } else {
              sum[q] = acc[r - r0];
            }
          }
        }
#pragma unroll
        for (int q = 0; q < RB; ++q) {
          const int64_t r = rr[q];
          if (r < r1) {
            const double nv = __dadd_rn(base, __dmul_rn(damping, sum[q]));
            const double dd = fabs(nv - old[q]);
            pr_out[r] = nv;
            if (od[q] > 0) {
              const double c = __ddiv_rn(nv, (double)od[q]);
              cur[r] = c;
              // multi-GPU part: the same store into every peer's replica (the
              // sweep is the exchange, as in kernels.cu kModePeers)
              for (int pq = 0; pq < peers.n; ++pq) peers.p[pq][r] = c;
            }
            lmax = fmax(lmax, dd);
            lsum += dd;
          }
        }
      }
      if (from_slots && threadIdx.x == 0) bin_done[b] = 0u;
      // the bin's residual pair, reduced in a fixed thread order
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        lmax = fmax(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
        lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
      }
      if (lane == 0) {
        s_pair[0][warp] = lmax;
        s_pair[1][warp] = lsum;
      }
      __syncthreads();
      if (warp == 0) {
        lmax = lane < NW ? s_pair[0][lane] : 0.0;
        lsum = lane < NW ? s_pair[1][lane] : 0.0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
          lmax = fmax(lmax, __shfl_xor_sync(0xffffffffu, lmax, o));
          lsum += __shfl_xor_sync(0xffffffffu, lsum, o);
        }
        if (lane == 0) {
          bin_pairs[2 * b] = lmax;
          bin_pairs[2 * b + 1] = lsum;
        }
      }
    }
    __syncthreads();
  }
}

__global__ void pb_bin_edges_kernel(const int64_t* row, int32_t n, int shift, int64_t nbins, int64_t* be) {
  const int64_t b = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (b <= nbins) be[b] = row[min((int64_t)n, b << shift)];
}

// Fixed-order reduction of the per-bin residual pairs: thread t folds a
// contiguous run of bins in order, then a fixed shuffle/shared tree.
constexpr int kReduceThreads = 1024;
__global__ void __launch_bounds__(kReduceThreads) pb_reduce_kernel(int64_t nbins, const double* bin_pairs,
                                                                   double* err, double* l1, const unsigned int* gate) {
  if (gate && *reinterpret_cast<const volatile unsigned int*>(gate)) return;  // stopped: no-op sweep
  const int64_t per = (nbins + kReduceThreads - 1) / kReduceThreads;
  const int64_t b0 = (int64_t)threadIdx.x * per, b1 = min(nbins, b0 + per);
  double mx = 0.0, sm = 0.0;
  for (int64_t b = b0; b < b1; ++b) {
    mx = fmax(mx, bin_pairs[2 * b]);
    sm += bin_pairs[2 * b + 1];
  }
  __shared__ double s[2][32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    sm += __shfl_xor_sync(0xffffffffu, sm, o);
  }
  if (lane == 0) {
    s[0][warp] = mx;
    s[1][warp] = sm;
  }
  __syncthreads();
  if (warp == 0) {
    mx = s[0][lane];
    sm = s[1][lane];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      sm += __shfl_xor_sync(0xffffffffu, sm, o);
    }
    if (lane == 0) {
      *err = mx;
      *l1 = sm;
    }
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
  S = (uint32_t)std::max<int64_t>(1, std::min<int64_t>(S, nbins));  // at most one wave per bin
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
  if (e == cudaSuccess) e = alloc((void**)&plan.item_ubase, off[W] * sizeof(int64_t));
  if (e == cudaSuccess) {
    pb_piece_fill_kernel<<<sms * 4, 256, 0, st>>>(pb.counts, pb.start, piece_off, pb.seg_piece0, pb.pbase, nseg,
                                                   d_wb, W, nbins, nchunks, plan.item_start, plan.item_len,
                                                   plan.item_ubase);
    e = cudaGetLastError();
  }
  if (e == cudaSuccess) e = alloc((void**)&plan.ctr, 2 * (size_t)W * sizeof(unsigned long long));
  for (void* q : {(void*)npieces, (void*)piece_off, (void*)d_wb, temp})
    if (q) cudaFreeAsync(q, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  if (e != cudaSuccess) {
    for (void* q : plan.allocs) cudaFreeAsync(q, st);
    cudaStreamSynchronize(st);
    return e;
  }
  {
    // phase-2 units: bins, heavy ones cut into runs of whole tiles of about
    // `piece` entries: small enough that each wave has several units per
    // CTA, never below twice the average bin (a split bin writes and re-reads
    // a slot of row sums per unit; splitting config 4's even bins cost 5-10%)
    const int64_t avg_bin = pb.nps / std::max<int64_t>(1, pb.nbins);
    int64_t piece = std::max<int64_t>({int64_t(1) << 16, 2 * avg_bin, pb.nps / ((int64_t)pb.p2_grid * 8 * W)});
    if (const char* v = std::getenv("FPR_B200_PB_PIECE")) piece = std::max<int64_t>(32, std::atoll(v));  // tests
    const int64_t piece_tiles = std::max<int64_t>(1, (piece + kTile - 1) / kTile);
    std::vector<int32_t> ubin, uk, uj, uslot;
    std::vector<int64_t> ue, ut;
    int64_t nslots = 0;
    plan.unit0.assign(W + 1, 0);
    for (int w = 0; w < W; ++w) {
      plan.unit0[w] = (int64_t)ubin.size();
      for (int64_t b = plan.wave_bin[w]; b < plan.wave_bin[w + 1]; ++b) {
        const int64_t p0 = pb.pbin_pos[b], p1 = pb.pbin_pos[b + 1];
        const int64_t tiles = std::max<int64_t>(1, (p1 - p0 + kTile - 1) / kTile);
        const int64_t k = (tiles + piece_tiles - 1) / piece_tiles;
        for (int64_t j = 0; j < k; ++j) {
          ubin.push_back((int32_t)b);
          uk.push_back((int32_t)k);
          uj.push_back((int32_t)j);
          uslot.push_back(k > 1 ? (int32_t)nslots : -1);
          ue.push_back(std::min(p1, p0 + tiles * j / k * kTile));
          ut.push_back(pb.tile_off[b] + tiles * j / k);
        }
        if (k > 1) nslots += k;
      }
    }
    plan.unit0[W] = (int64_t)ubin.size();
    // unit u ends where unit u + 1 starts, or at its bin's end
    std::vector<int64_t> uend(ubin.size() + 1);
    for (size_t u = 0; u < ubin.size(); ++u)
      uend[u] = (u + 1 < ubin.size() && ubin[u + 1] == ubin[u]) ? ue[u + 1] : pb.pbin_pos[ubin[u] + 1];
    // unit_e holds [start, end) pairs flattened: start of u at 2u, end at 2u + 1
    std::vector<int64_t> ue2(2 * ubin.size());
    for (size_t u = 0; u < ubin.size(); ++u) {
      ue2[2 * u] = ue[u];
      ue2[2 * u + 1] = uend[u];
    }
    const size_t U = ubin.size();
    e = alloc((void**)&plan.unit_bin, U * sizeof(int32_t));
    if (e == cudaSuccess) e = alloc((void**)&plan.unit_k, U * sizeof(int32_t));
    if (e == cudaSuccess) e = alloc((void**)&plan.unit_j, U * sizeof(int32_t));
    if (e == cudaSuccess) e = alloc((void**)&plan.unit_slot, U * sizeof(int32_t));
    if (e == cudaSuccess) e = alloc((void**)&plan.unit_e, ue2.size() * sizeof(int64_t));
    if (e == cudaSuccess) e = alloc((void**)&plan.unit_t, U * sizeof(int64_t));
    if (e == cudaSuccess) e = alloc((void**)&plan.slots, (size_t)std::max<int64_t>(1, nslots) * sizeof(double) << pb.shift);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(plan.unit_bin, ubin.data(), U * sizeof(int32_t), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(plan.unit_k, uk.data(), U * sizeof(int32_t), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(plan.unit_j, uj.data(), U * sizeof(int32_t), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(plan.unit_slot, uslot.data(), U * sizeof(int32_t), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(plan.unit_e, ue2.data(), ue2.size() * sizeof(int64_t), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(plan.unit_t, ut.data(), U * sizeof(int64_t), cudaMemcpyHostToDevice, st);
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

cudaError_t build_pb(const DevGraph& g, int64_t nsrc, int shift, int chunk_shift, cudaStream_t st, PbSet& pb,
                     const char** msg) {
  cudaError_t e = cudaSuccess;
  *msg = nullptr;
  pb = PbSet{};
  const int sms = sm_count();
  const int64_t n = g.n;
  const int64_t nbins = n > 0 ? (n + (1ll << shift) - 1) >> shift : 0;
  const int64_t nchunks = std::max<int64_t>(1, (nsrc + (1ll << chunk_shift) - 1) >> chunk_shift);
  const int64_t nseg = nbins * nchunks;
  // layout kernel: chunk counters + the bin's (2^shift + 1) relative row offsets
  const size_t hist_smem = ((size_t)(nchunks + 3) & ~(size_t)3) * sizeof(uint32_t) +
                           (((size_t)1 << std::min(shift, 20)) + 1) * sizeof(uint32_t) +
                           (nchunks <= kSplitMaxChunks ? (size_t)(nchunks + 1) * 32 * sizeof(uint32_t) : 0);
  const size_t acc_smem = ((size_t)sizeof(double) << shift) + (size_t)kStages * sizeof(PbStage);
  // layout temporaries: per-entry row offsets, tile offsets, per-bin run
  // counts, per-segment pieces and their scan, per-run row offsets
  uint16_t* dstl = nullptr;
  uint16_t* pkey = nullptr;
  int64_t *tile_off_d = nullptr, *bin_np = nullptr, *pbin_pos_d = nullptr;
  uint32_t* seg_np = nullptr;
  uint32_t *hot_bits = nullptr, *hot_wpre = nullptr;  // hot-source bitmap + rank prefix (layout only)
  int64_t hot_kc = 0;
  void* scan_tmp = nullptr;
  const unsigned tgrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(nbins, (int64_t)sms * 4));
  const unsigned sgrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>((nseg + 255) / 256, (int64_t)sms * 32));
  if (n == 0 || shift < 5 || shift > 13 || chunk_shift < 0 || chunk_shift > 31 || hist_smem > 192 * 1024 ||
      acc_smem + 2048 > 227 * 1024 || nseg > (1ll << 31) || nsrc > 0x7FFFFFFFll) {
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
  pb.m = g.m;
  {
    // bin edge offsets (host copy: wave plans cut waves from them) and the
    // bins' 8-aligned entry positions (16-B source loads)
    std::vector<int64_t> be;
    e = pb_bin_edges(g, shift, st, &be);
    if (e != cudaSuccess) goto out;
    pb.bin_edge = be;
    pb.bin_pos.assign(nbins + 1, 0);
    for (int64_t b = 0; b < nbins; ++b) {
      if (be[b + 1] - be[b] >= (1ll << 32)) {  // the layout kernel's uint32 in-bin offsets
        *msg = "a bin holds 2^32 or more edges (use a smaller FPR_B200_PB_SHIFT)";
        goto out;
      }
      pb.bin_pos[b + 1] = pb.bin_pos[b] + ((be[b + 1] - be[b] + 7) & ~int64_t(7));
    }
  }
  pb.mpad = pb.bin_pos[nbins];
  PK(alloc((void**)&pb.counts, nseg * sizeof(uint32_t)));
  PK(alloc((void**)&pb.start, nseg * sizeof(int64_t)));
  PK(alloc((void**)&pb.bin_pos_d, (nbins + 1) * sizeof(int64_t)));
  PK(cudaMemcpyAsync(pb.bin_pos_d, pb.bin_pos.data(), (nbins + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  // the gather's 16-B source loads read up to 3 entries past a piece
  PK(alloc((void**)&pb.esrc, std::max<int64_t>(pb.mpad, 1) * sizeof(int32_t) + 64));
  PK(cudaMallocAsync(&dstl, std::max<int64_t>(pb.mpad, 1) * sizeof(uint16_t), st));
  {
    int key_bits = 1;
    while ((1ll << key_bits) <= nchunks) ++key_bits;  // chunk ids and the sentinel nchunks
    // pieces of every bin's edges (hub bins spread over many CTAs)
    int64_t lpiece = kLayoutPiece;
    if (const char* v = std::getenv("FPR_B200_PB_LAYOUT_PIECE")) lpiece = std::max<int64_t>(1, std::atoll(v));  // tests
    std::vector<int32_t> hb;
    std::vector<int64_t> he, hp0(nbins + 1, 0);
    for (int64_t b = 0; b < nbins; ++b) {
      hp0[b] = (int64_t)hb.size();
      const int64_t len = pb.bin_edge[b + 1] - pb.bin_edge[b];
      const int64_t k = std::max<int64_t>(1, (len + lpiece - 1) / lpiece);
      for (int64_t j = 0; j < k; ++j) {
        hb.push_back((int32_t)b);
        he.push_back(pb.bin_edge[b] + j * lpiece);
      }
    }
    hp0[nbins] = (int64_t)hb.size();
    const int64_t npc = (int64_t)hb.size();
    int32_t* piece_bin = nullptr;
    int64_t *piece_e = nullptr, *bin_piece0 = nullptr;
    uint32_t *phist = nullptr, *pcur = nullptr;
    e = cudaMallocAsync(&piece_bin, npc * sizeof(int32_t), st);
    if (e == cudaSuccess) e = cudaMallocAsync(&piece_e, npc * sizeof(int64_t), st);
    if (e == cudaSuccess) e = cudaMallocAsync(&bin_piece0, (nbins + 1) * sizeof(int64_t), st);
    if (e == cudaSuccess) e = cudaMallocAsync(&phist, npc * nchunks * sizeof(uint32_t), st);
    if (e == cudaSuccess) e = cudaMallocAsync(&pcur, npc * nchunks * sizeof(uint32_t), st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(piece_bin, hb.data(), npc * sizeof(int32_t), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess) e = cudaMemcpyAsync(piece_e, he.data(), npc * sizeof(int64_t), cudaMemcpyHostToDevice, st);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(bin_piece0, hp0.data(), (nbins + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st);
    const size_t hsm = ((size_t)(nchunks + 3) & ~(size_t)3) * sizeof(uint32_t);
    if (e == cudaSuccess && hsm > 48 * 1024)
      e = cudaFuncSetAttribute(pb_piece_hist_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hsm);
    if (e == cudaSuccess)
      e = cudaFuncSetAttribute(pb_layout_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hist_smem);
    if (e == cudaSuccess) {
      const unsigned pgrid = (unsigned)std::max<int64_t>(1, std::min<int64_t>(npc, (int64_t)sms * 2));
      pb_piece_hist_kernel<<<pgrid, kPbThreads, hsm, st>>>(g.row, g.src, g.n, shift, chunk_shift, nchunks, piece_bin,
                                                           piece_e, npc, phist);
      pb_bin_scan_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(nbins, (int64_t)sms * 2)), kPbThreads, 0,
                           st>>>(pb.bin_pos_d, nbins, nchunks, bin_piece0, phist, pb.counts, pb.start, pcur);
      pb_layout_kernel<<<(unsigned)std::max<int64_t>(1, std::min<int64_t>(npc, (int64_t)sms)), kPbThreads, hist_smem,
                         st>>>(g.row, g.src, g.n, shift, chunk_shift, key_bits, nchunks, pb.bin_pos_d, piece_bin, piece_e,
                               npc, pcur, pb.esrc, dstl);
      e = cudaGetLastError();
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);  // the host piece vectors die here
    for (void* q : {(void*)piece_bin, (void*)piece_e, (void*)bin_piece0, (void*)phist, (void*)pcur})
      if (q) cudaFreeAsync(q, st);
    PK(e);
  }
  // runs per bin -> their 8-aligned positions and the accumulate's tiles
  PK(cudaMallocAsync(&bin_np, std::max<int64_t>(nbins, 1) * sizeof(int64_t), st));
  pb_close_count_kernel<<<tgrid, kAccThreads, 0, st>>>(pb.esrc, dstl, g.row, g.n, shift, pb.bin_pos_d, pb.start,
                                                      nbins, chunk_shift, bin_np);
  PK(cudaGetLastError());
  {
    std::vector<int64_t> np(nbins);
    PK(cudaMemcpyAsync(np.data(), bin_np, nbins * sizeof(int64_t), cudaMemcpyDeviceToHost, st));
    PK(cudaStreamSynchronize(st));
    pb.pbin_pos.assign(nbins + 1, 0);
    for (int64_t b = 0; b < nbins; ++b) pb.pbin_pos[b + 1] = pb.pbin_pos[b] + ((np[b] + 7) & ~int64_t(7));
  }
  pb.nps = pb.pbin_pos[nbins];
  pb.tile_off.assign(nbins + 1, 0);
  for (int64_t b = 0; b < nbins; ++b)
    pb.tile_off[b + 1] = pb.tile_off[b] + (pb.pbin_pos[b + 1] - pb.pbin_pos[b] + kTile - 1) / kTile;
  pb.ntiles = pb.tile_off[nbins];
  PK(cudaMallocAsync(&pbin_pos_d, (nbins + 1) * sizeof(int64_t), st));
  PK(cudaMemcpyAsync(pbin_pos_d, pb.pbin_pos.data(), (nbins + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  PK(cudaMallocAsync(&tile_off_d, (nbins + 1) * sizeof(int64_t), st));
  PK(cudaMemcpyAsync(tile_off_d, pb.tile_off.data(), (nbins + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, st));
  // the gather pieces of every segment (numbered segment by segment,
  // chunk-major) and the first run of each
  PK(cudaMallocAsync(&seg_np, std::max<int64_t>(nseg, 1) * sizeof(uint32_t), st));
  PK(alloc((void**)&pb.seg_piece0, std::max<int64_t>(nseg, 1) * sizeof(uint32_t)));
  pb_seg_pieces_kernel<<<sgrid, 256, 0, st>>>(pb.counts, nseg, seg_np);
  PK(cudaGetLastError());
  {
    size_t tb = 0;
    PK(cub::DeviceScan::ExclusiveSum(nullptr, tb, seg_np, pb.seg_piece0, nseg, st));
    PK(cudaMallocAsync(&scan_tmp, std::max<size_t>(tb, 16), st));
    PK(cub::DeviceScan::ExclusiveSum(scan_tmp, tb, seg_np, pb.seg_piece0, nseg, st));
    uint32_t last0 = 0, last1 = 0;
    PK(cudaMemcpyAsync(&last0, pb.seg_piece0 + nseg - 1, 4, cudaMemcpyDeviceToHost, st));
    PK(cudaMemcpyAsync(&last1, seg_np + nseg - 1, 4, cudaMemcpyDeviceToHost, st));
    PK(cudaStreamSynchronize(st));
    pb.npieces = (int64_t)last0 + last1;
  }
  PK(alloc((void**)&pb.pbase, std::max<int64_t>(pb.npieces, 1) * sizeof(int64_t)));
  PK(cudaMallocAsync(&pkey, std::max<int64_t>(pb.nps, 1) * sizeof(uint16_t), st));
  // hot sources per chunk, with a dense copy refreshed before every gather pass
  if (kHot > 0 && chunk_shift >= 5 && nsrc <= (int64_t)kIdMask + 1 && g.m > 0) {
    uint32_t *cnt = nullptr, *thr = nullptr;
    hot_kc = std::min<int64_t>(kHot, int64_t(1) << chunk_shift);  // slots per chunk
    pb.nhot = nchunks * hot_kc;
    const int64_t nw = (nsrc + 31) >> 5;
    e = alloc((void**)&pb.hot_src, pb.nhot * sizeof(int32_t));
    if (e == cudaSuccess) e = alloc((void**)&pb.hot_val, pb.nhot * sizeof(double));
    if (e == cudaSuccess) e = cudaMemsetAsync(pb.hot_src, 0xFF, pb.nhot * sizeof(int32_t), st);
    if (e == cudaSuccess) e = cudaMemsetAsync(pb.hot_val, 0, pb.nhot * sizeof(double), st);
    if (e == cudaSuccess) e = cudaMallocAsync(&cnt, nsrc * sizeof(uint32_t), st);
    if (e == cudaSuccess) e = cudaMallocAsync(&thr, nchunks * sizeof(uint32_t), st);
    if (e == cudaSuccess) e = cudaMallocAsync(&hot_bits, nw * sizeof(uint32_t), st);
    if (e == cudaSuccess) e = cudaMallocAsync(&hot_wpre, nw * sizeof(uint32_t), st);
    // a source's frequency among the entries is its out-degree on a whole
    // graph; a multi-GPU part counts its own entries
    const bool whole = nsrc == (int64_t)g.n;
    if (e == cudaSuccess && whole)
      e = cudaMemcpyAsync(cnt, g.outdeg, nsrc * sizeof(uint32_t), cudaMemcpyDeviceToDevice, st);
    if (e == cudaSuccess && !whole) e = cudaMemsetAsync(cnt, 0, nsrc * sizeof(uint32_t), st);
    if (e == cudaSuccess) {
      const unsigned grid = (unsigned)sms * 8;
      if (!whole) pb_src_hist_kernel<<<grid, 256, 0, st>>>(pb.esrc, pb.mpad, cnt);
      pb_hot_threshold_kernel<<<(unsigned)nchunks, 1024, 0, st>>>(cnt, nsrc, chunk_shift, hot_kc, thr);
      pb_hot_bits_kernel<<<grid, 256, 0, st>>>(cnt, nsrc, chunk_shift, thr, hot_bits);
      pb_hot_rank_kernel<<<(unsigned)nchunks, 1024, 0, st>>>(hot_bits, nsrc, chunk_shift, hot_wpre);
      pb_hot_src_kernel<<<grid, 256, 0, st>>>(hot_bits, hot_wpre, nsrc, chunk_shift, hot_kc, pb.hot_src);
      e = cudaGetLastError();
    }
    for (void* q : {(void*)cnt, (void*)thr})
      if (q) cudaFreeAsync(q, st);
    PK(e);
  }
  pb_psum_kernel<<<tgrid, kAccThreads, 0, st>>>(pb.esrc, dstl, g.row, g.n, shift, pb.bin_pos_d, pbin_pos_d, pb.start,
                                               pb.seg_piece0, nbins, chunk_shift, pkey, pb.pbase);
  PK(cudaGetLastError());
  if (hot_bits) {
    pb_hot_rewrite_kernel<<<(unsigned)sms * 8, 256, 0, st>>>(pb.esrc, pb.mpad, hot_bits, hot_wpre, chunk_shift,
                                                             hot_kc);
    PK(cudaGetLastError());
  }

  // the accumulate's side: per tile of runs, the row order
  PK(alloc((void**)&pb.vidx, std::max<int64_t>(pb.nps, 1) * sizeof(uint16_t)));
  PK(alloc((void**)&pb.skey, std::max<int64_t>(pb.nps, 1) * sizeof(uint16_t)));
  PK(alloc((void**)&pb.tile_meta, std::max<int64_t>(pb.ntiles, 1) * sizeof(uint64_t)));
  pb_tile_sort_kernel<<<tgrid, kAccThreads, 0, st>>>(pkey, pbin_pos_d, tile_off_d, nbins, shift, pb.vidx, pb.skey,
                                                    pb.tile_meta);
  PK(cudaGetLastError());
  // per-sweep scratch: the runs' partial sums (the stage's pair-rounded
  // copies read one past a tile)
  PK(alloc((void**)&pb.psum, std::max<int64_t>(pb.nps, 1) * sizeof(double) + 64));
  PK(cudaMemsetAsync(pb.psum, 0, std::max<int64_t>(pb.nps, 1) * sizeof(double) + 64, st));
  PK(alloc((void**)&pb.bin_pairs, 2 * nbins * sizeof(double)));
  PK(alloc((void**)&pb.live_rows, (size_t)nbins * sizeof(uint16_t) << shift));
  PK(alloc((void**)&pb.live_cnt, nbins * sizeof(int32_t)));
  pb_live_rows_kernel<<<tgrid, 1024, 0, st>>>(g.row, g.n, shift, nbins, pb.live_rows, pb.live_cnt);
  PK(cudaGetLastError());
  PK(alloc((void**)&pb.bin_done, nbins * sizeof(unsigned int)));
  PK(cudaMemsetAsync(pb.bin_done, 0, nbins * sizeof(unsigned int), st));
  PK(cudaFuncSetAttribute(pb_accum_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)acc_smem));
  {
    // phase-2 residency: the CTAs per SM that fit the bin's accumulators +
    // the staged tiles (two at 2^13-row bins), up to kAccCtas
    int per_sm = 0;
    PK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pb_accum_kernel, kAccThreads, acc_smem));
    per_sm = std::max(1, std::min(per_sm, kAccCtas));
    pb.p2_grid = (int)std::min<int64_t>(nbins, (int64_t)sms * per_sm);
    pb.p1_grid = sms * 8;
    pb.acc_smem = (int)acc_smem;
  }
  PK(cudaStreamSynchronize(st));
out:
  for (void* q : {(void*)dstl, (void*)pkey, (void*)tile_off_d, (void*)bin_np, (void*)pbin_pos_d, (void*)seg_np,
                  (void*)hot_bits, (void*)hot_wpre, scan_tmp})
    if (q) cudaFreeAsync(q, st);
  if (e != cudaSuccess || *msg) {
    free_pb(pb, st);
    cudaStreamSynchronize(st);
  }
  return e;
}

cudaError_t launch_pb_sweep(const PbSet& pb, const PbPlan& plan, const DevGraph& g, const double* prev,
                            const double* pr, double* pr_out, double* cur, const PbPeers& peers, double base,
                            double damping, double* err, double* l1, cudaStream_t st, const unsigned int* gate,
                            bool skip_empty) {
  const uint16_t* lrows = skip_empty && pb.live_rows ? pb.live_rows : nullptr;
  const int W = plan.nwaves;
  // work counters: [0, W) phase-1 pieces, [W, 2W) phase-2 units
  cudaError_t e = cudaMemsetAsync(plan.ctr, 0, 2 * (size_t)W * sizeof(unsigned long long), st);
  if (e != cudaSuccess) return e;
  for (int w = 0; w < W; ++w) {
    const int64_t i0 = plan.item0[w], u0 = plan.unit0[w];
    if (plan.item0[w + 1] > i0) {
      if (pb.nhot > 0) {
        pb_hot_refresh_kernel<<<(unsigned)std::min<int64_t>((pb.nhot + 255) / 256, (int64_t)pb.p1_grid), 256, 0,
                                st>>>(pb.hot_src, pb.nhot, prev, pb.hot_val, gate);
        if ((e = cudaGetLastError()) != cudaSuccess) return e;
      }
      pb_gather_kernel<<<pb.p1_grid, kGatherThreads, 0, st>>>(pb.esrc, plan.item_start + i0, plan.item_len + i0,
                                                              plan.item_ubase + i0, plan.item0[w + 1] - i0, prev,
                                                              pb.nhot > 0 ? pb.hot_val : nullptr, pb.psum,
                                                              plan.ctr + w, gate);
      if ((e = cudaGetLastError()) != cudaSuccess) return e;
    }
    pb_accum_kernel<<<pb.p2_grid, kAccThreads, pb.acc_smem, st>>>(
        pb.psum, pb.vidx, pb.skey, pb.tile_meta, plan.unit_bin + u0, plan.unit_e + 2 * u0, plan.unit_t + u0,
        plan.unit_k + u0, plan.unit_j + u0,
        plan.unit_slot + u0, plan.unit0[w + 1] - u0, pb.shift, g.n, g.outdeg, pr, pr_out, cur,
        peers, base, damping, plan.slots, pb.bin_done, plan.ctr + W + w, pb.bin_pairs, gate, lrows, pb.live_cnt);
    if ((e = cudaGetLastError()) != cudaSuccess) return e;
  }
  pb_reduce_kernel<<<1, kReduceThreads, 0, st>>>(pb.nbins, pb.bin_pairs, err, l1, gate);
  return cudaGetLastError();
}

}  // namespace fprb
