// blocked.cu -- source-blocked layout for graphs whose contribution vector
// does not fit in L2 (configs 4/5).
//
// The EC gather contrib[in_src[e]] is a random 8-B read.  While contrib fits
// in L2 it costs one L2 request; at config 5 (2.1 GB) most gathers miss to
// HBM, where a random 32-B sector read costs far more.  The blocked layout
// splits the source range into column blocks of 2^shift vertices, each block
// small enough to stay L2-resident while it is swept:
//   * every edge goes to the block of its source, keeping the row-major edge
//     order inside the block (a stable counting sort by block id);
//   * inside a block the rows that have edges there are compacted: local row
//     k is global row ids[k], with row_ptr over the block's edge slice;
//   * each block gets its own merge-path task partition, so one EC sweep is B
//     passes of the ordinary solve kernel in accumulate mode (partial[row] +=
//     in-block sum, blocks in order: one writer per (row, block)), then an
//     apply pass that turns partial[] into ranks, contributions and the
//     residual.
// Summation order per row: within a block ascending source (as the reference),
// blocks ascending -- a regrouping of the reference's left-to-right sum, well
// inside the 1e-12 per-iteration tolerance.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>
#include <vector>

#include "internal.cuh"

namespace fprb {

namespace {

constexpr int kTileEdges = 16384;  // edges per counting-sort tile (one CTA)
constexpr int kSortThreads = 256;
constexpr int kMaxBlocks = 256;    // column blocks (smem counters per CTA)

int grid_for(int64_t work) {
  const int64_t b = (work + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148ll * 16));
}

// Row id of every edge (warp per row, lanes stride the row's edges).
__global__ void edge_rows_kernel(const int64_t* row, int32_t n, int32_t* erow) {
  const int lane = threadIdx.x & 31;
  const int64_t w0 = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = w0; r < n; r += nw) {
    const int64_t a = row[r], b = row[r + 1];
    for (int64_t e = a + lane; e < b; e += 32) erow[e] = (int32_t)r;
  }
}

// Pass 1: per-tile histogram of block ids, stored block-major (hist[b*ntiles+tile]).
__global__ void __launch_bounds__(kSortThreads) tile_hist_kernel(const int32_t* src, int64_t m, int shift,
                                                                 int nblocks, int64_t ntiles,
                                                                 unsigned long long* hist) {
  __shared__ unsigned int h[kMaxBlocks];
  for (int b = threadIdx.x; b < nblocks; b += kSortThreads) h[b] = 0;
  __syncthreads();
  const int64_t e0 = (int64_t)blockIdx.x * kTileEdges;
  const int64_t e1 = e0 + kTileEdges < m ? e0 + kTileEdges : m;
  for (int64_t e = e0 + threadIdx.x; e < e1; e += kSortThreads)
    atomicAdd(&h[(uint32_t)src[e] >> shift], 1u);
  __syncthreads();
  for (int b = threadIdx.x; b < nblocks; b += kSortThreads)
    hist[(int64_t)b * ntiles + blockIdx.x] = h[b];
}

// Pass 2: stable scatter.  The tile is consumed in 256-edge chunks in edge
// order; inside a chunk, edges of the same block are ranked by warp
// (match_any) and by lane, so every block receives its edges in edge order.
__global__ void __launch_bounds__(kSortThreads) tile_scatter_kernel(
    const int32_t* src, const int32_t* erow, int64_t m, int shift, int nblocks, int64_t ntiles,
    const unsigned long long* offs, const long long* adjust, int32_t* out_src, int32_t* out_row) {
  constexpr int kWarps = kSortThreads / 32;
  __shared__ long long run[kMaxBlocks];
  __shared__ unsigned int wc[kWarps][kMaxBlocks];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int b = threadIdx.x; b < nblocks; b += kSortThreads) {
    run[b] = (long long)offs[(int64_t)b * ntiles + blockIdx.x] + adjust[b];
    for (int w = 0; w < kWarps; ++w) wc[w][b] = 0;
  }
  __syncthreads();
  const int64_t e0 = (int64_t)blockIdx.x * kTileEdges;
  const int64_t e1 = e0 + kTileEdges < m ? e0 + kTileEdges : m;
  for (int64_t c = e0; c < e1; c += kSortThreads) {
    const int64_t e = c + threadIdx.x;
    const bool valid = e < e1;
    const int32_t s = valid ? src[e] : 0;
    const int k = valid ? (int)((uint32_t)s >> shift) : -1;
    const unsigned peers = __match_any_sync(0xffffffffu, k);
    const int rank = __popc(peers & ((1u << lane) - 1u));
    if (valid && rank == 0) wc[warp][k] = __popc(peers);
    __syncthreads();
    if (valid) {
      long long pos = run[k] + rank;
      for (int w = 0; w < warp; ++w) pos += wc[w][k];
      out_src[pos] = s;
      out_row[pos] = erow[e];
    }
    __syncthreads();
    for (int b = threadIdx.x; b < nblocks; b += kSortThreads) {
      unsigned t = 0;
      for (int w = 0; w < kWarps; ++w) {
        t += wc[w][b];
        wc[w][b] = 0;
      }
      run[b] += t;
    }
    __syncthreads();
  }
}

__global__ void row_heads_kernel(const int32_t* rows, int64_t cnt, int32_t* flag) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += stride)
    flag[i] = (i == 0 || rows[i] != rows[i - 1]) ? 1 : 0;
}

__global__ void row_emit_kernel(const int32_t* rows, const int32_t* flag, const int32_t* pos, int64_t cnt,
                                int64_t* row_ptr, int32_t* ids) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < cnt; i += stride) {
    if (!flag[i]) continue;
    row_ptr[pos[i]] = i;
    ids[pos[i]] = rows[i];
  }
}

__global__ void set_last_kernel(int64_t* row_ptr, int32_t nrows, int64_t cnt) { row_ptr[nrows] = cnt; }

#define BK(x)                       \
  do {                              \
    e = (x);                        \
    if (e != cudaSuccess) goto out; \
  } while (0)

}  // namespace

// ------------------------------------------------------------ apply pass
// Every row from its accumulated sum: nv = base + d*partial (no FMA, as the
// unblocked finalize), contribution, residual; partial[] re-armed to 0.
// Per-CTA (max, sum) pairs in a fixed grid -> deterministic reduction.
__global__ void __launch_bounds__(256) apply_kernel(int32_t n, double* partial, const int32_t* outdeg,
                                                    double* pr, double* cur, double base, double damping,
                                                    double* cta_pairs) {
  double lmax = 0.0, lsum = 0.0;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n; r += stride) {
    const double s = partial[r];
    partial[r] = 0.0;
    const double nv = __dadd_rn(base, __dmul_rn(damping, s));
    const double d = fabs(nv - pr[r]);
    pr[r] = nv;
    const int od = outdeg[r];
    if (od > 0) cur[r] = __ddiv_rn(nv, (double)od);
    lmax = fmax(lmax, d);
    lsum += d;
  }
  __shared__ double sm[2][256];
  sm[0][threadIdx.x] = lmax;
  sm[1][threadIdx.x] = lsum;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      sm[0][threadIdx.x] = fmax(sm[0][threadIdx.x], sm[0][threadIdx.x + o]);
      sm[1][threadIdx.x] += sm[1][threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    cta_pairs[2 * blockIdx.x] = sm[0][0];
    cta_pairs[2 * blockIdx.x + 1] = sm[1][0];
  }
}

__global__ void __launch_bounds__(256) reduce_pairs_kernel(int nctas, const double* cta_pairs, double* err,
                                                           double* l1) {
  double lmax = 0.0, lsum = 0.0;
  for (int i = threadIdx.x; i < nctas; i += 256) {
    lmax = fmax(lmax, cta_pairs[2 * i]);
    lsum += cta_pairs[2 * i + 1];
  }
  __shared__ double sm[2][256];
  sm[0][threadIdx.x] = lmax;
  sm[1][threadIdx.x] = lsum;
  __syncthreads();
  for (int o = 128; o > 0; o >>= 1) {
    if (threadIdx.x < o) {
      sm[0][threadIdx.x] = fmax(sm[0][threadIdx.x], sm[0][threadIdx.x + o]);
      sm[1][threadIdx.x] += sm[1][threadIdx.x + o];
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    *err = sm[0][0];
    *l1 = sm[1][0];
  }
}

cudaError_t launch_apply(const BlockSet& bs, int32_t n, const int32_t* outdeg, double* pr, double* cur,
                         double base, double damping, double* err, double* l1, cudaStream_t st) {
  apply_kernel<<<bs.apply_grid, 256, 0, st>>>(n, bs.partial, outdeg, pr, cur, base, damping, bs.cta_pairs);
  reduce_pairs_kernel<<<1, 256, 0, st>>>(bs.apply_grid, bs.cta_pairs, err, l1);
  return cudaGetLastError();
}

void free_blocks(BlockSet& bs, cudaStream_t st) {
  for (void* p : bs.allocs)
    if (p) cudaFreeAsync(p, st);
  bs = BlockSet{};
}

cudaError_t build_blocks(const DevGraph& g, int shift, cudaStream_t st, BlockSet& bs, const char** msg) {
  cudaError_t e = cudaSuccess;
  bs = BlockSet{};
  const int64_t m = g.m;
  const int nblocks = (int)(((int64_t)g.n + (1ll << shift) - 1) >> shift);
  const int64_t ntiles = (m + kTileEdges - 1) / kTileEdges;
  int32_t* erow = nullptr;
  int32_t* rows = nullptr;
  unsigned long long* hist = nullptr;
  unsigned long long* offs = nullptr;
  long long* adjust = nullptr;
  int32_t* flag = nullptr;
  int32_t* pos = nullptr;
  void* temp = nullptr;
  size_t temp_bytes = 0;
  std::vector<unsigned long long> start(nblocks + 1), cnt(nblocks);
  std::vector<long long> adj(nblocks);
  std::vector<int64_t> base(nblocks + 1);
  int64_t maxcnt = 0;
  auto track = [&](void* p) { bs.allocs.push_back(p); };
  if (nblocks < 1 || nblocks > kMaxBlocks) {
    *msg = "blocked layout: block count outside [1, 256] (raise the block size)";
    return cudaSuccess;
  }
  bs.nblocks = nblocks;
  bs.shift = shift;
  BK(cudaMallocAsync(&erow, std::max<int64_t>(m, 1) * sizeof(int32_t), st));
  BK(cudaMallocAsync(&hist, (size_t)nblocks * ntiles * sizeof(unsigned long long) + 8, st));
  BK(cudaMallocAsync(&offs, (size_t)nblocks * ntiles * sizeof(unsigned long long) + 8, st));
  if (m > 0) {
    edge_rows_kernel<<<grid_for((int64_t)g.n * 32), 256, 0, st>>>(g.row, g.n, erow);
    BK(cudaGetLastError());
    tile_hist_kernel<<<(unsigned)ntiles, kSortThreads, 0, st>>>(g.src, m, shift, nblocks, ntiles, hist);
    BK(cudaGetLastError());
    BK(cub::DeviceScan::ExclusiveSum(nullptr, temp_bytes, hist, offs, (int64_t)nblocks * ntiles, st));
    BK(cudaMallocAsync(&temp, std::max<size_t>(temp_bytes, 16), st));
    BK(cub::DeviceScan::ExclusiveSum(temp, temp_bytes, hist, offs, (int64_t)nblocks * ntiles, st));
    for (int b = 0; b < nblocks; ++b)
      BK(cudaMemcpyAsync(&start[b], offs + (int64_t)b * ntiles, sizeof(unsigned long long),
                         cudaMemcpyDeviceToHost, st));
    BK(cudaStreamSynchronize(st));
  }
  start[nblocks] = (unsigned long long)m;
  // block b's slice of the pool starts 32-B aligned (LDG.256 source loads)
  base[0] = 0;
  for (int b = 0; b < nblocks; ++b) {
    cnt[b] = start[b + 1] - start[b];
    maxcnt = std::max<int64_t>(maxcnt, (int64_t)cnt[b]);
    base[b + 1] = base[b] + (((int64_t)cnt[b] + 7) & ~7ll);
    adj[b] = (long long)base[b] - (long long)start[b];
  }
  BK(cudaMallocAsync(&bs.src_pool, (base[nblocks] + 8) * sizeof(int32_t), st));
  track(bs.src_pool);
  BK(cudaMemsetAsync(bs.src_pool, 0, (base[nblocks] + 8) * sizeof(int32_t), st));
  BK(cudaMallocAsync(&rows, (base[nblocks] + 8) * sizeof(int32_t), st));
  BK(cudaMallocAsync(&adjust, nblocks * sizeof(long long), st));
  BK(cudaMemcpyAsync(adjust, adj.data(), nblocks * sizeof(long long), cudaMemcpyHostToDevice, st));
  if (m > 0) {
    tile_scatter_kernel<<<(unsigned)ntiles, kSortThreads, 0, st>>>(g.src, erow, m, shift, nblocks, ntiles, offs,
                                                                   adjust, bs.src_pool, rows);
    BK(cudaGetLastError());
  }
  cudaFreeAsync(erow, st);
  erow = nullptr;
  // per block: compacted rows, row_ptr, partition
  BK(cudaMallocAsync(&flag, std::max<int64_t>(maxcnt, 1) * sizeof(int32_t), st));
  BK(cudaMallocAsync(&pos, std::max<int64_t>(maxcnt, 1) * sizeof(int32_t), st));
  {
    size_t tb = 0;
    BK(cub::DeviceScan::ExclusiveSum(nullptr, tb, flag, pos, std::max<int64_t>(maxcnt, 1), st));
    if (tb > temp_bytes) {
      if (temp) cudaFreeAsync(temp, st);
      temp_bytes = tb;
      BK(cudaMallocAsync(&temp, temp_bytes, st));
    }
  }
  bs.blocks.resize(nblocks);
  for (int b = 0; b < nblocks; ++b) {
    BlockSet::Block& B = bs.blocks[b];
    const int64_t c = (int64_t)cnt[b];
    int32_t nrows = 0;
    if (c > 0) {
      row_heads_kernel<<<grid_for(c), 256, 0, st>>>(rows + base[b], c, flag);
      BK(cudaGetLastError());
      size_t tb = temp_bytes;
      BK(cub::DeviceScan::ExclusiveSum(temp, tb, flag, pos, c, st));
      int32_t lf = 0, lp = 0;
      BK(cudaMemcpyAsync(&lf, flag + c - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      BK(cudaMemcpyAsync(&lp, pos + c - 1, sizeof(int32_t), cudaMemcpyDeviceToHost, st));
      BK(cudaStreamSynchronize(st));
      nrows = lf + lp;
    }
    B.view.n = nrows;
    B.view.m = c;
    B.view.src = bs.src_pool + base[b];
    B.view.outdeg = nullptr;
    BK(cudaMallocAsync(&B.view.row, ((int64_t)nrows + 1) * sizeof(int64_t), st));
    track(B.view.row);
    BK(cudaMallocAsync(&B.ids, std::max<int64_t>(nrows, 1) * sizeof(int32_t), st));
    track(B.ids);
    if (c > 0) {
      row_emit_kernel<<<grid_for(c), 256, 0, st>>>(rows + base[b], flag, pos, c, B.view.row, B.ids);
      BK(cudaGetLastError());
    }
    set_last_kernel<<<1, 1, 0, st>>>(B.view.row, nrows, c);
    BK(cudaGetLastError());
    // merge-path task partition of the block (as finish_graph does for the graph)
    const int64_t items = (int64_t)nrows + c;
    const int64_t nt = (items + kTaskDiag - 1) / kTaskDiag;
    Partition& P = B.part;
    P.ntasks = (int32_t)nt;
    BK(cudaMallocAsync(&P.task_row, (nt + 1) * sizeof(int32_t), st));
    track(P.task_row);
    BK(cudaMallocAsync(&P.task_edge, (nt + 1) * sizeof(int64_t), st));
    track(P.task_edge);
    BK(cudaMallocAsync(&P.head_first, (nt + 1) * sizeof(int32_t), st));
    track(P.head_first);
    BK(cudaMallocAsync(&P.clean_start, (nt + 1) * sizeof(int32_t), st));
    track(P.clean_start);
    BK(cudaMallocAsync(&P.task_bits, 8 * (nt + 1) * sizeof(uint32_t), st));
    track(P.task_bits);
    if (nrows > 0) BK(launch_partition(B.view, P, st));
    {
      const int32_t w[4] = {0, (int32_t)nt, 0, 0};
      BK(cudaMallocAsync(&B.waves, sizeof(w), st));
      track(B.waves);
      BK(cudaMemcpyAsync(B.waves, w, sizeof(w), cudaMemcpyHostToDevice, st));
      BK(cudaStreamSynchronize(st));  // w is a stack array
    }
    bs.max_ntasks = std::max<int64_t>(bs.max_ntasks, nt);
    bs.pairs += nrows;
  }
  BK(cudaMallocAsync(&bs.partial, std::max<int64_t>(g.n, 1) * sizeof(double), st));
  track(bs.partial);
  BK(cudaMemsetAsync(bs.partial, 0, std::max<int64_t>(g.n, 1) * sizeof(double), st));
  BK(cudaMallocAsync(&bs.tail_partial, (bs.max_ntasks + 1) * sizeof(double), st));
  track(bs.tail_partial);
  BK(cudaMemsetAsync(bs.tail_partial, 0xFF, (bs.max_ntasks + 1) * sizeof(double), st));
  BK(cudaMallocAsync(&bs.scratch, 8 * sizeof(double), st));
  track(bs.scratch);
  bs.apply_grid = 148 * 8;
  BK(cudaMallocAsync(&bs.cta_pairs, 2 * bs.apply_grid * sizeof(double), st));
  track(bs.cta_pairs);
  BK(cudaStreamSynchronize(st));
out:
  for (void* p : {(void*)erow, (void*)rows, (void*)hist, (void*)offs, (void*)adjust, (void*)flag, (void*)pos, temp})
    if (p) cudaFreeAsync(p, st);
  cudaStreamSynchronize(st);
  if (e != cudaSuccess || *msg) free_blocks(bs, st);
  return e;
}

}  // namespace fprb
