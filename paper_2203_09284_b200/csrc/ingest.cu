// ingest.cu -- SNAP edge-list text -> EdgeSet on the device (SURVEY.md §8(f)
// rank 4; fpr::parse_edge_list, edge_list.hpp:33-80).
//
// The reference reads the text with std::getline, tokenises each line, parses
// the two ids with std::from_chars and compacts sparse ids through an
// unordered_map in first-appearance order, one line at a time.  Here:
//   1. newline positions (tile count, scan, tile write)        -> line bounds;
//   2. one thread per line classifies it exactly as the reference does
//      (empty / '#' / '%' / whitespace-only -> skipped; else two decimal u64
//      tokens separated by ' ', '\t', '\r', nothing after) and records the
//      first malformed line with an atomicMin, so the reported error is the
//      one the sequential parser throws;
//   3. edge lines are compacted in line order (CUB select);
//   4. first-appearance compaction of the 2m raw ids without a hash table:
//      stable radix sort of (raw id, position), segment heads mark first
//      occurrences, an exclusive scan over positions numbers them in
//      appearance order, and every occurrence takes its segment head's number.
// The result (2m int32 dense ids in edge order) feeds the K4 CSR build.
#include <cub/cub.cuh>

#include <algorithm>
#include <cstdint>

#include "internal.cuh"

namespace fprb {

namespace {

__device__ __forceinline__ bool is_ws(unsigned char c) { return c == ' ' || c == '\t' || c == '\r'; }

struct MaxU32 {
  __device__ __forceinline__ uint32_t operator()(uint32_t a, uint32_t b) const { return a > b ? a : b; }
};

__device__ __forceinline__ void line_bounds(const int64_t* nl, int64_t n_nl, int64_t len, int64_t k,
                                            int64_t& b, int64_t& e) {
  b = k == 0 ? 0 : __ldg(nl + k - 1) + 1;
  e = k < n_nl ? __ldg(nl + k) : len;
}

// One line, as edge_list.hpp:48-76 treats it.  Returns 0 skipped, 1 edge,
// or FPR_B200_PARSE_* + 1 ... encoded as kind + 1 (2 tokens, 3 bad token,
// 4 trailing); [tb, te) = the offending token for a bad token.
__device__ int parse_line(const unsigned char* t, int64_t b, int64_t e, uint64_t& v0, uint64_t& v1,
                          int64_t& tb, int64_t& te) {
  if (b == e) return 0;                          // line.empty()
  const unsigned char c0 = __ldg(t + b);
  if (c0 == '#' || c0 == '%') return 0;          // comment (first byte only)
  int64_t i = b;
  while (i < e && is_ws(__ldg(t + i))) ++i;
  if (i == e) return 0;                          // only " \t\r"
  uint64_t v[2];
  for (int k = 0; k < 2; ++k) {
    while (i < e && is_ws(__ldg(t + i))) ++i;
    if (i == e) return 2;                        // "expected two integer tokens"
    const int64_t s = i;
    while (i < e && !is_ws(__ldg(t + i))) ++i;
    // std::from_chars(base 10) over the whole token: digits only, no sign,
    // value <= 2^64-1.
    uint64_t x = 0;
    bool ok = true;
    for (int64_t j = s; j < i; ++j) {
      const unsigned d = (unsigned)__ldg(t + j) - (unsigned)'0';
      if (d > 9u || x > (~0ull - d) / 10ull) {
        ok = false;
        break;
      }
      x = x * 10ull + d;
    }
    if (!ok) {
      tb = s;
      te = i;
      return 3;                                  // "bad token '...'"
    }
    v[k] = x;
  }
  while (i < e && is_ws(__ldg(t + i))) ++i;
  if (i != e) return 4;                          // "trailing characters after edge"
  v0 = v[0];
  v1 = v[1];
  return 1;
}

// Newline positions without a per-byte select: tiles of kTile bytes (one CTA,
// 64 bytes per thread as four 16-B loads), counted in pass 1, scanned, then
// re-read in pass 2 where a block scan orders each thread's positions.
constexpr int kNlThreads = 256;
constexpr int kNlBytes = 64;  // per thread
constexpr int64_t kTile = (int64_t)kNlThreads * kNlBytes;

__device__ __forceinline__ int newline_mask16(const unsigned char* t, int64_t base, int64_t len, uint32_t& mask) {
  mask = 0;
  if (base + 16 <= len) {
    const uint4 w = __ldg(reinterpret_cast<const uint4*>(t + base));
    const unsigned x[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const unsigned eq = __vcmpeq4(x[q], 0x0a0a0a0au);  // 0xff per matching byte
      // bit b of the 4-bit group = byte b matches
      const unsigned nib = (eq & 1u) | ((eq >> 7) & 2u) | ((eq >> 14) & 4u) | ((eq >> 21) & 8u);
      mask |= nib << (4 * q);
    }
  } else {
    for (int64_t i = base; i < len && i < base + 16; ++i)
      if (__ldg(t + i) == '\n') mask |= 1u << (i - base);
  }
  return __popc(mask);
}

__global__ void __launch_bounds__(kNlThreads) nl_count_kernel(const unsigned char* t, int64_t len,
                                                              uint64_t* tile_count) {
  const int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kNlBytes;
  int c = 0;
#pragma unroll
  for (int q = 0; q < kNlBytes / 16; ++q) {
    uint32_t m;
    if (base + 16 * q < len) c += newline_mask16(t, base + 16 * q, len, m);
  }
  using BR = cub::BlockReduce<int, kNlThreads>;
  __shared__ typename BR::TempStorage tmp;
  const int total = BR(tmp).Sum(c);
  if (threadIdx.x == 0) tile_count[blockIdx.x] = (uint64_t)total;
}

__global__ void __launch_bounds__(kNlThreads) nl_write_kernel(const unsigned char* t, int64_t len,
                                                              const uint64_t* tile_off, int64_t* nl) {
  const int64_t base = (int64_t)blockIdx.x * kTile + (int64_t)threadIdx.x * kNlBytes;
  uint32_t masks[kNlBytes / 16];
  int c = 0;
#pragma unroll
  for (int q = 0; q < kNlBytes / 16; ++q) {
    masks[q] = 0;
    if (base + 16 * q < len) c += newline_mask16(t, base + 16 * q, len, masks[q]);
  }
  using BS = cub::BlockScan<int, kNlThreads>;
  __shared__ typename BS::TempStorage tmp;
  int off;
  BS(tmp).ExclusiveSum(c, off);
  int64_t* out = nl + tile_off[blockIdx.x] + off;
#pragma unroll
  for (int q = 0; q < kNlBytes / 16; ++q) {
    uint32_t m = masks[q];
    while (m) {
      const int b = __ffs(m) - 1;
      m &= m - 1;
      *out++ = base + 16 * q + b;
    }
  }
}

__global__ void parse_lines_kernel(const unsigned char* t, const int64_t* nl, int64_t n_nl, int64_t len,
                                   int64_t nlines, ulonglong2* vals, uint8_t* is_edge,
                                   unsigned long long* first_err) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nlines; k += stride) {
    int64_t b, e, tb, te;
    line_bounds(nl, n_nl, len, k, b, e);
    uint64_t v0 = 0, v1 = 0;
    const int r = parse_line(t, b, e, v0, v1, tb, te);
    is_edge[k] = r == 1;
    vals[k] = make_ulonglong2(v0, v1);
    if (r >= 2) atomicMin(first_err, (unsigned long long)k);
  }
}

// Re-parses the first malformed line for its error kind and token range.
__global__ void error_detail_kernel(const unsigned char* t, const int64_t* nl, int64_t n_nl, int64_t len,
                                    int64_t k, int64_t* out) {
  int64_t b, e, tb = 0, te = 0;
  line_bounds(nl, n_nl, len, k, b, e);
  uint64_t v0, v1;
  out[0] = parse_line(t, b, e, v0, v1, tb, te) - 1;  // FPR_B200_PARSE_*
  out[1] = tb;
  out[2] = te;
}

__global__ void iota_kernel(uint32_t* p, int64_t n) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) p[i] = (uint32_t)i;
}

// sorted (key, pos): first[pos] = 1 at a segment head (first occurrence of a
// raw id, the stable sort keeps positions ascending within a segment);
// hidx[i] = i at heads, else 0 (a max-scan then yields each i's head).
__global__ void heads_kernel(const uint64_t* keys, const uint32_t* pos, int64_t n, uint32_t* first,
                             uint32_t* hidx) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const bool h = i == 0 || keys[i] != keys[i - 1];
    if (h) first[pos[i]] = 1u;  // first[] zeroed: n scattered writes, not N
    hidx[i] = h ? (uint32_t)i : 0u;
  }
}

__global__ void dense_kernel(const uint32_t* pos, const uint32_t* head, const uint32_t* rank, int64_t n,
                             int32_t* dense) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    dense[pos[i]] = (int32_t)rank[pos[head[i]]];
}

int grid_for(int64_t work) {
  const int64_t b = (work + 255) / 256;
  return (int)std::max<int64_t>(1, std::min<int64_t>(b, 148ll * 16));
}

#define IK(x)                       \
  do {                              \
    e = (x);                        \
    if (e != cudaSuccess) goto out; \
  } while (0)

template <class T>
cudaError_t alloc(T** p, int64_t count, cudaStream_t st) {
  return cudaMallocAsync((void**)p, (size_t)std::max<int64_t>(count, 1) * sizeof(T), st);
}

}  // namespace

cudaError_t ingest_edge_list(const unsigned char* t, uint64_t len, bool ends_with_newline, cudaStream_t st,
                             Ingested& out, IngestError& err, const char** msg) {
  cudaError_t e = cudaSuccess;
  unsigned long long* scal = nullptr;  // [1] first error line
  uint64_t* tile_count = nullptr;
  uint64_t* tile_off = nullptr;
  int64_t* nl = nullptr;
  int64_t* d_sel = nullptr;
  ulonglong2* vals = nullptr;
  ulonglong2* pairs = nullptr;
  uint8_t* is_edge = nullptr;
  uint64_t* keys_alt = nullptr;
  uint32_t *pos = nullptr, *pos_alt = nullptr, *first = nullptr, *rank = nullptr, *hidx = nullptr;
  uint64_t* dmax = nullptr;
  int64_t* detail = nullptr;
  void* temp = nullptr;
  size_t temp_bytes = 0;
  unsigned long long h_scal[3] = {0, 0, 0};
  int64_t n_nl = 0, nlines = 0, m = 0, N = 0;
  out = Ingested{};
  err = IngestError{};

  IK(alloc(&scal, 3, st));
  IK(alloc(&d_sel, 1, st));
  IK(cudaMemsetAsync(scal, 0, 3 * sizeof(unsigned long long), st));
  IK(cudaMemsetAsync(scal + 1, 0xFF, sizeof(unsigned long long), st));
  if (len > 0) {
    const int64_t tiles = ((int64_t)len + kTile - 1) / kTile;
    if (tiles >= (1ll << 31)) {
      *msg = "edge-list text too large";
      goto out;
    }
    IK(alloc(&tile_count, tiles, st));
    IK(alloc(&tile_off, tiles + 1, st));
    nl_count_kernel<<<(unsigned)tiles, kNlThreads, 0, st>>>(t, (int64_t)len, tile_count);
    IK(cudaGetLastError());
    size_t tb = 0;
    IK(cub::DeviceScan::ExclusiveSum(nullptr, tb, tile_count, tile_off, tiles, st));
    IK(alloc((unsigned char**)&temp, (int64_t)tb, st));
    IK(cub::DeviceScan::ExclusiveSum(temp, tb, tile_count, tile_off, tiles, st));
    IK(cudaFreeAsync(temp, st));
    temp = nullptr;
    uint64_t last_off = 0;
    uint64_t last_cnt = 0;
    IK(cudaMemcpyAsync(&last_off, tile_off + tiles - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    IK(cudaMemcpyAsync(&last_cnt, tile_count + tiles - 1, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    IK(cudaStreamSynchronize(st));
    n_nl = (int64_t)(last_off + last_cnt);
    IK(alloc(&nl, n_nl, st));
    if (n_nl > 0) {
      nl_write_kernel<<<(unsigned)tiles, kNlThreads, 0, st>>>(t, (int64_t)len, tile_off, nl);
      IK(cudaGetLastError());
    }
  }
  // std::getline: one line per '\n', plus a final unterminated line.
  nlines = n_nl + ((len > 0 && !ends_with_newline) ? 1 : 0);
  if (nlines == 0) goto out;
  IK(alloc(&vals, nlines, st));
  IK(alloc(&is_edge, nlines, st));
  parse_lines_kernel<<<grid_for(nlines), 256, 0, st>>>(t, nl, n_nl, (int64_t)len, nlines, vals, is_edge,
                                                       scal + 1);
  IK(cudaGetLastError());
  IK(cudaMemcpyAsync(h_scal + 1, scal + 1, sizeof(unsigned long long), cudaMemcpyDeviceToHost, st));
  IK(cudaStreamSynchronize(st));
  if (h_scal[1] != ~0ull) {
    int64_t h_detail[3] = {0, 0, 0};
    IK(alloc(&detail, 3, st));
    error_detail_kernel<<<1, 1, 0, st>>>(t, nl, n_nl, (int64_t)len, (int64_t)h_scal[1], detail);
    IK(cudaGetLastError());
    IK(cudaMemcpyAsync(h_detail, detail, sizeof(h_detail), cudaMemcpyDeviceToHost, st));
    IK(cudaStreamSynchronize(st));
    err.line = h_scal[1] + 1;
    err.kind = (int)h_detail[0];
    if (err.kind == 2 && h_detail[2] > h_detail[1]) {
      err.token.resize((size_t)(h_detail[2] - h_detail[1]));
      IK(cudaMemcpyAsync(&err.token[0], t + h_detail[1], err.token.size(), cudaMemcpyDeviceToHost, st));
      IK(cudaStreamSynchronize(st));
    }
    goto out;
  }
  // edge lines, in line order
  IK(alloc(&pairs, nlines, st));
  {
    size_t tb = 0;
    IK(cub::DeviceSelect::Flagged(nullptr, tb, vals, is_edge, pairs, d_sel, nlines, st));
    IK(alloc((unsigned char**)&temp, (int64_t)tb, st));
    IK(cub::DeviceSelect::Flagged(temp, tb, vals, is_edge, pairs, d_sel, nlines, st));
    IK(cudaFreeAsync(temp, st));
    temp = nullptr;
  }
  IK(cudaFreeAsync(vals, st));
  vals = nullptr;
  IK(cudaMemcpyAsync(&m, d_sel, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  IK(cudaStreamSynchronize(st));
  if (m == 0) goto out;
  N = 2 * m;
  if (N >= (1ll << 32)) {
    *msg = "edge list has 2^31 or more edges (one call handles fewer)";
    goto out;
  }
  // first-appearance compaction of the N raw ids (positions 2e, 2e+1)
  {
    uint64_t* keys = reinterpret_cast<uint64_t*>(pairs);
    uint64_t hmax = 0;
    IK(alloc(&keys_alt, N, st));
    IK(alloc(&pos, N, st));
    IK(alloc(&pos_alt, N, st));
    IK(alloc(&dmax, 1, st));
    size_t tb = 0;
    IK(cub::DeviceReduce::Max(nullptr, tb, keys, dmax, N, st));
    temp_bytes = std::max(temp_bytes, tb);
    {
      cub::DoubleBuffer<uint64_t> dk(keys, keys_alt);
      cub::DoubleBuffer<uint32_t> dv(pos, pos_alt);
      tb = 0;
      IK(cub::DeviceRadixSort::SortPairs(nullptr, tb, dk, dv, N, 0, 64, st));
      temp_bytes = std::max(temp_bytes, tb);
    }
    tb = 0;
    IK(cub::DeviceScan::ExclusiveSum(nullptr, tb, pos, pos_alt, N, st));
    temp_bytes = std::max(temp_bytes, tb);
    tb = 0;
    IK(cub::DeviceScan::InclusiveScan(nullptr, tb, pos, pos_alt, MaxU32{}, N, st));
    temp_bytes = std::max(temp_bytes, tb);
    IK(alloc((unsigned char**)&temp, (int64_t)temp_bytes, st));
    tb = temp_bytes;
    IK(cub::DeviceReduce::Max(temp, tb, keys, dmax, N, st));
    IK(cudaMemcpyAsync(&hmax, dmax, sizeof(uint64_t), cudaMemcpyDeviceToHost, st));
    iota_kernel<<<grid_for(N), 256, 0, st>>>(pos, N);
    IK(cudaGetLastError());
    IK(cudaStreamSynchronize(st));
    int bits = 1;
    while (bits < 64 && (hmax >> bits) != 0) ++bits;
    cub::DoubleBuffer<uint64_t> dk(keys, keys_alt);
    cub::DoubleBuffer<uint32_t> dv(pos, pos_alt);
    tb = temp_bytes;
    IK(cub::DeviceRadixSort::SortPairs(temp, tb, dk, dv, N, 0, bits, st));
    const uint64_t* sk = dk.Current();
    const uint32_t* sp = dv.Current();
    // scratch reuse: the non-current buffers are free after the sort
    uint32_t* spare_pos = dv.Alternate();
    IK(alloc(&first, N, st));
    IK(alloc(&rank, N, st));
    hidx = spare_pos;
    IK(cudaMemsetAsync(first, 0, N * sizeof(uint32_t), st));
    heads_kernel<<<grid_for(N), 256, 0, st>>>(sk, sp, N, first, hidx);
    IK(cudaGetLastError());
    tb = temp_bytes;
    IK(cub::DeviceScan::ExclusiveSum(temp, tb, first, rank, N, st));
    tb = temp_bytes;
    uint32_t* head = reinterpret_cast<uint32_t*>(dk.Alternate());  // free after the sort
    IK(cub::DeviceScan::InclusiveScan(temp, tb, hidx, head, MaxU32{}, N, st));
    uint32_t last_first = 0, last_rank = 0;
    IK(cudaMemcpyAsync(&last_first, first + N - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    IK(cudaMemcpyAsync(&last_rank, rank + N - 1, sizeof(uint32_t), cudaMemcpyDeviceToHost, st));
    IK(alloc(&out.pairs, N, st));
    dense_kernel<<<grid_for(N), 256, 0, st>>>(sp, head, rank, N, out.pairs);
    IK(cudaGetLastError());
    IK(cudaStreamSynchronize(st));
    out.m = m;
    out.n = (uint64_t)last_rank + last_first;
  }
out:
  for (void* p : {(void*)scal, (void*)tile_count, (void*)tile_off, (void*)nl, (void*)d_sel, (void*)vals, (void*)pairs, (void*)is_edge,
                  (void*)keys_alt, (void*)pos, (void*)pos_alt, (void*)first, (void*)rank, (void*)dmax,
                  (void*)detail, temp})
    if (p) cudaFreeAsync(p, st);
  if (e != cudaSuccess || *msg || err.line) {
    if (out.pairs) cudaFreeAsync(out.pairs, st);
    out = Ingested{};
  }
  cudaStreamSynchronize(st);
  return e;
}

}  // namespace fprb
