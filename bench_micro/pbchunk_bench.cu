// Shared-memory-chunk propagation-blocking gather, measured in isolation:
// can a phase-1 pass that stages a source chunk in shared memory and gathers
// from it beat the L2-window gather pass (request-bound at ~263 G/s)?
// Entries are chunk-major; each holds a 16-bit source offset in its chunk and
// the int64 position of its value slot in the bin-major value array (runs of
// R consecutive slots, as the (bin, chunk) segments would be).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pbchunk_bench pbchunk_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

__global__ void fill(long long m, int C, int R, long long nruns, uint16_t* srcl, long long* pos, int scatter) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
    srcl[i] = (uint16_t)(hash32((uint32_t)i * 2654435761u + 7u) % (uint32_t)C);
    const long long run = i / R;
    const long long slot = scatter ? (long long)(((uint64_t)hash32((uint32_t)run) << 20 ^ hash32((uint32_t)run + 99u)) % (uint64_t)nruns) : run;
    pos[i] = slot * R + (i % R);
  }
}

// CTA per item (a piece of one chunk); the chunk's contributions are staged
// in shared memory, reloaded only when the chunk changes.
template <int U>
__global__ void __launch_bounds__(1024) phase1(const double* prev, const uint16_t* srcl, const long long* pos,
                                               long long per_chunk, long long piece, long long nitems, int C,
                                               double* val, unsigned long long* ctr) {
  extern __shared__ double chunk[];
  __shared__ long long s_item;
  long long have = -1;
  for (;;) {
    if (threadIdx.x == 0) s_item = (long long)atomicAdd(ctr, 1ull);
    __syncthreads();
    const long long it = s_item;
    if (it >= nitems) break;
    const long long pieces = per_chunk / piece;
    const long long c = it / pieces;
    if (c != have) {
      for (int i = threadIdx.x; i < C; i += blockDim.x) chunk[i] = __ldcs(prev + c * C + i);
      have = c;
    }
    __syncthreads();
    const long long e0 = c * per_chunk + (it % pieces) * piece, e1 = e0 + piece;
    for (long long e = e0 + threadIdx.x; e < e1; e += (long long)blockDim.x * U) {
      uint16_t s[U];
      long long p[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const long long k = e + (long long)u * blockDim.x;
        s[u] = k < e1 ? __ldcs(srcl + k) : 0;
        p[u] = k < e1 ? __ldcs(pos + k) : -1;
      }
#pragma unroll
      for (int u = 0; u < U; ++u)
        if (p[u] >= 0) __stcs(val + p[u], chunk[s[u]]);
    }
    __syncthreads();
  }
}

int main() {
  const int C = 1 << 14;            // sources per chunk: 128 KB of fp64
  const long long n = 1ll << 26;    // config 4's vertex count
  const long long m = 1ll << 30;    // ~config 4's edge count
  const long long nchunks = n / C, per_chunk = m / nchunks;
  double *prev, *val;
  uint16_t* srcl;
  long long* pos;
  unsigned long long* ctr;
  cudaMalloc(&prev, n * 8); cudaMalloc(&val, m * 8); cudaMalloc(&srcl, m * 2); cudaMalloc(&pos, m * 8);
  cudaMalloc(&ctr, 8);
  cudaMemset(prev, 0, n * 8);
  cudaFuncSetAttribute(phase1<4>, cudaFuncAttributeMaxDynamicSharedMemorySize, C * 8);
  cudaFuncSetAttribute(phase1<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, C * 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int scatter = 0; scatter < 2; ++scatter) {
    for (int R : {4, 8, 16, 32}) {
      if (!scatter && R != 8) continue;
      fill<<<sms * 8, 256>>>(m, C, R, m / R, srcl, pos, scatter);
      for (long long piece : {1ll << 16, 1ll << 18}) {
        for (int u : {4, 8}) {
          const long long nitems = m / piece;
          cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
          float best = 1e9;
          for (int rep = 0; rep < 4; ++rep) {
            cudaMemset(ctr, 0, 8);
            cudaEventRecord(a);
            if (u == 4) phase1<4><<<sms, 1024, C * 8>>>(prev, srcl, pos, per_chunk, piece, nitems, C, val, ctr);
            else phase1<8><<<sms, 1024, C * 8>>>(prev, srcl, pos, per_chunk, piece, nitems, C, val, ctr);
            cudaEventRecord(b); cudaEventSynchronize(b);
            float ms; cudaEventElapsedTime(&ms, a, b);
            if (rep && ms < best) best = ms;
          }
          const double bytes = (double)m * 18 + (double)nitems * C * 8;
          printf("scatter=%d run=%2d piece=2^%d U=%d: %.3f ms, %.1f G entries/s, %.0f GB/s (18 B/entry + chunk loads) %s\n",
                 scatter, R, piece == (1ll << 16) ? 16 : 18, u, best, m / best / 1e6, bytes / best / 1e6,
                 cudaGetErrorString(cudaGetLastError()));
        }
      }
    }
  }
  return 0;
}
