// Random 8-B gather throughput on B200: the hardware ceiling for the PageRank
// pull gather (contrib[in_src[e]]).  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
#include <cstdio>
#include <cstdint>
#include <vector>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

// idx stream read coalesced (like in_src), values gathered; U loads in flight per thread.
template <int U, int MODE>
__global__ void gather(const int* __restrict__ idx, const double* vals, long long m, double* out) {
  double acc = 0;
  long long stride = (long long)gridDim.x * blockDim.x * U;
  for (long long base = ((long long)blockIdx.x * blockDim.x) * U + threadIdx.x; base < m; base += stride) {
    int s[U];
#pragma unroll
    for (int u = 0; u < U; ++u) { long long e = base + (long long)u * blockDim.x; s[u] = e < m ? __ldg(idx + e) : 0; }
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      if (MODE == 0) v[u] = vals[s[u]];
      else if (MODE == 1) v[u] = __ldcg(vals + s[u]);
      else if (MODE == 2) { double2 t = __ldcg(reinterpret_cast<const double2*>(vals) + (s[u] >> 1)); v[u] = (s[u] & 1) ? t.y : t.x; }
      else { v[u] = __ldg(vals + s[u]); }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (acc == 12345.678) out[0] = acc;
}

__global__ void fill_idx(int* idx, long long m, int n, int sorted_run) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
    idx[i] = (int)(hash32((uint32_t)i * 2654435761u + 12345u) % (uint32_t)n);
  }
}

template <int U, int MODE>
float run(const int* idx, const double* vals, long long m, double* out, int blocks, int threads) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  gather<U, MODE><<<blocks, threads>>>(idx, vals, m, out);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) gather<U, MODE><<<blocks, threads>>>(idx, vals, m, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  return ms / 5;
}

int main(int argc, char** argv) {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  if (argc > 1) {  // "one": a single config-2-shaped launch (n = 2^22, 8 CTAs/SM, U=8, ld.cg) for ncu
    const long long m1 = 1ll << 26;
    const int n1 = 1 << 22;
    int* idx1; double* vals1; double* out1;
    cudaMalloc(&idx1, m1 * 4); cudaMalloc(&out1, 8); cudaMalloc(&vals1, (size_t)n1 * 8);
    cudaMemset(vals1, 0, (size_t)n1 * 8);
    fill_idx<<<1024, 256>>>(idx1, m1, n1, 0);
    cudaDeviceSynchronize();
    const float t = run<8, 1>(idx1, vals1, m1, out1, sms * 8, 256);
    printf("n=%d: %.1f G gathers/s (%.3f ms per 2^26 gathers)\n", n1, m1 / t / 1e6, t);
    if (argc > 2) {  // "one all": the load flavours side by side
      const float tl = run<8, 0>(idx1, vals1, m1, out1, sms * 8, 256);
      const float tg = run<8, 3>(idx1, vals1, m1, out1, sms * 8, 256);
      const float t20 = run<8, 1>(idx1, vals1, m1, out1, sms * 5, 128);
      printf("ld.ca %.1f  ld.nc(__ldg) %.1f  ld.cg at 20 warps/SM %.1f G/s\n", m1 / tl / 1e6, m1 / tg / 1e6,
             m1 / t20 / 1e6);
    }
    return 0;
  }
  const long long m = 1ll << 26;
  int* idx; double* vals; double* out;
  cudaMalloc(&idx, m * 4); cudaMalloc(&out, 8);
  const int nmax = 1 << 28;
  cudaMalloc(&vals, (size_t)nmax * 8);
  cudaMemset(vals, 0, (size_t)nmax * 8);
  for (int n : {1 << 16, 1 << 20, 1 << 22, 1 << 24, 1 << 26, 1 << 28}) {
    fill_idx<<<1024, 256>>>(idx, m, n, 0);
    cudaDeviceSynchronize();
    for (int occ : {4, 8, 16}) {
      int blocks = sms * occ, threads = 256;
      float t0 = run<8, 0>(idx, vals, m, out, blocks, threads);
      float t1 = run<8, 1>(idx, vals, m, out, blocks, threads);
      float t2 = run<8, 2>(idx, vals, m, out, blocks, threads);
      float t3 = run<16, 1>(idx, vals, m, out, blocks, threads);
      float t4 = run<4, 1>(idx, vals, m, out, blocks, threads);
      printf("n=%9d (%6.1f MB) blocks/SM=%2d  G gathers/s: ld %.1f  ldcg %.1f  ldcg16B %.1f  ldcg U16 %.1f  ldcg U4 %.1f\n",
             n, n * 8.0 / 1e6, occ, m / t0 / 1e6, m / t1 / 1e6, m / t2 / 1e6, m / t3 / 1e6, m / t4 / 1e6);
    }
  }
  cudaError_t e = cudaGetLastError();
  printf("status %s\n", cudaGetErrorString(e));
  return 0;
}
