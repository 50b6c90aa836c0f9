// Bin accumulation throughput on B200, the phase-2 cost of a propagation-
// blocked sweep: stream (val, dstl) of one bin and add val into the bin's row
// accumulator.  Modes: shared fp64 atomicAdd (a CAS loop on sm_100a), shared
// u64 / fp32 atomics (native), global fp64 RED into an L2-resident slice, and
// the plain stream as the bandwidth floor.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 satom_bench.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

__global__ void fill(double* v, uint16_t* d, long long m, int R) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x) {
    uint32_t h = hash32((uint32_t)i * 2654435761u + 7u);
    v[i] = (h & 1023) * 1e-9;
    d[i] = (uint16_t)(hash32(h) % (uint32_t)R);
  }
}

template <int MODE>
__global__ void accum(const double* v, const uint16_t* d, long long per_bin, long long nbins, int R, double* gacc,
                      double* out) {
  extern __shared__ double acc[];
  unsigned long long* iacc = reinterpret_cast<unsigned long long*>(acc);
  float* facc = reinterpret_cast<float*>(acc);
  double tot = 0;
  for (long long b = blockIdx.x; b < nbins; b += gridDim.x) {
    for (int i = threadIdx.x; i < R; i += blockDim.x) acc[i] = 0;
    __syncthreads();
    const long long e0 = b * per_bin, e1 = e0 + per_bin;
    double* g = gacc + (long long)blockIdx.x * R;
    for (long long e = e0 + threadIdx.x; e < e1; e += blockDim.x) {
      const double x = __ldg(v + e);
      const int k = __ldg(d + e);
      if (MODE == 0) atomicAdd(&acc[k], x);
      else if (MODE == 1) atomicAdd(&iacc[k], (unsigned long long)(x * 1e18));
      else if (MODE == 2) atomicAdd(&facc[k], (float)x);
      else if (MODE == 3) atomicAdd(&g[k], x);
      else tot += x + k;
    }
    __syncthreads();
    for (int i = threadIdx.x; i < R; i += blockDim.x) tot += acc[i] + (MODE == 3 ? g[i] : 0.0);
    __syncthreads();
  }
  if (tot == 12345.678) out[0] = tot;
}

template <int MODE>
float run(const double* v, const uint16_t* d, long long m, int R, int threads, int ctas_per_sm, int sms, double* gacc,
          double* out) {
  const long long per_bin = 1ll << 16;  // entries per bin
  const long long nbins = m / per_bin;
  const size_t smem = (size_t)R * 8;
  cudaFuncSetAttribute(accum<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  const int grid = sms * ctas_per_sm;
  accum<MODE><<<grid, threads, smem>>>(v, d, per_bin, nbins, R, gacc, out);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  for (int r = 0; r < 5; ++r) accum<MODE><<<grid, threads, smem>>>(v, d, per_bin, nbins, R, gacc, out);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) printf("error %s\n", cudaGetErrorString(e));
  return ms / 5;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const long long m = 1ll << 28;
  double* v; uint16_t* d; double* out; double* gacc;
  cudaMalloc(&v, m * 8); cudaMalloc(&d, m * 2); cudaMalloc(&out, 8);
  cudaMalloc(&gacc, (size_t)sms * 8 * 16384 * 8);
  cudaMemset(gacc, 0, (size_t)sms * 8 * 16384 * 8);
  const char* names[] = {"smem f64 CAS", "smem u64", "smem f32", "global RED f64 (L2)", "stream only"};
  for (int R : {16384, 8192, 4096}) {
    fill<<<1024, 256>>>(v, d, m, R);
    cudaDeviceSynchronize();
    for (int cps : {1, 2, 3}) {
      if ((size_t)R * 8 * cps > 220 * 1024) continue;
      float t[5];
      t[0] = run<0>(v, d, m, R, 1024, cps, sms, gacc, out);
      t[1] = run<1>(v, d, m, R, 1024, cps, sms, gacc, out);
      t[2] = run<2>(v, d, m, R, 1024, cps, sms, gacc, out);
      t[3] = run<3>(v, d, m, R, 1024, cps, sms, gacc, out);
      t[4] = run<4>(v, d, m, R, 1024, cps, sms, gacc, out);
      for (int i = 0; i < 5; ++i)
        printf("R=%5d ctas/sm=%d %-22s %8.3f ms  %7.1f G entries/s  %6.0f GB/s\n", R, cps, names[i], t[i],
               m / (t[i] * 1e6), m * 10.0 / (t[i] * 1e6));
    }
  }
  return 0;
}
