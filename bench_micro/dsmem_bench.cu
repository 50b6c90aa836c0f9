// Random 8-B gathers from a source chunk spread over a thread-block cluster's
// distributed shared memory (DSMEM): the candidate phase-1 gather of the
// propagation-blocked engine (pb.cu) with chunk = cluster x 128 KB.
// Index stream read coalesced (u32: rank << 14 | offset), values written
// sequentially, like phase 1's val stream.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dsmem_bench dsmem_bench.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

namespace cg = cooperative_groups;

constexpr int kPer = 1 << 14;  // doubles per CTA: 128 KB

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

__global__ void fill(long long m, int ranks, uint32_t* idx) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (long long)gridDim.x * blockDim.x)
    idx[i] = hash32((uint32_t)i * 2654435761u + 7u) % (uint32_t)(ranks * kPer);
}

template <int U>
__global__ void __launch_bounds__(1024) gather(const double* prev, const uint32_t* idx, long long m, double* val) {
  extern __shared__ double part[];
  cg::cluster_group cl = cg::this_cluster();
  const unsigned rank = cl.block_rank();
  for (int i = threadIdx.x; i < kPer; i += blockDim.x) part[i] = prev[rank * kPer + i];
  cl.sync();
  const long long nthreads = (long long)gridDim.x * blockDim.x;
  for (long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += nthreads * U) {
    uint32_t s[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long k = e + u * nthreads;
      s[u] = k < m ? __ldcs(idx + k) : 0u;
    }
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const double* p = cl.map_shared_rank(part, s[u] >> 14);
      v[u] = p[s[u] & (kPer - 1)];
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const long long k = e + u * nthreads;
      if (k < m) __stcs(val + k, v[u]);
    }
  }
  cl.sync();  // no CTA may exit while its shared memory can still be read
}

int main() {
  const long long m = 1ll << 30;
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double *prev, *val;
  uint32_t* idx;
  cudaMalloc(&prev, 16ll * kPer * 8); cudaMalloc(&val, m * 8); cudaMalloc(&idx, m * 4);
  cudaMemset(prev, 0, 16ll * kPer * 8);
  for (int cs : {1, 2, 4, 8, 16}) {
    fill<<<sms * 8, 256>>>(m, cs, idx);
    for (int threads : {512, 1024}) {
      cudaFuncSetAttribute(gather<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, kPer * 8);
      cudaFuncSetAttribute(gather<8>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
      cudaLaunchConfig_t cfg = {};
      cudaLaunchAttribute attr[1];
      attr[0].id = cudaLaunchAttributeClusterDimension;
      attr[0].val.clusterDim.x = cs; attr[0].val.clusterDim.y = 1; attr[0].val.clusterDim.z = 1;
      cfg.attrs = attr; cfg.numAttrs = 1;
      cfg.blockDim = dim3(threads);
      cfg.dynamicSmemBytes = kPer * 8;
      int nclusters = 0;
      cfg.gridDim = dim3(cs);
      cudaOccupancyMaxActiveClusters(&nclusters, gather<8>, &cfg);
      cfg.gridDim = dim3(nclusters * cs);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      float best = 1e9;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(a);
        cudaLaunchKernelEx(&cfg, gather<8>, (const double*)prev, (const uint32_t*)idx, m, val);
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        if (rep && ms < best) best = ms;
      }
      printf("cluster %2d x %4d threads, %3d clusters (%d CTAs): %.3f ms, %.1f G gathers/s (%s)\n", cs, threads,
             nclusters, nclusters * cs, best, m / best / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
