// Random-row gathers through the TMA unit (cp.async.bulk.tensor tile::gather4,
// sm_100a) against the LSU path's ~263 G random 8-B gathers/s ceiling: does
// the TMA unit fetch scattered 16-B rows of an L2-resident vector faster than
// one request per SM clock?
// contrib (2^22 doubles, config 2's 33.5 MB) is viewed as a 2-D tensor of
// 2^21 rows x 2 doubles; each gather4 lands 4 rows (64 B) in shared memory.
// Each warp: lane l issues one gather4 per batch into its 64-B slot, all
// lanes arrive on the warp's mbarrier with expect_tx; two batches in flight.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tma_gather_bench tma_gather_bench.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>
#include <algorithm>
#include <vector>

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

__global__ void fill(int64_t m, uint32_t rows, uint32_t* idx) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += (int64_t)gridDim.x * blockDim.x)
    idx[i] = hash32((uint32_t)i * 2654435761u + 11u) % rows;
}

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}

constexpr int kWarps = 4;
constexpr int kDepth = 2;  // batches in flight per warp

__global__ void __launch_bounds__(kWarps * 32) tma_gather(const __grid_constant__ CUtensorMap tmap, const uint32_t* idx,
                                                          int64_t nbatches_total, double* out) {
  // per warp: kDepth batches x 32 lanes x 64 B
  __shared__ __align__(128) double slot[kWarps][kDepth][32][16];  // 128-B aligned TMA destinations
  __shared__ __align__(8) uint64_t bar[kWarps][kDepth];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  if (lane == 0)
    for (int d = 0; d < kDepth; ++d)
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[warp][d])), "r"(32));
  __syncwarp();
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  const int64_t gw = (int64_t)blockIdx.x * kWarps + warp, nw = (int64_t)gridDim.x * kWarps;
  double acc = 0.0;
  uint32_t phase[kDepth] = {};
  auto issue = [&](int64_t b, int d) {
    const uint4 r = reinterpret_cast<const uint4*>(idx)[b * 32 + lane];
    const uint32_t mb = smem_u32(&bar[warp][d]);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(64) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(&slot[warp][d][lane][0])),
        "l"(&tmap), "r"(0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(mb)
        : "memory");
  };
  int64_t b = gw;
  int d = 0;
  for (int k = 0; k < kDepth && b + (int64_t)k * nw < nbatches_total; ++k) issue(b + (int64_t)k * nw, k);
  for (; b < nbatches_total; b += nw) {
    const uint32_t mb = smem_u32(&bar[warp][d]);
    asm volatile(
        "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(mb),
        "r"(phase[d])
        : "memory");
    phase[d] ^= 1u;
    acc += slot[warp][d][lane][0] + slot[warp][d][lane][3] + slot[warp][d][lane][5] + slot[warp][d][lane][6];
    __syncwarp();
    const int64_t nb = b + (int64_t)kDepth * nw;
    if (nb < nbatches_total) issue(nb, d);
    d = (d + 1) % kDepth;
  }
  if (acc == 12345.678) out[0] = acc;
}

// Mixed: in each 8-warp CTA, warps [0, tw) issue TMA gather4 batches (slots
// in dynamic shared memory, 8 KB per TMA warp); the others do LSU random
// 8-B gathers (ld.global.cg, 8 in flight per lane) of the same vector.
// Reports the aggregate: are the TMA and LSU paths additive?
constexpr int kMixWarps = 8;
__global__ void __launch_bounds__(kMixWarps * 32) mixed(const __grid_constant__ CUtensorMap tmap, const uint32_t* idx,
                                                        int64_t tma_batches, const uint32_t* idx2, int64_t lsu_m,
                                                        const double* vals, int tw, double* out) {
  extern __shared__ __align__(128) double dslot[];  // [tw][kDepth][32][16]
  __shared__ __align__(8) uint64_t bar[kMixWarps][kDepth];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  double acc = 0.0;
  if (warp < tw) {
    double* myslot = dslot + (size_t)warp * kDepth * 32 * 16;
    if (lane == 0)
      for (int d = 0; d < kDepth; ++d)
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[warp][d])), "r"(32));
    __syncwarp();
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const int64_t gw = (int64_t)blockIdx.x * tw + warp, nw = (int64_t)gridDim.x * tw;
    uint32_t phase[kDepth] = {};
    auto issue = [&](int64_t b, int d) {
      const uint4 r = reinterpret_cast<const uint4*>(idx)[b * 32 + lane];
      const uint32_t mb = smem_u32(&bar[warp][d]);
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(mb), "r"(64) : "memory");
      asm volatile(
          "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes"
          " [%0], [%1, {%2, %3, %4, %5, %6}], [%7];" ::"r"(smem_u32(myslot + (d * 32 + lane) * 16)),
          "l"(&tmap), "r"(0), "r"(r.x), "r"(r.y), "r"(r.z), "r"(r.w), "r"(mb)
          : "memory");
    };
    int64_t b = gw;
    int d = 0;
    for (int k = 0; k < kDepth && b + (int64_t)k * nw < tma_batches; ++k) issue(b + (int64_t)k * nw, k);
    for (; b < tma_batches; b += nw) {
      const uint32_t mb = smem_u32(&bar[warp][d]);
      asm volatile(
          "{ .reg .pred p; W: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1; @!p bra W; }" ::"r"(mb),
          "r"(phase[d])
          : "memory");
      phase[d] ^= 1u;
      acc += myslot[(d * 32 + lane) * 16] + myslot[(d * 32 + lane) * 16 + 3];
      __syncwarp();
      const int64_t nb = b + (int64_t)kDepth * nw;
      if (nb < tma_batches) issue(nb, d);
      d = (d + 1) % kDepth;
    }
  } else {
    constexpr int U = 8;
    const int lw = kMixWarps - tw;
    const int64_t t = ((int64_t)blockIdx.x * lw + (warp - tw)) * 32 + lane, nt = (int64_t)gridDim.x * lw * 32;
    for (int64_t e = t; e < lsu_m; e += nt * U) {
      uint32_t s[U];
#pragma unroll
      for (int u = 0; u < U; ++u) s[u] = e + u * nt < lsu_m ? __ldcs(idx2 + e + u * nt) : 0u;
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldcg(vals + s[u]);
#pragma unroll
      for (int u = 0; u < U; ++u) acc += v[u];
    }
  }
  if (acc == 12345.678) out[0] = acc;
}

int main() {
  const uint32_t n = 1u << 22, rows = n / 2;
  const int64_t batches = 1ll << 20;  // TMA-only runs; the mixed ones use up to 4x  // x 32 lanes x 4 rows = 2^27 rows
  const int64_t m = batches * 32 * 4;
  double *vals, *out;
  uint32_t* idx;
  cudaMalloc(&vals, (size_t)n * 8); cudaMalloc(&out, 8); cudaMalloc(&idx, (size_t)m * 4 * 4);
  cudaMemset(vals, 0, (size_t)n * 8);
  fill<<<1024, 256>>>(m * 4, rows, idx);

  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  using Enc = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                           const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                           CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  CUtensorMap tmap;
  cuuint64_t dims[2] = {2, rows};
  cuuint64_t strides[1] = {16};
  cuuint32_t box[2] = {2, 1};
  cuuint32_t estr[2] = {1, 1};
  CUresult cr = ((Enc)fn)(&tmap, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, vals, dims, strides, box, estr,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                          CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  printf("encode: %d\n", (int)cr);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int per_sm : {1, 2, 4, 8, 16}) {
    cudaEvent_t a, e; cudaEventCreate(&a); cudaEventCreate(&e);
    float best = 1e9;
    for (int rep = 0; rep < 4; ++rep) {
      cudaEventRecord(a);
      tma_gather<<<sms * per_sm, kWarps * 32>>>(tmap, idx, batches, out);
      cudaEventRecord(e); cudaEventSynchronize(e);
      float ms; cudaEventElapsedTime(&ms, a, e);
      if (rep && ms < best) best = ms;
    }
    printf("%2d CTAs/SM (%d warps/SM, %d batches in flight/warp): %.3f ms, %.1f G rows/s (%s)\n", per_sm,
           per_sm * kWarps, kDepth, best, m / best / 1e6, cudaGetErrorString(cudaGetLastError()));
  }
  // mixed runs: 6 CTAs of 8 warps per SM = 48 warps; t of each CTA's warps on TMA
  uint32_t* idx2;
  const int64_t lsu_m = 1ll << 29;
  cudaMalloc(&idx2, (size_t)lsu_m * 4);
  fill<<<1024, 256>>>(lsu_m, n, idx2);
  for (int tw : {0, 1, 2, 3}) {
    for (double tfrac : {0.0, 0.15, 0.3, 0.45}) {
      if ((tw == 0) != (tfrac == 0.0)) continue;
      const int64_t tb = (int64_t)(batches * 4 * tfrac);  // TMA rows: tb * 128
      const int64_t lm = (int64_t)(lsu_m * (1.0 - tfrac));
      const size_t dsm = (size_t)std::max(tw, 1) * kDepth * 32 * 16 * 8;
      cudaFuncSetAttribute(mixed, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsm);
      cudaEvent_t a, e; cudaEventCreate(&a); cudaEventCreate(&e);
      float best = 1e9;
      for (int rep = 0; rep < 4; ++rep) {
        cudaEventRecord(a);
        mixed<<<sms * 6, kMixWarps * 32, dsm>>>(tmap, idx, tb, idx2, lm, vals, tw, out);
        cudaEventRecord(e); cudaEventSynchronize(e);
        float ms; cudaEventElapsedTime(&ms, a, e);
        if (rep && ms < best) best = ms;
      }
      const double total = (double)tb * 128 + (double)lm;
      printf("mixed: %d/8 TMA warps, %.0f%% of fetches by TMA: %.3f ms, %.1f G fetches/s (%s)\n", tw,
             100.0 * tb * 128 / total, best, total / best / 1e6, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
