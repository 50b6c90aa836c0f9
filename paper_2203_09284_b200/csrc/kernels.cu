// kernels.cu -- the B200 PageRank hot path (sm_100a).
//
// K1 (EC Jacobi), K2 (FusEd block-async / wave-lockstep Gauss-Seidel) and K3
// (grid residual reduction) are ONE persistent cooperative kernel per solve:
// the convergence loop of pagerank_ec_seq / pagerank_fused_seq
// (/root/reference/proj/include/fpr/pagerank.hpp:136-142, :166-186) runs on
// the device, with one software grid barrier per sweep (plus one per wave in
// the lockstep schedule) and the stop predicate `error <= threshold`
// (:141, :185) evaluated identically by every CTA.
//
// Work unit: a warp task = kTaskItems consecutive items of the merge path of
// (row ends, edges) -- the pull restatement of scatter+gather:
//   * the task's in_src slice is streamed coalesced (4 B/edge, L1 no-allocate,
//     L2 evict-first so the rank vector stays L2-resident) and its
//     contrib[src] values gathered (8 B/edge) into a per-warp smem buffer;
//   * rows whose segment lies inside the task are summed lane-per-row in
//     ascending-src order (bit-identical to gather_ranks_jacobi, :85-87);
//     rows longer than 32 in-task edges are summed warp-cooperatively;
//   * rows split across tasks (hubs) publish per-task partials; the task that
//     holds the row's end combines them in task order -> deterministic;
//   * the update `base + damping*sum` (:88) uses __dmul_rn/__dadd_rn (no FMA
//     contraction, matching the reference's -O3 x86-64 build) and
//     contrib = value / (double)out_degree uses __ddiv_rn (:69,:177).
#include <cstdint>
#include <cstdio>

#include "internal.cuh"

namespace fprb {

#define FULL_MASK 0xffffffffu

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ int32_t ld_stream_i32(const int32_t* p, unsigned long long pol) {
  int32_t v;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
               : "=r"(v)
               : "l"(p), "l"(pol));
  return v;
}
__device__ __forceinline__ unsigned long long evict_first_policy() {
  unsigned long long pol;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
  return pol;
}
__device__ __forceinline__ double ld_relaxed_f64(const double* p) {
  double v;
  asm volatile("ld.relaxed.gpu.global.f64 %0, [%1];" : "=d"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed_f64(double* p, double v) {
  asm volatile("st.relaxed.gpu.global.f64 [%0], %1;" ::"l"(p), "d"(v) : "memory");
}
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release_u32(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned long long globaltimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(FULL_MASK, v, o);
  return v;
}
__device__ __forceinline__ double warp_max(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(FULL_MASK, v, o));
  return v;
}

// ------------------------------------------------------------- grid barrier
// Sense-by-generation barrier over co-resident CTAs (cooperative launch).
// Thread 0 of each CTA fences (release), arrives, and spins on the generation
// word with acquire loads; the trailing __threadfence invalidates this SM's L1
// so plain loads after the barrier observe every CTA's pre-barrier stores.
__device__ __forceinline__ void grid_sync(GridBar* bar) {
  __syncthreads();
  if (threadIdx.x == 0) {
    const unsigned gen = ld_acquire_u32(&bar->gen);
    __threadfence();
    const unsigned old = atomicAdd(&bar->count, 1u);
    if (old == gridDim.x - 1) {
      atomicExch(&bar->count, 0u);
      __threadfence();
      st_release_u32(&bar->gen, gen + 1);
    } else {
      while (ld_acquire_u32(&bar->gen) == gen) __nanosleep(20);
    }
    __threadfence();
  }
  __syncthreads();
}

// Block-reduce (max, sum) to thread 0, in a fixed order.
__device__ __forceinline__ void block_reduce(double& mx, double& sm, double* sred) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  mx = warp_max(mx);
  sm = warp_sum(sm);
  __syncthreads();
  if (lane == 0) {
    sred[2 * w] = mx;
    sred[2 * w + 1] = sm;
  }
  __syncthreads();
  if (w == 0) {
    const int nw = blockDim.x >> 5;
    mx = lane < nw ? sred[2 * lane] : 0.0;
    sm = lane < nw ? sred[2 * lane + 1] : 0.0;
    mx = warp_max(mx);
    sm = warp_sum(sm);
  }
}

// Grid barrier fused with the residual reduction (K3).  Every CTA publishes
// its (max, sum); the LAST CTA to arrive reduces all partials in a fixed order
// and writes totals before releasing the barrier, so every CTA reads the same
// two doubles afterwards and takes the same stop decision.
__device__ __forceinline__ void grid_sync_reduce(const SolveParams& p, double bmax, double bsum,
                                                 double& tmax, double& tsum, double* sred) {
  __shared__ unsigned s_gen;
  __shared__ int s_last;
  if (threadIdx.x == 0) {
    p.partials[2 * blockIdx.x] = bmax;
    p.partials[2 * blockIdx.x + 1] = bsum;
    const unsigned gen = ld_acquire_u32(&p.bar->gen);
    __threadfence();
    const unsigned old = atomicAdd(&p.bar->count, 1u);
    s_gen = gen;
    s_last = (old == gridDim.x - 1);
  }
  __syncthreads();
  if (s_last) {
    __threadfence();
    double mx = 0.0, sm = 0.0;
    for (unsigned i = threadIdx.x; i < gridDim.x; i += blockDim.x) {
      mx = fmax(mx, ld_relaxed_f64(p.partials + 2 * i));
      sm += ld_relaxed_f64(p.partials + 2 * i + 1);
    }
    block_reduce(mx, sm, sred);
    if (threadIdx.x == 0) {
      p.totals[0] = mx;
      p.totals[1] = sm;
      atomicExch(&p.bar->count, 0u);
      __threadfence();
      st_release_u32(&p.bar->gen, s_gen + 1);
    }
  } else if (threadIdx.x == 0) {
    while (ld_acquire_u32(&p.bar->gen) == s_gen) __nanosleep(20);
    __threadfence();
  }
  __syncthreads();
  tmax = ld_relaxed_f64(p.totals);
  tsum = ld_relaxed_f64(p.totals + 1);
}

// ------------------------------------------------------------ one warp task
// Per-warp shared memory: two in_src staging slices (16-B cp.async chunks, so
// up to 3 leading pad entries + kTaskItems + 3 trailing) and two gathered
// value buffers -- a 2-deep cp.async pipeline across the warp's tasks.
constexpr int kSrcSlots = kTaskItems + 8;
constexpr int kWarpSmemBytes = 2 * kSrcSlots * 4 + 2 * kTaskItems * 8;
constexpr int kSolveSmemBytes = kWarpsPerBlock * kWarpSmemBytes;

__device__ __forceinline__ void cp_async16(void* sdst, const void* gsrc, unsigned long long pol) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(s), "l"(gsrc),
               "l"(pol)
               : "memory");
}
__device__ __forceinline__ void cp_async8(void* sdst, const void* gsrc) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(sdst);
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(s), "l"(gsrc) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

struct TaskMeta {
  int i0, i1;
  int64_t j0, j1;
};

__device__ __forceinline__ TaskMeta load_meta(const SolveParams& p, int t) {
  TaskMeta m;
  m.i0 = __ldg(p.task_row + t);
  m.i1 = __ldg(p.task_row + t + 1);
  m.j0 = __ldg(p.task_edge + t);
  m.j1 = __ldg(p.task_edge + t + 1);
  return m;
}

// Row metadata of a task's first 32 rows, prefetched one pipeline step early.
struct RowPre {
  int64_t a, b;
  int od;
  double ov;
};

__device__ __forceinline__ RowPre load_rowpre(const SolveParams& p, const TaskMeta& m, int lane) {
  RowPre r{0, 0, 0, 0.0};
  const int row = m.i0 + lane;
  if (row < m.i1) {
    r.a = __ldg(p.row + row);
    r.b = __ldg(p.row + row + 1);
    r.od = __ldg(p.outdeg + row);
    r.ov = p.pr[row];
  }
  return r;
}

// Stage the task's in_src slice: 16-B chunks from the 4-element-aligned base.
__device__ __forceinline__ void issue_src(const SolveParams& p, const TaskMeta& m, int32_t* sbuf,
                                          int lane, unsigned long long pol) {
  const int64_t base = m.j0 & ~int64_t(3);
  const int nchunks = (int)((m.j1 - base + 3) >> 2);
  for (int c = lane; c < nchunks; c += 32) cp_async16(sbuf + 4 * c, p.src + base + 4 * c, pol);
}

// Gather contrib[src] for the task's edges straight into shared memory.
template <bool ASYNC>
__device__ __forceinline__ void issue_gathers(const TaskMeta& m, const int32_t* sbuf, double* vbuf,
                                              int fresh_below, const double* prev,
                                              const double* cur, int lane) {
  const int off = (int)(m.j0 & 3);
  const int nE = (int)(m.j1 - m.j0);
  for (int k = lane; k < nE; k += 32) {
    const int s = sbuf[off + k];
    const double* basep = ASYNC ? cur : ((s < fresh_below) ? cur : prev);
    cp_async8(vbuf + k, basep + s);
  }
}

__device__ __forceinline__ double tail_not_ready() { return __longlong_as_double(-1ll); }  // NaN

template <bool ASYNC>
__device__ __forceinline__ void process_task(const SolveParams& p, int t, const TaskMeta& m,
                                             const RowPre& pre, const double* vals, double* cur,
                                             int lane, double& lmax, double& lsum) {
  const int i0 = m.i0, i1 = m.i1;
  const int64_t j0 = m.j0;
  const int nE = (int)(m.j1 - m.j0);

  // (a) open row at the end of the task: publish this task's partial first,
  //     so a task waiting on it never waits on this task's own head (no chain).
  //     The partial IS the flag: ready iff >= 0 (sums of positive contributions).
  if (i1 < p.n) {
    const int64_t rs = __ldg(p.row + i1);
    const int lo = (int)((rs > j0 ? rs : j0) - j0);
    if (lo < nE) {
      double a = 0.0;
      for (int k = lo + lane; k < nE; k += 32) a += vals[k];
      a = warp_sum(a);
      if (lane == 0) st_relaxed_f64(p.tail_partial + t, a);
    }
  }
  // (b) head row split across earlier tasks: combine their partials in task order.
  bool has_head = false;
  double head_sum = 0.0;
  if (i0 < i1 && __shfl_sync(FULL_MASK, pre.a, 0) < j0) {
    has_head = true;
    const int ta = __ldg(p.head_first + t);
    double acc = 0.0;
    for (int tt = ta + lane; tt < t; tt += 32) {
      double v = ld_relaxed_f64(p.tail_partial + tt);
      while (!(v >= 0.0)) {
        __nanosleep(32);
        v = ld_relaxed_f64(p.tail_partial + tt);
      }
      acc += v;
      st_relaxed_f64(p.tail_partial + tt, tail_not_ready());  // consumed: re-arm for next sweep
    }
    acc = warp_sum(acc);
    const int hi = (int)(__shfl_sync(FULL_MASK, pre.b, 0) - j0);
    double own = 0.0;
    for (int k = lane; k < hi; k += 32) own += vals[k];
    head_sum = acc + warp_sum(own);
  }

  // (c) rows whose end marker lies in this task: lane per row, ascending-src
  //     sequential sums (the reference's order); long rows warp-cooperative.
  for (int rb = i0; rb < i1; rb += 32) {
    const int r = rb + lane;
    const bool act = r < i1;
    int64_t a = pre.a, b = pre.b;
    int od = pre.od;
    double ov = pre.ov;
    if (rb != i0 && act) {
      a = __ldg(p.row + r);
      b = __ldg(p.row + r + 1);
      od = __ldg(p.outdeg + r);
      ov = p.pr[r];
    }
    int lo = 0, hi = 0;
    if (act) {
      lo = (int)((a > j0 ? a : j0) - j0);
      hi = (int)(b - j0);
    }
    const bool head = has_head && r == i0;
    const bool is_long = act && !head && (hi - lo) > 32;
    double sum = 0.0;
    if (act && !head && !is_long) {
      for (int k = lo; k < hi; ++k) sum += vals[k];
    }
    unsigned lm = __ballot_sync(FULL_MASK, is_long);
    while (lm) {
      const int L = __ffs(lm) - 1;
      lm &= lm - 1;
      const int llo = __shfl_sync(FULL_MASK, lo, L), lhi = __shfl_sync(FULL_MASK, hi, L);
      double acc = 0.0;
      for (int k = llo + lane; k < lhi; k += 32) acc += vals[k];
      acc = warp_sum(acc);
      if (lane == L) sum = acc;
    }
    if (head) sum = head_sum;
    if (act) {
      const double nv = __dadd_rn(p.base, __dmul_rn(p.damping, sum));
      p.pr[r] = nv;
      if (od > 0) {
        const double c = __ddiv_rn(nv, (double)od);
        if (ASYNC)
          st_relaxed_f64(cur + r, c);
        else
          cur[r] = c;
      }
      const double d = fabs(nv - ov);
      lmax = fmax(lmax, d);
      lsum += d;
    }
  }
}

// All tasks t = tb + gwarp + k*nwarps < te of this warp, software-pipelined:
// step k waits for in_src(k), issues in_src(k+1) and gathers(k), prefetches
// meta(k+2) and row metadata(k), then processes task k-1 while gathers(k)
// are in flight.  cp.async group order: S0, [empty], S1, G0, S2, G1, ...
template <bool ASYNC>
__device__ __forceinline__ void run_tasks(const SolveParams& p, int tb, int te, int gwarp,
                                          int nwarps, int fresh_below, const double* prev,
                                          double* cur, int32_t* sb, double* vb, int lane,
                                          unsigned long long pol, double& lmax, double& lsum) {
  int tk = tb + gwarp;
  if (tk >= te) return;
  TaskMeta mA = load_meta(p, tk);
  issue_src(p, mA, sb, lane, pol);
  cp_async_commit();
  cp_async_commit();  // stands in for G_{-1}
  TaskMeta mB{0, 0, 0, 0};
  if (tk + nwarps < te) mB = load_meta(p, tk + nwarps);
  TaskMeta mP{0, 0, 0, 0};
  RowPre rpP{0, 0, 0, 0.0};
  int tP = -1;
  int k = 0;
  while (true) {
    const bool haveA = tk < te;
    cp_async_wait<1>();  // in_src(k) landed
    __syncwarp();
    if (haveA && tk + nwarps < te) issue_src(p, mB, sb + ((k + 1) & 1) * kSrcSlots, lane, pol);
    cp_async_commit();
    RowPre rpA{0, 0, 0, 0.0};
    TaskMeta mC{0, 0, 0, 0};
    if (haveA) {
      issue_gathers<ASYNC>(mA, sb + (k & 1) * kSrcSlots, vb + (k & 1) * kTaskItems, fresh_below,
                           prev, cur, lane);
      if (tk + 2 * nwarps < te) mC = load_meta(p, tk + 2 * nwarps);
      rpA = load_rowpre(p, mA, lane);
    }
    cp_async_commit();
    if (tP >= 0) {
      cp_async_wait<2>();  // gathers(k-1) landed
      __syncwarp();
      process_task<ASYNC>(p, tP, mP, rpP, vb + ((k - 1) & 1) * kTaskItems, cur, lane, lmax, lsum);
      __syncwarp();
    }
    if (!haveA) break;
    mP = mA;
    rpP = rpA;
    tP = tk;
    mA = mB;
    mB = mC;
    tk += nwarps;
    ++k;
  }
  cp_async_wait<0>();
  __syncwarp();
}

// ------------------------------------------------------ persistent solver
// ASYNC=false: Jacobi (nwaves == 1, EC) or wave-lockstep Gauss-Seidel.
// ASYNC=true : block-asynchronous Gauss-Seidel, in-place contributions.
template <bool ASYNC>
__global__ void __launch_bounds__(kBlockThreads, 2) solve_kernel(SolveParams p) {
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double sred[2 * kWarpsPerBlock];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  unsigned char* wsm = smem + wib * kWarpSmemBytes;
  int32_t* sb = reinterpret_cast<int32_t*>(wsm);
  double* vb = reinterpret_cast<double*>(wsm + 2 * kSrcSlots * 4);
  const int gwarp = blockIdx.x * kWarpsPerBlock + wib;
  const int nwarps = gridDim.x * kWarpsPerBlock;
  const unsigned long long pol = evict_first_policy();
  int par = p.parity0;
  if (blockIdx.x == 0 && threadIdx.x == 0) p.iter_ns[0] = globaltimer();

  for (uint32_t it = 0; it < p.max_iters; ++it) {
    double lmax = 0.0, lsum = 0.0;
    if (ASYNC) {
      run_tasks<true>(p, 0, p.ntasks, gwarp, nwarps, 0, p.contrib0, p.contrib0, sb, vb, lane, pol,
                      lmax, lsum);
    } else {
      const double* prev = par ? p.contrib1 : p.contrib0;
      double* cur = par ? p.contrib0 : p.contrib1;
      for (int w = 0; w < p.nwaves; ++w) {
        run_tasks<false>(p, __ldg(p.wave_task + w), __ldg(p.wave_task + w + 1), gwarp, nwarps,
                         __ldg(p.wave_row + w), prev, cur, sb, vb, lane, pol, lmax, lsum);
        if (w + 1 < p.nwaves) grid_sync(p.bar);
      }
      par ^= 1;
    }
    block_reduce(lmax, lsum, sred);
    double tmax, tsum;
    grid_sync_reduce(p, lmax, lsum, tmax, tsum, sred);
    if (blockIdx.x == 0 && threadIdx.x == 0) {
      p.errors[it] = tmax;
      p.l1errors[it] = tsum;
      p.iter_ns[it + 1] = globaltimer();
    }
    const double crit = p.norm ? tsum : tmax;
    if (crit <= p.threshold || it + 1 == p.max_iters) {
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        *p.out_iters = it + 1;
        *p.out_stop = crit <= p.threshold ? 1 : 0;
      }
      return;
    }
  }
}

// ------------------------------------------------------------ partitioning
// Merge-path search (Merrill & Garland): number of row-end markers consumed
// at `diag` when row ends (row[i+1]) are merged with edge indices.
__device__ __forceinline__ int64_t merge_path(int64_t diag, const int64_t* row, int64_t n,
                                              int64_t m) {
  int64_t lo = diag - m > 0 ? diag - m : 0;
  int64_t hi = diag < n ? diag : n;
  while (lo < hi) {
    const int64_t pivot = (lo + hi) >> 1;
    if (row[pivot + 1] <= diag - pivot - 1)
      lo = pivot + 1;
    else
      hi = pivot;
  }
  return lo;
}

__global__ void partition_kernel(const int64_t* row, int32_t n, int64_t m, int32_t ntasks,
                                 int32_t* task_row, int64_t* task_edge) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > ntasks) return;
  const int64_t total = (int64_t)n + m;
  int64_t diag = t * (int64_t)kTaskItems;
  if (diag > total) diag = total;
  const int64_t x = merge_path(diag, row, n, m);
  task_row[t] = (int32_t)x;
  task_edge[t] = diag - x;
}

__global__ void head_kernel(const int64_t* row, int32_t n, int32_t ntasks, const int32_t* task_row,
                            const int64_t* task_edge, int32_t* head_first, uint8_t* clean_start) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t > ntasks) return;
  const int32_t i0 = task_row[t];
  const int64_t j0 = task_edge[t];
  const bool mid = i0 < n && row[i0] < j0;  // task starts inside row i0
  clean_start[t] = mid ? 0 : 1;
  if (t == ntasks) return;
  int32_t hf = -1;
  if (mid && i0 < task_row[t + 1]) {
    // last task t' with task_edge[t'] <= row[i0]: the one holding edge row[i0]
    const int64_t key = row[i0];
    int64_t lo = 0, hi = ntasks + 1;  // upper_bound
    while (lo < hi) {
      const int64_t mid2 = (lo + hi) >> 1;
      if (task_edge[mid2] <= key)
        lo = mid2 + 1;
      else
        hi = mid2;
    }
    hf = (int32_t)(lo - 1);
  }
  head_first[t] = hf;
}

__global__ void init_kernel(int32_t n, const int32_t* outdeg, double init, double* pr,
                            double* contrib) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
       u += (int64_t)gridDim.x * blockDim.x) {
    pr[u] = init;
    const int od = outdeg[u];
    contrib[u] = od > 0 ? __ddiv_rn(init, (double)od) : 0.0;
  }
}

__global__ void narrow_kernel(const uint64_t* in, int32_t* out, int64_t count, uint64_t bound,
                              unsigned int* bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count;
       i += (int64_t)gridDim.x * blockDim.x) {
    const uint64_t v = in[i];
    if (v >= bound) atomicOr(bad, 1u);
    out[i] = (int32_t)v;
  }
}

__global__ void check_offsets_kernel(const int64_t* row, int32_t n, int64_t m, unsigned int* bad) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
       i += (int64_t)gridDim.x * blockDim.x) {
    if (row[i + 1] < row[i]) atomicOr(bad, 2u);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    if (row[0] != 0 || row[n] != m) atomicOr(bad, 4u);
  }
}

__global__ void widen_kernel(const int64_t* row, const int32_t* ids, uint64_t* out_row,
                             uint64_t* out_ids, int64_t nrow, int64_t nids) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nrow; i += stride)
    out_row[i] = (uint64_t)row[i];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nids; i += stride)
    out_ids[i] = (uint64_t)(uint32_t)ids[i];
}

static int grid_for(int64_t work, int threads = 256) {
  int64_t b = (work + threads - 1) / threads;
  if (b < 1) b = 1;
  if (b > 148 * 32) b = 148 * 32;
  return (int)b;
}

// ------------------------------------------------------------ host launchers
cudaError_t launch_partition(const DevGraph& g, Partition& p, cudaStream_t s) {
  const int64_t nt = p.ntasks;
  const int blocks = (int)((nt + 1 + 255) / 256);
  partition_kernel<<<blocks, 256, 0, s>>>(g.row, g.n, g.m, p.ntasks, p.task_row, p.task_edge);
  head_kernel<<<blocks, 256, 0, s>>>(g.row, g.n, p.ntasks, p.task_row, p.task_edge, p.head_first,
                                     p.clean_start);
  return cudaGetLastError();
}

cudaError_t launch_init(const DevGraph& g, double* pr, double* contrib, cudaStream_t s) {
  init_kernel<<<grid_for(g.n), 256, 0, s>>>(g.n, g.outdeg, 1.0 / (double)g.n, pr, contrib);
  return cudaGetLastError();
}

cudaError_t solve_grid(int engine, int num_sms, int* grid_out) {
  int per_sm = 0;
  for (const void* fn : {(const void*)solve_kernel<true>, (const void*)solve_kernel<false>}) {
    cudaError_t a = cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, kSolveSmemBytes);
    if (a != cudaSuccess) return a;
  }
  cudaError_t e = engine == kFused
                      ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_kernel<true>,
                                                                      kBlockThreads, kSolveSmemBytes)
                      : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, solve_kernel<false>,
                                                                      kBlockThreads, kSolveSmemBytes);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) return cudaErrorInvalidConfiguration;
  *grid_out = per_sm * num_sms;
  return cudaSuccess;
}

cudaError_t launch_solve(int engine, int grid, const SolveParams& p, cudaStream_t s) {
  SolveParams copy = p;
  void* args[] = {&copy};
  const void* fn = engine == kFused ? (const void*)solve_kernel<true> : (const void*)solve_kernel<false>;
  return cudaLaunchCooperativeKernel(fn, dim3(grid), dim3(kBlockThreads), args, kSolveSmemBytes, s);
}

cudaError_t launch_narrow_ids(const uint64_t* in, int32_t* out, int64_t count, uint64_t bound,
                              unsigned int* bad_flag, cudaStream_t s) {
  if (count <= 0) return cudaSuccess;
  narrow_kernel<<<grid_for(count), 256, 0, s>>>(in, out, count, bound, bad_flag);
  return cudaGetLastError();
}

cudaError_t launch_check_offsets(const int64_t* row, int32_t n, int64_t m, unsigned int* bad_flag,
                                 cudaStream_t s) {
  check_offsets_kernel<<<grid_for(n), 256, 0, s>>>(row, n, m, bad_flag);
  return cudaGetLastError();
}

cudaError_t launch_widen(const int64_t* row, const int32_t* ids32, uint64_t* out_row,
                         uint64_t* out_ids, int64_t nrow, int64_t nids, cudaStream_t s) {
  widen_kernel<<<grid_for(nrow > nids ? nrow : nids), 256, 0, s>>>(row, ids32, out_row, out_ids,
                                                                   nrow, nids);
  return cudaGetLastError();
}

}  // namespace fprb
