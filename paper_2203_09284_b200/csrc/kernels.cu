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
// Work unit: a warp task = ~kTaskDiag consecutive items of the merge path of
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
// A task covers ~kTaskDiag merge items (<= kTaskItems = 249 edges); its slice [j0, j1) is
// viewed in 32-B-aligned "position" space p = (e - (j0 & ~7)), so lane L owns
// positions [8L, 8L+8) and loads them as one aligned 32-B vector (coalesced 1 KB per
// warp), gathers its <= 8 contributions into registers, and reduces them
// lane-sequentially in ascending-src order.  Segments (rows) crossing lanes are
// combined by one warp segmented scan; rows crossing tasks by tail partials.
constexpr int kLaneItems = 8;
constexpr int kPos = 32 * kLaneItems;  // 256 positions per task


struct alignas(16) WarpSmem {
  double pacc[kPos];  // per position: lane-local running sum since the last segment start
  double carry[33];   // carry[L] = inclusive segmented scan of lane L-1's tail (0 for L=0)
  // the head row whose finish is deferred by one task (finish_head)
  double ph_sum;      // its sum inside the owner task
  double ph_ov;       // pr[r] before the sweep
  int ph_od;          // outdeg[r]
  int ph_r;           // the row
  int ph_t;           // the owner task, -1 = none
  int ph_pad;
};
// Launch shape per engine: Jacobi/lockstep run 20 warps/SM (160-thread CTAs,
// <= 102 registers, no spills); the async engine runs 16 warps/SM, which its
// relaxed in-place traffic prefers (measured).
#ifndef FPR_EC_BLOCK
#define FPR_EC_BLOCK 160
#endif
#ifndef FPR_EC_MINB
#define FPR_EC_MINB 4
#endif
#ifndef FPR_ASYNC_BLOCK
#define FPR_ASYNC_BLOCK 256
#endif
#ifndef FPR_ASYNC_MINB
#define FPR_ASYNC_MINB 2
#endif
template <int BT>
constexpr int solve_smem_bytes() { return (BT / 32) * (int)sizeof(WarpSmem); }

static_assert(kTaskItems + 7 <= 32 * kLaneItems, "task slice (+ alignment pad) must fit 256 positions");

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


// Lane's 8 source ids of a task: one aligned 32-B load (LDG.256) per lane, so
// the warp's 1 KB of in_src costs exactly one L2 request per sector.
struct Src8 {
  int4 a, b;
};
constexpr int kPosAlign = 8;
__device__ __forceinline__ Src8 load_src8(const SolveParams& p, const TaskMeta& m, int lane,
                                          unsigned long long pol) {
  Src8 s{{0, 0, 0, 0}, {0, 0, 0, 0}};
  const int64_t base = (m.j0 & ~int64_t(kPosAlign - 1)) + 8 * lane;
  if (base < m.j1) {
    asm volatile(
        "ld.global.nc.L1::no_allocate.L2::cache_hint.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8], %9;"
        : "=r"(s.a.x), "=r"(s.a.y), "=r"(s.a.z), "=r"(s.a.w), "=r"(s.b.x), "=r"(s.b.y),
          "=r"(s.b.z), "=r"(s.b.w)
        : "l"(p.src + base), "l"(pol));
  }
  return s;
}

__device__ __forceinline__ double tail_not_ready() { return __longlong_as_double(-1ll); }  // NaN

// Predicated gather into v (left untouched when !valid).  Inline PTX keeps the
// compiler from consuming the value (and stalling) before it is needed.
template <bool ASYNC>
__device__ __forceinline__ void gather1(double& v, bool valid, int s, int fresh_below,
                                        const double* prev, const double* cur) {
  const double* basep = ASYNC ? prev : ((s < fresh_below) ? cur : prev);
  const double* addr = basep + s;
  if (ASYNC) {  // value-atomic live read (pagerank.hpp:305)
#ifdef FPR_ASYNC_CG
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q ld.global.cg.f64 %0, [%1]; }"
                 : "+d"(v)
                 : "l"(addr), "r"((int)valid)
                 : "memory");
#else
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q ld.relaxed.gpu.global.f64 %0, [%1]; }"
                 : "+d"(v)
                 : "l"(addr), "r"((int)valid)
                 : "memory");
#endif
  } else {
    // L2 only: random 8-B gathers have no L1 reuse (an L1-allocating ld.ca
    // variant measured no faster even on R-MAT hubs)
    asm volatile("{ .reg .pred q; setp.ne.b32 q, %2, 0; @q ld.global.cg.f64 %0, [%1]; }"
                 : "+d"(v)
                 : "l"(addr), "r"((int)valid));
  }
}

// Finalize mode of a solve instantiation:
//   kModeFinal : rank update + contribution store (single GPU);
//   kModePeers : ... plus the store into every peer replica (fused exchange).
constexpr int kModeFinal = 0, kModePeers = 1;

// Row metadata of a task's first 32 rows (i0 .. i0+31, including the open
// row i1 when it falls in that window), prefetched one task ahead, with the
// row bounds already relative to the task's first edge j0.
struct RowPre {
  int lo;     // max(row[r], j0) - j0, or -1 when row r began before j0 (split head)
  int hi;     // row[r+1] - j0 (finalized rows) or j1 - j0 (open row)
  int od;     // outdeg[r] (finalized rows only)
  double ov;  // pr[r]     (finalized rows only)
};
template <int MODE>
__device__ __forceinline__ RowPre load_rowpre(const SolveParams& p, const TaskMeta& m, int lane) {
  RowPre r{0, 0, 0, 0.0};
  const int row = m.i0 + lane;
  if (row < m.i1) {
    const int64_t a = __ldg(p.row + row), b = __ldg(p.row + row + 1);
    r.lo = a < m.j0 ? -1 : (int)(a - m.j0);
    r.hi = (int)(b - m.j0);
    r.od = __ldg(p.outdeg + row);
    r.ov = p.pr[row];
  } else if (row == m.i1 && row < p.n) {
    const int64_t a = __ldg(p.row + row);
    r.lo = a < m.j0 ? -1 : (int)(a - m.j0);
    r.hi = (int)(m.j1 - m.j0);
  }
  return r;
}

// 1. gathers: position q of this lane holds edge q - off when off <= q < off + nE;
//    invalid positions keep 0 (predicated loads, nothing consumed early).
template <bool ASYNC>
__device__ __forceinline__ void issue_gathers8(const TaskMeta& m, const Src8& sx, int lane,
                                               int fresh_below, const double* prev,
                                               const double* cur, double (&v)[8]) {
  const int off = (int)(m.j0 & (kPosAlign - 1));
  const int valid_hi = off + (int)(m.j1 - m.j0);
  const int pos0 = 8 * lane;
  const int sids[8] = {sx.a.x, sx.a.y, sx.a.z, sx.a.w, sx.b.x, sx.b.y, sx.b.z, sx.b.w};
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const int q = pos0 + i;
    v[i] = 0.0;
    gather1<ASYNC>(v[i], q >= off && q < valid_hi, sids[i], fresh_below, prev, cur);
  }
}

// 2. lane-sequential running sums, reset at every segment start (ascending
//    source order inside a row, as gather_ranks_jacobi sums, :85-87); the 8
//    partial sums go to shared memory so v can take the next task's gathers.
__device__ __forceinline__ double task_sums(const double (&v)[8], unsigned bits8, WarpSmem& ws,
                                            int lane) {
  double acc = 0.0, w[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    if ((bits8 >> i) & 1u) acc = 0.0;
    acc += v[i];
    w[i] = acc;
  }
  double4* pa = reinterpret_cast<double4*>(ws.pacc + 8 * lane);
  pa[0] = make_double4(w[0], w[1], w[2], w[3]);
  pa[1] = make_double4(w[4], w[5], w[6], w[7]);
  return acc;
}

// A head row split across earlier tasks is finished one task LATER by the
// warp that holds its end (the owner): the partials of the earlier tasks are
// written while this warp runs its next task, so the combine rarely waits
// (waiting at once spun on partials of tasks running in parallel: 26% of
// config 3's stall samples).  The same warp finishes the row in the same
// place of its schedule on every run, so ranks and residuals keep their bits.
#ifndef FPR_DEFER_HEAD
#define FPR_DEFER_HEAD 1
#endif
template <bool ASYNC, int MODE>
__device__ __forceinline__ void finish_head(const SolveParams& p, WarpSmem& ws, double* cur, int lane,
                                            double& lmax, double& lsum) {
  const int t = ws.ph_t;
  if (t < 0) return;
  const int ta = __ldg(p.head_first + t);
  double accp = 0.0;
  for (int tt = ta + lane; tt < t; tt += 32) {
    double x = ld_relaxed_f64(p.tail_partial + tt);
    while (!(x >= 0.0)) {
      __nanosleep(64);
      x = ld_relaxed_f64(p.tail_partial + tt);
    }
    accp += x;
    st_relaxed_f64(p.tail_partial + tt, tail_not_ready());  // consumed: re-arm
  }
  const double head_extra = warp_sum(accp);
  if (lane == 0) {
    const int r = ws.ph_r, od = ws.ph_od;
    const double nv = __dadd_rn(p.base, __dmul_rn(p.damping, head_extra + ws.ph_sum));
    p.pr_out[r] = nv;
    if (od > 0) {
      const double c = __ddiv_rn(nv, (double)od);
      if (ASYNC)
        st_relaxed_f64(cur + r, c);
      else
        cur[r] = c;
      if (MODE == kModePeers)
        for (int q = 0; q < p.npeers; ++q) p.peer[q][r] = c;
    }
    const double d = fabs(nv - ws.ph_ov);
    lmax = fmax(lmax, d);
    lsum += d;
    ws.ph_t = -1;
  }
  __syncwarp();
}

template <bool ASYNC, int MODE>
__device__ __forceinline__ void task_finish(const SolveParams& p, int t, const TaskMeta& m,
                                            double acc, unsigned bits8, const RowPre& rp,
                                            double* cur, WarpSmem& ws, int lane, double& lmax,
                                            double& lsum) {
  const int i0 = m.i0, i1 = m.i1;
  const int64_t j0 = m.j0, j1 = m.j1;
  const int off = (int)(j0 & (kPosAlign - 1));
  const int valid_hi = off + (int)(j1 - j0);

  // 3. carries across lanes: inclusive segmented scan of the lane tails; a
  //    lane holding a segment start breaks the chain.
  double S = acc;
  bool brk = bits8 != 0u || lane == 0;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    if (__all_sync(FULL_MASK, brk)) break;  // every chain resolved (rows rarely span many lanes)
    const double up = __shfl_up_sync(FULL_MASK, S, d);
    const bool ub = __shfl_up_sync(FULL_MASK, brk, d);
    if (lane >= d) {
      if (!brk) S += up;
      brk = brk || ub;
    } else {
      brk = true;
    }
  }
  ws.carry[lane + 1] = S;
  if (lane == 0) ws.carry[0] = 0.0;
  // open row at the end of the task: publish its partial first (the partial
  // IS the flag: >= 0 once written), before waiting on any earlier task.
  {
    const int orr = i1 - i0;  // relative index of the open row
    bool has_piece = false;
    if (i1 < p.n) {
      if (orr < 32) {
        const int lo = __shfl_sync(FULL_MASK, rp.lo, orr), hi = __shfl_sync(FULL_MASK, rp.hi, orr);
        has_piece = (lo < 0 ? 0 : lo) < hi;
      } else {
        has_piece = __ldg(p.row + i1) < j1;
      }
    }
    if (has_piece && lane == ((valid_hi - 1) >> 3)) st_relaxed_f64(p.tail_partial + t, S);
  }
  __syncwarp();

  // 4. head row split across earlier tasks: combine their partials in task
  //    order -- deferred (finish_head): the previous task's head row now,
  //    this task's after the next task.
  double head_extra = 0.0;
  const bool has_head = i0 < i1 && __shfl_sync(FULL_MASK, rp.lo, 0) < 0;
#if FPR_DEFER_HEAD
  finish_head<ASYNC, MODE>(p, ws, cur, lane, lmax, lsum);
#else
  if (has_head) {
    const int ta = __ldg(p.head_first + t);
    double accp = 0.0;
    for (int tt = ta + lane; tt < t; tt += 32) {
      double x = ld_relaxed_f64(p.tail_partial + tt);
      while (!(x >= 0.0)) {
        __nanosleep(64);
        x = ld_relaxed_f64(p.tail_partial + tt);
      }
      accp += x;
      st_relaxed_f64(p.tail_partial + tt, tail_not_ready());  // consumed: re-arm
    }
    head_extra = warp_sum(accp);
  }
#endif

  // 5. finalize rows [i0, i1): lane per row.  A row's in-task sum is the
  //    running sum at its last position plus the carry into that lane when
  //    the row began in an earlier lane.
  for (int rb = i0; rb < i1; rb += 32) {
    const int r = rb + lane;
    if (r < i1) {
      int lo = rp.lo < 0 ? 0 : rp.lo, hi = rp.hi;
      int od = rp.od;
      double ov = rp.ov;
      if (rb != i0) {
        lo = (int)(__ldg(p.row + r) - j0);
        hi = (int)(__ldg(p.row + r + 1) - j0);
        od = __ldg(p.outdeg + r);
        ov = p.pr[r];
      }
      double sum = 0.0;
      if (lo < hi) {
        const int e = hi - 1 + off;
        sum = ws.pacc[e];
        if (lo + off < (e & ~7)) sum = ws.carry[e >> 3] + sum;
      }
#if FPR_DEFER_HEAD
      if (r == i0 && has_head) {  // finished after the next task (finish_head)
        ws.ph_r = r;
        ws.ph_sum = sum;
        ws.ph_od = od;
        ws.ph_ov = ov;
        ws.ph_t = t;
        continue;
      }
#else
      if (r == i0 && has_head) sum = head_extra + sum;
#endif
      const double nv = __dadd_rn(p.base, __dmul_rn(p.damping, sum));
      p.pr_out[r] = nv;
      if (od > 0) {
        const double c = __ddiv_rn(nv, (double)od);
        if (ASYNC)
          st_relaxed_f64(cur + r, c);
        else
          cur[r] = c;
        // fused exchange: the same (coalesced) store into every peer replica
        if (MODE == kModePeers && !(p.peer_skip_empty && lo == hi && !(r == i0 && has_head)))
          for (int q = 0; q < p.npeers; ++q) p.peer[q][r] = c;
      }
      const double d = fabs(nv - ov);
      lmax = fmax(lmax, d);
      lsum += d;
    }
  }
  __syncwarp();
}

// All tasks t = tb + gwarp + k*nwarps < te of this warp, software-pipelined
// without extra registers: once a task's gathered values are folded into
// shared memory, the next task's gathers are issued into the same registers
// and fly while this task's carry scan and row finalize run.  Source ids are
// prefetched two tasks ahead, row metadata and bitmaps one task ahead.
__device__ __forceinline__ unsigned load_bits8(const SolveParams& p, int t, int lane) {
  return (__ldg(p.task_bits + 8 * (int64_t)t + (lane >> 2)) >> ((lane & 3) * 8)) & 0xffu;
}

#ifdef FPR_CHECKS
// Debug build (make variant V=checks EXTRA=-DFPR_CHECKS): every task's
// metadata and source ids are bounds-checked before use; a violation traps.
__device__ __noinline__ void check_task(const SolveParams& p, int t, const TaskMeta& m, const Src8& sx, int lane) {
  const bool meta_ok = t >= 0 && t < p.ntasks && m.i0 >= 0 && m.i0 <= m.i1 && m.i1 <= p.n && m.j0 >= 0 &&
                       m.j0 <= m.j1 && m.j1 - m.j0 <= kTaskItems && __ldg(p.head_first + t) <= t;
  const int off = (int)(m.j0 & (kPosAlign - 1));
  const int valid_hi = off + (int)(m.j1 - m.j0);
  const int sids[8] = {sx.a.x, sx.a.y, sx.a.z, sx.a.w, sx.b.x, sx.b.y, sx.b.z, sx.b.w};
  bool ids_ok = true;
  for (int i = 0; i < 8; ++i) {
    const int q = 8 * lane + i;
    if (q >= off && q < valid_hi) ids_ok = ids_ok && sids[i] >= 0 && (int64_t)sids[i] < p.nsrc;
  }
  if (!meta_ok || !ids_ok) {
    printf("FPR_CHECKS: task %d lane %d meta_ok %d ids_ok %d i0 %d i1 %d j0 %lld j1 %lld\n", t, lane, (int)meta_ok,
           (int)ids_ok, m.i0, m.i1, (long long)m.j0, (long long)m.j1);
    __trap();
  }
}
#define FPR_CHECK_TASK(p, t, m, sx, lane) check_task(p, t, m, sx, lane)
#else
#define FPR_CHECK_TASK(p, t, m, sx, lane) ((void)0)
#endif

template <bool ASYNC, int MODE>
__device__ __forceinline__ void run_tasks(const SolveParams& p, int tb, int te, int gwarp,
                                          int nwarps, int fresh_below, const double* prev,
                                          double* cur, WarpSmem& ws, int lane,
                                          unsigned long long pol, double& lmax, double& lsum) {
  int t = tb + gwarp;
  if (t >= te) return;
  TaskMeta m = load_meta(p, t);
  double v[8];
  {
    const Src8 sx = load_src8(p, m, lane, pol);
    FPR_CHECK_TASK(p, t, m, sx, lane);
    issue_gathers8<ASYNC>(m, sx, lane, fresh_below, prev, cur, v);
  }
  RowPre rp = load_rowpre<MODE>(p, m, lane);
  unsigned bits = load_bits8(p, t, lane);
  if (lane == 0) ws.ph_t = -1;
  __syncwarp();
  TaskMeta mn{0, 0, 0, 0}, mnn{0, 0, 0, 0};
  Src8 sn{{0, 0, 0, 0}, {0, 0, 0, 0}};
  if (t + nwarps < te) {
    mn = load_meta(p, t + nwarps);
    sn = load_src8(p, mn, lane, pol);
    if (t + 2 * nwarps < te) mnn = load_meta(p, t + 2 * nwarps);
  }
  while (true) {
    const int tn = t + nwarps;
    const double acc = task_sums(v, bits, ws, lane);
    RowPre rpn{0, 0, 0, 0.0};
    unsigned bitsn = 0;
    Src8 snn{{0, 0, 0, 0}, {0, 0, 0, 0}};
    TaskMeta mnnn{0, 0, 0, 0};
    if (tn < te) {
      FPR_CHECK_TASK(p, tn, mn, sn, lane);
      issue_gathers8<ASYNC>(mn, sn, lane, fresh_below, prev, cur, v);
      rpn = load_rowpre<MODE>(p, mn, lane);
      bitsn = load_bits8(p, tn, lane);
      if (tn + nwarps < te) {
        snn = load_src8(p, mnn, lane, pol);
        if (tn + 2 * nwarps < te) mnnn = load_meta(p, tn + 2 * nwarps);
      }
    }
    task_finish<ASYNC, MODE>(p, t, m, acc, bits, rp, cur, ws, lane, lmax, lsum);
    if (tn >= te) break;
    t = tn;
    m = mn;
    rp = rpn;
    bits = bitsn;
    mn = mnn;
    sn = snn;
    mnn = mnnn;
  }
  finish_head<ASYNC, MODE>(p, ws, cur, lane, lmax, lsum);  // the last task's head row
}

// ------------------------------------------------------ persistent solver
// ASYNC=false: Jacobi (nwaves == 1, EC) or wave-lockstep Gauss-Seidel.
// ASYNC=true : block-asynchronous Gauss-Seidel, in-place contributions.
template <bool ASYNC, int BT, int MB, int MODE>
__global__ void __launch_bounds__(BT, MB) solve_kernel(SolveParams p) {
  constexpr int kWPB = BT / 32;
  extern __shared__ __align__(16) unsigned char smem[];
  __shared__ double sred[2 * kWPB];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  WarpSmem& ws = reinterpret_cast<WarpSmem*>(smem)[wib];
  const int gwarp = blockIdx.x * kWPB + wib;
  const int nwarps = gridDim.x * kWPB;
  const unsigned long long pol = evict_first_policy();
  if (p.gate && *reinterpret_cast<const volatile unsigned int*>(p.gate)) return;  // stopped: no-op sweep
  int par = p.parity0;
  if (blockIdx.x == 0 && threadIdx.x == 0) p.iter_ns[0] = globaltimer();

  for (uint32_t it = 0; it < p.max_iters; ++it) {
    double lmax = 0.0, lsum = 0.0;
    if (ASYNC) {
      // in place: reads through the full vector, writes to this part's slice
      run_tasks<true, MODE>(p, 0, p.ntasks, gwarp, nwarps, 0, p.contrib0, p.contrib0 + p.write_off, ws, lane, pol,
                      lmax, lsum);
    } else {
      const double* prev = par ? p.contrib1 : p.contrib0;
      double* cur = (par ? p.contrib0 : p.contrib1) + p.write_off;
      for (int w = 0; w < p.nwaves; ++w) {
        run_tasks<false, MODE>(p, __ldg(p.wave_task + w), __ldg(p.wave_task + w + 1), gwarp, nwarps,
                         __ldg(p.wave_row + w), prev, cur, ws, lane, pol, lmax, lsum);
        if (w + 1 < p.nwaves) grid_sync(p.bar);
      }
      par ^= 1;
    }
#ifdef FPR_TRACE_WARPS
    // diagnostic build (scripts/warp_tail.py): when each warp finished sweep 2,
    // stored past the tail partials (the runtime over-allocates that array)
    if (it == 2 && lane == 0)
      reinterpret_cast<unsigned long long*>(p.tail_partial)[p.ntasks + 1 + gwarp] = globaltimer();
#endif
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
        p.out_last[0] = tmax;
        p.out_last[1] = tsum;
      }
      if (MODE == kModePeers) __threadfence_system();  // peer-replica stores performed before exit
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
  int64_t diag = t * (int64_t)kTaskDiag;
  if (diag > total) diag = total;
  const int64_t x = merge_path(diag, row, n, m);
  int64_t y = diag - x;
  // Snap: never split a short row -- the boundary moves back to its first
  // edge, so only rows longer than kSnapEdges ever need cross-task partials.
  if (x < n && y > row[x] && row[x + 1] - row[x] <= kSnapEdges) y = row[x];
  task_row[t] = (int32_t)x;
  task_edge[t] = y;
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

// Per-task segment-start bitmap (iteration-invariant): in the task's
// position space p = e - (j0 & ~7), bit p is set when the in-task segment of
// one of the rows i0..i1 (i1 = the open row) starts at edge e.
__global__ void task_bits_kernel(const int64_t* row, int32_t n, int32_t ntasks,
                                 const int32_t* task_row, const int64_t* task_edge,
                                 uint32_t* bits) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= ntasks) return;
  const int32_t i0 = task_row[t], i1 = task_row[t + 1];
  const int64_t j0 = task_edge[t], j1 = task_edge[t + 1];
  const int off = (int)(j0 & 7);
  uint32_t w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  const int32_t last = i1 < n ? i1 : i1 - 1;
  for (int32_t r = i0; r <= last; ++r) {
    const int64_t a = row[r], b = r < i1 ? row[r + 1] : j1;
    const int64_t lo = (a > j0 ? a : j0) - j0, hi = (b < j1 ? b : j1) - j0;
    if (lo < hi) {
      const int q = (int)lo + off;
      w[q >> 5] |= 1u << (q & 31);
    }
  }
  uint4* out = reinterpret_cast<uint4*>(bits + 8 * t);
  out[0] = make_uint4(w[0], w[1], w[2], w[3]);
  out[1] = make_uint4(w[4], w[5], w[6], w[7]);
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

// Multi-GPU destination-range partition: part r owns rows
// [bounds[r], bounds[r+1]); its sources are remapped into the padded exchange
// space part(s)*slice + (s - bounds[part(s)]) so one equal-size all-gather per
// iteration rebuilds every part's view of the contribution vector.
__global__ void part_bounds_kernel(const int64_t* row, int32_t n, int64_t m, uint32_t nparts,
                                   int64_t* bounds) {
  const uint32_t r = blockIdx.x * blockDim.x + threadIdx.x;
  if (r > nparts) return;
  const int64_t total = (int64_t)n + m;
  const int64_t diag = (int64_t)((__int128)total * r / nparts);
  bounds[r] = r == nparts ? n : merge_path(diag, row, n, m);
}

__global__ void part_extract_kernel(const int64_t* row, const int32_t* src, const int32_t* outdeg,
                                    const int64_t* bounds, uint32_t nparts, uint32_t part,
                                    int64_t slice, int64_t* lrow, int32_t* lsrc, int32_t* lout) {
  __shared__ int64_t sb[65];
  for (uint32_t i = threadIdx.x; i <= nparts; i += blockDim.x) sb[i] = bounds[i];
  __syncthreads();
  const int64_t v0 = sb[part], v1 = sb[part + 1];
  const int64_t e0 = row[v0], e1 = row[v1];
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i <= v1 - v0; i += stride) {
    lrow[i] = row[v0 + i] - e0;
    if (i < v1 - v0) lout[i] = outdeg[v0 + i];
  }
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < e1 - e0; e += stride) {
    const int32_t s = src[e0 + e];
    uint32_t lo = 0, hi = nparts;  // last part with bounds[part] <= s
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (sb[mid] <= s)
        lo = mid;
      else
        hi = mid;
    }
    lsrc[e] = (int32_t)((int64_t)lo * slice + (s - sb[lo]));
  }
}

// In-place variants for a part uploaded directly from the host (part_create):
// row offsets made local, global source ids remapped into the exchange space.
__global__ void offset_shift_kernel(int64_t* row, int64_t count, int64_t e0) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride) row[i] -= e0;
}

__global__ void part_remap_kernel(int32_t* src, int64_t m, const int64_t* bounds, uint32_t nparts, int64_t slice) {
  __shared__ int64_t sb[65];
  for (uint32_t i = threadIdx.x; i <= nparts; i += blockDim.x) sb[i] = bounds[i];
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < m; e += stride) {
    const int32_t s = src[e];
    uint32_t lo = 0, hi = nparts;  // last part with bounds[part] <= s
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (sb[mid] <= s)
        lo = mid;
      else
        hi = mid;
    }
    src[e] = (int32_t)((int64_t)lo * slice + (s - sb[lo]));
  }
}

__global__ void part_init_kernel(int32_t n, const int32_t* outdeg, double init, double* pr,
                                 double* contrib_slice) {
  for (int64_t u = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; u < n;
       u += (int64_t)gridDim.x * blockDim.x) {
    pr[u] = init;
    const int od = outdeg[u];
    contrib_slice[u] = od > 0 ? __ddiv_rn(init, (double)od) : 0.0;
  }
}

// build_csr invariants (graph.hpp:20-30): offsets monotone with row[0]=0 and
// row[n]=m, ids in range, no self-loops, strictly ascending sources per row
// (sorted + deduplicated), out-degrees equal to the per-source edge counts.
__global__ void validate_kernel(const int64_t* row, const int32_t* src, int32_t n, int64_t m,
                                int32_t* recount, unsigned int* bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t d = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; d < n; d += stride) {
    const int64_t a = row[d], b = row[d + 1];
    if (b < a) atomicOr(bad, 1u);
    int32_t prev = -1;
    for (int64_t e = a; e < b; ++e) {
      const int32_t s = src[e];
      if (s < 0 || s >= n) {
        atomicOr(bad, 2u);
        continue;
      }
      if (s == (int32_t)d) atomicOr(bad, 4u);
      if (s <= prev) atomicOr(bad, 8u);
      prev = s;
      atomicAdd(&recount[s], 1);
    }
  }
  if (blockIdx.x == 0 && threadIdx.x == 0 && (row[0] != 0 || row[n] != m)) atomicOr(bad, 16u);
}

__global__ void compare_counts_kernel(const int32_t* a, const int32_t* b, int32_t n, unsigned int* bad) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    if (a[i] != b[i]) atomicOr(bad, 32u);
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
  task_bits_kernel<<<blocks, 256, 0, s>>>(g.row, g.n, p.ntasks, p.task_row, p.task_edge, p.task_bits);
  head_kernel<<<blocks, 256, 0, s>>>(g.row, g.n, p.ntasks, p.task_row, p.task_edge, p.head_first,
                                     p.clean_start);
  return cudaGetLastError();
}

cudaError_t launch_init(const DevGraph& g, double* pr, double* contrib, cudaStream_t s) {
  init_kernel<<<grid_for(g.n), 256, 0, s>>>(g.n, g.outdeg, 1.0 / (double)g.n, pr, contrib);
  return cudaGetLastError();
}

struct SolveShape {
  const void* fn;
  int block;
  int smem;
};

// One instantiation per finalize mode; the plain one carries no trace of the
// peer stores.
static SolveShape solve_shape(int engine, int mode) {
  if (engine == kFusedWide)
    return {mode == kModePeers ? (const void*)solve_kernel<true, FPR_EC_BLOCK, FPR_EC_MINB, kModePeers>
                               : (const void*)solve_kernel<true, FPR_EC_BLOCK, FPR_EC_MINB, kModeFinal>,
            FPR_EC_BLOCK, solve_smem_bytes<FPR_EC_BLOCK>()};
  if (engine == kFused)
    return {mode == kModePeers ? (const void*)solve_kernel<true, FPR_ASYNC_BLOCK, FPR_ASYNC_MINB, kModePeers>
                               : (const void*)solve_kernel<true, FPR_ASYNC_BLOCK, FPR_ASYNC_MINB, kModeFinal>,
            FPR_ASYNC_BLOCK, solve_smem_bytes<FPR_ASYNC_BLOCK>()};
  const void* fn = mode == kModePeers ? (const void*)solve_kernel<false, FPR_EC_BLOCK, FPR_EC_MINB, kModePeers>
                                      : (const void*)solve_kernel<false, FPR_EC_BLOCK, FPR_EC_MINB, kModeFinal>;
  return {fn, FPR_EC_BLOCK, solve_smem_bytes<FPR_EC_BLOCK>()};
}

int solve_block_threads(int engine) { return solve_shape(engine, kModeFinal).block; }

// Co-resident grid for the engine: the smallest of its instantiations'
// occupancy, so either can be launched cooperatively with it.
cudaError_t solve_grid(int engine, int num_sms, int* grid_out) {
  int best = 1 << 30;
  for (int mode : {kModeFinal, kModePeers}) {
    const SolveShape sh = solve_shape(engine, mode);
    cudaError_t e = cudaFuncSetAttribute(sh.fn, cudaFuncAttributeMaxDynamicSharedMemorySize, sh.smem);
    if (e != cudaSuccess) return e;
    int per_sm = 0;
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, sh.fn, sh.block, sh.smem);
    if (e != cudaSuccess) return e;
    best = std::min(best, per_sm);
  }
  if (best < 1) return cudaErrorInvalidConfiguration;
  *grid_out = best * num_sms;
  return cudaSuccess;
}

// ------------------------------------------------- device-side stop rule
// One thread: the parts' pairs in part order (max, then sum -- the order the
// host drivers use), the trace entry, and pagerank.hpp's predicate
// `error <= threshold` (:141, :216) or the iteration cap.  A stopped gate
// stays stopped (later updates and gated sweeps are no-ops).
__global__ void gate_update_kernel(GateHdr* g, PairPtrs pp, double threshold, int norm, uint64_t max_iterations) {
  if (g->stop) return;
  double err = 0.0, l1 = 0.0;
  for (int r = 0; r < pp.n; ++r) {
    const volatile double* q = pp.p[r];
    err = fmax(err, q[0]);
    l1 += q[1];
  }
  const unsigned long long it = g->iters;
  double* trace = reinterpret_cast<double*>(g + 1);
  if (it < g->cap) {
    trace[2 * it] = err;
    trace[2 * it + 1] = l1;
  }
  g->iters = it + 1;
  const double crit = norm ? l1 : err;  // FPR_B200_NORM_L1 = 1
  if (crit <= threshold || it + 1 >= max_iterations) g->stop = 1u;
}

__global__ void gate_init_kernel(GateHdr* g, uint64_t cap) {
  g->stop = 0u;
  g->pad = 0u;
  g->iters = 0ull;
  g->cap = cap;
  g->pad2 = 0ull;
}

cudaError_t launch_gate_init(GateHdr* g, uint64_t cap, cudaStream_t s) {
  gate_init_kernel<<<1, 1, 0, s>>>(g, cap);
  return cudaGetLastError();
}

cudaError_t launch_gate_update(GateHdr* g, const PairPtrs& pp, double threshold, int norm, uint64_t max_iterations,
                               cudaStream_t s) {
  gate_update_kernel<<<1, 1, 0, s>>>(g, pp, threshold, norm, max_iterations);
  return cudaGetLastError();
}

cudaError_t launch_solve(int engine, int grid, const SolveParams& p, cudaStream_t s) {
  const SolveShape sh = solve_shape(engine, p.npeers > 0 ? kModePeers : kModeFinal);
  SolveParams copy = p;
  void* args[] = {&copy};
  return cudaLaunchCooperativeKernel(sh.fn, dim3(grid), dim3(sh.block), args, sh.smem, s);
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

cudaError_t launch_part_bounds(const DevGraph& g, uint32_t nparts, int64_t* bounds, cudaStream_t s) {
  part_bounds_kernel<<<1, 128, 0, s>>>(g.row, g.n, g.m, nparts, bounds);
  return cudaGetLastError();
}

cudaError_t launch_part_extract(const DevGraph& g, const int64_t* bounds, uint32_t nparts,
                                uint32_t part, int64_t slice, int64_t nloc, int64_t mloc,
                                DevGraph& out, cudaStream_t s) {
  part_extract_kernel<<<grid_for(nloc > mloc ? nloc : mloc), 256, 0, s>>>(
      g.row, g.src, g.outdeg, bounds, nparts, part, slice, out.row, out.src, out.outdeg);
  return cudaGetLastError();
}

cudaError_t launch_offset_shift(int64_t* row, int64_t count, int64_t e0, cudaStream_t s) {
  if (count > 0) offset_shift_kernel<<<grid_for(count), 256, 0, s>>>(row, count, e0);
  return cudaGetLastError();
}

cudaError_t launch_part_remap(int32_t* src, int64_t m, const int64_t* bounds, uint32_t nparts, int64_t slice,
                              cudaStream_t s) {
  if (m > 0) part_remap_kernel<<<grid_for(m), 256, 0, s>>>(src, m, bounds, nparts, slice);
  return cudaGetLastError();
}

cudaError_t launch_part_init(const DevGraph& g, double init, double* pr, double* contrib_slice,
                             cudaStream_t s) {
  part_init_kernel<<<grid_for(g.n), 256, 0, s>>>(g.n, g.outdeg, init, pr, contrib_slice);
  return cudaGetLastError();
}

cudaError_t launch_validate(const DevGraph& g, int32_t* recount, unsigned int* bad, cudaStream_t s) {
  validate_kernel<<<grid_for(g.n), 256, 0, s>>>(g.row, g.src, g.n, g.m, recount, bad);
  compare_counts_kernel<<<grid_for(g.n), 256, 0, s>>>(recount, g.outdeg, g.n, bad);
  return cudaGetLastError();
}

__global__ void gather_ranks_kernel(const double* pr, const int32_t* new_of_old, int32_t n,
                                    double* out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = pr[new_of_old[i]];
}

cudaError_t launch_gather_ranks(const double* pr, const int32_t* new_of_old, int32_t n, double* out,
                               cudaStream_t s) {
  gather_ranks_kernel<<<grid_for(n), 256, 0, s>>>(pr, new_of_old, n, out);
  return cudaGetLastError();
}

cudaError_t launch_widen(const int64_t* row, const int32_t* ids32, uint64_t* out_row,
                         uint64_t* out_ids, int64_t nrow, int64_t nids, cudaStream_t s) {
  widen_kernel<<<grid_for(nrow > nids ? nrow : nids), 256, 0, s>>>(row, ids32, out_row, out_ids,
                                                                   nrow, nids);
  return cudaGetLastError();
}

}  // namespace fprb
