// runtime.cu -- C ABI (include/fpr_b200.h) and host runtime of libfpr_b200.so.
//
// Mirrors the reference's engine contract (pagerank.hpp): validation with the
// same predicates and messages (:40-53, :56), the convergence trace
// (errors[] = per-iteration max delta, iterations = errors.size(),
// converged = errors.back() <= threshold, detail::finish :104-109), and
// non-convergence as a result rather than an error.  There is no CPU
// fallback: every numeric step runs in the kernels of kernels.cu/generate.cu.
#include <cuda_runtime.h>
#include <omp.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/fpr_b200.h"
#include "internal.cuh"

using namespace fprb;

namespace {

thread_local std::string g_last_error;

int fail(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      return fail(e_ == cudaErrorMemoryAllocation ? FPR_B200_ENOMEM : FPR_B200_ECUDA,     \
                  std::string("fpr_b200: CUDA error '") + cudaGetErrorString(e_) + "' at " + \
                      __FILE__ + ":" + std::to_string(__LINE__) + " (" #call ")");         \
    }                                                                                     \
  } while (0)

constexpr uint32_t kChunkIters = 1u << 16;  // device trace capacity per launch

// Pinned host staging for the per-launch trace readback, pooled process-wide so
// a one-shot fpr_b200_pagerank() does not pay cudaMallocHost on every call.
struct HostStaging {
  SolveStatus* status = nullptr;
  unsigned int* iters = nullptr;
  int* stop = nullptr;
  double* errors = nullptr;
  double* l1 = nullptr;
  unsigned long long* ns = nullptr;
};
std::mutex g_staging_mu;
std::vector<HostStaging*> g_staging_free;

HostStaging* acquire_staging() {
  {
    std::lock_guard<std::mutex> lk(g_staging_mu);
    if (!g_staging_free.empty()) {
      HostStaging* s = g_staging_free.back();
      g_staging_free.pop_back();
      return s;
    }
  }
  auto* s = new HostStaging;
  if (cudaMallocHost(&s->status, sizeof(SolveStatus)) != cudaSuccess ||
      cudaMallocHost(&s->iters, sizeof(unsigned)) != cudaSuccess ||
      cudaMallocHost(&s->stop, sizeof(int)) != cudaSuccess ||
      cudaMallocHost(&s->errors, kChunkIters * sizeof(double)) != cudaSuccess ||
      cudaMallocHost(&s->l1, kChunkIters * sizeof(double)) != cudaSuccess ||
      cudaMallocHost(&s->ns, (kChunkIters + 1) * sizeof(unsigned long long)) != cudaSuccess) {
    for (void* p : {(void*)s->status, (void*)s->iters, (void*)s->stop, (void*)s->errors, (void*)s->l1,
                    (void*)s->ns})
      if (p) cudaFreeHost(p);
    delete s;
    return nullptr;
  }
  return s;
}

void release_staging(HostStaging* s) {
  if (!s) return;
  std::lock_guard<std::mutex> lk(g_staging_mu);
  g_staging_free.push_back(s);
}

// Pinned ring for uploads from PAGEABLE host memory (std::vector graphs of
// the C++ drop-in): host threads narrow u64 -> int32 (range-checking as they
// go) into a pinned buffer while the previous buffer's DMA is in flight, so
// the link carries 4 B per edge instead of 8.  One ring per device, reused.
constexpr int kRingBufs = 4;
constexpr double kHostNarrowShare = 0.9;  // measured default, see host_narrow_share()
constexpr int64_t kRingBytes = 32ll << 20;
struct UploadRing {
  int device = -1;
  void* buf[kRingBufs] = {};
  cudaEvent_t done[kRingBufs] = {};
  bool used[kRingBufs] = {};
  std::mutex mu;
};
std::mutex g_ring_mu;
std::vector<UploadRing*> g_rings;

UploadRing* get_ring(int device) {
  std::lock_guard<std::mutex> lk(g_ring_mu);
  for (auto* r : g_rings)
    if (r->device == device) return r;
  auto* r = new UploadRing;
  r->device = device;
  for (int k = 0; k < kRingBufs; ++k) {
    if (cudaMallocHost(&r->buf[k], kRingBytes) != cudaSuccess ||
        cudaEventCreateWithFlags(&r->done[k], cudaEventDisableTiming) != cudaSuccess) {
      for (int j = 0; j <= k; ++j) {
        if (r->buf[j]) cudaFreeHost(r->buf[j]);
        if (r->done[j]) cudaEventDestroy(r->done[j]);
      }
      delete r;
      return nullptr;
    }
  }
  g_rings.push_back(r);
  return r;
}

// Share of a PINNED in_src that host threads narrow (the rest is DMA'd raw
// and narrowed on the device).  Measured on the 16-core B200 hosts (config 2
// upload, scripts/narrow_sweep.py): 0 -> 11.2 ms, 0.7 -> 8.5, 0.9 -> 7.6,
// 1.0 -> 7.7 (host-bound).  Fewer host threads narrow proportionally less.
// FPR_B200_HOST_NARROW overrides (0..1).
double host_narrow_share() {
  const char* s = std::getenv("FPR_B200_HOST_NARROW");
  const double x = s ? std::atof(s) : kHostNarrowShare * std::min(1.0, omp_get_max_threads() / 16.0);
  return x < 0.0 ? 0.0 : (x > 1.0 ? 1.0 : x);
}

bool is_pinned(const void* p) {
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// Uploads `count` u64 values as T (int32 narrowed + range-checked against
// `bound`, or int64 verbatim) through the ring on stream s.  Returns false on
// an out-of-range value; *e receives CUDA errors.
template <class T>
bool ring_upload(UploadRing* r, const uint64_t* src, T* dst, int64_t count, uint64_t bound,
                 cudaStream_t s, int& k, cudaError_t* e) {
  const int64_t per = kRingBytes / (int64_t)sizeof(T);
  bool ok = true;
  for (int64_t off = 0; off < count && *e == cudaSuccess; off += per) {
    const int64_t cnt = std::min<int64_t>(per, count - off);
    if (r->used[k]) *e = cudaEventSynchronize(r->done[k]);
    if (*e != cudaSuccess) break;
    T* stage = static_cast<T*>(r->buf[k]);
    const uint64_t* in = src + off;
    if constexpr (sizeof(T) == 4) {
      ok = !host_narrow_ids(in, reinterpret_cast<int32_t*>(stage), cnt, bound) && ok;
    } else {
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < cnt; ++i) stage[i] = (T)in[i];
    }
    *e = cudaMemcpyAsync(dst + off, stage, cnt * sizeof(T), cudaMemcpyHostToDevice, s);
    if (*e == cudaSuccess) *e = cudaEventRecord(r->done[k], s);
    r->used[k] = true;
    k = (k + 1) % kRingBufs;
  }
  return ok;
}

// Uploads `len` bytes of PAGEABLE host memory through the ring (parallel
// memcpy into a pinned buffer while the previous one's DMA is in flight).
void ring_upload_bytes(UploadRing* r, const char* src, unsigned char* dst, int64_t len, cudaStream_t s,
                       cudaError_t* e) {
  int k = 0;
  for (int64_t off = 0; off < len && *e == cudaSuccess; off += kRingBytes) {
    const int64_t cnt = std::min<int64_t>(kRingBytes, len - off);
    if (r->used[k]) *e = cudaEventSynchronize(r->done[k]);
    if (*e != cudaSuccess) break;
    char* stage = static_cast<char*>(r->buf[k]);
    const int64_t piece = 1 << 20;
#pragma omp parallel for schedule(static)
    for (int64_t p = 0; p < cnt; p += piece) std::memcpy(stage + p, src + off + p, std::min(piece, cnt - p));
    *e = cudaMemcpyAsync(dst + off, stage, cnt, cudaMemcpyHostToDevice, s);
    if (*e == cudaSuccess) *e = cudaEventRecord(r->done[k], s);
    r->used[k] = true;
    k = (k + 1) % kRingBufs;
  }
}

struct Waves {
  int32_t nwaves = 0;
  int32_t* d_task = nullptr;
  int32_t* d_row = nullptr;
  std::vector<uint64_t> vertex_start;  // nwaves+1
};

}  // namespace

struct fpr_b200_graph {
  int device = 0;
  int num_sms = 148;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int norm = FPR_B200_NORM_LINF;
  uint32_t wave_count = 0;
  DevGraph g;
  Partition part;
  double* pr = nullptr;
  double* contrib[2] = {nullptr, nullptr};
  double* tail_partial = nullptr;
  int grid_full[2] = {0, 0};  // [0]=Jacobi/lockstep kernel, [1]=async kernel
  int async_shape = kFused;   // kFusedWide when the contributions exceed ~64 MB
  double* partials = nullptr;
  double* totals = nullptr;
  GridBar* bar = nullptr;
  SolveStatus* d_status = nullptr;  // iters, stop, last residual pair: one readback per launch
  double* d_errors = nullptr;
  double* d_l1 = nullptr;
  unsigned long long* d_ns = nullptr;
  // pinned host staging (pooled)
  HostStaging* hs = nullptr;
  unsigned int* h_iters = nullptr;
  int* h_stop = nullptr;
  double* h_errors = nullptr;
  double* h_l1 = nullptr;
  unsigned long long* h_ns = nullptr;
  cudaStream_t copy_stream = nullptr;  // H2D upload overlapped with narrowing
  cudaStream_t ring_stream = nullptr;  // host-narrowed share of a pinned upload
  cudaEvent_t ring_ev = nullptr;
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  cudaEvent_t up_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  std::map<uint32_t, Waves> waves;
  std::vector<void*> allocs;
  // multi-GPU part (fpr_b200_graph_partition); nparts == 1 for a whole graph
  uint32_t nparts = 1, part_id = 0;
  uint32_t flags = 0;
  int32_t* new_of_old = nullptr;  // FPR_B200_OPT_REORDER(_SOURCES): caller id -> internal id
  bool use_pb = false;            // propagation-blocked sweeps (decided at creation, pb_wanted)
  PbSet* pb = nullptr;            // their layout: built at the first EC / lockstep / FUSED run
  uint64_t part_sweeps = 0;       // part sweeps since fpr_b200_part_init
  double* part_pr[2] = {nullptr, nullptr};  // part ranks ping-pong ([0] = pr)
  int part_pr_cur = 0;                       // buffer holding the latest sweep
  const unsigned int* gate = nullptr;        // device-side stop flag (fpr_b200_part_set_gate)
  double* ranks_tmp = nullptr;    // reordered ranks gathered back to caller order
  uint64_t n_global = 0, row_begin = 0, slice = 0;
};

namespace {

int dalloc(fpr_b200_graph* h, void** p, size_t bytes) {
  if (bytes == 0) bytes = 8;
  cudaError_t e = cudaMallocAsync(p, bytes, h->stream);
  if (e != cudaSuccess) {
    *p = nullptr;
    return fail(e == cudaErrorMemoryAllocation ? FPR_B200_ENOMEM : FPR_B200_ECUDA,
                std::string("fpr_b200: device allocation of ") + std::to_string(bytes) +
                    " bytes failed: " + cudaGetErrorString(e));
  }
  h->allocs.push_back(*p);
  return FPR_B200_OK;
}

template <class T>
int dalloc_n(fpr_b200_graph* h, T** p, size_t count) {
  return dalloc(h, reinterpret_cast<void**>(p), count * sizeof(T));
}

void destroy_handle(fpr_b200_graph* h) {
  if (!h) return;
  cudaSetDevice(h->device);
  if (h->stream) cudaStreamSynchronize(h->stream);
  for (void* p : h->allocs) cudaFreeAsync(p, h->stream);
  if (h->pb) {
    free_pb(*h->pb, h->stream);
    delete h->pb;
    h->pb = nullptr;
  }
  if (h->stream) cudaStreamSynchronize(h->stream);
  release_staging(h->hs);
  for (auto& e : h->ev)
    if (e) cudaEventDestroy(e);
  for (auto& e : h->up_ev)
    if (e) cudaEventDestroy(e);
  if (h->copy_stream) cudaStreamDestroy(h->copy_stream);
  if (h->ring_ev) cudaEventDestroy(h->ring_ev);
  if (h->ring_stream) cudaStreamDestroy(h->ring_stream);
  if (h->own_stream && h->stream) cudaStreamDestroy(h->stream);
  delete h;
}

// Device selection, stream, pool and the per-handle capability checks.
int open_handle(const fpr_b200_options* opts, fpr_b200_graph** out) {
  fpr_b200_options o;
  fpr_b200_options_init(&o);
  if (opts) o = *opts;
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  if (e != cudaSuccess || ndev == 0)
    return fail(FPR_B200_ECUDA, std::string("fpr_b200: no CUDA device available (") +
                                    cudaGetErrorString(e) + ")");
  auto* h = new fpr_b200_graph;
  if (o.device >= 0) {
    h->device = o.device;
  } else {
    cudaGetDevice(&h->device);
  }
  *out = h;
  CK(cudaSetDevice(h->device));
  int coop = 0, cc_major = 0;
  CK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, h->device));
  CK(cudaDeviceGetAttribute(&h->num_sms, cudaDevAttrMultiProcessorCount, h->device));
  CK(cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, h->device));
  if (!coop) return fail(FPR_B200_ECUDA, "fpr_b200: device lacks cooperative launch");
  if (cc_major != 10)
    return fail(FPR_B200_ECUDA, "fpr_b200: built for sm_100a (B200); device compute capability " +
                                    std::to_string(cc_major) + ".x is not supported");
  if (o.stream) {
    h->stream = static_cast<cudaStream_t>(o.stream);
  } else {
    CK(cudaStreamCreateWithFlags(&h->stream, cudaStreamNonBlocking));
    h->own_stream = true;
  }
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, h->device) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  h->norm = o.norm;
  h->wave_count = o.wave_count;
  h->flags = o.flags;
  for (auto& ev : h->ev) CK(cudaEventCreate(&ev));
  h->hs = acquire_staging();
  if (!h->hs) return fail(FPR_B200_ENOMEM, "fpr_b200: pinned host staging allocation failed");
  h->h_iters = h->hs->iters;
  h->h_stop = h->hs->stop;
  h->h_errors = h->hs->errors;
  h->h_l1 = h->hs->l1;
  h->h_ns = h->hs->ns;
  return FPR_B200_OK;
}

// Partition + solver state, common to create/generate (after the optional
// locality reorder, which swaps in the renumbered CSR).
#ifdef FPR_TRACE_WARPS
constexpr int64_t kTraceWarps = 8192;  // per-warp timestamps after the tail partials
#else
constexpr int64_t kTraceWarps = 0;
#endif

// Sweep kind, fixed at creation: OPT_PULL / OPT_PB force it; by default
// propagation blocking when the contribution vector (8 n bytes) exceeds half
// the L2 -- past it the pull gathers start missing L2 (each miss moves ~64 B
// of DRAM for 8 useful bytes) and the run-sum PB sweep wins: config 3 (134 MB)
// 1.04 vs 1.61 ms, configs 4/5 3x; on config 2 (33.5 MB, L2-resident) the
// pull sweep wins, 0.32 vs 0.36 ms.
// A multi-GPU part gathers from the whole exchange space (nparts x slice
// contributions), so the rule uses that size.
int64_t source_space(const fpr_b200_graph* h) {
  return h->nparts > 1 ? (int64_t)h->nparts * (int64_t)h->slice : (int64_t)h->g.n;
}

void pb_geometry(int* shift, int* chunk_shift);

bool pb_wanted(const fpr_b200_graph* h) {
  if (h->flags & FPR_B200_OPT_PULL) return false;
  if (h->flags & FPR_B200_OPT_PB) return true;
  int l2 = 0;
  if (cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, h->device) != cudaSuccess || l2 <= 0) l2 = 126 << 20;
  const int64_t bytes = source_space(h) * (int64_t)sizeof(double);
  if (const char* v = std::getenv("FPR_B200_PB_AUTO_BYTES")) return bytes > std::atoll(v);  // tests
  return bytes > (int64_t)l2 / 2;
}

int finish_graph(fpr_b200_graph* h) {
  if ((h->flags & (FPR_B200_OPT_REORDER | FPR_B200_OPT_REORDER_SOURCES | FPR_B200_OPT_REORDER_BLOCKS)) &&
      h->g.n > 1) {
    DevGraph re;
    int32_t* perm = nullptr;
    const char* msg = nullptr;
    const bool by_degree = h->flags & (FPR_B200_OPT_REORDER | FPR_B200_OPT_REORDER_BLOCKS);
    // degree order inside blocks of the PB source chunk (unless OPT_REORDER)
    int shift = 0, chunk_shift = 0;
    pb_geometry(&shift, &chunk_shift);
    const int block_shift = (h->flags & FPR_B200_OPT_REORDER) ? 0 : std::max(1, std::min(chunk_shift, 23));
    CK(reorder_by_degree(h->g, !by_degree, by_degree ? block_shift : 0, re, &perm, h->stream, &msg));
    if (msg) return fail(FPR_B200_ENOMEM, std::string("fpr_b200 reorder: ") + msg);
    h->allocs.push_back(re.row);
    h->allocs.push_back(re.src);
    h->allocs.push_back(re.outdeg);
    h->allocs.push_back(perm);
    h->g = re;  // the original arrays stay owned by allocs until destroy
    h->new_of_old = perm;
    int rc2 = dalloc_n(h, &h->ranks_tmp, h->g.n);
    if (rc2) return rc2;
  }
  DevGraph& g = h->g;
  Partition& p = h->part;
  const int64_t items = (int64_t)g.n + g.m;
  const int64_t nt = (items + kTaskDiag - 1) / kTaskDiag;
  if (nt >= INT32_MAX) return fail(FPR_B200_ERANGE, "fpr_b200: graph too large for task index");
  p.ntasks = (int32_t)nt;
  int rc;
  if ((rc = dalloc_n(h, &p.task_row, nt + 1)) || (rc = dalloc_n(h, &p.task_edge, nt + 1)) ||
      (rc = dalloc_n(h, &p.head_first, nt + 1)) || (rc = dalloc_n(h, &p.clean_start, nt + 1)) ||
      (rc = dalloc_n(h, &p.task_bits, 8 * (nt + 1))))
    return rc;
  if (g.n > 0) CK(launch_partition(g, p, h->stream));
  if ((rc = dalloc_n(h, &h->pr, g.n)) || (rc = dalloc_n(h, &h->contrib[0], g.n)) ||
      (rc = dalloc_n(h, &h->contrib[1], g.n)) || (rc = dalloc_n(h, &h->tail_partial, nt + 1 + kTraceWarps)))
    return rc;
  // tail partials start "not ready" (NaN); each consumer re-arms what it reads.
  CK(cudaMemsetAsync(h->tail_partial, 0xFF, (nt + 1) * sizeof(double), h->stream));
  CK(solve_grid(kEC, h->num_sms, &h->grid_full[0]));
  h->async_shape = (int64_t)g.n * (int64_t)sizeof(double) > (64ll << 20) ? kFusedWide : kFused;
  CK(solve_grid(h->async_shape, h->num_sms, &h->grid_full[1]));
  const int gmax = std::max(h->grid_full[0], h->grid_full[1]);
  if ((rc = dalloc_n(h, &h->partials, 2 * gmax)) || (rc = dalloc_n(h, &h->totals, 2)) ||
      (rc = dalloc_n(h, &h->bar, 1)) || (rc = dalloc_n(h, &h->d_status, 1)) ||
      (rc = dalloc_n(h, &h->d_errors, kChunkIters)) ||
      (rc = dalloc_n(h, &h->d_l1, kChunkIters)) || (rc = dalloc_n(h, &h->d_ns, kChunkIters + 1)))
    return rc;
  CK(cudaMemsetAsync(h->bar, 0, sizeof(GridBar), h->stream));
  CK(cudaStreamSynchronize(h->stream));
  h->use_pb = pb_wanted(h);
  return FPR_B200_OK;
}

// Wave boundaries of the lockstep schedule: task indices where a task starts
// on a row boundary, so that no split row straddles two waves.
int get_waves(fpr_b200_graph* h, uint32_t wave_count, const Waves** out) {
  const int64_t items = (int64_t)h->g.n + h->g.m;
  uint32_t S = wave_count;
  if (S == 0) {
    // Auto: one wave per ~32M merge items.  Each wave costs a grid barrier
    // plus a pipeline drain/refill (8-25 us); more waves recover more of the
    // Gauss-Seidel gain.  Measured time-to-converge optima (scripts/
    // wave_probe.py): config 2 (71M items) 2 waves, config 3 (280M) 8,
    // config 4 (1.2G) 16-32, config 5 (4.5G) 16-32.
    const int64_t want = items >> 25;
    S = (uint32_t)std::min<int64_t>(32, std::max<int64_t>(2, want));
  }
  auto it = h->waves.find(S);
  if (it != h->waves.end()) {
    *out = &it->second;
    return FPR_B200_OK;
  }
  const int32_t nt = h->part.ntasks;
  if (S == 1) {  // Jacobi: one wave over every task, nothing to download
    Waves wv;
    wv.nwaves = 1;
    const int32_t wt[2] = {0, nt}, wr[2] = {0, h->g.n};
    wv.vertex_start = {0, (uint64_t)h->g.n};
    int rc;
    if ((rc = dalloc_n(h, &wv.d_task, 2)) || (rc = dalloc_n(h, &wv.d_row, 2))) return rc;
    CK(cudaMemcpyAsync(wv.d_task, wt, sizeof(wt), cudaMemcpyHostToDevice, h->stream));
    CK(cudaMemcpyAsync(wv.d_row, wr, sizeof(wr), cudaMemcpyHostToDevice, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    auto res = h->waves.emplace(S, std::move(wv));
    *out = &res.first->second;
    return FPR_B200_OK;
  }
  std::vector<uint8_t> clean(nt + 1);
  std::vector<int32_t> trow(nt + 1);
  CK(cudaMemcpyAsync(clean.data(), h->part.clean_start, nt + 1, cudaMemcpyDeviceToHost, h->stream));
  CK(cudaMemcpyAsync(trow.data(), h->part.task_row, (nt + 1) * sizeof(int32_t),
                     cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  std::vector<int32_t> wt{0};
  for (uint32_t w = 1; w < S; ++w) {
    int64_t t = (int64_t)nt * w / S;
    if (t <= wt.back()) t = wt.back() + 1;
    while (t < nt && !clean[t]) ++t;
    if (t >= nt) break;
    wt.push_back((int32_t)t);
  }
  wt.push_back(nt);
  Waves wv;
  wv.nwaves = (int32_t)wt.size() - 1;
  std::vector<int32_t> wr(wt.size());
  for (size_t i = 0; i < wt.size(); ++i) {
    wr[i] = trow[wt[i]];
    wv.vertex_start.push_back((uint64_t)wr[i]);
  }
  int rc;
  if ((rc = dalloc_n(h, &wv.d_task, wt.size())) || (rc = dalloc_n(h, &wv.d_row, wt.size())))
    return rc;
  CK(cudaMemcpyAsync(wv.d_task, wt.data(), wt.size() * sizeof(int32_t), cudaMemcpyHostToDevice,
                     h->stream));
  CK(cudaMemcpyAsync(wv.d_row, wr.data(), wr.size() * sizeof(int32_t), cudaMemcpyHostToDevice,
                     h->stream));
  CK(cudaStreamSynchronize(h->stream));
  auto res = h->waves.emplace(S, std::move(wv));
  *out = &res.first->second;
  return FPR_B200_OK;
}

int validate_config(const fpr_config* cfg) {
  // validate(PageRankConfig), pagerank.hpp:40-53 -- same predicates and text.
  if (!(cfg->damping > 0.0 && cfg->damping < 1.0))
    return fail(FPR_B200_EINVAL, "pagerank: damping must be in (0,1)");
  if (!(cfg->threshold > 0.0)) return fail(FPR_B200_EINVAL, "pagerank: threshold must be positive");
  if (cfg->max_iterations == 0)
    return fail(FPR_B200_EINVAL, "pagerank: max_iterations must be positive");
  if (cfg->thread_count == 0)
    return fail(FPR_B200_EINVAL, "pagerank: thread_count must be positive");
  return FPR_B200_OK;
}

// Propagation-blocked geometry: 2^13-row bins (64 KB of shared accumulators,
// 2 CTAs per SM) and 2^23-source chunks (a 64 MB contribution window: the
// larger the chunk, the longer a row's runs and the fewer partial sums, until
// the window stops fitting L2 -- 2^24 loses 30% on config 4's unordered
// ids); measured on configs 4/5.  The environment
// overrides are for tests and probes.
void pb_geometry(int* shift, int* chunk_shift) {
  *shift = 13;
  *chunk_shift = 23;
  if (const char* s = std::getenv("FPR_B200_PB_SHIFT")) *shift = std::atoi(s);
  if (const char* s = std::getenv("FPR_B200_PB_CHUNK_SHIFT")) *chunk_shift = std::atoi(s);
}

// Lockstep wave count: the requested one, or an auto rule.  Plain sweeps:
// the rule of get_waves.  Propagation-blocked sweeps: every wave re-walks
// all chunk windows and drains two launches, so fewer waves pay: one per
// 128 M merge items, 2-8 (measured optima: config 4 4-8 waves, config 5 8;
// DESIGN.md §3.4).
// EC on propagation-blocked sweeps: one wave (every bin reads the previous
// sweep's contributions).  FPR_B200_PB_EC_WAVES splits it for tests: the
// waves run one after the other (round 1 overlapped them on two streams,
// wave w+1's gather beside wave w's accumulate: slower).
uint32_t pb_ec_waves(const fpr_b200_graph* h) {
  (void)h;
  uint32_t w = 1;
  if (const char* v = std::getenv("FPR_B200_PB_EC_WAVES")) w = (uint32_t)std::max(1, std::min(64, std::atoi(v)));
  return w;
}

uint32_t lockstep_waves(const fpr_b200_graph* h) {
  if (h->wave_count) return h->wave_count;
  const int64_t items = (int64_t)h->g.n + h->g.m;
  if (h->use_pb) return (uint32_t)std::min<int64_t>(8, std::max<int64_t>(2, items >> 26));
  return (uint32_t)std::min<int64_t>(32, std::max<int64_t>(2, items >> 25));
}

}  // namespace

extern "C" {

void fpr_b200_options_init(fpr_b200_options* o) {
  if (!o) return;
  std::memset(o, 0, sizeof(*o));
  o->device = -1;
  o->norm = FPR_B200_NORM_LINF;
}

void fpr_b200_config_init(fpr_config* c) {
  if (!c) return;
  c->damping = 0.85;
  c->threshold = 1e-15;
  c->max_iterations = 10000;
  c->thread_count = 1;
}

const char* fpr_b200_last_error(void) { return g_last_error.c_str(); }

int fpr_b200_version(void) { return 1; }

// Pinned u64 id arrays -> int32 device arrays, range-checked against `bound`
// (a failure sets *bad).  The link is the bound at 8 B per id, so for arrays
// marked `split` host threads narrow the last host_narrow_share() to 4 B per
// id through the pinned ring (ring stream) while the DMA engine moves the rest
// raw into two device staging buffers that the main stream narrows, chunk i
// copying while chunk i-1 narrows (e2e).  An optional raw blob
// (in_start) goes first on the copy stream.  Ordered before later work on
// h->stream; returns a status code, CUDA errors in *e.
struct IdUpload {
  const uint64_t* host;
  int32_t* dev;
  int64_t count;
  bool split;
};

int upload_ids_pinned(fpr_b200_graph* h, const std::vector<IdUpload>& arrays, uint64_t bound, unsigned int* bad,
                      const void* raw_host, void* raw_dev, size_t raw_bytes, cudaError_t* e) {
  const int64_t chunk = 1 << 24;
  struct Piece {
    const uint64_t* host;
    int32_t* dst;
    int64_t count;
  };
  std::vector<Piece> pieces;
  struct HostPart {
    const uint64_t* host;
    int32_t* dst;
    int64_t count;
  };
  std::vector<HostPart> host_parts;
  const double share = host_narrow_share();
  int64_t most = 0;
  for (const IdUpload& a : arrays) {
    const int64_t nh = a.split ? (int64_t)((double)a.count * share) : 0;
    const int64_t nd = a.count - nh;
    for (int64_t off = 0; off < nd; off += chunk) pieces.push_back({a.host + off, a.dev + off, std::min(chunk, nd - off)});
    if (nh > 0) host_parts.push_back({a.host + nd, a.dev + nd, nh});
    most = std::max(most, std::min(chunk, nd));
  }
  UploadRing* ring = host_parts.empty() ? nullptr : get_ring(h->device);
  if (!host_parts.empty() && !ring) return fail(FPR_B200_ENOMEM, "fpr_b200: pinned upload ring allocation failed");
  uint64_t* stage = nullptr;
  if (*e == cudaSuccess && most > 0) *e = cudaMallocAsync((void**)&stage, 2 * most * sizeof(uint64_t), h->stream);
  if (*e == cudaSuccess && !h->copy_stream) *e = cudaStreamCreateWithFlags(&h->copy_stream, cudaStreamNonBlocking);
  for (auto& ev : h->up_ev)
    if (*e == cudaSuccess && !ev) *e = cudaEventCreateWithFlags(&ev, cudaEventDisableTiming);
  if (*e == cudaSuccess) *e = cudaEventRecord(h->up_ev[2], h->stream);  // destinations + staging allocated
  if (*e == cudaSuccess) *e = cudaStreamWaitEvent(h->copy_stream, h->up_ev[2], 0);
  if (*e == cudaSuccess && raw_bytes)
    *e = cudaMemcpyAsync(raw_dev, raw_host, raw_bytes, cudaMemcpyHostToDevice, h->copy_stream);
  for (size_t i = 0; *e == cudaSuccess && i < pieces.size(); ++i) {
    const int k = (int)(i & 1);
    uint64_t* buf = stage + k * most;
    if (i >= 2) *e = cudaStreamWaitEvent(h->copy_stream, h->up_ev[2 + k], 0);  // buf drained
    if (*e == cudaSuccess)
      *e = cudaMemcpyAsync(buf, pieces[i].host, pieces[i].count * sizeof(uint64_t), cudaMemcpyHostToDevice,
                           h->copy_stream);
    if (*e == cudaSuccess) *e = cudaEventRecord(h->up_ev[k], h->copy_stream);
    if (*e == cudaSuccess) *e = cudaStreamWaitEvent(h->stream, h->up_ev[k], 0);
    if (*e == cudaSuccess) *e = launch_narrow_ids(buf, pieces[i].dst, pieces[i].count, bound, bad, h->stream);
    if (*e == cudaSuccess) *e = cudaEventRecord(h->up_ev[2 + k], h->stream);
  }
  if (*e == cudaSuccess && raw_bytes && pieces.empty()) {  // raw blob alone: order it before later work
    *e = cudaEventRecord(h->up_ev[0], h->copy_stream);
    if (*e == cudaSuccess) *e = cudaStreamWaitEvent(h->stream, h->up_ev[0], 0);
  }
  if (*e == cudaSuccess && !host_parts.empty()) {
    if (!h->ring_stream) *e = cudaStreamCreateWithFlags(&h->ring_stream, cudaStreamNonBlocking);
    if (*e == cudaSuccess && !h->ring_ev) *e = cudaEventCreateWithFlags(&h->ring_ev, cudaEventDisableTiming);
    if (*e == cudaSuccess) *e = cudaEventRecord(h->ring_ev, h->stream);
    if (*e == cudaSuccess) *e = cudaStreamWaitEvent(h->ring_stream, h->ring_ev, 0);
    std::lock_guard<std::mutex> lk(ring->mu);
    int k = 0;
    bool ok = true;
    for (const HostPart& hp : host_parts)
      if (*e == cudaSuccess) ok = ring_upload<int32_t>(ring, hp.host, hp.dst, hp.count, bound, h->ring_stream, k, e) && ok;
    if (*e == cudaSuccess) *e = cudaEventRecord(h->ring_ev, h->ring_stream);
    if (*e == cudaSuccess) *e = cudaStreamWaitEvent(h->stream, h->ring_ev, 0);
    if (*e == cudaSuccess && !ok) *e = cudaMemsetAsync(bad, 1, 1, h->stream);  // reported with the device check
  }
  if (stage) cudaFreeAsync(stage, h->stream);  // after the last narrow on h->stream
  return FPR_B200_OK;
}

int fpr_b200_graph_create(const fpr_graph_view* v, const fpr_b200_options* opts,
                          fpr_b200_graph** out) {
  if (!v || !out) return fail(FPR_B200_EINVAL, "fpr_b200_graph_create: null argument");
  *out = nullptr;
  if (v->n >= (1ULL << 31))
    return fail(FPR_B200_ERANGE, "fpr_b200: n = " + std::to_string(v->n) +
                                     " exceeds the int32 vertex-id range (n < 2^31)");
  if (v->n > 0 && !v->in_start) return fail(FPR_B200_EINVAL, "fpr_b200: null in_start");
  if (v->m > 0 && !v->in_src) return fail(FPR_B200_EINVAL, "fpr_b200: null in_src");
  if (v->n > 0 && !v->out_degree) return fail(FPR_B200_EINVAL, "fpr_b200: null out_degree");
  fpr_b200_graph* h = nullptr;
  int rc = open_handle(opts, &h);
  if (rc) {
    destroy_handle(h);
    return rc;
  }
  auto bail = [&](int code) {
    destroy_handle(h);
    return code;
  };
  DevGraph& g = h->g;
  g.n = (int32_t)v->n;
  g.m = (int64_t)v->m;
  if ((rc = dalloc_n(h, &g.row, g.n + 1)) || (rc = dalloc_n(h, &g.src, g.m + 8)) ||
      (rc = dalloc_n(h, &g.outdeg, g.n)))
    return bail(rc);
  unsigned int* bad = nullptr;
  if ((rc = dalloc_n(h, &bad, 1))) return bail(rc);
  cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(unsigned), h->stream);
  const bool pinned = g.n > 0 && is_pinned(v->in_start) && (g.m == 0 || is_pinned(v->in_src)) &&
                      is_pinned(v->out_degree);
  if (e == cudaSuccess && g.n > 0 && !pinned) {
    // Pageable source: host-side narrowing through the pinned ring.
    UploadRing* ring = get_ring(h->device);
    if (!ring) return bail(fail(FPR_B200_ENOMEM, "fpr_b200: pinned upload ring allocation failed"));
    std::lock_guard<std::mutex> lk(ring->mu);
    int k = 0;
    bool ok = ring_upload<int64_t>(ring, v->in_start, g.row, (int64_t)g.n + 1, 0, h->stream, k, &e);
    ok = ring_upload<int32_t>(ring, v->in_src, g.src, g.m, v->n, h->stream, k, &e) && ok;
    ok = ring_upload<int32_t>(ring, v->out_degree, g.outdeg, g.n, v->n, h->stream, k, &e) && ok;
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);  // ring reusable once we return
    if (e == cudaSuccess && !ok)
      return bail(fail(FPR_B200_EINVAL, "fpr_b200: in_src/out_degree value outside [0," +
                                            std::to_string(v->n) + ")"));
  }
  if (e == cudaSuccess && g.n > 0 && pinned) {
    // in_src split between raw DMA and host narrowing; out_degree raw;
    // in_start (int64 as is) first on the copy stream.
    const std::vector<IdUpload> arrays = {{v->in_src, g.src, g.m, true}, {v->out_degree, g.outdeg, g.n, false}};
    if ((rc = upload_ids_pinned(h, arrays, v->n, bad, v->in_start, g.row, (g.n + 1) * sizeof(int64_t), &e)))
      return bail(rc);
  }
  if (e == cudaSuccess && g.n > 0) e = launch_check_offsets(g.row, g.n, g.m, bad, h->stream);
  unsigned hbad = 0;
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(h->h_iters, bad, sizeof(unsigned), cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess)
    return bail(fail(FPR_B200_ECUDA, std::string("fpr_b200_graph_create: ") + cudaGetErrorString(e)));
  hbad = *h->h_iters;
  if (hbad & 1u)
    return bail(fail(FPR_B200_EINVAL, "fpr_b200: in_src/out_degree value outside [0," +
                                          std::to_string(v->n) + ")"));
  if (hbad & 6u)
    return bail(fail(FPR_B200_EINVAL, "fpr_b200: in_start is not a valid CSR offset array "
                                      "(in_start[0]==0, non-decreasing, in_start[n]==m)"));
  if ((rc = finish_graph(h))) return bail(rc);
  *out = h;
  return FPR_B200_OK;
}

}  // extern "C"

namespace {
// validate(RmatParams) (rmat.hpp:24-35, same text) and the other generators' ranges.
int check_gen(const GenRequest& req) {
  if (req.kind == FPR_B200_GEN_RMAT) {
    // validate(RmatParams), rmat.hpp:24-35 -- same text.
    if (req.scale == 0 || req.scale > 32)
      return fail(FPR_B200_EINVAL, "rmat: scale must be in [1,32], got " + std::to_string(req.scale));
    if (req.edge_factor == 0) return fail(FPR_B200_EINVAL, "rmat: edge_factor must be positive");
    if (req.a < 0 || req.b < 0 || req.c < 0 || req.d < 0 ||
        std::abs(req.a + req.b + req.c + req.d - 1.0) > 1e-9)
      return fail(FPR_B200_EINVAL,
                  "rmat: quadrant probabilities must be non-negative and sum to 1");
    if (req.scale > 30)
      return fail(FPR_B200_ERANGE, "fpr_b200: rmat scale > 30 exceeds the int32 vertex-id range");
  } else if (req.kind == FPR_B200_GEN_UNIFORM) {
    if (req.n == 0) return fail(FPR_B200_EINVAL, "fpr_b200: uniform generator needs n > 0");
    if (req.n >= (1ULL << 31))
      return fail(FPR_B200_ERANGE, "fpr_b200: n exceeds the int32 vertex-id range");
  } else if (req.kind == FPR_B200_GEN_CHUNGLU) {
    if (req.n == 0) return fail(FPR_B200_EINVAL, "fpr_b200: chung-lu generator needs n > 0");
    if (req.n >= (1ULL << 31))
      return fail(FPR_B200_ERANGE, "fpr_b200: n exceeds the int32 vertex-id range");
    if (!(req.alpha > 1.0) || req.kmax == 0 || req.kmax > (1ull << 28))
      return fail(FPR_B200_EINVAL, "fpr_b200: chung-lu needs alpha > 1 and 1 <= kmax <= 2^28");
  } else {
    return fail(FPR_B200_EINVAL, "fpr_b200: unknown generator kind");
  }
  if (req.relabel_bfs) {
    const uint64_t nn = req.kind == FPR_B200_GEN_RMAT ? (1ull << req.scale) : req.n;
    if (req.bfs_root >= nn) return fail(FPR_B200_EINVAL, "fpr_b200: bfs_root outside [0,n)");
  }
  return FPR_B200_OK;
}

GenRequest gen_request(const fpr_gen_params* prm) {
  return GenRequest{prm->kind, prm->scale,      prm->edge_factor, prm->a,
                    prm->b,    prm->c,          prm->d,           prm->n,
                    prm->avg_degree, prm->seed, prm->draws,      prm->alpha,
                    prm->kmax, prm->relabel_bfs, prm->bfs_root};
}
}  // namespace

extern "C" {

int fpr_b200_generate_edges(const fpr_gen_params* prm, const fpr_b200_options* opts, uint64_t* src, uint64_t* dst,
                            uint64_t cap, uint64_t* count_out) {
  if (!prm || !count_out) return fail(FPR_B200_EINVAL, "fpr_b200_generate_edges: null argument");
  const GenRequest req = gen_request(prm);
  int rc = check_gen(req);
  if (rc) return rc;
  if (req.kind != FPR_B200_GEN_RMAT && req.kind != FPR_B200_GEN_UNIFORM)
    return fail(FPR_B200_EINVAL, "fpr_b200_generate_edges: raw draws exist for the rmat and uniform generators");
  const uint64_t draws = req.kind == FPR_B200_GEN_RMAT ? req.edge_factor << req.scale : req.n * req.avg_degree;
  fpr_b200_graph* h = nullptr;
  if ((rc = open_handle(opts, &h))) {
    destroy_handle(h);
    return rc;
  }
  const uint64_t chunk = std::min<uint64_t>(draws, 1ull << 24);
  uint64_t *d = nullptr, *hb = nullptr;
  uint64_t kept = 0;
  cudaError_t e = cudaMallocAsync(&d, 2 * std::max<uint64_t>(chunk, 1) * sizeof(uint64_t), h->stream);
  if (e == cudaSuccess) e = cudaMallocHost(&hb, 2 * std::max<uint64_t>(chunk, 1) * sizeof(uint64_t));
  for (uint64_t i0 = 0; e == cudaSuccess && i0 < draws; i0 += chunk) {
    const uint64_t cnt = std::min(chunk, draws - i0);
    e = generate_draws(req, i0, cnt, d, d + chunk, h->stream);
    if (e == cudaSuccess) e = cudaMemcpyAsync(hb, d, cnt * sizeof(uint64_t), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess)
      e = cudaMemcpyAsync(hb + chunk, d + chunk, cnt * sizeof(uint64_t), cudaMemcpyDeviceToHost, h->stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    for (uint64_t i = 0; e == cudaSuccess && i < cnt; ++i) {
      // generate_rmat keeps every draw; random_sparse skips self-loops
      if (req.kind == FPR_B200_GEN_UNIFORM && hb[i] == hb[chunk + i]) continue;
      if (src && dst && kept < cap) {
        src[kept] = hb[i];
        dst[kept] = hb[chunk + i];
      }
      ++kept;
    }
  }
  if (d) cudaFreeAsync(d, h->stream);
  if (h->stream) cudaStreamSynchronize(h->stream);
  if (hb) cudaFreeHost(hb);
  destroy_handle(h);
  if (e != cudaSuccess)
    return fail(FPR_B200_ECUDA, std::string("fpr_b200_generate_edges: ") + cudaGetErrorString(e));
  *count_out = kept;
  if (src && dst && kept > cap)
    return fail(FPR_B200_ERANGE, "fpr_b200_generate_edges: " + std::to_string(kept) + " edges, capacity " +
                                     std::to_string(cap));
  return FPR_B200_OK;
}

int fpr_b200_graph_generate(const fpr_gen_params* prm, const fpr_b200_options* opts,
                            fpr_b200_graph** out) {
  if (!prm || !out) return fail(FPR_B200_EINVAL, "fpr_b200_graph_generate: null argument");
  *out = nullptr;
  GenRequest req = gen_request(prm);
  int rc0 = check_gen(req);
  if (rc0) return rc0;
  fpr_b200_graph* h = nullptr;
  int rc = open_handle(opts, &h);
  if (rc) {
    destroy_handle(h);
    return rc;
  }
  const char* msg = nullptr;
  cudaError_t e = generate_graph(req, h->g, h->stream, &msg);
  if (e != cudaSuccess || msg) {
    destroy_handle(h);
    if (msg) return fail(FPR_B200_ENOMEM, std::string("fpr_b200_graph_generate: ") + msg);
    return fail(e == cudaErrorMemoryAllocation ? FPR_B200_ENOMEM : FPR_B200_ECUDA,
                std::string("fpr_b200_graph_generate: ") + cudaGetErrorString(e));
  }
  // generate_graph allocated g's arrays with cudaMallocAsync on h->stream.
  h->allocs.push_back(h->g.row);
  h->allocs.push_back(h->g.src);
  h->allocs.push_back(h->g.outdeg);
  if ((rc = finish_graph(h))) {
    destroy_handle(h);
    return rc;
  }
  *out = h;
  return FPR_B200_OK;
}

// fpr::build_csr(EdgeSet) (graph.hpp:35-70) on the device: the endpoints are
// narrowed to int32 with a range check while they upload (host threads through
// the pinned ring, or DMA + device narrowing for pinned input), then the K4
// build (sort by (dst, src), dedup, drop self-loops, degree scans).
int fpr_b200_graph_from_edges(uint64_t n, uint64_t m, const uint64_t* src, const uint64_t* dst,
                              const fpr_b200_options* opts, fpr_b200_graph** out) {
  if (!out) return fail(FPR_B200_EINVAL, "fpr_b200_graph_from_edges: null argument");
  *out = nullptr;
  if (m && (!src || !dst)) return fail(FPR_B200_EINVAL, "fpr_b200_graph_from_edges: null edge arrays");
  if (n >= (1ull << 31)) return fail(FPR_B200_ERANGE, "fpr_b200: n >= 2^31 exceeds the int32 vertex-id range");
  if (m >= (1ull << 40)) return fail(FPR_B200_ERANGE, "fpr_b200: too many edges");
  fpr_b200_graph* h = nullptr;
  int rc = open_handle(opts, &h);
  if (rc) {
    destroy_handle(h);
    return rc;
  }
  // temporaries (freed once the CSR is built)
  int32_t* ds = nullptr;
  int32_t* dd = nullptr;
  unsigned int* bad = nullptr;
  auto bail = [&](int code) {
    for (void* p : {(void*)ds, (void*)dd, (void*)bad})
      if (p) cudaFreeAsync(p, h->stream);
    destroy_handle(h);
    return code;
  };
  cudaError_t e = cudaMallocAsync((void**)&ds, (m + 1) * sizeof(int32_t), h->stream);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&dd, (m + 1) * sizeof(int32_t), h->stream);
  if (e == cudaSuccess) e = cudaMallocAsync((void**)&bad, sizeof(unsigned), h->stream);
  if (e != cudaSuccess) return bail(fail(FPR_B200_ENOMEM, "fpr_b200_graph_from_edges: device allocation failed"));
  e = cudaMemsetAsync(bad, 0, sizeof(unsigned), h->stream);
  bool ok = true;
  if (e == cudaSuccess && m > 0) {
    if (is_pinned(src) && is_pinned(dst)) {
      const std::vector<IdUpload> arrays = {{src, ds, (int64_t)m, true}, {dst, dd, (int64_t)m, true}};
      if ((rc = upload_ids_pinned(h, arrays, n, bad, nullptr, nullptr, 0, &e))) return bail(rc);
    } else {
      UploadRing* ring = get_ring(h->device);
      if (!ring) return bail(fail(FPR_B200_ENOMEM, "fpr_b200: pinned upload ring allocation failed"));
      std::lock_guard<std::mutex> lk(ring->mu);
      int k = 0;
      ok = ring_upload<int32_t>(ring, src, ds, (int64_t)m, n, h->stream, k, &e);
      ok = ring_upload<int32_t>(ring, dst, dd, (int64_t)m, n, h->stream, k, &e) && ok;
    }
  }
  unsigned hbad = 0;
  if (e == cudaSuccess) e = cudaMemcpyAsync(h->h_iters, bad, sizeof(unsigned), cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess)
    return bail(fail(FPR_B200_ECUDA, std::string("fpr_b200_graph_from_edges: ") + cudaGetErrorString(e)));
  hbad = *h->h_iters;
  if (!ok || hbad) {
    // The device saw an endpoint outside [0, n); name the first one the way
    // build_csr does (graph.hpp:39-43).  Error path only.
    for (uint64_t i = 0; i < m; ++i)
      if (src[i] >= n || dst[i] >= n)
        return bail(fail(FPR_B200_EINVAL, "build_csr: edge #" + std::to_string(i) + " (" + std::to_string(src[i]) +
                                              "," + std::to_string(dst[i]) + ") has endpoint outside [0," +
                                              std::to_string(n) + ")"));
  }
  const char* msg = nullptr;
  e = build_csr_from_arrays(ds, dd, (int64_t)m, n, h->g, h->stream, &msg);
  for (void* p : {(void*)ds, (void*)dd, (void*)bad})
    if (p) cudaFreeAsync(p, h->stream);
  ds = dd = nullptr;
  bad = nullptr;
  if (e != cudaSuccess || msg) {
    if (msg) return bail(fail(FPR_B200_ENOMEM, std::string("fpr_b200_graph_from_edges: ") + msg));
    return bail(fail(e == cudaErrorMemoryAllocation ? FPR_B200_ENOMEM : FPR_B200_ECUDA,
                     std::string("fpr_b200_graph_from_edges: ") + cudaGetErrorString(e)));
  }
  h->allocs.push_back(h->g.row);
  h->allocs.push_back(h->g.src);
  h->allocs.push_back(h->g.outdeg);
  if ((rc = finish_graph(h))) return bail(rc);
  *out = h;
  return FPR_B200_OK;
}

void fpr_b200_graph_destroy(fpr_b200_graph* h) { destroy_handle(h); }

int fpr_b200_graph_set_wave_count(fpr_b200_graph* h, uint32_t wave_count) {
  if (!h) return fail(FPR_B200_EINVAL, "fpr_b200_graph_set_wave_count: null graph");
  h->wave_count = wave_count;  // schedules are cached per wave count (get_waves)
  return FPR_B200_OK;
}

int fpr_b200_graph_layout_info(const fpr_b200_graph* h, int* sweep, uint64_t* runs, uint64_t* pieces,
                               uint64_t* tiles) {
  if (!h) return fail(FPR_B200_EINVAL, "fpr_b200_graph_layout_info: null graph");
  if (sweep) *sweep = h->use_pb ? FPR_B200_SWEEP_PB : FPR_B200_SWEEP_PULL;
  if (runs) *runs = h->pb ? (uint64_t)h->pb->nps : 0;
  if (pieces) *pieces = h->pb ? (uint64_t)h->pb->npieces : 0;
  if (tiles) *tiles = h->pb ? (uint64_t)h->pb->ntiles : 0;
  return FPR_B200_OK;
}

int fpr_b200_graph_info(const fpr_b200_graph* h, uint64_t* n, uint64_t* m, uint64_t* ntasks) {
  if (!h) return fail(FPR_B200_EINVAL, "fpr_b200_graph_info: null graph");
  if (n) *n = (uint64_t)h->g.n;
  if (m) *m = (uint64_t)h->g.m;
  if (ntasks) *ntasks = (uint64_t)h->part.ntasks;
  return FPR_B200_OK;
}

int fpr_b200_graph_download_csr(const fpr_b200_graph* hc, uint64_t* in_start, uint64_t* in_src,
                                uint64_t* out_degree) {
  auto* h = const_cast<fpr_b200_graph*>(hc);
  if (!h) return fail(FPR_B200_EINVAL, "fpr_b200_graph_download_csr: null graph");
  if (h->new_of_old)
    return fail(FPR_B200_EINVAL, "fpr_b200_graph_download_csr: graph was created with "
                                 "FPR_B200_OPT_REORDER / _SOURCES / _BLOCKS (resident CSR uses internal ids)");
  CK(cudaSetDevice(h->device));
  const DevGraph& g = h->g;
  const int64_t chunk = 1 << 24;
  uint64_t* tmp = nullptr;
  CK(cudaMallocAsync(&tmp, 2 * chunk * sizeof(uint64_t), h->stream));
  cudaError_t e = cudaSuccess;
  if (in_start && g.n >= 0) {
    for (int64_t off = 0; e == cudaSuccess && off < (int64_t)g.n + 1; off += chunk) {
      const int64_t cnt = std::min<int64_t>(chunk, (int64_t)g.n + 1 - off);
      e = launch_widen(g.row + off, nullptr, tmp, nullptr, cnt, 0, h->stream);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(in_start + off, tmp, cnt * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                            h->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    }
  }
  auto ids = [&](const int32_t* d, uint64_t* hout, int64_t count) {
    for (int64_t off = 0; e == cudaSuccess && off < count; off += chunk) {
      const int64_t cnt = std::min<int64_t>(chunk, count - off);
      e = launch_widen(nullptr, d + off, nullptr, tmp + chunk, 0, cnt, h->stream);
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(hout + off, tmp + chunk, cnt * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                            h->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    }
  };
  if (in_src) ids(g.src, in_src, g.m);
  if (out_degree) ids(g.outdeg, out_degree, g.n);
  cudaFreeAsync(tmp, h->stream);
  cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess)
    return fail(FPR_B200_ECUDA, std::string("fpr_b200_graph_download_csr: ") + cudaGetErrorString(e));
  return FPR_B200_OK;
}

int fpr_b200_graph_validate(fpr_b200_graph* h, uint32_t* flags) {
  if (!h || !flags) return fail(FPR_B200_EINVAL, "fpr_b200_graph_validate: null argument");
  CK(cudaSetDevice(h->device));
  int32_t* recount = nullptr;
  unsigned int* bad = nullptr;
  CK(cudaMallocAsync(&recount, std::max<int64_t>(h->g.n, 1) * sizeof(int32_t), h->stream));
  CK(cudaMallocAsync(&bad, sizeof(unsigned int), h->stream));
  CK(cudaMemsetAsync(recount, 0, std::max<int64_t>(h->g.n, 1) * sizeof(int32_t), h->stream));
  CK(cudaMemsetAsync(bad, 0, sizeof(unsigned int), h->stream));
  if (h->g.n > 0) CK(launch_validate(h->g, recount, bad, h->stream));
  CK(cudaMemcpyAsync(h->h_iters, bad, sizeof(unsigned int), cudaMemcpyDeviceToHost, h->stream));
  cudaFreeAsync(recount, h->stream);
  cudaFreeAsync(bad, h->stream);
  CK(cudaStreamSynchronize(h->stream));
  *flags = *h->h_iters;
  return FPR_B200_OK;
}

int fpr_b200_graph_bfs_order(fpr_b200_graph* h, uint64_t root, uint64_t* new_id) {
  if (!h || !new_id) return fail(FPR_B200_EINVAL, "fpr_b200_graph_bfs_order: null argument");
  if (root >= (uint64_t)h->g.n) return fail(FPR_B200_EINVAL, "fpr_b200: bfs root outside [0,n)");
  CK(cudaSetDevice(h->device));
  std::vector<int32_t> tmp(h->g.n);
  const char* msg = nullptr;
  CK(relabel_order_bfs(h->g, (int32_t)root, tmp.data(), h->stream, &msg));
  if (msg) return fail(FPR_B200_ENOMEM, std::string("fpr_b200_graph_bfs_order: ") + msg);
  for (int32_t i = 0; i < h->g.n; ++i) new_id[i] = (uint64_t)tmp[i];
  return FPR_B200_OK;
}

int fpr_b200_graph_wave_starts(fpr_b200_graph* h, uint32_t wave_count, uint64_t* wave_start,
                               uint64_t cap, uint64_t* nwaves) {
  if (!h) return fail(FPR_B200_EINVAL, "fpr_b200_graph_wave_starts: null graph");
  if (h->g.n == 0) return fail(FPR_B200_EINVAL, "pagerank: graph has no vertices");
  CK(cudaSetDevice(h->device));
  std::vector<uint64_t> vs;
  if (h->use_pb) {
    // propagation-blocked lockstep: waves of consecutive bins (run_pb)
    int shift = 0, chunk_shift = 0;
    pb_geometry(&shift, &chunk_shift);
    if (shift < 5 || shift > 14) return fail(FPR_B200_EINVAL, "fpr_b200 propagation-blocked layout: bin/chunk geometry out of range");
    std::vector<int64_t> be;
    if (h->pb && h->pb->shift == shift) {
      be = h->pb->bin_edge;
    } else {
      CK(pb_bin_edges(h->g, shift, h->stream, &be));
    }
    for (int64_t b : pb_wave_bins(be, wave_count ? wave_count : lockstep_waves(h)))
      vs.push_back((uint64_t)std::min<int64_t>(h->g.n, b << shift));
  } else {
    const Waves* wv = nullptr;
    int rc = get_waves(h, wave_count ? wave_count : h->wave_count, &wv);
    if (rc) return rc;
    vs = wv->vertex_start;
  }
  if (nwaves) *nwaves = (uint64_t)vs.size() - 1;
  if (wave_start) {
    if (cap < vs.size()) return fail(FPR_B200_EINVAL, "fpr_b200_graph_wave_starts: buffer too small");
    std::copy(vs.begin(), vs.end(), wave_start);
  }
  return FPR_B200_OK;
}

const double* fpr_b200_graph_ranks_device(const fpr_b200_graph* h) { return h ? h->pr : nullptr; }

namespace {
// Propagation-blocked sweeps (FPR_B200_OPT_PB, pb.cu).  EC: one wave, the
// gather reads contrib[par] and the rows write contrib[par ^ 1].  Lockstep
// (the deterministic FusEd schedule): S waves of consecutive bins, gathered
// from and written to contrib[0] in place, so wave w reads this sweep's
// contributions of waves < w (fo_pagerank_lockstep).  The host checks the
// stop rule after each sweep.
constexpr int kPbDeclined = -1;  // the auto-selected layout did not fit; run the pull sweep

// The propagation-blocked layout of h, built at its first use.
int ensure_pb(fpr_b200_graph* h) {
  if (!h->pb) {
    int shift = 0, chunk_shift = 0;
    pb_geometry(&shift, &chunk_shift);
    auto* pb = new PbSet;
    const char* msg = nullptr;
    cudaError_t e = build_pb(h->g, source_space(h), shift, chunk_shift, h->stream, *pb, &msg);
    if (e != cudaSuccess || msg) {
      delete pb;
      if (!(h->flags & FPR_B200_OPT_PB) && (msg || e == cudaErrorMemoryAllocation)) {
        // auto-selected and it does not fit (or the geometry does not apply):
        // the pull sweep runs instead -- a device engine choice, not a fallback
        cudaGetLastError();
        h->use_pb = false;
        return kPbDeclined;
      }
      if (msg) return fail(FPR_B200_EINVAL, std::string("fpr_b200 propagation-blocked layout: ") + msg);
      return fail(e == cudaErrorMemoryAllocation ? FPR_B200_ENOMEM : FPR_B200_ECUDA,
                  std::string("fpr_b200 propagation-blocked layout: ") + cudaGetErrorString(e));
    }
    h->pb = pb;
  }
  return FPR_B200_OK;
}

int run_pb(fpr_b200_graph* h, bool lockstep, const fpr_config* cfg, double* ranks_out, double* errors_out,
           double* l1_out, uint64_t* iter_ns_out, uint64_t errors_cap, fpr_b200_result* result) {
  const DevGraph& g = h->g;
  float setup_ms = 0.f, solve_ms = 0.f;
  uint64_t launches = 0;
  CK(cudaEventRecord(h->ev[0], h->stream));
  {
    const int rc = ensure_pb(h);
    if (rc) return rc;  // kPbDeclined included
  }
  const PbPlan* plan = nullptr;
  {
    cudaError_t e = get_pb_plan(*h->pb, lockstep ? lockstep_waves(h) : pb_ec_waves(h), h->stream, &plan);
    if (e != cudaSuccess)
      return fail(e == cudaErrorMemoryAllocation ? FPR_B200_ENOMEM : FPR_B200_ECUDA,
                  std::string("fpr_b200 propagation-blocked plan: ") + cudaGetErrorString(e));
  }
  CK(launch_init(g, h->pr, h->contrib[0], h->stream));
  ++launches;
  CK(cudaEventRecord(h->ev[1], h->stream));
  const double base = (1.0 - cfg->damping) / (double)g.n;  // pagerank.hpp:81
  uint64_t total = 0;
  int par = 0;
  double last_err = 1.0, last_l1 = 1.0;
  while (total < cfg->max_iterations) {
    CK(cudaEventRecord(h->ev[1], h->stream));
    double* prev = h->contrib[lockstep ? 0 : par];
    double* next = h->contrib[lockstep ? 0 : par ^ 1];
    // rows without in-edges are settled once both contribution buffers hold
    // their constant (after two sweeps of this run; lockstep after one)
    CK(launch_pb_sweep(*h->pb, *plan, g, prev, h->pr, h->pr, next, PbPeers{}, base, cfg->damping, h->d_errors,
                       h->d_l1, h->stream, nullptr, total >= 2));
    launches += (uint64_t)plan->nwaves + (uint64_t)(plan->item0.back() > 0 ? plan->nwaves : 0) + 1;
    CK(cudaEventRecord(h->ev[2], h->stream));
    CK(cudaMemcpyAsync(h->h_errors, h->d_errors, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaMemcpyAsync(h->h_l1, h->d_l1, sizeof(double), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (total == 0) cudaEventElapsedTime(&setup_ms, h->ev[0], h->ev[1]);
    float it_ms = 0.f;
    cudaEventElapsedTime(&it_ms, h->ev[1], h->ev[2]);
    solve_ms += it_ms;
    if (errors_out && errors_cap < total + 1)
      return fail(FPR_B200_EINVAL, "fpr_b200_run: errors buffer holds " + std::to_string(errors_cap) +
                                       " entries, need " + std::to_string(total + 1));
    last_err = h->h_errors[0];
    last_l1 = h->h_l1[0];
    if (errors_out) errors_out[total] = last_err;
    if (l1_out) l1_out[total] = last_l1;
    if (iter_ns_out) iter_ns_out[total] = (uint64_t)(it_ms * 1e6);
    ++total;
    par ^= 1;
    if ((h->norm == FPR_B200_NORM_L1 ? last_l1 : last_err) <= cfg->threshold) break;
  }
  if (ranks_out) {
    const double* src = h->pr;
    if (h->new_of_old) {
      CK(launch_gather_ranks(h->pr, h->new_of_old, g.n, h->ranks_tmp, h->stream));
      src = h->ranks_tmp;
    }
    CK(cudaMemcpyAsync(ranks_out, src, g.n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  }
  CK(cudaStreamSynchronize(h->stream));
  if (result) {
    result->iterations = total;
    const double crit = h->norm == FPR_B200_NORM_L1 ? last_l1 : last_err;
    result->converged = (total > 0 && crit <= cfg->threshold) ? 1 : 0;
    result->final_error = total > 0 ? last_err : 1.0;
    result->setup_ms = setup_ms;
    result->solve_ms = solve_ms;
    result->kernel_launches = launches;
    result->sweep = FPR_B200_SWEEP_PB;
  }
  return FPR_B200_OK;
}
}  // namespace

int fpr_b200_run(fpr_b200_graph* h, int engine, const fpr_config* cfg, double* ranks_out,
                 double* errors_out, double* l1_out, uint64_t* iter_ns_out, uint64_t errors_cap,
                 fpr_b200_result* result) {
  if (!h || !cfg) return fail(FPR_B200_EINVAL, "fpr_b200_run: null argument");
  int rc = validate_config(cfg);
  if (rc) return rc;
  if (h->g.n == 0) return fail(FPR_B200_EINVAL, "pagerank: graph has no vertices");
  if (engine != kEC && engine != kFused && engine != kLockstep)
    return fail(FPR_B200_EINVAL, "fpr_b200: unknown engine " + std::to_string(engine));
  CK(cudaSetDevice(h->device));
  // Propagation-blocked graphs: EC runs PB Jacobi sweeps; lockstep and FUSED
  // run the lockstep Gauss-Seidel schedule on PB sweeps (the fastest FusEd
  // schedule there, within the fused_par contract).
  if (h->use_pb) {
    rc = run_pb(h, engine != kEC, cfg, ranks_out, errors_out, l1_out, iter_ns_out, errors_cap, result);
    if (rc != kPbDeclined) return rc;
  }

  // Jacobi = one wave; lockstep = the cached wave schedule; async = all tasks.
  const Waves* wv = nullptr;
  if ((rc = get_waves(h, engine == kLockstep ? h->wave_count : 1u, &wv))) return rc;
  if (engine != kLockstep && wv->nwaves != 1) {
    return fail(FPR_B200_ECUDA, "fpr_b200: internal error (EC wave schedule)");
  }
  const int variant = engine == kFused ? 1 : 0;
  const int shape = engine == kFused ? h->async_shape : engine;
  const int wpb = solve_block_threads(shape) / 32;
  const int64_t want = (h->part.ntasks + wpb - 1) / wpb;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(h->grid_full[variant], want));


  const DevGraph& g = h->g;
  uint64_t launches = 0;
  CK(cudaEventRecord(h->ev[0], h->stream));
  CK(launch_init(g, h->pr, h->contrib[0], h->stream));
  ++launches;
  CK(cudaEventRecord(h->ev[1], h->stream));
  float setup_ms = 0.f, solve_ms = 0.f;
  bool setup_timed = false;

  SolveParams p{};
  p.n = g.n;
  p.row = g.row;
  p.src = g.src;
  p.outdeg = g.outdeg;
  p.task_row = h->part.task_row;
  p.task_edge = h->part.task_edge;
  p.head_first = h->part.head_first;
  p.task_bits = h->part.task_bits;
  p.ntasks = h->part.ntasks;
  p.wave_task = wv->d_task;
  p.wave_row = wv->d_row;
  p.nwaves = wv->nwaves;
  p.nsrc = g.n;
  p.pr = h->pr;
  p.pr_out = h->pr;
  p.contrib0 = h->contrib[0];
  p.contrib1 = h->contrib[1];
  p.tail_partial = h->tail_partial;
  p.damping = cfg->damping;
  p.base = (1.0 - cfg->damping) / (double)g.n;  // pagerank.hpp:81
  p.write_off = 0;
  p.threshold = cfg->threshold;
  p.norm = h->norm;
  p.errors = h->d_errors;
  p.l1errors = h->d_l1;
  p.iter_ns = h->d_ns;
  p.partials = h->partials;
  p.totals = h->totals;
  p.bar = h->bar;
  p.out_iters = &h->d_status->iters;
  p.out_stop = &h->d_status->stop;
  p.out_last = h->d_status->last;

  uint64_t total = 0;
  int parity = 0;
  int stop = 0;
  double last_err = 1.0, last_l1 = 1.0;
  while (total < cfg->max_iterations) {
    const uint64_t chunk = std::min<uint64_t>(cfg->max_iterations - total, kChunkIters);
    p.max_iters = (uint32_t)chunk;
    p.parity0 = parity;
    CK(cudaEventRecord(h->ev[1], h->stream));
    CK(launch_solve(shape, grid, p, h->stream));
    CK(cudaEventRecord(h->ev[2], h->stream));
    ++launches;
    CK(cudaMemcpyAsync(h->hs->status, h->d_status, sizeof(SolveStatus), cudaMemcpyDeviceToHost, h->stream));
    CK(cudaStreamSynchronize(h->stream));
    if (!setup_timed) {
      cudaEventElapsedTime(&setup_ms, h->ev[0], h->ev[1]);
      setup_timed = true;
    }
    float chunk_ms = 0.f;
    cudaEventElapsedTime(&chunk_ms, h->ev[1], h->ev[2]);
    solve_ms += chunk_ms;
    const uint64_t done = h->hs->status->iters;
    stop = h->hs->status->stop;
    if (done == 0 || done > chunk) return fail(FPR_B200_ECUDA, "fpr_b200: solver reported bad count");
    if (errors_out && errors_cap < total + done)
      return fail(FPR_B200_EINVAL, "fpr_b200_run: errors buffer holds " +
                                       std::to_string(errors_cap) + " entries, need " +
                                       std::to_string(total + done));
    if (errors_out || l1_out || iter_ns_out) {  // the trace: a second copy only when asked for
      if (errors_out)
        CK(cudaMemcpyAsync(h->h_errors, h->d_errors, done * sizeof(double), cudaMemcpyDeviceToHost,
                           h->stream));
      if (l1_out)
        CK(cudaMemcpyAsync(h->h_l1, h->d_l1, done * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
      if (iter_ns_out)
        CK(cudaMemcpyAsync(h->h_ns, h->d_ns, (done + 1) * sizeof(unsigned long long),
                           cudaMemcpyDeviceToHost, h->stream));
      CK(cudaStreamSynchronize(h->stream));
      if (errors_out) std::memcpy(errors_out + total, h->h_errors, done * sizeof(double));
      if (l1_out) std::memcpy(l1_out + total, h->h_l1, done * sizeof(double));
      if (iter_ns_out)
        for (uint64_t k = 0; k < done; ++k) iter_ns_out[total + k] = h->h_ns[k + 1] - h->h_ns[k];
    }
    last_err = h->hs->status->last[0];
    last_l1 = h->hs->status->last[1];
    total += done;
    parity ^= (int)(done & 1);
    if (stop) break;
  }
  if (ranks_out) {
    const double* src = h->pr;
    if (h->new_of_old) {  // back to the caller's vertex ids
      CK(launch_gather_ranks(h->pr, h->new_of_old, g.n, h->ranks_tmp, h->stream));
      src = h->ranks_tmp;
    }
    CK(cudaMemcpyAsync(ranks_out, src, g.n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  }
  CK(cudaStreamSynchronize(h->stream));
  if (result) {
    result->iterations = total;
    const double crit = h->norm == FPR_B200_NORM_L1 ? last_l1 : last_err;
    result->converged = (total > 0 && crit <= cfg->threshold) ? 1 : 0;
    result->final_error = total > 0 ? last_err : 1.0;
    result->setup_ms = setup_ms;
    result->solve_ms = solve_ms;
    result->kernel_launches = launches;
    result->sweep = FPR_B200_SWEEP_PULL;
  }
  return FPR_B200_OK;
}

// ------------------------------------------------------------ multi-GPU parts
int fpr_b200_graph_partition(const fpr_b200_graph* fullc, uint32_t nparts, uint32_t part,
                             const fpr_b200_options* opts, uint64_t* bounds_out,
                             uint64_t* slice_out, fpr_b200_graph** out) {
  auto* full = const_cast<fpr_b200_graph*>(fullc);
  if (!full || !out) return fail(FPR_B200_EINVAL, "fpr_b200_graph_partition: null argument");
  *out = nullptr;
  if (nparts == 0 || nparts > 64 || part >= nparts)
    return fail(FPR_B200_EINVAL, "fpr_b200_graph_partition: need 1 <= nparts <= 64, part < nparts");
  if (full->nparts != 1) return fail(FPR_B200_EINVAL, "fpr_b200_graph_partition: already a part");
  if (full->g.n == 0) return fail(FPR_B200_EINVAL, "pagerank: graph has no vertices");
  CK(cudaSetDevice(full->device));
  int64_t* d_bounds = nullptr;
  CK(cudaMallocAsync(&d_bounds, (nparts + 1) * sizeof(int64_t), full->stream));
  CK(launch_part_bounds(full->g, nparts, d_bounds, full->stream));
  std::vector<int64_t> b(nparts + 1);
  CK(cudaMemcpyAsync(b.data(), d_bounds, (nparts + 1) * sizeof(int64_t), cudaMemcpyDeviceToHost,
                     full->stream));
  CK(cudaStreamSynchronize(full->stream));
  int64_t slice = 0;
  for (uint32_t r = 0; r < nparts; ++r) slice = std::max<int64_t>(slice, b[r + 1] - b[r]);
  if ((int64_t)nparts * slice >= INT32_MAX) {
    cudaFreeAsync(d_bounds, full->stream);
    return fail(FPR_B200_ERANGE, "fpr_b200: padded exchange space exceeds int32 ids");
  }
  int64_t rows[2];
  CK(cudaMemcpyAsync(&rows[0], full->g.row + b[part], sizeof(int64_t), cudaMemcpyDeviceToHost, full->stream));
  CK(cudaMemcpyAsync(&rows[1], full->g.row + b[part + 1], sizeof(int64_t), cudaMemcpyDeviceToHost, full->stream));
  CK(cudaStreamSynchronize(full->stream));
  fpr_b200_graph* h = nullptr;
  fpr_b200_options o;
  fpr_b200_options_init(&o);
  if (opts) o = *opts;
  o.device = full->device;
  int rc = open_handle(&o, &h);
  auto bail = [&](int code) {
    cudaFreeAsync(d_bounds, full->stream);
    destroy_handle(h);
    return code;
  };
  if (rc) return bail(rc);
  const int64_t nloc = b[part + 1] - b[part], mloc = rows[1] - rows[0];
  h->g.n = (int32_t)nloc;
  h->g.m = mloc;
  if ((rc = dalloc_n(h, &h->g.row, nloc + 1)) || (rc = dalloc_n(h, &h->g.src, mloc + 8)) ||
      (rc = dalloc_n(h, &h->g.outdeg, std::max<int64_t>(nloc, 1))))
    return bail(rc);
  // the full graph's stream finished the bounds; order the extract after it
  CK(cudaStreamSynchronize(full->stream));
  cudaError_t e = launch_part_extract(full->g, d_bounds, nparts, part, slice, nloc, mloc, h->g, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess)
    return bail(fail(FPR_B200_ECUDA, std::string("fpr_b200_graph_partition: ") + cudaGetErrorString(e)));
  cudaFreeAsync(d_bounds, full->stream);
  d_bounds = nullptr;
  h->nparts = nparts;
  h->part_id = part;
  h->n_global = (uint64_t)full->g.n;
  h->row_begin = (uint64_t)b[part];
  h->slice = (uint64_t)slice;
  if ((rc = finish_graph(h))) {
    destroy_handle(h);
    return rc;
  }
  if (bounds_out)
    for (uint32_t r = 0; r <= nparts; ++r) bounds_out[r] = (uint64_t)b[r];
  if (slice_out) *slice_out = (uint64_t)slice;
  *out = h;
  return FPR_B200_OK;
}

// Host restatement of part_bounds_kernel / merge_path (same integer steps), so
// every rank derives the same bounds from its own copy of in_start.
namespace {
std::vector<int64_t> host_part_bounds(const uint64_t* in_start, int64_t n, int64_t m, uint32_t nparts) {
  std::vector<int64_t> b(nparts + 1);
  const int64_t total = n + m;
  for (uint32_t r = 0; r <= nparts; ++r) {
    if (r == nparts) {
      b[r] = n;
      continue;
    }
    const int64_t diag = (int64_t)((__int128)total * r / nparts);
    int64_t lo = diag - m > 0 ? diag - m : 0;
    int64_t hi = diag < n ? diag : n;
    while (lo < hi) {
      const int64_t pivot = (lo + hi) >> 1;
      if ((int64_t)in_start[pivot + 1] <= diag - pivot - 1)
        lo = pivot + 1;
      else
        hi = pivot;
    }
    b[r] = lo;
  }
  return b;
}
}  // namespace

int fpr_b200_part_create(const fpr_graph_view* v, uint32_t nparts, uint32_t part, const fpr_b200_options* opts,
                         uint64_t* bounds_out, uint64_t* slice_out, fpr_b200_graph** out) {
  if (!v || !out) return fail(FPR_B200_EINVAL, "fpr_b200_part_create: null argument");
  *out = nullptr;
  if (nparts == 0 || nparts > 64 || part >= nparts)
    return fail(FPR_B200_EINVAL, "fpr_b200_part_create: need 1 <= nparts <= 64, part < nparts");
  if (v->n == 0) return fail(FPR_B200_EINVAL, "pagerank: graph has no vertices");
  if (v->n >= (1ULL << 31))
    return fail(FPR_B200_ERANGE, "fpr_b200: n = " + std::to_string(v->n) +
                                     " exceeds the int32 vertex-id range (n < 2^31)");
  if (!v->in_start || !v->out_degree || (v->m > 0 && !v->in_src))
    return fail(FPR_B200_EINVAL, "fpr_b200_part_create: null array");
  if (v->in_start[0] != 0 || v->in_start[v->n] != v->m)
    return fail(FPR_B200_EINVAL, "fpr_b200: in_start is not a valid CSR offset array "
                                 "(in_start[0]==0, non-decreasing, in_start[n]==m)");
  const std::vector<int64_t> b = host_part_bounds(v->in_start, (int64_t)v->n, (int64_t)v->m, nparts);
  int64_t slice = 0;
  for (uint32_t r = 0; r < nparts; ++r) slice = std::max<int64_t>(slice, b[r + 1] - b[r]);
  if ((int64_t)nparts * slice >= INT32_MAX)
    return fail(FPR_B200_ERANGE, "fpr_b200: padded exchange space exceeds int32 ids");
  const int64_t b0 = b[part], b1 = b[part + 1];
  const int64_t e0 = (int64_t)v->in_start[b0], e1 = (int64_t)v->in_start[b1];
  if (e1 < e0) return fail(FPR_B200_EINVAL, "fpr_b200: in_start is not a valid CSR offset array "
                                            "(in_start[0]==0, non-decreasing, in_start[n]==m)");
  fpr_b200_graph* h = nullptr;
  int rc = open_handle(opts, &h);
  if (rc) {
    destroy_handle(h);
    return rc;
  }
  auto bail = [&](int code) {
    destroy_handle(h);
    return code;
  };
  DevGraph& g = h->g;
  g.n = (int32_t)(b1 - b0);
  g.m = e1 - e0;
  unsigned int* bad = nullptr;
  int64_t* d_bounds = nullptr;
  if ((rc = dalloc_n(h, &g.row, (int64_t)g.n + 1)) || (rc = dalloc_n(h, &g.src, g.m + 8)) ||
      (rc = dalloc_n(h, &g.outdeg, std::max<int64_t>(g.n, 1))) || (rc = dalloc_n(h, &bad, 1)) ||
      (rc = dalloc_n(h, &d_bounds, nparts + 1)))
    return bail(rc);
  cudaError_t e = cudaMemsetAsync(bad, 0, sizeof(unsigned), h->stream);
  if (e == cudaSuccess)
    e = cudaMemcpyAsync(d_bounds, b.data(), (nparts + 1) * sizeof(int64_t), cudaMemcpyHostToDevice, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);  // b is a host vector
  // Only this part's rows cross the link: in_start[b0..b1], in_src[e0..e1),
  // out_degree[b0..b1) -- ids range-checked against the global n.
  const bool pinned = is_pinned(v->in_start) && (g.m == 0 || is_pinned(v->in_src)) && is_pinned(v->out_degree);
  if (e == cudaSuccess && pinned) {
    const std::vector<IdUpload> arrays = {{v->in_src + e0, g.src, g.m, true}, {v->out_degree + b0, g.outdeg, g.n, false}};
    if ((rc = upload_ids_pinned(h, arrays, v->n, bad, v->in_start + b0, g.row, ((size_t)g.n + 1) * sizeof(int64_t),
                                &e)))
      return bail(rc);
  } else if (e == cudaSuccess) {
    UploadRing* ring = get_ring(h->device);
    if (!ring) return bail(fail(FPR_B200_ENOMEM, "fpr_b200: pinned upload ring allocation failed"));
    std::lock_guard<std::mutex> lk(ring->mu);
    int k = 0;
    bool ok = ring_upload<int64_t>(ring, v->in_start + b0, g.row, (int64_t)g.n + 1, 0, h->stream, k, &e);
    ok = ring_upload<int32_t>(ring, v->in_src + e0, g.src, g.m, v->n, h->stream, k, &e) && ok;
    ok = ring_upload<int32_t>(ring, v->out_degree + b0, g.outdeg, g.n, v->n, h->stream, k, &e) && ok;
    if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
    if (e == cudaSuccess && !ok) e = cudaMemsetAsync(bad, 1, 1, h->stream);
  }
  if (e == cudaSuccess) e = launch_offset_shift(g.row, (int64_t)g.n + 1, e0, h->stream);
  if (e == cudaSuccess && g.n > 0) e = launch_check_offsets(g.row, g.n, g.m, bad, h->stream);
  if (e == cudaSuccess) e = launch_part_remap(g.src, g.m, d_bounds, nparts, slice, h->stream);
  if (e == cudaSuccess) e = cudaMemcpyAsync(h->h_iters, bad, sizeof(unsigned), cudaMemcpyDeviceToHost, h->stream);
  if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
  if (e != cudaSuccess)
    return bail(fail(FPR_B200_ECUDA, std::string("fpr_b200_part_create: ") + cudaGetErrorString(e)));
  if (*h->h_iters & 1u)
    return bail(fail(FPR_B200_EINVAL, "fpr_b200: in_src/out_degree value outside [0," + std::to_string(v->n) + ")"));
  if (*h->h_iters & 6u)
    return bail(fail(FPR_B200_EINVAL, "fpr_b200: in_start is not a valid CSR offset array "
                                      "(in_start[0]==0, non-decreasing, in_start[n]==m)"));
  h->nparts = nparts;
  h->part_id = part;
  h->n_global = v->n;
  h->row_begin = (uint64_t)b0;
  h->slice = (uint64_t)slice;
  if ((rc = finish_graph(h))) return bail(rc);
  if (bounds_out)
    for (uint32_t r = 0; r <= nparts; ++r) bounds_out[r] = (uint64_t)b[r];
  if (slice_out) *slice_out = (uint64_t)slice;
  *out = h;
  return FPR_B200_OK;
}

int fpr_b200_part_init(fpr_b200_graph* h, double* exchange) {
  if (!h || !exchange) return fail(FPR_B200_EINVAL, "fpr_b200_part_init: null argument");
  CK(cudaSetDevice(h->device));
  const uint64_t ng = h->nparts > 1 ? h->n_global : (uint64_t)h->g.n;
  int rc = 0;
  if (!h->part_pr[1] && (rc = dalloc_n(h, &h->part_pr[1], std::max<int64_t>(h->g.n, 1)))) return rc;
  h->part_pr[0] = h->pr;
  h->part_pr_cur = 0;
  CK(launch_part_init(h->g, 1.0 / (double)ng, h->pr, exchange + (uint64_t)h->part_id * h->slice,
                      h->stream));
  h->part_sweeps = 0;
  return FPR_B200_OK;
}

int fpr_b200_part_sweep(fpr_b200_graph* h, int engine, const fpr_config* cfg,
                        const double* exch_read, double* exch_write, double* pair_out) {
  return fpr_b200_part_sweep_peers(h, engine, cfg, exch_read, exch_write, nullptr, 0, pair_out);
}

int fpr_b200_part_sweep_peers(fpr_b200_graph* h, int engine, const fpr_config* cfg,
                              const double* exch_read, double* exch_write,
                              double* const* peer_write, uint32_t npeer_bufs, double* pair_out) {
  if (!h || !cfg || !exch_read || !exch_write || !pair_out)
    return fail(FPR_B200_EINVAL, "fpr_b200_part_sweep: null argument");
  if (!h->part_pr[0]) return fail(FPR_B200_EINVAL, "fpr_b200_part_sweep: call fpr_b200_part_init first");
  if (npeer_bufs && (!peer_write || npeer_bufs != (uint32_t)h->nparts))
    return fail(FPR_B200_EINVAL, "fpr_b200_part_sweep_peers: need one exchange pointer per part");
  if (npeer_bufs && h->nparts - 1 > kMaxPeers)
    return fail(FPR_B200_EINVAL, "fpr_b200_part_sweep_peers: at most " + std::to_string(kMaxPeers + 1) +
                                     " parts");
  int rc = validate_config(cfg);
  if (rc) return rc;
  if (engine != kEC && engine != kFused)
    return fail(FPR_B200_EINVAL, "fpr_b200_part_sweep: engine must be EC or FUSED");
  if (engine == kFused && exch_read != exch_write)
    return fail(FPR_B200_EINVAL, "fpr_b200_part_sweep: FUSED updates the exchange vector in place");
  CK(cudaSetDevice(h->device));
  const uint64_t ng = h->nparts > 1 ? h->n_global : (uint64_t)h->g.n;
  if (h->use_pb) {
    // propagation-blocked part sweep: bins over the part's rows, chunks over
    // the exchange space; the accumulate's finalize stores each contribution
    // into the part's slice and into every peer's replica.  EC: one wave;
    // FUSED: the lockstep waves, in place.
    rc = ensure_pb(h);
    if (rc && rc != kPbDeclined) return rc;
    if (!rc) {
      const PbPlan* plan = nullptr;
      const cudaError_t e = get_pb_plan(*h->pb, engine == kFused ? lockstep_waves(h) : pb_ec_waves(h), h->stream, &plan);
      if (e != cudaSuccess)
        return fail(e == cudaErrorMemoryAllocation ? FPR_B200_ENOMEM : FPR_B200_ECUDA,
                    std::string("fpr_b200 propagation-blocked plan: ") + cudaGetErrorString(e));
      const int64_t off = (int64_t)h->part_id * (int64_t)h->slice;
      PbPeers peers;
      for (uint32_t q = 0; q < npeer_bufs; ++q) {
        if (q == h->part_id) continue;
        if (!peer_write[q]) return fail(FPR_B200_EINVAL, "fpr_b200_part_sweep_peers: null peer pointer");
        peers.p[peers.n++] = peer_write[q] + off;
      }
      ++h->part_sweeps;
      CK(launch_pb_sweep(*h->pb, *plan, h->g, exch_read, h->part_pr[h->part_pr_cur], h->part_pr[h->part_pr_cur ^ 1],
                         exch_write + off, peers, (1.0 - cfg->damping) / (double)ng, cfg->damping, h->d_errors,
                         h->d_l1, h->stream, h->gate, h->part_sweeps > 3));  // rows without in-edges: as the peer rule
      h->part_pr_cur ^= 1;
      CK(cudaMemcpyAsync(pair_out, h->d_errors, sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
      CK(cudaMemcpyAsync(pair_out + 1, h->d_l1, sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
      return FPR_B200_OK;
    }
  }
  const Waves* wv = nullptr;
  if ((rc = get_waves(h, 1u, &wv))) return rc;
  const int variant = engine == kFused ? 1 : 0;
  const int shape = engine == kFused ? h->async_shape : engine;
  const int wpb = solve_block_threads(shape) / 32;
  const int64_t want = (h->part.ntasks + wpb - 1) / wpb;
  const int grid = (int)std::max<int64_t>(1, std::min<int64_t>(h->grid_full[variant], want));
  SolveParams p{};
  p.n = h->g.n;
  p.row = h->g.row;
  p.src = h->g.src;
  p.outdeg = h->g.outdeg;
  p.task_row = h->part.task_row;
  p.task_edge = h->part.task_edge;
  p.head_first = h->part.head_first;
  p.task_bits = h->part.task_bits;
  p.ntasks = h->part.ntasks;
  p.wave_task = wv->d_task;
  p.wave_row = wv->d_row;
  p.nwaves = wv->nwaves;
  // ranks ping-pong between two buffers, so the state before the latest
  // sweep stays readable (fpr_b200_part_ranks_prev: speculative drivers)
  p.nsrc = (int64_t)h->nparts * (int64_t)(h->nparts > 1 ? h->slice : (uint64_t)h->g.n);
  p.pr = h->part_pr[h->part_pr_cur];
  p.pr_out = h->part_pr[h->part_pr_cur ^ 1];
  p.contrib0 = const_cast<double*>(exch_read);
  p.contrib1 = exch_write;
  p.parity0 = 0;
  p.write_off = (int64_t)h->part_id * (int64_t)h->slice;
  p.tail_partial = h->tail_partial;
  p.damping = cfg->damping;
  p.base = (1.0 - cfg->damping) / (double)ng;
  p.threshold = 0.0;  // one sweep; the caller decides after the all-reduce
  p.norm = h->norm;
  p.max_iters = 1;
  p.errors = h->d_errors;
  p.l1errors = h->d_l1;
  p.iter_ns = h->d_ns;
  p.partials = h->partials;
  p.totals = h->totals;
  p.bar = h->bar;
  p.out_iters = &h->d_status->iters;
  p.out_stop = &h->d_status->stop;
  p.out_last = h->d_status->last;
  p.npeers = 0;
  // Rows without in-edges have a constant contribution after the first sweep;
  // once every rotating exchange vector holds it (3 sweeps after part_init:
  // drivers rotate through 2, or 3 when speculating) peers are not sent it
  // again (SURVEY §8(e) exchange compaction).
  p.peer_skip_empty = h->part_sweeps >= 3 ? 1 : 0;
  p.gate = h->gate;
  ++h->part_sweeps;
  for (uint32_t q = 0; q < npeer_bufs; ++q) {
    if (q == (uint32_t)h->part_id) continue;
    if (!peer_write[q]) return fail(FPR_B200_EINVAL, "fpr_b200_part_sweep_peers: null peer pointer");
    p.peer[p.npeers++] = peer_write[q] + p.write_off;  // this part's slice in part q's replica
  }
  CK(launch_solve(shape, grid, p, h->stream));
  h->part_pr_cur ^= 1;
  CK(cudaMemcpyAsync(pair_out, h->d_errors, sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  CK(cudaMemcpyAsync(pair_out + 1, h->d_l1, sizeof(double), cudaMemcpyDeviceToDevice, h->stream));
  return FPR_B200_OK;
}

// ---- device-side stop rule (include/fpr_b200.h fpr_b200_gate_*) ----
uint64_t fpr_b200_gate_bytes(uint64_t trace_cap) { return sizeof(GateHdr) + 2 * trace_cap * sizeof(double); }

int fpr_b200_gate_init(void* gate, uint64_t trace_cap, int device, void* stream) {
  if (!gate) return fail(FPR_B200_EINVAL, "fpr_b200_gate_init: null gate");
  CK(cudaSetDevice(device));
  CK(launch_gate_init(static_cast<GateHdr*>(gate), trace_cap, static_cast<cudaStream_t>(stream)));
  return FPR_B200_OK;
}

int fpr_b200_gate_update(void* gate, const double* const* pairs, uint32_t npairs, const fpr_config* cfg, int norm,
                         int device, void* stream) {
  if (!gate || !pairs || !cfg) return fail(FPR_B200_EINVAL, "fpr_b200_gate_update: null argument");
  if (npairs < 1 || npairs > (uint32_t)kMaxPeers + 1)
    return fail(FPR_B200_EINVAL, "fpr_b200_gate_update: 1 to " + std::to_string(kMaxPeers + 1) + " residual pairs");
  int rc = validate_config(cfg);
  if (rc) return rc;
  PairPtrs pp;
  pp.n = (int)npairs;
  for (uint32_t r = 0; r < npairs; ++r) {
    if (!pairs[r]) return fail(FPR_B200_EINVAL, "fpr_b200_gate_update: null pair pointer");
    pp.p[r] = pairs[r];
  }
  CK(cudaSetDevice(device));
  CK(launch_gate_update(static_cast<GateHdr*>(gate), pp, cfg->threshold, norm, cfg->max_iterations,
                        static_cast<cudaStream_t>(stream)));
  return FPR_B200_OK;
}

int fpr_b200_gate_read(const void* gate, int device, void* stream, uint64_t* iterations, int* stopped,
                       double* errors_out, double* l1_out, uint64_t cap) {
  if (!gate) return fail(FPR_B200_EINVAL, "fpr_b200_gate_read: null gate");
  CK(cudaSetDevice(device));
  const cudaStream_t st = static_cast<cudaStream_t>(stream);
  GateHdr hdr{};
  CK(cudaMemcpyAsync(&hdr, gate, sizeof(hdr), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  if (iterations) *iterations = hdr.iters;
  if (stopped) *stopped = hdr.stop ? 1 : 0;
  const uint64_t k = std::min<uint64_t>(hdr.iters, std::min<uint64_t>(hdr.cap, cap));
  if ((errors_out || l1_out) && k > 0) {
    std::vector<double> tr(2 * k);
    CK(cudaMemcpyAsync(tr.data(), static_cast<const GateHdr*>(gate) + 1, 2 * k * sizeof(double),
                       cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    for (uint64_t i = 0; i < k; ++i) {
      if (errors_out) errors_out[i] = tr[2 * i];
      if (l1_out) l1_out[i] = tr[2 * i + 1];
    }
  }
  return FPR_B200_OK;
}

int fpr_b200_part_set_gate(fpr_b200_graph* h, const void* gate) {
  if (!h) return fail(FPR_B200_EINVAL, "fpr_b200_part_set_gate: null graph");
  h->gate = static_cast<const unsigned int*>(gate);  // GateHdr::stop is its first word
  return FPR_B200_OK;
}

int fpr_b200_part_ranks_after(fpr_b200_graph* h, uint64_t sweeps, double* ranks_out) {
  if (!h || !ranks_out) return fail(FPR_B200_EINVAL, "fpr_b200_part_ranks_after: null argument");
  if (!h->part_pr[0]) return fail(FPR_B200_EINVAL, "fpr_b200_part_ranks_after: call fpr_b200_part_init first");
  if (sweeps > h->part_sweeps)
    return fail(FPR_B200_EINVAL, "fpr_b200_part_ranks_after: " + std::to_string(sweeps) + " sweeps requested, " +
                                     std::to_string(h->part_sweeps) + " issued");
  if (sweeps + 1 < h->part_sweeps && !h->gate)
    return fail(FPR_B200_EINVAL, "fpr_b200_part_ranks_after: only the last two states are kept (no gate)");
  CK(cudaSetDevice(h->device));
  // part_init leaves the ranks in part_pr[0]; sweep k writes part_pr[k % 2];
  // gated no-op sweeps write nothing
  CK(cudaMemcpyAsync(ranks_out, h->part_pr[sweeps & 1], h->g.n * sizeof(double), cudaMemcpyDeviceToHost,
                     h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return FPR_B200_OK;
}

int fpr_b200_part_info(const fpr_b200_graph* h, uint64_t* n_global, uint64_t* row_begin,
                       uint64_t* slice, uint32_t* nparts, uint32_t* part) {
  if (!h) return fail(FPR_B200_EINVAL, "fpr_b200_part_info: null graph");
  if (n_global) *n_global = h->nparts > 1 ? h->n_global : (uint64_t)h->g.n;
  if (row_begin) *row_begin = h->row_begin;
  if (slice) *slice = h->nparts > 1 ? h->slice : (uint64_t)h->g.n;
  if (nparts) *nparts = h->nparts;
  if (part) *part = h->part_id;
  return FPR_B200_OK;
}

int fpr_b200_part_ranks(fpr_b200_graph* h, double* ranks_out) {
  if (!h || !ranks_out) return fail(FPR_B200_EINVAL, "fpr_b200_part_ranks: null argument");
  CK(cudaSetDevice(h->device));
  const double* src = h->part_pr[0] ? h->part_pr[h->part_pr_cur] : h->pr;
  CK(cudaMemcpyAsync(ranks_out, src, h->g.n * sizeof(double), cudaMemcpyDeviceToHost, h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return FPR_B200_OK;
}

int fpr_b200_part_ranks_prev(fpr_b200_graph* h, double* ranks_out) {
  if (!h || !ranks_out) return fail(FPR_B200_EINVAL, "fpr_b200_part_ranks_prev: null argument");
  if (!h->part_pr[0] || h->part_sweeps == 0)
    return fail(FPR_B200_EINVAL, "fpr_b200_part_ranks_prev: no sweep since fpr_b200_part_init");
  CK(cudaSetDevice(h->device));
  CK(cudaMemcpyAsync(ranks_out, h->part_pr[h->part_pr_cur ^ 1], h->g.n * sizeof(double), cudaMemcpyDeviceToHost,
                     h->stream));
  CK(cudaStreamSynchronize(h->stream));
  return FPR_B200_OK;
}

int fpr_b200_pagerank(const fpr_graph_view* view, int engine, const fpr_config* cfg,
                      const fpr_b200_options* opts, double* ranks_out, double* errors_out,
                      uint64_t errors_cap, fpr_b200_result* result) {
  if (!view || !cfg) return fail(FPR_B200_EINVAL, "fpr_b200_pagerank: null argument");
  int rc = validate_config(cfg);
  if (rc) return rc;
  if (view->n == 0) return fail(FPR_B200_EINVAL, "pagerank: graph has no vertices");
  if (opts && opts->ndevices > 1) {  // one host thread drives opts->ndevices parts
    fpr_b200_mgpu* mg = nullptr;
    if ((rc = fpr_b200_mgpu_create(view, opts, &mg))) return rc;
    rc = fpr_b200_mgpu_run(mg, engine, cfg, ranks_out, errors_out, nullptr, errors_cap, result);
    fpr_b200_mgpu_destroy(mg);
    return rc;
  }
  fpr_b200_graph* h = nullptr;
  if ((rc = fpr_b200_graph_create(view, opts, &h))) return rc;
  rc = fpr_b200_run(h, engine, cfg, ranks_out, errors_out, nullptr, nullptr, errors_cap, result);
  fpr_b200_graph_destroy(h);
  return rc;
}

}  // extern "C"

// ------------------------------------------------------------ edge-list ingest
namespace {

void set_parse_error(fpr_parse_error* err, uint64_t line, int kind, const std::string& what) {
  if (!err) return;
  err->line = line;
  err->kind = kind;
  // ParseError::what() is a C string: a NUL inside a bad token ends it.
  const size_t nbytes = std::min(std::strlen(what.c_str()), sizeof(err->message) - 1);
  err->message_len = (uint32_t)nbytes;
  std::memcpy(err->message, what.data(), nbytes);
  err->message[nbytes] = 0;
}

// Text -> device -> ingest_edge_list.  Returns a status; *ing owns device pairs.
int ingest_text(fpr_b200_graph* h, const char* text, uint64_t len, Ingested* ing, fpr_parse_error* perr) {
  set_parse_error(perr, 0, 0, "");
  if (!text && len) return fail(FPR_B200_EINVAL, "fpr_b200_parse_edge_list: null text");
  unsigned char* dtext = nullptr;
  cudaError_t e = cudaMallocAsync((void**)&dtext, std::max<uint64_t>(len, 1), h->stream);
  if (e == cudaSuccess && len) {
    if (is_pinned(text)) {
      e = cudaMemcpyAsync(dtext, text, len, cudaMemcpyHostToDevice, h->stream);
    } else {
      UploadRing* ring = get_ring(h->device);
      if (!ring) {
        cudaFreeAsync(dtext, h->stream);
        return fail(FPR_B200_ENOMEM, "fpr_b200: pinned upload ring allocation failed");
      }
      std::lock_guard<std::mutex> lk(ring->mu);
      ring_upload_bytes(ring, text, dtext, (int64_t)len, h->stream, &e);
      if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);  // ring reusable once we return
    }
  }
  const char* msg = nullptr;
  IngestError ie;
  if (e == cudaSuccess)
    e = ingest_edge_list(dtext, len, len > 0 && text[len - 1] == '\n', h->stream, *ing, ie, &msg);
  if (dtext) cudaFreeAsync(dtext, h->stream);
  if (e != cudaSuccess)
    return fail(e == cudaErrorMemoryAllocation ? FPR_B200_ENOMEM : FPR_B200_ECUDA,
                std::string("fpr_b200_parse_edge_list: ") + cudaGetErrorString(e));
  if (msg) return fail(FPR_B200_ERANGE, std::string("fpr_b200_parse_edge_list: ") + msg);
  if (ie.line) {
    // fpr::ParseError::what() (edge_list.hpp:17-21, 60-72)
    std::string what = ie.kind == FPR_B200_PARSE_TOKENS      ? std::string("expected two integer tokens")
                       : ie.kind == FPR_B200_PARSE_BAD_TOKEN ? "bad token '" + ie.token + "'"
                                                             : std::string("trailing characters after edge");
    what = "line " + std::to_string(ie.line) + ": " + what;
    what.resize(std::strlen(what.c_str()));  // what() semantics (C string)
    set_parse_error(perr, ie.line, ie.kind, what);
    return fail(FPR_B200_EPARSE, what);
  }
  if (ing->n >= (1ull << 31)) {
    if (ing->pairs) cudaFreeAsync(ing->pairs, h->stream);
    *ing = Ingested{};
    return fail(FPR_B200_ERANGE, "fpr_b200: edge list has 2^31 or more distinct ids (int32 vertex ids)");
  }
  return FPR_B200_OK;
}

__global__ void widen_pairs_kernel(const int32_t* in, int64_t count, uint64_t* out) {
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < count; i += stride)
    out[i] = (uint64_t)(uint32_t)in[i];
}

}  // namespace

extern "C" {

int fpr_b200_parse_edge_list(const char* text, uint64_t len, const fpr_b200_options* opts, uint64_t* n_out,
                             uint64_t* m_out, uint64_t* edges_out, uint64_t edges_cap, fpr_parse_error* err) {
  fpr_b200_graph* h = nullptr;
  int rc = open_handle(opts, &h);
  if (rc) {
    destroy_handle(h);
    return rc;
  }
  Ingested ing;
  rc = ingest_text(h, text, len, &ing, err);
  if (rc == FPR_B200_OK) {
    if (n_out) *n_out = ing.n;
    if (m_out) *m_out = (uint64_t)ing.m;
    if (edges_out && (uint64_t)ing.m > edges_cap) {
      rc = fail(FPR_B200_ERANGE, "fpr_b200_parse_edge_list: edges_cap " + std::to_string(edges_cap) +
                                     " < m " + std::to_string(ing.m));
    } else if (edges_out && ing.m > 0) {
      uint64_t* wide = nullptr;
      const int64_t cnt = 2 * ing.m;
      cudaError_t e = cudaMallocAsync((void**)&wide, cnt * sizeof(uint64_t), h->stream);
      if (e == cudaSuccess) {
        widen_pairs_kernel<<<(int)std::min<int64_t>((cnt + 255) / 256, 148 * 16), 256, 0, h->stream>>>(
            ing.pairs, cnt, wide);
        e = cudaGetLastError();
      }
      if (e == cudaSuccess)
        e = cudaMemcpyAsync(edges_out, wide, cnt * sizeof(uint64_t), cudaMemcpyDeviceToHost, h->stream);
      if (wide) cudaFreeAsync(wide, h->stream);
      if (e == cudaSuccess) e = cudaStreamSynchronize(h->stream);
      if (e != cudaSuccess)
        rc = fail(FPR_B200_ECUDA, std::string("fpr_b200_parse_edge_list: ") + cudaGetErrorString(e));
    }
  }
  if (ing.pairs) cudaFreeAsync(ing.pairs, h->stream);
  destroy_handle(h);
  return rc;
}

int fpr_b200_graph_from_edge_list(const char* text, uint64_t len, const fpr_b200_options* opts,
                                  fpr_b200_graph** out, fpr_parse_error* err) {
  if (!out) return fail(FPR_B200_EINVAL, "fpr_b200_graph_from_edge_list: null argument");
  *out = nullptr;
  fpr_b200_graph* h = nullptr;
  int rc = open_handle(opts, &h);
  if (rc) {
    destroy_handle(h);
    return rc;
  }
  Ingested ing;
  if ((rc = ingest_text(h, text, len, &ing, err))) {
    destroy_handle(h);
    return rc;
  }
  const char* msg = nullptr;
  cudaError_t e = build_csr_from_pairs(ing.pairs, ing.m, ing.n, h->g, h->stream, &msg);
  if (ing.pairs) cudaFreeAsync(ing.pairs, h->stream);
  if (e != cudaSuccess || msg) {
    destroy_handle(h);
    if (msg) return fail(FPR_B200_ENOMEM, std::string("fpr_b200_graph_from_edge_list: ") + msg);
    return fail(e == cudaErrorMemoryAllocation ? FPR_B200_ENOMEM : FPR_B200_ECUDA,
                std::string("fpr_b200_graph_from_edge_list: ") + cudaGetErrorString(e));
  }
  h->allocs.push_back(h->g.row);
  h->allocs.push_back(h->g.src);
  h->allocs.push_back(h->g.outdeg);
  if ((rc = finish_graph(h))) {
    destroy_handle(h);
    return rc;
  }
  *out = h;
  return FPR_B200_OK;
}

}  // extern "C"

// ------------------------------------------------------------ CUDA IPC (fused exchange)
namespace {
std::map<void*, void*> g_ipc_offsets;  // imported pointer -> mapped allocation base
std::mutex g_ipc_mu;
}  // namespace

extern "C" {

// A handle is the 64-B cudaIpcMemHandle of the ALLOCATION containing dev_ptr
// (caching allocators such as torch's sub-allocate) plus dev_ptr's byte
// offset inside it; the importer maps the allocation and adds the offset.
namespace {
using GetAddressRangeFn = int (*)(unsigned long long*, size_t*, unsigned long long);
cudaError_t allocation_base(const void* p, uintptr_t* base) {
  static GetAddressRangeFn fn = nullptr;
  if (!fn) {
    void* sym = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaError_t e = cudaGetDriverEntryPoint("cuMemGetAddressRange", &sym, cudaEnableDefault, &q);
    if (e != cudaSuccess || !sym) return e != cudaSuccess ? e : cudaErrorNotSupported;
    fn = reinterpret_cast<GetAddressRangeFn>(sym);
  }
  unsigned long long b = 0;
  size_t size = 0;
  if (fn(&b, &size, (unsigned long long)(uintptr_t)p) != 0) return cudaErrorInvalidValue;
  *base = (uintptr_t)b;
  return cudaSuccess;
}
}  // namespace

int fpr_b200_ipc_export(const void* dev_ptr, void* handle_out) {
  if (!dev_ptr || !handle_out) return fail(FPR_B200_EINVAL, "fpr_b200_ipc_export: null argument");
  cudaIpcMemHandle_t hd;
  uintptr_t base = 0;
  cudaError_t e = allocation_base(dev_ptr, &base);
  if (e == cudaSuccess) e = cudaIpcGetMemHandle(&hd, reinterpret_cast<void*>(base));
  if (e != cudaSuccess) return fail(FPR_B200_ECUDA, std::string("fpr_b200_ipc_export: ") + cudaGetErrorString(e));
  static_assert(sizeof(hd) + sizeof(uint64_t) == FPR_B200_IPC_HANDLE_BYTES, "IPC handle size");
  const uint64_t off = (uint64_t)((uintptr_t)dev_ptr - base);
  std::memcpy(handle_out, &hd, sizeof(hd));
  std::memcpy(static_cast<char*>(handle_out) + sizeof(hd), &off, sizeof(off));
  return FPR_B200_OK;
}

int fpr_b200_ipc_import(const void* handle, int device, void** dev_ptr_out) {
  if (!handle || !dev_ptr_out) return fail(FPR_B200_EINVAL, "fpr_b200_ipc_import: null argument");
  *dev_ptr_out = nullptr;
  cudaIpcMemHandle_t hd;
  uint64_t off = 0;
  std::memcpy(&hd, handle, sizeof(hd));
  std::memcpy(&off, static_cast<const char*>(handle) + sizeof(hd), sizeof(off));
  void* base = nullptr;
  cudaError_t e = device >= 0 ? cudaSetDevice(device) : cudaSuccess;
  // LazyEnablePeerAccess: a buffer on another GPU is reached over NVLink P2P
  if (e == cudaSuccess) e = cudaIpcOpenMemHandle(&base, hd, cudaIpcMemLazyEnablePeerAccess);
  if (e != cudaSuccess) return fail(FPR_B200_ECUDA, std::string("fpr_b200_ipc_import: ") + cudaGetErrorString(e));
  *dev_ptr_out = static_cast<char*>(base) + off;
  std::lock_guard<std::mutex> lk(g_ipc_mu);
  g_ipc_offsets[*dev_ptr_out] = base;
  return FPR_B200_OK;
}

int fpr_b200_ipc_close(void* dev_ptr) {
  if (!dev_ptr) return FPR_B200_OK;
  void* base = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_ipc_mu);
    auto it = g_ipc_offsets.find(dev_ptr);
    if (it == g_ipc_offsets.end()) return fail(FPR_B200_EINVAL, "fpr_b200_ipc_close: not an imported pointer");
    base = it->second;
    g_ipc_offsets.erase(it);
  }
  cudaError_t e = cudaIpcCloseMemHandle(base);
  if (e != cudaSuccess) return fail(FPR_B200_ECUDA, std::string("fpr_b200_ipc_close: ") + cudaGetErrorString(e));
  return FPR_B200_OK;
}

}  // extern "C"

#ifdef FPR_TRACE_WARPS
// Diagnostic build only: per-warp finish times of sweep 2 and the sweep stamps.
extern "C" int fpr_b200_debug_warp_times(fpr_b200_graph* h, uint64_t* out, uint64_t nwarps) {
  cudaMemcpy(out, reinterpret_cast<unsigned long long*>(h->tail_partial) + h->part.ntasks + 1, nwarps * 8,
             cudaMemcpyDeviceToHost);
  cudaMemcpy(out + nwarps, h->d_ns, 5 * 8, cudaMemcpyDeviceToHost);
  return 0;
}
#endif


namespace fprb {
int set_error(int code, const std::string& msg) { return fail(code, msg); }
cudaStream_t graph_stream(const void* h) { return static_cast<const fpr_b200_graph*>(h)->stream; }
int graph_device(const void* h) { return static_cast<const fpr_b200_graph*>(h)->device; }
bool graph_uses_pb(const void* h) { return static_cast<const fpr_b200_graph*>(h)->use_pb; }
}  // namespace fprb
