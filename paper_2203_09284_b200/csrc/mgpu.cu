// mgpu.cu -- the multi-device solve driven by ONE host thread
// (include/fpr_b200.h, fpr_b200_mgpu_*; SURVEY §8(b) Threading row, §8(e)).
//
// The reference's parallel engines cut the vertices into static blocks, one
// per thread (pagerank.hpp:111-122 block_for), separated by a barrier whose
// completion step reduces the per-thread maxima and applies the stop rule
// (:209-218, :276-286).  Here a block is an edge-balanced destination range
// of rows (the merge-path split of fpr_b200_part_create), one per device:
//   * part r lives on devices[r] with its rows, their in-edges (sources
//     remapped into the padded exchange space P x slice) and two exchange
//     vectors (EC ping-pongs them; FUSED updates the first in place);
//   * one sweep per part per iteration, on the part's stream; its epilogue
//     stores every new contribution into ALL parts' exchange vectors -- peer
//     stores over NVLink between distinct GPUs (peer access enabled here),
//     plain stores within one device -- so the sweep is the all-gather
//     (fpr_b200_part_sweep_peers: kernels.cu kModePeers for the pull sweep,
//     the accumulate's finalize in pb.cu for propagation-blocked parts, which
//     the library picks when the exchange space far exceeds L2);
//   * the stop rule runs on the devices: after each iteration every part's
//     stream waits (CUDA events, no host involvement) for all parts' sweeps,
//     then a one-thread gate kernel reduces the parts' 16-B (max, sum)
//     residual pairs in part order -- peer loads -- (the on_barrier step,
//     deterministic) and applies the reference's predicate
//     `error <= threshold` (:141, :216); once it holds, the parts' later
//     sweeps are no-ops (fpr_b200_part_set_gate).  The calling thread
//     enqueues batches of iterations and reads device 0's gate once per
//     batch, so no iteration waits on a host round trip.
// Parts that share a device run on their own streams one after the other;
// the test suite uses that to check P parts against one GPU.
#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "../../include/fpr_b200.h"
#include "internal.cuh"

struct fpr_b200_mgpu {
  uint32_t P = 0;
  uint64_t n = 0, m = 0, slice = 0;
  int norm = FPR_B200_NORM_LINF;
  std::vector<int> dev;
  std::vector<fpr_b200_graph*> parts;
  std::vector<uint64_t> bounds;    // P + 1 row bounds
  std::vector<double*> x[2];       // per part: exchange vectors (P * slice doubles, on the part's device)
  std::vector<double*> dpair;      // per part: its (max, sum) residual pair, two slots by iteration parity
  std::vector<void*> gate;         // per part: device-side stop rule (fpr_b200_gate_*) on its device
  uint64_t gate_cap = 0;           // trace capacity of the gates
  std::vector<cudaEvent_t> ev[2];  // per part: its sweep of an even / odd iteration finished
};

namespace {

using fprb::set_error;

#define MCK(call)                                                                                        \
  do {                                                                                                   \
    cudaError_t e_ = (call);                                                                             \
    if (e_ != cudaSuccess)                                                                               \
      return set_error(e_ == cudaErrorMemoryAllocation ? FPR_B200_ENOMEM : FPR_B200_ECUDA,               \
                       std::string("fpr_b200_mgpu: CUDA error '") + cudaGetErrorString(e_) + "' (" #call ")"); \
  } while (0)

int check_opts(const fpr_b200_options* opts) {
  if (!opts || opts->ndevices < 1 || !opts->devices)
    return set_error(FPR_B200_EINVAL, "fpr_b200_mgpu: opts->devices / opts->ndevices must name the parts' devices");
  if (opts->ndevices > 8)
    return set_error(FPR_B200_EINVAL, "fpr_b200_mgpu: at most 8 parts (one NVSwitch node)");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
    return set_error(FPR_B200_ECUDA, "fpr_b200_mgpu: no CUDA device available");
  for (uint32_t r = 0; r < opts->ndevices; ++r)
    if (opts->devices[r] < 0 || opts->devices[r] >= ndev)
      return set_error(FPR_B200_EINVAL, "fpr_b200_mgpu: device " + std::to_string(opts->devices[r]) +
                                            " out of range (" + std::to_string(ndev) + " devices)");
  return FPR_B200_OK;
}

// Peer access between every pair of distinct devices (NVLink through
// NVSwitch on a B200 node); parts on the same device need none.
int enable_peers(const std::vector<int>& dev) {
  for (int a : dev)
    for (int b : dev) {
      if (a == b) continue;
      int ok = 0;
      MCK(cudaDeviceCanAccessPeer(&ok, a, b));
      if (!ok)
        return set_error(FPR_B200_ECUDA, "fpr_b200_mgpu: device " + std::to_string(a) +
                                             " cannot access device " + std::to_string(b) + " (no P2P path)");
      MCK(cudaSetDevice(a));
      const cudaError_t e = cudaDeviceEnablePeerAccess(b, 0);
      if (e == cudaErrorPeerAccessAlreadyEnabled) {
        cudaGetLastError();
      } else if (e != cudaSuccess) {
        return set_error(FPR_B200_ECUDA, std::string("fpr_b200_mgpu: cudaDeviceEnablePeerAccess: ") +
                                             cudaGetErrorString(e));
      }
    }
  return FPR_B200_OK;
}

// Exchange vectors, residual pairs and peer access once the parts exist.
int finish(fpr_b200_mgpu* mg) {
  int rc = enable_peers(mg->dev);
  if (rc) return rc;
  for (auto& v : mg->x) v.assign(mg->P, nullptr);
  mg->dpair.assign(mg->P, nullptr);
  for (uint32_t r = 0; r < mg->P; ++r) {
    MCK(cudaSetDevice(mg->dev[r]));
    for (auto& v : mg->x) MCK(cudaMalloc(&v[r], (size_t)mg->P * mg->slice * sizeof(double)));
    // on the part's own stream: the library's streams are non-blocking, so a
    // legacy-stream cudaMemset could land after the first run's part_init
    const cudaStream_t st = fprb::graph_stream(mg->parts[r]);
    MCK(cudaMemsetAsync(mg->x[0][r], 0, (size_t)mg->P * mg->slice * sizeof(double), st));
    MCK(cudaMemsetAsync(mg->x[1][r], 0, (size_t)mg->P * mg->slice * sizeof(double), st));
    MCK(cudaMalloc(&mg->dpair[r], 4 * sizeof(double)));
    MCK(cudaMemsetAsync(mg->dpair[r], 0, 4 * sizeof(double), st));
    MCK(cudaStreamSynchronize(st));
  }
  mg->gate.assign(mg->P, nullptr);
  for (auto& v : mg->ev) {
    v.assign(mg->P, nullptr);
    for (uint32_t r = 0; r < mg->P; ++r) {
      MCK(cudaSetDevice(mg->dev[r]));
      MCK(cudaEventCreateWithFlags(&v[r], cudaEventDisableTiming));
    }
  }
  return FPR_B200_OK;
}

std::vector<int> devices_of(const fpr_b200_options* opts) {
  return std::vector<int>(opts->devices, opts->devices + opts->ndevices);
}

}  // namespace

extern "C" {

void fpr_b200_mgpu_destroy(fpr_b200_mgpu* mg) {
  if (!mg) return;
  for (uint32_t r = 0; r < mg->parts.size(); ++r) {
    cudaSetDevice(mg->dev[r]);
    cudaDeviceSynchronize();
    for (auto& v : mg->x)
      if (r < v.size() && v[r]) cudaFree(v[r]);
    if (r < mg->dpair.size() && mg->dpair[r]) cudaFree(mg->dpair[r]);
    if (r < mg->gate.size() && mg->gate[r]) cudaFree(mg->gate[r]);
    for (auto& v : mg->ev)
      if (r < v.size() && v[r]) cudaEventDestroy(v[r]);
    fpr_b200_graph_destroy(mg->parts[r]);
  }
  delete mg;
}

int fpr_b200_mgpu_create(const fpr_graph_view* view, const fpr_b200_options* opts, fpr_b200_mgpu** out) {
  if (!view || !out) return set_error(FPR_B200_EINVAL, "fpr_b200_mgpu_create: null argument");
  *out = nullptr;
  int rc = check_opts(opts);
  if (rc) return rc;
  auto* mg = new fpr_b200_mgpu;
  mg->P = opts->ndevices;
  mg->dev = devices_of(opts);
  mg->norm = opts->norm;
  mg->n = view->n;
  mg->m = view->m;
  mg->bounds.assign(mg->P + 1, 0);
  mg->parts.assign(mg->P, nullptr);
  for (uint32_t r = 0; r < mg->P && !rc; ++r) {
    fpr_b200_options o = *opts;
    o.device = mg->dev[r];
    o.devices = nullptr;
    o.ndevices = 0;
    o.stream = nullptr;  // every part on its own library stream
    // only this part's rows and in-edges cross its link
    rc = fpr_b200_part_create(view, mg->P, r, &o, mg->bounds.data(), &mg->slice, &mg->parts[r]);
  }
  if (!rc) rc = finish(mg);
  if (rc) {
    fpr_b200_mgpu_destroy(mg);
    return rc;
  }
  *out = mg;
  return FPR_B200_OK;
}

int fpr_b200_mgpu_generate(const fpr_gen_params* params, const fpr_b200_options* opts, fpr_b200_mgpu** out) {
  if (!params || !out) return set_error(FPR_B200_EINVAL, "fpr_b200_mgpu_generate: null argument");
  *out = nullptr;
  int rc = check_opts(opts);
  if (rc) return rc;
  auto* mg = new fpr_b200_mgpu;
  mg->P = opts->ndevices;
  mg->dev = devices_of(opts);
  mg->norm = opts->norm;
  mg->bounds.assign(mg->P + 1, 0);
  mg->parts.assign(mg->P, nullptr);
  // one full graph per distinct device (the generators are deterministic),
  // partitioned into that device's parts, then released
  std::vector<int> done;
  for (uint32_t r = 0; r < mg->P && !rc; ++r) {
    const int d = mg->dev[r];
    if (std::find(done.begin(), done.end(), d) != done.end()) continue;
    done.push_back(d);
    fpr_b200_options o = *opts;
    o.device = d;
    o.devices = nullptr;
    o.ndevices = 0;
    o.stream = nullptr;
    fpr_b200_graph* full = nullptr;
    if ((rc = fpr_b200_graph_generate(params, &o, &full))) break;
    uint64_t n = 0, m = 0, nt = 0;
    fpr_b200_graph_info(full, &n, &m, &nt);
    mg->n = n;
    mg->m = m;
    for (uint32_t q = 0; q < mg->P && !rc; ++q)
      if (mg->dev[q] == d) rc = fpr_b200_graph_partition(full, mg->P, q, &o, mg->bounds.data(), &mg->slice, &mg->parts[q]);
    fpr_b200_graph_destroy(full);
  }
  if (!rc) rc = finish(mg);
  if (rc) {
    fpr_b200_mgpu_destroy(mg);
    return rc;
  }
  *out = mg;
  return FPR_B200_OK;
}

int fpr_b200_mgpu_info(const fpr_b200_mgpu* mg, uint64_t* n, uint64_t* m, uint32_t* nparts, uint64_t* bounds) {
  if (!mg) return set_error(FPR_B200_EINVAL, "fpr_b200_mgpu_info: null handle");
  if (n) *n = mg->n;
  if (m) *m = mg->m;
  if (nparts) *nparts = mg->P;
  if (bounds) std::copy(mg->bounds.begin(), mg->bounds.end(), bounds);
  return FPR_B200_OK;
}

int fpr_b200_mgpu_run(fpr_b200_mgpu* mg, int engine, const fpr_config* cfg, double* ranks_out, double* errors_out,
                      double* l1_out, uint64_t errors_cap, fpr_b200_result* result) {
  if (!mg || !cfg) return set_error(FPR_B200_EINVAL, "fpr_b200_mgpu_run: null argument");
  // validate(PageRankConfig), pagerank.hpp:40-53 (the part sweep re-checks it)
  if (!(cfg->damping > 0.0 && cfg->damping < 1.0)) return set_error(FPR_B200_EINVAL, "pagerank: damping must be in (0,1)");
  if (!(cfg->threshold > 0.0)) return set_error(FPR_B200_EINVAL, "pagerank: threshold must be positive");
  if (cfg->max_iterations == 0) return set_error(FPR_B200_EINVAL, "pagerank: max_iterations must be positive");
  if (cfg->thread_count == 0) return set_error(FPR_B200_EINVAL, "pagerank: thread_count must be positive");
  if (engine != FPR_B200_ENGINE_EC && engine != FPR_B200_ENGINE_FUSED)
    return set_error(FPR_B200_EINVAL, "fpr_b200_mgpu_run: multi-device engines are EC and FUSED");
  const uint32_t P = mg->P;
  const size_t sl = (size_t)mg->slice;
  int rc;
  cudaEvent_t t0 = nullptr, t1 = nullptr;
  MCK(cudaSetDevice(mg->dev[0]));
  MCK(cudaEventCreate(&t0));
  MCK(cudaEventCreate(&t1));
  // init: every part writes 1/n ranks and its contribution slice into its own
  // first exchange vector, then the slices are copied to every other part
  for (uint32_t r = 0; r < P; ++r)
    if ((rc = fpr_b200_part_init(mg->parts[r], mg->x[0][r]))) return rc;
  for (uint32_t r = 0; r < P; ++r) {
    MCK(cudaSetDevice(mg->dev[r]));
    MCK(cudaStreamSynchronize(fprb::graph_stream(mg->parts[r])));
  }
  for (uint32_t q = 0; q < P; ++q)
    for (uint32_t r = 0; r < P; ++r)
      if (q != r)
        MCK(cudaMemcpyPeerAsync(mg->x[0][q] + r * sl, mg->dev[q], mg->x[0][r] + r * sl, mg->dev[r],
                                sl * sizeof(double), fprb::graph_stream(mg->parts[q])));
  for (uint32_t r = 0; r < P; ++r) {
    MCK(cudaSetDevice(mg->dev[r]));
    MCK(cudaStreamSynchronize(fprb::graph_stream(mg->parts[r])));
  }
  // gates: one per part on its device (every part reaches the same decision
  // from the same pairs in the same order); trace capacity = the iteration cap
  const uint64_t cap = std::min<uint64_t>(cfg->max_iterations, uint64_t(1) << 22);
  if (mg->gate_cap < cap) {
    for (uint32_t r = 0; r < P; ++r) {
      MCK(cudaSetDevice(mg->dev[r]));
      if (mg->gate[r]) MCK(cudaFree(mg->gate[r]));
      mg->gate[r] = nullptr;
      MCK(cudaMalloc(&mg->gate[r], fpr_b200_gate_bytes(cap)));
    }
    mg->gate_cap = cap;
  }
  for (uint32_t r = 0; r < P; ++r) {
    if ((rc = fpr_b200_gate_init(mg->gate[r], mg->gate_cap, mg->dev[r], fprb::graph_stream(mg->parts[r])))) return rc;
    if ((rc = fpr_b200_part_set_gate(mg->parts[r], mg->gate[r]))) return rc;
  }
  uint64_t batch = 8;
  if (const char* v = std::getenv("FPR_B200_MGPU_BATCH")) batch = (uint64_t)std::max(1, std::atoi(v));
  MCK(cudaSetDevice(mg->dev[0]));
  MCK(cudaEventRecord(t0, fprb::graph_stream(mg->parts[0])));
  std::vector<double*> peers(P);
  std::vector<const double*> pairs(P);
  uint64_t issued = 0, it = 0;
  int stopped = 0;
  while (!stopped && issued < cfg->max_iterations) {
    for (uint64_t k = 0; k < batch && issued < cfg->max_iterations; ++k, ++issued) {
      const int par = (int)(issued & 1);
      const int cur = engine == FPR_B200_ENGINE_EC ? par : 0;
      const int nxt = engine == FPR_B200_ENGINE_EC ? cur ^ 1 : cur;
      for (uint32_t q = 0; q < P; ++q) peers[q] = mg->x[nxt][q];
      for (uint32_t r = 0; r < P; ++r) {
        // gated: a no-op once the stop rule held
        if ((rc = fpr_b200_part_sweep_peers(mg->parts[r], engine, cfg, mg->x[cur][r], mg->x[nxt][r], peers.data(), P,
                                            mg->dpair[r] + 2 * par)))
          return rc;
        MCK(cudaSetDevice(mg->dev[r]));
        MCK(cudaEventRecord(mg->ev[par][r], fprb::graph_stream(mg->parts[r])));
      }
      // the barrier (stream waits on every part's sweep: its pair and its
      // peer stores are in place), then the stop rule on every device
      for (uint32_t q = 0; q < P; ++q) pairs[q] = mg->dpair[q] + 2 * par;
      for (uint32_t r = 0; r < P; ++r) {
        MCK(cudaSetDevice(mg->dev[r]));
        for (uint32_t q = 0; q < P; ++q)
          if (q != r) MCK(cudaStreamWaitEvent(fprb::graph_stream(mg->parts[r]), mg->ev[par][q], 0));
        if ((rc = fpr_b200_gate_update(mg->gate[r], pairs.data(), P, cfg, mg->norm, mg->dev[r],
                                       fprb::graph_stream(mg->parts[r]))))
          return rc;
      }
    }
    // one read per batch: device 0's gate (its stream has waited for every part)
    if ((rc = fpr_b200_gate_read(mg->gate[0], mg->dev[0], fprb::graph_stream(mg->parts[0]), &it, &stopped, nullptr,
                                 nullptr, 0)))
      return rc;
  }
  MCK(cudaSetDevice(mg->dev[0]));
  MCK(cudaEventRecord(t1, fprb::graph_stream(mg->parts[0])));
  MCK(cudaEventSynchronize(t1));
  for (uint32_t r = 0; r < P; ++r) {
    MCK(cudaSetDevice(mg->dev[r]));
    MCK(cudaStreamSynchronize(fprb::graph_stream(mg->parts[r])));
  }
  float ms = 0.f;
  cudaEventElapsedTime(&ms, t0, t1);
  cudaEventDestroy(t0);
  cudaEventDestroy(t1);
  std::vector<double> errs(it), l1s(it);
  if (it > 0 && (rc = fpr_b200_gate_read(mg->gate[0], mg->dev[0], fprb::graph_stream(mg->parts[0]), &it, &stopped,
                                         errs.data(), l1s.data(), it)))
    return rc;
  if (it > mg->gate_cap && (errors_out || l1_out))
    return set_error(FPR_B200_EINVAL, "fpr_b200_mgpu_run: trace longer than " + std::to_string(mg->gate_cap));
  if (errors_out) {
    if (errors_cap < it)
      return set_error(FPR_B200_EINVAL, "fpr_b200_mgpu_run: errors buffer holds " + std::to_string(errors_cap) +
                                            " entries, need " + std::to_string(it));
    std::copy(errs.begin(), errs.end(), errors_out);
  }
  if (l1_out && errors_cap >= it) std::copy(l1s.begin(), l1s.end(), l1_out);
  const double err = it > 0 ? errs[it - 1] : 1.0, l1 = it > 0 ? l1s[it - 1] : 1.0;
  if (ranks_out)
    for (uint32_t r = 0; r < P; ++r)
      if ((rc = fpr_b200_part_ranks_after(mg->parts[r], it, ranks_out + mg->bounds[r]))) return rc;
  for (uint32_t r = 0; r < P; ++r) fpr_b200_part_set_gate(mg->parts[r], nullptr);
  if (result) {
    result->iterations = it;
    result->converged = (it > 0 && (mg->norm == FPR_B200_NORM_L1 ? l1 : err) <= cfg->threshold) ? 1 : 0;
    result->sweep = fprb::graph_uses_pb(mg->parts[0]) ? FPR_B200_SWEEP_PB : FPR_B200_SWEEP_PULL;
    result->final_error = it > 0 ? err : 1.0;
    result->solve_ms = ms;  // device 0's stream: first sweep issued .. last residual read
    result->setup_ms = 0.0;
    result->kernel_launches = issued * P * 2 + P;  // sweeps (no-ops after the stop included) + gate updates
  }
  return FPR_B200_OK;
}

}  // extern "C"
