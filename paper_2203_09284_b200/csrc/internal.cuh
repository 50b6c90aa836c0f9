// internal.cuh -- shared device/host declarations of libfpr_b200.so.
//
// HBM layout of a resident graph (narrowed):
//   row      int64[n+1]   in-CSR offsets (fpr::Graph::in_start)
//   src      int32[m]     in-edge sources, dst-grouped, ascending (in_src)
//   outdeg   int32[n]     out-degrees (out_degree)
//   pr       fp64[n]      ranks, updated in place by their owning task
//   contrib  fp64[2][n]   pr/outdeg; EC/lockstep ping-pong, FUSED uses [0] in place
//   task_*   merge-path partition of the (n + m) row-end/edge items into
//            warp tasks of TASK_ITEMS items (Merrill & Garland merge-based SpMV)
#pragma once

#include <cstdint>
#include <string>
#include <map>
#include <vector>
#include <cuda_runtime.h>

namespace fprb {

#ifndef FPR_BLOCK_THREADS
#define FPR_BLOCK_THREADS 256
#endif
constexpr int kBlockThreads = FPR_BLOCK_THREADS;
constexpr int kWarpsPerBlock = kBlockThreads / 32;
#ifndef FPR_TASK_DIAG
#define FPR_TASK_DIAG 224
#endif
#ifndef FPR_SNAP_EDGES
#define FPR_SNAP_EDGES 25
#endif
constexpr int kTaskDiag = FPR_TASK_DIAG;    // merge-path diagonal stride between warp tasks
constexpr int kSnapEdges = FPR_SNAP_EDGES;  // a boundary inside a row of <= kSnapEdges edges moves to its start
constexpr int kTaskItems = kTaskDiag + kSnapEdges;  // max items (and edges) per task: 249 (+7 pad <= 256)

struct GridBar {
  unsigned int count;
  unsigned int gen;
};

struct DevGraph {
  int32_t n = 0;
  int64_t m = 0;
  int64_t* row = nullptr;
  int32_t* src = nullptr;  // m + 8 entries: aligned 32-B loads may overrun by 7
  int32_t* outdeg = nullptr;
};

struct Partition {
  int32_t ntasks = 0;
  int32_t* task_row = nullptr;    // ntasks+1: first row whose end marker lies in task t
  int64_t* task_edge = nullptr;   // ntasks+1: first edge of task t
  int32_t* head_first = nullptr;  // ntasks: first task holding a piece of t's split head row, -1 if none
  uint8_t* clean_start = nullptr; // ntasks+1: task t begins at a row boundary
  uint32_t* task_bits = nullptr;  // ntasks x 8 words: bit p = a row segment starts at position p
};

// Everything the persistent solve kernel needs (passed by value).
constexpr int kMaxPeers = 7;  // parts - 1 on one NVSwitch node of 8 GPUs

// Per-launch result the host reads back in ONE copy (pinned mirror).
struct SolveStatus {
  unsigned int iters;
  int stop;
  double last[2];
};

struct SolveParams {
  int32_t n;
  const int64_t* row;
  const int32_t* src;
  const int32_t* outdeg;
  const int32_t* task_row;
  const int64_t* task_edge;
  const int32_t* head_first;
  const uint32_t* task_bits;  // ntasks x 8
  int32_t ntasks;
  const int32_t* wave_task;  // nwaves+1
  const int32_t* wave_row;   // nwaves+1
  int32_t nwaves;
  int64_t nsrc;   // contributions addressable by a gather (n, or nparts*slice for a part)
  double* pr;      // ranks read (old value of each row)
  double* pr_out;  // ranks written: == pr except in multi-GPU part sweeps (ping-pong)
  double* contrib0;
  double* contrib1;
  int32_t parity0;  // contrib buffer holding the previous sweep at local iteration 0
  int64_t write_off;  // multi-GPU: this part's slice offset in the exchange vector (0 otherwise)
  double* tail_partial;  // per task: partial of its open row; NaN = not ready
  double damping;
  double base;
  double threshold;
  int32_t norm;
  uint32_t max_iters;
  double* errors;     // [max_iters]
  double* l1errors;   // [max_iters]
  unsigned long long* iter_ns;  // [max_iters+1] globaltimer stamps
  double* partials;   // 2 * gridDim.x
  double* totals;     // 2
  GridBar* bar;
  unsigned int* out_iters;
  int* out_stop;
  double* out_last;  // [2]: residual (max, sum) of the launch's last sweep
  // Fused exchange (multi-GPU): every finalized contribution is also stored
  // into each peer's replica (peer[q] = that replica at this part's slice,
  // P2P-mapped), so the sweep itself performs the all-gather over NVLink.
  int32_t npeers;
  int32_t peer_skip_empty;  // peers already hold the constant contribution of rows without in-edges
  double* peer[kMaxPeers];
  // device-side stop (multi-GPU drivers): the sweep is a no-op while *gate
  // != 0 (the stop flag of a GateHdr); nullptr = ungated
  const unsigned int* gate;
};

// Device-side stop rule (fpr_b200_gate_*): header, then 2 x cap doubles of
// trace (max |delta|, sum |delta| per iteration).
struct GateHdr {
  unsigned int stop;
  unsigned int pad;
  unsigned long long iters;
  unsigned long long cap;
  unsigned long long pad2;
};
struct PairPtrs {
  int n = 0;
  const double* p[kMaxPeers + 1] = {};
};
cudaError_t launch_gate_init(GateHdr* g, uint64_t cap, cudaStream_t s);
// One iteration's stop decision from the parts' residual pairs, reduced in
// part order (max, sum) -- the host driver's rule, on the device.
cudaError_t launch_gate_update(GateHdr* g, const PairPtrs& pp, double threshold, int norm, uint64_t max_iterations,
                               cudaStream_t s);

enum Engine { kEC = 0, kFused = 1, kLockstep = 2 };
// Launch-shape id of the async engine on graphs whose contributions exceed
// ~64 MB (20 warps/SM instead of 16: more gathers in flight for DRAM-bound
// sweeps; measured).  Internal only.
constexpr int kFusedWide = 3;

// kernels.cu
cudaError_t launch_partition(const DevGraph& g, Partition& p, cudaStream_t s);
cudaError_t launch_init(const DevGraph& g, double* pr, double* contrib, cudaStream_t s);
cudaError_t solve_grid(int engine, int num_sms, int* grid_out);
int solve_block_threads(int engine);  // threads per CTA of the engine's solve kernel
cudaError_t launch_solve(int engine, int grid, const SolveParams& p, cudaStream_t s);
cudaError_t launch_narrow_ids(const uint64_t* in, int32_t* out, int64_t count, uint64_t bound,
                              unsigned int* bad_flag, cudaStream_t s);
cudaError_t launch_check_offsets(const int64_t* row, int32_t n, int64_t m, unsigned int* bad_flag,
                                 cudaStream_t s);
cudaError_t launch_part_bounds(const DevGraph& g, uint32_t nparts, int64_t* bounds, cudaStream_t s);
cudaError_t launch_part_extract(const DevGraph& g, const int64_t* bounds, uint32_t nparts,
                                uint32_t part, int64_t slice, int64_t nloc, int64_t mloc,
                                DevGraph& out, cudaStream_t s);
cudaError_t launch_offset_shift(int64_t* row, int64_t count, int64_t e0, cudaStream_t s);
cudaError_t launch_part_remap(int32_t* src, int64_t m, const int64_t* bounds, uint32_t nparts, int64_t slice,
                              cudaStream_t s);
cudaError_t launch_part_init(const DevGraph& g, double init, double* pr, double* contrib_slice,
                             cudaStream_t s);
cudaError_t launch_validate(const DevGraph& g, int32_t* recount, unsigned int* bad, cudaStream_t s);
cudaError_t launch_gather_ranks(const double* pr, const int32_t* new_of_old, int32_t n, double* out,
                               cudaStream_t s);
cudaError_t launch_widen(const int64_t* row, const int32_t* ids32, uint64_t* out_row,
                         uint64_t* out_ids, int64_t nrow, int64_t nids, cudaStream_t s);

// generate.cu
struct GenRequest {
  int kind;  // 0 rmat, 1 uniform, 2 chung-lu
  uint32_t scale;
  uint64_t edge_factor;
  double a, b, c, d;
  uint64_t n;
  uint64_t avg_degree;
  uint64_t seed;
  uint64_t draws;    // chung-lu
  double alpha;      // chung-lu
  uint64_t kmax;     // chung-lu
  int relabel_bfs;   // config 3: BFS crawl-order relabel
  uint64_t bfs_root;
};
// Builds row/src/outdeg on the device (allocates them into g).  Returns a
// cudaError_t; *msg receives a static description on non-CUDA failures.
cudaError_t generate_graph(const GenRequest& req, DevGraph& g, cudaStream_t s, const char** msg);
// Raw draws [i0, i0 + count) of the rmat (kind 0) / uniform (kind 1) generator.
cudaError_t generate_draws(const GenRequest& req, uint64_t i0, uint64_t count, uint64_t* d_src, uint64_t* d_dst,
                           cudaStream_t s);
// Locality reorder by descending out-degree, or (sources_only) the stable
// partition with the out-degree > 0 vertices first: new CSR in `out`
// (allocated on stream s), *perm = device new_of_old (n int32, caller frees).
cudaError_t reorder_by_degree(const DevGraph& g, bool sources_only, int block_shift, DevGraph& out, int32_t** perm,
                              cudaStream_t s, const char** msg);
// BFS discovery order of g (config-3 relabel) into a host buffer of n int32.
cudaError_t relabel_order_bfs(const DevGraph& g, int32_t root, int32_t* new_id_out,
                              cudaStream_t s, const char** msg);

// host_narrow.cpp: out[i] = (int32)in[i]; true if any in[i] >= bound.
bool host_narrow_ids(const uint64_t* in, int32_t* out, int64_t count, uint64_t bound);

// ingest.cu: fpr::parse_edge_list on the device.  `t` = the text (device,
// len bytes).  On success out.pairs holds 2*out.m int32 dense ids (src, dst
// per edge, input order; cudaMallocAsync on st, caller frees) and out.n the
// number of distinct ids.  A malformed line sets err (line > 0) instead.
struct Ingested {
  int32_t* pairs = nullptr;
  int64_t m = 0;
  uint64_t n = 0;
};
struct IngestError {
  uint64_t line = 0;  // 1-based; 0 = none
  int kind = 0;       // FPR_B200_PARSE_*
  std::string token;  // the bad token's bytes
};
cudaError_t ingest_edge_list(const unsigned char* t, uint64_t len, bool ends_with_newline, cudaStream_t st,
                             Ingested& out, IngestError& err, const char** msg);
// generate.cu: build_csr over m edges given as two int32 arrays, ids in [0, n).
cudaError_t build_csr_from_arrays(const int32_t* src, const int32_t* dst, int64_t m, uint64_t n, DevGraph& g,
                                  cudaStream_t st, const char** msg);
// generate.cu: build_csr over m (src, dst) int32 pairs with ids in [0, n).
cudaError_t build_csr_from_pairs(const int32_t* pairs, int64_t m, uint64_t n, DevGraph& g, cudaStream_t st,
                                 const char** msg);

// pb.cu: propagation-blocked EC (FPR_B200_OPT_PB).
// A sweep plan: the bins cut into waves of consecutive bins (1 wave = EC,
// S waves = the lockstep Gauss-Seidel schedule), phase-1 pieces ordered
// (wave, chunk, bin) so each wave walks the chunks in order.
struct PbPlan {
  int nwaves = 0;
  std::vector<int64_t> wave_bin;  // nwaves + 1: first bin of each wave
  std::vector<int64_t> item0;     // nwaves + 1: first phase-1 piece of each wave
  std::vector<int64_t> unit0;     // nwaves + 1: first phase-2 unit of each wave
  // phase-2 units: whole bins, heavy bins cut into runs of whole tiles
  // (smaller pieces for more waves, so that every wave has a few units per CTA)
  int32_t* unit_bin = nullptr;
  int64_t* unit_e = nullptr;      // 2 x units: [first, end) run position of each unit
  int64_t* unit_t = nullptr;      // units: the unit's first tile
  int32_t* unit_k = nullptr;      // units of the unit's bin (1 = the bin is whole)
  int32_t* unit_j = nullptr;      // index of the unit within its bin
  int32_t* unit_slot = nullptr;   // split bins: the bin's first row-sum slot (-1 otherwise)
  double* slots = nullptr;        // split-bin units' row sums, 2^shift doubles per slot
  int64_t* item_start = nullptr;  // pieces: first entry, length and first run
  uint32_t* item_len = nullptr;
  int64_t* item_ubase = nullptr;
  unsigned long long* ctr = nullptr;  // 2 x nwaves work counters (reset per sweep)
  std::vector<void*> allocs;
};
struct PbSet {
  int shift = 0;         // destination bin = row >> shift (at most 2^16 rows: uint16 offsets)
  int chunk_shift = 0;   // source chunk = src >> chunk_shift
  int64_t nbins = 0, nchunks = 0, m = 0, mpad = 0;
  // Entries: bin b's (from bin_pos[b]) are the in-CSR's edges of its rows
  // regrouped by source chunk, in row order inside each (bin, chunk)
  // segment.  A run = the entries of one row in one segment piece; each run
  // is one partial sum (the gather pass sums it), numbered bin by bin from
  // pbin_pos[b].
  int64_t nps = 0, ntiles = 0, npieces = 0;
  int32_t* esrc = nullptr;       // mpad: the source of each entry; bit 31 = the entry closes its run
  double* psum = nullptr;        // nps: per-sweep scratch, the runs' partial sums
  uint16_t* vidx = nullptr;      // nps: per tile of runs, the tile index of the run at each sorted place
  uint16_t* skey = nullptr;      // nps: row offset (in the bin) at each sorted place of a tile; 0xFFFF = pad
  uint64_t* tile_meta = nullptr;  // ntiles: first run << 16 | runs of each tile
  std::vector<int64_t> tile_off;  // nbins + 1: first tile of each bin
  std::vector<int64_t> pbin_pos;  // nbins + 1: 8-aligned first run of each bin
  uint32_t* counts = nullptr;    // nchunks x nbins (chunk-major): entries of segment (bin, chunk)
  int64_t* start = nullptr;      // nchunks x nbins (chunk-major): first entry of segment (bin, chunk)
  uint32_t* seg_piece0 = nullptr;  // nchunks x nbins: the segment's first gather piece
  int64_t* pbase = nullptr;        // npieces: the first run of each piece
  // hot sources: per chunk up to kHot frequent sources whose entries read a
  // dense copy (hot_val[slot] = contribution of hot_src[slot], refreshed per wave)
  uint16_t* live_rows = nullptr;  // nbins << shift: per bin, its rows with in-edges (offsets)
  int32_t* live_cnt = nullptr;    // nbins
  int64_t nhot = 0;
  int32_t* hot_src = nullptr;
  double* hot_val = nullptr;
  std::vector<int64_t> bin_edge;  // nbins + 1: in-CSR edge offset of each bin's first row (waves)
  std::vector<int64_t> bin_pos;   // nbins + 1: 8-aligned entry position of each bin
  int64_t* bin_pos_d = nullptr;   // device copy
  double* bin_pairs = nullptr;   // nbins x (max, sum) residual of each bin's rows, reduced in bin order
  unsigned int* bin_done = nullptr;  // nbins: units of a split bin finished this sweep
  int p1_grid = 0, p2_grid = 0, acc_smem = 0;
  std::map<uint32_t, PbPlan> plans;  // by wave count
  std::vector<void*> allocs;
};
// Peer replicas a multi-GPU part's finalize also stores into (this part's
// slice in each peer's exchange vector; n = 0 on one GPU).
struct PbPeers {
  int n = 0;
  double* p[kMaxPeers] = {};
};
// Builds the layout from the resident in-CSR (duplicates and self loops kept
// exactly as the CSR holds them).  *msg set (no error) on bad geometry.
// nsrc: the source id space (n; nparts * slice for a multi-GPU part).
cudaError_t build_pb(const DevGraph& g, int64_t nsrc, int shift, int chunk_shift, cudaStream_t st, PbSet& pb,
                     const char** msg);
void free_pb(PbSet& pb, cudaStream_t st);
// First bin of each of (at most) S edge-balanced waves, from the bins' edge
// offsets (nbins + 1 values): S' + 1 values.
std::vector<int64_t> pb_wave_bins(const std::vector<int64_t>& bin_edge, uint32_t S);
// Edge offset of every 2^shift-row bin boundary of g (nbins + 1 values).
cudaError_t pb_bin_edges(const DevGraph& g, int shift, cudaStream_t st, std::vector<int64_t>* out);
// The plan for S waves, built on first use and cached in pb.plans.
cudaError_t get_pb_plan(PbSet& pb, uint32_t S, cudaStream_t st, const PbPlan** out);
// One propagation-blocked sweep: for each wave, gather from prev then
// finish the wave's rows into (pr, cur); residual into err/l1.  EC passes
// prev != cur with one wave; lockstep passes prev == cur (in place).
// Ranks are read from pr and written to pr_out (the same array except for a
// multi-GPU part's ping-pong); contributions go to cur (+ peers).
cudaError_t launch_pb_sweep(const PbSet& pb, const PbPlan& plan, const DevGraph& g, const double* prev,
                            const double* pr, double* pr_out, double* cur, const PbPeers& peers, double base,
                            double damping, double* err, double* l1, cudaStream_t st,
                            const unsigned int* gate = nullptr, bool skip_empty = false);

// runtime.cu hooks for mgpu.cu (the multi-device driver over the part API)
int set_error(int code, const std::string& msg);  // thread-local last error; returns code
cudaStream_t graph_stream(const void* graph_handle);
int graph_device(const void* graph_handle);
bool graph_uses_pb(const void* graph_handle);

}  // namespace fprb
