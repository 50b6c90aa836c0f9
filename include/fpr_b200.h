/*
 * fpr_b200.h -- C ABI of the B200-native FusEd-PageRank engines
 * (libfpr_b200.so, built from paper_2203_09284_b200/csrc/).
 *
 * The reference (/root/reference/proj/include/fpr) is a header-only C++20
 * library with no C ABI.  This header is what a foreign caller (ctypes, JNI,
 * cgo, or the C++ drop-in wrapper include/fpr/pagerank_b200.hpp) binds.  No
 * std:: or torch types cross it: plain pointers, sizes and PODs only.
 *
 * Entry point -> reference interface it replaces:
 *   fpr_b200_pagerank(view, FPR_B200_ENGINE_EC, ...)
 *        -> fpr::pagerank_ec_seq / pagerank_ec_par    (pagerank.hpp:128,147,195)
 *   fpr_b200_pagerank(view, FPR_B200_ENGINE_FUSED, ...)
 *        -> fpr::pagerank_fused_par                   (pagerank.hpp:261)
 *   fpr_b200_pagerank(view, FPR_B200_ENGINE_FUSED_LOCKSTEP, ...)
 *        -> fpr::pagerank_fused_seq-style deterministic schedule (pagerank.hpp:156)
 *   fpr_graph_view          -> fpr::Graph               (graph.hpp:20-30)
 *   fpr_config              -> fpr::PageRankConfig      (pagerank.hpp:17-22)
 *   fpr_b200_result + ranks/errors buffers
 *                           -> fpr::PageRankResult      (pagerank.hpp:24-38)
 *   fpr_b200_graph_generate -> fpr::generate_rmat + fpr::build_csr
 *                              (rmat.hpp:42, graph.hpp:35) and
 *                              testutil::random_sparse (tests/test_util.hpp:49)
 *   fpr_b200_graph_download_csr -> the fpr::Graph arrays of build_csr
 *   fpr_b200_graph_from_edges   -> fpr::build_csr(EdgeSet)  (graph.hpp:35-70)
 *   fpr_b200_parse_edge_list -> fpr::parse_edge_list     (edge_list.hpp:39-80)
 *   fpr_b200_graph_from_edge_list
 *                           -> fpr::build_csr(fpr::parse_edge_list(in))
 *
 * Errors: every function returns a status code; fpr_b200_last_error() gives
 * the thread-local message.  FPR_B200_EINVAL carries the reference's exact
 * std::invalid_argument text (pagerank.hpp:42-51,56,100; graph.hpp:39-43).
 * Non-convergence is not an error (converged = 0), as in the reference.
 *
 * Threading: calls are synchronous and blocking.  A graph handle is not
 * re-entrant; distinct handles are independent.  fpr_config.thread_count is
 * validated (must be > 0, as the reference requires) and otherwise ignored.
 */
#ifndef FPR_B200_H
#define FPR_B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define FPR_B200_OK 0
#define FPR_B200_EINVAL 1 /* bad argument; message = reference's text */
#define FPR_B200_ECUDA 2  /* CUDA runtime error or no usable device */
#define FPR_B200_ENCCL 3  /* collective error (multi-GPU path) */
#define FPR_B200_ENOMEM 4 /* device/host allocation failed */
#define FPR_B200_ERANGE 5 /* n >= 2^31 (int32 vertex ids) */
#define FPR_B200_EPARSE 6 /* fpr::ParseError (edge_list.hpp:17-21); see fpr_parse_error */

#define FPR_B200_ENGINE_EC 0             /* Jacobi, bit-deterministic */
#define FPR_B200_ENGINE_FUSED 1          /* block-asynchronous Gauss-Seidel */
#define FPR_B200_ENGINE_FUSED_LOCKSTEP 2 /* deterministic wave-lockstep GS */

#define FPR_B200_NORM_LINF 0 /* reference stop rule: max |delta| <= threshold */
#define FPR_B200_NORM_L1 1   /* sum |delta| <= threshold (BASELINE wording) */

#define FPR_B200_GEN_RMAT 0    /* fpr::generate_rmat (rmat.hpp:42-77) */
#define FPR_B200_GEN_UNIFORM 1 /* testutil::random_sparse (test_util.hpp:49-58) */
#define FPR_B200_GEN_CHUNGLU 2 /* config 4 (no reference generator) */

/* Borrowed view of an fpr::Graph (graph.hpp:20-30); host or pinned memory. */
typedef struct fpr_graph_view {
  uint64_t n;
  uint64_t m;
  const uint64_t* in_start;   /* n + 1 */
  const uint64_t* in_src;     /* m */
  const uint64_t* out_degree; /* n */
} fpr_graph_view;

/* fpr::PageRankConfig (pagerank.hpp:17-22). */
typedef struct fpr_config {
  double damping;          /* reference default 0.85 */
  double threshold;        /* reference default 1e-15 */
  uint64_t max_iterations; /* reference default 10000 */
  uint32_t thread_count;   /* validated, ignored on the GPU */
} fpr_config;

#define FPR_B200_OPT_REORDER 1u /* renumber vertices by descending out-degree inside
                                  the library (locality for contrib gathers); ranks
                                  and traces are reported in the caller's ids */
#define FPR_B200_OPT_REORDER_SOURCES 8u /* renumber inside the library so that the
                                  vertices with out-degree > 0 (the only ones whose
                                  contributions are ever read) come first, the
                                  caller's order otherwise kept: the gathered vector
                                  shrinks to the sources without losing a crawl
                                  order's locality; ranks and
                                  traces in the caller's ids.  OPT_REORDER wins if
                                  both are set */
#define FPR_B200_OPT_REORDER_BLOCKS 32u /* renumber by descending out-degree inside
                                  each block of 2^23 ids (the propagation-blocked
                                  sweep's source chunk): a chunk's hub
                                  contributions share cache lines, so more gathers
                                  hit L1, while the chunks keep their edges and the
                                  FusEd waves their order (for
                                  repeated solves: the renumbering costs a CSR
                                  rebuild at creation).  Ranks and traces in the
                                  caller's ids; OPT_REORDER wins if both are set */
/* Sweep kind.  By default the library picks it when the graph is created:
 * propagation-blocked sweeps (below) when the contribution vector (8 n bytes)
 * exceeds half the device's L2 -- configs 3-5, where the pull gathers start
 * missing L2 -- and the pull sweep otherwise.  The two flags force one kind. */
#define FPR_B200_OPT_PB 4u      /* EC and lockstep engines: propagation-blocked sweeps
                                  (bins of 2^13 rows, source chunks of 2^23;
                                  FPR_B200_PB_SHIFT / FPR_B200_PB_CHUNK_SHIFT override):
                                  two streaming passes instead of the random pull
                                  gather; row sums are exact
                                  fixed-point sums of fixed run partials, so runs are
                                  bit-reproducible.  Lockstep waves are then runs of
                                  whole bins (fpr_b200_graph_wave_starts reports
                                  them); FUSED runs that lockstep schedule too */
#define FPR_B200_OPT_PULL 16u   /* pull sweeps on every graph (no propagation blocking) */

typedef struct fpr_b200_options {
  int32_t device;       /* CUDA ordinal; -1 = current device */
  int32_t norm;         /* FPR_B200_NORM_* stop rule */
  uint32_t wave_count;  /* lockstep engine: waves per sweep (0 = auto) */
  uint32_t flags;       /* FPR_B200_OPT_* */
  void* stream;         /* cudaStream_t to run on; NULL = library stream */
  const int32_t* devices; /* multi-device solve: CUDA ordinal of each part (NULL = single device) */
  uint32_t ndevices;    /* number of parts; > 1 selects the multi-device path (fpr_b200_mgpu_*) */
  uint32_t reserved0;
} fpr_b200_options;

#define FPR_B200_SWEEP_PULL 0 /* fpr_b200_result.sweep: the pull sweep ran */
#define FPR_B200_SWEEP_PB 1   /* propagation-blocked sweeps ran */

typedef struct fpr_b200_result {
  uint64_t iterations;      /* == errors written (trace.iterations) */
  int32_t converged;        /* last error <= threshold (detail::finish) */
  int32_t sweep;            /* FPR_B200_SWEEP_* actually used */
  double final_error;       /* last error, 1.0 if none (RankVector::final_error) */
  double solve_ms;          /* device time of the convergence loop (CUDA events) */
  double setup_ms;          /* rank/contribution initialisation kernel time */
  uint64_t kernel_launches; /* library kernels launched by this call */
} fpr_b200_result;

typedef struct fpr_gen_params {
  int32_t kind;          /* FPR_B200_GEN_* */
  uint32_t scale;        /* rmat: n = 2^scale */
  uint64_t edge_factor;  /* rmat: draws = edge_factor * n */
  double a, b, c, d;     /* rmat quadrant probabilities */
  uint64_t n;            /* uniform / chung-lu: vertices */
  uint64_t avg_degree;   /* uniform: draws = n * avg_degree */
  uint64_t seed;
  uint64_t draws;        /* chung-lu: edge draws */
  double alpha;          /* chung-lu: power-law exponent (> 1) */
  uint64_t kmax;         /* chung-lu: max weight (min is 1) */
  int32_t relabel_bfs;   /* 1: relabel vertices in BFS order (config 3) */
  int32_t reserved0;
  uint64_t bfs_root;     /* BFS root (old id) */
} fpr_gen_params;

typedef struct fpr_b200_graph fpr_b200_graph;

void fpr_b200_options_init(fpr_b200_options* opts);
void fpr_b200_config_init(fpr_config* cfg); /* reference defaults */
const char* fpr_b200_last_error(void);
int fpr_b200_version(void);

/* Copies + narrows a host fpr::Graph to the device (u64 -> int64 offsets,
 * int32 ids, range-checked) and builds the merge-path task partition. */
int fpr_b200_graph_create(const fpr_graph_view* view, const fpr_b200_options* opts,
                          fpr_b200_graph** out);
/* Generates + normalises a graph on the device, bit-identical to
 * build_csr(generate_rmat(p)) / build_csr(random_sparse(...)). */
int fpr_b200_graph_generate(const fpr_gen_params* params, const fpr_b200_options* opts,
                            fpr_b200_graph** out);
/* The generator's EdgeSet before build_csr, in generation order: the draws of
 * fpr::generate_rmat (rmat.hpp:42-77; self-loops and duplicates kept) or of
 * testutil::random_sparse (test_util.hpp:49-58; self-loops skipped).  Drawn
 * on the device.  *count_out = edges; src/dst (cap entries each, or NULL to
 * count only) receive them, ERANGE when cap is smaller. */
int fpr_b200_generate_edges(const fpr_gen_params* params, const fpr_b200_options* opts, uint64_t* src,
                            uint64_t* dst, uint64_t cap, uint64_t* count_out);
/* fpr::build_csr(EdgeSet{n, edges}) (graph.hpp:35-70) on the device: m edges
 * as two u64 arrays (host or pinned memory).  EINVAL names the first edge
 * with an endpoint outside [0, n), in build_csr's words. */
int fpr_b200_graph_from_edges(uint64_t n, uint64_t m, const uint64_t* src, const uint64_t* dst,
                              const fpr_b200_options* opts, fpr_b200_graph** out);
void fpr_b200_graph_destroy(fpr_b200_graph* g);
/* Lockstep engine: waves per sweep for later runs (0 = auto). */
int fpr_b200_graph_set_wave_count(fpr_b200_graph* g, uint32_t wave_count);
int fpr_b200_graph_info(const fpr_b200_graph* g, uint64_t* n, uint64_t* m, uint64_t* ntasks);
/* The propagation-blocked layout of g (built by its first PB solve): runs
 * (one partial sum per row and segment piece, incl. pad places), gather
 * pieces, accumulate tiles; all 0 while no layout exists.  *sweep is the
 * sweep kind the graph uses (FPR_B200_SWEEP_*).  Instrumentation for the
 * roofline (bench.py), not part of the reference interface. */
int fpr_b200_graph_layout_info(const fpr_b200_graph* g, int* sweep, uint64_t* runs, uint64_t* pieces,
                               uint64_t* tiles);
/* Downloads the CSR as fpr::Graph arrays (u64).  EINVAL for a graph created
 * with FPR_B200_OPT_REORDER (its resident CSR is in internal ids). */
int fpr_b200_graph_download_csr(const fpr_b200_graph* g, uint64_t* in_start, uint64_t* in_src,
                                uint64_t* out_degree);
/* Checks build_csr's invariants on the device (graph.hpp:20-30): *flags = 0
 * when offsets are monotone (row[0]=0, row[n]=m), ids in range, no
 * self-loops, sources strictly ascending per row, out-degrees consistent. */
int fpr_b200_graph_validate(fpr_b200_graph* g, uint32_t* flags);

/* Config-3 crawl order of a resident graph: new_id[old] (n entries) of the
 * BFS from `root` over out-edges, neighbours ascending, unreached vertices
 * appended in ascending id (the definition fo_bfs_relabel restates). */
int fpr_b200_graph_bfs_order(fpr_b200_graph* g, uint64_t root, uint64_t* new_id);

/* Vertex boundaries of the lockstep engine's waves for wave_count (0 = auto):
 * writes *nwaves and wave_start[0..*nwaves] (capacity cap). */
int fpr_b200_graph_wave_starts(fpr_b200_graph* g, uint32_t wave_count, uint64_t* wave_start,
                               uint64_t cap, uint64_t* nwaves);

/* Runs one engine to convergence on a resident graph.  ranks_out (n doubles),
 * errors_out / l1_errors_out (errors_cap doubles, per-iteration max / sum of
 * |delta|) and iter_ns_out (per-iteration device ns) are host buffers or NULL
 * (results stay on the device).  Returns FPR_B200_EINVAL if errors_out is
 * non-NULL and errors_cap < iterations actually run. */
int fpr_b200_run(fpr_b200_graph* g, int engine, const fpr_config* cfg, double* ranks_out,
                 double* errors_out, double* l1_errors_out, uint64_t* iter_ns_out,
                 uint64_t errors_cap, fpr_b200_result* result);
/* Device pointer of the rank vector left by the last run (n doubles). */
const double* fpr_b200_graph_ranks_device(const fpr_b200_graph* g);

/* ---- multi-GPU destination-range partitioning -------------
 * Part r of nparts owns rows [bounds[r], bounds[r+1]) (edge-balanced merge-
 * path split) with its in-edges; source ids are remapped into a padded
 * exchange space of nparts*slice doubles (part(s)*slice + s - bounds[part(s)])
 * so each iteration's exchange is ONE equal-size all-gather (NCCL over
 * NVLink), plus an all-reduce of the (max, sum) residual pair.  The caller
 * owns the exchange vectors (device memory, nparts*slice doubles) and the
 * collectives (paper_2203_09284_b200/dist.py). */
int fpr_b200_graph_partition(const fpr_b200_graph* full, uint32_t nparts, uint32_t part,
                             const fpr_b200_options* opts, uint64_t* bounds_out,
                             uint64_t* slice_out, fpr_b200_graph** out);
int fpr_b200_part_info(const fpr_b200_graph* g, uint64_t* n_global, uint64_t* row_begin,
                       uint64_t* slice, uint32_t* nparts, uint32_t* part);
/* pr = 1/n_global for the part's rows; their contributions into exchange's slice. */
/* Part `part` of `nparts` straight from a host view: the same destination-
 * range bounds and slice as fpr_b200_graph_partition (computed on the host),
 * but only this part's rows, in-edges and out-degrees are uploaded -- each
 * rank of a multi-GPU job moves ~1/nparts of the graph over its own link. */
int fpr_b200_part_create(const fpr_graph_view* view, uint32_t nparts, uint32_t part,
                         const fpr_b200_options* opts, uint64_t* bounds_out, uint64_t* slice_out,
                         fpr_b200_graph** out);
int fpr_b200_part_init(fpr_b200_graph* g, double* exchange);
/* One sweep on the part's stream, reading sources through exch_read and
 * writing the part's contributions into exch_write's slice (EC: distinct
 * vectors; FUSED: the same vector, in place).  pair_out (device, 2 doubles)
 * receives this part's (max |delta|, sum |delta|).  Does not synchronise. */
int fpr_b200_part_sweep(fpr_b200_graph* g, int engine, const fpr_config* cfg,
                        const double* exch_read, double* exch_write, double* pair_out);
int fpr_b200_part_ranks(fpr_b200_graph* g, double* ranks_out);
/* The part's ranks one sweep before the latest (a speculative driver that ran
 * one sweep past the stopping iteration reports these). */
int fpr_b200_part_ranks_prev(fpr_b200_graph* g, double* ranks_out);

/* Fused exchange: part_sweep whose epilogue also stores every updated
 * contribution into the other parts' exchange vectors -- peer_write[q] is
 * part q's write vector (base of the whole padded exchange space) mapped into
 * this device (fpr_b200_ipc_import for another process/GPU; a plain device
 * pointer within one process), peer_write[part] is ignored, npeer_bufs must
 * equal nparts (<= 8).  The sweep thereby performs the all-gather over NVLink
 * P2P stores, tile by tile as rows finalize; only the 16-B residual pair is
 * left for a collective, and that collective doubles as the barrier.  Rows
 * without in-edges (constant contribution) are sent only in the first 3
 * sweeps after fpr_b200_part_init: a driver may rotate through up to 3
 * exchange vectors. */
int fpr_b200_part_sweep_peers(fpr_b200_graph* g, int engine, const fpr_config* cfg,
                              const double* exch_read, double* exch_write,
                              double* const* peer_write, uint32_t npeer_bufs, double* pair_out);

/* ---- device-side stop rule (multi-GPU drivers) -------------
 * The reference's parallel engines reduce the per-thread residuals and apply
 * `error <= threshold` in the barrier's completion step (pagerank.hpp:209-218,
 * :276-286).  A multi-GPU driver that does this on the host pays a device ->
 * host round trip per iteration.  A gate moves the rule onto the device: it
 * is fpr_b200_gate_bytes(trace_cap) bytes of device memory holding the
 * iteration count, a stop flag and the (max, sum) residual trace.
 *   * fpr_b200_part_set_gate binds a part to a gate: its sweeps become
 *     no-ops (nothing read or written) once the gate is stopped;
 *   * fpr_b200_gate_update, enqueued after an iteration's residual pairs are
 *     in place (all parts' pairs: pointers on `device` or peer-mapped), adds
 *     the iteration to the trace and sets the stop flag when the reference's
 *     predicate holds or max_iterations is reached;
 * so a driver enqueues a batch of iterations -- sweep, pair exchange, gate
 * update -- and reads the gate once per batch (fpr_b200_gate_read).  The
 * ranks after the stopping iteration k are fpr_b200_part_ranks_after(g, k). */
uint64_t fpr_b200_gate_bytes(uint64_t trace_cap);
int fpr_b200_gate_init(void* gate, uint64_t trace_cap, int device, void* stream);
int fpr_b200_gate_update(void* gate, const double* const* pairs, uint32_t npairs, const fpr_config* cfg, int norm,
                         int device, void* stream);
int fpr_b200_gate_read(const void* gate, int device, void* stream, uint64_t* iterations, int* stopped,
                       double* errors_out, double* l1_errors_out, uint64_t cap);
int fpr_b200_part_set_gate(fpr_b200_graph* g, const void* gate);
int fpr_b200_part_ranks_after(fpr_b200_graph* g, uint64_t sweeps, double* ranks_out);

/* CUDA IPC of exchange buffers between the per-GPU processes.  A handle is
 * the cudaIpcMemHandle of the allocation holding dev_ptr plus dev_ptr's
 * offset in it (buffers from caching allocators are sub-allocations). */
#define FPR_B200_IPC_HANDLE_BYTES 72
int fpr_b200_ipc_export(const void* dev_ptr, void* handle_out /* 72 B */);
int fpr_b200_ipc_import(const void* handle /* 72 B */, int device, void** dev_ptr_out);
int fpr_b200_ipc_close(void* dev_ptr);

/* ---- multi-device solve from ONE host thread (SURVEY §8(b) Threading) ----
 * The reference's parallel engines split the vertices into static blocks, one
 * per thread (pagerank.hpp:111-122 block_for, used by pagerank_ec_par :195 and
 * pagerank_fused_par :261).  Here the blocks are edge-balanced destination
 * ranges, one per device: with opts->ndevices = P > 1, part r of the graph
 * (rows [bounds[r], bounds[r+1]) and their in-edges) lives on
 * opts->devices[r] (entries may repeat: parts that share a GPU run on their
 * own streams, one after the other).  Each part's sweep stores every new
 * contribution into all parts' exchange vectors -- peer stores over NVLink
 * between distinct GPUs (peer access enabled at creation), plain stores
 * within one -- so the sweep IS the exchange; the calling thread then reduces
 * the parts' (max, sum) residual pairs in part order and applies the
 * reference's stop rule.  EC gives the single-device iteration count and
 * ranks within 1e-12; FUSED is block-asynchronous across parts, the
 * fused_par contract.  fpr_b200_pagerank() takes this path when
 * opts->ndevices > 1, so the C++ drop-in reaches P GPUs through its options. */
typedef struct fpr_b200_mgpu fpr_b200_mgpu;
int fpr_b200_mgpu_create(const fpr_graph_view* view, const fpr_b200_options* opts, fpr_b200_mgpu** out);
/* The same from a generator: every device generates the graph (the generators
 * are deterministic) and keeps only its parts. */
int fpr_b200_mgpu_generate(const fpr_gen_params* params, const fpr_b200_options* opts, fpr_b200_mgpu** out);
/* EC or FUSED to convergence; buffers as fpr_b200_run (ranks in global ids). */
int fpr_b200_mgpu_run(fpr_b200_mgpu* mg, int engine, const fpr_config* cfg, double* ranks_out,
                      double* errors_out, double* l1_errors_out, uint64_t errors_cap, fpr_b200_result* result);
/* n, m, parts and the row bounds (nparts + 1 entries; NULL allowed). */
int fpr_b200_mgpu_info(const fpr_b200_mgpu* mg, uint64_t* n, uint64_t* m, uint32_t* nparts, uint64_t* bounds);
void fpr_b200_mgpu_destroy(fpr_b200_mgpu* mg);

/* Edge-list text ingest (SNAP style, edge_list.hpp:33-80): '#'/'%' comment
 * lines and blank/whitespace-only lines skipped, every other line exactly two
 * decimal u64 tokens separated by ' ', '\t' or '\r'; ids compacted to [0, n)
 * in first-appearance order.  Parsing and compaction run on the device.
 * FPR_B200_EPARSE reports the reference's ParseError for the FIRST malformed
 * line: line = its 1-based number, message = ParseError::what(). */
#define FPR_B200_PARSE_TOKENS 1    /* "expected two integer tokens" */
#define FPR_B200_PARSE_BAD_TOKEN 2 /* "bad token '<token>'" (incl. u64 overflow) */
#define FPR_B200_PARSE_TRAILING 3  /* "trailing characters after edge" */
typedef struct fpr_parse_error {
  uint64_t line;       /* 1-based line number (ParseError::line_number); 0 = none */
  int32_t kind;         /* FPR_B200_PARSE_* ; 0 = none */
  uint32_t message_len; /* strlen(message) */
  char message[256];    /* ParseError::what() as a C string, truncated to 255 bytes */
} fpr_parse_error;

/* fpr::parse_edge_list: *n_out = EdgeSet::n, *m_out = edges.size().  When
 * edges_out is non-null it receives the m (src, dst) pairs in input order
 * (2*m u64); edges_cap (in edges) smaller than m returns FPR_B200_ERANGE
 * after setting *n_out / *m_out.  err may be null. */
int fpr_b200_parse_edge_list(const char* text, uint64_t len, const fpr_b200_options* opts,
                             uint64_t* n_out, uint64_t* m_out, uint64_t* edges_out,
                             uint64_t edges_cap, fpr_parse_error* err);
/* build_csr(parse_edge_list(text)) into a resident graph handle. */
int fpr_b200_graph_from_edge_list(const char* text, uint64_t len, const fpr_b200_options* opts,
                                  fpr_b200_graph** out, fpr_parse_error* err);

/* One-shot drop-in: create from host view, run, copy results, destroy. */
int fpr_b200_pagerank(const fpr_graph_view* view, int engine, const fpr_config* cfg,
                      const fpr_b200_options* opts, double* ranks_out, double* errors_out,
                      uint64_t errors_cap, fpr_b200_result* result);

#ifdef __cplusplus
}
#endif
#endif
