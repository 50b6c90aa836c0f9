/*
 * fpr_oracle.h -- CPU restatement of the FusEd-PageRank reference hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker, never the product: only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load it.  The product path (libfpr_b200.so) has no CPU
 * fallback and never links this file.
 *
 * Every function restates a reference function of
 * /root/reference/proj/include/fpr (cited per function in fpr_oracle.c).
 * Parity is pinned: tests/test_oracle.py checks these functions bit-exactly
 * against golden vectors produced by the reference itself compiled here
 * (oracle/_ref/libfpr_ref.so, recipe oracle/Makefile, fixtures
 * tests/golden/, generator tests/golden/make_golden.py).
 */
#ifndef FPR_ORACLE_H
#define FPR_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* status codes (mirror include/fpr_b200.h) */
#define FO_OK 0
#define FO_EINVAL 1
#define FO_ENOMEM 4
#define FO_ERANGE 5

#define FO_NORM_LINF 0 /* reference stop rule: max |delta| (pagerank.hpp:90) */
#define FO_NORM_L1 1   /* BASELINE.json wording: sum |delta| */

uint64_t fo_splitmix_next(uint64_t* state);

/* R-MAT edge draw i of generate_rmat (rmat.hpp:42-77), O(1) indexable. */
void fo_rmat_draw(uint32_t scale, double a, double ab, double abc, uint64_t seed, uint64_t i,
                  uint64_t* src, uint64_t* dst);
int fo_generate_rmat(uint32_t scale, uint64_t edge_factor, double a, double b, double c, double d,
                     uint64_t seed, uint64_t* src, uint64_t* dst);
/* testutil::random_sparse (tests/test_util.hpp:49-58), dangling_free=false.
 * Writes up to n*avg_degree edges, returns the number kept (self-loops skipped). */
uint64_t fo_random_sparse(uint64_t n, uint64_t avg_degree, uint64_t seed, uint64_t* src,
                          uint64_t* dst);

/* build_csr (graph.hpp:35-70).  in_src must hold ne entries.  On an
 * out-of-range endpoint returns FO_EINVAL and sets *bad_edge. */
int fo_build_csr(uint64_t n, uint64_t ne, const uint64_t* src, const uint64_t* dst,
                 uint64_t* in_start, uint64_t* in_src, uint64_t* out_degree, uint64_t* m_out,
                 uint64_t* bad_edge);

/* BASELINE config 3's crawl-order relabel (defined in SURVEY.md §8(d); no
 * reference generator exists): BFS from `root` over OUT-edges of the
 * normalised graph, neighbours in ascending old id, FIFO order; unreached
 * vertices appended in ascending old id.  new_id[old] = discovery index. */
int fo_bfs_relabel(uint64_t n, uint64_t m, const uint64_t* in_start, const uint64_t* in_src,
                   uint64_t root, uint64_t* new_id);

/* BASELINE config 4's Chung-Lu graph (definition in DESIGN.md §4.1; no
 * reference generator exists).  cdf: kmax doubles; draws raw edges with the
 * permuted ids (self-loops/duplicates kept; build_csr removes them). */
void fo_chunglu_cdf(double alpha, uint64_t kmax, double* cdf);
uint64_t fo_chunglu_weight(const double* cdf, uint64_t kmax, uint64_t seed, uint64_t i);
int fo_generate_chunglu(uint64_t n, uint64_t draws, double alpha, uint64_t kmax, uint64_t seed,
                        uint64_t* src, uint64_t* dst);

/* Engines.  ranks: n doubles out.  errors / l1_errors: max_iterations
 * doubles (per-iteration max and sum of |delta|); l1_errors may be NULL.
 * history: NULL or (history_cap x n) doubles, receives the rank vector
 * after every iteration k < history_cap.  Returns FO_OK or FO_EINVAL. */
int fo_pagerank_ec(uint64_t n, uint64_t m, const uint64_t* in_start, const uint64_t* in_src,
                   const uint64_t* out_degree, double damping, double threshold,
                   uint64_t max_iterations, int norm, double* ranks, double* errors,
                   double* l1_errors, uint64_t* iterations, double* history,
                   uint64_t history_cap);

int fo_pagerank_fused_seq(uint64_t n, uint64_t m, const uint64_t* in_start,
                          const uint64_t* in_src, const uint64_t* out_degree, double damping,
                          double threshold, uint64_t max_iterations, int norm, double* ranks,
                          double* errors, double* l1_errors, uint64_t* iterations,
                          double* history, uint64_t history_cap);

/* Wave-lockstep block Gauss-Seidel: the schedule of the GPU's deterministic
 * fused engine.  Waves are the vertex ranges [wave_start[w], wave_start[w+1]),
 * processed in ascending order; a vertex of wave w reads current-sweep
 * contributions for sources < wave_start[w] and previous-sweep ones
 * otherwise.  nwaves=1 is Jacobi (EC); one vertex per wave is fused_seq. */
int fo_pagerank_lockstep(uint64_t n, uint64_t m, const uint64_t* in_start,
                         const uint64_t* in_src, const uint64_t* out_degree, double damping,
                         double threshold, uint64_t max_iterations, int norm, uint64_t nwaves,
                         const uint64_t* wave_start, double* ranks, double* errors,
                         double* l1_errors, uint64_t* iterations, double* history,
                         uint64_t history_cap);

/* pagerank_dense_oracle (pagerank.hpp:338-370).  n <= 4096. */
int fo_dense_oracle(uint64_t n, const uint64_t* in_start, const uint64_t* in_src,
                    const uint64_t* out_degree, double damping, double threshold,
                    uint64_t max_iterations, double* ranks);

double fo_l1_norm(uint64_t n, const double* a, const double* b);

/* fpr::parse_edge_list (edge_list.hpp:39-80) over a text buffer: n = distinct
 * ids, m = edge lines; edges (2*cap u64, may be NULL) receive the dense
 * (src, dst) pairs in input order.  FO_EPARSE: the first malformed line's
 * 1-based number, kind (1 tokens, 2 bad token, 3 trailing) and, for a bad
 * token, its byte range.  FO_ERANGE: edges != NULL and cap < m. */
#define FO_EPARSE 6
int fo_parse_edge_list(const char* text, uint64_t len, uint64_t* n, uint64_t* m, uint64_t* edges,
                       uint64_t cap, uint64_t* err_line, int* err_kind, uint64_t* tok_off,
                       uint64_t* tok_len);
double fo_linf_norm(uint64_t n, const double* a, const double* b);

/* One EC iteration from `prev` (the pagerank_ec_seq loop body,
 * pagerank.hpp:137-140), OpenMP over rows, bit-identical to the sequential
 * iteration; *err_out / *l1_out = max / sum of |next - prev|. */
int fo_ec_step(uint64_t n, const uint64_t* in_start, const uint64_t* in_src,
               const uint64_t* out_degree, double damping, const double* prev, double* next,
               double* err_out, double* l1_out);

#ifdef __cplusplus
}
#endif
#endif
