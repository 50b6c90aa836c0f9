/*
 * fpr_oracle.c -- CPU restatement of the reference hot path (TEST
 * INFRASTRUCTURE ONLY; see fpr_oracle.h).  Parity pinned against the compiled
 * reference via tests/golden/ (see tests/test_oracle.py).
 *
 * Build (oracle/Makefile): gcc -std=c11 -O3 -ffp-contract=off -fPIC -shared.
 * No -march: the reference's Release build has none, and FMA contraction of
 * `base + damping*sum` would change result bits.
 */
#include "fpr_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define GAMMA 0x9e3779b97f4a7c15ULL

static inline uint64_t mix64(uint64_t z) {
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

/* SplitMix64::next (rng.hpp:15-20) */
uint64_t fo_splitmix_next(uint64_t* state) {
  *state += GAMMA;
  return mix64(*state);
}

/* generate_rmat draw i (rmat.hpp:54-75): the root stream's (i+1)-th output
 * seeds the child (SplitMix64::split, rng.hpp:22); level l uses the child's
 * (l+1)-th output through next_unit (rng.hpp:25). */
void fo_rmat_draw(uint32_t scale, double a, double ab, double abc, uint64_t seed, uint64_t i,
                  uint64_t* src_out, uint64_t* dst_out) {
  uint64_t child = mix64(seed + (i + 1) * GAMMA);
  uint64_t src = 0, dst = 0;
  for (uint32_t level = 0; level < scale; ++level) {
    uint64_t z = mix64(child + (uint64_t)(level + 1) * GAMMA);
    double r = (double)(z >> 11) * 0x1.0p-53;
    src <<= 1;
    dst <<= 1;
    if (r < a) {
    } else if (r < ab) {
      dst |= 1;
    } else if (r < abc) {
      src |= 1;
    } else {
      src |= 1;
      dst |= 1;
    }
  }
  *src_out = src;
  *dst_out = dst;
}

/* generate_rmat (rmat.hpp:24-77), including validate(RmatParams). */
int fo_generate_rmat(uint32_t scale, uint64_t edge_factor, double a, double b, double c, double d,
                     uint64_t seed, uint64_t* src, uint64_t* dst) {
  if (scale == 0 || scale > 32) return FO_EINVAL;
  if (edge_factor == 0) return FO_EINVAL;
  if (a < 0 || b < 0 || c < 0 || d < 0 || fabs(a + b + c + d - 1.0) > 1e-9) return FO_EINVAL;
  const uint64_t draws = edge_factor << scale;
  const double ab = a + b, abc = a + b + c;
  for (uint64_t i = 0; i < draws; ++i) fo_rmat_draw(scale, a, ab, abc, seed, i, &src[i], &dst[i]);
  return FO_OK;
}

/* testutil::random_sparse (tests/test_util.hpp:49-58). */
uint64_t fo_random_sparse(uint64_t n, uint64_t avg_degree, uint64_t seed, uint64_t* src,
                          uint64_t* dst) {
  uint64_t state = seed, kept = 0;
  const uint64_t draws = n * avg_degree;
  for (uint64_t i = 0; i < draws; ++i) {
    uint64_t u = fo_splitmix_next(&state) % n;
    uint64_t v = fo_splitmix_next(&state) % n;
    if (u != v) {
      src[kept] = u;
      dst[kept] = v;
      ++kept;
    }
  }
  return kept;
}

/* LSD radix sort of 64-bit keys on the low `bits` bits, 11-bit digits. */
static int radix_sort_u64(uint64_t* keys, uint64_t count, unsigned bits) {
  if (count < 2 || bits == 0) return FO_OK;
  uint64_t* tmp = (uint64_t*)malloc(count * sizeof(uint64_t));
  if (!tmp) return FO_ENOMEM;
  uint64_t* in = keys;
  uint64_t* out = tmp;
  for (unsigned shift = 0; shift < bits; shift += 11) {
    uint64_t hist[2048];
    memset(hist, 0, sizeof(hist));
    for (uint64_t i = 0; i < count; ++i) hist[(in[i] >> shift) & 2047]++;
    uint64_t sum = 0;
    for (int b = 0; b < 2048; ++b) {
      uint64_t h = hist[b];
      hist[b] = sum;
      sum += h;
    }
    for (uint64_t i = 0; i < count; ++i) out[hist[(in[i] >> shift) & 2047]++] = in[i];
    uint64_t* t = in;
    in = out;
    out = t;
  }
  if (in != keys) memcpy(keys, in, count * sizeof(uint64_t));
  free(tmp);
  return FO_OK;
}

/* build_csr (graph.hpp:35-70): range check (:37-44), drop self-loops, sort
 * by (dst, src), dedup (:48-54), count + prefix sum (:63-68).  The sort key
 * packs (dst, src) as dst*2^k + src with k = bit width of n-1, so the
 * restatement handles n <= 2^32. */
int fo_build_csr(uint64_t n, uint64_t ne, const uint64_t* src, const uint64_t* dst,
                 uint64_t* in_start, uint64_t* in_src, uint64_t* out_degree, uint64_t* m_out,
                 uint64_t* bad_edge) {
  for (uint64_t i = 0; i < ne; ++i) {
    if (src[i] >= n || dst[i] >= n) {
      if (bad_edge) *bad_edge = i;
      return FO_EINVAL;
    }
  }
  if (n > (1ULL << 32)) return FO_ERANGE;
  unsigned k = 0;
  while (k < 64 && (1ULL << k) < n) ++k;
  uint64_t* keys = (uint64_t*)malloc((ne ? ne : 1) * sizeof(uint64_t));
  if (!keys) return FO_ENOMEM;
  uint64_t cnt = 0;
  for (uint64_t i = 0; i < ne; ++i)
    if (src[i] != dst[i]) keys[cnt++] = (dst[i] << k) | src[i];
  int rc = radix_sort_u64(keys, cnt, 2 * k);
  if (rc) {
    free(keys);
    return rc;
  }
  uint64_t m = 0;
  for (uint64_t i = 0; i < cnt; ++i)
    if (m == 0 || keys[i] != keys[m - 1]) keys[m++] = keys[i];
  const uint64_t mask = (k == 0) ? 0 : ((1ULL << k) - 1);
  memset(in_start, 0, (n + 1) * sizeof(uint64_t));
  memset(out_degree, 0, n * sizeof(uint64_t));
  for (uint64_t s = 0; s < m; ++s) {
    uint64_t d = keys[s] >> k, sr = keys[s] & mask;
    in_start[d + 1]++;
    in_src[s] = sr;
    out_degree[sr]++;
  }
  for (uint64_t u = 0; u < n; ++u) in_start[u + 1] += in_start[u];
  *m_out = m;
  free(keys);
  return FO_OK;
}

/* Config-3 relabel: sequential FIFO BFS over out-edges. */
int fo_bfs_relabel(uint64_t n, uint64_t m, const uint64_t* in_start, const uint64_t* in_src,
                   uint64_t root, uint64_t* new_id) {
  if (n == 0 || root >= n) return FO_EINVAL;
  uint64_t* out_start = (uint64_t*)calloc(n + 1, sizeof(uint64_t));
  uint64_t* out_dst = (uint64_t*)malloc((m ? m : 1) * sizeof(uint64_t));
  uint64_t* cursor = (uint64_t*)malloc(n * sizeof(uint64_t));
  uint64_t* queue = (uint64_t*)malloc(n * sizeof(uint64_t));
  if (!out_start || !out_dst || !cursor || !queue) {
    free(out_start); free(out_dst); free(cursor); free(queue);
    return FO_ENOMEM;
  }
  for (uint64_t e = 0; e < m; ++e) out_start[in_src[e] + 1]++;
  for (uint64_t u = 0; u < n; ++u) out_start[u + 1] += out_start[u];
  memcpy(cursor, out_start, n * sizeof(uint64_t));
  /* walking destinations ascending leaves every out-list ascending */
  for (uint64_t d = 0; d < n; ++d)
    for (uint64_t e = in_start[d]; e < in_start[d + 1]; ++e) out_dst[cursor[in_src[e]]++] = d;
  for (uint64_t u = 0; u < n; ++u) new_id[u] = UINT64_MAX;
  uint64_t head = 0, tail = 0, next = 0;
  queue[tail++] = root;
  new_id[root] = next++;
  while (head < tail) {
    const uint64_t u = queue[head++];
    for (uint64_t e = out_start[u]; e < out_start[u + 1]; ++e) {
      const uint64_t v = out_dst[e];
      if (new_id[v] == UINT64_MAX) {
        new_id[v] = next++;
        queue[tail++] = v;
      }
    }
  }
  for (uint64_t u = 0; u < n; ++u)
    if (new_id[u] == UINT64_MAX) new_id[u] = next++;
  free(out_start); free(out_dst); free(cursor); free(queue);
  return FO_OK;
}

/* Config-4 Chung-Lu.  Discrete power law P(k) ~ k^-alpha on
 * [1, kmax]: cdf[k-1] = (sum_{j<=k} j^-alpha) / Z, summed in ascending k. */
void fo_chunglu_cdf(double alpha, uint64_t kmax, double* cdf) {
  double z = 0.0;
  for (uint64_t k = 1; k <= kmax; ++k) z += pow((double)k, -alpha);
  double acc = 0.0;
  for (uint64_t k = 1; k <= kmax; ++k) {
    acc += pow((double)k, -alpha);
    cdf[k - 1] = acc / z;
  }
}

/* weight of vertex i: smallest k with u_i < cdf[k-1] (kmax if none), where
 * u_i = next_unit of SplitMix64(mix(seed + (i+1) gamma)). */
uint64_t fo_chunglu_weight(const double* cdf, uint64_t kmax, uint64_t seed, uint64_t i) {
  const uint64_t child = mix64(seed + (i + 1) * GAMMA);
  const double u = (double)(mix64(child + GAMMA) >> 11) * 0x1.0p-53;
  uint64_t lo = 0, hi = kmax;  /* first index with cdf > u */
  while (lo < hi) {
    const uint64_t mid = (lo + hi) >> 1;
    if (cdf[mid] > u) hi = mid; else lo = mid + 1;
  }
  return lo < kmax ? lo + 1 : kmax;
}

#define CL_SEED_DRAW 0x632be59bd9b4e019ULL
#define CL_SEED_PERM 0x9e6c63d0676a9a99ULL

static int cmp_u64pair(const void* a, const void* b) {
  const uint64_t* x = (const uint64_t*)a;
  const uint64_t* y = (const uint64_t*)b;
  if (x[0] != y[0]) return x[0] < y[0] ? -1 : 1;
  return x[1] < y[1] ? -1 : (x[1] > y[1]);
}

/* Draw j: r = mix(seed_d + (2j+1) gamma) % W for the source (+2 for the
 * destination), vertex = first i with inclusive prefix C_i > r; ids then go
 * through the permutation new = rank of (mix(seed_p + (i+1) gamma), i). */
int fo_generate_chunglu(uint64_t n, uint64_t draws, double alpha, uint64_t kmax, uint64_t seed,
                        uint64_t* src, uint64_t* dst) {
  if (n == 0 || kmax == 0 || !(alpha > 1.0)) return FO_EINVAL;
  double* cdf = (double*)malloc(kmax * sizeof(double));
  uint64_t* C = (uint64_t*)malloc(n * sizeof(uint64_t));
  uint64_t* kp = (uint64_t*)malloc(2 * n * sizeof(uint64_t));
  uint64_t* perm = (uint64_t*)malloc(n * sizeof(uint64_t));
  if (!cdf || !C || !kp || !perm) {
    free(cdf); free(C); free(kp); free(perm);
    return FO_ENOMEM;
  }
  fo_chunglu_cdf(alpha, kmax, cdf);
  uint64_t W = 0;
  for (uint64_t i = 0; i < n; ++i) {
    W += fo_chunglu_weight(cdf, kmax, seed, i);
    C[i] = W;
  }
  for (uint64_t i = 0; i < n; ++i) {
    kp[2 * i] = mix64(seed + CL_SEED_PERM + (i + 1) * GAMMA);
    kp[2 * i + 1] = i;
  }
  qsort(kp, n, 2 * sizeof(uint64_t), cmp_u64pair);
  for (uint64_t r = 0; r < n; ++r) perm[kp[2 * r + 1]] = r;
  const uint64_t sd = seed + CL_SEED_DRAW;
  for (uint64_t j = 0; j < draws; ++j) {
    for (int side = 0; side < 2; ++side) {
      const uint64_t r = mix64(sd + (2 * j + 1 + (uint64_t)side) * GAMMA) % W;
      uint64_t lo = 0, hi = n;
      while (lo < hi) {
        const uint64_t mid = (lo + hi) >> 1;
        if (C[mid] > r) hi = mid; else lo = mid + 1;
      }
      (side ? dst : src)[j] = perm[lo];
    }
  }
  free(cdf); free(C); free(kp); free(perm);
  return FO_OK;
}

/* validate(PageRankConfig) (pagerank.hpp:40-53) and init_ranks' n>0 check
 * (:55-57).  thread_count has no meaning here. */
static int check_config(uint64_t n, double damping, double threshold, uint64_t max_iterations) {
  if (!(damping > 0.0 && damping < 1.0)) return FO_EINVAL;
  if (!(threshold > 0.0)) return FO_EINVAL;
  if (max_iterations == 0) return FO_EINVAL;
  if (n == 0) return FO_EINVAL;
  return FO_OK;
}

static inline double norm_of(int norm, double mx, double sm) {
  return norm == FO_NORM_L1 ? sm : mx;
}

/* Pull restatement of pagerank_ec_seq (pagerank.hpp:126-145): the per-edge
 * scatter_contributions (:63-74) writes pr[u]/outdeg[u] into every slot of
 * u, so every slot of in_src[e] holds contrib[in_src[e]]; gather_ranks_jacobi
 * (:76-93) sums a dst segment left to right in ascending-src order.  Reading
 * contrib[in_src[e]] in the same order is bit-identical. */
int fo_pagerank_ec(uint64_t n, uint64_t m, const uint64_t* in_start, const uint64_t* in_src,
                   const uint64_t* out_degree, double damping, double threshold,
                   uint64_t max_iterations, int norm, double* ranks, double* errors,
                   double* l1_errors, uint64_t* iterations, double* history,
                   uint64_t history_cap) {
  (void)m;
  int rc = check_config(n, damping, threshold, max_iterations);
  if (rc) return rc;
  double* next = (double*)malloc(n * sizeof(double));
  double* contrib = (double*)malloc(n * sizeof(double));
  if (!next || !contrib) {
    free(next);
    free(contrib);
    return FO_ENOMEM;
  }
  for (uint64_t i = 0; i < n; ++i) ranks[i] = 1.0 / (double)n;
  const double base = (1.0 - damping) / (double)n;
  uint64_t it = 0;
  for (; it < max_iterations;) {
    for (uint64_t u = 0; u < n; ++u)
      contrib[u] = out_degree[u] ? ranks[u] / (double)out_degree[u] : 0.0;
    double err = 0.0, l1 = 0.0;
    for (uint64_t u = 0; u < n; ++u) {
      double sum = 0.0;
      for (uint64_t s = in_start[u]; s < in_start[u + 1]; ++s) sum += contrib[in_src[s]];
      const double value = base + damping * sum;
      next[u] = value;
      const double delta = fabs(value - ranks[u]);
      err = err > delta ? err : delta;
      l1 += delta;
    }
    memcpy(ranks, next, n * sizeof(double));
    errors[it] = err;
    if (l1_errors) l1_errors[it] = l1;
    if (history && it < history_cap) memcpy(history + it * n, ranks, n * sizeof(double));
    ++it;
    if (norm_of(norm, err, l1) <= threshold) break;
  }
  *iterations = it;
  free(next);
  free(contrib);
  return FO_OK;
}

/* One EC (Jacobi) iteration from an arbitrary rank vector: the body of the
 * pagerank_ec_seq loop (pagerank.hpp:137-140) -- scatter_contributions
 * (:63-74) of `prev`, then gather_ranks_jacobi (:76-93) into `next` -- in the
 * pull form of fo_pagerank_ec.  Rows are independent and each row's sum runs
 * left to right exactly as in the sequential loop, so splitting the rows over
 * OpenMP threads changes no bit of `next` or of the max delta (only the L1
 * delta's summation order).  For full-size one-step parity checks (configs
 * 3-5): the GPU's iterate k-1 goes in, the reference's iterate k comes out. */
int fo_ec_step(uint64_t n, const uint64_t* in_start, const uint64_t* in_src,
               const uint64_t* out_degree, double damping, const double* prev, double* next,
               double* err_out, double* l1_out) {
  if (n == 0 || !(damping > 0.0 && damping < 1.0)) return FO_EINVAL;
  double* contrib = (double*)malloc(n * sizeof(double));
  if (!contrib) return FO_ENOMEM;
  const double base = (1.0 - damping) / (double)n;
  const int64_t nn = (int64_t)n;
#pragma omp parallel for schedule(static)
  for (int64_t u = 0; u < nn; ++u)
    contrib[u] = out_degree[u] ? prev[u] / (double)out_degree[u] : 0.0;
  double err = 0.0, l1 = 0.0;
#pragma omp parallel for schedule(dynamic, 4096) reduction(max : err) reduction(+ : l1)
  for (int64_t u = 0; u < nn; ++u) {
    double sum = 0.0;
    for (uint64_t s = in_start[u]; s < in_start[u + 1]; ++s) sum += contrib[in_src[s]];
    const double value = base + damping * sum;
    next[u] = value;
    const double delta = fabs(value - prev[u]);
    err = err > delta ? err : delta;
    l1 += delta;
  }
  free(contrib);
  if (err_out) *err_out = err;
  if (l1_out) *l1_out = l1;
  return FO_OK;
}

/* Pull restatement of pagerank_fused_seq (pagerank.hpp:152-189): one initial
 * scatter (:164), then per vertex in ascending order gather the live
 * contributions, update in place and republish immediately (:166-183). */
int fo_pagerank_fused_seq(uint64_t n, uint64_t m, const uint64_t* in_start,
                          const uint64_t* in_src, const uint64_t* out_degree, double damping,
                          double threshold, uint64_t max_iterations, int norm, double* ranks,
                          double* errors, double* l1_errors, uint64_t* iterations,
                          double* history, uint64_t history_cap) {
  (void)m;
  int rc = check_config(n, damping, threshold, max_iterations);
  if (rc) return rc;
  double* contrib = (double*)malloc(n * sizeof(double));
  if (!contrib) return FO_ENOMEM;
  for (uint64_t i = 0; i < n; ++i) ranks[i] = 1.0 / (double)n;
  const double base = (1.0 - damping) / (double)n;
  for (uint64_t u = 0; u < n; ++u)
    contrib[u] = out_degree[u] ? ranks[u] / (double)out_degree[u] : 0.0;
  uint64_t it = 0;
  for (; it < max_iterations;) {
    double err = 0.0, l1 = 0.0;
    for (uint64_t u = 0; u < n; ++u) {
      double sum = 0.0;
      for (uint64_t s = in_start[u]; s < in_start[u + 1]; ++s) sum += contrib[in_src[s]];
      const double value = base + damping * sum;
      const double delta = fabs(value - ranks[u]);
      ranks[u] = value;
      if (out_degree[u] > 0) contrib[u] = value / (double)out_degree[u];
      err = err > delta ? err : delta;
      l1 += delta;
    }
    errors[it] = err;
    if (l1_errors) l1_errors[it] = l1;
    if (history && it < history_cap) memcpy(history + it * n, ranks, n * sizeof(double));
    ++it;
    if (norm_of(norm, err, l1) <= threshold) break;
  }
  *iterations = it;
  free(contrib);
  return FO_OK;
}

/* The GPU fused engine's deterministic schedule (see header).  With one
 * vertex per wave it is exactly fo_pagerank_fused_seq; with one wave it is
 * exactly fo_pagerank_ec. */
int fo_pagerank_lockstep(uint64_t n, uint64_t m, const uint64_t* in_start,
                         const uint64_t* in_src, const uint64_t* out_degree, double damping,
                         double threshold, uint64_t max_iterations, int norm, uint64_t nwaves,
                         const uint64_t* wave_start, double* ranks, double* errors,
                         double* l1_errors, uint64_t* iterations, double* history,
                         uint64_t history_cap) {
  (void)m;
  int rc = check_config(n, damping, threshold, max_iterations);
  if (rc) return rc;
  if (nwaves == 0 || wave_start[0] != 0 || wave_start[nwaves] != n) return FO_EINVAL;
  for (uint64_t w = 0; w < nwaves; ++w)
    if (wave_start[w + 1] < wave_start[w]) return FO_EINVAL;
  double* contrib = (double*)malloc(n * sizeof(double));
  double* wave_val = (double*)malloc(n * sizeof(double));
  if (!contrib || !wave_val) {
    free(contrib);
    free(wave_val);
    return FO_ENOMEM;
  }
  for (uint64_t i = 0; i < n; ++i) ranks[i] = 1.0 / (double)n;
  const double base = (1.0 - damping) / (double)n;
  for (uint64_t u = 0; u < n; ++u)
    contrib[u] = out_degree[u] ? ranks[u] / (double)out_degree[u] : 0.0;
  uint64_t it = 0;
  for (; it < max_iterations;) {
    double err = 0.0, l1 = 0.0;
    for (uint64_t w = 0; w < nwaves; ++w) {
      const uint64_t lo = wave_start[w], hi = wave_start[w + 1];
      for (uint64_t u = lo; u < hi; ++u) {
        double sum = 0.0;
        for (uint64_t s = in_start[u]; s < in_start[u + 1]; ++s) sum += contrib[in_src[s]];
        wave_val[u] = base + damping * sum;
      }
      for (uint64_t u = lo; u < hi; ++u) {
        const double value = wave_val[u];
        const double delta = fabs(value - ranks[u]);
        ranks[u] = value;
        if (out_degree[u] > 0) contrib[u] = value / (double)out_degree[u];
        err = err > delta ? err : delta;
        l1 += delta;
      }
    }
    errors[it] = err;
    if (l1_errors) l1_errors[it] = l1;
    if (history && it < history_cap) memcpy(history + it * n, ranks, n * sizeof(double));
    ++it;
    if (norm_of(norm, err, l1) <= threshold) break;
  }
  *iterations = it;
  free(contrib);
  free(wave_val);
  return FO_OK;
}

/* pagerank_dense_oracle (pagerank.hpp:335-370). */
int fo_dense_oracle(uint64_t n, const uint64_t* in_start, const uint64_t* in_src,
                    const uint64_t* out_degree, double damping, double threshold,
                    uint64_t max_iterations, double* ranks) {
  int rc = check_config(n, damping, threshold, max_iterations);
  if (rc) return rc;
  if (n > 4096) return FO_EINVAL;
  double* matrix = (double*)calloc(n * n, sizeof(double));
  double* next = (double*)malloc(n * sizeof(double));
  if (!matrix || !next) {
    free(matrix);
    free(next);
    return FO_ENOMEM;
  }
  for (uint64_t u = 0; u < n; ++u)
    for (uint64_t s = in_start[u]; s < in_start[u + 1]; ++s) {
      const uint64_t v = in_src[s];
      matrix[u * n + v] = 1.0 / (double)out_degree[v];
    }
  const double base = (1.0 - damping) / (double)n;
  for (uint64_t i = 0; i < n; ++i) ranks[i] = 1.0 / (double)n;
  for (uint64_t it = 0; it < max_iterations; ++it) {
    double err = 0.0;
    for (uint64_t u = 0; u < n; ++u) {
      double sum = 0.0;
      const double* row = matrix + u * n;
      for (uint64_t v = 0; v < n; ++v) sum += row[v] * ranks[v];
      next[u] = base + damping * sum;
      const double d = fabs(next[u] - ranks[u]);
      err = err > d ? err : d;
    }
    memcpy(ranks, next, n * sizeof(double));
    if (err <= threshold) break;
  }
  free(matrix);
  free(next);
  return FO_OK;
}

/* l1_norm / linf_norm (metrics.hpp:54-75). */
double fo_l1_norm(uint64_t n, const double* a, const double* b) {
  double sum = 0.0;
  for (uint64_t i = 0; i < n; ++i) sum += fabs(a[i] - b[i]);
  return sum;
}

double fo_linf_norm(uint64_t n, const double* a, const double* b) {
  double worst = 0.0;
  for (uint64_t i = 0; i < n; ++i) {
    const double d = fabs(a[i] - b[i]);
    worst = worst > d ? worst : d;
  }
  return worst;
}

/* ------------------------------------------------------------------ ingest */
/* fpr::parse_edge_list (edge_list.hpp:39-80).  std::getline lines (split on
 * '\n', a final unterminated line counts); a line is skipped when empty, when
 * its FIRST byte is '#' or '%' (:50), or when it holds only " \t\r" (:51);
 * otherwise two tokens delimited by " \t\r" (:55-69), each parsed by
 * std::from_chars base 10 over the whole token (:25-30: digits only, no sign,
 * <= 2^64-1), then nothing but " \t\r" (:71-73).  Dense ids in
 * first-appearance order, src before dst (:41-45, :74-76): an open-addressing
 * table stands in for the unordered_map. */
typedef struct {
  uint64_t* key;
  uint64_t* val;
  unsigned char* used;
  uint64_t cap, size;
} fo_idmap;

static uint64_t fo_hash(uint64_t x) {
  x ^= x >> 33;
  x *= 0xff51afd7ed558ccdULL;
  x ^= x >> 33;
  return x;
}

static int fo_idmap_grow(fo_idmap* mp) {
  fo_idmap nw;
  nw.cap = mp->cap ? mp->cap * 2 : 1024;
  nw.size = mp->size;
  nw.key = (uint64_t*)malloc(nw.cap * sizeof(uint64_t));
  nw.val = (uint64_t*)malloc(nw.cap * sizeof(uint64_t));
  nw.used = (unsigned char*)calloc(nw.cap, 1);
  if (!nw.key || !nw.val || !nw.used) {
    free(nw.key);
    free(nw.val);
    free(nw.used);
    return FO_ENOMEM;
  }
  for (uint64_t i = 0; i < mp->cap; ++i) {
    if (!mp->used[i]) continue;
    uint64_t h = fo_hash(mp->key[i]) & (nw.cap - 1);
    while (nw.used[h]) h = (h + 1) & (nw.cap - 1);
    nw.used[h] = 1;
    nw.key[h] = mp->key[i];
    nw.val[h] = mp->val[i];
  }
  free(mp->key);
  free(mp->val);
  free(mp->used);
  *mp = nw;
  return FO_OK;
}

static int fo_dense_id(fo_idmap* mp, uint64_t raw, uint64_t* out) {
  if (2 * (mp->size + 1) > mp->cap && fo_idmap_grow(mp) != FO_OK) return FO_ENOMEM;
  uint64_t h = fo_hash(raw) & (mp->cap - 1);
  while (mp->used[h]) {
    if (mp->key[h] == raw) {
      *out = mp->val[h];
      return FO_OK;
    }
    h = (h + 1) & (mp->cap - 1);
  }
  mp->used[h] = 1;
  mp->key[h] = raw;
  mp->val[h] = mp->size;
  *out = mp->size++;
  return FO_OK;
}

static int fo_is_ws(char c) { return c == ' ' || c == '\t' || c == '\r'; }

int fo_parse_edge_list(const char* text, uint64_t len, uint64_t* n, uint64_t* m, uint64_t* edges,
                       uint64_t cap, uint64_t* err_line, int* err_kind, uint64_t* tok_off,
                       uint64_t* tok_len) {
  fo_idmap mp = {0, 0, 0, 0, 0};
  uint64_t line = 0, ne = 0, pos = 0;
  int rc = FO_OK;
  *err_line = 0;
  *err_kind = 0;
  *tok_off = *tok_len = 0;
  while (pos < len) {
    uint64_t b = pos, e = pos;
    while (e < len && text[e] != '\n') ++e;
    pos = e < len ? e + 1 : len;
    ++line;
    if (b == e || text[b] == '#' || text[b] == '%') continue;
    uint64_t i = b;
    while (i < e && fo_is_ws(text[i])) ++i;
    if (i == e) continue;
    uint64_t v[2];
    int kind = 0;
    for (int k = 0; k < 2 && !kind; ++k) {
      while (i < e && fo_is_ws(text[i])) ++i;
      if (i == e) {
        kind = 1;
        break;
      }
      const uint64_t s = i;
      while (i < e && !fo_is_ws(text[i])) ++i;
      uint64_t x = 0;
      for (uint64_t j = s; j < i; ++j) {
        const unsigned d = (unsigned)(unsigned char)text[j] - (unsigned)'0';
        if (d > 9u || x > (UINT64_MAX - d) / 10u) {
          kind = 2;
          *tok_off = s;
          *tok_len = i - s;
          break;
        }
        x = x * 10u + d;
      }
      v[k] = x;
    }
    if (!kind) {
      while (i < e && fo_is_ws(text[i])) ++i;
      if (i != e) kind = 3;
    }
    if (kind) {
      *err_line = line;
      *err_kind = kind;
      rc = FO_EPARSE;
      break;
    }
    uint64_t ds, dd;
    if (fo_dense_id(&mp, v[0], &ds) != FO_OK || fo_dense_id(&mp, v[1], &dd) != FO_OK) {
      rc = FO_ENOMEM;
      break;
    }
    if (edges && ne < cap) {
      edges[2 * ne] = ds;
      edges[2 * ne + 1] = dd;
    }
    ++ne;
  }
  *n = mp.size;
  *m = ne;
  free(mp.key);
  free(mp.val);
  free(mp.used);
  if (rc == FO_OK && edges && ne > cap) rc = FO_ERANGE;
  return rc;
}

