// ref_shim.cpp -- extern "C" shim over the UNMODIFIED reference headers
// (TEST INFRASTRUCTURE ONLY).  Compiled by oracle/Makefile against
// /root/reference/proj/include (+ proj/tests for testutil::random_sparse) with
// the reference's CMake Release flags (-std=c++20 -O3, no -march;
// proj/CMakeLists.txt:3-8) into oracle/_ref/libfpr_ref.so.  Nothing here
// restates the algorithm: every call goes straight into the reference.
// Used to generate tests/golden/ and as bench.py's cpu_baseline ("reference").
#include <chrono>
#include <cstdint>
#include <cstring>
#include <exception>
#include <string>

#include <sstream>

#include "fpr/edge_list.hpp"
#include "fpr/graph.hpp"
#include "fpr/graph_cache.hpp"
#include "fpr/layout.hpp"
#include "fpr/metrics.hpp"
#include "fpr/pagerank.hpp"
#include "fpr/rmat.hpp"
#include "test_util.hpp"

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

struct RefGraph {
  fpr::Graph g;
  fpr::EdgeCentricLayout layout;
};
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }
uint64_t ref_last_error_len(void) { return g_err.size(); }

int ref_generate_rmat(uint32_t scale, uint64_t ef, double a, double b, double c, double d,
                      uint64_t seed, uint64_t* src, uint64_t* dst) {
  return guarded([&] {
    fpr::RmatParams p;
    p.scale = scale;
    p.edge_factor = ef;
    p.a = a;
    p.b = b;
    p.c = c;
    p.d = d;
    p.seed = seed;
    fpr::EdgeSet es = fpr::generate_rmat(p);
    for (size_t i = 0; i < es.edges.size(); ++i) {
      src[i] = es.edges[i].src;
      dst[i] = es.edges[i].dst;
    }
  });
}

// testutil::random_sparse with a fresh SplitMix64(seed); returns kept count.
uint64_t ref_random_sparse(uint64_t n, uint64_t deg, uint64_t seed, uint64_t* src, uint64_t* dst) {
  fpr::SplitMix64 rng(seed);
  fpr::EdgeSet es = fpr::testutil::random_sparse(n, deg, rng);
  for (size_t i = 0; i < es.edges.size(); ++i) {
    src[i] = es.edges[i].src;
    dst[i] = es.edges[i].dst;
  }
  return es.edges.size();
}

int ref_build_csr(uint64_t n, uint64_t ne, const uint64_t* src, const uint64_t* dst,
                  uint64_t* in_start, uint64_t* in_src, uint64_t* out_degree, uint64_t* m_out) {
  return guarded([&] {
    fpr::EdgeSet es;
    es.n = n;
    es.edges.resize(ne);
    for (uint64_t i = 0; i < ne; ++i) es.edges[i] = {src[i], dst[i]};
    fpr::Graph g = fpr::build_csr(es);
    std::memcpy(in_start, g.in_start.data(), (n + 1) * sizeof(uint64_t));
    std::memcpy(in_src, g.in_src.data(), g.m * sizeof(uint64_t));
    std::memcpy(out_degree, g.out_degree.data(), n * sizeof(uint64_t));
    *m_out = g.m;
  });
}

// Graph + layout built once (build_layout excluded from engine timing).
void* ref_graph_create(uint64_t n, uint64_t m, const uint64_t* in_start, const uint64_t* in_src,
                       const uint64_t* out_degree) {
  auto* h = new RefGraph;
  h->g.n = n;
  h->g.m = m;
  h->g.in_start.assign(in_start, in_start + n + 1);
  h->g.in_src.assign(in_src, in_src + m);
  h->g.out_degree.assign(out_degree, out_degree + n);
  h->layout = fpr::build_layout(h->g);
  return h;
}

void ref_graph_destroy(void* h) { delete static_cast<RefGraph*>(h); }

// engine: 0 ec_seq, 1 fused_seq, 2 ec_par, 3 fused_par (metrics.hpp:14).
// errors: capacity max_iterations.  *seconds = wall time of the engine call.
int ref_graph_run(void* hp, int engine, double damping, double threshold, uint64_t max_iter,
                  unsigned threads, double* ranks, double* errors, uint64_t* iterations,
                  int* converged, double* final_error, double* seconds) {
  auto* h = static_cast<RefGraph*>(hp);
  return guarded([&] {
    fpr::PageRankConfig cfg;
    cfg.damping = damping;
    cfg.threshold = threshold;
    cfg.max_iterations = max_iter;
    cfg.thread_count = threads;
    fpr::PageRankResult r;
    auto t0 = std::chrono::steady_clock::now();
    switch (engine) {
      case 0: r = fpr::pagerank_ec_seq(h->g, h->layout, cfg); break;
      case 1: r = fpr::pagerank_fused_seq(h->g, h->layout, cfg); break;
      case 2: r = fpr::pagerank_ec_par(h->g, h->layout, cfg); break;
      case 3: r = fpr::pagerank_fused_par(h->g, h->layout, cfg); break;
      default: throw std::invalid_argument("ref_shim: unknown engine");
    }
    auto t1 = std::chrono::steady_clock::now();
    if (seconds) *seconds = std::chrono::duration<double>(t1 - t0).count();
    std::memcpy(ranks, r.ranks.values.data(), h->g.n * sizeof(double));
    std::memcpy(errors, r.trace.errors.data(), r.trace.errors.size() * sizeof(double));
    *iterations = r.trace.iterations;
    *converged = r.trace.converged ? 1 : 0;
    *final_error = r.ranks.final_error;
  });
}

int ref_dense_oracle(uint64_t n, uint64_t m, const uint64_t* in_start, const uint64_t* in_src,
                     const uint64_t* out_degree, double damping, double threshold,
                     uint64_t max_iter, double* ranks) {
  return guarded([&] {
    fpr::Graph g;
    g.n = n;
    g.m = m;
    g.in_start.assign(in_start, in_start + n + 1);
    g.in_src.assign(in_src, in_src + m);
    g.out_degree.assign(out_degree, out_degree + n);
    fpr::PageRankConfig cfg;
    cfg.damping = damping;
    cfg.threshold = threshold;
    cfg.max_iterations = max_iter;
    fpr::RankVector rv = fpr::pagerank_dense_oracle(g, cfg);
    std::memcpy(ranks, rv.values.data(), n * sizeof(double));
  });
}

// fpr::save_cache / load_cache (graph_cache.hpp:65-97) for format interop tests.
int ref_save_cache(uint64_t n, uint64_t m, const uint64_t* in_start, const uint64_t* in_src,
                   const uint64_t* out_degree, const char* path) {
  return guarded([&] {
    fpr::Graph g;
    g.n = n;
    g.m = m;
    g.in_start.assign(in_start, in_start + n + 1);
    g.in_src.assign(in_src, in_src + m);
    g.out_degree.assign(out_degree, out_degree + n);
    fpr::save_cache(g, path);
  });
}

// Returns 0 and fills *n, *m (arrays NULL) or the arrays (sized by a first call).
int ref_load_cache(const char* path, uint64_t* n, uint64_t* m, uint64_t* in_start,
                   uint64_t* in_src, uint64_t* out_degree) {
  return guarded([&] {
    fpr::Graph g = fpr::load_cache(path);
    *n = g.n;
    *m = g.m;
    if (in_start) std::memcpy(in_start, g.in_start.data(), (g.n + 1) * sizeof(uint64_t));
    if (in_src) std::memcpy(in_src, g.in_src.data(), g.m * sizeof(uint64_t));
    if (out_degree) std::memcpy(out_degree, g.out_degree.data(), g.n * sizeof(uint64_t));
  });
}

// fpr::parse_edge_list (edge_list.hpp:39-80) over a text buffer.  Returns 0
// with *n, *m and (when edges != NULL and cap >= m) the 2*m ids; 3 on
// fpr::ParseError with *line = line_number and ref_last_error() = what().
int ref_parse_edge_list(const char* text, uint64_t len, uint64_t* n, uint64_t* m, uint64_t* edges,
                        uint64_t cap, uint64_t* line) {
  *line = 0;
  try {
    std::istringstream in(std::string(text, len));
    fpr::EdgeSet es = fpr::parse_edge_list(in);
    *n = es.n;
    *m = es.edges.size();
    if (edges && es.edges.size() <= cap)
      for (size_t i = 0; i < es.edges.size(); ++i) {
        edges[2 * i] = es.edges[i].src;
        edges[2 * i + 1] = es.edges[i].dst;
      }
    return 0;
  } catch (const fpr::ParseError& e) {
    g_err = e.what();
    *line = e.line_number;
    return 3;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 2;
  }
}

}  // extern "C"
