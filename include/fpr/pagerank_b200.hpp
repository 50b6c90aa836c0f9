// pagerank_b200.hpp -- C++ drop-in for the reference's engine entry points.
//
// Include AFTER (or instead of) the reference's <fpr/pagerank.hpp>; it pulls
// that header in itself, so the reference's own types are used unchanged:
// fpr::Graph (graph.hpp:20-30), fpr::EdgeCentricLayout (layout.hpp:18-22),
// fpr::PageRankConfig / PageRankResult (pagerank.hpp:17-38).
//
//   fpr::pagerank_ec_b200(g, layout, cfg)      ~ pagerank_ec_seq / ec_par (pagerank.hpp:128,195)
//   fpr::pagerank_ec_b200(g, cfg)              ~ pagerank_ec_seq(g, cfg)   (pagerank.hpp:147)
//   fpr::pagerank_fused_b200(g, layout, cfg)   ~ pagerank_fused_par        (pagerank.hpp:261)
//   fpr::pagerank_fused_lockstep_b200(...)     ~ deterministic GS schedule  (pagerank.hpp:156)
//
// With FPR_B200_AS_PAR defined before inclusion, call sites written against
// the reference's parallel engines (fpr::pagerank_ec_par / pagerank_fused_par)
// compile to the GPU engines with no source edits.
//
// Semantics kept from the reference: validate(cfg) and require_layout run on
// the host before any device work and throw std::invalid_argument with the
// reference's messages; non-convergence returns converged=false; the trace
// holds every iteration's max delta.  The layout is validated, not read: the
// GPU engines use the pull formulation.  Link: -lfpr_b200
// (paper_2203_09284_b200/libfpr_b200.so).
#pragma once

#include <fpr/pagerank.hpp>

#include <stdexcept>
#include <string>
#include <vector>

#include "../fpr_b200.h"

namespace fpr {
namespace b200 {

inline void throw_status(int rc) {
  if (rc == FPR_B200_OK) return;
  const std::string msg = fpr_b200_last_error();
  if (rc == FPR_B200_EINVAL || rc == FPR_B200_ERANGE) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// Uploads g, runs `engine`, returns the reference-shaped result.
inline PageRankResult run(const Graph& g, int engine, const PageRankConfig& cfg,
                          const fpr_b200_options* opts = nullptr) {
  validate(cfg);                          // pagerank.hpp:40-53, same messages
  RankVector ranks = init_ranks(g.n);     // n == 0 throws as the reference does (:56)
  fpr_graph_view view{g.n, g.m, g.in_start.data(), g.in_src.data(), g.out_degree.data()};
  fpr_config c{cfg.damping, cfg.threshold, cfg.max_iterations, cfg.thread_count};
  PageRankResult result{std::move(ranks), {}};
  const std::uint64_t cap = cfg.max_iterations < (1ull << 24) ? cfg.max_iterations : (1ull << 24);
  std::vector<double> errors(cap);
  fpr_b200_result r{};
  throw_status(fpr_b200_pagerank(&view, engine, &c, opts, result.ranks.values.data(),
                                 errors.data(), cap, &r));
  errors.resize(r.iterations);
  result.trace.errors = std::move(errors);
  detail::finish(result, cfg.threshold);  // iterations/converged/final_error (:104-109)
  return result;
}

}  // namespace b200

inline PageRankResult pagerank_ec_b200(const Graph& g, EdgeCentricLayout& layout,
                                       const PageRankConfig& cfg) {
  validate(cfg);
  detail::require_layout(g, layout);
  return b200::run(g, FPR_B200_ENGINE_EC, cfg);
}

inline PageRankResult pagerank_ec_b200(const Graph& g, const PageRankConfig& cfg) {
  return b200::run(g, FPR_B200_ENGINE_EC, cfg);
}

inline PageRankResult pagerank_fused_b200(const Graph& g, EdgeCentricLayout& layout,
                                          const PageRankConfig& cfg) {
  validate(cfg);
  detail::require_layout(g, layout);
  return b200::run(g, FPR_B200_ENGINE_FUSED, cfg);
}

inline PageRankResult pagerank_fused_b200(const Graph& g, const PageRankConfig& cfg) {
  return b200::run(g, FPR_B200_ENGINE_FUSED, cfg);
}

// With library options: a device list (opts.devices / ndevices > 1) runs the
// multi-device solve from this thread (the reference's thread fan-out,
// pagerank.hpp:111-122, moved to GPUs); flags force a sweep kind.
inline PageRankResult pagerank_ec_b200(const Graph& g, EdgeCentricLayout& layout, const PageRankConfig& cfg,
                                       const fpr_b200_options& opts) {
  validate(cfg);
  detail::require_layout(g, layout);
  return b200::run(g, FPR_B200_ENGINE_EC, cfg, &opts);
}

inline PageRankResult pagerank_fused_b200(const Graph& g, EdgeCentricLayout& layout, const PageRankConfig& cfg,
                                          const fpr_b200_options& opts) {
  validate(cfg);
  detail::require_layout(g, layout);
  return b200::run(g, FPR_B200_ENGINE_FUSED, cfg, &opts);
}

inline PageRankResult pagerank_fused_lockstep_b200(const Graph& g, EdgeCentricLayout& layout,
                                                   const PageRankConfig& cfg) {
  validate(cfg);
  detail::require_layout(g, layout);
  return b200::run(g, FPR_B200_ENGINE_FUSED_LOCKSTEP, cfg);
}

}  // namespace fpr

#ifdef FPR_B200_AS_PAR
#define pagerank_ec_par pagerank_ec_b200
#define pagerank_fused_par pagerank_fused_b200
#endif
