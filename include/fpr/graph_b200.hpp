// graph_b200.hpp -- C++ drop-in for fpr::build_csr (graph.hpp:35-70).
//
//   fpr::build_csr_b200(const EdgeSet&)   ~ fpr::build_csr(const EdgeSet&)
//
// The same fpr::Graph (duplicates and self-loops dropped, in-segments in
// ascending source order, out_degree counted from the survivors) and the same
// std::invalid_argument text for an out-of-range endpoint; the sort, dedup
// and degree scans run on the GPU (libfpr_b200.so).
#pragma once

#include <fpr/graph.hpp>

#include <stdexcept>
#include <string>
#include <vector>

#include "../fpr_b200.h"

namespace fpr {

inline Graph build_csr_b200(const EdgeSet& raw, const fpr_b200_options* opts = nullptr) {
  std::vector<std::uint64_t> src(raw.edges.size()), dst(raw.edges.size());
  for (std::size_t i = 0; i < raw.edges.size(); ++i) {
    src[i] = raw.edges[i].src;
    dst[i] = raw.edges[i].dst;
  }
  fpr_b200_graph* h = nullptr;
  int rc = fpr_b200_graph_from_edges(raw.n, raw.edges.size(), src.data(), dst.data(), opts, &h);
  if (rc != FPR_B200_OK) {
    const std::string msg = fpr_b200_last_error();
    if (rc == FPR_B200_EINVAL || rc == FPR_B200_ERANGE) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
  }
  std::uint64_t n = 0, m = 0;
  fpr_b200_graph_info(h, &n, &m, nullptr);
  Graph g;
  g.n = n;
  g.m = m;
  g.in_start.resize(n + 1);
  g.in_src.resize(m);
  g.out_degree.resize(n);
  rc = fpr_b200_graph_download_csr(h, g.in_start.data(), g.in_src.data(), g.out_degree.data());
  fpr_b200_graph_destroy(h);
  if (rc != FPR_B200_OK) throw std::runtime_error(fpr_b200_last_error());
  return g;
}

}  // namespace fpr
