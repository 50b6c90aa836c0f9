// edge_list_b200.hpp -- C++ drop-in for fpr::parse_edge_list (edge_list.hpp:39-80).
//
//   fpr::parse_edge_list_b200(std::istream&)   ~ fpr::parse_edge_list(std::istream&)
//   fpr::parse_edge_list_b200(const char*, n)  ~ the same over an in-memory text
//
// Same EdgeSet (first-appearance id compaction, input edge order) and the same
// fpr::ParseError (line_number, what()) for the first malformed line; the
// tokenising and compaction run on the GPU (libfpr_b200.so).  A caller that
// already holds the text in pinned memory avoids the host staging copy.
#pragma once

#include <fpr/edge_list.hpp>

#include <istream>
#include <iterator>
#include <stdexcept>
#include <string>

#include "../fpr_b200.h"

namespace fpr {

inline EdgeSet parse_edge_list_b200(const char* text, std::uint64_t len,
                                    const fpr_b200_options* opts = nullptr) {
  std::uint64_t n = 0, m = 0;
  fpr_parse_error err{};
  EdgeSet es;
  // one device pass with an upper bound of one edge per 4 bytes ("1 2\n")
  std::vector<std::uint64_t> flat(2 * ((len + 3) / 4 + 1));
  int rc = fpr_b200_parse_edge_list(text, len, opts, &n, &m, flat.data(), flat.size() / 2, &err);
  if (rc == FPR_B200_EPARSE) {
    // ParseError(line, what) prepends "line L: " itself (edge_list.hpp:17-21);
    // the full text is fpr_b200_last_error() (err.message stops at 255 bytes)
    std::string what = fpr_b200_last_error();
    const std::string prefix = "line " + std::to_string(err.line) + ": ";
    if (what.compare(0, prefix.size(), prefix) == 0) what.erase(0, prefix.size());
    throw ParseError(err.line, what);
  }
  if (rc != FPR_B200_OK) {
    const std::string msg = fpr_b200_last_error();
    if (rc == FPR_B200_EINVAL || rc == FPR_B200_ERANGE) throw std::invalid_argument(msg);
    throw std::runtime_error(msg);
  }
  es.n = n;
  es.edges.resize(m);
  for (std::uint64_t i = 0; i < m; ++i) es.edges[i] = Edge{flat[2 * i], flat[2 * i + 1]};
  return es;
}

inline EdgeSet parse_edge_list_b200(std::istream& in, const fpr_b200_options* opts = nullptr) {
  const std::string text((std::istreambuf_iterator<char>(in)), std::istreambuf_iterator<char>());
  return parse_edge_list_b200(text.data(), text.size(), opts);
}

}  // namespace fpr
