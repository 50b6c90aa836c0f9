// Drop-in test: a reference-shaped call site (the reference's own generator,
// build_csr, build_layout and engines) swapping in the B200 engines by name.
// Built by tests/cpp/Makefile against /root/reference/proj/include in the build
// container; the binary travels to the GPU box (tests/test_gpu_dropin.py).
#include <cmath>
#include <cstdio>
#include <stdexcept>
#include <string>

#include <sstream>

#include "fpr/edge_list_b200.hpp"
#include "fpr/graph_b200.hpp"
#include "fpr/metrics.hpp"
#include "fpr/pagerank_b200.hpp"
#include "fpr/rmat.hpp"

static int failures = 0;
#define CHECK(cond, ...)                       \
  do {                                         \
    if (!(cond)) {                             \
      std::printf("FAIL %s:%d ", __FILE__, __LINE__); \
      std::printf(__VA_ARGS__);                \
      std::printf("\n");                       \
      ++failures;                              \
    }                                          \
  } while (0)

static double max_rel(const std::vector<double>& a, const std::vector<double>& b) {
  double w = 0;
  for (size_t i = 0; i < a.size(); ++i) w = std::max(w, std::abs(a[i] - b[i]) / std::abs(b[i]));
  return w;
}

int main() {
  fpr::RmatParams p;
  p.scale = 12;
  p.edge_factor = 16;
  p.seed = 7;
  const fpr::Graph g = fpr::build_csr(fpr::generate_rmat(p));
  fpr::EdgeCentricLayout layout = fpr::build_layout(g);
  fpr::PageRankConfig cfg;
  cfg.threshold = 1e-10;

  const fpr::PageRankResult ref = fpr::pagerank_ec_seq(g, layout, cfg);
  const fpr::PageRankResult gpu = fpr::pagerank_ec_b200(g, layout, cfg);
  CHECK(gpu.trace.iterations == ref.trace.iterations, "iterations %llu vs %llu",
        (unsigned long long)gpu.trace.iterations, (unsigned long long)ref.trace.iterations);
  CHECK(gpu.trace.converged && gpu.trace.errors.size() == gpu.trace.iterations, "trace shape");
  CHECK(max_rel(gpu.ranks.values, ref.ranks.values) <= 1e-12, "ec rel err %.3e",
        max_rel(gpu.ranks.values, ref.ranks.values));

  // the same call site with a device list: three parts driven from this
  // thread (all on device 0 here; distinct GPUs in production)
  {
    int32_t devs[3] = {0, 0, 0};
    fpr_b200_options o;
    fpr_b200_options_init(&o);
    o.devices = devs;
    o.ndevices = 3;
    const fpr::PageRankResult mg = fpr::pagerank_ec_b200(g, layout, cfg, o);
    CHECK(mg.trace.iterations == ref.trace.iterations, "multi-device iterations %llu vs %llu",
          (unsigned long long)mg.trace.iterations, (unsigned long long)ref.trace.iterations);
    CHECK(max_rel(mg.ranks.values, ref.ranks.values) <= 1e-12, "multi-device rel err %.3e",
          max_rel(mg.ranks.values, ref.ranks.values));
  }

  fpr::PageRankConfig tight = cfg;
  tight.threshold = 1e-13;
  const fpr::PageRankResult fref = fpr::pagerank_fused_seq(g, layout, tight);
  const fpr::PageRankResult fgpu = fpr::pagerank_fused_b200(g, layout, tight);
  CHECK(fpr::l1_norm(fgpu.ranks, fref.ranks) <= 1e-9, "fused L1 %.3e",
        fpr::l1_norm(fgpu.ranks, fref.ranks));

  // reference error behaviour, thrown before any device work
  fpr::PageRankConfig bad = cfg;
  bad.damping = 1.5;
  try {
    fpr::pagerank_ec_b200(g, layout, bad);
    CHECK(false, "no throw for damping");
  } catch (const std::invalid_argument& e) {
    CHECK(std::string(e.what()) == "pagerank: damping must be in (0,1)", "msg '%s'", e.what());
  }
  fpr::EdgeCentricLayout wrong;
  try {
    fpr::pagerank_ec_b200(g, wrong, cfg);
    CHECK(false, "no throw for layout");
  } catch (const std::invalid_argument& e) {
    CHECK(std::string(e.what()) == "pagerank: layout does not match graph", "msg '%s'", e.what());
  }
  fpr::PageRankConfig capped = cfg;
  capped.threshold = 1e-15;
  capped.max_iterations = 3;
  const fpr::PageRankResult nc = fpr::pagerank_ec_b200(g, capped);
  CHECK(nc.trace.iterations == 3 && !nc.trace.converged, "non-convergence is a result");

  // build_csr on the device vs the reference's build_csr (graph.hpp:35-70)
  {
    const fpr::EdgeSet raw = fpr::generate_rmat(p);
    const fpr::Graph a = fpr::build_csr(raw), b = fpr::build_csr_b200(raw);
    CHECK(a.n == b.n && a.m == b.m && a.in_start == b.in_start && a.in_src == b.in_src &&
              a.out_degree == b.out_degree,
          "build_csr_b200 differs (m %llu vs %llu)", (unsigned long long)a.m, (unsigned long long)b.m);
    fpr::EdgeSet bad{2, {{0, 1}, {0, 2}}};
    std::string want, got;
    try {
      fpr::build_csr(bad);
    } catch (const std::invalid_argument& e) {
      want = e.what();
    }
    try {
      fpr::build_csr_b200(bad);
    } catch (const std::invalid_argument& e) {
      got = e.what();
    }
    CHECK(!want.empty() && want == got, "build_csr error '%s' vs '%s'", want.c_str(), got.c_str());
  }

  // edge-list ingest: the reference's parse_edge_list vs the device parser
  {
    std::ostringstream text;
    fpr::write_edge_list(text, fpr::generate_rmat(p), {"drop-in ingest"});
    std::string t = text.str() + "% tail comment\r\n\n  \t\n77777777777 5\n";
    std::istringstream a(t), b(t);
    const fpr::EdgeSet ea = fpr::parse_edge_list(a);
    const fpr::EdgeSet eb = fpr::parse_edge_list_b200(b);
    CHECK(ea == eb, "EdgeSet differs (n %llu vs %llu, m %zu vs %zu)", (unsigned long long)ea.n,
          (unsigned long long)eb.n, ea.edges.size(), eb.edges.size());
    CHECK(fpr::build_csr(ea).in_src == fpr::build_csr(eb).in_src, "build_csr differs");
    const std::string badtext = t + "1 2 3\n4 x\n";
    std::string want, got;
    std::uint64_t wl = 0, gl = 0;
    try {
      std::istringstream in(badtext);
      fpr::parse_edge_list(in);
    } catch (const fpr::ParseError& e) {
      want = e.what();
      wl = e.line_number;
    }
    try {
      std::istringstream in(badtext);
      fpr::parse_edge_list_b200(in);
    } catch (const fpr::ParseError& e) {
      got = e.what();
      gl = e.line_number;
    }
    CHECK(wl > 0 && wl == gl && want == got, "ParseError '%s'@%llu vs '%s'@%llu", want.c_str(),
          (unsigned long long)wl, got.c_str(), (unsigned long long)gl);
  }

  std::printf("%s: ec %llu it, fused %llu it (ref fused_seq %llu)\n", failures ? "FAILED" : "OK",
              (unsigned long long)gpu.trace.iterations, (unsigned long long)fgpu.trace.iterations,
              (unsigned long long)fref.trace.iterations);
  return failures ? 1 : 0;
}
