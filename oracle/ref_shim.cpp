// TEST INFRASTRUCTURE ONLY — never linked into or called by the product.
//
// extern "C" wrapper around the UNMODIFIED reference library (`tgx`, compiled
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/). It lets
// the Python tests, the golden-vector script and bench.py's reference arm call
// the reference's own entry points through ctypes:
//   TemporalGraph::build           /root/reference/proj/include/tgx/engine.hpp:32-33
//   earliest_arrival / latest_departure / fastest_path / shortest_duration /
//   temporal_bfs                   /root/reference/proj/include/tgx/algorithms.hpp:46-66
//   oracle::enumerate_paths        /root/reference/proj/tests/support/oracle.hpp:27-29
//   set_workers / num_workers      /root/reference/proj/include/tgx/parallel.hpp:19-21
//   choose_access_method / fit_cost_constants / count_in_window
//                                  /root/reference/proj/include/tgx/selective_index.hpp:63-120,
//                                  /root/reference/proj/include/tgx/tcsr.hpp:72
// Exceptions are mapped to integer codes (1 out_of_range, 2 invalid_argument,
// 3 anything else) and the message is kept for tgxref_last_error().

#include <cstdint>
#include <cstring>
#include <exception>
#include <stdexcept>
#include <string>
#include <vector>

#include "support/oracle.hpp"
#include "tgx/algorithms.hpp"
#include "tgx/digest.hpp"
#include "tgx/engine.hpp"
#include "tgx/ingest.hpp"
#include "tgx/parallel.hpp"
#include "tgx/selective_index.hpp"

namespace {

thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
  try {
    f();
    return 0;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return 1;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

std::vector<tgx::TemporalEdge> edges_of(std::uint64_t m, const std::uint32_t* src,
                                        const std::uint32_t* dst, const std::uint64_t* start,
                                        const std::uint64_t* end,
                                        const double* weight = nullptr) {
  std::vector<tgx::TemporalEdge> edges(m);
  for (std::uint64_t i = 0; i < m; ++i) {
    edges[i] = tgx::TemporalEdge{src[i], dst[i], start[i], end[i], weight ? weight[i] : 1.0};
  }
  return edges;
}

tgx::Ordering ordering_of(int o) {
  switch (o) {
    case 0: return tgx::Ordering::Succeeds;
    case 2: return tgx::Ordering::Overlaps;
    default: return tgx::Ordering::StrictlySucceeds;
  }
}

}  // namespace

extern "C" {

const char* tgxref_last_error() { return g_err.c_str(); }

void tgxref_set_workers(int n) { tgx::set_workers(n); }
int tgxref_num_workers() { return tgx::num_workers(); }

int tgxref_build(std::uint32_t n, std::uint64_t m, const std::uint32_t* src,
                 const std::uint32_t* dst, const std::uint64_t* start, const std::uint64_t* end,
                 int directed, std::uint64_t index_cutoff, void** out) {
  *out = nullptr;
  return guarded([&] {
    tgx::EngineConfig cfg;
    if (index_cutoff != 0) cfg.index_cutoff = index_cutoff;
    auto* g = new tgx::TemporalGraph(
        tgx::TemporalGraph::build(edges_of(m, src, dst, start, end), n, directed != 0, cfg));
    *out = g;
  });
}

// Same, with per-edge weights (TemporalEdge::weight, types.hpp:29-40).
int tgxref_build_weighted(std::uint32_t n, std::uint64_t m, const std::uint32_t* src,
                          const std::uint32_t* dst, const std::uint64_t* start,
                          const std::uint64_t* end, const double* weight, int directed,
                          std::uint64_t index_cutoff, void** out) {
  *out = nullptr;
  return guarded([&] {
    tgx::EngineConfig cfg;
    if (index_cutoff != 0) cfg.index_cutoff = index_cutoff;
    auto* g = new tgx::TemporalGraph(tgx::TemporalGraph::build(
        edges_of(m, src, dst, start, end, weight), n, directed != 0, cfg));
    *out = g;
  });
}

void tgxref_free(void* g) { delete static_cast<tgx::TemporalGraph*>(g); }

// kind: 0 earliest arrival, 1 latest departure, 2 fastest, 3 shortest duration
// (unweighted), 4 temporal BFS, 5 shortest duration with AlgoOptions::weighted.
// force: -1 graph default, 0 auto, 1 index, 2 scan.
int tgxref_query(void* gp, int kind, std::uint32_t vertex, std::uint64_t ta, std::uint64_t tb,
                 int ordering, int force, std::int64_t* out) {
  return guarded([&] {
    const auto& g = *static_cast<const tgx::TemporalGraph*>(gp);
    tgx::AlgoOptions opts;
    opts.ordering = ordering_of(ordering);
    if (force >= 0) {
      opts.force_access = force == 1   ? tgx::ForceAccess::Index
                          : force == 2 ? tgx::ForceAccess::Scan
                                       : tgx::ForceAccess::Auto;
    }
    const tgx::QueryWindow w{ta, tb};
    tgx::PathResult r;
    switch (kind) {
      case 0: r = tgx::earliest_arrival(g, vertex, w, opts); break;
      case 1: r = tgx::latest_departure(g, vertex, w, opts); break;
      case 2: r = tgx::fastest_path(g, vertex, w, opts); break;
      case 3: r = tgx::shortest_duration(g, vertex, w, opts); break;
      case 4: r = tgx::temporal_bfs(g, vertex, w, opts); break;
      case 5:
        opts.weighted = true;
        r = tgx::shortest_duration(g, vertex, w, opts);
        break;
      default: throw std::invalid_argument("unknown query kind");
    }
    std::memcpy(out, r.values.data(), r.values.size() * sizeof(std::int64_t));
  });
}

// metric: 0 EA, 1 LD, 2 fastest, 3 shortest duration, 4 hops (oracle::PathMetric
// order, tests/support/oracle.hpp:19).
int tgxref_enumerate(std::uint32_t n, std::uint64_t m, const std::uint32_t* src,
                     const std::uint32_t* dst, const std::uint64_t* start,
                     const std::uint64_t* end, std::uint32_t vertex, std::uint64_t ta,
                     std::uint64_t tb, int ordering, int metric, std::int64_t* out) {
  return guarded([&] {
    const auto edges = edges_of(m, src, dst, start, end);
    const auto pm = static_cast<tgx::oracle::PathMetric>(metric);
    const tgx::PathResult r =
        tgx::oracle::enumerate_paths(edges, n, vertex, tgx::QueryWindow{ta, tb},
                                     ordering_of(ordering), pm);
    std::memcpy(out, r.values.data(), r.values.size() * sizeof(std::int64_t));
  });
}

// Edge-list IO (ingest.hpp): load into caller arrays of capacity `cap`
// (m and n_v are always reported; arrays are filled only when m <= cap).
int tgxref_load_edge_list(const char* path, int map_ids, std::uint64_t seed, std::uint64_t dmax,
                          std::uint64_t cap, std::uint64_t* m, std::uint32_t* n_v,
                          std::uint32_t* src, std::uint32_t* dst, std::uint64_t* start,
                          std::uint64_t* end, double* weight) {
  return guarded([&] {
    tgx::LoadOptions opt;
    opt.map_ids = map_ids != 0;
    opt.seed = seed;
    opt.end_sample_max = dmax;
    const tgx::LoadResult r = tgx::load_edge_list(path, opt);
    *m = r.edges.size();
    *n_v = r.meta.n_v;
    if (r.edges.size() > cap) return;
    for (std::size_t i = 0; i < r.edges.size(); ++i) {
      src[i] = r.edges[i].source;
      dst[i] = r.edges[i].destination;
      start[i] = r.edges[i].start;
      end[i] = r.edges[i].end;
      weight[i] = r.edges[i].weight;
    }
  });
}

int tgxref_write_edge_list(const char* path, std::uint64_t m, const std::uint32_t* src,
                           const std::uint32_t* dst, const std::uint64_t* start,
                           const std::uint64_t* end, const double* weight) {
  return guarded([&] {
    std::vector<tgx::TemporalEdge> e(m);
    for (std::uint64_t i = 0; i < m; ++i) e[i] = {src[i], dst[i], start[i], end[i], weight[i]};
    tgx::write_edge_list(path, e);
  });
}

int tgxref_sample_end_times(std::uint64_t m, const std::uint64_t* start, std::uint64_t seed,
                            std::uint64_t dmax, std::uint64_t* end) {
  return guarded([&] {
    std::vector<tgx::TemporalEdge> e(m);
    for (std::uint64_t i = 0; i < m; ++i) e[i] = {0, 0, start[i], start[i], 1.0};
    tgx::sample_end_times(e, seed, dmax);
    for (std::uint64_t i = 0; i < m; ++i) end[i] = e[i].end;
  });
}

int tgxref_window_for_recent_fraction(std::uint64_t m, const std::uint64_t* start,
                                      const std::uint64_t* end, double fraction,
                                      std::uint64_t* ta, std::uint64_t* tb) {
  return guarded([&] {
    std::vector<tgx::TemporalEdge> e(m);
    for (std::uint64_t i = 0; i < m; ++i) e[i] = {0, 0, start[i], end[i], 1.0};
    const tgx::QueryWindow w = tgx::window_for_recent_fraction(e, fraction);
    *ta = w.t_a;
    *tb = w.t_b;
  });
}

std::uint64_t tgxref_digest(const std::int64_t* values, std::uint64_t n) {
  return tgx::digest_of(std::span<const std::int64_t>(values, n));
}


// Selective-index cost model: decision (0 index lookup, 1 scan), beta_hat,
// k_hat and count_in_window for k (vertex, window) pairs of one direction.
int tgxref_access_decisions(void* gp, int dir, std::uint64_t k, const std::uint32_t* verts,
                            const std::uint64_t* ta, const std::uint64_t* tb, double theta,
                            std::int32_t* method, double* beta, double* khat,
                            std::uint64_t* matches) {
  return guarded([&] {
    const auto& g = *static_cast<const tgx::TemporalGraph*>(gp);
    const tgx::Direction d = dir == 0 ? tgx::Direction::Out : tgx::Direction::In;
    tgx::CostModelParams p;
    p.theta_sel = theta;
    for (std::uint64_t i = 0; i < k; ++i) {
      const tgx::QueryWindow w{ta[i], tb[i]};
      const tgx::AccessDecision a = tgx::choose_access_method(verts[i], g.registry(), d, w, p);
      method[i] = a.method == tgx::AccessMethod::IndexLookup ? 0 : 1;
      beta[i] = a.beta_hat;
      khat[i] = a.k_hat;
      matches[i] = g.csr(d).count_in_window(verts[i], w);
    }
  });
}

int tgxref_fit_cost_constants(std::uint64_t k, const std::uint64_t* degree,
                              const std::uint64_t* matches, const double* index_s,
                              const double* scan_s, double theta, double* out) {
  return guarded([&] {
    std::vector<tgx::CalibrationPoint> pts(k);
    for (std::uint64_t i = 0; i < k; ++i) pts[i] = {degree[i], matches[i], index_s[i], scan_s[i]};
    const tgx::CostModelParams p = tgx::fit_cost_constants(pts, theta);
    out[0] = p.c;
    out[1] = p.c_prime;
    out[2] = p.theta_sel;
  });
}
}  // extern "C"
