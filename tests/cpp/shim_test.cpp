// The reference's hand-computed path cases (test_algorithms.cpp:51-122),
// written against the drop-in C++ shim exactly as a reference user would.
#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <numeric>
#include <stdexcept>
#include <string>

#include "tgx_b200/tgx.hpp"

using namespace tgx_b200;

static int failures = 0;
#define CHECK(c)                                                   \
  do {                                                             \
    if (!(c)) {                                                    \
      std::printf("FAIL %s:%d %s\n", __FILE__, __LINE__, #c);      \
      ++failures;                                                  \
    }                                                              \
  } while (0)

constexpr std::int64_t kInf = PathResult::kUnreachedMin;
constexpr std::int64_t kNegInf = PathResult::kUnreachedMax;

// What the reference CLI does with a graph (tools/tgx.cpp:125-182): pick the
// top-k out-degree sources through out_csr().degree(v), then run an
// algorithm per source and digest its labels. Written here against the shim
// to show those call sites compile and behave unchanged.
static std::vector<VertexId> top_sources(const TemporalGraph& g, std::size_t k) {
  std::vector<VertexId> ids(g.vertex_count());
  std::iota(ids.begin(), ids.end(), VertexId{0});
  k = std::min(k, ids.size());
  std::partial_sort(ids.begin(), ids.begin() + static_cast<std::ptrdiff_t>(k), ids.end(),
                    [&](VertexId a, VertexId b) {
                      const EdgeId da = g.out_csr().degree(a), db = g.out_csr().degree(b);
                      return da != db ? da > db : a < b;
                    });
  ids.resize(k);
  return ids;
}

static std::uint64_t digest_run(const TemporalGraph& g, const std::string& algo, VertexId s,
                                const QueryWindow& w, const AlgoOptions& o) {
  if (algo == "earliest-arrival") return digest_of(earliest_arrival(g, s, w, o).values);
  if (algo == "latest-departure") return digest_of(latest_departure(g, s, w, o).values);
  if (algo == "fastest") return digest_of(fastest_path(g, s, w, o).values);
  if (algo == "shortest-duration") return digest_of(shortest_duration(g, s, w, o).values);
  return digest_of(temporal_bfs(g, s, w, o).values);
}

int main() {
  {  // graph inspection (engine.hpp:35-44, types.hpp:98-108, tcsr.hpp:36-50)
    const std::vector<TemporalEdge> es{{0, 1, 5, 6, 1.0}, {0, 2, 1, 3, 1.0}, {0, 1, 1, 2, 1.0},
                                       {2, 1, 4, 9, 1.0}, {3, 0, 0, 1, 1.0}};
    const auto g = TemporalGraph::build(es, 4, true);
    const GraphMeta& m = g.meta();
    CHECK(m.n_v == 4 && m.n_e == 5 && m.directed);
    CHECK(m.degree(0, Direction::Out) == 3 && m.degree(1, Direction::In) == 3);
    CHECK(g.degree(2, Direction::Out) == 1 && g.degree(0, Direction::In) == 1);
    CHECK(g.out_csr().edge_count() == 5 && g.in_csr().vertex_count() == 4);
    CHECK(g.out_csr().offsets()[1] == 3 && g.csr(Direction::In).degree(1) == 3);
    // segment order (start, end, neighbor): vertex 0's out-edges by start
    CHECK(g.out_csr().start_at(0) == 1 && g.out_csr().start_at(2) == 5);
    CHECK(g.out_csr().neighbor_at(2) == 1 && g.in_csr().neighbor_at(0) == 3);
    CHECK(g.out_csr().neighbor_at(0) == 1 && g.out_csr().end_at(1) == 3);  // (1,2) before (1,3)
    const auto top = top_sources(g, 2);
    CHECK(top.size() == 2 && top[0] == 0 && top[1] == 2);
    const auto u = TemporalGraph::build(es, 4, false);  // undirected: n_e stays logical
    CHECK(u.meta().n_e == 5 && u.out_csr().edge_count() == 10 && !u.meta().directed);
    // one run per source and algorithm, digests equal to the direct calls
    AlgoOptions o;
    EdgeMapStats st;
    o.stats = &st;
    for (const char* algo : {"earliest-arrival", "latest-departure", "fastest",
                             "shortest-duration", "bfs"})
      for (VertexId s : top) {
        const std::uint64_t d = digest_run(g, algo, s, QueryWindow{0, 100}, o);
        CHECK(d == digest_run(g, algo, s, QueryWindow{0, 100}, AlgoOptions{}));
      }
    CHECK(st.index_decisions + st.scan_decisions > 0);  // one per vertex expansion
  }
  {  // earliest arrival: no edges
    const auto g = TemporalGraph::build({}, 4, true);
    const auto r = earliest_arrival(g, 1, QueryWindow{5, 50});
    CHECK(r.values[1] == 5);
    CHECK(r.values[0] == kInf && r.values[2] == kInf && r.values[3] == kInf);
  }
  {  // single contained edge arrives at its end
    const auto g = TemporalGraph::build({{0, 1, 3, 5, 1.0}}, 2, true);
    CHECK(earliest_arrival(g, 0, QueryWindow{0, 10}).values[1] == 5);
  }
  {  // strict ordering rejects an equal handoff, weak accepts it
    const auto g = TemporalGraph::build({{0, 1, 1, 3, 1.0}, {1, 2, 3, 4, 1.0}}, 3, true);
    AlgoOptions strict, weak;
    strict.ordering = Ordering::StrictlySucceeds;
    weak.ordering = Ordering::Succeeds;
    CHECK(earliest_arrival(g, 0, QueryWindow{}, strict).values[2] == kInf);
    CHECK(earliest_arrival(g, 0, QueryWindow{}, weak).values[2] == 4);
  }
  {  // source out of range
    const auto g = TemporalGraph::build({}, 2, true);
    bool thrown = false;
    try {
      earliest_arrival(g, 5, QueryWindow{});
    } catch (const std::out_of_range&) {
      thrown = true;
    }
    CHECK(thrown);
  }
  {  // window with t_a > t_b
    const auto g = TemporalGraph::build({}, 2, true);
    bool thrown = false;
    try {
      earliest_arrival(g, 0, QueryWindow{9, 3});
    } catch (const std::invalid_argument&) {
      thrown = true;
    }
    CHECK(thrown);
  }
  {  // latest departure
    const auto g0 = TemporalGraph::build({}, 3, true);
    const auto r0 = latest_departure(g0, 1, QueryWindow{2, 9});
    CHECK(r0.values[1] == 9);
    CHECK(r0.values[0] == kNegInf);
    const auto g = TemporalGraph::build({{0, 1, 3, 5, 1.0}}, 2, true);
    CHECK(latest_departure(g, 1, QueryWindow{0, 10}).values[0] == 3);
  }
  {  // fastest: two-hop beats the direct edge
    const auto g =
        TemporalGraph::build({{0, 1, 2, 6, 1.0}, {0, 2, 3, 4, 1.0}, {2, 1, 4, 5, 1.0}}, 3, true);
    AlgoOptions weak;
    weak.ordering = Ordering::Succeeds;
    CHECK(fastest_path(g, 0, QueryWindow{}, weak).values[1] == 2);
    const auto g0 = TemporalGraph::build({}, 3, true);
    const auto r = fastest_path(g0, 2, QueryWindow{});
    CHECK(r.values[2] == 0);
    CHECK(r.values[0] == kInf);
  }
  {  // shortest duration (test_algorithms.cpp:124-146)
    const auto g1 = TemporalGraph::build({{0, 1, 3, 5, 1.0}}, 2, true);
    CHECK(shortest_duration(g1, 0, QueryWindow{}).values[1] == 2);
    const auto g =
        TemporalGraph::build({{0, 1, 0, 4, 1.0}, {0, 2, 0, 1, 1.0}, {2, 1, 5, 7, 1.0}}, 3, true);
    CHECK(shortest_duration(g, 0, QueryWindow{}).values[1] == 3);
    AlgoOptions w;
    w.weighted = true;
    CHECK(shortest_duration(g, 0, QueryWindow{}, w).values[1] == 1);  // weights 1.0
    // weighted: the sum of edge weights (path_algorithms.cpp:196-258)
    const auto gw = TemporalGraph::build(
        {{0, 1, 0, 4, 7.0}, {0, 2, 0, 1, 1.0}, {2, 1, 5, 7, 2.0}}, 3, true);
    CHECK(shortest_duration(gw, 0, QueryWindow{}, w).values[1] == 3);
    CHECK(shortest_duration(gw, 0, QueryWindow{}).values[1] == 3);
    const auto gbad = TemporalGraph::build({{0, 1, 0, 4, 1.5}}, 2, true);
    bool thrown = false;
    try {
      shortest_duration(gbad, 0, QueryWindow{}, w);
    } catch (const std::invalid_argument&) {
      thrown = true;
    }
    CHECK(thrown);
  }
  {  // temporal BFS (test_algorithms.cpp:149-168)
    const auto g = TemporalGraph::build(
        {{0, 1, 1, 2, 1.0}, {1, 2, 3, 4, 1.0}, {2, 3, 5, 6, 1.0}}, 4, true);
    const auto r = temporal_bfs(g, 0, QueryWindow{});
    CHECK(r.values == (std::vector<std::int64_t>{0, 1, 2, 3}));
    const auto g2 = TemporalGraph::build(
        {{0, 1, 9, 10, 1.0}, {0, 2, 0, 1, 1.0}, {2, 1, 2, 3, 1.0}, {1, 3, 5, 6, 1.0}}, 4, true);
    const auto r2 = temporal_bfs(g2, 0, QueryWindow{});
    CHECK(r2.values[1] == 1);
    CHECK(r2.values[3] == 3);
  }
  {  // Overlaps gate (test_engine.cpp:223-243 as a path query)
    const auto g = TemporalGraph::build({{0, 1, 2, 6, 1.0},
                                         {1, 2, 4, 9, 1.0},
                                         {1, 3, 7, 9, 1.0},
                                         {1, 4, 2, 8, 1.0},
                                         {1, 5, 3, 5, 1.0}},
                                        6, true);
    AlgoOptions ov;
    ov.ordering = Ordering::Overlaps;
    const auto r = earliest_arrival(g, 0, QueryWindow{}, ov);
    CHECK(r.values[2] == 9);
    CHECK(r.values[3] == kInf && r.values[4] == kInf && r.values[5] == kInf);
  }
  {  // edge validation (types.cpp:41-54)
    bool thrown = false;
    try {
      TemporalGraph::build({{0, 7, 1, 2, 1.0}}, 2, true);
    } catch (const std::out_of_range&) {
      thrown = true;
    }
    CHECK(thrown);
  }
  {  // views share the device graph (tgxd_graph_view)
    std::vector<TemporalEdge> es{{0, 1, 1, 2, 1.0}, {1, 2, 3, 4, 1.0}};
    const auto g = TemporalGraph::build(es, 3, true);
    const auto v = g.view(2);
    CHECK(earliest_arrival(v, 0, QueryWindow{}).values == earliest_arrival(g, 0, QueryWindow{}).values);
  }
  {  // selective-index cost model (selective_index.cpp:98-235)
    std::vector<TemporalEdge> es;
    for (std::uint64_t i = 0; i < 20; ++i) es.push_back({0, static_cast<VertexId>(1 + i % 3), 10 * i, 10 * i + 5, 1.0});
    EngineConfig cfg;
    cfg.index_cutoff = 8;
    const auto g = TemporalGraph::build(es, 4, true, cfg);
    const QueryWindow w{0, 1000};
    const AccessDecision a = choose_access_method(0, g, Direction::Out, w);
    CHECK(a.method == AccessMethod::Scan && a.k_hat == 20.0 && a.beta_hat == 1.0);
    CHECK(count_in_window(g, 0, Direction::Out, QueryWindow{10, 34}) == 2);
    const AccessDecision b = choose_access_method(1, g, Direction::Out, w);
    CHECK(b.beta_hat == -1.0 && b.k_hat == -1.0);
    const CostModelParams p = fit_cost_constants({{16, 0, 4.0, 16.0}});
    CHECK(p.c == 1.0 && p.c_prime == 1.0);
    bool thrown = false;
    try {
      fit_cost_constants({});
    } catch (const std::invalid_argument&) {
      thrown = true;
    }
    CHECK(thrown);
  }
  if (failures) return 1;
  std::printf("shim ok\n");
  return 0;
}
