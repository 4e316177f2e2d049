// The reference's hand-computed path cases (test_algorithms.cpp:51-122),
// written against the drop-in C++ shim exactly as a reference user would.
#include <cstdio>
#include <cstdlib>
#include <stdexcept>

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

int main() {
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
    bool thrown = false;
    AlgoOptions w;
    w.weighted = true;
    try {
      shortest_duration(g, 0, QueryWindow{}, w);
    } catch (const std::domain_error&) {
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
    for (std::uint64_t i = 0; i < 20; ++i) es.push_back({0, 1 + i % 3, 10 * i, 10 * i + 5, 1.0});
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
