// tgx_b200 — C++ drop-in for the reference's traversal entry points.
//
// Header-only shim over the C-ABI (include/tgxd.h, libtgxd.so). It keeps the
// reference signatures and semantics (/root/reference/proj/include/tgx/):
//   TemporalGraph::build(edges, n_v, directed, config)   engine.hpp:32-33
//   TemporalGraph::meta / degree / csr / out_csr / in_csr engine.hpp:35-44
//     (GraphMeta types.hpp:98-108; TemporalCsr read access tcsr.hpp:36-50,
//     materialized on the host from the device layout on first use)
//   earliest_arrival / latest_departure / fastest_path    algorithms.hpp:46-58
//   shortest_duration / temporal_bfs                      algorithms.hpp:62-67
//   PathResult (int64 values, INT64_MAX / INT64_MIN)       algorithms.hpp:16-21
//   digest_of                                             digest.hpp:42-52
// and re-throws the reference's exception types: std::out_of_range for a bad
// vertex or edge, std::invalid_argument for a bad window or (weighted
// shortest duration) a reachable edge whose weight is not a non-negative
// integer. Every ordering, Overlaps included, runs on the device. Times
// outside [0, 2^31 - 2] raise std::domain_error; there is no CPU fallback.
// force_access is accepted and ignored: results are access-invariant
// (test_algorithms.cpp:196-217). EdgeMapStats counts one access decision per
// vertex expansion (engine.hpp:316, 341): index_decisions for expansions that
// went through the selective index, scan_decisions for the others.
//
// A user of the reference switches by replacing `#include "tgx/..."` and
// `tgx::` with this header and `tgx_b200::`, and linking libtgxd.so.
#pragma once

#include <algorithm>
#include <cmath>
#include <numeric>
#include <cstdint>
#include <limits>
#include <memory>
#include <mutex>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../tgxd.h"

namespace tgx_b200 {

using Timestamp = std::uint64_t;
using VertexId = std::uint32_t;
using EdgeId = std::uint64_t;
inline constexpr Timestamp kMaxTimestamp = std::numeric_limits<Timestamp>::max();

struct TemporalEdge {
  VertexId source = 0;
  VertexId destination = 0;
  Timestamp start = 0;
  Timestamp end = 0;
  double weight = 1.0;
};

struct QueryWindow {
  Timestamp t_a = 0;
  Timestamp t_b = kMaxTimestamp;
  bool valid() const { return t_a <= t_b; }
};

enum class Ordering { Succeeds, StrictlySucceeds, Overlaps };
enum class ForceAccess { Auto, Index, Scan };
enum class Direction { Out, In };

struct GraphMeta {  // types.hpp:98-108
  VertexId n_v = 0;
  EdgeId n_e = 0;  // logical edge count (undirected: before symmetrization)
  bool directed = true;
  std::vector<EdgeId> out_degree;
  std::vector<EdgeId> in_degree;
  EdgeId degree(VertexId v, Direction d) const {
    return d == Direction::Out ? out_degree[v] : in_degree[v];
  }
};

struct EngineConfig {
  EdgeId index_cutoff = 2048;
  Ordering ordering = Ordering::StrictlySucceeds;
  ForceAccess force_access = ForceAccess::Auto;
};

struct EdgeMapStats {
  std::uint64_t index_decisions = 0;
  std::uint64_t scan_decisions = 0;
};

struct AlgoOptions {
  std::optional<Ordering> ordering;
  std::optional<ForceAccess> force_access;
  EdgeMapStats* stats = nullptr;
  bool weighted = false;  // shortest_duration only
};

struct PathResult {
  static constexpr std::int64_t kUnreachedMin = std::numeric_limits<std::int64_t>::max();
  static constexpr std::int64_t kUnreachedMax = std::numeric_limits<std::int64_t>::min();
  std::vector<std::int64_t> values;
};

namespace detail {
[[noreturn]] inline void raise(int code) {
  const std::string msg = tgxd_last_error();
  switch (code) {
    case TGXD_ERR_VERTEX_RANGE:
    case TGXD_ERR_EDGE:
      throw std::out_of_range(msg);
    case TGXD_ERR_WINDOW:
      throw std::invalid_argument(msg);
    case TGXD_ERR_TIME_RANGE:
    case TGXD_ERR_UNSUPPORTED:
      throw std::domain_error(msg);
    default:
      throw std::runtime_error(msg);
  }
}
inline void check(int code) {
  if (code != TGXD_OK) raise(code);
}
}  // namespace detail

// Host view of one device T-CSR layout (tcsr.hpp:27-85 read access):
// offsets and degrees from the device degrees, the edge arrays (segment
// order: start, end, neighbor) copied from the device on first use.
class TemporalCsr {
 public:
  VertexId vertex_count() const { return n_; }
  EdgeId edge_count() const { return offsets_.empty() ? 0 : offsets_.back(); }
  EdgeId degree(VertexId v) const { return offsets_[v + 1] - offsets_[v]; }
  std::span<const EdgeId> offsets() const { return offsets_; }
  std::span<const VertexId> neighbors() const { return edges().nbr; }
  std::span<const Timestamp> starts() const { return edges().st; }
  std::span<const Timestamp> ends() const { return edges().en; }
  VertexId neighbor_at(EdgeId i) const { return edges().nbr[i]; }
  Timestamp start_at(EdgeId i) const { return edges().st[i]; }
  Timestamp end_at(EdgeId i) const { return edges().en[i]; }

 private:
  friend class TemporalGraph;
  struct Edges {
    std::vector<VertexId> nbr;
    std::vector<Timestamp> st, en;
  };
  const Edges& edges() const {
    std::call_once(*once_, [this] {
      const EdgeId m = edge_count();
      std::vector<std::uint32_t> s(m), d(m);
      Edges e;
      e.st.resize(m);
      e.en.resize(m);
      if (m)
        detail::check(tgxd_graph_flatten(h_.get(), dir_ == Direction::Out ? 0 : 1, s.data(),
                                         d.data(), e.st.data(), e.en.data()));
      e.nbr = dir_ == Direction::Out ? std::move(d) : std::move(s);
      // the reference's segment order (start, end, neighbor), tcsr.cpp:12-15
      // (the device orders a segment by its search key only)
      std::vector<EdgeId> p;
      for (VertexId v = 0; v < n_; ++v) {
        const EdgeId lo = offsets_[v], hi = offsets_[v + 1];
        if (hi - lo < 2) continue;
        p.resize(hi - lo);
        std::iota(p.begin(), p.end(), lo);
        std::sort(p.begin(), p.end(), [&](EdgeId x, EdgeId y) {
          if (e.st[x] != e.st[y]) return e.st[x] < e.st[y];
          if (e.en[x] != e.en[y]) return e.en[x] < e.en[y];
          return e.nbr[x] < e.nbr[y];
        });
        std::vector<VertexId> nb(p.size());
        std::vector<Timestamp> a(p.size()), b(p.size());
        for (std::size_t i = 0; i < p.size(); ++i) {
          nb[i] = e.nbr[p[i]];
          a[i] = e.st[p[i]];
          b[i] = e.en[p[i]];
        }
        std::copy(nb.begin(), nb.end(), e.nbr.begin() + lo);
        std::copy(a.begin(), a.end(), e.st.begin() + lo);
        std::copy(b.begin(), b.end(), e.en.begin() + lo);
      }
      *edges_ = std::move(e);
    });
    return *edges_;
  }
  std::shared_ptr<tgxd_graph> h_;
  Direction dir_ = Direction::Out;
  VertexId n_ = 0;
  std::vector<EdgeId> offsets_;
  std::shared_ptr<std::once_flag> once_ = std::make_shared<std::once_flag>();
  std::shared_ptr<Edges> edges_ = std::make_shared<Edges>();
};

// Device-resident graph: both T-CSR layouts plus the selective index. Cheap
// to copy (shared handle); immutable after build.
class TemporalGraph {
 public:
  static TemporalGraph build(std::vector<TemporalEdge> edges, VertexId n_v, bool directed,
                             const EngineConfig& config = {}) {
    if (config.index_cutoff < 1) throw std::invalid_argument("index cutoff must be >= 1");
    const std::size_t m = edges.size();
    std::vector<std::uint32_t> s(m), d(m);
    std::vector<std::uint64_t> a(m), b(m);
    std::vector<double> w(m);
    bool weighted = false;
    for (std::size_t i = 0; i < m; ++i) {
      s[i] = edges[i].source;
      d[i] = edges[i].destination;
      a[i] = edges[i].start;
      b[i] = edges[i].end;
      w[i] = edges[i].weight;
      weighted = weighted || w[i] != 1.0;
    }
    tgxd_graph* h = nullptr;
    detail::check(tgxd_graph_build_weighted(n_v, m, s.data(), d.data(), a.data(), b.data(),
                                            weighted ? w.data() : nullptr, directed ? 1 : 0,
                                            config.index_cutoff, &h));
    TemporalGraph g;
    g.h_ = std::shared_ptr<tgxd_graph>(h, tgxd_graph_destroy);
    g.config_ = config;
    g.n_ = n_v;
    g.meta_ = std::make_shared<Layouts>();
    g.meta_->m_logical = m;
    g.meta_->directed = directed;
    return g;
  }

  // A handle on the same device graph with its own stream and workspace
  // (tgxd_graph_view): give each serving thread one; `share` of them run
  // side by side. Keeps this graph alive.
  TemporalGraph view(int share) const {
    tgxd_graph* v = nullptr;
    detail::check(tgxd_graph_view(h_.get(), share, &v));
    TemporalGraph g = *this;
    std::shared_ptr<tgxd_graph> parent = h_;
    g.h_ = std::shared_ptr<tgxd_graph>(v, [parent](tgxd_graph* p) { tgxd_graph_destroy(p); });
    return g;
  }

  VertexId vertex_count() const { return n_; }
  const EngineConfig& config() const { return config_; }
  Ordering ordering() const { return config_.ordering; }
  tgxd_graph* handle() const { return h_.get(); }

  // engine.hpp:35-44 (degrees read back from the device once per graph)
  const GraphMeta& meta() const { return layouts().meta; }
  const TemporalCsr& csr(Direction d) const { return d == Direction::Out ? out_csr() : in_csr(); }
  const TemporalCsr& out_csr() const { return layouts().out; }
  const TemporalCsr& in_csr() const { return layouts().in; }
  EdgeId degree(VertexId v, Direction d) const { return csr(d).degree(v); }

 private:
  struct Layouts {
    std::once_flag once;
    EdgeId m_logical = 0;
    bool directed = true;
    GraphMeta meta;
    TemporalCsr out, in;
  };
  const Layouts& layouts() const {
    std::call_once(meta_->once, [this] {
      Layouts& L = *meta_;
      L.meta.n_v = n_;
      L.meta.n_e = L.m_logical;
      L.meta.directed = L.directed;
      for (int dir = 0; dir < 2; ++dir) {
        std::vector<std::uint32_t> deg(n_);
        if (n_) detail::check(tgxd_graph_degrees(h_.get(), dir, deg.data()));
        std::vector<EdgeId>& md = dir == 0 ? L.meta.out_degree : L.meta.in_degree;
        md.assign(deg.begin(), deg.end());
        TemporalCsr& c = dir == 0 ? L.out : L.in;
        c.h_ = h_;
        c.dir_ = dir == 0 ? Direction::Out : Direction::In;
        c.n_ = n_;
        c.offsets_.assign(static_cast<std::size_t>(n_) + 1, 0);
        for (VertexId v = 0; v < n_; ++v) c.offsets_[v + 1] = c.offsets_[v] + deg[v];
      }
    });
    return *meta_;
  }
  std::shared_ptr<tgxd_graph> h_;
  EngineConfig config_;
  VertexId n_ = 0;
  std::shared_ptr<Layouts> meta_;
};

namespace detail {
inline PathResult run(int kind, const TemporalGraph& g, VertexId v, const QueryWindow& w,
                      const AlgoOptions& opts) {
  const Ordering ord = opts.ordering.value_or(g.ordering());
  PathResult r;
  r.values.resize(g.vertex_count());
  tgxd_stats st{};
  const std::uint64_t ta = w.t_a, tb = w.t_b;
  check(tgxd_query(g.handle(), kind, 1, &v, &ta, &tb, static_cast<int>(ord), TGXD_MODE_AUTO,
                   r.values.data(), 8, 0, &st));
  if (opts.stats) {
    opts.stats->index_decisions += st.index_lookups;
    opts.stats->scan_decisions += st.expansions - st.index_lookups;
  }
  return r;
}
}  // namespace detail

inline PathResult earliest_arrival(const TemporalGraph& g, VertexId source, const QueryWindow& w,
                                   const AlgoOptions& opts = {}) {
  return detail::run(TGXD_EARLIEST_ARRIVAL, g, source, w, opts);
}

inline PathResult latest_departure(const TemporalGraph& g, VertexId target, const QueryWindow& w,
                                   const AlgoOptions& opts = {}) {
  return detail::run(TGXD_LATEST_DEPARTURE, g, target, w, opts);
}

inline PathResult fastest_path(const TemporalGraph& g, VertexId source, const QueryWindow& w,
                               const AlgoOptions& opts = {}) {
  return detail::run(TGXD_FASTEST, g, source, w, opts);
}

// path_algorithms.cpp:196-258, 410-434: the least sum of end - start, or
// with opts.weighted of the edges' weights (weight 1.0 unless the graph was
// built with other weights).
inline PathResult shortest_duration(const TemporalGraph& g, VertexId source, const QueryWindow& w,
                                    const AlgoOptions& opts = {}) {
  return detail::run(opts.weighted ? TGXD_SHORTEST_DURATION_WEIGHTED : TGXD_SHORTEST_DURATION, g,
                     source, w, opts);
}

inline PathResult temporal_bfs(const TemporalGraph& g, VertexId source, const QueryWindow& w,
                               const AlgoOptions& opts = {}) {
  return detail::run(TGXD_TEMPORAL_BFS, g, source, w, opts);
}

// Selective-index cost model (selective_index.hpp:45-130). The registry is
// the graph's own (its index cutoff); histograms live on the device.
enum class AccessMethod { IndexLookup, Scan };
struct CostModelParams {
  double c = 1.0;
  double c_prime = 1.0;
  double theta_sel = 0.2;
};
struct AccessDecision {
  AccessMethod method = AccessMethod::Scan;
  double beta_hat = -1.0;
  double k_hat = -1.0;
};
struct CalibrationPoint {
  std::uint64_t degree = 0;
  std::uint64_t matches = 0;
  double index_seconds = 0.0;
  double scan_seconds = 0.0;
};

inline AccessDecision choose_access_method(VertexId v, const TemporalGraph& g, Direction d,
                                           const QueryWindow& w,
                                           const CostModelParams& params = {}) {
  std::int32_t m = 1;
  double beta = -1.0, kh = -1.0;
  std::uint64_t matches = 0;
  const std::uint64_t ta = w.t_a, tb = w.t_b;
  detail::check(tgxd_access_decisions(g.handle(), d == Direction::Out ? 0 : 1, 1, &v, &ta, &tb,
                                      params.theta_sel, &m, &beta, &kh, &matches));
  return AccessDecision{m == 0 ? AccessMethod::IndexLookup : AccessMethod::Scan, beta, kh};
}

inline std::uint64_t count_in_window(const TemporalGraph& g, VertexId v, Direction d,
                                     const QueryWindow& w) {
  std::int32_t m = 1;
  double beta = -1.0, kh = -1.0;
  std::uint64_t matches = 0;
  const std::uint64_t ta = w.t_a, tb = w.t_b;
  detail::check(tgxd_access_decisions(g.handle(), d == Direction::Out ? 0 : 1, 1, &v, &ta, &tb,
                                      0.2, &m, &beta, &kh, &matches));
  return matches;
}

inline CostModelParams fit_cost_constants(const std::vector<CalibrationPoint>& points,
                                          double theta_sel = 0.2) {
  std::vector<std::uint64_t> deg, mat;
  std::vector<double> ix, sc;
  for (const CalibrationPoint& p : points) {
    deg.push_back(p.degree);
    mat.push_back(p.matches);
    ix.push_back(p.index_seconds);
    sc.push_back(p.scan_seconds);
  }
  CostModelParams out;
  out.theta_sel = theta_sel;
  detail::check(tgxd_fit_cost_constants(points.size(), deg.data(), mat.data(), ix.data(),
                                        sc.data(), &out.c, &out.c_prime));
  return out;
}

inline double cost_index_lookup(std::uint64_t degree, double k, double c) {
  if (degree == 0) throw std::domain_error("cost_index_lookup: degree must be >= 1");
  return c * (std::log2(static_cast<double>(degree)) + k);
}

inline double cost_scan(std::uint64_t degree, double c_prime) {
  return c_prime * static_cast<double>(degree);
}

template <class T>
std::uint64_t digest_of(const std::vector<T>& values) {
  static_assert(sizeof(T) == 8, "labels are int64");
  return tgxd_digest(reinterpret_cast<const std::int64_t*>(values.data()), values.size());
}

}  // namespace tgx_b200
