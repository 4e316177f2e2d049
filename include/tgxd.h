/* tgxd — C-ABI of the B200-native temporal traversal engine.
 *
 * Drop-in boundary for the reference's traversal hot path (Kairos "tgx",
 * /root/reference/proj). Plain pointers and sizes only; no exceptions and no
 * torch types cross it. Every entry point names the reference interface it
 * replaces. Errors are integer codes plus tgxd_last_error() (thread-local
 * message); the codes map onto the reference's exception types:
 *   TGXD_ERR_VERTEX_RANGE  std::out_of_range   (path_algorithms.cpp:15-20)
 *   TGXD_ERR_EDGE          std::out_of_range   (types.cpp:41-54, tcsr.cpp:39-44)
 *   TGXD_ERR_WINDOW        std::invalid_argument (path_algorithms.cpp:22-25,
 *                                               internal.hpp:19-21)
 *   TGXD_ERR_TIME_RANGE    edge time outside the device's int32 time domain
 *                          [0, 2^31 - 2] (no reference equivalent: the
 *                          reference keeps u64 times)
 *   TGXD_ERR_UNSUPPORTED   a request outside the device path (e.g. the unit of
 *                          work of an edge-state query); no CPU fallback
 *   TGXD_ERR_CUDA          CUDA runtime failure, or no usable GPU
 *   TGXD_ERR_ARGUMENT      malformed call (null pointer, bad enum, ...)
 *
 * Threading: concurrent calls on one graph handle are serialized by the
 * handle's mutex (the reference allows concurrent const calls, SPEC.md:460;
 * here each handle owns one CUDA stream and one workspace).
 */
#ifndef TGXD_H
#define TGXD_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define TGXD_VERSION 1

typedef struct tgxd_graph tgxd_graph;

enum tgxd_status {
  TGXD_OK = 0,
  TGXD_ERR_VERTEX_RANGE = 1,
  TGXD_ERR_WINDOW = 2,
  TGXD_ERR_TIME_RANGE = 3,
  TGXD_ERR_UNSUPPORTED = 4,
  TGXD_ERR_CUDA = 5,
  TGXD_ERR_ARGUMENT = 6,
  TGXD_ERR_EDGE = 7
};

/* The reference's path metrics, algorithms.hpp:46-66 (EA / LD / fastest on
 * the hot path; shortest duration (unweighted) and temporal BFS next to it). */
enum tgxd_kind {
  TGXD_EARLIEST_ARRIVAL = 0,
  TGXD_LATEST_DEPARTURE = 1,
  TGXD_FASTEST = 2,
  TGXD_SHORTEST_DURATION = 3,
  TGXD_TEMPORAL_BFS = 4,
  /* shortest_duration with AlgoOptions::weighted (algorithms.hpp:36): the
   * sum of edge weights, which must be non-negative integers on every edge a
   * path can reach (else TGXD_ERR_WINDOW, the reference's invalid_argument,
   * path_algorithms.cpp:196-203); weights >= 2^62 give TGXD_ERR_TIME_RANGE.
   * A graph built without weights has weight 1.0 on every edge. */
  TGXD_SHORTEST_DURATION_WEIGHTED = 5
};

/* tgx::Ordering, types.hpp:64-68 (same numeric order). Overlaps runs every
 * metric on the edge-state engine (path_algorithms.cpp:40-191). */
enum tgxd_ordering { TGXD_SUCCEEDS = 0, TGXD_STRICTLY_SUCCEEDS = 1, TGXD_OVERLAPS = 2 };

/* Frontier representation policy (temporal_edge_map's representation switch,
 * engine.hpp:280-295). AUTO switches on frontier size; the forced modes exist
 * for the push/pull equivalence tests (test_engine.cpp:153-176). */
enum tgxd_mode {
  TGXD_MODE_AUTO = 0,    /* engine's choice */
  TGXD_MODE_SPARSE = 1,  /* round-based, queue frontier every round */
  TGXD_MODE_DENSE = 2,   /* round-based, implicit (dense) frontier every round */
  TGXD_MODE_ASYNC = 3,   /* barrier-free work queues (no rounds) */
  TGXD_MODE_PULL = 4,    /* round-based, every round pulled (dense bottom-up) */
  TGXD_MODE_LANES = 5    /* batches of 2..32 EA / LD queries: one warp lane per query,
                            vertex-major labels (AUTO's choice when they share one source) */
};

/* Output label width: 8 = int64 exactly as PathResult::values
 * (algorithms.hpp:16-21: INT64_MAX / INT64_MIN sentinels, exact seed values);
 * 4 = int32 device labels (INT32_MAX unreached for EA / fastest, INT32_MIN
 * for LD; the seed saturates to the int32 time domain). */

typedef struct tgxd_stats {
  uint32_t rounds;          /* frontier rounds (all candidates for fastest) */
  uint32_t candidates;      /* fastest: departure candidates swept */
  uint64_t expansions;      /* frontier vertices expanded: one per for_each_window_edge call
                               of the reference (engine.hpp:316, 341; a pull round visits
                               every slot) */
  uint64_t edges_relaxed;   /* edges relaxed by push plus entries scanned by pull rounds */
  uint64_t index_lookups;   /* expansions that used the selective index */
  float kernel_ms;          /* traversal kernel time (CUDA events) */
  float total_ms;           /* device time of the whole query incl. init/output */
} tgxd_stats;

/* Synthetic generator configuration (BASELINE.json configs). */
enum tgxd_gen_kind { TGXD_GEN_UNIFORM = 0, TGXD_GEN_RMAT = 1 };
enum tgxd_start_dist { TGXD_START_UNIFORM = 0, TGXD_START_CUBE_ROOT = 1 };
typedef struct tgxd_gen_config {
  int kind;            /* tgxd_gen_kind */
  uint32_t scale;      /* RMAT: n = 2^scale */
  uint32_t n;          /* uniform: vertex count */
  uint64_t m;          /* edges drawn (uniform: self-loops then dropped) */
  double a, b, c;      /* RMAT quadrant probabilities (d = 1 - a - b - c) */
  int start_dist;      /* tgxd_start_dist */
  uint32_t t_range;    /* starts in [0, t_range) */
  double geo_p;        /* duration = 1 + Geometric(geo_p) failures */
  uint64_t seed;
} tgxd_gen_config;

const char* tgxd_last_error(void);
int tgxd_version(void);
/* Number of visible CUDA devices (0 on a CPU-only host). */
int tgxd_device_count(int* count);

/* TemporalGraph::build(edges, n_v, directed, config), engine.hpp:32-33 /
 * engine.cpp:7-34. Validates like compute_meta (types.cpp:19-56), symmetrizes
 * undirected inputs, builds both device T-CSR layouts and the selective
 * index (vertices with degree >= index_cutoff; 0 = the reference default
 * 2048, selective_index.hpp:74). Host arrays of m edges. */
int tgxd_graph_build(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                     const uint64_t* start, const uint64_t* end, int directed,
                     uint64_t index_cutoff, tgxd_graph** out);

/* Same, with per-edge weights (TemporalEdge::weight, types.hpp:29-40):
 * stored on the device (int64, Out-layout order) for weighted shortest
 * duration; NULL = every weight 1.0. */
int tgxd_graph_build_weighted(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                              const uint64_t* start, const uint64_t* end, const double* weight,
                              int directed, uint64_t index_cutoff, tgxd_graph** out);

/* Same, but the edge list is generated on the device (no host copy). */
int tgxd_graph_generate(const tgxd_gen_config* cfg, int directed, uint64_t index_cutoff,
                        tgxd_graph** out);

/* The identical edge list on the host (for the oracle / reference side).
 * Writes at most `capacity` edges; *m_out receives the edge count. */
int tgxd_generate_host(const tgxd_gen_config* cfg, uint64_t capacity, uint64_t* m_out,
                       uint32_t* src, uint32_t* dst, uint64_t* start, uint64_t* end);

void tgxd_graph_destroy(tgxd_graph* g);

/* n, materialized edges per layout, and indexed vertices per direction
 * (VertexIndexRegistry::indexed_count, selective_index.hpp:93-96). */
int tgxd_graph_info(const tgxd_graph* g, uint32_t* n, uint64_t* m, uint64_t* indexed_out,
                    uint64_t* indexed_in);

/* Per-vertex degree in one direction (0 = Out, 1 = In) into a host array. */
int tgxd_graph_degrees(tgxd_graph* g, int direction, uint32_t* out);

/* The edge list back from one device layout (TemporalCsr::flatten,
 * tcsr.hpp:74-76), host arrays of m entries, segment order. */
int tgxd_graph_flatten(tgxd_graph* g, int direction, uint32_t* src, uint32_t* dst,
                       uint64_t* start, uint64_t* end);

/* earliest_arrival / latest_departure / fastest_path (algorithms.hpp:46-58):
 * one query, n int64 labels into a HOST array, exactly PathResult::values. */
int tgxd_earliest_arrival(tgxd_graph* g, uint32_t source, uint64_t t_a, uint64_t t_b,
                          int ordering, int64_t* out, tgxd_stats* stats);
int tgxd_latest_departure(tgxd_graph* g, uint32_t target, uint64_t t_a, uint64_t t_b,
                          int ordering, int64_t* out, tgxd_stats* stats);
int tgxd_fastest(tgxd_graph* g, uint32_t source, uint64_t t_a, uint64_t t_b, int ordering,
                 int64_t* out, tgxd_stats* stats);
/* shortest_duration (unweighted: sum of end - start; algorithms.hpp:62-63,
 * path_algorithms.cpp:410-434) and temporal_bfs (hops; algorithms.hpp:66-67,
 * path_algorithms.cpp:359-408). Same conventions: INT64_MAX unreached,
 * out[source] = 0. */
int tgxd_shortest_duration(tgxd_graph* g, uint32_t source, uint64_t t_a, uint64_t t_b,
                           int ordering, int64_t* out, tgxd_stats* stats);
int tgxd_temporal_bfs(tgxd_graph* g, uint32_t source, uint64_t t_a, uint64_t t_b, int ordering,
                      int64_t* out, tgxd_stats* stats);
/* shortest_duration with AlgoOptions::weighted = true (path_algorithms.cpp:196-258). */
int tgxd_shortest_duration_weighted(tgxd_graph* g, uint32_t source, uint64_t t_a, uint64_t t_b,
                                    int ordering, int64_t* out, tgxd_stats* stats);

/* General form: k queries of one kind run as one batched traversal
 * (configs 3 and 5). out holds k x n labels of `width` bytes (4 or 8),
 * host or device memory. mode is a tgxd_mode. */
int tgxd_query(tgxd_graph* g, int kind, uint32_t k, const uint32_t* vertices,
               const uint64_t* t_a, const uint64_t* t_b, int ordering, int mode, void* out,
               int width, int out_on_device, tgxd_stats* stats);

/* Unit of work of the LAST query on this handle (slot q of its batch):
 * E_adm and V_reached as SURVEY.md 8(d) defines them, counted on the device
 * from the final labels. For fastest, the arrival fixpoint is counted. */
int tgxd_last_work(tgxd_graph* g, uint32_t q, uint64_t* e_adm, uint64_t* v_reached);

/* Bytes the LAST host-result query moved device -> host: the int32 (or int64)
 * result copies plus, for the early copy of EA / LD results, the tail's
 * {slot, label} patch pairs (8 B each) written through mapped memory. */
int tgxd_last_d2h_bytes(tgxd_graph* g, uint64_t* bytes);

/* Bytes the LAST query moved host -> device: its parameters and seeds (only
 * when they differ from what the device already holds) and fastest's
 * candidate lists. */
int tgxd_last_h2d_bytes(tgxd_graph* g, uint64_t* bytes);

/* Kernels this handle's queries have launched so far (a running total;
 * measurement: bench.py's gpu_launches is the difference over its timed
 * loops). Not in the reference. */
int tgxd_launch_count(tgxd_graph* g, uint64_t* count);

/* Device time of `steps` back-to-back queries with device-resident output,
 * after `warmup` untimed ones: total ms (CUDA events on the handle's stream)
 * and the mean traversal-kernel ms per query. */
int tgxd_time_queries(tgxd_graph* g, int kind, uint32_t k, const uint32_t* vertices,
                      const uint64_t* t_a, const uint64_t* t_b, int ordering, int mode,
                      int warmup, int steps, float* total_ms, float* kernel_ms);

/* Same, but step i answers the single query i mod k (a rotation over k
 * sources / windows: every step uploads its own parameters and resets the
 * previous query's labels, as a stream of distinct queries does). */
int tgxd_time_rotation(tgxd_graph* g, int kind, uint32_t k, const uint32_t* vertices,
                       const uint64_t* t_a, const uint64_t* t_b, int ordering, int mode,
                       int warmup, int steps, float* total_ms, float* kernel_ms);

/* Diagnostics: record a per-round trace of the next queries, max_rounds = 0
 * disables. tgxd_get_trace writes 12 u64 per round: globaltimer (ns) at round
 * start / after expand / after relax, frontier size, chunks, small ranges,
 * pushes, flags, then the latest and (2^62 - earliest) warp completion time
 * of expand and of relax. Without with_device only the first 8 are filled
 * and the call is safe while a query is still running. */
int tgxd_set_trace(tgxd_graph* g, uint32_t max_rounds);
int tgxd_get_trace(tgxd_graph* g, uint64_t* out, uint32_t max_rounds, int with_device);

/* A second handle on g's device graph (no copy) with its own stream,
 * workspace and host staging, for serving queries side by side from several
 * host threads: its persistent grids take 1/share of the GPU, so `share`
 * views run concurrently (config 2: 4 views 1.35x the throughput of one
 * handle). Destroy views before g; no counterpart in the reference (its
 * concurrent const calls share the OpenMP pool). */
int tgxd_graph_view(tgxd_graph* g, int share, tgxd_graph** out);

/* Selective-index cost model (replaces choose_access_method,
 * selective_index.hpp:63-106 / selective_index.cpp:98-209, and
 * TemporalCsr::count_in_window, tcsr.hpp:72): for k (vertex, window) pairs of
 * one direction (0 out, 1 in), the access decision (0 index lookup, 1 scan),
 * beta_hat and k_hat from the vertex's 100x100 (start, duration) density
 * histogram (-1 and -1 for vertices below the index cutoff: no histogram),
 * and the exact number of window-contained edges. Bit-identical to the
 * reference's doubles. The histograms are built on the device on first use. */
int tgxd_access_decisions(tgxd_graph* g, int direction, uint32_t k, const uint32_t* vertices,
                          const uint64_t* t_a, const uint64_t* t_b, double theta_sel,
                          int32_t* method, double* beta_hat, double* k_hat, uint64_t* matches);

/* fit_cost_constants (selective_index.cpp:211-235): least-squares c (index:
 * seconds ~ c (log2 degree + matches)) and c' (scan: seconds ~ c' degree)
 * over k calibration points; INVALID_ARGUMENT for an empty sample or one
 * without degree >= 1 (TGXD_ERR_WINDOW: the reference throws std::invalid_argument). */
int tgxd_fit_cost_constants(uint64_t k, const uint64_t* degree, const uint64_t* matches,
                            const double* index_seconds, const double* scan_seconds,
                            double* c, double* c_prime);

/* FNV-1a digest of int64 labels (digest.hpp:12-52). */
uint64_t tgxd_digest(const int64_t* values, uint64_t n);

#ifdef __cplusplus
}
#endif
#endif
