/* TEST INFRASTRUCTURE ONLY — the checker, never the product.
 *
 * Plain-C restatement of the reference's temporal path algorithms
 * (earliest arrival, latest departure, fastest, shortest duration, temporal
 * BFS; every ordering including Overlaps) over a host T-CSR, with the
 * reference's u64 timestamps, int64 labels and sentinels. Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg may load it.
 * Pinned against the compiled reference (oracle/_ref/libtgxref.so) and the
 * golden vectors in tests/golden/ (see tests/test_oracle.py).
 */
#ifndef TGX_ORACLE_H
#define TGX_ORACLE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { TGXO_OK = 0, TGXO_OUT_OF_RANGE = 1, TGXO_INVALID_ARGUMENT = 2, TGXO_UNSUPPORTED = 3 };
/* kinds: the reference's five path metrics (algorithms.hpp:46-66) */
enum { TGXO_EA = 0, TGXO_LD = 1, TGXO_FASTEST = 2, TGXO_SD = 3, TGXO_BFS = 4 };
/* shortest duration with AlgoOptions::weighted (sum of edge weights) */
enum { TGXO_SD_WEIGHTED = 5 };
/* Ordering values follow tgx::Ordering (types.hpp:64-68). */
enum { TGXO_SUCCEEDS = 0, TGXO_STRICTLY_SUCCEEDS = 1, TGXO_OVERLAPS = 2 };

typedef struct tgxo_graph tgxo_graph;

int tgxo_graph_build(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                     const uint64_t* start, const uint64_t* end, int directed, tgxo_graph** out);
int tgxo_graph_build_weighted(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                              const uint64_t* start, const uint64_t* end, const double* weight,
                              int directed, tgxo_graph** out);
void tgxo_graph_free(tgxo_graph* g);
uint64_t tgxo_graph_edges(const tgxo_graph* g);

int tgxo_query(const tgxo_graph* g, int kind, uint32_t vertex, uint64_t ta, uint64_t tb,
               int ordering, int64_t* out);

/* SURVEY.md 8(d) unit of work from final labels: admissible window edges of
 * reached vertices, and the reached count. */
int tgxo_work(const tgxo_graph* g, int kind, uint32_t vertex, uint64_t ta, uint64_t tb,
              int ordering, const int64_t* labels, uint64_t* e_adm, uint64_t* v_reached);

uint64_t tgxo_digest(const int64_t* values, uint64_t n);

/* Selective-index cost model (selective_index.cpp:67-209): for k (vertex,
 * window) pairs of one direction (0 out, 1 in) of a graph indexed at
 * `cutoff`, choose_access_method's decision (0 index lookup, 1 scan),
 * beta_hat and k_hat (-1 / -1 below the cutoff), and count_in_window
 * (tcsr.cpp:124-128). */
int tgxo_access_decisions(const tgxo_graph* g, int dir, uint64_t cutoff, uint64_t k,
                          const uint32_t* verts, const uint64_t* ta, const uint64_t* tb,
                          double theta_sel, int32_t* method, double* beta_hat, double* k_hat,
                          uint64_t* matches);
/* fit_cost_constants (selective_index.cpp:211-235): least-squares c, c'. */
int tgxo_fit_cost_constants(uint64_t k, const uint64_t* degree, const uint64_t* matches,
                            const double* index_s, const double* scan_s, double* c,
                            double* c_prime);
const char* tgxo_last_error(void);

/* The BASELINE workload generator (tgx_gen.c); same field layout as the
 * product's tgxd_gen_config so one ctypes structure serves both. */
typedef struct tgxo_gen_config {
  int kind; /* 0 uniform, 1 RMAT */
  uint32_t scale;
  uint32_t n;
  uint64_t m;
  double a, b, c;
  int start_dist; /* 0 uniform, 1 cube root */
  uint32_t t_range;
  double geo_p;
  uint64_t seed;
} tgxo_gen_config;
int tgxo_generate(const tgxo_gen_config* c, uint64_t capacity, uint64_t* m_out, uint32_t* src,
                  uint32_t* dst, uint64_t* start, uint64_t* end);

#ifdef __cplusplus
}
#endif
#endif
