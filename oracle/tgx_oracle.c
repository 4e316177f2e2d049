/* TEST INFRASTRUCTURE ONLY — the checker, never the product.
 *
 * Plain-C restatement of the reference (Kairos "tgx", /root/reference/proj)
 * algorithms on the traversal hot path. Every function cites the reference
 * lines it follows. The restatement keeps the reference's data model
 * (u64 timestamps, int64 labels, INT64_MAX / INT64_MIN sentinels) and its
 * round-synchronous label-correcting schedule (snapshot per round, stamp
 * claim per round). Like the reference's engine it relaxes only a frontier
 * vertex's window edges; it always uses the sparse (push) representation —
 * the reference pins push/pull equivalence in test_engine.cpp:153-176 — and
 * it locates a segment's first admissible edge by binary search instead of
 * scanning from the segment start (tcsr.hpp:60-69 scans and filters; the set
 * of edges handed to `update` is identical because segments are sorted by
 * start).
 *
 * Pinned by tests/test_oracle.py against the compiled reference
 * (oracle/_ref/libtgxref.so) on thousands of random instances and against
 * the committed golden vectors in tests/golden/.
 */
#include "tgx_oracle.h"

#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#define INF64 ((int64_t)0x7fffffffffffffffLL)    /* PathResult::kUnreachedMin, algorithms.hpp:17 */
#define NEGINF64 ((int64_t)(-0x7fffffffffffffffLL - 1)) /* kUnreachedMax, algorithms.hpp:18 */
#define TIME_LIMIT ((uint64_t)0x7fffffffffffffffULL)    /* internal.hpp:17-25, types.cpp:29 */
#define TIME_MAX_U64 UINT64_MAX                          /* kMaxTimestamp, types.hpp */

static _Thread_local char g_err[256];

const char* tgxo_last_error(void) { return g_err; }

static int fail(int code, const char* msg) {
  snprintf(g_err, sizeof g_err, "%s", msg);
  return code;
}

/* One T-CSR layout (tcsr.hpp:27-85): offsets, neighbor, start, end. */
typedef struct {
  uint64_t* off;
  uint32_t* nbr;
  uint64_t* st;
  uint64_t* en;
  double* wt;
} ocsr;

struct tgxo_graph {
  uint32_t n;
  uint64_t m; /* materialized edge count per layout */
  ocsr out, in;
};

typedef struct {
  uint64_t s, e;
  uint32_t nbr;
  double w;
} orec;

/* Segment order (start, end, neighbor, weight), tcsr.cpp:12-15. */
static int rec_cmp(const void* a, const void* b) {
  const orec* x = (const orec*)a;
  const orec* y = (const orec*)b;
  if (x->s != y->s) return x->s < y->s ? -1 : 1;
  if (x->e != y->e) return x->e < y->e ? -1 : 1;
  if (x->nbr != y->nbr) return x->nbr < y->nbr ? -1 : 1;
  if (x->w != y->w) return x->w < y->w ? -1 : 1;
  return 0;
}

/* TemporalCsr::build, tcsr.cpp:19-84: count, exclusive scan, placement,
 * per-segment sort, split into flat arrays. */
static int build_csr(ocsr* c, uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                     const uint64_t* st, const uint64_t* en, const double* wt, int by_dst) {
  c->off = calloc((size_t)n + 1, sizeof(uint64_t));
  c->nbr = malloc((m ? m : 1) * sizeof(uint32_t));
  c->st = malloc((m ? m : 1) * sizeof(uint64_t));
  c->en = malloc((m ? m : 1) * sizeof(uint64_t));
  c->wt = malloc((m ? m : 1) * sizeof(double));
  orec* rec = malloc((m ? m : 1) * sizeof(orec));
  uint64_t* cur = malloc(((size_t)n + 1) * sizeof(uint64_t));
  if (!c->off || !c->nbr || !c->st || !c->en || !c->wt || !rec || !cur) {
    free(rec);
    free(cur);
    return fail(TGXO_INVALID_ARGUMENT, "oracle: out of host memory");
  }
  for (uint64_t i = 0; i < m; ++i) c->off[(by_dst ? dst[i] : src[i]) + 1]++;
  for (uint32_t v = 0; v < n; ++v) c->off[v + 1] += c->off[v];
  memcpy(cur, c->off, ((size_t)n + 1) * sizeof(uint64_t));
  for (uint64_t i = 0; i < m; ++i) {
    const uint32_t key = by_dst ? dst[i] : src[i];
    const uint64_t slot = cur[key]++;
    rec[slot].s = st[i];
    rec[slot].e = en[i];
    rec[slot].nbr = by_dst ? src[i] : dst[i];
    rec[slot].w = wt ? wt[i] : 1.0;
  }
  for (uint32_t v = 0; v < n; ++v) {
    const uint64_t lo = c->off[v], hi = c->off[v + 1];
    if (hi - lo > 1) qsort(rec + lo, hi - lo, sizeof(orec), rec_cmp);
  }
  for (uint64_t i = 0; i < m; ++i) {
    c->nbr[i] = rec[i].nbr;
    c->st[i] = rec[i].s;
    c->en[i] = rec[i].e;
    c->wt[i] = rec[i].w;
  }
  free(rec);
  free(cur);
  return TGXO_OK;
}

static void free_csr(ocsr* c) {
  free(c->off);
  free(c->nbr);
  free(c->st);
  free(c->en);
  free(c->wt);
}

void tgxo_graph_free(tgxo_graph* g) {
  if (!g) return;
  free_csr(&g->out);
  free_csr(&g->in);
  free(g);
}

uint64_t tgxo_graph_edges(const tgxo_graph* g) { return g->m; }

/* TemporalGraph::build, engine.cpp:7-34, with compute_meta's validation
 * (types.cpp:19-56): endpoints < n, end >= start, end <= 2^63-1, first
 * offending edge reported; undirected inputs materialize the reverse of every
 * non-self-loop edge (engine.cpp:13-22). */
int tgxo_graph_build(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                     const uint64_t* start, const uint64_t* end, int directed, tgxo_graph** out) {
  return tgxo_graph_build_weighted(n, m, src, dst, start, end, NULL, directed, out);
}

/* Same with per-edge weights (TemporalEdge::weight, types.hpp:29-40; NULL:
 * every weight 1.0, the TemporalEdge default). */
int tgxo_graph_build_weighted(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                              const uint64_t* start, const uint64_t* end, const double* weight,
                              int directed, tgxo_graph** out) {
  *out = NULL;
  for (uint64_t i = 0; i < m; ++i) {
    char msg[160];
    if (src[i] >= n || dst[i] >= n) {
      snprintf(msg, sizeof msg, "edge %llu: endpoint outside vertex range", (unsigned long long)i);
      return fail(TGXO_OUT_OF_RANGE, msg);
    }
    if (end[i] < start[i]) {
      snprintf(msg, sizeof msg, "edge %llu: end precedes start", (unsigned long long)i);
      return fail(TGXO_OUT_OF_RANGE, msg);
    }
    if (end[i] > TIME_LIMIT) {
      snprintf(msg, sizeof msg, "edge %llu: end beyond 2^63-1", (unsigned long long)i);
      return fail(TGXO_OUT_OF_RANGE, msg);
    }
  }
  const uint32_t* s = src;
  const uint32_t* d = dst;
  const uint64_t* a = start;
  const uint64_t* b = end;
  uint64_t mm = m;
  const double* w = weight;
  uint32_t *s2 = NULL, *d2 = NULL;
  uint64_t *a2 = NULL, *b2 = NULL;
  double* w2 = NULL;
  if (!directed) {
    uint64_t extra = 0;
    for (uint64_t i = 0; i < m; ++i) extra += src[i] != dst[i];
    mm = m + extra;
    s2 = malloc((mm ? mm : 1) * 4);
    d2 = malloc((mm ? mm : 1) * 4);
    a2 = malloc((mm ? mm : 1) * 8);
    b2 = malloc((mm ? mm : 1) * 8);
    w2 = malloc((mm ? mm : 1) * 8);
    memcpy(s2, src, m * 4);
    memcpy(d2, dst, m * 4);
    memcpy(a2, start, m * 8);
    memcpy(b2, end, m * 8);
    for (uint64_t i = 0; i < m; ++i) w2[i] = weight ? weight[i] : 1.0;
    uint64_t k = m;
    for (uint64_t i = 0; i < m; ++i) {
      if (src[i] == dst[i]) continue;
      s2[k] = dst[i];
      d2[k] = src[i];
      a2[k] = start[i];
      b2[k] = end[i];
      w2[k] = w2[i];
      ++k;
    }
    s = s2;
    d = d2;
    a = a2;
    b = b2;
    w = w2;
  }
  tgxo_graph* g = calloc(1, sizeof(tgxo_graph));
  g->n = n;
  g->m = mm;
  int rc = build_csr(&g->out, n, mm, s, d, a, b, w, 0);
  if (rc == TGXO_OK) rc = build_csr(&g->in, n, mm, s, d, a, b, w, 1);
  free(w2);
  free(s2);
  free(d2);
  free(a2);
  free(b2);
  if (rc != TGXO_OK) {
    tgxo_graph_free(g);
    return rc;
  }
  *out = g;
  return TGXO_OK;
}

/* First position in [lo, hi) whose start >= t (segment sorted by start). */
static uint64_t lower_start(const ocsr* c, uint64_t lo, uint64_t hi, uint64_t t) {
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (c->st[mid] < t) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

/* Growable vertex list. */
typedef struct {
  uint32_t* v;
  uint64_t n, cap;
} vlist;

static void vpush(vlist* l, uint32_t x) {
  if (l->n == l->cap) {
    l->cap = l->cap ? 2 * l->cap : 64;
    l->v = realloc(l->v, l->cap * sizeof(uint32_t));
  }
  l->v[l->n++] = x;
}

static int u32_cmp(const void* a, const void* b) {
  const uint32_t x = *(const uint32_t*)a, y = *(const uint32_t*)b;
  return x < y ? -1 : x > y;
}

/* VertexSubset::from_ids: sort + unique (engine.cpp:36-42). */
static void sort_unique(vlist* l) {
  if (l->n < 2) return;
  qsort(l->v, l->n, sizeof(uint32_t), u32_cmp);
  uint64_t k = 1;
  for (uint64_t i = 1; i < l->n; ++i)
    if (l->v[i] != l->v[k - 1]) l->v[k++] = l->v[i];
  l->n = k;
}

/* checked_window + clamp_window (path_algorithms.cpp:22-25,
 * internal.hpp:17-25). */
static int check_window(uint64_t* ta, uint64_t* tb) {
  if (*ta > *tb) return fail(TGXO_INVALID_ARGUMENT, "query window with t_a > t_b");
  if (*ta > TIME_LIMIT)
    return fail(TGXO_INVALID_ARGUMENT, "window start beyond the supported time range (2^63 - 1)");
  if (*tb > TIME_LIMIT) *tb = TIME_LIMIT;
  return TGXO_OK;
}

/* earliest_arrival, path_algorithms.cpp:262-308. Frontier expansion through
 * temporal_edge_map's sparse branch (engine.hpp:297-320); min_start hook
 * :287-291, update :294-304. */
static void earliest_arrival(const tgxo_graph* g, uint32_t source, uint64_t ta, uint64_t tb,
                             int strict, int64_t* L) {
  const uint32_t n = g->n;
  const ocsr* c = &g->out;
  for (uint32_t v = 0; v < n; ++v) L[v] = INF64;
  L[source] = (int64_t)ta;
  uint32_t* stamp = calloc(n ? n : 1, sizeof(uint32_t));
  uint32_t round = 0;
  vlist fr = {0}, nx = {0};
  int64_t* snapv = NULL;
  uint64_t snapcap = 0;
  vpush(&fr, source);
  while (fr.n) {
    ++round;
    if (fr.n > snapcap) {
      snapcap = fr.n;
      snapv = realloc(snapv, snapcap * sizeof(int64_t));
    }
    /* snap = r.values (:283), read only at frontier vertices */
    for (uint64_t i = 0; i < fr.n; ++i) snapv[i] = L[fr.v[i]];
    nx.n = 0;
    for (uint64_t i = 0; i < fr.n; ++i) {
      const uint32_t s = fr.v[i];
      const int64_t ps = snapv[i];
      uint64_t lo_t = ta;
      if (s != source) {
        const uint64_t b = (uint64_t)ps;
        lo_t = strict ? b + 1 : b;
      }
      if (lo_t < ta) lo_t = ta;
      if (lo_t > tb) continue; /* effective_window crossed, engine.hpp:264 */
      const uint64_t hi = c->off[s + 1];
      for (uint64_t e = lower_start(c, c->off[s], hi, lo_t); e < hi; ++e) {
        const uint64_t ts = c->st[e], te = c->en[e];
        if (ts > tb) break;
        if (te > tb) continue;
        if (s != source) {
          if (ps == INF64) continue;
          if (strict ? (int64_t)ts <= ps : (int64_t)ts < ps) continue;
        }
        const uint32_t d = c->nbr[e];
        if ((int64_t)te < L[d]) { /* write_min, parallel.hpp:91-99 */
          L[d] = (int64_t)te;
          if (stamp[d] != round) { /* claim_stamp, parallel.hpp:113-121 */
            stamp[d] = round;
            vpush(&nx, d);
          }
        }
      }
    }
    sort_unique(&nx);
    vlist t = fr;
    fr = nx;
    nx = t;
  }
  free(stamp);
  free(snapv);
  free(fr.v);
  free(nx.v);
}

/* First position in [lo, hi) whose start > t. */
static uint64_t upper_start(const ocsr* c, uint64_t lo, uint64_t hi, uint64_t t) {
  while (lo < hi) {
    const uint64_t mid = lo + (hi - lo) / 2;
    if (c->st[mid] <= t) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

/* latest_departure, path_algorithms.cpp:310-357: the mirror over the In
 * layout; max_end hook :337-342, update :344-352. */
static void latest_departure(const tgxo_graph* g, uint32_t target, uint64_t ta, uint64_t tb,
                             int strict, int64_t* L) {
  const uint32_t n = g->n;
  const ocsr* c = &g->in;
  for (uint32_t v = 0; v < n; ++v) L[v] = NEGINF64;
  L[target] = (int64_t)tb;
  uint32_t* stamp = calloc(n ? n : 1, sizeof(uint32_t));
  uint32_t round = 0;
  vlist fr = {0}, nx = {0};
  int64_t* snapv = NULL;
  uint64_t snapcap = 0;
  vpush(&fr, target);
  while (fr.n) {
    ++round;
    if (fr.n > snapcap) {
      snapcap = fr.n;
      snapv = realloc(snapv, snapcap * sizeof(int64_t));
    }
    for (uint64_t i = 0; i < fr.n; ++i) snapv[i] = L[fr.v[i]];
    nx.n = 0;
    for (uint64_t i = 0; i < fr.n; ++i) {
      const uint32_t s = fr.v[i];
      const int64_t ps = snapv[i];
      uint64_t hi_t = tb;
      if (s != target) {
        const uint64_t b = (uint64_t)ps;
        if (strict && b == 0) hi_t = 0;
        else hi_t = strict ? b - 1 : b;
      }
      if (hi_t > tb) hi_t = tb;
      if (ta > hi_t) continue;
      /* in-edges (u -> s) with start in [ta, hi_t] (ends are >= starts) */
      const uint64_t lo = lower_start(c, c->off[s], c->off[s + 1], ta);
      const uint64_t hi = upper_start(c, lo, c->off[s + 1], hi_t);
      for (uint64_t e = lo; e < hi; ++e) {
        const uint64_t ts = c->st[e], te = c->en[e];
        if (te > hi_t) continue;
        if (s != target) {
          if (ps == NEGINF64) continue;
          if (strict ? (int64_t)te >= ps : (int64_t)te > ps) continue;
        }
        const uint32_t u = c->nbr[e];
        if ((int64_t)ts > L[u]) { /* write_max, parallel.hpp:101-109 */
          L[u] = (int64_t)ts;
          if (stamp[u] != round) {
            stamp[u] = round;
            vpush(&nx, u);
          }
        }
      }
    }
    sort_unique(&nx);
    vlist t = fr;
    fr = nx;
    nx = t;
  }
  free(stamp);
  free(snapv);
  free(fr.v);
  free(nx.v);
}

typedef struct {
  uint64_t ts, te;
  uint32_t d;
} first_edge;

static int fe_desc(const void* a, const void* b) {
  const first_edge* x = (const first_edge*)a;
  const first_edge* y = (const first_edge*)b;
  return x->ts > y->ts ? -1 : x->ts < y->ts;
}

/* fastest_path, path_algorithms.cpp:436-528: candidate departures are the
 * distinct starts of the source's window out-edges (read from the T-CSR,
 * :452-458) in decreasing order; arrivals persist across candidates; each
 * candidate seeds its first edges (:476-486) then relaxes without a source
 * exemption (:489-517); touched vertices take r = min(r, arrival - depart)
 * (:519-524); r[source] = 0 last (:526). */
static void fastest(const tgxo_graph* g, uint32_t source, uint64_t ta, uint64_t tb, int strict,
                    int64_t* R) {
  const uint32_t n = g->n;
  const ocsr* c = &g->out;
  for (uint32_t v = 0; v < n; ++v) R[v] = INF64;
  R[source] = 0;
  uint64_t nfe = 0;
  first_edge* fe = malloc((c->off[source + 1] - c->off[source] + 1) * sizeof(first_edge));
  for (uint64_t e = c->off[source]; e < c->off[source + 1]; ++e) {
    if (c->st[e] > tb) break;
    if (c->st[e] >= ta && c->en[e] <= tb) {
      fe[nfe].ts = c->st[e];
      fe[nfe].te = c->en[e];
      fe[nfe].d = c->nbr[e];
      ++nfe;
    }
  }
  if (nfe == 0) {
    free(fe);
    return;
  }
  qsort(fe, nfe, sizeof(first_edge), fe_desc);
  int64_t* A = malloc((size_t)n * sizeof(int64_t));
  for (uint32_t v = 0; v < n; ++v) A[v] = INF64;
  uint32_t* stamp = calloc(n, sizeof(uint32_t));
  uint32_t* touch = calloc(n, sizeof(uint32_t));
  uint32_t round = 0, cand = 0;
  vlist fr = {0}, nx = {0}, touched = {0};
  int64_t* snapv = NULL;
  uint64_t snapcap = 0;
  uint64_t i = 0;
  while (i < nfe) {
    const uint64_t depart = fe[i].ts;
    ++cand;
    fr.n = 0;
    touched.n = 0;
    for (; i < nfe && fe[i].ts == depart; ++i) {
      const uint32_t d = fe[i].d;
      if ((int64_t)fe[i].te < A[d]) {
        A[d] = (int64_t)fe[i].te;
        if (touch[d] != cand) {
          touch[d] = cand;
          vpush(&touched, d);
        }
        vpush(&fr, d);
      }
    }
    sort_unique(&fr);
    while (fr.n) {
      ++round;
      if (fr.n > snapcap) {
        snapcap = fr.n;
        snapv = realloc(snapv, snapcap * sizeof(int64_t));
      }
      for (uint64_t k = 0; k < fr.n; ++k) snapv[k] = A[fr.v[k]];
      nx.n = 0;
      for (uint64_t k = 0; k < fr.n; ++k) {
        const uint32_t s = fr.v[k];
        const int64_t ps = snapv[k];
        if (ps == INF64) continue;
        uint64_t lo_t = strict ? (uint64_t)ps + 1 : (uint64_t)ps;
        if (lo_t < ta) lo_t = ta;
        if (lo_t > tb) continue;
        const uint64_t hi = c->off[s + 1];
        for (uint64_t e = lower_start(c, c->off[s], hi, lo_t); e < hi; ++e) {
          const uint64_t ts = c->st[e], te = c->en[e];
          if (ts > tb) break;
          if (te > tb) continue;
          if (strict ? (int64_t)ts <= ps : (int64_t)ts < ps) continue;
          const uint32_t d = c->nbr[e];
          if ((int64_t)te < A[d]) {
            A[d] = (int64_t)te;
            if (touch[d] != cand) {
              touch[d] = cand;
              vpush(&touched, d);
            }
            if (stamp[d] != round) {
              stamp[d] = round;
              vpush(&nx, d);
            }
          }
        }
      }
      sort_unique(&nx);
      vlist t = fr;
      fr = nx;
      nx = t;
    }
    const int64_t dep = (int64_t)depart;
    for (uint64_t k = 0; k < touched.n; ++k) {
      const uint32_t v = touched.v[k];
      if (A[v] - dep < R[v]) R[v] = A[v] - dep;
    }
  }
  R[source] = 0;
  free(fe);
  free(A);
  free(stamp);
  free(touch);
  free(snapv);
  free(fr.v);
  free(nx.v);
  free(touched.v);
}

/* ---- Edge-state traversals ------------------------------------------------
 * Growable edge-id list (flat positions of one layout). */
typedef struct {
  uint64_t* v;
  uint64_t n, cap;
} elist;

static void epush(elist* l, uint64_t x) {
  if (l->n == l->cap) {
    l->cap = l->cap ? 2 * l->cap : 64;
    l->v = realloc(l->v, l->cap * sizeof(uint64_t));
  }
  l->v[l->n++] = x;
}

static int u64_cmp(const void* a, const void* b) {
  const uint64_t x = *(const uint64_t*)a, y = *(const uint64_t*)b;
  return x < y ? -1 : x > y;
}

/* merge_edge_buffers: sort (path_algorithms.cpp:27-35; ids are unique by
 * construction of the callers). */
static void esort(elist* l) {
  if (l->n > 1) qsort(l->v, l->n, sizeof(uint64_t), u64_cmp);
}

/* ordering_holds, types.hpp:72-82 (a precedes b). */
static int holds(uint64_t as, uint64_t ae, uint64_t bs, uint64_t be, int ord) {
  switch (ord) {
    case TGXO_SUCCEEDS: return ae <= bs;
    case TGXO_STRICTLY_SUCCEEDS: return ae < bs;
    default: return as < bs && bs <= ae && ae < be;
  }
}

/* forward_window / backward_window, internal.hpp:33-77: the retrieval
 * window for edges that may follow (Out) or precede (In) interval [s, e];
 * returns 0 when empty. */
static int step_window(uint64_t s, uint64_t e, int ord, int out_dir, uint64_t* ta, uint64_t* tb) {
  if (out_dir) {
    uint64_t lo = *ta;
    switch (ord) {
      case TGXO_SUCCEEDS: lo = e; break;
      case TGXO_STRICTLY_SUCCEEDS:
        if (e == TIME_MAX_U64) return 0;
        lo = e + 1;
        break;
      default:
        if (s == TIME_MAX_U64) return 0;
        lo = s + 1;
        break;
    }
    if (lo > *ta) *ta = lo;
  } else {
    uint64_t hi = *tb;
    switch (ord) {
      case TGXO_SUCCEEDS: hi = s; break;
      case TGXO_STRICTLY_SUCCEEDS:
        if (s == 0) return 0;
        hi = s - 1;
        break;
      default:
        if (e == 0) return 0;
        hi = e - 1;
        break;
    }
    if (hi < *tb) *tb = hi;
  }
  return *ta <= *tb;
}

/* for_each_in_window over one segment (tcsr.hpp:60-69): start >= t_a and
 * end <= t_b, scanning from the first start >= t_a up to start > t_b. The
 * reference's index path yields the same set (test_algorithms.cpp:196-217). */
#define FOR_WINDOW(c, v, ta_, tb_, e)                                              \
  for (uint64_t e = lower_start((c), (c)->off[(v)], (c)->off[(v) + 1], (ta_));    \
       e < (c)->off[(v) + 1] && (c)->st[e] <= (tb_); ++e)                          \
    if ((c)->en[e] <= (tb_))

/* edge_reachability, path_algorithms.cpp:40-87: breadth-first search over
 * the edges of one layout under Overlaps; level[e] = the round an edge is
 * first reached (seeds: round 1), 0 if never. */
static uint32_t* edge_reachability(const tgxo_graph* g, uint64_t ta, uint64_t tb, int out_dir,
                                   uint32_t anchor) {
  const ocsr* c = out_dir ? &g->out : &g->in;
  uint32_t* level = calloc(g->m ? g->m : 1, sizeof(uint32_t));
  elist fr = {0}, nx = {0};
  FOR_WINDOW(c, anchor, ta, tb, f) {
    if (!level[f]) {
      level[f] = 1;
      epush(&fr, f);
    }
  }
  esort(&fr);
  uint32_t round = 1;
  while (fr.n) {
    ++round;
    nx.n = 0;
    for (uint64_t i = 0; i < fr.n; ++i) {
      const uint64_t e = fr.v[i];
      uint64_t wa = ta, wb = tb;
      if (!step_window(c->st[e], c->en[e], TGXO_OVERLAPS, out_dir, &wa, &wb)) continue;
      const uint32_t next = c->nbr[e];
      FOR_WINDOW(c, next, wa, wb, f) {
        const int ok = out_dir ? holds(c->st[e], c->en[e], c->st[f], c->en[f], TGXO_OVERLAPS)
                               : holds(c->st[f], c->en[f], c->st[e], c->en[e], TGXO_OVERLAPS);
        if (ok && !level[f]) {
          level[f] = round;
          epush(&nx, f);
        }
      }
    }
    esort(&nx);
    elist t = fr;
    fr = nx;
    nx = t;
  }
  free(fr.v);
  free(nx.v);
  return level;
}

/* earliest_arrival_overlaps / latest_departure_overlaps /
 * temporal_bfs_overlaps, path_algorithms.cpp:89-134. */
static void overlaps_reach(const tgxo_graph* g, int kind, uint32_t v, uint64_t ta, uint64_t tb,
                           int64_t* L) {
  const int out_dir = kind != TGXO_LD;
  const ocsr* c = out_dir ? &g->out : &g->in;
  uint32_t* level = edge_reachability(g, ta, tb, out_dir, v);
  for (uint32_t u = 0; u < g->n; ++u) L[u] = kind == TGXO_LD ? NEGINF64 : INF64;
  for (uint64_t e = 0; e < g->m; ++e) {
    if (!level[e]) continue;
    const uint32_t u = c->nbr[e];
    int64_t x;
    if (kind == TGXO_EA) {
      x = (int64_t)c->en[e];
      if (x < L[u]) L[u] = x;
    } else if (kind == TGXO_LD) {
      x = (int64_t)c->st[e];
      if (x > L[u]) L[u] = x;
    } else {
      x = (int64_t)level[e];
      if (x < L[u]) L[u] = x;
    }
  }
  L[v] = kind == TGXO_EA ? (int64_t)ta : kind == TGXO_LD ? (int64_t)tb : 0;
  free(level);
}

/* fastest_overlaps, path_algorithms.cpp:136-191: per out-edge the latest
 * first-edge start over valid paths ending with it (write_max + round stamp,
 * base read at the round's start); r[v] = min(end - depart). */
static void fastest_overlaps(const tgxo_graph* g, uint32_t source, uint64_t ta, uint64_t tb,
                             int64_t* R) {
  const ocsr* c = &g->out;
  const uint64_t m = g->m;
  int64_t* dep = malloc((m ? m : 1) * sizeof(int64_t));
  uint32_t* stamp = calloc(m ? m : 1, sizeof(uint32_t));
  for (uint64_t e = 0; e < m; ++e) dep[e] = NEGINF64;
  elist fr = {0}, nx = {0};
  int64_t* base = NULL;
  uint64_t bcap = 0;
  FOR_WINDOW(c, source, ta, tb, f) {
    if ((int64_t)c->st[f] > dep[f]) {
      dep[f] = (int64_t)c->st[f];
      epush(&fr, f);
    }
  }
  esort(&fr);
  uint32_t round = 0;
  while (fr.n) {
    ++round;
    if (fr.n > bcap) {
      bcap = fr.n;
      base = realloc(base, bcap * sizeof(int64_t));
    }
    for (uint64_t i = 0; i < fr.n; ++i) base[i] = dep[fr.v[i]];
    nx.n = 0;
    for (uint64_t i = 0; i < fr.n; ++i) {
      const uint64_t e = fr.v[i];
      uint64_t wa = ta, wb = tb;
      if (!step_window(c->st[e], c->en[e], TGXO_OVERLAPS, 1, &wa, &wb)) continue;
      FOR_WINDOW(c, c->nbr[e], wa, wb, f) {
        if (!holds(c->st[e], c->en[e], c->st[f], c->en[f], TGXO_OVERLAPS)) continue;
        if (base[i] > dep[f]) { /* write_max */
          dep[f] = base[i];
          if (stamp[f] != round) { /* claim_stamp */
            stamp[f] = round;
            epush(&nx, f);
          }
        }
      }
    }
    esort(&nx);
    elist t = fr;
    fr = nx;
    nx = t;
  }
  for (uint32_t u = 0; u < g->n; ++u) R[u] = INF64;
  for (uint64_t e = 0; e < m; ++e) {
    if (dep[e] == NEGINF64) continue;
    const int64_t d = (int64_t)c->en[e] - dep[e];
    if (d < R[c->nbr[e]]) R[c->nbr[e]] = d;
  }
  R[source] = 0;
  free(dep);
  free(stamp);
  free(base);
  free(fr.v);
  free(nx.v);
}

/* shortest_duration (unweighted), path_algorithms.cpp:205-258,410-434:
 * out-edge states value[f] = min over valid paths ending with f of the sum of
 * (end - start); frontier by write_min + round stamp with base read at the
 * round's start; r[v] = min over reached in-edges, r[source] = 0. */
/* duration_metric, path_algorithms.cpp:196-203: end - start, or the edge's
 * weight, which must be a non-negative integer (else invalid_argument). */
static int duration_metric(const ocsr* c, uint64_t f, int weighted, int64_t* d) {
  if (!weighted) {
    *d = (int64_t)(c->en[f] - c->st[f]);
    return TGXO_OK;
  }
  const double w = c->wt[f];
  const double r = nearbyint(w);
  if (w < 0.0 || r != w)
    return fail(TGXO_INVALID_ARGUMENT,
                "weighted shortest duration needs non-negative integer weights");
  *d = (int64_t)r;
  return TGXO_OK;
}

static int shortest_duration(const tgxo_graph* g, uint32_t source, uint64_t ta, uint64_t tb,
                             int ord, int weighted, int64_t* R) {
  int rc = TGXO_OK;
  const ocsr* c = &g->out;
  const uint64_t m = g->m;
  int64_t* val = malloc((m ? m : 1) * sizeof(int64_t));
  uint32_t* stamp = calloc(m ? m : 1, sizeof(uint32_t));
  uint8_t* touched = calloc(m ? m : 1, 1);
  for (uint64_t e = 0; e < m; ++e) val[e] = INF64;
  elist fr = {0}, nx = {0};
  int64_t* base = NULL;
  uint64_t bcap = 0;
  uint32_t round = 1;
  FOR_WINDOW(c, source, ta, tb, f) {
    int64_t d;
    if ((rc = duration_metric(c, f, weighted, &d))) goto done;
    if (d < val[f]) {
      val[f] = d;
      touched[f] = 1;
      if (stamp[f] != round) {
        stamp[f] = round;
        epush(&fr, f);
      }
    }
  }
  esort(&fr);
  while (fr.n) {
    ++round;
    if (fr.n > bcap) {
      bcap = fr.n;
      base = realloc(base, bcap * sizeof(int64_t));
    }
    for (uint64_t i = 0; i < fr.n; ++i) base[i] = val[fr.v[i]];
    nx.n = 0;
    for (uint64_t i = 0; i < fr.n; ++i) {
      const uint64_t e = fr.v[i];
      uint64_t wa = ta, wb = tb;
      if (!step_window(c->st[e], c->en[e], ord, 1, &wa, &wb)) continue;
      FOR_WINDOW(c, c->nbr[e], wa, wb, f) {
        if (!holds(c->st[e], c->en[e], c->st[f], c->en[f], ord)) continue;
        int64_t dm;
        if ((rc = duration_metric(c, f, weighted, &dm))) goto done;
        const int64_t cand = base[i] + dm;
        if (cand < val[f]) {
          val[f] = cand;
          touched[f] = 1;
          if (stamp[f] != round) {
            stamp[f] = round;
            epush(&nx, f);
          }
        }
      }
    }
    esort(&nx);
    elist t = fr;
    fr = nx;
    nx = t;
  }
  for (uint32_t u = 0; u < g->n; ++u) R[u] = INF64;
  for (uint64_t e = 0; e < m; ++e)
    if (touched[e] && val[e] < R[c->nbr[e]]) R[c->nbr[e]] = val[e];
  R[source] = 0;
done:
  free(val);
  free(stamp);
  free(touched);
  free(base);
  free(fr.v);
  free(nx.v);
  return rc;
}

/* temporal_bfs, path_algorithms.cpp:359-408: round-synchronous earliest
 * arrival (snapshot per round) recording the first round a vertex's arrival
 * improves; r[source] = 0. */
static void temporal_bfs(const tgxo_graph* g, uint32_t source, uint64_t ta, uint64_t tb,
                         int strict, int64_t* H) {
  const uint32_t n = g->n;
  const ocsr* c = &g->out;
  int64_t* A = malloc((size_t)(n ? n : 1) * sizeof(int64_t));
  int64_t* snap = malloc((size_t)(n ? n : 1) * sizeof(int64_t));
  uint32_t* stamp = calloc(n ? n : 1, sizeof(uint32_t));
  for (uint32_t v = 0; v < n; ++v) {
    A[v] = INF64;
    H[v] = INF64;
  }
  H[source] = 0;
  uint32_t round = 0;
  vlist fr = {0}, nx = {0};
  vpush(&fr, source);
  while (fr.n) {
    ++round;
    memcpy(snap, A, (size_t)n * sizeof(int64_t));
    nx.n = 0;
    for (uint64_t i = 0; i < fr.n; ++i) {
      const uint32_t s = fr.v[i];
      const int64_t ps = snap[s];
      uint64_t lo_t = ta;
      if (s != source) {
        if (ps == INF64) continue;
        lo_t = strict ? (uint64_t)ps + 1 : (uint64_t)ps;
      }
      if (lo_t < ta) lo_t = ta;
      if (lo_t > tb) continue;
      FOR_WINDOW(c, s, lo_t, tb, e) {
        const uint64_t ts = c->st[e], te = c->en[e];
        if (s != source && (strict ? (int64_t)ts <= ps : (int64_t)ts < ps)) continue;
        const uint32_t d = c->nbr[e];
        if ((int64_t)te < A[d]) {
          A[d] = (int64_t)te;
          if (H[d] == INF64) H[d] = round;
          if (stamp[d] != round) {
            stamp[d] = round;
            vpush(&nx, d);
          }
        }
      }
    }
    sort_unique(&nx);
    vlist t = fr;
    fr = nx;
    nx = t;
  }
  H[source] = 0;
  free(A);
  free(snap);
  free(stamp);
  free(fr.v);
  free(nx.v);
}

int tgxo_query(const tgxo_graph* g, int kind, uint32_t vertex, uint64_t ta, uint64_t tb,
               int ordering, int64_t* out) {
  if (vertex >= g->n) return fail(TGXO_OUT_OF_RANGE, "vertex outside vertex range");
  int rc = check_window(&ta, &tb);
  if (rc) return rc;
  const int strict = ordering == TGXO_STRICTLY_SUCCEEDS;
  if (ordering == TGXO_OVERLAPS) { /* path_algorithms.cpp:267,315,366,443 */
    switch (kind) {
      case TGXO_EA:
      case TGXO_LD:
      case TGXO_BFS: overlaps_reach(g, kind, vertex, ta, tb, out); return TGXO_OK;
      case TGXO_FASTEST: fastest_overlaps(g, vertex, ta, tb, out); return TGXO_OK;
      case TGXO_SD: return shortest_duration(g, vertex, ta, tb, ordering, 0, out);
      case TGXO_SD_WEIGHTED: return shortest_duration(g, vertex, ta, tb, ordering, 1, out);
      default: return fail(TGXO_INVALID_ARGUMENT, "unknown query kind");
    }
  }
  switch (kind) {
    case TGXO_EA: earliest_arrival(g, vertex, ta, tb, strict, out); break;
    case TGXO_LD: latest_departure(g, vertex, ta, tb, strict, out); break;
    case TGXO_FASTEST: fastest(g, vertex, ta, tb, strict, out); break;
    case TGXO_SD: return shortest_duration(g, vertex, ta, tb, ordering, 0, out);
    case TGXO_SD_WEIGHTED: return shortest_duration(g, vertex, ta, tb, ordering, 1, out);
    case TGXO_BFS: temporal_bfs(g, vertex, ta, tb, strict, out); break;
    default: return fail(TGXO_INVALID_ARGUMENT, "unknown query kind");
  }
  return TGXO_OK;
}

/* E_adm = sum over reached u of the window edges of u that
 * are admissible under u's final label (all window edges for the root);
 * V_reached = finite labels. kind is TGXO_EA or TGXO_LD; a fastest sweep
 * relaxes exactly the edges its earliest-arrival fixpoint admits (every
 * source window edge is a seed), so callers count it with TGXO_EA. */
int tgxo_work(const tgxo_graph* g, int kind, uint32_t vertex, uint64_t ta, uint64_t tb,
              int ordering, const int64_t* labels, uint64_t* e_adm, uint64_t* v_reached) {
  if (vertex >= g->n) return fail(TGXO_OUT_OF_RANGE, "vertex outside vertex range");
  int rc = check_window(&ta, &tb);
  if (rc) return rc;
  if (kind != TGXO_EA && kind != TGXO_LD) return fail(TGXO_INVALID_ARGUMENT, "work: EA or LD");
  const int strict = ordering == TGXO_STRICTLY_SUCCEEDS;
  uint64_t ea = 0, vr = 0;
  const int ld = kind == TGXO_LD;
  const ocsr* c = ld ? &g->in : &g->out;
  for (uint32_t u = 0; u < g->n; ++u) {
    const int64_t x = labels[u];
    if (x == (ld ? NEGINF64 : INF64)) continue;
    ++vr;
    for (uint64_t e = c->off[u]; e < c->off[u + 1]; ++e) {
      const uint64_t ts = c->st[e], te = c->en[e];
      if (ts < ta || te > tb) continue;
      if (u != vertex) {
        if (ld) {
          if (strict ? (int64_t)te >= x : (int64_t)te > x) continue;
        } else {
          if (strict ? (int64_t)ts <= x : (int64_t)ts < x) continue;
        }
      }
      ++ea;
    }
  }
  *e_adm = ea;
  *v_reached = vr;
  return TGXO_OK;
}

/* Digest (FNV-1a over the little-endian label bytes), digest.hpp:12-52. */
uint64_t tgxo_digest(const int64_t* values, uint64_t n) {
  uint64_t h = 0xcbf29ce484222325ULL;
  const unsigned char* p = (const unsigned char*)values;
  for (uint64_t i = 0; i < n * 8; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

/* ------------------------------------------------------------------------
 * Selective-index cost model, selective_index.cpp:67-209 (DensityHistogram
 * build / estimate, choose_access_method) and :211-235 (fit_cost_constants).
 * Same double operations in the same order (x86-64 baseline: no FMA
 * contraction), so results are bit-identical to the reference's. */

#define HB 100 /* DensityHistogram::kBucketsPerDim, selective_index.hpp:21 */

static int bucket_of(uint64_t x, uint64_t lo, uint64_t hi, int buckets) {
  if (buckets == 1 || hi == lo) return 0;
  const unsigned __int128 num = (unsigned __int128)(x - lo) * (unsigned)buckets;
  int b = (int)(num / (hi - lo));
  if (b >= buckets) b = buckets - 1;
  return b;
}

static double dmin2(double a, double b) { return b < a ? b : a; } /* std::min */
static double dmax2(double a, double b) { return a < b ? b : a; } /* std::max */

static double region_fraction(double s0, double s1, double d0, double d1, double ta, double tb) {
  const int s_point = s1 <= s0;
  const int d_point = d1 <= d0;
  if (s_point && d_point) return (s0 >= ta && s0 + d0 <= tb) ? 1.0 : 0.0;
  if (s_point) {
    if (s0 < ta) return 0.0;
    const double dmax = dmin2(d1, tb - s0);
    if (dmax <= d0) return 0.0;
    return (dmax - d0) / (d1 - d0);
  }
  if (d_point) {
    const double a = dmax2(s0, ta);
    const double b = dmin2(s1, tb - d0);
    if (b <= a) return 0.0;
    return (b - a) / (s1 - s0);
  }
  const double a = dmax2(s0, ta);
  if (a >= s1) return 0.0;
  const double height = d1 - d0;
  const double full_hi = dmin2(s1, tb - d1);
  double area = 0.0;
  if (full_hi > a) area += (full_hi - a) * height;
  const double lin_lo = dmax2(a, tb - d1);
  const double lin_hi = dmin2(s1, tb - d0);
  if (lin_hi > lin_lo) {
    const double h_lo = tb - d0 - lin_lo;
    const double h_hi = tb - d0 - lin_hi;
    area += 0.5 * (h_lo + h_hi) * (lin_hi - lin_lo);
  }
  return area / ((s1 - s0) * height);
}

/* DensityHistogram::build + estimate over one segment [lo, hi). */
static double hist_estimate(const ocsr* c, uint64_t lo, uint64_t hi, uint64_t wta, uint64_t wtb) {
  const uint64_t total = hi - lo;
  if (total == 0) return 0.0;
  uint64_t smin = UINT64_MAX, smax = 0, dmin = UINT64_MAX, dmax = 0;
  for (uint64_t e = lo; e < hi; ++e) {
    const uint64_t d = c->en[e] - c->st[e];
    if (c->st[e] < smin) smin = c->st[e];
    if (c->st[e] > smax) smax = c->st[e];
    if (d < dmin) dmin = d;
    if (d > dmax) dmax = d;
  }
  const int sb = smin == smax ? 1 : HB;
  const int db = dmin == dmax ? 1 : HB;
  static _Thread_local uint32_t counts[HB * HB];
  static _Thread_local uint64_t rows[HB];
  memset(counts, 0, sizeof counts);
  memset(rows, 0, sizeof rows);
  for (uint64_t e = lo; e < hi; ++e) {
    const int i = bucket_of(c->st[e], smin, smax, sb);
    const int j = bucket_of(c->en[e] - c->st[e], dmin, dmax, db);
    ++counts[i * db + j];
    ++rows[i];
  }
  const double ta = (double)wta;
  const double tb = (double)wtb;
  const double s_lo = (double)smin;
  const double s_span = (double)(smax - smin);
  const double d_lo = (double)dmin;
  const double d_span = (double)(dmax - dmin);
  const double s_width = sb == 1 ? 0.0 : s_span / sb;
  const double d_width = db == 1 ? 0.0 : d_span / db;
  const double d_top = db == 1 ? d_lo : d_lo + d_span;
  double acc = 0.0;
  for (int i = 0; i < sb; ++i) {
    if (rows[i] == 0) continue;
    const double s0 = s_lo + i * s_width;
    const double s1 = sb == 1 ? s0 : s_lo + (i + 1) * s_width;
    double s_frac;
    if (s1 <= s0) {
      s_frac = s0 >= ta ? 1.0 : 0.0;
    } else {
      s_frac = (s1 - dmax2(s0, ta)) / (s1 - s0);
      s_frac = s_frac < 0.0 ? 0.0 : (1.0 < s_frac ? 1.0 : s_frac); /* std::clamp */
    }
    if (s_frac == 0.0) continue;
    if (s1 + d_top <= tb) {
      acc += (double)rows[i] * s_frac;
      continue;
    }
    for (int j = 0; j < db; ++j) {
      const uint32_t count = counts[i * db + j];
      if (count == 0) continue;
      const double d0 = d_lo + j * d_width;
      const double d1 = db == 1 ? d0 : d_lo + (j + 1) * d_width;
      acc += count * region_fraction(s0, s1, d0, d1, ta, tb);
    }
  }
  const double tot = (double)total;
  return acc < 0.0 ? 0.0 : (tot < acc ? tot : acc);
}

int tgxo_access_decisions(const tgxo_graph* g, int dir, uint64_t cutoff, uint64_t k,
                          const uint32_t* verts, const uint64_t* ta, const uint64_t* tb,
                          double theta_sel, int32_t* method, double* beta_hat, double* k_hat,
                          uint64_t* matches) {
  if (cutoff < 1) return fail(TGXO_INVALID_ARGUMENT, "index cutoff must be >= 1");
  const ocsr* c = dir == 0 ? &g->out : &g->in;
  for (uint64_t i = 0; i < k; ++i) {
    const uint32_t v = verts[i];
    if (v >= g->n) return fail(TGXO_OUT_OF_RANGE, "vertex outside vertex range");
    const uint64_t lo = c->off[v], hi = c->off[v + 1];
    uint64_t cnt = 0; /* count_in_window: window_contains, types.hpp:55-57 */
    for (uint64_t e = lo; e < hi; ++e) cnt += c->st[e] >= ta[i] && c->en[e] <= tb[i];
    matches[i] = cnt;
    if (hi - lo < cutoff) { /* no histogram: Scan, -1, -1 (selective_index.cpp:202) */
      method[i] = 1;
      beta_hat[i] = -1.0;
      k_hat[i] = -1.0;
      continue;
    }
    const double kh = hist_estimate(c, lo, hi, ta[i], tb[i]);
    const double beta = kh / (double)(hi - lo);
    method[i] = beta <= theta_sel ? 0 : 1;
    beta_hat[i] = beta;
    k_hat[i] = kh;
  }
  return TGXO_OK;
}

int tgxo_fit_cost_constants(uint64_t k, const uint64_t* degree, const uint64_t* matches,
                            const double* index_s, const double* scan_s, double* c,
                            double* c_prime) {
  if (k == 0) return fail(TGXO_INVALID_ARGUMENT, "cost calibration needs a nonempty sample");
  double num_c = 0.0, den_c = 0.0, num_cp = 0.0, den_cp = 0.0;
  for (uint64_t i = 0; i < k; ++i) {
    if (degree[i] == 0) continue;
    const double x = log2((double)degree[i]) + (double)matches[i];
    num_c += index_s[i] * x;
    den_c += x * x;
    const double y = (double)degree[i];
    num_cp += scan_s[i] * y;
    den_cp += y * y;
  }
  if (den_c == 0.0 || den_cp == 0.0)
    return fail(TGXO_INVALID_ARGUMENT, "cost calibration needs samples with degree >= 1");
  *c = num_c / den_c;
  *c_prime = num_cp / den_cp;
  return TGXO_OK;
}
