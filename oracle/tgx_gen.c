/* TEST INFRASTRUCTURE ONLY — the checker's own copy of the BASELINE
 * workload generator, so the reference arm of bench.py (and the tests) can
 * build the same edge list without loading the product library.
 *
 * The reference has no RMAT / uniform generator (ingest.cpp
 * only has a log-normal / Poisson one); the workloads follow BASELINE.json's
 * config text with SURVEY.md §8(d)'s pinned conventions. Every draw is a pure
 * function of (seed, stream, counter): a splitmix64 finaliser over
 * seed ^ mix(stream << 56 ^ counter). This file states that definition
 * independently in C; tests/test_oracle.py checks it against the product's
 * generator (tgxd_generate_host) edge for edge and against the committed
 * golden edge-list digests (tests/golden/*.npz), so the two cannot drift.
 *
 *   RMAT:    scale levels, one draw per level (stream 1, counter 64 i + lvl);
 *            quadrant a / b / c / d by cumulative thresholds floor(p 2^64);
 *            ids through a seeded 3-round xorshift-multiply-add bijection
 *            of [0, 2^scale); self-loops and duplicates kept.
 *   uniform: src / dst = mulhi(draw, n) on streams 4 / 5; self-loops dropped.
 *   start:   stream 2; uniform mulhi(draw, t_range) or floor(t_range u^(1/3))
 *            evaluated exactly (the largest s with s^3 2^64 <= r t_range^3).
 *   end:     start + 1 + Geometric(p) failures, inverse CDF over the table
 *            thr[k] = floor(2^64 (1-p)^k) (stream 3).
 */
#include "tgx_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define GEO_MAX 32768

typedef unsigned __int128 u128;

static uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

static uint64_t draw(uint64_t seed, uint64_t stream, uint64_t ctr) {
  return mix64(seed ^ mix64((stream << 56) ^ ctr));
}

static uint64_t mulhi(uint64_t a, uint64_t b) { return (uint64_t)(((u128)a * b) >> 64); }

static uint64_t threshold(long double x) {
  if (x <= 0) return 0;
  if (x >= 1) return ~0ULL;
  return (uint64_t)floorl(x * 18446744073709551616.0L);
}

typedef struct {
  const tgxo_gen_config* c;
  uint64_t ta, tab, tabc;
  uint64_t pm[3], pa[3];
  uint64_t* thr;
  int geo_len;
} genp;

static uint32_t permute(const genp* p, uint32_t v) {
  const uint32_t scale = p->c->scale;
  if (scale == 0) return 0;
  const uint64_t mask = (1ULL << scale) - 1;
  const uint32_t sh = (scale + 1) / 2;
  uint64_t x = v;
  for (int r = 0; r < 3; ++r) {
    x ^= x >> sh;
    x = (x * p->pm[r] + p->pa[r]) & mask;
  }
  return (uint32_t)x;
}

static u128 cube_shift(int64_t x) {
  const u128 c = (u128)x * (u128)x * (u128)x;
  return c << 64;
}

static uint32_t cube_root_start(uint64_t r, uint32_t t_range) {
  const double u = (double)(r >> 11) * 0x1.0p-53;
  int64_t s = (int64_t)((double)t_range * cbrt(u));
  if (s < 0) s = 0;
  const u128 rhs = (u128)r * ((u128)t_range * t_range * t_range);
  while (s > 0 && cube_shift(s) > rhs) --s;
  while ((uint64_t)(s + 1) < t_range && cube_shift(s + 1) <= rhs) ++s;
  if ((uint64_t)s >= t_range) s = t_range - 1;
  return (uint32_t)s;
}

static uint32_t geometric(const genp* p, uint64_t r) {
  int lo = 1, hi = p->geo_len; /* first k with thr[k] <= r */
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (p->thr[mid] > r) lo = mid + 1;
    else hi = mid;
  }
  return (uint32_t)(lo - 1);
}

static void edge(const genp* p, uint64_t i, uint32_t* s_out, uint32_t* d_out, uint64_t* st_out,
                 uint64_t* en_out) {
  const tgxo_gen_config* c = p->c;
  uint32_t s = 0, d = 0;
  if (c->kind == 1) {
    for (uint32_t lvl = 0; lvl < c->scale; ++lvl) {
      const uint64_t r = draw(c->seed, 1, i * 64 + lvl);
      s = (s << 1) | (r >= p->tab ? 1u : 0u);
      d = (d << 1) | (((r >= p->ta && r < p->tab) || r >= p->tabc) ? 1u : 0u);
    }
    s = permute(p, s);
    d = permute(p, d);
  } else {
    s = (uint32_t)mulhi(draw(c->seed, 4, i), c->n);
    d = (uint32_t)mulhi(draw(c->seed, 5, i), c->n);
  }
  const uint64_t rs = draw(c->seed, 2, i);
  const uint32_t st = c->start_dist == 1 ? cube_root_start(rs, c->t_range)
                                         : (uint32_t)mulhi(rs, c->t_range);
  *s_out = s;
  *d_out = d;
  *st_out = st;
  *en_out = (uint64_t)st + 1 + geometric(p, draw(c->seed, 3, i));
}

int tgxo_generate(const tgxo_gen_config* c, uint64_t capacity, uint64_t* m_out, uint32_t* src,
                  uint32_t* dst, uint64_t* start, uint64_t* end) {
  if (!c || !m_out) return TGXO_INVALID_ARGUMENT;
  if (c->t_range == 0 || c->t_range > (1u << 30)) return TGXO_INVALID_ARGUMENT;
  if (!(c->geo_p > 0.0 && c->geo_p <= 1.0)) return TGXO_INVALID_ARGUMENT;
  genp p;
  memset(&p, 0, sizeof p);
  p.c = c;
  if (c->kind == 1) {
    if (c->scale > 31) return TGXO_INVALID_ARGUMENT;
    p.ta = threshold((long double)c->a);
    p.tab = threshold((long double)c->a + (long double)c->b);
    p.tabc = threshold((long double)c->a + (long double)c->b + (long double)c->c);
    for (int r = 0; r < 3; ++r) {
      p.pm[r] = mix64(c->seed ^ (0x5851f42d4c957f2dULL * (uint64_t)(r + 1))) | 1ULL;
      p.pa[r] = mix64(c->seed + 0x14057b7ef767814fULL * (uint64_t)(r + 7));
    }
  } else if (c->kind != 0 || c->n == 0) {
    return TGXO_INVALID_ARGUMENT;
  }
  p.thr = (uint64_t*)malloc(sizeof(uint64_t) * GEO_MAX);
  if (!p.thr) return TGXO_INVALID_ARGUMENT;
  p.thr[0] = ~0ULL;
  p.geo_len = 0;
  {
    const long double q = 1.0L - (long double)c->geo_p;
    long double cur = 18446744073709551616.0L;
    for (int k = 1; k < GEO_MAX; ++k) {
      cur *= q;
      const long double f = floorl(cur);
      p.thr[k] = f >= 18446744073709551615.0L ? ~0ULL : (uint64_t)f;
      if (p.thr[k] == 0) {
        p.geo_len = k + 1;
        break;
      }
    }
  }
  if (p.geo_len == 0) {
    free(p.thr);
    return TGXO_INVALID_ARGUMENT;
  }
  const uint64_t m = c->m;
  const int drop = c->kind == 0;
  uint64_t k = 0;
  if (!drop) {
    /* RMAT: one output per draw, in parallel */
    if (src && capacity >= m) {
#pragma omp parallel for schedule(static)
      for (int64_t i = 0; i < (int64_t)m; ++i)
        edge(&p, (uint64_t)i, &src[i], &dst[i], &start[i], &end[i]);
    }
    k = m;
  } else {
    for (uint64_t i = 0; i < m; ++i) {
      uint32_t s, d;
      uint64_t a, b;
      edge(&p, i, &s, &d, &a, &b);
      if (s == d) continue;
      if (src && k < capacity) {
        src[k] = s;
        dst[k] = d;
        start[k] = a;
        end[k] = b;
      }
      ++k;
    }
  }
  free(p.thr);
  *m_out = k;
  if (src && k > capacity) return TGXO_INVALID_ARGUMENT;
  return TGXO_OK;
}
