// Deterministic temporal-graph generators shared by host (C++) and device
// (CUDA). Every draw is a pure function of (seed, stream, counter), so the
// host and device generators produce the same edge list bit for bit, and any
// edge can be regenerated independently (no sequential RNG state).
//
// The reference has no RMAT or uniform generator (ingest.cpp
// only has a log-normal/Poisson one); these follow BASELINE.json's config
// text with the conventions pinned in SURVEY.md §8(d):
//   * geometric = number of failures (support >= 0), duration = 1 + Geo(p);
//   * "start = floor(1e6 * u^(1/3))" is evaluated exactly in integers;
//   * uniform configs drop self-loops, RMAT keeps self-loops and duplicates;
//   * RMAT vertex ids go through a seeded bijection of [0, 2^scale).
#pragma once

#include <cmath>
#include <cstdint>

#ifdef __CUDACC__
#define TGX_HD __host__ __device__ __forceinline__
#else
#define TGX_HD inline
#endif

namespace tgxd {

enum GenKind : int { kGenUniform = 0, kGenRmat = 1 };
enum StartDist : int { kStartUniform = 0, kStartCubeRoot = 1 };

// Geometric inverse-CDF table: thr[k] = floor(2^64 (1-p)^k) for k >= 1
// (thr[0] unused). G = #{k >= 1 : r < thr[k]}. Built once on the host and
// shared with the device so both sides draw identical durations.
constexpr int kGeoTableMax = 32768;

struct GenParams {
  int kind;            // GenKind
  uint32_t scale;      // n = 2^scale (RMAT) ; uniform uses n_vertices
  uint32_t n_vertices;
  uint64_t m_draws;    // candidate edges drawn (uniform drops self-loops)
  uint64_t thr_a, thr_ab, thr_abc;  // RMAT cumulative quadrant thresholds * 2^64
  int start_dist;      // StartDist
  uint32_t t_range;    // starts in [0, t_range)
  uint64_t seed;
  uint64_t perm_mul[3], perm_add[3];  // vertex bijection (RMAT)
  int geo_len;         // entries of the geometric table in use
};

TGX_HD uint64_t mix64(uint64_t z) {
  z += 0x9e3779b97f4a7c15ULL;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
  return z ^ (z >> 31);
}

TGX_HD uint64_t draw(uint64_t seed, uint64_t stream, uint64_t ctr) {
  return mix64(seed ^ mix64((stream << 56) ^ ctr));
}

TGX_HD uint64_t mulhi64(uint64_t a, uint64_t b) {
#ifdef __CUDA_ARCH__
  return __umul64hi(a, b);
#else
  return (uint64_t)(((unsigned __int128)a * b) >> 64);
#endif
}

// Seeded bijection of [0, 2^scale): three rounds of xorshift, odd multiply,
// add, all mod 2^scale (each step invertible).
TGX_HD uint32_t permute_vertex(const GenParams& p, uint32_t v) {
  if (p.scale == 0) return 0;
  const uint64_t mask = (p.scale >= 64) ? ~0ULL : ((1ULL << p.scale) - 1);
  uint64_t x = v;
  const uint32_t sh = (p.scale + 1) / 2;
  for (int r = 0; r < 3; ++r) {
    x ^= x >> sh;
    x = (x * p.perm_mul[r] + p.perm_add[r]) & mask;
  }
  return (uint32_t)x;
}

// floor(1e6 * (r / 2^64)^(1/3)) exactly: the largest s with
// s^3 * 2^64 <= r * 1e18 (128-bit integer check around a double estimate).
TGX_HD uint32_t cube_root_start(uint64_t r, uint32_t t_range) {
  const double u = (double)(r >> 11) * 0x1.0p-53;
  int64_t s = (int64_t)((double)t_range * cbrt(u));
  if (s < 0) s = 0;
  const unsigned __int128 rhs = (unsigned __int128)r * ((unsigned __int128)t_range * t_range * t_range);
  auto cube_shift = [](int64_t x) -> unsigned __int128 {
    const unsigned __int128 c = (unsigned __int128)x * (unsigned __int128)x * (unsigned __int128)x;
    return c << 64;
  };
  while (s > 0 && cube_shift(s) > rhs) --s;
  while ((uint64_t)(s + 1) < t_range && cube_shift(s + 1) <= rhs) ++s;
  if ((uint64_t)s >= t_range) s = t_range - 1;
  return (uint32_t)s;
}

TGX_HD uint32_t geometric(const uint64_t* thr, int len, uint64_t r) {
  // count of k in [1, len) with r < thr[k]; thr strictly non-increasing
  int lo = 1, hi = len;  // first k with thr[k] <= r
  while (lo < hi) {
    const int mid = (lo + hi) >> 1;
    if (thr[mid] > r) lo = mid + 1;
    else hi = mid;
  }
  return (uint32_t)(lo - 1);
}

struct GenEdge {
  uint32_t src, dst;
  int32_t start, end;
};

// Candidate edge i; for uniform graphs the caller drops self-loops.
TGX_HD GenEdge gen_edge(const GenParams& p, const uint64_t* thr, uint64_t i) {
  GenEdge e;
  if (p.kind == kGenRmat) {
    uint32_t s = 0, d = 0;
    for (uint32_t lvl = 0; lvl < p.scale; ++lvl) {
      const uint64_t r = draw(p.seed, 1, i * 64 + lvl);
      const uint32_t sb = r >= p.thr_ab ? 1u : 0u;
      const uint32_t db = (r >= p.thr_a && r < p.thr_ab) || r >= p.thr_abc ? 1u : 0u;
      s = (s << 1) | sb;
      d = (d << 1) | db;
    }
    e.src = permute_vertex(p, s);
    e.dst = permute_vertex(p, d);
  } else {
    e.src = (uint32_t)mulhi64(draw(p.seed, 4, i), p.n_vertices);
    e.dst = (uint32_t)mulhi64(draw(p.seed, 5, i), p.n_vertices);
  }
  const uint64_t rs = draw(p.seed, 2, i);
  const uint32_t st = p.start_dist == kStartCubeRoot ? cube_root_start(rs, p.t_range)
                                                     : (uint32_t)mulhi64(rs, p.t_range);
  const uint32_t dur = 1u + geometric(thr, p.geo_len, draw(p.seed, 3, i));
  e.start = (int32_t)st;
  e.end = (int32_t)(st + dur);
  return e;
}

}  // namespace tgxd
