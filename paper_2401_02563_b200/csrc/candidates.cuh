// Candidate departures of a fastest query on the device
// (path_algorithms.cpp:449-458): the distinct start times of the source's
// window out-edges. The reference collects them on the host before its
// sweep; here one CTA extracts them on the query's stream, so a fastest
// query never synchronises with the host and a hub source with tens of
// thousands of candidates costs one short kernel.
//
// A key group (equal starts) is a candidate iff klo <= key <= vhi and one of
// its edges ends by vhi (an edge of the group lies inside the window). The
// device layout orders a segment by key only (build.cuh: equal keys keep
// input order), so the group's first thread looks for such an end.
// Candidates are written in ascending key order with their whole group
// ({lo, count, key}); the sweep walks them from the top (descending,
// path_algorithms.cpp:460).
#pragma once

#include <cub/block/block_scan.cuh>

#include "tgxd_internal.cuh"

namespace tgxd {

constexpr int kCandThreads = 512;
constexpr int kCandPerThread = 4;
constexpr uint32_t kCandTile = kCandThreads * kCandPerThread;

// First index in [lo, hi) whose key is > x (keys ascending).
__device__ __forceinline__ uint32_t cand_upper(const int32_t* key, uint32_t lo, uint32_t hi,
                                               int32_t x) {
  while (lo < hi) {
    const uint32_t mid = lo + ((hi - lo) >> 1);
    if (__ldg(key + mid) <= x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

// First index in [lo, hi) whose key is >= x.
__device__ __forceinline__ uint32_t cand_lower(const int32_t* key, uint32_t lo, uint32_t hi,
                                               int32_t x) {
  while (lo < hi) {
    const uint32_t mid = lo + ((hi - lo) >> 1);
    if (__ldg(key + mid) < x) lo = mid + 1;
    else hi = mid;
  }
  return lo;
}

__global__ void __launch_bounds__(kCandThreads) candidates_kernel(
    DevCsr g, const QueryParam* qp, uint32_t src, uint32_t* cand_lo, uint32_t* cand_cnt,
    int32_t* cand_key, uint32_t* n_cand) {
  using Scan = cub::BlockScan<uint32_t, kCandThreads>;
  __shared__ typename Scan::TempStorage tmp;
  const int32_t klo = qp[0].klo, vhi = qp[0].vhi;
  const uint32_t s0 = g.off[src], s1 = g.off[src + 1];
  // only key groups inside [klo, vhi] can qualify
  const uint32_t a = cand_lower(g.key, s0, s1, klo);
  const uint32_t b = cand_upper(g.key, a, s1, vhi);
  uint32_t base = 0;
  for (uint32_t t0 = a; t0 < b; t0 += kCandTile) {
    uint32_t flag[kCandPerThread], gend[kCandPerThread];
    uint32_t cnt = 0;
#pragma unroll
    for (int k = 0; k < kCandPerThread; ++k) {
      const uint32_t j = t0 + threadIdx.x * kCandPerThread + k;
      flag[k] = 0;
      gend[k] = j;
      if (j < b) {
        const int32_t kv = __ldg(g.key + j);
        if (j == s0 || __ldg(g.key + j - 1) != kv) {  // first edge of its key group
          const uint32_t e = cand_upper(g.key, j, b, kv);
          for (uint32_t i = j; i < e; ++i)
            if ((int32_t)__ldg(&g.pay[i].y) <= vhi) {
              flag[k] = 1;
              break;
            }
          gend[k] = e;
        }
      }
      cnt += flag[k];
    }
    uint32_t pos, total;
    Scan(tmp).ExclusiveSum(cnt, pos, total);
#pragma unroll
    for (int k = 0; k < kCandPerThread; ++k) {
      if (!flag[k]) continue;
      const uint32_t j = t0 + threadIdx.x * kCandPerThread + k;
      cand_lo[base + pos] = j;
      cand_cnt[base + pos] = gend[k] - j;
      cand_key[base + pos] = __ldg(g.key + j);
      ++pos;
    }
    base += total;
    __syncthreads();  // tmp is reused by the next tile
  }
  if (threadIdx.x == 0) *n_cand = base;
}

}  // namespace tgxd
