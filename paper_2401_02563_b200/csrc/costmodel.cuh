// Selective-index cost model on the device (selective_index.cpp:67-209):
// a 100 x 100 (start, duration) density histogram per indexed vertex and
// direction (DensityHistogram::build), the window-count estimate k_hat
// (DensityHistogram::estimate), beta = k_hat / degree and the decision
// beta <= theta_sel -> index lookup (choose_access_method), plus the exact
// window count (TemporalCsr::count_in_window, tcsr.cpp:124-128).
//
// Results-neutral for the traversals (their window lookup always uses the
// fence index); this serves the reference's
// estimator / calibration callers. Bit-exact: the estimate performs the
// reference's double operations in the reference's order, each rounded on
// its own (__d*_rn intrinsics: no FMA contraction — the reference is built
// for baseline x86-64, which has none).
#pragma once

#include "traverse.cuh"

namespace tgxd {

constexpr int kHistB = 100;              // DensityHistogram::kBucketsPerDim
constexpr uint32_t kNoSlot = 0xffffffffu;

struct HistHdr {
  long long smin, smax, dmin, dmax;  // start / duration extremes
  unsigned long long total;          // edges (degree)
  int sb, db;                        // buckets per dimension (1 if degenerate)
};

// Edge times of one layout position (Out: key = start, val = end; In:
// key = -end, val = -start).
__device__ __forceinline__ void edge_times(const DevCsr& g, int dir, uint32_t e, long long& s,
                                           long long& t) {
  const long long k = g.key[e];
  const long long v = (int32_t)g.pay[e].y;
  if (dir == 0) {
    s = k;
    t = v;
  } else {
    s = -v;
    t = -k;
  }
}

// bucket_of (selective_index.cpp:15-22); times fit 32 bits, so 64-bit
// arithmetic is exact.
__device__ __forceinline__ int hist_bucket(long long x, long long lo, long long hi, int buckets) {
  if (buckets == 1 || hi == lo) return 0;
  const unsigned long long num = (unsigned long long)(x - lo) * (unsigned)buckets;
  int b = (int)(num / (unsigned long long)(hi - lo));
  if (b >= buckets) b = buckets - 1;
  return b;
}

// One block per indexed vertex: extremes, then bucket counts in shared memory.
__global__ void hist_build_kernel(DevCsr g, int dir, const uint32_t* ids, HistHdr* hdr,
                                  uint32_t* counts, unsigned long long* rows) {
  extern __shared__ uint32_t s_cnt[];  // kHistB * kHistB
  __shared__ long long s_red[4][kWarps];
  __shared__ HistHdr s_h;
  const uint32_t v = ids[blockIdx.x];
  const uint32_t lo = g.off[v], hi = g.off[v + 1];
  long long smin = LLONG_MAX, smax = LLONG_MIN, dmin = LLONG_MAX, dmax = LLONG_MIN;
  for (uint32_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
    long long s, t;
    edge_times(g, dir, e, s, t);
    smin = min(smin, s);
    smax = max(smax, s);
    dmin = min(dmin, t - s);
    dmax = max(dmax, t - s);
  }
  for (int o = 16; o > 0; o >>= 1) {
    smin = min(smin, __shfl_xor_sync(0xffffffffu, smin, o));
    smax = max(smax, __shfl_xor_sync(0xffffffffu, smax, o));
    dmin = min(dmin, __shfl_xor_sync(0xffffffffu, dmin, o));
    dmax = max(dmax, __shfl_xor_sync(0xffffffffu, dmax, o));
  }
  const uint32_t w = threadIdx.x >> 5;
  if ((threadIdx.x & 31) == 0) {
    s_red[0][w] = smin;
    s_red[1][w] = smax;
    s_red[2][w] = dmin;
    s_red[3][w] = dmax;
  }
  for (uint32_t i = threadIdx.x; i < kHistB * kHistB; i += blockDim.x) s_cnt[i] = 0;
  __syncthreads();
  if (threadIdx.x == 0) {
    HistHdr h;
    h.smin = s_red[0][0];
    h.smax = s_red[1][0];
    h.dmin = s_red[2][0];
    h.dmax = s_red[3][0];
    for (int k = 1; k < kWarps; ++k) {
      h.smin = min(h.smin, s_red[0][k]);
      h.smax = max(h.smax, s_red[1][k]);
      h.dmin = min(h.dmin, s_red[2][k]);
      h.dmax = max(h.dmax, s_red[3][k]);
    }
    h.total = hi - lo;
    h.sb = h.smin == h.smax ? 1 : kHistB;
    h.db = h.dmin == h.dmax ? 1 : kHistB;
    s_h = h;
    hdr[blockIdx.x] = h;
  }
  __syncthreads();
  const HistHdr h = s_h;
  for (uint32_t e = lo + threadIdx.x; e < hi; e += blockDim.x) {
    long long s, t;
    edge_times(g, dir, e, s, t);
    const int i = hist_bucket(s, h.smin, h.smax, h.sb);
    const int j = hist_bucket(t - s, h.dmin, h.dmax, h.db);
    atomicAdd(&s_cnt[i * h.db + j], 1u);
  }
  __syncthreads();
  uint32_t* c = counts + (size_t)blockIdx.x * kHistB * kHistB;
  for (uint32_t i = threadIdx.x; i < kHistB * kHistB; i += blockDim.x) c[i] = s_cnt[i];
  for (int i = threadIdx.x; i < h.sb; i += blockDim.x) {
    unsigned long long r = 0;
    for (int j = 0; j < h.db; ++j) r += s_cnt[i * h.db + j];
    rows[(size_t)blockIdx.x * kHistB + i] = r;
  }
}

__device__ __forceinline__ double dmn(double a, double b) { return b < a ? b : a; }  // std::min
__device__ __forceinline__ double dmx(double a, double b) { return a < b ? b : a; }  // std::max

// region_fraction (selective_index.cpp:27-63).
__device__ double region_fraction_dev(double s0, double s1, double d0, double d1, double ta,
                                      double tb) {
  const bool s_point = s1 <= s0;
  const bool d_point = d1 <= d0;
  if (s_point && d_point) return (s0 >= ta && __dadd_rn(s0, d0) <= tb) ? 1.0 : 0.0;
  if (s_point) {
    if (s0 < ta) return 0.0;
    const double dmax = dmn(d1, __dsub_rn(tb, s0));
    if (dmax <= d0) return 0.0;
    return __ddiv_rn(__dsub_rn(dmax, d0), __dsub_rn(d1, d0));
  }
  if (d_point) {
    const double a = dmx(s0, ta);
    const double b = dmn(s1, __dsub_rn(tb, d0));
    if (b <= a) return 0.0;
    return __ddiv_rn(__dsub_rn(b, a), __dsub_rn(s1, s0));
  }
  const double a = dmx(s0, ta);
  if (a >= s1) return 0.0;
  const double height = __dsub_rn(d1, d0);
  const double full_hi = dmn(s1, __dsub_rn(tb, d1));
  double area = 0.0;
  if (full_hi > a) area = __dadd_rn(area, __dmul_rn(__dsub_rn(full_hi, a), height));
  const double lin_lo = dmx(a, __dsub_rn(tb, d1));
  const double lin_hi = dmn(s1, __dsub_rn(tb, d0));
  if (lin_hi > lin_lo) {
    const double h_lo = __dsub_rn(__dsub_rn(tb, d0), lin_lo);
    const double h_hi = __dsub_rn(__dsub_rn(tb, d0), lin_hi);
    area = __dadd_rn(area, __dmul_rn(__dmul_rn(0.5, __dadd_rn(h_lo, h_hi)),
                                     __dsub_rn(lin_hi, lin_lo)));
  }
  return __ddiv_rn(area, __dmul_rn(__dsub_rn(s1, s0), height));
}

// DensityHistogram::estimate (selective_index.cpp:98-142).
__device__ double hist_estimate_dev(const HistHdr& h, const uint32_t* counts,
                                    const unsigned long long* rows, unsigned long long wta,
                                    unsigned long long wtb) {
  if (h.total == 0) return 0.0;
  const double ta = __ull2double_rn(wta);
  const double tb = __ull2double_rn(wtb);
  const double s_lo = __ll2double_rn(h.smin);
  const double s_span = __ll2double_rn(h.smax - h.smin);
  const double d_lo = __ll2double_rn(h.dmin);
  const double d_span = __ll2double_rn(h.dmax - h.dmin);
  const double s_width = h.sb == 1 ? 0.0 : __ddiv_rn(s_span, (double)h.sb);
  const double d_width = h.db == 1 ? 0.0 : __ddiv_rn(d_span, (double)h.db);
  const double d_top = h.db == 1 ? d_lo : __dadd_rn(d_lo, d_span);
  double acc = 0.0;
  for (int i = 0; i < h.sb; ++i) {
    if (rows[i] == 0) continue;
    const double s0 = __dadd_rn(s_lo, __dmul_rn((double)i, s_width));
    const double s1 = h.sb == 1 ? s0 : __dadd_rn(s_lo, __dmul_rn((double)(i + 1), s_width));
    double s_frac;
    if (s1 <= s0) {
      s_frac = s0 >= ta ? 1.0 : 0.0;
    } else {
      s_frac = __ddiv_rn(__dsub_rn(s1, dmx(s0, ta)), __dsub_rn(s1, s0));
      s_frac = s_frac < 0.0 ? 0.0 : (1.0 < s_frac ? 1.0 : s_frac);  // std::clamp
    }
    if (s_frac == 0.0) continue;
    if (__dadd_rn(s1, d_top) <= tb) {
      acc = __dadd_rn(acc, __dmul_rn(__ull2double_rn(rows[i]), s_frac));
      continue;
    }
    for (int j = 0; j < h.db; ++j) {
      const uint32_t count = counts[i * h.db + j];
      if (count == 0) continue;
      const double d0 = __dadd_rn(d_lo, __dmul_rn((double)j, d_width));
      const double d1 = h.db == 1 ? d0 : __dadd_rn(d_lo, __dmul_rn((double)(j + 1), d_width));
      acc = __dadd_rn(acc, __dmul_rn((double)count, region_fraction_dev(s0, s1, d0, d1, ta, tb)));
    }
  }
  const double tot = __ull2double_rn(h.total);
  return acc < 0.0 ? 0.0 : (tot < acc ? tot : acc);
}

// One warp per (vertex, window): the lanes count the window-contained edges
// (window_contains, types.hpp:55-57); lane 0 runs the estimate and the
// decision (choose_access_method, selective_index.cpp:200-209).
__global__ void access_decision_kernel(DevCsr g, int dir, uint32_t k, const uint32_t* verts,
                                       const unsigned long long* ta, const unsigned long long* tb,
                                       double theta, const uint32_t* slot, const HistHdr* hdr,
                                       const uint32_t* counts, const unsigned long long* rows,
                                       int32_t* method, double* beta, double* khat,
                                       unsigned long long* matches) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  for (uint32_t q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; q < k; q += nw) {
    const uint32_t v = verts[q];
    const unsigned long long a = ta[q], b = tb[q];
    // times are in [0, 2^31 - 2]: the window's ends compare exactly as int64
    const long long la = a > (1ull << 62) ? (1ll << 62) : (long long)a;
    const long long lb = b > (1ull << 62) ? (1ll << 62) : (long long)b;
    const uint32_t lo = g.off[v], hi = g.off[v + 1];
    unsigned long long cnt = 0;
    for (uint32_t e = lo + lane; e < hi; e += 32) {
      long long s, t;
      edge_times(g, dir, e, s, t);
      cnt += (s >= la && t <= lb) ? 1 : 0;
    }
    for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
    if (lane == 0) {
      matches[q] = cnt;
      const uint32_t sl = slot[v];
      if (sl == kNoSlot) {  // no histogram: Scan, -1, -1
        method[q] = 1;
        beta[q] = -1.0;
        khat[q] = -1.0;
      } else {
        const HistHdr h = hdr[sl];
        const double kh = hist_estimate_dev(h, counts + (size_t)sl * kHistB * kHistB,
                                            rows + (size_t)sl * kHistB, a, b);
        const double bt = h.total == 0 ? 0.0 : __ddiv_rn(kh, __ull2double_rn(h.total));
        method[q] = bt <= theta ? 0 : 1;
        beta[q] = bt;
        khat[q] = kh;
      }
    }
  }
}

}  // namespace tgxd
