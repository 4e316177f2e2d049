// Cluster tail engine: the last, thin rounds of an EA / LD traversal on ONE
// thread-block cluster (16 CTAs x 1024 threads, non-portable size; 8 when 16
// does not fit), synchronised by the cluster barrier instead of a grid
// barrier.
//
// After its heavy rounds a query's frontier shrinks over a dozen or more
// dependent rounds that each relax a few thousand edges (config 2: 160K ->
// 58K -> 24K -> ... -> 6 vertices). On the full grid every such round pays
// two grid barriers, counter reads through L2 and the phases' completion
// spread (~20 us per round for a 200-vertex frontier, against ~7 us for the
// same work on one CTA). Here a round is:
//
//   1. every warp takes 32 frontier slots, expands them (the same key-range
//      search, expansion bounds and selective index as traverse.cuh) and
//      relaxes the short ranges itself, 32 edges per step packed over the
//      warp's lanes; ranges longer than kTailInline edges become 128-edge
//      chunks in a list;
//   2. (only when the round emitted chunks) one cluster barrier, then every
//      warp relaxes chunks;
//   3. one cluster barrier; the next frontier's size is read from CTA 0's
//      shared memory (the counters live there: pushes and chunks are
//      distributed-shared-memory atomics, no L2 round trip).
//
// Expansion and relaxation run concurrently within a round, so the round
// engine's "first improvement" rule (bound(old) == Ex) does not hold here;
// instead an improved slot is queued when its stamp for this round is
// claimed (atomicExch: the reference's claim_stamp, parallel.hpp:113-121).
// A slot improved while it is being expanded is simply expanded again next
// round (the second expansion walks only [new bound, old bound)), so the
// result is the same least fixpoint and every admissible edge is still
// relaxed once.
#pragma once

#include <cooperative_groups.h>

#include "traverse.cuh"

namespace tgxd {

constexpr int kTailThreads = 1024;
constexpr int kTailWarps = kTailThreads / 32;
constexpr uint32_t kTailInline = 96;   // longer ranges go to the chunk list
constexpr uint32_t kTailChunk = 128;   // edges per chunk

struct TailCtl {
  unsigned int epoch;        // stamp base: every round of every tail run has its own value
  unsigned int rounds;       // rounds of the last run
  unsigned int error;        // watchdog
  unsigned int pad;
  unsigned long long edges;  // edges handed to the relax step
  unsigned long long visits; // vertex expansions
  unsigned long long index_lookups;
  unsigned long long t_entry, t_end;
};

struct TailArgs {
  DevCsr g;
  const QueryParam* qp;
  int32_t* X;
  int2* EP;
  uint32_t* fa;              // frontier queues (the round kernel's)
  uint32_t* fb;
  uint2* chunks;             // {lo, q << 10 | len}
  uint32_t* stamp;           // per slot: round it was last queued (epoch-based)
  const Control* hctl;       // the round kernel's handoff: size and queue parity
  TailCtl* tc;
  uint32_t n, Q;
  int strict;
  uint32_t cutoff;
  uint32_t round_limit;
  unsigned long long slots;
  uint32_t fresh;            // the round kernel's queue-item mark (cleared on read)
  // early host copy: every slot the tail lowers is listed (api.cu)
  uint32_t* chg;
  unsigned long long* chg_n;
  unsigned long long chg_cap;
  // optional per-round trace (mapped host memory, rows after the round
  // kernel's): t0, t after phase 1, t end, F, chunks, -, -, kind 4
  unsigned long long* trace;
  uint32_t trace_cap;
};

__device__ __forceinline__ void tail_trace(const TailArgs& a, uint32_t row, int slot,
                                           unsigned long long v) {
  if (a.trace && row < a.trace_cap) {
    volatile unsigned long long* t = a.trace;
    t[row * 8 + slot] = v;
  }
}

namespace cgt = cooperative_groups;

// kTailU relax steps of 32 edges (lane's edge f[u] of query q[u] when
// act[u]), every load and atomic of the batch in flight together; the
// improved slots whose stamp this round claims are queued with one DSMEM
// reservation for the whole batch.
constexpr int kTailU = 4;
__device__ __forceinline__ void tail_relax(const TailArgs& a, const bool (&act)[kTailU],
                                           const uint32_t (&f)[kTailU],
                                           const uint32_t (&q)[kTailU], uint32_t epoch,
                                           uint64_t pol_stream, uint64_t pol_keep,
                                           unsigned long long* push_cnt, uint32_t* fout) {
  uint2 pl[kTailU];
#pragma unroll
  for (int u = 0; u < kTailU; ++u)
    pl[u] = act[u] ? ld_stream2(a.g.pay + f[u], pol_stream) : make_uint2(0u, (uint32_t)kInf);
  uint32_t d[kTailU];
  int32_t v[kTailU], cur[kTailU];
#pragma unroll
  for (int u = 0; u < kTailU; ++u) {
    d[u] = q[u] * a.n + pl[u].x;
    v[u] = (int32_t)pl[u].y;
    const int32_t vhi = a.Q == 1 ? a.qp[0].vhi : __ldg(&a.qp[q[u]].vhi);
    if (!(act[u] && v[u] <= vhi)) v[u] = kInf;  // window containment, types.hpp:55-57
    cur[u] = v[u] != kInf ? ld_state(a.X + d[u], pol_keep) : kInf;
  }
  int32_t old[kTailU];
#pragma unroll
  for (int u = 0; u < kTailU; ++u)
    old[u] = v[u] < cur[u] ? atomicMin(a.X + d[u], v[u]) : v[u];  // write_min, parallel.hpp:91-99
  bool imp[kTailU], push[kTailU];
#pragma unroll
  for (int u = 0; u < kTailU; ++u) {
    imp[u] = v[u] < old[u];
    // claim_stamp (parallel.hpp:113-121): queued once per round
    push[u] = imp[u] && atomicExch(a.stamp + d[u], epoch) != epoch;
  }
  const uint32_t lane = lane_id();
  const uint32_t below = (1u << lane) - 1;
  uint32_t pm[kTailU], tot = 0;
#pragma unroll
  for (int u = 0; u < kTailU; ++u) {
    pm[u] = __ballot_sync(0xffffffffu, push[u]);
    tot += __popc(pm[u]);
  }
  if (tot) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(push_cnt, (unsigned long long)tot);
    base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
    for (int u = 0; u < kTailU; ++u) {
      if (push[u]) fout[base + __popc(pm[u] & below)] = d[u];
      base += __popc(pm[u]);
    }
#if TGXD_PF_TAIL
#pragma unroll
    for (int u = 0; u < kTailU; ++u)
      if (push[u]) prefetch_expansion<TGXD_PF_TAIL>(a.g.okm, a.g.key, a.g.pay, pl[u].x);
#endif
  }
  if (a.chg) {  // early host copy: every lowered slot is listed
    uint32_t im[kTailU], itot = 0;
#pragma unroll
    for (int u = 0; u < kTailU; ++u) {
      im[u] = __ballot_sync(0xffffffffu, imp[u]);
      itot += __popc(im[u]);
    }
    if (itot) {
      unsigned long long base = 0;
      if (lane == 0) base = atomicAdd(a.chg_n, (unsigned long long)itot);
      base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
      for (int u = 0; u < kTailU; ++u) {
        const unsigned long long k = base + __popc(im[u] & below);
        if (imp[u] && k < a.chg_cap) a.chg[k] = d[u];
        base += __popc(im[u]);
      }
    }
  }
}

__global__ void __launch_bounds__(kTailThreads, 1) tail_kernel(TailArgs a) {
  // CTA 0's counters, reached by every CTA of the cluster through DSMEM:
  // pushes of the round's output queue (3 rotating slots: the one a round
  // reads, the one it fills, the one rank 0 clears for the next round) and
  // chunks emitted in the round (same rotation)
  __shared__ unsigned long long s_cnt[6];
  cgt::cluster_group cluster = cgt::this_cluster();
  const unsigned long long nh = __ldcg(&a.hctl->handoff_n);
  // the round kernel finished the query itself, or handed it to the async
  // engine (uniform)
  if (nh == 0 || __ldcg(&a.hctl->handoff_kind) != 1) return;
  const uint32_t rank = cluster.block_rank();
  const uint32_t ncta = cluster.num_blocks();
  const bool lead = rank == 0 && threadIdx.x == 0;
  if (threadIdx.x < 6) s_cnt[threadIdx.x] = threadIdx.x == 0 ? nh : 0ull;
  unsigned long long* cnt = cluster.map_shared_rank(s_cnt, 0);
  const uint32_t lane = lane_id();
  const uint32_t gw = rank * kTailWarps + (threadIdx.x >> 5);
  const uint32_t nw = ncta * kTailWarps;
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();
  uint32_t base_epoch = __ldcg(&a.tc->epoch);
  if (base_epoch > 0xe0000000u) {  // stamps would wrap: start them over
    for (unsigned long long i = (unsigned long long)rank * kTailThreads + threadIdx.x; i < a.slots;
         i += (unsigned long long)ncta * kTailThreads)
      a.stamp[i] = 0;
    base_epoch = 0;
  }
  if (lead) a.tc->t_entry = gtimer();
  cluster.sync();
  uint32_t* qin = __ldcg(&a.hctl->handoff_flip) ? a.fb : a.fa;
  uint32_t* qout = qin == a.fa ? a.fb : a.fa;
  unsigned long long work = 0, ix = 0;
  uint32_t r = 0;
  const uint32_t row0 = a.trace ? __ldcg(&a.hctl->rounds) : 0u;
  for (;; ++r) {
    const unsigned long long F = *(volatile unsigned long long*)&cnt[r % 3];
    if (lead) {
      tail_trace(a, row0 + r, 0, gtimer());
      tail_trace(a, row0 + r, 3, F);
      tail_trace(a, row0 + r, 7, 4);
    }
    if (F == 0) break;
    if (r >= a.round_limit) {
      if (lead) a.tc->error = 1;
      break;
    }
    if (lead) {  // the slots round r + 1 fills next were last read in round r - 1
      cnt[(r + 2) % 3] = 0;
      cnt[3 + (r + 2) % 3] = 0;
    }
    unsigned long long* push_cnt = &cnt[(r + 1) % 3];
    unsigned long long* ch_cnt = &cnt[3 + r % 3];
    const uint32_t epoch = base_epoch + r + 1;
    // (1) each warp expands up to 32 slots (spread over all warps when the
    // frontier is small) and relaxes their short ranges in place
    const uint32_t ipw = (uint32_t)min(32ull, max(1ull, (F + nw - 1) / nw));
    for (unsigned long long b = (unsigned long long)gw * ipw; b < F; b += (unsigned long long)nw * ipw) {
      const unsigned long long i = b + lane;
      uint32_t q = 0, p0 = 0, cnt_e = 0;
      if (lane < ipw && i < F) {
        const uint32_t item = __ldcg(qin + i) & ~a.fresh;  // (round kernel's marks)
        q = a.Q == 1 ? 0u : item / a.n;
        const uint32_t v = item - q * a.n;
        const int32_t x = ld_state(a.X + item, pol_keep);
        const int2 ep = __ldcg(a.EP + item);
#if TGXD_OKM_ENGINES
        // segment bounds and last key from one {off, kmax} line
        const uint2 ok = __ldg(a.g.okm + v);
        const uint32_t s = ok.x, t = __ldg(&a.g.okm[v + 1].x);
        const int32_t km = (int32_t)ok.y;
#else
        const uint32_t s = __ldg(a.g.off + v), t = __ldg(a.g.off + v + 1);
        const int32_t km = __ldg(a.g.kmax + v);
#endif
        const QueryParam& qp = a.qp[q];
        // min_start / max_end hooks (path_algorithms.cpp:287-291, :337-342)
        int32_t lb = (v == qp.root) ? qp.klo : bound_of(x, a.strict);
        if (lb < qp.klo) lb = qp.klo;
        const int32_t old = ep.x;
        if (x != kInf && lb < old) {
          const int32_t hik = min(old, qp.vhi + 1);
          uint32_t pos = kNoPos, p1 = 0;
          if (lb < hik) {
            ix += 1ull << 32;
            if (t > s && km >= lb) {
              const bool fence = a.cutoff != 0 && t - s >= a.cutoff;
              ix += fence ? 1 : 0;
              if (old <= qp.vhi + 1 && ep.y != (int32_t)kNoPos) p1 = (uint32_t)ep.y;
              else p1 = km < hik ? t : lane_lower_bound(a.g, s, t, hik, fence);
              p0 = p1 > s ? lane_lower_bound(a.g, s, p1, lb, fence) : s;
              pos = p0;
              cnt_e = p1 - p0;
            }
          }
          a.EP[item] = make_int2(lb, (int32_t)pos);
        }
      }
      work += cnt_e;
      // long ranges -> chunks (warp-cooperative, one reservation per 32)
      const bool big = cnt_e > kTailInline;
      uint32_t bigs = __ballot_sync(0xffffffffu, big);
      while (bigs) {
        const uint32_t src = __ffs(bigs) - 1;
        bigs &= bigs - 1;
        const uint32_t B0 = __shfl_sync(0xffffffffu, p0, src);
        const uint32_t BC = __shfl_sync(0xffffffffu, cnt_e, src);
        const uint32_t BQ = __shfl_sync(0xffffffffu, q, src);
        const uint32_t bn = (BC + kTailChunk - 1) / kTailChunk;
        for (uint32_t k0 = 0; k0 < bn; k0 += 32) {
          const uint32_t m = min(32u, bn - k0);
          unsigned long long cb = 0;
          if (lane == 0) cb = atomicAdd(ch_cnt, (unsigned long long)m);
          cb = __shfl_sync(0xffffffffu, cb, 0);
          if (lane < m) {
            const uint32_t off = (k0 + lane) * kTailChunk;
            a.chunks[cb + lane] = make_uint2(B0 + off, (BQ << 10) | min(kTailChunk, BC - off));
          }
        }
      }
      // short ranges: the warp's ranges packed 32 edges per step, kTailU
      // steps in flight (the owner lane of edge t is found from the mask of
      // range starts)
      const uint32_t c = big ? 0u : cnt_e;
      uint32_t incl = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= (uint32_t)o) incl += y;
      }
      const uint32_t start = incl - c;
      const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
      const uint32_t nonempty = __ballot_sync(0xffffffffu, c != 0);
      for (uint32_t sb0 = 0; sb0 < total; sb0 += 32 * kTailU) {
        bool act[kTailU];
        uint32_t f[kTailU], oqs[kTailU];
#pragma unroll
        for (int u = 0; u < kTailU; ++u) {
          const uint32_t sb = sb0 + 32 * u;
          const uint32_t before = __ballot_sync(0xffffffffu, c != 0 && start <= sb);
          const uint32_t i0 = before ? 31 - __clz(before) : 0;
          const uint32_t rel = start - sb;
          const uint32_t bit = (c != 0 && start > sb && rel < 32) ? (1u << rel) : 0u;
          const uint32_t mask = __reduce_or_sync(0xffffffffu, bit);
          const uint32_t k = __popc(mask & ((2u << lane) - 1));
          const uint32_t own = k ? __fns(nonempty, i0, (int)k + 1) & 31 : i0;
          const uint32_t olo = __shfl_sync(0xffffffffu, p0, own);
          const uint32_t ost = __shfl_sync(0xffffffffu, start, own);
          oqs[u] = __shfl_sync(0xffffffffu, q, own);
          const uint32_t tt = sb + lane;
          act[u] = tt < total;
          f[u] = olo + (tt - ost);
        }
        tail_relax(a, act, f, oqs, epoch, pol_stream, pol_keep, push_cnt, qout);
      }
    }
    cluster.sync();
    // (2) chunks, when the round emitted any (the count is final after the barrier)
    const unsigned long long nch = *(volatile unsigned long long*)ch_cnt;
    if (lead) {
      tail_trace(a, row0 + r, 1, gtimer());
      tail_trace(a, row0 + r, 4, nch);
    }
    if (nch) {
      static_assert(kTailChunk == 32 * kTailU, "a chunk is one relax batch");
      for (unsigned long long cix = gw; cix < nch; cix += nw) {
        const uint2 ch = __ldcg(a.chunks + cix);
        const uint32_t cq = ch.y >> 10, len = ch.y & 1023u;
        bool act[kTailU];
        uint32_t f[kTailU], qs[kTailU];
#pragma unroll
        for (int u = 0; u < kTailU; ++u) {
          act[u] = 32 * u + lane < len;
          f[u] = ch.x + 32 * u + lane;
          qs[u] = cq;
        }
        tail_relax(a, act, f, qs, epoch, pol_stream, pol_keep, push_cnt, qout);
      }
      cluster.sync();
    }
    if (lead) tail_trace(a, row0 + r, 2, gtimer());
    uint32_t* tq = qin;
    qin = qout;
    qout = tq;
  }
  // the loop leaves with every CTA past the same barrier; sum the counters
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    work += __shfl_xor_sync(0xffffffffu, work, o);
    ix += __shfl_xor_sync(0xffffffffu, ix, o);
  }
  if (lane == 0) {
    if (work) atomicAdd(&a.tc->edges, work);
    if (ix & 0xffffffffull) atomicAdd(&a.tc->index_lookups, ix & 0xffffffffull);
    if (ix >> 32) atomicAdd(&a.tc->visits, ix >> 32);
  }
  if (lead) {
    a.tc->rounds = r;
    a.tc->epoch = base_epoch + r + 2;
    a.tc->t_end = gtimer();
  }
  cluster.sync();  // no CTA leaves while others may still touch CTA 0's counters
}

// Query start: the tail's statistics (the epoch persists across queries).
__global__ void tail_reset_kernel(TailCtl* tc) {
  tc->rounds = 0;
  tc->error = 0;
  tc->edges = tc->visits = tc->index_lookups = 0;
}

}  // namespace tgxd
