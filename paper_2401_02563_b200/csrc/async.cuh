// Asynchronous (barrier-free) traversal — the same fixpoint as traverse.cuh
// without rounds.
//
// All warps share ONE ticket queue of 64-byte work units:
//   * a vertex batch — up to kBatch slots whose label improved since their
//     last expansion, or
//   * an edge chunk — up to kAChunk edges of one vertex's admissible range.
// A warp takes the next ticket with one atomicAdd, waits on that unit's
// header (its own address: no hot spot), and processes it: a chunk is
// relaxed; a batch is expanded (the same key-range search and selective
// index as the round kernel), its short ranges relaxed by the warp itself
// (packed 32 ranges per warp) and its long ranges published as chunks.
// Label and "queued" bit share one 64-bit word per slot (XQ): an improver
// lowers the label and sets the bit in one CAS and enqueues the slot only if
// the bit was clear; the expander clears the bit with atomicAnd, whose
// return value is the label it expands with. All of it is ordered by the
// coherence of that single address — no fences — so no improvement is ever
// left unexpanded. Labels are copied back to X when the query is done.
//
// Work efficiency is unchanged: an expansion only walks keys in
// [bound, previous bound), so every admissible edge is relaxed once per
// query (concurrent expansions of one vertex can at worst repeat a range,
// which is idempotent). Labels are the unique least fixpoint
// — bit-identical to the reference.
//
// Termination: `tail` counts published units, `completed` finished ones. A
// warp adds its finished units only while it waits with nothing staged, so
// `completed` can equal `tail` only when no unit is unfinished (a
// producer's own unit always completes after what it published). The warp
// whose addition makes them equal raises `quiesce`; waiting warps abandon
// their tickets (the next query or candidate restarts the queue at its tail).
#pragma once

#include <cooperative_groups.h>

#include "traverse.cuh"

namespace tgxd {

#ifndef TGXD_ASYNC_SLEEP
#define TGXD_ASYNC_SLEEP 256  // ns between polls of a long-waiting ticket
#endif
#ifndef TGXD_A_CHUNK
#define TGXD_A_CHUNK 512
#endif
#ifndef TGXD_A_INLINE
#define TGXD_A_INLINE 64
#endif
constexpr uint32_t kAChunk = TGXD_A_CHUNK;    // edges per chunk unit (4 x 128-edge bursts)
constexpr uint32_t kAInline = TGXD_A_INLINE;  // shorter ranges are relaxed by the expanding warp
constexpr uint32_t kUnitWords = 16;      // 64-byte units
constexpr uint32_t kBatch = kUnitWords - 1;  // vertices per batch unit
constexpr uint32_t kEmpty = 0xffffffffu;
constexpr uint32_t kChunkTag = 0x80000000u;  // header: tag | q << 10 | len (len <= 512)

struct alignas(128) PaddedCounter {
  unsigned long long v;
  unsigned long long pad[15];
};

struct AsyncCtl {
  PaddedCounter head, tail, completed;  // units claimed / published / finished
  alignas(128) unsigned int quiesce;  // epoch whose work is complete
  unsigned int abort;
  unsigned int error;
  unsigned int pad0;
  unsigned long long edges;
  unsigned long long index_lookups;
  unsigned long long visits;  // vertex expansions (for_each_window_edge calls)
  unsigned long long batches, chunks;
  unsigned long long wait_ns, busy_ns, t_first, t_last;  // time accounting
  unsigned long long t_entry, t_loop;  // handoff: kernel entry, queue ready
  unsigned long long bad[4];  // TGXD_VALIDATE: first violation {kind, a, b, c}
};

struct AsyncArgs {
  DevCsr g;
  const QueryParam* qp;
  int32_t* X;       // final labels (copied from XQ at the end)
  unsigned long long* XQ;  // per slot: label << 32 | queued bit
  int2* EP;
  int32_t* R;
  uint32_t* units;  // ring of 64-byte units, header word kEmpty when free
  unsigned long long umask;
  AsyncCtl* c;
  uint32_t n, Q;
  int strict;
  uint32_t cutoff;
  int fastest;
  const uint32_t* n_cand;  // device count (candidates.cuh), ascending lists
  const uint32_t* cand_lo;
  const uint32_t* cand_cnt;
  const int32_t* cand_key;
  unsigned long long time_limit_ns;  // watchdog
  // host results copied early (api.cu): every label the tail lowers is
  // listed here (slot ids, repeats allowed) so the host can patch its copy
  uint32_t* chg;
  unsigned long long* chg_n;
  unsigned long long chg_cap;
  // tail handoff from the round kernel: its frontier queue and labels
  const Control* hctl;  // nullptr: a query of its own
  const uint32_t* hfa;
  const uint32_t* hfb;
  uint32_t hfresh;       // the round kernel's queue-item mark (cleared on read)
};

__device__ __forceinline__ void st_volatile(uint32_t* p, uint32_t v) {
  *reinterpret_cast<volatile uint32_t*>(p) = v;
}
__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
  return *reinterpret_cast<const volatile uint32_t*>(p);
}
// Release / acquire primitives (PTX memory model): cheaper than the full
// fences they replace, and exactly the orderings the handoffs need.
__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
// Label word: (label with its sign bit flipped) << 32 | queued bit, so the
// unsigned order of words is the signed order of labels (LD labels are
// negative in key space) and one 64-bit atomicMin both lowers the label and
// sets the bit.
__device__ __forceinline__ unsigned long long xq_pack(int32_t label, uint32_t queued) {
  return ((unsigned long long)((uint32_t)label ^ 0x80000000u) << 32) | queued;
}
__device__ __forceinline__ int32_t xq_label(unsigned long long w) {
  return (int32_t)((uint32_t)(w >> 32) ^ 0x80000000u);
}

__device__ __forceinline__ uint32_t* unit_ptr(const AsyncArgs& a, unsigned long long pos) {
  return a.units + (pos & a.umask) * kUnitWords;
}

// Reserves k units (one atomic on the publish counter).
__device__ __forceinline__ unsigned long long reserve_units(const AsyncArgs& a, uint32_t k) {
  return atomicAdd(&a.c->tail.v, (unsigned long long)k);
}

// Per-warp staging of vertex pushes (64 entries of shared memory).
struct VBuf {
  uint32_t* buf;
  uint32_t n;  // warp-uniform
};

// Publishes the first `count` (<= kBatch) staged vertices as one batch unit.
__device__ __forceinline__ void vb_publish(const AsyncArgs& a, VBuf& vb, uint32_t count) {
  const uint32_t lane = lane_id();
  __syncwarp();
  const uint32_t v = vb.buf[lane];
  const uint32_t rest = vb.buf[(lane + count) & 63];
  unsigned long long pos = 0;
  if (lane == 0) pos = reserve_units(a, 1);
  pos = __shfl_sync(0xffffffffu, pos, 0);
  uint32_t* u = unit_ptr(a, pos);
  if (lane < count) u[1 + lane] = v;
  __syncwarp();                            // payload words happen-before ...
  if (lane == 0) st_release(u, count);     // ... the releasing header store
  if (lane + count < vb.n) vb.buf[lane] = rest;
  vb.n -= count;
  __syncwarp();
}

__device__ __forceinline__ void vb_append(const AsyncArgs& a, VBuf& vb, bool p, uint32_t item) {
  const uint32_t bal = __ballot_sync(0xffffffffu, p);
  if (bal == 0) return;
  if (p) vb.buf[vb.n + __popc(bal & ((1u << lane_id()) - 1))] = item;
  vb.n += __popc(bal);
  while (vb.n >= kBatch) vb_publish(a, vb, kBatch);
}

struct ARelax {
  int32_t vhi0;
  int32_t depart;
  uint64_t pol_stream, pol_keep;
};

// Relax kUnroll 32-edge steps (see relax_steps in traverse.cuh); an
// improvement enqueues its vertex when its queued bit was clear.
__device__ __forceinline__ void relax_async(const AsyncArgs& a, const uint32_t (&e)[kUnroll],
                                            const uint32_t (&q)[kUnroll],
                                            const bool (&act)[kUnroll], const ARelax& rx,
                                            VBuf& vb) {
  int32_t v[kUnroll];
  uint32_t idx[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    const uint2 pl = act[u] ? ld_stream2(a.g.pay + e[u], rx.pol_stream) : make_uint2(0u, kInf);
    idx[u] = q[u] * a.n + pl.x;
    v[u] = (int32_t)pl.y;
  }
  unsigned long long cur[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    const int32_t vhi = a.Q == 1 ? rx.vhi0 : __ldg(&a.qp[q[u]].vhi);
#ifdef TGXD_VALIDATE
    if (act[u] && __ldg(a.g.key + e[u]) < a.qp[q[u]].klo && atomicCAS(&a.c->bad[0], 0ull, 1ull) == 0)
      a.c->bad[1] = e[u], a.c->bad[2] = (unsigned long long)(long long)__ldg(a.g.key + e[u]),
      a.c->bad[3] = q[u];
#endif
    if (!(act[u] && v[u] <= vhi)) v[u] = kInf;  // window containment (types.hpp:55-57)
    cur[u] = v[u] != kInf ? __ldcg(a.XQ + idx[u]) : xq_pack(kInf, 1u);
  }
  // write_min (parallel.hpp:91-99) and the queued bit in one 64-bit
  // atomicMin: a lower label wins whatever the bit, and the new word carries
  // the bit set; all atomics of the batch are issued before any result is used
  bool imp[kUnroll];
  uint32_t was[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    imp[u] = v[u] < xq_label(cur[u]);
    was[u] = 1u;
    if (imp[u]) {
      const unsigned long long prev = atomicMin(a.XQ + idx[u], xq_pack(v[u], 1u));
      imp[u] = v[u] < xq_label(prev);
      if (imp[u]) was[u] = (uint32_t)(prev & 1ull);
    }
  }
  if (a.chg) {  // every label the tail lowers, for the early host copy's patch
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t m = __ballot_sync(0xffffffffu, imp[u]);
      if (m == 0) continue;
      unsigned long long cb = 0;
      if (lane_id() == 0) cb = atomicAdd(a.chg_n, (unsigned long long)__popc(m));
      cb = __shfl_sync(0xffffffffu, cb, 0) + __popc(m & ((1u << lane_id()) - 1));
      if (imp[u] && cb < a.chg_cap) a.chg[cb] = idx[u];
    }
  }
#pragma unroll
  for (int u = 0; u < kUnroll; ++u)
    if (imp[u] && a.R) atomicMin(a.R + idx[u], v[u] - rx.depart);
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) vb_append(a, vb, was[u] == 0u, idx[u]);
#if TGXD_PF_ASYNC
#pragma unroll
  for (int u = 0; u < kUnroll; ++u)
    if (was[u] == 0u) prefetch_expansion<TGXD_PF_ASYNC>(a.g.okm, a.g.key, a.g.pay, idx[u] - q[u] * a.n);
#endif
}

// Relax ranges given one per lane (lo, cnt, q), packed 32 per warp: range l
// sits in lane l, items are numbered densely and each lane finds its owner
// from the redux.or mask of range starts (as phase_b's small windows).
__device__ __forceinline__ void relax_ranges_packed(const AsyncArgs& a, uint32_t lo, uint32_t cnt,
                                                    uint32_t rq, const ARelax& rx, VBuf& vb) {
  const uint32_t lane = lane_id();
  // compact the non-empty ranges into the low lanes
  const uint32_t nz = __ballot_sync(0xffffffffu, cnt != 0);
  const uint32_t k = __popc(nz);
  const uint32_t src = lane < k ? __fns(nz, 0, lane + 1) : 0u;
  lo = __shfl_sync(0xffffffffu, lo, src);
  rq = __shfl_sync(0xffffffffu, rq, src);
  cnt = __shfl_sync(0xffffffffu, cnt, src);
  if (lane >= k) cnt = 0;
  uint32_t incl = cnt;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const uint32_t start = incl - cnt;
  const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
  for (uint32_t base = 0; base < total; base += 32 * kUnroll) {
    uint32_t e[kUnroll], q[kUnroll];
    bool act[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t sb = base + u * 32;
      const uint32_t before = __ballot_sync(0xffffffffu, cnt != 0 && start <= sb);
      const uint32_t i0 = before ? 31 - __clz(before) : 0;
      const uint32_t rel = start - sb;
      const uint32_t bit = (cnt != 0 && start > sb && rel < 32) ? (1u << rel) : 0u;
      const uint32_t mask = __reduce_or_sync(0xffffffffu, bit);
      const uint32_t own = (i0 + __popc(mask & ((2u << lane) - 1))) & 31;
      const uint32_t olo = __shfl_sync(0xffffffffu, lo, own);
      const uint32_t ost = __shfl_sync(0xffffffffu, start, own);
      const uint32_t oq = __shfl_sync(0xffffffffu, rq, own);
      const uint32_t t = sb + lane;
      act[u] = t < total;
      e[u] = olo + (t - ost);
      q[u] = oq;
    }
    relax_async(a, e, q, act, rx, vb);
  }
}

// Relax one contiguous range [lo, lo + len) of query slot q (a chunk, or a
// seed piece), 128 edges per step.
__device__ __forceinline__ void relax_span(const AsyncArgs& a, uint32_t lo, uint32_t len,
                                           uint32_t q, const ARelax& rx, VBuf& vb) {
  const uint32_t lane = lane_id();
  for (uint32_t b = 0; b < len; b += 32 * kUnroll) {
    uint32_t e[kUnroll], qq[kUnroll];
    bool act[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t off = b + u * 32 + lane;
      act[u] = off < len;
      e[u] = lo + off;
      qq[u] = q;
    }
    relax_async(a, e, qq, act, rx, vb);
  }
}

// Expansion of one batch (one slot per lane, `valid` lanes only).
__device__ __forceinline__ void expand_batch(const AsyncArgs& a, bool valid, uint32_t item,
                                             const ARelax& rx, VBuf& vb,
                                             unsigned long long& work, unsigned long long& ix) {
  const uint32_t lane = lane_id();
  uint32_t q = 0, p0 = 0, p1 = 0;
  bool act = false;
  if (valid) {
    // clear the queued bit; the returned word holds the label to expand
    // with (an improvement after this point re-enqueues the slot)
    q = a.Q == 1 ? 0u : item / a.n;
    const uint32_t v = item - q * a.n;
    // label, bounds and the segment's extent all issued together
    const int32_t x = xq_label(atomicAnd(a.XQ + item, ~1ull));
    const int2 ep = __ldcg(a.EP + item);
#if TGXD_OKM_ENGINES
    // segment bounds and last key from one {off, kmax} line
    const uint2 ok = __ldg(a.g.okm + v);
    const uint32_t s = ok.x, t = __ldg(&a.g.okm[v + 1].x);
    const int32_t km = (int32_t)ok.y;
#else
    const uint32_t s = __ldg(a.g.off + v), t = __ldg(a.g.off + v + 1);
    const int32_t km = __ldg(a.g.kmax + v);  // no key at or above lb: nothing to do
#endif
    const QueryParam& qp = a.qp[q];
    // min_start / max_end hooks (path_algorithms.cpp:287-291, :337-342)
    int32_t lb = (v == qp.root) ? qp.klo : bound_of(x, a.strict);
    if (lb < qp.klo) lb = qp.klo;
    const int32_t old = ep.x;
    if (x != kInf && lb < old) {
      const int32_t hik = min(old, qp.vhi + 1);
      uint32_t pos = kNoPos;
      if (lb < hik) {
        ix += 1ull << 32;  // a vertex expansion (high word), index lookups (low word)
        if (t > s && km >= lb) {
          act = true;
          const bool fence = a.cutoff != 0 && t - s >= a.cutoff;
          ix += fence ? 1 : 0;
          if (old <= qp.vhi + 1 && ep.y != (int32_t)kNoPos) {
            p1 = (uint32_t)ep.y;
          } else {
            p1 = km < hik ? t : lane_lower_bound(a.g, s, t, hik, fence);
          }
          p0 = p1 > s ? lane_lower_bound(a.g, s, p1, lb, fence) : s;
          pos = p0;
        }
      }
      a.EP[item] = make_int2(lb, (int32_t)pos);
    }
  }
  const uint32_t cnt = act ? p1 - p0 : 0u;
  work += cnt;
  // long ranges: chunk units (one reservation for the whole warp)
  const uint32_t nch = cnt >= kAInline ? (cnt + kAChunk - 1) / kAChunk : 0u;
  uint32_t incl = nch;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += y;
  }
  const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
  if (tot) {
    unsigned long long base = 0;
    if (lane == 0) base = reserve_units(a, tot);
    base = __shfl_sync(0xffffffffu, base, 0) + incl - nch;
    for (uint32_t j = 0; j < nch; ++j) {
      uint32_t* cu = unit_ptr(a, base + j);
      cu[1] = p0 + j * kAChunk;
      st_release(cu, kChunkTag | (q << 10) | min(kAChunk, cnt - j * kAChunk));
    }
  }
  // short ranges: relaxed right here
  const bool inl = cnt != 0 && cnt < kAInline;
  if (__any_sync(0xffffffffu, inl))
    relax_ranges_packed(a, inl ? p0 : 0u, inl ? cnt : 0u, q, rx, vb);
}

// Takes tickets and processes their units until the epoch's work is done.
__device__ void async_loop(const AsyncArgs& a, const ARelax& rx, VBuf& vb, uint32_t epoch,
                           unsigned long long t_deadline, unsigned long long& done,
                           unsigned long long& work, unsigned long long& ix,
                           unsigned long long& nb, unsigned long long& nc,
                           unsigned long long& wait_ns, unsigned long long& busy_ns) {
  const uint32_t lane = lane_id();
  for (;;) {
    const unsigned long long t0 = gtimer();
    unsigned long long h = 0;
    if (lane == 0) h = atomicAdd(&a.c->head.v, 1ull);
    h = __shfl_sync(0xffffffffu, h, 0);
    uint32_t* u = unit_ptr(a, h);
    uint32_t hdr = kEmpty;
    uint32_t polls = 0;
    for (;;) {  // wait for the ticket's unit
      if (lane == 0) hdr = ld_acquire(u);
      hdr = __shfl_sync(0xffffffffu, hdr, 0);
      if (hdr != kEmpty) break;
      // nothing staged or unsubtracted may be held while waiting
      if (vb.n) {
        vb_publish(a, vb, vb.n);
        continue;
      }
      if (done) {
        // completions are published lazily, only from here: `completed`
        // can reach `tail` only when no unit is unfinished (a producer's own
        // unit completes after everything it published was reserved)
        if (lane == 0) {
          const unsigned long long c = atomicAdd(&a.c->completed.v, done) + done;
          if (c == __ldcg(&a.c->tail.v)) st_volatile(&a.c->quiesce, epoch);
        }
        done = 0;
        continue;
      }
      ++polls;
      uint32_t stop = 0;
      if (lane == 0 && (polls & 15) == 0) {
        stop = ld_volatile(&a.c->quiesce) == epoch || ld_volatile(&a.c->abort);
        if (!stop && gtimer() > t_deadline) {
          a.c->error = 1;
          st_volatile(&a.c->abort, 1u);
          stop = 1;
        }
      }
      if (__shfl_sync(0xffffffffu, stop, 0)) {
        wait_ns += gtimer() - t0;
        return;
      }
      __nanosleep(polls < 64 ? 64 : TGXD_ASYNC_SLEEP);
    }
    const unsigned long long t1 = gtimer();
    wait_ns += t1 - t0;
    __syncwarp();  // lane 0's acquire orders the payload reads of every lane
    if (hdr & kChunkTag) {
      const uint32_t lo = ld_volatile(u + 1);
      __syncwarp();
      if (lane == 0) st_volatile(u, kEmpty);
      relax_span(a, lo, hdr & 1023u, (hdr & ~kChunkTag) >> 10, rx, vb);
      ++nc;
    } else {
      const uint32_t item = lane < hdr ? ld_volatile(u + 1 + lane) : 0u;
      __syncwarp();
      if (lane == 0) st_volatile(u, kEmpty);
      expand_batch(a, lane < hdr, item, rx, vb, work, ix);
      ++nb;
    }
    ++done;
    busy_ns += gtimer() - t1;
  }
}

__global__ void __launch_bounds__(kThreads, TGXD_MIN_BLOCKS) async_kernel(AsyncArgs a) {
  __shared__ uint32_t s_vb[kWarps][64];
  cg::grid_group grid = cg::this_grid();
  VBuf vb{s_vb[threadIdx.x >> 5], 0};
  const unsigned long long t_deadline = gtimer() + a.time_limit_ns;
  ARelax rx{a.qp[0].vhi, 0, policy_evict_first(), policy_evict_last()};
  unsigned long long done = 0, work = 0, ix = 0, nb = 0, nc = 0, wait_ns = 0, busy_ns = 0;
  const uint32_t gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint32_t nw = gridDim.x * kWarps;
  if (a.hctl) {
    // Continuation of a round-kernel query (traverse.cuh, tail handoff):
    // labels become label words, the handed-over queue becomes batch units.
    const unsigned long long nh = __ldcg(&a.hctl->handoff_n);
    // the round kernel finished the query itself, or handed it to the
    // cluster engine
    if (nh == 0 || __ldcg(&a.hctl->handoff_kind) != 2) return;
    if (blockIdx.x == 0 && threadIdx.x == 0) a.c->t_entry = gtimer();
    const uint32_t* fin = __ldcg(&a.hctl->handoff_flip) ? a.hfb : a.hfa;
    const unsigned long long t0 = __ldcg(&a.c->tail.v);
    const size_t slots = (size_t)a.Q * a.n;
    const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t nthr = (size_t)gridDim.x * blockDim.x;
    // label words from the labels, 4 slots per thread and step (16-byte
    // accesses; X and XQ are 256-byte aligned allocations)
    for (size_t i = tid; i < slots / 4; i += nthr) {
      const int4 x = reinterpret_cast<const int4*>(a.X)[i];
      ulonglong2* d = reinterpret_cast<ulonglong2*>(a.XQ) + 2 * i;
      d[0] = make_ulonglong2(xq_pack(x.x, 0u), xq_pack(x.y, 0u));
      d[1] = make_ulonglong2(xq_pack(x.z, 0u), xq_pack(x.w, 0u));
    }
    for (size_t i = slots / 4 * 4 + tid; i < slots; i += nthr) a.XQ[i] = xq_pack(a.X[i], 0u);
    grid.sync();
    for (size_t k = tid; k < nh; k += nthr) {
      const uint32_t item = __ldcg(fin + k) & ~a.hfresh;  // (round kernel's marks)
      a.XQ[item] = xq_pack(a.X[item], 1u);
      uint32_t* u = unit_ptr(a, t0 + k / kBatch);
      u[1 + k % kBatch] = item;
      if (k % kBatch == 0) u[0] = (uint32_t)min((unsigned long long)kBatch, nh - k);
    }
    if (tid == 0) {
      a.c->abort = 0;
      a.c->error = 0;
      a.c->quiesce = 0;
      a.c->edges = a.c->index_lookups = a.c->visits = a.c->batches = a.c->chunks = 0;
      a.c->wait_ns = a.c->busy_ns = 0;
      a.c->head.v = a.c->completed.v = t0;
      a.c->tail.v = t0 + (nh + kBatch - 1) / kBatch;
      a.c->t_last = 0;
    }
    grid.sync();
    if (tid == 0) a.c->t_loop = gtimer();
    async_loop(a, rx, vb, 1, t_deadline, done, work, ix, nb, nc, wait_ns, busy_ns);
  } else if (!a.fastest) {
    async_loop(a, rx, vb, 1, t_deadline, done, work, ix, nb, nc, wait_ns, busy_ns);
  } else {
    const uint32_t n_cand = __ldcg(a.n_cand);
    for (uint32_t cand = 0; cand < n_cand; ++cand) {
      // Seeds (path_algorithms.cpp:476-486): the candidate's first edges,
      // relaxed without an admissibility check, 128-edge pieces over warps
      // (descending: the lists are ascending).
      const uint32_t ci = n_cand - 1 - cand;
      rx.depart = a.cand_key[ci];
      const uint32_t lo = a.cand_lo[ci], cnt = a.cand_cnt[ci];
      const uint32_t pieces = (cnt + 127) / 128;
      const uint32_t mine = gw < pieces ? (pieces - gw + nw - 1) / nw : 0u;
      grid.sync();  // the previous candidate is drained everywhere
      if (blockIdx.x == 0 && threadIdx.x == 0) {
        // drop idle tickets; the seed pieces count as work to complete
        a.c->head.v = a.c->tail.v;
        a.c->completed.v = a.c->tail.v - pieces;
      }
      grid.sync();
      for (uint32_t pc = gw; pc < pieces; pc += nw) {
        relax_span(a, lo + pc * 128, min(128u, cnt - pc * 128), 0, rx, vb);
        ++done;
      }
      async_loop(a, rx, vb, cand + 1, t_deadline, done, work, ix, nb, nc, wait_ns, busy_ns);
      if (ld_volatile(&a.c->abort)) break;
    }
  }
  if (lane_id() == 0) atomicMax(&a.c->t_last, gtimer());
  grid.sync();  // every label is final: copy them out (4 slots per thread and step)
  {
    const size_t slots = (size_t)a.Q * a.n;
    const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
    const size_t nthr = (size_t)gridDim.x * blockDim.x;
    for (size_t i = tid; i < slots / 4; i += nthr) {
      const ulonglong2* q = reinterpret_cast<const ulonglong2*>(a.XQ) + 2 * i;
      const ulonglong2 w0 = __ldcg(q), w1 = __ldcg(q + 1);
      reinterpret_cast<int4*>(a.X)[i] =
          make_int4(xq_label(w0.x), xq_label(w0.y), xq_label(w1.x), xq_label(w1.y));
    }
    for (size_t i = slots / 4 * 4 + tid; i < slots; i += nthr) a.X[i] = xq_label(__ldcg(a.XQ + i));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    work += __shfl_xor_sync(0xffffffffu, work, o);
    ix += __shfl_xor_sync(0xffffffffu, ix, o);
  }
  if (lane_id() == 0) {
    if (work) atomicAdd(&a.c->edges, work);
    if (ix & 0xffffffffull) atomicAdd(&a.c->index_lookups, ix & 0xffffffffull);
    if (ix >> 32) atomicAdd(&a.c->visits, ix >> 32);
    if (nb) atomicAdd(&a.c->batches, nb);
    if (nc) atomicAdd(&a.c->chunks, nc);
    atomicAdd(&a.c->wait_ns, wait_ns);
    atomicAdd(&a.c->busy_ns, busy_ns);
  }
}

// Query start: counters, and for EA / LD the roots as the first batch units.
__global__ void async_seed_kernel(const QueryParam* qp, uint32_t Q, uint32_t n,
                                  unsigned long long* XQ, uint32_t* units,
                                  unsigned long long umask, AsyncCtl* c, int fastest) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  c->abort = 0;
  c->error = 0;
  c->quiesce = 0;
  c->edges = 0;
  c->index_lookups = 0;
  c->visits = 0;
  c->batches = 0;
  c->chunks = 0;
  c->wait_ns = 0;
  c->busy_ns = 0;
  c->bad[0] = c->bad[1] = c->bad[2] = c->bad[3] = 0;
  c->head.v = c->tail.v;  // tickets left waiting by the previous query are void
  c->completed.v = c->tail.v;
  if (fastest) return;
  unsigned long long t = c->tail.v;
  uint32_t nu = 0;
  for (uint32_t q0 = 0; q0 < Q; q0 += kBatch, ++nu) {
    uint32_t* u = units + ((t + nu) & umask) * kUnitWords;
    const uint32_t k = min(kBatch, Q - q0);
    for (uint32_t j = 0; j < k; ++j) {
      const uint32_t item = (q0 + j) * n + qp[q0 + j].root;
      XQ[item] = ((unsigned long long)((uint32_t)qp[q0 + j].klo ^ 0x80000000u) << 32) | 1ull;
      u[1 + j] = item;
    }
    u[0] = k;
  }
  c->tail.v = t + nu;
}

// The tail's changed labels for the host (mapped memory): out[0] = count,
// then {slot, label} pairs (count <= cap; a larger count means the host
// copies the labels again).
__global__ void tail_patch_kernel(const uint32_t* chg, const unsigned long long* chg_n,
                                  unsigned long long cap, const int32_t* X,
                                  unsigned long long* out) {
  const unsigned long long n = *chg_n;
  const unsigned long long k = n < cap ? n : cap;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < k; i += stride) {
    const uint32_t v = chg[i];
    out[1 + i] = (unsigned long long)v | ((unsigned long long)(uint32_t)X[v] << 32);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) out[0] = n;
}

// Fresh (or post-abort) queue state: every unit free.
__global__ void async_reset_kernel(uint32_t* units, size_t nunits, AsyncCtl* c) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nunits; i += stride)
    units[i * kUnitWords] = kEmpty;
  if (blockIdx.x == 0 && threadIdx.x == 0) c->head.v = c->tail.v = c->completed.v = 0;
}

// Per-query label words: INF, not queued.
__global__ void async_init_kernel(unsigned long long* XQ, size_t slots) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const unsigned long long w = (unsigned long long)((uint32_t)kInf ^ 0x80000000u) << 32;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < slots; i += stride) XQ[i] = w;
}

}  // namespace tgxd
