// Asynchronous (barrier-free) traversal — the same fixpoint as traverse.cuh
// without rounds.
//
// Every warp loops over two multi-producer / multi-consumer ring queues:
//   CQ  edge chunks (up to kAChunk edges of one vertex's admissible range),
//   VQ  vertex slots whose label improved since their last expansion.
// A warp pops a chunk and relaxes it, or pops up to 32 vertices, expands
// them (the same key-range search and selective index as the round kernel),
// relaxes their short ranges itself (packed 32 ranges per warp) and pushes
// long ranges to CQ as chunks. Improved vertices are enqueued once per
// improvement "epoch": a per-slot queued flag is set with atomicExch by the
// improver and cleared (then fenced) by the expander before it reads the
// label, so no improvement is ever left unexpanded.
//
// Work efficiency is unchanged: an expansion only walks keys in
// [bound, previous bound), so every admissible edge is relaxed once per
// query (concurrent expansions of one vertex can at worst repeat a range,
// which is idempotent). Labels are the unique least fixpoint
// — bit-identical to the reference.
//
// Termination: `pending` counts items that exist (queued, staged or being
// processed). Producers add before publishing; a warp subtracts what it has
// completed only when it is idle with empty staging buffers, so pending
// reaches zero exactly when all work is done.
#pragma once

#include <cooperative_groups.h>

#include "traverse.cuh"

namespace tgxd {

constexpr uint32_t kAChunk = 512;        // edges per async chunk (4 x 128-edge bursts)
constexpr uint32_t kAInline = 64;        // shorter ranges are relaxed by the expanding warp
constexpr uint32_t kAChunkLenBits = 10;  // len <= 512
constexpr uint32_t kEmpty = 0xffffffffu;

struct alignas(128) PaddedCounter {
  unsigned long long v;
  unsigned long long pad[15];
};

struct AsyncCtl {
  PaddedCounter vhead, vtail, chead, ctail, pending;
  unsigned int abort;
  unsigned int error;
  unsigned long long expansions;
  unsigned long long edges;
  unsigned long long index_lookups;
  unsigned long long vpops, cpops;
  unsigned long long bad[4];  // TGXD_VALIDATE: first violation {kind, a, b, c}
};

struct AsyncArgs {
  DevCsr g;
  const QueryParam* qp;
  int32_t* X;
  int2* EP;
  int32_t* R;
  uint32_t* flag;   // per slot: 1 while queued
  uint32_t* vq;     // vertex ring, kEmpty when free
  uint2* cq;        // chunk ring, .y == kEmpty when free
  uint32_t vmask, cmask;
  AsyncCtl* c;
  uint32_t n, Q;
  int strict;
  uint32_t cutoff;
  int fastest;
  uint32_t n_cand;
  const uint32_t* cand_lo;
  const uint32_t* cand_cnt;
  const int32_t* cand_key;
  unsigned long long time_limit_ns;  // watchdog
};

__device__ __forceinline__ void st_volatile(uint32_t* p, uint32_t v) {
  *reinterpret_cast<volatile uint32_t*>(p) = v;
}
__device__ __forceinline__ uint32_t ld_volatile(const uint32_t* p) {
  return *reinterpret_cast<const volatile uint32_t*>(p);
}

// Per-warp staging of vertex pushes (64 entries of shared memory).
struct VBuf {
  uint32_t* buf;
  uint32_t n;  // warp-uniform
};

__device__ __forceinline__ void vq_flush(const AsyncArgs& a, VBuf& vb, uint32_t count) {
  const uint32_t lane = lane_id();
  __syncwarp();
  const uint32_t v = vb.buf[lane];
  const uint32_t tail = vb.buf[32 + lane];
  unsigned long long base = 0;
  if (lane == 0) {
    atomicAdd(&a.c->pending.v, (unsigned long long)count);  // before the items exist
    __threadfence();
    base = atomicAdd(&a.c->vtail.v, (unsigned long long)count);
  }
  base = __shfl_sync(0xffffffffu, base, 0);
  if (lane < count) st_volatile(a.vq + ((base + lane) & a.vmask), v);
  __syncwarp();
  if (lane + count < vb.n) vb.buf[lane] = tail;
  vb.n -= count;
  __syncwarp();
}

__device__ __forceinline__ void vq_append(const AsyncArgs& a, VBuf& vb, bool p, uint32_t item) {
  const uint32_t bal = __ballot_sync(0xffffffffu, p);
  if (bal == 0) return;
  if (p) vb.buf[vb.n + __popc(bal & ((1u << lane_id()) - 1))] = item;
  vb.n += __popc(bal);
  if (vb.n >= 32) vq_flush(a, vb, 32);
}

struct ARelax {
  int32_t vhi0;
  int32_t depart;
  uint64_t pol_stream, pol_keep;
};

// Relax kUnroll 32-edge steps (see relax_steps in traverse.cuh); an
// improvement enqueues its vertex when the queued flag was clear.
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
  int32_t cur[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    const int32_t vhi = a.Q == 1 ? rx.vhi0 : __ldg(&a.qp[q[u]].vhi);
#ifdef TGXD_VALIDATE
    if (act[u] && __ldg(a.g.key + e[u]) < a.qp[q[u]].klo && atomicCAS(&a.c->bad[0], 0ull, 1ull) == 0)
      a.c->bad[1] = e[u], a.c->bad[2] = (unsigned long long)(long long)__ldg(a.g.key + e[u]),
      a.c->bad[3] = q[u];
#endif
    if (!(act[u] && v[u] <= vhi)) v[u] = kInf;  // window containment (types.hpp:55-57)
    cur[u] = v[u] != kInf ? ld_state(a.X + idx[u], rx.pol_keep) : kInf;
  }
  int32_t old[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u)
    old[u] = v[u] < cur[u] ? atomicMin(a.X + idx[u], v[u]) : kInf;  // write_min
  uint32_t was[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    was[u] = 1u;
    if (v[u] < old[u]) {
      if (a.R) atomicMin(a.R + idx[u], v[u] - rx.depart);
      was[u] = atomicExch(a.flag + idx[u], 1u);
    }
  }
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) vq_append(a, vb, was[u] == 0u, idx[u]);
}

// Relax ranges given one per lane (lo, cnt, q), packed 32 per warp: lane l
// owns range l, items are numbered densely and each lane finds its owner
// from the redux.or mask of range starts (as phase_b's small windows).
__device__ __forceinline__ void relax_ranges_packed(const AsyncArgs& a, uint32_t lo, uint32_t cnt,
                                                    uint32_t rq, const ARelax& rx, VBuf& vb) {
  const uint32_t lane = lane_id();
  // compact the non-empty ranges into the low lanes: the owner search below
  // needs range l in lane l
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
// seed range), 128 edges per step.
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

// Expansion of up to 32 popped slots (one per lane).
__device__ __forceinline__ void expand_batch(const AsyncArgs& a, bool valid, uint32_t item,
                                             const ARelax& rx, VBuf& vb,
                                             unsigned long long& work, unsigned long long& ix) {
  const uint32_t lane = lane_id();
  uint32_t q = 0, p0 = 0, p1 = 0;
  bool act = false;
  if (valid) {
    // clear the queued flag before reading the label: an improvement after
    // this point re-enqueues the slot
    st_volatile(a.flag + item, 0u);
    __threadfence();
    const int32_t x = __ldcg(a.X + item);
    const int2 ep = __ldcg(a.EP + item);
    q = a.Q == 1 ? 0u : item / a.n;
    const uint32_t v = item - q * a.n;
    const QueryParam& qp = a.qp[q];
    int32_t lb = (v == qp.root) ? qp.klo : bound_of(x, a.strict);
    if (lb < qp.klo) lb = qp.klo;
    const int32_t old = ep.x;
    if (x != kInf && lb < old) {
      const int32_t hik = min(old, qp.vhi + 1);
      uint32_t pos = kNoPos;
      if (lb < hik) {
        const uint32_t s = __ldg(a.g.off + v), t = __ldg(a.g.off + v + 1);
        if (t > s) {
          act = true;
          const bool fence = a.cutoff != 0 && t - s >= a.cutoff;
          ix += fence ? 1 : 0;
          if (old <= qp.vhi + 1 && ep.y != (int32_t)kNoPos) {
            p1 = (uint32_t)ep.y;
          } else {
            p1 = __ldg(a.g.key + t - 1) < hik ? t : lane_lower_bound(a.g, s, t, hik, fence);
          }
          p0 = p1 > s ? lane_lower_bound(a.g, s, p1, lb, fence) : s;
          pos = p0;
#ifdef TGXD_VALIDATE
          bool badr = p0 > p1 || p1 > t || p0 < s;
          if (!badr && p0 < p1) badr = __ldg(a.g.key + p0) < lb || __ldg(a.g.key + p1 - 1) >= hik;
          if (!badr && p0 > s) badr = __ldg(a.g.key + p0 - 1) >= lb;
          if (badr && atomicCAS(&a.c->bad[0], 0ull, 2ull) == 0)
            a.c->bad[1] = item, a.c->bad[2] = ((unsigned long long)p0 << 32) | p1,
            a.c->bad[3] = ((unsigned long long)(uint32_t)lb << 32) | (uint32_t)hik;
#endif
        }
      }
      a.EP[item] = make_int2(lb, (int32_t)pos);
    }
  }
  const uint32_t cnt = act ? p1 - p0 : 0u;
  work += cnt;
  // long ranges: chunks to CQ (one reservation for the whole warp)
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
    if (lane == 0) {
      atomicAdd(&a.c->pending.v, (unsigned long long)tot);
      __threadfence();
      base = atomicAdd(&a.c->ctail.v, (unsigned long long)tot);
    }
    base = __shfl_sync(0xffffffffu, base, 0) + incl - nch;
    for (uint32_t j = 0; j < nch; ++j)  // payload words first ...
      a.cq[(base + j) & a.cmask].x = p0 + j * kAChunk;
    __threadfence();
    for (uint32_t j = 0; j < nch; ++j)  // ... then the words that publish them
      st_volatile(&a.cq[(base + j) & a.cmask].y,
                  (q << kAChunkLenBits) | min(kAChunk, cnt - j * kAChunk));
  }
  // short ranges: relaxed right here
  const bool inl = cnt != 0 && cnt < kAInline;
  if (__any_sync(0xffffffffu, inl))
    relax_ranges_packed(a, inl ? p0 : 0u, inl ? cnt : 0u, q, rx, vb);
}

// Claims up to `want` consecutive queue positions; returns how many (uniform).
__device__ __forceinline__ uint32_t claim(unsigned long long* head, unsigned long long* tailp,
                                          uint32_t want, unsigned long long& h_out) {
  unsigned long long h = 0;
  uint32_t take = 0;
  if (lane_id() == 0) {
    h = __ldcg(head);
    const unsigned long long t = __ldcg(tailp);
    if (t > h) {
      take = (uint32_t)((t - h) < want ? (t - h) : want);
      if (atomicCAS(head, h, h + take) != h) take = 0;
    }
  }
  take = __shfl_sync(0xffffffffu, take, 0);
  h_out = __shfl_sync(0xffffffffu, h, 0);
  return take;
}

__device__ void async_loop(const AsyncArgs& a, const ARelax& rx, VBuf& vb,
                           unsigned long long t_deadline, unsigned long long& done,
                           unsigned long long& work, unsigned long long& ix,
                           unsigned long long& vpops, unsigned long long& cpops) {
  const uint32_t lane = lane_id();
  uint32_t idle_ns = 0;
  for (;;) {
    if (ld_volatile(&a.c->abort)) return;
    unsigned long long h;
    // chunks first: edge work that is ready
    if (claim(&a.c->chead.v, &a.c->ctail.v, 1, h)) {
      uint2* slot = a.cq + (h & a.cmask);
      uint32_t y = kEmpty;
      uint32_t x = 0;
      if (lane == 0) {
        while ((y = ld_volatile(&slot->y)) == kEmpty) {}
        __threadfence();
        x = ld_volatile(&slot->x);
        st_volatile(&slot->y, kEmpty);
      }
      y = __shfl_sync(0xffffffffu, y, 0);
      x = __shfl_sync(0xffffffffu, x, 0);
      relax_span(a, x, y & ((1u << kAChunkLenBits) - 1), y >> kAChunkLenBits, rx, vb);
      ++done;
      ++cpops;
      idle_ns = 0;
      continue;
    }
    const uint32_t take = claim(&a.c->vhead.v, &a.c->vtail.v, 32, h);
    if (take) {
      uint32_t item = 0;
      if (lane < take) {
        uint32_t* slot = a.vq + ((h + lane) & a.vmask);
        while ((item = ld_volatile(slot)) == kEmpty) {}
        st_volatile(slot, kEmpty);
      }
      expand_batch(a, lane < take, item, rx, vb, work, ix);
      done += take;
      ++vpops;
      idle_ns = 0;
      continue;
    }
    // idle: publish staged pushes and completed work, then test for the end
    if (vb.n) vq_flush(a, vb, vb.n);
    if (done) {
      if (lane == 0) {
        __threadfence();
        atomicAdd(&a.c->pending.v, (unsigned long long)(0ull - done));
      }
      done = 0;
      continue;  // look again before sleeping: others may be waiting on us
    }
    unsigned long long p = 0;
    if (lane == 0) p = __ldcg(&a.c->pending.v);
    p = __shfl_sync(0xffffffffu, p, 0);
    if (p == 0) return;
    if (idle_ns) __nanosleep(idle_ns);
    idle_ns = min(2 * idle_ns + 64, 2048u);
    if (lane == 0 && gtimer() > t_deadline) {
      a.c->error = 1;
      a.c->abort = 1;
    }
  }
}

__global__ void __launch_bounds__(kThreads, TGXD_MIN_BLOCKS) async_kernel(AsyncArgs a) {
  __shared__ uint32_t s_vb[kWarps][64];
  cg::grid_group grid = cg::this_grid();
  VBuf vb{s_vb[threadIdx.x >> 5], 0};
  const unsigned long long t_deadline = gtimer() + a.time_limit_ns;
  ARelax rx{a.qp[0].vhi, 0, policy_evict_first(), policy_evict_last()};
  unsigned long long done = 0, work = 0, ix = 0, vpops = 0, cpops = 0;
  const uint32_t gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint32_t nw = gridDim.x * kWarps;
  if (!a.fastest) {
    async_loop(a, rx, vb, t_deadline, done, work, ix, vpops, cpops);
  } else {
    for (uint32_t cand = 0; cand < a.n_cand; ++cand) {
      // Seeds (path_algorithms.cpp:476-486): the candidate's first edges,
      // relaxed without an admissibility check, 128-edge pieces over warps.
      rx.depart = a.cand_key[cand];
      const uint32_t lo = a.cand_lo[cand], cnt = a.cand_cnt[cand];
      const uint32_t pieces = (cnt + 127) / 128;
      const uint32_t mine = gw < pieces ? (pieces - gw + nw - 1) / nw : 0u;
      grid.sync();  // the previous candidate is fully drained everywhere
      if (lane_id() == 0 && mine) atomicAdd(&a.c->pending.v, (unsigned long long)mine);
      grid.sync();  // no warp sees pending == 0 before all seeds are counted
      for (uint32_t pc = gw; pc < pieces; pc += nw) {
        relax_span(a, lo + pc * 128, min(128u, cnt - pc * 128), 0, rx, vb);
        ++done;
      }
      async_loop(a, rx, vb, t_deadline, done, work, ix, vpops, cpops);
      if (ld_volatile(&a.c->abort)) break;
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    work += __shfl_xor_sync(0xffffffffu, work, o);
    ix += __shfl_xor_sync(0xffffffffu, ix, o);
  }
  if (lane_id() == 0) {
    if (work) atomicAdd(&a.c->edges, work);
    if (ix) atomicAdd(&a.c->index_lookups, ix);
    if (vpops) atomicAdd(&a.c->vpops, vpops);
    if (cpops) atomicAdd(&a.c->cpops, cpops);
  }
}

// Seeds of an async EA / LD query: X[root] = klo, roots queued.
__global__ void async_seed_kernel(const QueryParam* qp, uint32_t Q, uint32_t n, int32_t* X,
                                  uint32_t* flag, uint32_t* vq, uint32_t vmask, AsyncCtl* c,
                                  int fastest) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  c->abort = 0;
  c->error = 0;
  c->edges = 0;
  c->index_lookups = 0;
  c->vpops = 0;
  c->cpops = 0;
  c->bad[0] = c->bad[1] = c->bad[2] = c->bad[3] = 0;
  c->pending.v = 0;
  c->vhead.v = c->vtail.v;
  c->chead.v = c->ctail.v;
  if (fastest) return;
  const unsigned long long t = c->vtail.v;
  for (uint32_t q = 0; q < Q; ++q) {
    const uint32_t item = q * n + qp[q].root;
    X[item] = qp[q].klo;
    flag[item] = 1u;
    vq[(t + q) & vmask] = item;
  }
  c->vtail.v = t + Q;
  c->pending.v = Q;
}

// After a watchdog abort the rings and flags may hold stale entries.
__global__ void async_reset_kernel(uint32_t* flag, size_t slots, uint32_t* vq, size_t vcap,
                                   uint2* cq, size_t ccap, AsyncCtl* c) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < slots; i += stride) flag[i] = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < vcap; i += stride) vq[i] = kEmpty;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < ccap; i += stride)
    cq[i] = make_uint2(0u, kEmpty);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    c->vhead.v = c->vtail.v = c->chead.v = c->ctail.v = 0;
    c->pending.v = 0;
  }
}

}  // namespace tgxd
