// Shortest duration under Succeeds / StrictlySucceeds, priced per out-edge.
//
// The reference relaxes edge states (shortest_duration_edges,
// path_algorithms.cpp:205-258): every reached edge e scans all out-edges of
// its head that start after it ends. Under the two "succeeds" orderings the
// best predecessor of an out-edge g of w depends only on g.start:
//
//   value[g] = (g.end - g.start) + B_w(g.start),
//   B_w(t)   = min{ value[e] : e reached in-edge of w, e.end < t (strict) or
//                   e.end <= t (weak) }     (value = duration for the root's edges)
//
// In w's In segment (key = -end ascending) the in-edges ending before t form
// a suffix [lower_bound(1 - t), end) (weak: lower_bound(-t)), so B_w is a
// suffix minimum of a per-position array that only ever decreases: a
// Fenwick tree per segment (suffix-min, point decrease) answers it in
// O(log deg) independent loads and takes an improvement in O(log deg)
// atomicMins. A round re-prices the window out-edges of the vertices whose
// trees changed (chunks of kChunk out-edges spread over all warps); an
// improved out-edge updates its head's tree and queues the head. Same least
// fixpoint as the edge-state relaxation without its O(successors) scan per
// edge. The fold to vertex results is the edge engine's (edges.cuh).
#pragma once

#include "edges.cuh"
#include "tgxd_internal.cuh"
#include "traverse.cuh"

namespace tgxd {

struct SdArgs {
  DevCsr out, in;
  const uint32_t* out2in;  // Out position -> In position of the same edge
  QueryParam qp;           // root, klo = t_a, vhi = t_b (Out key space)
  int strict;
  long long* val;          // per Out position: least duration sum (kInf64: none)
  long long* tree;         // per In position: Fenwick suffix-min over the segment
  uint32_t* stamp;         // per vertex: round it was last queued
  uint32_t* fa;            // vertex queues
  uint32_t* fb;
  uint2* chunks;           // {first out position, vertex}: one round's work list
  EdgeCtl* ctl;
  unsigned long long* nchunks;  // chunk counter (monotone)
  uint32_t n;
  uint32_t round_limit;
  int weighted;            // price = weight (w; null: 1) instead of end - start
  const long long* w;
};

// Out -> In position map: the In entry of the same (src, dst, start, end)
// (duplicates may share one entry: they carry the same value and end).
__global__ void out2in_kernel(DevCsr out, DevCsr in, uint32_t* map) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t f = blockIdx.x * blockDim.x + threadIdx.x; f < out.m; f += stride) {
    // owner u of Out position f: last vertex whose segment starts at or before f
    uint32_t lo = 0, hi = out.n;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(out.off + mid) <= f) lo = mid;
      else hi = mid;
    }
    const uint32_t u = lo;
    const int32_t st = __ldg(out.key + f);
    const uint2 pf = __ldg(out.pay + f);  // {dst w, end}
    const uint32_t w = pf.x;
    const int32_t k = -(int32_t)pf.y;     // In key of the edge
    const uint32_t a = __ldg(in.off + w), b = __ldg(in.off + w + 1);
    uint32_t p = lane_lower_bound(in, a, b, k, in.fence != nullptr && b - a >= 64);
    while (p < b && __ldg(in.key + p) == k &&
           !(__ldg(in.pay + p).x == u && -(int32_t)__ldg(in.pay + p).y == st))
      ++p;
    map[f] = p;
  }
}

// Fenwick tree over one In segment [s, t), reversed so that a suffix of the
// segment is a prefix of the tree: position pos <-> rank r = t - 1 - pos.
__device__ __forceinline__ void fen_update(long long* tree, uint32_t s, uint32_t t, uint32_t pos,
                                           long long v) {
  const uint32_t L = t - s;
  for (uint32_t i = t - pos; i <= L; i += i & (0u - i)) {
    long long* cell = tree + s + i - 1;
    if (v < (long long)__ldcg(reinterpret_cast<const unsigned long long*>(cell))) atomicMin(cell, v);
  }
}

// min over segment positions [p, t)
__device__ __forceinline__ long long fen_query(const long long* tree, uint32_t s, uint32_t t,
                                               uint32_t p) {
  long long r = kInf64;
  for (uint32_t i = t - p; i > 0; i -= i & (0u - i))
    r = min(r, (long long)__ldcg(reinterpret_cast<const unsigned long long*>(tree + s + i - 1)));
  return r;
}

// Prices out-edge g (position f) of vertex w; true when g improved (its head
// is returned in *head).
__device__ __forceinline__ bool sd_price(const SdArgs& a, uint32_t w, uint32_t f, uint32_t* head) {
  const int32_t st = __ldg(a.out.key + f);
  const uint2 pf = __ldg(a.out.pay + f);
  *head = pf.x;
  if (st < a.qp.klo || st > a.qp.vhi || (int32_t)pf.y > a.qp.vhi) return false;
  long long best = kInf64;
  if (w == a.qp.root) {
    best = 0;  // the root's window edges start paths (path_algorithms.cpp:214-224)
  } else {
    const uint32_t si = __ldg(a.in.off + w), ti = __ldg(a.in.off + w + 1);
    if (ti > si) {
      const int32_t x = a.strict ? 1 - st : -st;  // in-edges ending before / by st
      const uint32_t p = __ldg(a.in.kmax + w) < x
                             ? ti
                             : lane_lower_bound(a.in, si, ti, x,
                                                a.in.fence != nullptr && ti - si >= 64);
      if (p < ti) best = fen_query(a.tree, si, ti, p);
    }
  }
  if (best == kInf64) return false;
  // g is an admissible successor: the reference evaluates its cost here
  long long cost;
  if (!edge_cost(a.weighted, a.w, f, st, (int32_t)pf.y, &a.ctl->weight_err, &cost)) return false;
  const long long c = best + cost;
  if (!(c < (long long)__ldcg(reinterpret_cast<const unsigned long long*>(a.val + f)))) return false;
  if (!(c < atomicMin(a.val + f, c))) return false;
  const uint32_t h = pf.x;
  fen_update(a.tree, __ldg(a.in.off + h), __ldg(a.in.off + h + 1), __ldg(a.out2in + f), c);
  return true;
}

__global__ void __launch_bounds__(kThreads, TGXD_MIN_BLOCKS) sd_kernel(SdArgs a) {
  __shared__ uint32_t s_buf[kWarps][64];
  __shared__ uint2 s_cbuf[kWarps][kListCap];
  uint32_t* wbuf = s_buf[threadIdx.x >> 5];
  GridBarrier grid{&a.ctl->bar_count, &a.ctl->bar_gen, gridDim.x, 0};
  EdgeCtl* ctl = a.ctl;
  const uint32_t lane = lane_id();
  const uint32_t gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint32_t nw = gridDim.x * kWarps;
  const bool tr = blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long checked = 0;
  if (tr) {
    a.fa[0] = a.qp.root;  // round 1 prices the root's window edges (the seeds)
    ctl->pushes = 1;
  }
  grid.sync();
  unsigned long long prev = 0, now = edge_pushes(ctl);
  unsigned long long c_cur = 0;
  uint32_t round = 0, flip = 0;
  while (now > prev) {
    if (round >= a.round_limit) {
      if (tr) ctl->error = 1;
      break;
    }
    const uint32_t* fin = flip ? a.fb : a.fa;
    uint32_t* fout = flip ? a.fa : a.fb;
    grid.sync();  // every block's counter reads are over before anyone moves them
    // (1) each frontier vertex: its window out-edges as kChunk-edge chunks
    {
      WarpList cl{s_cbuf[threadIdx.x >> 5], 0};
      const uint32_t F = (uint32_t)(now - prev);
      for (uint32_t base = gw * 32; base < F; base += nw * 32) {
        const uint32_t i = base + lane;
        uint32_t w = 0, p0 = 0, cnt = 0;
        if (i < F) {
          w = __ldcg(fin + i);
          const uint32_t so = __ldg(a.out.off + w), to = __ldg(a.out.off + w + 1);
          if (to > so && __ldg(a.out.kmax + w) >= a.qp.klo) {
            p0 = lane_lower_bound(a.out, so, to, a.qp.klo, a.out.fence != nullptr && to - so >= 64);
            const uint32_t p1 = a.qp.vhi == kInf ? to
                                                 : lane_lower_bound(a.out, p0, to, a.qp.vhi + 1,
                                                                    a.out.fence != nullptr &&
                                                                        to - so >= 64);
            cnt = p1 - p0;
          }
        }
        const uint32_t nch = (cnt + kChunk - 1) / kChunk;
        uint32_t todo = __ballot_sync(0xffffffffu, nch != 0);
        while (todo) {
          const uint32_t L = __ffs(todo) - 1;
          todo &= todo - 1;
          const uint32_t W = __shfl_sync(0xffffffffu, w, L);
          const uint32_t P = __shfl_sync(0xffffffffu, p0, L);
          const uint32_t bn = __shfl_sync(0xffffffffu, nch, L);
          for (uint32_t k0 = 0; k0 < bn; k0 += 32) {
            const uint32_t k = k0 + lane;
            list_append(cl, k < bn, make_uint2(P + k * kChunk, W), a.nchunks, c_cur, a.chunks);
          }
        }
      }
      list_drain(cl, a.nchunks, c_cur, a.chunks);
    }
    grid.sync();
    unsigned long long c_end;
    {
      __shared__ unsigned long long s_c;
      if (threadIdx.x == 0) s_c = __ldcg(a.nchunks);
      __syncthreads();
      c_end = s_c;
      __syncthreads();
    }
    // (2) every chunk: its out-edges priced, improved heads queued
    {
      uint32_t nb = 0;
      for (unsigned long long c = gw; c < c_end - c_cur; c += nw) {
        const uint2 ch = __ldcg(a.chunks + c);
        const uint32_t w = ch.y;
        const uint32_t to = __ldg(a.out.off + w + 1);
#pragma unroll 1
        for (uint32_t u = 0; u < kChunk; u += 32) {
          const uint32_t f = ch.x + u + lane;
          bool push = false;
          uint32_t head = 0;
          if (f < to && f < ch.x + kChunk) {
            ++checked;
            if (sd_price(a, w, f, &head))
              push = atomicExch(a.stamp + head, round + 1) != round + 1;
          }
          edge_push(wbuf, nb, push, head, ctl, now, fout);
        }
      }
      edge_push_drain(wbuf, nb, ctl, now, fout);
    }
    c_cur = c_end;
    grid.sync();
    prev = now;
    now = edge_pushes(ctl);
    ++round;
    flip ^= 1u;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) checked += __shfl_xor_sync(0xffffffffu, checked, o);
  if (lane == 0 && checked) atomicAdd(&ctl->checked, checked);
  if (tr) {
    ctl->rounds = round;
    ctl->expanded = prev;
  }
}

}  // namespace tgxd
