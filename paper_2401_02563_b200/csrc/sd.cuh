// Shortest duration under Succeeds / StrictlySucceeds, vertex-driven.
//
// The reference relaxes edge states (shortest_duration_edges,
// path_algorithms.cpp:205-258): every reached edge e scans all out-edges of
// its head that start after it ends. Under the two "succeeds" orderings the
// best predecessor of an out-edge f of u depends only on f.start:
//
//   value[f] = (f.end - f.start) + B_u(f.start),
//   B_u(t)   = min{ value[e] : e reached in-edge of u, e.end < t (strict) or
//                   e.end <= t (weak) }     (0 for the source's edges)
//
// and in u's In segment (key = -end ascending) the in-edges ending before t
// form a suffix [lower_bound(1 - t), end) (weak: lower_bound(-t)), so B_u(t)
// is a suffix minimum. A round takes the vertices whose in-edge values
// changed, rebuilds their suffix minima (warp scan over the In segment,
// values gathered through the In -> Out position map) and re-prices their
// out-edges (one search + one read each); an improved out-edge queues its
// head. Same least fixpoint as the edge-state relaxation, without the
// O(successors) scan per edge. The fold to vertex results is the edge
// engine's (edges.cuh).
#pragma once

#include "edges.cuh"
#include "tgxd_internal.cuh"
#include "traverse.cuh"

namespace tgxd {

struct SdArgs {
  DevCsr out, in;
  const uint32_t* in2out;  // In position -> Out position of the same edge
  QueryParam qp;           // root, klo = t_a, vhi = t_b (Out key space)
  int strict;
  long long* val;          // per Out position: least duration sum (kInf64: none)
  long long* sm;           // per In position: suffix minimum of in-edge values
  uint32_t* stamp;         // per vertex: round it was last queued
  uint32_t* fa;
  uint32_t* fb;
  EdgeCtl* ctl;
  uint32_t n;
  uint32_t round_limit;
};

// In -> Out position map: the Out entry of the same (src, dst, start, end)
// (duplicates map to their first copy, which carries the same value).
__global__ void in2out_kernel(DevCsr out, DevCsr in, uint32_t* map) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < in.m; j += stride) {
    // owner u of In position j: last vertex whose segment starts at or before j
    uint32_t lo = 0, hi = in.n;
    while (hi - lo > 1) {
      const uint32_t mid = (lo + hi) >> 1;
      if (__ldg(in.off + mid) <= j) lo = mid;
      else hi = mid;
    }
    const uint32_t u = lo;
    const uint2 pj = __ldg(in.pay + j);  // {src w, -start}
    const int32_t st = -(int32_t)pj.y, en = -__ldg(in.key + j);
    const uint32_t w = pj.x;
    const uint32_t a = __ldg(out.off + w), b = __ldg(out.off + w + 1);
    uint32_t p = lane_lower_bound(out, a, b, st, out.fence != nullptr && b - a >= 64);
    while (p < b && __ldg(out.key + p) == st &&
           !(__ldg(out.pay + p).x == u && (int32_t)__ldg(out.pay + p).y == en))
      ++p;
    map[j] = p;
  }
}

// One frontier vertex per warp: suffix minima over its in-edges, then its
// window out-edges re-priced.
__device__ void sd_vertex(const SdArgs& a, uint32_t u, uint32_t round, unsigned long long pstart,
                          uint32_t* fout, uint32_t* wbuf, uint32_t& nb,
                          unsigned long long& checked) {
  const uint32_t lane = lane_id();
  const uint32_t si = __ldg(a.in.off + u), ti = __ldg(a.in.off + u + 1);
  // suffix minimum from the segment's end (smallest ends) backward
  long long carry = kInf64;
  for (uint32_t top = ti; top > si;) {
    const uint32_t lo = top > si + 32 ? top - 32 : si;
    const uint32_t j = top - 1 - lane;  // lane 0 holds the smallest end of the step
    long long v = kInf64;
    if (j >= lo && j < top)
      v = (long long)__ldcg(reinterpret_cast<const unsigned long long*>(a.val + __ldg(a.in2out + j)));
    // inclusive prefix minimum over lanes 0..lane (ascending end)
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const long long y = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= (uint32_t)o) v = min(v, y);
    }
    v = min(v, carry);
    if (j >= lo && j < top) a.sm[j] = v;
    carry = __shfl_sync(0xffffffffu, v, 31);
    top = lo;
  }
  __syncwarp();
  // window out-edges: start in [t_a, t_b], end <= t_b
  const uint32_t so = __ldg(a.out.off + u), to = __ldg(a.out.off + u + 1);
  if (to <= so) return;
  const bool root = u == a.qp.root;
  uint32_t p0 = so;
  if (lane == 0)
    p0 = __ldg(a.out.kmax + u) < a.qp.klo
             ? to
             : lane_lower_bound(a.out, so, to, a.qp.klo, a.out.fence != nullptr && to - so >= 64);
  p0 = __shfl_sync(0xffffffffu, p0, 0);
  for (uint32_t b = p0; b < to; b += 32) {
    const uint32_t f = b + lane;
    bool push = false;
    uint32_t w = 0;
    if (f < to) {
      const int32_t st = __ldg(a.out.key + f);
      const uint2 pf = __ldg(a.out.pay + f);
      w = pf.x;
      if (st <= a.qp.vhi && (int32_t)pf.y <= a.qp.vhi) {
        ++checked;
        long long best = root ? 0 : kInf64;
        if (!root && ti > si) {
          // in-edges ending before st (strict) or by st (weak): key >= bound
          const int32_t x = a.strict ? 1 - st : -st;
          const uint32_t p = __ldg(a.in.key + ti - 1) < x
                                 ? ti
                                 : lane_lower_bound(a.in, si, ti, x,
                                                    a.in.fence != nullptr && ti - si >= 64);
          if (p < ti) best = __ldcg(reinterpret_cast<const unsigned long long*>(a.sm + p));
        }
        if (best != kInf64) {
          const long long c = best + (long long)((int32_t)pf.y - st);
          if (c < (long long)__ldcg(reinterpret_cast<const unsigned long long*>(a.val + f)) &&
              c < atomicMin(a.val + f, c))
            push = atomicExch(a.stamp + w, round + 1) != round + 1;
        }
      }
    }
    edge_push(wbuf, nb, push, w, a.ctl, pstart, fout);
  }
}

__global__ void __launch_bounds__(kThreads, TGXD_MIN_BLOCKS) sd_kernel(SdArgs a) {
  __shared__ uint32_t s_buf[kWarps][64];
  uint32_t* wbuf = s_buf[threadIdx.x >> 5];
  GridBarrier grid{&a.ctl->bar_count, &a.ctl->bar_gen, gridDim.x, 0};
  EdgeCtl* ctl = a.ctl;
  const uint32_t lane = lane_id();
  const uint32_t gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint32_t nw = gridDim.x * kWarps;
  const bool tr = blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long checked = 0;
  // round 0: the root alone (its window out-edges are the seeds, value = duration)
  if (tr) {
    a.fa[0] = a.qp.root;
    ctl->pushes = 1;
  }
  grid.sync();
  unsigned long long prev = 0, now = edge_pushes(ctl);
  uint32_t round = 0, flip = 0;
  while (now > prev) {
    if (round >= a.round_limit) {
      if (tr) ctl->error = 1;
      break;
    }
    const uint32_t* fin = flip ? a.fb : a.fa;
    uint32_t* fout = flip ? a.fa : a.fb;
    grid.sync();  // every block's read of `pushes` is over before anyone pushes
    uint32_t nb = 0;
    for (unsigned long long i = gw; i < now - prev; i += nw)
      sd_vertex(a, __ldcg(fin + i), round + 1, now, fout, wbuf, nb, checked);
    edge_push_drain(wbuf, nb, ctl, now, fout);
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
