// Edge-state traversals: the Overlaps ordering (earliest arrival, latest
// departure, temporal BFS, fastest) and shortest duration (every ordering).
//
// Under Overlaps a path's admissibility depends on the interval of the edge
// that reached a vertex, not on a per-vertex label, so the reference walks
// edges instead of vertices (edge_reachability, path_algorithms.cpp:40-87;
// fastest_overlaps :136-191; shortest_duration_edges :205-258). Same here: the
// frontier holds flat edge positions of one layout, and an edge e's
// successors are a contiguous key range of its far endpoint's segment:
//
//   Overlaps   keys in (key_e, val_e] and val_f > val_e
//              Out (key = start, val = end): e.start < f.start <= e.end < f.end
//              In (key = -end, val = -start) is the same test mirrored:
//              f.start < e.start <= f.end < e.end (backward_window, holds(f, e))
//   Strict     keys >= val_e + 1   (e.end < f.start), Out only (shortest duration)
//   Succeeds   keys >= val_e       (e.end <= f.start)
//
// each further limited by the window (key <= vhi, val <= vhi). One round
// expands the frontier edges (one per lane, the selective-index search for
// the range), and the warp walks its 32 ranges packed 32 candidates per step.
//
//   reach (EA / LD / BFS under Overlaps)  a bit per edge (atomicOr claims it
//       once); the far endpoint's label takes min(val_f) — earliest end
//       (EA), latest start (LD, mirrored) — or the BFS level
//   fastest (Overlaps)  per edge the latest first-edge start over paths
//       ending with it (atomicMax), queued once per round (stamp)
//   shortest duration  per edge the least sum of durations (64-bit
//       atomicMin), queued once per round (stamp)
//
// The fixpoints are unique (reachability sets; max / min over paths), so the
// in-round order of updates cannot change a result. A final pass folds edge
// states into vertex results (min over reached in-edges).
#pragma once

#include "tgxd_internal.cuh"
#include "traverse.cuh"

namespace tgxd {

enum EdgeKind : int { kEdgeReach = 0, kEdgeFastest = 1, kEdgeShortest = 2 };

struct EdgeCtl {
  unsigned long long pushes;   // frontier appends (queue position)
  unsigned long long expanded; // frontier edges expanded
  unsigned long long checked;  // candidate edges examined
  unsigned long long nchunks;  // shortest duration: out-edge chunks emitted
  unsigned int rounds;
  unsigned int error;
  unsigned int weight_err;     // weighted: 1 a reachable edge's weight is invalid, 2 too large
  alignas(128) unsigned int bar_count;
  alignas(128) unsigned int bar_gen;
  unsigned int bar_pad[31];
};

struct EdgeArgs {
  DevCsr g;               // Out, or In for latest departure (key space)
  QueryParam qp;          // one query: root, klo, vhi
  int kind;               // EdgeKind
  int ord;                // tgxd_ordering
  int bfs;                // reach kind: label = BFS level instead of val
  int32_t* X;             // reach: per-vertex label (key space) or level
  uint32_t* reached;      // reach: one bit per edge
  int32_t* dep;           // fastest: per-edge departure (INT32_MIN: none)
  long long* val;         // shortest: per-edge duration sum (LLONG_MAX: none)
  uint32_t* stamp;        // fastest / shortest: round an edge was last queued
  uint32_t* fa;
  uint32_t* fb;
  EdgeCtl* ctl;
  uint32_t n, m;
  uint32_t round_limit;
  int weighted;           // shortest: sum edge weights (w; null: every weight 1)
  const long long* w;     // per position (Out layout) weight code, see tgxd_graph::out_w
};

constexpr long long kInf64 = 0x7fffffffffffffffLL;

// The pushes counter, read once per block right after a barrier.
__device__ __forceinline__ unsigned long long edge_pushes(const EdgeCtl* ctl) {
  __shared__ unsigned long long s_p;
  if (threadIdx.x == 0) s_p = __ldcg(&ctl->pushes);
  __syncthreads();
  const unsigned long long p = s_p;
  __syncthreads();
  return p;
}

// Successor key range [lo_key, hi_key] of edge (key_e, val_e); false if empty.
__device__ __forceinline__ bool succ_keys(const EdgeArgs& a, int32_t key_e, int32_t val_e,
                                          int32_t& lo_key, int32_t& hi_key) {
  hi_key = a.qp.vhi;
  if (a.ord == TGXD_OVERLAPS) {
    lo_key = key_e + 1;
    hi_key = min(hi_key, val_e);
  } else {
    lo_key = val_e + (a.ord == TGXD_STRICTLY_SUCCEEDS ? 1 : 0);
  }
  return lo_key <= hi_key;
}

// Candidate f (payload pl, key kf) of edge e: window + ordering filter.
__device__ __forceinline__ bool succ_ok(const EdgeArgs& a, int32_t val_e, int32_t vf) {
  if (vf > a.qp.vhi) return false;
  return a.ord != TGXD_OVERLAPS || vf > val_e;
}

__device__ __forceinline__ void edge_push(uint32_t* buf, uint32_t& nb, bool p, uint32_t f,
                                          EdgeCtl* ctl, unsigned long long pstart,
                                          uint32_t* fout) {
  const uint32_t bal = __ballot_sync(0xffffffffu, p);
  if (!bal) return;
  const uint32_t lane = lane_id();
  if (p) buf[nb + __popc(bal & ((1u << lane) - 1))] = f;
  nb += __popc(bal);
  __syncwarp();
  if (nb >= 32) {
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&ctl->pushes, 32ull);
    base = __shfl_sync(0xffffffffu, base, 0);
    if (TGXD_IN_CAP(base - pstart + lane, 0)) fout[base - pstart + lane] = buf[lane];
    __syncwarp();
    const uint32_t t = buf[32 + lane];
    __syncwarp();
    if (lane + 32 < nb) buf[lane] = t;
    nb -= 32;
    __syncwarp();
  }
}

__device__ __forceinline__ void edge_push_drain(uint32_t* buf, uint32_t& nb, EdgeCtl* ctl,
                                                unsigned long long pstart, uint32_t* fout) {
  if (!nb) return;
  const uint32_t lane = lane_id();
  __syncwarp();
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(&ctl->pushes, (unsigned long long)nb);
  base = __shfl_sync(0xffffffffu, base, 0);
  if (lane < nb && TGXD_IN_CAP(base - pstart + lane, 0)) fout[base - pstart + lane] = buf[lane];
  nb = 0;
  __syncwarp();
}

// The cost of edge f for shortest duration: its duration, or (weighted) its
// weight; an invalid weight code records the reference's error
// (path_algorithms.cpp:196-203) and the edge is not taken.
__device__ __forceinline__ bool edge_cost(int weighted, const long long* w, uint32_t f, int32_t key,
                                          int32_t val, unsigned int* err, long long* cost) {
  if (!weighted) {
    *cost = (long long)(val - key);
    return true;
  }
  const long long c = w ? __ldg(w + f) : 1ll;
  if (c < 0) {
    atomicMax(err, c == -1 ? 1u : 2u);
    return false;
  }
  *cost = c;
  return true;
}

// Applies candidate f to its edge state; returns true when f joins the next
// frontier. base: the expanding edge's departure (fastest) or sum (shortest).
__device__ __forceinline__ bool edge_update(const EdgeArgs& a, uint32_t f, uint2 pf, int32_t kf,
                                            long long base, uint32_t round) {
  if (a.kind == kEdgeReach) {
    const uint32_t bit = 1u << (f & 31);
    if (__ldcg(a.reached + (f >> 5)) & bit) return false;
    if (atomicOr(a.reached + (f >> 5), bit) & bit) return false;
    const int32_t lab = a.bfs ? (int32_t)round + 1 : (int32_t)pf.y;
    if (lab < __ldcg(a.X + pf.x)) atomicMin(a.X + pf.x, lab);
    return true;
  }
  bool improved = false;
  if (a.kind == kEdgeFastest) {
    const int32_t b = (int32_t)base;
    if (b > __ldcg(a.dep + f)) improved = b > atomicMax(a.dep + f, b);
  } else {
    long long cost;
    if (!edge_cost(a.weighted, a.w, f, kf, (int32_t)pf.y, &a.ctl->weight_err, &cost)) return false;
    const long long c = base + cost;
    if (c < (long long)__ldcg(reinterpret_cast<const unsigned long long*>(a.val + f)))
      improved = c < atomicMin(a.val + f, c);
  }
  return improved && atomicExch(a.stamp + f, round + 1) != round + 1;
}

// Expands one round of frontier edges [0, F) of fin.
__device__ void edge_round(const EdgeArgs& a, const uint32_t* fin, uint32_t F, uint32_t round,
                           unsigned long long pstart, uint32_t* fout, uint32_t* wbuf,
                           unsigned long long& checked) {
  const uint32_t lane = lane_id();
  const uint32_t gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint32_t nw = gridDim.x * kWarps;
  uint32_t nb = 0;
  for (uint32_t base = gw * 32; base < F; base += nw * 32) {
    const uint32_t i = base + lane;
    uint32_t lo = 0, cnt = 0;
    int32_t val_e = 0;
    long long bval = 0;
    if (i < F) {
      const uint32_t e = __ldcg(fin + i);
      const int32_t key_e = __ldg(a.g.key + e);
      const uint2 pe = __ldg(a.g.pay + e);
      val_e = (int32_t)pe.y;
      if (a.kind == kEdgeFastest) bval = __ldcg(a.dep + e);
      else if (a.kind == kEdgeShortest)
        bval = (long long)__ldcg(reinterpret_cast<const unsigned long long*>(a.val + e));
      int32_t lk, hk;
      if (succ_keys(a, key_e, val_e, lk, hk)) {
        const uint32_t v = pe.x;
        const uint32_t s = __ldg(a.g.off + v), t = __ldg(a.g.off + v + 1);
        if (t > s && __ldg(a.g.kmax + v) >= lk) {
          const bool fence = a.g.fence != nullptr && t - s >= 64;
          const uint32_t p0 = lane_lower_bound(a.g, s, t, lk, fence);
          const uint32_t p1 = hk == kInf ? t : lane_lower_bound(a.g, p0, t, hk + 1, fence);
          lo = p0;
          cnt = p1 - p0;
        }
      }
    }
    // the warp's 32 ranges, packed 32 candidates per step (owner lane from
    // the mask of range starts, as phase_b's small windows)
    uint32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t start = incl - cnt;
    const uint32_t total = __shfl_sync(0xffffffffu, incl, 31);
    // lanes with an empty range are interleaved: the owner of item t is the
    // k-th non-empty lane after the last one starting at or before the step
    const uint32_t nonempty = __ballot_sync(0xffffffffu, cnt != 0);
    for (uint32_t sb = 0; sb < total; sb += 32) {
      const uint32_t before = __ballot_sync(0xffffffffu, cnt != 0 && start <= sb);
      const uint32_t i0 = before ? 31 - __clz(before) : 0;
      const uint32_t rel = start - sb;
      const uint32_t bit = (cnt != 0 && start > sb && rel < 32) ? (1u << rel) : 0u;
      const uint32_t mask = __reduce_or_sync(0xffffffffu, bit);
      const uint32_t k = __popc(mask & ((2u << lane) - 1));
      const uint32_t own = k ? __fns(nonempty, i0, (int)k + 1) & 31 : i0;
      const uint32_t olo = __shfl_sync(0xffffffffu, lo, own);
      const uint32_t ost = __shfl_sync(0xffffffffu, start, own);
      const int32_t oval = __shfl_sync(0xffffffffu, val_e, own);
      const long long ob = __shfl_sync(0xffffffffu, bval, own);
      const uint32_t t = sb + lane;
      bool push = false;
      uint32_t f = 0;
      if (t < total) {
        f = olo + (t - ost);
        ++checked;
        const uint2 pf = __ldg(a.g.pay + f);
        if (succ_ok(a, oval, (int32_t)pf.y)) {
          const int32_t kf = a.kind == kEdgeShortest ? __ldg(a.g.key + f) : 0;
          push = edge_update(a, f, pf, kf, ob, round);
        }
      }
      edge_push(wbuf, nb, push, f, a.ctl, pstart, fout);
    }
  }
  edge_push_drain(wbuf, nb, a.ctl, pstart, fout);
}

__global__ void __launch_bounds__(kThreads, TGXD_MIN_BLOCKS) edge_kernel(EdgeArgs a) {
  __shared__ uint32_t s_buf[kWarps][64];
  uint32_t* wbuf = s_buf[threadIdx.x >> 5];
  GridBarrier grid{&a.ctl->bar_count, &a.ctl->bar_gen, gridDim.x, 0};
  EdgeCtl* ctl = a.ctl;
  const uint32_t lane = lane_id();
  const uint32_t gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint32_t nw = gridDim.x * kWarps;
  unsigned long long checked = 0;
  // Seeds (path_algorithms.cpp:49-58,143-153,214-224): the root's window
  // edges, keys in [klo, vhi] with val <= vhi.
  {
    const uint32_t r = a.qp.root;
    const uint32_t s = __ldg(a.g.off + r), t = __ldg(a.g.off + r + 1);
    uint32_t p0 = t;
    if (t > s && __ldg(a.g.kmax + r) >= a.qp.klo)
      p0 = lane_lower_bound(a.g, s, t, a.qp.klo, a.g.fence != nullptr && t - s >= 64);
    uint32_t nb = 0;
    for (uint32_t b = p0 + gw * 32; b < t; b += nw * 32) {
      const uint32_t f = b + lane;
      bool push = false;
      if (f < t) {
        const int32_t kf = __ldg(a.g.key + f);
        const uint2 pf = __ldg(a.g.pay + f);
        if (kf <= a.qp.vhi && (int32_t)pf.y <= a.qp.vhi) {
          if (a.kind == kEdgeReach) {
            push = edge_update(a, f, pf, kf, 0, 0);
          } else if (a.kind == kEdgeFastest) {
            a.dep[f] = kf;  // write_max over an untouched edge (seeds are distinct)
            push = true;
          } else {
            long long cost;
            push = edge_cost(a.weighted, a.w, f, kf, (int32_t)pf.y, &ctl->weight_err, &cost);
            if (push) a.val[f] = cost;  // write_min over an untouched edge
          }
        }
      }
      edge_push(wbuf, nb, push, f, ctl, 0, a.fa);
    }
    edge_push_drain(wbuf, nb, ctl, 0, a.fa);
  }
  grid.sync();
  unsigned long long prev = 0, now = edge_pushes(ctl);
  uint32_t round = 0, flip = 0;
  const bool tr = blockIdx.x == 0 && threadIdx.x == 0;
  while (now > prev) {
    if (round >= a.round_limit) {  // identical in every block
      if (tr) ctl->error = 1;
      break;
    }
    uint32_t* fin = flip ? a.fb : a.fa;
    uint32_t* fout = flip ? a.fa : a.fb;
    grid.sync();  // every block's read of `pushes` is over before anyone pushes
    edge_round(a, fin, (uint32_t)(now - prev), round + 1, now, fout, wbuf, checked);
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

// Folds edge states into vertex results: fastest R[v] = min(end - departure)
// (path_algorithms.cpp:182-188), shortest Y[v] = min(sum) (:425-430), over
// the edges that reach v.
__global__ void edge_fold_kernel(DevCsr g, int kind, const int32_t* dep, const long long* val,
                                 int32_t* R, long long* Y) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t e = blockIdx.x * blockDim.x + threadIdx.x; e < g.m; e += stride) {
    const uint2 pe = __ldg(g.pay + e);
    if (kind == kEdgeFastest) {
      const int32_t d = dep[e];
      if (d != INT32_MIN) atomicMin(R + pe.x, (int32_t)pe.y - d);
    } else {
      const long long v = val[e];
      if (v != kInf64) atomicMin(Y + pe.x, v);
    }
  }
}

// Per-query reset of the edge states and the control block.
__global__ void edge_init_kernel(int kind, uint32_t m, uint32_t* reached, int32_t* dep,
                                 long long* val, uint32_t* stamp, long long* Y, uint32_t n,
                                 EdgeCtl* ctl, long long* tree = nullptr, uint32_t tree_n = 0) {
  const uint32_t stride = gridDim.x * blockDim.x;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  if (kind == kEdgeReach) {
    for (uint32_t i = tid; i < (m + 31) / 32; i += stride) reached[i] = 0;
  } else {
    for (uint32_t i = tid; i < m; i += stride) {
      if (kind == kEdgeFastest) dep[i] = INT32_MIN;
      else val[i] = kInf64;
      stamp[i] = 0;
    }
    if (Y)
      for (uint32_t i = tid; i < n; i += stride) Y[i] = kInf64;
    if (tree)
      for (uint32_t i = tid; i < tree_n; i += stride) tree[i] = kInf64;
  }
  if (tid == 0) {
    ctl->pushes = 0;
    ctl->expanded = 0;
    ctl->checked = 0;
    ctl->nchunks = 0;
    ctl->rounds = 0;
    ctl->error = 0;
    ctl->weight_err = 0;
    ctl->bar_count = 0;
    ctl->bar_gen = 0;
  }
}

}  // namespace tgxd
