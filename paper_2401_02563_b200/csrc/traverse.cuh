// Frontier traversal on the device T-CSR — the hot path of
// earliest_arrival / latest_departure / fastest_path
// (reference: path_algorithms.cpp:262-357,436-528 driving temporal_edge_map,
// engine.hpp:239-353).
//
// One persistent cooperative kernel runs the whole query: every round is
//   A1  expand: per frontier item, locate the not-yet-relaxed admissible key
//       range of its segment (selective index: fence search for hubs, plain
//       binary search otherwise) and record its size;
//   A2  scan: grid-wide exclusive scan of range sizes, compacting non-empty
//       ranges into a merge-path table;
//   B   relax: every warp takes an equal slab of the round's edge work,
//       resolves its lanes' ranges with shuffles, streams dst/val coalesced,
//       relaxes labels with atomicMin and appends improved vertices to the
//       next frontier (bitmap dedup + warp-aggregated append);
// separated by grid barriers. No host round trip per round.
//
// Work efficiency. Labels only decrease (key space) and the relaxed value of
// an edge (its val) does not depend on the label that admitted it, so once an
// edge has been relaxed it never needs relaxing again. Each vertex remembers
// the bound it was last expanded with (Ex); a re-expansion only walks the
// keys in [new bound, old bound). Every admissible edge is relaxed exactly
// once per query (once per sweep for fastest), whatever the schedule — the
// labels are the unique least fixpoint the reference's round-synchronous
// loop also reaches, so results are bit-identical.
#include <cooperative_groups.h>

#include "tgxd_internal.cuh"

namespace cg = cooperative_groups;

namespace tgxd {

constexpr int kThreads = 256;
constexpr int kWarps = kThreads / 32;
constexpr int kUnroll = 4;

struct TravArgs {
  DevCsr g;
  const QueryParam* qp;
  int32_t* X;         // labels, Q x n (key space)
  int32_t* Ex;        // bound each vertex was last expanded with
  int32_t* R;         // fastest durations (nullptr otherwise)
  uint32_t* bitmap;   // queued flags, Q x n bits
  uint32_t* fa;       // frontier queues (items = q * n + v)
  uint32_t* fb;
  uint32_t* cnt;      // per frontier slot: range size
  uint32_t* lo;       // per frontier slot: range start
  RangeEntry* ranges; // compacted non-empty ranges + sentinel
  unsigned long long* bsum;
  uint32_t* bnz;
  uint32_t* bidx;
  Control* ctl;
  uint32_t n;
  uint32_t Q;
  int strict;
  uint32_t cutoff;
  int mode;           // tgxd_mode
  // fastest sweep (Q == 1)
  int fastest;
  uint32_t n_cand;
  const uint32_t* cand_lo;
  const uint32_t* cand_cnt;
  const int32_t* cand_key;
};

__device__ __forceinline__ int32_t ld_nc(const int32_t* p) {
  int32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ld_nc(const uint32_t* p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}

// First position in [s, t) whose key >= x. Vertices at or above the index
// cutoff first search the fence array (every 32nd key of the layout, a
// compact "bucketed timeline"), which narrows the search to one 128-byte key
// line; the rest binary-search their segment directly. Results-neutral, like
// the reference's TGER-vs-scan choice (test_algorithms.cpp:196-217).
__device__ __forceinline__ uint32_t lower_key(const DevCsr& g, uint32_t s, uint32_t t, int32_t x,
                                              bool use_index) {
  if (use_index && t > s) {
    const uint32_t jlo = (s + kFenceStride - 1) >> kFenceShift;
    const uint32_t jhi = (t - 1) >> kFenceShift;
    if (jlo <= jhi) {
      uint32_t a = jlo, b = jhi + 1;
      while (a < b) {
        const uint32_t mid = (a + b) >> 1;
        if (__ldg(g.fence + mid) < x) a = mid + 1;
        else b = mid;
      }
      if (a > jlo) s = max(s, ((a - 1) << kFenceShift) + 1);
      if (a <= jhi) t = min(t, a << kFenceShift);
    }
  }
  while (s < t) {
    const uint32_t mid = (s + t) >> 1;
    if (__ldg(g.key + mid) < x) s = mid + 1;
    else t = mid;
  }
  return s;
}

struct Sums {
  unsigned long long w;
  uint32_t nz;
  uint32_t ix;
};

// Block-wide exclusive scan of (w, nz) pairs; returns the block totals.
__device__ __forceinline__ void block_scan2(unsigned long long w, uint32_t nz,
                                            unsigned long long& ew, uint32_t& enz,
                                            unsigned long long& tw, uint32_t& tnz) {
  __shared__ unsigned long long s_w[kWarps];
  __shared__ uint32_t s_nz[kWarps];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  unsigned long long iw = w;
  uint32_t inz = nz;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const unsigned long long yw = __shfl_up_sync(0xffffffffu, iw, o);
    const uint32_t ynz = __shfl_up_sync(0xffffffffu, inz, o);
    if (lane >= o) {
      iw += yw;
      inz += ynz;
    }
  }
  if (lane == 31) {
    s_w[wid] = iw;
    s_nz[wid] = inz;
  }
  __syncthreads();
  unsigned long long bw = 0, totw = 0;
  uint32_t bnz = 0, totnz = 0;
#pragma unroll
  for (int k = 0; k < kWarps; ++k) {
    if (k < wid) {
      bw += s_w[k];
      bnz += s_nz[k];
    }
    totw += s_w[k];
    totnz += s_nz[k];
  }
  __syncthreads();
  ew = bw + iw - w;
  enz = bnz + inz - nz;
  tw = totw;
  tnz = totnz;
}

__device__ __forceinline__ void block_sum2(unsigned long long& w, uint32_t& nz) {
  __shared__ unsigned long long r_w[kWarps];
  __shared__ uint32_t r_nz[kWarps];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    w += __shfl_xor_sync(0xffffffffu, w, o);
    nz += __shfl_xor_sync(0xffffffffu, nz, o);
  }
  if ((threadIdx.x & 31) == 0) {
    r_w[threadIdx.x >> 5] = w;
    r_nz[threadIdx.x >> 5] = nz;
  }
  __syncthreads();
  w = 0;
  nz = 0;
#pragma unroll
  for (int k = 0; k < kWarps; ++k) {
    w += r_w[k];
    nz += r_nz[k];
  }
  __syncthreads();
}

// Expansion of one frontier item: clears its queued flag, computes the range
// of keys [bound, previous bound) still to relax and records it.
__device__ __forceinline__ uint32_t expand_item(const TravArgs& a, uint32_t item, uint32_t& lo_out,
                                                uint32_t& ix) {
  const uint32_t q = a.Q == 1 ? 0u : item / a.n;
  const uint32_t v = item - q * a.n;
  const QueryParam qp = a.qp[q];
  const int32_t x = __ldcg(a.X + item);
  // min_start / max_end hook (path_algorithms.cpp:287-291, :337-342): the
  // root leaves at any time inside the window; everyone else strictly
  // (or weakly) after its own label.
  int32_t lb = (v == qp.root) ? qp.klo : (x == kInf ? kInf : x + a.strict);
  if (lb < qp.klo) lb = qp.klo;
  const int32_t old = __ldcg(a.Ex + item);
  lo_out = 0;
  if (lb >= old) return 0;
  a.Ex[item] = lb;
  const int32_t hik = min(old, qp.vhi + 1);  // keys above vhi cannot fit the window
  if (lb >= hik) return 0;
  const uint32_t s = __ldg(a.g.off + v), t = __ldg(a.g.off + v + 1);
  const bool idx = a.cutoff != 0 && t - s >= a.cutoff;
  ix += idx;
  const uint32_t p0 = lower_key(a.g, s, t, lb, idx);
  const uint32_t p1 = lower_key(a.g, p0, t, hik, idx);
  lo_out = p0;
  return p1 - p0;
}

// Phase A1: contiguous frontier chunk per block.
__device__ void phase_a1(const TravArgs& a, const uint32_t* fin, uint32_t F) {
  const uint32_t chunk = (F + gridDim.x - 1) / gridDim.x;
  const uint32_t beg = min(F, blockIdx.x * chunk), end = min(F, beg + chunk);
  unsigned long long w = 0;
  uint32_t nz = 0, ix = 0;
  for (uint32_t i = beg + threadIdx.x; i < end; i += blockDim.x) {
    const uint32_t item = __ldcg(fin + i);
    a.bitmap[item >> 5] = 0u;  // every set bit belongs to a frontier item
    uint32_t lo;
    const uint32_t c = expand_item(a, item, lo, ix);
    a.cnt[i] = c;
    a.lo[i] = lo;
    w += c;
    nz += c != 0;
  }
  block_sum2(w, nz);
  unsigned long long dummy = ix;
  uint32_t ixs = 0;
  block_sum2(dummy, ixs);
  if (threadIdx.x == 0) {
    a.bsum[blockIdx.x] = w;
    a.bnz[blockIdx.x] = nz;
    a.bidx[blockIdx.x] = (uint32_t)dummy;
  }
}

// Phase A2: block offsets from the per-block sums, then an in-order scan of
// the block's chunk writing compacted, prefix-annotated ranges.
__device__ void phase_a2(const TravArgs& a, const uint32_t* fin, uint32_t F,
                         unsigned long long& W, uint32_t& NR, uint32_t& IX) {
  __shared__ unsigned long long s_pre_w, s_tot_w;
  __shared__ uint32_t s_pre_nz, s_tot_nz, s_tot_ix;
  unsigned long long pw = 0, tw = 0, ix = 0;
  uint32_t pnz = 0, tnz = 0, dz = 0;
  for (uint32_t j = threadIdx.x; j < gridDim.x; j += blockDim.x) {
    const unsigned long long bw = __ldcg(a.bsum + j);
    const uint32_t bn = __ldcg(a.bnz + j);
    if (j < blockIdx.x) {
      pw += bw;
      pnz += bn;
    }
    tw += bw;
    tnz += bn;
    ix += __ldcg(a.bidx + j);
  }
  block_sum2(pw, pnz);
  block_sum2(tw, tnz);
  block_sum2(ix, dz);
  if (threadIdx.x == 0) {
    s_pre_w = pw;
    s_pre_nz = pnz;
    s_tot_w = tw;
    s_tot_nz = tnz;
    s_tot_ix = (uint32_t)ix;
  }
  __syncthreads();
  unsigned long long base_w = s_pre_w;
  uint32_t base_nz = s_pre_nz;
  W = s_tot_w;
  NR = s_tot_nz;
  IX = s_tot_ix;
  const uint32_t chunk = (F + gridDim.x - 1) / gridDim.x;
  const uint32_t beg = min(F, blockIdx.x * chunk), end = min(F, beg + chunk);
  for (uint32_t tile = beg; tile < end; tile += blockDim.x) {
    const uint32_t i = tile + threadIdx.x;
    const uint32_t c = i < end ? __ldcg(a.cnt + i) : 0u;
    unsigned long long ew, bw;
    uint32_t enz, bnz;
    block_scan2(c, c != 0, ew, enz, bw, bnz);
    if (c != 0) {
      const uint32_t item = __ldcg(fin + i);
      RangeEntry r;
      r.pfx = base_w + ew;
      r.lo = __ldcg(a.lo + i);
      r.item = a.Q == 1 ? 0u : item / a.n;
      a.ranges[base_nz + enz] = r;
    }
    base_w += bw;
    base_nz += bnz;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    a.ranges[NR].pfx = W;  // merge-path sentinel
  }
}

// Phase B: merge-path relax of W edge-work items over NR ranges. With
// `single`, the table is the one explicit range (lo0, q = 0) — the seed
// edges of a fastest candidate.
__device__ void phase_b(const TravArgs& a, unsigned long long W, uint32_t NR, bool single,
                        uint32_t lo0, int32_t depart, uint32_t* fout, unsigned int* fcn) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint32_t nw = gridDim.x * kWarps;
  unsigned long long S = (W + nw - 1) / nw;
  S = (S + 31) & ~31ull;
  if (S < 32) S = 32;
  const unsigned long long s0 = (unsigned long long)gw * S;
  if (s0 >= W) return;
  const unsigned long long s1 = min(W, s0 + S);

  uint32_t i = 0;
  if (!single) {
    uint32_t lo = 0, hi = NR;  // first range with pfx > s0
    if (lane == 0) {
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (__ldcg(&a.ranges[mid].pfx) <= s0) lo = mid + 1;
        else hi = mid;
      }
    }
    i = __shfl_sync(0xffffffffu, lo, 0) - 1;
  }
  const int32_t vhi0 = a.qp[0].vhi;
  uint32_t wi = 0xffffffffu;
  unsigned long long endP = 0, Pi = 0;
  uint32_t wlo = 0, wq = 0;

  for (unsigned long long base = s0; base < s1; base += 32ull * kUnroll) {
    uint32_t e[kUnroll], qq[kUnroll];
    bool act[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const unsigned long long b = base + 32ull * u;
      act[u] = false;
      e[u] = 0;
      qq[u] = 0;
      if (b < s1) {
        if (i != wi) {  // (re)load the 32-range window starting at range i
          wi = i;
          if (single) {
            endP = lane == 0 ? W : ~0ull;
            wlo = lo0;
            wq = 0;
            Pi = 0;
          } else {
            const uint32_t r = i + lane;
            unsigned long long p = ~0ull;
            if (r <= NR) {
              const RangeEntry re = a.ranges[r];
              p = re.pfx;
              wlo = re.lo;
              wq = re.item;
            }
            Pi = __shfl_sync(0xffffffffu, p, 0);
            endP = __shfl_down_sync(0xffffffffu, p, 1);
            if (lane == 31) endP = (r + 1 <= NR) ? __ldcg(&a.ranges[r + 1].pfx) : ~0ull;
            if (r >= NR) endP = ~0ull;
          }
        }
        const unsigned long long t = b + lane;
        uint32_t pos = 0;
#pragma unroll
        for (uint32_t step = 16; step >= 1; step >>= 1) {
          const unsigned long long ev = __shfl_sync(0xffffffffu, endP, pos + step - 1);
          if (ev <= t) pos += step;
        }
        const unsigned long long prev = __shfl_sync(0xffffffffu, endP, pos > 0 ? pos - 1 : 0);
        const unsigned long long startP = pos ? prev : Pi;
        const uint32_t rlo = __shfl_sync(0xffffffffu, wlo, pos);
        const uint32_t rq = __shfl_sync(0xffffffffu, wq, pos);
        act[u] = t < s1;
        e[u] = rlo + (uint32_t)(t - startP);
        qq[u] = rq;
        i += __popc(__ballot_sync(0xffffffffu, endP <= b + 32));
      }
    }
    int32_t v[kUnroll];
    uint32_t d[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      if (act[u]) {
        v[u] = ld_nc(a.g.val + e[u]);
        d[u] = ld_nc(a.g.nbr + e[u]);
      }
    }
    uint32_t idx[kUnroll];
    bool cand[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      cand[u] = false;
      idx[u] = 0;
      if (act[u]) {
        const int32_t vhi = a.Q == 1 ? vhi0 : a.qp[qq[u]].vhi;
        if (v[u] <= vhi) {  // window containment: end <= t_b (types.hpp:55-57)
          idx[u] = qq[u] * a.n + d[u];
          cand[u] = true;
        }
      }
    }
    int32_t cur[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) cur[u] = cand[u] ? __ldcg(a.X + idx[u]) : kInf;
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      bool push = false;
      if (cand[u] && v[u] < cur[u]) {
        const int32_t old = atomicMin(a.X + idx[u], v[u]);  // write_min, parallel.hpp:91-99
        if (v[u] < old) {
          if (a.R) atomicMin(a.R + idx[u], v[u] - depart);
          const uint32_t m = 1u << (idx[u] & 31);
          const uint32_t ob = atomicOr(a.bitmap + (idx[u] >> 5), m);  // frontier claim
          push = (ob & m) == 0;
        }
      }
      const uint32_t bal = __ballot_sync(0xffffffffu, push);
      if (bal) {
        uint32_t basep = 0;
        const uint32_t leader = __ffs(bal) - 1;
        if (lane == leader) basep = atomicAdd(fcn, __popc(bal));
        basep = __shfl_sync(0xffffffffu, basep, leader);
        if (push) fout[basep + __popc(bal & ((1u << lane) - 1))] = idx[u];
      }
    }
  }
}

__global__ void __launch_bounds__(kThreads) traverse_kernel(TravArgs a) {
  cg::grid_group grid = cg::this_grid();
  uint32_t* fin = a.fa;
  uint32_t* fout = a.fb;
  uint32_t round = 0;
  unsigned long long work = 0, expansions = 0, index_lookups = 0;
  Control* ctl = a.ctl;
  for (uint32_t cand = 0;; ++cand) {
    if (a.fastest) {
      if (cand >= a.n_cand) break;
      // Seed round (path_algorithms.cpp:476-486): the candidate's first
      // edges, relaxed without an admissibility check.
      const uint32_t c0 = a.cand_cnt[cand];
      phase_b(a, c0, 1, true, a.cand_lo[cand], a.cand_key[cand], fout, &ctl->fc[(round + 1) & 1]);
      work += c0;
      grid.sync();
      ++round;
      uint32_t* t = fin;
      fin = fout;
      fout = t;
    }
    const int32_t depart = a.fastest ? a.cand_key[cand] : 0;
    for (;;) {
      const uint32_t F = __ldcg(&ctl->fc[round & 1]);
      if (F == 0) break;
      phase_a1(a, fin, F);
      grid.sync();
      if (blockIdx.x == 0 && threadIdx.x == 0) ctl->fc[round & 1] = 0;
      unsigned long long W;
      uint32_t NR, IX;
      phase_a2(a, fin, F, W, NR, IX);
      grid.sync();
      if (W) phase_b(a, W, NR, false, 0, depart, fout, &ctl->fc[(round + 1) & 1]);
      work += W;
      expansions += NR;
      index_lookups += IX;
      grid.sync();
      ++round;
      uint32_t* t = fin;
      fin = fout;
      fout = t;
    }
    if (!a.fastest) break;
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->rounds = round;
    ctl->work_all = work;
    ctl->expansions = expansions;
    ctl->index_lookups = index_lookups;
    ctl->candidates = a.fastest ? a.n_cand : 0;
  }
}

// Labels to INF, expansion bounds to INF, durations to INF, flags cleared.
__global__ void init_kernel(int32_t* X, int32_t* Ex, int32_t* R, uint32_t* bitmap, size_t nl,
                            size_t nwords) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += stride) {
    X[i] = kInf;
    Ex[i] = kInf;
    if (R) R[i] = kInf;
  }
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nwords; i += stride)
    bitmap[i] = 0u;
}

// Seeds: X[root] = klo (EA: t_a, LD: -t_b), root queued as round-0 frontier.
__global__ void seed_kernel(const QueryParam* qp, uint32_t Q, uint32_t n, int32_t* X,
                            uint32_t* bitmap, uint32_t* fa, Control* ctl, int fastest) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q == 0) {
    ctl->fc[0] = fastest ? 0u : Q;
    ctl->fc[1] = 0u;
  }
  if (q >= Q || fastest) return;
  const uint32_t item = q * n + qp[q].root;
  X[item] = qp[q].klo;
  atomicOr(bitmap + (item >> 5), 1u << (item & 31));
  fa[q] = item;
}

}  // namespace tgxd
