// Batched queries with one warp lane per query (configs 3 and 5: up to 32
// earliest-arrival or latest-departure queries sharing one graph).
//
// The slot-major batch (traverse.cuh with Q > 1) gives every (query, vertex)
// its own label slot, so a relaxation touches one random 4-byte label per
// query: Q queries cost Q random L2/DRAM accesses per edge, and for config 5
// (32 x 2^24 labels, 2.1 GB) every one misses L2. Here the labels of one
// vertex for all queries share one 128-byte line, XM[v * 32 + q], and a warp
// relaxes one edge for the whole batch at once — lane q is query q — so an
// edge costs ONE line access however many queries admit it (the warp's 32
// probes / atomicMins coalesce into one request).
//
// Round-synchronous, like the reference's temporal_edge_map rounds
// (engine.hpp:239-353) run for every query in lock step:
//   A  expand: per frontier vertex v, lane q computes its query's bound
//      (bound_of(label) or the window start at the root, path_algorithms.cpp
//      :287-291 / :337-342) and its not-yet-relaxed key range [bound, upper)
//      (upper = the bound v was last expanded with, capped by the window);
//      the warp searches the UNION of the lanes' ranges once (same tiered
//      search and selective index as traverse.cuh) and emits 128-edge chunks.
//      EB[v * 32 + q] = {new bound, upper} records each lane's range.
//   B  relax: a warp takes a chunk, each lane loads its query's range of the
//      chunk's vertex, and the warp walks the edges (coalesced loads of 32,
//      then shuffled out one at a time): lane q admits the edge iff its key
//      lies in lane q's range and val <= the window end (types.hpp:55-57),
//      probes its label in the edge's destination line and atomicMins
//      (write_min, parallel.hpp:91-99). The lanes that improved are OR-ed
//      into the destination's dirty mask with one atomic; the lane whose OR
//      found the mask empty queues the destination for the next round (the
//      claim_stamp of parallel.hpp:113-121, per vertex for the whole batch).
// Every query's labels are its unique least fixpoint (SURVEY.md Appendix
// A.7), reached here round by round exactly as in the single-query engine;
// per query every admissible edge is relaxed once (ranges only shrink).
#pragma once

#include "traverse.cuh"

namespace tgxd {

constexpr uint32_t kLanesMaxN = 1u << 24;  // chunk records carry v in 24 bits
constexpr uint32_t kLChunk = 128;          // edges per chunk (len - 1 in 7 bits)
constexpr int kLUnroll = 8;                // edges whose probes are in flight together

struct LanesArgs {
  DevCsr g;
  const QueryParam* qp;  // Q entries (key space)
  uint32_t Q, n;
  int strict;
  uint32_t cutoff;
  int32_t* XM;           // n x 32 labels, lane q = query q
  int2* EB;              // n x 32 {bound last expanded with, end of this round's range}
  uint32_t* dirty;       // n: queries improved since the vertex's last expansion
  uint32_t* fa;          // frontier queues (vertex ids)
  uint32_t* fb;
  uint2* chunks;         // {first edge, v | (len - 1) << 24}
  Control* ctl;          // pushes / chunks / edges counters, round count, barrier
  uint32_t round_limit;
};

// Chunk emission of one lane's range [p0, p0 + cnt) of vertex v.
__device__ __forceinline__ void lanes_emit(const LanesArgs& a, WarpList& wl, unsigned long long cstart,
                                           uint32_t v, uint32_t p0, uint32_t cnt) {
  const uint32_t lane = lane_id();
  const uint32_t nch = (cnt + kLChunk - 1) / kLChunk;
  uint32_t bigs = __ballot_sync(0xffffffffu, nch != 0 && nch <= 32);
  while (bigs) {
    const uint32_t src = __ffs(bigs) - 1;
    bigs &= bigs - 1;
    const uint32_t B0 = __shfl_sync(0xffffffffu, p0, src), BC = __shfl_sync(0xffffffffu, cnt, src);
    const uint32_t BV = __shfl_sync(0xffffffffu, v, src);
    const uint32_t bn = __shfl_sync(0xffffffffu, nch, src);
    const uint32_t off = lane * kLChunk;
    const uint32_t len = lane < bn ? min(kLChunk, BC - off) : 1u;
    list_append(wl, lane < bn, make_uint2(B0 + off, BV | ((len - 1) << 24)), &a.ctl->chunks,
                cstart, a.chunks);
  }
  uint32_t huge = __ballot_sync(0xffffffffu, nch > 32);
  while (huge) {
    const uint32_t src = __ffs(huge) - 1;
    huge &= huge - 1;
    const uint32_t B0 = __shfl_sync(0xffffffffu, p0, src), BC = __shfl_sync(0xffffffffu, cnt, src);
    const uint32_t BV = __shfl_sync(0xffffffffu, v, src);
    const uint32_t bn = __shfl_sync(0xffffffffu, nch, src);
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&a.ctl->chunks, (unsigned long long)bn);
    base = __shfl_sync(0xffffffffu, base, 0) - cstart;
    for (uint32_t j = lane; j < bn; j += 32) {
      const uint32_t off = j * kLChunk;
      const uint32_t len = min(kLChunk, BC - off);
      if (TGXD_IN_CAP(base + j, 1)) a.chunks[base + j] = make_uint2(B0 + off, BV | ((len - 1) << 24));
    }
  }
}

// Phase A: 32 frontier vertices per warp iteration. Lanes = queries for the
// label lines (8 vertices' lines in flight), lanes = vertices for the search.
__device__ TGXD_PHASE void lanes_expand(const LanesArgs& a, const uint32_t* fin, uint32_t F,
                                        unsigned long long cstart, uint2* ebuf,
                                        const QueryParam& qp, bool qv,
                                        unsigned long long& work, unsigned long long& ix) {
  const uint32_t lane = lane_id();
  const uint32_t gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint32_t nw = gridDim.x * kWarps;
  WarpList wl{ebuf, 0};
  for (uint32_t base = gw * 32; base < F; base += nw * 32) {
    const uint32_t nv = min(32u, F - base);
    const bool valid = lane < nv;
    const uint32_t v = valid ? __ldcg(fin + base + lane) : 0u;
    uint32_t s = 0, t = 0;
    int32_t km = INT32_MIN;
    if (valid) {
      s = __ldg(a.g.off + v);
      t = __ldg(a.g.off + v + 1);
      km = __ldg(a.g.kmax + v);
      a.dirty[v] = 0u;  // improvements from this round's relax on re-queue v
    }
    int32_t klo = kInf, khi = INT32_MIN;  // this lane's vertex: union of the queries' ranges
    for (uint32_t j0 = 0; j0 < nv; j0 += kLUnroll) {
      int32_t x[kLUnroll];
      int2 eb[kLUnroll];
      uint32_t vj[kLUnroll];
#pragma unroll
      for (int u = 0; u < kLUnroll; ++u) {
        vj[u] = __shfl_sync(0xffffffffu, v, (j0 + u) & 31);
        const bool in = j0 + u < nv;
        x[u] = in ? __ldcg(a.XM + (size_t)vj[u] * 32 + lane) : kInf;
        eb[u] = in ? __ldcg(a.EB + (size_t)vj[u] * 32 + lane) : make_int2(kInf, kInf);
      }
#pragma unroll
      for (int u = 0; u < kLUnroll; ++u) {
        const bool in = j0 + u < nv;
        // min_start / max_end hooks (path_algorithms.cpp:287-291, :337-342)
        int32_t lb = vj[u] == qp.root ? qp.klo : bound_of(x[u], a.strict);
        if (lb < qp.klo) lb = qp.klo;
        const int32_t old = eb[u].x;
        const bool moved = qv && x[u] != kInf && lb < old;
        const int32_t hi = min(old, qp.vhi + 1);  // keys above vhi cannot fit the window
        const bool act = moved && lb < hi;
        const int32_t nb = moved ? lb : old;
        if (in && qv) a.EB[(size_t)vj[u] * 32 + lane] = make_int2(nb, act ? hi : nb);
        const int32_t mlo = __reduce_min_sync(0xffffffffu, act ? lb : kInf);
        const int32_t mhi = __reduce_max_sync(0xffffffffu, act ? hi : INT32_MIN);
        if (lane == j0 + u) {
          klo = mlo;
          khi = mhi;
        }
      }
    }
    uint32_t p0 = 0, p1 = 0;
    const bool act = valid && klo < khi && t > s && km >= klo;
    if (act) {
      const bool fence = a.cutoff != 0 && t - s >= a.cutoff;
      ix += fence ? 1 : 0;
      p1 = km < khi ? t : lane_lower_bound(a.g, s, t, khi, fence);
      p0 = p1 > s ? lane_lower_bound(a.g, s, p1, klo, fence) : s;
    }
    const uint32_t cnt = act ? p1 - p0 : 0u;
    work += cnt;
    lanes_emit(a, wl, cstart, v, p0, cnt);
  }
  list_drain(wl, &a.ctl->chunks, cstart, a.chunks);
}

// Phase B: one chunk per warp iteration.
__device__ TGXD_PHASE void lanes_relax(const LanesArgs& a, unsigned long long nchunks,
                                       unsigned long long pstart, uint32_t* fout, uint32_t* wbuf,
                                       const QueryParam& qp, uint64_t pol_stream) {
  const uint32_t lane = lane_id();
  const uint32_t gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint32_t nw = gridDim.x * kWarps;
  PushBuf pb{wbuf, 0};
  for (unsigned long long c = gw; c < nchunks; c += nw) {
    const uint2 ch = __ldcg(a.chunks + c);
    const uint32_t v = ch.y & 0xffffffu;
    const uint32_t len = (ch.y >> 24) + 1;
    const int2 rng = __ldcg(a.EB + (size_t)v * 32 + lane);  // this lane's [bound, upper)
    for (uint32_t e0 = 0; e0 < len; e0 += 32) {
      const uint32_t ne = min(32u, len - e0);
      const bool in = lane < ne;
      const int32_t k = in ? ld_stream(a.g.key + ch.x + e0 + lane, pol_stream) : kInf;
      const uint2 pl = in ? ld_stream2(a.g.pay + ch.x + e0 + lane, pol_stream) : make_uint2(0u, kInf);
      for (uint32_t j0 = 0; j0 < ne; j0 += kLUnroll) {
        uint32_t d[kLUnroll];
        int32_t val[kLUnroll], cur[kLUnroll];
        bool ad[kLUnroll];
#pragma unroll
        for (int u = 0; u < kLUnroll; ++u) {
          const uint32_t j = (j0 + u) & 31;
          const int32_t kj = __shfl_sync(0xffffffffu, k, j);
          d[u] = __shfl_sync(0xffffffffu, pl.x, j);
          val[u] = (int32_t)__shfl_sync(0xffffffffu, pl.y, j);
          // admissible for this lane's query: inside its range and its window
          ad[u] = j0 + u < ne && kj >= rng.x && kj < rng.y && val[u] <= qp.vhi;
          cur[u] = ad[u] ? __ldcg(a.XM + (size_t)d[u] * 32 + lane) : kInf;
        }
#pragma unroll
        for (int u = 0; u < kLUnroll; ++u) {
          bool imp = false;
          if (ad[u] && val[u] < cur[u]) {
            const int32_t old = atomicMin(a.XM + (size_t)d[u] * 32 + lane, val[u]);
            imp = val[u] < old;
          }
          const uint32_t mask = __ballot_sync(0xffffffffu, imp);
          bool push = false;
          if (mask && lane == (uint32_t)(__ffs(mask) - 1))
            push = atomicOr(a.dirty + d[u], mask) == 0u;
          const uint32_t pbal = __ballot_sync(0xffffffffu, push);
          if (pbal) {
            if (push) pb.buf[pb.n] = d[u];
            pb.n += 1;
            if (pb.n >= 32) push_flush32(pb, a.ctl, pstart, fout);
          }
        }
      }
    }
  }
  push_drain(pb, a.ctl, pstart, fout);
}

__global__ void __launch_bounds__(kThreads, TGXD_MIN_BLOCKS) lanes_kernel(LanesArgs a) {
  __shared__ uint2 s_ebuf[kWarps][kListCap];
  __shared__ uint32_t s_pbuf[kWarps][64];
  GridBarrier grid{&a.ctl->bar_count, &a.ctl->bar_gen, gridDim.x, 0};
  const uint32_t lane = lane_id();
  const bool qv = lane < a.Q;
  QueryParam qp;
  if (qv) {
    qp = a.qp[lane];
  } else {  // lanes without a query admit nothing
    qp.root = kNoRoot;
    qp.klo = kInf;
    qp.vhi = INT32_MIN;
    qp.depart = 0;
  }
  const uint64_t pol_stream = policy_evict_first();
  Control* ctl = a.ctl;
  unsigned long long p_prev = 0, p_known = block_read(&ctl->pushes), c_known = 0;
  unsigned long long work = 0, ix = 0;
  uint32_t flip = 0, rounds = 0;
  for (;;) {
    const unsigned long long F = p_known - p_prev;
    if (F == 0) break;
    if (rounds > a.round_limit) {  // identical in every block
      if (blockIdx.x == 0 && threadIdx.x == 0) ctl->error = 1;
      break;
    }
    const uint32_t* fin = flip ? a.fb : a.fa;
    uint32_t* fout = flip ? a.fa : a.fb;
    lanes_expand(a, fin, (uint32_t)F, c_known, s_ebuf[threadIdx.x >> 5], qp, qv, work, ix);
    grid.sync();
    const unsigned long long c_end = block_read(&ctl->chunks);
    lanes_relax(a, c_end - c_known, p_known, fout, s_pbuf[threadIdx.x >> 5], qp, pol_stream);
    grid.sync();
    p_prev = p_known;
    p_known = block_read(&ctl->pushes);
    c_known = c_end;
    flip ^= 1u;
    ++rounds;
  }
  flush_work(ctl, work);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) ix += __shfl_xor_sync(0xffffffffu, ix, o);
  if (lane == 0 && ix) atomicAdd(&ctl->index_lookups, ix);
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->rounds = rounds;
    ctl->expansions = __ldcg(&ctl->chunks);
    ctl->candidates = 0;
    ctl->t_end = gtimer();
  }
}

// Labels and ranges to INF, dirty masks to 0.
__global__ void lanes_init_kernel(int32_t* XM, int2* EB, uint32_t* dirty, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const int4 inf4 = make_int4(kInf, kInf, kInf, kInf);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n * 8; i += stride) {
    reinterpret_cast<int4*>(XM)[i] = inf4;
    reinterpret_cast<int4*>(EB)[2 * i] = inf4;
    reinterpret_cast<int4*>(EB)[2 * i + 1] = inf4;
    if (i < n) dirty[i] = 0u;
  }
}

// Seeds: X[root_q][q] = klo_q, each distinct root queued once.
__global__ void lanes_seed_kernel(const QueryParam* qp, uint32_t Q, int32_t* XM, uint32_t* dirty,
                                  uint32_t* fa, Control* ctl) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  unsigned long long f = 0;
  for (uint32_t q = 0; q < Q; ++q) {
    const uint32_t r = qp[q].root;
    XM[(size_t)r * 32 + q] = qp[q].klo;
    if (dirty[r] == 0u) fa[f++] = r;
    dirty[r] |= 1u << q;
  }
  ctl->pushes = f;
  ctl->improved = 0;
  ctl->chunks = 0;
  ctl->smalls = 0;
  ctl->edges = 0;
  ctl->expansions = 0;
  ctl->index_lookups = 0;
  ctl->pull_scanned = 0;
  ctl->pchunks = 0;
  ctl->handoff_n = 0;
  ctl->handoff_kind = 0;
  ctl->error = 0;
  ctl->bar_count = 0;
  ctl->bar_gen = 0;
}

// Vertex-major labels -> the slot-major X (Q x n) the rest of the library
// reads (results, work counters): 32 x 32 tiles through shared memory.
__global__ void lanes_transpose_kernel(const int32_t* XM, int32_t* X, uint32_t n, uint32_t Q) {
  __shared__ int32_t tile[32][33];
  const uint32_t lane = threadIdx.x & 31, wy = threadIdx.x >> 5;  // 8 warps
  for (uint32_t v0 = blockIdx.x * 32; v0 < n; v0 += gridDim.x * 32) {
    for (uint32_t r = wy; r < 32; r += 8) {
      const uint32_t v = v0 + r;
      tile[r][lane] = v < n ? XM[(size_t)v * 32 + lane] : kInf;
    }
    __syncthreads();
    for (uint32_t q = wy; q < Q; q += 8) {
      const uint32_t v = v0 + lane;
      if (v < n) X[(size_t)q * n + v] = tile[lane][q];
    }
    __syncthreads();
  }
}

}  // namespace tgxd
