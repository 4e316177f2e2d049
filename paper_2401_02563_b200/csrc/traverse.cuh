// Frontier traversal on the device T-CSR — the hot path of
// earliest_arrival / latest_departure / fastest_path
// (reference: path_algorithms.cpp:262-357,436-528 driving temporal_edge_map,
// engine.hpp:239-353).
//
// One persistent cooperative kernel runs the whole query. Each round is
//   A  expand: every frontier item locates the not-yet-relaxed admissible key
//      range of its segment (selective index: fence search for hubs, plain
//      binary search otherwise) and emits it as work: ranges of >= 32 edges
//      as fixed-size chunks, shorter ones into a small-range list
//      (warp-aggregated atomic emission — no ordered scan needed);
//   B  relax: warps stream chunks (coalesced, unrolled) and pack 32 small
//      ranges per warp (lane ownership from a redux.or start mask), relax
//      labels with atomicMin and append improved vertices to the next
//      frontier through per-warp shared-memory push buffers;
// separated by grid barriers. No host round trip per round. All counters
// are monotone, so no round ever resets one (no extra barrier).
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
constexpr int kUnroll = 4;                       // 32-edge steps in flight per warp
constexpr uint32_t kChunk = 32u * kUnroll;       // edges per chunk of a big range
constexpr uint32_t kSmall = 32;                  // ranges below this go to the small list
constexpr uint32_t kChunkLenBits = 9;            // kChunk <= 256
constexpr uint32_t kSmallCntBits = 6;

struct TravArgs {
  DevCsr g;
  const QueryParam* qp;
  int32_t* X;          // labels, Q x n (key space)
  int32_t* Ex;         // bound each vertex was last expanded with
  int32_t* R;          // fastest durations (nullptr otherwise)
  uint32_t* bitmap;    // queued flags, Q x n bits
  uint32_t* fa;        // frontier queues (items = q * n + v)
  uint32_t* fb;
  uint2* chunks;       // {lo, q << 9 | len}
  uint2* smalls;       // {lo, q << 6 | cnt}
  Control* ctl;
  uint32_t n;
  uint32_t Q;
  int strict;
  uint32_t cutoff;
  int mode;            // tgxd_mode
  // fastest sweep (Q == 1)
  int fastest;
  uint32_t n_cand;
  const uint32_t* cand_lo;
  const uint32_t* cand_cnt;
  const int32_t* cand_key;
  // optional per-round trace (block 0): {t_start, t_after_A, t_after_B, F,
  // chunks, smalls, pushes, 0} per round, globaltimer ns
  unsigned long long* trace;
  uint32_t trace_cap;
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

__device__ __forceinline__ int32_t ld_stream(const int32_t* p) {
  int32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.b32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p) {
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

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

// Per-warp push buffer: improved vertices are staged in shared memory and
// appended to the next frontier 32 at a time (one global atomic per 32).
struct PushBuf {
  uint32_t* buf;  // 64 entries of this warp
  uint32_t n;     // staged entries (warp-uniform)
};

__device__ __forceinline__ void push_flush32(PushBuf& pb, Control* ctl,
                                             unsigned long long pstart, uint32_t* fout) {
  const uint32_t lane = lane_id();
  __syncwarp();
  const uint32_t v = pb.buf[lane];
  const uint32_t tail = pb.buf[32 + lane];
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(&ctl->pushes, 32ull);
  base = __shfl_sync(0xffffffffu, base, 0);
  fout[base - pstart + lane] = v;
  __syncwarp();
  if (lane + 32 < pb.n) pb.buf[lane] = tail;
  pb.n -= 32;
  __syncwarp();
}

__device__ __forceinline__ void push(PushBuf& pb, bool p, uint32_t item, Control* ctl,
                                     unsigned long long pstart, uint32_t* fout) {
  const uint32_t bal = __ballot_sync(0xffffffffu, p);
  if (bal == 0) return;
  const uint32_t lane = lane_id();
  if (p) pb.buf[pb.n + __popc(bal & ((1u << lane) - 1))] = item;
  pb.n += __popc(bal);
  if (pb.n >= 32) push_flush32(pb, ctl, pstart, fout);
}

__device__ __forceinline__ void push_drain(PushBuf& pb, Control* ctl, unsigned long long pstart,
                                           uint32_t* fout) {
  if (pb.n == 0) return;
  const uint32_t lane = lane_id();
  __syncwarp();
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(&ctl->pushes, (unsigned long long)pb.n);
  base = __shfl_sync(0xffffffffu, base, 0);
  if (lane < pb.n) fout[base - pstart + lane] = pb.buf[lane];
  pb.n = 0;
  __syncwarp();
}

// Relax kUnroll 32-edge steps: e[u] edge ids, q[u] query slots, act[u] lane
// validity. write_min (parallel.hpp:91-99) + claim_stamp (:113-121) become a
// plain label probe, atomicMin, and an atomicOr on the queued bitmap.
__device__ __forceinline__ void relax_steps(const TravArgs& a, const uint32_t (&e)[kUnroll],
                                            const uint32_t (&q)[kUnroll],
                                            const bool (&act)[kUnroll], int32_t vhi0,
                                            int32_t depart, PushBuf& pb,
                                            unsigned long long pstart, uint32_t* fout) {
  int32_t v[kUnroll];
  uint32_t d[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    v[u] = act[u] ? ld_stream(a.g.val + e[u]) : kInf;
    d[u] = act[u] ? ld_stream(a.g.nbr + e[u]) : 0u;
  }
  uint32_t idx[kUnroll];
  int32_t cur[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    const int32_t vhi = a.Q == 1 ? vhi0 : __ldg(&a.qp[q[u]].vhi);
    // window containment: end <= t_b (types.hpp:55-57)
    const bool ok = act[u] && v[u] <= vhi;
    idx[u] = q[u] * a.n + d[u];
    cur[u] = ok ? __ldcg(a.X + idx[u]) : kInf;
    if (!ok) v[u] = kInf;
  }
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    bool p = false;
    if (v[u] < cur[u]) {
      const int32_t old = atomicMin(a.X + idx[u], v[u]);
      if (v[u] < old) {
        if (a.R) atomicMin(a.R + idx[u], v[u] - depart);
        const uint32_t m = 1u << (idx[u] & 31);
        p = (atomicOr(a.bitmap + (idx[u] >> 5), m) & m) == 0;
      }
    }
    push(pb, p, idx[u], a.ctl, pstart, fout);
  }
}

// Phase A: expand the frontier and emit work.
__device__ void phase_a(const TravArgs& a, const uint32_t* fin, uint32_t F,
                        unsigned long long cstart, unsigned long long sstart,
                        unsigned long long& work, unsigned long long& ix) {
  const uint32_t lane = lane_id();
  const uint32_t nthreads = gridDim.x * blockDim.x;
  const uint32_t tbase = blockIdx.x * blockDim.x + (threadIdx.x & ~31u);
  for (uint32_t base = tbase; base < F; base += nthreads) {
    const uint32_t i = base + lane;
    uint32_t cnt = 0, lo = 0, q = 0;
    if (i < F) {
      const uint32_t item = __ldcg(fin + i);
      a.bitmap[item >> 5] = 0u;  // every set bit belongs to a frontier item
      q = a.Q == 1 ? 0u : item / a.n;
      const uint32_t v = item - q * a.n;
      const QueryParam qp = a.qp[q];
      const int32_t x = __ldcg(a.X + item);
      // min_start / max_end hooks (path_algorithms.cpp:287-291, :337-342):
      // the root leaves at any time inside the window; everyone else
      // strictly (or weakly) after its own label.
      int32_t lb = (v == qp.root) ? qp.klo : (x == kInf ? kInf : x + a.strict);
      if (lb < qp.klo) lb = qp.klo;
      const int32_t old = __ldcg(a.Ex + item);
      if (lb < old) {
        a.Ex[item] = lb;
        const int32_t hik = min(old, qp.vhi + 1);  // keys above vhi cannot fit the window
        if (lb < hik) {
          const uint32_t s = __ldg(a.g.off + v), t = __ldg(a.g.off + v + 1);
          const bool use_idx = a.cutoff != 0 && t - s >= a.cutoff;
          ix += use_idx;
          const uint32_t p0 = lower_key(a.g, s, t, lb, use_idx);
          const uint32_t p1 = lower_key(a.g, p0, t, hik, use_idx);
          lo = p0;
          cnt = p1 - p0;
          work += cnt;
        }
      }
    }
    // warp-aggregated emission
    const bool small = cnt != 0 && cnt < kSmall;
    const uint32_t nch = cnt >= kSmall ? (cnt + kChunk - 1) / kChunk : 0u;
    const uint32_t sbal = __ballot_sync(0xffffffffu, small);
    uint32_t incl = nch;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, incl, 31);
    unsigned long long cb = 0, sb = 0;
    if (lane == 0) {
      if (tot) cb = atomicAdd(&a.ctl->chunks, (unsigned long long)tot);
      if (sbal) sb = atomicAdd(&a.ctl->smalls, (unsigned long long)__popc(sbal));
    }
    cb = __shfl_sync(0xffffffffu, cb, 0);
    sb = __shfl_sync(0xffffffffu, sb, 0);
    if (small) {
      const uint64_t pos = sb - sstart + __popc(sbal & ((1u << lane) - 1));
      a.smalls[pos] = make_uint2(lo, (q << kSmallCntBits) | cnt);
    }
    if (nch) {
      uint64_t pos = cb - cstart + incl - nch;
      for (uint32_t c = 0; c < nch; ++c, ++pos) {
        const uint32_t off = c * kChunk;
        const uint32_t len = min(kChunk, cnt - off);
        a.chunks[pos] = make_uint2(lo + off, (q << kChunkLenBits) | len);
      }
    }
  }
}

// Phase B: relax the round's chunks and small ranges (plus, for a fastest
// seed round, the virtual chunks of one explicit range).
__device__ void phase_b(const TravArgs& a, unsigned long long nchunks, unsigned long long nsmall,
                        uint32_t xlo, uint32_t xcnt, int32_t depart, unsigned long long pstart,
                        uint32_t* fout, uint32_t* wbuf) {
  const uint32_t lane = lane_id();
  const uint32_t gw = blockIdx.x * kWarps + (threadIdx.x >> 5);
  const uint32_t nw = gridDim.x * kWarps;
  const int32_t vhi0 = a.qp[0].vhi;
  PushBuf pb{wbuf, 0};

  // explicit range (fastest seeds), split into virtual chunks
  const uint32_t nx = (xcnt + kChunk - 1) / kChunk;
  for (uint32_t c = gw; c < nx; c += nw) {
    uint32_t e[kUnroll], q[kUnroll];
    bool act[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t off = c * kChunk + u * 32 + lane;
      act[u] = off < xcnt;
      e[u] = xlo + off;
      q[u] = 0;
    }
    relax_steps(a, e, q, act, vhi0, depart, pb, pstart, fout);
  }

  // chunks of big ranges: coalesced kChunk-edge bursts
  for (unsigned long long c = gw; c < nchunks; c += nw) {
    const uint2 ch = a.chunks[c];
    const uint32_t len = ch.y & ((1u << kChunkLenBits) - 1);
    const uint32_t cq = ch.y >> kChunkLenBits;
    uint32_t e[kUnroll], q[kUnroll];
    bool act[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t off = u * 32 + lane;
      act[u] = off < len;
      e[u] = ch.x + off;
      q[u] = cq;
    }
    relax_steps(a, e, q, act, vhi0, depart, pb, pstart, fout);
  }

  // small ranges: 32 per warp window; lane l owns range l, items are packed
  // densely and each lane finds its owner from the mask of range starts.
  const unsigned long long nwin = (nsmall + 31) / 32;
  for (unsigned long long w = gw; w < nwin; w += nw) {
    const unsigned long long r = w * 32 + lane;
    uint32_t lo = 0, cnt = 0, rq = 0;
    if (r < nsmall) {
      const uint2 s = a.smalls[r];
      lo = s.x;
      cnt = s.y & ((1u << kSmallCntBits) - 1);
      rq = s.y >> kSmallCntBits;
    }
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
        // owner of item sb: last range starting at or before it
        const uint32_t before = __ballot_sync(0xffffffffu, cnt != 0 && start <= sb);
        const uint32_t i0 = before ? 31 - __clz(before) : 0;
        // ranges starting strictly inside (sb, sb + 32)
        const uint32_t rel = start - sb;
        const uint32_t bit = (cnt != 0 && start > sb && rel < 32) ? (1u << rel) : 0u;
        const uint32_t mask = __reduce_or_sync(0xffffffffu, bit);
        const uint32_t own = i0 + __popc(mask & ((2u << lane) - 1));
        const uint32_t olo = __shfl_sync(0xffffffffu, lo, own & 31);
        const uint32_t ost = __shfl_sync(0xffffffffu, start, own & 31);
        const uint32_t oq = __shfl_sync(0xffffffffu, rq, own & 31);
        const uint32_t t = sb + lane;
        act[u] = t < total;
        e[u] = olo + (t - ost);
        q[u] = oq;
      }
      relax_steps(a, e, q, act, vhi0, depart, pb, pstart, fout);
    }
  }
  push_drain(pb, a.ctl, pstart, fout);
}

__global__ void __launch_bounds__(kThreads, 3) traverse_kernel(TravArgs a) {
  __shared__ uint32_t s_buf[kWarps][64];
  cg::grid_group grid = cg::this_grid();
  uint32_t* wbuf = s_buf[threadIdx.x >> 5];
  uint32_t* fin = a.fa;
  uint32_t* fout = a.fb;
  Control* ctl = a.ctl;
  uint32_t rounds = 0;
  unsigned long long work = 0, ix = 0, expansions = 0;
  // Counter discipline: `pushes` only grows in phase B and is read at round
  // start (phase A); `chunks` / `smalls` only grow in phase A and are read
  // in phase B. A counter is never read while another block may be moving
  // it, so every block sees the same round boundaries.
  unsigned long long prev_p = 0;         // queue position where fin's items start
  unsigned long long c_cur = 0, s_cur = 0;
  for (uint32_t cand = 0;; ++cand) {
    int32_t depart = 0;
    if (a.fastest) {
      if (cand >= a.n_cand) break;
      // Seed round (path_algorithms.cpp:476-486): the candidate's first
      // edges, relaxed without an admissibility check. The queue is empty
      // here, so pushes == prev_p for every block.
      depart = a.cand_key[cand];
      const uint32_t c0 = a.cand_cnt[cand];
      phase_b(a, 0, 0, a.cand_lo[cand], c0, depart, prev_p, fout, wbuf);
      if (blockIdx.x == 0 && threadIdx.x == 0) work += c0;
      grid.sync();
      ++rounds;
      uint32_t* t = fin;
      fin = fout;
      fout = t;
    }
    for (;;) {
      const unsigned long long p_now = __ldcg(&ctl->pushes);
      const uint32_t F = (uint32_t)(p_now - prev_p);
      if (F == 0) break;
      const bool tr = a.trace && blockIdx.x == 0 && threadIdx.x == 0 && rounds < a.trace_cap;
      if (tr) {
        a.trace[rounds * 8 + 0] = gtimer();
        a.trace[rounds * 8 + 3] = F;
      }
      phase_a(a, fin, F, c_cur, s_cur, work, ix);
      grid.sync();
      const unsigned long long c_end = __ldcg(&ctl->chunks), s_end = __ldcg(&ctl->smalls);
      if (tr) {
        a.trace[rounds * 8 + 1] = gtimer();
        a.trace[rounds * 8 + 4] = c_end - c_cur;
        a.trace[rounds * 8 + 5] = s_end - s_cur;
      }
      phase_b(a, c_end - c_cur, s_end - s_cur, 0, 0, depart, p_now, fout, wbuf);
      expansions += (c_end - c_cur) + (s_end - s_cur);
      c_cur = c_end;
      s_cur = s_end;
      prev_p = p_now;
      grid.sync();
      if (tr) {
        a.trace[rounds * 8 + 2] = gtimer();
        a.trace[rounds * 8 + 6] = __ldcg(&ctl->pushes) - p_now;
      }
      ++rounds;
      uint32_t* t = fin;
      fin = fout;
      fout = t;
    }
    if (!a.fastest) break;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    work += __shfl_xor_sync(0xffffffffu, work, o);
    ix += __shfl_xor_sync(0xffffffffu, ix, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (work) atomicAdd(&ctl->work_all, work);
    if (ix) atomicAdd(&ctl->index_lookups, ix);
  }
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    ctl->rounds = rounds;
    ctl->expansions = expansions;
    ctl->candidates = a.fastest ? a.n_cand : 0;
  }
}

// Labels to INF, expansion bounds to INF, durations to INF, flags cleared.
__global__ void init_kernel(int32_t* X, int32_t* Ex, int32_t* R, uint32_t* bitmap, size_t nl,
                            size_t nwords) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t n4 = nl / 4;
  const int4 inf4 = make_int4(kInf, kInf, kInf, kInf);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    reinterpret_cast<int4*>(X)[i] = inf4;
    reinterpret_cast<int4*>(Ex)[i] = inf4;
    if (R) reinterpret_cast<int4*>(R)[i] = inf4;
  }
  for (size_t i = n4 * 4 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += stride) {
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
    ctl->pushes = fastest ? 0ull : Q;
    ctl->chunks = 0;
    ctl->smalls = 0;
    ctl->work_all = 0;
    ctl->expansions = 0;
    ctl->index_lookups = 0;
  }
  if (q >= Q || fastest) return;
  const uint32_t item = q * n + qp[q].root;
  X[item] = qp[q].klo;
  atomicOr(bitmap + (item >> 5), 1u << (item & 31));
  fa[q] = item;
}

}  // namespace tgxd
