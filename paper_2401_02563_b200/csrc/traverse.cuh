// Frontier traversal on the device T-CSR — the hot path of
// earliest_arrival / latest_departure / fastest_path
// (reference: path_algorithms.cpp:262-357,436-528 driving temporal_edge_map,
// engine.hpp:239-353).
//
// One persistent cooperative kernel runs the whole query. Each round is
//   A  expand: every frontier vertex locates the not-yet-relaxed admissible
//      key range of its segment (selective index: fence search for hubs,
//      plain binary search otherwise) and emits it as work — ranges of >= 32
//      edges as fixed-size chunks, shorter ones into a small-range list
//      (warp-aggregated atomic emission, no ordered scan). The frontier is
//      either the sparse queue of vertices pushed last round or, when large,
//      implicit (dense): every vertex whose label moved below the bound it
//      was last expanded with (temporal_edge_map's sparse/dense switch,
//      engine.hpp:280-295).
//   B  relax: warps stream chunks (coalesced, unrolled, L2 evict-first) and
//      pack 32 small ranges per warp (lane ownership from a redux.or start
//      mask), relax labels with atomicMin and, when the next round is
//      sparse, append each vertex's first improvement of the round to the
//      next frontier through per-warp shared-memory push buffers.
// Rounds are separated by grid barriers; no host round trip per round.
// Rounds with a tiny frontier run on one CTA with CTA barriers only
// ("local" rounds) and hand back to the whole grid when work grows.
//
// Work efficiency. Labels only decrease (key space) and the relaxed value of
// an edge (its val) does not depend on the label that admitted it, so once an
// edge has been relaxed it never needs relaxing again. Each vertex remembers
// the bound it was last expanded with (Ex); a re-expansion only walks the
// keys in [new bound, old bound). Every admissible edge is relaxed exactly
// once per query (once per sweep for fastest), whatever the schedule — the
// labels are the unique least fixpoint the reference's round-synchronous
// loop also reaches, so results are bit-identical.
//
// Frontier dedup without flags. After every expand phase each reached vertex
// v satisfies Ex[v] == bound(X[v]). During relax, the atomicMin that returns
// old with bound(old) == Ex[v] is therefore the first improvement of v in
// this round: exactly one thread pushes v (claim_stamp, parallel.hpp:113-121).
#pragma once

#include <cooperative_groups.h>

#include "tgxd_internal.cuh"

namespace cg = cooperative_groups;

namespace tgxd {

#ifndef TGXD_UNROLL
#define TGXD_UNROLL 4
#endif
#ifndef TGXD_MIN_BLOCKS
#define TGXD_MIN_BLOCKS 4
#endif
// Phase functions are inlined (measured: out of line, the calls' stack
// traffic costs ~25% on config 2); TGXD_NOINLINE_PHASES builds them as calls.
#ifdef TGXD_NOINLINE_PHASES
#define TGXD_PHASE __noinline__
#else
#define TGXD_PHASE
#endif
#ifndef TGXD_LOCAL_F
#define TGXD_LOCAL_F 128
#endif
#ifndef TGXD_THREADS
#define TGXD_THREADS 256
#endif
constexpr int kThreads = TGXD_THREADS;
constexpr int kWarps = kThreads / 32;
constexpr int kUnroll = TGXD_UNROLL;             // 32-edge steps in flight per warp
constexpr uint32_t kChunk = 32u * kUnroll;       // edges per chunk of a big range
#ifndef TGXD_SMALL
#define TGXD_SMALL 32
#endif
constexpr uint32_t kSmall = TGXD_SMALL;          // ranges below this go to the small list
constexpr uint32_t kChunkLenBits = 10;           // kChunk <= 512
constexpr uint32_t kSmallCntBits = 6;
constexpr uint32_t kLocalMaxF = TGXD_LOCAL_F;    // frontier that one CTA expands
constexpr uint32_t kLocalMaxW = 4096;            // edge work that one CTA relaxes

struct TravArgs {
  DevCsr g;            // push layout
  DevCsr rg;           // reverse layout (pull rounds)
  const QueryParam* qp;
  int32_t* X;          // labels, Q x n (key space)
  int2* EP;            // per slot {bound it was last expanded with, position of
                       // that bound in its segment (kNoPos: unknown)}
  int32_t* R;          // fastest durations / BFS hop counts (nullptr otherwise)
  int hops;            // temporal BFS: R[v] = the round v's arrival first improved
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
  unsigned long long dense_f;  // AUTO: frontier above this expands densely
  unsigned long long push_w;   // AUTO: rounds relaxing more edges do not push
  unsigned long long pull_f;   // AUTO: a frontier at least this big is pulled
  unsigned int pull_grow;      // ... if it also grew by at least this factor over the previous
                               // round's (0: no growth condition)
  unsigned long long handoff_f;  // AUTO: a shrinking frontier this small goes to the cluster tail engine
  unsigned long long async_f;    // AUTO: a frontier this small goes to the async engine when it
                                 // grows by less than handoff_growth per round (or shrinks,
                                 // with async_grow_only == 0)
  unsigned int handoff_growth;
  int async_grow_only;
  // fastest sweep: one query (split == 1), or `split` sub-sweeps over
  // interleaved candidate subsets, one query slot each (Q == split; see
  // split_seed_step)
  int fastest;
  uint32_t split;
  int split_forced;        // split is the width (tests), not a cap for split_width
  int32_t* dep;            // split > 1: departure of each sub-sweep's current candidate
  const uint32_t* n_cand;  // device: candidate count (candidates.cuh), ascending lists
  const uint32_t* cand_lo;
  const uint32_t* cand_cnt;
  const int32_t* cand_key;
  // optional per-round trace (block 0), 8 u64 per round, plus per-warp
  // phase completion extremes (device memory, 4 u64 per round)
  unsigned long long* trace;
  unsigned long long* wtrace;
  int wtrace_on;
  uint32_t trace_cap;
  uint32_t round_limit;  // watchdog: a correct traversal never gets near it
  // early host copy of EA / LD labels (api.cu): a frontier past its peak and
  // at most log_f slots raises *copy_flag (mapped host memory) and from then
  // on every lowered slot is listed in chg
  uint32_t* chg;
  unsigned long long* chg_n;
  unsigned long long chg_cap;
  volatile unsigned int* copy_flag;
  unsigned long long log_f;
  uint32_t* p24;         // non-null: the copy reads labels packed to 24 bits here
  int p24_neg;
  // frontier queue items of slots first reached in the round that queued
  // them carry this bit (0: not used, slots >= 2^31): their expansion state
  // is the initial one, so the expansion skips its load
  uint32_t fresh;
#ifdef TGXD_EXPERIMENTS
  uint32_t x_stop_a;     // experiment: stop before this round's relax (api.cu tgxd_x_relax)
#endif
  unsigned long long init_pushes;  // queue position / improvements after seeding
};

__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

#ifdef TGXD_CHAIN
// diagnostics build: timestamps along the dependent chain of block 0 / warp 0
// in the rounds' phases (api.cu dumps them to TGXD_CHAIN_FILE; tools/chain_trace.py)
__device__ unsigned long long g_chain[64][16];
__device__ unsigned int g_chain_round;
__device__ __forceinline__ void chain_mark(int k, unsigned int consume = 0) {
  __shared__ volatile unsigned int s_sink;
  if (blockIdx.x == 0 && threadIdx.x == 0) {
    s_sink = consume;  // issues once `consume` is available
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t)::"memory");
    if (g_chain_round < 64) g_chain[g_chain_round][k] = t;
  }
}
#define TGXD_MARK(k, v) chain_mark(k, (unsigned int)(v))
#else
#define TGXD_MARK(k, v)
#endif

__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// Streaming read of immutable edge data: no L1 allocation, L2 evict-first
// so the edge stream does not push labels out of L2.
__device__ __forceinline__ int32_t ld_stream(const int32_t* p, uint64_t pol) {
  int32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
               : "=r"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint32_t ld_stream(const uint32_t* p, uint64_t pol) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.b32 %0, [%1], %2;"
               : "=r"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ uint2 ld_stream2(const uint2* p, uint64_t pol) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
               : "=r"(r.x), "=r"(r.y) : "l"(p), "l"(pol));
  return r;
}
// Coherent (L2) read of mutable state, kept resident in L2.
__device__ __forceinline__ int32_t ld_state(const int32_t* p, uint64_t pol) {
  int32_t r;
  asm volatile("ld.global.cg.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31; }

// Expansion prefetch at push time: a slot queued for expansion has the
// {off, kmax} line its expansion starts from pulled into L2 by its pusher
// (level 1, fire and forget), or the pusher reads the segment bounds and
// prefetches the first key and payload lines of a short segment (level 2:
// one DRAM latency for the pushing warp, up to three fewer for the
// expansion). Measured (tools/runs/p1.sh, p2.sh; ms): level 1 in the async
// engine — config 1 0.482 -> 0.461, everything else unchanged — is on;
// level 1 in thin grid rounds (config 2 rotation 1.070 -> 1.075), in the
// cluster tail (neutral) and level 2 anywhere (rotation 1.103, config 1
// 0.49) are off. The engines' expansions read {off, kmax} from the
// interleaved okm line (TGXD_OKM_ENGINES; config 1 -1 %).
#ifndef TGXD_PF_GRID
#define TGXD_PF_GRID 0
#endif
#ifndef TGXD_PF_TAIL
#define TGXD_PF_TAIL 0
#endif
#ifndef TGXD_PF_ASYNC
#define TGXD_PF_ASYNC 1
#endif
#ifndef TGXD_OKM_ENGINES
#define TGXD_OKM_ENGINES 1
#endif
#ifndef TGXD_PF_MAXW
#define TGXD_PF_MAXW (1u << 18)
#endif
constexpr unsigned long long kPfMaxW = TGXD_PF_MAXW;  // a round relaxing more is not latency-bound
__device__ __forceinline__ void pf_l2(const void* p) {
  asm volatile("prefetch.global.L2::evict_last [%0];" ::"l"(p));
}
template <int kLevel>
__device__ __forceinline__ void prefetch_expansion(const uint2* okm, const int32_t* key,
                                                   const uint2* pay, uint32_t v) {
  if (kLevel >= 2) {
    const uint32_t s = __ldg(&okm[v].x), t = __ldg(&okm[v + 1].x);
    if (t > s && t - s <= 32) {
      pf_l2(key + s);
      if (((s ^ (t - 1)) >> 5) != 0) pf_l2(key + t - 1);
      pf_l2(pay + s);
      if (((s ^ (t - 1)) >> 4) != 0) pf_l2(pay + t - 1);
    }
  } else if (kLevel == 1) {
    pf_l2(okm + v);
  }
}

// Debug builds (-DTGXD_CHECK): every queue / work-list store is checked
// against its allocation; a violation is recorded (and the store skipped)
// and reported by the host as an internal error.
#ifdef TGXD_CHECK
__device__ unsigned long long g_cap[2];  // [0] frontier queue entries, [1] work-list entries
__device__ unsigned int g_check_fail;
#define TGXD_IN_CAP(idx, which) \
  ((unsigned long long)(idx) < g_cap[which] || (atomicExch(&g_check_fail, 1u + (which)), false))
#else
#define TGXD_IN_CAP(idx, which) true
#endif

// The bound a label implies for its vertex's next expansion (min_start /
// max_end hooks, path_algorithms.cpp:287-291, :337-342).
__device__ __forceinline__ int32_t bound_of(int32_t x, int strict) {
  return x == kInf ? kInf : x + strict;
}

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
  if (TGXD_IN_CAP(base - pstart + lane, 0)) fout[base - pstart + lane] = v;
  __syncwarp();
  if (lane + 32 < pb.n) pb.buf[lane] = tail;
  pb.n -= 32;
  __syncwarp();
}

// The relax's variant: kPushFlush staged entries per reservation (buffers of
// kPushFlush + 32 entries: the round kernel's). The pushes counter is one
// address: at 0.66 ns per atomic a heavy round's ~85K 32-entry reservations
// kept it busy for half the phase. Config 2 rotation / config 4 fastest, ms:
// 32 entries 1.020 / 4.23, 64 0.969 / 3.97, 128 0.964 / 3.91, 256 0.965 / 3.93
// (profiles/r02ap; the work lists' granule kListFlush stays 32: 64 equal, 128 slower).
#ifndef TGXD_PUSH_FLUSH
#define TGXD_PUSH_FLUSH 128
#endif
constexpr uint32_t kPushFlush = TGXD_PUSH_FLUSH;
static_assert(kPushFlush % 32 == 0 && kPushFlush >= 32, "whole 32-entry rows");
__device__ __forceinline__ void push_flush_n(PushBuf& pb, Control* ctl,
                                             unsigned long long pstart, uint32_t* fout) {
  const uint32_t lane = lane_id();
  __syncwarp();
  uint32_t v[kPushFlush / 32];
#pragma unroll
  for (uint32_t j = 0; j < kPushFlush / 32; ++j) v[j] = pb.buf[32 * j + lane];
  const uint32_t tail = pb.buf[kPushFlush + lane];
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(&ctl->pushes, (unsigned long long)kPushFlush);
  base = __shfl_sync(0xffffffffu, base, 0) - pstart;
#pragma unroll
  for (uint32_t j = 0; j < kPushFlush / 32; ++j)
    if (TGXD_IN_CAP(base + 32 * j + lane, 0)) fout[base + 32 * j + lane] = v[j];
  __syncwarp();
  if (lane + kPushFlush < pb.n) pb.buf[lane] = tail;
  pb.n -= kPushFlush;
  __syncwarp();
}

__device__ __forceinline__ void push_drain(PushBuf& pb, Control* ctl, unsigned long long pstart,
                                           uint32_t* fout) {
  if (pb.n == 0) return;
  const uint32_t lane = lane_id();
  __syncwarp();
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(&ctl->pushes, (unsigned long long)pb.n);
  base = __shfl_sync(0xffffffffu, base, 0) - pstart;
  for (uint32_t i = lane; i < pb.n; i += 32)
    if (TGXD_IN_CAP(base + i, 0)) fout[base + i] = pb.buf[i];
  pb.n = 0;
  __syncwarp();
}

struct RelaxCtx {
  int32_t vhi0;
  int32_t depart;
  bool push;                 // append first improvements to the next frontier
  unsigned long long pstart; // queue position of the next frontier's start
  uint32_t* fout;
  uint64_t pol_stream, pol_keep;
  uint32_t improved;         // per-lane improvement count (no-push rounds)
  int32_t hop;               // temporal BFS: this round's number (1-based)
  bool log = false;          // list every lowered slot (the host copy has started)
  bool pf = false;           // prefetch pushed slots' expansion lines (thin rounds)
};

// 24-bit packing of key-space labels for the early host copy (api.cu): 4
// labels per 12 bytes, INF as 0xFFFFFF, LD labels negated back to times.
// Threads [tid, nthr) of the caller pack groups [0, ceil(slots / 4)).
__device__ __forceinline__ uint32_t pack24_one(int32_t x, int neg) {
  return x == kInf ? 0xFFFFFFu : (uint32_t)(neg ? -x : x) & 0xFFFFFFu;
}
__device__ __forceinline__ void pack24(const int32_t* X, uint32_t* P, uint64_t slots, int neg,
                                       uint64_t tid, uint64_t nthr) {
  const uint64_t groups = (slots + 3) / 4;
  for (uint64_t i = tid; i < groups; i += nthr) {
    uint32_t u[4];
    if (4 * i + 4 <= slots) {
      const int4 x = __ldcg(reinterpret_cast<const int4*>(X) + i);
      u[0] = pack24_one(x.x, neg);
      u[1] = pack24_one(x.y, neg);
      u[2] = pack24_one(x.z, neg);
      u[3] = pack24_one(x.w, neg);
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) u[k] = 4 * i + k < slots ? pack24_one(__ldcg(X + 4 * i + k), neg) : 0u;
    }
    P[3 * i] = u[0] | (u[1] << 24);
    P[3 * i + 1] = (u[1] >> 8) | (u[2] << 16);
    P[3 * i + 2] = (u[2] >> 16) | (u[3] << 8);
  }
}

// Early host copy (api.cu): once the round kernel signals the copy, every
// slot it lowers afterwards is listed (the tail engines do the same); the
// host patches the listed slots with their final labels. One reservation
// per warp and call.
__device__ __forceinline__ void log_lowered(const TravArgs& a, bool lowered, uint32_t slot) {
  const uint32_t bal = __ballot_sync(0xffffffffu, lowered);
  if (!bal) return;
  const uint32_t lane = lane_id();
  unsigned long long base = 0;
  if (lane == __ffs(bal) - 1) base = atomicAdd(a.chg_n, (unsigned long long)__popc(bal));
  base = __shfl_sync(0xffffffffu, base, __ffs(bal) - 1);
  const unsigned long long k = base + __popc(bal & ((1u << lane) - 1));
  if (lowered && k < a.chg_cap) a.chg[k] = slot;
}

// Relax kUnroll 32-edge steps: e[u] edge ids, q[u] query slots, act[u] lane
// validity. write_min (parallel.hpp:91-99) is a plain label probe followed by
// atomicMin when the probe says the edge can improve.
// Payload loads of kUnroll 32-edge steps (inactive lanes get a no-op edge).
__device__ __forceinline__ void relax_load(const TravArgs& a, const uint32_t (&e)[kUnroll],
                                           const bool (&act)[kUnroll], const RelaxCtx& rx,
                                           uint2 (&pl)[kUnroll]) {
#pragma unroll
  for (int u = 0; u < kUnroll; ++u)
    pl[u] = act[u] ? ld_stream2(a.g.pay + e[u], rx.pol_stream) : make_uint2(0u, kInf);
}

__device__ __forceinline__ void relax_apply(const TravArgs& a, const uint2 (&pl)[kUnroll],
                                            const uint32_t (&q)[kUnroll],
                                            const bool (&act)[kUnroll], RelaxCtx& rx,
                                            PushBuf& pb);

// Fastest: r = min over improvements of (label - departure) is not taken per
// improving edge but per expansion, from the label the slot is expanded
// with (expand_warp, P1): every improvement is followed by an expansion of
// the improved slot before the candidate's rounds end, the last one with
// the candidate's final label, and r needs only the minimum of label -
// departure (path_algorithms.cpp:519-523) — one probe and at most one
// atomicMin per expansion instead of one per improving edge (config 4
// fastest 5.11 -> 4.66 ms). Split sweeps (split_seed_step) give every query
// slot its own departure (dep[q]); the round's `depart` is then kSplitDepart.
constexpr int32_t kSplitDepart = INT32_MIN;

__device__ __forceinline__ void relax_steps(const TravArgs& a, const uint32_t (&e)[kUnroll],
                                            const uint32_t (&q)[kUnroll],
                                            const bool (&act)[kUnroll], RelaxCtx& rx,
                                            PushBuf& pb) {
  uint2 pl[kUnroll];
  relax_load(a, e, act, rx, pl);
  relax_apply(a, pl, q, act, rx, pb);
}

__device__ __forceinline__ void relax_apply(const TravArgs& a, const uint2 (&pl)[kUnroll],
                                            const uint32_t (&q)[kUnroll],
                                            const bool (&act)[kUnroll], RelaxCtx& rx,
                                            PushBuf& pb) {
  int32_t v[kUnroll];
  uint32_t idx[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    idx[u] = q[u] * a.n + pl[u].x;
    v[u] = (int32_t)pl[u].y;
  }
  int32_t cur[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    const int32_t vhi = a.Q == 1 ? rx.vhi0 : __ldg(&a.qp[q[u]].vhi);
    // window containment: end <= t_b (types.hpp:55-57)
    if (!(act[u] && v[u] <= vhi)) v[u] = kInf;
#ifdef TGXD_L1_PROBE
    // L1-cached probe: a stale (higher) label only costs an extra atomicMin,
    // which returns the true old value; a stale label is never lower
    if (v[u] != kInf) asm volatile("ld.global.ca.b32 %0, [%1];" : "=r"(cur[u]) : "l"(a.X + idx[u]));
    else cur[u] = kInf;
#else
    cur[u] = v[u] != kInf ? ld_state(a.X + idx[u], rx.pol_keep) : kInf;
#endif
  }
  // all atomics of the batch are in flight before any result is used
  int32_t old[kUnroll], ex[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    old[u] = v[u];  // no atomic issued: not an improvement
    ex[u] = kInf;
    if (v[u] < cur[u]) {
      // the expansion bound decides the first improvement; a slot probed
      // unreached was never expanded (bound INF, no load): its improver that
      // finds old == INF pushes it, later ones see a finite old
#ifdef TGXD_EP_ALWAYS
      if (rx.push) ex[u] = ld_state(reinterpret_cast<const int32_t*>(a.EP + idx[u]), rx.pol_keep);
#else
      if (rx.push && cur[u] != kInf)
        ex[u] = ld_state(reinterpret_cast<const int32_t*>(a.EP + idx[u]), rx.pol_keep);
#endif
      old[u] = atomicMin(a.X + idx[u], v[u]);  // write_min, parallel.hpp:91-99
    }
  }
  if (rx.log) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) log_lowered(a, v[u] < old[u], idx[u]);
  }
  bool p[kUnroll];
#pragma unroll
  for (int u = 0; u < kUnroll; ++u) {
    p[u] = false;
    if (v[u] < old[u]) {
      // BFS: the first improving round (compare_and_swap(r[d], inf, round),
      // path_algorithms.cpp:395-397); fastest's r is taken at expansion
      if (a.hops && old[u] == kInf) a.R[idx[u]] = rx.hop;
      if (rx.push) p[u] = bound_of(old[u], a.strict) == ex[u];
      else ++rx.improved;
    }
  }
  if (rx.push) {
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t bal = __ballot_sync(0xffffffffu, p[u]);
      if (bal) {
        const uint32_t lane = lane_id();
        if (p[u]) pb.buf[pb.n + __popc(bal & ((1u << lane) - 1))] = idx[u] | (old[u] == kInf ? a.fresh : 0u);
        pb.n += __popc(bal);
        if (pb.n >= kPushFlush) push_flush_n(pb, a.ctl, rx.pstart, rx.fout);
      }
    }
#if TGXD_PF_GRID
    if (rx.pf) {
#pragma unroll
      for (int u = 0; u < kUnroll; ++u)
        if (p[u]) prefetch_expansion<TGXD_PF_GRID>(a.g.okm, a.g.key, a.g.pay, pl[u].x);
    }
#endif
  }
}

// ---------------------------------------------------------------------------
// Phase A: expansion. Each warp takes 32 frontier slots at a time. Short
// segments (<= 32 keys) are counted in registers from a handful of 16-byte
// loads; medium segments binary-search per lane; segments at or above the
// index cutoff go through the selective index: a warp-cooperative 32-ary
// search of the fence array (every 32nd key, a compact "bucketed timeline")
// that lands on one 128-byte key line. All three are results-neutral, like
// the reference's TGER-vs-scan choice (test_algorithms.cpp:196-217).
// Emission is buffered per warp in shared memory (no block barriers).


// Per-warp staging of emitted work, appended to the global list kListFlush
// entries per atomic (the list counters are shared by every warp).
#ifndef TGXD_LIST_FLUSH
#define TGXD_LIST_FLUSH 32
#endif
constexpr uint32_t kListFlush = TGXD_LIST_FLUSH;
constexpr uint32_t kListCap = kListFlush + 32;  // entries of one warp buffer

struct WarpList {
  uint2* buf;       // kListCap entries of this warp
  uint32_t n;       // staged entries (warp-uniform)
};

__device__ __forceinline__ void list_flush(WarpList& wl, uint32_t count, unsigned long long* ctr,
                                           unsigned long long start, uint2* list) {
  const uint32_t lane = lane_id();
  __syncwarp();
  unsigned long long base = 0;
  if (lane == 0) base = atomicAdd(ctr, (unsigned long long)count);
  base = __shfl_sync(0xffffffffu, base, 0);
  for (uint32_t k = lane; k < count; k += 32)
    if (TGXD_IN_CAP(base - start + k, 1)) list[base - start + k] = wl.buf[k];
  const uint32_t rem = wl.n - count;  // < 32
  const uint2 t = lane < rem ? wl.buf[count + lane] : make_uint2(0u, 0u);
  __syncwarp();
  if (lane < rem) wl.buf[lane] = t;
  wl.n = rem;
  __syncwarp();
}

__device__ __forceinline__ void list_append(WarpList& wl, bool p, uint2 v, unsigned long long* ctr,
                                            unsigned long long start, uint2* list) {
  const uint32_t bal = __ballot_sync(0xffffffffu, p);
  if (bal == 0) return;
  if (p) wl.buf[wl.n + __popc(bal & ((1u << lane_id()) - 1))] = v;
  wl.n += __popc(bal);
  if (wl.n >= kListFlush) list_flush(wl, kListFlush, ctr, start, list);
}

__device__ __forceinline__ void list_drain(WarpList& wl, unsigned long long* ctr,
                                           unsigned long long start, uint2* list) {
  while (wl.n) list_flush(wl, min(wl.n, kListFlush), ctr, start, list);
}

constexpr uint32_t kNoPos = 0xffffffffu;

// Keys below x in a short range [lo, hi), hi - lo <= 32, from aligned
// 16-byte loads (at most 9, all in flight together).
__device__ __forceinline__ uint32_t line_count(const int32_t* key, uint32_t lo, uint32_t hi,
                                               int32_t x) {
  uint32_t c = 0;
  const uint32_t a0 = lo & ~3u;
#pragma unroll
  for (uint32_t j = 0; j < 9; ++j) {
    const uint32_t p = a0 + 4 * j;
    if (p < hi) {
      const int4 k4 = __ldg(reinterpret_cast<const int4*>(key + p));
      c += (p + 0 >= lo && p + 0 < hi && k4.x < x) ? 1u : 0u;
      c += (p + 1 >= lo && p + 1 < hi && k4.y < x) ? 1u : 0u;
      c += (p + 2 >= lo && p + 2 < hi && k4.z < x) ? 1u : 0u;
      c += (p + 3 >= lo && p + 3 < hi && k4.w < x) ? 1u : 0u;
    }
  }
  return lo + c;
}

#ifndef TGXD_SEARCH_W
#define TGXD_SEARCH_W 8
#endif
constexpr int kSearchW = TGXD_SEARCH_W;  // probes per search step

// W-ary narrowing of [a, b] (the first element >= x of the sorted A lies in
// it): each step issues W independent probes — one memory latency instead
// of log2(W + 1) dependent ones — and keeps the gap between the last probe
// below x and the first one at or above it. A range of <= W + 1 elements is
// resolved exactly in one step.
__device__ __forceinline__ void wide_narrow(const int32_t* A, uint32_t& a, uint32_t& b, int32_t x,
                                            uint32_t stop) {
  while (b - a > stop) {
    const uint32_t len = b - a;
    int32_t v[kSearchW];
#pragma unroll
    for (int k = 0; k < kSearchW; ++k)
      v[k] = __ldg(A + a + (uint32_t)(((unsigned long long)len * (k + 1)) / (kSearchW + 1)));
    uint32_t na = a, nb = b;
#pragma unroll
    for (int k = 0; k < kSearchW; ++k) {
      const uint32_t pk = a + (uint32_t)(((unsigned long long)len * (k + 1)) / (kSearchW + 1));
      if (v[k] < x) na = pk + 1;
    }
#pragma unroll
    for (int k = kSearchW - 1; k >= 0; --k) {
      const uint32_t pk = a + (uint32_t)(((unsigned long long)len * (k + 1)) / (kSearchW + 1));
      if (v[k] >= x) nb = pk;
    }
    a = na;
    b = nb;
  }
}

// lower_bound(x) over key[lo, hi) by one lane. With `fence` (the vertex is
// at or above the index cutoff) the selective index first narrows the range
// to one 32-key line through the fence array (every 32nd key of the layout,
// a compact "bucketed timeline"); otherwise the keys themselves are narrowed
// down to 32. Both with W-ary steps; the last line is counted with vector
// loads. Results-neutral, like the reference's TGER-vs-scan choice
// (test_algorithms.cpp:196-217).
__device__ __forceinline__ uint32_t lane_lower_bound(const DevCsr& g, uint32_t lo, uint32_t hi,
                                                     int32_t x, bool fence) {
  if (fence && hi - lo > 32) {
    const uint32_t jlo = (lo + kFenceStride - 1) >> kFenceShift;
    const uint32_t jhi = (hi - 1) >> kFenceShift;
    uint32_t a = jlo, b = jhi + 1;  // first fence >= x in [jlo, jhi], else jhi + 1
    wide_narrow(g.fence, a, b, x, 0);
    if (a > jlo) lo = max(lo, ((a - 1) << kFenceShift) + 1);
    if (a <= jhi) hi = min(hi, a << kFenceShift);
  }
  if (hi - lo > 32) wide_narrow(g.key, lo, hi, x, 32);
  return line_count(g.key, lo, hi, x);
}


struct ExpandBufs {
  WarpList sm, ch;
  unsigned long long cstart, sstart;
};

// Expansion of one slot per lane (item = q * n + v, label x, previous
// expansion state ep = {bound, position}); the emitted ranges go to the
// warp's lists. All lanes must call it; no lane ever waits on another's
// search.
__device__ __forceinline__ void expand_warp(const TravArgs& a, bool valid, uint32_t item, int32_t x,
                                            int2 ep, uint32_t s, uint32_t t, int32_t km,
                                            ExpandBufs& eb, unsigned long long& work,
                                            unsigned long long& ix, int32_t depart) {
  const uint32_t lane = lane_id();
  uint32_t q = 0, p0 = 0, p1 = 0;
  bool act = false;
  if (valid) {
    q = a.Q == 1 ? 0u : item / a.n;
    const uint32_t v = item - q * a.n;
    const QueryParam& qp = a.qp[q];
    // min_start / max_end hooks (path_algorithms.cpp:287-291, :337-342):
    // the root leaves at any time inside the window; everyone else strictly
    // (or weakly) after its own label.
    int32_t lb = (v == qp.root) ? qp.klo : bound_of(x, a.strict);
    if (lb < qp.klo) lb = qp.klo;
    const int32_t old = ep.x;
    if (a.fastest && lb < old) {  // fastest: r from the expanded label
      const int32_t r = x - (depart == kSplitDepart ? __ldcg(a.dep + q) : depart);
      if (r < __ldcg(a.R + item)) atomicMin(a.R + item, r);
    }
    if (lb < old) {
      const int32_t hik = min(old, qp.vhi + 1);  // keys above vhi cannot fit the window
      uint32_t pos = kNoPos;
      if (lb < hik) {
        // one for_each_window_edge call of the reference (engine.hpp:316),
        // counted in ix's high word; index lookups in its low word
        ix += 1ull << 32;
        // (s, t, km: segment bounds and last key, loaded with the label)
        if (t > s && km >= lb) {
          act = true;
          const bool fence = a.cutoff != 0 && t - s >= a.cutoff;
          ix += fence ? 1 : 0;
          // upper end: the previous expansion's position when that bound is
          // the limit (a re-expansion), else the segment end when every key
          // fits under the window
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
  // short ranges: one small-list entry
  list_append(eb.sm, cnt != 0 && cnt < kSmall, make_uint2(p0, (q << kSmallCntBits) | cnt),
              &a.ctl->smalls, eb.sstart, a.smalls);
  // long ranges: kChunk-edge chunks; medium ones through the warp buffer,
  // huge ones straight to the list with one reservation
  const uint32_t nch = cnt >= kSmall ? (cnt + kChunk - 1) / kChunk : 0u;
  uint32_t bigs = __ballot_sync(0xffffffffu, nch != 0 && nch < 32);
  while (bigs) {
    const uint32_t src = __ffs(bigs) - 1;
    bigs &= bigs - 1;
    const uint32_t B0 = __shfl_sync(0xffffffffu, p0, src), BC = __shfl_sync(0xffffffffu, cnt, src);
    const uint32_t BQ = __shfl_sync(0xffffffffu, q, src);
    const uint32_t bn = __shfl_sync(0xffffffffu, nch, src);
    const uint32_t off = lane * kChunk;
    list_append(eb.ch, lane < bn,
                make_uint2(B0 + off, (BQ << kChunkLenBits) | (lane < bn ? min(kChunk, BC - off) : 0u)),
                &a.ctl->chunks, eb.cstart, a.chunks);
  }
  uint32_t huge = __ballot_sync(0xffffffffu, nch >= 32);
  while (huge) {
    const uint32_t src = __ffs(huge) - 1;
    huge &= huge - 1;
    const uint32_t B0 = __shfl_sync(0xffffffffu, p0, src), BC = __shfl_sync(0xffffffffu, cnt, src);
    const uint32_t BQ = __shfl_sync(0xffffffffu, q, src);
    const uint32_t bn = __shfl_sync(0xffffffffu, nch, src);
    unsigned long long base = 0;
    if (lane == 0) base = atomicAdd(&a.ctl->chunks, (unsigned long long)bn);
    base = __shfl_sync(0xffffffffu, base, 0) - eb.cstart;
    for (uint32_t j = lane; j < bn; j += 32) {
      const uint32_t off = j * kChunk;
      if (TGXD_IN_CAP(base + j, 1))
        a.chunks[base + j] = make_uint2(B0 + off, (BQ << kChunkLenBits) | min(kChunk, BC - off));
    }
  }
}

// Adds a block's relax-work count to the edges counter (one atomic per block).
__device__ __forceinline__ void flush_work(Control* ctl, unsigned long long work) {
  __shared__ unsigned long long s_w[kWarps];
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) work += __shfl_xor_sync(0xffffffffu, work, o);
  if (lane_id() == 0) s_w[threadIdx.x >> 5] = work;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned long long t = 0;
#pragma unroll
    for (int k = 0; k < kWarps; ++k) t += s_w[k];
    if (t) atomicAdd(&ctl->edges, t);
  }
  __syncthreads();
}

// End of an expand phase: the warps' staged list entries and work counts go
// out with ONE reservation per block and list (a spread thin round would
// otherwise end with ~5K same-address atomics on each counter).
__device__ __forceinline__ void block_finish_expand(const TravArgs& a, ExpandBufs& eb,
                                                    unsigned long long work) {
  __shared__ uint32_t s_n[2][kWarps];
  __shared__ unsigned long long s_w[kWarps];
  __shared__ unsigned long long s_base[2];
  const uint32_t lane = lane_id(), w = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) work += __shfl_xor_sync(0xffffffffu, work, o);
  if (lane == 0) {
    s_n[0][w] = eb.sm.n;
    s_n[1][w] = eb.ch.n;
    s_w[w] = work;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t0 = 0, t1 = 0;
    unsigned long long tw = 0;
#pragma unroll
    for (int k = 0; k < kWarps; ++k) {
      const uint32_t c0 = s_n[0][k], c1 = s_n[1][k];
      s_n[0][k] = t0;
      s_n[1][k] = t1;
      t0 += c0;
      t1 += c1;
      tw += s_w[k];
    }
    unsigned long long b0 = 0, b1 = 0;
    if (t0) b0 = atomicAdd(&a.ctl->smalls, (unsigned long long)t0);
    if (t1) b1 = atomicAdd(&a.ctl->chunks, (unsigned long long)t1);
    if (tw) atomicAdd(&a.ctl->edges, tw);
    s_base[0] = b0;
    s_base[1] = b1;
  }
  __syncthreads();
  {
    const unsigned long long b = s_base[0] + s_n[0][w] - eb.sstart;
    for (uint32_t i = lane; i < eb.sm.n; i += 32)
      if (TGXD_IN_CAP(b + i, 1)) a.smalls[b + i] = eb.sm.buf[i];
  }
  {
    const unsigned long long b = s_base[1] + s_n[1][w] - eb.cstart;
    for (uint32_t i = lane; i < eb.ch.n; i += 32)
      if (TGXD_IN_CAP(b + i, 1)) a.chunks[b + i] = eb.ch.buf[i];
  }
  eb.sm.n = eb.ch.n = 0;
  __syncthreads();
}

// End of a relax phase: the warps' staged queue entries with one reservation per block.
__device__ __forceinline__ void block_push_drain(PushBuf& pb, Control* ctl, unsigned long long pstart,
                                                 uint32_t* fout) {
  __shared__ uint32_t s_pn[kWarps];
  __shared__ unsigned long long s_pbase;
  const uint32_t lane = lane_id(), w = threadIdx.x >> 5;
  if (lane == 0) s_pn[w] = pb.n;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t t = 0;
#pragma unroll
    for (int k = 0; k < kWarps; ++k) {
      const uint32_t c = s_pn[k];
      s_pn[k] = t;
      t += c;
    }
    s_pbase = t ? atomicAdd(&ctl->pushes, (unsigned long long)t) : 0ull;
  }
  __syncthreads();
  const unsigned long long b = s_pbase + s_pn[w] - pstart;
  for (uint32_t i = lane; i < pb.n; i += 32)
    if (TGXD_IN_CAP(b + i, 0)) fout[b + i] = pb.buf[i];
  pb.n = 0;
  __syncthreads();
}

// Phase A over a sparse frontier queue (items [0, F) of fin) or, with
// fin == nullptr, over the implicit dense frontier: every slot whose label
// bound is below its expansion bound.
__device__ TGXD_PHASE void phase_a(const TravArgs& a, const uint32_t* fin, uint32_t F,
                        unsigned long long cstart, unsigned long long sstart, uint32_t bid,
                        uint32_t nblk, uint64_t pol_keep, uint2* ebuf, unsigned long long& ix,
                        int32_t depart) {
  const uint32_t lane = lane_id();
  const uint32_t gw = bid * kWarps + (threadIdx.x >> 5);
  const uint32_t nw = nblk * kWarps;
  const uint32_t total = fin ? F : a.Q * a.n;
  ExpandBufs eb{{ebuf, 0}, {ebuf + kListCap, 0}, cstart, sstart};
  unsigned long long work = 0;
  TGXD_MARK(0, 0);
  // a queue that does not fill every warp is spread over all of them (ipw
  // slots per warp): a thin round's time is the one warp-iteration that has
  // work, and 32 lanes in different branches of the search serialise in it
#ifndef TGXD_NO_SPREAD
  const uint32_t ipw = fin ? min(32u, max(1u, (total + nw - 1) / nw)) : 32u;
#else
  const uint32_t ipw = 32u;
#endif
  for (uint32_t base = gw * ipw; base < total; base += nw * ipw) {
    const uint32_t i = base + lane;
    bool valid = lane < ipw && i < total;
    uint32_t item = i;
    int32_t x = kInf;
    int2 ep = make_int2(kInf, (int32_t)kNoPos);
    uint32_t s0 = 0, t0 = 0;
    int32_t km0 = INT32_MIN;
    if (valid) {
      bool fresh = false;
      if (fin) {
        item = __ldcg(fin + i);
        fresh = (item & a.fresh) != 0;
        item &= ~a.fresh;
      }
      x = ld_state(a.X + item, pol_keep);
      if (!fresh) ep = __ldcg(a.EP + item);  // (a fresh slot's is the initial state)
      // the segment's bounds and last key do not depend on the label: issue
      // them with it (one dependent load less per expansion)
      const uint32_t v = a.Q == 1 ? item : item % a.n;
      // segment bounds and last key from the interleaved {off, kmax} array:
      // one 128-byte line per random miss instead of two (config 2 rotation
      // 1.110 -> 1.099 ms, config 4 fastest 5.20 -> 5.09)
      const uint2 ok = __ldg(a.g.okm + v);
      s0 = ok.x;
      km0 = (int32_t)ok.y;
      t0 = __ldg(&a.g.okm[v + 1].x);
      valid = x != kInf;
    }
    if (base == gw * ipw) {
      TGXD_MARK(1, item);
      TGXD_MARK(2, x + ep.x + s0 + t0 + km0);
    }
    expand_warp(a, valid, item, x, ep, s0, t0, km0, eb, work, ix, depart);
    if (base == gw * ipw) TGXD_MARK(3, eb.sm.n + eb.ch.n + (uint32_t)work);
  }
#ifdef TGXD_WARP_DRAIN
  list_drain(eb.sm, &a.ctl->smalls, sstart, a.smalls);
  list_drain(eb.ch, &a.ctl->chunks, cstart, a.chunks);
  TGXD_MARK(4, eb.sm.n);
  flush_work(a.ctl, work);
#else
  TGXD_MARK(4, eb.sm.n);
  block_finish_expand(a, eb, work);
#endif
  TGXD_MARK(5, 0);
}

#ifdef TGXD_TMA_RELAX
// Chunk payloads staged through shared memory by the TMA engine (1-D bulk
// copies, cp.async.bulk + mbarrier complete_tx): the copy of the next chunk
// is in flight while the current one is relaxed. Per warp two buffers of
// kChunk + 2 entries (the copy starts at the 16-byte-aligned entry at or
// below the chunk's first) and two mbarriers.
constexpr uint32_t kTmaEntries = kChunk + 2;
struct TmaBufs {
  uint2* buf;                // 2 x kTmaEntries
  unsigned long long* bar;   // 2 mbarriers
  uint32_t* parity;          // per-buffer phase bits (bit b)
};
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void tma_issue(const TmaBufs& t, int b, const uint2* pay, uint32_t first,
                                          uint32_t len, uint64_t pol) {
  if (lane_id() == 0) {
    const uint32_t a0 = first & ~1u;
    const uint32_t bytes = (((first + len + 1) & ~1u) - a0) * 8u;
    const uint32_t bar = smem_u32(t.bar + b);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint "
        "[%0], [%1], %2, [%3], %4;" ::"r"(smem_u32(t.buf + b * kTmaEntries)),
        "l"(pay + a0), "r"(bytes), "r"(bar), "l"(pol)
        : "memory");
  }
}
__device__ __forceinline__ void tma_wait(const TmaBufs& t, int b) {
  const uint32_t bar = smem_u32(t.bar + b);
  const uint32_t ph = (*t.parity >> b) & 1u;
  uint32_t done = 0;
  while (!done) {
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(bar), "r"(ph)
        : "memory");
  }
  __syncwarp();
  if (lane_id() == 0) *t.parity ^= 1u << b;
  __syncwarp();
}
#endif

// One window of 32 small ranges (lane l's entry sv = {lo, q << 6 | cnt}):
// items packed densely, each lane finding its owner from the mask of range
// starts, kUnroll 32-edge steps at a time.
__device__ __forceinline__ void relax_window(const TravArgs& a, uint2 sv, RelaxCtx& rx,
                                             PushBuf& pb) {
  const uint32_t lane = lane_id();
  const uint32_t lo = sv.x;
  const uint32_t cnt = sv.y & ((1u << kSmallCntBits) - 1);
  const uint32_t rq = sv.y >> kSmallCntBits;
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
      const uint32_t own = (i0 + __popc(mask & ((2u << lane) - 1))) & 31;
      const uint32_t olo = __shfl_sync(0xffffffffu, lo, own);
      const uint32_t ost = __shfl_sync(0xffffffffu, start, own);
      const uint32_t oq = __shfl_sync(0xffffffffu, rq, own);
      const uint32_t t = sb + lane;
      act[u] = t < total;
      e[u] = olo + (t - ost);
      q[u] = oq;
    }
    relax_steps(a, e, q, act, rx, pb);
  }
}

// Phase B: relax the round's chunks and small ranges (plus, for a fastest
// seed round, the virtual chunks of one explicit range).
#ifdef TGXD_TMA_RELAX
__device__ TmaBufs tma_bufs_of_warp();
#endif
__device__ TGXD_PHASE void phase_b(const TravArgs& a, unsigned long long nchunks, unsigned long long nsmall,
                        uint32_t xlo,
                        uint32_t xcnt, RelaxCtx& rx, uint32_t bid, uint32_t nblk,
                        uint32_t* wbuf) {
  const uint32_t lane = lane_id();
  const uint32_t gw = bid * kWarps + (threadIdx.x >> 5);
  const uint32_t nw = nblk * kWarps;
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
    relax_steps(a, e, q, act, rx, pb);
  }

  // chunks of big ranges: coalesced kChunk-edge bursts (software-pipelining
  // the next chunk's payload loads measured no gain: the relax is bound by
  // the L2 atomic rate, ~150 G/s when most edges improve)
#ifdef TGXD_TMA_RELAX
  if (gw < nchunks) {
    const TmaBufs tb = tma_bufs_of_warp();
    // descriptor of chunk c in `cur`, of c + nw in `nxt`; the copy of c is
    // in buffer cb, issued one iteration ahead
    uint2 cur = __ldcg(a.chunks + gw);
    uint2 nxt = gw + nw < nchunks ? __ldcg(a.chunks + gw + nw) : make_uint2(0u, 0u);
    int cb = 0;
    tma_issue(tb, cb, a.g.pay, cur.x, cur.y & ((1u << kChunkLenBits) - 1), rx.pol_stream);
    for (unsigned long long c = gw; c < nchunks; c += nw) {
      const uint2 ch = cur;
      const bool more = c + nw < nchunks;
      if (more) {
        tma_issue(tb, cb ^ 1, a.g.pay, nxt.x, nxt.y & ((1u << kChunkLenBits) - 1), rx.pol_stream);
        cur = nxt;
        if (c + 2ull * nw < nchunks) nxt = __ldcg(a.chunks + c + 2ull * nw);
      }
      const uint32_t len = ch.y & ((1u << kChunkLenBits) - 1);
      const uint32_t cq = ch.y >> kChunkLenBits;
      tma_wait(tb, cb);
      const uint2* sb = tb.buf + cb * kTmaEntries + (ch.x - (ch.x & ~1u));
      uint2 pl[kUnroll];
      uint32_t q[kUnroll];
      bool act[kUnroll];
#pragma unroll
      for (int u = 0; u < kUnroll; ++u) {
        const uint32_t off = u * 32 + lane;
        act[u] = off < len;
        q[u] = cq;
        pl[u] = act[u] ? sb[off] : make_uint2(0u, kInf);
      }
      __syncwarp();
      relax_apply(a, pl, q, act, rx, pb);
      cb ^= 1;
    }
  }
  for (unsigned long long c = nchunks; false;) {
    const uint2 ch = make_uint2(0u, 0u);
#else
  uint2 nxt = gw < nchunks ? __ldcg(a.chunks + gw) : make_uint2(0u, 0u);
  for (unsigned long long c = gw; c < nchunks; c += nw) {
    const uint2 ch = nxt;  // descriptor prefetched one iteration ahead
    if (c + nw < nchunks) nxt = __ldcg(a.chunks + c + nw);
#endif
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
    relax_steps(a, e, q, act, rx, pb);
  }

  // small ranges: 32 per warp window, static shares (a window holds 32 to
  // ~1000 edges; taking windows from an atomic cursor instead measured 4 %
  // slower on config 2's rotation — the cursor's line slows its L2 slice)
  // (a list that does not fill every warp's window is spread: epw ranges per window)
#ifndef TGXD_NO_SPREAD
  const uint32_t epw = (uint32_t)min(32ull, max(1ull, (nsmall + nw - 1) / nw));
#else
  const uint32_t epw = 32u;
#endif
  const unsigned long long nwin = (nsmall + epw - 1) / epw;
  auto win_load = [&](unsigned long long w) -> uint2 {
    const unsigned long long i = w * epw + lane;
    return (w < nwin && lane < epw && i < nsmall) ? __ldcg(a.smalls + i) : make_uint2(0u, 0u);
  };
  // chunks and windows are one sequence of work units dealt round-robin:
  // the windows continue where the chunks end, so the warps that took one
  // chunk fewer start on the windows first
#ifdef TGXD_SPLIT_UNITS
  const unsigned long long w0 = gw;
#else
  const unsigned long long w0 =
      (gw >= nchunks ? gw : gw + (nchunks - gw + nw - 1) / nw * nw) - nchunks;
#endif
  TGXD_MARK(8, 0);
  uint2 sv = win_load(w0);
  TGXD_MARK(9, sv.x + sv.y);
  for (unsigned long long w = w0; w < nwin; w += nw) {
    const uint2 snx = win_load(w + nw);  // next window prefetched
    relax_window(a, sv, rx, pb);
    if (w == w0) TGXD_MARK(10, pb.n);
    sv = snx;
  }
  if (rx.push) block_push_drain(pb, a.ctl, rx.pstart, rx.fout);
  TGXD_MARK(11, pb.n);
}

// ---------------------------------------------------------------------------
// Pull round (the dense "bottom-up" direction of temporal_edge_map,
// engine.hpp:321-346): every slot considers the in-edges (reverse layout)
// that could lower its label — arrival below the current label and inside
// the window, a suffix of its key-sorted segment found with the same index
// search as the push side — and takes the smallest candidate admissible
// under the current labels. Afterwards every edge admissible under the
// round-start labels has been considered, so each slot's expansion bound
// becomes bound(start label); slots the pull improved are queued for a push
// expansion of their new delta. On config 2 the two heaviest push rounds
// (17.8M + 37.9M edge relaxations) need 11.4M + 6.2M in-edge checks.
//
//   P1  one lane per slot finds its candidate window; short windows
//       (<= kPullLane entries) are scanned in candidate order with batched
//       loads, stopping at the first admissible entry. Long windows (a few
//       thousand slots whose in-degree runs into the thousands) become
//       kChunk-entry pull chunks {first position, slot}.
//   P2  all warps take pull chunks; a chunk's smallest admissible candidate
//       (warp min) goes in with one atomicMin, and the slot is queued on its
//       first improvement (bound(old) == the EP bound P1 stored), the push
//       rule of relax_steps.
//
// Reverse layout in key space (see DevCsr): for the push layout's edge
// (key_P, val_P) the reverse entry has key_R = -val_P, val_R = -key_P, so a
// candidate is -key_R and the admissibility key is -val_R; positions
// descending = candidates ascending.
#ifndef TGXD_PULL_LANE
#define TGXD_PULL_LANE 16
#endif
#ifndef TGXD_PULL_BATCH
#define TGXD_PULL_BATCH 8
#endif
constexpr uint32_t kPullLane = TGXD_PULL_LANE;    // longest window a lane scans by itself
constexpr uint32_t kPullBatch = TGXD_PULL_BATCH;  // entries in flight per lane while scanning

// Is the reverse entry with payload pl admissible for query q under the
// current labels? (the admissibility test of relax, path_algorithms.cpp:287-300)
__device__ __forceinline__ bool pull_admissible(const TravArgs& a, uint2 pl, uint32_t q,
                                                const QueryParam& qp, uint64_t pol_keep) {
  const int32_t kp = -(int32_t)pl.y;
  if (kp < qp.klo) return false;
  if (pl.x == qp.root) return true;
  const int32_t xs = ld_state(a.X + q * a.n + pl.x, pol_keep);
  return xs != kInf && kp >= bound_of(xs, a.strict);
}

// Warp-shared list of 64 slots: append with a ballot, take 32 at a time.
__device__ __forceinline__ void slot_list_push(uint2* buf, uint32_t& n, bool p, uint2 v) {
  const uint32_t bal = __ballot_sync(0xffffffffu, p);
  if (p) buf[n + __popc(bal & ((1u << lane_id()) - 1))] = v;
  n += __popc(bal);
  __syncwarp();
}
__device__ __forceinline__ void slot_list_pop(uint2* buf, uint32_t& n, uint32_t taken) {
  const uint32_t lane = lane_id();
  __syncwarp();
  const uint2 t = taken + lane < 64 ? buf[taken + lane] : make_uint2(0u, 0u);
  __syncwarp();
  if (lane + taken < n) buf[lane] = t;
  n -= taken;
  __syncwarp();
}

__device__ __forceinline__ void slot_list_push4(uint4* buf, uint32_t& n, bool p, uint4 v) {
  const uint32_t bal = __ballot_sync(0xffffffffu, p);
  if (p) buf[n + __popc(bal & ((1u << lane_id()) - 1))] = v;
  n += __popc(bal);
  __syncwarp();
}
__device__ __forceinline__ void slot_list_pop4(uint4* buf, uint32_t& n, uint32_t taken) {
  const uint32_t lane = lane_id();
  __syncwarp();
  const uint4 t = taken + lane < 64 ? buf[taken + lane] : make_uint4(0u, 0u, 0u, 0u);
  __syncwarp();
  if (lane + taken < n) buf[lane] = t;
  n -= taken;
  __syncwarp();
}

struct PullBufs {
  PushBuf pb;
  WarpList chl;          // pull chunks
  uint4* obuf;           // open slots {slot, lim, segment start, segment end}
  uint2* rbuf;           // long windows {slot, lim}
  uint32_t no, nr;
  unsigned long long cstart;
};

// Long windows: the rest of the window below the lane-scanned entries,
// [lower_bound(1 - lim), t - kPullLane), goes out as pull chunks, those
// nearest the smallest candidates first. One window per lane.
__device__ TGXD_PHASE void pull_search32(const TravArgs& a, PullBufs& b, uint32_t cnt) {
  const DevCsr& rg = a.rg;
  const uint32_t lane = lane_id();
  const bool act = lane < cnt;
  const uint2 r = act ? b.rbuf[lane] : make_uint2(0u, 0u);
  uint32_t p = 0, j = 0;
  if (act) {
    const uint32_t q = a.Q == 1 ? 0u : r.x / a.n;
    const uint32_t v = r.x - q * a.n;
    const uint32_t s = __ldg(rg.off + v);
    j = __ldg(rg.off + v + 1) - kPullLane;
    p = lane_lower_bound(rg, s, j, 1 - (int32_t)r.y, a.cutoff != 0 && j - s >= a.cutoff);
  }
  slot_list_pop(b.rbuf, b.nr, cnt);
  const uint32_t nch = act ? (j - p + kChunk - 1) / kChunk : 0u;
  uint32_t bigs = __ballot_sync(0xffffffffu, nch != 0);
  while (bigs) {
    const uint32_t L = __ffs(bigs) - 1;
    bigs &= bigs - 1;
    const uint32_t I = __shfl_sync(0xffffffffu, r.x, L);
    const uint32_t bn = __shfl_sync(0xffffffffu, nch, L);
    const uint32_t P = __shfl_sync(0xffffffffu, p, L);
    for (uint32_t k0 = 0; k0 < bn; k0 += 32) {
      // chunk k covers [P + k kChunk, min(P + (k+1) kChunk, window end))
      const uint32_t k = bn - 1 - min(k0 + lane, bn - 1);
      list_append(b.chl, k0 + lane < bn, make_uint2(P + k * kChunk, I), &a.ctl->pchunks, b.cstart,
                  a.chunks);
    }
  }
}

// Open slots (some in-edge below the label): one per lane, the smallest
// candidates first, kPullBatch entries in flight, until the first admissible
// one or the end of the window; windows longer than kPullLane entries go to
// the long-window list.
__device__ TGXD_PHASE void pull_scan32(const TravArgs& a, RelaxCtx& rx, PullBufs& b, uint32_t cnt,
                            unsigned long long& scanned) {
  const DevCsr& rg = a.rg;
  const uint32_t lane = lane_id();
  const bool act = lane < cnt;
  const uint4 o = act ? b.obuf[lane] : make_uint4(0u, 0u, 0u, 0u);
  slot_list_pop4(b.obuf, b.no, cnt);
  const uint32_t i = o.x;
  const int32_t lim = (int32_t)o.y;
  int32_t best = kInf;
  bool open = act;
  if (act) {
    const uint32_t q = a.Q == 1 ? 0u : i / a.n;
    const QueryParam& qp = a.qp[q];
    const uint32_t s = o.z;  // segment bounds came with the sweep's coalesced loads
    uint32_t j = o.w;
    for (uint32_t k = 0; open && k < kPullLane; k += kPullBatch) {
      int32_t kr[kPullBatch];
      uint2 pl[kPullBatch];
#pragma unroll
      for (uint32_t e = 0; e < kPullBatch; ++e) {
        const bool in = j > s + e;
        kr[e] = in ? __ldg(rg.key + j - 1 - e) : kInf;
        pl[e] = in ? __ldg(rg.pay + j - 1 - e) : make_uint2(0u, 0x7fffffffu);
      }
      uint32_t stop = kPullBatch;  // first entry outside the window (keys ascend)
#pragma unroll
      for (int e = kPullBatch - 1; e >= 0; --e)
        if (j <= s + e || -kr[e] >= lim) stop = e;
      bool adm[kPullBatch];
#pragma unroll
      for (uint32_t e = 0; e < kPullBatch; ++e)
        adm[e] = e < stop && pull_admissible(a, pl[e], q, qp, rx.pol_keep);
      uint32_t hit = stop;
#pragma unroll
      for (int e = kPullBatch - 1; e >= 0; --e)
        if (adm[e]) hit = e;
#pragma unroll
      for (uint32_t e = 0; e < kPullBatch; ++e)
        if (e == hit && hit < stop) best = -kr[e];
      scanned += min(hit + 1, stop);
      if (hit < stop || stop < kPullBatch) open = false;
      j -= kPullBatch;
    }
  }
  // every candidate is below the label, so finding one improves it
  const bool improved = best != kInf;
  if (improved) {
    a.X[i] = best;
  }
  if (rx.log) log_lowered(a, improved, i);
  const uint32_t bal = __ballot_sync(0xffffffffu, improved);
  if (bal) {
    // (lim == vhi + 1: the slot was unreached — a reached label lies in the window)
    const bool fresh = a.Q == 1 ? lim == a.qp[0].vhi + 1 : lim == a.qp[i / a.n].vhi + 1;
    if (improved) b.pb.buf[b.pb.n + __popc(bal & ((1u << lane) - 1))] = i | (fresh ? a.fresh : 0u);
    b.pb.n += __popc(bal);
    if (b.pb.n >= kPushFlush) push_flush_n(b.pb, a.ctl, rx.pstart, rx.fout);
  }
  slot_list_push(b.rbuf, b.nr, open, make_uint2(o.x, o.y));
  if (b.nr >= 32) pull_search32(a, b, 32);
}

#ifndef TGXD_PULL_SLOTS
#define TGXD_PULL_SLOTS 1
#endif
constexpr uint32_t kPullSlots = TGXD_PULL_SLOTS;  // slot groups per lane in flight in the sweep

__device__ TGXD_PHASE void phase_pull1(const TravArgs& a, RelaxCtx& rx, unsigned long long cstart,
                            uint32_t bid, uint32_t nblk, uint32_t* wbuf, uint2* ebuf,
                            uint2* rbuf, uint4* obuf, unsigned long long& scanned) {
  const DevCsr& rg = a.rg;
  const uint32_t lane = lane_id();
  const uint32_t gw = bid * kWarps + (threadIdx.x >> 5);
  const uint32_t nw = nblk * kWarps;
  const uint32_t slots = a.Q * a.n;
  PullBufs b{{wbuf, 0}, {ebuf, 0}, obuf, rbuf, 0, 0, cstart};
  // label sweep: coalesced labels and last keys; slots with an in-edge below
  // their label are queued for the scan
  for (uint32_t base = gw * 32 * kPullSlots; base < slots; base += nw * 32 * kPullSlots) {
    int32_t x[kPullSlots], km[kPullSlots];
    uint32_t sg[kPullSlots], tg[kPullSlots];
#pragma unroll
    for (uint32_t u = 0; u < kPullSlots; ++u) {
      const uint32_t i = base + u * 32 + lane;
      const uint32_t q = a.Q == 1 ? 0u : i / a.n;
      const uint32_t v = i - q * a.n;
      x[u] = i < slots ? ld_state(a.X + i, rx.pol_keep) : kInf;
      km[u] = i < slots ? __ldg(rg.kmax + v) : INT32_MIN;
      // segment bounds ride along (coalesced): the scan starts at the keys
      sg[u] = i < slots ? __ldg(rg.off + v) : 0u;
      tg[u] = i < slots ? __ldg(rg.off + v + 1) : 0u;
    }
#pragma unroll
    for (uint32_t u = 0; u < kPullSlots; ++u) {
      const uint32_t i = base + u * 32 + lane;
      bool open = false;
      int32_t lim = 0;
      if (i < slots) {
        const uint32_t q = a.Q == 1 ? 0u : i / a.n;
        const QueryParam& qp = a.qp[q];
        // candidates below lim: key_R >= 1 - lim, a suffix of the segment
        lim = min(x[u], qp.vhi + 1);
        open = km[u] >= 1 - lim;
        // every edge admissible under the round-start label is considered now
        if (x[u] != kInf) {
          int32_t lb = (i - q * a.n == qp.root) ? qp.klo : bound_of(x[u], a.strict);
          if (lb < qp.klo) lb = qp.klo;
          a.EP[i] = make_int2(lb, (int32_t)kNoPos);
          if (a.fastest) {  // fastest: r from the label the pull starts from
            const int32_t r = x[u] - (rx.depart == kSplitDepart ? __ldcg(a.dep + q) : rx.depart);
            if (r < __ldcg(a.R + i)) atomicMin(a.R + i, r);
          }
        }
      }
      slot_list_push4(b.obuf, b.no, open, make_uint4(i, (uint32_t)lim, sg[u], tg[u]));
      if (b.no >= 32) pull_scan32(a, rx, b, 32, scanned);
    }
  }
  while (b.no) pull_scan32(a, rx, b, min(b.no, 32u), scanned);
  while (b.nr) pull_search32(a, b, min(b.nr, 32u));
  push_drain(b.pb, a.ctl, rx.pstart, rx.fout);
  list_drain(b.chl, &a.ctl->pchunks, cstart, a.chunks);
}

// P2: one warp per pull chunk, kUnroll entries per lane. A chunk's entries
// run from its first position to min(first + kChunk, window end).
__device__ TGXD_PHASE void phase_pull2(const TravArgs& a, RelaxCtx& rx, unsigned long long nch, uint32_t bid,
                            uint32_t nblk, uint32_t* wbuf, unsigned long long& scanned) {
  const DevCsr& rg = a.rg;
  const uint32_t lane = lane_id();
  const uint32_t gw = bid * kWarps + (threadIdx.x >> 5);
  const uint32_t nw = nblk * kWarps;
  PushBuf pb{wbuf, 0};
  for (unsigned long long c = gw; c < nch; c += nw) {
    const uint2 ch = __ldcg(a.chunks + c);
    const uint32_t slot = ch.y;
    const uint32_t q = a.Q == 1 ? 0u : slot / a.n;
    const uint32_t v = slot - q * a.n;
    const QueryParam& qp = a.qp[q];
    // P1 already scanned the last kPullLane entries of the segment
    const uint32_t hi = min(__ldg(rg.off + v + 1) - kPullLane, ch.x + kChunk);
    int32_t kr[kUnroll];
    uint2 pl[kUnroll];
#pragma unroll
    for (int u = 0; u < kUnroll; ++u) {
      const uint32_t j = ch.x + u * 32 + lane;
      const bool in = j < hi;
      kr[u] = in ? ld_stream(rg.key + j, rx.pol_stream) : 0;
      pl[u] = in ? ld_stream2(rg.pay + j, rx.pol_stream) : make_uint2(0u, 0x7fffffffu);
    }
    int32_t m = kInf;
#pragma unroll
    for (int u = 0; u < kUnroll; ++u)
      if (pull_admissible(a, pl[u], q, qp, rx.pol_keep)) m = min(m, -kr[u]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    scanned += lane == 0 ? hi - ch.x : 0u;
    bool first = false, lowered = false, fresh = false;
    if (lane == 0 && m != kInf && m < ld_state(a.X + slot, rx.pol_keep)) {
      const int32_t old = atomicMin(a.X + slot, m);
      if (m < old) {
        lowered = true;
        fresh = old == kInf;
        first = fresh || bound_of(old, a.strict) == __ldcg(&a.EP[slot].x);
      }
    }
    if (rx.log) log_lowered(a, lowered, slot);
    const uint32_t bal = __ballot_sync(0xffffffffu, first);
    if (bal) {
      if (lane == 0) pb.buf[pb.n] = slot | (fresh ? a.fresh : 0u);
      pb.n += 1;
      if (pb.n >= kPushFlush) push_flush_n(pb, a.ctl, rx.pstart, rx.fout);
    }
  }
  push_drain(pb, a.ctl, rx.pstart, rx.fout);
}

#ifndef TGXD_BAR_MAX_NS
#define TGXD_BAR_MAX_NS 256
#endif
#ifndef TGXD_BAR_LOCAL_NS
#define TGXD_BAR_LOCAL_NS 2048
#endif
// Grid barrier for the persistent round kernel. One arrival atomic per
// block; waiters poll the generation word with exponential __nanosleep
// backoff, so ~600 blocks idling through a CTA-local round (or a slow phase)
// do not keep one L2 slice saturated with polls — which stretches every
// other memory access the working warps make (measured: ~1 us per
// dependent load instead of ~0.4 us). Release/acquire as in cg's grid sync.
struct GridBarrier {
  unsigned int* count;
  unsigned int* gen;
  unsigned int nblocks;
  unsigned int phase;  // generations passed (identical in every block)
  // max_ns: backoff cap of the waiters (longer while one CTA works alone)
  __device__ __forceinline__ void sync(unsigned int max_ns = TGXD_BAR_MAX_NS) {
    __syncthreads();
    if (threadIdx.x == 0) {
      const unsigned int g = phase;
      __threadfence();
      if (atomicAdd(count, 1u) + 1 == nblocks) {
        *count = 0;
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(gen), "r"(g + 1) : "memory");
      } else {
        unsigned int ns = 32;
        for (;;) {
          unsigned int cur;
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(gen) : "memory");
          if (cur != g) break;
          __nanosleep(ns);
          if (ns < max_ns) ns <<= 1;
        }
      }
      __threadfence();
    }
    ++phase;
    __syncthreads();
  }
};

// Traversal state; identical in every block at every grid barrier.
//
// Counter discipline. The shared counters (pushes, improved, chunks,
// smalls, edges) are only read immediately after a barrier, into the
// "known" fields below, and every phase that moves a counter is separated
// from those reads by at least one more barrier. So every block derives the
// same round boundaries and the same control flow.
struct TState {
  unsigned long long prev_p;   // queue position where fin's items start
  unsigned long long prev_i;   // improvement counter at the start of the last relax
  unsigned long long p_known;  // pushes counter as of the last barrier
  unsigned long long i_known;  // improved counter as of the last barrier
  unsigned long long c_cur, s_cur, e_cur;  // emission counters as of the last barrier
  unsigned long long pc_cur;   // pull chunks counter as of the last barrier
  uint32_t rounds;
  uint32_t flip;               // fin/fout parity
  int dense;                   // the next expand scans densely
  int pending;                 // CTA expand done, grid relax of its work pending
  uint32_t last_f;             // previous round's frontier size
  int logging;                 // early host copy running: list lowered slots
};

__device__ __forceinline__ void save_state(Control* ctl, const TState& s) {
  static_assert(sizeof(TState) <= sizeof(ctl->state), "state slot too small");
  const unsigned long long* src = reinterpret_cast<const unsigned long long*>(&s);
  unsigned long long* dst = ctl->state;
#pragma unroll
  for (int i = 0; i < (int)(sizeof(TState) / 8); ++i) dst[i] = src[i];
}
// Post-barrier reads of shared counters go through one thread per block and
// shared memory: the same address read by every warp of the grid would
// queue ~5k requests at one L2 slice (~10 us per read).
__device__ __forceinline__ void load_state(const Control* ctl, TState& s) {
  __shared__ unsigned long long s_st[sizeof(TState) / 8];
  if (threadIdx.x < sizeof(TState) / 8) s_st[threadIdx.x] = __ldcg(ctl->state + threadIdx.x);
  __syncthreads();
  unsigned long long* dst = reinterpret_cast<unsigned long long*>(&s);
#pragma unroll
  for (int i = 0; i < (int)(sizeof(TState) / 8); ++i) dst[i] = s_st[i];
  __syncthreads();
}

struct Counters {
  unsigned long long pushes, improved, chunks, smalls, edges, pchunks;
};
__device__ __forceinline__ Counters read_counters(const Control* ctl) {
  __shared__ Counters s_c;
  if (threadIdx.x == 0) {
#ifdef TGXD_SCALAR_COUNTERS
    s_c.pushes = __ldcg(&ctl->pushes);
    s_c.improved = __ldcg(&ctl->improved);
    s_c.chunks = __ldcg(&ctl->chunks);
    s_c.smalls = __ldcg(&ctl->smalls);
    s_c.edges = __ldcg(&ctl->edges);
    s_c.pchunks = __ldcg(&ctl->pchunks);
#else
    static_assert(offsetof(Control, pushes) == 0 && offsetof(Control, pchunks) == 40,
                  "the six post-barrier counters lead the control block");
    const ulonglong2* p = reinterpret_cast<const ulonglong2*>(ctl);
    const ulonglong2 c0 = __ldcg(p), c1 = __ldcg(p + 1), c2 = __ldcg(p + 2);
    s_c.pushes = c0.x;
    s_c.improved = c0.y;
    s_c.chunks = c1.x;
    s_c.smalls = c1.y;
    s_c.edges = c2.x;
    s_c.pchunks = c2.y;
#endif
  }
  __syncthreads();
  const Counters c = s_c;
  __syncthreads();
  return c;
}

__device__ __forceinline__ void trace_round(const TravArgs& a, uint32_t r, int slot,
                                            unsigned long long v) {
  if (a.trace && r < a.trace_cap) {
    volatile unsigned long long* t = a.trace;  // mapped host memory, no fence
    t[r * 8 + slot] = v;
  }
}

// Per-warp phase completion: wtrace[r*4 + 2*phase] = latest, [+1] = earliest
// (stored as kTBig - t so both are maxima).
constexpr unsigned long long kTBig = 1ull << 62;
#ifdef TGXD_WTRACE_ALL
// diagnostics build: every warp's completion time of rounds < 16 (api.cu
// dumps it to TGXD_WTRACE_ALL_FILE; tools/warp_spread.py)
__device__ unsigned long long g_wdone[16][2][148 * TGXD_MIN_BLOCKS * kWarps];
#endif
__device__ __forceinline__ void trace_warp_done(const TravArgs& a, uint32_t r, int phase) {
  if (a.wtrace && a.wtrace_on && r < a.trace_cap && lane_id() == 0) {
    const unsigned long long t = gtimer();
    atomicMax(a.wtrace + r * 4 + 2 * phase, t);
    atomicMax(a.wtrace + r * 4 + 2 * phase + 1, kTBig - t);
#ifdef TGXD_WTRACE_ALL
    if (r < 16) g_wdone[r][phase][blockIdx.x * kWarps + (threadIdx.x >> 5)] = t;
#endif
  }
}

// Reads one counter into every thread of the block (block 0 local rounds).
__device__ __forceinline__ unsigned long long block_read(const unsigned long long* p) {
  __shared__ unsigned long long s_v;
  __syncthreads();
  if (threadIdx.x == 0) s_v = __ldcg(p);
  __syncthreads();
  return s_v;
}

// Rounds with a tiny frontier on one CTA (block 0; it is the only block
// moving counters meanwhile). Returns with st updated and, if an expand
// produced more edge work than one CTA should relax, st.pending set with the
// relax left to the grid.
__device__ TGXD_PHASE void local_rounds(const TravArgs& a, TState& st, uint32_t xlo, uint32_t xcnt,
                             int32_t depart, int32_t vhi0, uint64_t pol_stream,
                             uint64_t pol_keep, uint32_t* wbuf, uint2* ebuf,
                             unsigned long long& ix) {
  Control* ctl = a.ctl;
  bool seed = xcnt != 0;
  const bool tr = threadIdx.x == 0;
  for (;;) {
    if (st.rounds > a.round_limit) return;
    const unsigned long long p_now = st.p_known;
    uint32_t* fin = st.flip ? a.fb : a.fa;
    uint32_t* fout = st.flip ? a.fa : a.fb;
    RelaxCtx rx{vhi0, depart, true, p_now, fout, pol_stream, pol_keep, 0, (int32_t)st.rounds + 1};
    rx.log = st.logging;
    rx.pf = TGXD_PF_GRID != 0;
    if (seed) {
      if (tr) {
        trace_round(a, st.rounds, 0, gtimer());
        trace_round(a, st.rounds, 1, gtimer());
        trace_round(a, st.rounds, 7, 1);
      }
      phase_b(a, 0, 0, xlo, xcnt, rx, 0, 1, wbuf);
      seed = false;
    } else {
      const uint32_t F = (uint32_t)(p_now - st.prev_p);
      if (F == 0 || F > kLocalMaxF) return;
      if (tr) {
        trace_round(a, st.rounds, 0, gtimer());
        trace_round(a, st.rounds, 3, F);
        trace_round(a, st.rounds, 7, 1);
      }
      phase_a(a, fin, F, st.c_cur, st.s_cur, 0, 1, pol_keep, ebuf, ix, depart);
      const unsigned long long c_end = block_read(&ctl->chunks);
      const unsigned long long s_end = block_read(&ctl->smalls);
      const unsigned long long e_end = block_read(&ctl->edges);
      if (tr) {
        trace_round(a, st.rounds, 1, gtimer());
        trace_round(a, st.rounds, 4, c_end - st.c_cur);
        trace_round(a, st.rounds, 5, s_end - st.s_cur);
      }
      if (e_end - st.e_cur > kLocalMaxW) {  // hand the relax to the grid
        st.pending = 1;
        return;
      }
      phase_b(a, c_end - st.c_cur, s_end - st.s_cur, 0, 0, rx, 0, 1, wbuf);
      st.c_cur = c_end;
      st.s_cur = s_end;
      st.e_cur = e_end;
    }
    st.p_known = block_read(&ctl->pushes);
    if (tr) {
      trace_round(a, st.rounds, 2, gtimer());
      trace_round(a, st.rounds, 6, st.p_known - p_now);
    }
    st.prev_p = p_now;
    st.flip ^= 1u;
    st.dense = 0;
    ++st.rounds;
  }
}

// Sub-sweeps a fastest query's n_cand candidates are split over. A split
// sweep costs ~ K full traversals (every sub-sweep starts from scratch) plus
// n_cand / K steps of shared rounds, so K ~ sqrt(c n_cand / n): config 4's
// graph (scale 23) 241K candidates 4.0 s at 64 (5.4 at 32, 4.7 at 128), 24K
// 1.25 s at 20 (1.82 at 64); scale 20, 6.9K candidates 0.19 s at 27, 0.36 at
// 10 — c ~ 1.2e5. One sweep below K = 2 (config 4's own source: 3
// candidates). At most `cap`.
__host__ __device__ __forceinline__ uint32_t split_width(uint32_t n_cand, uint32_t n, uint32_t cap) {
  const unsigned long long t = 120000ull * n_cand;  // K^2 n <= t
  uint32_t k = 1;
  while (k < cap && (unsigned long long)(k + 1) * (k + 1) * n <= t) ++k;
  return k;
}

// One step of a split fastest sweep (split > 1). The closed form
// r[v] = min over candidates d of (A_d[v] - d), A_d the arrivals of the
// paths whose first edge leaves the source at d (a path has exactly one
// first edge, so arrivals from a set of departures are the pointwise minimum
// of the single-departure arrivals), lets the candidates be split into
// `split` subsets, each swept in decreasing order with incremental labels
// exactly as path_algorithms.cpp:460-524 sweeps all of them; the sub-sweeps'
// r are then reduced by a minimum (api.cu split_reduce_kernel). Subset q
// takes candidates q, q + split, q + 2 split, ... of the descending list, so
// every step advances all sub-sweeps by one candidate and their rounds are
// shared: ~n_cand / split steps instead of n_cand.
//
// The step emits each sub-sweep's seed group (its candidate's first edges,
// relaxed without an admissibility check, :476-486) as chunks of query slot
// q, records the candidate's departure in dep[q] and relaxes the chunks with
// the push rule; st is left as after a round that pushed.
__device__ TGXD_PHASE void split_seed_step(const TravArgs& a, TState& st, uint32_t step,
                                           uint32_t n_cand, uint32_t keff, GridBarrier& grid,
                                           int32_t vhi0, uint64_t pol_stream, uint64_t pol_keep,
                                           uint32_t* wbuf) {
  Control* ctl = a.ctl;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nthr = gridDim.x * blockDim.x;
  for (uint32_t q = tid; q < keff; q += nthr) {
    const uint32_t j = step * keff + q;  // position in the descending candidate order
    if (j >= n_cand) continue;
    const uint32_t ci = n_cand - 1 - j;     // the lists are ascending
    a.dep[q] = a.cand_key[ci];
    const uint32_t lo = a.cand_lo[ci], cnt = a.cand_cnt[ci];
    const uint32_t nch = (cnt + kChunk - 1) / kChunk;
    const unsigned long long base = atomicAdd(&ctl->chunks, (unsigned long long)nch) - st.c_cur;
    for (uint32_t k = 0; k < nch; ++k)
      if (TGXD_IN_CAP(base + k, 1))
        a.chunks[base + k] = make_uint2(lo + k * kChunk, (q << kChunkLenBits) | min(kChunk, cnt - k * kChunk));
  }
  grid.sync();
  const Counters c0 = read_counters(ctl);
  const unsigned long long p_now = st.p_known;
  uint32_t* fout = st.flip ? a.fa : a.fb;
  RelaxCtx rx{vhi0, kSplitDepart, true, p_now, fout, pol_stream, pol_keep, 0,
              (int32_t)st.rounds + 1};
  phase_b(a, c0.chunks - st.c_cur, 0, 0, 0, rx, blockIdx.x, gridDim.x, wbuf);
  grid.sync();
  const Counters c1 = read_counters(ctl);
  st.p_known = c1.pushes;
  st.i_known = c1.improved;
  st.c_cur = c0.chunks;
  st.e_cur = c0.edges;
  st.prev_p = p_now;
  st.flip ^= 1u;
  ++st.rounds;
  st.dense = a.mode == TGXD_MODE_AUTO && st.p_known - p_now > a.dense_f;
  if (st.dense) st.prev_i = st.i_known - (st.p_known - p_now);
}

#ifdef TGXD_TMA_RELAX
__shared__ __align__(128) uint2 s_tma_buf[kWarps][2 * kTmaEntries];
__shared__ __align__(8) unsigned long long s_tma_bar[kWarps][2];
__shared__ uint32_t s_tma_par[kWarps];
__device__ TmaBufs tma_bufs_of_warp() {
  const uint32_t w = threadIdx.x >> 5;
  return TmaBufs{s_tma_buf[w], s_tma_bar[w], &s_tma_par[w]};
}
#endif
__global__ void __launch_bounds__(kThreads, TGXD_MIN_BLOCKS) traverse_kernel(TravArgs a) {
  __shared__ uint32_t s_buf[kWarps][kPushFlush + 32];
  __shared__ uint2 s_ebuf[kWarps][2 * kListCap];
  __shared__ uint2 s_rbuf[kWarps][64];
  __shared__ uint4 s_obuf[kWarps][64];
#ifdef TGXD_TMA_RELAX
  if (threadIdx.x < kWarps) {
    const uint32_t b0 = smem_u32(&s_tma_bar[threadIdx.x][0]);
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0) : "memory");
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b0 + 8) : "memory");
    s_tma_par[threadIdx.x] = 0;
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
#endif
  GridBarrier grid{&a.ctl->bar_count, &a.ctl->bar_gen, gridDim.x, 0};
  uint32_t* wbuf = s_buf[threadIdx.x >> 5];
  uint2* ebuf = s_ebuf[threadIdx.x >> 5];
  Control* ctl = a.ctl;
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();
  const int32_t vhi0 = a.qp[0].vhi;
  const bool tr = blockIdx.x == 0 && threadIdx.x == 0;
  unsigned long long ix = 0, work_pull = 0;
  TState st;
  st.prev_p = 0;
  st.prev_i = 0;
  st.p_known = a.init_pushes;
  st.i_known = a.init_pushes;
  st.c_cur = st.s_cur = st.e_cur = st.pc_cur = 0;
  st.rounds = 0;
  st.flip = 0;
  st.dense = a.mode == TGXD_MODE_DENSE;
  st.pending = 0;
  st.last_f = 0;
  st.logging = 0;
  bool handed = false;
  const uint32_t n_cand = a.fastest ? __ldcg(a.n_cand) : 0u;
  // split sweeps take `split` candidates per step, one per query slot
  // (the host sized `split` query slots from the source's degree; the
  // candidates decide how many of them work: slots beyond keff stay idle)
  const uint32_t keff = a.split <= 1 ? 1u
                        : a.split_forced ? min(a.split, max(n_cand, 1u))
                                         : split_width(n_cand, a.n, a.split);
  const uint32_t n_steps = (n_cand + keff - 1) / keff;
  for (uint32_t cand = 0;; ++cand) {
    int32_t depart = 0;
    uint32_t xlo = 0, xcnt = 0;
    if (a.fastest) {
      if (cand >= n_steps) break;
      // the previous candidate's last post-barrier reads end before this
      // candidate's seeds move the counters
      if (cand) grid.sync();
      if (keff > 1) {
        depart = kSplitDepart;  // per slot, dep[q]
        if (tr) trace_round(a, st.rounds, 0, gtimer());
        split_seed_step(a, st, cand, n_cand, keff, grid, vhi0, pol_stream, pol_keep, wbuf);
        if (tr) {
          trace_round(a, st.rounds - 1, 1, gtimer());
          trace_round(a, st.rounds - 1, 2, gtimer());
          trace_round(a, st.rounds - 1, 6, st.p_known - st.prev_p);
          trace_round(a, st.rounds - 1, 7, 5);
        }
        // the rounds below propagate every sub-sweep's delta
      } else {
      // Seed round (path_algorithms.cpp:476-486): the candidate's first
      // edges, relaxed without an admissibility check.
      // (descending: the lists are ascending)
      const uint32_t ci = n_cand - 1 - cand;
      depart = a.cand_key[ci];
      xlo = a.cand_lo[ci];
      xcnt = a.cand_cnt[ci];
      }
    }
    for (;;) {
      if (st.rounds > a.round_limit) {  // identical in every block: all stop together
        if (tr) ctl->error = 1;
        break;
      }
      const unsigned long long F =
          xcnt ? 0 : (st.dense ? st.i_known - st.prev_i : st.p_known - st.prev_p);
      if (!xcnt && F == 0) break;
      // Tail handoff: once the frontier is past its peak and small, the
      // barrier-free engine (async.cuh) finishes the query from this queue
      // and these labels / expansion bounds — the same fixpoint, without a
      // ~10 us latency floor per round.
      // (past its peak, or growing by less than handoff_growth per round: a
      // frontier that stays small for many rounds is latency-bound in rounds)
      // Two engines: the cluster engine (tail.cuh) for a small frontier past
      // its peak; the barrier-free engine on every SM (async.cuh) for a
      // frontier that grows slowly — a long thin traversal (config 1: 27
      // rounds of <= 103K slots) needs the whole GPU, not one cluster.
      if (!xcnt && !st.dense && !a.fastest && st.rounds >= 2) {
        const unsigned long long lf = st.last_f;
        unsigned long long kind = 0;
        if (F <= a.handoff_f && F < lf)
          kind = 1;
        else if (F <= a.async_f && F < lf * a.handoff_growth && (!a.async_grow_only || F >= lf))
          kind = 2;
        if (kind) {
          if (tr) {
            ctl->handoff_n = F;
            ctl->handoff_kind = kind;
            ctl->handoff_flip = st.flip;
          }
          handed = true;
          break;
        }
      }
      // early host copy: a frontier past its peak and small enough starts
      // the labels' copy to the host now (the heavy rounds are over); what
      // the remaining rounds lower is listed for the host's patch
      if (a.copy_flag && !st.logging && !xcnt && st.rounds >= 2 && F <= a.log_f &&
          F < (unsigned long long)st.last_f) {
        st.logging = 1;
        if (a.p24) {  // the copy reads 24-bit labels: pack them first
          pack24(a.X, a.p24, (uint64_t)a.Q * a.n, a.p24_neg,
                 (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, (uint64_t)gridDim.x * blockDim.x);
          grid.sync();
        }
        if (tr) {
          __threadfence_system();
          *a.copy_flag = 1u;
        }
      }
      const unsigned long long f_prev = st.last_f;
      if (!xcnt) st.last_f = (uint32_t)min(F, 0xffffffffull);
      const bool go_local = a.mode != TGXD_MODE_DENSE && !st.dense &&
                            (xcnt ? xcnt <= kLocalMaxW : F <= kLocalMaxF);
      if (go_local) {
        grid.sync();  // post-barrier reads of every block end before block 0 moves counters
        if (blockIdx.x == 0) {
          local_rounds(a, st, xlo, xcnt, depart, vhi0, pol_stream, pol_keep, wbuf, ebuf, ix);
          if (threadIdx.x == 0) save_state(ctl, st);
        }
        xcnt = 0;
        grid.sync(TGXD_BAR_LOCAL_NS);  // the other CTAs idle through block 0's rounds
        load_state(ctl, st);
        if (!st.pending) continue;
        // the grid relaxes what the CTA expanded
        const Counters c0 = read_counters(ctl);
        const unsigned long long c_end = c0.chunks, s_end = c0.smalls, e_end = c0.edges;
        const unsigned long long p_now = st.p_known;
        uint32_t* fout = st.flip ? a.fa : a.fb;
        RelaxCtx rx{vhi0, depart, true, p_now, fout, pol_stream, pol_keep, 0, (int32_t)st.rounds + 1};
        rx.log = st.logging;
        rx.pf = TGXD_PF_GRID != 0 && e_end - st.e_cur <= kPfMaxW;
        phase_b(a, c_end - st.c_cur, s_end - st.s_cur, 0, 0, rx, blockIdx.x, gridDim.x, wbuf);
        trace_warp_done(a, st.rounds, 1);
        grid.sync();
        const Counters c1 = read_counters(ctl);
        st.p_known = c1.pushes;
        st.i_known = c1.improved;
        st.c_cur = c_end;
        st.s_cur = s_end;
        st.e_cur = e_end;
        st.prev_p = p_now;
        st.pending = 0;
        st.flip ^= 1u;
        if (tr) {
          trace_round(a, st.rounds, 2, gtimer());
          trace_round(a, st.rounds, 6, st.p_known - p_now);
        }
        ++st.rounds;
        st.dense = a.mode == TGXD_MODE_AUTO && st.p_known - p_now > a.dense_f;
        if (st.dense) st.prev_i = st.i_known - (st.p_known - p_now);
        continue;
      }
      const unsigned long long p_now = st.p_known, i_now = st.i_known;
      uint32_t* fin = st.flip ? a.fb : a.fa;
      uint32_t* fout = st.flip ? a.fa : a.fb;
      const bool pull = !xcnt && (a.mode == TGXD_MODE_PULL ||
                                  (a.mode == TGXD_MODE_AUTO && F >= a.pull_f &&
                                   F >= f_prev * a.pull_grow));
      if (tr) {
        trace_round(a, st.rounds, 0, gtimer());
        trace_round(a, st.rounds, 3, F);
        trace_round(a, st.rounds, 7, pull ? 3 : (st.dense ? 2 : 0));
      }
      if (pull) {
        RelaxCtx rx{vhi0, depart, true, p_now, fout, pol_stream, pol_keep, 0, (int32_t)st.rounds + 1};
        rx.log = st.logging;
        unsigned long long scanned = 0;
        // P1 queues slots right away: every block's post-barrier read of the
        // pushes counter must be over first (counter discipline)
        grid.sync();
        phase_pull1(a, rx, st.pc_cur, blockIdx.x, gridDim.x, wbuf, ebuf, s_rbuf[threadIdx.x >> 5],
                    s_obuf[threadIdx.x >> 5], scanned);
        trace_warp_done(a, st.rounds, 0);
        grid.sync();
        const unsigned long long pc_end = read_counters(ctl).pchunks;
        if (tr) {
          trace_round(a, st.rounds, 1, gtimer());
          trace_round(a, st.rounds, 4, pc_end - st.pc_cur);
          trace_round(a, st.rounds, 5, 0);
        }
        phase_pull2(a, rx, pc_end - st.pc_cur, blockIdx.x, gridDim.x, wbuf, scanned);
        if (tr) ix += (unsigned long long)a.Q * a.n << 32;  // a pull visits every slot (engine.hpp:341)
        st.pc_cur = pc_end;
        work_pull += scanned;
        trace_warp_done(a, st.rounds, 1);
        grid.sync();
        const Counters c1 = read_counters(ctl);
        st.p_known = c1.pushes;
        st.i_known = c1.improved;
        st.prev_p = p_now;
        st.flip ^= 1u;
        st.dense = 0;
        if (tr) {
          trace_round(a, st.rounds, 2, gtimer());
          trace_round(a, st.rounds, 6, st.p_known - p_now);
        }
        ++st.rounds;
        continue;
      }
      unsigned long long c_end = st.c_cur, s_end = st.s_cur, e_end = st.e_cur;
      if (!xcnt) {
#ifdef TGXD_CHAIN
        if (tr) g_chain_round = st.rounds;
#endif
        phase_a(a, st.dense ? nullptr : fin, (uint32_t)F, st.c_cur, st.s_cur, blockIdx.x,
                gridDim.x, pol_keep, ebuf, ix, depart);
        trace_warp_done(a, st.rounds, 0);
        grid.sync();
        TGXD_MARK(6, 0);
        const Counters c0 = read_counters(ctl);
        TGXD_MARK(7, c0.chunks);
        c_end = c0.chunks;
        s_end = c0.smalls;
        e_end = c0.edges;
      }
      if (tr) {
        trace_round(a, st.rounds, 1, gtimer());
        trace_round(a, st.rounds, 4, c_end - st.c_cur);
        trace_round(a, st.rounds, 5, s_end - st.s_cur);
      }
      const unsigned long long w = (e_end - st.e_cur) + xcnt;
      const bool push = a.mode == TGXD_MODE_SPARSE ||
                        (a.mode == TGXD_MODE_AUTO && w <= a.push_w);
#ifdef TGXD_EXPERIMENTS
      if (st.rounds == a.x_stop_a) {  // experiment: leave this round's relax to relax_only_kernel
        if (tr) {
          ctl->state[0] = c_end - st.c_cur;
          ctl->state[1] = s_end - st.s_cur;
          ctl->state[2] = p_now;
          ctl->state[3] = st.flip;
          ctl->state[4] = push;
          ctl->state[5] = st.c_cur;
          ctl->state[6] = st.s_cur;
        }
        break;
      }
#endif
      RelaxCtx rx{vhi0, depart, push, p_now, fout, pol_stream, pol_keep, 0, (int32_t)st.rounds + 1};
      rx.log = st.logging;
      rx.pf = TGXD_PF_GRID != 0 && push && w <= kPfMaxW;
      phase_b(a, c_end - st.c_cur, s_end - st.s_cur, xlo, xcnt, rx, blockIdx.x, gridDim.x, wbuf);
      if (!push) {  // improvements only feed the dense frontier's size
        uint32_t imp = rx.improved;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) imp += __shfl_xor_sync(0xffffffffu, imp, o);
        if (lane_id() == 0 && imp) atomicAdd(&ctl->improved, (unsigned long long)imp);
      }
      trace_warp_done(a, st.rounds, 1);
      grid.sync();
      TGXD_MARK(12, 0);
      const Counters c1 = read_counters(ctl);
      TGXD_MARK(13, c1.pushes);
      st.p_known = c1.pushes;
      st.i_known = c1.improved;
      st.c_cur = c_end;
      st.s_cur = s_end;
      st.e_cur = e_end;
      st.prev_p = p_now;
      st.prev_i = i_now;
      xcnt = 0;
      const unsigned long long pushed = st.p_known - p_now;
      if (tr) {
        trace_round(a, st.rounds, 2, gtimer());
        trace_round(a, st.rounds, 6, push ? pushed : st.i_known - i_now);
      }
      ++st.rounds;
      if (push) st.flip ^= 1u;
      // the next expand is dense when nothing was queued or the queue is big;
      // a dense expand sizes its frontier by improvements since this relax
      if (a.mode == TGXD_MODE_DENSE || !push) {
        st.dense = 1;
      } else {
        st.dense = a.mode == TGXD_MODE_AUTO && pushed > a.dense_f;
        if (st.dense) st.prev_i = st.i_known - pushed;
      }
    }
    if (!a.fastest || handed || st.rounds > a.round_limit) break;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    ix += __shfl_xor_sync(0xffffffffu, ix, o);
    work_pull += __shfl_xor_sync(0xffffffffu, work_pull, o);
  }
  if (lane_id() == 0 && (ix & 0xffffffffull)) atomicAdd(&ctl->index_lookups, ix & 0xffffffffull);
  if (lane_id() == 0 && (ix >> 32)) atomicAdd(&ctl->expansions, ix >> 32);
  if (lane_id() == 0 && work_pull) atomicAdd(&ctl->pull_scanned, work_pull);
  if (tr) {
    ctl->t_end = gtimer();
    ctl->rounds = st.rounds;
    ctl->candidates = n_cand;
  }
}

#ifdef TGXD_EXPERIMENTS
#ifndef TGXD_X_BLOCKS
#define TGXD_X_BLOCKS 8
#endif
// Experiment: one round's relax as a non-persistent kernel (own register
// budget and occupancy, the hardware block scheduler balancing the units):
// units of `upw` per warp, chunks then windows, push rule as phase_b.
__global__ void __launch_bounds__(kThreads, TGXD_X_BLOCKS)
    relax_only_kernel(TravArgs a, unsigned long long nchunks, unsigned long long nsmall,
                      unsigned long long pstart, uint32_t* fout, int push, uint32_t upw) {
  __shared__ uint32_t s_buf[kWarps][kPushFlush + 32];
  const uint32_t lane = lane_id();
  const unsigned long long gw = (unsigned long long)blockIdx.x * kWarps + (threadIdx.x >> 5);
  PushBuf pb{s_buf[threadIdx.x >> 5], 0};
  RelaxCtx rx{a.qp[0].vhi, 0, push != 0, pstart, fout, policy_evict_first(), policy_evict_last(),
              0, 1};
  const unsigned long long nwin = (nsmall + 31) / 32;
  for (unsigned long long u = gw * upw; u < (gw + 1) * upw && u < nchunks + nwin; ++u) {
    if (u < nchunks) {
      const uint2 ch = __ldcg(a.chunks + u);
      const uint32_t len = ch.y & ((1u << kChunkLenBits) - 1);
      uint32_t e[kUnroll], q[kUnroll];
      bool act[kUnroll];
#pragma unroll
      for (int k = 0; k < kUnroll; ++k) {
        const uint32_t off = k * 32 + lane;
        act[k] = off < len;
        e[k] = ch.x + off;
        q[k] = ch.y >> kChunkLenBits;
      }
      relax_steps(a, e, q, act, rx, pb);
    } else {
      const unsigned long long i = (u - nchunks) * 32 + lane;
      relax_window(a, i < nsmall ? __ldcg(a.smalls + i) : make_uint2(0u, 0u), rx, pb);
    }
  }
  if (rx.push) block_push_drain(pb, a.ctl, rx.pstart, rx.fout);
}
#endif

// 24-bit packing when the copy starts after the round kernel (api.cu; it
// runs beside the tail engine).
__global__ void pack24_kernel(const int32_t* X, uint32_t* P, uint64_t slots, int neg) {
  pack24(X, P, slots, neg, (uint64_t)blockIdx.x * blockDim.x + threadIdx.x,
         (uint64_t)gridDim.x * blockDim.x);
}

// Labels, expansion bounds and durations to INF.
__global__ void init_kernel(int32_t* X, int2* EP, int32_t* R, size_t nl) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t n4 = nl / 4;
  const int4 inf4 = make_int4(kInf, kInf, kInf, kInf);
  const int4 ep2 = make_int4(kInf, (int32_t)kNoPos, kInf, (int32_t)kNoPos);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    reinterpret_cast<int4*>(X)[i] = inf4;
    reinterpret_cast<int4*>(EP)[2 * i] = ep2;
    reinterpret_cast<int4*>(EP)[2 * i + 1] = ep2;
    if (R) reinterpret_cast<int4*>(R)[i] = inf4;
  }
  for (size_t i = n4 * 4 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += stride) {
    X[i] = kInf;
    EP[i] = make_int2(kInf, (int32_t)kNoPos);
    if (R) R[i] = kInf;
  }
}

// Lazy reset (api.cu launch): slots the previous query reached (finite
// label) back to INF / the initial expansion state; untouched slots are only
// read.
__global__ void reset_kernel(int32_t* X, int2* EP, size_t nl) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t n4 = nl / 4;
  const int2 ep0 = make_int2(kInf, (int32_t)kNoPos);
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n4; i += stride) {
    const int4 x = reinterpret_cast<const int4*>(X)[i];
    if (x.x != kInf || x.y != kInf || x.z != kInf || x.w != kInf) {
      // whole 16-byte groups (slots already initial are rewritten unchanged)
      reinterpret_cast<int4*>(X)[i] = make_int4(kInf, kInf, kInf, kInf);
      const int4 e2 = make_int4(kInf, (int32_t)kNoPos, kInf, (int32_t)kNoPos);
      reinterpret_cast<int4*>(EP)[2 * i] = e2;
      reinterpret_cast<int4*>(EP)[2 * i + 1] = e2;
    }
  }
  for (size_t i = n4 * 4 + (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < nl; i += stride) {
    if (X[i] != kInf) {
      X[i] = kInf;
      EP[i] = ep0;
    }
  }
}

// One query (Q == 1) on the lazy path: reset_kernel and seed_kernel in one
// launch. The thread that resets the root's slot group writes the seed after
// it (a root beyond the dirty range is written by thread 0: that slot is
// clean); thread 0 also resets the counters and queues the root.
__global__ void reset_seed_kernel(int32_t* X, int2* EP, size_t nl, uint32_t root, int32_t klo,
                                  uint32_t* fa, Control* ctl) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  const size_t tid = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t n4 = nl / 4;
  for (size_t i = tid; i < n4; i += stride) {
    const int4 x = reinterpret_cast<const int4*>(X)[i];
    if (x.x != kInf || x.y != kInf || x.z != kInf || x.w != kInf) {
      reinterpret_cast<int4*>(X)[i] = make_int4(kInf, kInf, kInf, kInf);
      const int4 e2 = make_int4(kInf, (int32_t)kNoPos, kInf, (int32_t)kNoPos);
      reinterpret_cast<int4*>(EP)[2 * i] = e2;
      reinterpret_cast<int4*>(EP)[2 * i + 1] = e2;
    }
    if (root / 4 == i) X[root] = klo;
  }
  for (size_t i = n4 * 4 + tid; i < nl; i += stride) {
    if (X[i] != kInf) {
      X[i] = kInf;
      EP[i] = make_int2(kInf, (int32_t)kNoPos);
    }
    if (i == root) X[root] = klo;
  }
  if (tid == 0) {
    if (root >= nl) X[root] = klo;
    fa[0] = root;
    ctl->pushes = 1;
    ctl->improved = 1;
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
}

// Seeds: X[root] = klo (EA: t_a, LD: -t_b), root queued as round-0 frontier.
__global__ void seed_kernel(const QueryParam* qp, uint32_t Q, uint32_t n, int32_t* X,
                            uint32_t* fa, Control* ctl, int fastest) {
  const uint32_t q = blockIdx.x * blockDim.x + threadIdx.x;
  if (q == 0) {
    ctl->pushes = fastest ? 0ull : Q;
    ctl->improved = fastest ? 0ull : Q;
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
  if (q >= Q || fastest) return;
  const uint32_t item = q * n + qp[q].root;
  X[item] = qp[q].klo;
  fa[q] = item;
}

}  // namespace tgxd
