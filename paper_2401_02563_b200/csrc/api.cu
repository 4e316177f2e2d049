// C-ABI of the B200 temporal traversal engine (include/tgxd.h).
//
// Host orchestration only: argument validation with the reference's error
// semantics, workspace management, kernel launches on the handle's stream,
// output widening. All per-edge work is in build.cuh / traverse.cuh.
#include <cuda_runtime.h>
#include <immintrin.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "build.cuh"
#include "gen.cuh"
#include "tgxd_internal.cuh"
#include "traverse.cuh"
#include "async.cuh"
#include "edges.cuh"
#include "sd.cuh"
#include "lanes.cuh"
#include "candidates.cuh"
#include "tail.cuh"
#include "costmodel.cuh"

namespace tgxd {

namespace {

thread_local std::string g_err;

int fail(int code, const std::string& msg) {
  g_err = msg;
  return code;
}

#define TGXD_CUDA(expr)                                                          \
  do {                                                                           \
    cudaError_t _e = (expr);                                                     \
    if (_e != cudaSuccess)                                                       \
      return fail(TGXD_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e)); \
  } while (0)

constexpr uint64_t kTimeLimit63 = 0x7fffffffffffffffULL;

struct Seed {
  uint32_t root;
  uint32_t pad;
  long long value;
};

// Geometric table thr[k] = floor(2^64 (1 - p)^k), k >= 1, until it reaches 0.
int geo_table(double p, std::vector<uint64_t>& thr) {
  if (!(p > 0.0 && p <= 1.0)) return fail(TGXD_ERR_ARGUMENT, "geo_p must lie in (0, 1]");
  thr.assign(1, ~0ULL);
  const long double q = 1.0L - (long double)p;
  long double cur = 18446744073709551616.0L;  // 2^64
  for (int k = 1; k < kGeoTableMax; ++k) {
    cur *= q;
    const long double f = floorl(cur);
    const uint64_t t = f >= 18446744073709551615.0L ? ~0ULL : (uint64_t)f;
    thr.push_back(t);
    if (t == 0) return TGXD_OK;
  }
  return fail(TGXD_ERR_ARGUMENT, "geo_p too small for the duration table");
}

uint64_t prob_threshold(long double x) {
  if (x <= 0) return 0;
  if (x >= 1) return ~0ULL;
  return (uint64_t)floorl(x * 18446744073709551616.0L);
}

int gen_params(const tgxd_gen_config* c, GenParams& p, std::vector<uint64_t>& thr) {
  if (!c) return fail(TGXD_ERR_ARGUMENT, "null generator config");
  std::memset(&p, 0, sizeof p);
  p.kind = c->kind;
  p.seed = c->seed;
  p.start_dist = c->start_dist;
  p.t_range = c->t_range;
  p.m_draws = c->m;
  if (c->t_range == 0 || c->t_range > 1u << 30)
    return fail(TGXD_ERR_ARGUMENT, "t_range must lie in [1, 2^30]");
  if (c->kind == TGXD_GEN_RMAT) {
    if (c->scale > 31) return fail(TGXD_ERR_ARGUMENT, "RMAT scale must be <= 31");
    p.scale = c->scale;
    p.n_vertices = c->scale == 32 ? 0 : (1u << c->scale);
    if (c->a < 0 || c->b < 0 || c->c < 0 || c->a + c->b + c->c > 1.0)
      return fail(TGXD_ERR_ARGUMENT, "RMAT probabilities must be non-negative and sum <= 1");
    p.thr_a = prob_threshold((long double)c->a);
    p.thr_ab = prob_threshold((long double)c->a + (long double)c->b);
    p.thr_abc = prob_threshold((long double)c->a + (long double)c->b + (long double)c->c);
    for (int r = 0; r < 3; ++r) {
      p.perm_mul[r] = mix64(c->seed ^ (0x5851f42d4c957f2dULL * (r + 1))) | 1ULL;
      p.perm_add[r] = mix64(c->seed + 0x14057b7ef767814fULL * (r + 7));
    }
  } else if (c->kind == TGXD_GEN_UNIFORM) {
    if (c->n == 0) return fail(TGXD_ERR_ARGUMENT, "uniform generator needs n >= 1");
    p.n_vertices = c->n;
  } else {
    return fail(TGXD_ERR_ARGUMENT, "unknown generator kind");
  }
  int rc = geo_table(c->geo_p, thr);
  if (rc) return rc;
  p.geo_len = (int)thr.size();
  return TGXD_OK;
}

template <class T>
T* dalloc(DeviceBuffer& b, size_t count) {
  if (b.ensure(count * sizeof(T) + 16) != cudaSuccess) return nullptr;
  return b.as<T>();
}

}  // namespace

DeviceBuffer::~DeviceBuffer() { release(); }

void DeviceBuffer::release() {
  if (p) cudaFree(p);
  p = nullptr;
  bytes = 0;
}

cudaError_t DeviceBuffer::ensure(size_t nbytes) {
  if (nbytes <= bytes && p) return cudaSuccess;
  release();
  cudaError_t e = cudaMalloc(&p, nbytes);
  if (e != cudaSuccess) {
    p = nullptr;
    return e;
  }
  bytes = nbytes;
  return cudaSuccess;
}

// Builds both layouts from device edge arrays (m edges, already validated and
// materialized). Frees nothing it does not own.
__global__ void gather_weights(const uint32_t* idx, const long long* w, uint64_t m,
                               long long* out) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += stride)
    out[j] = w[idx[j]];
}

// (d_w / out_w: optional per-edge weight codes, gathered into Out order)
static int build_layouts(tgxd_graph* G, const uint32_t* d_src, const uint32_t* d_dst,
                         const int32_t* d_st, const int32_t* d_en, uint64_t m,
                         const long long* d_w = nullptr, long long* out_w = nullptr) {
  cudaStream_t s = G->stream;
  const uint32_t n = G->n;
  G->m = m;
  DeviceBuffer keys_a, keys_b, idx_a, idx_b, temp, cnt, counter;
  unsigned long long* ka = dalloc<unsigned long long>(keys_a, m);
  unsigned long long* kb = dalloc<unsigned long long>(keys_b, m);
  uint32_t* ia = dalloc<uint32_t>(idx_a, m);
  uint32_t* ib = dalloc<uint32_t>(idx_b, m);
  uint32_t* dc = dalloc<uint32_t>(cnt, (size_t)n + 1);
  unsigned long long* dctr = dalloc<unsigned long long>(counter, 2);
  if (!ka || !kb || !ia || !ib || !dc || !dctr)
    return fail(TGXD_ERR_CUDA, "device allocation failed while building the graph");
  int end_bit = 32;
  while (end_bit < 64 && (1ULL << (end_bit - 32)) < (uint64_t)n) ++end_bit;
  if (end_bit == 32) end_bit = 33;
  // without weights the sort moves the payloads (keys + 8-byte values; no
  // random gathers after it: config 2's two gathers took 4.5 ms each); with
  // weights it moves edge indices, which also order the weights
  const bool kv = d_w == nullptr && !getenv("TGXD_BUILD_GATHER");
  DeviceBuffer vals_a;
  unsigned long long* va = kv ? dalloc<unsigned long long>(vals_a, std::max<uint64_t>(m, 1)) : nullptr;
  if (kv && !va) return fail(TGXD_ERR_CUDA, "device allocation failed while building the graph");
  size_t temp_bytes = 0, scan_bytes = 0;
  if (kv) {
    TGXD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, ka, kb, va, va, (int64_t)m, 0,
                                              end_bit, s));
  } else {
    TGXD_CUDA(cub::DeviceRadixSort::SortPairs(nullptr, temp_bytes, ka, kb, ia, ib, (int64_t)m, 0,
                                              end_bit, s));
  }
  TGXD_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, dc, dc, (int64_t)n + 1, s));
  if (temp.ensure(std::max(temp_bytes, scan_bytes) + 16) != cudaSuccess)
    return fail(TGXD_ERR_CUDA, "device allocation failed (sort scratch)");
  TGXD_CUDA(cudaMemsetAsync(dctr, 0, 16, s));
  const int gb = grid_for(m, G->sm_count);
  const uint64_t nf = (m + kFenceStride - 1) >> kFenceShift;
  for (int dir = 0; dir < 2; ++dir) {
    const uint32_t* owner = dir == 0 ? d_src : d_dst;
    const uint32_t* other = dir == 0 ? d_dst : d_src;
    const int32_t* kk = dir == 0 ? d_st : d_en;
    const int32_t* vv = dir == 0 ? d_en : d_st;
    DeviceBuffer& b_off = dir == 0 ? G->out_off : G->in_off;
    DeviceBuffer& b_key = dir == 0 ? G->out_key : G->in_key;
    DeviceBuffer& b_pay = dir == 0 ? G->out_pay : G->in_pay;
    DeviceBuffer& b_fence = dir == 0 ? G->out_fence : G->in_fence;
    DeviceBuffer& b_kmax = dir == 0 ? G->out_kmax : G->in_kmax;
    int32_t* kmax = dalloc<int32_t>(b_kmax, (size_t)n + 1);
    uint2* okm = dalloc<uint2>(dir == 0 ? G->out_okm : G->in_okm, (size_t)n + 1);
    uint32_t* off = dalloc<uint32_t>(b_off, (size_t)n + 1);
    int32_t* key = dalloc<int32_t>(b_key, m);
    uint2* pay = dalloc<uint2>(b_pay, m);
    int32_t* fence = dalloc<int32_t>(b_fence, nf);
    if (!off || !key || !pay || !fence || !kmax || !okm)
      return fail(TGXD_ERR_CUDA, "device allocation failed (T-CSR arrays)");
    if (m) {
      if (kv) {
        make_sort_kv<<<gb, 256, 0, s>>>(owner, other, kk, vv, dir, m, ka, va);
        TGXD_CUDA(cub::DeviceRadixSort::SortPairs(temp.p, temp_bytes, ka, kb, va,
                                                  reinterpret_cast<unsigned long long*>(pay),
                                                  (int64_t)m, 0, end_bit, s));
        keys_from_sorted<<<gb, 256, 0, s>>>(kb, m, key);
      } else {
        make_sort_keys<<<gb, 256, 0, s>>>(owner, kk, dir, m, ka, ia);
        TGXD_CUDA(cub::DeviceRadixSort::SortPairs(temp.p, temp_bytes, ka, kb, ia, ib, (int64_t)m,
                                                  0, end_bit, s));
        gather_layout<<<gb, 256, 0, s>>>(ib, other, kk, vv, dir, m, key, pay);
      }
      if (dir == 0 && d_w && out_w) gather_weights<<<gb, 256, 0, s>>>(ib, d_w, m, out_w);
      make_fences<<<grid_for(nf, G->sm_count), 256, 0, s>>>(key, m, fence);
    }
    TGXD_CUDA(cudaMemsetAsync(dc, 0, ((size_t)n + 1) * 4, s));
    if (m) degree_count<<<gb, 256, 0, s>>>(owner, m, dc);
    size_t sb = scan_bytes;
    TGXD_CUDA(cub::DeviceScan::ExclusiveSum(temp.p, sb, dc, off, (int64_t)n + 1, s));
    if (n) count_indexed<<<grid_for(n, G->sm_count), 256, 0, s>>>(off, n, G->index_cutoff, dctr + dir);
    if (n) segment_kmax<<<grid_for(n, G->sm_count), 256, 0, s>>>(off, key, n, kmax);
    make_okm<<<grid_for((size_t)n + 1, G->sm_count), 256, 0, s>>>(off, kmax, n, okm);
    DevCsr& c = dir == 0 ? G->out : G->in;
    c.off = off;
    c.key = key;
    c.pay = pay;
    c.fence = fence;
    c.kmax = kmax;
    c.okm = okm;
    c.n = n;
    c.m = (uint32_t)m;
  }
  unsigned long long h[2];
  TGXD_CUDA(cudaMemcpyAsync(h, dctr, 16, cudaMemcpyDeviceToHost, s));
  TGXD_CUDA(cudaStreamSynchronize(s));
  TGXD_CUDA(cudaGetLastError());
  G->indexed[0] = h[0];
  G->indexed[1] = h[1];
  return TGXD_OK;
}

// The cluster tail engine's size: 16 CTAs (non-portable) when the device can
// co-schedule them, else the portable 8, else 0 (the async engine finishes
// tails). TGXD_TAIL=async forces the async engine; TGXD_TAIL_CLUSTER=8/16.
static int tail_cluster_size() {
  static const int size = [] {
    const char* e = getenv("TGXD_TAIL");
    if (e && std::string(e) == "async") return 0;
    int want = 16;
    if (const char* c = getenv("TGXD_TAIL_CLUSTER")) want = atoi(c);
    cudaFuncSetAttribute(tail_kernel, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    for (int c : {16, 8}) {
      if (c > want) continue;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(c);
      cfg.blockDim = dim3(kTailThreads);
      cudaLaunchAttribute at;
      at.id = cudaLaunchAttributeClusterDimension;
      at.val.clusterDim.x = c;
      at.val.clusterDim.y = 1;
      at.val.clusterDim.z = 1;
      cfg.attrs = &at;
      cfg.numAttrs = 1;
      int clusters = 0;
      if (cudaOccupancyMaxActiveClusters(&clusters, tail_kernel, &cfg) == cudaSuccess &&
          clusters > 0)
        return c;
      cudaGetLastError();
    }
    return 0;
  }();
  return size;
}

static int new_graph(uint32_t n, uint64_t index_cutoff, int directed, tgxd_graph** out) {
  int dev = 0, count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return fail(TGXD_ERR_CUDA, "no CUDA device available (the engine has no CPU fallback)");
  TGXD_CUDA(cudaGetDevice(&dev));
  auto* G = new tgxd_graph();
  G->device = dev;
  G->n = n;
  G->directed = directed ? 1 : 0;
  G->index_cutoff = index_cutoff ? index_cutoff : 2048;
  cudaError_t e = cudaStreamCreateWithFlags(&G->stream, cudaStreamNonBlocking);
  if (e == cudaSuccess) e = cudaDeviceGetAttribute(&G->sm_count, cudaDevAttrMultiProcessorCount, dev);
  int per_sm = 0;
  if (e == cudaSuccess)
    e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, traverse_kernel, kThreads, 0);
  for (int i = 0; e == cudaSuccess && i < 4; ++i) e = cudaEventCreate(&G->ws.ev[i]);
  if (e != cudaSuccess) {
    delete G;
    return fail(TGXD_ERR_CUDA, std::string("graph setup: ") + cudaGetErrorString(e));
  }
  if (const char* b = getenv("TGXD_BLOCKS_PER_SM"))  // experiments: fewer resident CTAs
    per_sm = std::min(per_sm, std::max(1, atoi(b)));
  G->coop_blocks = std::max(1, per_sm) * G->sm_count;
  // the tail runs on fewer CTAs: its frontier is small, and every idle warp
  // polls a queue ticket (measured on config 2: 3 CTAs per SM 0.91 ms, all 4
  // 1.02 ms, 1 1.01 ms; TGXD_TAIL_BLOCKS_PER_SM overrides)
  {
    const char* t = getenv("TGXD_TAIL_BLOCKS_PER_SM");
    G->tail_per_sm = t ? std::max(1, atoi(t)) : 3;
  }
  int per_sm_a = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_a, async_kernel, kThreads, 0);
  G->coop_blocks_async = std::max(1, per_sm_a) * G->sm_count;
  int per_sm_e = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_e, edge_kernel, kThreads, 0);
  G->coop_blocks_edge = std::max(1, per_sm_e) * G->sm_count;
  int per_sm_s = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_s, sd_kernel, kThreads, 0);
  G->coop_blocks_sd = std::max(1, per_sm_s) * G->sm_count;
  int per_sm_l = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_l, lanes_kernel, kThreads, 0);
  G->coop_blocks_lanes = std::max(1, per_sm_l) * G->sm_count;
  G->tail_cluster = tail_cluster_size();
  *out = G;
  return TGXD_OK;
}

// ---------------------------------------------------------------------------
// Queries

struct Prepared {
  int kind;
  int strict;
  int ordering;
  bool edge;  // edge-state engine (edges.cuh): Overlaps, or shortest duration
  bool weighted = false;  // shortest duration summing edge weights
  uint32_t Q;
  std::vector<QueryParam> qp;
  std::vector<Seed> seeds;
};

// Validation in the reference's order: require_vertex (out_of_range), then
// checked_window (invalid_argument), then the ordering.
static int prepare(tgxd_graph* G, int kind, uint32_t k, const uint32_t* verts, const uint64_t* ta,
                   const uint64_t* tb, int ordering, Prepared& P) {
  if (kind < 0 || kind > 5) return fail(TGXD_ERR_ARGUMENT, "unknown query kind");
  P.weighted = kind == TGXD_SHORTEST_DURATION_WEIGHTED;
  if (P.weighted) kind = TGXD_SHORTEST_DURATION;
  if (k == 0 || !verts || !ta || !tb) return fail(TGXD_ERR_ARGUMENT, "empty or null query batch");
  if ((uint64_t)k * G->n >= 0xffffffffULL)
    return fail(TGXD_ERR_ARGUMENT, "batch too large: k * n must stay below 2^32");
  if (ordering < 0 || ordering > 2) return fail(TGXD_ERR_ARGUMENT, "unknown ordering");
  P.kind = kind;
  P.Q = k;
  P.strict = ordering == TGXD_STRICTLY_SUCCEEDS ? 1 : 0;
  P.ordering = ordering;
  P.edge = ordering == TGXD_OVERLAPS || kind == TGXD_SHORTEST_DURATION;
  if (P.edge && k != 1) return fail(TGXD_ERR_ARGUMENT, "edge-state queries run one at a time");
  P.qp.resize(k);
  P.seeds.resize(k);
  for (uint32_t q = 0; q < k; ++q) {
    const char* what = kind == TGXD_LATEST_DEPARTURE ? "target " : "source ";
    if (verts[q] >= G->n)
      return fail(TGXD_ERR_VERTEX_RANGE, std::string(what) + std::to_string(verts[q]) +
                                             " outside vertex range [0, " + std::to_string(G->n) +
                                             ")");
    if (ta[q] > tb[q]) return fail(TGXD_ERR_WINDOW, "query window with t_a > t_b");
    if (ta[q] > kTimeLimit63)
      return fail(TGXD_ERR_WINDOW, "window start beyond the supported time range (2^63 - 1)");
  }
  for (uint32_t q = 0; q < k; ++q) {
    const uint64_t tb63 = std::min<uint64_t>(tb[q], kTimeLimit63);
    const int64_t ta_c = (int64_t)std::min<uint64_t>(ta[q], (uint64_t)kTimeMax + 1);
    const int64_t tb_c = (int64_t)std::min<uint64_t>(tb63, (uint64_t)kTimeMax);
    QueryParam& p = P.qp[q];
    p.depart = 0;
    Seed& sd = P.seeds[q];
    sd.root = verts[q];
    sd.pad = 0;
    if (kind == TGXD_LATEST_DEPARTURE) {
      p.root = verts[q];
      p.klo = (int32_t)(-tb_c);
      p.vhi = (int32_t)(-ta_c);
      sd.value = (long long)tb63;
    } else {
      // fastest sweeps have no source exemption (path_algorithms.cpp:497-500);
      // the edge engine seeds from the root's window edges
      p.root = kind == TGXD_FASTEST && !P.edge ? kNoRoot : verts[q];
      p.klo = (int32_t)ta_c;  // == kInf when t_a lies beyond every edge time
      p.vhi = (int32_t)tb_c;
      // r[source]: t_a (EA), 0 (fastest :526, shortest duration :432, BFS :406)
      sd.value = kind == TGXD_EARLIEST_ARRIVAL ? (long long)ta[q] : 0;
    }
  }
  return TGXD_OK;
}

__global__ void max_degree_kernel(const uint32_t* off, uint32_t n, unsigned int* out) {
  unsigned int m = 0;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x)
    m = max(m, off[v + 1] - off[v]);
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if ((threadIdx.x & 31) == 0 && m) atomicMax(out, m);
}

// Largest out-degree (once per graph): sizes the device candidate lists of
// fastest queries (candidates.cuh) and bounds their watchdog.
static int ensure_max_out_degree(tgxd_graph* G) {
  if (G->max_out_deg_known) return TGXD_OK;
  DeviceBuffer tmp;
  unsigned int* d = dalloc<unsigned int>(tmp, 1);
  if (!d) return fail(TGXD_ERR_CUDA, "allocation (max degree)");
  TGXD_CUDA(cudaMemsetAsync(d, 0, 4, G->stream));
  if (G->n)
    max_degree_kernel<<<grid_for(G->n, G->sm_count), 256, 0, G->stream>>>(G->out.off, G->n, d);
  unsigned int h = 0;
  TGXD_CUDA(cudaMemcpyAsync(&h, d, 4, cudaMemcpyDeviceToHost, G->stream));
  TGXD_CUDA(cudaStreamSynchronize(G->stream));
  G->max_out_deg = h;
  G->max_out_deg_known = true;
  return TGXD_OK;
}

static int ensure_workspace(tgxd_graph* G, uint32_t Q, bool need_r) {
  Workspace& w = G->ws;
  const uint64_t slots = (uint64_t)Q * G->n;
  // chunks per round <= frontier items + edges / kChunk (per query slot)
  const uint64_t max_chunks = slots + (uint64_t)Q * (G->m / kChunk + 1);
  bool ok = dalloc<int32_t>(w.X, slots) && dalloc<int2>(w.EP, slots) &&
            dalloc<uint32_t>(w.fa, slots) &&
            dalloc<uint32_t>(w.fb, slots) && dalloc<uint2>(w.chunks, max_chunks) &&
            dalloc<uint2>(w.smalls, slots) && dalloc<Control>(w.ctl, 1) &&
            dalloc<QueryParam>(w.params, Q) && dalloc<Seed>(w.seeds, Q);
  if (ok && need_r) ok = dalloc<int32_t>(w.R, slots) != nullptr;
  if (!ok) return fail(TGXD_ERR_CUDA, "device allocation failed (traversal workspace)");
  if (slots > w.slots) {  // X / EP / params / seeds may have been reallocated
    w.xinv = false;
    w.up_valid = false;
  }
  w.slots = std::max(w.slots, slots);
  return TGXD_OK;
}

// Device labels -> PathResult values. form 0: int32, INT32_MAX -> INT64_MAX
// (EA, fastest durations, BFS hops); form 1: LD key space (negated,
// INT32_MAX -> INT64_MIN); form 2: int64 as is (shortest duration). The
// root's value is written exactly (Seed).
enum ConvertForm : int { kFormMin = 0, kFormLd = 1, kFormI64 = 2 };

__device__ __forceinline__ long long convert_one(int form, int32_t x) {
  if (form == kFormLd) return x == kInf ? (-0x7fffffffffffffffLL - 1) : -(long long)x;
  return x == kInf ? 0x7fffffffffffffffLL : (long long)x;
}
__device__ __forceinline__ int32_t clamp32(long long o) {
  return (int32_t)(o > 0x7fffffffLL ? 0x7fffffffLL : (o < -0x80000000LL ? -0x80000000LL : o));
}

__global__ void convert_kernel(int form, const int32_t* V, const long long* V64, uint64_t total,
                               uint32_t n, const Seed* seeds, void* out, int width) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  uint64_t done = 0;
  // int32 labels, 4 slots per thread and step with 16-byte accesses (the
  // output must be 16-byte aligned; a step crosses at most one query)
  if (form != kFormI64 && n >= 4 && (reinterpret_cast<uintptr_t>(out) & 15) == 0) {
    const uint64_t n4 = total / 4;
    for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n4; j += stride) {
      const int4 x4 = reinterpret_cast<const int4*>(V)[j];
      const int32_t xs[4] = {x4.x, x4.y, x4.z, x4.w};
      const uint64_t i0 = 4 * j;
      const uint32_t q0 = (uint32_t)(i0 / n);
      const uint32_t v0 = (uint32_t)(i0 - (uint64_t)q0 * n);
      long long o[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        uint32_t q = q0, v = v0 + k;
        if (v >= n) {
          ++q;
          v -= n;
        }
        o[k] = convert_one(form, xs[k]);
        const Seed sd = seeds[q];
        if (v == sd.root) o[k] = sd.value;
      }
      if (width == 8) {
        longlong2* d = reinterpret_cast<longlong2*>(out) + 2 * j;
        d[0] = make_longlong2(o[0], o[1]);
        d[1] = make_longlong2(o[2], o[3]);
      } else {
        reinterpret_cast<int4*>(out)[j] = make_int4(clamp32(o[0]), clamp32(o[1]), clamp32(o[2]),
                                                    clamp32(o[3]));
      }
    }
    done = n4 * 4;
  }
  for (uint64_t i = done + (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total; i += stride) {
    const uint32_t q = (uint32_t)(i / n);
    const uint32_t v = (uint32_t)(i - (uint64_t)q * n);
    long long o = form == kFormI64 ? V64[i] : convert_one(form, V[i]);
    if (v == seeds[q].root) o = seeds[q].value;
    if (width == 8) {
      static_cast<long long*>(out)[i] = o;
    } else {
      static_cast<int32_t*>(out)[i] = clamp32(o);
    }
  }
}

// The form and source array of a query's result.
static void convert_for(tgxd_graph* G, const Prepared& P, void* out_dev, int width) {
  Workspace& w = G->ws;
  const uint64_t slots = (uint64_t)P.Q * G->n;
  int form = kFormMin;
  const int32_t* V = w.X.as<int32_t>();
  const long long* V64 = nullptr;
  if (P.kind == TGXD_LATEST_DEPARTURE) form = kFormLd;
  if (P.kind == TGXD_FASTEST) V = w.R.as<int32_t>();
  if (P.kind == TGXD_TEMPORAL_BFS && !P.edge) V = w.R.as<int32_t>();
  if (P.kind == TGXD_SHORTEST_DURATION) {
    form = kFormI64;
    V64 = w.ey.as<long long>();
  }
  convert_kernel<<<grid_for(slots, G->sm_count), 256, 0, G->stream>>>(
      form, V, V64, slots, G->n, w.seeds.as<Seed>(), out_dev, width);
  ++G->ws.launches;
}

static uint64_t next_pow2(uint64_t x) {
  uint64_t p = 1;
  while (p < x) p <<= 1;
  return p;
}

// The asynchronous engine: rings and flags persist across queries (every
// query leaves them empty and clear); the kernel runs after init_kernel.
// Label words and the unit ring of the async engine (allocated on first use).
static int ensure_async(tgxd_graph* G, uint32_t Q, bool required = true) {
  Workspace& w = G->ws;
  cudaStream_t s = G->stream;
  const uint64_t slots = (uint64_t)Q * G->n;
  // outstanding units <= batches (<= one per queued slot) + chunks (ranges of
  // >= kAInline edges and their 512-edge pieces) + staging slack
  const uint64_t nunits =
      next_pow2(slots + (uint64_t)Q * (G->m / kAInline + G->m / kAChunk) +
                4ull * G->coop_blocks_async * kWarps + 64);
  if (nunits > (1ull << 26)) {
    if (!required) return TGXD_ERR_UNSUPPORTED;
    return fail(TGXD_ERR_UNSUPPORTED, "async engine: batch too large (use a round-based mode)");
  }
  if (w.a_slots < slots || w.a_units < nunits) {
    if (!dalloc<unsigned long long>(w.axq, slots) ||
        !dalloc<uint32_t>(w.aunits, nunits * kUnitWords) || !dalloc<AsyncCtl>(w.actl, 1))
      return fail(TGXD_ERR_CUDA, "device allocation failed (async queue)");
    TGXD_CUDA(cudaMemsetAsync(w.actl.p, 0, sizeof(AsyncCtl), s));
    async_reset_kernel<<<grid_for(nunits, G->sm_count), 256, 0, s>>>(
        w.aunits.as<uint32_t>(), nunits, w.actl.as<AsyncCtl>());
    ++G->ws.launches;
    w.a_slots = slots;
    w.a_units = nunits;
  }
  return TGXD_OK;
}

// The cluster tail engine's per-slot stamps (zeroed once; epochs keep them
// valid across queries) and control block.
static int ensure_tail(tgxd_graph* G, uint32_t Q) {
  Workspace& w = G->ws;
  const uint64_t slots = (uint64_t)Q * G->n;
  if (w.t_slots < slots || !w.tctl.p) {
    if (!dalloc<uint32_t>(w.tstamp, slots) || !dalloc<TailCtl>(w.tctl, 1))
      return fail(TGXD_ERR_CUDA, "device allocation failed (tail engine)");
    TGXD_CUDA(cudaMemsetAsync(w.tstamp.p, 0, slots * 4, G->stream));
    TGXD_CUDA(cudaMemsetAsync(w.tctl.p, 0, sizeof(TailCtl), G->stream));
    w.t_slots = slots;
  }
  return TGXD_OK;
}

static int launch_async(tgxd_graph* G, const Prepared& P, const DevCsr& g,
                        cudaEvent_t ev_k0, cudaEvent_t ev_k1) {
  Workspace& w = G->ws;
  cudaStream_t s = G->stream;
  const bool fast = P.kind == TGXD_FASTEST;
  const uint64_t slots = (uint64_t)P.Q * G->n;
  if (const int rc = ensure_async(G, P.Q)) return rc;
  async_init_kernel<<<grid_for(slots, G->sm_count), 256, 0, s>>>(
      w.axq.as<unsigned long long>(), slots);
  ++G->ws.launches;
  async_seed_kernel<<<1, 32, 0, s>>>(w.params.as<QueryParam>(), P.Q, G->n,
                                     w.axq.as<unsigned long long>(), w.aunits.as<uint32_t>(),
                                     w.a_units - 1, w.actl.as<AsyncCtl>(), fast);
  ++G->ws.launches;
  AsyncArgs a;
  a.g = g;
  a.qp = w.params.as<QueryParam>();
  a.X = w.X.as<int32_t>();
  a.EP = w.EP.as<int2>();
  a.R = fast ? w.R.as<int32_t>() : nullptr;
  a.XQ = w.axq.as<unsigned long long>();
  a.units = w.aunits.as<uint32_t>();
  a.umask = w.a_units - 1;
  a.c = w.actl.as<AsyncCtl>();
  a.n = G->n;
  a.Q = P.Q;
  a.strict = P.strict;
  a.cutoff = (uint32_t)std::min<uint64_t>(G->index_cutoff, 0xffffffffULL);
  a.fastest = fast ? 1 : 0;
  a.n_cand = w.cand_n.as<uint32_t>();
  a.cand_lo = w.cand_lo.as<uint32_t>();
  a.cand_cnt = w.cand_cnt.as<uint32_t>();
  a.cand_key = w.cand_key.as<int32_t>();
  a.time_limit_ns = 20ull * 1000 * 1000 * 1000;  // watchdog: 20 s
  a.chg = nullptr;
  a.chg_n = nullptr;
  a.chg_cap = 0;
  a.hctl = nullptr;
  a.hfa = a.hfb = nullptr;
  a.hfresh = 0;
  if (ev_k0) TGXD_CUDA(cudaEventRecord(ev_k0, s));
  {
    void* args[] = {&a};
    // 3 CTAs per SM: every idle warp polls a queue ticket, and with all 4
    // resident the polls slow the working warps (config 2: 1.7 vs 3.4 ms)
    static const int per_sm = [] {
      const char* e = getenv("TGXD_ASYNC_BLOCKS_PER_SM");
      return e ? std::max(1, atoi(e)) : 3;
    }();
    const int blocks = std::min(G->coop_blocks_async, per_sm * G->sm_count);
    TGXD_CUDA(cudaLaunchCooperativeKernel((const void*)async_kernel, dim3(blocks), dim3(kThreads),
                                          args, 0, s));
    ++G->ws.launches;
  }
  if (ev_k1) TGXD_CUDA(cudaEventRecord(ev_k1, s));
  w.last_async = true;
  return TGXD_OK;
}

// The one writer of the device's query parameters and seeds: uploads P's
// unless the buffers already hold exactly these (a repeated query skips two
// small copies). ensure_workspace drops the record whenever it may have
// reallocated the buffers.
static int upload_query(tgxd_graph* G, const Prepared& P) {
  Workspace& w = G->ws;
  const size_t nq = P.Q * sizeof(QueryParam), ns = P.Q * sizeof(Seed);
  const bool same = w.up_valid && w.up_qp.size() == nq && w.up_seeds.size() == ns &&
                    std::memcmp(w.up_qp.data(), P.qp.data(), nq) == 0 &&
                    std::memcmp(w.up_seeds.data(), P.seeds.data(), ns) == 0;
  if (same) return TGXD_OK;
  TGXD_CUDA(cudaMemcpyAsync(w.params.p, P.qp.data(), nq, cudaMemcpyHostToDevice, G->stream));
  TGXD_CUDA(cudaMemcpyAsync(w.seeds.p, P.seeds.data(), ns, cudaMemcpyHostToDevice, G->stream));
  const char* a = reinterpret_cast<const char*>(P.qp.data());
  const char* b = reinterpret_cast<const char*>(P.seeds.data());
  w.up_qp.assign(a, a + nq);
  w.up_seeds.assign(b, b + ns);
  w.up_valid = true;
  w.last_h2d += nq + ns;
  return TGXD_OK;
}

// Edge-state queries (edges.cuh): Overlaps for every metric, shortest
// duration for every ordering. One query (Q == 1).
static int launch_edges(tgxd_graph* G, const Prepared& P, void* out_dev, int width,
                        cudaEvent_t ev_k0, cudaEvent_t ev_k1) {
  Workspace& w = G->ws;
  cudaStream_t s = G->stream;
  const DevCsr& g = P.kind == TGXD_LATEST_DEPARTURE ? G->in : G->out;
  const uint32_t m = g.m;
  const int kind = P.kind == TGXD_SHORTEST_DURATION ? kEdgeShortest
                   : P.kind == TGXD_FASTEST          ? kEdgeFastest
                                                     : kEdgeReach;
  // shortest duration under the succeeds orderings: vertex-driven (sd.cuh)
  const bool sd = kind == kEdgeShortest && P.ordering != TGXD_OVERLAPS;
  const size_t qcap = (size_t)std::max<uint64_t>(m, G->n) + 1;  // edge or vertex queues
  bool ok = dalloc<uint32_t>(w.efa, qcap) && dalloc<uint32_t>(w.efb, qcap) &&
            dalloc<EdgeCtl>(w.ectl, 1);
  if (ok && kind == kEdgeReach) ok = dalloc<uint32_t>(w.ereached, (size_t)m / 32 + 1) != nullptr;
  if (ok && kind != kEdgeReach) ok = dalloc<uint32_t>(w.estamp, qcap) != nullptr;
  if (ok && sd) ok = dalloc<long long>(w.esm, (size_t)G->in.m + 1) != nullptr;
  if (ok && sd && !G->out2in_ready) {
    ok = dalloc<uint32_t>(G->out2in, (size_t)G->out.m + 1) != nullptr;
    if (ok && G->out.m) {
      out2in_kernel<<<grid_for(G->out.m, G->sm_count), 256, 0, s>>>(G->out, G->in,
                                                                    G->out2in.as<uint32_t>());
      ++G->ws.launches;
      G->out2in_ready = true;
    }
  }
  if (ok && kind == kEdgeFastest) ok = dalloc<int32_t>(w.edep, (size_t)m + 1) != nullptr;
  if (ok && kind == kEdgeShortest)
    ok = dalloc<long long>(w.eval, qcap) && dalloc<long long>(w.ey, G->n + 1);
  if (!ok) return fail(TGXD_ERR_CUDA, "device allocation failed (edge-state workspace)");
  {
    const int rc = upload_query(G, P);
    if (rc) return rc;
  }
  init_kernel<<<grid_for(G->n, G->sm_count), 256, 0, s>>>(
      w.X.as<int32_t>(), w.EP.as<int2>(), kind == kEdgeFastest ? w.R.as<int32_t>() : nullptr,
      G->n);
  ++G->ws.launches;
  edge_init_kernel<<<grid_for(qcap, G->sm_count), 256, 0, s>>>(
      kind, sd ? (uint32_t)(qcap - 1) : m, w.ereached.as<uint32_t>(), w.edep.as<int32_t>(),
      w.eval.as<long long>(), w.estamp.as<uint32_t>(),
      kind == kEdgeShortest ? w.ey.as<long long>() : nullptr, G->n, w.ectl.as<EdgeCtl>(),
      sd ? w.esm.as<long long>() : nullptr, sd ? G->in.m : 0u);
  ++G->ws.launches;
#ifdef TGXD_CHECK
  {
    const unsigned long long caps[2] = {qcap, (uint64_t)G->n + (uint64_t)(G->m / kChunk + 1)};
    const unsigned int zero = 0;
    TGXD_CUDA(cudaMemcpyToSymbolAsync(g_cap, caps, sizeof caps, 0, cudaMemcpyHostToDevice, s));
    TGXD_CUDA(cudaMemcpyToSymbolAsync(g_check_fail, &zero, 4, 0, cudaMemcpyHostToDevice, s));
  }
#endif
  if (sd) {
    SdArgs d;
    d.out = G->out;
    d.in = G->in;
    d.out2in = G->out2in.as<uint32_t>();
    d.qp = P.qp[0];
    d.strict = P.strict;
    d.val = w.eval.as<long long>();
    d.tree = w.esm.as<long long>();
    d.stamp = w.estamp.as<uint32_t>();
    d.fa = w.efa.as<uint32_t>();
    d.fb = w.efb.as<uint32_t>();
    d.chunks = w.chunks.as<uint2>();
    d.ctl = w.ectl.as<EdgeCtl>();
    d.nchunks = &w.ectl.as<EdgeCtl>()->nchunks;
    d.n = G->n;
    d.round_limit = m + 16;
    d.weighted = P.weighted ? 1 : 0;
    d.w = G->out_w;
    if (ev_k0) TGXD_CUDA(cudaEventRecord(ev_k0, s));
    void* sargs[] = {&d};
    TGXD_CUDA(cudaLaunchCooperativeKernel((const void*)sd_kernel, dim3(G->coop_blocks_sd),
                                          dim3(kThreads), sargs, 0, s));
    ++G->ws.launches;
    edge_fold_kernel<<<grid_for(m, G->sm_count), 256, 0, s>>>(
        g, kEdgeShortest, nullptr, d.val, w.R.as<int32_t>(), w.ey.as<long long>());
    ++G->ws.launches;
    if (ev_k1) TGXD_CUDA(cudaEventRecord(ev_k1, s));
    if (out_dev) convert_for(G, P, out_dev, width);
    TGXD_CUDA(cudaGetLastError());
    w.last_edge = true;
    w.last_async = false;
    w.last_handoff = false;
    w.last_kind = P.kind;
    w.last_q = P.Q;
    w.last_strict = P.strict;
    w.last_params = P.qp;
    return TGXD_OK;
  }
  EdgeArgs a;
  a.g = g;
  a.qp = P.qp[0];
  a.kind = kind;
  a.ord = P.ordering;
  a.bfs = P.kind == TGXD_TEMPORAL_BFS ? 1 : 0;
  a.X = w.X.as<int32_t>();
  a.reached = w.ereached.as<uint32_t>();
  a.dep = w.edep.as<int32_t>();
  a.val = w.eval.as<long long>();
  a.stamp = w.estamp.as<uint32_t>();
  a.fa = w.efa.as<uint32_t>();
  a.fb = w.efb.as<uint32_t>();
  a.ctl = w.ectl.as<EdgeCtl>();
  a.n = G->n;
  a.m = m;
  a.round_limit = m + 16;  // every round queues an edge state that strictly improved
  a.weighted = P.weighted ? 1 : 0;
  a.w = P.kind == TGXD_LATEST_DEPARTURE ? nullptr : G->out_w;
  if (ev_k0) TGXD_CUDA(cudaEventRecord(ev_k0, s));
  void* args[] = {&a};
  TGXD_CUDA(cudaLaunchCooperativeKernel((const void*)edge_kernel, dim3(G->coop_blocks_edge),
                                        dim3(kThreads), args, 0, s));
  ++G->ws.launches;
  if (kind != kEdgeReach)
    edge_fold_kernel<<<grid_for(m, G->sm_count), 256, 0, s>>>(
        g, kind, a.dep, a.val, w.R.as<int32_t>(), w.ey.as<long long>());
  if (kind != kEdgeReach) ++G->ws.launches;
  if (ev_k1) TGXD_CUDA(cudaEventRecord(ev_k1, s));
  if (out_dev) convert_for(G, P, out_dev, width);
  TGXD_CUDA(cudaGetLastError());
  w.last_edge = true;
  w.last_async = false;
  w.last_handoff = false;
  w.last_kind = P.kind;
  w.last_q = P.Q;
  w.last_strict = P.strict;
  w.last_params = P.qp;
  return TGXD_OK;
}

// A batch on the lane-per-query engine (lanes.cuh); params already uploaded.
static int launch_lanes(tgxd_graph* G, const Prepared& P, const DevCsr& g, void* out_dev,
                        int width, cudaEvent_t ev_k0, cudaEvent_t ev_k1) {
  Workspace& w = G->ws;
  w.xinv = false;  // X is rewritten by the transpose
  cudaStream_t s = G->stream;
  const size_t n = G->n;
  if (!dalloc<int32_t>(w.lxm, n * 32) || !dalloc<int2>(w.leb, n * 32) ||
      !dalloc<uint32_t>(w.ldirty, n))
    return fail(TGXD_ERR_CUDA, "device allocation failed (lane-per-query labels)");
  lanes_init_kernel<<<grid_for(n * 8, G->sm_count), 256, 0, s>>>(
      w.lxm.as<int32_t>(), w.leb.as<int2>(), w.ldirty.as<uint32_t>(), n);
  ++G->ws.launches;
  lanes_seed_kernel<<<1, 32, 0, s>>>(w.params.as<QueryParam>(), P.Q, w.lxm.as<int32_t>(),
                                     w.ldirty.as<uint32_t>(), w.fa.as<uint32_t>(),
                                     w.ctl.as<Control>());
  ++G->ws.launches;
#ifdef TGXD_CHECK
  {  // frontier: distinct vertices; chunks: segments / 128 + one per vertex
    const unsigned long long caps[2] = {(uint64_t)P.Q * G->n,
                                        (uint64_t)P.Q * G->n + (uint64_t)P.Q * (G->m / kChunk + 1)};
    const unsigned int zero = 0;
    TGXD_CUDA(cudaMemcpyToSymbolAsync(g_cap, caps, sizeof caps, 0, cudaMemcpyHostToDevice, s));
    TGXD_CUDA(cudaMemcpyToSymbolAsync(g_check_fail, &zero, 4, 0, cudaMemcpyHostToDevice, s));
  }
#endif
  LanesArgs a;
  a.g = g;
  a.qp = w.params.as<QueryParam>();
  a.Q = P.Q;
  a.n = G->n;
  a.strict = P.strict;
  a.cutoff = (uint32_t)std::min<uint64_t>(G->index_cutoff, 0xffffffffULL);
  a.XM = w.lxm.as<int32_t>();
  a.EB = w.leb.as<int2>();
  a.dirty = w.ldirty.as<uint32_t>();
  a.fa = w.fa.as<uint32_t>();
  a.fb = w.fb.as<uint32_t>();
  a.chunks = w.chunks.as<uint2>();
  a.ctl = w.ctl.as<Control>();
  // every round lowers some (vertex, query) label
  a.round_limit = (uint32_t)std::min<uint64_t>(0xfffffff0ULL, (uint64_t)P.Q * G->n + 16);
  if (ev_k0) TGXD_CUDA(cudaEventRecord(ev_k0, s));
  void* args[] = {&a};
  TGXD_CUDA(cudaLaunchCooperativeKernel((const void*)lanes_kernel, dim3(G->coop_blocks_lanes),
                                        dim3(kThreads), args, 0, s));
  ++G->ws.launches;
  if (ev_k1) TGXD_CUDA(cudaEventRecord(ev_k1, s));
  lanes_transpose_kernel<<<std::min<uint64_t>((n + 31) / 32, 8ull * G->sm_count), 256, 0, s>>>(
      w.lxm.as<int32_t>(), w.X.as<int32_t>(), G->n, P.Q);
  ++G->ws.launches;
  if (out_dev) convert_for(G, P, out_dev, width);
  TGXD_CUDA(cudaGetLastError());
  w.last_edge = false;
  w.last_async = false;
  w.last_handoff = false;
  w.last_kind = P.kind;
  w.last_q = P.Q;
  w.last_strict = P.strict;
  w.last_params = P.qp;
  return TGXD_OK;
}

// Query slots of a fastest query's split sweep (traverse.cuh
// split_seed_step): sized from the source's out-degree, which bounds its
// candidate count, so no read back is needed; the kernel decides from the
// candidates how many slots work (split_width). TGXD_FASTEST_SPLIT forces a
// width (1 = one sweep).
static int fastest_split(tgxd_graph* G, uint32_t src, uint32_t* split, int* forced) {
  const char* e = getenv("TGXD_FASTEST_SPLIT");  // read per query (tests vary it)
  *forced = e != nullptr;
  if (e) {
    *split = (uint32_t)std::max(1, atoi(e));
    return TGXD_OK;
  }
  if (G->h_out_off.size() != (size_t)G->n + 1) {  // once per handle
    G->h_out_off.resize((size_t)G->n + 1);
    TGXD_CUDA(cudaMemcpyAsync(G->h_out_off.data(), G->out.off, ((size_t)G->n + 1) * 4,
                              cudaMemcpyDeviceToHost, G->stream));
    TGXD_CUDA(cudaStreamSynchronize(G->stream));
  }
  *split = split_width(G->h_out_off[src + 1] - G->h_out_off[src], G->n, 64);
  return TGXD_OK;
}

// r[v] = min over the sub-sweeps of their r (and the arrival labels, for the
// work count: the minimum over the subsets is the sweep over all candidates).
__global__ void split_reduce_kernel(int32_t* R, int32_t* X, uint32_t n, uint32_t k) {
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += gridDim.x * blockDim.x) {
    int32_t r = R[v], x = X[v];
    for (uint32_t q = 1; q < k; ++q) {
      r = min(r, R[(size_t)q * n + v]);
      x = min(x, X[(size_t)q * n + v]);
    }
    R[v] = r;
    X[v] = x;
  }
}

static int launch_body(tgxd_graph* G, const Prepared& P, const Prepared& Pout, uint32_t split,
                       int forced, int mode, void* out_dev, int width, cudaEvent_t ev_k0,
                       cudaEvent_t ev_k1);

// Enqueues one traversal (init, seeds, the persistent kernel, widening into
// out_dev). ev_k0/ev_k1 bracket the traversal kernel when non-null.
static int launch(tgxd_graph* G, const Prepared& P, int mode, void* out_dev, int width,
                  cudaEvent_t ev_k0, cudaEvent_t ev_k1) {
  if (P.edge) {
    G->ws.xinv = false;
    return launch_edges(G, P, out_dev, width, ev_k0, ev_k1);
  }
  uint32_t split = 1;
  int forced = 0;
  if (P.kind == TGXD_FASTEST && P.Q == 1 && mode != TGXD_MODE_ASYNC)
    if (const int rc = fastest_split(G, P.seeds[0].root, &split, &forced)) return rc;
  if (split <= 1) return launch_body(G, P, P, 1, 0, mode, out_dev, width, ev_k0, ev_k1);
  Prepared Pk = P;
  Pk.Q = split;
  Pk.qp.assign(split, P.qp[0]);
  Pk.seeds.assign(split, P.seeds[0]);
  if (const int rc = ensure_workspace(G, split, true)) return rc;
  if (!dalloc<int32_t>(G->ws.dep, split))
    return fail(TGXD_ERR_CUDA, "device allocation failed (split sweep)");
  return launch_body(G, Pk, P, split, forced, mode, out_dev, width, ev_k0, ev_k1);
}

static int launch_body(tgxd_graph* G, const Prepared& P, const Prepared& Pout, uint32_t split,
                       int forced, int mode, void* out_dev, int width, cudaEvent_t ev_k0,
                       cudaEvent_t ev_k1) {
  Workspace& w = G->ws;
  w.last_edge = false;
  cudaStream_t s = G->stream;
  const bool fast = P.kind == TGXD_FASTEST;
  // temporal BFS is hop-minimal only with round-synchronous admission
  // (path_algorithms.cpp:368-371): queue-driven or dense rounds, no pulls,
  // no barrier-free engine
  const bool bfs = P.kind == TGXD_TEMPORAL_BFS;
  if (bfs && mode != TGXD_MODE_DENSE) mode = TGXD_MODE_SPARSE;
  const DevCsr& g = P.kind == TGXD_LATEST_DEPARTURE ? G->in : G->out;
  const uint64_t slots = (uint64_t)P.Q * G->n;
  {
    const int rc = upload_query(G, P);
    if (rc) return rc;
  }
  if (fast) {  // candidate departures, extracted on the device (candidates.cuh)
    if (const int rc = ensure_max_out_degree(G)) return rc;
    const size_t cap = (size_t)G->max_out_deg + 1;
    if (!dalloc<uint32_t>(w.cand_lo, cap) || !dalloc<uint32_t>(w.cand_cnt, cap) ||
        !dalloc<int32_t>(w.cand_key, cap) || !dalloc<uint32_t>(w.cand_n, 1))
      return fail(TGXD_ERR_CUDA, "device allocation failed (candidates)");
    candidates_kernel<<<1, kCandThreads, 0, s>>>(
        G->out, w.params.as<QueryParam>(), P.seeds[0].root, w.cand_lo.as<uint32_t>(),
        w.cand_cnt.as<uint32_t>(), w.cand_key.as<int32_t>(), w.cand_n.as<uint32_t>());
    ++G->ws.launches;
  }
  // batches of EA / LD queries: one warp lane per query (AUTO's choice)
  const bool lanes_ok = P.Q >= 2 && P.Q <= 32 && G->n <= kLanesMaxN && !fast && !bfs &&
                        (P.kind == TGXD_EARLIEST_ARRIVAL || P.kind == TGXD_LATEST_DEPARTURE);
  if (mode == TGXD_MODE_LANES && !lanes_ok)
    return fail(TGXD_ERR_UNSUPPORTED,
                "lane-per-query mode: 2..32 earliest-arrival or latest-departure queries, "
                "n <= 2^24");
  // AUTO takes it for window sweeps from one source: their rounds advance
  // together, so a vertex's ranges for all queries are scanned at once
  // (config-2 graph, 32 nested / shifted full windows: 9.3 ms vs 25 ms
  // slot-major). Independent sources reach a vertex in different rounds and
  // its union range is rescanned per query (32 random sources: 43 vs 36 ms;
  // config 5: 94 vs 55 ms), so those stay slot-major.
  bool one_root = true;
  for (uint32_t q = 1; q < P.Q; ++q) one_root = one_root && P.qp[q].root == P.qp[0].root;
  if (lanes_ok && (mode == TGXD_MODE_LANES ||
                   (mode == TGXD_MODE_AUTO && one_root && !getenv("TGXD_NO_LANES"))))
    return launch_lanes(G, P, g, out_dev, width, ev_k0, ev_k1);
  if (mode == TGXD_MODE_LANES) mode = TGXD_MODE_AUTO;
  // EA / LD on the round kernel: reset only what the previous such query
  // touched (X finite) instead of initializing every slot (config 3's batch:
  // 134M slots, 1.6 GB of writes); everything else initializes in full
  const bool lazy = !fast && !bfs && mode != TGXD_MODE_ASYNC && !getenv("TGXD_FULL_INIT");
  bool seeded = false;
  if (lazy) {
    if (!w.xinv) {
      init_kernel<<<grid_for(w.slots, G->sm_count), 256, 0, s>>>(w.X.as<int32_t>(),
                                                                  w.EP.as<int2>(), nullptr, w.slots);
      ++G->ws.launches;
      w.xinv = true;
    } else if (P.Q == 1) {  // reset + seed in one launch
      reset_seed_kernel<<<grid_for(std::max<uint64_t>(w.xdirty / 4, 1), G->sm_count), 256, 0, s>>>(
          w.X.as<int32_t>(), w.EP.as<int2>(), w.xdirty, P.qp[0].root, P.qp[0].klo,
          w.fa.as<uint32_t>(), w.ctl.as<Control>());
      ++G->ws.launches;
      seeded = true;
    } else if (w.xdirty) {
      reset_kernel<<<grid_for(w.xdirty, G->sm_count), 256, 0, s>>>(w.X.as<int32_t>(),
                                                                    w.EP.as<int2>(), w.xdirty);
      ++G->ws.launches;
    }
    w.xdirty = slots;
  } else {
    init_kernel<<<grid_for(slots, G->sm_count), 256, 0, s>>>(
        w.X.as<int32_t>(), w.EP.as<int2>(), fast || bfs ? w.R.as<int32_t>() : nullptr, slots);
    ++G->ws.launches;
    w.xinv = false;
  }
  if (!seeded)
    seed_kernel<<<(P.Q + 127) / 128, 128, 0, s>>>(w.params.as<QueryParam>(), P.Q, G->n,
                                                   w.X.as<int32_t>(), w.fa.as<uint32_t>(),
                                                   w.ctl.as<Control>(), fast);
  if (!seeded) ++G->ws.launches;
  if (mode == TGXD_MODE_ASYNC) {
    const int rc = launch_async(G, P, g, ev_k0, ev_k1);
    if (rc) return rc;
    if (out_dev) convert_for(G, P, out_dev, width);
    TGXD_CUDA(cudaGetLastError());
    w.last_kind = P.kind;
    w.last_q = P.Q;
    w.last_strict = P.strict;
    w.last_params = P.qp;
    if (fast) w.last_params[0].root = P.seeds[0].root;
    return TGXD_OK;
  }
  w.last_async = false;
#ifdef TGXD_CHECK
  {
    const unsigned long long caps[2] = {slots, slots + (uint64_t)P.Q * (G->m / kChunk + 1)};
    const unsigned int zero = 0;
    TGXD_CUDA(cudaMemcpyToSymbolAsync(g_cap, caps, sizeof caps, 0, cudaMemcpyHostToDevice, s));
    TGXD_CUDA(cudaMemcpyToSymbolAsync(g_check_fail, &zero, 4, 0, cudaMemcpyHostToDevice, s));
  }
#endif
  TravArgs a;
  a.g = g;
  a.qp = w.params.as<QueryParam>();
  a.X = w.X.as<int32_t>();
  a.EP = w.EP.as<int2>();
  a.R = fast || bfs ? w.R.as<int32_t>() : nullptr;
  a.hops = bfs ? 1 : 0;
  a.fa = w.fa.as<uint32_t>();
  a.fb = w.fb.as<uint32_t>();
  a.chunks = w.chunks.as<uint2>();
  a.smalls = w.smalls.as<uint2>();
  a.ctl = w.ctl.as<Control>();
  a.n = G->n;
  a.Q = P.Q;
  a.strict = P.strict;
  a.cutoff = (uint32_t)std::min<uint64_t>(G->index_cutoff, 0xffffffffULL);
  a.mode = mode;
  // AUTO: push every round unless a round relaxes more edges than 4x the
  // slot count; expand densely only when the queue holds half the slots
  // (measured on config 2: the queue-driven expand is cheaper below that).
  a.dense_f = std::max<uint64_t>(1024, slots / 2);
  if (const char* dd = getenv("TGXD_DENSE_DIV"))  // experiments: dense expand above slots / div
    a.dense_f = std::max<uint64_t>(1024, slots / (uint64_t)std::max(1, atoi(dd)));
  a.push_w = std::max<uint64_t>(4096, slots * 4);
  // a frontier holding half the slots is pulled (direction switch; a quarter
  // for fastest sweeps). Measured over config 2's 8-source rotation: pulling
  // from a quarter 1.255 ms per query, a third 1.136, half 1.102, never
  // 1.144 — a pull scans every open slot's in-edges, which is wasted on the
  // many vertices still unreachable; config 4 fastest 5.14 (quarter) vs 5.31
  // ms (half) (TGXD_PULL_DIV overrides the divisor; 0 turns AUTO's pulls off)
  const char* pf = getenv("TGXD_PULL_DIV");
  const int pdiv = pf ? atoi(pf) : (fast ? 4 : 2);
  a.pull_f = pdiv <= 0 ? ~0ull : std::max<uint64_t>(1024, slots / pdiv);
  if (const char* pfx = getenv("TGXD_PULL_F")) a.pull_f = strtoull(pfx, nullptr, 10);  // tests
  // ... and only when it jumped there from a much smaller frontier. A big
  // frontier reached by a jump (config 2's own source: 43K -> 2.58M slots)
  // is about to push the bulk of the query's edges at labels the pull can
  // prune against; one reached by steady growth (config 4 LD: 1.17M -> 5.44M)
  // follows a round that already relaxed most of them, and the pull then
  // rescans long in-segments for little (621 vs 473 us for that round,
  // profiles/r02at). Fastest sweeps keep the plain size rule.
  a.pull_grow = fast ? 0u : 6u;
  if (const char* pg = getenv("TGXD_PULL_GROW")) a.pull_grow = (unsigned)std::max(0, atoi(pg));
  // AUTO tail handoff (traverse.cuh): a frontier past its peak and at most
  // 16K slots goes to the cluster tail engine — its 16 SMs are fast per round
  // (5-7 us for a few hundred slots against ~20 us on the grid) but a ninth
  // of the GPU's throughput (config 2's rotation: handoff at 16K 1.096 ms,
  // 32K 1.101, 64K 1.123); a frontier of at most 1/16 of the slots that grows
  // by less than 8x per round goes to the async engine on every SM (config 1:
  // 27 such rounds, 0.45 ms there against 0.76 ms on the cluster engine).
  // Without a cluster, the async engine takes both (the round-1 rule).
  // TGXD_HANDOFF_F / TGXD_ASYNC_F override the sizes (0 turns one off).
  a.handoff_f = 0;
  a.async_f = 0;
  a.async_grow_only = 0;
  const bool cluster_tail = G->tail_cluster > 0;
  if (mode == TGXD_MODE_AUTO && !fast) {
    const char* hf = getenv("TGXD_HANDOFF_F");
    const char* af = getenv("TGXD_ASYNC_F");
    const uint64_t sixteenth = std::max<uint64_t>(4096, slots / 16);
    const uint64_t want_c = !cluster_tail ? 0
                            : hf          ? strtoull(hf, nullptr, 10)
                                          : std::min<uint64_t>(16384, sixteenth);
    const uint64_t want_a = af ? strtoull(af, nullptr, 10) : sixteenth;
    if (want_c && ensure_tail(G, P.Q) == TGXD_OK) a.handoff_f = want_c;
    if (want_a && ensure_async(G, P.Q, false) == TGXD_OK) a.async_f = want_a;
    a.async_grow_only = a.handoff_f != 0;
  }
  w.last_handoff = a.handoff_f != 0 || a.async_f != 0;
  if (a.handoff_f) tail_reset_kernel<<<1, 1, 0, s>>>(w.tctl.as<TailCtl>());
  if (a.handoff_f) ++G->ws.launches;
  {
    const char* hg = getenv("TGXD_HANDOFF_GROWTH");
    a.handoff_growth = hg ? (unsigned)std::max(1, atoi(hg)) : 8u;
  }
  a.rg = P.kind == TGXD_LATEST_DEPARTURE ? G->out : G->in;
  a.fastest = fast ? 1 : 0;
  a.split = split;
  a.split_forced = forced;
  a.dep = split > 1 ? w.dep.as<int32_t>() : nullptr;
  a.n_cand = w.cand_n.as<uint32_t>();
  a.cand_lo = w.cand_lo.as<uint32_t>();
  a.cand_cnt = w.cand_cnt.as<uint32_t>();
  a.cand_key = w.cand_key.as<int32_t>();
  a.init_pushes = fast ? 0ull : P.Q;
  a.trace = w.trace_dev;
  a.wtrace = w.trace_cap ? w.wtrace.as<unsigned long long>() : nullptr;
  a.wtrace_on = getenv("TGXD_WTRACE") != nullptr;
  a.trace_cap = w.trace_cap;
  a.round_limit = (uint32_t)std::min<uint64_t>(
      0xfffffff0ULL, ((uint64_t)(fast ? G->max_out_deg : 0) + 1) * ((uint64_t)slots + 2) + 16);
  // profiling only: stop after this many rounds (tools/phase_profile.sh takes
  // per-round differences of ncu captures); the labels are then incomplete
  if (const char* sr = getenv("TGXD_STOP_ROUND")) a.round_limit = (uint32_t)atoi(sr);
  {
    // early host copy from inside the round kernel (traverse.cuh): EA / LD
    // with a host result; TGXD_LOG_F overrides the frontier size (0 = off:
    // the copy starts after the round kernel)
    const bool early = w.early_req && !fast && !bfs;
    const char* lf = getenv("TGXD_LOG_F");
    const uint64_t log_f = lf ? strtoull(lf, nullptr, 10) : std::max<uint64_t>(4096, slots / 16);
    const bool in_kernel = early && log_f && G->copy_flag_dev;
    a.copy_flag = in_kernel ? G->copy_flag_dev : nullptr;
    a.log_f = log_f;
    a.fresh = slots < (1ull << 31) && !getenv("TGXD_NO_FRESH") ? 0x80000000u : 0u;
#ifdef TGXD_EXPERIMENTS
    const char* xs = getenv("TGXD_X_STOP_A");
    a.x_stop_a = xs ? (uint32_t)atoi(xs) : 0xffffffffu;
#endif
    a.p24 = early && w.p24_req ? w.p24.as<uint32_t>() : nullptr;
    a.p24_neg = P.kind == TGXD_LATEST_DEPARTURE ? 1 : 0;
    a.chg = early ? w.chg.as<uint32_t>() : nullptr;
    a.chg_n = early ? w.chg_n.as<unsigned long long>() : nullptr;
    a.chg_cap = early ? w.chg_cap : 0;
  }
  if (w.trace_host) {
    TGXD_CUDA(cudaStreamSynchronize(s));
    std::memset(w.trace_host, 0, w.trace_cap * 64ull);
    TGXD_CUDA(cudaMemsetAsync(w.wtrace.p, 0, w.trace_cap * 32ull, s));
  }
  if (ev_k0) TGXD_CUDA(cudaEventRecord(ev_k0, s));
  {
    void* args[] = {&a};
    const bool early = w.early_req && !fast && !bfs;
    if (early) TGXD_CUDA(cudaMemsetAsync(w.chg_n.p, 0, 8, s));
    TGXD_CUDA(cudaLaunchCooperativeKernel((const void*)traverse_kernel, dim3(G->coop_blocks),
                                          dim3(kThreads), args, 0, s));
    ++G->ws.launches;
    if (early) {  // the caller's copy of the labels may start now
      TGXD_CUDA(cudaEventRecord(G->early_ev, s));
      w.early_done = true;
    }
    if (a.handoff_f) {  // exits at once unless the round kernel handed off to it
      TailArgs t;
      t.g = g;
      t.qp = a.qp;
      t.X = a.X;
      t.EP = a.EP;
      t.fa = a.fa;
      t.fb = a.fb;
      t.chunks = a.chunks;
      t.stamp = w.tstamp.as<uint32_t>();
      t.hctl = a.ctl;
      t.tc = w.tctl.as<TailCtl>();
      t.n = G->n;
      t.Q = P.Q;
      t.strict = P.strict;
      t.cutoff = a.cutoff;
      t.round_limit = (uint32_t)std::min<uint64_t>(0xfffffff0ULL, slots + 16);
      t.slots = slots;
      t.fresh = a.fresh;
      t.chg = early ? w.chg.as<uint32_t>() : nullptr;
      t.chg_n = early ? w.chg_n.as<unsigned long long>() : nullptr;
      t.chg_cap = early ? w.chg_cap : 0;
      t.trace = w.trace_dev;
      t.trace_cap = w.trace_cap;
      cudaLaunchConfig_t cfg = {};
      cfg.gridDim = dim3(G->tail_cluster);
      cfg.blockDim = dim3(kTailThreads);
      cfg.stream = s;
      cudaLaunchAttribute at;
      at.id = cudaLaunchAttributeClusterDimension;
      at.val.clusterDim.x = G->tail_cluster;
      at.val.clusterDim.y = 1;
      at.val.clusterDim.z = 1;
      cfg.attrs = &at;
      cfg.numAttrs = 1;
      TGXD_CUDA(cudaLaunchKernelEx(&cfg, tail_kernel, t));
      ++G->ws.launches;
    }
    if (a.async_f) {  // the continuation exits at once unless the round kernel handed off to it
      AsyncArgs h;
      h.g = g;
      h.qp = a.qp;
      h.X = a.X;
      h.EP = a.EP;
      h.R = nullptr;
      h.XQ = w.axq.as<unsigned long long>();
      h.units = w.aunits.as<uint32_t>();
      h.umask = w.a_units - 1;
      h.c = w.actl.as<AsyncCtl>();
      h.n = G->n;
      h.Q = P.Q;
      h.strict = P.strict;
      h.cutoff = a.cutoff;
      h.fastest = 0;
      h.n_cand = nullptr;
      h.cand_lo = nullptr;
      h.cand_cnt = nullptr;
      h.cand_key = nullptr;
      h.time_limit_ns = 20ull * 1000 * 1000 * 1000;
      h.chg = early ? w.chg.as<uint32_t>() : nullptr;
      h.chg_n = early ? w.chg_n.as<unsigned long long>() : nullptr;
      h.chg_cap = early ? w.chg_cap : 0;
      h.hctl = a.ctl;
      h.hfa = a.fa;
      h.hfb = a.fb;
      h.hfresh = a.fresh;
      void* hargs[] = {&h};
      // the tail on fewer CTAs per SM (new_graph: G->tail_per_sm)
      const int tail_blocks = std::min(G->coop_blocks_async, G->tail_per_sm * G->sm_count);
      TGXD_CUDA(cudaLaunchCooperativeKernel((const void*)async_kernel, dim3(tail_blocks),
                                            dim3(kThreads), hargs, 0, s));
      ++G->ws.launches;
    }
    if (early)  // the labels lowered after the early copy started (round kernel, tail engine)
      tail_patch_kernel<<<2 * G->sm_count, 256, 0, s>>>(
          w.chg.as<uint32_t>(), w.chg_n.as<unsigned long long>(), w.chg_cap, a.X, G->patch_dev);
    if (early) ++G->ws.launches;
  }
  if (split > 1)
    split_reduce_kernel<<<grid_for(G->n, G->sm_count), 256, 0, s>>>(
        w.R.as<int32_t>(), w.X.as<int32_t>(), G->n, split);
  if (split > 1) ++G->ws.launches;
  if (ev_k1) TGXD_CUDA(cudaEventRecord(ev_k1, s));
  if (out_dev && !w.early_done) convert_for(G, Pout, out_dev, width);
  TGXD_CUDA(cudaGetLastError());
  w.last_kind = Pout.kind;
  w.last_q = Pout.Q;
  w.last_strict = Pout.strict;
  w.last_params = Pout.qp;
  if (fast) {  // count the arrival fixpoint with the source as root (all seeds)
    w.last_params[0].root = P.seeds[0].root;
  }
  return TGXD_OK;
}

static int read_stats(tgxd_graph* G, tgxd_stats* st, float kernel_ms, float total_ms) {
#ifdef TGXD_CHECK
  {
    unsigned int bad = 0;
    TGXD_CUDA(cudaMemcpyFromSymbol(&bad, g_check_fail, 4));
    if (bad)
      return fail(TGXD_ERR_CUDA, bad == 1 ? "check: frontier queue overflow"
                                          : "check: work list overflow");
  }
#endif
  if (G->ws.last_edge) {
    EdgeCtl c;
    TGXD_CUDA(cudaMemcpyAsync(&c, G->ws.ectl.p, sizeof c, cudaMemcpyDeviceToHost, G->stream));
    TGXD_CUDA(cudaStreamSynchronize(G->stream));
    if (c.error) return fail(TGXD_ERR_CUDA, "edge traversal watchdog: round limit exceeded");
    if (c.weight_err == 1)  // path_algorithms.cpp:196-203
      return fail(TGXD_ERR_WINDOW,
                  "weighted shortest duration needs non-negative integer weights");
    if (c.weight_err == 2)
      return fail(TGXD_ERR_TIME_RANGE, "edge weight beyond the device range (2^62)");
    if (!st) return TGXD_OK;
    st->rounds = c.rounds;
    st->candidates = 0;
    st->expansions = c.expanded;
    st->edges_relaxed = c.checked;
    st->index_lookups = 0;
    st->kernel_ms = kernel_ms;
    st->total_ms = total_ms;
    return TGXD_OK;
  }
  if (G->ws.last_async) {
    AsyncCtl c;
    TGXD_CUDA(cudaMemcpyAsync(&c, G->ws.actl.p, sizeof c, cudaMemcpyDeviceToHost, G->stream));
    TGXD_CUDA(cudaStreamSynchronize(G->stream));
    if (c.error) {
      Workspace& w = G->ws;
      async_reset_kernel<<<grid_for(w.a_units, G->sm_count), 256, 0, G->stream>>>(
          w.aunits.as<uint32_t>(), w.a_units, w.actl.as<AsyncCtl>());
      cudaStreamSynchronize(G->stream);
      return fail(TGXD_ERR_CUDA, "async traversal watchdog expired");
    }
    if (c.bad[0]) {
      char msg[256];
      snprintf(msg, sizeof msg, "async validation failed: kind %llu a=%llu b=%llx c=%llx", c.bad[0],
               c.bad[1], c.bad[2], c.bad[3]);
      return fail(TGXD_ERR_CUDA, msg);
    }
    if (getenv("TGXD_ASTATS"))
      fprintf(stderr, "async: batches %llu chunks %llu edges %llu wait %.3f ms busy %.3f ms (warp-sum)\n",
              c.batches, c.chunks, c.edges, c.wait_ns / 1e6, c.busy_ns / 1e6);
    if (!st) return TGXD_OK;
    st->rounds = 0;
    st->candidates = 0;
    st->expansions = c.visits;
    st->edges_relaxed = c.edges;
    st->index_lookups = c.index_lookups;
    st->kernel_ms = kernel_ms;
    st->total_ms = total_ms;
    return TGXD_OK;
  }
  Control c;
  TGXD_CUDA(cudaMemcpyAsync(&c, G->ws.ctl.p, sizeof c, cudaMemcpyDeviceToHost, G->stream));
  TGXD_CUDA(cudaStreamSynchronize(G->stream));
  if (c.error && !getenv("TGXD_STOP_ROUND"))
    return fail(TGXD_ERR_CUDA, "traversal watchdog: round limit exceeded");
  AsyncCtl ac;
  std::memset(&ac, 0, sizeof ac);
  uint32_t tail_rounds = 0;
  if (G->ws.last_handoff && c.handoff_n && c.handoff_kind == 1) {  // the cluster engine finished it
    TailCtl tc;
    TGXD_CUDA(cudaMemcpyAsync(&tc, G->ws.tctl.p, sizeof tc, cudaMemcpyDeviceToHost, G->stream));
    TGXD_CUDA(cudaStreamSynchronize(G->stream));
    if (tc.error) return fail(TGXD_ERR_CUDA, "tail traversal watchdog: round limit exceeded");
    if (getenv("TGXD_ASTATS"))
      fprintf(stderr, "tail %llu: rounds %u edges %llu visits %llu gap %.1f us loop %.1f us\n",
              c.handoff_n, tc.rounds, tc.edges, tc.visits, (tc.t_entry - c.t_end) / 1e3,
              (tc.t_end - tc.t_entry) / 1e3);
    tail_rounds = tc.rounds;
    ac.edges = tc.edges;
    ac.visits = tc.visits;
    ac.index_lookups = tc.index_lookups;
  } else if (G->ws.last_handoff && c.handoff_n) {  // the async engine finished it
    TGXD_CUDA(cudaMemcpyAsync(&ac, G->ws.actl.p, sizeof ac, cudaMemcpyDeviceToHost, G->stream));
    TGXD_CUDA(cudaStreamSynchronize(G->stream));
    if (ac.error) {
      Workspace& w = G->ws;
      async_reset_kernel<<<grid_for(w.a_units, G->sm_count), 256, 0, G->stream>>>(
          w.aunits.as<uint32_t>(), w.a_units, w.actl.as<AsyncCtl>());
      cudaStreamSynchronize(G->stream);
      return fail(TGXD_ERR_CUDA, "async traversal watchdog expired");
    }
    if (getenv("TGXD_ASTATS"))
      fprintf(stderr,
              "handoff %llu: batches %llu chunks %llu edges %llu wait %.3f ms busy %.3f ms "
              "gap %.1f us prep %.1f us loop %.1f us\n",
              c.handoff_n, ac.batches, ac.chunks, ac.edges, ac.wait_ns / 1e6, ac.busy_ns / 1e6,
              (ac.t_entry - c.t_end) / 1e3, (ac.t_loop - ac.t_entry) / 1e3,
              (ac.t_last - ac.t_loop) / 1e3);
  }
  if (!st) return TGXD_OK;
  st->rounds = c.rounds + tail_rounds;
  st->candidates = c.candidates;
  st->expansions = c.expansions + ac.visits;
  st->edges_relaxed = c.edges + c.pull_scanned + ac.edges;
  st->index_lookups = c.index_lookups + ac.index_lookups;
  st->kernel_ms = kernel_ms;
  st->total_ms = total_ms;
  return TGXD_OK;
}

// Host widening of int32 labels into the caller's int64 PathResult values
// (INT32_MAX -> INT64_MAX / INT32_MIN -> INT64_MIN; LD key space: negated,
// INT32_MAX -> INT64_MIN), 8 labels per AVX2 step when the host has it (the
// widening is the e2e limit once the copies overlap the tail). Returns the
// first index left to the scalar loop.
__attribute__((target("avx2"))) static uint64_t widen_avx2(const int32_t* src, int64_t* dst,
                                                         uint64_t a, uint64_t b, bool neg) {
  const __m256i imax32 = _mm256_set1_epi32(INT32_MAX);
  const __m256i imin32 = _mm256_set1_epi32(INT32_MIN);
  const __m256i imax64 = _mm256_set1_epi64x(INT64_MAX);
  const __m256i imin64 = _mm256_set1_epi64x(INT64_MIN);
  const __m256i zero = _mm256_setzero_si256();
  uint64_t i = a;
  for (; i + 8 <= b; i += 8) {
    const __m256i x = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + i));
    const __m256i is_max = _mm256_cmpeq_epi32(x, imax32);
    __m256i lo = _mm256_cvtepi32_epi64(_mm256_castsi256_si128(x));
    __m256i hi = _mm256_cvtepi32_epi64(_mm256_extracti128_si256(x, 1));
    const __m256i mlo = _mm256_cvtepi32_epi64(_mm256_castsi256_si128(is_max));
    const __m256i mhi = _mm256_cvtepi32_epi64(_mm256_extracti128_si256(is_max, 1));
    if (neg) {
      lo = _mm256_blendv_epi8(_mm256_sub_epi64(zero, lo), imin64, mlo);
      hi = _mm256_blendv_epi8(_mm256_sub_epi64(zero, hi), imin64, mhi);
    } else {
      const __m256i is_min = _mm256_cmpeq_epi32(x, imin32);
      const __m256i nlo = _mm256_cvtepi32_epi64(_mm256_castsi256_si128(is_min));
      const __m256i nhi = _mm256_cvtepi32_epi64(_mm256_extracti128_si256(is_min, 1));
      lo = _mm256_blendv_epi8(_mm256_blendv_epi8(lo, imax64, mlo), imin64, nlo);
      hi = _mm256_blendv_epi8(_mm256_blendv_epi8(hi, imax64, mhi), imin64, nhi);
    }
    _mm256_storeu_si256(reinterpret_cast<__m256i*>(dst + i), lo);
    _mm256_storeu_si256(reinterpret_cast<__m256i*>(dst + i + 4), hi);
  }
  return i;
}

// 24-bit labels (pack24, traverse.cuh) -> int64 PathResult values: 8 per
// step (bytes 0-11 of the group to the low lane, 12-23 to the high lane, one
// byte shuffle, the 0xFFFFFF sentinel blended). `src` is readable 8 bytes
// past the last group.
__attribute__((target("avx2"))) static uint64_t widen24_avx2(const uint8_t* src, int64_t* dst,
                                                           uint64_t a, uint64_t b, bool neg) {
  const __m256i perm = _mm256_setr_epi32(0, 1, 2, 3, 3, 4, 5, 6);
  const __m256i shuf = _mm256_setr_epi8(0, 1, 2, -1, 3, 4, 5, -1, 6, 7, 8, -1, 9, 10, 11, -1,
                                        0, 1, 2, -1, 3, 4, 5, -1, 6, 7, 8, -1, 9, 10, 11, -1);
  const __m256i sent = _mm256_set1_epi32(0xFFFFFF);
  const __m256i inf64 = _mm256_set1_epi64x(neg ? INT64_MIN : INT64_MAX);
  uint64_t i = a;
  for (; i + 8 <= b; i += 8) {
    const __m256i raw = _mm256_loadu_si256(reinterpret_cast<const __m256i*>(src + 3 * i));
    const __m256i x = _mm256_shuffle_epi8(_mm256_permutevar8x32_epi32(raw, perm), shuf);
    const __m256i is_inf = _mm256_cmpeq_epi32(x, sent);
    const __m256i lo = _mm256_cvtepu32_epi64(_mm256_castsi256_si128(x));
    const __m256i hi = _mm256_cvtepu32_epi64(_mm256_extracti128_si256(x, 1));
    const __m256i mlo = _mm256_cvtepi32_epi64(_mm256_castsi256_si128(is_inf));
    const __m256i mhi = _mm256_cvtepi32_epi64(_mm256_extracti128_si256(is_inf, 1));
    _mm256_storeu_si256(reinterpret_cast<__m256i*>(dst + i), _mm256_blendv_epi8(lo, inf64, mlo));
    _mm256_storeu_si256(reinterpret_cast<__m256i*>(dst + i + 4), _mm256_blendv_epi8(hi, inf64, mhi));
  }
  return i;
}

static inline int64_t widen24_one(const uint8_t* src, uint64_t i, bool neg) {
  const uint32_t u = (uint32_t)src[3 * i] | ((uint32_t)src[3 * i + 1] << 8) |
                     ((uint32_t)src[3 * i + 2] << 16);
  return u == 0xFFFFFFu ? (neg ? INT64_MIN : INT64_MAX) : (int64_t)u;
}

static bool host_avx2() {
  static const bool has = [] {
    if (const char* e = getenv("TGXD_HOST_AVX2")) return atoi(e) != 0;
    __builtin_cpu_init();
    return __builtin_cpu_supports("avx2") != 0;
  }();
  return has;
}

static int query_impl(tgxd_graph* G, int kind, uint32_t k, const uint32_t* verts,
                      const uint64_t* ta, const uint64_t* tb, int ordering, int mode, void* out,
                      int width, int out_on_device, tgxd_stats* stats);

// Label bytes (4 per slot) above which a wide-window AUTO batch is split
// (TGXD_BATCH_BUDGET_MB overrides). Config 5's 16-query groups (device ms):
// budget 64 MiB (one query at a time) 41.9, 128 (2) 42.9, 256 (4) 43.9,
// 512 (8) 47.5, one batch 53.1.
static uint64_t batch_label_budget() {
  const char* e = getenv("TGXD_BATCH_BUDGET_MB");
  return e ? std::max<uint64_t>(1, strtoull(e, nullptr, 10)) << 20 : 64ull << 20;
}

__global__ void time_span_kernel(DevCsr g, int* span) {
  int lo = INT32_MAX, hi = INT32_MIN;
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < g.m; i += gridDim.x * blockDim.x) {
    lo = min(lo, __ldg(g.key + i));
    hi = max(hi, (int32_t)__ldg(&g.pay[i].y));
  }
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMin(span, lo);
    atomicMax(span + 1, hi);
  }
}

// [earliest start, latest end] of the graph's edges (once per graph).
static int ensure_time_span(tgxd_graph* G) {
  if (G->span_known) return TGXD_OK;
  DeviceBuffer tmp;
  int* d = dalloc<int>(tmp, 2);
  if (!d) return fail(TGXD_ERR_CUDA, "allocation (time span)");
  const int init[2] = {INT32_MAX, INT32_MIN};
  TGXD_CUDA(cudaMemcpyAsync(d, init, 8, cudaMemcpyHostToDevice, G->stream));
  if (G->out.m)
    time_span_kernel<<<grid_for(G->out.m, G->sm_count), 256, 0, G->stream>>>(G->out, d);
  TGXD_CUDA(cudaMemcpyAsync(G->span, d, 8, cudaMemcpyDeviceToHost, G->stream));
  TGXD_CUDA(cudaStreamSynchronize(G->stream));
  G->span_known = true;
  return TGXD_OK;
}

// AUTO batches of wide-window EA / LD queries whose labels exceed
// batch_label_budget() run in groups within it: a batch's rounds are shared,
// but when its queries reach most of the graph every label probe of a Q x n
// batch goes to DRAM (config 5: 32 queries x 2^24 slots = 2.1 GB of labels;
// slot-major batch 50.9 ms, one by one 46.5). Narrow windows (config 3, 1% of
// the timeline) reach little and keep the shared rounds. *group = 0: no split.
// (`locked`: the caller already holds G->mu)
static int split_group(tgxd_graph* G, int kind, uint32_t k, const uint64_t* ta,
                       const uint64_t* tb, int mode, bool locked, uint32_t* group) {
  *group = 0;
  if (!(k > 1 && mode == TGXD_MODE_AUTO && ta && tb &&
        (kind == TGXD_EARLIEST_ARRIVAL || kind == TGXD_LATEST_DEPARTURE) &&
        (uint64_t)k * G->n * 4 > batch_label_budget() && !getenv("TGXD_NO_SPLIT")))
    return TGXD_OK;
  if (!G->span_known) {
    std::unique_lock<std::mutex> lock(G->mu, std::defer_lock);
    if (!locked) lock.lock();
    TGXD_CUDA(cudaSetDevice(G->device));
    if (const int rc = ensure_time_span(G)) return rc;
  }
  const double span = std::max(1.0, (double)G->span[1] - (double)G->span[0]);
  double frac = 0;
  for (uint32_t q = 0; q < k; ++q) {
    const double lo = std::max<double>((double)ta[q], G->span[0]);
    const double hi = std::min<double>((double)std::min<uint64_t>(tb[q], kTimeLimit63), G->span[1]);
    frac += std::max(0.0, hi - lo) / span;
  }
  if (frac / k < 0.05) return TGXD_OK;
  const uint32_t g = (uint32_t)std::max<uint64_t>(1, batch_label_budget() / ((uint64_t)G->n * 4));
  if (g < k) *group = g;
  return TGXD_OK;
}

// Queries of a batch in groups of `group`, one traversal per group, results
// and statistics accumulated (tgxd_last_work then refers to the last group).
static int run_groups(tgxd_graph* G, int kind, uint32_t k, const uint32_t* verts,
                      const uint64_t* ta, const uint64_t* tb, int ordering, int mode, void* out,
                      int width, int out_on_device, tgxd_stats* stats, uint32_t group) {
  if (!verts || !ta || !tb) return fail(TGXD_ERR_ARGUMENT, "null query arrays");
  tgxd_stats acc;
  std::memset(&acc, 0, sizeof acc);
  uint64_t h2d = 0, d2h = 0;
  for (uint32_t q = 0; q < k; q += group) {
    const uint32_t kq = std::min(group, k - q);
    char* o = static_cast<char*>(out) + (size_t)q * G->n * width;
    tgxd_stats one;
    const int rc = query_impl(G, kind, kq, verts + q, ta + q, tb + q, ordering, mode, o, width,
                              out_on_device, &one);
    if (rc) return rc;
    h2d += G->ws.last_h2d;
    d2h += G->ws.last_d2h;
    G->ws.last_h2d = h2d;
    G->ws.last_d2h = d2h;
    acc.rounds += one.rounds;
    acc.candidates += one.candidates;
    acc.expansions += one.expansions;
    acc.edges_relaxed += one.edges_relaxed;
    acc.index_lookups += one.index_lookups;
    acc.kernel_ms += one.kernel_ms;
    acc.total_ms += one.total_ms;
  }
  if (stats) *stats = acc;
  return TGXD_OK;
}

static int query_impl(tgxd_graph* G, int kind, uint32_t k, const uint32_t* verts,
                      const uint64_t* ta, const uint64_t* tb, int ordering, int mode, void* out,
                      int width, int out_on_device, tgxd_stats* stats) {
  if (!G) return fail(TGXD_ERR_ARGUMENT, "null graph");
  if (!out) return fail(TGXD_ERR_ARGUMENT, "null output");
  if (width != 4 && width != 8) return fail(TGXD_ERR_ARGUMENT, "width must be 4 or 8");
  const bool edge_kind = ordering == TGXD_OVERLAPS || kind == TGXD_SHORTEST_DURATION ||
                         kind == TGXD_SHORTEST_DURATION_WEIGHTED;
  if ((kind == TGXD_FASTEST || edge_kind) && k > 1)  // one sweep / edge traversal per source
    return run_groups(G, kind, k, verts, ta, tb, ordering, mode, out, width, out_on_device, stats,
                      1);
  {
    uint32_t group = 0;
    if (const int rc = split_group(G, kind, k, ta, tb, mode, false, &group)) return rc;
    if (group)
      return run_groups(G, kind, k, verts, ta, tb, ordering, mode, out, width, out_on_device,
                        stats, group);
  }
  std::lock_guard<std::mutex> lock(G->mu);
  TGXD_CUDA(cudaSetDevice(G->device));
  G->ws.last_h2d = 0;
  Prepared P;
  int rc = prepare(G, kind, k, verts, ta, tb, ordering, P);
  if (rc) return rc;
  rc = ensure_workspace(G, P.Q, kind == TGXD_FASTEST || kind == TGXD_TEMPORAL_BFS);
  if (rc) return rc;
  Workspace& w = G->ws;
  const uint64_t slots = (uint64_t)P.Q * G->n;
  // Large int64 results for the host travel as int32 (every label but the
  // root's fits; the root's exact value is written on the host) in chunks,
  // widened by the handle's host threads while later chunks are still
  // crossing PCIe: half the bytes on the link, the widening hidden behind it.
  // (up to 2^26 slots: the pinned staging stays <= 256 MB per handle)
  const bool staged = !out_on_device && width == 8 && slots >= (1u << 20) &&
                      slots <= (1ull << 26) && P.kind != TGXD_SHORTEST_DURATION;
  void* dout = out;
  if (!out_on_device) {
    if (!dalloc<char>(w.timing_out, slots * width))
      return fail(TGXD_ERR_CUDA, "device allocation failed (output staging)");
    dout = w.timing_out.p;
  }
  if (staged && G->pinned_n < slots) {
    if (G->pinned) cudaFreeHost(G->pinned);
    G->pinned = nullptr;
    G->pinned_n = 0;
    TGXD_CUDA(cudaHostAlloc(&G->pinned, slots * 4, cudaHostAllocDefault));
    G->pinned_n = slots;
  }
  static const int kChunks = [] {
    const char* e = getenv("TGXD_HOST_CHUNKS");
    return e ? std::max(1, std::min(16, atoi(e))) : 8;
  }();
  if (staged && !G->chunk_ev[kChunks - 1])
    for (int c = 0; c < kChunks; ++c)
      if (!G->chunk_ev[c])
      TGXD_CUDA(cudaEventCreateWithFlags(&G->chunk_ev[c], cudaEventDisableTiming));
  // Early copy (EA / LD through the round kernel): the labels leave for the
  // host on a second stream as soon as the round kernel is done, while the
  // async engine finishes the tail; the few labels the tail changes come
  // back afterwards as a patch list in mapped memory.
  const bool early_ok = staged && !P.edge && !getenv("TGXD_NO_EARLY_COPY") &&
                        (kind == TGXD_EARLIEST_ARRIVAL || kind == TGXD_LATEST_DEPARTURE);
  if (early_ok) {
    size_t cap = std::min<size_t>(1ull << 24, std::max<size_t>(1ull << 16, slots / 4));
    if (const char* e = getenv("TGXD_PATCH_CAP")) cap = std::max(1, atoi(e));  // tests: the re-copy
    if (!G->copy_stream)
      TGXD_CUDA(cudaStreamCreateWithFlags(&G->copy_stream, cudaStreamNonBlocking));
    if (!G->early_ev) TGXD_CUDA(cudaEventCreateWithFlags(&G->early_ev, cudaEventDisableTiming));
    if (G->patch_cap < cap) {
      if (G->patch_host) cudaFreeHost(G->patch_host);
      G->patch_host = nullptr;
      G->patch_cap = 0;
      void* hp = nullptr;
      TGXD_CUDA(cudaHostAlloc(&hp, (cap + 1) * 8, cudaHostAllocMapped));
      G->patch_host = static_cast<unsigned long long*>(hp);
      void* dp = nullptr;
      TGXD_CUDA(cudaHostGetDevicePointer(&dp, hp, 0));
      G->patch_dev = static_cast<unsigned long long*>(dp);
      G->patch_cap = cap;
    }
    if (!G->copy_flag_host) {
      void* hp = nullptr;
      TGXD_CUDA(cudaHostAlloc(&hp, 64, cudaHostAllocMapped));
      G->copy_flag_host = static_cast<volatile unsigned int*>(hp);
      void* dp = nullptr;
      TGXD_CUDA(cudaHostGetDevicePointer(&dp, hp, 0));
      G->copy_flag_dev = static_cast<unsigned int*>(dp);
    }
    *G->copy_flag_host = 0u;
    if (!dalloc<uint32_t>(w.chg, cap) || !dalloc<unsigned long long>(w.chg_n, 1))
      return fail(TGXD_ERR_CUDA, "device allocation failed (tail patch list)");
    w.chg_cap = cap;
    G->patch_host[0] = 0;  // no tail: nothing to patch
  }
  // the early copy moves 24-bit labels when every time of the graph fits
  // (config 2: 12.6 MB over PCIe instead of 16.8; TGXD_NO_PACK24 turns it off)
  bool pack = false;
  if (early_ok && !getenv("TGXD_NO_PACK24")) {
    if (const int rc2 = ensure_time_span(G)) return rc2;
    pack = G->span[0] >= 0 && G->span[1] < 0xFFFFFE;
    if (pack && !dalloc<uint32_t>(w.p24, (slots * 3 + 3) / 4 + 16))
      return fail(TGXD_ERR_CUDA, "device allocation failed (packed labels)");
  }
  w.p24_req = pack;
  w.early_req = early_ok;
  w.early_done = false;
  // TGXD_E2E_TRACE: host timeline of this call on stderr (diagnostics)
  static const bool e2e_trace = getenv("TGXD_E2E_TRACE") != nullptr;
  auto host_us = [] {
    return std::chrono::duration<double, std::micro>(
               std::chrono::steady_clock::now().time_since_epoch()).count();
  };
  const double h0 = e2e_trace ? host_us() : 0.0;
  double h_flag = 0, h_enq = 0, h_c0 = 0, h_clast = 0, h_widen = 0;
  bool by_flag = false;
  TGXD_CUDA(cudaEventRecord(w.ev[2], G->stream));
  rc = launch(G, P, mode, dout, staged ? 4 : width, w.ev[0], w.ev[1]);
  const double h_launched = e2e_trace ? host_us() : 0.0;
  w.early_req = false;
  w.p24_req = false;
  if (rc) return rc;
  const bool early = w.early_done;  // the traversal took the round kernel
  const bool p24 = early && pack;
  // chunk c covers [bound(c), bound(c + 1)): shrinking chunks (1 - ((K - c) / K)^2
  // of the slots before chunk c), so the widening exposed after the last copy
  // is short (config 2: the last of 8 chunks is 1.6 % of the labels instead
  // of 12.5 %); TGXD_FLAT_CHUNKS=1 makes them equal
  static const bool flat = getenv("TGXD_FLAT_CHUNKS") != nullptr;
  auto bound = [&](int c) -> uint64_t {
    if (c >= kChunks) return slots;
    if (flat) return std::min<uint64_t>(slots, c * ((slots + kChunks - 1) / kChunks));
    const double r = (double)(kChunks - c) / kChunks;
    return std::min<uint64_t>(slots, (uint64_t)((1.0 - r * r) * (double)slots) & ~(uint64_t)7);
  };
  cudaStream_t cs = early ? G->copy_stream : G->stream;
  const int32_t* csrc = early ? w.X.as<int32_t>() : static_cast<int32_t*>(dout);
  if (early) {
    // the copies may start once the round kernel raises the copy flag (its
    // heavy rounds are over; later changes are listed for the patch) or,
    // at the latest, when it is done
    for (;;) {
      if (*G->copy_flag_host) {
        by_flag = true;
        break;
      }
      const cudaError_t q = cudaEventQuery(G->early_ev);
      if (q == cudaSuccess) break;
      if (q != cudaErrorNotReady) return fail(TGXD_ERR_CUDA, cudaGetErrorString(q));
    }
    if (e2e_trace) h_flag = host_us();
    if (p24 && !by_flag) {  // the round kernel ended without packing: pack beside the tail
      TGXD_CUDA(cudaStreamWaitEvent(cs, G->early_ev, 0));
      pack24_kernel<<<grid_for((slots + 3) / 4, G->sm_count), 256, 0, cs>>>(
          w.X.as<int32_t>(), w.p24.as<uint32_t>(), slots, kind == TGXD_LATEST_DEPARTURE ? 1 : 0);
      ++G->ws.launches;
    }
  }
  if (staged) {
    for (int c = 0; c < kChunks; ++c) {
      const uint64_t lo = bound(c);
      const uint64_t len = bound(c + 1) - lo;
      if (len && p24)
        TGXD_CUDA(cudaMemcpyAsync(reinterpret_cast<char*>(G->pinned) + 3 * lo,
                                  w.p24.as<char>() + 3 * lo, len * 3, cudaMemcpyDeviceToHost, cs));
      else if (len)
        TGXD_CUDA(cudaMemcpyAsync(G->pinned + lo, csrc + lo, len * 4, cudaMemcpyDeviceToHost, cs));
      TGXD_CUDA(cudaEventRecord(G->chunk_ev[c], cs));
    }
    if (early) TGXD_CUDA(cudaStreamWaitEvent(G->stream, G->chunk_ev[kChunks - 1], 0));
  } else if (!out_on_device) {
    TGXD_CUDA(cudaMemcpyAsync(out, dout, slots * width, cudaMemcpyDeviceToHost, G->stream));
  }
  TGXD_CUDA(cudaEventRecord(w.ev[3], G->stream));
  if (e2e_trace) h_enq = host_us();
  if (staged) {
    if (G->pool.size() == 0)
      G->pool.start([&] {
        const char* e = getenv("TGXD_HOST_THREADS");
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        // the widening is the e2e limit once the copies overlap the tail:
        // config 2 on a 16-core host, 12 threads 1.28-1.33 ms vs 8 threads
        // 1.43-1.53 (non-temporal stores measured 2.9-3.6 ms); views that
        // run side by side split the host threads
        if (e) return std::max(1, atoi(e));
        const int t = (int)std::max(1u, std::min(12u, hw > 4 ? hw - 4 : hw));
        return std::max(1, t / std::max(1, G->share));
      }());
    const int T = G->pool.size();
    int64_t* o64 = static_cast<int64_t*>(out);
    const int32_t* src = G->pinned;
    // early copies carry key-space labels: LD's are negated (DevCsr In layout)
    const bool neg = early && kind == TGXD_LATEST_DEPARTURE;
    auto widen = [neg](int32_t v) -> int64_t {
      if (neg) return v == INT32_MAX ? INT64_MIN : -(int64_t)v;
      return v == INT32_MAX ? INT64_MAX : v == INT32_MIN ? INT64_MIN : (int64_t)v;
    };
    std::atomic<int> bad{0};
    std::atomic<int> widened{0};
    std::atomic<int> recopy{0};
    const volatile unsigned long long* ph = G->patch_host;
    G->pool.run([&](int wi) {
      for (int c = 0; c < kChunks; ++c) {
        const uint64_t lo = bound(c);
        const uint64_t hi = bound(c + 1);
        const uint64_t per = (hi - lo + T - 1) / T;
        const uint64_t a = std::min(hi, lo + wi * per), b = std::min(hi, a + per);
        if (cudaEventSynchronize(G->chunk_ev[c]) != cudaSuccess) {
          bad = 1;
          break;
        }
        if (e2e_trace && wi == 0 && c == 0) h_c0 = host_us();
        if (e2e_trace && wi == 0 && c == kChunks - 1) h_clast = host_us();
        uint64_t i = a;
        if (p24) {  // 24-bit labels (times, sentinel 0xFFFFFF)
          const uint8_t* s8 = reinterpret_cast<const uint8_t*>(src);
          // the vector loads read 8 bytes past their 8 labels: stay clear of
          // the staging's end
          const uint64_t vb = b + 8 <= slots ? b : (b > 8 ? b - 8 : a);
          if (host_avx2() && vb > a) i = widen24_avx2(s8, o64, a, vb, neg);
          for (; i < b; ++i) o64[i] = widen24_one(s8, i, neg);
          continue;
        }
        if (host_avx2()) i = widen_avx2(src, o64, a, b, neg);  // 8 labels per step
        if (neg) {
          for (; i < b; ++i) o64[i] = widen(src[i]);
        } else {
          for (; i < b; ++i) {
            const int32_t v = src[i];
            o64[i] = v == INT32_MAX   ? INT64_MAX
                     : v == INT32_MIN ? INT64_MIN
                                      : (int64_t)v;
          }
        }
      }
      if (!early) return;
      // the tail's patch list, in the same dispatch: once every worker has
      // widened (a patched slot may lie in another worker's share) and the
      // tail and its list are done
      widened.fetch_add(1);
      if (cudaEventSynchronize(w.ev[3]) != cudaSuccess) bad = 1;
      while (widened.load() < T) std::this_thread::yield();
      if (bad) return;
      const unsigned long long np = ph[0];
      if (np > w.chg_cap) {  // too many changes to list: the caller copies the labels again
        recopy = 1;
        return;
      }
      const uint64_t per = (np + T - 1) / T;
      const uint64_t a = std::min<uint64_t>(np, wi * per), b = std::min<uint64_t>(np, a + per);
      for (uint64_t i = a; i < b; ++i) {
        const unsigned long long e = ph[1 + i];
        o64[(uint32_t)e] = widen((int32_t)(uint32_t)(e >> 32));
      }
    });
    if (e2e_trace) h_widen = host_us();
    if (bad) return fail(TGXD_ERR_CUDA, "result copy failed");
    if (recopy) {
      TGXD_CUDA(cudaMemcpyAsync(G->pinned, w.X.p, slots * 4, cudaMemcpyDeviceToHost, G->stream));
      TGXD_CUDA(cudaStreamSynchronize(G->stream));
      G->pool.run([&](int wi) {
        const uint64_t per = (slots + T - 1) / T;
        const uint64_t a = std::min<uint64_t>(slots, wi * per), b = std::min(slots, a + per);
        for (uint64_t i = a; i < b; ++i) o64[i] = widen(src[i]);
      });
    }
    for (uint32_t q = 0; q < P.Q; ++q)  // the roots' exact values (t_a, t_b, 0)
      o64[(uint64_t)q * G->n + P.seeds[q].root] = P.seeds[q].value;
    w.last_d2h = slots * (p24 ? 3 : 4);
    if (early) {
      const unsigned long long np = G->patch_host[0];
      w.last_d2h += np > w.chg_cap ? slots * 4 : 8 * (np + 1);
    }
  } else {
    w.last_d2h = out_on_device ? 0 : slots * (uint64_t)width;
  }
  TGXD_CUDA(cudaStreamSynchronize(G->stream));
  float km = 0, tm = 0;
  TGXD_CUDA(cudaEventElapsedTime(&km, w.ev[0], w.ev[1]));
  TGXD_CUDA(cudaEventElapsedTime(&tm, w.ev[2], w.ev[3]));
  if (e2e_trace)
    fprintf(stderr,
            "e2e us: launched %.0f copy-start %.0f (%s) enqueued %.0f chunk0 %.0f last-chunk %.0f "
            "widened+patched %.0f end %.0f | kernels %.0f span %.0f patch %llu\n",
            h_launched - h0, h_flag - h0, by_flag ? "flag" : "event", h_enq - h0, h_c0 - h0,
            h_clast - h0, h_widen - h0, host_us() - h0, km * 1e3, tm * 1e3,
            G->patch_host ? (unsigned long long)G->patch_host[0] : 0ull);
  return read_stats(G, stats, km, tm);
}

// E_adm / V_reached of slot q from the final labels; warp
// per vertex.
__global__ void work_kernel(DevCsr g, const int32_t* X, QueryParam qp, int strict,
                            unsigned long long* acc) {
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t nw = (gridDim.x * blockDim.x) >> 5;
  unsigned long long e_adm = 0, reached = 0;
  for (uint32_t v = (blockIdx.x * blockDim.x + threadIdx.x) >> 5; v < g.n; v += nw) {
    const int32_t x = X[v];
    if (x == kInf && v != qp.root) continue;
    if (lane == 0) ++reached;
    int32_t lb = v == qp.root ? qp.klo : x + strict;
    if (lb < qp.klo) lb = qp.klo;
    const uint32_t s = g.off[v], t = g.off[v + 1];
    for (uint32_t j = s + lane; j < t; j += 32) {
      const int32_t k = g.key[j];
      e_adm += (k >= lb && (int32_t)g.pay[j].y <= qp.vhi) ? 1 : 0;
    }
  }
  for (int o = 16; o > 0; o >>= 1) {
    e_adm += __shfl_xor_sync(0xffffffffu, e_adm, o);
    reached += __shfl_xor_sync(0xffffffffu, reached, o);
  }
  if (lane == 0) {
    atomicAdd(acc, e_adm);
    atomicAdd(acc + 1, reached);
  }
}

}  // namespace tgxd

using namespace tgxd;

extern "C" {

const char* tgxd_last_error(void) { return g_err.c_str(); }
int tgxd_version(void) { return TGXD_VERSION; }

int tgxd_device_count(int* count) {
  if (!count) return fail(TGXD_ERR_ARGUMENT, "null count");
  *count = 0;
  if (cudaGetDeviceCount(count) != cudaSuccess) *count = 0;
  cudaGetLastError();
  return TGXD_OK;
}

int tgxd_generate_host(const tgxd_gen_config* cfg, uint64_t capacity, uint64_t* m_out,
                       uint32_t* src, uint32_t* dst, uint64_t* start, uint64_t* end) {
  GenParams p;
  std::vector<uint64_t> thr;
  int rc = gen_params(cfg, p, thr);
  if (rc) return rc;
  if (!m_out) return fail(TGXD_ERR_ARGUMENT, "null m_out");
  const uint64_t m = cfg->m;
  const bool drop = cfg->kind == TGXD_GEN_UNIFORM;
  std::vector<GenEdge> tmp(m);
  const unsigned nt = std::max(1u, std::min(64u, std::thread::hardware_concurrency()));
  std::vector<std::thread> th;
  for (unsigned t = 0; t < nt; ++t) {
    th.emplace_back([&, t] {
      const uint64_t b = m * t / nt, e = m * (t + 1) / nt;
      for (uint64_t i = b; i < e; ++i) tmp[i] = gen_edge(p, thr.data(), i);
    });
  }
  for (auto& x : th) x.join();
  uint64_t k = 0;
  for (uint64_t i = 0; i < m; ++i) {
    const GenEdge& e = tmp[i];
    if (drop && e.src == e.dst) continue;
    if (k < capacity && src) {
      src[k] = e.src;
      dst[k] = e.dst;
      start[k] = (uint64_t)e.start;
      end[k] = (uint64_t)e.end;
    }
    ++k;
  }
  *m_out = k;
  if (k > capacity && src) return fail(TGXD_ERR_ARGUMENT, "capacity smaller than the edge count");
  return TGXD_OK;
}

int tgxd_graph_generate(const tgxd_gen_config* cfg, int directed, uint64_t index_cutoff,
                        tgxd_graph** out) {
  if (!out) return fail(TGXD_ERR_ARGUMENT, "null out");
  *out = nullptr;
  GenParams p;
  std::vector<uint64_t> thr;
  int rc = gen_params(cfg, p, thr);
  if (rc) return rc;
  const uint32_t n = p.n_vertices;
  const uint64_t m = cfg->m;
  const uint64_t cap = directed ? m : 2 * m;
  if (cap >= 0xffffffffULL) return fail(TGXD_ERR_ARGUMENT, "edge count must stay below 2^32");
  tgxd_graph* G = nullptr;
  rc = new_graph(n, index_cutoff, directed, &G);
  if (rc) return rc;
  G->m_logical = m;
  cudaStream_t s = G->stream;
  DeviceBuffer bthr, bs, bd, bst, ben, bflag, bpos, cs, cd, cst, cen, temp;
  uint64_t* dthr = dalloc<uint64_t>(bthr, thr.size());
  uint32_t* ds = dalloc<uint32_t>(bs, cap);
  uint32_t* dd = dalloc<uint32_t>(bd, cap);
  int32_t* dst_ = dalloc<int32_t>(bst, cap);
  int32_t* den = dalloc<int32_t>(ben, cap);
  uint32_t* fl = dalloc<uint32_t>(bflag, m + 1);
  uint32_t* pos = dalloc<uint32_t>(bpos, m + 1);
  if (!dthr || !ds || !dd || !dst_ || !den || !fl || !pos) {
    tgxd_graph_destroy(G);
    return fail(TGXD_ERR_CUDA, "device allocation failed (generator)");
  }
  auto cleanup = [&](int code) {
    if (code) tgxd_graph_destroy(G);
    return code;
  };
#define GEN_CUDA(expr)                                                                     \
  do {                                                                                     \
    cudaError_t _e = (expr);                                                               \
    if (_e != cudaSuccess)                                                                 \
      return cleanup(fail(TGXD_ERR_CUDA, std::string(#expr) + ": " + cudaGetErrorString(_e))); \
  } while (0)
  GEN_CUDA(cudaMemcpyAsync(dthr, thr.data(), thr.size() * 8, cudaMemcpyHostToDevice, s));
  const int gb = grid_for(m, G->sm_count);
  if (m) gen_kernel<<<gb, 256, 0, s>>>(p, dthr, m, ds, dd, dst_, den);
  uint64_t mm = m;
  size_t tb = 0;
  GEN_CUDA(cub::DeviceScan::ExclusiveSum(nullptr, tb, fl, pos, (int64_t)m + 1, s));
  if (temp.ensure(tb + 16) != cudaSuccess) return cleanup(fail(TGXD_ERR_CUDA, "scan scratch"));
  auto count_non_loops = [&](const uint32_t* a, const uint32_t* b) -> int {
    if (m) non_loop_flags<<<gb, 256, 0, s>>>(a, b, m, fl);
    GEN_CUDA(cudaMemsetAsync(fl + m, 0, 4, s));
    size_t t2 = tb;
    GEN_CUDA(cub::DeviceScan::ExclusiveSum(temp.p, t2, fl, pos, (int64_t)m + 1, s));
    return TGXD_OK;
  };
  if (cfg->kind == TGXD_GEN_UNIFORM) {  // self-loops dropped (BASELINE config 1)
    if ((rc = count_non_loops(ds, dd))) return cleanup(rc);
    uint32_t kept = 0;
    GEN_CUDA(cudaMemcpyAsync(&kept, pos + m, 4, cudaMemcpyDeviceToHost, s));
    GEN_CUDA(cudaStreamSynchronize(s));
    uint32_t* o_s = dalloc<uint32_t>(cs, cap);
    uint32_t* o_d = dalloc<uint32_t>(cd, cap);
    int32_t* o_st = dalloc<int32_t>(cst, cap);
    int32_t* o_en = dalloc<int32_t>(cen, cap);
    if (!o_s || !o_d || !o_st || !o_en) return cleanup(fail(TGXD_ERR_CUDA, "allocation (compact)"));
    if (m) compact_edges<<<gb, 256, 0, s>>>(ds, dd, dst_, den, fl, pos, m, o_s, o_d, o_st, o_en);
    std::swap(bs.p, cs.p);
    std::swap(bs.bytes, cs.bytes);
    std::swap(bd.p, cd.p);
    std::swap(bd.bytes, cd.bytes);
    std::swap(bst.p, cst.p);
    std::swap(bst.bytes, cst.bytes);
    std::swap(ben.p, cen.p);
    std::swap(ben.bytes, cen.bytes);
    ds = bs.as<uint32_t>();
    dd = bd.as<uint32_t>();
    dst_ = bst.as<int32_t>();
    den = ben.as<int32_t>();
    mm = kept;
    G->m_logical = kept;
  }
  if (!directed) {
    const uint64_t m0 = mm;
    if (m0) non_loop_flags<<<grid_for(m0, G->sm_count), 256, 0, s>>>(ds, dd, m0, fl);
    GEN_CUDA(cudaMemsetAsync(fl + m0, 0, 4, s));
    size_t t2 = tb;
    GEN_CUDA(cub::DeviceScan::ExclusiveSum(temp.p, t2, fl, pos, (int64_t)m0 + 1, s));
    uint32_t extra = 0;
    GEN_CUDA(cudaMemcpyAsync(&extra, pos + m0, 4, cudaMemcpyDeviceToHost, s));
    GEN_CUDA(cudaStreamSynchronize(s));
    if (m0) append_reverse<<<grid_for(m0, G->sm_count), 256, 0, s>>>(ds, dd, dst_, den, fl, pos, m0);
    mm = m0 + extra;
  }
  bflag.release();
  bpos.release();
  temp.release();
  rc = build_layouts(G, ds, dd, dst_, den, mm);
  if (rc) return cleanup(rc);
  *out = G;
  return TGXD_OK;
#undef GEN_CUDA
}

int tgxd_graph_build(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                     const uint64_t* start, const uint64_t* end, int directed,
                     uint64_t index_cutoff, tgxd_graph** out) {
  return tgxd_graph_build_weighted(n, m, src, dst, start, end, nullptr, directed, index_cutoff,
                                   out);
}

int tgxd_graph_build_weighted(uint32_t n, uint64_t m, const uint32_t* src, const uint32_t* dst,
                              const uint64_t* start, const uint64_t* end, const double* weight,
                              int directed, uint64_t index_cutoff, tgxd_graph** out) {
  if (!out) return fail(TGXD_ERR_ARGUMENT, "null out");
  *out = nullptr;
  if (m && (!src || !dst || !start || !end)) return fail(TGXD_ERR_ARGUMENT, "null edge arrays");
  // Host passes over the m input edges run on up to 16 threads (config 5:
  // 268M edges; one thread took seconds per pass).
  const unsigned nthreads = (unsigned)std::max<uint64_t>(
      1, std::min<uint64_t>({16, std::max(1u, std::thread::hardware_concurrency()), m / 65536 + 1}));
  auto par = [&](auto&& fn) {  // fn(t, lo, hi) over nthreads contiguous ranges
    std::vector<std::thread> th;
    const uint64_t per = (m + nthreads - 1) / nthreads;
    for (unsigned t = 0; t < nthreads; ++t)
      th.emplace_back([&, t] { fn(t, std::min<uint64_t>(m, t * per), std::min<uint64_t>(m, (t + 1) * per)); });
    for (auto& x : th) x.join();
  };
  // compute_meta (types.cpp:29-54): first offending edge, reference wording.
  {
    std::vector<uint64_t> bad(nthreads, UINT64_MAX), far(nthreads, UINT64_MAX);
    par([&](unsigned t, uint64_t lo, uint64_t hi) {
      for (uint64_t i = lo; i < hi; ++i)
        if (src[i] >= n || dst[i] >= n || end[i] < start[i] || end[i] > kTimeLimit63) {
          bad[t] = i;
          break;
        }
      for (uint64_t i = lo; i < hi; ++i)
        if (end[i] > (uint64_t)kTimeMax) {
          far[t] = i;
          break;
        }
    });
    const uint64_t i = *std::min_element(bad.begin(), bad.end());
    if (i != UINT64_MAX) {
      if (src[i] >= n || dst[i] >= n)
        return fail(TGXD_ERR_EDGE, "edge " + std::to_string(i) + ": endpoint (" +
                                       std::to_string(src[i]) + " -> " + std::to_string(dst[i]) +
                                       ") outside vertex range [0, " + std::to_string(n) + ")");
      if (end[i] < start[i])
        return fail(TGXD_ERR_EDGE, "edge " + std::to_string(i) + ": end " +
                                       std::to_string(end[i]) + " precedes start " +
                                       std::to_string(start[i]));
      return fail(TGXD_ERR_EDGE, "edge " + std::to_string(i) + ": end " + std::to_string(end[i]) +
                                     " beyond the supported time range (2^63 - 1)");
    }
    const uint64_t j = *std::min_element(far.begin(), far.end());
    if (j != UINT64_MAX)
      return fail(TGXD_ERR_TIME_RANGE, "edge " + std::to_string(j) + ": end " +
                                           std::to_string(end[j]) +
                                           " outside the device time domain [0, 2^31 - 2]");
  }
  // undirected graphs add the reverse of every non-loop edge (engine.cpp:13-22),
  // in input order after the originals: per-thread counts give each range's slot
  std::vector<uint64_t> extra(nthreads + 1, 0);
  if (!directed)
    par([&](unsigned t, uint64_t lo, uint64_t hi) {
      uint64_t c = 0;
      for (uint64_t i = lo; i < hi; ++i) c += src[i] != dst[i];
      extra[t + 1] = c;
    });
  for (unsigned t = 0; t < nthreads; ++t) extra[t + 1] += extra[t];
  const uint64_t mm = m + extra[nthreads];
  if (mm >= 0xffffffffULL) return fail(TGXD_ERR_ARGUMENT, "edge count must stay below 2^32");
  std::vector<uint32_t> hs(mm), hd(mm);
  std::vector<int32_t> hst(mm), hen(mm);
  // weights as int64 codes: the value when a non-negative integer below 2^62,
  // -1 when not a non-negative integer (duration_metric's invalid_argument,
  // raised only if a query reaches the edge), -2 when too large
  std::vector<long long> hw(weight ? mm : 0);
  par([&](unsigned t, uint64_t lo, uint64_t hi) {
    uint64_t k = m + extra[t];
    for (uint64_t i = lo; i < hi; ++i) {
      hs[i] = src[i];
      hd[i] = dst[i];
      hst[i] = (int32_t)start[i];
      hen[i] = (int32_t)end[i];
      if (weight) {
        const double x = weight[i], r = std::nearbyint(x);
        hw[i] = (x < 0.0 || r != x) ? -1ll : (r >= 4611686018427387904.0 ? -2ll : (long long)r);
      }
      if (!directed && src[i] != dst[i]) {
        hs[k] = dst[i];
        hd[k] = src[i];
        hst[k] = hst[i];
        hen[k] = hen[i];
        if (weight) hw[k] = hw[i];
        ++k;
      }
    }
  });
  tgxd_graph* G = nullptr;
  int rc = new_graph(n, index_cutoff, directed, &G);
  if (rc) return rc;
  G->m_logical = m;
  DeviceBuffer bs, bd, bst, ben;
  uint32_t* ds = dalloc<uint32_t>(bs, mm);
  uint32_t* dd = dalloc<uint32_t>(bd, mm);
  int32_t* dst_ = dalloc<int32_t>(bst, mm);
  int32_t* den = dalloc<int32_t>(ben, mm);
  cudaError_t e = (ds && dd && dst_ && den) ? cudaSuccess : cudaErrorMemoryAllocation;
  if (e == cudaSuccess && mm) e = cudaMemcpyAsync(ds, hs.data(), mm * 4, cudaMemcpyHostToDevice, G->stream);
  if (e == cudaSuccess && mm) e = cudaMemcpyAsync(dd, hd.data(), mm * 4, cudaMemcpyHostToDevice, G->stream);
  if (e == cudaSuccess && mm) e = cudaMemcpyAsync(dst_, hst.data(), mm * 4, cudaMemcpyHostToDevice, G->stream);
  if (e == cudaSuccess && mm) e = cudaMemcpyAsync(den, hen.data(), mm * 4, cudaMemcpyHostToDevice, G->stream);
  if (e != cudaSuccess) {
    tgxd_graph_destroy(G);
    return fail(TGXD_ERR_CUDA, std::string("edge upload: ") + cudaGetErrorString(e));
  }
  DeviceBuffer bw;
  long long* dw = nullptr;
  if (weight) {
    dw = dalloc<long long>(bw, mm);
    long long* ow = dalloc<long long>(G->out_wbuf, mm);
    if (!dw || !ow ||
        (mm && cudaMemcpyAsync(dw, hw.data(), mm * 8, cudaMemcpyHostToDevice, G->stream) !=
                   cudaSuccess)) {
      tgxd_graph_destroy(G);
      return fail(TGXD_ERR_CUDA, "edge weight upload failed");
    }
    G->out_w = ow;
  }
  rc = build_layouts(G, ds, dd, dst_, den, mm, dw, G->out_wbuf.as<long long>());
  if (rc) {
    tgxd_graph_destroy(G);
    return rc;
  }
  *out = G;
  return TGXD_OK;
}

void tgxd_graph_destroy(tgxd_graph* g) {
  if (!g) return;
  cudaSetDevice(g->device);
  if (g->stream) cudaStreamSynchronize(g->stream);
  for (auto& e : g->ws.ev)
    if (e) cudaEventDestroy(e);
  if (g->ws.trace_host) cudaFreeHost(g->ws.trace_host);
  if (g->pinned) cudaFreeHost(g->pinned);
  if (g->patch_host) cudaFreeHost(g->patch_host);
  if (g->copy_flag_host) cudaFreeHost(const_cast<unsigned int*>(g->copy_flag_host));
  if (g->early_ev) cudaEventDestroy(g->early_ev);
  if (g->copy_stream) cudaStreamDestroy(g->copy_stream);
  for (auto& e : g->chunk_ev)
    if (e) cudaEventDestroy(e);
  if (g->stream) cudaStreamDestroy(g->stream);
  delete g;
}

int tgxd_graph_view(tgxd_graph* g, int share, tgxd_graph** out) {
  if (!g || !out) return fail(TGXD_ERR_ARGUMENT, "null argument");
  if (share < 1 || share > 16) return fail(TGXD_ERR_ARGUMENT, "share must lie in [1, 16]");
  if (g->parent) return fail(TGXD_ERR_ARGUMENT, "a view of a view: use the owning handle");
  *out = nullptr;
  TGXD_CUDA(cudaSetDevice(g->device));
  tgxd_graph* v = nullptr;
  int rc = new_graph(g->n, g->index_cutoff, g->directed, &v);
  if (rc) return rc;
  v->m_logical = g->m_logical;
  v->m = g->m;
  v->indexed[0] = g->indexed[0];
  v->indexed[1] = g->indexed[1];
  v->out = g->out;  // the device graph is the parent's: no buffers owned here
  v->in = g->in;
  v->out_w = g->out_w;
  v->parent = g;
  v->share = share;
  // grids sized so `share` views fit on the GPU side by side
  auto div = [&](int blocks) { return std::max(1, blocks / v->sm_count / share) * v->sm_count; };
  v->coop_blocks = div(v->coop_blocks);
  v->coop_blocks_async = div(v->coop_blocks_async);
  v->coop_blocks_edge = div(v->coop_blocks_edge);
  v->coop_blocks_sd = div(v->coop_blocks_sd);
  v->coop_blocks_lanes = div(v->coop_blocks_lanes);
  v->tail_per_sm = std::max(1, std::min(v->tail_per_sm, v->coop_blocks / v->sm_count));
  *out = v;
  return TGXD_OK;
}

int tgxd_graph_info(const tgxd_graph* g, uint32_t* n, uint64_t* m, uint64_t* indexed_out,
                    uint64_t* indexed_in) {
  if (!g) return fail(TGXD_ERR_ARGUMENT, "null graph");
  if (n) *n = g->n;
  if (m) *m = g->m;
  if (indexed_out) *indexed_out = g->indexed[0];
  if (indexed_in) *indexed_in = g->indexed[1];
  return TGXD_OK;
}

int tgxd_graph_degrees(tgxd_graph* g, int direction, uint32_t* out) {
  if (!g || !out) return fail(TGXD_ERR_ARGUMENT, "null argument");
  std::lock_guard<std::mutex> lock(g->mu);
  TGXD_CUDA(cudaSetDevice(g->device));
  const DevCsr& c = direction == 0 ? g->out : g->in;
  DeviceBuffer b;
  uint32_t* d = dalloc<uint32_t>(b, g->n);
  if (!d) return fail(TGXD_ERR_CUDA, "allocation");
  if (g->n) degrees_kernel<<<grid_for(g->n, g->sm_count), 256, 0, g->stream>>>(c.off, g->n, d);
  TGXD_CUDA(cudaMemcpyAsync(out, d, g->n * 4ull, cudaMemcpyDeviceToHost, g->stream));
  TGXD_CUDA(cudaStreamSynchronize(g->stream));
  return TGXD_OK;
}

// Histograms of the indexed vertices of one direction (costmodel.cuh).
static int ensure_hist(tgxd_graph* g, int dir) {
  tgxd_graph::Hist& H = g->hist[dir];
  if (H.built) return TGXD_OK;
  const DevCsr& c = dir == 0 ? g->out : g->in;
  std::vector<uint32_t> off((size_t)g->n + 1);
  TGXD_CUDA(cudaMemcpyAsync(off.data(), c.off, off.size() * 4, cudaMemcpyDeviceToHost, g->stream));
  TGXD_CUDA(cudaStreamSynchronize(g->stream));
  // VertexIndexRegistry::build (selective_index.cpp:153-186): degree >= cutoff, ascending ids
  std::vector<uint32_t> ids, slot(g->n, kNoSlot);
  for (uint32_t v = 0; v < g->n; ++v)
    if ((uint64_t)(off[v + 1] - off[v]) >= g->index_cutoff) {
      slot[v] = (uint32_t)ids.size();
      ids.push_back(v);
    }
  const size_t K = ids.size();
  if (!dalloc<uint32_t>(H.ids, std::max<size_t>(K, 1)) || !dalloc<uint32_t>(H.slot, g->n) ||
      !dalloc<HistHdr>(H.hdr, std::max<size_t>(K, 1)) ||
      !dalloc<uint32_t>(H.counts, std::max<size_t>(K, 1) * kHistB * kHistB) ||
      !dalloc<unsigned long long>(H.rows, std::max<size_t>(K, 1) * kHistB))
    return fail(TGXD_ERR_CUDA, "device allocation failed (density histograms)");
  if (K)
    TGXD_CUDA(cudaMemcpyAsync(H.ids.p, ids.data(), K * 4, cudaMemcpyHostToDevice, g->stream));
  if (g->n)
    TGXD_CUDA(cudaMemcpyAsync(H.slot.p, slot.data(), (size_t)g->n * 4, cudaMemcpyHostToDevice,
                              g->stream));
  const int smem = kHistB * kHistB * 4;
  TGXD_CUDA(cudaFuncSetAttribute(hist_build_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 smem));
  if (K)
    hist_build_kernel<<<(unsigned)K, 256, smem, g->stream>>>(
        c, dir, H.ids.as<uint32_t>(), H.hdr.as<HistHdr>(), H.counts.as<uint32_t>(),
        H.rows.as<unsigned long long>());
  TGXD_CUDA(cudaGetLastError());
  TGXD_CUDA(cudaStreamSynchronize(g->stream));
  H.count = (uint32_t)K;
  H.built = true;
  return TGXD_OK;
}

int tgxd_access_decisions(tgxd_graph* g, int direction, uint32_t k, const uint32_t* vertices,
                          const uint64_t* t_a, const uint64_t* t_b, double theta_sel,
                          int32_t* method, double* beta_hat, double* k_hat, uint64_t* matches) {
  if (!g) return fail(TGXD_ERR_ARGUMENT, "null graph");
  if (direction != 0 && direction != 1) return fail(TGXD_ERR_ARGUMENT, "direction must be 0 or 1");
  if (k == 0) return TGXD_OK;
  if (!vertices || !t_a || !t_b || !method || !beta_hat || !k_hat || !matches)
    return fail(TGXD_ERR_ARGUMENT, "null argument");
  for (uint32_t i = 0; i < k; ++i)
    if (vertices[i] >= g->n) {
      char msg[128];
      snprintf(msg, sizeof msg, "vertex %u outside vertex range [0, %u)", vertices[i], g->n);
      return fail(TGXD_ERR_VERTEX_RANGE, msg);
    }
  std::lock_guard<std::mutex> lock(g->mu);
  TGXD_CUDA(cudaSetDevice(g->device));
  int rc = ensure_hist(g, direction);
  if (rc) return rc;
  const tgxd_graph::Hist& H = g->hist[direction];
  const DevCsr& c = direction == 0 ? g->out : g->in;
  // vertices (padded to 8), windows, beta, k_hat, matches, method: 56 bytes per query
  DeviceBuffer b;
  char* d = dalloc<char>(b, (size_t)k * 56 + 64);
  if (!d) return fail(TGXD_ERR_CUDA, "allocation");
  uint32_t* dv = reinterpret_cast<uint32_t*>(d);
  unsigned long long* dta = reinterpret_cast<unsigned long long*>(d + (size_t)k * 8);
  unsigned long long* dtb = dta + k;
  double* dbeta = reinterpret_cast<double*>(dtb + k);
  double* dkh = dbeta + k;
  unsigned long long* dm = reinterpret_cast<unsigned long long*>(dkh + k);
  int32_t* dmeth = reinterpret_cast<int32_t*>(dm + k);
  cudaStream_t s = g->stream;
  TGXD_CUDA(cudaMemcpyAsync(dv, vertices, (size_t)k * 4, cudaMemcpyHostToDevice, s));
  TGXD_CUDA(cudaMemcpyAsync(dta, t_a, (size_t)k * 8, cudaMemcpyHostToDevice, s));
  TGXD_CUDA(cudaMemcpyAsync(dtb, t_b, (size_t)k * 8, cudaMemcpyHostToDevice, s));
  access_decision_kernel<<<grid_for((uint64_t)k * 32, g->sm_count), 256, 0, s>>>(
      c, direction, k, dv, dta, dtb, theta_sel, H.slot.as<uint32_t>(), H.hdr.as<HistHdr>(),
      H.counts.as<uint32_t>(), H.rows.as<unsigned long long>(), dmeth, dbeta, dkh, dm);
  TGXD_CUDA(cudaGetLastError());
  TGXD_CUDA(cudaMemcpyAsync(method, dmeth, (size_t)k * 4, cudaMemcpyDeviceToHost, s));
  TGXD_CUDA(cudaMemcpyAsync(beta_hat, dbeta, (size_t)k * 8, cudaMemcpyDeviceToHost, s));
  TGXD_CUDA(cudaMemcpyAsync(k_hat, dkh, (size_t)k * 8, cudaMemcpyDeviceToHost, s));
  TGXD_CUDA(cudaMemcpyAsync(matches, dm, (size_t)k * 8, cudaMemcpyDeviceToHost, s));
  TGXD_CUDA(cudaStreamSynchronize(s));
  return TGXD_OK;
}

// fit_cost_constants (selective_index.cpp:211-235), the same host arithmetic.
int tgxd_fit_cost_constants(uint64_t k, const uint64_t* degree, const uint64_t* matches,
                            const double* index_seconds, const double* scan_seconds, double* c,
                            double* c_prime) {
  if (k == 0) return fail(TGXD_ERR_WINDOW, "cost calibration needs a nonempty sample");
  if (!degree || !matches || !index_seconds || !scan_seconds || !c || !c_prime)
    return fail(TGXD_ERR_ARGUMENT, "null argument");
  double num_c = 0.0, den_c = 0.0, num_cp = 0.0, den_cp = 0.0;
  for (uint64_t i = 0; i < k; ++i) {
    if (degree[i] == 0) continue;
    const double x = std::log2(static_cast<double>(degree[i])) + static_cast<double>(matches[i]);
    num_c += index_seconds[i] * x;
    den_c += x * x;
    const double y = static_cast<double>(degree[i]);
    num_cp += scan_seconds[i] * y;
    den_cp += y * y;
  }
  if (den_c == 0.0 || den_cp == 0.0)
    return fail(TGXD_ERR_WINDOW, "cost calibration needs samples with degree >= 1");
  *c = num_c / den_c;
  *c_prime = num_cp / den_cp;
  return TGXD_OK;
}

int tgxd_graph_flatten(tgxd_graph* g, int direction, uint32_t* src, uint32_t* dst,
                       uint64_t* start, uint64_t* end) {
  if (!g || !src || !dst || !start || !end) return fail(TGXD_ERR_ARGUMENT, "null argument");
  std::lock_guard<std::mutex> lock(g->mu);
  TGXD_CUDA(cudaSetDevice(g->device));
  const DevCsr& c = direction == 0 ? g->out : g->in;
  const uint64_t m = g->m;
  DeviceBuffer b;
  uint32_t* own = dalloc<uint32_t>(b, m);
  if (!own) return fail(TGXD_ERR_CUDA, "allocation");
  if (g->n) owners_kernel<<<grid_for(g->n, g->sm_count), 256, 0, g->stream>>>(c.off, g->n, own);
  std::vector<uint32_t> o(m), nb(m);
  std::vector<int32_t> k(m), v(m);
  std::vector<uint2> pay(m);
  if (m) {
    TGXD_CUDA(cudaMemcpyAsync(o.data(), own, m * 4, cudaMemcpyDeviceToHost, g->stream));
    TGXD_CUDA(cudaMemcpyAsync(k.data(), c.key, m * 4, cudaMemcpyDeviceToHost, g->stream));
    TGXD_CUDA(cudaMemcpyAsync(pay.data(), c.pay, m * 8, cudaMemcpyDeviceToHost, g->stream));
  }
  TGXD_CUDA(cudaStreamSynchronize(g->stream));
  for (uint64_t i = 0; i < m; ++i) {
    nb[i] = pay[i].x;
    v[i] = (int32_t)pay[i].y;
  }
  for (uint64_t i = 0; i < m; ++i) {
    if (direction == 0) {
      src[i] = o[i];
      dst[i] = nb[i];
      start[i] = (uint64_t)k[i];
      end[i] = (uint64_t)v[i];
    } else {
      src[i] = nb[i];
      dst[i] = o[i];
      start[i] = (uint64_t)(-(int64_t)v[i]);
      end[i] = (uint64_t)(-(int64_t)k[i]);
    }
  }
  return TGXD_OK;
}

int tgxd_query(tgxd_graph* g, int kind, uint32_t k, const uint32_t* vertices, const uint64_t* t_a,
               const uint64_t* t_b, int ordering, int mode, void* out, int width,
               int out_on_device, tgxd_stats* stats) {
  return query_impl(g, kind, k, vertices, t_a, t_b, ordering, mode, out, width, out_on_device,
                    stats);
}

int tgxd_earliest_arrival(tgxd_graph* g, uint32_t source, uint64_t t_a, uint64_t t_b,
                          int ordering, int64_t* out, tgxd_stats* stats) {
  return query_impl(g, TGXD_EARLIEST_ARRIVAL, 1, &source, &t_a, &t_b, ordering, TGXD_MODE_AUTO,
                    out, 8, 0, stats);
}

int tgxd_latest_departure(tgxd_graph* g, uint32_t target, uint64_t t_a, uint64_t t_b,
                          int ordering, int64_t* out, tgxd_stats* stats) {
  return query_impl(g, TGXD_LATEST_DEPARTURE, 1, &target, &t_a, &t_b, ordering, TGXD_MODE_AUTO,
                    out, 8, 0, stats);
}

int tgxd_fastest(tgxd_graph* g, uint32_t source, uint64_t t_a, uint64_t t_b, int ordering,
                 int64_t* out, tgxd_stats* stats) {
  return query_impl(g, TGXD_FASTEST, 1, &source, &t_a, &t_b, ordering, TGXD_MODE_AUTO, out, 8, 0,
                    stats);
}

int tgxd_shortest_duration(tgxd_graph* g, uint32_t source, uint64_t t_a, uint64_t t_b,
                           int ordering, int64_t* out, tgxd_stats* stats) {
  return query_impl(g, TGXD_SHORTEST_DURATION, 1, &source, &t_a, &t_b, ordering, TGXD_MODE_AUTO,
                    out, 8, 0, stats);
}

int tgxd_shortest_duration_weighted(tgxd_graph* g, uint32_t source, uint64_t t_a, uint64_t t_b,
                                    int ordering, int64_t* out, tgxd_stats* stats) {
  return query_impl(g, TGXD_SHORTEST_DURATION_WEIGHTED, 1, &source, &t_a, &t_b, ordering,
                    TGXD_MODE_AUTO, out, 8, 0, stats);
}

int tgxd_temporal_bfs(tgxd_graph* g, uint32_t source, uint64_t t_a, uint64_t t_b, int ordering,
                      int64_t* out, tgxd_stats* stats) {
  return query_impl(g, TGXD_TEMPORAL_BFS, 1, &source, &t_a, &t_b, ordering, TGXD_MODE_AUTO, out,
                    8, 0, stats);
}

int tgxd_last_d2h_bytes(tgxd_graph* g, uint64_t* bytes) {
  if (!g || !bytes) return fail(TGXD_ERR_ARGUMENT, "null argument");
  std::lock_guard<std::mutex> lock(g->mu);
  *bytes = g->ws.last_d2h;
  return TGXD_OK;
}

#ifdef TGXD_EXPERIMENTS
// Experiment (tools/x_relax.py): runs an EA query whose round kernel stops
// before round `round`'s relax (TGXD_X_STOP_A), then times that relax as
// relax_only_kernel with `upw` units per warp. out: {ms, chunks, smalls, push}.
extern "C" int tgxd_x_relax(tgxd_graph* G, uint32_t src, uint32_t round, uint32_t upw,
                            double* out) {
  std::lock_guard<std::mutex> lock(G->mu);
  TGXD_CUDA(cudaSetDevice(G->device));
  const uint64_t ta = 0, tb = 999999;
  Prepared P;
  int rc = prepare(G, TGXD_EARLIEST_ARRIVAL, 1, &src, &ta, &tb, 1, P);
  if (rc) return rc;
  if ((rc = ensure_workspace(G, 1, false))) return rc;
  setenv("TGXD_X_STOP_A", std::to_string(round).c_str(), 1);
  setenv("TGXD_HANDOFF_F", "0", 1);
  setenv("TGXD_ASYNC_F", "0", 1);
  rc = launch(G, P, TGXD_MODE_AUTO, nullptr, 4, nullptr, nullptr);
  unsetenv("TGXD_X_STOP_A");
  unsetenv("TGXD_HANDOFF_F");
  unsetenv("TGXD_ASYNC_F");
  if (rc) return rc;
  Workspace& w = G->ws;
  Control c;
  TGXD_CUDA(cudaMemcpyAsync(&c, w.ctl.p, sizeof c, cudaMemcpyDeviceToHost, G->stream));
  TGXD_CUDA(cudaStreamSynchronize(G->stream));
  const unsigned long long nch = c.state[0], nsm = c.state[1], pstart = c.state[2];
  const int flip = (int)c.state[3], push = (int)c.state[4];
  TravArgs a;
  std::memset(&a, 0, sizeof a);
  a.g = G->out;
  a.qp = w.params.as<QueryParam>();
  a.X = w.X.as<int32_t>();
  a.EP = w.EP.as<int2>();
  a.chunks = w.chunks.as<uint2>();
  a.smalls = w.smalls.as<uint2>();
  a.ctl = w.ctl.as<Control>();
  a.n = G->n;
  a.Q = 1;
  a.strict = P.strict;
  a.fresh = 0x80000000u;
  const unsigned long long units = nch + (nsm + 31) / 32;
  const unsigned long long warps = (units + upw - 1) / upw;
  const unsigned blocks = (unsigned)std::max<unsigned long long>(1, (warps + kWarps - 1) / kWarps);
  uint32_t* fout = flip ? w.fa.as<uint32_t>() : w.fb.as<uint32_t>();
  TGXD_CUDA(cudaEventRecord(w.ev[0], G->stream));
  relax_only_kernel<<<blocks, kThreads, 0, G->stream>>>(a, nch, nsm, pstart, fout, push, upw);
  TGXD_CUDA(cudaEventRecord(w.ev[1], G->stream));
  TGXD_CUDA(cudaStreamSynchronize(G->stream));
  TGXD_CUDA(cudaGetLastError());
  float ms = 0;
  TGXD_CUDA(cudaEventElapsedTime(&ms, w.ev[0], w.ev[1]));
  out[0] = ms;
  out[1] = (double)nch;
  out[2] = (double)nsm;
  out[3] = push;
  w.xinv = false;  // the labels are a partial traversal's: the next query initializes
  return TGXD_OK;
}
#endif

int tgxd_launch_count(tgxd_graph* g, uint64_t* count) {
  if (!g || !count) return fail(TGXD_ERR_ARGUMENT, "null argument");
  std::lock_guard<std::mutex> lock(g->mu);
  *count = g->ws.launches;
  return TGXD_OK;
}

int tgxd_last_h2d_bytes(tgxd_graph* g, uint64_t* bytes) {
  if (!g || !bytes) return fail(TGXD_ERR_ARGUMENT, "null argument");
  std::lock_guard<std::mutex> lock(g->mu);
  *bytes = g->ws.last_h2d;
  return TGXD_OK;
}

int tgxd_last_work(tgxd_graph* g, uint32_t q, uint64_t* e_adm, uint64_t* v_reached) {
  if (!g || !e_adm || !v_reached) return fail(TGXD_ERR_ARGUMENT, "null argument");
  std::lock_guard<std::mutex> lock(g->mu);
  Workspace& w = g->ws;
  if (w.last_kind < 0 || q >= w.last_q) return fail(TGXD_ERR_ARGUMENT, "no such query slot");
  if (w.last_edge)
    return fail(TGXD_ERR_UNSUPPORTED, "the unit of work is defined for vertex-label traversals");
  TGXD_CUDA(cudaSetDevice(g->device));
  const DevCsr& c = w.last_kind == TGXD_LATEST_DEPARTURE ? g->in : g->out;
  DeviceBuffer acc;
  unsigned long long* d = dalloc<unsigned long long>(acc, 2);
  if (!d) return fail(TGXD_ERR_CUDA, "allocation");
  TGXD_CUDA(cudaMemsetAsync(d, 0, 16, g->stream));
  work_kernel<<<g->sm_count * 8, 256, 0, g->stream>>>(
      c, w.X.as<int32_t>() + (size_t)q * g->n, w.last_params[q], w.last_strict, d);
  unsigned long long h[2];
  TGXD_CUDA(cudaMemcpyAsync(h, d, 16, cudaMemcpyDeviceToHost, g->stream));
  TGXD_CUDA(cudaStreamSynchronize(g->stream));
  *e_adm = h[0];
  *v_reached = h[1];
  return TGXD_OK;
}

// Device time of `steps` launches after `warmup` untimed ones, outputs in
// HBM. rotate = false: every step is the whole k-query batch; rotate =
// true: step i is the single query i mod k (parameters uploaded per step).
static int time_impl(tgxd_graph* g, int kind, uint32_t k, const uint32_t* vertices,
                     const uint64_t* t_a, const uint64_t* t_b, int ordering, int mode, int warmup,
                     int steps, bool rotate, float* total_ms, float* kernel_ms) {
  if (!g || !total_ms || !kernel_ms || steps < 1 || warmup < 0 || k == 0 || !vertices || !t_a ||
      !t_b)
    return fail(TGXD_ERR_ARGUMENT, "bad timing arguments");
  if (kind == TGXD_FASTEST && k != 1 && !rotate)
    return fail(TGXD_ERR_ARGUMENT, "timed fastest: one source");
  std::lock_guard<std::mutex> lock(g->mu);
  TGXD_CUDA(cudaSetDevice(g->device));
  uint32_t group = 0;
  int rc = rotate ? TGXD_OK : split_group(g, kind, k, t_a, t_b, mode, true, &group);
  if (rc) return rc;
  // rotate: one Prepared per query, step i runs query i mod k; a split batch:
  // one per group, every step runs all groups; else one for the whole batch
  const uint32_t np = rotate ? k : (group ? (k + group - 1) / group : 1);
  const uint32_t per_step = rotate ? 1 : np;
  std::vector<Prepared> Ps(np);
  uint32_t qmax = 1;
  for (uint32_t i = 0; i < np; ++i) {
    Prepared& P = Ps[i];
    const uint32_t q0 = rotate ? i : i * (group ? group : k);
    const uint32_t kq = rotate ? 1 : std::min(group ? group : k, k - q0);
    rc = prepare(g, kind, kq, vertices + q0, t_a + q0, t_b + q0, ordering, P);
    if (rc) return rc;
    qmax = std::max(qmax, P.Q);
  }
  rc = ensure_workspace(g, qmax, kind == TGXD_FASTEST || kind == TGXD_TEMPORAL_BFS);
  if (rc) return rc;
  Workspace& w = g->ws;
  const uint64_t slots = (uint64_t)qmax * g->n;
  if (!dalloc<int32_t>(w.timing_out, slots)) return fail(TGXD_ERR_CUDA, "allocation (output)");
  std::vector<cudaEvent_t> ev(2 * (size_t)steps);
  for (auto& e : ev) TGXD_CUDA(cudaEventCreate(&e));
  auto destroy = [&] {
    for (auto& e : ev) cudaEventDestroy(e);
  };
  for (int i = 0; i < warmup; ++i)
    for (uint32_t j = 0; j < per_step; ++j)
      if ((rc = launch(g, Ps[(i * per_step + j) % np], mode, w.timing_out.p, 4, nullptr, nullptr)))
        return destroy(), rc;
  TGXD_CUDA(cudaEventRecord(w.ev[2], g->stream));
  for (int i = 0; i < steps; ++i)
    for (uint32_t j = 0; j < per_step; ++j)
      if ((rc = launch(g, Ps[(i * per_step + j) % np], mode, w.timing_out.p, 4,
                       j == 0 ? ev[2 * i] : nullptr, j + 1 == per_step ? ev[2 * i + 1] : nullptr)))
        return destroy(), rc;
  TGXD_CUDA(cudaEventRecord(w.ev[3], g->stream));
  TGXD_CUDA(cudaStreamSynchronize(g->stream));
  float tot = 0, ksum = 0;
  TGXD_CUDA(cudaEventElapsedTime(&tot, w.ev[2], w.ev[3]));
  for (int i = 0; i < steps; ++i) {
    float x = 0;
    TGXD_CUDA(cudaEventElapsedTime(&x, ev[2 * i], ev[2 * i + 1]));
    ksum += x;
  }
  destroy();
  *total_ms = tot;
  *kernel_ms = ksum / steps;
  return read_stats(g, nullptr, 0, 0);
}

int tgxd_time_queries(tgxd_graph* g, int kind, uint32_t k, const uint32_t* vertices,
                      const uint64_t* t_a, const uint64_t* t_b, int ordering, int mode, int warmup,
                      int steps, float* total_ms, float* kernel_ms) {
  return time_impl(g, kind, k, vertices, t_a, t_b, ordering, mode, warmup, steps, false, total_ms,
                   kernel_ms);
}

int tgxd_time_rotation(tgxd_graph* g, int kind, uint32_t k, const uint32_t* vertices,
                       const uint64_t* t_a, const uint64_t* t_b, int ordering, int mode,
                       int warmup, int steps, float* total_ms, float* kernel_ms) {
  return time_impl(g, kind, k, vertices, t_a, t_b, ordering, mode, warmup, steps, true, total_ms,
                   kernel_ms);
}

// The trace lives in mapped pinned host memory: the device writes it
// directly, so it stays readable even while a traversal is still running.
int tgxd_set_trace(tgxd_graph* g, uint32_t max_rounds) {
  if (!g) return fail(TGXD_ERR_ARGUMENT, "null graph");
  std::lock_guard<std::mutex> lock(g->mu);
  TGXD_CUDA(cudaSetDevice(g->device));
  if (g->ws.trace_host) {
    cudaFreeHost(g->ws.trace_host);
    g->ws.trace_host = nullptr;
  }
  g->ws.trace_cap = 0;
  g->ws.trace_dev = nullptr;
  if (max_rounds) {
    void* h = nullptr;
    TGXD_CUDA(cudaHostAlloc(&h, max_rounds * 64ull, cudaHostAllocMapped));
    std::memset(h, 0, max_rounds * 64ull);
    void* d = nullptr;
    TGXD_CUDA(cudaHostGetDevicePointer(&d, h, 0));
    g->ws.trace_host = static_cast<unsigned long long*>(h);
    g->ws.trace_dev = static_cast<unsigned long long*>(d);
    g->ws.trace_cap = max_rounds;
    if (!dalloc<unsigned long long>(g->ws.wtrace, max_rounds * 4ull))
      return fail(TGXD_ERR_CUDA, "allocation (trace)");
  }
  return TGXD_OK;
}

// Rows of 12 u64: the 8 block-0 fields (read from mapped host memory, no
// lock: usable while a query is still running) and the 4 per-warp phase
// extremes (device memory; copied only when `with_device` is set).
int tgxd_get_trace(tgxd_graph* g, uint64_t* out, uint32_t max_rounds, int with_device) {
  if (!g || !out) return fail(TGXD_ERR_ARGUMENT, "null argument");
#ifdef TGXD_CHAIN
  if (const char* path = getenv("TGXD_CHAIN_FILE")) {  // diagnostics: block 0 / warp 0 chain marks
    std::vector<unsigned long long> all(sizeof(g_chain) / 8);
    TGXD_CUDA(cudaMemcpyFromSymbol(all.data(), g_chain, sizeof(g_chain)));
    if (FILE* f = fopen(path, "wb")) {
      fwrite(all.data(), 8, all.size(), f);
      fclose(f);
    }
  }
#endif
#ifdef TGXD_WTRACE_ALL
  if (const char* path = getenv("TGXD_WTRACE_ALL_FILE")) {  // diagnostics: every warp's times
    std::vector<unsigned long long> all(sizeof(g_wdone) / 8);
    TGXD_CUDA(cudaMemcpyFromSymbol(all.data(), g_wdone, sizeof(g_wdone)));
    if (FILE* f = fopen(path, "wb")) {
      fwrite(all.data(), 8, all.size(), f);
      fclose(f);
    }
  }
#endif
  const uint32_t r = std::min(max_rounds, g->ws.trace_cap);
  volatile unsigned long long* src = g->ws.trace_host;
  std::vector<unsigned long long> wt(r * 4ull, 0);
  if (with_device && r) {
    TGXD_CUDA(cudaMemcpy(wt.data(), g->ws.wtrace.p, r * 32ull, cudaMemcpyDeviceToHost));
  }
  for (uint64_t i = 0; i < r; ++i) {
    for (int j = 0; j < 8; ++j) out[i * 12 + j] = src[i * 8 + j];
    for (int j = 0; j < 4; ++j) out[i * 12 + 8 + j] = wt[i * 4 + j];
  }
  return TGXD_OK;
}

uint64_t tgxd_digest(const int64_t* values, uint64_t n) {
  uint64_t h = 0xcbf29ce484222325ULL;
  const unsigned char* p = reinterpret_cast<const unsigned char*>(values);
  for (uint64_t i = 0; i < n * 8; ++i) {
    h ^= p[i];
    h *= 0x100000001b3ULL;
  }
  return h;
}

}  // extern "C"
