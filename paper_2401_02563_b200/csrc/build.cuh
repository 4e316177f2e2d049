// Device T-CSR build (TemporalCsr::build, tcsr.cpp:19-84; TemporalGraph::build,
// engine.cpp:7-34) and the device edge generator.
//
// Each layout is one stable radix sort of 64-bit (owner << 32 | key) keys
// carrying the edge index, followed by a gather into the SoA arrays, a
// degree histogram + exclusive scan for the offsets, and the fence array of
// the selective index. The stable sort keeps equal (owner, key) edges in
// input order, so a layout is a deterministic function of the edge list.
#pragma once

#include <cub/device/device_radix_sort.cuh>
#include <cub/device/device_scan.cuh>

#include "gen.cuh"
#include "tgxd_internal.cuh"

namespace tgxd {

__global__ void gen_kernel(GenParams p, const uint64_t* thr, uint64_t m, uint32_t* src,
                           uint32_t* dst, int32_t* st, int32_t* en) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const GenEdge e = gen_edge(p, thr, i);
    src[i] = e.src;
    dst[i] = e.dst;
    st[i] = e.start;
    en[i] = e.end;
  }
}

// flags[i] = (src != dst); used to drop self-loops (uniform configs) and to
// count the reversed copies of an undirected graph.
__global__ void non_loop_flags(const uint32_t* src, const uint32_t* dst, uint64_t m,
                               uint32_t* flags) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride)
    flags[i] = src[i] != dst[i] ? 1u : 0u;
}

// Stable compaction of non-self-loop edges: out[pos[i]] = in[i] where flag.
__global__ void compact_edges(const uint32_t* src, const uint32_t* dst, const int32_t* st,
                              const int32_t* en, const uint32_t* flags, const uint32_t* pos,
                              uint64_t m, uint32_t* o_src, uint32_t* o_dst, int32_t* o_st,
                              int32_t* o_en) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    if (!flags[i]) continue;
    const uint32_t j = pos[i];
    o_src[j] = src[i];
    o_dst[j] = dst[i];
    o_st[j] = st[i];
    o_en[j] = en[i];
  }
}

// Undirected materialization (engine.cpp:13-22): the reverse of every
// non-self-loop edge is appended after the original m edges, in input order.
__global__ void append_reverse(uint32_t* src, uint32_t* dst, int32_t* st, int32_t* en,
                               const uint32_t* flags, const uint32_t* pos, uint64_t m) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    if (!flags[i]) continue;
    const uint64_t j = m + pos[i];
    src[j] = dst[i];
    dst[j] = src[i];
    st[j] = st[i];
    en[j] = en[i];
  }
}

__device__ __forceinline__ uint32_t key_bits(int32_t k) { return (uint32_t)k ^ 0x80000000u; }

// Sort keys of one layout. Out: owner = src, key = start. In: owner = dst,
// key = -end (segments by end descending, the latest-departure mirror).
__global__ void make_sort_keys(const uint32_t* owner, const int32_t* kk, int negate, uint64_t m,
                               unsigned long long* keys, uint32_t* idx) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const int32_t k = negate ? -kk[i] : kk[i];
    keys[i] = ((unsigned long long)owner[i] << 32) | key_bits(k);
    idx[i] = (uint32_t)i;
  }
}

// Sort keys and their payloads {other, val} as one 64-bit value (the sort
// moves the payload: no random gathers afterwards; used without weights).
__global__ void make_sort_kv(const uint32_t* owner, const uint32_t* other, const int32_t* kk,
                             const int32_t* vv, int negate, uint64_t m, unsigned long long* keys,
                             unsigned long long* vals) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride) {
    const int32_t k = negate ? -kk[i] : kk[i];
    keys[i] = ((unsigned long long)owner[i] << 32) | key_bits(k);
    const uint32_t v = (uint32_t)(negate ? -vv[i] : vv[i]);
    vals[i] = ((unsigned long long)v << 32) | other[i];  // = uint2 {other, val}
  }
}

// The layout's keys from the sorted sort keys.
__global__ void keys_from_sorted(const unsigned long long* keys, uint64_t m, int32_t* key) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += stride)
    key[j] = (int32_t)((uint32_t)keys[j] ^ 0x80000000u);
}

__global__ void gather_layout(const uint32_t* idx, const uint32_t* other, const int32_t* kk,
                              const int32_t* vv, int negate, uint64_t m, int32_t* key,
                              uint2* pay) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < m; j += stride) {
    const uint32_t i = idx[j];
    key[j] = negate ? -kk[i] : kk[i];
    pay[j] = make_uint2(other[i], (uint32_t)(negate ? -vv[i] : vv[i]));
  }
}

__global__ void degree_count(const uint32_t* owner, uint64_t m, uint32_t* cnt) {
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; i < m; i += stride)
    atomicAdd(cnt + owner[i], 1u);
}

__global__ void make_fences(const int32_t* key, uint64_t m, int32_t* fence) {
  const uint64_t nf = (m + kFenceStride - 1) >> kFenceShift;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < nf; j += stride)
    fence[j] = key[j << kFenceShift];
}

// Last key of every segment (the pull side's "any candidate?" test and the
// expansion's "anything at or above the bound?" test without a dependent load).
__global__ void segment_kmax(const uint32_t* off, const int32_t* key, uint32_t n, int32_t* kmax) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride) {
    const uint32_t s = off[v], t = off[v + 1];
    kmax[v] = t > s ? key[t - 1] : INT32_MIN;
  }
}

__global__ void make_okm(const uint32_t* off, const int32_t* kmax, uint32_t n, uint2* okm) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v <= n; v += stride)
    okm[v] = make_uint2(off[v], v < n ? (uint32_t)kmax[v] : (uint32_t)INT32_MIN);
}

__global__ void count_indexed(const uint32_t* off, uint32_t n, uint64_t cutoff,
                              unsigned long long* out) {
  unsigned long long c = 0;
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride)
    c += (uint64_t)(off[v + 1] - off[v]) >= cutoff;
  for (int o = 16; o > 0; o >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o);
  if ((threadIdx.x & 31) == 0 && c) atomicAdd(out, c);
}

__global__ void degrees_kernel(const uint32_t* off, uint32_t n, uint32_t* deg) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride)
    deg[v] = off[v + 1] - off[v];
}

// Inverse of the layout: owner of every position (for flatten).
__global__ void owners_kernel(const uint32_t* off, uint32_t n, uint32_t* own) {
  const uint32_t stride = gridDim.x * blockDim.x;
  for (uint32_t v = blockIdx.x * blockDim.x + threadIdx.x; v < n; v += stride)
    for (uint32_t j = off[v]; j < off[v + 1]; ++j) own[j] = v;
}

inline int grid_for(uint64_t work, int sms) {
  uint64_t b = (work + 255) / 256;
  const uint64_t cap = (uint64_t)sms * 16;
  if (b > cap) b = cap;
  if (b < 1) b = 1;
  return (int)b;
}

}  // namespace tgxd
