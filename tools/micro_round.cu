// Grid-round overhead microbenchmark: a persistent grid (148 x 4 CTAs x 256
// threads, like traverse_kernel) runs rounds of "W working warps each do D
// dependent random L2 loads + one counter atomic, then a grid barrier, then
// every block reads the counters". Variants of the barrier / counter read:
//   0  one generation word polled by every block (traverse.cuh GridBarrier),
//      then 6 counter loads per block
//   1  as 0 without the counter loads
//   2  generation replicated in 32 records 1 KB apart (block b polls b % 32),
//      6 counter loads per block
//   3  replicated generation + counter snapshot in the record (last arriver
//      copies the counters; blocks read their record)
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/micro_round tools/micro_round.cu
#include <cstdio>
#include <cstdint>
#include <vector>
#include <random>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

struct alignas(128) Ctl {
  unsigned long long ctr[8];
  alignas(128) unsigned int count;
  alignas(128) unsigned int gen;
};

constexpr int kReps = 32, kStride = 128;

template <int V>
__device__ __forceinline__ void barrier(Ctl* c, unsigned long long* rec, unsigned long long& tag,
                                        unsigned long long* snap, unsigned max_ns) {
  __shared__ int s_last;
  __syncthreads();
  const unsigned long long want = tag + 1;
  if (V <= 1) {
    if (threadIdx.x == 0) {
      __threadfence();
      if (atomicAdd(&c->count, 1u) + 1 == gridDim.x) {
        c->count = 0;
        __threadfence();
        asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(&c->gen), "r"((unsigned)want) : "memory");
      } else {
        unsigned ns = 32;
        for (;;) {
          unsigned cur;
          asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(cur) : "l"(&c->gen) : "memory");
          if (cur == (unsigned)want) break;
          __nanosleep(ns);
          if (ns < max_ns) ns <<= 1;
        }
      }
      __threadfence();
      if (V == 0) {
        for (int k = 0; k < 6; ++k) snap[k] = __ldcg(&c->ctr[k]);
      }
    }
  } else if (V == 4) {
    // tagged snapshot words: tag16 << 48 | value48, polled word-per-lane
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = atomicAdd(&c->count, 1u) + 1 == gridDim.x;
    }
    __syncthreads();
    const unsigned long long t16 = (want % 65535ull) + 1;
    if (threadIdx.x < 32) {
      const int lane = threadIdx.x;
      if (s_last) {
        if (lane == 0) c->count = 0;
        __threadfence();
        const unsigned long long v = lane < 6 ? __ldcg(&c->ctr[lane]) : 0ull;
        const unsigned long long w = t16 << 48 | (v & ((1ull << 48) - 1));
        unsigned long long* r = rec + blockIdx.x * 0;  // (placeholder)
        for (int k = 0; k < kReps; ++k) {
          const unsigned long long wk = __shfl_sync(0xffffffffu, w, lane & 7);
          (void)wk;
        }
        // lane l writes word (l % 8) of replicas l/8, l/8 + 4, ...
        const int word = lane & 7;
        const unsigned long long mine = __shfl_sync(0xffffffffu, w, word);
        for (int rr = lane >> 3; rr < kReps; rr += 4)
          asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(rec + rr * kStride + word), "l"(mine) : "memory");
        (void)r;
      }
      const unsigned long long* r = rec + (blockIdx.x % kReps) * kStride;
      unsigned long long cur = 0;
      unsigned ns = 32;
      for (;;) {
        if (lane < 6) asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(cur) : "l"(r + lane) : "memory");
        if (__all_sync(0xffffffffu, lane >= 6 || (cur >> 48) == t16)) break;
        __nanosleep(ns);
        if (ns < max_ns) ns <<= 1;
      }
      __threadfence();
      if (lane < 6) snap[lane] = cur & ((1ull << 48) - 1);
    }
  } else {
    if (threadIdx.x == 0) {
      __threadfence();
      s_last = atomicAdd(&c->count, 1u) + 1 == gridDim.x;
    }
    __syncthreads();
    if (s_last && threadIdx.x < 32) {
      const int lane = threadIdx.x;
      if (lane == 0) c->count = 0;
      __threadfence();
      unsigned long long* r = rec + lane * kStride;
      if (V == 3) {
        unsigned long long v = lane < 6 ? __ldcg(&c->ctr[lane]) : 0ull;
        unsigned long long w[6];
#pragma unroll
        for (int k = 0; k < 6; ++k) w[k] = __shfl_sync(0xffffffffu, v, k);
#pragma unroll
        for (int k = 0; k < 6; k += 2)
          asm volatile("st.global.cg.v2.u64 [%0], {%1, %2};" ::"l"(r + 2 + k), "l"(w[k]), "l"(w[k + 1]) : "memory");
      }
      asm volatile("st.release.gpu.global.u64 [%0], %1;" ::"l"(r), "l"(want) : "memory");
    }
    if (threadIdx.x == 0) {
      const unsigned long long* r = rec + (blockIdx.x % kReps) * kStride;
      unsigned ns = 32;
      for (;;) {
        unsigned long long cur;
        asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(cur) : "l"(r) : "memory");
        if (cur == want) break;
        __nanosleep(ns);
        if (ns < max_ns) ns <<= 1;
      }
      __threadfence();
      if (V == 2) {
        for (int k = 0; k < 6; ++k) snap[k] = __ldcg(&c->ctr[k]);
      } else {
        for (int k = 0; k < 6; ++k) snap[k] = __ldcg(r + 2 + k);
      }
    }
  }
  tag = want;
  __syncthreads();
}

template <int V>
__global__ void __launch_bounds__(256, 4) rounds(const unsigned* __restrict__ nxt, unsigned mask,
                                                 int nrounds, int work_warps, int deps, Ctl* c,
                                                 unsigned long long* rec, unsigned long long tag0,
                                                 unsigned max_ns, unsigned* out) {
  __shared__ unsigned long long snap[8];
  unsigned long long tag = tag0;
  const unsigned gw = blockIdx.x * 8 + (threadIdx.x >> 5);
  const unsigned lane = threadIdx.x & 31;
  unsigned p = (gw * 2654435761u + lane * 40503u) & mask;
  unsigned acc = 0;
  for (int r = 0; r < nrounds; ++r) {
    // spread the working warps over the grid like a frontier of 32-slot groups
    const unsigned stride = (gridDim.x * 8) / (work_warps ? work_warps : 1);
    if (work_warps && gw % (stride ? stride : 1) == 0 && gw / (stride ? stride : 1) < (unsigned)work_warps) {
      for (int d = 0; d < deps; ++d) p = __ldcg(nxt + p) & mask;
      if (lane == 0) atomicAdd(&c->ctr[r % 6], 1ull);
      acc += p;
    }
    barrier<V>(c, rec, tag, snap, max_ns);
    acc += (unsigned)snap[r % 6];
  }
  if (acc == 0x12345678u) out[0] = acc;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int blocks = sms * 4;
  const size_t n = 1 << 22;  // 16 MB chase array (L2 resident)
  std::vector<unsigned> h(n);
  std::mt19937 rng(1);
  for (size_t i = 0; i < n; ++i) h[i] = rng() & (n - 1);
  unsigned* d_nxt;
  Ctl* c;
  unsigned long long* rec;
  unsigned* out;
  CK(cudaMalloc(&d_nxt, n * 4));
  CK(cudaMemcpy(d_nxt, h.data(), n * 4, cudaMemcpyHostToDevice));
  CK(cudaMalloc(&c, sizeof(Ctl)));
  CK(cudaMalloc(&rec, kReps * kStride * 8));
  CK(cudaMalloc(&out, 4));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int nr = 2000;
  for (int deps : {0, 8}) {
    for (int ww : {0, 128}) {
      if (deps == 0 && ww) continue;
      for (unsigned max_ns : {256u, 1024u}) {
        for (int v = 0; v < 5; ++v) {
          float best = 1e9f;
          for (int rep = 0; rep < 3; ++rep) {
            CK(cudaMemset(c, 0, sizeof(Ctl)));
            CK(cudaMemset(rec, 0, kReps * kStride * 8));
            cudaEventRecord(e0);
            const unsigned long long tag0 = 0;
            if (v == 0) rounds<0><<<blocks, 256>>>(d_nxt, n - 1, nr, ww, deps, c, rec, tag0, max_ns, out);
            if (v == 1) rounds<1><<<blocks, 256>>>(d_nxt, n - 1, nr, ww, deps, c, rec, tag0, max_ns, out);
            if (v == 2) rounds<2><<<blocks, 256>>>(d_nxt, n - 1, nr, ww, deps, c, rec, tag0, max_ns, out);
            if (v == 4) rounds<4><<<blocks, 256>>>(d_nxt, n - 1, nr, ww, deps, c, rec, tag0, max_ns, out);
            if (v == 3) rounds<3><<<blocks, 256>>>(d_nxt, n - 1, nr, ww, deps, c, rec, tag0, max_ns, out);
            CK(cudaGetLastError());
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best) best = ms;
          }
          printf("deps=%d work_warps=%3d max_ns=%4u variant %d: %.2f us/round\n", deps, ww, max_ns, v,
                 best * 1e3 / nr);
        }
      }
    }
  }
  // dependent-load latency alone (one warp)
  {
    cudaEventRecord(e0);
    CK(cudaMemset(c, 0, sizeof(Ctl)));
    rounds<1><<<1, 256>>>(d_nxt, n - 1, 1, 1, 20000, c, rec, 0, 256, out);
    CK(cudaGetLastError());
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("one warp, dependent L2 load: %.0f ns\n", ms * 1e6 / 20000);
  }
  return 0;
}
