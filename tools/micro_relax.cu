// Ceiling of the relax step in isolation: stream {nbr, val} payloads of
// 128-edge chunks, probe the label, atomicMin when it improves.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o micro_relax micro_relax.cu
#include <cstdio>
#include <cstdint>
#include <vector>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

template <int U, bool HINT>
__global__ void relax(const uint2* __restrict__ pay, const uint2* __restrict__ chunks, size_t nch,
                      int* X, unsigned long long* imp) {
  const unsigned lane = threadIdx.x & 31;
  const size_t gw = (blockIdx.x * (size_t)blockDim.x + threadIdx.x) >> 5;
  const size_t nw = (gridDim.x * (size_t)blockDim.x) >> 5;
  unsigned long long cnt = 0;
  uint64_t pf, pk;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pf));
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pk));
  for (size_t c = gw; c < nch; c += nw) {
    const uint2 ch = __ldg(chunks + c);
    for (unsigned b = 0; b < ch.y; b += 32 * U) {
      uint2 p[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const unsigned off = b + u * 32 + lane;
        if (off < ch.y) {
          if (HINT)
            asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.u32 {%0, %1}, [%2], %3;"
                         : "=r"(p[u].x), "=r"(p[u].y) : "l"(pay + ch.x + off), "l"(pf));
          else
            p[u] = __ldg(pay + ch.x + off);
        } else {
          p[u] = make_uint2(0, 0x7fffffff);
        }
      }
      int cur[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        if (HINT)
          asm volatile("ld.global.cg.L2::cache_hint.b32 %0, [%1], %2;" : "=r"(cur[u]) : "l"(X + p[u].x), "l"(pk));
        else
          cur[u] = __ldcg(X + p[u].x);
      }
      int old[U];
#pragma unroll
      for (int u = 0; u < U; ++u) old[u] = (int)p[u].y < cur[u] ? atomicMin(X + p[u].x, (int)p[u].y) : 0x7fffffff;
#pragma unroll
      for (int u = 0; u < U; ++u) cnt += (int)p[u].y < old[u];
    }
  }
  if (cnt) atomicAdd(imp, cnt);
}

int main() {
  const size_t n = 1 << 22, m = 1ull << 26, nch = m / 128;
  std::vector<uint2> hp(m);
  std::vector<uint2> hc(nch);
  uint64_t s = 88172645463325252ull;
  for (size_t i = 0; i < m; ++i) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    hp[i] = make_uint2((unsigned)(s % n), (unsigned)((s >> 32) % 1000000));
  }
  // chunks in random order (frontier order is not memory order)
  for (size_t c = 0; c < nch; ++c) hc[c] = make_uint2((unsigned)(c * 128), 128u);
  for (size_t c = nch - 1; c > 0; --c) {
    s ^= s << 13; s ^= s >> 7; s ^= s << 17;
    std::swap(hc[c], hc[s % (c + 1)]);
  }
  uint2 *pay, *chunks;
  int* X;
  unsigned long long* imp;
  CK(cudaMalloc(&pay, m * 8));
  CK(cudaMalloc(&chunks, nch * 8));
  CK(cudaMalloc(&X, n * 4));
  CK(cudaMalloc(&imp, 8));
  CK(cudaMemcpy(pay, hp.data(), m * 8, cudaMemcpyHostToDevice));
  CK(cudaMemcpy(chunks, hc.data(), nch * 8, cudaMemcpyHostToDevice));
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&](auto kern, const char* name, int bps, int fill) {
    for (int rep = 0; rep < 2; ++rep) {
      cudaMemset(X, fill, n * 4);  // 0x7f..: every probe improves; 0: none do
      cudaEventRecord(e0);
      kern<<<sms * bps, 256>>>(pay, chunks, nch, X, imp);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms;
      cudaEventElapsedTime(&ms, e0, e1);
      if (rep) printf("%-22s %d blk/SM labels %s: %.3f ms  %.0f G edges/s\n", name, bps,
                      fill ? "INF " : "zero", ms, m / (ms * 1e6));
    }
  };
  for (int bps : {2, 4, 6, 8}) {
    for (int fill : {0, 0x7f}) {
      run(relax<4, true>, "U=4 hints", bps, fill);
      run(relax<4, false>, "U=4 no hints", bps, fill);
      run(relax<8, true>, "U=8 hints", bps, fill);
    }
  }
  return 0;
}
