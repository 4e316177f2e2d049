// Random-access ceilings of this B200 for the traversal's access shapes:
// every warp lane reads G contiguous bytes (G = 4, 32, 64, 128) at a random
// G-aligned offset of a buffer of B bytes, U independent reads in flight per
// lane. B = 16 MB stays in L2 (the label probes); B = 2 GB misses it (key
// lines, payload ranges and per-vertex records of a graph larger than L2).
// Prints requests/s and useful GB/s; DRAM sectors are whatever the memory
// system fetches for them (run under ncu for dram__bytes).
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o micro_gather micro_gather.cu
#include <cstdio>
#include <cstdint>

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__device__ __forceinline__ uint64_t mix(uint64_t x) {
  x ^= x >> 33; x *= 0xff51afd7ed558ccdull; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ull;
  return x ^ (x >> 33);
}

template <int G, int U>
__global__ void gather(const uint4* __restrict__ buf, uint64_t units, int iters, uint32_t* sink) {
  const uint64_t tid = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x;
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
    uint32_t v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t r = mix(tid * 1315423911ull + (uint64_t)it * U + u) % units;
      if (G == 4) {
        v[u] = __ldcg(reinterpret_cast<const uint32_t*>(buf) + r);
      } else {
        const uint4* p = buf + r * (G / 16);
        uint32_t s = 0;
#pragma unroll
        for (int k = 0; k < G / 16; ++k) {
          const uint4 q = __ldcg(p + k);
          s += q.x ^ q.y ^ q.z ^ q.w;
        }
        v[u] = s;
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (acc == 0x12345678u) sink[0] = acc;
}

template <int G, int U>
int run(const uint4* buf, uint64_t bytes, int sms, uint32_t* sink) {
  const uint64_t units = bytes / G;
  const int blocks = sms * 8, threads = 256, iters = 64;
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  gather<G, U><<<blocks, threads>>>(buf, units, 4, sink);
  CK(cudaEventRecord(a));
  gather<G, U><<<blocks, threads>>>(buf, units, iters, sink);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms = 0;
  CK(cudaEventElapsedTime(&ms, a, b));
  const double reqs = (double)blocks * threads * iters * U;
  printf("buffer %6llu MB  granule %3d B  in flight/lane %d: %7.1f G req/s  %7.0f GB/s useful\n",
         (unsigned long long)(bytes >> 20), G, U, reqs / ms / 1e6, reqs * G / ms / 1e6);
  return 0;
}

int main() {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const uint64_t big = 2ull << 30, small = 16ull << 20;
  uint4* buf = nullptr;
  uint32_t* sink = nullptr;
  CK(cudaMalloc(&buf, big));
  CK(cudaMalloc(&sink, 4));
  CK(cudaMemset(buf, 1, big));
  for (uint64_t bytes : {small, big}) {
    run<4, 4>(buf, bytes, sms, sink);
    run<4, 8>(buf, bytes, sms, sink);
    run<32, 4>(buf, bytes, sms, sink);
    run<32, 8>(buf, bytes, sms, sink);
    run<64, 4>(buf, bytes, sms, sink);
    run<128, 2>(buf, bytes, sms, sink);
    run<128, 4>(buf, bytes, sms, sink);
  }
  return 0;
}
