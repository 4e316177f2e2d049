// Latency of dependent L2-resident loads from ONE warp lane to random lines of a 16 MB
// buffer (warmed through L2 by the whole grid, then by this lane itself): is there one latency
// or two (lines homed in the SM's near L2 partition / in the other die's)?
// build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o tools/micro_l2_home tools/micro_l2_home.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <cuda_runtime.h>

__global__ void warm(const uint32_t* buf, size_t n, uint32_t* sink) {
  uint32_t acc = 0;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
    acc += __ldcg(buf + i);
  if (acc == 0x12345678u) *sink = acc;
}

__global__ void probe(const uint32_t* buf, size_t lines, uint32_t* lat, uint32_t* smid, int reps,
                      int fresh) {
  __shared__ volatile uint32_t sh[2];
  if (threadIdx.x != 0) return;
  uint32_t sm;
  asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
  smid[blockIdx.x] = sm;
  uint32_t x = 12345u + blockIdx.x * 7919u;
  for (int pass = 0; pass < 2; ++pass) {  // pass 0 warms this lane's own path
    uint32_t s = fresh && pass ? x ^ 0x9e3779b9u : x;  // fresh: the timed pass touches new lines (DRAM)
    for (int i = 0; i < reps; ++i) {
      s = s * 1664525u + 1013904223u;
      const size_t line = (size_t)(s >> 8) % lines;
      const uint32_t* p = buf + line * 32;
      const long long t0 = clock64();
      const uint32_t v = __ldcg(p);
      sh[0] = v;  // volatile store of the loaded value: issues when the load has returned
      const long long t1 = clock64();
      s += sh[0] & 1u;  // dependent
      if (pass == 1) lat[(size_t)blockIdx.x * reps + i] = (uint32_t)(t1 - t0) + (s & 0u);
    }
  }
}

int main(int argc, char** argv) {
  const size_t bytes = (size_t)(argc > 1 ? atoi(argv[1]) : 16) << 20, n = bytes / 4, lines = bytes / 128;
  const int reps = 4096, blocks = 8;
  uint32_t *buf, *lat, *smid, *sink;
  cudaMalloc(&buf, bytes);
  cudaMemset(buf, 0, bytes);
  cudaMalloc(&lat, (size_t)blocks * reps * 4);
  cudaMalloc(&smid, blocks * 4);
  cudaMalloc(&sink, 4);
  warm<<<592, 256>>>(buf, n, sink);
  probe<<<blocks, 32>>>(buf, lines, lat, smid, reps, bytes > (64u << 20));
  cudaDeviceSynchronize();
  std::vector<uint32_t> h((size_t)blocks * reps), sm(blocks);
  cudaMemcpy(h.data(), lat, h.size() * 4, cudaMemcpyDeviceToHost);
  cudaMemcpy(sm.data(), smid, blocks * 4, cudaMemcpyDeviceToHost);
  for (int b = 0; b < blocks; ++b) {
    std::vector<uint32_t> v(h.begin() + (size_t)b * reps, h.begin() + (size_t)(b + 1) * reps);
    std::sort(v.begin(), v.end());
    printf("sm %3u: latency cycles p5 %u p25 %u p50 %u p75 %u p95 %u | histogram (50-cycle bins from 200, %zu MB):", sm[b],
           v[reps / 20], v[reps / 4], v[reps / 2], v[3 * reps / 4], v[19 * reps / 20], bytes >> 20);
    int hist[40] = {0};
    for (uint32_t x : v) { int k = x < 200 ? 0 : std::min(39, (int)((x - 200) / 50)); ++hist[k]; }
    for (int k = 0; k < 40; ++k) printf(" %d", hist[k]);
    printf("\n");
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
