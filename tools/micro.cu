// Microbenchmarks of the primitives the traversal is built from (B200):
// grid barrier cost, same-address atomics, random L2 probes vs in-flight
// loads. nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o micro micro.cu
#include <cooperative_groups.h>
#include <cstdio>
#include <cstdint>
#include <vector>
namespace cg = cooperative_groups;

#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e)); return 1; } } while (0)

__global__ void gsync_kernel(int iters, unsigned* sink) {
  cg::grid_group g = cg::this_grid();
  for (int i = 0; i < iters; ++i) g.sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) sink[0] = iters;
}

__global__ void atom_hot(unsigned long long* c, int iters) {
  for (int i = 0; i < iters; ++i)
    if ((threadIdx.x & 31) == 0) atomicAdd(c, 1ull);
}

__global__ void atom_hot_block(unsigned long long* c, int iters) {
  for (int i = 0; i < iters; ++i) {
    if (threadIdx.x == 0) atomicAdd(c, 1ull);
    __syncthreads();
  }
}

template <int U>
__global__ void probe_kernel(const int* __restrict__ X, const unsigned* __restrict__ idx, size_t n,
                             unsigned long long* out) {
  unsigned long long acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i + (U - 1) * stride < n;
       i += U * stride) {
    unsigned id[U];
#pragma unroll
    for (int u = 0; u < U; ++u) id[u] = __ldg(idx + i + u * stride);
    int v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcg(X + id[u]);
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  if (acc == 42) out[0] = acc;
}

template <int U>
__global__ void probe_atomic_kernel(int* X, const unsigned* __restrict__ idx, size_t n) {
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i + (U - 1) * stride < n;
       i += U * stride) {
    unsigned id[U];
#pragma unroll
    for (int u = 0; u < U; ++u) id[u] = __ldg(idx + i + u * stride);
    int r[U];
#pragma unroll
    for (int u = 0; u < U; ++u) r[u] = atomicMin(X + id[u], (int)(i & 1023));
    if (r[0] == -5) X[0] = 1;
  }
}

__global__ void stream_kernel(const uint2* __restrict__ p, size_t n, unsigned long long* out) {
  unsigned long long acc = 0;
  const size_t stride = (size_t)gridDim.x * blockDim.x;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    uint2 v = __ldg(p + i);
    acc += v.x ^ v.y;
  }
  if (acc == 42) out[0] = acc;
}

int latency_main();
int main() {
  latency_main();
  int dev = 0, sms = 0;
  CK(cudaSetDevice(dev));
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  unsigned* sink;
  unsigned long long* c;
  CK(cudaMalloc(&sink, 64));
  CK(cudaMalloc(&c, 64));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  // grid barrier cost vs grid size
  for (int per : {1, 2, 3, 4}) {
    for (int thr : {256, 512}) {
      int maxb = 0;
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&maxb, gsync_kernel, thr, 0);
      if (per > maxb) continue;
      int iters = 2000;
      void* args[] = {&iters, &sink};
      CK(cudaLaunchCooperativeKernel((void*)gsync_kernel, sms * per, thr, args, 0, 0));
      CK(cudaDeviceSynchronize());
      cudaEventRecord(e0);
      CK(cudaLaunchCooperativeKernel((void*)gsync_kernel, sms * per, thr, args, 0, 0));
      cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1));
      cudaEventElapsedTime(&ms, e0, e1);
      printf("grid.sync: %4d blocks x %d thr: %.2f us/sync\n", sms * per, thr, ms * 1e3 / iters);
    }
  }
  // hot atomics
  {
    int iters = 200;
    atom_hot<<<sms * 4, 256>>>(c, iters);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    atom_hot<<<sms * 4, 256>>>(c, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    double n = (double)sms * 4 * 8 * iters;
    printf("same-address atomicAdd (1 lane/warp, all warps): %.2f ns/op, %.0f Mop/s\n",
           ms * 1e6 / n, n / (ms * 1e3));
    atom_hot_block<<<sms * 4, 256>>>(c, iters);
    CK(cudaDeviceSynchronize());
    cudaEventRecord(e0);
    atom_hot_block<<<sms * 4, 256>>>(c, iters);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    n = (double)sms * 4 * iters;
    printf("same-address atomicAdd (1 per block + syncthreads): %.2f ns/op\n", ms * 1e6 / n);
  }
  // random probes into a 16.8 MB label array
  {
    const size_t nl = 1 << 22, np = 64u << 20;
    int* X;
    unsigned* idx;
    CK(cudaMalloc(&X, nl * 4));
    CK(cudaMalloc(&idx, np * 4));
    std::vector<unsigned> h(np);
    uint64_t s = 88172645463325252ull;
    for (size_t i = 0; i < np; ++i) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      h[i] = (unsigned)(s % nl);
    }
    CK(cudaMemcpy(idx, h.data(), np * 4, cudaMemcpyHostToDevice));
    CK(cudaMemset(X, 0, nl * 4));
    for (int blocks_per : {3, 4, 8}) {
      auto run = [&](auto kern, const char* name) {
        kern<<<sms * blocks_per, 256>>>(X, idx, np, c);
        cudaDeviceSynchronize();
        cudaEventRecord(e0);
        kern<<<sms * blocks_per, 256>>>(X, idx, np, c);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        printf("random L2 probe %s, %d blk/SM: %.1f Gprobe/s\n", name, blocks_per, np / (ms * 1e6));
      };
      run(probe_kernel<1>, "U=1");
      run(probe_kernel<4>, "U=4");
      run(probe_kernel<8>, "U=8");
    }
    for (int blocks_per : {4, 8}) {
      probe_atomic_kernel<4><<<sms * blocks_per, 256>>>(X, idx, np);
      cudaDeviceSynchronize();
      cudaEventRecord(e0);
      probe_atomic_kernel<4><<<sms * blocks_per, 256>>>(X, idx, np);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      printf("random atomicMin U=4, %d blk/SM: %.1f Gop/s\n", blocks_per, np / (ms * 1e6));
    }
    CK(cudaGetLastError());
  }
  // streaming 8-byte payload
  {
    const size_t n = 128u << 20;
    uint2* p;
    CK(cudaMalloc(&p, n * 8));
    CK(cudaMemset(p, 1, n * 8));
    stream_kernel<<<sms * 8, 256>>>(p, n, c);
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    stream_kernel<<<sms * 8, 256>>>(p, n, c);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1);
    printf("stream 8B loads: %.0f GB/s\n", n * 8 / (ms * 1e6));
  }
  return 0;
}

// ---- latency probes (appended) ----
__global__ void chase(const unsigned* __restrict__ nxt, int steps, unsigned* out, long long* cyc) {
  unsigned p = 0;
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) p = __ldcg(nxt + p);
  long long t1 = clock64();
  out[0] = p;
  cyc[0] = t1 - t0;
}
__global__ void chase_atomic(unsigned* nxt, int steps, unsigned* out, long long* cyc) {
  unsigned p = 0;
  long long t0 = clock64();
  for (int i = 0; i < steps; ++i) p = atomicAdd(nxt + p, 0u);
  long long t1 = clock64();
  out[0] = p;
  cyc[0] = t1 - t0;
}
// a round = grid.sync + a dependent chain of `deps` L2 loads in one warp per block
__global__ void rounds_kernel(const unsigned* __restrict__ nxt, int rounds, int deps, unsigned* out) {
  cg::grid_group g = cg::this_grid();
  unsigned p = blockIdx.x;
  for (int r = 0; r < rounds; ++r) {
    if (threadIdx.x < 32)
      for (int d = 0; d < deps; ++d) p = __ldcg(nxt + (p & 1023));
    g.sync();
  }
  if (p == 12345) out[0] = p;
}
int latency_main() {
  const size_t n_small = 1 << 20, n_big = 1u << 28;  // 4 MB (L2) and 1 GB (DRAM)
  unsigned *a, *out;
  long long* cyc;
  CK(cudaMalloc(&a, n_big * 4));
  CK(cudaMalloc(&out, 64));
  CK(cudaMalloc(&cyc, 64));
  for (size_t n : {n_small, n_big}) {
    std::vector<unsigned> h(n);
    // random cyclic permutation with large strides
    uint64_t s = 1234567;
    std::vector<unsigned> perm(n);
    for (size_t i = 0; i < n; ++i) perm[i] = i;
    for (size_t i = n - 1; i > 0; --i) {
      s ^= s << 13; s ^= s >> 7; s ^= s << 17;
      size_t j = s % (i + 1);
      std::swap(perm[i], perm[j]);
    }
    for (size_t i = 0; i < n; ++i) h[perm[i]] = perm[(i + 1) % n];
    CK(cudaMemcpy(a, h.data(), n * 4, cudaMemcpyHostToDevice));
    const int steps = 20000;
    chase<<<1, 1>>>(a, 1000, out, cyc);  // warm
    CK(cudaDeviceSynchronize());
    chase<<<1, 1>>>(a, steps, out, cyc);
    long long c;
    CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    printf("dependent load latency, %zu MB footprint: %.0f cycles (%.0f ns @1.965GHz)\n",
           n * 4 >> 20, (double)c / steps, (double)c / steps / 1.965);
    chase_atomic<<<1, 1>>>(a, steps, out, cyc);
    CK(cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost));
    printf("dependent atomic latency, %zu MB footprint: %.0f cycles\n", n * 4 >> 20,
           (double)c / steps);
  }
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int deps : {0, 4, 8}) {
    int rounds = 500;
    void* args[] = {&a, &rounds, &deps, &out};
    CK(cudaLaunchCooperativeKernel((void*)rounds_kernel, sms * 3, 256, args, 0, 0));
    cudaEventRecord(e0);
    CK(cudaLaunchCooperativeKernel((void*)rounds_kernel, sms * 3, 256, args, 0, 0));
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    printf("round = %d dependent L2 loads + grid.sync (444 CTAs): %.2f us\n", deps,
           ms * 1e3 / rounds);
  }
  return 0;
}
