// Cold vs warm instruction fetch: one warp runs a long straight-line ALU
// sequence twice and times each pass with clock64.
// nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o icache icache.cu
#include <cstdio>
#define OP(i) x = x * 1664525u + (i); y ^= x >> 3;
#define OP8(i) OP(i) OP(i+1) OP(i+2) OP(i+3) OP(i+4) OP(i+5) OP(i+6) OP(i+7)
#define OP64(i) OP8(i) OP8(i+8) OP8(i+16) OP8(i+24) OP8(i+32) OP8(i+40) OP8(i+48) OP8(i+56)
#define OP512(i) OP64(i) OP64(i+64) OP64(i+128) OP64(i+192) OP64(i+256) OP64(i+320) OP64(i+384) OP64(i+448)
__global__ void k(unsigned* out, long long* t) {
  unsigned x = threadIdx.x, y = 0;
  long long t0 = clock64();
  for (int pass = 0; pass < 3; ++pass) {
    OP512(0) OP512(512) OP512(1024) OP512(1536)
    long long t1 = clock64();
    if (threadIdx.x == 0 && blockIdx.x == 0) t[pass] = t1 - t0;
    t0 = clock64();
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x ^ y;
}
int main() {
  unsigned* o; long long* t; cudaMalloc(&o, 1 << 20); cudaMalloc(&t, 64);
  for (int r = 0; r < 3; ++r) {
    k<<<1, 32>>>(o, t);
    long long h[3]; cudaMemcpy(h, t, 24, cudaMemcpyDeviceToHost);
    printf("run %d: pass cycles %lld %lld %lld (code ~%d instr)\n", r, h[0], h[1], h[2], 2048 * 3);
  }
  return 0;
}
