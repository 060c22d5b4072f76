// Do DMMA (mma.sync f64) and DFMA issue concurrently on sm_100a?  Even warps
// run a DMMA loop, odd warps a DFMA loop; compare with each alone.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void mix(double* out, int iters, int mode) {
  const int warp = threadIdx.x >> 5;
  const bool do_mma = mode == 0 ? true : mode == 1 ? false : (warp & 1) == 0;
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999, s = 0;
  if (do_mma) {
    double c[4][2] = {};
    for (int it = 0; it < iters; ++it)
#pragma unroll
      for (int i = 0; i < 4; ++i)
        asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                     : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
    for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  } else {
    double acc[8];
    for (int c = 0; c < 8; ++c) acc[c] = a + c;
    for (int it = 0; it < iters * 16; ++it)
#pragma unroll
      for (int c = 0; c < 8; ++c) acc[c] = fma(acc[c], b, 1e-7);
    for (int c = 0; c < 8; ++c) s += acc[c];
  }
  if (s == 12345.678) out[0] = s;
}
int main() {
  double* out; cudaMalloc(&out, 8);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int blocks = 148 * 4, threads = 512, iters = 4096;
  // per warp: DMMA warp does 4*iters DMMA = 4*iters*512 flops; DFMA warp does 16*iters*8*32*2 flops
  const double f_mma = 4.0 * iters * 512, f_fma = 16.0 * iters * 8 * 32 * 2;
  for (int mode = 0; mode < 3; ++mode) {
    mix<<<blocks, threads>>>(out, iters, mode); cudaDeviceSynchronize();
    float best = 1e9;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); mix<<<blocks, threads>>>(out, iters, mode); cudaEventRecord(e1);
      cudaEventSynchronize(e1); float ms; cudaEventElapsedTime(&ms, e0, e1); if (ms < best) best = ms;
    }
    const int warps = blocks * threads / 32;
    double flops = mode == 0 ? warps * f_mma : mode == 1 ? warps * f_fma : warps / 2 * (f_mma + f_fma);
    printf("{\"mode\": \"%s\", \"ms\": %.3f, \"tflops\": %.2f}\n", mode == 0 ? "dmma" : mode == 1 ? "dfma" : "mixed",
           best, flops / (best * 1e-3) / 1e12);
  }
  return 0;
}
