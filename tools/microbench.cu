// Microbenchmarks for the B200 FP64 roofline denominators used by this repo:
// DFMA peak, DMMA (mma.sync f64 m8n8k4) peak, FP64 RED throughput at L2,
// and a double-precision copy bandwidth. Prints one JSON object.
#include <cstdio>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){fprintf(stderr,"%s:%d %s\n",__FILE__,__LINE__,cudaGetErrorString(e)); return 1;}}while(0)

template<int CH>
__global__ void dfma_kernel(double* out, int iters, double a, double b) {
  double acc[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) acc[c] = threadIdx.x * 1e-9 + c;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int c = 0; c < CH; ++c) acc[c] = fma(acc[c], a, b);
  }
  double s = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) s += acc[c];
  if (s == 12345.678) out[0] = s;
}

__global__ void dmma_kernel(double* out, int iters) {
  double a = 1.0 + threadIdx.x * 1e-9, b = 0.999;
  double c[4][2];
  for (int i = 0; i < 4; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 4; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
  for (int i = 0; i < 4; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

__global__ void red_kernel(double* y, const int* idx, long n) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long stride = (long)gridDim.x * blockDim.x;
  for (; i < n; i += stride) atomicAdd(&y[idx[i]], 1.0);
}
__global__ void copy_kernel(double2* __restrict__ d, const double2* __restrict__ s, long n) {
  long i = blockIdx.x * (long)blockDim.x + threadIdx.x;
  long stride = (long)gridDim.x * blockDim.x;
  for (; i < n; i += stride) d[i] = s[i];
}

int main() {
  int dev = 0; cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, dev));
  double* out; CK(cudaMalloc(&out, 8));
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  printf("{\"gpu\": \"%s\", \"sms\": %d, \"l2_bytes\": %d", p.name, p.multiProcessorCount, p.l2CacheSize);
  // DFMA
  {
    int iters = 1 << 14, threads = 256, blocks = p.multiProcessorCount * 8;
    for (int w = 0; w < 2; ++w) dfma_kernel<8><<<blocks, threads>>>(out, iters, 0.9999, 1e-7);
    CK(cudaDeviceSynchronize());
    double best = 0;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dfma_kernel<8><<<blocks, threads>>>(out, iters, 0.9999, 1e-7); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      double tf = 2.0 * 8 * iters * (double)threads * blocks / (ms * 1e-3) / 1e12; if (tf > best) best = tf;
    }
    printf(", \"dfma_tflops\": %.3f", best);
    // sustained: 3 s back to back
    int n = 0; cudaEventRecord(e0);
    for (;;) { dfma_kernel<8><<<blocks, threads>>>(out, iters, 0.9999, 1e-7); ++n;
      if (n % 20 == 0) { cudaEventRecord(e1); cudaEventSynchronize(e1); cudaEventElapsedTime(&ms, e0, e1); if (ms > 3000) break; } }
    printf(", \"dfma_tflops_sustained\": %.3f", 2.0 * 8 * iters * (double)threads * blocks * n / (ms * 1e-3) / 1e12);
  }
  // DMMA
  {
    int iters = 1 << 13, threads = 256, blocks = p.multiProcessorCount * 8;
    for (int w = 0; w < 2; ++w) dmma_kernel<<<blocks, threads>>>(out, iters);
    CK(cudaDeviceSynchronize());
    double best = 0;
    for (int r = 0; r < 5; ++r) {
      cudaEventRecord(e0); dmma_kernel<<<blocks, threads>>>(out, iters); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      double tf = 2.0 * 256 * 4 * iters * (double)(threads / 32) * blocks / (ms * 1e-3) / 1e12; if (tf > best) best = tf;
    }
    printf(", \"dmma_tflops\": %.3f", best);
  }
  // RED f64: 64M atomics onto targets of varying footprint
  {
    long n = 1L << 26;
    int* hidx = (int*)malloc(n * 4); int* didx; double* y;
    CK(cudaMalloc(&didx, n * 4)); CK(cudaMalloc(&y, (1L << 25) * 8));
    const long foots[3] = {1L << 18, 1L << 22, 1L << 25};
    const char* names[3] = {"red_f64_2MB_gops", "red_f64_32MB_gops", "red_f64_256MB_gops"};
    for (int f = 0; f < 3; ++f) {
      unsigned long long s = 88172645463325252ULL;
      // locality pattern similar to a FE scatter: runs of nearby indices
      for (long i = 0; i < n; ++i) { s ^= s << 13; s ^= s >> 7; s ^= s << 17; hidx[i] = (int)(((i / 10) * 7 + (s % 64)) % foots[f]); }
      CK(cudaMemcpy(didx, hidx, n * 4, cudaMemcpyHostToDevice));
      CK(cudaMemset(y, 0, foots[f] * 8));
      red_kernel<<<p.multiProcessorCount * 16, 256>>>(y, didx, n); CK(cudaDeviceSynchronize());
      double best = 0;
      for (int r = 0; r < 3; ++r) {
        cudaEventRecord(e0); red_kernel<<<p.multiProcessorCount * 16, 256>>>(y, didx, n); cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
        double g = n / (ms * 1e-3) / 1e9; if (g > best) best = g;
      }
      printf(", \"%s\": %.2f", names[f], best);
    }
    free(hidx); cudaFree(didx); cudaFree(y);
  }
  // copy bandwidth (double2), 2 GiB
  {
    long n = (1L << 31) / 16; double2 *a, *b; CK(cudaMalloc(&a, n * 16)); CK(cudaMalloc(&b, n * 16));
    cudaMemset(a, 0, n * 16);
    copy_kernel<<<p.multiProcessorCount * 8, 512>>>(b, a, n); CK(cudaDeviceSynchronize());
    double best = 0;
    for (int r = 0; r < 10; ++r) {
      cudaEventRecord(e0); copy_kernel<<<p.multiProcessorCount * 8, 512>>>(b, a, n); cudaEventRecord(e1);
      CK(cudaEventSynchronize(e1)); cudaEventElapsedTime(&ms, e0, e1);
      double g = 2.0 * n * 16 / (ms * 1e-3) / 1e9; if (g > best) best = g;
    }
    printf(", \"copy_gbs\": %.1f", best);
  }
  printf("}\n");
  return 0;
}
