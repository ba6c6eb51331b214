// Latency calibration of FP64 dependent chains on the device (profiling aid):
// DFMA, DMUL+DADD, division, sqrt, hypot, shared-memory store->load round trip.
#include <cstdio>
#include <cuda_runtime.h>
__device__ unsigned long long now() { unsigned long long t; asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t)); return t; }
__global__ void k(double* out, double a, double b, int n) {
  __shared__ double sm[64];
  double x = a;
  unsigned long long t0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, b, a);
  unsigned long long t1 = clock64();
  for (int i = 0; i < n; ++i) x = a / x + b;
  unsigned long long t2 = clock64();
  for (int i = 0; i < n; ++i) x = sqrt(x) + a;
  unsigned long long t3 = clock64();
  for (int i = 0; i < n; ++i) x = hypot(x, b) * 0.5;
  unsigned long long t4 = clock64();
  sm[threadIdx.x] = x;
  for (int i = 0; i < n; ++i) { sm[(i + 1) & 31] = sm[i & 31] * b + a; }
  unsigned long long t5 = clock64();
  for (int i = 0; i < n; ++i) x = rsqrt(x) + a;
  unsigned long long t6 = clock64();
  if (threadIdx.x == 0)
    printf("cycles per op: dfma %.1f  div %.1f  sqrt %.1f  hypot %.1f  smem-chain %.1f  rsqrt %.1f  (x=%g %g)\n",
           double(t1 - t0) / n, double(t2 - t1) / n, double(t3 - t2) / n, double(t4 - t3) / n, double(t5 - t4) / n,
           double(t6 - t5) / n, x, sm[5]);
  out[threadIdx.x] = x;
}
int main() {
  double* d;
  cudaMalloc(&d, 1024);
  k<<<1, 32>>>(d, 1.000001, 0.999999, 2000);
  cudaDeviceSynchronize();
  k<<<1, 32>>>(d, 1.000001, 0.999999, 2000);
  cudaDeviceSynchronize();
  return 0;
}
