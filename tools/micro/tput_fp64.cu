// FP64 throughput calibration (profiling aid): DFMA on the FP64 pipe against DMMA
// (mma.sync m8n8k4 f64) on the tensor pipe, all SMs, independent accumulators.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_dfma(double* out, double a, double b, int n) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = a + j;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) x[j] = fma(x[j], b, a);
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

__global__ void k_dmma(double* out, double a, double b, int n) {
  double acc[8][2];
#pragma unroll
  for (int j = 0; j < 8; ++j) acc[j][0] = acc[j][1] = 0;
  double fa = a + threadIdx.x * 1e-3, fb = b - threadIdx.x * 1e-3;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(acc[j][0]), "+d"(acc[j][1])
                   : "d"(fa), "d"(fb));
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += acc[j][0] + acc[j][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// F2F.F64.F32 conversions interleaved with DFMA: 8 DFMA per conversion (the validation
// convolution's window loads would convert FP32 tile values in the inner loop)
__global__ void k_f2f(double* out, const float* in, int n) {
  double x[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) x[j] = j;
  float f = in[threadIdx.x & 31];
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const double v = double(f);
      f = __int_as_float(__float_as_int(f) ^ 1);
      x[j] = fma(x[j], v, 1.0);
    }
  }
  double s = 0;
#pragma unroll
  for (int j = 0; j < 8; ++j) s += x[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  double* d;
  cudaMalloc(&d, sizeof(double) * sms * 8 * 1024);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int n = 4096;
  for (int threads : {256, 512, 1024}) {
    for (int rep = 0; rep < 2; ++rep) {
      float ms = 0;
      cudaEventRecord(e0);
      k_dfma<<<sms * 2, threads>>>(d, 1.0000001, 0.9999999, n);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double dfma_tf = 2.0 * 8 * n * double(sms) * 2 * threads / (ms * 1e-3) / 1e12;
      cudaEventRecord(e0);
      k_dmma<<<sms * 2, threads>>>(d, 1.0000001, 0.9999999, n);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      float ms2 = 0;
      cudaEventElapsedTime(&ms2, e0, e1);
      // one m8n8k4 = 256 FMAs per warp
      const double dmma_tf = 2.0 * 256 * 8 * n * double(sms) * 2 * (threads / 32) / (ms2 * 1e-3) / 1e12;
      if (rep) printf("threads/CTA %4d: DFMA %.1f TFLOP/s  DMMA %.1f TFLOP/s\n", threads, dfma_tf, dmma_tf);
    }
  }
  {
    float* fin;
    cudaMalloc(&fin, 128);
    cudaMemset(fin, 0, 128);
    for (int rep = 0; rep < 2; ++rep) {
      float ms = 0;
      cudaEventRecord(e0);
      k_f2f<<<sms * 2, 512>>>(d, fin, n);
      cudaEventRecord(e1);
      cudaEventSynchronize(e1);
      cudaEventElapsedTime(&ms, e0, e1);
      const double gops = 8.0 * n * double(sms) * 2 * 512 / (ms * 1e-3) / 1e9;
      if (rep) printf("F2F.F64.F32 + DFMA pairs: %.0f G pairs/s (DFMA alone at peak: %.0f G/s)\n", gops, 37.0e3 / 2);
    }
  }
  printf("err %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
