// Vendor baseline for the deconvolution (not part of the product): the same 2-D Wiener
// deconvolution of a batch of planes with planned cuFFT R2C / C2R and callbacks (load
// callback zero-pads the pitched blurred planes into the Gr x Gc grid, store callback of the
// R2C multiplies by the filter table, store callback of the C2R crops to the latent region).
// Built by tools/cufft/build.sh into tools/cufft/libcufft_baseline.so (cuFFT static + callbacks).
#include <cstdio>
#include <cuda_runtime.h>
#include <cufft.h>
#include <cufftXt.h>

struct InInfo {
  const float* in;  // planes of Mb rows x ld floats (plane stride in_plane)
  long long in_plane;
  int ld, Mb, Nb, Gr, Gc;
};
struct MulInfo {
  const float2* H;  // Gr x Hc filter (scaled by 1/(Gr Gc)), shared by every plane
  int Hc;
  long long hplane;  // Gr * Hc
};
struct OutInfo {
  float* out;  // planes of M rows x ld_out floats
  long long out_plane;
  int ld_out, M, N, Gr, Gc;
};

__device__ cufftReal cb_load(void* dataIn, size_t offset, void* callerInfo, void* sharedPtr) {
  const InInfo* a = static_cast<const InInfo*>(callerInfo);
  const unsigned g = unsigned(a->Gr) * unsigned(a->Gc), off = unsigned(offset);  // < 2^32 elements
  const unsigned p = off / g, rem = off - p * g;
  const unsigned r = rem / unsigned(a->Gc), c = rem - r * unsigned(a->Gc);
  return (r < unsigned(a->Mb) && c < unsigned(a->Nb)) ? a->in[p * a->in_plane + (long long)r * a->ld + c] : 0.f;
}
__device__ void cb_mul(void* dataOut, size_t offset, cufftComplex element, void* callerInfo, void* sharedPtr) {
  const MulInfo* m = static_cast<const MulInfo*>(callerInfo);
  const float2 h = m->H[unsigned(offset) % unsigned(m->hplane)];
  static_cast<cufftComplex*>(dataOut)[offset] =
      make_float2(element.x * h.x - element.y * h.y, element.x * h.y + element.y * h.x);
}
__device__ void cb_crop(void* dataOut, size_t offset, cufftReal element, void* callerInfo, void* sharedPtr) {
  const OutInfo* o = static_cast<const OutInfo*>(callerInfo);
  const unsigned g = unsigned(o->Gr) * unsigned(o->Gc), off = unsigned(offset);
  const unsigned p = off / g, rem = off - p * g;
  const unsigned r = rem / unsigned(o->Gc), c = rem - r * unsigned(o->Gc);
  if (r < unsigned(o->M) && c < unsigned(o->N)) o->out[p * o->out_plane + (long long)r * o->ld_out + c] = element;
}
__device__ cufftCallbackLoadR d_load = cb_load;
__device__ cufftCallbackStoreC d_mul = cb_mul;
__device__ cufftCallbackStoreR d_crop = cb_crop;

// explicit passes (no callbacks): zero-padded copy, R2C, filter multiply, C2R, crop
__global__ void k_pad(const float* in, long long in_plane, int ld, int Mb, int Nb, int Gr, int Gc, float* x, int planes) {
  const long long g = (long long)Gr * Gc, n = g * planes;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long p = i / g, rem = i - p * g;
    const int r = int(rem / Gc), c = int(rem - (long long)r * Gc);
    x[i] = (r < Mb && c < Nb) ? in[p * in_plane + (long long)r * ld + c] : 0.f;
  }
}
__global__ void k_mul(float2* X, const float2* H, long long hplane, long long n) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const float2 e = X[i], h = H[i % hplane];
    X[i] = make_float2(e.x * h.x - e.y * h.y, e.x * h.y + e.y * h.x);
  }
}
__global__ void k_crop(const float* x, int Gr, int Gc, float* out, long long out_plane, int ld_out, int M, int N, int planes) {
  const long long n = (long long)M * N * planes;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const long long p = i / ((long long)M * N), rem = i - p * M * N;
    const int r = int(rem / N), c = int(rem - (long long)r * N);
    out[p * out_plane + (long long)r * ld_out + c] = x[(p * Gr + r) * (long long)Gc + c];
  }
}

extern "C" int cufft_deblur_plain(const float* in, long long in_plane, int ld, int Mb, int Nb, const float2* H, int Gr,
                                  int Gc, float* out, long long out_plane, int ld_out, int M, int N, int planes,
                                  int reps, float* ms_per_rep) {
  const int Hc = Gc / 2 + 1;
  cufftHandle fwd, inv;
  int n[2] = {Gr, Gc};
  if (cufftPlanMany(&fwd, 2, n, nullptr, 1, Gr * Gc, nullptr, 1, Gr * Hc, CUFFT_R2C, planes) != CUFFT_SUCCESS) return 1;
  if (cufftPlanMany(&inv, 2, n, nullptr, 1, Gr * Hc, nullptr, 1, Gr * Gc, CUFFT_C2R, planes) != CUFFT_SUCCESS) return 2;
  float* x = nullptr;
  cufftComplex* spec = nullptr;
  if (cudaMalloc(&x, size_t(planes) * Gr * Gc * sizeof(float)) != cudaSuccess) return 6;
  if (cudaMalloc(&spec, size_t(planes) * Gr * Hc * sizeof(cufftComplex)) != cudaSuccess) return 7;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto run = [&] {
    k_pad<<<148 * 8, 256>>>(in, in_plane, ld, Mb, Nb, Gr, Gc, x, planes);
    cufftExecR2C(fwd, x, spec);
    k_mul<<<148 * 8, 256>>>(spec, H, (long long)Gr * Hc, (long long)Gr * Hc * planes);
    cufftExecC2R(inv, spec, x);
    k_crop<<<148 * 8, 256>>>(x, Gr, Gc, out, out_plane, ld_out, M, N, planes);
  };
  for (int w = 0; w < 2; ++w) run();
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) run();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms_per_rep, e0, e1);
  *ms_per_rep /= float(reps);
  const cudaError_t err = cudaGetLastError();
  cudaFree(x);
  cudaFree(spec);
  cufftDestroy(fwd);
  cufftDestroy(inv);
  return err == cudaSuccess ? 0 : 8;
}

static void* dev_copy(const void* h, size_t n) {
  void* d = nullptr;
  cudaMalloc(&d, n);
  cudaMemcpy(d, h, n, cudaMemcpyHostToDevice);
  return d;
}

extern "C" int cufft_deblur(const float* in, long long in_plane, int ld, int Mb, int Nb, const float2* H, int Gr,
                            int Gc, float* out, long long out_plane, int ld_out, int M, int N, int planes, int reps,
                            float* ms_per_rep) {
  const int Hc = Gc / 2 + 1;
  cufftHandle fwd, inv;
  int n[2] = {Gr, Gc};
  if (cufftPlanMany(&fwd, 2, n, nullptr, 1, Gr * Gc, nullptr, 1, Gr * Hc, CUFFT_R2C, planes) != CUFFT_SUCCESS) return 1;
  if (cufftPlanMany(&inv, 2, n, nullptr, 1, Gr * Hc, nullptr, 1, Gr * Gc, CUFFT_C2R, planes) != CUFFT_SUCCESS) return 2;
  InInfo ii{in, in_plane, ld, Mb, Nb, Gr, Gc};
  MulInfo mi{H, Hc, (long long)Gr * Hc};
  OutInfo oi{out, out_plane, ld_out, M, N, Gr, Gc};
  void* dii = dev_copy(&ii, sizeof ii);
  void* dmi = dev_copy(&mi, sizeof mi);
  void* doi = dev_copy(&oi, sizeof oi);
  cufftCallbackLoadR h_load;
  cufftCallbackStoreC h_mul;
  cufftCallbackStoreR h_crop;
  cudaMemcpyFromSymbol(&h_load, d_load, sizeof h_load);
  cudaMemcpyFromSymbol(&h_mul, d_mul, sizeof h_mul);
  cudaMemcpyFromSymbol(&h_crop, d_crop, sizeof h_crop);
  if (cufftXtSetCallback(fwd, (void**)&h_load, CUFFT_CB_LD_REAL, &dii) != CUFFT_SUCCESS) return 3;
  if (cufftXtSetCallback(fwd, (void**)&h_mul, CUFFT_CB_ST_COMPLEX, &dmi) != CUFFT_SUCCESS) return 4;
  if (cufftXtSetCallback(inv, (void**)&h_crop, CUFFT_CB_ST_REAL, &doi) != CUFFT_SUCCESS) return 5;
  // the R2C input buffer is never read (the load callback reads the pitched planes); the C2R
  // output buffer is never written (the store callback writes the latent region)
  float* dummy_r = nullptr;
  cufftComplex* spec = nullptr;
  if (cudaMalloc(&dummy_r, size_t(planes) * Gr * Gc * sizeof(float)) != cudaSuccess) return 6;
  if (cudaMalloc(&spec, size_t(planes) * Gr * Hc * sizeof(cufftComplex)) != cudaSuccess) return 7;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  for (int w = 0; w < 2; ++w) {
    cufftExecR2C(fwd, dummy_r, spec);
    cufftExecC2R(inv, spec, dummy_r);
  }
  cudaEventRecord(e0);
  for (int r = 0; r < reps; ++r) {
    cufftExecR2C(fwd, dummy_r, spec);
    cufftExecC2R(inv, spec, dummy_r);
  }
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms_per_rep, e0, e1);
  *ms_per_rep /= float(reps);
  const cudaError_t err = cudaGetLastError();
  cudaFree(dummy_r);
  cudaFree(spec);
  cudaFree(dii);
  cudaFree(dmi);
  cudaFree(doi);
  cufftDestroy(fwd);
  cufftDestroy(inv);
  return err == cudaSuccess ? 0 : 8;
}
