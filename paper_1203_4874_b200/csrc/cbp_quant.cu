// Quantized-stream tier (reference encoder.cpp:105-139, acceptance.cpp:366-403).
//
// The reference keeps quantized frames as doubles k / (2^bits - 1) tagged u8/u16. On the
// device a quantized frame is its integer codes (1 or 2 bytes per sample), which is also
// what travels over PCIe in the host pipeline: half (u16) or a quarter (u8) of the FP32
// bytes. Decoding dequantizes into FP32 device frames, float(double(k) / maxv): the same
// value the FP32 tier gets from the reference's double, so the decode itself is unchanged.
//   quantize_frame:  k = round(clamp(x, 0, 1) * maxv), range check [-1e-9, 1 + 1e-9]
//   degrade_bits:    k & ~(2^drop - 1)
#include <algorithm>
#include <cstdint>
#include <cstring>
#include <string>
#include <vector>

#include "cbp_ctx.cuh"

using namespace cbp_host;

namespace cbp_dev {

template <class T>
__global__ void k_quantize(const float* in, int planes, int rows, int cols, int ld, double maxv, T* out, int ldq,
                           int* bad) {
  const size_t total = size_t(planes) * rows * cols;
  int b = 0;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
    const size_t pr = i / cols, n = i - pr * cols;  // plane-row, column
    const double x = in[pr * ld + n];
    b |= !(x >= -1e-9 && x <= 1.0 + 1e-9);
    const double c = fmin(1.0, fmax(0.0, x));
    out[pr * ldq + n] = T(round(c * maxv));
  }
  if (b) atomicOr(bad, 1);
}

template <class T>
__global__ void k_dequantize(const T* in, int planes, int rows, int cols, int ldq, double maxv, float* out,
                             int ld) {
  const size_t total = size_t(planes) * rows * cols;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
    const size_t pr = i / cols, n = i - pr * cols;
    out[pr * ld + n] = float(double(in[pr * ldq + n]) / maxv);
  }
}

template <class T>
__global__ void k_degrade(T* codes, int planes, int rows, int cols, int ldq, unsigned mask) {
  const size_t total = size_t(planes) * rows * cols;
  for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < total; i += size_t(gridDim.x) * blockDim.x) {
    const size_t pr = i / cols, n = i - pr * cols;
    codes[pr * ldq + n] = T(unsigned(codes[pr * ldq + n]) & mask);
  }
}

}  // namespace cbp_dev

namespace {

int check_bits(cbp_ctx* ctx, int bits) {
  if (bits != 8 && bits != 16)
    return set_error(ctx, CBP_INVALID_ARGUMENT, "quantization depth must be u8 or u16");  // encoder.cpp:107
  return 0;
}

int grid_for(size_t n) { return int(std::min<size_t>((n + 255) / 256, 148 * 16)); }

// codes (bits) -> FP32 frames; returns 0 or a status
int dequantize(cbp_ctx* ctx, const void* codes, int bits, int planes, int rows, int cols, int ldq, float* out, int ld,
               cudaStream_t s) {
  const double maxv = double((1u << bits) - 1);
  const size_t n = size_t(planes) * rows * cols;
  if (n == 0) return 0;
  if (bits == 8)
    cbp_dev::k_dequantize<<<grid_for(n), 256, 0, s>>>(static_cast<const uint8_t*>(codes), planes, rows, cols, ldq,
                                                        maxv, out, ld);
  else
    cbp_dev::k_dequantize<<<grid_for(n), 256, 0, s>>>(static_cast<const uint16_t*>(codes), planes, rows, cols, ldq,
                                                        maxv, out, ld);
  ++ctx->launches;
  return cuda_check(ctx, cudaGetLastError(), "dequantize launch");
}

}  // namespace

extern "C" {

int cbp_decode_frames(cbp_ctx* ctx, const float* pub_dev, const float* prv_dev, int batch, int channels, int rows,
                      int cols, int ld, const int* width_hints, const cbp_decode_cfg* cfg, float* latent_dev,
                      int ld_out, cbp_decode_info* info, void* stream);
int cbp_decode_frames_async(cbp_ctx* ctx, const float* pub_dev, const float* prv_dev, int batch, int channels,
                            int rows, int cols, int ld, const int* width_hints, const cbp_decode_cfg* cfg,
                            float* latent_dev, int ld_out, cbp_kernel_slot* slots_dev, void* stream);
int cbp_spectral_deblur_slot(cbp_ctx* ctx, const float* blurred_dev, int batch, int channels, int rows, int cols,
                             int ld, const cbp_kernel_slot* slot_dev, float* latent_dev, int ld_out, void* stream);

int cbp_quantize_frames(cbp_ctx* ctx, const float* in_dev, int planes, int rows, int cols, int ld, int bits,
                        void* codes_dev, int ld_codes, void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx || !in_dev || !codes_dev) return CBP_INVALID_ARGUMENT;
  int st;
  if ((st = check_bits(ctx, bits))) return st;
  if (planes < 0 || rows < 1 || cols < 1 || ld < cols || ld_codes < cols)
    return set_error(ctx, CBP_INVALID_ARGUMENT, "bad frame geometry");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int* bad = static_cast<int*>(workspace(ctx, WS_RED, 64));
  if (!bad) return set_error(ctx, CBP_CUDA_ERROR, "workspace allocation failed");
  cudaMemsetAsync(bad, 0, sizeof(int), s);
  const double maxv = double((1u << bits) - 1);
  const size_t n = size_t(planes) * rows * cols;
  if (n) {
    if (bits == 8)
      cbp_dev::k_quantize<<<grid_for(n), 256, 0, s>>>(in_dev, planes, rows, cols, ld, maxv,
                                                      static_cast<uint8_t*>(codes_dev), ld_codes, bad);
    else
      cbp_dev::k_quantize<<<grid_for(n), 256, 0, s>>>(in_dev, planes, rows, cols, ld, maxv,
                                                      static_cast<uint16_t*>(codes_dev), ld_codes, bad);
    ++ctx->launches;
  }
  int hb = 0;
  cudaMemcpyAsync(&hb, bad, sizeof(int), cudaMemcpyDeviceToHost, s);
  if ((st = cuda_check(ctx, cudaStreamSynchronize(s), "quantize"))) return st;
  if (hb) return set_error(ctx, CBP_RANGE_EXCEEDED, "samples outside [0,1]");  // encoder.cpp:112-113
  return 0;
}

int cbp_dequantize_frames(cbp_ctx* ctx, const void* codes_dev, int bits, int planes, int rows, int cols,
                          int ld_codes, float* out_dev, int ld, void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx || !codes_dev || !out_dev) return CBP_INVALID_ARGUMENT;
  int st;
  if ((st = check_bits(ctx, bits))) return st;
  if (planes < 0 || rows < 1 || cols < 1 || ld < cols || ld_codes < cols)
    return set_error(ctx, CBP_INVALID_ARGUMENT, "bad frame geometry");
  return dequantize(ctx, codes_dev, bits, planes, rows, cols, ld_codes, out_dev, ld, static_cast<cudaStream_t>(stream));
}

int cbp_degrade_bits(cbp_ctx* ctx, void* codes_dev, int bits, int planes, int rows, int cols, int ld_codes, int drop,
                     void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx || !codes_dev) return CBP_INVALID_ARGUMENT;
  int st;
  if ((st = check_bits(ctx, bits))) return st;
  if (!(drop >= 0 && drop < bits))
    return set_error(ctx, CBP_INVALID_ARGUMENT, "drop must lie in [0, bit width)");  // encoder.cpp:128-129
  if (drop == 0) return 0;
  const unsigned mask = ~((1u << drop) - 1u);
  const size_t n = size_t(planes) * rows * cols;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  if (n) {
    if (bits == 8)
      cbp_dev::k_degrade<<<grid_for(n), 256, 0, s>>>(static_cast<uint8_t*>(codes_dev), planes, rows, cols, ld_codes,
                                                     mask);
    else
      cbp_dev::k_degrade<<<grid_for(n), 256, 0, s>>>(static_cast<uint16_t*>(codes_dev), planes, rows, cols, ld_codes,
                                                     mask);
    ++ctx->launches;
  }
  return cuda_check(ctx, cudaGetLastError(), "degrade launch");
}

// decode_frame on quantized device frames: dequantize into pitched FP32 workspaces, then
// the FP32 decode (same results as decoding the dequantized values).
int cbp_decode_frames_q(cbp_ctx* ctx, const void* pub_codes, const void* prv_codes, int bits, int batch,
                        int channels, int rows, int cols, int ld_codes, const int* width_hints,
                        const cbp_decode_cfg* cfg, float* latent_dev, int ld_out, cbp_decode_info* info,
                        void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx || !pub_codes || !prv_codes || !cfg) return CBP_INVALID_ARGUMENT;
  int st;
  if ((st = check_bits(ctx, bits))) return st;
  if (batch < 0 || rows < 1 || cols < 1 || ld_codes < cols || !(channels == 1 || channels == 3))
    return set_error(ctx, CBP_INVALID_ARGUMENT, "bad frame geometry");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int ldf = (cols + 3) & ~3;
  const int planes = batch * channels;
  const size_t bytes = sizeof(float) * size_t(planes) * rows * ldf;
  float* pub = static_cast<float*>(workspace(ctx, WS_QPUB, std::max<size_t>(bytes, 256)));
  float* prv = static_cast<float*>(workspace(ctx, WS_QPRV, std::max<size_t>(bytes, 256)));
  if (!pub || !prv) return set_error(ctx, CBP_CUDA_ERROR, "workspace allocation failed");
  if ((st = dequantize(ctx, pub_codes, bits, planes, rows, cols, ld_codes, pub, ldf, s))) return st;
  if ((st = dequantize(ctx, prv_codes, bits, planes, rows, cols, ld_codes, prv, ldf, s))) return st;
  return cbp_decode_frames(ctx, pub, prv, batch, channels, rows, cols, ldf, width_hints, cfg, latent_dev, ld_out,
                           info, stream);
}

}  // extern "C"
