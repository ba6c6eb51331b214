// Host-buffer decode pipeline (the end-to-end path): the reference CLI decodes a run
// of frames held in host memory (tools/cbp.cpp:130-207). Here H2D copies, device
// decode and D2H copies of consecutive frames overlap on three streams through a
// ring of device frame buffers; recovered kernels stay on the device (slots) and are
// reused by the following frames (spectral_deblur_slot), with no host round trip.
#include <cstdlib>
#include <cstring>
#include <string>
#include <vector>

#include "cbp_ctx.cuh"

namespace {
// ring depth: H2D runs up to kRing frames ahead, so the ~1 ms recovery of a frame hides
// under the transfers of the following ones (the path is PCIe-bound)
#ifndef CBP_E2E_RING
#define CBP_E2E_RING 6
#endif
constexpr int kRing = CBP_E2E_RING;

struct Pipe {
  cudaStream_t h2d = nullptr, comp = nullptr, d2h = nullptr;
  cudaEvent_t in[kRing], done[kRing], out[kRing];
  bool ready = false;
};

Pipe& pipe_of(cbp_ctx* ctx) {
  static thread_local std::vector<std::pair<cbp_ctx*, Pipe>> pipes;
  for (auto& p : pipes)
    if (p.first == ctx) return p.second;
  pipes.push_back({ctx, Pipe{}});
  Pipe& p = pipes.back().second;
  cudaStreamCreateWithFlags(&p.h2d, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&p.comp, cudaStreamNonBlocking);
  cudaStreamCreateWithFlags(&p.d2h, cudaStreamNonBlocking);
  for (int r = 0; r < kRing; ++r) {
    cudaEventCreateWithFlags(&p.in[r], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&p.done[r], cudaEventDisableTiming);
    cudaEventCreateWithFlags(&p.out[r], cudaEventDisableTiming);
  }
  p.ready = true;
  return p;
}
}  // namespace

using namespace cbp_host;

extern "C" {

int cbp_decode_frames_async(cbp_ctx* ctx, const float* pub_dev, const float* prv_dev, int batch, int channels,
                            int rows, int cols, int ld, const int* width_hints, const cbp_decode_cfg* cfg,
                            float* latent_dev, int ld_out, cbp_kernel_slot* slots_dev, void* stream);
int cbp_spectral_deblur_slot(cbp_ctx* ctx, const float* blurred_dev, int batch, int channels, int rows, int cols,
                             int ld, const cbp_kernel_slot* slot_dev, float* latent_dev, int ld_out, void* stream);

int cbp_dequantize_frames(cbp_ctx* ctx, const void* codes_dev, int bits, int planes, int rows, int cols,
                          int ld_codes, float* out_dev, int ld, void* stream);

}  // extern "C"

namespace {

// bits = 0: FP32 host frames; 8 / 16: quantized codes (uint8 / uint16), copied as codes and
// dequantized on the device (cbp_quant.cu), so PCIe carries 1 or 2 bytes per sample.
int run_host(cbp_ctx* ctx, const void* pub, const void* prv, int bits, int n_frames, int channels, int rows,
             int cols, const int* recover, int width_hint, const cbp_decode_cfg* cfg, float* latent,
             cbp_kernel_slot* slots_host) {
  if (!ctx || !pub || !recover || !cfg || !latent) return CBP_INVALID_ARGUMENT;
  if (bits != 0 && bits != 8 && bits != 16)
    return set_error(ctx, CBP_INVALID_ARGUMENT, "quantization depth must be u8 or u16");
  if (n_frames <= 0) return 0;
  if (!recover[0]) return set_error(ctx, CBP_INVALID_ARGUMENT, "the first frame of a run must recover the kernel");
  int n_rec = 0;
  for (int j = 0; j < n_frames; ++j) n_rec += recover[j] ? 1 : 0;
  if (n_rec > 0 && !prv) return set_error(ctx, CBP_INVALID_ARGUMENT, "recovery frames need the private stream");
  Pipe& P = pipe_of(ctx);
  const size_t frame = size_t(channels) * rows * cols;
  const size_t esz = bits == 0 ? sizeof(float) : bits == 8 ? 1 : 2;
  float* dpub = static_cast<float*>(workspace(ctx, WS_PUB, sizeof(float) * frame * kRing));
  float* dprv = static_cast<float*>(workspace(ctx, WS_PRV, sizeof(float) * frame * kRing));
  float* dout = static_cast<float*>(workspace(ctx, WS_OUT, sizeof(float) * frame * kRing));
  char* codes = bits ? static_cast<char*>(workspace(ctx, WS_QCODES, esz * frame * kRing * 2)) : nullptr;
  cbp_kernel_slot* slots = static_cast<cbp_kernel_slot*>(workspace(ctx, WS_SOLVE, sizeof(cbp_kernel_slot) * n_rec));
  if (!dpub || !dprv || !dout || !slots || (bits && !codes))
    return set_error(ctx, CBP_CUDA_ERROR, "pipeline allocation failed");
  const char* hpub = static_cast<const char*>(pub);
  const char* hprv = static_cast<const char*>(prv);
  int rec = -1;
  const int hint = width_hint;
  int tlo = hint > 0 && cfg->trust_hint ? hint : cfg->search_min;
  tlo = tlo < 1 ? 1 : (tlo > rows || tlo > cols ? 1 : tlo);
  // Frames move in groups of G consecutive frames (consecutive ring slots: kRing % G == 0):
  // one H2D copy of the group's public frames and one D2H copy of its latents. Copies of two
  // 1080p RGB frames (50 MB) keep the PCIe link busier than per-frame ones (tools/
  // copy_pattern_probe.py, copies alone: 1.76k against 1.70k frames/s); the decode of a
  // group's first frame waits for its second frame's transfer (latency, not throughput).
  static const int G = [] {  // CBP_E2E_GROUP: A/B switch (1, 2 or 3)
    const char* e = getenv("CBP_E2E_GROUP");
    const int g = e ? atoi(e) : 2;
    return g == 1 || g == 3 ? g : 2;
  }();
  static_assert(kRing % 2 == 0 && kRing % 3 == 0, "ring slots must split into groups");
  for (int j0 = 0; j0 < n_frames; j0 += G) {
    const int g = n_frames - j0 < G ? n_frames - j0 : G;
    const int r0 = j0 % kRing;
    if (j0 >= kRing) cudaStreamWaitEvent(P.h2d, P.out[r0], 0);  // the group's ring slots drained
    char* cpub0 = bits ? codes + esz * frame * r0 : reinterpret_cast<char*>(dpub + r0 * frame);
    cudaMemcpyAsync(cpub0, hpub + esz * frame * j0, esz * frame * g, cudaMemcpyHostToDevice, P.h2d);
    for (int k = 0; k < g; ++k) {
      char* cprv = bits ? codes + esz * frame * (kRing + r0 + k) : reinterpret_cast<char*>(dprv + (r0 + k) * frame);
      if (recover[j0 + k])
        cudaMemcpyAsync(cprv, hprv + esz * frame * (j0 + k), esz * frame, cudaMemcpyHostToDevice, P.h2d);
    }
    cudaEventRecord(P.in[r0], P.h2d);
    cudaStreamWaitEvent(P.comp, P.in[r0], 0);
    for (int k = 0; k < g; ++k) {
      const int j = j0 + k, r = r0 + k;
      char* cpub = bits ? codes + esz * frame * r : reinterpret_cast<char*>(dpub + r * frame);
      char* cprv = bits ? codes + esz * frame * (kRing + r) : reinterpret_cast<char*>(dprv + r * frame);
      int st = 0;
      if (bits) {
        st = cbp_dequantize_frames(ctx, cpub, bits, channels, rows, cols, cols, dpub + r * frame, cols, P.comp);
        if (!st && recover[j])
          st = cbp_dequantize_frames(ctx, cprv, bits, channels, rows, cols, cols, dprv + r * frame, cols, P.comp);
        if (st) return st;
      }
      if (recover[j]) {
        ++rec;
        st = cbp_decode_frames_async(ctx, dpub + r * frame, dprv + r * frame, 1, channels, rows, cols, cols,
                                     hint > 0 ? &hint : nullptr, cfg, dout + r * frame, cols, slots + rec, P.comp);
      } else {
        st = cbp_spectral_deblur_slot(ctx, dpub + r * frame, 1, channels, rows, cols, cols, slots + rec,
                                      dout + r * frame, cols, P.comp);
      }
      if (st) return st;
    }
    cudaEventRecord(P.done[r0], P.comp);
    cudaStreamWaitEvent(P.d2h, P.done[r0], 0);
    // D2H as ONE contiguous copy per group, ending at the last row a latent can occupy in the
    // group's last plane (rows - tlo + 1 rows, tlo = the smallest width the frame can decode
    // with: trusted hint, else search_min). One block sustains more of the link than three
    // per-plane copies of the latent rows per frame (copies alone: 1.70k against 1.59k
    // frames/s), for 0.2% more bytes (the t - 1 rows between planes).
    static const bool full_d2h = getenv("CBP_E2E_FULL_D2H") != nullptr;  // A/B switch: whole frames
    const size_t n_d2h = full_d2h ? frame * g
                                  : frame * (g - 1) + size_t(channels - 1) * rows * cols + size_t(rows - tlo + 1) * cols;
    cudaMemcpyAsync(latent + j0 * frame, dout + r0 * frame, sizeof(float) * n_d2h, cudaMemcpyDeviceToHost, P.d2h);
    cudaEventRecord(P.out[r0], P.d2h);
  }
  int st = cuda_check(ctx, cudaStreamSynchronize(P.d2h), "pipeline");
  if (st) return st;
  if ((st = cuda_check(ctx, cudaStreamSynchronize(P.comp), "pipeline"))) return st;
  std::vector<cbp_kernel_slot> hs(n_rec);
  cudaMemcpy(hs.data(), slots, sizeof(cbp_kernel_slot) * n_rec, cudaMemcpyDeviceToHost);
  if (slots_host) std::memcpy(slots_host, hs.data(), sizeof(cbp_kernel_slot) * n_rec);
  for (int k = 0; k < n_rec; ++k)
    if (hs[k].status) return set_error(ctx, hs[k].status, "recovery frame " + std::to_string(k) + " failed");
  return 0;
}

}  // namespace

extern "C" {

int cbp_decode_run_host(cbp_ctx* ctx, const float* pub, const float* prv, int n_frames, int channels, int rows,
                        int cols, const int* recover, int width_hint, const cbp_decode_cfg* cfg, float* latent,
                        cbp_kernel_slot* slots_host) {
  cbp_host::DeviceGuard device_guard(ctx);
  return run_host(ctx, pub, prv, 0, n_frames, channels, rows, cols, recover, width_hint, cfg, latent, slots_host);
}

int cbp_decode_run_host_q(cbp_ctx* ctx, const void* pub_codes, const void* prv_codes, int bits, int n_frames,
                          int channels, int rows, int cols, const int* recover, int width_hint,
                          const cbp_decode_cfg* cfg, float* latent, cbp_kernel_slot* slots_host) {
  cbp_host::DeviceGuard device_guard(ctx);
  if (bits != 8 && bits != 16) return ctx ? set_error(ctx, CBP_INVALID_ARGUMENT, "quantization depth must be u8 or u16")
                                          : CBP_INVALID_ARGUMENT;
  return run_host(ctx, pub_codes, prv_codes, bits, n_frames, channels, rows, cols, recover, width_hint, cfg, latent,
                  slots_host);
}

}  // extern "C"
