// Host-buffer decode pipeline (the end-to-end path): the reference CLI decodes a run
// of frames held in host memory (tools/cbp.cpp:130-207). Here H2D copies, device
// decode and D2H copies of consecutive frames overlap on three streams through a
// ring of device frame buffers; recovered kernels stay on the device (slots) and are
// reused by the following frames (spectral_deblur_slot), with no host round trip.
#include <cstring>
#include <string>
#include <vector>

#include "cbp_ctx.cuh"

namespace {
constexpr int kRing = 3;

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

int cbp_decode_run_host(cbp_ctx* ctx, const float* pub, const float* prv, int n_frames, int channels, int rows,
                        int cols, const int* recover, int width_hint, const cbp_decode_cfg* cfg, float* latent,
                        cbp_kernel_slot* slots_host) {
  if (!ctx || !pub || !recover || !cfg || !latent) return CBP_INVALID_ARGUMENT;
  if (n_frames <= 0) return 0;
  if (!recover[0]) return set_error(ctx, CBP_INVALID_ARGUMENT, "the first frame of a run must recover the kernel");
  int n_rec = 0;
  for (int j = 0; j < n_frames; ++j) n_rec += recover[j] ? 1 : 0;
  if (n_rec > 0 && !prv) return set_error(ctx, CBP_INVALID_ARGUMENT, "recovery frames need the private stream");
  Pipe& P = pipe_of(ctx);
  const size_t frame = size_t(channels) * rows * cols;
  float* dpub = static_cast<float*>(workspace(ctx, WS_PUB, sizeof(float) * frame * kRing));
  float* dprv = static_cast<float*>(workspace(ctx, WS_PRV, sizeof(float) * frame * kRing));
  float* dout = static_cast<float*>(workspace(ctx, WS_OUT, sizeof(float) * frame * kRing));
  cbp_kernel_slot* slots = static_cast<cbp_kernel_slot*>(workspace(ctx, WS_SOLVE, sizeof(cbp_kernel_slot) * n_rec));
  if (!dpub || !dprv || !dout || !slots) return set_error(ctx, CBP_CUDA_ERROR, "pipeline allocation failed");
  int rec = -1;
  const int hint = width_hint;
  for (int j = 0; j < n_frames; ++j) {
    const int r = j % kRing;
    if (j >= kRing) cudaStreamWaitEvent(P.h2d, P.out[r], 0);  // ring slot drained
    cudaMemcpyAsync(dpub + r * frame, pub + j * frame, sizeof(float) * frame, cudaMemcpyHostToDevice, P.h2d);
    if (recover[j])
      cudaMemcpyAsync(dprv + r * frame, prv + j * frame, sizeof(float) * frame, cudaMemcpyHostToDevice, P.h2d);
    cudaEventRecord(P.in[r], P.h2d);
    cudaStreamWaitEvent(P.comp, P.in[r], 0);
    int st;
    if (recover[j]) {
      ++rec;
      st = cbp_decode_frames_async(ctx, dpub + r * frame, dprv + r * frame, 1, channels, rows, cols, cols,
                                   hint > 0 ? &hint : nullptr, cfg, dout + r * frame, cols, slots + rec, P.comp);
    } else {
      st = cbp_spectral_deblur_slot(ctx, dpub + r * frame, 1, channels, rows, cols, cols, slots + rec,
                                    dout + r * frame, cols, P.comp);
    }
    if (st) return st;
    cudaEventRecord(P.done[r], P.comp);
    cudaStreamWaitEvent(P.d2h, P.done[r], 0);
    cudaMemcpyAsync(latent + j * frame, dout + r * frame, sizeof(float) * frame, cudaMemcpyDeviceToHost, P.d2h);
    cudaEventRecord(P.out[r], P.d2h);
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

}  // extern "C"
