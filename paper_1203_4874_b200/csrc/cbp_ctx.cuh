// Host-side context shared by the C-ABI translation units.
#pragma once

#include <cstdlib>
#include <map>
#include <mutex>
#include <string>
#include <vector>

#include "cbp_deblur.cuh"
#include "cbp_fft.cuh"

struct cbp_ctx {
  int device = 0;
  std::string err;
  std::map<int, float2*> tw;  // n -> exp(-2 pi i k / n), k < n (device, FP64-rounded)
  // device workspaces, grown on demand (never inside a launch sequence)
  void* ws[20] = {};
  size_t ws_bytes[20] = {};
  cbp_kernel_slot* host_slot = nullptr;  // pinned staging
  cudaEvent_t ev[8] = {};
  int num_sms = 148;
  int sm_reserve = 0;  // cbp_set_sm_reserve
  int chain = 1;       // cbp_set_launch_chaining
  void* slot_event = nullptr;  // cudaEvent_t recorded when the kernel slots are final (_async_ev)
  // optional per-pass timing of the deconvolution (cbp_profile)
  int prof = 0;
  std::vector<cudaEvent_t> prof_ev;
  int prof_used = 0;
  long long prof_planes = 0;
  long long launches = 0;  // kernels enqueued by this context
  unsigned* tile_ctr = nullptr;  // dynamic-tile counters of the deconvolution passes (device), 4 per side stream
  // side streams of the deconvolution (launch groups alternate between them, so one group's
  // launch tails overlap the next group's passes); created on first use
  static constexpr int kSideStreams = 4;
  cudaStream_t side[kSideStreams] = {};
  cudaEvent_t side_ev[kSideStreams + 1] = {};
  // stream ordering of the context's shared scratch: the last stream that enqueued work and
  // an event recorded there; a call on another stream first waits on it (StreamOrder)
  cudaEvent_t order_ev = nullptr;
  cudaStream_t order_stream = nullptr;
  bool order_valid = false;
};

namespace cbp_host {

// Makes ctx's device current for the duration of a C-ABI call (restored on return), so a
// thread can drive contexts of several GPUs and a context never allocates or launches on
// whatever device the calling thread happened to have current.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(const cbp_ctx* ctx) {
    if (ctx && cudaGetDevice(&prev) == cudaSuccess && prev != ctx->device) cudaSetDevice(ctx->device);
    else prev = -1;
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DeviceGuard(const DeviceGuard&) = delete;
  DeviceGuard& operator=(const DeviceGuard&) = delete;
};

// A context's workspaces, Wiener tables, tile counters and staging slot are shared by all its
// calls. Work enqueued on a new stream first waits for the work the context enqueued on the
// previous stream (an event), so using one context from several streams serializes instead
// of racing on the scratch; one context per stream keeps them concurrent.
struct StreamOrder {
  cbp_ctx* c;
  cudaStream_t s;
  StreamOrder(cbp_ctx* ctx, void* stream) : c(ctx), s(static_cast<cudaStream_t>(stream)) {
    static const bool off = getenv("CBP_NO_STREAM_ORDER") != nullptr;  // A/B switch
    if (off) c = nullptr;
    if (c && c->order_ev && c->order_valid && c->order_stream != s) cudaStreamWaitEvent(s, c->order_ev, 0);
  }
  ~StreamOrder() {
    if (c && c->order_ev) {
      cudaEventRecord(c->order_ev, s);
      c->order_stream = s;
      c->order_valid = true;
    }
  }
  StreamOrder(const StreamOrder&) = delete;
  StreamOrder& operator=(const StreamOrder&) = delete;
};

enum Workspace {
  WS_X = 0,       // deconvolution half spectrum
  WS_SLOTS = 1,   // kernel slots owned by the context
  WS_PART = 2,    // fold partial sums
  WS_FOLD = 3,    // folds
  WS_SLICES = 4,  // unit-circle slices
  WS_SOLVE = 5,   // cofactor solutions
  WS_MISC = 6,
  WS_PUB = 7,     // host-pipeline staging
  WS_PRV = 8,
  WS_OUT = 9,
  WS_RED = 10,    // validation partial sums
  // 11, 12: Wiener filter tables (WS_RED + 1, WS_RED + 2)
  WS_QPUB = 13,   // dequantized frames (cbp_decode_frames_q)
  WS_QPRV = 14,
  WS_QCODES = 15, // host-pipeline code rings (cbp_decode_run_host_q)
  WS_FUSED = 16,  // fused deconvolution ticket and per-plane completion counters
};

const char* errc_name(int status);
int set_error(cbp_ctx* ctx, int status, const std::string& msg);
int cuda_check(cbp_ctx* ctx, cudaError_t e, const char* what);
void* workspace(cbp_ctx* ctx, int id, size_t bytes);
const float2* twiddles(cbp_ctx* ctx, int n);
cbp_dev::FftPlan make_plan(int n);
int friendly_size(int n);

// Fills the deconvolution geometry (grid, plans, tables) for a Mb x Nb plane.
int deblur_setup(cbp_ctx* ctx, int Mb, int Nb, cbp_dev::DeblurArgs& a);
// Runs passes A/B/C over `planes` planes of one batch in L2-sized groups.
int deblur_run(cbp_ctx* ctx, cbp_dev::DeblurArgs a, int planes, size_t in_plane_stride,
               size_t out_plane_stride, cudaStream_t stream);

}  // namespace cbp_host
