// C ABI: decode_frame orchestration (reference decoder.cpp:280-378) and the
// stage-level entry points (decoder.hpp:29-86, poly.hpp:51-55, encoder.hpp:36-37).
// Every stage is a device kernel; the host only checks arguments, sizes workspaces,
// enqueues launches and formats the reference's error messages.
#include <cmath>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "cbp_ctx.cuh"
#include "cbp_recover.cuh"

using namespace cbp_dev;
using namespace cbp_host;

namespace {

constexpr int kDeviceMaxWidth = kWideMaxWidth;  // the reference's bound (decoder.cpp:32-33, 305-306)

const char* stage_name(int s) {
  switch (s) {
    case CBP_STAGE_POLYNOMIAL_EVALUATION: return "polynomial_evaluation";
    case CBP_STAGE_KERNEL_DEGREE_ESTIMATION: return "kernel_degree_estimation";
    case CBP_STAGE_KERNEL_ESTIMATION_1D: return "kernel_estimation_1d";
    case CBP_STAGE_KERNEL_ESTIMATION_2D_FFT: return "kernel_estimation_2d_fft";
    default: return "";
  }
}

std::string fmtd(double v) { return std::to_string(v); }  // std::to_string like the reference

// Inner message (what the failing reference function throws) for a slot failure.
std::string inner_message(const cbp_kernel_slot& s) {
  const std::string name = errc_name(s.status);
  const std::string ax = s.fail_axis == 1 ? "z2" : "z1";
  switch (s.fail_reason) {
    case CBP_REASON_GAP:  // decoder.cpp:108-109 wrapping poly.cpp:111-113
      return name + ": " + ax + " slice " + std::to_string(s.fail_slice) +
             ": IllConditioned: cofactor null space not one-dimensional (gap " + fmtd(s.fail_value) + ")";
    case CBP_REASON_VANISHING_COFACTOR:
      return name + ": " + ax + " slice " + std::to_string(s.fail_slice) + ": vanishing cofactor estimate";
    case CBP_REASON_SCALE_RATIO: return name + ": near-zero per-slice scale (ratio " + fmtd(s.fail_value) + ")";
    case CBP_REASON_SCALE_ZERO: return name + ": zero scale entry";
    case CBP_REASON_VANISHING_MASS: return name + ": kernel estimate has vanishing mass";
    case CBP_REASON_ZERO_KERNEL: return name + ": kernel estimate is zero";
    case CBP_REASON_IMAG_ENERGY: return name + ": imaginary energy fraction " + fmtd(s.fail_value);
    case CBP_REASON_NO_POSITIVE: return name + ": kernel estimate has no positive weight";
    case CBP_REASON_NEGATIVE_WEIGHT:
      return name + ": negative weight beyond tolerance (min " + fmtd(s.fail_value) + " of max)";
    case CBP_REASON_AXES_DISAGREE:
      return name + ": width estimates disagree: z1 gives " + std::to_string(s.width_z1) + ", z2 gives " +
             std::to_string(s.width_z2);
    case CBP_REASON_ZERO_POLY: return name + ": bezout of an all-zero polynomial";
    case CBP_REASON_NONFINITE: return name + ": frame contains non-finite samples";
    case CBP_REASON_TOO_SMALL: return name + ": frame smaller than the kernel width";
    case CBP_REASON_ZERO_PUBLIC: return name + ": public frame is identically zero";
    case CBP_REASON_SIGNED:
      return name + ": signed-content width search (decoder.cpp:65-82) is not implemented on the device";
    case CBP_REASON_WIDTH_LIMIT:
      return name + ": kernel width " + std::to_string(s.width) + " exceeds the device solver limit (" +
             std::to_string(kDeviceMaxWidth) + ")";
    default: return name + ": decode failed";
  }
}

// decode_frame rethrows stage errors as Error(code, "<stage>: " + what) (decoder.cpp:294-360)
std::string full_message(const cbp_kernel_slot& s) {
  std::string inner = inner_message(s);
  if (s.fail_stage >= CBP_STAGE_POLYNOMIAL_EVALUATION && s.fail_stage <= CBP_STAGE_KERNEL_ESTIMATION_2D_FFT)
    return std::string(errc_name(s.status)) + ": " + stage_name(s.fail_stage) + ": " + inner;
  return inner;
}

}  // namespace

// The reference's error text for a failed slot (what decode_frame would throw), for
// pipelines that read slots instead of cbp_decode_info.
extern "C" int cbp_slot_message(const cbp_kernel_slot* slot, char* buf, int len) {
  if (!slot) return CBP_INVALID_ARGUMENT;
  if (buf && len > 0) {
    const std::string m = slot->status == 0 ? std::string() : full_message(*slot);
    std::snprintf(buf, size_t(len), "%s", m.c_str());
  }
  return slot->status;
}

namespace {

int check_search(cbp_ctx* ctx, int smin, int smax) {  // decoder.cpp:31-34
  if (!(smin >= 3 && smax <= 63 && smin <= smax && smin % 2 == 1 && smax % 2 == 1))
    return set_error(ctx, CBP_INVALID_ARGUMENT, "width search range must be odd values within [3,63]");
  return 0;
}

int check_geometry(cbp_ctx* ctx, int batch, int channels, int rows, int cols, int ld) {
  if (batch < 0) return set_error(ctx, CBP_INVALID_ARGUMENT, "batch must be >= 0");
  if (!(channels == 1 || channels == 3)) return set_error(ctx, CBP_DIM_MISMATCH, "frame must have 1 or 3 planes");
  if (rows < 1 || cols < 1) return set_error(ctx, CBP_DIM_MISMATCH, "empty frame plane");
  if (ld < cols) return set_error(ctx, CBP_INVALID_ARGUMENT, "row pitch smaller than the row");
  return 0;
}

int check_kernel(cbp_ctx* ctx, const double* w, int t) {  // kernel.cpp:7-17
  if (!(t >= 1 && t % 2 == 1 && t <= CBP_MAX_WIDTH))
    return set_error(ctx, CBP_INVALID_ARGUMENT, "kernel width must be odd and >= 1");
  double s = 0.0;
  for (int i = 0; i < t * t; ++i) {
    if (!std::isfinite(w[i])) return set_error(ctx, CBP_INVALID_ARGUMENT, "kernel weights must be finite");
    if (w[i] < 0.0) return set_error(ctx, CBP_INVALID_ARGUMENT, "kernel weights must be nonnegative");
  }
  for (int n = 0; n < t; ++n)
    for (int m = 0; m < t; ++m) s += w[m * t + n];
  if (std::abs(s - 1.0) > 1e-9) return set_error(ctx, CBP_INVALID_ARGUMENT, "kernel weights must sum to 1");
  return 0;
}

template <class T>
T* ws(cbp_ctx* ctx, int id, size_t count) {
  return static_cast<T*>(workspace(ctx, id, count * sizeof(T)));
}

// All per-batch device workspaces carved from WS_MISC.
struct RecoverPlan {
  RecoverArgs a;
  double* vpart = nullptr;
  int vtiles = 0;
};

int plan_recover(cbp_ctx* ctx, RecoverPlan& P, const float* pub, const float* prv, int batch, int channels,
                 int rows, int cols, int ld, int t_max, int smin, int smax, double tau, int trust_hint,
                 const cbp_decode_cfg* cfg, bool want_validate) {
  RecoverArgs& a = P.a;
  std::memset(&a, 0, sizeof(a));
  a.pub = pub;
  a.prv = prv;
  a.batch = batch;
  a.channels = channels;
  a.rows = rows;
  a.cols = cols;
  a.ld = ld;
  a.t_max = t_max;
  a.lmax = std::max(rows, cols);
  fold_plan(batch, rows, cols, t_max, a.ncb, a.fold_rh, a.part_stride);
  a.search_min = smin;
  a.search_max = smax;
  a.nsizes = smax >= smin ? (smax - smin) / 2 + 1 : 0;
  a.tau = tau;
  a.chain = ctx->chain;
  a.trust_hint = trust_hint;
  a.gap_threshold = cfg ? cfg->gap_threshold : 1e-9;
  a.max_imag_energy = cfg ? cfg->max_imag_energy : 0.01;
  a.negative_weight_tol = cfg ? cfg->negative_weight_tol : 0.01;
  a.has_epsilon = cfg ? cfg->has_epsilon : 0;
  a.epsilon = cfg ? cfg->epsilon : 0.0;
  const size_t B = size_t(batch), T = size_t(t_max), L = size_t(a.lmax);
  // the tile count is largest for the widest kernel the batch allows
  P.vtiles = want_validate ? validate_tiles(rows, cols, std::min(t_max, kDeviceMaxWidth)) : 0;
  // carve one allocation (256-byte aligned pieces)
  size_t off = 0;
  auto take = [&](size_t bytes) {
    size_t o = off;
    off += (bytes + 255) & ~size_t(255);
    return o;
  };
  const size_t o_part = take(B * 2 * a.part_stride * sizeof(double));
  const size_t o_part2 = take(B * 2 * a.ncb * T * rows * sizeof(double));
  const size_t o_slices = take(B * 4 * T * L * sizeof(double2));
  const size_t o_values = take(B * 2 * T * T * sizeof(double2));
  const size_t o_gaps = take(B * 2 * T * sizeof(double));
  const size_t o_sstat = take(B * 2 * T * sizeof(int));
  const size_t o_scratch = take(B * 2 * T * (L + T) * sizeof(double2));
  const size_t o_ratios = take(B * 2 * std::max(a.nsizes, 1) * sizeof(double));
  const size_t o_flags = take(B * sizeof(int));
  const size_t o_vpart = take(B * channels * std::max(P.vtiles, 1) * sizeof(double2) + 64);
  const size_t o_roots = take(size_t(rows + cols) * sizeof(double2));
  const size_t o_epart = take(signed_energy_doubles(batch, rows, cols) * sizeof(double));
  // widths above the shared-memory solvers: per-CTA global scratch (k_solve_wide, k_compose_wide)
  a.wide_ctas = t_max > kSmemMaxWidth ? 64 : 0;
  a.wide_stride = wide_scratch_elems();
  const size_t o_wide = take(size_t(a.wide_ctas) * a.wide_stride * sizeof(double2));
  char* base = static_cast<char*>(workspace(ctx, WS_MISC, off));
  if (!base) return set_error(ctx, CBP_CUDA_ERROR, "workspace allocation failed");
  a.part = reinterpret_cast<double*>(base + o_part);
  a.part2 = reinterpret_cast<double*>(base + o_part2);
  a.slices = reinterpret_cast<double2*>(base + o_slices);
  a.values = reinterpret_cast<double2*>(base + o_values);
  a.gaps = reinterpret_cast<double*>(base + o_gaps);
  a.slice_status = reinterpret_cast<int*>(base + o_sstat);
  a.scratch = reinterpret_cast<double2*>(base + o_scratch);
  a.ratios = reinterpret_cast<double*>(base + o_ratios);
  a.flags = reinterpret_cast<int*>(base + o_flags);
  P.vpart = reinterpret_cast<double*>(base + o_vpart);
  a.roots = reinterpret_cast<double2*>(base + o_roots);
  a.epart = reinterpret_cast<double*>(base + o_epart);
  a.wide = a.wide_ctas ? reinterpret_cast<double2*>(base + o_wide) : nullptr;
  a.epart_z2 = size_t(batch) * 2 * ((cols + 31) / 32) * (rows / 2 + 1);  // z1 part (cbp_signed.cu)
  return 0;
}

// pinned host staging, grown on demand
template <class T>
T* pinned(cbp_ctx* ctx, size_t count) {
  static thread_local std::vector<std::pair<cbp_ctx*, std::pair<void*, size_t>>> pool;
  for (auto& e : pool)
    if (e.first == ctx && e.second.second >= count * sizeof(T)) return static_cast<T*>(e.second.first);
  for (auto it = pool.begin(); it != pool.end(); ++it)
    if (it->first == ctx) {
      cudaFreeHost(it->second.first);
      pool.erase(it);
      break;
    }
  void* p = nullptr;
  if (cudaMallocHost(&p, std::max<size_t>(count * sizeof(T), 64)) != cudaSuccess) return nullptr;
  pool.push_back({ctx, {p, std::max<size_t>(count * sizeof(T), 64)}});
  return static_cast<T*>(p);
}

// Enqueues the whole decode for a batch (no synchronization).
// stages: which parts of decode_frame (decoder.cpp:280-378) to enqueue
constexpr int kStageRecover = 1, kStageDeblur = 2, kStageValidate = 4, kStageAll = 7;
int enqueue_decode(cbp_ctx* ctx, const float* pub, const float* prv, int batch, int channels, int rows, int cols,
                   int ld, const int* hints, const cbp_decode_cfg* cfg, float* latent, int ld_out,
                   cbp_kernel_slot* slots, cudaStream_t s, bool record_events, int stages = kStageAll) {
  int st;
  if ((st = check_geometry(ctx, batch, channels, rows, cols, ld))) return st;
  if (ld_out < cols) return set_error(ctx, CBP_INVALID_ARGUMENT, "output row pitch smaller than the row");
  if ((st = check_search(ctx, cfg->search_min, cfg->search_max))) return st;
  if (!(cfg->tau > 0.0 && cfg->tau < 1.0)) return set_error(ctx, CBP_INVALID_ARGUMENT, "tau must lie in (0,1)");
  bool need_est = false;
  int t_max = 1;
  for (int b = 0; b < batch; ++b) {
    const int h = hints ? hints[b] : 0;
    if (h > 0 && h % 2 == 0)  // check_pair, decoder.cpp:26-28
      return set_error(ctx, CBP_INVALID_ARGUMENT, "kernel width hint must be odd and >= 1");
    if (cfg->trust_hint && h > 0) {
      if (h > 63)
        return set_error(ctx, CBP_INVALID_ARGUMENT,
                         "kernel_degree_estimation: InvalidArgument: kernel width hint must be odd, within [1,63]");
      if (rows < h || cols < h)
        return set_error(ctx, CBP_FRAME_TOO_SMALL,
                         "polynomial_evaluation: FrameTooSmall: frame smaller than the kernel width");
      t_max = std::max(t_max, h);
    } else {
      need_est = true;
    }
  }
  if (need_est) {
    if (!(std::min(rows, cols) > cfg->search_max))  // decoder.cpp:47
      return set_error(ctx, CBP_FRAME_TOO_SMALL,
                       "kernel_degree_estimation: FrameTooSmall: frame too small for the width search bound");
    t_max = std::max(t_max, cfg->search_max);
  }
  if (cfg->has_epsilon && !(cfg->epsilon >= 0.0))
    return set_error(ctx, CBP_INVALID_ARGUMENT,
                     "kernel_estimation_2d_fft: InvalidArgument: epsilon must be nonnegative");
  if (batch == 0) return 0;
  const int t_solve = std::min(t_max, kDeviceMaxWidth);
  RecoverPlan P;
  if ((st = plan_recover(ctx, P, pub, prv, batch, channels, rows, cols, ld, t_max, cfg->search_min,
                         cfg->search_max, cfg->tau, cfg->trust_hint, cfg, cfg->validate != 0)))
    return st;
  RecoverArgs& a = P.a;
  a.slots = slots;
  if (record_events) cudaEventRecord(ctx->ev[0], s);
  cudaError_t e = launch_init_slots(a, hints, s);
  ctx->launches += (batch + HintChunk::kMax - 1) / HintChunk::kMax;
  if (e == cudaSuccess && need_est) e = launch_fold(a, 1, s);  // DC slices (decoder.cpp:58-64)
  if (e == cudaSuccess && need_est) e = launch_signed_slices(a, s);  // signed content (65-82)
  if (e == cudaSuccess && need_est) e = launch_width(a, s);
  if (need_est) ctx->launches += 5;
  if (record_events) cudaEventRecord(ctx->ev[1], s);
  // widths <= 31 solve in shared memory, wider ones (<= 63) on the per-CTA global scratch
  if (e == cudaSuccess) e = launch_fold(a, 0, s);  // axis_roots_dft x4 (decoder.cpp:323-326)
  ctx->launches += 5;  // fold x3, solve, compose
  if (record_events) cudaEventRecord(ctx->ev[2], s);
  if (e == cudaSuccess) e = launch_solve(a, s);
  if (record_events) cudaEventRecord(ctx->ev[3], s);
  if (e == cudaSuccess) e = launch_compose(a, s);
  if ((st = cuda_check(ctx, e, "recovery launch"))) return st;
  // kernels, widths and epsilons are final here; the frame's own deconvolution and the
  // validation residual follow on this stream, consumers of the slots need not wait for them
  if (ctx->slot_event) cudaEventRecord(static_cast<cudaEvent_t>(ctx->slot_event), s);
  if (!(stages & kStageDeblur)) return 0;  // cbp_recover_kernels_async
  DeblurArgs d;
  if ((st = deblur_setup(ctx, rows, cols, d))) return st;
  d.in = pub;
  d.in_ld = ld;
  d.out = latent;
  d.out_ld = ld_out;
  d.slot = slots;
  d.slot_per_frame = 1;
  d.channels = channels;
  if ((st = deblur_run(ctx, d, batch * channels, size_t(rows) * ld, size_t(rows) * ld_out, s))) return st;
  if (record_events) cudaEventRecord(ctx->ev[4], s);
  if (cfg->validate && (stages & kStageValidate)) {
    a.pub = pub;
    if ((st = cuda_check(ctx, launch_validate(a, latent, ld_out, P.vpart, P.vtiles, s), "validation launch")))
      return st;
    ctx->launches += 2;
  }
  (void)t_solve;
  return 0;
}

void fill_info(const cbp_kernel_slot& s, cbp_decode_info& info) {
  std::memset(&info, 0, sizeof(info));
  info.status = s.status;
  info.fail_stage = s.fail_stage;
  info.fail_axis = s.fail_axis;
  info.fail_slice = s.fail_slice;
  info.width_used = s.width;
  info.width_clamped = s.clamped;
  info.validation_residual = s.residual;
  info.epsilon_used = s.epsilon;
  info.fail_value = s.fail_value;
  if (s.status == 0 && s.width > 0 && s.width <= CBP_MAX_WIDTH)
    std::memcpy(info.kernel, s.weights, sizeof(double) * s.width * s.width);
}

}  // namespace

extern "C" {

int cbp_decode_frames_async(cbp_ctx* ctx, const float* pub_dev, const float* prv_dev, int batch, int channels,
                            int rows, int cols, int ld, const int* width_hints, const cbp_decode_cfg* cfg,
                            float* latent_dev, int ld_out, cbp_kernel_slot* slots_dev, void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx || !cfg || !slots_dev) return CBP_INVALID_ARGUMENT;
  return enqueue_decode(ctx, pub_dev, prv_dev, batch, channels, rows, cols, ld, width_hints, cfg, latent_dev,
                        ld_out, slots_dev, static_cast<cudaStream_t>(stream), false);
}

int cbp_recover_kernels_async(cbp_ctx* ctx, const float* pub_dev, const float* prv_dev, int batch, int channels,
                              int rows, int cols, int ld, const int* width_hints, const cbp_decode_cfg* cfg,
                              cbp_kernel_slot* slots_dev, void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx || !cfg || !slots_dev) return CBP_INVALID_ARGUMENT;
  return enqueue_decode(ctx, pub_dev, prv_dev, batch, channels, rows, cols, ld, width_hints, cfg, nullptr, ld,
                        slots_dev, static_cast<cudaStream_t>(stream), false, kStageRecover);
}

int cbp_validate_frames_async(cbp_ctx* ctx, const float* pub_dev, const float* latent_dev, int batch, int channels,
                              int rows, int cols, int ld, int ld_out, cbp_kernel_slot* slots_dev, void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx || !slots_dev || !latent_dev) return CBP_INVALID_ARGUMENT;
  int st;
  if ((st = check_geometry(ctx, batch, channels, rows, cols, ld))) return st;
  if (ld_out < cols) return set_error(ctx, CBP_INVALID_ARGUMENT, "output row pitch smaller than the row");
  if (batch == 0) return 0;
  RecoverArgs a;
  std::memset(&a, 0, sizeof(a));
  a.pub = pub_dev;
  a.batch = batch;
  a.channels = channels;
  a.rows = rows;
  a.cols = cols;
  a.ld = ld;
  a.t_max = kDeviceMaxWidth;  // slot widths are <= 63
  a.slots = slots_dev;
  const int vtiles = validate_tiles(rows, cols, kDeviceMaxWidth);
  double* vpart = ws<double>(ctx, WS_RED, size_t(2) * batch * channels * vtiles + 8);
  if (!vpart) return set_error(ctx, CBP_CUDA_ERROR, "workspace allocation failed");
  st = cuda_check(ctx, launch_validate(a, latent_dev, ld_out, vpart, vtiles, static_cast<cudaStream_t>(stream)),
                  "validation launch");
  ctx->launches += 2;
  return st;
}

int cbp_decode_frames_async_ev(cbp_ctx* ctx, const float* pub_dev, const float* prv_dev, int batch, int channels,
                               int rows, int cols, int ld, const int* width_hints, const cbp_decode_cfg* cfg,
                               float* latent_dev, int ld_out, cbp_kernel_slot* slots_dev, void* stream,
                               void* slot_ready_event) {
  cbp_host::DeviceGuard device_guard(ctx);
  if (!ctx || !cfg || !slots_dev) return CBP_INVALID_ARGUMENT;
  ctx->slot_event = slot_ready_event;
  const int st = enqueue_decode(ctx, pub_dev, prv_dev, batch, channels, rows, cols, ld, width_hints, cfg,
                                latent_dev, ld_out, slots_dev, static_cast<cudaStream_t>(stream), false);
  ctx->slot_event = nullptr;
  return st;
}

int cbp_decode_frames(cbp_ctx* ctx, const float* pub_dev, const float* prv_dev, int batch, int channels, int rows,
                      int cols, int ld, const int* width_hints, const cbp_decode_cfg* cfg, float* latent_dev,
                      int ld_out, cbp_decode_info* info, void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx || !cfg) return CBP_INVALID_ARGUMENT;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cbp_kernel_slot* slots = ws<cbp_kernel_slot>(ctx, WS_SLOTS, std::max(batch, 64));
  if (!slots) return set_error(ctx, CBP_CUDA_ERROR, "workspace allocation failed");
  int st = enqueue_decode(ctx, pub_dev, prv_dev, batch, channels, rows, cols, ld, width_hints, cfg, latent_dev,
                          ld_out, slots, s, true);
  if (st) return st;
  if (batch == 0) return 0;
  cbp_kernel_slot* h = pinned<cbp_kernel_slot>(ctx, size_t(batch));
  if (!h) return set_error(ctx, CBP_CUDA_ERROR, "pinned allocation failed");
  cudaMemcpyAsync(h, slots, sizeof(cbp_kernel_slot) * batch, cudaMemcpyDeviceToHost, s);
  if ((st = cuda_check(ctx, cudaStreamSynchronize(s), "decode"))) return st;
  float ms[4] = {0, 0, 0, 0}, total = 0;
  cudaEventElapsedTime(&ms[0], ctx->ev[1], ctx->ev[2]);  // polynomial_evaluation
  cudaEventElapsedTime(&ms[1], ctx->ev[0], ctx->ev[1]);  // kernel_degree_estimation
  cudaEventElapsedTime(&ms[2], ctx->ev[2], ctx->ev[3]);  // kernel_estimation_1d
  cudaEventElapsedTime(&ms[3], ctx->ev[3], ctx->ev[4]);  // kernel_estimation_2d_fft
  cudaEventElapsedTime(&total, ctx->ev[0], ctx->ev[4]);
  int first = -1;
  for (int b = 0; b < batch; ++b) {
    if (info) {
      fill_info(h[b], info[b]);
      for (int k = 0; k < 4; ++k) info[b].stage_ms[k] = ms[k];
      info[b].stage_ms[4] = total;
    }
    if (h[b].status != 0 && first < 0) first = b;
  }
  if (first >= 0) {
    ctx->err = full_message(h[first]);
    return h[first].status;
  }
  return 0;
}

int cbp_estimate_kernel_width(cbp_ctx* ctx, const float* pub_dev, const float* prv_dev, int channels, int rows,
                              int cols, int ld, int search_min, int search_max, double tau, int* width,
                              int* clamped, void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx) return CBP_INVALID_ARGUMENT;
  int st;
  if ((st = check_geometry(ctx, 1, channels, rows, cols, ld))) return st;
  if ((st = check_search(ctx, search_min, search_max))) return st;
  if (!(tau > 0.0 && tau < 1.0)) return set_error(ctx, CBP_INVALID_ARGUMENT, "tau must lie in (0,1)");
  if (!(std::min(rows, cols) > search_max))
    return set_error(ctx, CBP_FRAME_TOO_SMALL, "frame too small for the width search bound");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cbp_decode_cfg cfg;
  cbp_decode_cfg_default(&cfg);
  RecoverPlan P;
  if ((st = plan_recover(ctx, P, pub_dev, prv_dev, 1, channels, rows, cols, ld, search_max, search_min,
                         search_max, tau, 0, &cfg, false)))
    return st;
  cbp_kernel_slot* slots = ws<cbp_kernel_slot>(ctx, WS_SLOTS, 64);
  P.a.slots = slots;
  cudaError_t e = launch_init_slots(P.a, nullptr, s);
  if (e == cudaSuccess) e = launch_fold(P.a, 1, s);
  if (e == cudaSuccess) e = launch_signed_slices(P.a, s);
  if (e == cudaSuccess) e = launch_width(P.a, s);
  if ((st = cuda_check(ctx, e, "width launch"))) return st;
  cbp_kernel_slot* h = pinned<cbp_kernel_slot>(ctx, 1);
  cudaMemcpyAsync(h, slots, sizeof(cbp_kernel_slot), cudaMemcpyDeviceToHost, s);
  if ((st = cuda_check(ctx, cudaStreamSynchronize(s), "width"))) return st;
  if (h->status) {
    ctx->err = inner_message(*h);
    return h->status;
  }
  *width = h->width;
  *clamped = h->clamped;
  return 0;
}

int cbp_sample_slices(cbp_ctx* ctx, const float* pub_dev, const float* prv_dev, int channels, int rows, int cols,
                      int ld, int t, int axis, double* slices_pub, double* slices_prv, void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx) return CBP_INVALID_ARGUMENT;
  int st;
  if ((st = check_geometry(ctx, 1, channels, rows, cols, ld))) return st;
  if (t < 1) return set_error(ctx, CBP_INVALID_ARGUMENT, "axis_roots_dft needs t >= 1");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cbp_decode_cfg cfg;
  cbp_decode_cfg_default(&cfg);
  RecoverPlan P;
  if ((st = plan_recover(ctx, P, pub_dev, prv_dev, 1, channels, rows, cols, ld, t, 3, 3, 0.5, 0, &cfg, false)))
    return st;
  cbp_kernel_slot* slots = ws<cbp_kernel_slot>(ctx, WS_SLOTS, 64);
  P.a.slots = slots;
  cudaError_t e = launch_init_slots(P.a, nullptr, s);
  if (e == cudaSuccess) e = launch_fold(P.a, t, s);
  if ((st = cuda_check(ctx, e, "fold launch"))) return st;
  const int L = axis == 0 ? cols : rows;
  for (int q = 0; q < 2; ++q)
    cudaMemcpy2DAsync(q ? slices_prv : slices_pub, sizeof(double2) * L,
                      P.a.slices + slice_offset(P.a, 0, axis, q, 0), sizeof(double2) * P.a.lmax,
                      sizeof(double2) * L, t, cudaMemcpyDeviceToHost, s);
  return cuda_check(ctx, cudaStreamSynchronize(s), "fold");
}

int cbp_sample_cofactors(cbp_ctx* ctx, const float* pub_dev, const float* prv_dev, int channels, int rows,
                         int cols, int ld, int width, int axis, double gap_threshold, double* values,
                         double* gaps, void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx) return CBP_INVALID_ARGUMENT;
  int st;
  if ((st = check_geometry(ctx, 1, channels, rows, cols, ld))) return st;
  if (!(width >= 1 && width % 2 == 1)) return set_error(ctx, CBP_INVALID_ARGUMENT, "width must be odd and >= 1");
  if (rows < width || cols < width)
    return set_error(ctx, CBP_FRAME_TOO_SMALL, "frame smaller than the kernel width");
  if (width > kDeviceMaxWidth)
    return set_error(ctx, CBP_UNSUPPORTED, "kernel width exceeds the device solver limit (63)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cbp_decode_cfg cfg;
  cbp_decode_cfg_default(&cfg);
  cfg.gap_threshold = gap_threshold;
  RecoverPlan P;
  if ((st = plan_recover(ctx, P, pub_dev, prv_dev, 1, channels, rows, cols, ld, width, 3, 3, 0.5, 1, &cfg,
                         false)))
    return st;
  cbp_kernel_slot* slots = ws<cbp_kernel_slot>(ctx, WS_SLOTS, 64);
  P.a.slots = slots;
  const int hint = width;
  cudaError_t e = launch_init_slots(P.a, &hint, s);
  if (e == cudaSuccess) e = launch_fold(P.a, 0, s);
  if (e == cudaSuccess) e = launch_solve(P.a, s);
  if ((st = cuda_check(ctx, e, "solve launch"))) return st;
  std::vector<double2> vals(size_t(width) * width);
  std::vector<double> g(width);
  std::vector<int> ss(width);
  const size_t base = size_t(axis) * P.a.t_max;
  cudaMemcpyAsync(vals.data(), P.a.values + base * P.a.t_max, sizeof(double2) * width * width,
                  cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(g.data(), P.a.gaps + base, sizeof(double) * width, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(ss.data(), P.a.slice_status + base, sizeof(int) * width, cudaMemcpyDeviceToHost, s);
  cbp_kernel_slot* h = pinned<cbp_kernel_slot>(ctx, 1);
  cudaMemcpyAsync(h, slots, sizeof(cbp_kernel_slot), cudaMemcpyDeviceToHost, s);
  if ((st = cuda_check(ctx, cudaStreamSynchronize(s), "solve"))) return st;
  if (h->status) {
    ctx->err = inner_message(*h);
    return h->status;
  }
  for (int i = 0; i < width; ++i)
    if (ss[i]) {  // first failing slice (decoder.cpp:100-110)
      cbp_kernel_slot f{};
      f.status = CBP_ILL_CONDITIONED_SLICE;
      f.fail_axis = axis;
      f.fail_slice = i;
      f.fail_reason = ss[i];
      f.fail_value = g[i];
      ctx->err = inner_message(f);
      return f.status;
    }
  std::memcpy(values, vals.data(), sizeof(double2) * width * width);
  std::memcpy(gaps, g.data(), sizeof(double) * width);
  return 0;
}

int cbp_cofactor_solve_batch(cbp_ctx* ctx, const double* p, const double* q, int batch, int len, int t,
                             double gap_threshold, double* k1, double* k2, double* gaps, int* status, void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx) return CBP_INVALID_ARGUMENT;
  if (t < 1) return set_error(ctx, CBP_INVALID_ARGUMENT, "cofactor width must be >= 1");
  if (len < t) return set_error(ctx, CBP_INVALID_ARGUMENT, "slice degree below cofactor degree");
  if (t > kDeviceMaxWidth) return set_error(ctx, CBP_UNSUPPORTED, "cofactor width exceeds the device limit (63)");
  if (batch <= 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t nb = size_t(batch);
  const size_t wide_bytes = t > kSmemMaxWidth ? nb * wide_scratch_elems() * sizeof(double2) : 0;
  const size_t bytes = (2 * nb * len + 2 * nb * t + nb * (len + t)) * sizeof(double2) + nb * (sizeof(double) + sizeof(int)) +
                       1024 + wide_bytes;
  char* base = static_cast<char*>(workspace(ctx, WS_SOLVE, bytes));
  if (!base) return set_error(ctx, CBP_CUDA_ERROR, "workspace allocation failed");
  double2* dp = reinterpret_cast<double2*>(base);
  double2* dq = dp + nb * len;
  double2* d1 = dq + nb * len;
  double2* d2 = d1 + nb * t;
  double2* sc = d2 + nb * t;
  double* dg = reinterpret_cast<double*>(sc + nb * (len + t));
  int* ds = reinterpret_cast<int*>(dg + nb);
  double2* wide = wide_bytes ? reinterpret_cast<double2*>(base + ((bytes - wide_bytes) & ~size_t(255))) : nullptr;
  cudaMemcpyAsync(dp, p, sizeof(double2) * nb * len, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(dq, q, sizeof(double2) * nb * len, cudaMemcpyHostToDevice, s);
  int st = cuda_check(ctx, launch_cofactor_batch(dp, len, dq, len, batch, t, gap_threshold, d1, d2, dg, ds, sc, wide, s),
                      "cofactor launch");
  if (st) return st;
  cudaMemcpyAsync(k1, d1, sizeof(double2) * nb * t, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(k2, d2, sizeof(double2) * nb * t, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(gaps, dg, sizeof(double) * nb, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(status, ds, sizeof(int) * nb, cudaMemcpyDeviceToHost, s);
  if ((st = cuda_check(ctx, cudaStreamSynchronize(s), "cofactor solve"))) return st;
  for (int b = 0; b < batch; ++b)
    if (status[b]) {
      ctx->err = "IllConditioned: cofactor null space not one-dimensional (gap " + fmtd(gaps[b]) + ")";
      return status[b];
    }
  return 0;
}

int cbp_complete_to_spectrum(cbp_ctx* ctx, const double* values, int t, int axis, double* out, void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx) return CBP_INVALID_ARGUMENT;
  if (t < 1) return set_error(ctx, CBP_DIM_MISMATCH, "scaled kernel transform must be square");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double2* d = ws<double2>(ctx, WS_SOLVE, size_t(2) * t * t);
  cudaMemcpyAsync(d, values, sizeof(double2) * t * t, cudaMemcpyHostToDevice, s);
  int st = cuda_check(ctx, launch_complete(d, t, axis, d + t * t, s), "complete launch");
  if (st) return st;
  cudaMemcpyAsync(out, d + t * t, sizeof(double2) * t * t, cudaMemcpyDeviceToHost, s);
  return cuda_check(ctx, cudaStreamSynchronize(s), "complete");
}

int cbp_resolve_scales(cbp_ctx* ctx, const double* a_values, const double* b_values, int t, double* lambda,
                       double* mu, double* residual, void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx) return CBP_INVALID_ARGUMENT;
  if (t < 1) return set_error(ctx, CBP_DIM_MISMATCH, "transforms disagree on size");
  if (t > kDeviceMaxWidth) return set_error(ctx, CBP_UNSUPPORTED, "width exceeds the device limit (63)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t wide_off = (sizeof(double2) * (2 * t * t + 2 * t) + 64 + 255) & ~size_t(255);
  char* base = static_cast<char*>(workspace(ctx, WS_SOLVE, wide_off + (t > kSmemMaxWidth ? wide_scratch_elems() * sizeof(double2) : 0)));
  if (!base) return set_error(ctx, CBP_CUDA_ERROR, "workspace allocation failed");
  double2* wide = t > kSmemMaxWidth ? reinterpret_cast<double2*>(base + wide_off) : nullptr;
  double2* da = reinterpret_cast<double2*>(base);
  double2* db = da + t * t;
  double2* dl = db + t * t;
  double2* dm = dl + t;
  double* dr = reinterpret_cast<double*>(dm + t);
  int* dst = reinterpret_cast<int*>(dr + 2);
  cudaMemcpyAsync(da, a_values, sizeof(double2) * t * t, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(db, b_values, sizeof(double2) * t * t, cudaMemcpyHostToDevice, s);
  int st = cuda_check(ctx, launch_resolve(da, db, t, dl, dm, dr, dst, dr + 1, wide, s), "resolve launch");
  if (st) return st;
  double r[2];
  int status = 0;
  cudaMemcpyAsync(lambda, dl, sizeof(double2) * t, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(mu, dm, sizeof(double2) * t, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(r, dr, sizeof(double) * 2, cudaMemcpyDeviceToHost, s);
  cudaMemcpyAsync(&status, dst, sizeof(int), cudaMemcpyDeviceToHost, s);
  if ((st = cuda_check(ctx, cudaStreamSynchronize(s), "resolve"))) return st;
  *residual = r[0];
  if (status) {
    cbp_kernel_slot f{};
    f.status = status;
    f.fail_reason = CBP_REASON_SCALE_RATIO;
    f.fail_value = r[1];
    ctx->err = inner_message(f);
    return status;
  }
  return 0;
}

int cbp_assemble_kernel(cbp_ctx* ctx, const double* a_spectrum, const double* b_spectrum, const double* lambda,
                        const double* mu, int t, double max_imag_energy, double negative_weight_tol,
                        double* weights, void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx) return CBP_INVALID_ARGUMENT;
  if (t < 1) return set_error(ctx, CBP_DIM_MISMATCH, "spectrum estimates must be square and equal-sized");
  if (t > kDeviceMaxWidth) return set_error(ctx, CBP_UNSUPPORTED, "width exceeds the device limit (63)");
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const size_t wide_off = (sizeof(double2) * (2 * t * t + 2 * t) + sizeof(cbp_kernel_slot) + 64 + 255) & ~size_t(255);
  char* base = static_cast<char*>(workspace(ctx, WS_SOLVE, wide_off + (t > kSmemMaxWidth ? wide_scratch_elems() * sizeof(double2) : 0)));
  if (!base) return set_error(ctx, CBP_CUDA_ERROR, "workspace allocation failed");
  double2* wide = t > kSmemMaxWidth ? reinterpret_cast<double2*>(base + wide_off) : nullptr;
  double2* da = reinterpret_cast<double2*>(base);
  double2* db = da + t * t;
  double2* dl = db + t * t;
  double2* dm = dl + t;
  cbp_kernel_slot* slot = reinterpret_cast<cbp_kernel_slot*>(dm + t);
  cudaMemcpyAsync(da, a_spectrum, sizeof(double2) * t * t, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(db, b_spectrum, sizeof(double2) * t * t, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(dl, lambda, sizeof(double2) * t, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(dm, mu, sizeof(double2) * t, cudaMemcpyHostToDevice, s);
  int st = cuda_check(ctx, launch_assemble(da, db, dl, dm, t, max_imag_energy, negative_weight_tol, slot, wide, s),
                      "assemble launch");
  if (st) return st;
  cbp_kernel_slot* h = pinned<cbp_kernel_slot>(ctx, 1);
  cudaMemcpyAsync(h, slot, sizeof(cbp_kernel_slot), cudaMemcpyDeviceToHost, s);
  if ((st = cuda_check(ctx, cudaStreamSynchronize(s), "assemble"))) return st;
  if (h->status) {
    ctx->err = inner_message(*h);
    return h->status;
  }
  std::memcpy(weights, h->weights, sizeof(double) * t * t);
  return 0;
}

int cbp_validate_pair(cbp_ctx* ctx, const float* pub_dev, const float* prv_dev, int channels, int rows, int cols,
                      int ld, const double* k1, const double* k2, int t, double* residual, void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx) return CBP_INVALID_ARGUMENT;
  int st;
  if ((st = check_geometry(ctx, 1, channels, rows, cols, ld))) return st;
  if ((st = check_kernel(ctx, k1, t))) return st;
  if ((st = check_kernel(ctx, k2, t))) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  const int nt = validate_tiles(rows + t - 1, cols + t - 1, t);
  char* base = static_cast<char*>(
      workspace(ctx, WS_RED, sizeof(double2) * (size_t(nt) * channels + 2) + 2 * sizeof(double) * t * t + 256));
  double* part = reinterpret_cast<double*>(base);
  double* dk1 = part + 2 * (size_t(nt) * channels + 2);
  double* dk2 = dk1 + t * t;
  cudaMemcpyAsync(dk1, k1, sizeof(double) * t * t, cudaMemcpyHostToDevice, s);
  cudaMemcpyAsync(dk2, k2, sizeof(double) * t * t, cudaMemcpyHostToDevice, s);
  if ((st = cuda_check(ctx, launch_validate_pair(pub_dev, prv_dev, channels, rows, cols, ld, dk1, dk2, t, part, s),
                       "validate launch")))
    return st;
  double r = 0.0;
  cudaMemcpyAsync(&r, part + 2 * size_t(nt) * channels, sizeof(double), cudaMemcpyDeviceToHost, s);
  if ((st = cuda_check(ctx, cudaStreamSynchronize(s), "validate"))) return st;
  if (r < 0.0) return set_error(ctx, CBP_DEGENERATE_INPUT, "cross-convolution is identically zero");
  *residual = r;
  return 0;
}

int cbp_encode_frames(cbp_ctx* ctx, const float* latent_dev, int batch, int channels, int rows, int cols, int ld,
                      const double* k1, const double* k2, int t, float* pub_dev, float* prv_dev, int ld_out,
                      void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx) return CBP_INVALID_ARGUMENT;
  int st;
  if ((st = check_geometry(ctx, batch, channels, rows, cols, ld))) return st;
  if ((st = check_kernel(ctx, k1, t))) return st;
  if ((st = check_kernel(ctx, k2, t))) return st;
  if (rows < t || cols < t) return set_error(ctx, CBP_FRAME_TOO_SMALL, "latent frame smaller than the blur kernel");
  if (ld_out < cols + t - 1) return set_error(ctx, CBP_INVALID_ARGUMENT, "output row pitch too small");
  if (batch == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  double* dk = ws<double>(ctx, WS_RED, size_t(2) * t * t);
  double* hk = pinned<double>(ctx, size_t(2) * t * t);
  std::memcpy(hk, k1, sizeof(double) * t * t);
  std::memcpy(hk + t * t, k2, sizeof(double) * t * t);
  cudaMemcpyAsync(dk, hk, sizeof(double) * 2 * t * t, cudaMemcpyHostToDevice, s);
  cudaError_t e = launch_encode(latent_dev, batch * channels, rows, cols, ld, dk, t, pub_dev, ld_out, s);
  if (e == cudaSuccess) e = launch_encode(latent_dev, batch * channels, rows, cols, ld, dk + t * t, t, prv_dev, ld_out, s);
  st = cuda_check(ctx, e, "encode launch");
  if (st) return st;
  // the pinned staging buffer is reused by the next call: finish the upload first
  return cuda_check(ctx, cudaStreamSynchronize(s), "encode");
}

int cbp_synth_frames(cbp_ctx* ctx, float* out_dev, int planes, int rows, int cols, int ld, uint64_t seed,
                     void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx) return CBP_INVALID_ARGUMENT;
  return cuda_check(ctx, launch_synth(out_dev, planes, rows, cols, ld, seed, static_cast<cudaStream_t>(stream)),
                    "synth launch");
}

}  // extern "C"
