// C ABI: context, workspaces, FFT plans/tables and the fixed-kernel deconvolution
// entry points (reference decoder.cpp:273-278 spectral_deblur).
#include <cmath>
#include <cstdlib>
#include <cstdio>
#include <cstring>

#include "cbp_ctx.cuh"

using namespace cbp_dev;

namespace cbp_dev {
bool pdl_enabled() {
  static const bool on = getenv("CBP_NO_PDL") == nullptr;  // A/B switch
  return on;
}
}  // namespace cbp_dev

namespace cbp_host {

const char* errc_name(int status) {  // error.cpp:5-27, status = 1 + Errc
  static const char* names[] = {
      "InvalidArgument", "NonUnitSamplePoint", "DegenerateInput", "IllConditioned",
      "CoprimalityFailure", "FrameTooSmall", "RangeExceeded", "NotQuantized",
      "InconsistentAxes", "IllConditionedSlice", "DegenerateScales", "NonRealKernel",
      "DimMismatch", "IoFailure", "CorruptManifest", "MissingFrame", "FormatViolation",
      "PairMismatch"};
  if (status >= 1 && status <= 18) return names[status - 1];
  if (status == CBP_CUDA_ERROR) return "CudaError";
  if (status == CBP_UNSUPPORTED) return "Unsupported";
  return status == 0 ? "Ok" : "Error";
}

int set_error(cbp_ctx* ctx, int status, const std::string& msg) {
  if (ctx) ctx->err = std::string(errc_name(status)) + ": " + msg;
  return status;
}

int cuda_check(cbp_ctx* ctx, cudaError_t e, const char* what) {
  if (e == cudaSuccess) return 0;
  return set_error(ctx, CBP_CUDA_ERROR, std::string(what) + ": " + cudaGetErrorString(e));
}

void* workspace(cbp_ctx* ctx, int id, size_t bytes) {
  if (bytes == 0) bytes = 16;
  if (ctx->ws_bytes[id] >= bytes) return ctx->ws[id];
  if (ctx->ws[id]) {
    cudaDeviceSynchronize();  // growth is rare: never inside a steady-state loop
    cudaFree(ctx->ws[id]);
  }
  ctx->ws[id] = nullptr;
  ctx->ws_bytes[id] = 0;
  size_t want = bytes + bytes / 8;
  if (cudaMalloc(&ctx->ws[id], want) != cudaSuccess) return nullptr;
  ctx->ws_bytes[id] = want;
  return ctx->ws[id];
}

// Per-stage twiddles of a compile-time plan, DIT stage order; stage s (radix R, sub-length
// PP, PS = PP*R, NB = n/R) holds W_PS^{i*(b % PP)} at [(i-1)*NB + b]. See cbp_fft_ct.cuh.
const float2* stage_twiddles(cbp_ctx* ctx, int n, bool column) {
  std::vector<int> rad;
  if (!ct_radices(n, column, rad)) return nullptr;
  const int key = column ? -2 * n - 1 : -2 * n - 2;
  auto it = ctx->tw.find(key);
  if (it != ctx->tw.end()) return it->second;
  std::vector<float2> h;
  int pp = 1;
  for (int r : rad) {
    const int ps = pp * r, nb = n / r;
    for (int i = 1; i < r; ++i)
      for (int b = 0; b < nb; ++b) {
        const long e = long(i) * (b % pp);
        const double ang = -2.0 * M_PI * double(e % ps) / double(ps);
        h.push_back(make_float2(float(std::cos(ang)), float(std::sin(ang))));
      }
    pp = ps;
  }
  float2* d = nullptr;
  if (cudaMalloc(&d, std::max<size_t>(h.size(), 1) * sizeof(float2)) != cudaSuccess) return nullptr;
  cudaMemcpy(d, h.data(), h.size() * sizeof(float2), cudaMemcpyHostToDevice);
  ctx->tw[key] = d;
  return d;
}

// slot(u) of the compile-time column plan's DIF output order (null: no plan, natural
// order); the Wiener table is stored in that order so pass B filters element-wise
// bmajor: slot b*R1 + i (butterfly b of the first DIT radix R1) is stored at i*(n/R1) + b
const short* column_slots(cbp_ctx* ctx, int n, bool bmajor) {
  std::vector<int> rad;
  if (!ct_radices(n, true, rad)) return nullptr;
  const int key = -(n + (1 << 24) + (bmajor ? (1 << 25) : 0));  // distinct from the twiddle keys
  auto it = ctx->tw.find(key);
  if (it != ctx->tw.end()) return reinterpret_cast<const short*>(it->second);
  // [slot of u (n)][u of slot (n)]: the inverse lets the Wiener-table kernel write slots in order
  std::vector<short> h(2 * static_cast<size_t>(n));
  for (int u = 0; u < n; ++u) {
    const int sl = ct_pos(rad, u);
    h[u] = short(bmajor ? (sl % rad[0]) * (n / rad[0]) + sl / rad[0] : sl);
    h[n + h[u]] = short(u);
  }
  float2* d = nullptr;
  if (cudaMalloc(&d, h.size() * sizeof(short) + sizeof(float2)) != cudaSuccess) return nullptr;
  cudaMemcpy(d, h.data(), h.size() * sizeof(short), cudaMemcpyHostToDevice);
  ctx->tw[key] = d;
  return reinterpret_cast<const short*>(d);
}

const float2* twiddles(cbp_ctx* ctx, int n) {
  auto it = ctx->tw.find(n);
  if (it != ctx->tw.end()) return it->second;
  std::vector<float2> h(size_t(std::max(n, 1)));
  for (int k = 0; k < n; ++k) {
    const double ang = -2.0 * M_PI * double(k) / double(n);
    h[k] = make_float2(float(std::cos(ang)), float(std::sin(ang)));
  }
  float2* d = nullptr;
  if (cudaMalloc(&d, h.size() * sizeof(float2)) != cudaSuccess) return nullptr;
  cudaMemcpy(d, h.data(), h.size() * sizeof(float2), cudaMemcpyHostToDevice);
  ctx->tw[n] = d;
  return d;
}

FftPlan make_plan(int n) {
  FftPlan p{};
  p.n = n;
  p.nst = 0;
  int r = n;
  while (r % 8 == 0 && r != 16) p.radix[p.nst++] = 8, r /= 8;  // 16 -> 4 x 4
  while (r % 4 == 0) p.radix[p.nst++] = 4, r /= 4;
  while (r % 2 == 0) p.radix[p.nst++] = 2, r /= 2;
  while (r % 9 == 0) p.radix[p.nst++] = 9, r /= 9;
  while (r % 3 == 0) p.radix[p.nst++] = 3, r /= 3;
  while (r % 5 == 0) p.radix[p.nst++] = 5, r /= 5;
  while (r % 7 == 0) p.radix[p.nst++] = 7, r /= 7;
  if (r != 1) p.nst = -1;  // not 2/3/5/7-smooth
  return p;
}

int friendly_size(int n) {  // fft.cpp:272-280
  if (n < 1) return -1;
  for (int m = n;; ++m) {
    int r = m;
    for (int f : {2, 3, 5, 7})
      while (r % f == 0) r /= f;
    if (r == 1) return m;
  }
}

int deblur_setup(cbp_ctx* ctx, int Mb, int Nb, DeblurArgs& a) {
  std::memset(&a, 0, sizeof(a));
  a.frames_per_slot = 1;
  a.Mb = Mb;
  a.Nb = Nb;
  a.Gr = friendly_size(Mb);
  a.Gc = friendly_size(Nb);
  a.Hc = a.Gc / 2 + 1;
  a.even = (a.Gc % 2 == 0) ? 1 : 0;
  const int L = a.even ? a.Gc / 2 : a.Gc;
  a.plan_row = make_plan(L);
  a.plan_col = make_plan(a.Gr);
  if (a.plan_row.nst < 0 || a.plan_col.nst < 0)
    return set_error(ctx, CBP_UNSUPPORTED, "transform grid is not 2/3/5/7-smooth");
  a.xp = (a.Mb + 3) & ~3;  // XT column pitch
  a.hp = (a.Gr + 3) & ~3;
  static const int variant = getenv("CBP_FFT_VARIANT") ? atoi(getenv("CBP_FFT_VARIANT")) : 0;
  static const bool dyn = !getenv("CBP_STATIC_TILES");
  a.tile_ctr = dyn ? ctx->tile_ctr : nullptr;
  a.hpos = column_slots(ctx, a.Gr, true);  // compile-time column plans: butterfly-major filter
  a.h_bmajor = a.hpos != nullptr;
  // rows per CTA for passes A/C: keep 2*rpc*L*8 bytes <= 64 KB, at most 8 rows
  int rpc = 8;
  while (rpc > 1 && size_t(2) * rpc * L * sizeof(float2) > 64 * 1024) rpc /= 2;
  a.rows_per_cta = rpc;
  a.col_width = deblur_col_width(a.Gr, CBP_MAX_WIDTH);
  a.sm_reserve = ctx->sm_reserve;
  a.chain = ctx->chain;
  a.tw_row = twiddles(ctx, L);
  a.tw_post = twiddles(ctx, a.Gc);
  a.tw_col = twiddles(ctx, a.Gr);
  a.twst_row = a.even ? stage_twiddles(ctx, L, false) : nullptr;
  a.twst_col = stage_twiddles(ctx, a.Gr, true);
  static const int dbg = getenv("CBP_DEBLUR_DBG") ? atoi(getenv("CBP_DEBLUR_DBG")) : 0;
  a.dbg = dbg;
  a.variant = variant;
  if (!a.tw_row || !a.tw_post || !a.tw_col)
    return set_error(ctx, CBP_CUDA_ERROR, "twiddle table allocation failed");
  if (size_t(2) * rpc * L * sizeof(float2) > 200 * 1024)
    return set_error(ctx, CBP_UNSUPPORTED, "frame too wide for the shared-memory row transform");
  return 0;
}

int deblur_run(cbp_ctx* ctx, DeblurArgs a, int planes, size_t in_plane_stride,
               size_t out_plane_stride, cudaStream_t stream) {
  // Group whole frames into as few launches as the workspace budget allows: measured on
  // B200 (tools/deblur_micro.py, 1080p RGB), launch boundaries cost more than keeping the
  // half spectrum L2-resident (3 planes per launch: 29.0 us/plane; 87 planes: 18.9 us/plane,
  // spectrum in HBM). CBP_GROUP_BUDGET_MB caps the spectrum workspace (default 1 GB).
  const size_t plane_bytes = size_t(a.Hc) * a.xp * sizeof(float2);
  const int ch = std::max(a.channels, 1);
  static const size_t budget = [] {
    const char* e = getenv("CBP_GROUP_BUDGET_MB");
    return size_t(e ? atoi(e) : 1024) << 20;
  }();
  int frames_per_group = int(std::max<size_t>(1, budget / (plane_bytes * ch)));
  const int frames = planes / ch;
  frames_per_group = std::min(frames_per_group, std::max(frames, 1));
  const int fps = a.slot_per_frame ? std::max(a.frames_per_slot, 1) : 1;
  a.frames_per_slot = fps;
  if (fps > 1 && frames_per_group >= fps) frames_per_group -= frames_per_group % fps;  // groups start on a slot
  const int group_planes = frames_per_group * ch;
  a.x_plane = size_t(a.Hc) * a.xp;
  a.in_plane = in_plane_stride;
  a.out_plane = out_plane_stride;
  // Wiener filter table(s) H[u][v] for the kernel slot(s) of this batch
  const int nslots = a.slot_per_frame ? std::max((frames + fps - 1) / fps, 1) : 1;
  a.s_frame = size_t(a.Hc) * CBP_MAX_WIDTH;
  a.h_frame = size_t(a.Hc) * a.hp;
  a.S = static_cast<double2*>(workspace(ctx, WS_RED + 1, sizeof(double2) * a.s_frame * nslots));
  a.H = static_cast<float2*>(workspace(ctx, WS_RED + 2, sizeof(float2) * a.h_frame * nslots));
  if (!a.S || !a.H) return set_error(ctx, CBP_CUDA_ERROR, "workspace allocation failed");
  if (int st = cuda_check(ctx, launch_wiener_tables(a, nslots, stream), "filter table launch")) return st;
  ctx->launches += 2;
  // Fused persistent launch (one kernel for passes A, B, C over the whole batch, the
  // spectrum in an L2-resident ring of plane slots), where the grid has a fused plan
  static const bool fused_off = getenv("CBP_FUSED") == nullptr;  // measured slower: opt-in experiment
  int nA = 0, nB = 0, nC = 0;
  if (!fused_off && planes > 0 && deblur_fused_shape(a, nA, nB, nC)) {
    static const int ring_env = getenv("CBP_FUSED_RING") ? atoi(getenv("CBP_FUSED_RING")) : 6;
    FusedCtl f{};
    f.planes = planes;
    f.ring = std::min(std::max(ring_env, 2), planes);
    f.nA = nA, f.nB = nB, f.nC = nC;
    f.nsm = ctx->num_sms;
    a.X = static_cast<float2*>(workspace(ctx, WS_X, plane_bytes * f.ring));
    const size_t nctl = 4 + 3 * size_t(planes);
    unsigned* ctl = static_cast<unsigned*>(workspace(ctx, WS_FUSED, sizeof(unsigned) * (nctl + f.nsm)));
    if (!a.X || !ctl) return set_error(ctx, CBP_CUDA_ERROR, "workspace allocation failed");
    f.ticket = ctl;
    f.done = ctl + 4;
    f.sm_role = reinterpret_cast<int*>(ctl + nctl);
    a.frame0 = 0;
    a.in_vec2 = (reinterpret_cast<uintptr_t>(a.in) % 8 == 0) && a.in_ld % 2 == 0 && in_plane_stride % 2 == 0;
    a.out_vec2 = (reinterpret_cast<uintptr_t>(a.out) % 8 == 0) && a.out_ld % 2 == 0 && out_plane_stride % 2 == 0;
    a.in_vec4 = (reinterpret_cast<uintptr_t>(a.in) % 16 == 0) && a.in_ld % 4 == 0 && in_plane_stride % 4 == 0;
    cudaEvent_t* ev = nullptr;
    if (ctx->prof) {
      if (ctx->prof_used + 4 > int(ctx->prof_ev.size())) {
        for (int k = 0; k < 256; ++k) {
          cudaEvent_t e;
          cudaEventCreate(&e);
          ctx->prof_ev.push_back(e);
        }
      }
      ev = &ctx->prof_ev[ctx->prof_used];
      ctx->prof_used += 4;
      ctx->prof_planes += planes;
    }
    cudaMemsetAsync(ctl, 0, sizeof(unsigned) * nctl, stream);
    cudaMemsetAsync(f.sm_role, 0xff, sizeof(int) * f.nsm, stream);  // -1: no role claimed
    if (ev) cudaEventRecord(ev[0], stream);
    if (launch_deblur_fused(a, f, stream)) {
      if (ev)  // one launch: the whole duration is reported as pass A, B and C as zero
        for (int k = 1; k < 4; ++k) cudaEventRecord(ev[k], stream);
      ++ctx->launches;
      return cuda_check(ctx, cudaGetLastError(), "deconvolution launch");
    }
    if (ev) cudaEventRecord(ev[1], stream), cudaEventRecord(ev[2], stream), cudaEventRecord(ev[3], stream);
  }
  // Several launch groups in flight on side streams: each group's spectrum (1 frame by
  // default) stays L2-resident between its passes, and the fill/drain of one group's
  // persistent passes overlaps the passes of the group on the other stream.
  static const int side_env = getenv("CBP_DEBLUR_STREAMS") ? atoi(getenv("CBP_DEBLUR_STREAMS")) : 1;
  static const int group_mb = getenv("CBP_GROUP_MB") ? atoi(getenv("CBP_GROUP_MB")) : 28;
  int ns = std::min(std::max(side_env, 1), cbp_ctx::kSideStreams);
  int gp = group_planes;
  if (ns > 1) {
    const int fpg = std::max(1, int((size_t(std::max(group_mb, 1)) << 20) / (plane_bytes * ch)));
    gp = std::min(fpg, std::max(frames, 1));
    if (fps > 1 && gp >= fps) gp -= gp % fps;
    gp *= ch;
    if (planes <= gp) ns = 1, gp = group_planes;  // one group: no fork
  }
  for (int k = 0; ns > 1 && k < ns; ++k) {
    if (!ctx->side[k] && cudaStreamCreateWithFlags(&ctx->side[k], cudaStreamNonBlocking) != cudaSuccess) ns = 1;
    if (!ctx->side_ev[k] && cudaEventCreateWithFlags(&ctx->side_ev[k], cudaEventDisableTiming) != cudaSuccess) ns = 1;
  }
  if (ns > 1 && !ctx->side_ev[cbp_ctx::kSideStreams] &&
      cudaEventCreateWithFlags(&ctx->side_ev[cbp_ctx::kSideStreams], cudaEventDisableTiming) != cudaSuccess)
    ns = 1;
  if (ns == 1) gp = group_planes;
  float2* X = static_cast<float2*>(workspace(ctx, WS_X, plane_bytes * gp * ns));
  if (!X) return set_error(ctx, CBP_CUDA_ERROR, "workspace allocation failed");
  a.X = X;
  if (ns > 1) {
    const int fpg = gp / ch;
    cudaEvent_t* ev = nullptr;
    if (ctx->prof) {
      if (ctx->prof_used + 4 > int(ctx->prof_ev.size())) {
        for (int k = 0; k < 256; ++k) {
          cudaEvent_t e;
          cudaEventCreate(&e);
          ctx->prof_ev.push_back(e);
        }
      }
      ev = &ctx->prof_ev[ctx->prof_used];
      ctx->prof_used += 4;
      ctx->prof_planes += planes;
      cudaEventRecord(ev[0], stream);
    }
    cudaEventRecord(ctx->side_ev[cbp_ctx::kSideStreams], stream);  // fork: inputs and filter tables ready
    for (int k = 0; k < ns; ++k) cudaStreamWaitEvent(ctx->side[k], ctx->side_ev[cbp_ctx::kSideStreams], 0);
    const float* in0 = a.in;
    float* out0 = a.out;
    const cbp_kernel_slot* slot0 = a.slot;
    float2* const H0 = a.H;
    int used = 0;
    for (int p0 = 0, g = 0; p0 < planes; p0 += gp, ++g) {
      const int k = g % ns;
      cudaStream_t sk = ctx->side[k];
      used = std::max(used, k + 1);
      const int np = std::min(gp, planes - p0);
      a.in = in0 + size_t(p0) * in_plane_stride;
      a.out = out0 + size_t(p0) * out_plane_stride;
      const int s0 = a.slot_per_frame && fpg % fps == 0 ? (p0 / ch) / fps : 0;
      a.slot = slot0 + s0;
      a.H = H0 + size_t(s0) * (a.slot_per_frame ? a.h_frame : 0);
      a.frame0 = a.slot_per_frame && fpg % fps != 0 ? p0 / ch : 0;
      a.X = X + size_t(k) * gp * a.x_plane;
      a.tile_ctr = ctx->tile_ctr && a.tile_ctr ? ctx->tile_ctr + 4 * k : nullptr;
      a.in_vec2 = (reinterpret_cast<uintptr_t>(a.in) % 8 == 0) && a.in_ld % 2 == 0 && in_plane_stride % 2 == 0;
      a.out_vec2 = (reinterpret_cast<uintptr_t>(a.out) % 8 == 0) && a.out_ld % 2 == 0 && out_plane_stride % 2 == 0;
      a.in_vec4 = (reinterpret_cast<uintptr_t>(a.in) % 16 == 0) && a.in_ld % 4 == 0 && in_plane_stride % 4 == 0;
      if (a.tile_ctr) cudaMemsetAsync(a.tile_ctr, 0, 3 * sizeof(unsigned), sk);
      for (int pass = 0; pass < 3; ++pass) {
        int st = cuda_check(ctx, launch_deblur_pass(a, np, pass, sk), "deconvolution launch");
        if (st) return st;
        ++ctx->launches;
      }
    }
    for (int k = 0; k < used; ++k) {  // join
      cudaEventRecord(ctx->side_ev[k], ctx->side[k]);
      cudaStreamWaitEvent(stream, ctx->side_ev[k], 0);
    }
    if (ev)
      for (int k = 1; k < 4; ++k) cudaEventRecord(ev[k], stream);
    return 0;
  }
  const float* in0 = a.in;
  float* out0 = a.out;
  const cbp_kernel_slot* slot0 = a.slot;
  double2* const S0 = a.S;
  float2* const H0 = a.H;
  for (int p0 = 0; p0 < planes; p0 += group_planes) {
    const int np = std::min(group_planes, planes - p0);
    a.in = in0 + size_t(p0) * in_plane_stride;
    a.out = out0 + size_t(p0) * out_plane_stride;
    // a group starts on a slot boundary when it can (frames_per_group a multiple of fps);
    // otherwise (fps > frames per group) slot indices stay global: base slot 0
    const int s0 = a.slot_per_frame && frames_per_group % fps == 0 ? (p0 / ch) / fps : 0;
    a.slot = slot0 + s0;
    a.S = S0 + size_t(s0) * (a.slot_per_frame ? a.s_frame : 0);
    a.H = H0 + size_t(s0) * (a.slot_per_frame ? a.h_frame : 0);
    a.frame0 = a.slot_per_frame && frames_per_group % fps != 0 ? p0 / ch : 0;
    a.in_vec2 = (reinterpret_cast<uintptr_t>(a.in) % 8 == 0) && a.in_ld % 2 == 0 && in_plane_stride % 2 == 0;
    a.out_vec2 = (reinterpret_cast<uintptr_t>(a.out) % 8 == 0) && a.out_ld % 2 == 0 && out_plane_stride % 2 == 0;
    a.in_vec4 = (reinterpret_cast<uintptr_t>(a.in) % 16 == 0) && a.in_ld % 4 == 0 && in_plane_stride % 4 == 0;
    cudaEvent_t* ev = nullptr;
    if (ctx->prof) {
      if (ctx->prof_used + 4 > int(ctx->prof_ev.size())) {
        for (int k = 0; k < 256; ++k) {
          cudaEvent_t e;
          cudaEventCreate(&e);
          ctx->prof_ev.push_back(e);
        }
      }
      ev = &ctx->prof_ev[ctx->prof_used];
      ctx->prof_used += 4;
      ctx->prof_planes += np;
      cudaEventRecord(ev[0], stream);
    }
    if (a.tile_ctr) cudaMemsetAsync(a.tile_ctr, 0, 3 * sizeof(unsigned), stream);
    for (int pass = 0; pass < 3; ++pass) {
      int st = cuda_check(ctx, launch_deblur_pass(a, np, pass, stream), "deconvolution launch");
      if (st) return st;
      ++ctx->launches;
      if (ev) cudaEventRecord(ev[pass + 1], stream);
    }
  }
  return 0;
}

}  // namespace cbp_host

using namespace cbp_host;

extern "C" {

void cbp_decode_cfg_default(cbp_decode_cfg* c) {  // decoder.hpp:10-20
  c->search_min = 9;
  c->search_max = 25;
  c->tau = 1e-6;
  c->has_epsilon = 0;
  c->epsilon = 0.0;
  c->gap_threshold = 1e-9;
  c->trust_hint = 0;
  c->max_imag_energy = 0.01;
  c->negative_weight_tol = 0.01;
  c->validate = 1;
}

const char* cbp_errc_name(int status) { return errc_name(status); }
int cbp_friendly_size(int n) { return friendly_size(n); }

int cbp_create(int device, cbp_ctx** out) {
  if (!out) return CBP_INVALID_ARGUMENT;
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) return CBP_CUDA_ERROR;
  if (device < 0 || device >= n) return CBP_INVALID_ARGUMENT;
  if (cudaSetDevice(device) != cudaSuccess) return CBP_CUDA_ERROR;
  cbp_ctx* ctx = new cbp_ctx();
  ctx->device = device;
  cudaDeviceGetAttribute(&ctx->num_sms, cudaDevAttrMultiProcessorCount, device);
  if (cudaMallocHost(&ctx->host_slot, sizeof(cbp_kernel_slot)) != cudaSuccess) {
    delete ctx;
    return CBP_CUDA_ERROR;
  }
  for (auto& e : ctx->ev) cudaEventCreate(&e);
  cudaEventCreateWithFlags(&ctx->order_ev, cudaEventDisableTiming);
  if (cudaMalloc(&ctx->tile_ctr, 4 * cbp_ctx::kSideStreams * sizeof(unsigned)) != cudaSuccess)
    ctx->tile_ctr = nullptr;  // static tiles then
  *out = ctx;
  return 0;
}

void cbp_destroy(cbp_ctx* ctx) {
  cbp_host::DeviceGuard device_guard(ctx);
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  for (auto& kv : ctx->tw) cudaFree(kv.second);
  for (void* p : ctx->ws)
    if (p) cudaFree(p);
  if (ctx->host_slot) cudaFreeHost(ctx->host_slot);
  if (ctx->tile_ctr) cudaFree(ctx->tile_ctr);
  for (auto& e : ctx->ev)
    if (e) cudaEventDestroy(e);
  if (ctx->order_ev) cudaEventDestroy(ctx->order_ev);
  for (auto& st : ctx->side)
    if (st) cudaStreamDestroy(st);
  for (auto& e : ctx->side_ev)
    if (e) cudaEventDestroy(e);
  delete ctx;
}

const char* cbp_last_error(const cbp_ctx* ctx) { return ctx ? ctx->err.c_str() : ""; }

long long cbp_launch_count(const cbp_ctx* ctx) { return ctx ? ctx->launches : 0; }

int cbp_set_launch_chaining(cbp_ctx* ctx, int on) {
  cbp_host::DeviceGuard device_guard(ctx);
  if (!ctx) return CBP_INVALID_ARGUMENT;
  ctx->chain = on ? 1 : 0;
  return 0;
}

int cbp_set_sm_reserve(cbp_ctx* ctx, int sms) {
  cbp_host::DeviceGuard device_guard(ctx);
  if (!ctx || sms < 0) return CBP_INVALID_ARGUMENT;
  ctx->sm_reserve = sms;
  return 0;
}

int cbp_profile(cbp_ctx* ctx, int enable) {
  cbp_host::DeviceGuard device_guard(ctx);
  if (!ctx) return CBP_INVALID_ARGUMENT;
  ctx->prof = enable;
  ctx->prof_used = 0;
  ctx->prof_planes = 0;
  return 0;
}

// Sums the per-pass device times recorded since cbp_profile(ctx, 1); call after the
// work has completed. pass_ms[3] = A, B, C totals; *planes = planes processed.
int cbp_profile_read(cbp_ctx* ctx, double* pass_ms, long long* planes, int* groups) {
  cbp_host::DeviceGuard device_guard(ctx);
  if (!ctx) return CBP_INVALID_ARGUMENT;
  pass_ms[0] = pass_ms[1] = pass_ms[2] = 0.0;
  for (int g = 0; g + 4 <= ctx->prof_used; g += 4)
    for (int p = 0; p < 3; ++p) {
      float ms = 0.f;
      if (cudaEventElapsedTime(&ms, ctx->prof_ev[g + p], ctx->prof_ev[g + p + 1]) != cudaSuccess)
        return cuda_check(ctx, cudaGetLastError(), "profile read");
      pass_ms[p] += ms;
    }
  *planes = ctx->prof_planes;
  *groups = ctx->prof_used / 4;
  return 0;
}

// validate_kernel (kernel.cpp:7-17)
static int check_kernel(cbp_ctx* ctx, const double* w, int t) {
  if (!(t >= 1 && t % 2 == 1 && t <= CBP_MAX_WIDTH))
    return set_error(ctx, CBP_INVALID_ARGUMENT, "kernel width must be odd and >= 1");
  double s = 0.0, mn = 1e300;
  for (int i = 0; i < t * t; ++i) {
    if (!std::isfinite(w[i])) return set_error(ctx, CBP_INVALID_ARGUMENT, "kernel weights must be finite");
    mn = std::min(mn, w[i]);
  }
  if (mn < 0.0) return set_error(ctx, CBP_INVALID_ARGUMENT, "kernel weights must be nonnegative");
  for (int n = 0; n < t; ++n)
    for (int m = 0; m < t; ++m) s += w[m * t + n];
  if (std::abs(s - 1.0) > 1e-9)
    return set_error(ctx, CBP_INVALID_ARGUMENT, "kernel weights must sum to 1");
  return 0;
}

static int check_geometry(cbp_ctx* ctx, int batch, int channels, int rows, int cols, int ld) {
  if (batch < 0) return set_error(ctx, CBP_INVALID_ARGUMENT, "batch must be >= 0");
  if (!(channels == 1 || channels == 3))
    return set_error(ctx, CBP_DIM_MISMATCH, "frame must have 1 or 3 planes");
  if (rows < 1 || cols < 1) return set_error(ctx, CBP_DIM_MISMATCH, "empty frame plane");
  if (ld < cols) return set_error(ctx, CBP_INVALID_ARGUMENT, "row pitch smaller than the row");
  return 0;
}

int cbp_spectral_deblur(cbp_ctx* ctx, const float* blurred_dev, int batch, int channels, int rows,
                        int cols, int ld, const double* kernel, int t, double epsilon,
                        float* latent_dev, int ld_out, void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx) return CBP_INVALID_ARGUMENT;
  int st = check_kernel(ctx, kernel, t);
  if (st) return st;
  if (!(epsilon >= 0.0)) return set_error(ctx, CBP_INVALID_ARGUMENT, "epsilon must be nonnegative");
  if ((st = check_geometry(ctx, batch, channels, rows, cols, ld))) return st;
  if (rows < t || cols < t)
    return set_error(ctx, CBP_FRAME_TOO_SMALL, "blurred frame smaller than the kernel");
  if (batch == 0) return 0;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  cbp_kernel_slot* slot = static_cast<cbp_kernel_slot*>(workspace(ctx, WS_SLOTS, sizeof(cbp_kernel_slot) * 64));
  if (!slot) return set_error(ctx, CBP_CUDA_ERROR, "workspace allocation failed");
  // stage the fixed kernel into a context-owned slot (pinned, stream-ordered)
  if ((st = cuda_check(ctx, cudaStreamSynchronize(s), "stream sync"))) return st;
  cbp_kernel_slot* h = ctx->host_slot;
  std::memset(h, 0, offsetof(cbp_kernel_slot, weights));
  h->width = t;
  h->epsilon = epsilon;
  std::memcpy(h->weights, kernel, sizeof(double) * t * t);
  if ((st = cuda_check(ctx, cudaMemcpyAsync(slot, h, sizeof(cbp_kernel_slot), cudaMemcpyHostToDevice, s),
                       "slot upload")))
    return st;
  DeblurArgs a;
  if ((st = deblur_setup(ctx, rows, cols, a))) return st;
  a.in = blurred_dev;
  a.in_ld = ld;
  a.out = latent_dev;
  a.out_ld = ld_out;
  a.slot = slot;
  a.slot_per_frame = 0;
  a.channels = channels;
  return deblur_run(ctx, a, batch * channels, size_t(rows) * ld, size_t(rows) * ld_out, s);
}

int cbp_spectral_deblur_slots(cbp_ctx* ctx, const float* blurred_dev, int batch, int channels, int rows, int cols,
                              int ld, const cbp_kernel_slot* slots_dev, int frames_per_slot, float* latent_dev,
                              int ld_out, void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx || !slots_dev) return CBP_INVALID_ARGUMENT;
  if (frames_per_slot < 1) return set_error(ctx, CBP_INVALID_ARGUMENT, "frames_per_slot must be >= 1");
  int st = check_geometry(ctx, batch, channels, rows, cols, ld);
  if (st) return st;
  if (batch == 0) return 0;
  DeblurArgs a;
  if ((st = deblur_setup(ctx, rows, cols, a))) return st;
  a.in = blurred_dev;
  a.in_ld = ld;
  a.out = latent_dev;
  a.out_ld = ld_out;
  a.slot = slots_dev;
  a.slot_per_frame = 1;
  a.frames_per_slot = frames_per_slot;
  a.channels = channels;
  return deblur_run(ctx, a, batch * channels, size_t(rows) * ld, size_t(rows) * ld_out,
                    static_cast<cudaStream_t>(stream));
}

int cbp_spectral_deblur_slot(cbp_ctx* ctx, const float* blurred_dev, int batch, int channels,
                             int rows, int cols, int ld, const cbp_kernel_slot* slot_dev,
                             float* latent_dev, int ld_out, void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx || !slot_dev) return CBP_INVALID_ARGUMENT;
  int st = check_geometry(ctx, batch, channels, rows, cols, ld);
  if (st) return st;
  if (batch == 0) return 0;
  DeblurArgs a;
  if ((st = deblur_setup(ctx, rows, cols, a))) return st;
  a.in = blurred_dev;
  a.in_ld = ld;
  a.out = latent_dev;
  a.out_ld = ld_out;
  a.slot = slot_dev;
  a.slot_per_frame = 0;
  a.channels = channels;
  return deblur_run(ctx, a, batch * channels, size_t(rows) * ld, size_t(rows) * ld_out,
                    static_cast<cudaStream_t>(stream));
}

int cbp_device_alloc(cbp_ctx* ctx, size_t bytes, void** dev) {
  cbp_host::DeviceGuard device_guard(ctx);
  if (!ctx || !dev) return CBP_INVALID_ARGUMENT;
  cudaSetDevice(ctx->device);
  return cuda_check(ctx, cudaMalloc(dev, bytes ? bytes : 16), "device allocation");
}

void cbp_device_free(cbp_ctx* ctx, void* dev) {
  cbp_host::DeviceGuard device_guard(ctx);
  if (ctx && dev) cudaFree(dev);
}

int cbp_copy_to_device(cbp_ctx* ctx, void* dev, const void* host, size_t bytes) {
  cbp_host::DeviceGuard device_guard(ctx);
  if (!ctx) return CBP_INVALID_ARGUMENT;
  return cuda_check(ctx, cudaMemcpy(dev, host, bytes, cudaMemcpyHostToDevice), "copy to device");
}

int cbp_copy_to_host(cbp_ctx* ctx, void* host, const void* dev, size_t bytes) {
  cbp_host::DeviceGuard device_guard(ctx);
  if (!ctx) return CBP_INVALID_ARGUMENT;
  return cuda_check(ctx, cudaMemcpy(host, dev, bytes, cudaMemcpyDeviceToHost), "copy to host");
}

int cbp_read_slots(cbp_ctx* ctx, const cbp_kernel_slot* slots_dev, int count,
                   cbp_kernel_slot* slots_host, void* stream) {
  cbp_host::DeviceGuard device_guard(ctx);
  cbp_host::StreamOrder stream_order(ctx, stream);
  if (!ctx) return CBP_INVALID_ARGUMENT;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  int st = cuda_check(ctx, cudaMemcpyAsync(slots_host, slots_dev, sizeof(cbp_kernel_slot) * count,
                                           cudaMemcpyDeviceToHost, s), "slot read");
  if (st) return st;
  return cuda_check(ctx, cudaStreamSynchronize(s), "slot read sync");
}

}  // extern "C"

#ifdef CBP_PHASES
namespace cbp_dev {
__device__ unsigned long long g_phase[64];
}
extern "C" int cbp_debug_phases(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, cbp_dev::g_phase, sizeof(unsigned long long) * 64) == cudaSuccess ? 0 : 1;
}
#endif
