// Shared device helpers for the CBP sm_100a kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <mutex>

#include "../../include/cbp_cuda.h"

namespace cbp_dev {

// First-launch setup (cudaFuncSetAttribute, occupancy queries) is per device and must be
// thread-safe: the reference's callers decode from a pool of host threads
// (tools/cbp.cpp:141-164). CBP_ONCE_PER_DEVICE runs its body once per (call site, device).
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d < 0 || d >= kMaxDevices ? 0 : d;
}
#define CBP_ONCE_PER_DEVICE(...)                                    \
  do {                                                              \
    static std::once_flag cbp_once_[cbp_dev::kMaxDevices];          \
    std::call_once(cbp_once_[cbp_dev::current_device()], [&] __VA_ARGS__); \
  } while (0)

// Programmatic dependent launch for the latency-bound recovery chain (a dozen dependent
// kernels of one or a few CTAs each): kernels launched with launch_chain may be scheduled
// while their predecessor in the stream still runs; pdl_enter() (first statement of every
// such kernel) waits for the predecessor's completion and memory (griddepcontrol.wait, a
// no-op for ordinary launches), so the next kernel is scheduled as this one drains and the
// launch latency of each link overlaps the previous kernel instead of adding to the chain
// (c1 decode latency 0.290 -> 0.255 ms). cbp_set_launch_chaining turns it off per context.
__device__ __forceinline__ void pdl_enter() {
  // no early griddepcontrol.launch_dependents: the implicit trigger at CTA exit already
  // overlaps the dependent's launch with the predecessor's drain, while an early trigger
  // makes the dependents resident (holding registers and shared memory) during the whole
  // predecessor (c4 batch of 4: 2.12k vs 2.30k frames/s; c1 0.260 vs 0.255 ms)
  asm volatile("griddepcontrol.wait;\n" ::: "memory");
}
bool pdl_enabled();  // CBP_NO_PDL unset (cbp_capi.cu)
template <typename... KArgs, typename... Args>
inline cudaError_t launch_chain(void (*kernel)(KArgs...), bool chain, dim3 grid, dim3 block, size_t smem,
                                cudaStream_t s, Args... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  // only small grids launch early: the waiting CTAs of a large one would hold SM slots that
  // a concurrent stream's kernels (the video pipeline's deconvolution) could use
  const unsigned blocks = grid.x * grid.y * grid.z;
  cfg.numAttrs = chain && pdl_enabled() && blocks <= 2 * 148 ? 1 : 0;
  return cudaLaunchKernelEx(&cfg, kernel, args...);
}

// ---------------------------------------------------------------- complex math
__host__ __device__ __forceinline__ float2 cadd(float2 a, float2 b) { return make_float2(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ float2 csub(float2 a, float2 b) { return make_float2(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ float2 cmul(float2 a, float2 b) {
  return make_float2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
__host__ __device__ __forceinline__ float2 cconj(float2 a) { return make_float2(a.x, -a.y); }
__host__ __device__ __forceinline__ float2 cscale(float2 a, float s) { return make_float2(a.x * s, a.y * s); }

__host__ __device__ __forceinline__ double2 zadd(double2 a, double2 b) { return make_double2(a.x + b.x, a.y + b.y); }
__host__ __device__ __forceinline__ double2 zsub(double2 a, double2 b) { return make_double2(a.x - b.x, a.y - b.y); }
__host__ __device__ __forceinline__ double2 zmul(double2 a, double2 b) {
  return make_double2(a.x * b.x - a.y * b.y, a.x * b.y + a.y * b.x);
}
// conj(a) * b
__host__ __device__ __forceinline__ double2 zcmul(double2 a, double2 b) {
  return make_double2(a.x * b.x + a.y * b.y, a.x * b.y - a.y * b.x);
}
__host__ __device__ __forceinline__ double2 zconj(double2 a) { return make_double2(a.x, -a.y); }
__host__ __device__ __forceinline__ double2 zscale(double2 a, double s) { return make_double2(a.x * s, a.y * s); }
__host__ __device__ __forceinline__ double zabs2(double2 a) { return a.x * a.x + a.y * a.y; }
__device__ __forceinline__ double zabs(double2 a) { return hypot(a.x, a.y); }
__device__ __forceinline__ double2 zdiv(double2 a, double2 b) {
  double d = b.x * b.x + b.y * b.y;
  return make_double2((a.x * b.x + a.y * b.y) / d, (a.y * b.x - a.x * b.y) / d);
}
// exp(-2*pi*i * k / n) in FP64
__device__ __forceinline__ double2 zroot(long k, long n) {
  double s, c;
  sincospi(-2.0 * double(k % n) / double(n), &s, &c);
  return make_double2(c, s);
}

// ------------------------------------------------------------- frame geometry
struct FrameGeom {
  int batch, channels, rows, cols, ld;
  __host__ __device__ size_t plane_elems() const { return size_t(rows) * ld; }
  __host__ __device__ const float* plane(const float* base, int b, int c) const {
    return base + (size_t(b) * channels + c) * plane_elems();
  }
};

// Rec.601 luma on the fly (image.cpp:41-45): identity for gray, same association
// order as Eigen's 0.299*R + 0.587*G + 0.114*B.
__device__ __forceinline__ double luma_at(const float* p0, size_t plane, int channels, size_t off) {
  if (channels == 1) return double(__ldg(p0 + off));
  double r = __ldg(p0 + off), g = __ldg(p0 + plane + off), b = __ldg(p0 + 2 * plane + off);
  // unfused, like the reference's Eigen expression (bit-identical to the CPU restatement)
  return __dadd_rn(__dadd_rn(__dmul_rn(0.299, r), __dmul_rn(0.587, g)), __dmul_rn(0.114, b));
}

// Record the first failure on a slot (status stays the first error).
__device__ __forceinline__ void slot_fail(cbp_kernel_slot* s, int status, int stage, int axis,
                                          int slice, double value, int reason) {
  if (atomicCAS(&s->status, 0, status) == 0) {
    s->fail_stage = stage;
    s->fail_axis = axis;
    s->fail_slice = slice;
    s->fail_value = value;
    s->fail_reason = reason;
  }
}

// Phase timestamps for kernel-internal profiling (build with -DCBP_PHASES; read with
// cbp_debug_phases). Compiled out otherwise.
#ifdef CBP_PHASES
extern __device__ unsigned long long g_phase[64];
__device__ __forceinline__ void phase_mark(int i, bool who) {
  if (who && threadIdx.x == 0) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_phase[i] = t;
  }
}
#define CBP_PHASE(i, who) ::cbp_dev::phase_mark((i), (who))
#else
#define CBP_PHASE(i, who) ((void)(who))
#endif

// ---------------------------------------------------------------- cp.async
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async8(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
// 16-byte copy that bypasses L1 (.cg); src_bytes < 16 zero-fills the tail
__device__ __forceinline__ void cp_async16(void* smem, const void* gmem, int src_bytes) {
  const unsigned s = static_cast<unsigned>(__cvta_generic_to_shared(smem));
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;\n" ::"r"(s), "l"(gmem), "r"(src_bytes));
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;\n" ::"n"(N));
}

}  // namespace cbp_dev
