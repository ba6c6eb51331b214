/* cbp_cuda.h — C ABI of the B200-native CBP decryption path.
 *
 * This is the drop-in boundary for the reference's public C++ API
 * (/root/reference/proj/core/include/cbp/decoder.hpp, fft.hpp, poly.hpp, encoder.hpp).
 * The reference has no FFI of its own; its callers are C++ (tools/cbp.cpp:151,
 * core/src/bench.cpp:30-37). The C++ shim in include/cbp/ restores the exact
 * reference signatures on top of these entry points; INTEGRATION.md shows the
 * ctypes / C++ bindings.
 *
 * Conventions
 *  - Frames are row-major FP32 planes: element (m, n) of plane c of frame b sits at
 *    ptr[((b * channels + c) * rows + m) * ld + n]. Row index m is the z1 power,
 *    column index n the z2 power (reference types.hpp:15-17).
 *  - "_dev" pointers are device memory; everything else is host memory.
 *  - Every call is enqueued on `stream` (a cudaStream_t, NULL = legacy default).
 *    Calls that return results in host memory synchronize that stream.
 *  - Return value: 0 on success, otherwise 1 + the index of cbp::Errc
 *    (reference error.hpp:8-27), or CBP_CUDA_ERROR / CBP_UNSUPPORTED.
 *    cbp_last_error() returns "<ErrcName>: <stage>: <detail>" exactly like the
 *    reference's cbp::Error::what() (error.hpp:31-39, decoder.cpp:294-360).
 *  - There is no CPU fallback: without a CUDA device every compute entry point
 *    fails with CBP_CUDA_ERROR.
 *  - Threading: a context owns its scratch (workspaces, Wiener tables, dynamic-tile
 *    counters, a pinned staging slot). Use a context from one host thread and one
 *    stream at a time; work for another stream or thread needs its own context (the
 *    reference's callers run one decode per host thread, tools/cbp.cpp:141-164). Every
 *    entry point makes ctx's device current for the call, so contexts of different GPUs
 *    can be driven from one thread.
 */
#ifndef CBP_CUDA_H
#define CBP_CUDA_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ---- status codes: 1 + cbp::Errc (error.hpp:8-27) ------------------------ */
enum {
  CBP_OK = 0,
  CBP_INVALID_ARGUMENT = 1,
  CBP_NON_UNIT_SAMPLE_POINT = 2,
  CBP_DEGENERATE_INPUT = 3,
  CBP_ILL_CONDITIONED = 4,
  CBP_COPRIMALITY_FAILURE = 5,
  CBP_FRAME_TOO_SMALL = 6,
  CBP_RANGE_EXCEEDED = 7,
  CBP_NOT_QUANTIZED = 8,
  CBP_INCONSISTENT_AXES = 9,
  CBP_ILL_CONDITIONED_SLICE = 10,
  CBP_DEGENERATE_SCALES = 11,
  CBP_NON_REAL_KERNEL = 12,
  CBP_DIM_MISMATCH = 13,
  CBP_IO_FAILURE = 14,
  CBP_CORRUPT_MANIFEST = 15,
  CBP_MISSING_FRAME = 16,
  CBP_FORMAT_VIOLATION = 17,
  CBP_PAIR_MISMATCH = 18,
  CBP_CUDA_ERROR = 100,
  CBP_UNSUPPORTED = 101
};

/* decode_frame stage ids, used for the "<stage>: " error prefix (decoder.cpp:294-360) */
enum {
  CBP_STAGE_NONE = 0,
  CBP_STAGE_POLYNOMIAL_EVALUATION = 1,
  CBP_STAGE_KERNEL_DEGREE_ESTIMATION = 2,
  CBP_STAGE_KERNEL_ESTIMATION_1D = 3,
  CBP_STAGE_KERNEL_ESTIMATION_2D_FFT = 4,
  CBP_STAGE_VALIDATION = 5
};

/* fail_reason values: select the reference's message text for a status */
enum {
  CBP_REASON_NONE = 0,
  CBP_REASON_GAP = 1,              /* cofactor null space not one-dimensional (gap %f) */
  CBP_REASON_VANISHING_COFACTOR = 2,
  CBP_REASON_SCALE_RATIO = 3,      /* near-zero per-slice scale (ratio %f) */
  CBP_REASON_VANISHING_MASS = 4,   /* kernel estimate has vanishing mass */
  CBP_REASON_ZERO_KERNEL = 5,      /* kernel estimate is zero */
  CBP_REASON_IMAG_ENERGY = 6,      /* imaginary energy fraction %f */
  CBP_REASON_NO_POSITIVE = 7,      /* kernel estimate has no positive weight */
  CBP_REASON_NEGATIVE_WEIGHT = 8,  /* negative weight beyond tolerance (min %f of max) */
  CBP_REASON_AXES_DISAGREE = 9,    /* width estimates disagree: z1 gives %d, z2 gives %d */
  CBP_REASON_ZERO_POLY = 10,       /* bezout of an all-zero polynomial */
  CBP_REASON_NONFINITE = 11,       /* frame contains non-finite samples */
  CBP_REASON_TOO_SMALL = 12,       /* frame smaller than the kernel width */
  CBP_REASON_ZERO_PUBLIC = 13,     /* public frame is identically zero */
  CBP_REASON_SIGNED = 14,          /* signed-content width search (not on the device yet) */
  CBP_REASON_SCALE_ZERO = 15,      /* zero scale entry */
  CBP_REASON_WIDTH_LIMIT = 16      /* width above the device solver limit */
};

#define CBP_MAX_WIDTH 63 /* decoder.cpp:32 search bound, decoder.cpp:305 hint bound */
#define CBP_AXIS_Z1 0
#define CBP_AXIS_Z2 1

typedef struct cbp_ctx cbp_ctx;

/* Mirror of cbp::DecodeConfig (decoder.hpp:10-20), field for field. */
typedef struct {
  int search_min, search_max; /* odd, within [3,63] */
  double tau;                 /* singularity threshold in (0,1) */
  int has_epsilon;            /* 0: epsilon = 1e-8 * peak|K|^2 (decoder.cpp:198-199) */
  double epsilon;
  double gap_threshold; /* poly.hpp:40 */
  int trust_hint;
  double max_imag_energy, negative_weight_tol;
  int validate;
} cbp_decode_cfg;

/* Per-frame decode state in device memory. Written by cbp_decode_frames_async and
 * consumed by cbp_spectral_deblur_slot, so kernel recovery and reuse chain on the
 * device without a host round trip. */
typedef struct {
  int status;       /* 0 ok, else CBP_* code */
  int fail_stage;   /* CBP_STAGE_* of the failure */
  int fail_axis;    /* CBP_AXIS_* for ill_conditioned_slice, else -1 */
  int fail_slice;   /* slice index for ill_conditioned_slice, else -1 */
  int width;        /* t */
  int clamped;      /* WidthEstimate::clamped (decoder.cpp:89) */
  int width_z1, width_z2;
  int fail_reason;  /* which check failed inside the stage (CBP_REASON_*) */
  int reserved;
  double fail_value; /* numeric detail for the error message (gap, ratio, ...) */
  double epsilon;    /* spectral guard used for the deconvolution */
  double residual;   /* validation_residual (decoder.cpp:367-376) */
  double scale_residual; /* ScaleResolution::residual */
  double weights[CBP_MAX_WIDTH * CBP_MAX_WIDTH]; /* kernel estimate, t x t row-major */
} cbp_kernel_slot;

/* Host-side mirror of cbp::DecodedFrame metadata (decoder.hpp:65-80). */
typedef struct {
  int status, fail_stage, fail_axis, fail_slice;
  int width_used, width_clamped;
  double validation_residual, epsilon_used, fail_value;
  double stage_ms[5]; /* polynomial_evaluation, kernel_degree_estimation,
                         kernel_estimation_1d, kernel_estimation_2d_fft, total
                         (StageTimings, decoder.hpp:65-71); batch-level CUDA-event times */
  double kernel[CBP_MAX_WIDTH * CBP_MAX_WIDTH]; /* t x t row-major */
} cbp_decode_info;

/* ---- context ------------------------------------------------------------ */
void cbp_decode_cfg_default(cbp_decode_cfg* cfg);
int cbp_create(int device, cbp_ctx** out);
void cbp_destroy(cbp_ctx* ctx);
const char* cbp_last_error(const cbp_ctx* ctx);
const char* cbp_errc_name(int status);
int cbp_friendly_size(int n); /* fft_internal.hpp:22-24 */

/* ---- decode (replaces cbp::decode_frame, decoder.hpp:82) ------------------
 * Decodes `batch` independent blurred pairs. width_hints (host, may be NULL) is
 * BlurredPair::kernel_width_hint per frame (<= 0: none). latent_dev has the input
 * geometry (planes of rows x ld_out floats, plane pitch rows*ld_out); the top-left
 * (rows-t+1) x (cols-t+1) region of each plane is written. info (host, batch
 * entries) receives per-frame results.
 * Returns the status of the first failing frame (its message in cbp_last_error). */
int cbp_decode_frames(cbp_ctx* ctx, const float* pub_dev, const float* prv_dev, int batch,
                      int channels, int rows, int cols, int ld, const int* width_hints,
                      const cbp_decode_cfg* cfg, float* latent_dev, int ld_out,
                      cbp_decode_info* info, void* stream);

/* Asynchronous variant: per-frame results go to slots_dev (device, batch entries);
 * nothing is synchronized. Argument errors are still reported synchronously. */
int cbp_decode_frames_async(cbp_ctx* ctx, const float* pub_dev, const float* prv_dev, int batch,
                            int channels, int rows, int cols, int ld, const int* width_hints,
                            const cbp_decode_cfg* cfg, float* latent_dev, int ld_out,
                            cbp_kernel_slot* slots_dev, void* stream);

/* Writes the reference's error text for a failed slot (host copy) into buf: the message
 * decode_frame would throw, "<Errc>: <stage>: <Errc>: <detail>" (decoder.cpp:294-360);
 * "" for a successful slot. Returns the slot's status. */
int cbp_slot_message(const cbp_kernel_slot* slot_host, char* buf, int len);

/* Copies `count` slots to host memory (synchronizes the stream). */
int cbp_read_slots(cbp_ctx* ctx, const cbp_kernel_slot* slots_dev, int count,
                   cbp_kernel_slot* slots_host, void* stream);

/* ---- fixed-kernel deconvolution (replaces cbp::spectral_deblur, decoder.hpp:63) ---
 * kernel: host t x t row-major FP64 weights (validated like validate_kernel,
 * kernel.cpp:7-17). latent_dev has the input geometry (plane pitch rows*ld_out);
 * the top-left (rows-t+1) x (cols-t+1) region of each plane is written. */
int cbp_spectral_deblur(cbp_ctx* ctx, const float* blurred_dev, int batch, int channels, int rows,
                        int cols, int ld, const double* kernel, int t, double epsilon,
                        float* latent_dev, int ld_out, void* stream);

/* Same, with kernel, width and epsilon read on the device from a slot written by
 * cbp_decode_frames_async (a failed slot leaves its outputs untouched). */
/* As cbp_decode_frames_async, and records `slot_ready_event` (a cudaEvent_t) on `stream` as
 * soon as the slots hold their final kernel, width and epsilon, before the batch's own
 * deconvolution and validation residual: a pipeline can start cbp_spectral_deblur_slot on
 * the following frames while those finish (the residual and any validation failure land
 * in the slot when `stream` completes). */
int cbp_decode_frames_async_ev(cbp_ctx* ctx, const float* pub_dev, const float* prv_dev, int batch,
                               int channels, int rows, int cols, int ld, const int* width_hints,
                               const cbp_decode_cfg* cfg, float* latent_dev, int ld_out,
                               cbp_kernel_slot* slots_dev, void* stream, void* slot_ready_event);
/* Many kernels in one call: frame f of the batch is deconvolved with slots_dev[f /
 * frames_per_slot] (e.g. S camera streams x n frames, stream-major, frames_per_slot = n:
 * one launch group and one Wiener-table launch for all streams instead of S calls). A
 * failed slot leaves its frames' outputs untouched. */
int cbp_spectral_deblur_slots(cbp_ctx* ctx, const float* blurred_dev, int batch, int channels,
                              int rows, int cols, int ld, const cbp_kernel_slot* slots_dev,
                              int frames_per_slot, float* latent_dev, int ld_out, void* stream);
/* decode_frame split at its stage boundaries (decoder.cpp:280-378), for pipelines that batch
 * the recovery frame's deconvolution with the frames that reuse its kernel:
 *  - cbp_recover_kernels_async: width estimation, unit-circle sampling, cofactor solves and
 *    kernel composition (decoder.cpp:290-352) into slots_dev; no deconvolution, no residual;
 *  - cbp_validate_frames_async: the validation residual (decoder.cpp:367-376) of latents
 *    already deconvolved with the slots' kernels (e.g. by cbp_spectral_deblur_slot) into
 *    slots_dev[b].residual.
 * recover -> spectral_deblur_slot -> validate gives bit-identical slots and latents to
 * cbp_decode_frames_async. */
int cbp_recover_kernels_async(cbp_ctx* ctx, const float* pub_dev, const float* prv_dev, int batch,
                              int channels, int rows, int cols, int ld, const int* width_hints,
                              const cbp_decode_cfg* cfg, cbp_kernel_slot* slots_dev, void* stream);
int cbp_validate_frames_async(cbp_ctx* ctx, const float* pub_dev, const float* latent_dev, int batch,
                              int channels, int rows, int cols, int ld, int ld_out,
                              cbp_kernel_slot* slots_dev, void* stream);
int cbp_spectral_deblur_slot(cbp_ctx* ctx, const float* blurred_dev, int batch, int channels,
                             int rows, int cols, int ld, const cbp_kernel_slot* slot_dev,
                             float* latent_dev, int ld_out, void* stream);

/* ---- stage-level entry points (host in/out; synchronize) -------------------- */
/* estimate_kernel_width (decoder.hpp:29-30) */
int cbp_estimate_kernel_width(cbp_ctx* ctx, const float* pub_dev, const float* prv_dev,
                              int channels, int rows, int cols, int ld, int search_min,
                              int search_max, double tau, int* width, int* clamped, void* stream);
/* axis_roots_dft of luma(pub) and luma(prv) (fft.hpp:15-18): slices_pub/prv receive t
 * slices of length L (L = cols for Z1, rows for Z2), complex interleaved, slice-major. */
int cbp_sample_slices(cbp_ctx* ctx, const float* pub_dev, const float* prv_dev, int channels,
                      int rows, int cols, int ld, int t, int axis, double* slices_pub,
                      double* slices_prv, void* stream);
/* cofactor_null_solve (poly.hpp:51-52) over `batch` slice pairs of length len (host,
 * complex interleaved). Outputs k1/k2 (batch x t complex) and gaps; per-problem
 * status (0 or CBP_ILL_CONDITIONED). */
int cbp_cofactor_solve_batch(cbp_ctx* ctx, const double* p, const double* q, int batch, int len,
                             int t, double gap_threshold, double* k1, double* k2, double* gaps,
                             int* status, void* stream);
/* sample_cofactors (decoder.hpp:40-41): values t x t complex, gaps t. */
int cbp_sample_cofactors(cbp_ctx* ctx, const float* pub_dev, const float* prv_dev, int channels,
                         int rows, int cols, int ld, int width, int axis, double gap_threshold,
                         double* values, double* gaps, void* stream);
/* complete_to_spectrum (decoder.hpp:45) */
int cbp_complete_to_spectrum(cbp_ctx* ctx, const double* values, int t, int axis, double* out,
                             void* stream);
/* resolve_scales (decoder.hpp:54) */
int cbp_resolve_scales(cbp_ctx* ctx, const double* a_values, const double* b_values, int t,
                       double* lambda, double* mu, double* residual, void* stream);
/* assemble_kernel (decoder.hpp:57-59) */
int cbp_assemble_kernel(cbp_ctx* ctx, const double* a_spectrum, const double* b_spectrum,
                        const double* lambda, const double* mu, int t, double max_imag_energy,
                        double negative_weight_tol, double* weights, void* stream);
/* validate_pair (decoder.hpp:85-86) */
int cbp_validate_pair(cbp_ctx* ctx, const float* pub_dev, const float* prv_dev, int channels,
                      int rows, int cols, int ld, const double* k1, const double* k2, int t,
                      double* residual, void* stream);

/* ---- polynomial / transform utilities (poly.hpp:30-55, fft.hpp:9-13) -------------
 * Stand-alone device versions of functions the decode path runs fused inside its kernels.
 * Complex arrays: interleaved (re, im) FP64, host memory; matrices row-major; synchronous.
 * cbp_bezout_leading_block: B[i][j] = sum_{k<=min(i,j)} p[i+j+1-k] q[k] - q[i+j+1-k] p[k]
 *   (poly.cpp:66-79): CBP_DEGENERATE_INPUT for an all-zero p or q.
 * cbp_numerical_singularity: one-sided Jacobi singular values of the n x n matrix m;
 *   ratio = sigma_min / sigma_max (0 and singular for the zero matrix), singular = ratio < tau
 *   (poly.cpp:81-91).
 * cbp_homogeneous_lsq: the unit right singular vector of the smallest singular value of the
 *   rows x cols matrix a (rows >= cols), largest |x_i| rotated real positive (poly.cpp:123-130).
 * cbp_fft2: the rows x cols 2D DFT, exponent -2 pi i (inverse = 0), or +2 pi i with the
 *   1/(rows cols) normalization (inverse = 1) (fft.cpp:170-195); any size. */
int cbp_bezout_leading_block(cbp_ctx* ctx, const double* p, int np, const double* q, int nq, int size,
                             double* out, void* stream);
int cbp_numerical_singularity(cbp_ctx* ctx, const double* m, int n, double tau, int* singular,
                              double* ratio, void* stream);
int cbp_homogeneous_lsq(cbp_ctx* ctx, const double* a, int rows, int cols, double* x, void* stream);
int cbp_fft2(cbp_ctx* ctx, const double* in, int rows, int cols, int inverse, double* out, void* stream);

/* ---- CBP generation on the device (encoder.hpp:36-37, poly.hpp:14) ----------
 * encode_frame: pub = latent (*) k1, prv = latent (*) k2 per plane, FP64 accumulation,
 * FP32 output of size (rows+t-1) x (cols+t-1) with row pitch ld_out. */
int cbp_encode_frames(cbp_ctx* ctx, const float* latent_dev, int batch, int channels, int rows,
                      int cols, int ld, const double* k1, const double* k2, int t, float* pub_dev,
                      float* prv_dev, int ld_out, void* stream);
/* Synthetic uniform [0,1) frames for benchmarking (counter-based splitmix64 hash of
 * (seed, plane, m, n); NOT bit-identical to the reference's mt19937_64 random_frame). */
int cbp_synth_frames(cbp_ctx* ctx, float* out_dev, int planes, int rows, int cols, int ld,
                     uint64_t seed, void* stream);

/* ---- host-buffer pipeline (the e2e path) ------------------------------------
 * Decodes a run of frames held in host memory, like the reference CLI
 * (tools/cbp.cpp:130-207): frame j uses pub[j] and, when recover[j] != 0, prv[j]
 * (frames packed [n_frames][channels][rows][cols]). Recovery frames run decode_frame
 * (width_hint > 0 with cfg->trust_hint skips the width search); the others reuse the
 * most recent recovered kernel through spectral_deblur on the device. H2D, compute
 * and D2H overlap on internal streams. latent receives frames in the input geometry
 * (the latent is the top-left (rows-t+1) x (cols-t+1) of each plane). Frames are
 * transferred in pairs, each pair as one block that ends at row rows-tlo of the second
 * frame's last plane, tlo = width_hint when cfg->trust_hint, else cfg->search_min: the
 * rows after it are left untouched, other samples outside the latents hold unspecified
 * values. slots_host (may be NULL) gets
 * one cbp_kernel_slot per recovery frame. Synchronizes before returning.
 * Pinned host memory gives full PCIe bandwidth. recover[0] must be nonzero. */
int cbp_decode_run_host(cbp_ctx* ctx, const float* pub, const float* prv, int n_frames,
                        int channels, int rows, int cols, const int* recover, int width_hint,
                        const cbp_decode_cfg* cfg, float* latent, cbp_kernel_slot* slots_host);

/* ---- quantized-stream tier (encoder.cpp:105-139) ---------------------------------
 * Quantized frames are integer codes k (uint8 for bits = 8, uint16 for bits = 16) with
 * value k / (2^bits - 1): the device form of the reference's u8/u16 frames.
 * cbp_quantize_frames: k = round(clamp(x, 0, 1) * maxv) (quantize_frame, encoder.cpp:105-120);
 *   CBP_RANGE_EXCEEDED ("samples outside [0,1]") if a sample lies outside [-1e-9, 1+1e-9].
 *   Synchronizes (the range check is reported on the host).
 * cbp_dequantize_frames: float(k / maxv) into FP32 frames (async).
 * cbp_degrade_bits: k & ~(2^drop - 1) in place, drop in [0, bits) (degrade_bits,
 *   encoder.cpp:124-139; async).
 * cbp_decode_frames_q: cbp_decode_frames on quantized device frames (dequantized into
 *   context workspaces first; same results as decoding the dequantized FP32 values).
 * cbp_decode_run_host_q: cbp_decode_run_host with host codes: PCIe carries 1 or 2 bytes per
 *   sample, dequantization runs on the device. */
int cbp_quantize_frames(cbp_ctx* ctx, const float* in_dev, int planes, int rows, int cols, int ld, int bits,
                        void* codes_dev, int ld_codes, void* stream);
int cbp_dequantize_frames(cbp_ctx* ctx, const void* codes_dev, int bits, int planes, int rows, int cols,
                          int ld_codes, float* out_dev, int ld, void* stream);
int cbp_degrade_bits(cbp_ctx* ctx, void* codes_dev, int bits, int planes, int rows, int cols, int ld_codes,
                     int drop, void* stream);
int cbp_decode_frames_q(cbp_ctx* ctx, const void* pub_codes, const void* prv_codes, int bits, int batch,
                        int channels, int rows, int cols, int ld_codes, const int* width_hints,
                        const cbp_decode_cfg* cfg, float* latent_dev, int ld_out, cbp_decode_info* info,
                        void* stream);
int cbp_decode_run_host_q(cbp_ctx* ctx, const void* pub_codes, const void* prv_codes, int bits, int n_frames,
                          int channels, int rows, int cols, const int* recover, int width_hint,
                          const cbp_decode_cfg* cfg, float* latent, cbp_kernel_slot* slots_host);

/* ---- reference-exact input generators (host; untimed) ------------------------
 * frame_seed / splitmix64 (rng.hpp:8-29), random_frame (synth.cpp:12-22: mt19937_64,
 * column-major draw, returned row-major FP32), coprimality_check and
 * generate_coprime_pair (encoder.cpp:45-81; k1/k2 t x t row-major). */
uint64_t cbp_frame_seed(uint64_t stream_seed, int frame_index);
uint64_t cbp_splitmix64(uint64_t x);
int cbp_random_frame(int rows, int cols, int channels, uint64_t seed, float* out);
double cbp_coprimality_check(const double* k1, const double* k2, int t, int trials);
int cbp_generate_coprime_pair(int width, uint64_t seed, int max_retries, double margin_threshold,
                              int trials, double* k1, double* k2, double* margin);

/* ---- device memory helpers (used by the C++ shim, include/cbp/) ---------------- */
int cbp_device_alloc(cbp_ctx* ctx, size_t bytes, void** dev);
void cbp_device_free(cbp_ctx* ctx, void* dev);
int cbp_copy_to_device(cbp_ctx* ctx, void* dev, const void* host, size_t bytes);
int cbp_copy_to_host(cbp_ctx* ctx, void* host, const void* dev, size_t bytes);

/* ---- scheduling ----------------------------------------------------------------
 * The deconvolution passes run persistent grids sized to fill the GPU. A context whose
 * deconvolution overlaps work of another stream (the next epoch's kernel recovery in a
 * video pipeline) can leave `sms` SMs to that stream. No reference counterpart
 * (the reference parallelizes frames over host threads, tools/cbp.cpp:141-164). */
int cbp_set_sm_reserve(cbp_ctx* ctx, int sms);
/* Programmatic dependent launch of the context's small latency-chain kernels (kernel
 * recovery, Wiener tables, validation reduction): on (default) each kernel is scheduled as
 * its predecessor drains instead of after it (c1 decode_frame 0.290 -> 0.255 ms). */
int cbp_set_launch_chaining(cbp_ctx* ctx, int on);

/* ---- instrumentation ----------------------------------------------------------
 * Kernels enqueued by this context so far; optional CUDA-event timing of the three
 * deconvolution passes (A rows forward, B columns + filter, C rows inverse). */
long long cbp_launch_count(const cbp_ctx* ctx);
int cbp_profile(cbp_ctx* ctx, int enable);
int cbp_profile_read(cbp_ctx* ctx, double* pass_ms, long long* planes, int* groups);

#ifdef __cplusplus
}
#endif
#endif /* CBP_CUDA_H */
