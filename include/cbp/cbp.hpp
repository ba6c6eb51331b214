// cbp::core public API for the B200 build: the reference's headers
// (proj/core/include/cbp/{error,image,kernel,encoder,decoder,fft,poly,synth,metrics}.hpp)
// with the same names, fields, defaults and error behaviour. Every compute function runs
// on the GPU through the C ABI of include/cbp_cuda.h (libcbp_cuda.so); there is no CPU
// fallback: without a CUDA device those calls throw std::runtime_error("CudaError: ...").
// Host-only helpers (input generators, validate_*, luma, psnr, quantize_frame,
// conv2_full) are plain C++ like the reference's; none of them is on the decode path.
// The per-module headers error.hpp, image.hpp, ... include this file, so reference code
// that includes "cbp/decoder.hpp" compiles unchanged.
#pragma once

#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

#include "cbp/types.hpp"

namespace cbp {

// ------------------------------------------------------------ error.hpp:8-45
enum class Errc {
  invalid_argument,
  non_unit_sample_point,
  degenerate_input,
  ill_conditioned,
  coprimality_failure,
  frame_too_small,
  range_exceeded,
  not_quantized,
  inconsistent_axes,
  ill_conditioned_slice,
  degenerate_scales,
  non_real_kernel,
  dim_mismatch,
  io_failure,
  corrupt_manifest,
  missing_frame,
  format_violation,
  pair_mismatch,
};

const char* errc_name(Errc c);

class Error : public std::runtime_error {
 public:
  Error(Errc code, const std::string& what)
      : std::runtime_error(std::string(errc_name(code)) + ": " + what), code_(code) {}
  // message already prefixed (as produced by the C ABI)
  Error(Errc code, const std::string& full, bool) : std::runtime_error(full), code_(code) {}
  Errc code() const { return code_; }

 private:
  Errc code_;
};

[[noreturn]] inline void fail(Errc code, const std::string& what) { throw Error(code, what); }
inline void require(bool ok, Errc code, const std::string& what) {
  if (!ok) fail(code, what);
}

// ------------------------------------------------------------ image.hpp:10-32
enum class BitDepth { f32, u16, u8 };
int bit_depth_bits(BitDepth d);
const char* bit_depth_name(BitDepth d);              // "float32", "u16", "u8"
BitDepth bit_depth_from_name(const std::string& s);  // InvalidArgument for other names

struct Frame {
  std::vector<ImagePlane> planes;
  BitDepth bit_depth = BitDepth::f32;
  int index = 0;
  int rows() const { return planes.empty() ? 0 : int(planes[0].rows()); }
  int cols() const { return planes.empty() ? 0 : int(planes[0].cols()); }
  int channels() const { return int(planes.size()); }
};

void validate_frame(const Frame& f);
Mat luma(const Frame& f);

// ----------------------------------------------------------- kernel.hpp:13-24
struct BlurKernel {
  int width = 1;
  Mat weights;
};
void validate_kernel(const BlurKernel& k, double sum_tol = 1e-9);
struct CoprimePair {
  BlurKernel k1, k2;
  double coprimality_margin = 0.0;
  std::uint64_t seed = 0;
};

// ---------------------------------------------------------- encoder.hpp:12-43
inline constexpr double kDefaultMarginThreshold = 1e-6;
inline constexpr int kDefaultCoprimalityTrials = 4;
inline constexpr int kDefaultMaxRetries = 16;
double coprimality_check(const BlurKernel& k1, const BlurKernel& k2, int trials = kDefaultCoprimalityTrials);
CoprimePair generate_coprime_pair(int width, std::uint64_t seed, int max_retries = kDefaultMaxRetries,
                                  double margin_threshold = kDefaultMarginThreshold,
                                  int trials = kDefaultCoprimalityTrials);
struct BlurredPair {
  Frame public_frame, private_frame;
  std::optional<int> kernel_width_hint;
  std::string pair_id;
};
BlurredPair encode_frame(const Frame& latent, const CoprimePair& pair);  // on the GPU
Frame quantize_frame(const Frame& f, BitDepth depth);
// zero the `drop` least significant bits of every quantized sample (encoder.hpp:43;
// device: cbp_degrade_bits on the frame's integer codes)
Frame degrade_bits(const Frame& f, int drop);

// -------------------------------------------------------------- poly.hpp:14-62
inline constexpr double kDefaultGapThreshold = 1e-9;
Mat conv2_full(const Mat& a, const Mat& b);  // host utility (the device blur is encode_frame)
struct CofactorSolution {
  CVec k1, k2;
  double gap = 0.0;
};
CofactorSolution cofactor_null_solve(const CVec& p, const CVec& q, int t,
                                     double gap_threshold = kDefaultGapThreshold);
// 1D restrictions at arbitrary unit-circle points (poly.hpp:16-27; host utility)
struct SpectralSliceSet {
  Axis axis = Axis::Z1;
  std::vector<cplx> points;
  std::vector<CVec> slices;
};
SpectralSliceSet axis_dft(const Mat& plane, Axis axis, const std::vector<cplx>& points);
// leading size x size Bezout block (poly.hpp:30; device: cbp_bezout_leading_block)
CMat bezout_leading_block(const CVec& p, const CVec& q, int size);
struct SingularityResult {
  bool singular = true;
  double ratio = 0.0;  // sigma_min / sigma_max, 0 for the zero matrix
};
// sigma_min / sigma_max < tau (poly.hpp:38; device: cbp_numerical_singularity)
SingularityResult numerical_singularity(const CMat& m, double tau);
// unit-norm minimizer of |A x|, phase-normalized (poly.hpp:55; device: cbp_homogeneous_lsq)
CVec homogeneous_lsq(const CMat& a);
CMat sylvester_matrix(const CVec& p, const CVec& q);       // poly.hpp:59 (host utility)
int numerical_degree(const CVec& p, double rel_tol = 1e-12);  // poly.hpp:62 (host utility)

// --------------------------------------------------------------- fft.hpp:9-18
// unnormalized forward 2D DFT of any size and its 1/(M N)-normalized inverse (FP64, device:
// cbp_fft2)
CMat fft2(const CMat& x);
CMat fft2(const Mat& x);
CMat ifft2(const CMat& x);
CMat axis_roots_dft(const Mat& plane, Axis axis, int t);

// ---------------------------------------------------------- decoder.hpp:10-86
struct DecodeConfig {
  int search_min = 9;
  int search_max = 25;
  double tau = 1e-6;
  std::optional<double> epsilon;
  double gap_threshold = kDefaultGapThreshold;
  bool trust_hint = false;
  double max_imag_energy = 0.01;
  double negative_weight_tol = 0.01;
  bool validate = true;
};
struct WidthEstimate {
  int width = 0;
  bool clamped = false;
};
WidthEstimate estimate_kernel_width(const BlurredPair& pair, int search_min, int search_max, double tau);
struct ScaledKernelTransform {
  Axis axis = Axis::Z1;
  CMat values;
  Vec gaps;
};
ScaledKernelTransform sample_cofactors(const BlurredPair& pair, int width, Axis axis,
                                       double gap_threshold = kDefaultGapThreshold);
CMat complete_to_spectrum(const ScaledKernelTransform& skt);
struct ScaleResolution {
  CVec lambda, mu;
  double residual = 0.0;
};
ScaleResolution resolve_scales(const ScaledKernelTransform& a, const ScaledKernelTransform& b);
BlurKernel assemble_kernel(const CMat& a_spectrum, const CMat& b_spectrum, const ScaleResolution& scales,
                           double max_imag_energy = 0.01, double negative_weight_tol = 0.01);
Mat spectral_deblur(const Mat& blurred, const BlurKernel& k1, double epsilon);
struct StageTimings {
  double polynomial_evaluation_ms = 0.0;
  double kernel_degree_estimation_ms = 0.0;
  double kernel_estimation_1d_ms = 0.0;
  double kernel_estimation_2d_fft_ms = 0.0;
  double total_ms = 0.0;
};
struct DecodedFrame {
  Frame latent;
  BlurKernel kernel_estimate;
  int width_used = 0;
  bool width_clamped = false;
  StageTimings stage_timings;
  double validation_residual = 0.0;
};
DecodedFrame decode_frame(const BlurredPair& pair, const DecodeConfig& cfg = {});
double validate_pair(const BlurredPair& pair, const BlurKernel& k1_hat, const BlurKernel& k2_hat);

// ------------------------------------------------------------- synth.hpp:10-13
std::uint64_t frame_seed(std::uint64_t stream_seed, int frame_index);
Frame random_frame(int rows, int cols, int channels, std::uint64_t seed);

// ----------------------------------------------------------- metrics.hpp:8-10
double psnr(const Frame& reference, const Frame& test);
double psnr(const Mat& reference, const Mat& test);

}  // namespace cbp
