// ============================================================================
// CBP ORACLE — TEST INFRASTRUCTURE ONLY. NOT PART OF THE PRODUCT PATH.
//
// A CPU, FP64 restatement of the reference CBP decryption path
// (/root/reference/proj/core/src/{decoder,poly,fft,image,kernel,encoder,synth}.cpp
// and rng.hpp). Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline /
// --impl reference leg may load it, and only as the checker or the timed CPU
// baseline. The CUDA product path (paper_1203_4874_b200/csrc) never calls it.
//
// The reference links Eigen3 (JacobiSVD) and FFTW3, neither of which is present
// in this image, so the reference cannot be compiled here. This restatement
// replaces them with an in-house complex Householder-QR + one-sided Jacobi SVD and
// a mixed-radix (2/3/4/5/7/generic) FFT, both FP64. It is pinned against the
// reference's own known-answer tests (tests/test_oracle_kat.py) and against an
// independent numpy/LAPACK restatement (oracle/np_ref.py).
// ============================================================================
#pragma once

#include <complex>
#include <cstdint>
#include <optional>
#include <stdexcept>
#include <string>
#include <vector>

namespace orc {

using cplx = std::complex<double>;

// Dense row-major matrices. Index (m, n): m = row = z1 power, n = col = z2 power
// (reference types.hpp:15-17). Storage order differs from Eigen's column-major
// but every loop that fixes an order (RNG fills, folds) follows the reference.
template <class T>
struct Dense {
  int r = 0, c = 0;
  std::vector<T> v;
  Dense() = default;
  Dense(int rows, int cols, T fill = T()) : r(rows), c(cols), v(size_t(rows) * cols, fill) {}
  T& operator()(int i, int j) { return v[size_t(i) * c + j]; }
  const T& operator()(int i, int j) const { return v[size_t(i) * c + j]; }
  int rows() const { return r; }
  int cols() const { return c; }
  size_t size() const { return v.size(); }
  T* data() { return v.data(); }
  const T* data() const { return v.data(); }
};
using Mat = Dense<double>;
using CMat = Dense<cplx>;
using Vec = std::vector<double>;
using CVec = std::vector<cplx>;

enum class Axis { Z1, Z2 };
inline const char* axis_name(Axis a) { return a == Axis::Z1 ? "z1" : "z2"; }

// error.hpp:8-27 — order matters: C-ABI status = 1 + index.
enum class Errc {
  invalid_argument, non_unit_sample_point, degenerate_input, ill_conditioned,
  coprimality_failure, frame_too_small, range_exceeded, not_quantized, inconsistent_axes,
  ill_conditioned_slice, degenerate_scales, non_real_kernel, dim_mismatch, io_failure,
  corrupt_manifest, missing_frame, format_violation, pair_mismatch,
};
const char* errc_name(Errc c);

class Error : public std::runtime_error {
 public:
  Error(Errc code, const std::string& what)
      : std::runtime_error(std::string(errc_name(code)) + ": " + what), code_(code) {}
  Errc code() const { return code_; }

 private:
  Errc code_;
};
[[noreturn]] inline void fail(Errc code, const std::string& what) { throw Error(code, what); }
inline void require(bool ok, Errc code, const std::string& what) {
  if (!ok) fail(code, what);
}

// ---- rng.hpp / synth.cpp ----
uint64_t splitmix64(uint64_t x);
uint64_t frame_seed(uint64_t stream_seed, int frame_index);
struct Frame {
  std::vector<Mat> planes;
  int bit_depth = 0;  // 0 f32, 16 u16, 8 u8
  int index = 0;
  int rows() const { return planes.empty() ? 0 : planes[0].r; }
  int cols() const { return planes.empty() ? 0 : planes[0].c; }
  int channels() const { return int(planes.size()); }
};
Frame random_frame(int rows, int cols, int channels, uint64_t seed);
// tests/support.hpp:31-39 (libstdc++ uniform_real_distribution, bit-identical here)
Mat random_mat(int rows, int cols, uint64_t seed, double lo, double hi);

// ---- kernel.hpp / image.cpp ----
struct BlurKernel {
  int width = 1;
  Mat weights;
};
struct CoprimePair {
  BlurKernel k1, k2;
  double coprimality_margin = 0.0;
  uint64_t seed = 0;
};
struct BlurredPair {
  Frame public_frame, private_frame;
  std::optional<int> kernel_width_hint;
};
void validate_kernel(const BlurKernel& k, double sum_tol = 1e-9);
void validate_frame(const Frame& f);
Mat luma(const Frame& f);

// ---- poly.hpp ----
inline constexpr double kDefaultGapThreshold = 1e-9;
Mat conv2_full(const Mat& a, const Mat& b);
CVec axis_dft_slice(const Mat& plane, Axis axis, cplx w);
CMat bezout_leading_block(const CVec& p, const CVec& q, int size);
struct SingularityResult {
  bool singular = true;
  double ratio = 0.0;
};
SingularityResult numerical_singularity(const CMat& m, double tau);
struct CofactorSolution {
  CVec k1, k2;
  double gap = 0.0;
};
CofactorSolution cofactor_null_solve(const CVec& p, const CVec& q, int t,
                                     double gap_threshold = kDefaultGapThreshold);
CVec homogeneous_lsq(const CMat& a);
CMat sylvester_matrix(const CVec& p, const CVec& q);
int numerical_degree(const CVec& p, double rel_tol = 1e-12);

// SVD helper: singular values (descending) and, optionally, the full V.
void svd(const CMat& a, Vec& sv, CMat* v);

// ---- fft.hpp ----
CMat fft2(const CMat& x);
CMat ifft2(const CMat& x);
CMat axis_roots_dft(const Mat& plane, Axis axis, int t);
CMat axis_spectrum_half(const Mat& plane, Axis axis);
int friendly_size(int n);
void fft1(cplx* x, int n, int sign);  // in place, unnormalized

// ---- encoder.hpp ----
double coprimality_check(const BlurKernel& k1, const BlurKernel& k2, int trials = 4);
CoprimePair generate_coprime_pair(int width, uint64_t seed, int max_retries = 16,
                                  double margin_threshold = 1e-6, int trials = 4);
BlurredPair encode_frame(const Frame& latent, const CoprimePair& pair);
Frame quantize_frame(const Frame& f, int bits);
Frame degrade_bits(const Frame& f, int drop);

// ---- decoder.hpp ----
struct DecodeConfig {
  int search_min = 9, search_max = 25;
  double tau = 1e-6;
  std::optional<double> epsilon;
  double gap_threshold = kDefaultGapThreshold;
  bool trust_hint = false;
  double max_imag_energy = 0.01, negative_weight_tol = 0.01;
  bool validate = true;
};
struct WidthEstimate {
  int width = 0;
  bool clamped = false;
};
struct ScaledKernelTransform {
  Axis axis = Axis::Z1;
  CMat values;
  Vec gaps;
};
struct ScaleResolution {
  CVec lambda, mu;
  double residual = 0.0;
};
struct StageTimings {
  double polynomial_evaluation_ms = 0, kernel_degree_estimation_ms = 0,
         kernel_estimation_1d_ms = 0, kernel_estimation_2d_fft_ms = 0, total_ms = 0;
};
struct DecodedFrame {
  Frame latent;
  BlurKernel kernel_estimate;
  int width_used = 0;
  bool width_clamped = false;
  StageTimings stage_timings;
  double validation_residual = 0.0;
  double epsilon_used = 0.0;
};
WidthEstimate estimate_kernel_width(const BlurredPair& pair, int search_min, int search_max,
                                    double tau);
ScaledKernelTransform sample_cofactors(const BlurredPair& pair, int width, Axis axis,
                                       double gap_threshold = kDefaultGapThreshold);
CMat complete_to_spectrum(const ScaledKernelTransform& skt);
ScaleResolution resolve_scales(const ScaledKernelTransform& a, const ScaledKernelTransform& b);
ScaleResolution resolve_completed(const CMat& a_spec, const CMat& b_spec);
BlurKernel assemble_kernel(const CMat& a_spectrum, const CMat& b_spectrum,
                           const ScaleResolution& scales, double max_imag_energy = 0.01,
                           double negative_weight_tol = 0.01);
Mat spectral_deblur(const Mat& blurred, const BlurKernel& k1, double epsilon);
DecodedFrame decode_frame(const BlurredPair& pair, const DecodeConfig& cfg = {});
double validate_pair(const BlurredPair& pair, const BlurKernel& k1_hat, const BlurKernel& k2_hat);
double psnr(const Mat& reference, const Mat& test);

}  // namespace orc
