// cbp::core C++ API over the C ABI (include/cbp_cuda.h). Mirrors the reference
// implementation files proj/core/src/{decoder,encoder,image,kernel,error,synth,metrics}.cpp
// at the interface level: same argument checks and messages, same Errc codes, same value
// types. Device work (decode, deblur, sampling, solves, encode, validation) happens in
// libcbp_cuda.so; this file converts column-major FP64 planes to the device's row-major
// FP32 frames and back.
#include <algorithm>
#include <cmath>
#include <cstring>
#include <limits>
#include <random>
#include <string>

#include "cbp/cbp.hpp"
#include "cbp_cuda.h"

namespace cbp {
namespace {

struct Ctx {
  cbp_ctx* ptr = nullptr;
  Ctx() {
    const int st = cbp_create(0, &ptr);
    if (st) throw std::runtime_error(std::string(cbp_errc_name(st)) + ": no usable CUDA device (no CPU fallback)");
  }
  ~Ctx() { cbp_destroy(ptr); }
};

cbp_ctx* ctx() {
  thread_local Ctx c;
  return c.ptr;
}

[[noreturn]] void throw_status(int st) {
  const std::string msg = cbp_last_error(ctx());
  if (st >= 1 && st <= 18) throw Error(Errc(st - 1), msg, true);
  throw std::runtime_error(msg);
}

void check(int st) {
  if (st) throw_status(st);
}

struct DevBuf {
  void* p = nullptr;
  explicit DevBuf(size_t bytes) { check(cbp_device_alloc(ctx(), bytes, &p)); }
  ~DevBuf() { cbp_device_free(ctx(), p); }
  float* f() { return static_cast<float*>(p); }
};

// column-major FP64 planes -> row-major FP32 [channels][rows][cols]
std::vector<float> pack(const Frame& f) {
  const int r = f.rows(), c = f.cols();
  std::vector<float> out(size_t(f.channels()) * r * c);
  for (int k = 0; k < f.channels(); ++k)
    for (int i = 0; i < r; ++i)
      for (int j = 0; j < c; ++j) out[(size_t(k) * r + i) * c + j] = float(f.planes[k](i, j));
  return out;
}

Mat unpack_plane(const float* p, int rows, int cols, int ld, int out_rows, int out_cols) {
  Mat m(out_rows, out_cols);
  for (int i = 0; i < out_rows; ++i)
    for (int j = 0; j < out_cols; ++j) m(i, j) = double(p[size_t(i) * ld + j]);
  return m;
}

std::vector<double> rowmajor(const Mat& m) {
  std::vector<double> v(size_t(m.size()));
  for (long i = 0; i < m.rows(); ++i)
    for (long j = 0; j < m.cols(); ++j) v[size_t(i * m.cols() + j)] = m(i, j);
  return v;
}

std::vector<cplx> rowmajor(const CMat& m) {
  std::vector<cplx> v(size_t(m.size()));
  for (long i = 0; i < m.rows(); ++i)
    for (long j = 0; j < m.cols(); ++j) v[size_t(i * m.cols() + j)] = m(i, j);
  return v;
}

CMat from_rowmajor(const cplx* v, int rows, int cols) {
  CMat m(rows, cols);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) m(i, j) = v[size_t(i) * cols + j];
  return m;
}

void check_pair(const BlurredPair& pair) {  // decoder.cpp:19-29
  validate_frame(pair.public_frame);
  validate_frame(pair.private_frame);
  require(pair.public_frame.rows() == pair.private_frame.rows() &&
              pair.public_frame.cols() == pair.private_frame.cols() &&
              pair.public_frame.channels() == pair.private_frame.channels(),
          Errc::dim_mismatch, "pair frames disagree on dimensions");
  if (pair.kernel_width_hint)
    require(*pair.kernel_width_hint >= 1 && *pair.kernel_width_hint % 2 == 1, Errc::invalid_argument,
            "kernel width hint must be odd and >= 1");
}

cbp_decode_cfg to_c(const DecodeConfig& c) {
  cbp_decode_cfg o;
  o.search_min = c.search_min;
  o.search_max = c.search_max;
  o.tau = c.tau;
  o.has_epsilon = c.epsilon ? 1 : 0;
  o.epsilon = c.epsilon.value_or(0.0);
  o.gap_threshold = c.gap_threshold;
  o.trust_hint = c.trust_hint;
  o.max_imag_energy = c.max_imag_energy;
  o.negative_weight_tol = c.negative_weight_tol;
  o.validate = c.validate;
  return o;
}

struct DevPair {
  int ch, rows, cols;
  DevBuf pub, prv;
  explicit DevPair(const BlurredPair& p)
      : ch(p.public_frame.channels()), rows(p.public_frame.rows()), cols(p.public_frame.cols()),
        pub(sizeof(float) * size_t(ch) * rows * cols), prv(sizeof(float) * size_t(ch) * rows * cols) {
    const auto a = pack(p.public_frame), b = pack(p.private_frame);
    check(cbp_copy_to_device(ctx(), pub.p, a.data(), a.size() * sizeof(float)));
    check(cbp_copy_to_device(ctx(), prv.p, b.data(), b.size() * sizeof(float)));
  }
};

}  // namespace

const char* errc_name(Errc c) { return cbp_errc_name(int(c) + 1); }  // error.cpp:5-27

int bit_depth_bits(BitDepth d) { return d == BitDepth::u16 ? 16 : d == BitDepth::u8 ? 8 : 0; }

const char* bit_depth_name(BitDepth d) {  // image.cpp:5-12
  return d == BitDepth::u16 ? "u16" : d == BitDepth::u8 ? "u8" : "float32";
}

BitDepth bit_depth_from_name(const std::string& s) {  // image.cpp:14-19
  if (s == "float32") return BitDepth::f32;
  if (s == "u16") return BitDepth::u16;
  if (s == "u8") return BitDepth::u8;
  fail(Errc::invalid_argument, "unknown bit depth '" + s + "'");
}

void validate_frame(const Frame& f) {  // image.cpp:30-39
  require(f.channels() == 1 || f.channels() == 3, Errc::dim_mismatch, "frame must have 1 or 3 planes");
  for (const auto& p : f.planes) {
    require(p.rows() == f.rows() && p.cols() == f.cols(), Errc::dim_mismatch, "frame planes disagree on dimensions");
    require(p.rows() >= 1 && p.cols() >= 1, Errc::dim_mismatch, "empty frame plane");
    for (long i = 0; i < p.size(); ++i)
      require(std::isfinite(p.data()[i]), Errc::range_exceeded, "frame contains non-finite samples");
  }
}

Mat luma(const Frame& f) {  // image.cpp:41-45
  validate_frame(f);
  if (f.channels() == 1) return f.planes[0];
  Mat out(f.rows(), f.cols());
  for (long i = 0; i < out.size(); ++i)
    out.data()[i] = 0.299 * f.planes[0].data()[i] + 0.587 * f.planes[1].data()[i] + 0.114 * f.planes[2].data()[i];
  return out;
}

void validate_kernel(const BlurKernel& k, double sum_tol) {  // kernel.cpp:7-17
  require(k.width >= 1 && k.width % 2 == 1, Errc::invalid_argument, "kernel width must be odd and >= 1");
  require(k.weights.rows() == k.width && k.weights.cols() == k.width, Errc::dim_mismatch,
          "kernel weights must be width x width");
  double mn = std::numeric_limits<double>::infinity();
  for (long i = 0; i < k.weights.size(); ++i) {
    require(std::isfinite(k.weights.data()[i]), Errc::invalid_argument, "kernel weights must be finite");
    mn = std::min(mn, k.weights.data()[i]);
  }
  require(mn >= 0.0, Errc::invalid_argument, "kernel weights must be nonnegative");
  require(std::abs(k.weights.sum() - 1.0) <= sum_tol, Errc::invalid_argument, "kernel weights must sum to 1");
}

double coprimality_check(const BlurKernel& k1, const BlurKernel& k2, int trials) {  // encoder.cpp:45-64
  validate_kernel(k1);
  validate_kernel(k2);
  require(k1.width == k2.width, Errc::dim_mismatch, "kernel widths differ");
  require(trials >= 1, Errc::invalid_argument, "trials must be >= 1");
  const auto a = rowmajor(k1.weights), b = rowmajor(k2.weights);
  return cbp_coprimality_check(a.data(), b.data(), k1.width, trials);
}

CoprimePair generate_coprime_pair(int width, std::uint64_t seed, int max_retries, double margin_threshold,
                                  int trials) {  // encoder.cpp:66-81
  require(width >= 3 && width <= 63 && width % 2 == 1, Errc::invalid_argument,
          "kernel width must be odd, within [3,63]");
  require(max_retries >= 1, Errc::invalid_argument, "max_retries must be >= 1");
  require(margin_threshold > 0.0, Errc::invalid_argument, "margin threshold must be positive");
  std::vector<double> a(size_t(width) * width), b(a.size());
  double margin = 0.0;
  const int st = cbp_generate_coprime_pair(width, seed, max_retries, margin_threshold, trials, a.data(), b.data(),
                                           &margin);
  if (st == CBP_COPRIMALITY_FAILURE)
    fail(Errc::coprimality_failure, "no coprime pair of width " + std::to_string(width) + " within " +
                                        std::to_string(max_retries) + " draws");
  CoprimePair p;
  p.k1 = {width, Mat(width, width)};
  p.k2 = {width, Mat(width, width)};
  for (int i = 0; i < width; ++i)
    for (int j = 0; j < width; ++j) p.k1.weights(i, j) = a[size_t(i) * width + j], p.k2.weights(i, j) = b[size_t(i) * width + j];
  p.coprimality_margin = margin;
  p.seed = seed;
  return p;
}

BlurredPair encode_frame(const Frame& latent, const CoprimePair& pair) {  // encoder.cpp:83-103
  validate_frame(latent);
  validate_kernel(pair.k1);
  validate_kernel(pair.k2);
  require(pair.k1.width == pair.k2.width, Errc::dim_mismatch, "kernel widths differ");
  const int t = pair.k1.width, ch = latent.channels(), r = latent.rows(), c = latent.cols();
  require(r >= t && c >= t, Errc::frame_too_small, "latent frame smaller than the blur kernel");
  const int ro = r + t - 1, co = c + t - 1;
  DevBuf lat(sizeof(float) * size_t(ch) * r * c), pub(sizeof(float) * size_t(ch) * ro * co),
      prv(sizeof(float) * size_t(ch) * ro * co);
  const auto packed = pack(latent);
  check(cbp_copy_to_device(ctx(), lat.p, packed.data(), packed.size() * sizeof(float)));
  const auto k1 = rowmajor(pair.k1.weights), k2 = rowmajor(pair.k2.weights);
  check(cbp_encode_frames(ctx(), lat.f(), 1, ch, r, c, c, k1.data(), k2.data(), t, pub.f(), prv.f(), co, nullptr));
  std::vector<float> hp(size_t(ch) * ro * co), hq(hp.size());
  check(cbp_copy_to_host(ctx(), hp.data(), pub.p, hp.size() * sizeof(float)));
  check(cbp_copy_to_host(ctx(), hq.data(), prv.p, hq.size() * sizeof(float)));
  BlurredPair out;
  out.public_frame.index = out.private_frame.index = latent.index;
  for (int k = 0; k < ch; ++k) {
    out.public_frame.planes.push_back(unpack_plane(hp.data() + size_t(k) * ro * co, ro, co, co, ro, co));
    out.private_frame.planes.push_back(unpack_plane(hq.data() + size_t(k) * ro * co, ro, co, co, ro, co));
  }
  out.kernel_width_hint = t;
  std::uint64_t h = cbp_splitmix64(pair.seed ^ (0xb1e55ed * std::uint64_t(t)));
  static const char* digits = "0123456789abcdef";
  out.pair_id.assign(16, '0');
  for (int i = 15; i >= 0; --i, h >>= 4) out.pair_id[size_t(i)] = digits[h & 0xf];
  return out;
}

Frame quantize_frame(const Frame& f, BitDepth depth) {  // encoder.cpp:105-120
  validate_frame(f);
  require(depth != BitDepth::f32, Errc::invalid_argument, "quantization depth must be u8 or u16");
  const double maxv = double((1u << bit_depth_bits(depth)) - 1);
  Frame out = f;
  out.bit_depth = depth;
  for (auto& plane : out.planes)
    for (long i = 0; i < plane.size(); ++i) {
      const double x = plane.data()[i];
      require(x >= -1e-9 && x <= 1.0 + 1e-9, Errc::range_exceeded, "samples outside [0,1]");
      plane.data()[i] = std::round(std::min(1.0, std::max(0.0, x)) * maxv) / maxv;
    }
  return out;
}

Frame degrade_bits(const Frame& f, int drop) {  // encoder.cpp:124-139
  validate_frame(f);
  require(f.bit_depth != BitDepth::f32, Errc::not_quantized, "bit-precision degradation needs a quantized frame");
  const int bits = bit_depth_bits(f.bit_depth);
  require(drop >= 0 && drop < bits, Errc::invalid_argument, "drop must lie in [0, bit width)");
  if (drop == 0) return f;
  const double maxv = double((1u << bits) - 1);
  const int r = f.rows(), c = f.cols(), planes = f.channels();
  const size_t n = size_t(planes) * r * c;
  // the frame's integer codes (lround(x * maxv), encoder.cpp:134) masked on the device
  std::vector<unsigned short> c16(bits == 16 ? n : 0);
  std::vector<unsigned char> c8(bits == 8 ? n : 0);
  for (int k = 0; k < planes; ++k)
    for (int i = 0; i < r; ++i)
      for (int j = 0; j < c; ++j) {
        const long code = std::lround(f.planes[k](i, j) * maxv);
        const size_t at = (size_t(k) * r + i) * c + j;
        if (bits == 16) c16[at] = static_cast<unsigned short>(code);
        else c8[at] = static_cast<unsigned char>(code);
      }
  const size_t bytes = n * (bits == 16 ? 2 : 1);
  DevBuf d(bytes);
  void* host = bits == 16 ? static_cast<void*>(c16.data()) : static_cast<void*>(c8.data());
  check(cbp_copy_to_device(ctx(), d.p, host, bytes));
  check(cbp_degrade_bits(ctx(), d.p, bits, planes, r, c, c, drop, nullptr));
  check(cbp_copy_to_host(ctx(), host, d.p, bytes));
  Frame out = f;
  for (int k = 0; k < planes; ++k)
    for (int i = 0; i < r; ++i)
      for (int j = 0; j < c; ++j) {
        const size_t at = (size_t(k) * r + i) * c + j;
        out.planes[k](i, j) = double(bits == 16 ? c16[at] : c8[at]) / maxv;
      }
  return out;
}

Mat conv2_full(const Mat& a, const Mat& b) {  // poly.cpp:27-38 (host utility)
  require(a.size() > 0 && b.size() > 0, Errc::dim_mismatch, "conv2_full needs nonempty inputs");
  const Mat& big = a.size() >= b.size() ? a : b;
  const Mat& small = a.size() >= b.size() ? b : a;
  Mat out = Mat::Zero(a.rows() + b.rows() - 1, a.cols() + b.cols() - 1);
  for (long n = 0; n < small.cols(); ++n)
    for (long m = 0; m < small.rows(); ++m) {
      const double w = small(m, n);
      if (w == 0.0) continue;
      for (long j = 0; j < big.cols(); ++j)
        for (long i = 0; i < big.rows(); ++i) out(m + i, n + j) += w * big(i, j);
    }
  return out;
}

CofactorSolution cofactor_null_solve(const CVec& p, const CVec& q, int t, double gap_threshold) {
  require(t >= 1, Errc::invalid_argument, "cofactor width must be >= 1");
  require(p.size() >= t && q.size() >= t, Errc::invalid_argument, "slice degree below cofactor degree");
  const long L = std::max(p.size(), q.size());  // zero padding leaves the system unchanged
  std::vector<cplx> pp(static_cast<size_t>(L), cplx(0.0)), qq(static_cast<size_t>(L), cplx(0.0)), k1(static_cast<size_t>(t)), k2(static_cast<size_t>(t));
  for (long i = 0; i < p.size(); ++i) pp[size_t(i)] = p[i];
  for (long i = 0; i < q.size(); ++i) qq[size_t(i)] = q[i];
  double gap = 0.0;
  int status = 0;
  check(cbp_cofactor_solve_batch(ctx(), reinterpret_cast<double*>(pp.data()), reinterpret_cast<double*>(qq.data()), 1,
                                 int(L), t, gap_threshold, reinterpret_cast<double*>(k1.data()),
                                 reinterpret_cast<double*>(k2.data()), &gap, &status, nullptr));
  CofactorSolution s;
  s.k1 = CVec(t);
  s.k2 = CVec(t);
  for (int i = 0; i < t; ++i) s.k1[i] = k1[size_t(i)], s.k2[i] = k2[size_t(i)];
  s.gap = gap;
  return s;
}

SpectralSliceSet axis_dft(const Mat& plane, Axis axis, const std::vector<cplx>& points) {  // poly.cpp:40-64
  require(plane.size() > 0, Errc::invalid_argument, "axis_dft needs a nonempty plane");
  for (const cplx& w : points)
    require(std::abs(std::abs(w) - 1.0) <= 1e-12, Errc::non_unit_sample_point, "sample point off the unit circle");
  const long d = axis == Axis::Z1 ? plane.rows() : plane.cols();
  const long len = axis == Axis::Z1 ? plane.cols() : plane.rows();
  SpectralSliceSet out;
  out.axis = axis;
  out.points = points;
  for (const cplx& w : points) {
    const double theta = std::arg(w);
    std::vector<double> pr(static_cast<size_t>(d)), pi(static_cast<size_t>(d));
    for (long m = 0; m < d; ++m) pr[size_t(m)] = std::cos(theta * double(m)), pi[size_t(m)] = std::sin(theta * double(m));
    CVec slice(len);
    for (long n = 0; n < len; ++n) {
      double re = 0.0, im = 0.0;
      for (long m = 0; m < d; ++m) {
        const double x = axis == Axis::Z1 ? plane(m, n) : plane(n, m);
        re += x * pr[size_t(m)];
        im += x * pi[size_t(m)];
      }
      slice[n] = cplx(re, im);
    }
    out.slices.push_back(slice);
  }
  return out;
}

CMat bezout_leading_block(const CVec& p, const CVec& q, int size) {  // poly.cpp:66-79
  CMat out(size > 0 ? size : 0, size > 0 ? size : 0);
  std::vector<cplx> o(size_t(size > 0 ? size : 0) * (size > 0 ? size : 0));
  check(cbp_bezout_leading_block(ctx(), reinterpret_cast<const double*>(p.data()), int(p.size()),
                                 reinterpret_cast<const double*>(q.data()), int(q.size()), size,
                                 reinterpret_cast<double*>(o.data()), nullptr));
  return from_rowmajor(o.data(), size, size);
}

SingularityResult numerical_singularity(const CMat& m, double tau) {  // poly.cpp:81-91
  require(m.rows() == m.cols() && m.rows() >= 1, Errc::invalid_argument, "singularity test needs a square matrix");
  const auto a = rowmajor(m);
  int singular = 1;
  double ratio = 0.0;
  check(cbp_numerical_singularity(ctx(), reinterpret_cast<const double*>(a.data()), int(m.rows()), tau, &singular,
                                  &ratio, nullptr));
  return {singular != 0, ratio};
}

CVec homogeneous_lsq(const CMat& a) {  // poly.cpp:123-130
  require(a.rows() >= a.cols() && a.cols() >= 1, Errc::invalid_argument, "homogeneous system needs rows >= cols");
  const auto v = rowmajor(a);
  std::vector<cplx> x(size_t(a.cols()));
  check(cbp_homogeneous_lsq(ctx(), reinterpret_cast<const double*>(v.data()), int(a.rows()), int(a.cols()),
                            reinterpret_cast<double*>(x.data()), nullptr));
  CVec out(a.cols());
  for (long i = 0; i < a.cols(); ++i) out[i] = x[size_t(i)];
  return out;
}

CMat sylvester_matrix(const CVec& p, const CVec& q) {  // poly.cpp:132-141
  require(p.size() >= 1 && q.size() >= 1, Errc::invalid_argument, "empty polynomial");
  const long m = p.size() - 1, n = q.size() - 1;
  CMat s = CMat::Zero(m + n, m + n);
  for (long r = 0; r < n; ++r)
    for (long k = 0; k <= m; ++k) s(r, r + k) = p[m - k];
  for (long r = 0; r < m; ++r)
    for (long k = 0; k <= n; ++k) s(n + r, r + k) = q[n - k];
  return s;
}

int numerical_degree(const CVec& p, double rel_tol) {  // poly.cpp:143-150
  if (p.size() == 0) return -1;
  double mx = 0.0;
  for (long i = 0; i < p.size(); ++i) mx = std::max(mx, std::abs(p[i]));
  if (mx == 0.0) return -1;
  for (long i = p.size() - 1; i >= 0; --i)
    if (std::abs(p[i]) > rel_tol * mx) return int(i);
  return -1;
}

static CMat fft2_device(const CMat& x, int inverse) {
  require(x.rows() >= 1 && x.cols() >= 1, Errc::invalid_argument, "fft2 needs a nonempty matrix");
  const auto v = rowmajor(x);
  std::vector<cplx> o(v.size());
  check(cbp_fft2(ctx(), reinterpret_cast<const double*>(v.data()), int(x.rows()), int(x.cols()), inverse,
                 reinterpret_cast<double*>(o.data()), nullptr));
  return from_rowmajor(o.data(), int(x.rows()), int(x.cols()));
}

CMat fft2(const CMat& x) { return fft2_device(x, 0); }  // fft.cpp:166-168

CMat fft2(const Mat& x) {  // fft.cpp:170-179
  CMat c(x.rows(), x.cols());
  for (long j = 0; j < x.cols(); ++j)
    for (long i = 0; i < x.rows(); ++i) c(i, j) = cplx(x(i, j), 0.0);
  return fft2_device(c, 0);
}

CMat ifft2(const CMat& x) { return fft2_device(x, 1); }  // fft.cpp:191-195

CMat axis_roots_dft(const Mat& plane, Axis axis, int t) {  // fft.cpp:197-213
  require(plane.rows() >= 1 && plane.cols() >= 1, Errc::invalid_argument, "axis_roots_dft needs a nonempty plane");
  require(t >= 1, Errc::invalid_argument, "axis_roots_dft needs t >= 1");
  Frame f;
  f.planes.push_back(plane);
  BlurredPair bp;
  bp.public_frame = bp.private_frame = f;
  DevPair d(bp);
  const int ax = axis == Axis::Z1 ? CBP_AXIS_Z1 : CBP_AXIS_Z2;
  const int L = axis == Axis::Z1 ? d.cols : d.rows;
  std::vector<cplx> s1(size_t(t) * L), s2(s1.size());
  check(cbp_sample_slices(ctx(), d.pub.f(), d.prv.f(), 1, d.rows, d.cols, d.cols, t, ax,
                          reinterpret_cast<double*>(s1.data()), reinterpret_cast<double*>(s2.data()), nullptr));
  if (axis == Axis::Z1) return from_rowmajor(s1.data(), t, L);  // t x N, row i = slice
  CMat out(L, t);                                                // M x t, column i = slice
  for (int i = 0; i < t; ++i)
    for (int m = 0; m < L; ++m) out(m, i) = s1[size_t(i) * L + m];
  return out;
}

WidthEstimate estimate_kernel_width(const BlurredPair& pair, int search_min, int search_max, double tau) {
  check_pair(pair);
  DevPair d(pair);
  int w = 0, cl = 0;
  check(cbp_estimate_kernel_width(ctx(), d.pub.f(), d.prv.f(), d.ch, d.rows, d.cols, d.cols, search_min, search_max,
                                  tau, &w, &cl, nullptr));
  return {w, cl != 0};
}

ScaledKernelTransform sample_cofactors(const BlurredPair& pair, int width, Axis axis, double gap_threshold) {
  check_pair(pair);
  DevPair d(pair);
  std::vector<cplx> vals(size_t(width) * std::max(width, 1));
  std::vector<double> gaps(size_t(std::max(width, 1)));
  check(cbp_sample_cofactors(ctx(), d.pub.f(), d.prv.f(), d.ch, d.rows, d.cols, d.cols, width,
                             axis == Axis::Z1 ? CBP_AXIS_Z1 : CBP_AXIS_Z2, gap_threshold,
                             reinterpret_cast<double*>(vals.data()), gaps.data(), nullptr));
  ScaledKernelTransform s;
  s.axis = axis;
  s.values = from_rowmajor(vals.data(), width, width);
  s.gaps = Vec(width);
  for (int i = 0; i < width; ++i) s.gaps[i] = gaps[size_t(i)];
  return s;
}

CMat complete_to_spectrum(const ScaledKernelTransform& skt) {  // decoder.cpp:240-246
  const int t = int(skt.values.rows());
  require(skt.values.cols() == t && t >= 1, Errc::dim_mismatch, "scaled kernel transform must be square");
  const auto v = rowmajor(skt.values);
  std::vector<cplx> out(v.size());
  check(cbp_complete_to_spectrum(ctx(), reinterpret_cast<const double*>(v.data()), t,
                                 skt.axis == Axis::Z1 ? CBP_AXIS_Z1 : CBP_AXIS_Z2,
                                 reinterpret_cast<double*>(out.data()), nullptr));
  return from_rowmajor(out.data(), t, t);
}

ScaleResolution resolve_scales(const ScaledKernelTransform& a, const ScaledKernelTransform& b) {
  require(a.axis == Axis::Z1 && b.axis == Axis::Z2, Errc::invalid_argument,
          "resolve_scales expects a z1 transform and a z2 transform");
  require(a.values.rows() == b.values.rows() && a.values.cols() == b.values.cols(), Errc::dim_mismatch,
          "transforms disagree on size");
  const int t = int(a.values.rows());
  const auto av = rowmajor(a.values), bv = rowmajor(b.values);
  std::vector<cplx> lam(static_cast<size_t>(t)), mu(static_cast<size_t>(t));
  ScaleResolution r;
  check(cbp_resolve_scales(ctx(), reinterpret_cast<const double*>(av.data()), reinterpret_cast<const double*>(bv.data()),
                           t, reinterpret_cast<double*>(lam.data()), reinterpret_cast<double*>(mu.data()), &r.residual,
                           nullptr));
  r.lambda = CVec(t);
  r.mu = CVec(t);
  for (int i = 0; i < t; ++i) r.lambda[i] = lam[size_t(i)], r.mu[i] = mu[size_t(i)];
  return r;
}

BlurKernel assemble_kernel(const CMat& a_spectrum, const CMat& b_spectrum, const ScaleResolution& scales,
                           double max_imag_energy, double negative_weight_tol) {  // decoder.cpp:256-271
  const int t = int(a_spectrum.rows());
  require(a_spectrum.cols() == t && b_spectrum.rows() == t && b_spectrum.cols() == t, Errc::dim_mismatch,
          "spectrum estimates must be square and equal-sized");
  require(scales.lambda.size() == t && scales.mu.size() == t, Errc::dim_mismatch,
          "scale vectors must match the kernel width");
  const auto A = rowmajor(a_spectrum), B = rowmajor(b_spectrum);
  std::vector<double> w(size_t(t) * t);
  check(cbp_assemble_kernel(ctx(), reinterpret_cast<const double*>(A.data()), reinterpret_cast<const double*>(B.data()),
                            reinterpret_cast<const double*>(scales.lambda.data()),
                            reinterpret_cast<const double*>(scales.mu.data()), t, max_imag_energy, negative_weight_tol,
                            w.data(), nullptr));
  BlurKernel k{t, Mat(t, t)};
  for (int i = 0; i < t; ++i)
    for (int j = 0; j < t; ++j) k.weights(i, j) = w[size_t(i) * t + j];
  return k;
}

Mat spectral_deblur(const Mat& blurred, const BlurKernel& k1, double epsilon) {  // decoder.cpp:273-278
  validate_kernel(k1);
  require(epsilon >= 0.0, Errc::invalid_argument, "epsilon must be nonnegative");
  Frame f;
  f.planes.push_back(blurred);
  const int r = int(blurred.rows()), c = int(blurred.cols()), t = k1.width;
  require(r >= t && c >= t, Errc::frame_too_small, "blurred frame smaller than the kernel");
  DevBuf in(sizeof(float) * size_t(r) * c), out(sizeof(float) * size_t(r) * c);
  const auto packed = pack(f);
  check(cbp_copy_to_device(ctx(), in.p, packed.data(), packed.size() * sizeof(float)));
  const auto k = rowmajor(k1.weights);
  check(cbp_spectral_deblur(ctx(), in.f(), 1, 1, r, c, c, k.data(), t, epsilon, out.f(), c, nullptr));
  std::vector<float> h(size_t(r) * c);
  check(cbp_copy_to_host(ctx(), h.data(), out.p, h.size() * sizeof(float)));
  return unpack_plane(h.data(), r, c, c, r - t + 1, c - t + 1);
}

DecodedFrame decode_frame(const BlurredPair& pair, const DecodeConfig& cfg) {  // decoder.cpp:280-378
  check_pair(pair);
  DevPair d(pair);
  DevBuf out(sizeof(float) * size_t(d.ch) * d.rows * d.cols);
  const cbp_decode_cfg c = to_c(cfg);
  const int hint = pair.kernel_width_hint.value_or(0);
  cbp_decode_info info;
  check(cbp_decode_frames(ctx(), d.pub.f(), d.prv.f(), 1, d.ch, d.rows, d.cols, d.cols, &hint, &c, out.f(), d.cols,
                          &info, nullptr));
  std::vector<float> h(size_t(d.ch) * d.rows * d.cols);
  check(cbp_copy_to_host(ctx(), h.data(), out.p, h.size() * sizeof(float)));
  const int t = info.width_used;
  DecodedFrame res;
  for (int k = 0; k < d.ch; ++k)
    res.latent.planes.push_back(
        unpack_plane(h.data() + size_t(k) * d.rows * d.cols, d.rows, d.cols, d.cols, d.rows - t + 1, d.cols - t + 1));
  res.latent.bit_depth = BitDepth::f32;
  res.latent.index = pair.public_frame.index;
  res.kernel_estimate = {t, Mat(t, t)};
  for (int i = 0; i < t; ++i)
    for (int j = 0; j < t; ++j) res.kernel_estimate.weights(i, j) = info.kernel[i * t + j];
  res.width_used = t;
  res.width_clamped = info.width_clamped != 0;
  res.stage_timings = {info.stage_ms[0], info.stage_ms[1], info.stage_ms[2], info.stage_ms[3], info.stage_ms[4]};
  res.validation_residual = info.validation_residual;
  return res;
}

double validate_pair(const BlurredPair& pair, const BlurKernel& k1_hat, const BlurKernel& k2_hat) {
  check_pair(pair);  // decoder.cpp:380-395
  validate_kernel(k1_hat);
  validate_kernel(k2_hat);
  require(k1_hat.width == k2_hat.width, Errc::dim_mismatch, "kernel widths differ");
  DevPair d(pair);
  const auto a = rowmajor(k1_hat.weights), b = rowmajor(k2_hat.weights);
  double r = 0.0;
  check(cbp_validate_pair(ctx(), d.pub.f(), d.prv.f(), d.ch, d.rows, d.cols, d.cols, a.data(), b.data(), k1_hat.width,
                          &r, nullptr));
  return r;
}

std::uint64_t frame_seed(std::uint64_t stream_seed, int frame_index) {  // synth.cpp / rng.hpp:27-29
  return cbp_frame_seed(stream_seed, frame_index);
}

Frame random_frame(int rows, int cols, int channels, std::uint64_t seed) {  // synth.cpp:12-22
  require(rows > 0 && cols > 0, Errc::invalid_argument, "bad frame geometry");
  require(channels == 1 || channels == 3, Errc::invalid_argument, "channels must be 1 or 3");
  std::mt19937_64 eng(seed);
  Frame f;
  f.planes.assign(size_t(channels), ImagePlane(rows, cols));
  for (ImagePlane& p : f.planes)
    for (int c = 0; c < cols; ++c)
      for (int r = 0; r < rows; ++r) p(r, c) = double(eng() >> 11) * 0x1.0p-53;
  return f;
}

static double psnr_from(double sq, double count) {  // metrics.cpp:11-14
  return sq == 0.0 ? std::numeric_limits<double>::infinity() : 10.0 * std::log10(count / sq);
}

double psnr(const Mat& reference, const Mat& test) {
  require(reference.rows() == test.rows() && reference.cols() == test.cols(), Errc::dim_mismatch,
          "psnr operands differ in shape");
  require(reference.size() > 0, Errc::invalid_argument, "psnr of empty image");
  double sq = 0.0;
  for (long i = 0; i < reference.size(); ++i) {
    const double d = reference.data()[i] - test.data()[i];
    sq += d * d;
  }
  return psnr_from(sq, double(reference.size()));
}

double psnr(const Frame& reference, const Frame& test) {
  validate_frame(reference);
  validate_frame(test);
  require(reference.channels() == test.channels() && reference.rows() == test.rows() &&
              reference.cols() == test.cols(),
          Errc::dim_mismatch, "psnr operands differ in shape");
  double sq = 0.0;
  for (int c = 0; c < reference.channels(); ++c)
    for (long i = 0; i < reference.planes[c].size(); ++i) {
      const double d = reference.planes[c].data()[i] - test.planes[c].data()[i];
      sq += d * d;
    }
  return psnr_from(sq, double(reference.rows()) * reference.cols() * reference.channels());
}

}  // namespace cbp
