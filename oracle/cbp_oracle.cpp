// CBP ORACLE — TEST INFRASTRUCTURE ONLY (see cbp_oracle.hpp header).
// FP64 CPU restatement of the reference decode path; every function cites the
// reference file:line it follows (paths relative to /root/reference/proj).
#include "cbp_oracle.hpp"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <map>
#include <numbers>
#include <random>

namespace orc {

const char* errc_name(Errc c) {  // core/src/error.cpp:5-27
  static const char* names[] = {
      "InvalidArgument", "NonUnitSamplePoint", "DegenerateInput", "IllConditioned",
      "CoprimalityFailure", "FrameTooSmall", "RangeExceeded", "NotQuantized",
      "InconsistentAxes", "IllConditionedSlice", "DegenerateScales", "NonRealKernel",
      "DimMismatch", "IoFailure", "CorruptManifest", "MissingFrame", "FormatViolation",
      "PairMismatch"};
  int i = int(c);
  return (i >= 0 && i < 18) ? names[i] : "Error";
}

// ------------------------------------------------------------------ rng.hpp
uint64_t splitmix64(uint64_t x) {  // core/src/rng.hpp:8-13
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

namespace {
class UniformRng {  // core/src/rng.hpp:17-25
 public:
  explicit UniformRng(uint64_t seed) : eng_(seed) {}
  double next() { return double(eng_() >> 11) * 0x1.0p-53; }

 private:
  std::mt19937_64 eng_;
};
}  // namespace

uint64_t frame_seed(uint64_t stream_seed, int frame_index) {  // rng.hpp:27-29
  return splitmix64(stream_seed ^ (0x9E3779B97F4A7C15ull * uint64_t(frame_index) + 1));
}

Frame random_frame(int rows, int cols, int channels, uint64_t seed) {  // synth.cpp:12-22
  require(rows > 0 && cols > 0, Errc::invalid_argument, "bad frame geometry");
  require(channels == 1 || channels == 3, Errc::invalid_argument, "channels must be 1 or 3");
  UniformRng rng(seed);
  Frame f;
  f.planes.assign(size_t(channels), Mat(rows, cols));
  for (Mat& p : f.planes)
    for (int c = 0; c < cols; ++c)
      for (int r = 0; r < rows; ++r) p(r, c) = rng.next();  // column-major draw order
  return f;
}

Mat random_mat(int rows, int cols, uint64_t seed, double lo, double hi) {  // support.hpp:31-39
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(lo, hi);
  Mat m(rows, cols);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) m(i, j) = dist(rng);
  return m;
}

// ------------------------------------------------------------ image / kernel
static bool all_finite(const Mat& m) {
  for (double x : m.v)
    if (!std::isfinite(x)) return false;
  return true;
}

void validate_kernel(const BlurKernel& k, double sum_tol) {  // kernel.cpp:7-17
  require(k.width >= 1 && k.width % 2 == 1, Errc::invalid_argument,
          "kernel width must be odd and >= 1");
  require(k.weights.r == k.width && k.weights.c == k.width, Errc::dim_mismatch,
          "kernel weights must be width x width");
  require(all_finite(k.weights), Errc::invalid_argument, "kernel weights must be finite");
  double mn = *std::min_element(k.weights.v.begin(), k.weights.v.end());
  require(mn >= 0.0, Errc::invalid_argument, "kernel weights must be nonnegative");
  double s = 0;
  for (double x : k.weights.v) s += x;
  require(std::abs(s - 1.0) <= sum_tol, Errc::invalid_argument, "kernel weights must sum to 1");
}

void validate_frame(const Frame& f) {  // image.cpp:30-39
  require(f.channels() == 1 || f.channels() == 3, Errc::dim_mismatch,
          "frame must have 1 or 3 planes");
  for (const auto& p : f.planes) {
    require(p.r == f.rows() && p.c == f.cols(), Errc::dim_mismatch,
            "frame planes disagree on dimensions");
    require(p.r >= 1 && p.c >= 1, Errc::dim_mismatch, "empty frame plane");
    require(all_finite(p), Errc::range_exceeded, "frame contains non-finite samples");
  }
}

Mat luma(const Frame& f) {  // image.cpp:41-45 (Rec.601)
  validate_frame(f);
  if (f.channels() == 1) return f.planes[0];
  Mat out(f.rows(), f.cols());
  for (size_t i = 0; i < out.size(); ++i)
    out.v[i] = 0.299 * f.planes[0].v[i] + 0.587 * f.planes[1].v[i] + 0.114 * f.planes[2].v[i];
  return out;
}

// ---------------------------------------------------------------- poly.cpp
static cplx coef(const CVec& v, long i) {  // poly.cpp:10-12
  return (i >= 0 && i < long(v.size())) ? v[size_t(i)] : cplx(0.0, 0.0);
}
static bool all_zero(const CVec& v) {  // poly.cpp:14
  for (const cplx& c : v)
    if (std::abs(c) != 0.0) return false;
  return true;
}
static void normalize_phase(CVec& x) {  // poly.cpp:18-23 (first max index, like Eigen)
  size_t imax = 0;
  double best = -1;
  for (size_t i = 0; i < x.size(); ++i) {
    double a = std::abs(x[i]);
    if (a > best) best = a, imax = i;
  }
  double a = std::abs(x[imax]);
  if (a > 0.0) {
    cplx rot = std::conj(x[imax]) / a;
    for (auto& c : x) c *= rot;
  }
}
static double norm2(const CVec& v) {
  double s = 0;
  for (const cplx& c : v) s += std::norm(c);
  return std::sqrt(s);
}

Mat conv2_full(const Mat& a, const Mat& b) {  // poly.cpp:27-38
  require(a.size() > 0 && b.size() > 0, Errc::dim_mismatch, "conv2_full needs nonempty inputs");
  const Mat& big = a.size() >= b.size() ? a : b;
  const Mat& small = a.size() >= b.size() ? b : a;
  Mat out(a.r + b.r - 1, a.c + b.c - 1, 0.0);
  for (int n = 0; n < small.c; ++n)
    for (int m = 0; m < small.r; ++m) {
      double w = small(m, n);
      if (w == 0.0) continue;
      for (int i = 0; i < big.r; ++i) {
        double* o = &out(m + i, n);
        const double* s = &big(i, 0);
        for (int j = 0; j < big.c; ++j) o[j] += w * s[j];
      }
    }
  return out;
}

CVec axis_dft_slice(const Mat& plane, Axis axis, cplx w) {  // poly.cpp:40-64 (one point)
  require(plane.size() > 0, Errc::invalid_argument, "axis_dft needs a nonempty plane");
  require(std::abs(std::abs(w) - 1.0) <= 1e-12, Errc::non_unit_sample_point,
          "sample point off the unit circle");
  const int d = axis == Axis::Z1 ? plane.r : plane.c;
  const double theta = std::arg(w);
  std::vector<double> pr(d), pi(d);
  for (int m = 0; m < d; ++m) {
    cplx pw = std::polar(1.0, theta * double(m));
    pr[m] = pw.real(), pi[m] = pw.imag();
  }
  if (axis == Axis::Z1) {
    CVec out(static_cast<size_t>(plane.c));
    for (int n = 0; n < plane.c; ++n) {
      double re = 0, im = 0;
      for (int m = 0; m < plane.r; ++m) re += plane(m, n) * pr[m], im += plane(m, n) * pi[m];
      out[n] = cplx(re, 0) + cplx(0, 1) * cplx(im, 0);
    }
    return out;
  }
  CVec out(static_cast<size_t>(plane.r));
  for (int m = 0; m < plane.r; ++m) {
    double re = 0, im = 0;
    for (int n = 0; n < plane.c; ++n) re += plane(m, n) * pr[n], im += plane(m, n) * pi[n];
    out[m] = cplx(re, 0) + cplx(0, 1) * cplx(im, 0);
  }
  return out;
}

CMat bezout_leading_block(const CVec& p, const CVec& q, int size) {  // poly.cpp:66-79
  require(size >= 1, Errc::invalid_argument, "bezout block size must be >= 1");
  require(!all_zero(p) && !all_zero(q), Errc::degenerate_input,
          "bezout of an all-zero polynomial");
  CMat b(size, size);
  for (int i = 0; i < size; ++i)
    for (int j = 0; j < size; ++j) {
      cplx s(0.0, 0.0);
      for (int k = 0; k <= std::min(i, j); ++k)
        s += coef(p, i + j + 1 - k) * coef(q, k) - coef(q, i + j + 1 - k) * coef(p, k);
      b(i, j) = s;
    }
  return b;
}

// --- SVD (replaces Eigen::JacobiSVD, poly.cpp:85,103,126): complex Householder
// QR preconditioning for tall inputs, then one-sided (Hestenes) Jacobi.
static CMat householder_r(const CMat& a) {
  const int m = a.r, n = a.c;
  CMat r = a;
  std::vector<cplx> v(static_cast<size_t>(m));
  for (int k = 0; k < n && k < m; ++k) {
    double xn = 0;
    for (int i = k; i < m; ++i) xn += std::norm(r(i, k));
    xn = std::sqrt(xn);
    if (xn == 0.0) continue;
    cplx x0 = r(k, k);
    cplx ph = std::abs(x0) > 0 ? x0 / std::abs(x0) : cplx(1, 0);
    cplx alpha = -ph * xn;
    for (int i = k; i < m; ++i) v[i] = r(i, k);
    v[k] -= alpha;
    double vn = 0;
    for (int i = k; i < m; ++i) vn += std::norm(v[i]);
    if (vn == 0.0) continue;
    for (int j = k; j < n; ++j) {
      cplx d(0, 0);
      for (int i = k; i < m; ++i) d += std::conj(v[i]) * r(i, j);
      d *= 2.0 / vn;
      for (int i = k; i < m; ++i) r(i, j) -= v[i] * d;
    }
  }
  CMat out(n, n, cplx(0, 0));
  for (int i = 0; i < std::min(m, n); ++i)
    for (int j = i; j < n; ++j) out(i, j) = r(i, j);
  return out;
}

void svd(const CMat& a, Vec& sv, CMat* vout) {
  const int m = a.r, n = a.c;
  CMat g;
  if (m > n) {
    g = householder_r(a);
  } else {
    g = CMat(n, n, cplx(0, 0));  // wide: zero-pad to square (implicit zero singular values)
    for (int i = 0; i < m; ++i)
      for (int j = 0; j < n; ++j) g(i, j) = a(i, j);
  }
  CMat v(n, n, cplx(0, 0));
  for (int i = 0; i < n; ++i) v(i, i) = 1.0;
  const double tol = 1e-15;
  for (int sweep = 0; sweep < 80; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double al = 0, be = 0;
        cplx ga(0, 0);
        for (int k = 0; k < n; ++k) {
          al += std::norm(g(k, p));
          be += std::norm(g(k, q));
          ga += std::conj(g(k, p)) * g(k, q);
        }
        double ag = std::abs(ga);
        if (ag == 0.0 || ag <= tol * std::sqrt(al * be)) continue;
        rotated = true;
        double zeta = (be - al) / (2.0 * ag);
        double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1.0 + zeta * zeta));
        double c = 1.0 / std::sqrt(1.0 + t * t), s = c * t;
        cplx e = std::conj(ga / ag);
        for (int k = 0; k < n; ++k) {
          cplx gp = g(k, p), gq = e * g(k, q);
          g(k, p) = c * gp - s * gq;
          g(k, q) = s * gp + c * gq;
          cplx vp = v(k, p), vq = e * v(k, q);
          v(k, p) = c * vp - s * vq;
          v(k, q) = s * vp + c * vq;
        }
      }
    if (!rotated) break;
  }
  std::vector<double> s(n);
  for (int j = 0; j < n; ++j) {
    double acc = 0;
    for (int k = 0; k < n; ++k) acc += std::norm(g(k, j));
    s[j] = std::sqrt(acc);
  }
  std::vector<int> order(n);
  for (int j = 0; j < n; ++j) order[j] = j;
  std::stable_sort(order.begin(), order.end(), [&](int x, int y) { return s[x] > s[y]; });
  sv.assign(n, 0.0);
  for (int j = 0; j < n; ++j) sv[j] = s[order[j]];
  if (vout) {
    *vout = CMat(n, n);
    for (int j = 0; j < n; ++j)
      for (int k = 0; k < n; ++k) (*vout)(k, j) = v(k, order[j]);
  }
}

SingularityResult numerical_singularity(const CMat& m, double tau) {  // poly.cpp:81-91
  require(m.r == m.c && m.r >= 1, Errc::invalid_argument,
          "singularity test needs a square matrix");
  require(tau > 0.0 && tau < 1.0, Errc::invalid_argument, "tau must lie in (0,1)");
  Vec sv;
  svd(m, sv, nullptr);
  double smax = sv[0];
  if (smax == 0.0) return {true, 0.0};
  double ratio = sv.back() / smax;
  return {ratio < tau, ratio};
}

CofactorSolution cofactor_null_solve(const CVec& p, const CVec& q, int t,
                                     double gap_threshold) {  // poly.cpp:93-121
  require(t >= 1, Errc::invalid_argument, "cofactor width must be >= 1");
  require(int(p.size()) >= t && int(q.size()) >= t, Errc::invalid_argument,
          "slice degree below cofactor degree");
  const int rows = int(std::max(p.size(), q.size())) + t - 1;
  CMat a(rows, 2 * t, cplx(0, 0));
  for (int j = 0; j < t; ++j) {
    for (size_t i = 0; i < p.size(); ++i) a(j + int(i), j) = p[i];       // p * k2
    for (size_t i = 0; i < q.size(); ++i) a(j + int(i), t + j) = -q[i];  // -q * k1
  }
  Vec sv;
  CMat v;
  svd(a, sv, &v);
  const int n = 2 * t;
  double smax = sv[0];
  // zero-padding makes the implicit zero singular values explicit (poly.cpp:106-109)
  double second_smallest = n >= 2 ? sv[n - 2] : 0.0;
  double gap = smax == 0.0 ? 0.0 : second_smallest / smax;
  if (gap < gap_threshold)
    fail(Errc::ill_conditioned,
         "cofactor null space not one-dimensional (gap " + std::to_string(gap) + ")");
  CVec x(n);
  for (int k = 0; k < n; ++k) x[k] = v(k, n - 1);
  normalize_phase(x);
  CofactorSolution sol;
  sol.k2.assign(x.begin(), x.begin() + t);
  sol.k1.assign(x.begin() + t, x.end());
  sol.gap = gap;
  return sol;
}

CVec homogeneous_lsq(const CMat& a) {  // poly.cpp:123-130
  require(a.r >= a.c && a.c >= 1, Errc::invalid_argument, "homogeneous system needs rows >= cols");
  Vec sv;
  CMat v;
  svd(a, sv, &v);
  CVec x(static_cast<size_t>(a.c));
  for (int k = 0; k < a.c; ++k) x[k] = v(k, a.c - 1);
  normalize_phase(x);
  return x;
}

CMat sylvester_matrix(const CVec& p, const CVec& q) {  // poly.cpp:132-141
  require(p.size() >= 1 && q.size() >= 1, Errc::invalid_argument, "empty polynomial");
  const int m = int(p.size()) - 1, n = int(q.size()) - 1;
  CMat s(m + n, m + n, cplx(0, 0));
  for (int r = 0; r < n; ++r)
    for (int k = 0; k <= m; ++k) s(r, r + k) = p[m - k];
  for (int r = 0; r < m; ++r)
    for (int k = 0; k <= n; ++k) s(n + r, r + k) = q[n - k];
  return s;
}

int numerical_degree(const CVec& p, double rel_tol) {  // poly.cpp:143-150
  if (p.empty()) return -1;
  double mx = 0;
  for (const cplx& c : p) mx = std::max(mx, std::abs(c));
  if (mx == 0.0) return -1;
  for (int i = int(p.size()) - 1; i >= 0; --i)
    if (std::abs(p[i]) > rel_tol * mx) return i;
  return -1;
}

// ----------------------------------------------------------------- fft.cpp
// Mixed-radix Stockham FFT (replaces FFTW, fft.cpp:23-109). Plans cached per
// thread: radix list and the n-point root table exp(-2*pi*i*k/n).
namespace {
struct FftPlan {
  int n = 0;
  std::vector<int> radices;
  std::vector<cplx> root;  // root[k] = exp(-2*pi*i*k/n)
};
const FftPlan& fft_plan(int n) {
  thread_local std::map<int, FftPlan> cache;
  auto it = cache.find(n);
  if (it != cache.end()) return it->second;
  FftPlan p;
  p.n = n;
  int r = n;
  for (int f : {4, 2, 3, 5, 7})
    while (r % f == 0) p.radices.push_back(f), r /= f;
  for (int f = 11; r > 1; f += 2)
    while (r % f == 0) p.radices.push_back(f), r /= f;
  p.root.resize(size_t(n));
  for (int k = 0; k < n; ++k) {
    double ang = -2.0 * std::numbers::pi * double(k) / double(n);
    p.root[k] = cplx(std::cos(ang), std::sin(ang));
  }
  return cache.emplace(n, std::move(p)).first->second;
}
}  // namespace

void fft1(cplx* x, int n, int sign) {
  if (n <= 1) return;
  const FftPlan& pl = fft_plan(n);
  thread_local std::vector<cplx> work;
  if (int(work.size()) < n) work.resize(size_t(n));
  cplx* in = x;
  cplx* out = work.data();
  int ns = 1;
  cplx v[64], y[64];
  std::vector<cplx> big_v, big_y;
  for (int r : pl.radices) {
    const int stride = n / r;
    cplx* vv = v;
    cplx* yy = y;
    if (r > 64) {
      big_v.resize(size_t(r)), big_y.resize(size_t(r));
      vv = big_v.data(), yy = big_y.data();
    }
    const int tw_step = n / (ns * r);
    for (int j = 0; j < stride; ++j) {
      const int k = j % ns;
      for (int i = 0; i < r; ++i) {
        cplx w = pl.root[size_t((long(i) * k * tw_step) % n)];
        if (sign > 0) w = std::conj(w);
        vv[i] = in[j + i * stride] * w;
      }
      if (r == 2) {
        yy[0] = vv[0] + vv[1], yy[1] = vv[0] - vv[1];
      } else if (r == 4) {
        cplx a = vv[0] + vv[2], b = vv[0] - vv[2], c = vv[1] + vv[3], d = vv[1] - vv[3];
        cplx jd = sign < 0 ? cplx(d.imag(), -d.real()) : cplx(-d.imag(), d.real());
        yy[0] = a + c, yy[2] = a - c, yy[1] = b + jd, yy[3] = b - jd;
      } else {
        const int rstep = n / r;
        for (int o = 0; o < r; ++o) {
          cplx acc = vv[0];
          for (int i = 1; i < r; ++i) {
            cplx w = pl.root[size_t((long(o) * i % r) * rstep)];
            if (sign > 0) w = std::conj(w);
            acc += vv[i] * w;
          }
          yy[o] = acc;
        }
      }
      const int base = (j / ns) * ns * r + k;
      for (int i = 0; i < r; ++i) out[base + i * ns] = yy[i];
    }
    std::swap(in, out);
    ns *= r;
  }
  if (in != x) std::copy(in, in + n, x);
}

// Real forward transform of length n: out[0..n/2]. Half-length complex trick for even n.
static void rfft(const double* x, int n, cplx* out) {
  thread_local std::vector<cplx> z;
  if (n % 2 == 0 && n >= 2) {
    const int h = n / 2;
    z.resize(size_t(h));
    for (int i = 0; i < h; ++i) z[i] = cplx(x[2 * i], x[2 * i + 1]);
    fft1(z.data(), h, -1);
    const FftPlan& pl = fft_plan(n);
    for (int k = 0; k <= h; ++k) {
      cplx zk = z[k % h], zc = std::conj(z[(h - k) % h]);
      cplx e = 0.5 * (zk + zc), o = cplx(0, -0.5) * (zk - zc);
      out[k] = e + pl.root[size_t(k)] * o;
    }
    return;
  }
  z.resize(size_t(n));
  for (int i = 0; i < n; ++i) z[i] = cplx(x[i], 0);
  fft1(z.data(), n, -1);
  for (int k = 0; k <= n / 2; ++k) out[k] = z[k];
}

// Inverse of rfft (unnormalized): real out[0..n-1] from X[0..n/2].
static void irfft(const cplx* X, int n, double* out) {
  thread_local std::vector<cplx> z;
  if (n % 2 == 0 && n >= 2) {
    const int h = n / 2;
    z.resize(size_t(h));
    const FftPlan& pl = fft_plan(n);
    for (int k = 0; k < h; ++k) {
      cplx a = X[k], b = std::conj(X[h - k]);
      cplx e = a + b, o = (a - b) * std::conj(pl.root[size_t(k)]);
      z[k] = e + cplx(0, 1) * o;
    }
    fft1(z.data(), h, +1);
    for (int i = 0; i < h; ++i) out[2 * i] = z[i].real(), out[2 * i + 1] = z[i].imag();
    return;
  }
  z.resize(size_t(n));
  for (int k = 0; k <= n / 2; ++k) z[k] = X[k];
  for (int k = n / 2 + 1; k < n; ++k) z[k] = std::conj(X[n - k]);
  fft1(z.data(), n, +1);
  for (int i = 0; i < n; ++i) out[i] = z[i].real();
}

static void fft2_inplace(CMat& y, int sign) {
  const int M = y.r, N = y.c;
  for (int m = 0; m < M; ++m) fft1(&y(m, 0), N, sign);
  std::vector<cplx> col(static_cast<size_t>(M));
  for (int n = 0; n < N; ++n) {
    for (int m = 0; m < M; ++m) col[m] = y(m, n);
    fft1(col.data(), M, sign);
    for (int m = 0; m < M; ++m) y(m, n) = col[m];
  }
}

CMat fft2(const CMat& x) {  // fft.cpp:177 (unnormalized forward)
  require(x.r >= 1 && x.c >= 1, Errc::invalid_argument, "fft2 needs a nonempty array");
  CMat y = x;
  fft2_inplace(y, -1);
  return y;
}

CMat ifft2(const CMat& x) {  // fft.cpp:191-195 (1/(M*N))
  require(x.r >= 1 && x.c >= 1, Errc::invalid_argument, "fft2 needs a nonempty array");
  CMat y = x;
  fft2_inplace(y, +1);
  const double s = 1.0 / (double(x.r) * double(x.c));
  for (auto& c : y.v) c *= s;
  return y;
}

static CMat dft_matrix(int t) {  // decoder.cpp:125-131 and fft.cpp:203-204
  constexpr double tau = 2.0 * std::numbers::pi;
  CMat w(t, t);
  for (int i = 0; i < t; ++i)
    for (int j = 0; j < t; ++j) w(i, j) = std::polar(1.0, -tau * double((i * j) % t) / double(t));
  return w;
}

CMat axis_roots_dft(const Mat& plane, Axis axis, int t) {  // fft.cpp:197-213
  const int M = plane.r, N = plane.c;
  require(M >= 1 && N >= 1, Errc::invalid_argument, "axis_roots_dft needs a nonempty plane");
  require(t >= 1, Errc::invalid_argument, "axis_roots_dft needs t >= 1");
  CMat w = dft_matrix(t);
  if (axis == Axis::Z1) {
    Mat fold(t, N, 0.0);
    for (int m = 0; m < M; ++m)
      for (int n = 0; n < N; ++n) fold(m % t, n) += plane(m, n);
    CMat out(t, N, cplx(0, 0));
    for (int i = 0; i < t; ++i)
      for (int n = 0; n < N; ++n) {
        cplx acc(0, 0);
        for (int r = 0; r < t; ++r) acc += w(i, r) * fold(r, n);
        out(i, n) = acc;
      }
    return out;
  }
  Mat fold(M, t, 0.0);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) fold(m, n % t) += plane(m, n);
  CMat out(M, t, cplx(0, 0));
  for (int m = 0; m < M; ++m)
    for (int i = 0; i < t; ++i) {
      cplx acc(0, 0);
      for (int r = 0; r < t; ++r) acc += fold(m, r) * w(r, i);
      out(m, i) = acc;
    }
  return out;
}

CMat axis_spectrum_half(const Mat& plane, Axis axis) {  // fft.cpp:217-240
  const int M = plane.r, N = plane.c;
  require(M >= 1 && N >= 1, Errc::invalid_argument, "axis_spectrum_half needs a nonempty plane");
  if (axis == Axis::Z1) {
    const int half = M / 2 + 1;
    CMat y(half, N);
    std::vector<double> col(static_cast<size_t>(M));
    std::vector<cplx> sp(static_cast<size_t>(half));
    for (int n = 0; n < N; ++n) {
      for (int m = 0; m < M; ++m) col[m] = plane(m, n);
      rfft(col.data(), M, sp.data());
      for (int i = 0; i < half; ++i) y(i, n) = sp[i];
    }
    return y;
  }
  const int half = N / 2 + 1;
  CMat y(M, half);
  for (int m = 0; m < M; ++m) rfft(&plane(m, 0), N, &y(m, 0));
  return y;
}

int friendly_size(int n) {  // fft.cpp:272-280
  require(n >= 1, Errc::invalid_argument, "extent must be positive");
  for (int m = n;; ++m) {
    int r = m;
    for (int f : {2, 3, 5, 7})
      while (r % f == 0) r /= f;
    if (r == 1) return m;
  }
}

// ------------------------------------------------------------- encoder.cpp
static double restriction_margin(const CVec& p, const CVec& q) {  // encoder.cpp:16-24
  int dp = numerical_degree(p), dq = numerical_degree(q);
  if (dp < 0 || dq < 0) return 0.0;
  if (dp == 0 && dq == 0) return 1.0;
  CMat s = sylvester_matrix(CVec(p.begin(), p.begin() + dp + 1), CVec(q.begin(), q.begin() + dq + 1));
  Vec sv;
  svd(s, sv, nullptr);
  return sv[0] == 0.0 ? 0.0 : sv.back() / sv[0];
}

static BlurKernel draw_kernel(int width, UniformRng& rng) {  // encoder.cpp:26-34
  Mat w(width, width);
  for (int n = 0; n < width; ++n)
    for (int m = 0; m < width; ++m) w(m, n) = rng.next();
  double s = 0;
  for (int n = 0; n < width; ++n)  // column-major summation order
    for (int m = 0; m < width; ++m) s += w(m, n);
  require(s > 0.0, Errc::degenerate_input, "drew an all-zero kernel");
  for (double& x : w.v) x /= s;
  return BlurKernel{width, w};
}

double coprimality_check(const BlurKernel& k1, const BlurKernel& k2, int trials) {  // 45-64
  validate_kernel(k1);
  validate_kernel(k2);
  require(k1.width == k2.width, Errc::dim_mismatch, "kernel widths differ");
  require(trials >= 1, Errc::invalid_argument, "trials must be >= 1");
  UniformRng rng(0x5ca1ab1e0ddba11ull);
  constexpr double tau = 2.0 * std::numbers::pi;
  double margin = 1.0;
  for (int trial = 0; trial < trials; ++trial) {
    cplx w = std::polar(1.0, tau * rng.next());
    for (Axis axis : {Axis::Z1, Axis::Z2}) {
      CVec p = axis_dft_slice(k1.weights, axis, w);
      CVec q = axis_dft_slice(k2.weights, axis, w);
      margin = std::min(margin, restriction_margin(p, q));
    }
  }
  return margin;
}

CoprimePair generate_coprime_pair(int width, uint64_t seed, int max_retries,
                                  double margin_threshold, int trials) {  // encoder.cpp:66-81
  require(width >= 3 && width <= 63 && width % 2 == 1, Errc::invalid_argument,
          "kernel width must be odd, within [3,63]");
  require(max_retries >= 1, Errc::invalid_argument, "max_retries must be >= 1");
  require(margin_threshold > 0.0, Errc::invalid_argument, "margin threshold must be positive");
  UniformRng rng(seed);
  for (int attempt = 0; attempt < max_retries; ++attempt) {
    BlurKernel k1 = draw_kernel(width, rng);
    BlurKernel k2 = draw_kernel(width, rng);
    double margin = coprimality_check(k1, k2, trials);
    if (margin > margin_threshold) return CoprimePair{k1, k2, margin, seed};
  }
  fail(Errc::coprimality_failure, "no coprime pair of width " + std::to_string(width) +
                                      " within " + std::to_string(max_retries) + " draws");
}

BlurredPair encode_frame(const Frame& latent, const CoprimePair& pair) {  // encoder.cpp:83-103
  validate_frame(latent);
  validate_kernel(pair.k1);
  validate_kernel(pair.k2);
  require(pair.k1.width == pair.k2.width, Errc::dim_mismatch, "kernel widths differ");
  const int t = pair.k1.width;
  require(latent.rows() >= t && latent.cols() >= t, Errc::frame_too_small,
          "latent frame smaller than the blur kernel");
  BlurredPair out;
  out.public_frame.index = out.private_frame.index = latent.index;
  for (const auto& plane : latent.planes) {
    out.public_frame.planes.push_back(conv2_full(plane, pair.k1.weights));
    out.private_frame.planes.push_back(conv2_full(plane, pair.k2.weights));
  }
  out.kernel_width_hint = t;
  return out;
}

Frame quantize_frame(const Frame& f, int bits) {  // encoder.cpp:105-120
  validate_frame(f);
  require(bits == 8 || bits == 16, Errc::invalid_argument, "quantization depth must be u8 or u16");
  const double maxv = double((1u << bits) - 1);
  Frame out = f;
  out.bit_depth = bits;
  for (auto& plane : out.planes) {
    double mn = *std::min_element(plane.v.begin(), plane.v.end());
    double mx = *std::max_element(plane.v.begin(), plane.v.end());
    require(mn >= -1e-9 && mx <= 1.0 + 1e-9, Errc::range_exceeded, "samples outside [0,1]");
    for (double& x : plane.v) {
      double c = std::min(1.0, std::max(0.0, x));
      x = std::round(c * maxv) / maxv;
    }
  }
  return out;
}

Frame degrade_bits(const Frame& f, int drop) {  // encoder.cpp:124-139
  validate_frame(f);
  require(f.bit_depth != 0, Errc::not_quantized, "bit-precision degradation needs a quantized frame");
  const int bits = f.bit_depth;
  require(drop >= 0 && drop < bits, Errc::invalid_argument, "drop must lie in [0, bit width)");
  if (drop == 0) return f;
  const double maxv = double((1u << bits) - 1);
  const std::uint32_t mask = ~((1u << drop) - 1u);
  Frame out = f;
  for (auto& plane : out.planes)
    for (double& x : plane.v) {
      const auto k = static_cast<std::uint32_t>(std::lround(x * maxv));
      x = double(k & mask) / maxv;
    }
  return out;
}

// ------------------------------------------------------------- decoder.cpp
namespace {
using Clock = std::chrono::steady_clock;
double ms_since(Clock::time_point t0) {
  return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

void check_pair(const BlurredPair& pair) {  // decoder.cpp:19-29
  validate_frame(pair.public_frame);
  validate_frame(pair.private_frame);
  require(pair.public_frame.rows() == pair.private_frame.rows() &&
              pair.public_frame.cols() == pair.private_frame.cols() &&
              pair.public_frame.channels() == pair.private_frame.channels(),
          Errc::dim_mismatch, "pair frames disagree on dimensions");
  if (pair.kernel_width_hint)
    require(*pair.kernel_width_hint >= 1 && *pair.kernel_width_hint % 2 == 1,
            Errc::invalid_argument, "kernel width hint must be odd and >= 1");
}

void check_search(int smin, int smax) {  // decoder.cpp:31-34
  require(smin >= 3 && smax <= 63 && smin <= smax && smin % 2 == 1 && smax % 2 == 1,
          Errc::invalid_argument, "width search range must be odd values within [3,63]");
}

WidthEstimate width_from_slices(const CVec& p, const CVec& q, int smin, int smax,
                                double tau) {  // decoder.cpp:38-44
  for (int s = smin; s <= smax; s += 2) {
    CMat block = bezout_leading_block(p, q, s);
    if (numerical_singularity(block, tau).singular) return {s, false};
  }
  return {smax, true};
}

WidthEstimate estimate_from_lumas(const Mat& l1, const Mat& l2, int smin, int smax,
                                  double tau) {  // decoder.cpp:46-90
  require(std::min(l1.r, l1.c) > smax, Errc::frame_too_small,
          "frame too small for the width search bound");
  double mn1 = *std::min_element(l1.v.begin(), l1.v.end());
  double mn2 = *std::min_element(l2.v.begin(), l2.v.end());
  const bool nonneg = mn1 >= 0.0 && mn2 >= 0.0;
  WidthEstimate est[2];
  for (Axis axis : {Axis::Z1, Axis::Z2}) {
    const int idx = axis == Axis::Z1 ? 0 : 1;
    CVec p, q;
    if (nonneg) {
      if (axis == Axis::Z1) {  // column sums, length N
        p.assign(size_t(l1.c), 0.0), q.assign(size_t(l1.c), 0.0);
        for (int m = 0; m < l1.r; ++m)
          for (int n = 0; n < l1.c; ++n) p[n] += l1(m, n), q[n] += l2(m, n);
      } else {  // row sums, length M
        p.assign(size_t(l1.r), 0.0), q.assign(size_t(l1.r), 0.0);
        for (int m = 0; m < l1.r; ++m) {
          double a = 0, b = 0;
          for (int n = 0; n < l1.c; ++n) a += l1(m, n), b += l2(m, n);
          p[m] = a, q[m] = b;
        }
      }
    } else {  // signed content: maximum joint energy slice (decoder.cpp:65-82)
      CMat s1 = axis_spectrum_half(l1, axis), s2 = axis_spectrum_half(l2, axis);
      int pick = 0;
      double best = -1;
      if (axis == Axis::Z1) {
        for (int i = 0; i < s1.r; ++i) {
          double e = 0;
          for (int n = 0; n < s1.c; ++n) e += std::norm(s1(i, n)) + std::norm(s2(i, n));
          if (e > best) best = e, pick = i;
        }
        p.resize(size_t(s1.c)), q.resize(size_t(s1.c));
        for (int n = 0; n < s1.c; ++n) p[n] = s1(pick, n), q[n] = s2(pick, n);
      } else {
        for (int j = 0; j < s1.c; ++j) {
          double e = 0;
          for (int m = 0; m < s1.r; ++m) e += std::norm(s1(m, j)) + std::norm(s2(m, j));
          if (e > best) best = e, pick = j;
        }
        p.resize(size_t(s1.r)), q.resize(size_t(s1.r));
        for (int m = 0; m < s1.r; ++m) p[m] = s1(m, pick), q[m] = s2(m, pick);
      }
    }
    est[idx] = width_from_slices(p, q, smin, smax, tau);
  }
  if (est[0].width != est[1].width)
    fail(Errc::inconsistent_axes, "width estimates disagree: z1 gives " +
                                      std::to_string(est[0].width) + ", z2 gives " +
                                      std::to_string(est[1].width));
  return {est[0].width, est[0].clamped && est[1].clamped};
}

ScaledKernelTransform solve_axis(const CMat& s1, const CMat& s2, int t, Axis axis,
                                 double gap_threshold) {  // decoder.cpp:94-123
  ScaledKernelTransform out;
  out.axis = axis;
  out.values = CMat(t, t);
  out.gaps.assign(size_t(t), 0.0);
  for (int i = 0; i < t; ++i) {
    CVec p, q;
    if (axis == Axis::Z1) {
      p.resize(size_t(s1.c)), q.resize(size_t(s1.c));
      for (int n = 0; n < s1.c; ++n) p[n] = s1(i, n), q[n] = s2(i, n);
    } else {
      p.resize(size_t(s1.r)), q.resize(size_t(s1.r));
      for (int m = 0; m < s1.r; ++m) p[m] = s1(m, i), q[m] = s2(m, i);
    }
    CofactorSolution sol;
    try {
      sol = cofactor_null_solve(p, q, t, gap_threshold);
    } catch (const Error& e) {
      if (e.code() != Errc::ill_conditioned) throw;
      fail(Errc::ill_conditioned_slice,
           std::string(axis_name(axis)) + " slice " + std::to_string(i) + ": " + e.what());
    }
    double norm = norm2(sol.k1);
    if (norm == 0.0)
      fail(Errc::ill_conditioned_slice, std::string(axis_name(axis)) + " slice " +
                                            std::to_string(i) + ": vanishing cofactor estimate");
    for (int k = 0; k < t; ++k) {
      cplx v = sol.k1[k] / norm;
      if (axis == Axis::Z1)
        out.values(i, k) = v;
      else
        out.values(k, i) = v;
    }
    out.gaps[i] = sol.gap;
  }
  return out;
}

Mat realize_kernel(CMat k, double max_imag_energy, double negative_weight_tol) {  // 159-176
  cplx mass(0, 0);
  for (const cplx& c : k.v) mass += c;
  require(std::abs(mass) > 0.0, Errc::non_real_kernel, "kernel estimate has vanishing mass");
  cplx rot = std::conj(mass) / std::abs(mass);
  for (cplx& c : k.v) c *= rot;
  double total = 0, imag = 0;
  for (const cplx& c : k.v) total += std::norm(c), imag += c.imag() * c.imag();
  require(total > 0.0, Errc::non_real_kernel, "kernel estimate is zero");
  if (imag > max_imag_energy * total)
    fail(Errc::non_real_kernel, "imaginary energy fraction " + std::to_string(imag / total));
  Mat w(k.r, k.c);
  for (size_t i = 0; i < w.size(); ++i) w.v[i] = k.v[i].real();
  double mx = *std::max_element(w.v.begin(), w.v.end());
  double mn = *std::min_element(w.v.begin(), w.v.end());
  require(mx > 0.0, Errc::non_real_kernel, "kernel estimate has no positive weight");
  if (mn < -negative_weight_tol * mx)
    fail(Errc::non_real_kernel,
         "negative weight beyond tolerance (min " + std::to_string(mn / mx) + " of max)");
  double s = 0;
  for (double& x : w.v) x = std::max(x, 0.0), s += x;
  for (double& x : w.v) x /= s;
  return w;
}

struct DeblurPlan {  // decoder.cpp:178-182
  int work_rows = 0, work_cols = 0;
  CMat kernel_half;  // work_rows x (work_cols/2+1): row-major grid halves the column axis
  double epsilon = 0.0;
};

// 2-D real forward transform of a zero-padded array; only rows < nz_rows are nonzero.
CMat fft2_real_half(const Mat& src, int G_r, int G_c) {
  const int H = G_c / 2 + 1;
  CMat y(G_r, H, cplx(0, 0));
  std::vector<double> row(size_t(G_c), 0.0);
  for (int m = 0; m < src.r; ++m) {
    std::fill(row.begin(), row.end(), 0.0);
    for (int n = 0; n < src.c; ++n) row[n] = src(m, n);
    rfft(row.data(), G_c, &y(m, 0));
  }
  std::vector<cplx> col(static_cast<size_t>(G_r));
  for (int v = 0; v < H; ++v) {
    for (int u = 0; u < G_r; ++u) col[u] = y(u, v);
    fft1(col.data(), G_r, -1);
    for (int u = 0; u < G_r; ++u) y(u, v) = col[u];
  }
  return y;
}

DeblurPlan make_deblur_plan(int rows, int cols, const BlurKernel& k,
                            std::optional<double> epsilon) {  // decoder.cpp:187-202
  const int t = k.width;
  require(rows >= t && cols >= t, Errc::frame_too_small, "blurred frame smaller than the kernel");
  DeblurPlan plan;
  plan.work_rows = friendly_size(rows);
  plan.work_cols = friendly_size(cols);
  plan.kernel_half = fft2_real_half(k.weights, plan.work_rows, plan.work_cols);
  double peak = 0;
  for (const cplx& c : plan.kernel_half.v) peak = std::max(peak, std::abs(c));
  plan.epsilon = epsilon.value_or(1e-8 * peak * peak);
  require(plan.epsilon >= 0.0, Errc::invalid_argument, "epsilon must be nonnegative");
  return plan;
}

Mat run_deblur(const Mat& blurred, const DeblurPlan& plan, int t) {  // decoder.cpp:204-214
  const int G_r = plan.work_rows, G_c = plan.work_cols, H = G_c / 2 + 1;
  const int out_r = blurred.r - t + 1, out_c = blurred.c - t + 1;
  CMat fb = fft2_real_half(blurred, G_r, G_c);
  std::vector<cplx> col(static_cast<size_t>(G_r));
  for (int v = 0; v < H; ++v) {
    for (int u = 0; u < G_r; ++u) {
      cplx fk = plan.kernel_half(u, v);
      col[u] = fb(u, v) * std::conj(fk) / (std::norm(fk) + plan.epsilon);
    }
    fft1(col.data(), G_r, +1);
    for (int u = 0; u < out_r; ++u) fb(u, v) = col[u];
  }
  Mat out(out_r, out_c);
  std::vector<double> row(static_cast<size_t>(G_c));
  const double scale = 1.0 / (double(G_r) * double(G_c));  // fft.cpp:268
  for (int m = 0; m < out_r; ++m) {
    irfft(&fb(m, 0), G_c, row.data());
    for (int n = 0; n < out_c; ++n) out(m, n) = row[n] * scale;
  }
  return out;
}
}  // namespace

WidthEstimate estimate_kernel_width(const BlurredPair& pair, int search_min, int search_max,
                                    double tau) {  // decoder.cpp:218-225
  check_pair(pair);
  check_search(search_min, search_max);
  require(tau > 0.0 && tau < 1.0, Errc::invalid_argument, "tau must lie in (0,1)");
  return estimate_from_lumas(luma(pair.public_frame), luma(pair.private_frame), search_min,
                             search_max, tau);
}

ScaledKernelTransform sample_cofactors(const BlurredPair& pair, int width, Axis axis,
                                       double gap_threshold) {  // decoder.cpp:227-238
  check_pair(pair);
  require(width >= 1 && width % 2 == 1, Errc::invalid_argument, "width must be odd and >= 1");
  Mat l1 = luma(pair.public_frame), l2 = luma(pair.private_frame);
  require(l1.r >= width && l1.c >= width, Errc::frame_too_small,
          "frame smaller than the kernel width");
  CMat s1 = axis_roots_dft(l1, axis, width), s2 = axis_roots_dft(l2, axis, width);
  return solve_axis(s1, s2, width, axis, gap_threshold);
}

CMat complete_to_spectrum(const ScaledKernelTransform& skt) {  // decoder.cpp:240-246
  const int t = skt.values.r;
  require(skt.values.c == t && t >= 1, Errc::dim_mismatch, "scaled kernel transform must be square");
  CMat w = dft_matrix(t);
  CMat out(t, t, cplx(0, 0));
  for (int i = 0; i < t; ++i)
    for (int j = 0; j < t; ++j) {
      cplx acc(0, 0);
      for (int k = 0; k < t; ++k)
        acc += skt.axis == Axis::Z1 ? skt.values(i, k) * w(k, j) : w(i, k) * skt.values(k, j);
      out(i, j) = acc;
    }
  return out;
}

ScaleResolution resolve_completed(const CMat& a_spec, const CMat& b_spec) {  // 133-155
  const int t = a_spec.r;
  require(a_spec.c == t && b_spec.r == t && b_spec.c == t, Errc::dim_mismatch,
          "spectrum estimates must be square and equal-sized");
  CMat sys(t * t, 2 * t, cplx(0, 0));
  for (int i = 0; i < t; ++i)
    for (int j = 0; j < t; ++j) {
      int r = i * t + j;
      sys(r, i) = -b_spec(i, j);
      sys(r, t + j) = a_spec(i, j);
    }
  CVec x = homogeneous_lsq(sys);
  ScaleResolution out;
  out.lambda.assign(x.begin(), x.begin() + t);
  out.mu.assign(x.begin() + t, x.end());
  double rr = 0;
  for (int r = 0; r < t * t; ++r) {
    cplx acc(0, 0);
    for (int c = 0; c < 2 * t; ++c) acc += sys(r, c) * x[c];
    rr += std::norm(acc);
  }
  out.residual = std::sqrt(rr);
  double mx = 0, mn = 1e300;
  for (const cplx& c : x) mx = std::max(mx, std::abs(c)), mn = std::min(mn, std::abs(c));
  if (mx == 0.0 || mn < 1e-10 * mx)
    fail(Errc::degenerate_scales, "near-zero per-slice scale (ratio " +
                                      std::to_string(mx == 0.0 ? 0.0 : mn / mx) + ")");
  return out;
}

ScaleResolution resolve_scales(const ScaledKernelTransform& a,
                               const ScaledKernelTransform& b) {  // decoder.cpp:248-254
  require(a.axis == Axis::Z1 && b.axis == Axis::Z2, Errc::invalid_argument,
          "resolve_scales expects a z1 transform and a z2 transform");
  require(a.values.r == b.values.r && a.values.c == b.values.c, Errc::dim_mismatch,
          "transforms disagree on size");
  return resolve_completed(complete_to_spectrum(a), complete_to_spectrum(b));
}

BlurKernel assemble_kernel(const CMat& a_spectrum, const CMat& b_spectrum,
                           const ScaleResolution& scales, double max_imag_energy,
                           double negative_weight_tol) {  // decoder.cpp:256-271
  const int t = a_spectrum.r;
  require(a_spectrum.c == t && b_spectrum.r == t && b_spectrum.c == t, Errc::dim_mismatch,
          "spectrum estimates must be square and equal-sized");
  require(int(scales.lambda.size()) == t && int(scales.mu.size()) == t, Errc::dim_mismatch,
          "scale vectors must match the kernel width");
  double mnl = 1e300, mnm = 1e300;
  for (const cplx& c : scales.lambda) mnl = std::min(mnl, std::abs(c));
  for (const cplx& c : scales.mu) mnm = std::min(mnm, std::abs(c));
  require(mnl > 0.0 && mnm > 0.0, Errc::degenerate_scales, "zero scale entry");
  CMat ka(t, t), kb(t, t);
  for (int i = 0; i < t; ++i)
    for (int j = 0; j < t; ++j) {
      ka(i, j) = (1.0 / scales.lambda[i]) * a_spectrum(i, j);
      kb(i, j) = b_spectrum(i, j) * (1.0 / scales.mu[j]);
    }
  Mat wa = realize_kernel(ifft2(ka), max_imag_energy, negative_weight_tol);
  Mat wb = realize_kernel(ifft2(kb), max_imag_energy, negative_weight_tol);
  BlurKernel k{t, Mat(t, t)};
  for (size_t i = 0; i < k.weights.size(); ++i) k.weights.v[i] = 0.5 * (wa.v[i] + wb.v[i]);
  return k;
}

Mat spectral_deblur(const Mat& blurred, const BlurKernel& k1, double epsilon) {  // 273-278
  validate_kernel(k1);
  require(epsilon >= 0.0, Errc::invalid_argument, "epsilon must be nonnegative");
  DeblurPlan plan = make_deblur_plan(blurred.r, blurred.c, k1, epsilon);
  return run_deblur(blurred, plan, k1.width);
}

DecodedFrame decode_frame(const BlurredPair& pair, const DecodeConfig& cfg) {  // 280-378
  check_pair(pair);
  check_search(cfg.search_min, cfg.search_max);
  require(cfg.tau > 0.0 && cfg.tau < 1.0, Errc::invalid_argument, "tau must lie in (0,1)");
  StageTimings tm;
  const auto t_begin = Clock::now();
  auto t0 = Clock::now();
  Mat l1, l2;
  try {
    l1 = luma(pair.public_frame);
    l2 = luma(pair.private_frame);
  } catch (const Error& e) {
    throw Error(e.code(), std::string("polynomial_evaluation: ") + e.what());
  }
  tm.polynomial_evaluation_ms += ms_since(t0);

  t0 = Clock::now();
  WidthEstimate est;
  if (cfg.trust_hint && pair.kernel_width_hint) {
    est.width = *pair.kernel_width_hint;
    est.clamped = false;
    require(est.width >= 1 && est.width % 2 == 1 && est.width <= 63, Errc::invalid_argument,
            "kernel width hint must be odd, within [1,63]");
  } else {
    try {
      est = estimate_from_lumas(l1, l2, cfg.search_min, cfg.search_max, cfg.tau);
    } catch (const Error& e) {
      throw Error(e.code(), std::string("kernel_degree_estimation: ") + e.what());
    }
  }
  const int t = est.width;
  tm.kernel_degree_estimation_ms += ms_since(t0);

  t0 = Clock::now();
  CMat s1z1, s2z1, s1z2, s2z2;
  try {
    require(l1.r >= t && l1.c >= t, Errc::frame_too_small, "frame smaller than the kernel width");
    s1z1 = axis_roots_dft(l1, Axis::Z1, t);
    s2z1 = axis_roots_dft(l2, Axis::Z1, t);
    s1z2 = axis_roots_dft(l1, Axis::Z2, t);
    s2z2 = axis_roots_dft(l2, Axis::Z2, t);
  } catch (const Error& e) {
    throw Error(e.code(), std::string("polynomial_evaluation: ") + e.what());
  }
  tm.polynomial_evaluation_ms += ms_since(t0);

  t0 = Clock::now();
  ScaledKernelTransform a, b;
  try {
    a = solve_axis(s1z1, s2z1, t, Axis::Z1, cfg.gap_threshold);
    b = solve_axis(s1z2, s2z2, t, Axis::Z2, cfg.gap_threshold);
  } catch (const Error& e) {
    throw Error(e.code(), std::string("kernel_estimation_1d: ") + e.what());
  }
  tm.kernel_estimation_1d_ms += ms_since(t0);

  t0 = Clock::now();
  DecodedFrame out;
  try {
    CMat a_spec = complete_to_spectrum(a);
    CMat b_spec = complete_to_spectrum(b);
    ScaleResolution scales = resolve_completed(a_spec, b_spec);
    out.kernel_estimate =
        assemble_kernel(a_spec, b_spec, scales, cfg.max_imag_energy, cfg.negative_weight_tol);
    DeblurPlan plan = make_deblur_plan(l1.r, l1.c, out.kernel_estimate, cfg.epsilon);
    out.epsilon_used = plan.epsilon;
    for (const auto& plane : pair.public_frame.planes)
      out.latent.planes.push_back(run_deblur(plane, plan, t));
    out.latent.index = pair.public_frame.index;
  } catch (const Error& e) {
    throw Error(e.code(), std::string("kernel_estimation_2d_fft: ") + e.what());
  }
  tm.kernel_estimation_2d_fft_ms += ms_since(t0);
  tm.total_ms = ms_since(t_begin);
  out.width_used = t;
  out.width_clamped = est.clamped;
  out.stage_timings = tm;
  if (cfg.validate) {  // decoder.cpp:367-376
    double num = 0.0, den = 0.0;
    for (size_t c = 0; c < pair.public_frame.planes.size(); ++c) {
      Mat reblur = conv2_full(out.latent.planes[c], out.kernel_estimate.weights);
      const Mat& pub = pair.public_frame.planes[c];
      for (size_t i = 0; i < reblur.size(); ++i) {
        double d = reblur.v[i] - pub.v[i];
        num += d * d;
        den += pub.v[i] * pub.v[i];
      }
    }
    require(den > 0.0, Errc::degenerate_input, "public frame is identically zero");
    out.validation_residual = std::sqrt(num / den);
  }
  return out;
}

double validate_pair(const BlurredPair& pair, const BlurKernel& k1_hat,
                     const BlurKernel& k2_hat) {  // decoder.cpp:380-395
  check_pair(pair);
  validate_kernel(k1_hat);
  validate_kernel(k2_hat);
  require(k1_hat.width == k2_hat.width, Errc::dim_mismatch, "kernel widths differ");
  double num = 0.0, den = 0.0;
  for (size_t c = 0; c < pair.public_frame.planes.size(); ++c) {
    Mat lhs = conv2_full(pair.public_frame.planes[c], k2_hat.weights);
    Mat rhs = conv2_full(pair.private_frame.planes[c], k1_hat.weights);
    for (size_t i = 0; i < lhs.size(); ++i) {
      double d = lhs.v[i] - rhs.v[i];
      num += d * d;
      den += lhs.v[i] * lhs.v[i];
    }
  }
  require(den > 0.0, Errc::degenerate_input, "cross-convolution is identically zero");
  return std::sqrt(num / den);
}

double psnr(const Mat& reference, const Mat& test) {  // metrics.cpp:11-25
  require(reference.r == test.r && reference.c == test.c, Errc::dim_mismatch,
          "psnr operands differ in shape");
  require(reference.size() > 0, Errc::invalid_argument, "psnr of empty image");
  double sq = 0;
  for (size_t i = 0; i < reference.size(); ++i) {
    double d = reference.v[i] - test.v[i];
    sq += d * d;
  }
  if (sq == 0.0) return std::numeric_limits<double>::infinity();
  return 10.0 * std::log10(double(reference.size()) / sq);
}

}  // namespace orc
