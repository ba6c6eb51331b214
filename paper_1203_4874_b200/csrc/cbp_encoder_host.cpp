// CBP generation inputs on the host: the seeded kernel-pair draw with its coprimality
// check (reference encoder.cpp:16-81) and the deterministic synthetic frames
// (synth.cpp:12-22, rng.hpp:8-29). Untimed input generation, API-kept by the north
// star; the blur itself (encode_frame) runs on the device (cbp_encode_frames).
#include <algorithm>
#include <cmath>
#include <complex>
#include <cstring>
#include <random>
#include <string>
#include <vector>

#include "../../include/cbp_cuda.h"

namespace {

using cplx = std::complex<double>;

uint64_t splitmix64(uint64_t x) {
  x += 0x9E3779B97F4A7C15ull;
  x = (x ^ (x >> 30)) * 0xBF58476D1CE4E5B9ull;
  x = (x ^ (x >> 27)) * 0x94D049BB133111EBull;
  return x ^ (x >> 31);
}

// mt19937_64 with the reference's hand-rolled [0,1) mapping (rng.hpp:17-25)
struct Uniform {
  std::mt19937_64 eng;
  explicit Uniform(uint64_t seed) : eng(seed) {}
  double next() { return double(eng() >> 11) * 0x1.0p-53; }
};

// Singular values of a small square complex matrix (one-sided Jacobi; columns in a).
std::vector<double> singular_values(std::vector<cplx> a, int n) {
  auto col = [&](int j) { return a.data() + size_t(j) * n; };
  for (int sweep = 0; sweep < 60; ++sweep) {
    bool rotated = false;
    for (int p = 0; p < n - 1; ++p)
      for (int q = p + 1; q < n; ++q) {
        double al = 0, be = 0;
        cplx ga = 0;
        for (int i = 0; i < n; ++i) {
          al += std::norm(col(p)[i]);
          be += std::norm(col(q)[i]);
          ga += std::conj(col(p)[i]) * col(q)[i];
        }
        const double ag = std::abs(ga);
        if (ag == 0.0 || ag <= 1e-15 * std::sqrt(al * be)) continue;
        rotated = true;
        const double zeta = (be - al) / (2 * ag);
        const double t = (zeta >= 0 ? 1.0 : -1.0) / (std::abs(zeta) + std::sqrt(1 + zeta * zeta));
        const double c = 1 / std::sqrt(1 + t * t), s = c * t;
        const cplx e = std::conj(ga / ag);
        for (int i = 0; i < n; ++i) {
          const cplx x = col(p)[i], y = e * col(q)[i];
          col(p)[i] = c * x - s * y;
          col(q)[i] = s * x + c * y;
        }
      }
    if (!rotated) break;
  }
  std::vector<double> sv(n);
  for (int j = 0; j < n; ++j) {
    double acc = 0;
    for (int i = 0; i < n; ++i) acc += std::norm(col(j)[i]);
    sv[j] = std::sqrt(acc);
  }
  std::sort(sv.begin(), sv.end(), std::greater<double>());
  return sv;
}

// numerical_degree (poly.cpp:143-150)
int degree(const std::vector<cplx>& p) {
  double mx = 0;
  for (const cplx& c : p) mx = std::max(mx, std::abs(c));
  if (mx == 0.0) return -1;
  for (int i = int(p.size()) - 1; i >= 0; --i)
    if (std::abs(p[i]) > 1e-12 * mx) return i;
  return -1;
}

// restriction_margin (encoder.cpp:16-24) via the Sylvester matrix (poly.cpp:132-141)
double restriction_margin(const std::vector<cplx>& p, const std::vector<cplx>& q) {
  const int dp = degree(p), dq = degree(q);
  if (dp < 0 || dq < 0) return 0.0;
  if (dp == 0 && dq == 0) return 1.0;
  const int n = dp + dq;
  std::vector<cplx> s(size_t(n) * n, 0.0);  // column-major
  auto at = [&](int r, int c) -> cplx& { return s[size_t(c) * n + r]; };
  for (int r = 0; r < dq; ++r)
    for (int k = 0; k <= dp; ++k) at(r, r + k) = p[dp - k];
  for (int r = 0; r < dp; ++r)
    for (int k = 0; k <= dq; ++k) at(dq + r, r + k) = q[dq - k];
  const std::vector<double> sv = singular_values(s, n);
  return sv[0] == 0.0 ? 0.0 : sv.back() / sv[0];
}

// One-point axis_dft restriction of a t x t row-major kernel (poly.cpp:40-64)
std::vector<cplx> restrict_axis(const double* w, int t, int axis, cplx pt) {
  const double theta = std::arg(pt);
  std::vector<double> pr(t), pi(t);
  for (int m = 0; m < t; ++m) {
    const cplx z = std::polar(1.0, theta * double(m));
    pr[m] = z.real(), pi[m] = z.imag();
  }
  std::vector<cplx> out(t);
  for (int o = 0; o < t; ++o) {
    double re = 0, im = 0;
    for (int m = 0; m < t; ++m) {
      const double v = axis == 0 ? w[m * t + o] : w[o * t + m];
      re += v * pr[m];
      im += v * pi[m];
    }
    out[o] = cplx(re, im);
  }
  return out;
}

double margin_of(const double* k1, const double* k2, int t, int trials) {  // encoder.cpp:45-64
  Uniform rng(0x5ca1ab1e0ddba11ull);
  double margin = 1.0;
  for (int trial = 0; trial < trials; ++trial) {
    const cplx w = std::polar(1.0, 2.0 * M_PI * rng.next());
    for (int axis = 0; axis < 2; ++axis)
      margin = std::min(margin, restriction_margin(restrict_axis(k1, t, axis, w), restrict_axis(k2, t, axis, w)));
  }
  return margin;
}

void draw_kernel(int t, Uniform& rng, double* w) {  // encoder.cpp:26-34 (column-major draw)
  for (int n = 0; n < t; ++n)
    for (int m = 0; m < t; ++m) w[m * t + n] = rng.next();
  double s = 0;
  for (int n = 0; n < t; ++n)
    for (int m = 0; m < t; ++m) s += w[m * t + n];
  for (int i = 0; i < t * t; ++i) w[i] /= s;
}

}  // namespace

extern "C" {

uint64_t cbp_frame_seed(uint64_t stream_seed, int frame_index) {  // rng.hpp:27-29
  return splitmix64(stream_seed ^ (0x9E3779B97F4A7C15ull * uint64_t(frame_index) + 1));
}

uint64_t cbp_splitmix64(uint64_t x) { return splitmix64(x); }

int cbp_random_frame(int rows, int cols, int channels, uint64_t seed, float* out) {  // synth.cpp:12-22
  if (rows <= 0 || cols <= 0) return CBP_INVALID_ARGUMENT;
  if (channels != 1 && channels != 3) return CBP_INVALID_ARGUMENT;
  Uniform rng(seed);
  for (int c = 0; c < channels; ++c)
    for (int n = 0; n < cols; ++n)
      for (int m = 0; m < rows; ++m) out[(size_t(c) * rows + m) * cols + n] = float(rng.next());
  return 0;
}

double cbp_coprimality_check(const double* k1, const double* k2, int t, int trials) {
  return margin_of(k1, k2, t, trials);
}

int cbp_generate_coprime_pair(int width, uint64_t seed, int max_retries, double margin_threshold, int trials,
                              double* k1, double* k2, double* margin) {  // encoder.cpp:66-81
  if (!(width >= 3 && width <= 63 && width % 2 == 1)) return CBP_INVALID_ARGUMENT;
  if (max_retries < 1 || !(margin_threshold > 0.0) || trials < 1) return CBP_INVALID_ARGUMENT;
  Uniform rng(seed);
  for (int attempt = 0; attempt < max_retries; ++attempt) {
    draw_kernel(width, rng, k1);
    draw_kernel(width, rng, k2);
    const double m = margin_of(k1, k2, width, trials);
    if (m > margin_threshold) {
      *margin = m;
      return 0;
    }
  }
  return CBP_COPRIMALITY_FAILURE;
}

}  // extern "C"
