// CBP ORACLE — TEST INFRASTRUCTURE ONLY. Flat C entry points over cbp_oracle.cpp
// for ctypes (tests/, smoke(), bench.py cpu_baseline / --impl reference).
// Arrays are row-major; complex arrays are interleaved (re, im) doubles.
// Return value: 0 = ok, otherwise 1 + Errc index; orc_last_error() has the text.
#include <atomic>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "cbp_oracle.hpp"

using namespace orc;

namespace {
thread_local std::string g_err;

template <class F>
int guard(F&& f) {
  try {
    f();
    g_err.clear();
    return 0;
  } catch (const Error& e) {
    g_err = e.what();
    return 1 + int(e.code());
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1000;
  }
}

Mat mat_in(const double* p, int r, int c) {
  Mat m(r, c);
  std::memcpy(m.data(), p, sizeof(double) * size_t(r) * c);
  return m;
}
void mat_out(const Mat& m, double* p) { std::memcpy(p, m.data(), sizeof(double) * m.size()); }
CVec cvec_in(const double* p, int n) {
  CVec v(static_cast<size_t>(n));
  for (int i = 0; i < n; ++i) v[i] = cplx(p[2 * i], p[2 * i + 1]);
  return v;
}
void cvec_out(const CVec& v, double* p) {
  for (size_t i = 0; i < v.size(); ++i) p[2 * i] = v[i].real(), p[2 * i + 1] = v[i].imag();
}
CMat cmat_in(const double* p, int r, int c) {
  CMat m(r, c);
  for (size_t i = 0; i < m.size(); ++i) m.v[i] = cplx(p[2 * i], p[2 * i + 1]);
  return m;
}
void cmat_out(const CMat& m, double* p) {
  for (size_t i = 0; i < m.size(); ++i) p[2 * i] = m.v[i].real(), p[2 * i + 1] = m.v[i].imag();
}
Frame frame_in(const double* p, int ch, int r, int c) {
  Frame f;
  for (int k = 0; k < ch; ++k) f.planes.push_back(mat_in(p + size_t(k) * r * c, r, c));
  return f;
}
BlurKernel kernel_in(const double* w, int t) { return BlurKernel{t, mat_in(w, t, t)}; }
}  // namespace

extern "C" {

// Mirrors cbp_decode_cfg in include/cbp_cuda.h field for field.
struct orc_decode_cfg {
  int search_min, search_max;
  double tau;
  int has_epsilon;
  double epsilon;
  double gap_threshold;
  int trust_hint;
  double max_imag_energy, negative_weight_tol;
  int validate;
};
struct orc_decode_info {
  int width_used, width_clamped;
  double validation_residual, epsilon_used;
  double stage_ms[5];
};

const char* orc_last_error() { return g_err.c_str(); }
uint64_t orc_splitmix64(uint64_t x) { return splitmix64(x); }
uint64_t orc_frame_seed(uint64_t s, int i) { return frame_seed(s, i); }
int orc_friendly_size(int n) {
  int out = 0;
  int st = guard([&] { out = friendly_size(n); });
  return st ? -st : out;
}

int orc_random_frame(int rows, int cols, int channels, uint64_t seed, double* out) {
  return guard([&] {
    Frame f = random_frame(rows, cols, channels, seed);
    for (int k = 0; k < channels; ++k) mat_out(f.planes[k], out + size_t(k) * rows * cols);
  });
}
int orc_random_mat(int rows, int cols, uint64_t seed, double lo, double hi, double* out) {
  return guard([&] { mat_out(random_mat(rows, cols, seed, lo, hi), out); });
}

int orc_generate_coprime_pair(int width, uint64_t seed, int max_retries, double margin_threshold,
                              int trials, double* k1, double* k2, double* margin) {
  return guard([&] {
    CoprimePair p = generate_coprime_pair(width, seed, max_retries, margin_threshold, trials);
    mat_out(p.k1.weights, k1);
    mat_out(p.k2.weights, k2);
    *margin = p.coprimality_margin;
  });
}
int orc_coprimality_check(const double* k1, const double* k2, int t, int trials, double* margin) {
  return guard([&] { *margin = coprimality_check(kernel_in(k1, t), kernel_in(k2, t), trials); });
}
int orc_conv2_full(const double* a, int ar, int ac, const double* b, int br, int bc, double* out) {
  return guard([&] { mat_out(conv2_full(mat_in(a, ar, ac), mat_in(b, br, bc)), out); });
}
// Full encode: latent (channels planes) -> public (k1), private (k2).
int orc_encode_frame(const double* latent, int channels, int rows, int cols, const double* k1,
                     const double* k2, int t, double* pub, double* prv) {
  return guard([&] {
    Frame f = frame_in(latent, channels, rows, cols);
    CoprimePair p{kernel_in(k1, t), kernel_in(k2, t), 1.0, 0};
    BlurredPair bp = encode_frame(f, p);
    const size_t plane = size_t(rows + t - 1) * (cols + t - 1);
    for (int k = 0; k < channels; ++k) {
      mat_out(bp.public_frame.planes[k], pub + k * plane);
      mat_out(bp.private_frame.planes[k], prv + k * plane);
    }
  });
}
int orc_quantize(double* planes, int channels, int rows, int cols, int bits) {
  return guard([&] {
    Frame f = quantize_frame(frame_in(planes, channels, rows, cols), bits);
    for (int k = 0; k < channels; ++k) mat_out(f.planes[k], planes + size_t(k) * rows * cols);
  });
}

// degrade_bits on frames quantized to `bits` (values k / (2^bits - 1))
int orc_degrade_bits(double* planes, int channels, int rows, int cols, int bits, int drop) {
  return guard([&] {
    Frame f = frame_in(planes, channels, rows, cols);
    f.bit_depth = bits;
    Frame d = degrade_bits(f, drop);
    for (int k = 0; k < channels; ++k) mat_out(d.planes[k], planes + size_t(k) * rows * cols);
  });
}

int orc_bezout_leading_block(const double* p, int lp, const double* q, int lq, int size,
                             double* out) {
  return guard([&] { cmat_out(bezout_leading_block(cvec_in(p, lp), cvec_in(q, lq), size), out); });
}
int orc_numerical_singularity(const double* m, int n, double tau, double* ratio, int* singular) {
  return guard([&] {
    SingularityResult r = numerical_singularity(cmat_in(m, n, n), tau);
    *ratio = r.ratio;
    *singular = r.singular;
  });
}
int orc_svd(const double* a, int rows, int cols, double* sv, double* v) {
  return guard([&] {
    Vec s;
    CMat vv;
    svd(cmat_in(a, rows, cols), s, v ? &vv : nullptr);
    std::memcpy(sv, s.data(), sizeof(double) * s.size());
    if (v) cmat_out(vv, v);
  });
}
int orc_cofactor_null_solve(const double* p, int lp, const double* q, int lq, int t,
                            double gap_threshold, double* k1, double* k2, double* gap) {
  return guard([&] {
    CofactorSolution s = cofactor_null_solve(cvec_in(p, lp), cvec_in(q, lq), t, gap_threshold);
    cvec_out(s.k1, k1);
    cvec_out(s.k2, k2);
    *gap = s.gap;
  });
}
int orc_homogeneous_lsq(const double* a, int rows, int cols, double* x) {
  return guard([&] { cvec_out(homogeneous_lsq(cmat_in(a, rows, cols)), x); });
}
int orc_sylvester_matrix(const double* p, int lp, const double* q, int lq, double* out) {
  return guard([&] { cmat_out(sylvester_matrix(cvec_in(p, lp), cvec_in(q, lq)), out); });
}
int orc_numerical_degree(const double* p, int lp, double rel_tol) {
  return numerical_degree(cvec_in(p, lp), rel_tol);
}

int orc_fft2(const double* x, int rows, int cols, int inverse, double* out) {
  return guard([&] {
    CMat m = cmat_in(x, rows, cols);
    cmat_out(inverse ? ifft2(m) : fft2(m), out);
  });
}
int orc_axis_roots_dft(const double* plane, int rows, int cols, int axis, int t, double* out) {
  return guard([&] {
    cmat_out(axis_roots_dft(mat_in(plane, rows, cols), axis ? Axis::Z2 : Axis::Z1, t), out);
  });
}
int orc_axis_spectrum_half(const double* plane, int rows, int cols, int axis, double* out) {
  return guard(
      [&] { cmat_out(axis_spectrum_half(mat_in(plane, rows, cols), axis ? Axis::Z2 : Axis::Z1), out); });
}
int orc_luma(const double* planes, int channels, int rows, int cols, double* out) {
  return guard([&] { mat_out(luma(frame_in(planes, channels, rows, cols)), out); });
}

static BlurredPair pair_in(const double* pub, const double* prv, int ch, int rows, int cols,
                           int hint) {
  BlurredPair bp;
  bp.public_frame = frame_in(pub, ch, rows, cols);
  bp.private_frame = frame_in(prv, ch, rows, cols);
  if (hint > 0) bp.kernel_width_hint = hint;
  return bp;
}
static DecodeConfig cfg_in(const orc_decode_cfg* c) {
  DecodeConfig d;
  if (!c) return d;
  d.search_min = c->search_min;
  d.search_max = c->search_max;
  d.tau = c->tau;
  if (c->has_epsilon) d.epsilon = c->epsilon;
  d.gap_threshold = c->gap_threshold;
  d.trust_hint = c->trust_hint != 0;
  d.max_imag_energy = c->max_imag_energy;
  d.negative_weight_tol = c->negative_weight_tol;
  d.validate = c->validate != 0;
  return d;
}

int orc_estimate_kernel_width(const double* pub, const double* prv, int ch, int rows, int cols,
                              int smin, int smax, double tau, int* width, int* clamped) {
  return guard([&] {
    WidthEstimate e = estimate_kernel_width(pair_in(pub, prv, ch, rows, cols, 0), smin, smax, tau);
    *width = e.width;
    *clamped = e.clamped;
  });
}
int orc_sample_cofactors(const double* pub, const double* prv, int ch, int rows, int cols,
                         int width, int axis, double gap_threshold, double* values, double* gaps) {
  return guard([&] {
    ScaledKernelTransform s = sample_cofactors(pair_in(pub, prv, ch, rows, cols, 0), width,
                                               axis ? Axis::Z2 : Axis::Z1, gap_threshold);
    cmat_out(s.values, values);
    std::memcpy(gaps, s.gaps.data(), sizeof(double) * s.gaps.size());
  });
}
int orc_complete_to_spectrum(const double* values, int t, int axis, double* out) {
  return guard([&] {
    ScaledKernelTransform s;
    s.axis = axis ? Axis::Z2 : Axis::Z1;
    s.values = cmat_in(values, t, t);
    cmat_out(complete_to_spectrum(s), out);
  });
}
int orc_resolve_scales(const double* a_values, const double* b_values, int t, double* lambda,
                       double* mu, double* residual) {
  return guard([&] {
    ScaledKernelTransform a, b;
    a.axis = Axis::Z1, b.axis = Axis::Z2;
    a.values = cmat_in(a_values, t, t), b.values = cmat_in(b_values, t, t);
    ScaleResolution r = resolve_scales(a, b);
    cvec_out(r.lambda, lambda);
    cvec_out(r.mu, mu);
    *residual = r.residual;
  });
}
int orc_assemble_kernel(const double* a_spec, const double* b_spec, const double* lambda,
                        const double* mu, int t, double max_imag, double neg_tol, double* out) {
  return guard([&] {
    ScaleResolution s;
    s.lambda = cvec_in(lambda, t), s.mu = cvec_in(mu, t);
    mat_out(assemble_kernel(cmat_in(a_spec, t, t), cmat_in(b_spec, t, t), s, max_imag, neg_tol)
                .weights,
            out);
  });
}
int orc_spectral_deblur(const double* blurred, int rows, int cols, const double* kernel, int t,
                        double epsilon, double* out) {
  return guard([&] {
    mat_out(spectral_deblur(mat_in(blurred, rows, cols), kernel_in(kernel, t), epsilon), out);
  });
}
int orc_decode_frame(const double* pub, const double* prv, int ch, int rows, int cols, int hint,
                     const orc_decode_cfg* cfg, double* latent, double* kernel,
                     orc_decode_info* info) {
  return guard([&] {
    DecodedFrame d = decode_frame(pair_in(pub, prv, ch, rows, cols, hint), cfg_in(cfg));
    const int t = d.width_used;
    const size_t plane = size_t(rows - t + 1) * (cols - t + 1);
    for (int k = 0; k < ch; ++k) mat_out(d.latent.planes[k], latent + k * plane);
    mat_out(d.kernel_estimate.weights, kernel);
    info->width_used = t;
    info->width_clamped = d.width_clamped;
    info->validation_residual = d.validation_residual;
    info->epsilon_used = d.epsilon_used;
    const StageTimings& s = d.stage_timings;
    double ms[5] = {s.polynomial_evaluation_ms, s.kernel_degree_estimation_ms,
                    s.kernel_estimation_1d_ms, s.kernel_estimation_2d_fft_ms, s.total_ms};
    std::memcpy(info->stage_ms, ms, sizeof(ms));
  });
}
int orc_validate_pair(const double* pub, const double* prv, int ch, int rows, int cols,
                      const double* k1, const double* k2, int t, double* out) {
  return guard([&] {
    *out = validate_pair(pair_in(pub, prv, ch, rows, cols, 0), kernel_in(k1, t), kernel_in(k2, t));
  });
}
double orc_psnr(const double* a, const double* b, int rows, int cols) {
  return psnr(mat_in(a, rows, cols), mat_in(b, rows, cols));
}

// CPU baseline (reference CLI semantics, tools/cbp.cpp:141-164): `threads`
// workers pull frames from an atomic cursor. Each job is one epoch frame:
// job j < n_recover runs decode_frame on (pub_j, prv_j); otherwise
// spectral_deblur of every plane of pub_j with the given kernel.
// Inputs are float32 planes (the same FP32 values the GPU consumes).
int orc_bench_frames(const float* pub, const float* prv, int n_frames, int ch, int rows, int cols,
                     const int* recover, const double* kernel, int t, double epsilon,
                     const orc_decode_cfg* cfg, int threads, double* seconds) {
  return guard([&] {
    const size_t plane = size_t(rows) * cols, frame = plane * ch;
    std::atomic<int> cursor{0};
    std::atomic<int> failed{0};
    auto worker = [&] {
      for (;;) {
        int j = cursor.fetch_add(1);
        if (j >= n_frames) return;
        try {
          Frame fp, fq;
          for (int k = 0; k < ch; ++k) {
            Mat a(rows, cols), b(rows, cols);
            for (size_t i = 0; i < plane; ++i) a.v[i] = pub[j * frame + k * plane + i];
            fp.planes.push_back(std::move(a));
            if (recover[j]) {
              for (size_t i = 0; i < plane; ++i) b.v[i] = prv[j * frame + k * plane + i];
              fq.planes.push_back(std::move(b));
            }
          }
          if (recover[j]) {
            BlurredPair bp;
            bp.public_frame = std::move(fp), bp.private_frame = std::move(fq);
            bp.kernel_width_hint = t;
            decode_frame(bp, cfg_in(cfg));
          } else {
            BlurKernel k = kernel_in(kernel, t);
            for (auto& p : fp.planes) spectral_deblur(p, k, epsilon);
          }
        } catch (...) {
          failed.fetch_add(1);
        }
      }
    };
    auto t0 = std::chrono::steady_clock::now();
    std::vector<std::thread> pool;
    for (int i = 0; i < threads; ++i) pool.emplace_back(worker);
    for (auto& th : pool) th.join();
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    require(failed.load() == 0, Errc::invalid_argument, "a baseline frame failed to decode");
  });
}

}  // extern "C"
