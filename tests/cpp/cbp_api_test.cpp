// C++ API tests for the B200 build, written against the reference's public headers
// (include/cbp/*.hpp keeps their names) and mirroring proj/tests/unit/decoder_test.cpp,
// encoder_test.cpp and poly_test.cpp cases with the reference's tolerances. Built by
// __graft_entry__.build(); run by tests/test_cpp_api.py on a GPU box.
#include <cmath>
#include <cstdio>
#include <filesystem>
#include <fstream>
#include <iterator>
#include <random>
#include <string>

#include "cbp/decoder.hpp"
#include "cbp/encoder.hpp"
#include "cbp/fft.hpp"
#include "cbp/metrics.hpp"
#include "cbp/poly.hpp"
#include "cbp/stream_io.hpp"
#include "cbp/synth.hpp"

using namespace cbp;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                                              \
  do {                                                                           \
    if (cond) {                                                                  \
      ++g_pass;                                                                  \
    } else {                                                                     \
      ++g_fail;                                                                  \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);                \
    }                                                                            \
  } while (0)
#define CHECK_THROWS_CODE(expr, errc)                                            \
  do {                                                                           \
    bool threw = false;                                                          \
    try {                                                                        \
      (void)(expr);                                                              \
    } catch (const Error& e) {                                                   \
      threw = e.code() == errc;                                                  \
    }                                                                            \
    CHECK(threw);                                                                \
  } while (0)

namespace fs = std::filesystem;

namespace {
// tests/support.hpp:31-39
Mat random_mat(int rows, int cols, std::uint64_t seed, double lo = 0.0, double hi = 1.0) {
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<double> dist(lo, hi);
  Mat m(rows, cols);
  for (int i = 0; i < rows; ++i)
    for (int j = 0; j < cols; ++j) m(i, j) = dist(rng);
  return m;
}
Frame gray(const Mat& m) {
  Frame f;
  f.planes = {m};
  return f;
}
double max_abs_diff(const Mat& a, const Mat& b) {
  double d = 0;
  for (long i = 0; i < a.size(); ++i) d = std::max(d, std::abs(a.data()[i] - b.data()[i]));
  return d;
}
double aligned_error(const CVec& e1, const CVec& e2, const CVec& r1, const CVec& r2) {
  cplx num = 0, den = 0;
  for (long i = 0; i < e1.size(); ++i) num += std::conj(e1[i]) * r1[i], den += std::conj(e1[i]) * e1[i];
  for (long i = 0; i < e2.size(); ++i) num += std::conj(e2[i]) * r2[i], den += std::conj(e2[i]) * e2[i];
  const cplx c = num / den;
  double m = 0;
  for (long i = 0; i < e1.size(); ++i) m = std::max(m, std::abs(c * e1[i] - r1[i]));
  for (long i = 0; i < e2.size(); ++i) m = std::max(m, std::abs(c * e2[i] - r2[i]));
  return m;
}
DecodeConfig small_search(int lo = 3, int hi = 9) {
  DecodeConfig c;
  c.search_min = lo;
  c.search_max = hi;
  return c;
}
}  // namespace

// public/private streams of `n` encoded frames (the `cbp encode` layout, tools/cbp.cpp:60-114)
void write_pair_streams(const fs::path& dir, int n, int rows, int cols, int ch, int t, BitDepth depth,
                        std::vector<Frame>* latents = nullptr) {
  std::vector<Frame> pub, prv;
  std::string id;
  for (int i = 0; i < n; ++i) {
    const Frame lat = random_frame(rows, cols, ch, frame_seed(11, i));
    BlurredPair bp = encode_frame(lat, generate_coprime_pair(t, frame_seed(12, i)));
    if (depth != BitDepth::f32) {
      bp.public_frame = quantize_frame(bp.public_frame, depth);
      bp.private_frame = quantize_frame(bp.private_frame, depth);
    }
    if (i == 0) id = bp.pair_id;
    pub.push_back(bp.public_frame);
    prv.push_back(bp.private_frame);
    if (latents) latents->push_back(lat);
  }
  StreamManifest m;
  m.frame_count = n;
  m.width = pub.front().cols();
  m.height = pub.front().rows();
  m.bit_depth = depth;
  m.pair_id = id;
  m.kernel_width_hint = t;
  m.role = StreamRole::Public;
  write_stream(pub, m, dir / "public");
  m.role = StreamRole::Private;
  write_stream(prv, m, dir / "private");
}

int main(int argc, char** argv) {
  if (argc == 3 && std::string(argv[1]) == "--write-streams") {  // fixture for the cbp-decode CLI test
    write_pair_streams(argv[2], 3, 40, 48, 3, 5, BitDepth::u16);
    return 0;
  }
  // decoder_test.cpp:311-331 round trip on a midsize scene
  {
    const Mat latent = random_mat(64, 64, 137);
    const CoprimePair pair = generate_coprime_pair(5, 137);
    const BlurredPair bp = encode_frame(gray(latent), pair);
    CHECK(bp.kernel_width_hint == 5 && !bp.pair_id.empty());
    const DecodedFrame dec = decode_frame(bp, small_search());
    CHECK(dec.width_used == 5);
    CHECK(!dec.width_clamped);
    CHECK(dec.latent.rows() == 64 && dec.latent.cols() == 64);
    CHECK(psnr(latent, dec.latent.planes[0]) >= 40.0);
    CHECK(dec.validation_residual <= 1e-4);
    CHECK(max_abs_diff(dec.kernel_estimate.weights, pair.k1.weights) <= 1e-6);
    const StageTimings& st = dec.stage_timings;
    CHECK(st.total_ms >= 0.95 * (st.polynomial_evaluation_ms + st.kernel_degree_estimation_ms +
                                 st.kernel_estimation_1d_ms + st.kernel_estimation_2d_fft_ms));
  }
  // decoder_test.cpp:333-346 trusted hint gives the same result
  {
    const Mat latent = random_mat(48, 40, 139);
    const CoprimePair pair = generate_coprime_pair(5, 139);
    const BlurredPair bp = encode_frame(gray(latent), pair);
    DecodeConfig cfg = small_search();
    const DecodedFrame est = decode_frame(bp, cfg);
    cfg.trust_hint = true;
    const DecodedFrame hinted = decode_frame(bp, cfg);
    CHECK(hinted.width_used == 5);
    CHECK(max_abs_diff(hinted.latent.planes[0], est.latent.planes[0]) == 0.0);
    CHECK(max_abs_diff(hinted.kernel_estimate.weights, est.kernel_estimate.weights) == 0.0);
  }
  // decoder_test.cpp:40-83 width estimation
  {
    const BlurredPair bp = encode_frame(gray(random_mat(24, 24, 101)), generate_coprime_pair(5, 101));
    const WidthEstimate e = estimate_kernel_width(bp, 3, 7, 1e-6);
    CHECK(e.width == 5 && !e.clamped);
    const BlurredPair wide = encode_frame(gray(random_mat(64, 64, 104)), generate_coprime_pair(27, 101));
    const WidthEstimate c = estimate_kernel_width(wide, 9, 25, 1e-6);
    CHECK(c.width == 25 && c.clamped);
    BlurredPair ns;
    const Mat lat = random_mat(16, 16, 105);
    ns.public_frame = gray(conv2_full(lat, random_mat(3, 5, 106, 0.05, 1.0)));
    ns.private_frame = gray(conv2_full(lat, random_mat(3, 5, 107, 0.05, 1.0)));
    CHECK_THROWS_CODE(estimate_kernel_width(ns, 3, 7, 1e-6), Errc::inconsistent_axes);
  }
  // decoder_test.cpp:107-130 sample_cofactors through a real scene, zero scene
  {
    const CoprimePair pair = generate_coprime_pair(3, 113);
    const BlurredPair bp = encode_frame(gray(random_mat(16, 16, 113)), pair);
    const ScaledKernelTransform skt = sample_cofactors(bp, 3, Axis::Z1);
    const CMat ref = axis_roots_dft(pair.k1.weights, Axis::Z1, 3);
    for (int i = 0; i < 3; ++i) {
      CVec got(3), want(3), none;
      double nrm = 0;
      for (int k = 0; k < 3; ++k) got[k] = skt.values(i, k), want[k] = ref(i, k), nrm += std::norm(got[k]);
      CHECK(std::abs(std::sqrt(nrm) - 1.0) <= 1e-9);
      CHECK(aligned_error(got, none, want, none) <= 1e-5);  // FP32 device inputs
      CHECK(skt.gaps[i] > 1e-6);
    }
    BlurredPair z;
    z.public_frame = gray(Mat::Zero(8, 8));
    z.private_frame = gray(Mat::Zero(8, 8));
    CHECK_THROWS_CODE(sample_cofactors(z, 3, Axis::Z1), Errc::ill_conditioned_slice);
  }
  // decoder_test.cpp:143-156 resolve_scales on consistent transforms; 224-247 assemble
  {
    const CoprimePair pair = generate_coprime_pair(3, 117);
    ScaledKernelTransform a, b;
    a.axis = Axis::Z1, b.axis = Axis::Z2;
    a.values = axis_roots_dft(pair.k1.weights, Axis::Z1, 3);
    b.values = axis_roots_dft(pair.k1.weights, Axis::Z2, 3);
    const ScaleResolution res = resolve_scales(a, b);
    CHECK(res.residual <= 1e-12);
    for (int i = 0; i < 3; ++i) CHECK(std::abs(res.lambda[i] - res.lambda[0]) <= 1e-12 && std::abs(res.mu[i] - res.mu[0]) <= 1e-12);
    const BlurKernel k = assemble_kernel(complete_to_spectrum(a), complete_to_spectrum(b), res);
    CHECK(max_abs_diff(k.weights, pair.k1.weights) <= 1e-8);
  }
  // decoder_test.cpp:278-294 spectral_deblur identity and inverse
  {
    const Mat b = random_mat(9, 7, 131);
    BlurKernel id{1, Mat::Ones(1, 1)};
    CHECK(max_abs_diff(spectral_deblur(b, id, 0.0), b) <= 1e-6);  // FP32 device path
    const Mat latent = random_mat(16, 16, 133);
    const CoprimePair pair = generate_coprime_pair(3, 133);
    const Mat back = spectral_deblur(conv2_full(latent, pair.k1.weights), pair.k1, 1e-12);
    CHECK(back.rows() == 16 && back.cols() == 16);
    CHECK(psnr(latent, back) >= 80.0);
  }
  // decoder_test.cpp:401-409 RGB via luma; 411-417 hopeless scene; 441-450 validate_pair
  {
    Frame rgb;
    rgb.planes = {random_mat(24, 24, 147), random_mat(24, 24, 148), random_mat(24, 24, 149)};
    const DecodedFrame dec = decode_frame(encode_frame(rgb, generate_coprime_pair(3, 147)), small_search(3, 7));
    CHECK(dec.latent.channels() == 3 && psnr(rgb, dec.latent) >= 40.0);
    BlurredPair z;
    z.public_frame = gray(Mat::Zero(12, 12));
    z.private_frame = gray(Mat::Zero(12, 12));
    z.kernel_width_hint = 3;
    DecodeConfig cfg = small_search(3, 7);
    cfg.trust_hint = true;
    bool threw = false;
    try {
      decode_frame(z, cfg);
    } catch (const Error& e) {
      threw = std::string(e.what()).rfind("IllConditionedSlice: kernel_estimation_1d: ", 0) == 0;
    }
    CHECK(threw);
    const CoprimePair pair = generate_coprime_pair(3, 155);
    const BlurredPair bp = encode_frame(gray(random_mat(16, 16, 155)), pair);
    CHECK(validate_pair(bp, pair.k1, pair.k2) <= 1e-6);
  }
  // poly_test.cpp:335-384 cofactor_null_solve known answers
  {
    const CofactorSolution s = cofactor_null_solve(CVec{1, 3, 2}, CVec{3, 4, 1}, 2);
    CHECK(aligned_error(s.k1, s.k2, CVec{1, 2}, CVec{3, 1}) <= 1e-12);
    CHECK(s.gap > 1e-3);
    CHECK_THROWS_CODE(cofactor_null_solve(CVec{1, 2, 1}, CVec{1, 2, 1}, 2), Errc::ill_conditioned);
  }
  // poly_test.cpp:134-287 and fft_test.cpp:32-74: the stand-alone device utilities
  {
    const CMat b1 = bezout_leading_block(CVec{1, 2}, CVec{3, 1}, 1);  // resultant of a linear pair
    CHECK(b1.rows() == 1 && b1(0, 0) == cplx(5, 0));
    const CMat b2 = bezout_leading_block(CVec{1, 3, 2}, CVec{3, 4, 1}, 2);  // shared root z = -1
    bool all5 = true;
    for (int i = 0; i < 2; ++i)
      for (int j = 0; j < 2; ++j) all5 = all5 && b2(i, j) == cplx(5, 0);
    CHECK(all5);
    CHECK(numerical_singularity(b2, 1e-8).singular);
    CHECK_THROWS_CODE(bezout_leading_block(CVec{0, 0}, CVec{1, 2}, 2), Errc::degenerate_input);
    CMat id = CMat::Zero(3, 3);
    for (int i = 0; i < 3; ++i) id(i, i) = 1.0;
    const SingularityResult si = numerical_singularity(id, 1e-8);
    CHECK(!si.singular && std::abs(si.ratio - 1.0) <= 1e-12);
    const SingularityResult sf = numerical_singularity(CMat(2, 2, cplx(5, 0)), 1e-8);
    CHECK(sf.singular && sf.ratio <= 1e-15);
    const SingularityResult sz = numerical_singularity(CMat::Zero(4, 4), 1e-8);
    CHECK(sz.singular && sz.ratio == 0.0);
    CMat a = CMat::Zero(2, 2);
    a(0, 0) = 1.0;
    const CVec x = homogeneous_lsq(a);
    CHECK(std::abs(x[0]) <= 1e-12 && std::abs(std::abs(x[1]) - 1.0) <= 1e-12);
    CHECK_THROWS_CODE(homogeneous_lsq(CMat::Ones(2, 3)), Errc::invalid_argument);
    Mat delta = Mat::Zero(3, 4);
    delta(0, 0) = 1.0;
    const CMat f = fft2(delta);
    double err = 0.0;
    for (int i = 0; i < 3; ++i)
      for (int j = 0; j < 4; ++j) err = std::max(err, std::abs(f(i, j) - cplx(1, 0)));
    CHECK(err <= 1e-12);
    const Mat r = random_mat(61, 97, 18);
    const CMat back = ifft2(fft2(r));
    double rt = 0.0;
    for (int j = 0; j < 97; ++j)
      for (int i = 0; i < 61; ++i) rt = std::max(rt, std::abs(back(i, j) - cplx(r(i, j), 0.0)));
    CHECK(rt <= 1e-10);
    const CMat s = sylvester_matrix(CVec{1, 2}, CVec{3, 1});
    CHECK(std::abs(s(0, 0) * s(1, 1) - s(0, 1) * s(1, 0)) == 5.0);
    CHECK(numerical_degree(CVec{0, 1, 1e-15}) == 1 && numerical_degree(CVec{0, 0}) == -1);
    // encoder_test.cpp:190-215 degrade_bits on a u8 frame
    Frame q;
    q.bit_depth = BitDepth::u8;
    q.planes.push_back(Mat(1, 2, 255.0 / 255.0));
    q.planes[0](0, 1) = 7.0 / 255.0;
    const Frame d = degrade_bits(q, 2);
    CHECK(d.planes[0](0, 0) == 252.0 / 255.0 && d.planes[0](0, 1) == 4.0 / 255.0);
    CHECK_THROWS_CODE(degrade_bits(q, 8), Errc::invalid_argument);
    Frame f32 = q;
    f32.bit_depth = BitDepth::f32;
    CHECK_THROWS_CODE(degrade_bits(f32, 1), Errc::not_quantized);
  }
  // encoder_test.cpp:28-54 determinism and validation
  {
    const CoprimePair a = generate_coprime_pair(9, 42), b = generate_coprime_pair(9, 42);
    CHECK(a.coprimality_margin > 1e-6 && max_abs_diff(a.k1.weights, b.k1.weights) == 0.0);
    CHECK_THROWS_CODE(generate_coprime_pair(4, 1), Errc::invalid_argument);
  }
  // disk-to-disk decode (tools/cbp.cpp:130-207): f32 and u16 streams, sidecars, exit codes
  for (BitDepth depth : {BitDepth::f32, BitDepth::u16}) {
    const fs::path dir = fs::temp_directory_path() / ("cbp_dec_" + std::to_string(int(depth)));
    fs::remove_all(dir);
    std::vector<Frame> lat;
    write_pair_streams(dir, 4, 48, 56, depth == BitDepth::f32 ? 1 : 3, 5, depth, &lat);
    DecodeStreamOptions o;
    o.pub = dir / "public";
    o.prv = dir / "private";
    o.out = dir / "latent";
    o.width_min = 3;
    o.width_max = 9;
    o.batch = 3;  // two device batches
    o.trust_hint = depth != BitDepth::f32;  // quantization noise swamps the width search (acceptance.cpp:379)
    o.verbose = false;
    CHECK(decode_stream(o) == 0);
    auto [back, m] = read_stream(o.out);
    CHECK(m.role == StreamRole::Latent && m.frame_count == 4 && m.bit_depth == BitDepth::f32);
    for (int i = 0; i < 4; ++i) CHECK(psnr(lat[size_t(i)], back[size_t(i)]) >= 40.0);
    char side[64];
    std::snprintf(side, sizeof(side), "frame_%06d.json", 3);
    std::ifstream sf(o.out / side);
    const std::string text((std::istreambuf_iterator<char>(sf)), std::istreambuf_iterator<char>());
    CHECK(text.find("\"width_used\": 5") != std::string::npos && text.find("\"total_ms\"") != std::string::npos);
    o.max_residual = 1e-30;  // every residual above it: status 4
    CHECK(decode_stream(o) == 4);
    o.prv = o.pub;  // two public streams do not pair
    CHECK_THROWS_CODE(decode_stream(o), Errc::pair_mismatch);
    fs::remove_all(dir);
  }
  std::printf("cbp_api_test: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail == 0 ? 0 : 1;
}
