// Stream I/O tests (no GPU needed): the behaviours pinned by the reference's
// proj/tests/unit/stream_io_test.cpp and acceptance criterion 9 (byte-exact persistence),
// exercised through include/cbp/stream_io.hpp. Run by tests/test_cpp_api.py.
#include <cstdio>
#include <cstring>
#include <filesystem>
#include <fstream>
#include <random>
#include <sstream>
#include <string>

#include "cbp/stream_io.hpp"

using namespace cbp;
namespace fs = std::filesystem;

static int g_fail = 0, g_pass = 0;
#define CHECK(cond)                                               \
  do {                                                            \
    if (cond) {                                                   \
      ++g_pass;                                                   \
    } else {                                                      \
      ++g_fail;                                                   \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond); \
    }                                                             \
  } while (0)

namespace {

template <class F>
Errc code_of(F&& f) {  // Errc thrown by f (invalid_argument if none: the test then fails)
  try {
    f();
  } catch (const Error& e) {
    return e.code();
  }
  return Errc(-1);
}

struct Tmp {
  fs::path p;
  explicit Tmp(const std::string& tag) {
    p = fs::temp_directory_path() / ("cbp_stream_" + tag + "_" + std::to_string(std::random_device{}()));
    fs::remove_all(p);
  }
  ~Tmp() { fs::remove_all(p); }
  operator const fs::path&() const { return p; }
  fs::path operator/(const std::string& s) const { return p / s; }
};

std::string bytes_of(const fs::path& p) {
  std::ifstream in(p, std::ios::binary);
  std::stringstream ss;
  ss << in.rdbuf();
  return ss.str();
}

void put_bytes(const fs::path& p, const std::string& s) { std::ofstream(p, std::ios::binary) << s; }

// frames with samples on the depth's grid (u8/u16) or arbitrary floats
std::vector<Frame> frames_of(int n, int rows, int cols, int ch, BitDepth d, unsigned seed) {
  std::mt19937 rng(seed);
  std::uniform_real_distribution<double> u(0.0, 1.0);
  const double maxv = d == BitDepth::u8 ? 255.0 : d == BitDepth::u16 ? 65535.0 : 0.0;
  std::vector<Frame> out(static_cast<size_t>(n));
  for (auto& f : out) {
    f.bit_depth = d;
    for (int k = 0; k < ch; ++k) {
      ImagePlane p(rows, cols);
      for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c) {
          double v = u(rng);
          if (maxv > 0) v = std::round(v * maxv) / maxv;
          else v = double(float(v));
          p(r, c) = v;
        }
      f.planes.push_back(p);
    }
  }
  return out;
}

StreamManifest manifest(const std::vector<Frame>& f, StreamRole role, const std::string& id = "pair-test") {
  StreamManifest m;
  m.role = role;
  m.frame_count = int(f.size());
  m.width = f.front().cols();
  m.height = f.front().rows();
  m.bit_depth = f.front().bit_depth;
  m.pair_id = id;
  return m;
}

bool same(const Frame& a, const Frame& b) {
  if (a.channels() != b.channels() || a.rows() != b.rows() || a.cols() != b.cols()) return false;
  for (int k = 0; k < a.channels(); ++k)
    for (int r = 0; r < a.rows(); ++r)
      for (int c = 0; c < a.cols(); ++c)
        if (a.planes[size_t(k)](r, c) != b.planes[size_t(k)](r, c)) return false;
  return true;
}

}  // namespace

int main() {
  {  // PFM layout: header, little-endian floats, bottom row first
    Tmp d("pfm");
    Frame f;
    ImagePlane p(2, 2);
    p(0, 0) = 0.1, p(0, 1) = 0.2, p(1, 0) = 0.3, p(1, 1) = 0.4;
    f.planes = {p};
    write_stream({f}, manifest({f}, StreamRole::Latent), d);
    const std::string b = bytes_of(d / "frame_000000.pfm");
    const std::string h = "Pf\n2 2\n-1.0\n";
    CHECK(b.size() == h.size() + 16 && b.compare(0, h.size(), h) == 0);
    float v = 0;
    std::memcpy(&v, b.data() + h.size(), 4);
    CHECK(v == 0.3f);
  }
  {  // 16-bit PGM samples are big-endian
    Tmp d("pgm16");
    Frame f;
    f.bit_depth = BitDepth::u16;
    ImagePlane p(2, 2, 0.0);
    p(0, 0) = 258.0 / 65535.0;
    f.planes = {p};
    write_stream({f}, manifest({f}, StreamRole::Latent), d);
    const std::string b = bytes_of(d / "frame_000000.pgm");
    const std::string h = "P5\n2 2\n65535\n";
    CHECK(b.size() == h.size() + 8 && b.compare(0, h.size(), h) == 0);
    CHECK((unsigned char)b[h.size()] == 0x01 && (unsigned char)b[h.size() + 1] == 0x02);
  }
  // round trips for every depth and channel layout, and byte-exact re-writes (criterion 9)
  for (BitDepth depth : {BitDepth::f32, BitDepth::u16, BitDepth::u8})
    for (int ch : {1, 3}) {
      Tmp a("rt_a"), b("rt_b");
      auto fr = frames_of(3, 5, 7, ch, depth, 11 + ch);
      StreamManifest m = manifest(fr, StreamRole::Public);
      m.kernel_width_hint = 9;
      m.seed = 12345678901234567890ull;
      write_stream(fr, m, a);
      auto [back, got] = read_stream(a);
      CHECK(back.size() == fr.size());
      for (size_t i = 0; i < fr.size(); ++i) CHECK(same(back[i], fr[i]) && back[i].index == int(i));
      CHECK(got.bit_depth == depth && got.role == StreamRole::Public && got.kernel_width_hint == 9);
      CHECK(got.seed && *got.seed == 12345678901234567890ull);
      write_stream(back, got, b);
      for (const auto& e : fs::directory_iterator(a.p))
        CHECK(bytes_of(e.path()) == bytes_of(b / e.path().filename().string()));
    }
  {  // manifest keys sorted (the reference's nlohmann dump order)
    Tmp d("keys");
    auto fr = frames_of(1, 3, 3, 1, BitDepth::f32, 31);
    StreamManifest m = manifest(fr, StreamRole::Private, "pair-keys");
    m.kernel_width_hint = 5;
    m.seed = 99;
    write_stream(fr, m, d);
    const std::string text = bytes_of(d / "manifest.json");
    size_t last = 0;
    bool ordered = true;
    for (const char* k : {"bit_depth", "frame_count", "height", "kernel_width_hint", "pair_id", "role", "seed",
                          "version", "width"}) {
      const size_t at = text.find(std::string("\"") + k + "\"");
      ordered = ordered && at != std::string::npos && at > last;
      last = at;
    }
    CHECK(ordered);
  }
  {  // pair_streams: order, role symmetry, hint agreement, mismatches
    Tmp a("pa"), b("pb");
    auto fa = frames_of(2, 4, 4, 1, BitDepth::f32, 1), fb = frames_of(2, 4, 4, 1, BitDepth::f32, 2);
    StreamManifest ma = manifest(fa, StreamRole::Public), mb = manifest(fb, StreamRole::Private);
    ma.kernel_width_hint = 5;
    mb.kernel_width_hint = 5;
    write_stream(fa, ma, a);
    write_stream(fb, mb, b);
    auto pairs = pair_streams(a, b);
    CHECK(pairs.size() == 2 && same(pairs[1].public_frame, fa[1]) && same(pairs[1].private_frame, fb[1]));
    CHECK(pairs[0].kernel_width_hint == 5 && pairs[0].pair_id == "pair-test");
    auto rev = pair_streams(b, a);  // either order pairs
    CHECK(same(rev[0].public_frame, fb[0]));
    mb.kernel_width_hint = 7;
    write_stream(fb, mb, b);
    CHECK(!pair_streams(a, b)[0].kernel_width_hint);
    CHECK(code_of([&] { pair_streams(a, a); }) == Errc::pair_mismatch);  // public + public
    mb.pair_id = "other";
    write_stream(fb, mb, b);
    CHECK(code_of([&] { pair_streams(a, b); }) == Errc::pair_mismatch);
    Tmp c("pc");
    auto fc = frames_of(3, 4, 4, 1, BitDepth::f32, 3);
    write_stream(fc, manifest(fc, StreamRole::Private), c);
    CHECK(code_of([&] { pair_streams(a, c); }) == Errc::pair_mismatch);  // frame count
  }
  {  // precise read failures
    auto fr = frames_of(2, 4, 4, 1, BitDepth::f32, 45);
    const StreamManifest m = manifest(fr, StreamRole::Latent);
    Tmp d1("garbled");
    write_stream(fr, m, d1);
    put_bytes(d1 / "manifest.json", "{not json");
    CHECK(code_of([&] { read_stream(d1); }) == Errc::corrupt_manifest);
    Tmp d2("version");
    write_stream(fr, m, d2);
    std::string t = bytes_of(d2 / "manifest.json");
    t.replace(t.find("\"version\": 1"), 12, "\"version\": 2");
    put_bytes(d2 / "manifest.json", t);
    CHECK(code_of([&] { read_stream(d2); }) == Errc::corrupt_manifest);
    Tmp d3("gone");
    write_stream(fr, m, d3);
    fs::remove(d3 / "frame_000001.pfm");
    CHECK(code_of([&] { read_stream(d3); }) == Errc::missing_frame);
    Tmp d4("short");
    write_stream(fr, m, d4);
    const std::string b = bytes_of(d4 / "frame_000000.pfm");
    put_bytes(d4 / "frame_000000.pfm", b.substr(0, b.size() - 7));
    CHECK(code_of([&] { read_stream(d4); }) == Errc::format_violation);
    Tmp d5("maxval");
    auto q = frames_of(1, 2, 2, 1, BitDepth::u8, 46);
    write_stream(q, manifest(q, StreamRole::Latent), d5);
    put_bytes(d5 / "frame_000000.pgm", std::string("P5\n2 2\n2\n\0\0\0\0", 13));
    CHECK(code_of([&] { read_stream(d5); }) == Errc::format_violation);
    CHECK(code_of([&] { read_stream(fs::temp_directory_path() / "cbp_no_such_stream_dir"); }) == Errc::io_failure);
  }
  {  // write-side validation is a caller error
    Tmp d("validate");
    auto fr = frames_of(2, 4, 4, 1, BitDepth::f32, 47);
    StreamManifest m = manifest(fr, StreamRole::Latent);
    m.width = 5;
    CHECK(code_of([&] { write_stream(fr, m, d); }) == Errc::invalid_argument);
    StreamManifest e = manifest(fr, StreamRole::Latent);
    e.frame_count = 0;
    CHECK(code_of([&] { write_stream({}, e, d); }) == Errc::invalid_argument);
  }
  {  // PNM header comments
    Tmp d("comments");
    auto q = frames_of(1, 2, 3, 1, BitDepth::u8, 48);
    write_stream(q, manifest(q, StreamRole::Latent), d);
    const std::string b = bytes_of(d / "frame_000000.pgm");
    const std::string h = "P5\n3 2\n255\n";
    CHECK(b.compare(0, h.size(), h) == 0);
    put_bytes(d / "frame_000000.pgm", "P5\n# a comment\n3 2\n255\n" + b.substr(h.size()));
    auto [back, got] = read_stream(d);
    CHECK(same(back[0], q[0]));
  }
  CHECK(exit_code_for(Errc::pair_mismatch) == 5 && exit_code_for(Errc::missing_frame) == 3 &&
        exit_code_for(Errc::invalid_argument) == 1 && exit_code_for(Errc::ill_conditioned_slice) == 4);
  std::printf("cbp_stream_test: %d passed, %d failed\n", g_pass, g_fail);
  return g_fail ? 1 : 0;
}
