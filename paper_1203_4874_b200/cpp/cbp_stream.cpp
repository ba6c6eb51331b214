// Stream I/O (PFM / PGM / PPM frames + manifest.json) and the disk-to-disk decode driver,
// behaviour of the reference's proj/core/src/stream_io.cpp and tools/cbp.cpp:130-207.
// Host code only; decode_stream hands whole batches of frames to the device through the
// C ABI (cbp_decode_frames, or cbp_decode_frames_q for quantized streams, which moves
// 1 or 2 bytes per sample to the GPU instead of 4).
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <iostream>
#include <map>
#include <sstream>
#include <variant>

#include "cbp/stream_io.hpp"
#include "cbp_cuda.h"

namespace cbp {
namespace {

namespace fs = std::filesystem;

std::string stem(int index) {
  char buf[32];
  std::snprintf(buf, sizeof(buf), "frame_%06d", index);
  return buf;
}

// --------------------------------------------------------------- flat JSON objects
// The manifest and the sidecars are flat objects (plus one nested object of numbers for the
// stage timings); keys are written sorted with a 2-space indent, the layout of the
// reference's nlohmann::json dump(2).
using JVal = std::variant<std::string, double, long long, unsigned long long, bool>;

std::string num(double v) {
  char buf[64];
  auto r = std::to_chars(buf, buf + sizeof(buf), v);  // shortest round-trip form
  std::string s(buf, r.ptr);
  if (s.find_first_of(".eEn") == std::string::npos) s += ".0";
  return s;
}

std::string quote(const std::string& s) {
  std::string o = "\"";
  for (char c : s) {
    if (c == '"' || c == '\\') o += '\\', o += c;
    else if (c == '\n') o += "\\n";
    else o += c;
  }
  return o + "\"";
}

std::string jval(const JVal& v) {
  if (auto p = std::get_if<std::string>(&v)) return quote(*p);
  if (auto p = std::get_if<double>(&v)) return num(*p);
  if (auto p = std::get_if<long long>(&v)) return std::to_string(*p);
  if (auto p = std::get_if<unsigned long long>(&v)) return std::to_string(*p);
  return std::get<bool>(v) ? "true" : "false";
}

std::string dump_object(const std::map<std::string, std::string>& fields, int indent) {
  const std::string pad(size_t(indent + 2), ' ');
  std::string o = "{\n";
  size_t i = 0;
  for (const auto& [k, v] : fields) o += pad + quote(k) + ": " + v + (++i < fields.size() ? ",\n" : "\n");
  return o + std::string(size_t(indent), ' ') + "}";
}

// parser for a flat object of strings / numbers / booleans / null
struct JsonReader {
  const std::string& s;
  const std::string& name;
  size_t i = 0;
  [[noreturn]] void bad(const std::string& what) {
    fail(Errc::corrupt_manifest, name + ": " + what + " at byte " + std::to_string(i));
  }
  void ws() {
    while (i < s.size() && std::isspace(static_cast<unsigned char>(s[i]))) ++i;
  }
  char peek() {
    ws();
    if (i >= s.size()) bad("unexpected end of input");
    return s[i];
  }
  void expect(char c) {
    if (peek() != c) bad(std::string("expected '") + c + "'");
    ++i;
  }
  std::string str() {
    expect('"');
    std::string o;
    while (true) {
      if (i >= s.size()) bad("unterminated string");
      char c = s[i++];
      if (c == '"') break;
      if (c == '\\') {
        if (i >= s.size()) bad("bad escape");
        char e = s[i++];
        switch (e) {
          case 'n': o += '\n'; break;
          case 't': o += '\t'; break;
          case 'r': o += '\r'; break;
          case 'b': o += '\b'; break;
          case 'f': o += '\f'; break;
          case 'u': {
            if (i + 4 > s.size()) bad("bad escape");
            o += char(std::stoi(s.substr(i, 4), nullptr, 16) & 0x7f);
            i += 4;
            break;
          }
          default: o += e;
        }
      } else {
        o += c;
      }
    }
    return o;
  }
  std::map<std::string, JVal> object() {
    std::map<std::string, JVal> m;
    expect('{');
    if (peek() == '}') {
      ++i;
      return m;
    }
    while (true) {
      std::string k = str();
      expect(':');
      const char c = peek();
      if (c == '"') {
        m[k] = str();
      } else if (c == 't' || c == 'f') {
        const bool v = s.compare(i, 4, "true") == 0;
        if (!v && s.compare(i, 5, "false") != 0) bad("bad literal");
        i += v ? 4 : 5;
        m[k] = v;
      } else if (c == 'n') {
        if (s.compare(i, 4, "null") != 0) bad("bad literal");
        i += 4;
      } else {
        size_t j = i;
        while (j < s.size() && (std::isdigit(static_cast<unsigned char>(s[j])) || std::strchr("+-.eE", s[j]))) ++j;
        const std::string tok = s.substr(i, j - i);
        if (tok.empty()) bad("unexpected character");
        i = j;
        if (tok.find_first_of(".eE") != std::string::npos) {
          m[k] = std::stod(tok);
        } else if (tok[0] == '-') {
          m[k] = std::stoll(tok);
        } else {
          m[k] = std::stoull(tok);
        }
      }
      if (peek() == ',') {
        ++i;
        continue;
      }
      expect('}');
      break;
    }
    ws();
    if (i != s.size()) bad("trailing characters");
    return m;
  }
};

// --------------------------------------------------------------- PFM (FP32)
void write_pfm(const Frame& f, const fs::path& path) {
  const int rows = f.rows(), cols = f.cols(), ch = f.channels();
  std::ofstream out(path, std::ios::binary);
  require(out.good(), Errc::io_failure, "cannot open " + path.string());
  out << (ch == 3 ? "PF" : "Pf") << "\n" << cols << " " << rows << "\n-1.0\n";  // negative scale: little-endian
  std::vector<float> line(size_t(cols) * ch);
  for (int r = rows - 1; r >= 0; --r) {  // bottom row first
    for (int c = 0; c < cols; ++c)
      for (int k = 0; k < ch; ++k) line[size_t(c) * ch + k] = float(f.planes[size_t(k)](r, c));
    out.write(reinterpret_cast<const char*>(line.data()), std::streamsize(line.size() * sizeof(float)));
  }
  require(out.good(), Errc::io_failure, "short write on " + path.string());
}

Frame read_pfm(std::istream& in, const std::string& name) {
  std::string magic;
  int cols = 0, rows = 0;
  double scale = 0.0;
  in >> magic >> cols >> rows >> scale;
  require(in.good() && (magic == "Pf" || magic == "PF"), Errc::format_violation, name + ": bad float map header");
  require(cols > 0 && rows > 0, Errc::format_violation, name + ": bad dimensions");
  require(scale < 0.0, Errc::format_violation, name + ": big-endian float maps unsupported");
  in.get();  // the one whitespace byte that ends the header
  const int ch = magic == "PF" ? 3 : 1;
  Frame f;
  f.planes.assign(size_t(ch), ImagePlane(rows, cols));
  std::vector<float> line(size_t(cols) * ch);
  for (int r = rows - 1; r >= 0; --r) {
    in.read(reinterpret_cast<char*>(line.data()), std::streamsize(line.size() * sizeof(float)));
    require(in.good(), Errc::format_violation, name + ": truncated raster");
    for (int c = 0; c < cols; ++c)
      for (int k = 0; k < ch; ++k) f.planes[size_t(k)](r, c) = line[size_t(c) * ch + k];
  }
  return f;
}

// --------------------------------------------------------------- PGM / PPM (u8, u16)
void write_pnm(const Frame& f, const fs::path& path) {
  const int rows = f.rows(), cols = f.cols(), ch = f.channels();
  const int maxv = f.bit_depth == BitDepth::u8 ? 255 : 65535;
  const int bytes = maxv > 255 ? 2 : 1;
  std::ofstream out(path, std::ios::binary);
  require(out.good(), Errc::io_failure, "cannot open " + path.string());
  out << (ch == 3 ? "P6" : "P5") << "\n" << cols << " " << rows << "\n" << maxv << "\n";
  std::vector<unsigned char> line(size_t(cols) * ch * bytes);
  for (int r = 0; r < rows; ++r) {
    unsigned char* o = line.data();
    for (int c = 0; c < cols; ++c)
      for (int k = 0; k < ch; ++k) {
        const long v = std::clamp<long>(std::lround(f.planes[size_t(k)](r, c) * maxv), 0, maxv);
        if (bytes == 2) *o++ = static_cast<unsigned char>(v >> 8);  // big-endian
        *o++ = static_cast<unsigned char>(v & 0xff);
      }
    out.write(reinterpret_cast<const char*>(line.data()), std::streamsize(line.size()));
  }
  require(out.good(), Errc::io_failure, "short write on " + path.string());
}

// header token; '#' comments run to the end of the line; consumes one trailing whitespace
std::string pnm_token(std::istream& in) {
  int c = in.get();
  while (c != EOF) {
    if (c == '#') {
      while (c != EOF && c != '\n') c = in.get();
    } else if (!std::isspace(c)) {
      break;
    }
    c = in.get();
  }
  std::string tok;
  while (c != EOF && !std::isspace(c)) {
    tok += char(c);
    c = in.get();
  }
  return tok;
}

int pnm_int(std::istream& in, const std::string& name) {
  const std::string tok = pnm_token(in);
  int v = 0;
  auto r = std::from_chars(tok.data(), tok.data() + tok.size(), v);
  if (tok.empty() || r.ec != std::errc() || r.ptr != tok.data() + tok.size())
    fail(Errc::format_violation, name + ": bad header token '" + tok + "'");
  return v;
}

Frame read_pnm(std::istream& in, const std::string& name) {
  const std::string magic = pnm_token(in);
  require(magic == "P5" || magic == "P6", Errc::format_violation, name + ": bad pixmap header");
  const int ch = magic == "P6" ? 3 : 1;
  const int cols = pnm_int(in, name), rows = pnm_int(in, name), maxv = pnm_int(in, name);
  require(cols > 0 && rows > 0, Errc::format_violation, name + ": bad dimensions");
  require(maxv == 255 || maxv == 65535, Errc::format_violation, name + ": unsupported maxval " + std::to_string(maxv));
  const int bytes = maxv > 255 ? 2 : 1;
  Frame f;
  f.bit_depth = maxv == 255 ? BitDepth::u8 : BitDepth::u16;
  f.planes.assign(size_t(ch), ImagePlane(rows, cols));
  std::vector<unsigned char> line(size_t(cols) * ch * bytes);
  for (int r = 0; r < rows; ++r) {
    in.read(reinterpret_cast<char*>(line.data()), std::streamsize(line.size()));
    require(in.good(), Errc::format_violation, name + ": truncated raster");
    const unsigned char* p = line.data();
    for (int c = 0; c < cols; ++c)
      for (int k = 0; k < ch; ++k) {
        int v = *p++;
        if (bytes == 2) v = (v << 8) | *p++;
        f.planes[size_t(k)](r, c) = double(v) / maxv;
      }
  }
  return f;
}

// --------------------------------------------------------------- manifest.json
std::string manifest_json(const StreamManifest& m) {
  std::map<std::string, std::string> f;
  f["version"] = jval(JVal((long long)m.version));
  f["role"] = jval(JVal(std::string(stream_role_name(m.role))));
  f["frame_count"] = jval(JVal((long long)m.frame_count));
  f["width"] = jval(JVal((long long)m.width));
  f["height"] = jval(JVal((long long)m.height));
  f["bit_depth"] = jval(JVal(std::string(bit_depth_name(m.bit_depth))));
  f["pair_id"] = jval(JVal(m.pair_id));
  if (m.kernel_width_hint) f["kernel_width_hint"] = jval(JVal((long long)*m.kernel_width_hint));
  if (m.seed) f["seed"] = jval(JVal((unsigned long long)*m.seed));
  return dump_object(f, 0);
}

long long as_int(const std::map<std::string, JVal>& j, const std::string& key, const std::string& name) {
  auto it = j.find(key);
  if (it == j.end()) fail(Errc::corrupt_manifest, name + ": missing key '" + key + "'");
  if (auto p = std::get_if<long long>(&it->second)) return *p;
  if (auto p = std::get_if<unsigned long long>(&it->second)) return (long long)*p;
  fail(Errc::corrupt_manifest, name + ": key '" + key + "' is not an integer");
}

std::string as_str(const std::map<std::string, JVal>& j, const std::string& key, const std::string& name) {
  auto it = j.find(key);
  if (it == j.end()) fail(Errc::corrupt_manifest, name + ": missing key '" + key + "'");
  if (auto p = std::get_if<std::string>(&it->second)) return *p;
  fail(Errc::corrupt_manifest, name + ": key '" + key + "' is not a string");
}

StreamManifest read_manifest(const fs::path& dir) {
  const fs::path path = dir / "manifest.json";
  std::ifstream in(path, std::ios::binary);
  require(in.good(), Errc::io_failure, "cannot open " + path.string());
  std::stringstream ss;
  ss << in.rdbuf();
  const std::string text = ss.str(), name = path.string();
  JsonReader rd{text, name};
  const auto j = rd.object();
  StreamManifest m;
  m.version = int(as_int(j, "version", name));
  require(m.version == 1, Errc::corrupt_manifest, name + ": unsupported version " + std::to_string(m.version));
  m.role = stream_role_from_name(as_str(j, "role", name));
  m.frame_count = int(as_int(j, "frame_count", name));
  m.width = int(as_int(j, "width", name));
  m.height = int(as_int(j, "height", name));
  m.bit_depth = bit_depth_from_name(as_str(j, "bit_depth", name));
  m.pair_id = as_str(j, "pair_id", name);
  if (j.count("kernel_width_hint")) m.kernel_width_hint = int(as_int(j, "kernel_width_hint", name));
  if (j.count("seed")) {
    const JVal& v = j.at("seed");
    if (auto p = std::get_if<unsigned long long>(&v)) m.seed = *p;
    else fail(Errc::corrupt_manifest, name + ": key 'seed' is not an unsigned integer");
  }
  require(m.frame_count >= 0 && m.width > 0 && m.height > 0, Errc::corrupt_manifest, name + ": bad geometry");
  return m;
}

const char* extension(BitDepth d, int channels) { return d == BitDepth::f32 ? "pfm" : channels == 3 ? "ppm" : "pgm"; }

}  // namespace

const char* stream_role_name(StreamRole r) {
  switch (r) {
    case StreamRole::Latent: return "latent";
    case StreamRole::Public: return "public";
    case StreamRole::Private: return "private";
  }
  fail(Errc::invalid_argument, "bad stream role");
}

StreamRole stream_role_from_name(const std::string& s) {
  if (s == "latent") return StreamRole::Latent;
  if (s == "public") return StreamRole::Public;
  if (s == "private") return StreamRole::Private;
  fail(Errc::corrupt_manifest, "unknown stream role '" + s + "'");
}

void write_stream(const std::vector<Frame>& frames, const StreamManifest& manifest, const fs::path& dir) {
  require(manifest.frame_count == int(frames.size()), Errc::invalid_argument,
          "manifest frame_count disagrees with frame list");
  require(manifest.frame_count > 0, Errc::invalid_argument, "empty stream");
  const int ch = frames.front().channels();
  for (const Frame& f : frames) {
    validate_frame(f);
    require(f.rows() == manifest.height && f.cols() == manifest.width, Errc::invalid_argument,
            "frame dimensions disagree with manifest");
    require(f.channels() == ch, Errc::invalid_argument, "mixed channel counts in stream");
    require(f.bit_depth == manifest.bit_depth, Errc::invalid_argument, "frame bit depth disagrees with manifest");
  }
  std::error_code ec;
  fs::create_directories(dir, ec);
  require(!ec, Errc::io_failure, "cannot create " + dir.string() + ": " + ec.message());
  const char* ext = extension(manifest.bit_depth, ch);
  for (int i = 0; i < manifest.frame_count; ++i) {
    const fs::path path = dir / (stem(i) + "." + ext);
    if (manifest.bit_depth == BitDepth::f32) write_pfm(frames[size_t(i)], path);
    else write_pnm(frames[size_t(i)], path);
  }
  const fs::path mpath = dir / "manifest.json";
  std::ofstream out(mpath, std::ios::binary);
  require(out.good(), Errc::io_failure, "cannot open " + mpath.string());
  out << manifest_json(manifest) << "\n";
  require(out.good(), Errc::io_failure, "short write on " + mpath.string());
}

std::pair<std::vector<Frame>, StreamManifest> read_stream(const fs::path& dir) {
  const StreamManifest m = read_manifest(dir);
  std::vector<Frame> frames;
  frames.reserve(size_t(m.frame_count));
  for (int i = 0; i < m.frame_count; ++i) {
    fs::path path = dir / (stem(i) + (m.bit_depth == BitDepth::f32 ? ".pfm" : ".pgm"));
    if (m.bit_depth != BitDepth::f32 && !fs::exists(path)) path = dir / (stem(i) + ".ppm");
    require(fs::exists(path), Errc::missing_frame, "missing " + (dir / (stem(i) + ".*")).string());
    std::ifstream in(path, std::ios::binary);
    require(in.good(), Errc::io_failure, "cannot open " + path.string());
    Frame f = m.bit_depth == BitDepth::f32 ? read_pfm(in, path.string()) : read_pnm(in, path.string());
    require(f.rows() == m.height && f.cols() == m.width, Errc::format_violation,
            path.string() + ": dimensions disagree with manifest");
    if (m.bit_depth != BitDepth::f32)
      require(f.bit_depth == m.bit_depth, Errc::format_violation, path.string() + ": sample depth disagrees with manifest");
    f.bit_depth = m.bit_depth;
    f.index = i;
    if (i > 0)
      require(f.channels() == frames.front().channels(), Errc::format_violation,
              path.string() + ": mixed channel counts in stream");
    frames.push_back(std::move(f));
  }
  return {std::move(frames), m};
}

std::vector<BlurredPair> pair_streams(const fs::path& public_dir, const fs::path& private_dir) {
  auto [a, am] = read_stream(public_dir);
  auto [b, bm] = read_stream(private_dir);
  // either role order pairs; the directory order decides which plays public when decoding
  const bool ok = (am.role == StreamRole::Public && bm.role == StreamRole::Private) ||
                  (am.role == StreamRole::Private && bm.role == StreamRole::Public);
  require(ok, Errc::pair_mismatch, "streams do not form a public/private pair");
  require(!am.pair_id.empty() && am.pair_id == bm.pair_id, Errc::pair_mismatch,
          "pair id mismatch: '" + am.pair_id + "' vs '" + bm.pair_id + "'");
  require(am.frame_count == bm.frame_count, Errc::pair_mismatch, "frame count mismatch");
  require(am.width == bm.width && am.height == bm.height, Errc::pair_mismatch, "frame geometry mismatch");
  require(am.bit_depth == bm.bit_depth, Errc::pair_mismatch, "bit depth mismatch");
  std::optional<int> hint;
  if (am.kernel_width_hint && bm.kernel_width_hint && *am.kernel_width_hint == *bm.kernel_width_hint)
    hint = am.kernel_width_hint;
  std::vector<BlurredPair> pairs(a.size());
  for (size_t i = 0; i < a.size(); ++i) {
    require(a[i].channels() == b[i].channels(), Errc::pair_mismatch, "channel count mismatch");
    pairs[i].public_frame = std::move(a[i]);
    pairs[i].private_frame = std::move(b[i]);
    pairs[i].kernel_width_hint = hint;
    pairs[i].pair_id = am.pair_id;
  }
  return pairs;
}

int exit_code_for(Errc code) {  // tools/cbp.cpp:30-46
  switch (code) {
    case Errc::invalid_argument: return 1;
    case Errc::coprimality_failure: return 2;
    case Errc::io_failure:
    case Errc::corrupt_manifest:
    case Errc::missing_frame:
    case Errc::format_violation: return 3;
    case Errc::pair_mismatch: return 5;
    default: return 4;
  }
}

namespace {

struct StreamCtx {
  cbp_ctx* ptr = nullptr;
  StreamCtx() {
    const int st = cbp_create(0, &ptr);
    if (st) throw std::runtime_error(std::string(cbp_errc_name(st)) + ": no usable CUDA device (no CPU fallback)");
  }
  ~StreamCtx() { cbp_destroy(ptr); }
};

void ck(cbp_ctx* c, int st) {
  if (!st) return;
  const std::string msg = cbp_last_error(c);
  if (st >= 1 && st <= 18) throw Error(Errc(st - 1), msg, true);
  throw std::runtime_error(msg);
}

}  // namespace

int decode_stream(const DecodeStreamOptions& o) {  // tools/cbp.cpp:130-207
  std::vector<BlurredPair> pairs = pair_streams(o.pub, o.prv);
  require(!pairs.empty(), Errc::invalid_argument, "streams have no frames");
  const int n = int(pairs.size());
  const int ch = pairs[0].public_frame.channels(), rows = pairs[0].public_frame.rows(),
            cols = pairs[0].public_frame.cols();
  const BitDepth depth = pairs[0].public_frame.bit_depth;
  const int bits = bit_depth_bits(depth);
  for (const BlurredPair& p : pairs) {  // decoder.cpp:19-29 per frame
    validate_frame(p.public_frame);
    validate_frame(p.private_frame);
    if (p.kernel_width_hint)
      require(*p.kernel_width_hint >= 1 && *p.kernel_width_hint % 2 == 1, Errc::invalid_argument,
              "kernel width hint must be odd and >= 1");
  }
  cbp_decode_cfg cfg;
  cbp_decode_cfg_default(&cfg);
  cfg.tau = o.tau;
  cfg.has_epsilon = o.epsilon ? 1 : 0;
  cfg.epsilon = o.epsilon.value_or(0.0);
  cfg.trust_hint = o.trust_hint;
  cfg.search_min = o.width_min;
  cfg.search_max = o.width_max;

  thread_local StreamCtx sc;
  cbp_ctx* c = sc.ptr;
  const int B = std::max(1, std::min(o.batch, n));
  const size_t plane = size_t(rows) * cols, frame = plane * ch;
  const size_t esz = bits == 0 ? sizeof(float) : bits == 8 ? 1 : 2;
  void *dpub = nullptr, *dprv = nullptr, *dout = nullptr;
  ck(c, cbp_device_alloc(c, esz * frame * B, &dpub));
  ck(c, cbp_device_alloc(c, esz * frame * B, &dprv));
  ck(c, cbp_device_alloc(c, sizeof(float) * frame * B, &dout));
  struct Free {
    cbp_ctx* c;
    void *a, *b, *d;
    ~Free() {
      cbp_device_free(c, a);
      cbp_device_free(c, b);
      cbp_device_free(c, d);
    }
  } guard{c, dpub, dprv, dout};
  std::vector<unsigned char> hp(esz * frame * B), hq(esz * frame * B);
  std::vector<float> hout(frame * B);
  std::vector<cbp_decode_info> info(static_cast<size_t>(B));
  std::vector<Frame> latents(static_cast<size_t>(n));
  std::vector<cbp_decode_info> all(static_cast<size_t>(n));
  const double maxv = bits ? double((1u << bits) - 1) : 1.0;
  auto put = [&](const Frame& f, unsigned char* dst) {  // row-major [ch][rows][cols]
    for (int k = 0; k < ch; ++k)
      for (int r = 0; r < rows; ++r)
        for (int x = 0; x < cols; ++x) {
          const double v = f.planes[size_t(k)](r, x);
          const size_t at = size_t(k) * plane + size_t(r) * cols + x;
          if (bits == 0) reinterpret_cast<float*>(dst)[at] = float(v);
          else if (bits == 8) dst[at] = static_cast<unsigned char>(std::lround(v * maxv));
          else reinterpret_cast<uint16_t*>(dst)[at] = static_cast<uint16_t>(std::lround(v * maxv));
        }
  };
  for (int f0 = 0; f0 < n; f0 += B) {
    const int nb = std::min(B, n - f0);
    std::vector<int> hints(static_cast<size_t>(nb));
    for (int j = 0; j < nb; ++j) {
      put(pairs[size_t(f0 + j)].public_frame, hp.data() + esz * frame * j);
      put(pairs[size_t(f0 + j)].private_frame, hq.data() + esz * frame * j);
      hints[size_t(j)] = pairs[size_t(f0 + j)].kernel_width_hint.value_or(0);
    }
    ck(c, cbp_copy_to_device(c, dpub, hp.data(), esz * frame * nb));
    ck(c, cbp_copy_to_device(c, dprv, hq.data(), esz * frame * nb));
    int st;
    if (bits == 0)
      st = cbp_decode_frames(c, static_cast<float*>(dpub), static_cast<float*>(dprv), nb, ch, rows, cols, cols,
                             hints.data(), &cfg, static_cast<float*>(dout), cols, info.data(), nullptr);
    else
      st = cbp_decode_frames_q(c, dpub, dprv, bits, nb, ch, rows, cols, cols, hints.data(), &cfg,
                               static_cast<float*>(dout), cols, info.data(), nullptr);
    ck(c, st);  // first failing frame of the batch, reference message
    ck(c, cbp_copy_to_host(c, hout.data(), dout, sizeof(float) * frame * nb));
    for (int j = 0; j < nb; ++j) {
      const cbp_decode_info& inf = info[size_t(j)];
      const int t = inf.width_used, lr = rows - t + 1, lc = cols - t + 1;
      Frame L;
      L.bit_depth = BitDepth::f32;
      L.index = f0 + j;
      for (int k = 0; k < ch; ++k) {
        ImagePlane p(lr, lc);
        const float* src = hout.data() + frame * j + plane * k;
        for (int r = 0; r < lr; ++r)
          for (int x = 0; x < lc; ++x) p(r, x) = src[size_t(r) * cols + x];
        L.planes.push_back(std::move(p));
      }
      latents[size_t(f0 + j)] = std::move(L);
      all[size_t(f0 + j)] = inf;
    }
  }
  StreamManifest m;
  m.role = StreamRole::Latent;
  m.frame_count = n;
  m.width = latents.front().cols();
  m.height = latents.front().rows();
  m.bit_depth = BitDepth::f32;
  m.pair_id = pairs.front().pair_id;
  write_stream(latents, m, o.out);

  bool within = true;
  for (int i = 0; i < n; ++i) {
    const cbp_decode_info& d = all[size_t(i)];
    std::map<std::string, std::string> st;
    st["polynomial_evaluation_ms"] = num(d.stage_ms[0]);
    st["kernel_degree_estimation_ms"] = num(d.stage_ms[1]);
    st["kernel_estimation_1d_ms"] = num(d.stage_ms[2]);
    st["kernel_estimation_2d_fft_ms"] = num(d.stage_ms[3]);
    st["total_ms"] = num(d.stage_ms[4]);
    std::map<std::string, std::string> j;
    j["width_used"] = std::to_string(d.width_used);
    j["width_clamped"] = d.width_clamped ? "true" : "false";
    j["validation_residual"] = num(d.validation_residual);
    j["stage_timings"] = dump_object(st, 2);
    const fs::path side = o.out / (stem(i) + ".json");
    std::ofstream sf(side, std::ios::binary);
    require(sf.good(), Errc::io_failure, "cannot open " + side.string());
    sf << dump_object(j, 0) << "\n";
    require(sf.good(), Errc::io_failure, "short write on " + side.string());
    if (o.verbose)
      std::cout << stem(i) << ": width " << d.width_used << ", residual " << d.validation_residual << "\n";
    if (!(d.validation_residual <= o.max_residual)) within = false;
  }
  if (!within) {
    std::cerr << "error: validation residual above " << o.max_residual << "\n";
    return 4;
  }
  return 0;
}

}  // namespace cbp
