// cbp stream I/O and the disk-to-disk decode driver for the B200 build.
//
// Same interface as the reference's proj/core/include/cbp/stream_io.hpp: a stream is a
// directory with manifest.json and frame_000000.{pfm,pgm,ppm}, ... (PFM little-endian
// FP32 rows bottom-up; PGM/PPM maxval 255 or 65535, 16-bit big-endian, rows top-down).
// decode_stream() is the `cbp decode` command of tools/cbp.cpp:130-207 as a library call:
// pair the streams, decode every frame on the GPU (kernel recovery per frame, batched),
// write the latent stream and one JSON sidecar per frame, return the CLI exit code.
#pragma once

#include <cstdint>
#include <filesystem>
#include <optional>
#include <string>
#include <utility>
#include <vector>

#include "cbp/cbp.hpp"

namespace cbp {

enum class StreamRole { Latent, Public, Private };

const char* stream_role_name(StreamRole r);
StreamRole stream_role_from_name(const std::string& s);

struct StreamManifest {
  int version = 1;
  StreamRole role = StreamRole::Latent;
  int frame_count = 0;
  int width = 0;   // columns
  int height = 0;  // rows
  BitDepth bit_depth = BitDepth::f32;
  std::string pair_id;
  std::optional<int> kernel_width_hint;
  std::optional<std::uint64_t> seed;
};

void write_stream(const std::vector<Frame>& frames, const StreamManifest& manifest,
                  const std::filesystem::path& dir);
std::pair<std::vector<Frame>, StreamManifest> read_stream(const std::filesystem::path& dir);

// Per-index public/private pairs; roles may come in either order, pair_id, frame count,
// geometry and bit depth must agree; the width hint survives only if both manifests agree.
std::vector<BlurredPair> pair_streams(const std::filesystem::path& public_dir,
                                      const std::filesystem::path& private_dir);

// `cbp decode` options (tools/cbp.cpp:117-128) and driver. Returns the CLI's exit status:
// 0 ok, 4 when a frame's validation residual exceeds max_residual; errors are thrown as
// cbp::Error (exit_code_for maps them like tools/cbp.cpp:30-46).
struct DecodeStreamOptions {
  std::filesystem::path pub, prv, out;
  double tau = 1e-6;
  std::optional<double> epsilon;
  bool trust_hint = false;
  double max_residual = 1e-2;
  int width_min = 9;
  int width_max = 25;
  int batch = 16;       // frames per device batch
  bool verbose = true;  // per-frame "frame_000000: width 11, residual ..." lines on stdout
};
int decode_stream(const DecodeStreamOptions& o);
int exit_code_for(Errc code);

}  // namespace cbp
