// cbp-decode: the `cbp decode` command (reference tools/cbp.cpp:85-99, 130-207) over the
// B200 library. Same options and exit codes (0 ok, 1 invalid argument, 3 I/O / format,
// 4 pipeline failure or residual above --max-residual, 5 pair mismatch).
#include <cstdlib>
#include <cstring>
#include <iostream>
#include <string>

#include "cbp/stream_io.hpp"

namespace {

void usage() {
  std::cerr << "usage: cbp-decode --public DIR --private DIR --out DIR [--tau X] [--epsilon X] [--trust-hint]\n"
               "                  [--max-residual X] [--width-min N] [--width-max N] [--workers N] [--batch N]\n";
}

}  // namespace

int main(int argc, char** argv) {
  cbp::DecodeStreamOptions o;
  bool have_pub = false, have_prv = false, have_out = false;
  for (int i = 1; i < argc; ++i) {
    const std::string a = argv[i];
    auto value = [&]() -> const char* {
      if (i + 1 >= argc) {
        std::cerr << "error: " << a << " needs a value\n";
        usage();
        std::exit(1);
      }
      return argv[++i];
    };
    try {
      if (a == "--public") o.pub = value(), have_pub = true;
      else if (a == "--private") o.prv = value(), have_prv = true;
      else if (a == "--out") o.out = value(), have_out = true;
      else if (a == "--tau") o.tau = std::stod(value());
      else if (a == "--epsilon") o.epsilon = std::stod(value());
      else if (a == "--trust-hint") o.trust_hint = true;
      else if (a == "--max-residual") o.max_residual = std::stod(value());
      else if (a == "--width-min") o.width_min = std::stoi(value());
      else if (a == "--width-max") o.width_max = std::stoi(value());
      else if (a == "--workers") (void)std::stoi(value());  // host threads: batching replaces them
      else if (a == "--batch") o.batch = std::stoi(value());
      else if (a == "-h" || a == "--help") return usage(), 0;
      else {
        std::cerr << "error: unknown option " << a << "\n";
        usage();
        return 1;
      }
    } catch (const std::exception&) {
      std::cerr << "error: bad value for " << a << "\n";
      return 1;
    }
  }
  if (!have_pub || !have_prv || !have_out) {
    usage();
    return 1;
  }
  try {
    return cbp::decode_stream(o);
  } catch (const cbp::Error& e) {
    std::cerr << "error: " << e.what() << "\n";
    return cbp::exit_code_for(e.code());
  } catch (const std::exception& e) {
    std::cerr << "error: " << e.what() << "\n";
    return 4;
  }
}
