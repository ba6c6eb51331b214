"""The C++ host layer (include/cbp/*.hpp, the reference's cbp:: API over the C ABI):
it builds and links here; on a GPU box its test program (tests/cpp/cbp_api_test.cpp,
mirroring the reference's unit tests) passes."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1203_4874_b200", "_lib")


def test_cpp_shim_built_and_linked():
    for f in ("libcbp.so", "libcbp_cuda.so", "cbp_api_test"):
        assert os.path.exists(os.path.join(LIB, f)), f
    out = subprocess.run(["nm", "-DC", "--defined-only", os.path.join(LIB, "libcbp.so")], capture_output=True,
                         text=True, check=True).stdout
    for sym in ("cbp::decode_frame(", "cbp::spectral_deblur(", "cbp::estimate_kernel_width(",
                "cbp::sample_cofactors(", "cbp::complete_to_spectrum(", "cbp::resolve_scales(",
                "cbp::assemble_kernel(", "cbp::validate_pair(", "cbp::encode_frame(",
                "cbp::generate_coprime_pair(", "cbp::cofactor_null_solve(", "cbp::axis_roots_dft("):
        assert sym in out, sym


@pytest.mark.gpu
def test_cpp_api_suite_on_gpu():
    r = subprocess.run([os.path.join(LIB, "cbp_api_test")], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout
