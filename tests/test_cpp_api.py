"""The C++ host layer (include/cbp/*.hpp, the reference's cbp:: API over the C ABI):
it builds and links here; on a GPU box its test program (tests/cpp/cbp_api_test.cpp,
mirroring the reference's unit tests) passes."""
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_1203_4874_b200", "_lib")


def test_cpp_shim_built_and_linked():
    for f in ("libcbp.so", "libcbp_cuda.so", "cbp_api_test", "cbp_stream_test", "cbp-decode"):
        assert os.path.exists(os.path.join(LIB, f)), f
    out = subprocess.run(["nm", "-DC", "--defined-only", os.path.join(LIB, "libcbp.so")], capture_output=True,
                         text=True, check=True).stdout
    for sym in ("cbp::decode_frame(", "cbp::spectral_deblur(", "cbp::estimate_kernel_width(",
                "cbp::sample_cofactors(", "cbp::complete_to_spectrum(", "cbp::resolve_scales(",
                "cbp::assemble_kernel(", "cbp::validate_pair(", "cbp::encode_frame(",
                "cbp::generate_coprime_pair(", "cbp::cofactor_null_solve(", "cbp::axis_roots_dft(",
                "cbp::read_stream(", "cbp::write_stream(", "cbp::pair_streams(", "cbp::decode_stream("):
        assert sym in out, sym


def test_stream_io_suite():
    """PFM/PGM/PPM + manifest.json I/O and pair_streams (stream_io_test.cpp behaviours, byte-exact
    persistence): host code, no GPU."""
    r = subprocess.run([os.path.join(LIB, "cbp_stream_test")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


def test_decode_cli_usage_errors():
    """cbp-decode argument errors exit with status 1 before touching the GPU."""
    r = subprocess.run([os.path.join(LIB, "cbp-decode"), "--public", "a"], capture_output=True, text=True)
    assert r.returncode == 1 and "usage" in r.stderr
    r = subprocess.run([os.path.join(LIB, "cbp-decode"), "--bogus"], capture_output=True, text=True)
    assert r.returncode == 1


@pytest.mark.gpu
def test_cpp_api_suite_on_gpu():
    r = subprocess.run([os.path.join(LIB, "cbp_api_test")], capture_output=True, text=True, timeout=600)
    print(r.stdout, r.stderr)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "0 failed" in r.stdout


@pytest.mark.gpu
def test_decode_cli_on_gpu(tmp_path):
    """The `cbp decode` contract (tools/cbp.cpp:130-207) through the cbp-decode binary: u16
    RGB streams in, latent stream + sidecars out, exit codes 0 / 4 / 5 / 3."""
    subprocess.run([os.path.join(LIB, "cbp_api_test"), "--write-streams", str(tmp_path)], check=True, timeout=300)
    cli = os.path.join(LIB, "cbp-decode")
    base = [cli, "--public", str(tmp_path / "public"), "--private", str(tmp_path / "private"),
            "--width-min", "3", "--width-max", "9", "--trust-hint"]  # u16: the manifest hint carries the width
    r = subprocess.run(base + ["--out", str(tmp_path / "latent")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stdout + r.stderr
    assert r.stdout.count("width 5, residual") == 3
    assert sorted(p.name for p in (tmp_path / "latent").iterdir()) == [
        "frame_000000.json", "frame_000000.pfm", "frame_000001.json", "frame_000001.pfm",
        "frame_000002.json", "frame_000002.pfm", "manifest.json"]
    r = subprocess.run(base + ["--out", str(tmp_path / "l2"), "--max-residual", "1e-30"], capture_output=True,
                       text=True, timeout=300)
    assert r.returncode == 4 and "validation residual above" in r.stderr
    r = subprocess.run([cli, "--public", str(tmp_path / "public"), "--private", str(tmp_path / "public"),
                        "--out", str(tmp_path / "l3")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 5 and "PairMismatch" in r.stderr
    r = subprocess.run([cli, "--public", str(tmp_path / "nope"), "--private", str(tmp_path / "private"),
                        "--out", str(tmp_path / "l4")], capture_output=True, text=True, timeout=300)
    assert r.returncode == 3
