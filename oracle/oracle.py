"""CBP ORACLE — TEST INFRASTRUCTURE ONLY.

ctypes front end of ``oracle/_build/libcbp_oracle.so``: the FP64 CPU restatement of
the reference CBP decryption path (reference ``proj/core/src/decoder.cpp``,
``poly.cpp``, ``fft.cpp``, ``image.cpp``, ``encoder.cpp``, ``synth.cpp``).
Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s CPU baseline leg may
import this module, and only as the checker / timed CPU baseline. The CUDA product
path never imports it.

Parity status: the reference cannot be compiled in this image (Eigen3 and FFTW3 are
absent), so this restatement is pinned by porting the reference's own known-answer
tests (tests/test_oracle_kat.py) and by an independent numpy/LAPACK restatement
(oracle/np_ref.py, tests/test_oracle_vs_numpy.py).

Arrays are row-major numpy; index (m, n) is (z1 power, z2 power) as in the reference
(types.hpp:15-17).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(HERE, "_build", "libcbp_oracle.so")

ERRC_NAMES = [
    "InvalidArgument", "NonUnitSamplePoint", "DegenerateInput", "IllConditioned",
    "CoprimalityFailure", "FrameTooSmall", "RangeExceeded", "NotQuantized",
    "InconsistentAxes", "IllConditionedSlice", "DegenerateScales", "NonRealKernel",
    "DimMismatch", "IoFailure", "CorruptManifest", "MissingFrame", "FormatViolation",
    "PairMismatch",
]


class OracleError(RuntimeError):
    """Mirror of cbp::Error: ``code`` is the Errc name, message is "<Name>: detail"."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status
        self.code = ERRC_NAMES[status - 1] if 1 <= status <= len(ERRC_NAMES) else "Unknown"


def build() -> str:
    subprocess.run(["make", "-s", "-C", HERE], check=True)
    return LIB_PATH


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        _lib = C.CDLL(LIB_PATH)
        _lib.orc_last_error.restype = C.c_char_p
        _lib.orc_frame_seed.restype = C.c_uint64
        _lib.orc_frame_seed.argtypes = [C.c_uint64, C.c_int]
        _lib.orc_splitmix64.restype = C.c_uint64
        _lib.orc_splitmix64.argtypes = [C.c_uint64]
        _lib.orc_random_frame.argtypes = [C.c_int, C.c_int, C.c_int, C.c_uint64, C.c_void_p]
        _lib.orc_random_mat.argtypes = [C.c_int, C.c_int, C.c_uint64, C.c_double, C.c_double, C.c_void_p]
        _lib.orc_generate_coprime_pair.argtypes = [C.c_int, C.c_uint64, C.c_int, C.c_double, C.c_int,
                                                   C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.orc_psnr.restype = C.c_double
        for name in ("orc_numerical_singularity", "orc_cofactor_null_solve", "orc_spectral_deblur",
                     "orc_estimate_kernel_width", "orc_sample_cofactors", "orc_assemble_kernel",
                     "orc_coprimality_check", "orc_homogeneous_lsq"):
            getattr(_lib, name).restype = C.c_int
        _lib.orc_numerical_singularity.argtypes = [C.c_void_p, C.c_int, C.c_double, C.c_void_p, C.c_void_p]
        _lib.orc_cofactor_null_solve.argtypes = [C.c_void_p, C.c_int, C.c_void_p, C.c_int, C.c_int,
                                                 C.c_double, C.c_void_p, C.c_void_p, C.c_void_p]
        _lib.orc_spectral_deblur.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_void_p, C.c_int,
                                             C.c_double, C.c_void_p]
        _lib.orc_estimate_kernel_width.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                                   C.c_int, C.c_int, C.c_double, C.c_void_p, C.c_void_p]
        _lib.orc_sample_cofactors.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                              C.c_int, C.c_double, C.c_void_p, C.c_void_p]
        _lib.orc_assemble_kernel.argtypes = [C.c_void_p] * 4 + [C.c_int, C.c_double, C.c_double, C.c_void_p]
        _lib.orc_coprimality_check.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_void_p]
        _lib.orc_bench_frames.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int, C.c_int, C.c_int,
                                          C.c_void_p, C.c_void_p, C.c_int, C.c_double, C.c_void_p,
                                          C.c_int, C.c_void_p]
    return _lib


def _check(status: int):
    if status != 0:
        raise OracleError(status, lib().orc_last_error().decode())


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.complex128)


# ----------------------------------------------------------------- synth / rng
def frame_seed(stream_seed: int, index: int) -> int:
    return int(lib().orc_frame_seed(stream_seed, index))


def splitmix64(x: int) -> int:
    return int(lib().orc_splitmix64(x))


def random_frame(rows: int, cols: int, channels: int, seed: int) -> np.ndarray:
    """synth.cpp:12-22 -> (channels, rows, cols) float64."""
    out = np.empty((channels, rows, cols), np.float64)
    _check(lib().orc_random_frame(rows, cols, channels, seed, _p(out)))
    return out


def random_mat(rows: int, cols: int, seed: int, lo: float = 0.0, hi: float = 1.0) -> np.ndarray:
    """tests/support.hpp:31-39 (libstdc++ uniform_real_distribution)."""
    out = np.empty((rows, cols), np.float64)
    _check(lib().orc_random_mat(rows, cols, seed, lo, hi, _p(out)))
    return out


# -------------------------------------------------------------------- encoder
@dataclass
class CoprimePair:
    k1: np.ndarray
    k2: np.ndarray
    coprimality_margin: float
    seed: int

    @property
    def width(self) -> int:
        return self.k1.shape[0]


def generate_coprime_pair(width: int, seed: int, max_retries: int = 16,
                          margin_threshold: float = 1e-6, trials: int = 4) -> CoprimePair:
    k1 = np.empty((width, width)); k2 = np.empty((width, width)); m = np.zeros(1)
    _check(lib().orc_generate_coprime_pair(width, seed, max_retries, margin_threshold, trials,
                                           _p(k1), _p(k2), _p(m)))
    return CoprimePair(k1, k2, float(m[0]), seed)


def coprimality_check(k1, k2, trials: int = 4) -> float:
    k1 = _f64(k1); k2 = _f64(k2); m = np.zeros(1)
    _check(lib().orc_coprimality_check(_p(k1), _p(k2), k1.shape[0], trials, _p(m)))
    return float(m[0])


def conv2_full(a, b) -> np.ndarray:
    a = _f64(a); b = _f64(b)
    out = np.empty((a.shape[0] + b.shape[0] - 1, a.shape[1] + b.shape[1] - 1))
    _check(lib().orc_conv2_full(_p(a), a.shape[0], a.shape[1], _p(b), b.shape[0], b.shape[1], _p(out)))
    return out


def encode_frame(latent, k1, k2):
    """encoder.cpp:83-103 -> (public, private), each (channels, rows+t-1, cols+t-1)."""
    lat = _f64(latent)
    if lat.ndim == 2:
        lat = lat[None]
    k1 = _f64(k1); k2 = _f64(k2); t = k1.shape[0]
    ch, r, c = lat.shape
    pub = np.empty((ch, r + t - 1, c + t - 1)); prv = np.empty_like(pub)
    _check(lib().orc_encode_frame(_p(lat), ch, r, c, _p(k1), _p(k2), t, _p(pub), _p(prv)))
    return pub, prv


def quantize(planes, bits: int) -> np.ndarray:
    x = _f64(planes).copy()
    if x.ndim == 2:
        x = x[None]
    _check(lib().orc_quantize(_p(x), x.shape[0], x.shape[1], x.shape[2], bits))
    return x


def degrade_bits(planes, bits: int, drop: int) -> np.ndarray:
    """encoder.cpp:124-139 on frames quantized to `bits` (values k / (2^bits - 1))."""
    x = _f64(planes).copy()
    if x.ndim == 2:
        x = x[None]
    _check(lib().orc_degrade_bits(_p(x), x.shape[0], x.shape[1], x.shape[2], bits, drop))
    return x


# ----------------------------------------------------------------------- poly
def bezout_leading_block(p, q, size: int) -> np.ndarray:
    p = _c128(p); q = _c128(q)
    out = np.empty((size, size), np.complex128)
    _check(lib().orc_bezout_leading_block(_p(p), len(p), _p(q), len(q), size, _p(out)))
    return out


def numerical_singularity(m, tau: float):
    m = _c128(m); ratio = np.zeros(1); sing = np.zeros(1, np.int32)
    _check(lib().orc_numerical_singularity(_p(m), m.shape[0], tau, _p(ratio), _p(sing)))
    return bool(sing[0]), float(ratio[0])


def svd(a):
    a = _c128(a); n = a.shape[1]
    sv = np.empty(n); v = np.empty((n, n), np.complex128)
    _check(lib().orc_svd(_p(a), a.shape[0], a.shape[1], _p(sv), _p(v)))
    return sv, v


def cofactor_null_solve(p, q, t: int, gap_threshold: float = 1e-9):
    p = _c128(p); q = _c128(q)
    k1 = np.empty(t, np.complex128); k2 = np.empty(t, np.complex128); gap = np.zeros(1)
    _check(lib().orc_cofactor_null_solve(_p(p), len(p), _p(q), len(q), t, gap_threshold,
                                         _p(k1), _p(k2), _p(gap)))
    return k1, k2, float(gap[0])


def homogeneous_lsq(a) -> np.ndarray:
    a = _c128(a); x = np.empty(a.shape[1], np.complex128)
    _check(lib().orc_homogeneous_lsq(_p(a), a.shape[0], a.shape[1], _p(x)))
    return x


def sylvester_matrix(p, q) -> np.ndarray:
    p = _c128(p); q = _c128(q); n = len(p) + len(q) - 2
    out = np.empty((n, n), np.complex128)
    _check(lib().orc_sylvester_matrix(_p(p), len(p), _p(q), len(q), _p(out)))
    return out


def numerical_degree(p, rel_tol: float = 1e-12) -> int:
    p = _c128(p)
    return int(lib().orc_numerical_degree(_p(p), len(p), C.c_double(rel_tol)))


# ------------------------------------------------------------------------ fft
def fft2(x, inverse: bool = False) -> np.ndarray:
    x = _c128(x); out = np.empty_like(x)
    _check(lib().orc_fft2(_p(x), x.shape[0], x.shape[1], int(inverse), _p(out)))
    return out


def ifft2(x) -> np.ndarray:
    return fft2(x, inverse=True)


def axis_roots_dft(plane, axis: int, t: int) -> np.ndarray:
    """fft.cpp:197-213. axis 0 = Z1 (t x N, row i = slice), 1 = Z2 (M x t, column i)."""
    plane = _f64(plane); M, N = plane.shape
    out = np.empty((t, N) if axis == 0 else (M, t), np.complex128)
    _check(lib().orc_axis_roots_dft(_p(plane), M, N, axis, t, _p(out)))
    return out


def axis_spectrum_half(plane, axis: int) -> np.ndarray:
    plane = _f64(plane); M, N = plane.shape
    out = np.empty((M // 2 + 1, N) if axis == 0 else (M, N // 2 + 1), np.complex128)
    _check(lib().orc_axis_spectrum_half(_p(plane), M, N, axis, _p(out)))
    return out


def friendly_size(n: int) -> int:
    r = lib().orc_friendly_size(n)
    if r < 0:
        _check(-r)
    return r


def luma(planes) -> np.ndarray:
    x = _f64(planes)
    if x.ndim == 2:
        x = x[None]
    out = np.empty(x.shape[1:])
    _check(lib().orc_luma(_p(x), x.shape[0], x.shape[1], x.shape[2], _p(out)))
    return out


# -------------------------------------------------------------------- decoder
class DecodeCfg(C.Structure):
    """Mirror of DecodeConfig (decoder.hpp:10-20) and of cbp_decode_cfg."""
    _fields_ = [("search_min", C.c_int), ("search_max", C.c_int), ("tau", C.c_double),
                ("has_epsilon", C.c_int), ("epsilon", C.c_double), ("gap_threshold", C.c_double),
                ("trust_hint", C.c_int), ("max_imag_energy", C.c_double),
                ("negative_weight_tol", C.c_double), ("validate", C.c_int)]


def make_cfg(search_min=9, search_max=25, tau=1e-6, epsilon=None, gap_threshold=1e-9,
             trust_hint=False, max_imag_energy=0.01, negative_weight_tol=0.01, validate=True) -> DecodeCfg:
    return DecodeCfg(search_min, search_max, tau, int(epsilon is not None),
                     0.0 if epsilon is None else float(epsilon), gap_threshold, int(trust_hint),
                     max_imag_energy, negative_weight_tol, int(validate))


class DecodeInfo(C.Structure):
    _fields_ = [("width_used", C.c_int), ("width_clamped", C.c_int),
                ("validation_residual", C.c_double), ("epsilon_used", C.c_double),
                ("stage_ms", C.c_double * 5)]


@dataclass
class DecodedFrame:
    latent: np.ndarray          # (channels, M, N)
    kernel: np.ndarray          # (t, t)
    width_used: int
    width_clamped: bool
    validation_residual: float
    epsilon_used: float
    stage_ms: list = field(default_factory=list)


def _planes(x) -> np.ndarray:
    x = _f64(x)
    return x[None] if x.ndim == 2 else x


def estimate_kernel_width(pub, prv, search_min: int, search_max: int, tau: float):
    pub = _planes(pub); prv = _planes(prv); ch, r, c = pub.shape
    w = np.zeros(1, np.int32); cl = np.zeros(1, np.int32)
    _check(lib().orc_estimate_kernel_width(_p(pub), _p(prv), ch, r, c, search_min, search_max, tau,
                                           _p(w), _p(cl)))
    return int(w[0]), bool(cl[0])


def sample_cofactors(pub, prv, width: int, axis: int, gap_threshold: float = 1e-9):
    pub = _planes(pub); prv = _planes(prv); ch, r, c = pub.shape
    vals = np.empty((width, width), np.complex128); gaps = np.empty(width)
    _check(lib().orc_sample_cofactors(_p(pub), _p(prv), ch, r, c, width, axis, gap_threshold,
                                      _p(vals), _p(gaps)))
    return vals, gaps


def complete_to_spectrum(values, axis: int) -> np.ndarray:
    v = _c128(values); t = v.shape[0]; out = np.empty_like(v)
    _check(lib().orc_complete_to_spectrum(_p(v), t, axis, _p(out)))
    return out


def resolve_scales(a_values, b_values):
    a = _c128(a_values); b = _c128(b_values); t = a.shape[0]
    lam = np.empty(t, np.complex128); mu = np.empty(t, np.complex128); res = np.zeros(1)
    _check(lib().orc_resolve_scales(_p(a), _p(b), t, _p(lam), _p(mu), _p(res)))
    return lam, mu, float(res[0])


def assemble_kernel(a_spec, b_spec, lam, mu, max_imag_energy=0.01, negative_weight_tol=0.01):
    a = _c128(a_spec); b = _c128(b_spec); lam = _c128(lam); mu = _c128(mu); t = a.shape[0]
    out = np.empty((t, t))
    _check(lib().orc_assemble_kernel(_p(a), _p(b), _p(lam), _p(mu), t, max_imag_energy,
                                     negative_weight_tol, _p(out)))
    return out


def spectral_deblur(blurred, kernel, epsilon: float) -> np.ndarray:
    b = _f64(blurred); k = _f64(kernel); t = k.shape[0]
    out = np.empty((b.shape[0] - t + 1, b.shape[1] - t + 1))
    _check(lib().orc_spectral_deblur(_p(b), b.shape[0], b.shape[1], _p(k), t, epsilon, _p(out)))
    return out


def decode_frame(pub, prv, hint: int | None = None, cfg: DecodeCfg | None = None) -> DecodedFrame:
    pub = _planes(pub); prv = _planes(prv); ch, r, c = pub.shape
    cfg = cfg or make_cfg()
    tmax = 63
    latent = np.empty(ch * r * c)  # oversized; trimmed below
    kernel = np.empty(tmax * tmax)
    info = DecodeInfo()
    _check(lib().orc_decode_frame(_p(pub), _p(prv), ch, r, c, -1 if hint is None else hint,
                                  C.byref(cfg), _p(latent), _p(kernel), C.byref(info)))
    t = info.width_used
    M, N = r - t + 1, c - t + 1
    return DecodedFrame(latent[: ch * M * N].reshape(ch, M, N).copy(), kernel[: t * t].reshape(t, t).copy(),
                        t, bool(info.width_clamped), info.validation_residual, info.epsilon_used,
                        list(info.stage_ms))


def validate_pair(pub, prv, k1, k2) -> float:
    pub = _planes(pub); prv = _planes(prv); ch, r, c = pub.shape
    k1 = _f64(k1); k2 = _f64(k2); out = np.zeros(1)
    _check(lib().orc_validate_pair(_p(pub), _p(prv), ch, r, c, _p(k1), _p(k2), k1.shape[0], _p(out)))
    return float(out[0])


def psnr(a, b) -> float:
    a = _f64(a); b = _f64(b)
    if a.ndim == 3:  # metrics.cpp:27-37, frame version
        sq = float(((a - b) ** 2).sum())
        return float("inf") if sq == 0 else 10 * np.log10(a.size / sq)
    return float(lib().orc_psnr(_p(a), _p(b), a.shape[0], a.shape[1]))


def bench_frames(pub32: np.ndarray, prv32: np.ndarray, recover: np.ndarray, kernel, epsilon: float,
                 cfg: DecodeCfg, threads: int) -> float:
    """CPU baseline with reference CLI semantics; returns wall seconds."""
    pub32 = np.ascontiguousarray(pub32, np.float32); prv32 = np.ascontiguousarray(prv32, np.float32)
    n, ch, r, c = pub32.shape
    rec = np.ascontiguousarray(recover, np.int32); k = _f64(kernel); secs = np.zeros(1)
    _check(lib().orc_bench_frames(_p(pub32), _p(prv32), n, ch, r, c, _p(rec), _p(k), k.shape[0],
                                  epsilon, C.byref(cfg), threads, _p(secs)))
    return float(secs[0])
