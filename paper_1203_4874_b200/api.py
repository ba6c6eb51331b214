"""Python host API mirroring the reference ``cbp::`` decoder interface.

Same function names, argument meaning and error behaviour as
/root/reference/proj/core/include/cbp/decoder.hpp (decode_frame, spectral_deblur,
estimate_kernel_width, sample_cofactors, complete_to_spectrum, resolve_scales,
assemble_kernel, validate_pair) and encoder.hpp (encode_frame). All compute runs in
libcbp_cuda.so through the C ABI of include/cbp_cuda.h; torch only supplies device
memory and the current CUDA stream. Errors raise ``CbpError`` whose ``code`` is the
reference ``Errc`` name and whose message carries the reference's
"<Name>: <stage>: <detail>" text.

Frames are numpy arrays or torch tensors shaped (rows, cols) or (channels, rows, cols);
row index m is the z1 power (types.hpp:15-17).
"""
from __future__ import annotations

import ctypes as C
import threading
from dataclasses import dataclass, field

import numpy as np
import torch

from . import _native as N
from ._native import CbpError, DecodeCfg, DecodeInfo, KernelSlot  # noqa: F401

AXIS_Z1, AXIS_Z2 = 0, 1

_tls = threading.local()


def context(device: int | None = None) -> N.Context:
    """Per-thread, per-device context (decode_frame is reentrant)."""
    if device is None:
        device = torch.cuda.current_device()
    ctxs = getattr(_tls, "ctxs", None)
    if ctxs is None:
        ctxs = _tls.ctxs = {}
    if device not in ctxs:
        ctxs[device] = N.Context(device)
    return ctxs[device]


def _stream_ptr(device) -> C.c_void_p:
    return C.c_void_p(torch.cuda.current_stream(device).cuda_stream)


def _dev_planes(x, device=None) -> torch.Tensor:
    """float32, contiguous, on the GPU, shaped (..., channels, rows, cols)."""
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    if not isinstance(x, torch.Tensor):
        x = torch.as_tensor(x)
    if device is None:
        device = torch.device("cuda", torch.cuda.current_device())
    x = x.to(device=device, dtype=torch.float32)
    if x.dim() == 2:
        x = x.unsqueeze(0)
    return x.contiguous()


def make_cfg(search_min=9, search_max=25, tau=1e-6, epsilon=None, gap_threshold=1e-9,
             trust_hint=False, max_imag_energy=0.01, negative_weight_tol=0.01,
             validate=True) -> DecodeCfg:
    """DecodeConfig with the reference defaults (decoder.hpp:10-20)."""
    return DecodeCfg(int(search_min), int(search_max), float(tau), int(epsilon is not None),
                     0.0 if epsilon is None else float(epsilon), float(gap_threshold),
                     int(bool(trust_hint)), float(max_imag_energy), float(negative_weight_tol),
                     int(bool(validate)))


def friendly_size(n: int) -> int:
    return int(N.lib().cbp_friendly_size(int(n)))


# ------------------------------------------------------------------ deconvolution
def spectral_deblur(blurred, kernel, epsilon: float, out: torch.Tensor | None = None) -> torch.Tensor:
    """cbp::spectral_deblur (decoder.hpp:63, decoder.cpp:273-278).

    ``blurred``: (rows, cols), (channels, rows, cols) or (batch, channels, rows, cols);
    ``kernel``: t x t nonnegative weights summing to 1. Returns the latent on the GPU,
    shaped like the input with rows-t+1 x cols-t+1 planes.
    """
    ndim = blurred.dim() if isinstance(blurred, torch.Tensor) else np.ndim(blurred)
    x = blurred if _pitched_ok(blurred) else _dev_planes(blurred)
    x4 = x.unsqueeze(0) if x.dim() == 3 else x
    if x4.dim() == 2:
        x4 = x4.unsqueeze(0).unsqueeze(0)
    B, ch, rows, cols = x4.shape
    ld = x4.stride(-2)
    k = np.ascontiguousarray(np.asarray(kernel, dtype=np.float64))
    if k.ndim != 2 or k.shape[0] != k.shape[1]:
        raise CbpError(13, "DimMismatch: kernel weights must be width x width")
    t = k.shape[0]
    ctx = context(x4.device.index)
    M, Nc = rows - t + 1, cols - t + 1
    if out is None:  # output planes keep the input geometry; the top-left M x N is written
        out = torch.empty((B, ch, rows, cols), dtype=torch.float32, device=x4.device)
    if not _pitched_ok(out) or out.shape[-2] != rows:
        raise CbpError(13, "DimMismatch: out must be float32 planes of the input geometry")
    ctx.check(N.lib().cbp_spectral_deblur(ctx.ptr, C.c_void_p(x4.data_ptr()), B, ch, rows, cols, ld,
                                          k.ctypes.data_as(C.c_void_p), t, float(epsilon),
                                          C.c_void_p(out.data_ptr()), out.stride(-2),
                                          _stream_ptr(x4.device)))
    out = out[..., :M, :Nc]
    if ndim == 2:
        return out[0, 0]
    if ndim == 3:
        return out[0]
    return out


# ----------------------------------------------------------------------- decode
@dataclass
class StageTimings:
    """decoder.hpp:65-71 (CUDA-event milliseconds of the batch the frame was in)."""
    polynomial_evaluation_ms: float = 0.0
    kernel_degree_estimation_ms: float = 0.0
    kernel_estimation_1d_ms: float = 0.0
    kernel_estimation_2d_fft_ms: float = 0.0
    total_ms: float = 0.0


@dataclass
class DecodedFrame:
    """decoder.hpp:73-80. ``latent`` is a GPU tensor (channels, M, N)."""
    latent: torch.Tensor
    kernel_estimate: np.ndarray
    width_used: int
    width_clamped: bool
    stage_timings: StageTimings = field(default_factory=StageTimings)
    validation_residual: float = 0.0
    epsilon_used: float = 0.0


def _pitched_ok(x) -> bool:
    """A CUDA float32 tensor the C ABI can read in place: unit column stride and planes of
    rows x ld (ld = row stride >= cols, e.g. a [..., :cols] view of pitched rows)."""
    if not (isinstance(x, torch.Tensor) and x.is_cuda and x.dtype == torch.float32 and x.dim() >= 2):
        return False
    rows, ld = x.shape[-2], x.stride(-2)
    if x.stride(-1) != 1 or ld < x.shape[-1]:
        return False
    expect = rows * ld
    for d in range(x.dim() - 3, -1, -1):
        if x.shape[d] > 1 and x.stride(d) != expect:
            return False
        expect *= x.shape[d]
    return True


def _check_planes(name: str, x, shape=None, device=None):
    """Raw device pointers go straight into the C ABI: reject tensors it would misread."""
    if not (_pitched_ok(x) and x.dim() == 4):
        raise CbpError(1, f"InvalidArgument: {name} must be a CUDA float32 (batch, channels, rows, cols) tensor "
                          f"with unit column stride and pitched planes")
    if shape is not None and tuple(x.shape) != tuple(shape):
        raise CbpError(13, f"DimMismatch: {name} is {tuple(x.shape)}, expected {tuple(shape)}")
    if device is not None and x.device != device:
        raise CbpError(1, f"InvalidArgument: {name} is on {x.device}, expected {device}")


def _check_slots(slots, count: int, device=None):
    if not (isinstance(slots, torch.Tensor) and slots.is_cuda and slots.dtype == torch.uint8
            and slots.is_contiguous()):
        raise CbpError(1, "InvalidArgument: slots must be a contiguous uint8 CUDA tensor")
    if slots.numel() < count * SLOT_BYTES:
        raise CbpError(1, f"InvalidArgument: slots hold {slots.numel() // SLOT_BYTES} kernel slots, {count} needed")
    if device is not None and slots.device != device:
        raise CbpError(1, f"InvalidArgument: slots are on {slots.device}, expected {device}")


def _slot_arg(slot, count: int, device) -> int:
    """A slot given as a uint8 tensor (checked) or as a raw device address (trusted)."""
    if isinstance(slot, torch.Tensor):
        _check_slots(slot, count, device)
        return slot.data_ptr()
    return int(slot)


def _as_batch(x) -> tuple[torch.Tensor, int]:
    ndim = x.dim() if isinstance(x, torch.Tensor) else np.ndim(x)
    t = _dev_planes(x)
    if t.dim() == 3:
        t = t.unsqueeze(0)
    return t.contiguous(), ndim


def decode_frames(pub, prv, hints=None, cfg: DecodeCfg | None = None) -> list[DecodedFrame]:
    """Batched cbp::decode_frame: pub/prv shaped (batch, channels, rows, cols)."""
    P, _ = _as_batch(pub)
    Q, _ = _as_batch(prv)
    if P.shape != Q.shape:
        raise CbpError(13, "DimMismatch: pair frames disagree on dimensions")
    B, ch, rows, cols = P.shape
    cfg = cfg or make_cfg()
    ctx = context(P.device.index)
    out = torch.empty((B, ch, rows, cols), dtype=torch.float32, device=P.device)
    hint_arr = None
    if hints is not None:
        hs = [hints] * B if np.isscalar(hints) else list(hints)
        hint_arr = (C.c_int * B)(*[int(h) if h is not None else 0 for h in hs])
    infos = (DecodeInfo * max(B, 1))()
    ctx.check(N.lib().cbp_decode_frames(ctx.ptr, C.c_void_p(P.data_ptr()), C.c_void_p(Q.data_ptr()), B, ch,
                                        rows, cols, cols, hint_arr, C.byref(cfg), C.c_void_p(out.data_ptr()),
                                        cols, infos, _stream_ptr(P.device)))
    res = []
    for b in range(B):
        inf = infos[b]
        t = inf.width_used
        k = np.array(inf.kernel[: t * t]).reshape(t, t)
        res.append(DecodedFrame(out[b, :, : rows - t + 1, : cols - t + 1], k, t, bool(inf.width_clamped),
                                StageTimings(*list(inf.stage_ms)), inf.validation_residual, inf.epsilon_used))
    return res


def decode_frame(pub, prv, hint: int | None = None, cfg: DecodeCfg | None = None) -> DecodedFrame:
    """cbp::decode_frame (decoder.hpp:82, decoder.cpp:280-378)."""
    return decode_frames(pub, prv, None if hint is None else [hint], cfg)[0]


# ------------------------------------------------------ quantized-stream tier
_QDTYPE = {8: torch.uint8, 16: torch.uint16}


def _bits_of(codes: torch.Tensor) -> int:
    for bits, dt in _QDTYPE.items():
        if codes.dtype == dt:
            return bits
    raise CbpError(1, "InvalidArgument: quantized frames must be uint8 or uint16 codes")


def _dev_codes(x) -> torch.Tensor:
    if isinstance(x, np.ndarray):
        x = torch.from_numpy(np.ascontiguousarray(x))
    x = x.to(device=torch.device("cuda", torch.cuda.current_device()))
    if x.dim() == 2:
        x = x.unsqueeze(0)
    return x.contiguous()


def quantize_frames(frames, bits: int) -> torch.Tensor:
    """cbp::quantize_frame (encoder.cpp:105-120) on the device: integer codes
    k = round(clamp(x, 0, 1) * (2^bits - 1)) as uint8 / uint16; RangeExceeded outside [0, 1]."""
    X = _dev_planes(frames)
    if bits not in _QDTYPE:
        raise CbpError(1, "InvalidArgument: quantization depth must be u8 or u16")
    rows, cols = X.shape[-2:]
    planes = X.numel() // (rows * cols)
    out = torch.empty(X.shape, dtype=_QDTYPE[bits], device=X.device)
    ctx = context(X.device.index)
    ctx.check(N.lib().cbp_quantize_frames(ctx.ptr, C.c_void_p(X.data_ptr()), planes, rows, cols, cols, bits,
                                          C.c_void_p(out.data_ptr()), cols, _stream_ptr(X.device)))
    return out


def dequantize_frames(codes) -> torch.Tensor:
    """FP32 frames float(k / (2^bits - 1)) from uint8 / uint16 codes."""
    Q = _dev_codes(codes)
    bits = _bits_of(Q)
    rows, cols = Q.shape[-2:]
    planes = Q.numel() // (rows * cols)
    out = torch.empty(Q.shape, dtype=torch.float32, device=Q.device)
    ctx = context(Q.device.index)
    ctx.check(N.lib().cbp_dequantize_frames(ctx.ptr, C.c_void_p(Q.data_ptr()), bits, planes, rows, cols, cols,
                                            C.c_void_p(out.data_ptr()), cols, _stream_ptr(Q.device)))
    return out


def degrade_bits(codes, drop: int) -> torch.Tensor:
    """cbp::degrade_bits (encoder.cpp:124-139) on codes: k & ~(2^drop - 1) (returns a copy)."""
    Q = _dev_codes(codes).clone()
    bits = _bits_of(Q)
    rows, cols = Q.shape[-2:]
    planes = Q.numel() // (rows * cols)
    ctx = context(Q.device.index)
    ctx.check(N.lib().cbp_degrade_bits(ctx.ptr, C.c_void_p(Q.data_ptr()), bits, planes, rows, cols, cols, int(drop),
                                       _stream_ptr(Q.device)))
    return Q


def decode_frames_q(pub_codes, prv_codes, hints=None, cfg: DecodeCfg | None = None) -> list[DecodedFrame]:
    """Batched decode_frame of quantized pairs (uint8 / uint16 codes, batch x ch x rows x cols)."""
    P = _dev_codes(pub_codes)
    Q = _dev_codes(prv_codes)
    if P.dim() == 3:
        P, Q = P.unsqueeze(0), Q.unsqueeze(0)
    if P.shape != Q.shape or P.dtype != Q.dtype:
        raise CbpError(13, "DimMismatch: pair frames disagree on dimensions")
    bits = _bits_of(P)
    B, ch, rows, cols = P.shape
    cfg = cfg or make_cfg()
    ctx = context(P.device.index)
    out = torch.empty((B, ch, rows, cols), dtype=torch.float32, device=P.device)
    hint_arr = None
    if hints is not None:
        hs = [hints] * B if np.isscalar(hints) else list(hints)
        hint_arr = (C.c_int * B)(*[int(h) if h is not None else 0 for h in hs])
    infos = (DecodeInfo * max(B, 1))()
    ctx.check(N.lib().cbp_decode_frames_q(ctx.ptr, C.c_void_p(P.data_ptr()), C.c_void_p(Q.data_ptr()), bits, B, ch,
                                          rows, cols, cols, hint_arr, C.byref(cfg), C.c_void_p(out.data_ptr()),
                                          cols, infos, _stream_ptr(P.device)))
    res = []
    for b in range(B):
        inf = infos[b]
        t = inf.width_used
        k = np.array(inf.kernel[: t * t]).reshape(t, t)
        res.append(DecodedFrame(out[b, :, : rows - t + 1, : cols - t + 1], k, t, bool(inf.width_clamped),
                                StageTimings(*list(inf.stage_ms)), inf.validation_residual, inf.epsilon_used))
    return res


def estimate_kernel_width(pub, prv, search_min: int, search_max: int, tau: float) -> tuple[int, bool]:
    """cbp::estimate_kernel_width (decoder.hpp:29-30) -> (width, clamped)."""
    P, _ = _as_batch(pub)
    Q, _ = _as_batch(prv)
    _, ch, rows, cols = P.shape
    ctx = context(P.device.index)
    w = C.c_int(); c = C.c_int()
    ctx.check(N.lib().cbp_estimate_kernel_width(ctx.ptr, C.c_void_p(P.data_ptr()), C.c_void_p(Q.data_ptr()), ch,
                                                rows, cols, cols, search_min, search_max, tau, C.byref(w),
                                                C.byref(c), _stream_ptr(P.device)))
    return w.value, bool(c.value)


def sample_slices(pub, prv, t: int, axis: int) -> tuple[np.ndarray, np.ndarray]:
    """axis_roots_dft of luma(pub) / luma(prv) (fft.hpp:15-18): (t, L) complex each."""
    P, _ = _as_batch(pub)
    Q, _ = _as_batch(prv)
    _, ch, rows, cols = P.shape
    L = cols if axis == AXIS_Z1 else rows
    sp = np.empty((t, L), np.complex128); sq = np.empty((t, L), np.complex128)
    ctx = context(P.device.index)
    ctx.check(N.lib().cbp_sample_slices(ctx.ptr, C.c_void_p(P.data_ptr()), C.c_void_p(Q.data_ptr()), ch, rows,
                                        cols, cols, t, axis, sp.ctypes.data_as(C.c_void_p),
                                        sq.ctypes.data_as(C.c_void_p), _stream_ptr(P.device)))
    return sp, sq


def sample_cofactors(pub, prv, width: int, axis: int, gap_threshold: float = 1e-9):
    """cbp::sample_cofactors (decoder.hpp:40-41) -> (values t x t complex, gaps)."""
    P, _ = _as_batch(pub)
    Q, _ = _as_batch(prv)
    _, ch, rows, cols = P.shape
    vals = np.empty((width, width), np.complex128); gaps = np.empty(width)
    ctx = context(P.device.index)
    ctx.check(N.lib().cbp_sample_cofactors(ctx.ptr, C.c_void_p(P.data_ptr()), C.c_void_p(Q.data_ptr()), ch,
                                           rows, cols, cols, width, axis, gap_threshold,
                                           vals.ctypes.data_as(C.c_void_p), gaps.ctypes.data_as(C.c_void_p),
                                           _stream_ptr(P.device)))
    return vals, gaps


def cofactor_solve_batch(p, q, t: int, gap_threshold: float = 1e-9):
    """Batched cbp::cofactor_null_solve (poly.hpp:51-52): p, q (batch, len) complex."""
    p = np.ascontiguousarray(np.atleast_2d(p), np.complex128)
    q = np.ascontiguousarray(np.atleast_2d(q), np.complex128)
    B, L = p.shape
    k1 = np.empty((B, t), np.complex128); k2 = np.empty((B, t), np.complex128)
    gaps = np.empty(B); st = np.zeros(B, np.int32)
    ctx = context()
    ctx.check(N.lib().cbp_cofactor_solve_batch(ctx.ptr, p.ctypes.data_as(C.c_void_p), q.ctypes.data_as(C.c_void_p),
                                               B, L, t, gap_threshold, k1.ctypes.data_as(C.c_void_p),
                                               k2.ctypes.data_as(C.c_void_p), gaps.ctypes.data_as(C.c_void_p),
                                               st.ctypes.data_as(C.c_void_p), _stream_ptr(None)))
    return k1, k2, gaps


def cofactor_null_solve(p, q, t: int, gap_threshold: float = 1e-9):
    """cbp::cofactor_null_solve for one pair -> (k1, k2, gap); p and q may differ in length."""
    p = np.asarray(p, np.complex128).ravel(); q = np.asarray(q, np.complex128).ravel()
    if len(p) < t or len(q) < t:
        raise CbpError(1, "InvalidArgument: slice degree below cofactor degree")
    L = max(len(p), len(q))  # zero padding leaves the stacked convolution system unchanged
    pp = np.zeros(L, np.complex128); pp[: len(p)] = p
    qq = np.zeros(L, np.complex128); qq[: len(q)] = q
    k1, k2, g = cofactor_solve_batch(pp[None], qq[None], t, gap_threshold)
    return k1[0], k2[0], float(g[0])


def _c128(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.complex128))


def bezout_leading_block(p, q, size: int) -> np.ndarray:
    """cbp::bezout_leading_block (poly.hpp:30, poly.cpp:66-79) on the device."""
    p, q = _c128(p), _c128(q)
    out = np.empty((max(int(size), 0), max(int(size), 0)), np.complex128)
    ctx = context()
    ctx.check(N.lib().cbp_bezout_leading_block(ctx.ptr, p.ctypes.data_as(C.c_void_p), len(p),
                                               q.ctypes.data_as(C.c_void_p), len(q), int(size),
                                               out.ctypes.data_as(C.c_void_p), _stream_ptr(None)))
    return out


def numerical_singularity(m, tau: float) -> tuple[bool, float]:
    """cbp::numerical_singularity (poly.hpp:38, poly.cpp:81-91): (singular, sigma_min/sigma_max)."""
    m = _c128(m)
    if m.ndim != 2 or m.shape[0] != m.shape[1] or m.shape[0] < 1:
        raise CbpError(1, "InvalidArgument: singularity test needs a square matrix")
    sing, ratio = C.c_int(), C.c_double()
    ctx = context()
    ctx.check(N.lib().cbp_numerical_singularity(ctx.ptr, m.ctypes.data_as(C.c_void_p), m.shape[0], float(tau),
                                                C.byref(sing), C.byref(ratio), _stream_ptr(None)))
    return bool(sing.value), float(ratio.value)


def homogeneous_lsq(a) -> np.ndarray:
    """cbp::homogeneous_lsq (poly.hpp:55, poly.cpp:123-130): unit minimizer of |A x|, phase-normalized."""
    a = _c128(a)
    if a.ndim != 2:
        raise CbpError(1, "InvalidArgument: homogeneous system needs a matrix")
    x = np.empty(a.shape[1], np.complex128)
    ctx = context()
    ctx.check(N.lib().cbp_homogeneous_lsq(ctx.ptr, a.ctypes.data_as(C.c_void_p), a.shape[0], a.shape[1],
                                          x.ctypes.data_as(C.c_void_p), _stream_ptr(None)))
    return x


def fft2(x, inverse: bool = False) -> np.ndarray:
    """cbp::fft2 (fft.hpp:9-10): unnormalized forward 2D DFT of any size, FP64, on the device;
    ``inverse`` gives cbp::ifft2 (fft.hpp:13, 1/(M N) normalization)."""
    x = _c128(x)
    if x.ndim != 2:
        raise CbpError(1, "InvalidArgument: fft2 needs a matrix")
    out = np.empty_like(x)
    ctx = context()
    ctx.check(N.lib().cbp_fft2(ctx.ptr, x.ctypes.data_as(C.c_void_p), x.shape[0], x.shape[1], int(bool(inverse)),
                               out.ctypes.data_as(C.c_void_p), _stream_ptr(None)))
    return out


def ifft2(x) -> np.ndarray:
    return fft2(x, inverse=True)


def complete_to_spectrum(values, axis: int) -> np.ndarray:
    """cbp::complete_to_spectrum (decoder.hpp:45)."""
    v = np.ascontiguousarray(values, np.complex128); t = v.shape[0]
    out = np.empty_like(v)
    ctx = context()
    ctx.check(N.lib().cbp_complete_to_spectrum(ctx.ptr, v.ctypes.data_as(C.c_void_p), t, axis,
                                               out.ctypes.data_as(C.c_void_p), _stream_ptr(None)))
    return out


def resolve_scales(a_values, b_values):
    """cbp::resolve_scales (decoder.hpp:54) -> (lambda, mu, residual)."""
    a = np.ascontiguousarray(a_values, np.complex128); b = np.ascontiguousarray(b_values, np.complex128)
    t = a.shape[0]
    lam = np.empty(t, np.complex128); mu = np.empty(t, np.complex128); res = C.c_double()
    ctx = context()
    ctx.check(N.lib().cbp_resolve_scales(ctx.ptr, a.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p), t,
                                         lam.ctypes.data_as(C.c_void_p), mu.ctypes.data_as(C.c_void_p),
                                         C.byref(res), _stream_ptr(None)))
    return lam, mu, res.value


def assemble_kernel(a_spectrum, b_spectrum, lam, mu, max_imag_energy=0.01, negative_weight_tol=0.01) -> np.ndarray:
    """cbp::assemble_kernel (decoder.hpp:57-59) -> t x t weights."""
    a = np.ascontiguousarray(a_spectrum, np.complex128); b = np.ascontiguousarray(b_spectrum, np.complex128)
    lam = np.ascontiguousarray(lam, np.complex128); mu = np.ascontiguousarray(mu, np.complex128)
    t = a.shape[0]
    w = np.empty((t, t))
    ctx = context()
    ctx.check(N.lib().cbp_assemble_kernel(ctx.ptr, a.ctypes.data_as(C.c_void_p), b.ctypes.data_as(C.c_void_p),
                                          lam.ctypes.data_as(C.c_void_p), mu.ctypes.data_as(C.c_void_p), t,
                                          max_imag_energy, negative_weight_tol, w.ctypes.data_as(C.c_void_p),
                                          _stream_ptr(None)))
    return w


def validate_pair(pub, prv, k1, k2) -> float:
    """cbp::validate_pair (decoder.hpp:85-86)."""
    P, _ = _as_batch(pub)
    Q, _ = _as_batch(prv)
    _, ch, rows, cols = P.shape
    k1 = np.ascontiguousarray(k1, np.float64); k2 = np.ascontiguousarray(k2, np.float64)
    if k1.shape != k2.shape:
        raise CbpError(13, "DimMismatch: kernel widths differ")
    r = C.c_double()
    ctx = context(P.device.index)
    ctx.check(N.lib().cbp_validate_pair(ctx.ptr, C.c_void_p(P.data_ptr()), C.c_void_p(Q.data_ptr()), ch, rows, cols,
                                        cols, k1.ctypes.data_as(C.c_void_p), k2.ctypes.data_as(C.c_void_p),
                                        k1.shape[0], C.byref(r), _stream_ptr(P.device)))
    return r.value


def encode_frame(latent, k1, k2) -> tuple[torch.Tensor, torch.Tensor]:
    """cbp::encode_frame on the device (encoder.cpp:83-103): (public, private) FP32 planes."""
    X, ndim = _as_batch(latent)
    B, ch, rows, cols = X.shape
    k1 = np.ascontiguousarray(k1, np.float64); k2 = np.ascontiguousarray(k2, np.float64)
    t = k1.shape[0]
    ro, co = rows + t - 1, cols + t - 1
    pub = torch.empty((B, ch, ro, co), dtype=torch.float32, device=X.device)
    prv = torch.empty_like(pub)
    ctx = context(X.device.index)
    ctx.check(N.lib().cbp_encode_frames(ctx.ptr, C.c_void_p(X.data_ptr()), B, ch, rows, cols, cols,
                                        k1.ctypes.data_as(C.c_void_p), k2.ctypes.data_as(C.c_void_p), t,
                                        C.c_void_p(pub.data_ptr()), C.c_void_p(prv.data_ptr()), co,
                                        _stream_ptr(X.device)))
    if ndim == 2:
        return pub[0, 0], prv[0, 0]
    if ndim == 3:
        return pub[0], prv[0]
    return pub, prv


def synth_frames(planes: int, rows: int, cols: int, seed: int, device=None) -> torch.Tensor:
    """Device-generated U[0,1) planes for benchmarking (not the reference's mt19937_64 stream)."""
    dev = torch.device("cuda", torch.cuda.current_device() if device is None else device)
    out = torch.empty((planes, rows, cols), dtype=torch.float32, device=dev)
    ctx = context(dev.index)
    ctx.check(N.lib().cbp_synth_frames(ctx.ptr, C.c_void_p(out.data_ptr()), planes, rows, cols, cols,
                                       C.c_uint64(seed), _stream_ptr(dev)))
    return out


# ------------------------------------------------------- CBP generation inputs
def frame_seed(stream_seed: int, frame_index: int) -> int:
    """rng.hpp:27-29."""
    return int(N.lib().cbp_frame_seed(C.c_uint64(stream_seed), int(frame_index)))


def splitmix64(x: int) -> int:
    return int(N.lib().cbp_splitmix64(C.c_uint64(x)))


def random_frame(rows: int, cols: int, channels: int, seed: int) -> np.ndarray:
    """synth.cpp:12-22 (mt19937_64, column-major draw) as float32 (channels, rows, cols)."""
    out = np.empty((channels, rows, cols), np.float32)
    st = N.lib().cbp_random_frame(rows, cols, channels, C.c_uint64(seed), out.ctypes.data_as(C.c_void_p))
    if st:
        raise CbpError(st, "InvalidArgument: bad frame geometry")
    return out


def coprimality_check(k1, k2, trials: int = 4) -> float:
    k1 = np.ascontiguousarray(k1, np.float64); k2 = np.ascontiguousarray(k2, np.float64)
    return float(N.lib().cbp_coprimality_check(k1.ctypes.data_as(C.c_void_p), k2.ctypes.data_as(C.c_void_p),
                                               k1.shape[0], trials))


@dataclass
class CoprimePair:
    """kernel.hpp:19-24."""
    k1: np.ndarray
    k2: np.ndarray
    coprimality_margin: float
    seed: int


def generate_coprime_pair(width: int, seed: int, max_retries: int = 16, margin_threshold: float = 1e-6,
                          trials: int = 4) -> CoprimePair:
    """encoder.cpp:66-81 (host: seeded draw + Sylvester coprimality check)."""
    k1 = np.empty((width, width)); k2 = np.empty((width, width)); m = C.c_double()
    st = N.lib().cbp_generate_coprime_pair(width, C.c_uint64(seed), max_retries, margin_threshold, trials,
                                           k1.ctypes.data_as(C.c_void_p), k2.ctypes.data_as(C.c_void_p),
                                           C.byref(m))
    if st == 5:
        raise CbpError(st, f"CoprimalityFailure: no coprime pair of width {width} within {max_retries} draws")
    if st:
        raise CbpError(st, "InvalidArgument: kernel width must be odd, within [3,63]")
    return CoprimePair(k1, k2, m.value, seed)


def decode_run_host(pub: torch.Tensor, prv: torch.Tensor, recover, cfg: DecodeCfg | None = None,
                    width_hint: int = 0, out: torch.Tensor | None = None, device: int | None = None):
    """Host-buffer run decode (the end-to-end path): pub/prv are CPU float32 tensors, or
    uint8 / uint16 quantized codes, (n, channels, rows, cols), ideally pinned; returns
    (latent CPU float32 tensor in the input geometry, list of KernelSlot for the recovery
    frames)."""
    assert pub.device.type == "cpu" and pub.is_contiguous()
    n, ch, rows, cols = pub.shape
    rec = np.ascontiguousarray(np.asarray(recover, np.int32))
    cfg = cfg or make_cfg()
    if out is None:
        out = torch.empty(pub.shape, dtype=torch.float32, pin_memory=pub.is_pinned())
    nrec = int((rec != 0).sum())
    slots = (KernelSlot * max(nrec, 1))()
    ctx = context(device)
    prv_p = C.c_void_p(prv.data_ptr()) if prv is not None else None
    if pub.dtype == torch.float32:
        ctx.check(N.lib().cbp_decode_run_host(ctx.ptr, C.c_void_p(pub.data_ptr()), prv_p, n, ch, rows, cols,
                                              rec.ctypes.data_as(C.c_void_p), int(width_hint), C.byref(cfg),
                                              C.c_void_p(out.data_ptr()), slots))
    else:  # quantized codes: 1 or 2 bytes per sample over PCIe, dequantized on the device
        ctx.check(N.lib().cbp_decode_run_host_q(ctx.ptr, C.c_void_p(pub.data_ptr()), prv_p, _bits_of(pub), n, ch,
                                                rows, cols, rec.ctypes.data_as(C.c_void_p), int(width_hint),
                                                C.byref(cfg), C.c_void_p(out.data_ptr()), slots))
    return out, [slots[i] for i in range(nrec)]


def launch_count(device: int | None = None) -> int:
    return int(N.lib().cbp_launch_count(context(device).ptr))


def decode_frames_async(pub: torch.Tensor, prv: torch.Tensor, cfg: DecodeCfg, out: torch.Tensor,
                        slots: torch.Tensor, hints=None, ctx: N.Context | None = None, stream=None,
                        slot_ready: "torch.cuda.Event | None" = None):
    """cbp_decode_frames_async on device tensors (batch, ch, rows, cols); ``slots`` is a
    uint8 device tensor of batch * sizeof(KernelSlot) bytes receiving the per-frame state.
    ``ctx`` / ``stream`` select the context (workspaces) and CUDA stream (default: the
    thread's context and torch's current stream)."""
    _check_planes("pub", pub)
    B, ch, rows, cols = pub.shape
    _check_planes("prv", prv, pub.shape, pub.device)
    _check_planes("out", out, pub.shape, pub.device)
    _check_slots(slots, B, pub.device)
    ctx = ctx or context(pub.device.index)
    hint_arr = None
    if hints is not None:
        hint_arr = (C.c_int * B)(*[int(h) for h in hints])
    st = C.c_void_p(stream.cuda_stream) if stream is not None else _stream_ptr(pub.device)
    if slot_ready is not None:  # recorded as soon as the kernels are final (cbp_decode_frames_async_ev)
        ev = C.c_void_p(slot_ready.cuda_event)
        ctx.check(N.lib().cbp_decode_frames_async_ev(ctx.ptr, C.c_void_p(pub.data_ptr()),
                                                     C.c_void_p(prv.data_ptr()), B, ch, rows, cols, pub.stride(-2),
                                                     hint_arr, C.byref(cfg), C.c_void_p(out.data_ptr()),
                                                     out.stride(-2), C.c_void_p(slots.data_ptr()), st, ev))
        return
    ctx.check(N.lib().cbp_decode_frames_async(ctx.ptr, C.c_void_p(pub.data_ptr()), C.c_void_p(prv.data_ptr()), B,
                                              ch, rows, cols, pub.stride(-2), hint_arr, C.byref(cfg),
                                              C.c_void_p(out.data_ptr()), out.stride(-2),
                                              C.c_void_p(slots.data_ptr()), st))


def recover_kernels_async(pub: torch.Tensor, prv: torch.Tensor, cfg: DecodeCfg, slots: torch.Tensor, hints=None,
                          ctx: N.Context | None = None, stream=None):
    """cbp_recover_kernels_async: decode_frame's recovery stages only (decoder.cpp:290-352),
    kernels, widths and epsilons into ``slots``; deconvolve with spectral_deblur_slot and
    finish with validate_frames_async for the same results as decode_frames_async."""
    _check_planes("pub", pub)
    B, ch, rows, cols = pub.shape
    _check_planes("prv", prv, pub.shape, pub.device)
    _check_slots(slots, B, pub.device)
    ctx = ctx or context(pub.device.index)
    hint_arr = (C.c_int * B)(*[int(h) for h in hints]) if hints is not None else None
    st = C.c_void_p(stream.cuda_stream) if stream is not None else _stream_ptr(pub.device)
    ctx.check(N.lib().cbp_recover_kernels_async(ctx.ptr, C.c_void_p(pub.data_ptr()), C.c_void_p(prv.data_ptr()), B,
                                                ch, rows, cols, pub.stride(-2), hint_arr, C.byref(cfg),
                                                C.c_void_p(slots.data_ptr()), st))


def validate_frames_async(pub: torch.Tensor, latent: torch.Tensor, slots: torch.Tensor, ctx: N.Context | None = None,
                          stream=None):
    """cbp_validate_frames_async: validation residual (decoder.cpp:367-376) of deconvolved
    latents into ``slots[b].residual``."""
    _check_planes("pub", pub)
    B, ch, rows, cols = pub.shape
    _check_planes("latent", latent, pub.shape, pub.device)
    _check_slots(slots, B, pub.device)
    ctx = ctx or context(pub.device.index)
    st = C.c_void_p(stream.cuda_stream) if stream is not None else _stream_ptr(pub.device)
    ctx.check(N.lib().cbp_validate_frames_async(ctx.ptr, C.c_void_p(pub.data_ptr()), C.c_void_p(latent.data_ptr()), B,
                                                ch, rows, cols, pub.stride(-2), latent.stride(-2),
                                                C.c_void_p(slots.data_ptr()), st))


def spectral_deblur_slots(blurred: torch.Tensor, slots: torch.Tensor, frames_per_slot: int, out: torch.Tensor,
                          ctx: N.Context | None = None, stream=None):
    """cbp_spectral_deblur_slots: frame f of ``blurred`` (batch, ch, rows, cols) is deconvolved
    with slot ``f // frames_per_slot`` of ``slots`` (uint8 device tensor of kernel slots)."""
    _check_planes("blurred", blurred)
    B, ch, rows, cols = blurred.shape
    _check_planes("out", out, blurred.shape, blurred.device)
    if int(frames_per_slot) < 1:
        raise CbpError(1, "InvalidArgument: frames_per_slot must be >= 1")
    _check_slots(slots, (B + int(frames_per_slot) - 1) // int(frames_per_slot), blurred.device)
    ctx = ctx or context(blurred.device.index)
    st = C.c_void_p(stream.cuda_stream) if stream is not None else _stream_ptr(blurred.device)
    ctx.check(N.lib().cbp_spectral_deblur_slots(ctx.ptr, C.c_void_p(blurred.data_ptr()), B, ch, rows, cols,
                                                blurred.stride(-2), C.c_void_p(slots.data_ptr()),
                                                int(frames_per_slot), C.c_void_p(out.data_ptr()), out.stride(-2), st))


def spectral_deblur_slot(blurred: torch.Tensor, slot_ptr, out: torch.Tensor, ctx: N.Context | None = None,
                         stream=None):
    """cbp_spectral_deblur_slot: kernel, width and epsilon read on the device. ``slot_ptr`` is a
    uint8 slot tensor (checked) or a raw device address of one cbp_kernel_slot."""
    _check_planes("blurred", blurred)
    B, ch, rows, cols = blurred.shape
    _check_planes("out", out, blurred.shape, blurred.device)
    slot_ptr = _slot_arg(slot_ptr, 1, blurred.device)
    ctx = ctx or context(blurred.device.index)
    st = C.c_void_p(stream.cuda_stream) if stream is not None else _stream_ptr(blurred.device)
    ctx.check(N.lib().cbp_spectral_deblur_slot(ctx.ptr, C.c_void_p(blurred.data_ptr()), B, ch, rows, cols,
                                               blurred.stride(-2), C.c_void_p(slot_ptr),
                                               C.c_void_p(out.data_ptr()), out.stride(-2), st))


def read_slots(slots: torch.Tensor, count: int) -> list:
    _check_slots(slots, count)
    host = (KernelSlot * count)()
    ctx = context(slots.device.index)
    ctx.check(N.lib().cbp_read_slots(ctx.ptr, C.c_void_p(slots.data_ptr()), count, host, _stream_ptr(slots.device)))
    return [host[i] for i in range(count)]


def slot_message(slot) -> str:
    """The reference's error text for a failed slot (cbp_slot_message): what decode_frame
    throws for that frame, "<Errc>: <stage>: <Errc>: <detail>"; "" for a good slot."""
    buf = C.create_string_buffer(512)
    N.lib().cbp_slot_message(C.byref(slot), buf, 512)
    return buf.value.decode()


def set_sm_reserve(sms: int, ctx: N.Context | None = None, device: int | None = None):
    """cbp_set_sm_reserve: SMs the deconvolution passes of this context leave to other streams."""
    ctx = ctx or context(device)
    ctx.check(N.lib().cbp_set_sm_reserve(ctx.ptr, int(sms)))


def set_launch_chaining(on: bool, ctx: N.Context | None = None, device: int | None = None):
    """cbp_set_launch_chaining: programmatic dependent launch of this context's small
    latency-chain kernels (default on)."""
    ctx = ctx or context(device)
    ctx.check(N.lib().cbp_set_launch_chaining(ctx.ptr, int(bool(on))))


def profile(enable: bool, device: int | None = None):
    N.lib().cbp_profile(context(device).ptr, int(enable))


def profile_read(device: int | None = None):
    ms = (C.c_double * 3)(); planes = C.c_longlong(); groups = C.c_int()
    ctx = context(device)
    ctx.check(N.lib().cbp_profile_read(ctx.ptr, ms, C.byref(planes), C.byref(groups)))
    return list(ms), planes.value, groups.value


SLOT_BYTES = C.sizeof(KernelSlot)
