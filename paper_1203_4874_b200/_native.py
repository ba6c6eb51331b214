"""ctypes binding of the C ABI in include/cbp_cuda.h (libcbp_cuda.so, sm_100a).

The library is built in-tree by ``__graft_entry__.build()`` (``make -C
paper_1203_4874_b200/csrc``). There is no CPU fallback: if the library or a CUDA
device is missing every call raises.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# CBP_CUDA_LIB: load another build of the same library (A/B kernel experiments)
LIB_PATH = os.environ.get("CBP_CUDA_LIB") or os.path.join(HERE, "_lib", "libcbp_cuda.so")

CBP_MAX_WIDTH = 63

ERRC_NAMES = [
    "InvalidArgument", "NonUnitSamplePoint", "DegenerateInput", "IllConditioned",
    "CoprimalityFailure", "FrameTooSmall", "RangeExceeded", "NotQuantized",
    "InconsistentAxes", "IllConditionedSlice", "DegenerateScales", "NonRealKernel",
    "DimMismatch", "IoFailure", "CorruptManifest", "MissingFrame", "FormatViolation",
    "PairMismatch",
]
CBP_CUDA_ERROR = 100
CBP_UNSUPPORTED = 101

STAGE_NAMES = {1: "polynomial_evaluation", 2: "kernel_degree_estimation",
               3: "kernel_estimation_1d", 4: "kernel_estimation_2d_fft", 5: "validation"}


class DecodeCfg(C.Structure):
    """cbp_decode_cfg == cbp::DecodeConfig (decoder.hpp:10-20)."""
    _fields_ = [("search_min", C.c_int), ("search_max", C.c_int), ("tau", C.c_double),
                ("has_epsilon", C.c_int), ("epsilon", C.c_double), ("gap_threshold", C.c_double),
                ("trust_hint", C.c_int), ("max_imag_energy", C.c_double),
                ("negative_weight_tol", C.c_double), ("validate", C.c_int)]


class KernelSlot(C.Structure):
    _fields_ = [("status", C.c_int), ("fail_stage", C.c_int), ("fail_axis", C.c_int),
                ("fail_slice", C.c_int), ("width", C.c_int), ("clamped", C.c_int),
                ("width_z1", C.c_int), ("width_z2", C.c_int), ("fail_reason", C.c_int),
                ("reserved", C.c_int), ("fail_value", C.c_double),
                ("epsilon", C.c_double), ("residual", C.c_double), ("scale_residual", C.c_double),
                ("weights", C.c_double * (CBP_MAX_WIDTH * CBP_MAX_WIDTH))]


class DecodeInfo(C.Structure):
    _fields_ = [("status", C.c_int), ("fail_stage", C.c_int), ("fail_axis", C.c_int),
                ("fail_slice", C.c_int), ("width_used", C.c_int), ("width_clamped", C.c_int),
                ("validation_residual", C.c_double), ("epsilon_used", C.c_double),
                ("fail_value", C.c_double), ("stage_ms", C.c_double * 5),
                ("kernel", C.c_double * (CBP_MAX_WIDTH * CBP_MAX_WIDTH))]


class CbpError(RuntimeError):
    """Mirror of cbp::Error: ``code`` is the Errc name; str() is "<Name>: <detail>"."""

    def __init__(self, status: int, message: str):
        super().__init__(message)
        self.status = status
        if 1 <= status <= len(ERRC_NAMES):
            self.code = ERRC_NAMES[status - 1]
        else:
            self.code = {CBP_CUDA_ERROR: "CudaError", CBP_UNSUPPORTED: "Unsupported"}.get(status, "Error")


_lib = None

_P = C.c_void_p
_I = C.c_int
_D = C.c_double

_SIGS = {
    "cbp_create": (_I, [_I, C.POINTER(_P)]),
    "cbp_destroy": (None, [_P]),
    "cbp_last_error": (C.c_char_p, [_P]),
    "cbp_errc_name": (C.c_char_p, [_I]),
    "cbp_friendly_size": (_I, [_I]),
    "cbp_decode_cfg_default": (None, [_P]),
    "cbp_decode_frames": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _I, _P, _P]),
    "cbp_decode_frames_async": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _I, _P, _P]),
    "cbp_decode_frames_async_ev": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _I, _P, _P, _P]),
    "cbp_read_slots": (_I, [_P, _P, _I, _P, _P]),
    "cbp_slot_message": (_I, [_P, C.c_char_p, _I]),
    "cbp_spectral_deblur": (_I, [_P, _P, _I, _I, _I, _I, _I, _P, _I, _D, _P, _I, _P]),
    "cbp_spectral_deblur_slot": (_I, [_P, _P, _I, _I, _I, _I, _I, _P, _P, _I, _P]),
    "cbp_recover_kernels_async": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _P, _P, _P, _P]),
    "cbp_spectral_deblur_slots": (_I, [_P, _P, _I, _I, _I, _I, _I, _P, _I, _P, _I, _P]),
    "cbp_validate_frames_async": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _I, _P, _P]),
    "cbp_estimate_kernel_width": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _I, _D, _P, _P, _P]),
    "cbp_sample_slices": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _I, _P, _P, _P]),
    "cbp_cofactor_solve_batch": (_I, [_P, _P, _P, _I, _I, _I, _D, _P, _P, _P, _P, _P]),
    "cbp_sample_cofactors": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _I, _D, _P, _P, _P]),
    "cbp_complete_to_spectrum": (_I, [_P, _P, _I, _I, _P, _P]),
    "cbp_resolve_scales": (_I, [_P, _P, _P, _I, _P, _P, _P, _P]),
    "cbp_assemble_kernel": (_I, [_P, _P, _P, _P, _P, _I, _D, _D, _P, _P]),
    "cbp_validate_pair": (_I, [_P, _P, _P, _I, _I, _I, _I, _P, _P, _I, _P, _P]),
    "cbp_bezout_leading_block": (_I, [_P, _P, _I, _P, _I, _I, _P, _P]),
    "cbp_numerical_singularity": (_I, [_P, _P, _I, _D, _P, _P, _P]),
    "cbp_homogeneous_lsq": (_I, [_P, _P, _I, _I, _P, _P]),
    "cbp_fft2": (_I, [_P, _P, _I, _I, _I, _P, _P]),
    "cbp_encode_frames": (_I, [_P, _P, _I, _I, _I, _I, _I, _P, _P, _I, _P, _P, _I, _P]),
    "cbp_synth_frames": (_I, [_P, _P, _I, _I, _I, _I, C.c_uint64, _P]),
    "cbp_decode_run_host": (_I, [_P, _P, _P, _I, _I, _I, _I, _P, _I, _P, _P, _P]),
    "cbp_decode_run_host_q": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _P, _I, _P, _P, _P]),
    "cbp_quantize_frames": (_I, [_P, _P, _I, _I, _I, _I, _I, _P, _I, _P]),
    "cbp_dequantize_frames": (_I, [_P, _P, _I, _I, _I, _I, _I, _P, _I, _P]),
    "cbp_degrade_bits": (_I, [_P, _P, _I, _I, _I, _I, _I, _I, _P]),
    "cbp_decode_frames_q": (_I, [_P, _P, _P, _I, _I, _I, _I, _I, _I, _P, _P, _P, _I, _P, _P]),
    "cbp_frame_seed": (C.c_uint64, [C.c_uint64, _I]),
    "cbp_splitmix64": (C.c_uint64, [C.c_uint64]),
    "cbp_random_frame": (_I, [_I, _I, _I, C.c_uint64, _P]),
    "cbp_coprimality_check": (_D, [_P, _P, _I, _I]),
    "cbp_generate_coprime_pair": (_I, [_I, C.c_uint64, _I, _D, _I, _P, _P, _P]),
    "cbp_launch_count": (C.c_longlong, [_P]),
    "cbp_profile": (_I, [_P, _I]),
    "cbp_set_sm_reserve": (_I, [_P, _I]),
    "cbp_set_launch_chaining": (_I, [_P, _I]),
    "cbp_profile_read": (_I, [_P, _P, _P, _P]),
}


def lib():
    """Load libcbp_cuda.so (raises if it was not built: there is no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeError(f"{LIB_PATH} missing: run __graft_entry__.build() first")
        handle = C.CDLL(LIB_PATH)
        for name, (res, args) in _SIGS.items():
            fn = getattr(handle, name, None)
            if fn is None:
                continue
            fn.restype = res
            fn.argtypes = args
        _lib = handle
    return _lib


def exported_symbols() -> list[str]:
    return list(_SIGS)


class Context:
    """Owns one cbp_ctx (per device, per host thread)."""

    def __init__(self, device: int = 0):
        self.ptr = _P()
        st = lib().cbp_create(device, C.byref(self.ptr))
        if st != 0:
            raise CbpError(st, f"{lib().cbp_errc_name(st).decode()}: cbp_create(device={device}) failed")
        self.device = device

    def check(self, status: int):
        if status != 0:
            raise CbpError(status, lib().cbp_last_error(self.ptr).decode())

    def close(self):
        if self.ptr:
            lib().cbp_destroy(self.ptr)
            self.ptr = _P()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
