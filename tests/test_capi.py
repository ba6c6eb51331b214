"""The C ABI library (libcbp_cuda.so) loads on CPU and exports every entry point that
include/cbp_cuda.h declares; the host-side generators are bit-identical to the
reference's (checked against the oracle). No device compute is called here."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_1203_4874_b200 import _native

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _declared():
    src = open(os.path.join(ROOT, "include", "cbp_cuda.h")).read()
    return sorted(set(re.findall(r"\b(cbp_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = C.CDLL(_native.LIB_PATH)
    declared = _declared()
    assert len(declared) >= 30
    missing = [s for s in declared if not hasattr(lib, s)]
    assert not missing, missing
    assert set(_native.exported_symbols()) <= set(declared)


def test_errc_names_map_one_to_one():
    lib = _native.lib()
    names = [lib.cbp_errc_name(i + 1).decode() for i in range(18)]
    assert names == _native.ERRC_NAMES
    assert lib.cbp_errc_name(0).decode() == "Ok"


def test_friendly_size_host(oracle):
    lib = _native.lib()
    for n in [1, 7, 11, 97, 262, 488, 1090, 1930, 2174, 3854, 4099]:
        assert lib.cbp_friendly_size(n) == oracle.friendly_size(n)


def test_cfg_defaults_mirror_decoder_hpp():
    cfg = _native.DecodeCfg()
    _native.lib().cbp_decode_cfg_default(C.byref(cfg))
    assert (cfg.search_min, cfg.search_max, cfg.tau, cfg.has_epsilon, cfg.gap_threshold,
            cfg.trust_hint, cfg.max_imag_energy, cfg.negative_weight_tol, cfg.validate) == \
        (9, 25, 1e-6, 0, 1e-9, 0, 0.01, 0.01, 1)


def test_no_device_means_loud_failure():
    """Without a GPU the product path fails; it never falls back to the CPU."""
    import torch
    if torch.cuda.is_available():
        pytest.skip("a CUDA device is present")
    ptr = C.c_void_p()
    assert _native.lib().cbp_create(0, C.byref(ptr)) == _native.CBP_CUDA_ERROR
    with pytest.raises(_native.CbpError):
        _native.Context(0)


def test_generators_match_reference(oracle):
    from paper_1203_4874_b200 import api
    for s, i in [(1, 0), (2, 5), (0xdeadbeef, 123)]:
        assert api.frame_seed(s, i) == oracle.frame_seed(s, i)
    f = api.random_frame(13, 11, 3, 77)
    ref = oracle.random_frame(13, 11, 3, 77)
    assert np.array_equal(f, ref.astype(np.float32))
    for t, seed in [(3, 7), (5, 101), (9, 42), (11, 1234), (15, 9)]:
        p = api.generate_coprime_pair(t, seed)
        q = oracle.generate_coprime_pair(t, seed)
        assert np.array_equal(p.k1, q.k1) and np.array_equal(p.k2, q.k2)
        assert abs(p.coprimality_margin - q.coprimality_margin) <= 1e-9 * q.coprimality_margin
