"""Cross-checks the C++ oracle against an independent numpy/LAPACK/pocketfft
restatement (oracle/np_ref.py) on identical inputs."""
import numpy as np
import pytest

from oracle import np_ref as N


def _case(oracle, rows, cols, t, ch, seed):
    lat = oracle.random_frame(rows, cols, ch, oracle.frame_seed(1, seed))
    pair = oracle.generate_coprime_pair(t, oracle.frame_seed(2, seed))
    pub, prv = oracle.encode_frame(lat, pair.k1, pair.k2)
    # the GPU consumes FP32 frames: compare on FP32-rounded inputs
    return lat, pair, pub.astype(np.float32).astype(np.float64), prv.astype(np.float32).astype(np.float64)


@pytest.mark.parametrize("rows,cols,t,ch,lo,hi", [(64, 64, 5, 1, 3, 9), (48, 56, 7, 3, 3, 9), (96, 80, 9, 1, 3, 25)])
def test_decode_agrees_with_numpy(oracle, rows, cols, t, ch, lo, hi):
    lat, pair, pub, prv = _case(oracle, rows, cols, t, ch, rows + t)
    d = oracle.decode_frame(pub, prv, cfg=oracle.make_cfg(lo, hi))
    lat_n, k_n, t_n = N.decode_frame(pub, prv, lo, hi)
    assert d.width_used == t_n == t
    assert np.linalg.norm(d.kernel - k_n) / np.linalg.norm(k_n) <= 1e-9
    assert np.abs(d.latent - lat_n).max() <= 1e-7


def test_pieces_agree_with_numpy(oracle):
    rng = np.random.default_rng(3)
    plane = rng.uniform(0, 1, (37, 41))
    for axis in (0, 1):
        assert np.abs(oracle.axis_roots_dft(plane, axis, 7) - N.axis_roots_dft(plane, axis, 7)).max() <= 1e-11
    x = rng.uniform(-1, 1, (30, 42)) + 1j * rng.uniform(-1, 1, (30, 42))
    assert np.abs(oracle.fft2(x) - np.fft.fft2(x)).max() <= 1e-10
    b = rng.uniform(0, 1, (40, 50))
    k = rng.uniform(0, 1, (5, 5)); k /= k.sum()
    assert np.abs(oracle.spectral_deblur(b, k, 1e-8) - N.spectral_deblur(b, k, 1e-8)).max() <= 1e-8
    p = rng.uniform(-1, 1, 30) + 1j * rng.uniform(-1, 1, 30)
    q = rng.uniform(-1, 1, 30) + 1j * rng.uniform(-1, 1, 30)
    l = rng.uniform(-1, 1, 20)
    p, q = np.convolve(l, p[:5]), np.convolve(l, q[:5])
    a1, a2, g = oracle.cofactor_null_solve(p, q, 5)
    b1, b2, h = N.cofactor_null_solve(p, q, 5)
    e = np.concatenate([a2, a1]); r = np.concatenate([b2, b1])
    c = np.vdot(e, r) / np.vdot(e, e)
    assert np.abs(c * e - r).max() <= 1e-9 and abs(g - h) <= 1e-9 * max(1.0, h)
    m = oracle.bezout_leading_block(p, q, 6)
    assert abs(oracle.numerical_singularity(m, 0.5)[1] - N.singular_ratio(m)) <= 1e-12
