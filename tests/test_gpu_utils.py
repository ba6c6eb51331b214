"""The polynomial / transform utilities of the reference's public headers as stand-alone
device calls (cbp_bezout_leading_block, cbp_numerical_singularity, cbp_homogeneous_lsq,
cbp_fft2): the reference's own known answers (poly_test.cpp:134-287, fft_test.cpp:32-74),
the exact-arithmetic rank law, and agreement with the FP64 oracle."""
import math

import numpy as np
import pytest

import exact as X

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def api():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_1203_4874_b200 import api as A
    torch.cuda.set_device(0)
    return A


def _rand_int_poly(rng, deg, bound=5):
    p = [int(v) for v in rng.integers(-bound, bound + 1, deg + 1)]
    while p[-1] == 0:
        p[-1] = int(rng.integers(-bound, bound + 1))
    if p[0] == 0:
        p[0] = 1
    return [X.Q(v) for v in p]


def test_bezout_known_answers(oracle, api):
    assert api.bezout_leading_block([1, 2], [3, 1], 1)[0, 0] == 5  # poly_test.cpp:134-138
    b = api.bezout_leading_block([1, 3, 2], [3, 4, 1], 2)          # :140-147
    assert np.array_equal(b, np.full((2, 2), 5.0 + 0j))
    assert api.numerical_singularity(b, 1e-8)[0]
    rng = np.random.default_rng(44)
    p = rng.uniform(-1, 1, 6) + 1j * rng.uniform(-1, 1, 6)
    assert np.abs(api.bezout_leading_block(p, p, 5)).max() == 0.0  # :149-153
    q = rng.uniform(-1, 1, 9) + 1j * rng.uniform(-1, 1, 9)
    for size in (1, 4, 8, 12):  # same sums in the same order (FMA contraction: last-bit differences)
        ref = oracle.bezout_leading_block(p, q, size)
        assert np.abs(api.bezout_leading_block(p, q, size) - ref).max() <= 1e-14 * max(1.0, np.abs(ref).max())
    with pytest.raises(api.CbpError) as e:
        api.bezout_leading_block([0, 0], [1, 2], 2)
    assert e.value.code == "DegenerateInput" and "all-zero" in str(e.value)
    with pytest.raises(api.CbpError) as e:
        api.bezout_leading_block([1, 2], [1, 2], 0)
    assert e.value.code == "InvalidArgument"


def test_bezout_antisymmetry_and_rank_law(api):
    """poly_test.cpp:155-191: bitwise antisymmetry; rank = degree - gcd degree against
    exact rational arithmetic, every leading block classified correctly at tau = 1e-9."""
    rng = np.random.default_rng(7)
    for _ in range(12):
        p = [float(v) for v in _rand_int_poly(rng, 3 + int(rng.integers(0, 4)))]
        q = [float(v) for v in _rand_int_poly(rng, 3 + int(rng.integers(0, 4)))]
        size = max(len(p), len(q)) - 1
        assert np.abs(api.bezout_leading_block(p, q, size) + api.bezout_leading_block(q, p, size)).max() == 0.0
    rng = np.random.default_rng(13)
    done = 0
    while done < 20:
        dg = int(rng.integers(0, 4))
        g = _rand_int_poly(rng, dg)
        u = _rand_int_poly(rng, 1 + int(rng.integers(0, 3)))
        v = _rand_int_poly(rng, 1 + int(rng.integers(0, 3)))
        if X.degree(X.gcd(u, v)) != 0:
            continue
        p, q = X.mul(g, u), X.mul(g, v)
        deg = max(X.degree(p), X.degree(q))
        pf, qf = [float(c) for c in p], [float(c) for c in q]
        for s in range(1, deg + 1):
            exact_singular = X.rank(X.bezout_block(p, q, s)) < s
            assert api.numerical_singularity(api.bezout_leading_block(pf, qf, s), 1e-9)[0] == exact_singular
        done += 1


def test_numerical_singularity(oracle, api):
    sing, ratio = api.numerical_singularity(np.eye(3), 1e-8)  # poly_test.cpp:196-209
    assert not sing and abs(ratio - 1.0) <= 1e-12
    sing, ratio = api.numerical_singularity(np.full((2, 2), 5.0), 1e-8)
    assert sing and ratio <= 1e-15
    sing, ratio = api.numerical_singularity(np.zeros((4, 4)), 1e-8)
    assert sing and ratio == 0.0
    rng = np.random.default_rng(3)
    for n in (3, 9, 25, 40):
        m = rng.uniform(-1, 1, (n, n)) + 1j * rng.uniform(-1, 1, (n, n))
        s_ref, r_ref = oracle.numerical_singularity(m, 1e-6)
        s, r = api.numerical_singularity(m, 1e-6)
        assert s == s_ref and abs(r - r_ref) <= 1e-9 * max(r_ref, 1e-300)
    with pytest.raises(api.CbpError) as e:
        api.numerical_singularity(np.eye(2), 1.5)
    assert e.value.code == "InvalidArgument"


def test_homogeneous_lsq(oracle, api):
    x = api.homogeneous_lsq(np.array([[1, 0], [0, 0]], complex))  # poly_test.cpp:262-268
    assert abs(x[0]) <= 1e-12 and abs(abs(x[1]) - 1) <= 1e-12
    rng = np.random.default_rng(5)                                 # :270-283
    c0 = rng.uniform(-1, 1, 6) + 1j * rng.uniform(-1, 1, 6)
    a = np.stack([c0, 2 * c0, rng.uniform(-1, 1, 6) + 0j], axis=1)
    x = api.homogeneous_lsq(a)
    assert np.linalg.norm(a @ x) <= 1e-12 * np.linalg.norm(a)
    assert abs(np.linalg.norm(x) - 1) <= 1e-12
    with pytest.raises(api.CbpError) as e:                         # :285-287
        api.homogeneous_lsq(np.ones((2, 3), complex))
    assert e.value.code == "InvalidArgument"
    # the scale system of a decode (t^2 x 2t at t = 7): same phase-normalized vector as the oracle
    for n_rows, n_cols in ((49, 14), (30, 30), (121, 22)):
        a = rng.uniform(-1, 1, (n_rows, n_cols)) + 1j * rng.uniform(-1, 1, (n_rows, n_cols))
        null = rng.uniform(-1, 1, n_cols) + 1j * rng.uniform(-1, 1, n_cols)
        a -= np.outer(a @ null, null.conj()) / np.vdot(null, null)  # planted null direction
        got, ref = api.homogeneous_lsq(a), oracle.homogeneous_lsq(a)
        assert np.abs(got - ref).max() <= 1e-10
        assert np.linalg.norm(a @ got) <= 1e-12 * np.linalg.norm(a)


def test_fft2_known_answers(oracle, api):
    d = np.zeros((3, 4)); d[0, 0] = 1                                 # fft_test.cpp:32-37
    assert np.abs(api.fft2(d) - 1).max() <= 1e-12
    i, j = np.meshgrid(np.arange(4), np.arange(5), indexing="ij")     # :39-45
    x = np.sin(0.7 * i + 0.3 * j) + 1j * np.cos(1.1 * i - 0.2 * j)
    u = np.arange(4)[:, None]
    v = np.arange(5)[:, None]
    direct = np.exp(-2j * np.pi * u * u.T / 4) @ x @ np.exp(-2j * np.pi * v * v.T / 5)
    assert np.abs(api.fft2(x) - direct).max() <= 1e-10
    for (r, c, seed) in [(5, 7, 17), (61, 97, 18)]:                   # :47-58
        x = oracle.random_mat(r, c, seed, -1, 1)
        back = api.ifft2(api.fft2(x))
        assert np.abs(back.real - x).max() <= 1e-10 and np.abs(back.imag).max() <= 1e-10
        assert np.abs(api.fft2(x) - oracle.fft2(x)).max() <= 1e-10 * max(1.0, np.abs(oracle.fft2(x)).max())
    a = oracle.random_mat(6, 5, 19)                                   # :60-71
    b = oracle.random_mat(3, 4, 20)
    pa = np.zeros((8, 8)); pa[:6, :5] = a
    pb = np.zeros((8, 8)); pb[:3, :4] = b
    back = api.ifft2(api.fft2(pa) * api.fft2(pb))
    assert np.abs(back.real - oracle.conv2_full(a, b)).max() <= 1e-10
    big = oracle.random_mat(270, 270, 21, -1, 1)  # a deblur grid (c1), vs numpy's pocketfft
    assert np.abs(api.fft2(big) - np.fft.fft2(big)).max() <= 1e-9
    assert math.isclose(abs(api.fft2(np.ones((7, 11)))[0, 0]), 77.0, rel_tol=1e-14)
