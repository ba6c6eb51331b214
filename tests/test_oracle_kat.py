"""Pins the CPU oracle (oracle/cbp_oracle.cpp) against the reference's own known-answer
tests: proj/tests/unit/{poly,fft,decoder,encoder}_test.cpp and acceptance criteria 2, 3,
5, 7 (proj/tests/acceptance/acceptance.cpp), with the same tolerances. Exact-arithmetic
oracles (rational / cyclotomic) come from tests/exact.py."""
import math

import numpy as np
import pytest

import exact as X


def aligned_error(est, ref):
    """support.hpp:70-82: best complex scale aligning est to ref, then max abs error."""
    est = np.asarray(est, np.complex128).ravel()
    ref = np.asarray(ref, np.complex128).ravel()
    c = np.vdot(est, ref) / np.vdot(est, est)
    return float(np.abs(c * est - ref).max())


def aligned_error2(e1, e2, r1, r2):
    return aligned_error(np.concatenate([e1, e2]), np.concatenate([r1, r2]))


# ----------------------------------------------------------------- poly_test.cpp
def test_conv2_identity_and_hand_product(oracle):
    a = np.array([[1.0, 2], [3, 4]])
    assert np.array_equal(oracle.conv2_full(a, [[1.0]]), a)
    assert np.array_equal(oracle.conv2_full([[1.0]], a), a)
    assert np.array_equal(oracle.conv2_full(a, np.eye(2)), [[1, 2, 0], [3, 5, 2], [0, 3, 4]])
    c = oracle.conv2_full(np.ones((3, 3)), np.ones((2, 2)))
    assert c.shape == (4, 4) and abs(c.sum() - 36.0) <= 1e-12


def test_conv2_exact_on_integer_grids(oracle):
    rng = np.random.default_rng(11)
    for _ in range(8):
        a = rng.integers(-9, 10, size=(6, 5)).astype(float)
        b = rng.integers(-9, 10, size=(4, 3)).astype(float)
        ex = X.conv2([[X.Q(int(v)) for v in r] for r in a], [[X.Q(int(v)) for v in r] for r in b])
        got = oracle.conv2_full(a, b)
        assert np.array_equal(got, np.array([[float(v) for v in r] for r in ex]))


def test_conv2_commutative_and_direct_loop(oracle):
    a = oracle.random_mat(7, 4, 21)
    b = oracle.random_mat(3, 6, 22)
    ab = oracle.conv2_full(a, b)
    assert np.abs(ab - oracle.conv2_full(b, a)).max() <= 1e-12
    direct = np.zeros_like(ab, dtype=np.longdouble)
    for i in range(a.shape[0]):
        for j in range(a.shape[1]):
            direct[i:i + 3, j:j + 6] += np.longdouble(a[i, j]) * b.astype(np.longdouble)
    assert np.abs(ab - direct.astype(float)).max() <= 1e-12


def test_bezout_known_answers(oracle):
    assert oracle.bezout_leading_block([1, 2], [3, 1], 1)[0, 0] == 5
    b = oracle.bezout_leading_block([1, 3, 2], [3, 4, 1], 2)
    assert np.array_equal(b, np.full((2, 2), 5.0 + 0j))
    assert oracle.numerical_singularity(b, 1e-8)[0]
    rng = np.random.default_rng(44)
    p = rng.uniform(-1, 1, 6) + 1j * rng.uniform(-1, 1, 6)
    assert np.abs(oracle.bezout_leading_block(p, p, 5)).max() == 0.0


def _rand_int_poly(rng, deg, bound=5):
    p = [int(v) for v in rng.integers(-bound, bound + 1, deg + 1)]
    while p[-1] == 0:
        p[-1] = int(rng.integers(-bound, bound + 1))
    if p[0] == 0:
        p[0] = 1
    return [X.Q(v) for v in p]


def test_bezout_antisymmetry_bitwise(oracle):
    rng = np.random.default_rng(7)
    for _ in range(12):
        p = _rand_int_poly(rng, 3 + int(rng.integers(0, 4)))
        q = _rand_int_poly(rng, 3 + int(rng.integers(0, 4)))
        size = max(X.degree(p), X.degree(q))
        pf = [float(v) for v in p]
        qf = [float(v) for v in q]
        pq = oracle.bezout_leading_block(pf, qf, size)
        qp = oracle.bezout_leading_block(qf, pf, size)
        assert np.abs(pq + qp).max() == 0.0


def test_bezout_rank_law_against_exact_arithmetic(oracle):
    """poly_test.cpp:193-218 and acceptance criterion 4 (rank = degree - gcd degree)."""
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
        assert X.rank(X.bezout_block(p, q, deg)) == deg - dg
        pf, qf = [float(c) for c in p], [float(c) for c in q]
        for s in range(1, deg + 1):
            exact_singular = X.rank(X.bezout_block(p, q, s)) < s
            assert oracle.numerical_singularity(oracle.bezout_leading_block(pf, qf, s), 1e-9)[0] == exact_singular
        done += 1


def test_numerical_singularity_cases(oracle):
    sing, ratio = oracle.numerical_singularity(np.eye(3), 1e-8)
    assert not sing and abs(ratio - 1.0) <= 1e-12
    sing, ratio = oracle.numerical_singularity(np.full((2, 2), 5.0), 1e-8)
    assert sing and ratio <= 1e-15
    sing, ratio = oracle.numerical_singularity(np.zeros((4, 4)), 1e-8)
    assert sing and ratio == 0.0


def test_cofactor_known_answers(oracle):
    k1, k2, gap = oracle.cofactor_null_solve([1, 3, 2], [3, 4, 1], 2)
    assert aligned_error2(k1, k2, [1, 2], [3, 1]) <= 1e-12
    assert gap > 1e-3
    k1, k2, _ = oracle.cofactor_null_solve([1, 1], [1, 1], 1)
    assert abs(k1[0] - k2[0]) <= 1e-14 and abs(abs(k1[0]) - 1 / math.sqrt(2)) <= 1e-12
    b1, b2, _ = oracle.cofactor_null_solve([1, 3, 2], [3, 4, 1], 2)
    s1, s2, _ = oracle.cofactor_null_solve(2j * np.array([1, 3, 2]), 2j * np.array([3, 4, 1]), 2)
    assert aligned_error2(s1, s2, b1, b2) <= 1e-12
    with pytest.raises(oracle.OracleError) as e:
        oracle.cofactor_null_solve([1, 2, 1], [1, 2, 1], 2)
    assert e.value.code == "IllConditioned"


def test_cofactor_planted_common_factor(oracle):
    rng = np.random.default_rng(99)
    for _ in range(6):
        l = rng.uniform(-1, 1, 7) + 1j * rng.uniform(-1, 1, 7)
        u = rng.uniform(-1, 1, 3) + 1j * rng.uniform(-1, 1, 3)
        v = rng.uniform(-1, 1, 3) + 1j * rng.uniform(-1, 1, 3)
        k1, k2, _ = oracle.cofactor_null_solve(np.convolve(l, u), np.convolve(l, v), 3)
        assert aligned_error2(k1, k2, u, v) <= 1e-8


def test_homogeneous_lsq(oracle):
    x = oracle.homogeneous_lsq(np.array([[1, 0], [0, 0]], complex))
    assert abs(x[0]) <= 1e-12 and abs(abs(x[1]) - 1) <= 1e-12
    rng = np.random.default_rng(5)
    c0 = rng.uniform(-1, 1, 6) + 1j * rng.uniform(-1, 1, 6)
    a = np.stack([c0, 2 * c0, rng.uniform(-1, 1, 6) + 0j], axis=1)
    x = oracle.homogeneous_lsq(a)
    assert np.linalg.norm(a @ x) <= 1e-12 * np.linalg.norm(a)
    assert abs(np.linalg.norm(x) - 1) <= 1e-12
    with pytest.raises(oracle.OracleError):
        oracle.homogeneous_lsq(np.ones((2, 3), complex))


def test_sylvester_and_degree(oracle):
    s = oracle.sylvester_matrix([1, 2], [3, 1])
    assert abs(abs(np.linalg.det(s)) - 5.0) <= 1e-12
    s = oracle.sylvester_matrix([1, 3, 2], [3, 4, 1])
    assert oracle.numerical_singularity(s, 1e-10)[0]
    assert oracle.numerical_degree([0, 1, 1e-15]) == 1
    assert oracle.numerical_degree([5]) == 0
    assert oracle.numerical_degree([0, 0, 0, 0]) == -1


# ------------------------------------------------------------------ fft_test.cpp
def _direct_dft2(x):
    m, n = x.shape
    u = np.arange(m)[:, None]
    v = np.arange(n)[:, None]
    return np.exp(-2j * np.pi * u * u.T / m) @ x @ np.exp(-2j * np.pi * v * v.T / n)


def test_fft2_known_answers(oracle):
    d = np.zeros((3, 4)); d[0, 0] = 1
    assert np.abs(oracle.fft2(d) - 1).max() <= 1e-12
    i, j = np.meshgrid(np.arange(4), np.arange(5), indexing="ij")
    x = np.sin(0.7 * i + 0.3 * j) + 1j * np.cos(1.1 * i - 0.2 * j)
    assert np.abs(oracle.fft2(x) - _direct_dft2(x)).max() <= 1e-10
    for (r, c, seed) in [(5, 7, 17), (61, 97, 18)]:
        x = oracle.random_mat(r, c, seed, -1, 1)
        back = oracle.ifft2(oracle.fft2(x))
        assert np.abs(back.real - x).max() <= 1e-10 and np.abs(back.imag).max() <= 1e-10


def test_fft_convolution_theorem(oracle):
    a = oracle.random_mat(6, 5, 19)
    b = oracle.random_mat(3, 4, 20)
    pa = np.zeros((8, 8)); pa[:6, :5] = a
    pb = np.zeros((8, 8)); pb[:3, :4] = b
    back = oracle.ifft2(oracle.fft2(pa) * oracle.fft2(pb))
    assert np.abs(back.real - oracle.conv2_full(a, b)).max() <= 1e-10


def test_axis_roots_dft_known_answers(oracle):
    plane = oracle.random_mat(6, 7, 23)
    for axis in (0, 1):
        got = oracle.axis_roots_dft(plane, axis, 5)
        pts = np.exp(-2j * np.pi * np.arange(5) / 5)
        for i, w in enumerate(pts):
            if axis == 0:
                ref = (plane * (w ** np.arange(6))[:, None]).sum(axis=0)
                assert np.abs(got[i] - ref).max() <= 1e-12
            else:
                ref = (plane * (w ** np.arange(7))[None, :]).sum(axis=1)
                assert np.abs(got[:, i] - ref).max() <= 1e-12
    plane = oracle.random_mat(8, 6, 29, -1, 1)
    s = oracle.axis_roots_dft(plane, 0, 8)
    w = np.exp(2j * np.pi * np.arange(8)[:, None] * np.arange(8)[None, :] / 8)
    back = (w @ s) / 8
    assert np.abs(back.real - plane).max() <= 1e-10 and np.abs(back.imag).max() <= 1e-10
    plane = oracle.random_mat(4, 5, 31)
    assert np.abs(oracle.axis_roots_dft(plane, 0, 1)[0].real - plane.sum(axis=0)).max() <= 1e-12
    assert np.abs(oracle.axis_roots_dft(plane, 1, 1)[:, 0].real - plane.sum(axis=1)).max() <= 1e-12


def test_friendly_size(oracle):
    assert [oracle.friendly_size(n) for n in (1, 11, 262, 488, 648, 1090, 1930, 2174, 3854)] == \
        [1, 12, 270, 490, 648, 1120, 1944, 2187, 3888]


# -------------------------------------------------------------- decoder_test.cpp
def _encode(oracle, latent, pair):
    return oracle.encode_frame(latent, pair.k1, pair.k2)


@pytest.mark.parametrize("size,t,lo,hi,want,clamped,kseed,lseed", [
    (24, 5, 3, 7, 5, False, 101, 101), (20, 3, 3, 9, 3, False, 102, 102),
    (64, 25, 9, 25, 25, None, 101, 103), (64, 27, 9, 25, 25, True, 101, 104)])
def test_estimate_width(oracle, size, t, lo, hi, want, clamped, kseed, lseed):
    lat = oracle.random_mat(size, size, lseed)
    pair = oracle.generate_coprime_pair(t, kseed)
    pub, prv = _encode(oracle, lat, pair)
    w, c = oracle.estimate_kernel_width(pub, prv, lo, hi, 1e-6)
    assert w == want
    if clamped is not None:
        assert c == clamped


def test_estimate_width_inconsistent_axes(oracle):
    lat = oracle.random_mat(16, 16, 105)
    a1 = oracle.random_mat(3, 5, 106, 0.05, 1.0)
    a2 = oracle.random_mat(3, 5, 107, 0.05, 1.0)
    with pytest.raises(oracle.OracleError) as e:
        oracle.estimate_kernel_width(oracle.conv2_full(lat, a1), oracle.conv2_full(lat, a2), 3, 7, 1e-6)
    assert e.value.code == "InconsistentAxes"


def test_sample_cofactors(oracle):
    pair = oracle.generate_coprime_pair(3, 111)
    z1, _ = oracle.sample_cofactors(pair.k1, pair.k2, 3, 0)
    ref1 = oracle.axis_roots_dft(pair.k1, 0, 3)
    for i in range(3):
        assert aligned_error(z1[i], ref1[i]) <= 1e-10
    z2, _ = oracle.sample_cofactors(pair.k1, pair.k2, 3, 1)
    ref2 = oracle.axis_roots_dft(pair.k1, 1, 3)
    for j in range(3):
        assert aligned_error(z2[:, j], ref2[:, j]) <= 1e-10
    lat = oracle.random_mat(16, 16, 113)
    pair = oracle.generate_coprime_pair(3, 113)
    pub, prv = _encode(oracle, lat, pair)
    vals, gaps = oracle.sample_cofactors(pub, prv, 3, 0)
    ref = oracle.axis_roots_dft(pair.k1, 0, 3)
    for i in range(3):
        assert abs(np.linalg.norm(vals[i]) - 1) <= 1e-9
        assert aligned_error(vals[i], ref[i]) <= 1e-8
        assert gaps[i] > 1e-6
    with pytest.raises(oracle.OracleError) as e:
        oracle.sample_cofactors(np.zeros((8, 8)), np.zeros((8, 8)), 3, 0)
    assert e.value.code == "IllConditionedSlice"


def test_complete_resolve_assemble(oracle):
    pair = oracle.generate_coprime_pair(5, 115)
    spec = np.fft.fft2(pair.k1)
    for axis in (0, 1):
        got = oracle.complete_to_spectrum(oracle.axis_roots_dft(pair.k1, axis, 5), axis)
        assert np.abs(got - spec).max() <= 1e-10
    pair = oracle.generate_coprime_pair(3, 117)
    lam, mu, res = oracle.resolve_scales(oracle.axis_roots_dft(pair.k1, 0, 3), oracle.axis_roots_dft(pair.k1, 1, 3))
    assert res <= 1e-12
    assert np.abs(lam - lam[0]).max() <= 1e-12 and np.abs(mu - mu[0]).max() <= 1e-12
    assert abs(lam[0] - mu[0]) <= 1e-12
    assert abs(math.sqrt(np.linalg.norm(lam) ** 2 + np.linalg.norm(mu) ** 2) - 1) <= 1e-12
    # planted scales (decoder_test.cpp:158-177)
    pair = oracle.generate_coprime_pair(3, 119)
    a = oracle.axis_roots_dft(pair.k1, 0, 3)
    b = oracle.axis_roots_dft(pair.k1, 1, 3)
    s = np.array([0.5 + 0.3 * i for i in range(3)]) * np.exp(1j * 0.7 * np.arange(3))
    r = np.array([1.1 - 0.2 * i for i in range(3)]) * np.exp(1j * (-0.4 * np.arange(3) + 0.2))
    lam, mu, res = oracle.resolve_scales(a * s[:, None], b * r[None, :])
    assert res <= 1e-9
    c0 = lam[0] / s[0]
    assert np.abs(lam - c0 * s).max() <= 1e-9 and np.abs(mu - c0 * r).max() <= 1e-9
    # degenerate scales
    pair = oracle.generate_coprime_pair(3, 121)
    a = oracle.axis_roots_dft(pair.k1, 0, 3)
    a[0] = 0
    with pytest.raises(oracle.OracleError) as e:
        oracle.resolve_scales(a, oracle.axis_roots_dft(pair.k1, 1, 3))
    assert e.value.code == "DegenerateScales"
    # assemble undoes planted scales (decoder_test.cpp:224-247)
    pair = oracle.generate_coprime_pair(3, 123)
    spec = np.fft.fft2(pair.k1)
    lam = np.array([0.8 + 0.2 * i for i in range(3)]) * np.exp(1j * (0.3 * np.arange(3) - 0.5))
    mu = np.array([1.2 - 0.1 * i for i in range(3)]) * np.exp(1j * (0.6 - 0.2 * np.arange(3)))
    joint = math.sqrt(np.linalg.norm(lam) ** 2 + np.linalg.norm(mu) ** 2)
    lam, mu = lam / joint, mu / joint
    k = oracle.assemble_kernel(lam[:, None] * spec, spec * mu[None, :], lam, mu)
    assert np.abs(k - pair.k1).max() <= 1e-8 and abs(k.sum() - 1) <= 1e-9 and k.min() >= 0
    junk = np.array([[math.sin(i + 2.0 * j) + 1j * math.cos(3.0 * i - j) for j in range(3)] for i in range(3)])
    c = 1 / math.sqrt(6)
    with pytest.raises(oracle.OracleError) as e:
        oracle.assemble_kernel(c * junk, junk * c, np.full(3, c), np.full(3, c))
    assert e.value.code == "NonRealKernel"


def test_spectral_deblur_known_answers(oracle):
    b = oracle.random_mat(9, 7, 131)
    assert np.abs(oracle.spectral_deblur(b, [[1.0]], 0.0) - b).max() <= 1e-12
    lat = oracle.random_mat(16, 16, 133)
    pair = oracle.generate_coprime_pair(3, 133)
    back = oracle.spectral_deblur(oracle.conv2_full(lat, pair.k1), pair.k1, 1e-12)
    assert back.shape == (16, 16) and oracle.psnr(lat, back) >= 80.0
    one = np.array([[0.5, 0.0, 0.5]])
    comb = oracle.conv2_full(one.T, one)
    lat = oracle.random_mat(6, 6, 135)
    back = oracle.spectral_deblur(oracle.conv2_full(lat, comb), comb, 1e-8)
    assert np.isfinite(back).all() and np.abs(back).max() <= 10.0


def test_decode_frame_round_trip_and_hint(oracle):
    lat = oracle.random_mat(64, 64, 137)
    pair = oracle.generate_coprime_pair(5, 137)
    pub, prv = _encode(oracle, lat, pair)
    d = oracle.decode_frame(pub, prv, hint=5, cfg=oracle.make_cfg(3, 9))
    assert d.width_used == 5 and not d.width_clamped
    assert oracle.psnr(lat, d.latent[0]) >= 40.0
    assert d.validation_residual <= 1e-4
    assert np.abs(d.kernel - pair.k1).max() <= 1e-6
    lat = oracle.random_mat(48, 40, 139)
    pair = oracle.generate_coprime_pair(5, 139)
    pub, prv = _encode(oracle, lat, pair)
    est = oracle.decode_frame(pub, prv, hint=5, cfg=oracle.make_cfg(3, 9))
    hinted = oracle.decode_frame(pub, prv, hint=5, cfg=oracle.make_cfg(3, 9, trust_hint=True))
    assert hinted.width_used == 5
    assert np.array_equal(hinted.latent, est.latent) and np.array_equal(hinted.kernel, est.kernel)


def test_decode_frame_adversarial_and_equivariance(oracle):
    la, lb = oracle.random_mat(24, 24, 141), oracle.random_mat(24, 24, 142)
    pair = oracle.generate_coprime_pair(3, 141)
    pub, prv = oracle.conv2_full(la, pair.k1), oracle.conv2_full(lb, pair.k2)
    try:
        d = oracle.decode_frame(pub, prv, hint=3, cfg=oracle.make_cfg(3, 7, trust_hint=True))
        flagged = d.validation_residual > 0.1
    except oracle.OracleError:
        flagged = True
    assert flagged
    lat = oracle.random_mat(32, 32, 143)
    pair = oracle.generate_coprime_pair(3, 143)
    pub, prv = _encode(oracle, lat, pair)
    ref = oracle.decode_frame(pub, prv, cfg=oracle.make_cfg(3, 7))
    got = oracle.decode_frame(2 * pub, 2 * prv, cfg=oracle.make_cfg(3, 7))
    assert np.abs(got.kernel - ref.kernel).max() <= 1e-9
    assert np.linalg.norm(got.latent - 2 * ref.latent) / np.linalg.norm(2 * ref.latent) <= 1e-6
    lat = oracle.random_mat(32, 32, 145)
    pair = oracle.generate_coprime_pair(3, 145)
    pub, prv = _encode(oracle, lat, pair)
    cfg = oracle.make_cfg(3, 7, epsilon=1e-12)
    ref = oracle.decode_frame(pub, prv, cfg=cfg)
    sw = oracle.decode_frame(prv, pub, cfg=cfg)
    assert np.abs(ref.kernel - pair.k1).max() <= 1e-8 and np.abs(sw.kernel - pair.k2).max() <= 1e-8
    assert np.linalg.norm(sw.latent - ref.latent) / np.linalg.norm(ref.latent) <= 1e-6


def test_decode_frame_rgb_u16_zero_and_validate(oracle):
    lat = np.stack([oracle.random_mat(24, 24, s) for s in (147, 148, 149)])
    pair = oracle.generate_coprime_pair(3, 147)
    pub, prv = _encode(oracle, lat, pair)
    d = oracle.decode_frame(pub, prv, cfg=oracle.make_cfg(3, 7))
    assert d.latent.shape[0] == 3 and oracle.psnr(lat, d.latent) >= 40.0
    lat = oracle.random_mat(48, 48, 153)
    pair = oracle.generate_coprime_pair(5, 153)
    pub, prv = _encode(oracle, lat, pair)
    d = oracle.decode_frame(oracle.quantize(pub, 16), oracle.quantize(prv, 16), hint=5,
                            cfg=oracle.make_cfg(3, 9, trust_hint=True))
    assert oracle.psnr(lat, d.latent[0]) >= 40.0 and d.validation_residual <= 1e-2
    with pytest.raises(oracle.OracleError):
        oracle.decode_frame(np.zeros((12, 12)), np.zeros((12, 12)), hint=3, cfg=oracle.make_cfg(3, 7, trust_hint=True))
    lat = oracle.random_mat(24, 24, 151)
    pair = oracle.generate_coprime_pair(3, 151)
    pub, prv = _encode(oracle, lat, pair)
    assert oracle.decode_frame(pub, prv, cfg=oracle.make_cfg(3, 7, validate=False)).validation_residual == 0.0


def test_validate_pair(oracle):
    lat = oracle.random_mat(16, 16, 155)
    pair = oracle.generate_coprime_pair(3, 155)
    pub, prv = _encode(oracle, lat, pair)
    assert oracle.validate_pair(pub, prv, pair.k1, pair.k2) <= 1e-10
    bad = oracle.conv2_full(oracle.random_mat(16, 16, 156), pair.k2)
    assert oracle.validate_pair(pub, bad, pair.k1, pair.k2) > 0.1


# -------------------------------------------------------------- encoder_test.cpp
def test_generate_coprime_pair(oracle):
    a = oracle.generate_coprime_pair(9, 42)
    b = oracle.generate_coprime_pair(9, 42)
    assert a.coprimality_margin > 1e-6 and np.array_equal(a.k1, b.k1) and np.array_equal(a.k2, b.k2)
    p = oracle.generate_coprime_pair(3, 7)
    for k in (p.k1, p.k2):
        assert k.shape == (3, 3) and k.min() >= 0 and abs(k.sum() - 1) <= 1e-9
    for w in (4, 1, 65):
        with pytest.raises(oracle.OracleError):
            oracle.generate_coprime_pair(w, 1)
    rejected = 0
    for seed in range(200):
        try:
            oracle.generate_coprime_pair(5, seed, max_retries=1)
        except oracle.OracleError as e:
            assert e.code == "CoprimalityFailure"
            rejected += 1
    assert rejected < 5


def test_coprimality_check(oracle):
    center = np.zeros((3, 3)); center[1, 1] = 1
    corner = np.zeros((3, 3)); corner[0, 0] = 1
    assert oracle.coprimality_check(center, corner) > 1e-3
    assert oracle.coprimality_check(center, center) <= 1e-12
    shared = np.array([[0.3, 0.1], [0.2, 0.4]])
    k1 = oracle.conv2_full(oracle.random_mat(2, 2, 61, 0.05, 1.0), shared)
    k2 = oracle.conv2_full(oracle.random_mat(2, 2, 62, 0.05, 1.0), shared)
    assert oracle.coprimality_check(k1 / k1.sum(), k2 / k2.sum()) <= 1e-8


def test_encode_frame(oracle):
    lat = np.array([[1.0, 2], [3, 4]]) / 4
    pub, prv = oracle.encode_frame(lat, [[1.0]], [[1.0]])
    assert np.array_equal(pub[0], lat) and np.array_equal(prv[0], lat)
    pair = oracle.generate_coprime_pair(3, 5)
    pub, prv = oracle.encode_frame(np.ones((8, 8)), pair.k1, pair.k2)
    for f in (pub, prv):
        assert f.shape == (1, 10, 10) and np.abs(f[0, 2:8, 2:8] - 1).max() <= 1e-9


# ------------------------------------------------------------- acceptance.cpp
def _int_instance(rng, t):
    """acceptance.cpp:99-146 (integer latent and kernels, exact rational blur)."""
    rows = 8 if t == 1 else 6 + int(rng.integers(0, 3))
    cols = 8 if t == 1 else 6 + int(rng.integers(0, 3))
    lat = rng.integers(0, 10, size=(rows, cols)).astype(float)
    lat[0, 0] = max(lat[0, 0], 1.0)
    lat[-1, -1] = max(lat[-1, -1], 1.0)
    k1 = rng.integers(1, 10, size=(t, t)).astype(float)
    k2 = rng.integers(1, 10, size=(t, t)).astype(float)
    lr = [[X.Q(int(v)) for v in r] for r in lat]
    k1r = [[X.Q(int(v)) / int(k1.sum()) for v in r] for r in k1]
    k2r = [[X.Q(int(v)) / int(k2.sum()) for v in r] for r in k2]
    b1r, b2r = X.conv2(lr, k1r), X.conv2(lr, k2r)
    return t, lat, k1 / k1.sum(), k2 / k2.sum(), b1r, b2r


def test_acceptance_2_cofactors_vs_cyclotomic_oracle(oracle):
    """Criterion 2: cofactor solves at the cube roots of unity agree with exact GCD
    cofactors (aligned error <= 1e-8); exact widths are recovered."""
    rng = np.random.default_rng(20250203)
    cases = 0
    while cases < 12:
        t = 1 if cases % 6 == 5 else 3
        t, lat, k1, k2, b1r, b2r = _int_instance(rng, t)
        b1f, b2f = oracle.conv2_full(lat, k1), oracle.conv2_full(lat, k2)
        refs, ok = [], True
        for axis in (0, 1):
            for pt in range(t):
                p = X.cube_root_slice(b1r, axis, 0 if t == 1 else pt)
                q = X.cube_root_slice(b2r, axis, 0 if t == 1 else pt)
                g = X.gcd(p, q)
                u, v = X.divexact(p, g), X.divexact(q, g)
                if X.degree(u) != t - 1 or X.degree(v) != t - 1:
                    ok = False
                refs.append((X.to_complex_list(u), X.to_complex_list(v)))
        w1 = X.exact_width_from_slices(X.dc_slice(b1r, 0), X.dc_slice(b2r, 0), 3, 7)
        w2 = X.exact_width_from_slices(X.dc_slice(b1r, 1), X.dc_slice(b2r, 1), 3, 7)
        if not ok or w1 != w2 or w1 > 7:
            continue
        slot = 0
        for axis in (0, 1):
            s1 = oracle.axis_roots_dft(b1f, axis, t)
            s2 = oracle.axis_roots_dft(b2f, axis, t)
            for pt in range(t):
                p = s1[pt] if axis == 0 else s1[:, pt]
                q = s2[pt] if axis == 0 else s2[:, pt]
                c1, c2, _ = oracle.cofactor_null_solve(p, q, t)
                assert aligned_error2(c1, c2, refs[slot][0], refs[slot][1]) <= 1e-8
                slot += 1
        w, clamped = oracle.estimate_kernel_width(b1f, b2f, 3, 7, 1e-6)
        assert w == w1 and not clamped
        cases += 1


def test_acceptance_3_width_recovery_rate(oracle):
    """Criterion 3 (subset): width recovered in >= 98% of trials."""
    correct = total = 0
    for t in (3, 5, 7, 9):
        for s in range(1, 6):
            seed = oracle.frame_seed(300 + t, s)
            lat = oracle.random_frame(96, 96, 1, seed)
            pair = oracle.generate_coprime_pair(t, oracle.frame_seed(seed, 9001))
            pub, prv = oracle.encode_frame(lat, pair.k1, pair.k2)
            total += 1
            try:
                w, c = oracle.estimate_kernel_width(pub, prv, 3, 9, 1e-6)
                correct += int(w == t and not c)
            except oracle.OracleError:
                pass
    assert correct / total >= 0.98


def test_acceptance_5_validation_separation(oracle):
    worst_true, best_adv = 0.0, float("inf")
    for i in range(8):
        t = (3, 5, 9)[i % 3]
        n = (16, 20, 24, 28, 32)[i % 5]
        lat = oracle.random_frame(n, n, 1, oracle.frame_seed(500, i))
        pair = oracle.generate_coprime_pair(t, oracle.frame_seed(501, i))
        pub, prv = oracle.encode_frame(lat, pair.k1, pair.k2)
        worst_true = max(worst_true, oracle.validate_pair(pub, prv, pair.k1, pair.k2))
        ta = 3 if i % 2 == 0 else 5
        pa = oracle.generate_coprime_pair(ta, oracle.frame_seed(503, i))
        other = oracle.random_frame(n, n, 1, oracle.frame_seed(502, i))
        fp, _ = oracle.encode_frame(lat, pa.k1, pa.k2)
        _, fq = oracle.encode_frame(other, pa.k1, pa.k2)
        best_adv = min(best_adv, oracle.validate_pair(fp, fq, pa.k1, pa.k2))
    assert worst_true <= 1e-10 and best_adv > 0.1


def test_acceptance_7_equivariance(oracle):
    lat = oracle.random_mat(48, 48, 700)
    pair = oracle.generate_coprime_pair(5, 701)
    pub, prv = oracle.encode_frame(lat, pair.k1, pair.k2)
    cfg = oracle.make_cfg(3, 9, epsilon=1e-12)
    base = oracle.decode_frame(pub, prv, cfg=cfg)
    for c in (0.5, 2.0):
        d = oracle.decode_frame(c * pub, c * prv, cfg=cfg)
        assert np.linalg.norm(d.latent - c * base.latent) / np.linalg.norm(c * base.latent) <= 1e-6
        assert np.abs(d.kernel - base.kernel).max() <= 1e-9
    m = oracle.decode_frame(prv, pub, cfg=cfg)
    assert np.linalg.norm(m.latent - base.latent) / np.linalg.norm(base.latent) <= 1e-6


def test_acceptance_1_reconstruction_subset(oracle):
    """Criterion 1 (subset): PSNR >= 40 dB and residual <= 1e-4 at 64x64, t in {3,5,9}."""
    for t in (3, 5, 9):
        for s in (1, 2, 3):
            lat = oracle.random_frame(64, 64, 1, oracle.frame_seed(100 + t, s))
            pair = oracle.generate_coprime_pair(t, oracle.frame_seed(100 + 31 * t, s))
            pub, prv = oracle.encode_frame(lat, pair.k1, pair.k2)
            d = oracle.decode_frame(pub, prv, cfg=oracle.make_cfg(3, 9))
            assert oracle.psnr(lat, d.latent) >= 40.0 and d.validation_residual <= 1e-4


def test_signed_content_width_and_decode(oracle):
    """Signed latents (decoder.cpp:65-82): the maximum-energy axis_spectrum_half slices
    carry the planted width; the decode reconstructs (the reference's planted-width and
    round-trip checks, decoder_test.cpp:40-83, 311-331, on zero-mean content)."""
    for rows, cols, t, hi in ((64, 64, 5, 9), (96, 128, 9, 25)):
        lat = oracle.random_frame(rows, cols, 1, oracle.frame_seed(3, rows + t)) - 0.5
        pair = oracle.generate_coprime_pair(t, oracle.frame_seed(4, cols + t))
        pub, prv = oracle.encode_frame(lat, pair.k1, pair.k2)
        assert oracle.estimate_kernel_width(pub, prv, 3, hi, 1e-6) == (t, False)
        d = oracle.decode_frame(pub, prv, cfg=oracle.make_cfg(3, hi))
        assert d.width_used == t and oracle.psnr(lat, d.latent) >= 40.0
        # the spectra the slices come from: axis_spectrum_half == numpy rfft along the axis
        luma = pub[0]
        np.testing.assert_allclose(oracle.axis_spectrum_half(luma, 0), np.fft.rfft(luma, axis=0), rtol=0, atol=1e-10)
        np.testing.assert_allclose(oracle.axis_spectrum_half(luma, 1), np.fft.rfft(luma, axis=1), rtol=0, atol=1e-10)


def test_quantize_and_degrade_kats(oracle):
    """encoder_test.cpp:170-215: rounding to the nearest level, idempotence, half-level error
    bound, range check, degrade_bits masking."""
    half = np.full((1, 2, 2), 0.5)
    assert oracle.quantize(half, 8)[0, 0, 0] == 128.0 / 255.0
    assert oracle.quantize(half, 16)[0, 0, 0] == 32768.0 / 65535.0
    f = oracle.random_mat(6, 6, 91)
    once = oracle.quantize(f, 8)
    assert np.array_equal(once, oracle.quantize(once, 8))
    g = oracle.random_mat(16, 16, 92)
    assert np.abs(oracle.quantize(g, 16)[0] - g).max() <= 0.5 / 65535.0 + 1e-15
    for bad in (1.1, -0.5):
        with pytest.raises(oracle.OracleError) as e:
            oracle.quantize(np.full((1, 2, 2), bad), 8)
        assert e.value.status == 7  # 1 + Errc::range_exceeded
    assert oracle.quantize(np.full((1, 2, 2), 1.0 + 5e-10), 8)[0, 0, 0] == 1.0
    assert oracle.degrade_bits(np.full((1, 1, 1), 183.0 / 255.0), 8, 3)[0, 0, 0] == 176.0 / 255.0
    assert oracle.degrade_bits(np.full((1, 1, 1), 258.0 / 65535.0), 16, 8)[0, 0, 0] == 256.0 / 65535.0
    with pytest.raises(oracle.OracleError) as e:
        oracle.degrade_bits(np.full((1, 1, 1), 0.5), 8, 8)
    assert e.value.status == 1  # 1 + Errc::invalid_argument: drop outside [0, bits)
