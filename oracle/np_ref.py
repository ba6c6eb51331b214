"""CBP ORACLE CROSS-CHECK — TEST INFRASTRUCTURE ONLY.

An independent numpy restatement of the reference decode path that uses LAPACK
(numpy.linalg.svd) and pocketfft (numpy.fft) instead of the in-house Jacobi SVD and
mixed-radix FFT of oracle/cbp_oracle.cpp. Agreement between the two pins the C++
oracle's arithmetic (tests/test_oracle_vs_numpy.py). Follows the same reference
citations as the C++ oracle (proj/core/src/decoder.cpp, poly.cpp, fft.cpp).
"""
from __future__ import annotations

import numpy as np


def friendly_size(n: int) -> int:  # fft.cpp:272-280
    m = n
    while True:
        r = m
        for f in (2, 3, 5, 7):
            while r % f == 0:
                r //= f
        if r == 1:
            return m
        m += 1


def luma(planes: np.ndarray) -> np.ndarray:  # image.cpp:41-45
    if planes.shape[0] == 1:
        return planes[0].astype(np.float64)
    return 0.299 * planes[0] + 0.587 * planes[1] + 0.114 * planes[2]


def dft_matrix(t: int) -> np.ndarray:  # decoder.cpp:125-131
    i = np.arange(t)
    return np.exp(-2j * np.pi * ((i[:, None] * i[None, :]) % t) / t)


def axis_roots_dft(plane: np.ndarray, axis: int, t: int) -> np.ndarray:  # fft.cpp:197-213
    M, N = plane.shape
    W = dft_matrix(t)
    if axis == 0:
        fold = np.zeros((t, N))
        for r in range(t):
            fold[r] = plane[r::t].sum(axis=0)
        return W @ fold
    fold = np.zeros((M, t))
    for r in range(t):
        fold[:, r] = plane[:, r::t].sum(axis=1)
    return fold @ W


def bezout_leading_block(p, q, size: int) -> np.ndarray:  # poly.cpp:66-79
    def c(v, i):
        return v[i] if 0 <= i < len(v) else 0.0
    B = np.zeros((size, size), np.complex128)
    for i in range(size):
        for j in range(size):
            s = 0j
            for k in range(min(i, j) + 1):
                s += c(p, i + j + 1 - k) * c(q, k) - c(q, i + j + 1 - k) * c(p, k)
            B[i, j] = s
    return B


def singular_ratio(m: np.ndarray) -> float:  # poly.cpp:81-91
    sv = np.linalg.svd(m, compute_uv=False)
    return 0.0 if sv[0] == 0 else sv[-1] / sv[0]


def normalize_phase(x: np.ndarray) -> np.ndarray:  # poly.cpp:18-23
    i = int(np.argmax(np.abs(x)))
    a = abs(x[i])
    return x * (np.conj(x[i]) / a) if a > 0 else x


def cofactor_null_solve(p, q, t: int, gap_threshold: float = 1e-9):  # poly.cpp:93-121
    p = np.asarray(p, np.complex128); q = np.asarray(q, np.complex128)
    rows = max(len(p), len(q)) + t - 1
    A = np.zeros((rows, 2 * t), np.complex128)
    for j in range(t):
        A[j:j + len(p), j] = p
        A[j:j + len(q), t + j] = -q
    _, sv, vh = np.linalg.svd(A)
    full = np.zeros(2 * t)
    full[: len(sv)] = sv
    gap = 0.0 if full[0] == 0 else full[2 * t - 2] / full[0]
    if gap < gap_threshold:
        raise ArithmeticError("IllConditioned")
    x = normalize_phase(vh.conj().T[:, 2 * t - 1])
    return x[t:], x[:t], gap


def homogeneous_lsq(A: np.ndarray) -> np.ndarray:  # poly.cpp:123-130
    _, _, vh = np.linalg.svd(A)
    return normalize_phase(vh.conj().T[:, A.shape[1] - 1])


def estimate_width(l1, l2, smin, smax, tau):  # decoder.cpp:38-90 (nonnegative content)
    out = []
    for axis in (0, 1):
        p = (l1.sum(axis=0) if axis == 0 else l1.sum(axis=1)).astype(np.complex128)
        q = (l2.sum(axis=0) if axis == 0 else l2.sum(axis=1)).astype(np.complex128)
        w, clamped = smax, True
        for s in range(smin, smax + 1, 2):
            if singular_ratio(bezout_leading_block(p, q, s)) < tau:
                w, clamped = s, False
                break
        out.append((w, clamped))
    if out[0][0] != out[1][0]:
        raise ArithmeticError("InconsistentAxes")
    return out[0][0], out[0][1] and out[1][1]


def solve_axis(s1, s2, t, axis, gap_threshold=1e-9):  # decoder.cpp:94-123
    vals = np.zeros((t, t), np.complex128)
    gaps = np.zeros(t)
    for i in range(t):
        p = s1[i] if axis == 0 else s1[:, i]
        q = s2[i] if axis == 0 else s2[:, i]
        k1, _, g = cofactor_null_solve(p, q, t, gap_threshold)
        k1 = k1 / np.linalg.norm(k1)
        if axis == 0:
            vals[i] = k1
        else:
            vals[:, i] = k1
        gaps[i] = g
    return vals, gaps


def realize_kernel(k, max_imag=0.01, neg_tol=0.01):  # decoder.cpp:159-176
    mass = k.sum()
    k = k * (np.conj(mass) / abs(mass))
    total = (np.abs(k) ** 2).sum()
    if (k.imag ** 2).sum() > max_imag * total:
        raise ArithmeticError("NonRealKernel")
    w = k.real
    if w.min() < -neg_tol * w.max():
        raise ArithmeticError("NonRealKernel")
    w = np.maximum(w, 0.0)
    return w / w.sum()


def spectral_deblur(blurred, kernel, eps):  # decoder.cpp:187-214
    t = kernel.shape[0]
    Mb, Nb = blurred.shape
    Gr, Gc = friendly_size(Mb), friendly_size(Nb)
    FB = np.fft.rfft2(blurred, s=(Gr, Gc))
    FK = np.fft.rfft2(kernel, s=(Gr, Gc))
    full = np.fft.irfft2(FB * np.conj(FK) / (np.abs(FK) ** 2 + eps), s=(Gr, Gc))
    return full[: Mb - t + 1, : Nb - t + 1]


def decode_frame(pub, prv, smin=9, smax=25, tau=1e-6, epsilon=None, hint=None):
    """decoder.cpp:280-378 with LAPACK / pocketfft. pub, prv: (channels, M, N)."""
    l1, l2 = luma(pub), luma(prv)
    t = hint if hint is not None else estimate_width(l1, l2, smin, smax, tau)[0]
    a, _ = solve_axis(axis_roots_dft(l1, 0, t), axis_roots_dft(l2, 0, t), t, 0)
    b, _ = solve_axis(axis_roots_dft(l1, 1, t), axis_roots_dft(l2, 1, t), t, 1)
    W = dft_matrix(t)
    A, B = a @ W, W @ b
    sys_ = np.zeros((t * t, 2 * t), np.complex128)
    for i in range(t):
        for j in range(t):
            sys_[i * t + j, i] = -B[i, j]
            sys_[i * t + j, t + j] = A[i, j]
    x = homogeneous_lsq(sys_)
    lam, mu = x[:t], x[t:]
    ka = np.fft.ifft2(A / lam[:, None])
    kb = np.fft.ifft2(B / mu[None, :])
    k = 0.5 * (realize_kernel(ka) + realize_kernel(kb))
    Gr, Gc = friendly_size(pub.shape[1]), friendly_size(pub.shape[2])
    peak = np.abs(np.fft.rfft2(k, s=(Gr, Gc))).max()
    eps = 1e-8 * peak * peak if epsilon is None else epsilon
    latent = np.stack([spectral_deblur(pl, k, eps) for pl in pub])
    return latent, k, t
