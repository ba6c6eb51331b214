"""Exact-arithmetic known-answer helpers for the tests (restating the reference's test
oracle, proj/tests/oracle/exact.hpp, with Python's fractions instead of
Boost.Multiprecision): rationals Q and the cyclotomic field Q(w), w = exp(-2 pi i / 3),
polynomial GCD, exact rank, Bezout blocks, cube-root and DC slices."""
from __future__ import annotations

from fractions import Fraction as Q
import math


class Eis:
    """a + b*w with w^2 = -1 - w (exact.hpp:28-75)."""
    __slots__ = ("a", "b")

    def __init__(self, a=0, b=0):
        self.a = Q(a)
        self.b = Q(b)

    def __add__(self, o):
        o = _eis(o)
        return Eis(self.a + o.a, self.b + o.b)

    __radd__ = __add__

    def __sub__(self, o):
        o = _eis(o)
        return Eis(self.a - o.a, self.b - o.b)

    def __rsub__(self, o):
        return _eis(o) - self

    def __neg__(self):
        return Eis(-self.a, -self.b)

    def __mul__(self, o):
        o = _eis(o)
        return Eis(self.a * o.a - self.b * o.b, self.a * o.b + self.b * o.a - self.b * o.b)

    __rmul__ = __mul__

    def conj(self):
        return Eis(self.a - self.b, -self.b)

    def norm(self):
        return self.a * self.a - self.a * self.b + self.b * self.b

    def inv(self):
        n = self.norm()
        c = self.conj()
        return Eis(c.a / n, c.b / n)

    def __truediv__(self, o):
        return self * _eis(o).inv()

    def is_zero(self):
        return self.a == 0 and self.b == 0

    def __eq__(self, o):
        o = _eis(o)
        return self.a == o.a and self.b == o.b

    def to_complex(self):
        s = math.sqrt(3.0) / 2.0
        return complex(float(self.a) - 0.5 * float(self.b), -s * float(self.b))


def _eis(x):
    return x if isinstance(x, Eis) else Eis(x, 0)


def is_zero(x):
    return x.is_zero() if isinstance(x, Eis) else x == 0


def inv(x):
    return x.inv() if isinstance(x, Eis) else 1 / Q(x)


def trim(p):
    p = list(p)
    while p and is_zero(p[-1]):
        p.pop()
    return p


def degree(p):
    return len(trim(p)) - 1


def mul(p, q):
    if not p or not q:
        return []
    out = [0 * p[0]] * (len(p) + len(q) - 1)
    out = [Q(0) if not isinstance(p[0], Eis) else Eis() for _ in range(len(p) + len(q) - 1)]
    for i, a in enumerate(p):
        for j, b in enumerate(q):
            out[i + j] = out[i + j] + a * b
    return trim(out)


def divmod_poly(a, b):
    a = trim(a)
    b = trim(b)
    if not b:
        raise ZeroDivisionError
    quo = [Q(0) if not isinstance(b[0], Eis) else Eis() for _ in range(max(len(a) - len(b) + 1, 1))]
    r = list(a)
    lead_inv = inv(b[-1])
    while len(trim(r)) >= len(b) and trim(r):
        r = trim(r)
        shift = len(r) - len(b)
        c = r[-1] * lead_inv
        quo[shift] = c
        for i, bc in enumerate(b):
            r[shift + i] = r[shift + i] - c * bc
        r = trim(r)
    return trim(quo), trim(r)


def gcd(a, b):
    a, b = trim(a), trim(b)
    while b:
        _, r = divmod_poly(a, b)
        a, b = b, r
    if not a:
        return []
    li = inv(a[-1])
    return [c * li for c in a]


def divexact(a, b):
    q, r = divmod_poly(a, b)
    assert not r
    return q


def bezout_block(p, q, size):
    """exact.hpp:175-190, same indexing as poly.cpp:66-79."""
    def c(v, i):
        return v[i] if 0 <= i < len(v) else Q(0)
    return [[sum((c(p, i + j + 1 - k) * c(q, k) - c(q, i + j + 1 - k) * c(p, k)
                  for k in range(min(i, j) + 1)), Q(0)) for j in range(size)] for i in range(size)]


def rank(m):
    """Exact rank by Gaussian elimination (exact.hpp:193-219)."""
    a = [list(r) for r in m]
    rows = len(a)
    cols = len(a[0]) if rows else 0
    rk = 0
    for c in range(cols):
        piv = next((r for r in range(rk, rows) if not is_zero(a[r][c])), None)
        if piv is None:
            continue
        a[rk], a[piv] = a[piv], a[rk]
        pi = inv(a[rk][c])
        for r in range(rows):
            if r != rk and not is_zero(a[r][c]):
                f = a[r][c] * pi
                a[r] = [x - f * y for x, y in zip(a[r], a[rk])]
        rk += 1
    return rk


def conv2(a, b):
    """Exact full 2-D convolution (exact.hpp:251-262)."""
    ra, ca, rb, cb = len(a), len(a[0]), len(b), len(b[0])
    out = [[Q(0)] * (ca + cb - 1) for _ in range(ra + rb - 1)]
    for i in range(ra):
        for j in range(ca):
            if a[i][j] == 0:
                continue
            for k in range(rb):
                for l in range(cb):
                    out[i + k][j + l] += a[i][j] * b[k][l]
    return out


def omega_pow(k):
    k %= 3
    return Eis(1, 0) if k == 0 else (Eis(0, 1) if k == 1 else Eis(-1, -1))


def cube_root_slice(m, axis, point):
    """exact.hpp:267-289: restriction at w^point along the axis (0 = Z1, 1 = Z2)."""
    rows, cols = len(m), len(m[0])
    if axis == 0:
        return trim([sum((Eis(m[r][n]) * omega_pow(point * r) for r in range(rows)), Eis()) for n in range(cols)])
    return trim([sum((Eis(m[r][n]) * omega_pow(point * n) for n in range(cols)), Eis()) for r in range(rows)])


def dc_slice(m, axis):
    rows, cols = len(m), len(m[0])
    if axis == 0:
        return trim([sum((m[r][n] for r in range(rows)), Q(0)) for n in range(cols)])
    return trim([sum((m[r][n] for n in range(cols)), Q(0)) for r in range(rows)])


def exact_width_from_slices(p, q, lo, hi):
    for s in range(lo, hi + 1, 2):
        if rank(bezout_block(p, q, s)) < s:
            return s
    return hi + 2


def to_complex_list(p):
    return [x.to_complex() if isinstance(x, Eis) else complex(float(x)) for x in p]
