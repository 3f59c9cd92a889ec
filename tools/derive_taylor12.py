"""Derive coefficients of a degree-12 Taylor evaluation in 4 matrix products
(Bader-Blanes-Casas-type scheme; A15):
    A2 = A^2, A3 = A2 A
    B4 = b1 A + b2 A2 + b3 A3
    A6 = B3 + B4^2,            B3 = a0 I + a1 A + a2 A2 + a3 A3
    T12 = B1 + (B2 + A6) A6,   B1, B2 = x0 I + x1 A + x2 A2 + x3 A3
    T12 == sum_{k<=12} A^k / k!   (exactly, as polynomials)
Write p = B3 + B4^2 (degree 6) and q = B2 + p.  Degrees 12..7 of q p fix p6, p5, p4 and the sums
s_i = q_i + p_i (i = 3, 2, 1) top-down; degrees 6, 5, 4 leave 3 polynomial equations in
(p0, p1, p2, p3, q0): a two-parameter family.  For a grid of (p0, p1) the remaining unknowns are solved
in 50-digit arithmetic; every solution is tested in double precision for rounding stability on random
matrices of 1-norm theta12 (and anti-Hermitian ones, the generators' character); the most stable one is
printed as C literals.  B1 = the degrees 0..3 that q p does not produce.  theta12 is the largest theta
with sum_{k>12} theta^k/k! <= 2^-53 e^-theta (the rule of THETA_T8 / THETA_T18).
"""
import itertools
import math

import mpmath as mp
import numpy as np

mp.mp.dps = 50
c = [mp.mpf(1) / mp.factorial(k) for k in range(13)]


def top(s6):
    p6 = s6 * mp.sqrt(c[12])
    p5 = c[11] / (2 * p6)
    p4 = (c[10] - p5 ** 2) / (2 * p6)
    s3 = (c[9] - 2 * p4 * p5) / p6
    s2 = (c[8] - p5 * s3 - p4 ** 2) / p6
    s1 = (c[7] - p5 * s2 - p4 * s3) / p6
    return p6, p5, p4, s3, s2, s1


def build(s6, p0, p1, p2, p3, q0):
    p6, p5, p4, s3, s2, s1 = top(s6)
    p = [p0, p1, p2, p3, p4, p5, p6]
    q = [q0, s1 - p1, s2 - p2, s3 - p3, p4, p5, p6]
    return p, q


def prod(p, q):
    r = [mp.mpf(0)] * 13
    for i in range(7):
        for j in range(7):
            r[i + j] += q[i] * p[j]
    return r


def resid(s6, p0, p1):
    def f(p2, p3, q0):
        p, q = build(s6, p0, p1, p2, p3, q0)
        r = prod(p, q)
        return [r[6] - c[6], r[5] - c[5], r[4] - c[4]]
    return f


def coeffs(s6, p0, p1, p2, p3, q0):
    p, q = build(s6, p0, p1, p2, p3, q0)
    r = prod(p, q)
    for k in range(4, 13):
        assert abs(r[k] - c[k]) < mp.mpf(10) ** -40 * max(1, abs(c[k])), (k, r[k], c[k])
    b3 = mp.sqrt(p[6]) if p[6] > 0 else None
    if b3 is None:
        return None
    b2 = p[5] / (2 * b3)
    b1 = (p[4] - b2 ** 2) / (2 * b3)
    B4 = [mp.mpf(0), b1, b2, b3]
    sq = [mp.mpf(0)] * 7
    for i in range(4):
        for j in range(4):
            sq[i + j] += B4[i] * B4[j]
    for k in range(4, 7):
        assert abs(sq[k] - p[k]) < mp.mpf(10) ** -40 * max(1, abs(p[k]))
    B3 = [p[k] - sq[k] for k in range(4)]
    B2 = [q[k] - p[k] for k in range(4)]
    B1 = [c[k] - r[k] for k in range(4)]
    return dict(B1=B1, B2=B2, B3=B3, B4=B4)


def scheme(A, co):
    I = np.eye(A.shape[0], dtype=A.dtype)
    A2 = A @ A
    A3 = A2 @ A
    P = [I, A, A2, A3]
    lin = lambda v: sum(float(x) * P[k] for k, x in enumerate(v))  # noqa: E731
    B4 = lin(co["B4"])
    A6 = lin(co["B3"]) + B4 @ B4
    return lin(co["B1"]) + (lin(co["B2"]) + A6) @ A6


def taylor_ref(A, m=12):
    Al = A.astype(np.clongdouble)
    S = np.eye(A.shape[0], dtype=np.clongdouble)
    term = S.copy()
    for k in range(1, m + 1):
        term = term @ Al / k
        S = S + term
    return S


def theta(m):
    f = lambda t: sum(mp.mpf(t) ** k / mp.factorial(k) for k in range(m + 1, m + 60)) - mp.mpf(2) ** -53 * mp.e ** (-t)  # noqa: E731
    return mp.findroot(f, 0.3)


def main():
    th = theta(12)
    print("theta12 =", mp.nstr(th, 17))
    rng = np.random.default_rng(0)
    mats = []
    for k in range(6):
        A = rng.standard_normal((64, 64)) + 1j * rng.standard_normal((64, 64))
        A *= float(th) / np.abs(A).sum(0).max()
        mats.append(A)
        B = 1j * (A + A.conj().T) / 2
        B *= float(th) / np.abs(B).sum(0).max()
        mats.append(B)
    refs = [taylor_ref(A) for A in mats]
    best = None
    seen = []
    for s6 in (1, -1):
        for p0, p1 in itertools.product([mp.mpf(x) for x in (-1, -0.5, 0, 0.5, 1, 2)],
                                        [mp.mpf(x) for x in (-2, -1, -0.5, 0, 0.5, 1, 2)]):
            for g in itertools.product([-1, -0.1, 0.1, 1], [-1, -0.1, 0.1, 1], [-1, 0.1, 1]):
                try:
                    r = mp.findroot(resid(s6, p0, p1), [mp.mpf(x) for x in g], tol=mp.mpf(10) ** -45, maxsteps=100)
                except (ZeroDivisionError, ValueError):
                    continue
                p2, p3, q0 = r[0], r[1], r[2]
                key = (s6, float(p0), float(p1), round(float(p2), 9), round(float(p3), 9))
                if key in seen:
                    continue
                seen.append(key)
                co = coeffs(s6, p0, p1, p2, p3, q0)
                if co is None:
                    continue
                err = max(float(np.abs(scheme(A, co) - R).max() / np.abs(R).max()) for A, R in zip(mats, refs))
                mag = max(abs(float(v)) for d in co.values() for v in d)
                if best is None or err < best[0]:
                    best = (err, mag, co, key)
    err, mag, co, key = best
    print(f"{len(seen)} solutions; chosen {key}: max rel err {err:.2e}, max |coef| {mag:.2e}")
    for name in ("B1", "B2", "B3", "B4"):
        print(name, [mp.nstr(v, 20) for v in co[name]])
    print("// C literals (columns I, A, A2, A3)")
    for name in ("B1", "B2", "B3", "B4"):
        print(name, ", ".join(repr(float(v)) for v in co[name]))


if __name__ == "__main__":
    main()
