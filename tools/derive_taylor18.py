"""Derive coefficients of a degree-18 Taylor evaluation in 5 matrix products
(Bader-Blanes-Casas-type scheme; A15):
    A2 = A^2, A3 = A2 A, A6 = A3^2
    B1 = a1 A + a2 A2 + a3 A3,  B5 = e1 A + e2 A2 + A6,  B4 = f0 I + f1 A + f2 A2 + f3 A3 + f6 A6
    A9 = B1 B5 + B4
    B3 = b0 I + b1 A + b2 A2 + b3 A3 + b6 A6,  B2 = g0 I + g1 A + g2 A2 + g3 A3 + g6 A6
    T18 = B2 + (B3 + A9) A9  ==  sum_{k<=18} A^k / k!   (exactly, as polynomials)
The Taylor match leaves a one-parameter family; eliminating top-down leaves two polynomial
equations in (t = alpha6, alpha3), solved here in 50-digit arithmetic.  Every real root is
then tested in double precision for rounding stability on random matrices of 1-norm up to
theta18 and on the configs' slice generators; the most stable one is printed as C literals.
"""
import itertools
import math

import mpmath as mp
import numpy as np

mp.mp.dps = 50
c = [mp.mpf(1) / mp.factorial(k) for k in range(19)]


def chain(t, a3, s9):
    """top-down elimination; returns all alpha/beta given (t = alpha6, alpha3) and the sign of alpha9."""
    a9 = s9 * mp.sqrt(c[18])
    a8 = c[17] / (2 * a9)
    a7 = (c[16] - a8 ** 2) / (2 * a9)
    g6 = (c[15] - 2 * a7 * a8) / a9
    a5 = (c[14] - g6 * a8 - a7 ** 2) / (2 * a9)
    a4 = (c[13] - 2 * a5 * a8 - g6 * a7) / (2 * a9)
    b6 = g6 - 2 * t
    g3 = (c[12] - 2 * a4 * a8 - 2 * a5 * a7 - t * (g6 - t)) / a9
    g2 = (c[11] - g3 * a8 - 2 * a4 * a7 - a5 * g6) / a9
    g1 = (c[10] - g2 * a8 - g3 * a7 - a4 * g6 - a5 ** 2) / a9
    g0 = (c[9] - g1 * a8 - g2 * a7 - g3 * t - b6 * a3 - 2 * a4 * a5) / a9
    a2 = (c[8] - g0 * a8 - g1 * a7 - g2 * t - g3 * a5 - a4 ** 2) / b6
    a1 = (c[7] - g0 * a7 - g1 * t - g2 * a5 - g3 * a4) / b6
    return dict(a9=a9, a8=a8, a7=a7, a6=t, a5=a5, a4=a4, a3=a3, a2=a2, a1=a1, g0=g0, g1=g1, g2=g2, g3=g3,
                g6=g6, b6=b6)


def resid(t, a3, s9):
    v = chain(t, a3, s9)
    e5 = v["g0"] * v["a5"] + v["g1"] * v["a4"] + v["g2"] * v["a3"] + v["g3"] * v["a2"] - 2 * v["a2"] * v["a3"] - c[5]
    e4 = (v["g0"] * v["a4"] + v["g1"] * v["a3"] + v["a2"] * (v["g2"] - v["a2"]) + (v["g3"] - 2 * v["a3"]) * v["a1"]
          - c[4])
    return e5, e4


def full_coeffs(v):
    """alpha0 = 0; beta_k = gamma_k - 2 alpha_k; B2 from the absorbed degrees; B1, B5, B4 from alpha."""
    a = [mp.mpf(0)] + [v[f"a{k}"] for k in range(1, 10)]
    beta = {0: v["g0"], 1: v["g1"] - 2 * a[1], 2: v["g2"] - 2 * a[2], 3: v["g3"] - 2 * a[3], 6: v["b6"]}
    # (B3 + A9) A9 coefficients
    prod = [mp.mpf(0)] * 19
    for i in range(10):
        for j in range(10):
            prod[i + j] += a[i] * a[j]
    for k, b in beta.items():
        for j in range(10):
            prod[k + j] += b * a[j]
    for k in list(range(4, 6)) + list(range(7, 19)):
        assert abs(prod[k] - c[k]) < mp.mpf(10) ** -40 * max(1, abs(c[k])), (k, prod[k], c[k])
    g = {k: c[k] - prod[k] for k in (0, 1, 2, 3, 6)}
    # A9 = B1 B5 + B4 with a0 = 0, e6 = 1, e3 = e0 = 0
    B1 = {1: a[7], 2: a[8], 3: a[9]}
    e2 = a[5] / a[9]
    e1 = (a[4] - a[8] * e2) / a[9]
    B5 = {1: e1, 2: e2, 6: mp.mpf(1)}
    f = {6: a[6], 3: a[3] - (a[7] * e2 + a[8] * e1), 2: a[2] - a[7] * e1, 1: a[1], 0: a[0]}
    return dict(B1=B1, B5=B5, B4=f, B3=beta, B2=g)


def poly_eval_scheme(A, co):
    """the 5-product scheme in double precision (numpy)"""
    I = np.eye(A.shape[0], dtype=A.dtype)
    A2 = A @ A
    A3 = A2 @ A
    A6 = A3 @ A3
    P = {0: I, 1: A, 2: A2, 3: A3, 6: A6}
    lin = lambda d: sum(float(v) * P[k] for k, v in d.items())  # noqa: E731
    A9 = lin(co["B1"]) @ lin(co["B5"]) + lin(co["B4"])
    return lin(co["B2"]) + (lin(co["B3"]) + A9) @ A9


def taylor_ref(A, m=18):
    """truncated Taylor polynomial in extended precision (numpy longdouble)"""
    Al = A.astype(np.clongdouble)
    S = np.eye(A.shape[0], dtype=np.clongdouble)
    term = S.copy()
    for k in range(1, m + 1):
        term = term @ Al / k
        S = S + term
    return S


def main():
    sols = []
    for s9 in (1, -1):
        for t0, x0 in itertools.product([-1e-3, -1e-4, -1e-5, 1e-5, 1e-4, 1e-3],
                                        [-1e-2, -1e-3, -1e-4, 1e-4, 1e-3, 1e-2]):
            try:
                r = mp.findroot(lambda t, x: resid(t, x, s9), (mp.mpf(t0), mp.mpf(x0)), tol=mp.mpf(10) ** -45,
                                maxsteps=200)
            except (ZeroDivisionError, ValueError):
                continue
            t, x = r[0], r[1]
            if any(abs(float(t) - float(q[1])) < 1e-12 * max(1, abs(float(t))) and q[0] == s9 for q in sols):
                continue
            sols.append((s9, t, x))
    print(len(sols), "real roots")
    rng = np.random.default_rng(0)
    mats = []
    for k in range(6):
        A = rng.standard_normal((64, 64)) + 1j * rng.standard_normal((64, 64))
        A *= 1.08 / np.abs(A).sum(0).max()
        mats.append(A)
        B = 1j * (A + A.conj().T) / 2
        B *= 1.08 / np.abs(B).sum(0).max()
        mats.append(B)
    refs = [taylor_ref(A) for A in mats]
    best = None
    for s9, t, x in sols:
        co = full_coeffs(chain(t, x, s9))
        err = max(float(np.abs(poly_eval_scheme(A, co) - R).max() / np.abs(R).max()) for A, R in zip(mats, refs))
        mag = max(abs(float(v)) for d in co.values() for v in d.values())
        print(f"s9={s9:+d} t={float(t):+.6e} a3={float(x):+.6e}  max rel err {err:.2e}  max |coef| {mag:.2e}")
        if best is None or err < best[0]:
            best = (err, co)
    err, co = best
    print("chosen: max rel err", err)
    for name in ("B1", "B5", "B4", "B3", "B2"):
        print(name, {k: mp.nstr(v, 20) for k, v in sorted(co[name].items())})
    print("// C literals")
    for name in ("B1", "B5", "B4", "B3", "B2"):
        print(name, ", ".join(repr(float(co[name].get(k, 0))) for k in (0, 1, 2, 3, 6)))


if __name__ == "__main__":
    main()
