"""Degree-8 Taylor polynomial in 3 matrix products (A15):
    A2 = A^2,  Y = A2 (c1 A + c2 A2),
    T8 = (Y + c3 A2 + c4 A)(Y + c5 A2) + c6 Y + c7 A2 + A + I  ==  sum_{k<=8} A^k / k!
Matching degrees 8..2 gives c2^2 = 1/8!, 2 c1 c2 = 1/7!, then sigma = c3 + c5 and c4 linearly,
and a quadratic for c5 (c6 from the degree-3 equation).  Each real root is checked for rounding
stability in double precision; the best is printed as C literals."""
import mpmath as mp
import numpy as np

mp.mp.dps = 50
c = [mp.mpf(1) / mp.factorial(k) for k in range(9)]


def solutions():
    out = []
    for s2 in (1, -1):
        c2 = s2 * mp.sqrt(c[8])
        c1 = c[7] / (2 * c2)
        sig = (c[6] - c1 ** 2) / c2
        c4 = (c[5] - c1 * sig) / c2
        # degree 4: c3 c5 + c1 c4 + c2 c6 = c4';  degree 3: c4 c5 + c1 c6 = c3'
        # with c3 = sig - c5 and c6 = (c[3] - c4 c5)/c1:
        #   (sig - c5) c5 + c1 c4 + c2 (c[3] - c4 c5)/c1 - c[4] = 0
        qa = -1
        qb = sig - c2 * c4 / c1
        qc = c1 * c4 + c2 * c[3] / c1 - c[4]
        disc = qb ** 2 - 4 * qa * qc
        if disc < 0:
            continue
        for sg in (1, -1):
            c5 = (-qb + sg * mp.sqrt(disc)) / (2 * qa)
            c3 = sig - c5
            c6 = (c[3] - c4 * c5) / c1
            out.append(dict(c1=c1, c2=c2, c3=c3, c4=c4, c5=c5, c6=c6, c7=c[2]))
    return out


def check_exact(s):
    # expand the scheme symbolically (polynomial coefficients) and compare with 1/k!
    P = lambda *pairs: {k: v for k, v in pairs}  # noqa: E731
    Y = {3: s["c1"], 4: s["c2"]}
    L = dict(Y); L[2] = L.get(2, 0) + s["c3"]; L[1] = L.get(1, 0) + s["c4"]
    R = dict(Y); R[2] = R.get(2, 0) + s["c5"]
    T = {}
    for i, a in L.items():
        for j, b in R.items():
            T[i + j] = T.get(i + j, 0) + a * b
    for k, v in Y.items():
        T[k] = T.get(k, 0) + s["c6"] * v
    T[2] = T.get(2, 0) + s["c7"]
    T[1] = T.get(1, 0) + 1
    T[0] = T.get(0, 0) + 1
    return max(abs(T.get(k, 0) - c[k]) / c[k] for k in range(9))


def scheme(A, s):
    I = np.eye(A.shape[0], dtype=A.dtype)
    A2 = A @ A
    Y = A2 @ (float(s["c1"]) * A + float(s["c2"]) * A2)
    return ((Y + float(s["c3"]) * A2 + float(s["c4"]) * A) @ (Y + float(s["c5"]) * A2) + float(s["c6"]) * Y
            + float(s["c7"]) * A2 + A + I)


def taylor_ref(A, m=8):
    Al = A.astype(np.clongdouble)
    S = np.eye(A.shape[0], dtype=np.clongdouble)
    term = S.copy()
    for k in range(1, m + 1):
        term = term @ Al / k
        S = S + term
    return S


def main():
    rng = np.random.default_rng(0)
    mats = []
    for _ in range(6):
        A = rng.standard_normal((64, 64)) + 1j * rng.standard_normal((64, 64))
        mats.append(A * 0.0694 / np.abs(A).sum(0).max())
    best = None
    for s in solutions():
        exact = check_exact(s)
        err = max(float(np.abs(scheme(A, s) - taylor_ref(A)).max()) for A in mats)
        print({k: mp.nstr(v, 12) for k, v in s.items()}, f"poly match {float(exact):.1e}  max abs err {err:.2e}")
        if best is None or err < best[0]:
            best = (err, s)
    print("C literals:", ", ".join(repr(float(best[1][k])) for k in ("c1", "c2", "c3", "c4", "c5", "c6", "c7")))


if __name__ == "__main__":
    main()
