"""Coefficients of the FAST-mode log (csrc/fdg_fast.cuh: log_fast).

log(m) for m in [sqrt(1/2), sqrt(2)) is written as log(1+f) = f - s (f - T(z)),
s = f / (2 + f), z = s^2, with T(z) = 2 (atanh(s)/s - 1) = 2z/3 + 2z^2/5 + ...
T is fitted here as z * (c1 + c2 z + ... + cK z^(K-1)) by a near-minimax
(Chebyshev-node, relative-weighted) least-squares fit in 60-digit arithmetic,
then the error of the whole double-precision evaluation is checked against
mpmath on random inputs.

Usage: python scripts/gen_logfast.py [K]   (prints the coefficient block)
"""

import sys

import mpmath as mp
import numpy as np

mp.mp.dps = 60


def target(z):
    if z == 0:
        return mp.mpf(0)
    s = mp.sqrt(z)
    return 2 * (mp.atanh(s) / s - 1)


def fit(K, zmax):
    # nodes: Chebyshev on [0, zmax]; fit T(z)/z with weight 1 (abs error of T/z ~ abs error of T / z)
    n = 4 * K + 20
    nodes = [zmax / 2 * (1 - mp.cos(mp.pi * (i + mp.mpf(1) / 2) / n)) for i in range(n)]
    A = mp.matrix(n, K)
    b = mp.matrix(n, 1)
    for i, z in enumerate(nodes):
        # weight by z: we care about the error of T = z * poly, not of poly
        for j in range(K):
            A[i, j] = z * z**j
        b[i] = target(z)
    # least squares via normal equations in high precision
    At = A.T
    c = mp.lu_solve(At * A, At * b)
    # iterate a few Lawson-style reweightings towards minimax
    w = [mp.mpf(1)] * n
    for _ in range(30):
        r = [abs(sum(A[i, j] * c[j] for j in range(K)) - b[i]) for i in range(n)]
        w = [w[i] * (r[i] + mp.mpf(10) ** -70) for i in range(n)]
        tot = sum(w)
        w = [x / tot for x in w]
        W = mp.diag(w)
        c = mp.lu_solve(At * W * A, At * W * b)
    return [c[j] for j in range(K)]


def eval_double(x, coef, ln2_hi, ln2_lo):
    """The CUDA sequence in float64 (numpy, with fma emulated exactly via mpmath rounding)."""
    def fma(a, b, c):
        return float(mp.mpf(a) * mp.mpf(b) + mp.mpf(c))

    m, e = np.frexp(x)  # x = m 2^e, m in [0.5, 1)
    m *= 2.0
    e -= 1
    if m >= np.sqrt(2.0):
        m /= 2.0
        e += 1
    f = m - 1.0
    den = 2.0 + f
    r = 1.0 / den  # rcp_fast is within 1 ulp of this
    s = f * r
    z = s * s
    if len(coef) == 7:  # the Estrin order of log_fast
        z2 = z * z
        p01 = fma(coef[1], z, coef[0])
        p23 = fma(coef[3], z, coef[2])
        p45 = fma(coef[5], z, coef[4])
        p47 = fma(coef[6], z2, p45)
        p03 = fma(p23, z2, p01)
        p = fma(p47, z2 * z2, p03)
    else:
        p = coef[-1]
        for cj in reversed(coef[:-1]):
            p = fma(p, z, cj)
    corr = s * fma(-z, p, f)
    ed = float(e)
    lo = fma(ed, ln2_lo, -corr)
    return fma(ed, ln2_hi, f) + lo


def main():
    K = int(sys.argv[1]) if len(sys.argv) > 1 else 7
    smax = (mp.sqrt(2) - 1) / (mp.sqrt(2) + 1)
    zmax = smax**2 * (1 + mp.mpf(2) ** -18)
    coef_mp = fit(K, zmax)
    coef = [float(c) for c in coef_mp]
    zs = [zmax * i / 2000 for i in range(1, 2001)]
    err = max(abs(sum(mp.mpf(c) * z ** (j + 1) for j, c in enumerate(coef)) - target(z)) for z in zs)
    ln2 = mp.log(2)
    ln2_hi = float(ln2)
    ln2_lo = float(ln2 - mp.mpf(ln2_hi))
    rng = np.random.default_rng(7)
    xs = np.concatenate([
        np.exp(rng.uniform(-700, 700, 3000)),
        rng.uniform(0.5, 2.0, 3000),
        1.0 + rng.uniform(-1e-6, 1e-6, 500),
        rng.uniform(0.1, 10.0, 2000),
    ])
    worst = 0.0
    for x in xs:
        got = eval_double(float(x), coef, ln2_hi, ln2_lo)
        want = mp.log(mp.mpf(float(x)))
        ulp = np.spacing(abs(float(want))) if want != 0 else 5e-324
        worst = max(worst, float(abs(mp.mpf(got) - want) / ulp))
    print("// K = %d, max |T - T_fit| on [0, zmax] = %.3e, max error of the double sequence = %.2f ulp" % (
        K, float(err), worst))
    for j, c in enumerate(coef):
        print("constexpr double LOGF_C%d = %s;" % (j + 1, repr(c)))
    print("constexpr double LOGF_LN2_HI = %r;" % ln2_hi)
    print("constexpr double LOGF_LN2_LO = %r;" % ln2_lo)


if __name__ == "__main__":
    main()
