"""Provenance of the frozen polynomial coefficients in spec/RNG.md.

Run once (python spec/fit_coeffs.py); the printed hex-floats were copied by
hand into spec/RNG.md, oracle/distill_oracle.c and the CUDA sources.  Neither
side imports this script.  Fits are weighted least squares on dense grids
followed by a few Lawson (IRLS) iterations toward minimax, in float64, then
rounded to float32.
"""
import numpy as np


def lawson(xs, target, basis, weight, iters=60):
    A = basis(xs)
    w = np.ones_like(xs)
    for _ in range(iters):
        W = np.sqrt(w)[:, None]
        c, *_ = np.linalg.lstsq(A * W * weight[:, None], target * W[:, 0] * weight, rcond=None)
        err = np.abs((A @ c - target) * weight)
        w = w * (err + 1e-30)
        w /= w.sum()
    return c, err.max()


def fit_log():
    # log1p(f) = f + f^2 * P(f),  f in [sqrt(1/2)-1, sqrt(2)-1]
    lo, hi = np.sqrt(0.5) - 1, np.sqrt(2.0) - 1
    f = np.linspace(lo, hi, 200001)
    f = f[np.abs(f) > 1e-6]
    target = (np.log1p(f) - f) / f**2
    deg = 7
    basis = lambda x: np.vander(x, deg + 1, increasing=True)
    # relative error of log(x) when e == 0 is f^2 dP / f = f dP -> weight |f|
    c, e = lawson(f, target, basis, np.abs(f))
    return c, e


def fit_sin():
    # sin(pi r) = r * S(r^2), r in [-1/2, 1/2] (half-turn reduction, RNG.md §5)
    r = np.linspace(1e-6, 0.5, 200001)
    t = r * r
    target = np.sin(np.pi * r) / r
    basis = lambda x: np.vander(x, 5, increasing=True)
    c, e = lawson(t, target, basis, r)          # absolute error of sin
    return c, e


def fit_cos():
    # cos(pi r) = 1 + r^2 C(r^2)
    r = np.linspace(0, 0.5, 200001)
    t = r * r
    target = np.cos(np.pi * r)
    tt = t[1:]
    tg = (target[1:] - 1) / tt
    basis = lambda x: np.vander(x, 5, increasing=True)
    c, e = lawson(tt, tg, basis, tt)             # absolute error of cos
    return c, e


def hexf(v):
    return float(np.float32(v)).hex()


if __name__ == "__main__":
    for name, fn in [("log P", fit_log), ("sin S", fit_sin), ("cos C", fit_cos)]:
        c, e = fn()
        print(name, "max weighted err %.3e" % e)
        for k, v in enumerate(c):
            print("  c%d = %s  (%r)" % (k, hexf(v), float(np.float32(v))))
