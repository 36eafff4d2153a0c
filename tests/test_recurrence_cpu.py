"""Error bounds of the FP64 kernel's sine recurrences (nbx_kernels.cu: step / to_cheb),
emulated in IEEE double with NumPy against an 80-bit long-double truth (CPU only).

The segmented kernel advances s_k = sin(pi (x0 + k y)) / pi along a uniform run in one of two forms:
  * Reinsch:   d <- fma(-alpha, s, d); s <- s + d          (alpha = 4 sin^2(pi y / 2); the denominators,
                                                           and numerators whose step angle is small)
  * Chebyshev: s' = fma(c2, s, -s_prev)                    (c2 = 2 - alpha; numerators on warp-runs whose
                                                           step angles all have |sin(pi y)| >= 0.02)
DESIGN states the Chebyshev form's error as <= ~k eps / sin(theta): <= 7e-13 (in sin units) over a
128-channel run at the threshold (measured max 4e-13), against ~2e-14 for Reinsch's form.  These tests check those
figures on random starts and steps (the FMA is emulated through long double, whose 64-bit
significand makes the product's rounding negligible next to the double result's).
"""
import numpy as np

LD = np.longdouble
EPS_RUN = 128  # the host cuts runs at <= 128 channels (nbx_runtime.cu)


def truth(x0, y, k):
    return np.sin(LD(np.pi) * (LD(x0) + LD(k) * LD(y))) / LD(np.pi)


def fma(a, b, c):
    return (LD(a) * LD(b) + LD(c)).astype(np.float64)


def start(x0, y):
    """Anchors rounded to double, as the kernel's (correctly rounded to ~1 ulp) polynomial anchors."""
    s0 = truth(x0, y, 0).astype(np.float64)
    sm1 = truth(x0, y, -1).astype(np.float64)
    alpha = (4 * np.sin(LD(np.pi) * LD(y) / 2) ** 2).astype(np.float64)
    return s0, sm1, alpha


def run_reinsch(x0, y, n):
    s, sm1, alpha = start(x0, y)
    d = (LD(s) - LD(sm1)).astype(np.float64)  # s0 - s_{-1}, as the kernel's product form gives it
    err = np.zeros_like(s)
    for k in range(1, n):
        d = fma(-alpha, s, d)
        s = s + d
        err = np.maximum(err, np.abs((LD(s) - truth(x0, y, k)).astype(np.float64)))
    return err * np.pi  # in sin units


def run_cheb(x0, y, n):
    s, sp, alpha = start(x0, y)
    s, sp = s, (LD(s) - (LD(s) - LD(sp))).astype(np.float64)  # to_cheb: s_{-1} = s - d
    c2 = 2.0 - alpha
    err = np.zeros_like(s)
    for k in range(1, n):
        s, sp = fma(c2, s, -sp), s
        err = np.maximum(err, np.abs((LD(s) - truth(x0, y, k)).astype(np.float64)))
    return err * np.pi


def test_chebyshev_numerator_error_bound_at_threshold():
    rng = np.random.default_rng(2205)
    m = 4000
    x0 = rng.uniform(-0.5, 0.5, m)
    # step angles theta = pi y with |sin theta| in [0.02, 1] (the kernel's eligibility), half near the threshold
    th = np.concatenate([rng.uniform(np.arcsin(0.02), 0.05, m // 2), rng.uniform(0.05, np.pi / 2, m - m // 2)])
    y = th / np.pi * rng.choice([-1.0, 1.0], m)
    err = run_cheb(x0, y, EPS_RUN)
    bound = EPS_RUN * 2.3e-16 / (2 * np.abs(np.sin(th)))  # k eps / (2 sin theta), eps = ulp(c2) / 2 ~ 1.1e-16..2.2e-16
    assert err.max() <= 7e-13, err.max()
    assert np.all(err <= 4 * bound + 5e-15), float(np.max(err / (bound + 5e-15)))


def test_reinsch_error_small_steps():
    rng = np.random.default_rng(76)
    m = 4000
    x0 = rng.uniform(-0.5, 0.5, m)
    # denominator steps: |y| <= 0.9 / (len - 1) for the run's span rule; numerators below the threshold too
    y = rng.uniform(-0.0075, 0.0075, m)
    err = run_reinsch(x0, y, EPS_RUN)
    assert err.max() <= 3e-14, err.max()  # measured 2.1e-14
