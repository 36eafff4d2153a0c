"""Fit Q(s) = sin(pi*sqrt(s)) / (pi*sqrt(s)) on s in [0, S_MAX] with Q(0) = 1 fixed.

Used to generate the polynomial constants in csrc/nbx_math.cuh.  Minimax in
relative error via a few Remez-style reweighted least-squares passes on a
dense grid evaluated with mpmath at 60 digits.
"""
import sys
import mpmath as mp
import numpy as np

mp.mp.dps = 60
S_MAX = 0.2704  # x <= 0.52 covers |t| <= 0.5 plus the 1e-12 bias and slop


def q_exact(s):
    if s == 0:
        return mp.mpf(1)
    x = mp.pi * mp.sqrt(s)
    return mp.sin(x) / x


def fit(deg, iters=30):
    # unknowns c1..c_deg ; Q(s) ~ 1 + sum c_k s^k
    grid = [mp.mpf(S_MAX) * (1 - mp.cos(mp.pi * (i + 0.5) / 4000)) / 2 for i in range(4000)]
    ex = [q_exact(s) for s in grid]
    w = np.ones(len(grid))
    for _ in range(iters):
        A = mp.matrix(len(grid), deg)
        b = mp.matrix(len(grid), 1)
        for i, s in enumerate(grid):
            wi = mp.mpf(w[i]) / ex[i]
            for k in range(deg):
                A[i, k] = wi * s ** (k + 1)
            b[i] = wi * (ex[i] - 1)
        c = mp.lu_solve(A.T * A, A.T * b)
        err = np.array([float((1 + sum(c[k] * s ** (k + 1) for k in range(deg)) - e) / e)
                        for s, e in zip(grid, ex)])
        w = w * (1 + 8 * np.abs(err) / np.abs(err).max())
    return [c[k] for k in range(deg)], np.abs(err).max()


if __name__ == "__main__":
    for deg in map(int, sys.argv[1:]):
        c, e = fit(deg)
        print(f"deg {deg}: max rel err {e:.3e}")
        for k, ck in enumerate(c):
            print(f"  c{k+1} = {mp.nstr(ck, 25)}")
