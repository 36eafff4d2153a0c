"""Poisson photon noise against an independent distribution: scipy.stats.poisson.

The bit-exact test (test_gpu_spots.py) pins the device sampler to its host twin, which is
the SAME header compiled for the CPU -- it cannot see a wrong constant.  Here the draws are
checked against scipy's Poisson pmf with a chi-square goodness-of-fit test at means on both
sides of the sampler's switch (inversion below 12, PTRS at and above 12,
csrc/nbx_poisson.h) and deep in the PTRS range, 400,000 draws each, plus mean, variance
and lag-1 independence of consecutive pixels.  The reference has no noise model
(SPEC.md:12, 252), so the Poisson law itself is the oracle.
"""
import numpy as np
import pytest
from scipy import stats

from paper_2205_07976_b200 import PixelBuffer, add_noise

pytestmark = pytest.mark.gpu

N_DRAWS = 400_000


def chi2_pvalue(draws: np.ndarray, mu: float, min_expected: float = 50.0) -> tuple[float, int]:
    """Chi-square p-value of integer draws against Poisson(mu); bins merged to >= min_expected."""
    k = draws.astype(np.int64)
    assert np.array_equal(k, draws), "Poisson draws must be integers"
    lo = int(stats.poisson.ppf(1e-9, mu))
    hi = int(stats.poisson.isf(1e-9, mu))
    support = np.arange(lo, hi + 1)
    expected = stats.poisson.pmf(support, mu) * k.size
    expected[0] += stats.poisson.cdf(lo - 1, mu) * k.size if lo > 0 else 0.0  # left tail into the first bin
    expected[-1] += stats.poisson.sf(hi, mu) * k.size  # right tail into the last
    observed = np.bincount(np.clip(k, lo, hi) - lo, minlength=support.size).astype(float)
    # merge adjacent values until every bin expects >= min_expected
    edges, acc_e, acc_o, obs, exp = [], 0.0, 0.0, [], []
    for o, e in zip(observed, expected):
        acc_e += e
        acc_o += o
        if acc_e >= min_expected:
            exp.append(acc_e)
            obs.append(acc_o)
            acc_e = acc_o = 0.0
    if acc_e > 0:
        exp[-1] += acc_e
        obs[-1] += acc_o
    obs, exp = np.array(obs), np.array(exp)
    chi2 = float(((obs - exp) ** 2 / exp).sum())
    dof = len(exp) - 1
    return float(stats.chi2.sf(chi2, dof)), dof


@pytest.mark.parametrize("mu", [0.3, 3.0, 11.9, 12.0, 12.1, 40.0, 1e3, 1e5])
@pytest.mark.parametrize("prec", ["f64", "f32"])
def test_poisson_draws_follow_scipy_poisson(gpu, mu, prec):
    buf = PixelBuffer((1, N_DRAWS), prec, np.full(N_DRAWS, mu))
    draws = add_noise(buf, seed=20220507, image=int(mu * 10) % 997).data.astype(np.float64)
    p, dof = chi2_pvalue(draws, mu)
    assert dof >= 2 or mu < 1
    # fixed seed: deterministic; a correct sampler fails this with probability 1e-4
    assert p > 1e-4, (mu, prec, p, dof)
    se = np.sqrt(mu / N_DRAWS)
    assert abs(draws.mean() - mu) < 5 * se, (draws.mean(), mu)
    # variance of the sample variance for Poisson: (mu + 2 mu^2) / n (fourth central moment mu + 3 mu^2)
    assert abs(draws.var() - mu) < 5 * np.sqrt((mu + 2 * mu * mu) / N_DRAWS), (draws.var(), mu)
    # neighbouring pixels are independent draws (Philox counter = pixel)
    d = draws - draws.mean()
    r1 = float((d[1:] * d[:-1]).mean() / d.var())
    assert abs(r1) < 5 / np.sqrt(N_DRAWS), r1


def test_poisson_images_are_independent(gpu):
    """Same means, different image counters: uncorrelated draws; same counter: identical."""
    mu = np.full(N_DRAWS, 7.5)
    buf = PixelBuffer((1, N_DRAWS), "f64", mu)
    a = add_noise(buf, seed=5, image=0).data
    b = add_noise(buf, seed=5, image=1).data
    c = add_noise(buf, seed=6, image=0).data
    assert np.array_equal(a, add_noise(buf, seed=5, image=0).data)
    for other in (b, c):
        r = np.corrcoef(a, other)[0, 1]
        assert abs(r) < 5 / np.sqrt(N_DRAWS), r


def test_poisson_zero_and_tiny_means(gpu):
    buf = PixelBuffer((1, 6), "f64", [0.0, 0.0, 1e-300, 1e-12, 0.0, 0.0])
    out = add_noise(buf, seed=1).data
    assert out[0] == out[1] == out[4] == out[5] == 0.0
    assert set(out.tolist()) <= {0.0, 1.0}
