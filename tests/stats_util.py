"""Test-side statistics: the reference's chi-square policy (stats.hpp:35-79)
with our own quantile (the reference uses Boost.Math, absent here).

Quantile: scipy's chi2.ppf, pinned in test_oracle.py against the reference's
known answers (test_stats.cpp:10-29: df=1 -> 10.828, df=9 -> 27.877,
df=99 -> 148.23 at p=1e-3).
"""
from __future__ import annotations

import numpy as np


def chi2_critical(df: int, p: float) -> float:
    from scipy.stats import chi2
    return float(chi2.isf(p, df))


def chi_square(observed, expected_prob, p: float = 1e-3, min_expect: float = 5.0):
    """Pearson statistic with cells of expected count < min_expect pooled into
    one tail cell first, exactly as stats.hpp:35-79.  Returns
    (statistic, critical, df, passed)."""
    obs = np.asarray(observed, dtype=np.float64)
    prob = np.asarray(expected_prob, dtype=np.float64)
    trials = obs.sum()
    e = prob * trials
    small = e < min_expect
    big = ~small
    d = obs[big] - e[big]
    stat = float(np.sum(d * d / e[big]))
    cells = int(big.sum())
    pool_exp = float(e[small].sum())
    if pool_exp > 0.0:
        pd = float(obs[small].sum()) - pool_exp
        stat += pd * pd / pool_exp
        cells += 1
    if cells < 2:
        return stat, 0.0, 0, True
    df = cells - 1
    crit = chi2_critical(df, p)
    return stat, crit, df, stat < crit
