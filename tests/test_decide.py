"""The certified ADMM decisions (paper_1607_00531_b200/decide.py, the twin of
csrc/admm_decide.h): the enclosure of the reference's sequential sum holds
for adversarial term sets, certified decisions never differ from the ones
taken on the sequential sums, and near-ties are left undecided."""
import math

import numpy as np
import pytest

from paper_1607_00531_b200 import decide


def seq(t):
    return float(np.add.accumulate(np.concatenate(([0.0], t)))[-1])


def tree(t):
    # a different order: pairwise (numpy's sum) over a permutation
    return float(np.sum(t[::-1].reshape(-1)))


@pytest.mark.parametrize("seed", range(6))
def test_enclosure_contains_sequential_sum(seed):
    rng = np.random.default_rng(seed)
    n = int(rng.integers(1, 200000))
    kind = seed % 3
    if kind == 0:
        t = rng.uniform(0, 1, n) ** 2
    elif kind == 1:  # wide dynamic range
        t = np.exp(rng.uniform(-60, 60, n))
    else:  # one huge term first, then tiny ones (the sequential chain loses them)
        t = np.concatenate(([1e16], rng.uniform(0, 1, n - 1)))
    s, tr = seq(t), tree(t)
    lo, hi = decide.enclose_seq(tr, n)
    assert lo <= s <= hi, (lo, s, hi)
    assert decide.enclose_seq(0.0, n) == (0.0, 0.0)
    assert decide.enclose_seq(math.inf, n) is None


def test_certified_matches_exact_and_declines_ties():
    rng = np.random.default_rng(5)
    n = 5000
    agree = undecided = 0
    for trial in range(400):
        scale = np.exp(rng.uniform(-3, 3, 5))
        terms = [rng.uniform(0, 1, n) * s for s in scale]
        rho = float(np.exp(rng.uniform(0, 12)))
        eps = float(rng.choice([1e-300, 1e-3, 0.2]))
        # sometimes force a near-tie pr ~ mu * du (sqrt(s0) ~ 10 rho sqrt(s1))
        if trial % 4 == 0:
            eps = 1e-300
            terms[0] = terms[1] * (10.0 * rho) ** 2 * (1 + 1e-13 * rng.uniform(-1, 1))
        tr = [tree(t) for t in terms]
        sq = [seq(t) for t in terms]
        kw = dict(rho=rho, V=1.0, sqrt_n=math.sqrt(n), eps_abs=eps, eps_rel=eps, mu=10.0,
                  adaptive=True)
        c = decide.certified(tr, n, **kw)
        e = decide.exact(sq, **kw)
        if c is None:
            undecided += 1
        else:
            assert c == e
            agree += 1
    assert agree >= 250 and undecided >= 50


def test_rho_apply_matches_reference_schedule():
    FIXED, ADAPT, BOUNDED = 0, 1, 2
    assert decide.rho_apply(FIXED, 5.0, 1.0, 1, 2.0, 2.0, FIXED, BOUNDED) == 5.0
    assert decide.rho_apply(ADAPT, 5.0, 10.0, -1, 2.0, 2.0, FIXED, BOUNDED) == 2.5
    assert decide.rho_apply(BOUNDED, 5.0, 10.0, -1, 2.0, 2.0, FIXED, BOUNDED) == 10.0
    assert decide.rho_apply(BOUNDED, 5.0, 1.0, 1, 2.0, 2.0, FIXED, BOUNDED) == 10.0
