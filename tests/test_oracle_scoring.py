"""Pins for oracle.score_argmin (eviction choice on an explicit node table).

* α = 0 is LRU: the pick is the candidate with the smallest (t_last, id).
* Degenerate ranges (all t equal, all eff equal) give u = 0.5 + 0.5 α for every
  candidate (SURVEY c.3 #2), so ties fall to the smallest id.
* Exact-rational argmin: utilities evaluated in exact rational arithmetic from
  the same double inputs; whenever the best two exact utilities are separated by
  far more than fp64 rounding, the oracle must pick the exact minimiser.
* E1 (SURVEY c.5): α = 0 evicts A, α = 1 evicts B.
"""
from fractions import Fraction

import numpy as np

import oracle as O
import tracegen as tg


def _rand_table(rng, n):
    t = rng.integers(1, 1000, n).astype(np.uint32)
    eff = rng.uniform(1e3, 3e5, n)
    cand = (rng.random(n) < 0.7).astype(np.uint8)
    ids = rng.permutation(n).astype(np.uint32) + 1
    return t, cand, ids, eff


def test_alpha0_is_lru():
    rng = np.random.default_rng(5)
    for _ in range(300):
        n = int(rng.integers(1, 60))
        t, cand, ids, eff = _rand_table(rng, n)
        t[rng.integers(0, n, n // 3)] = t[0]  # force timestamp ties
        b, u = O.score_argmin(t, cand, ids, eff, 0.0)
        c = np.nonzero(cand)[0]
        if len(c) == 0:
            assert b is None
            continue
        want = min(c, key=lambda i: (int(t[i]), int(ids[i])))
        assert b == want


def test_degenerate_ranges():
    for a in tg.ALPHA_GRID16:
        t = np.full(5, 7, np.uint32)
        eff = np.full(5, 123.5)
        ids = np.array([9, 4, 6, 2, 8], np.uint32)
        cand = np.array([1, 1, 1, 0, 1], np.uint8)
        b, u = O.score_argmin(t, cand, ids, eff, a)
        assert b == 1 and u == 0.5 + a * 0.5


def test_exact_rational_argmin():
    rng = np.random.default_rng(11)
    checked = 0
    for _ in range(400):
        n = int(rng.integers(2, 50))
        t, cand, ids, eff = _rand_table(rng, n)
        alpha = float(rng.choice(tg.ALPHA_GRID16))
        c = np.nonzero(cand)[0]
        if len(c) < 2:
            continue
        tmin, tmax = int(t.min()), int(t.max())
        emin, emax = Fraction(float(eff.min())), Fraction(float(eff.max()))
        ex = {}
        for i in c:
            rec = Fraction(1, 2) if tmax == tmin else Fraction(int(t[i]) - tmin, tmax - tmin)
            effn = Fraction(1, 2) if emax == emin else (Fraction(float(eff[i])) - emin) / (emax - emin)
            ex[i] = rec + Fraction(alpha) * effn
        srt = sorted(c, key=lambda i: ex[i])
        gap = ex[srt[1]] - ex[srt[0]]
        if gap <= Fraction(1, 10 ** 9) * (1 + Fraction(alpha)):
            continue
        b, u = O.score_argmin(t, cand, ids, eff, alpha)
        assert b == srt[0]
        assert abs(u - float(ex[srt[0]])) <= 1e-14 * (1 + alpha)
        checked += 1
    assert checked > 300


def test_e1_table():
    M = tg.MODEL_7B
    eff = [O.node_cost(M, 0, L, True)[2] for L in (1000, 200, 4000)]
    t = np.array([1, 2, 3], np.uint32)
    ids = np.array([1, 2, 3], np.uint32)
    cand = np.ones(3, np.uint8)
    assert O.score_argmin(t, cand, ids, eff, 0.0)[0] == 0
    b, u = O.score_argmin(t, cand, ids, eff, 1.0)
    assert b == 1 and u == 0.5
