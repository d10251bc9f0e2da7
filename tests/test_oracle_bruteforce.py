"""Pin the oracle against independent brute-force models on micro traces.

* flat-list simulator (tests/flatlist.py):
  same hits, same eviction log (ids, kinds, utility bits), same final cache.
* independent LRU: α = 0 falls back to LRU.
* OPT search: Σ reuse(α) <= OPT for every α (SURVEY.md c.1 "OPT search").
* pure-Transformer collapse: with n_ssm = 0 the hit is the textbook longest
  common prefix with any stored sequence, clipped to the input.
"""
import math

import numpy as np
import pytest

import flatlist as FL
import oracle as O
import tracegen as tg

GRID = tg.ALPHA_GRID16
SSMB = FL.SSMB(tg.MODEL_7B)
KVT = FL.KVT(tg.MODEL_7B)


def _cap(seed):
    """Alternate node-count and byte capacities so both trigger paths are exercised."""
    k = seed % 3
    if k == 0:
        return tg.UNLIMITED_BYTES, 2 + seed % 6
    if k == 1:
        return (2 + seed % 4) * SSMB + (seed % 50) * KVT, 0
    return (3 + seed % 3) * SSMB, 3 + seed % 5


def _oracle_run(tr, model, capb, capn, a, with_ctr=False):
    o = O.Oracle(tr, model, capb, capn, a)
    h, f, b = o.run(1, tr.n_requests)
    lg = o.log()
    d, _ = o.dump()
    ctr = o.counters()
    o.close()
    return (h, f, b, lg, d, ctr) if with_ctr else (h, f, b, lg, d)


@pytest.mark.parametrize("block", range(10))
def test_flatlist_equivalence(block):
    """500 micro traces (50 per block) x rotating α: identical hits, logs and final caches."""
    for seed in range(block * 50, block * 50 + 50):
        tr = tg.micro_trace(seed, n_req=20, max_len=64, alphabet=2 + seed % 3)
        model = tg.MODEL_7B if seed % 2 else tg.MODEL_TOY
        capb, capn = _cap(seed)
        a = GRID[seed % len(GRID)]
        h, f, b, lg, d, ctr = _oracle_run(tr, model, capb, capn, a, with_ctr=True)
        res, fc = FL.replay(tr, model, capb, capn, a)
        assert [int(x) for x in h] == [x[0] for x in res], seed
        assert [int(x) for x in f] == [x[1] for x in res], seed
        assert [int(x) for x in b] == [x[2] for x in res], seed
        got = [(int(x["req"]), int(x["node_id"]), int(x["kind"])) for x in lg]
        assert got == [(r, i, k) for r, i, k, _ in fc.log], seed
        # utility bits equal (both are IEEE fp64 with separately rounded ops)
        assert [float(x["utility"]).hex() for x in lg] == [u.hex() for *_, u in fc.log], seed
        dd = [(int(x["id"]), int(x["parent_id"]), int(x["d_start"]), int(x["d_end"]), int(x["has_ssm"]),
               int(x["t_last"])) for x in d]
        assert dd == fc.dump(), seed
        # the d.3 algorithmic-byte counters (numerator of roofline.frac), derived
        # independently from the brute-force relations
        assert [int(x) for x in ctr] == fc.ctr, (seed, ctr, fc.ctr)


def test_counters_pin_closed_form():
    """Hand-derived d.3 counters of worked example S1, c_r = min(m+1, n),
    v_r = |P| + 1, w_r = records written: r1 into an empty cache has m = 0 (c = 1), visits
    only the root (v = 1) and writes its leaf (w = 1); r2 matches 16 of 32 tokens inside
    r1's leaf (c = 17, P = {leaf}: v = 2), splits it at 16 (w = 2) and adds its leaf (w = 1);
    r3 walks the stateful 16-token node and stops at its boundary (c = 17, v = 2), touches
    the hit (w = 1) and adds its leaf (w = 1).  No evictions (unlimited capacity)."""
    P = list(range(100, 116))
    a, b, c = [200 + i for i in range(8)], [300 + i for i in range(8)], [400 + i for i in range(8)]
    x, y, z = [500 + i for i in range(8)], [600 + i for i in range(8)], [700 + i for i in range(8)]
    tr = tg.from_sequences([(P + a, x), (P + b, y), (P + c, z)])
    h, f, bb, lg, d, ctr = _oracle_run(tr, tg.MODEL_7B, tg.UNLIMITED_BYTES, 0, 0.0, with_ctr=True)
    assert [int(v) for v in h] == [0, 0, 16]
    assert [int(v) for v in ctr] == [1 + 17 + 17, 1 + 2 + 2, 0, 1 + 3 + 2]


def test_lru_equivalence_alpha0():
    """α = 0 evicts exactly like an independent LRU over the same candidates."""
    n = 0
    for seed in range(1000, 1120):
        tr = tg.micro_trace(seed, n_req=20, max_len=48, alphabet=2 + seed % 2)
        capb, capn = _cap(seed)
        h, f, b, lg, d = _oracle_run(tr, tg.MODEL_7B, capb, capn, 0.0)
        res, fc = FL.replay(tr, tg.MODEL_7B, capb, capn, 0.0, policy="lru")
        assert [(int(x["req"]), int(x["node_id"]), int(x["kind"])) for x in lg] == \
            [(r, i, k) for r, i, k, _ in fc.log], seed
        assert [int(x) for x in h] == [x[0] for x in res]
        n += len(lg)
    assert n > 200  # the traces really do evict


def test_opt_upper_bound():
    """Σ reuse(α) <= OPT on tiny traces, for every α in the grid."""
    checked = 0
    for seed in range(2000, 2040):
        tr = tg.micro_trace(seed, n_req=7, max_len=24, alphabet=2)
        capn = 2 + seed % 3
        opt = FL.opt_reuse(tr, tg.MODEL_7B, tg.UNLIMITED_BYTES, capn)
        for a in GRID[::3]:
            h, *_ = _oracle_run(tr, tg.MODEL_7B, tg.UNLIMITED_BYTES, capn, a)
            assert int(h.sum()) <= opt, (seed, a)
        checked += 1
    assert checked == 40


def test_pure_transformer_is_textbook_lcp():
    """n_ssm = 0: reuse = min(L_in, longest common prefix with any cached sequence).
    Unlimited capacity keeps every sequence, so the cache holds all previous ones."""
    attn = tg.Model(4, 0, 4)
    for seed in range(3000, 3100):
        tr = tg.micro_trace(seed, n_req=20, max_len=64, alphabet=2 + seed % 3)
        h, *_ = _oracle_run(tr, attn, tg.UNLIMITED_BYTES, 0, 0.0)
        seqs = [list(tr.seq(r)) for r in range(1, tr.n_requests + 1)]
        for r in range(1, tr.n_requests + 1):
            S = seqs[r - 1]
            best = 0
            for T in seqs[:r - 1]:
                k = 0
                while k < min(len(S), len(T)) and S[k] == T[k]:
                    k += 1
                best = max(best, k)
            assert int(h[r - 1]) == min(best, int(tr.lin[r - 1])), (seed, r)


def test_hybrid_hit_is_a_checkpointed_prefix():
    """Hybrid: the hit is exactly the longest prefix of the input that some earlier request
    checkpointed AND that is still cached -- with unlimited capacity nothing is evicted, so
    the hit must be <= the KV-only LCP and must equal a depth that holds a state."""
    for seed in range(3100, 3160):
        tr = tg.micro_trace(seed, n_req=20, max_len=64, alphabet=2)
        o = O.Oracle(tr, tg.MODEL_7B, tg.UNLIMITED_BYTES, 0, 0.0)
        for r in range(1, tr.n_requests + 1):
            d, _ = o.dump()
            ssm_depths = {int(x["d_end"]) for x in d if x["has_ssm"]}
            h, _, _ = o.step(r)
            assert h == 0 or h in ssm_depths
            assert h <= int(tr.lin[r - 1])
        o.close()
