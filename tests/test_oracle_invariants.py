"""Invariant pins for the oracle on session-structured traces.

* capacity never exceeded after admission; hits never exceed the input
  (north_star) -- the oracle also asserts byte
  conservation (incremental total == full walk) at every step internally;
* at most two SSM checkpoints admitted per request;
* α = 0 replay of segment k from snapshot S_k is bitwise the live LRU pass
  over window k (SURVEY.md c.4 "α-grid");
* snapshot dump -> load round-trips;
* α-grid selection: grid {0} -> 0; permuting the grid or
  re-sharding chains does not change α* (SPEC:365-370).
"""
import numpy as np
import pytest

import oracle as O
import tracegen as tg

GB = tg.GB


@pytest.fixture(scope="module")
def small():
    w = tg.workload(3, R=2400)
    v = tg.Variant(tg.MODEL_7B, 4 * GB)
    return w.trace, v


def test_capacity_and_hit_bounds(small):
    tr, v = small
    o = O.Oracle(tr, v.model, v.capacity_bytes, 0, 1.0)
    h, f, b = o.run(1, tr.n_requests)
    assert (h <= tr.lin).all()
    tot, cnt = o.total()
    assert tot <= v.capacity_bytes
    assert len(o.log()) > 100          # the cache is under contention
    assert h.sum() > 0


def test_at_most_two_checkpoints_per_request():
    tr = tg.workload(3, R=600).trace
    o = O.Oracle(tr, tg.MODEL_7B, tg.UNLIMITED_BYTES, 0, 0.0)
    prev = 0
    for r in range(1, tr.n_requests + 1):
        o.step(r)
        d, _ = o.dump()
        k = int(d["has_ssm"].sum())
        assert 0 <= k - prev <= 2, r
        prev = k


def test_third_occurrence_long_prompt():
    """Three sessions sharing a 1000-token prompt: hits (0, 0, 1000)."""
    prompt = list(range(1, 1001))
    reqs = [(prompt + [5000 + 10 * i + j for j in range(30)], [9000 + 10 * i + j for j in range(20)])
            for i in range(3)]
    tr = tg.from_sequences(reqs)
    o = O.Oracle(tr, tg.MODEL_7B, 60 * GB, 0, 0.0)
    assert [o.step(r)[0] for r in (1, 2, 3)] == [0, 0, 1000]


def test_segment_replay_alpha0_equals_live_pass(small):
    tr, v = small
    W = 300
    snaps, h_live, f_live, b_live = O.live_pass(tr, v, W)
    segs = [(k * W + 1, min(W, tr.n_requests - k * W)) for k in range(len(snaps))]
    chains = [(0, 0.0, a, n, k) for k, (a, n) in enumerate(segs)]
    hit, fl, by, hs, ctr = O.run_chains(tr, [v], chains, snaps, n_threads=4)
    assert np.array_equal(np.concatenate(hit), h_live)
    assert np.array_equal(np.concatenate(fl), f_live)
    assert np.array_equal(np.concatenate(by), b_live)


def test_dump_load_roundtrip(small):
    tr, v = small
    o = O.Oracle(tr, v.model, v.capacity_bytes, 0, 0.5)
    o.run(1, 1000)
    d, nid = o.dump()
    o2 = O.Oracle(tr, v.model, v.capacity_bytes, 0, 0.5)
    o2.load(d, nid)
    d2, nid2 = o2.dump()
    assert nid2 == nid and np.array_equal(d, d2)
    assert o.total() == o2.total()
    h1 = o.run(1001, 300)
    h2 = o2.run(1001, 300)
    for a, b in zip(h1, h2):
        assert np.array_equal(a, b)


def test_alpha_selection_rules(small):
    tr, v = small
    W = 600
    snaps, *_ = O.live_pass(tr, v, W)
    segs = [(k * W + 1, min(W, tr.n_requests - k * W)) for k in range(len(snaps))]
    grid = [0.0, 0.25, 1.0, 4.0, 64.0]

    def grid_sums(alphas, threads):
        chains = [(0, a, s, n, k) for a in alphas for k, (s, n) in enumerate(segs)]
        _, _, _, hs, _ = O.run_chains(tr, [v], chains, snaps, n_threads=threads)
        sums = {}
        for (vv, a, *_), x in zip(chains, hs):
            sums[a] = sums.get(a, 0) + int(x)
        return sums

    s1 = grid_sums(grid, 1)
    s2 = grid_sums(list(reversed(grid)), 8)
    assert s1 == s2
    a1 = O.select_alpha(list(s1), list(s1.values()))
    a2 = O.select_alpha(list(reversed(list(s1))), list(reversed(list(s1.values()))))
    assert a1 == a2
    assert O.select_alpha([0.0], [123]) == 0.0
    assert O.select_alpha([2.0, 1.0, 0.5], [7, 7, 7]) == 0.5


def test_symmetric_trace_selects_alpha0():
    """Uniformly short equal-length independent sequences: every α gives equal hits ->
    α* = 0 by tie-break."""
    reqs = [([100 * i + j for j in range(16)], [7000 + 100 * i + j for j in range(8)]) for i in range(40)]
    reqs += reqs[:10]
    tr = tg.from_sequences(reqs)
    sums = []
    for a in tg.ALPHA_GRID16:
        o = O.Oracle(tr, tg.MODEL_7B, tg.UNLIMITED_BYTES, 8, a)
        sums.append(int(o.run(1, tr.n_requests)[0].sum()))
    assert len(set(sums)) == 1
    assert O.select_alpha(tg.ALPHA_GRID16, sums) == 0.0
