"""Pins for oracle.live_tune, the paper's online tuning loop (§4.2).

* grid {0}: tuning can only adopt α = 0, so the result is the pure α = 0 (LRU) live
  pass;
* r_F is the first request whose admission evicted a node (cross-checked against an
  independent α = 0 run's eviction log); the window is (r_F, r_F + 10 r_F] (R16);
* no eviction ever -> α stays 0;
* α* is the argmax of the window's grid hit sums, ties to the smallest α; the hits after
  the window equal an α* replay from the tree at the window's end.
"""
import numpy as np

import oracle as O
import tracegen as tg


def _small():
    w = tg.workload(3, R=3000)
    return w.trace, tg.Variant(tg.MODEL_7B, 4 * tg.GB)


def test_grid_zero_is_pure_lru():
    tr, v = _small()
    h, f, info = O.live_tune(tr, v, [0.0])
    o = O.Oracle(tr, v.model, v.capacity_bytes, 0, 0.0)
    h0, f0, _ = o.run(1, tr.n_requests)
    assert np.array_equal(h, h0) and np.array_equal(f, f0)
    assert info["alpha_star"] == 0.0


def test_first_eviction_and_window():
    tr, v = _small()
    h, f, info = O.live_tune(tr, v, [0.0, 1.0, 64.0])
    o = O.Oracle(tr, v.model, v.capacity_bytes, 0, 0.0)
    o.run(1, tr.n_requests)
    r_f = int(o.log()[0]["req"])
    assert info["r_first_evict"] == r_f
    assert info["window"] == (r_f + 1, min(11 * r_f, tr.n_requests))
    sums = info["grid_hit_sums"]
    assert info["alpha_star"] == O.select_alpha([0.0, 1.0, 64.0], sums)
    # hits up to the window end are the α = 0 live pass's
    o2 = O.Oracle(tr, v.model, v.capacity_bytes, 0, 0.0)
    hl, _, _ = o2.run(1, info["window"][1])
    assert np.array_equal(h[: info["window"][1]], hl)


def test_no_eviction_keeps_alpha0():
    tr, _ = _small()
    v = tg.Variant(tg.MODEL_7B, tg.UNLIMITED_BYTES)
    h, f, info = O.live_tune(tr, v, [0.0, 1.0])
    assert info["r_first_evict"] == 0 and info["alpha_star"] == 0.0


def test_vllm_variant_keeps_its_policy_after_adoption():
    """Regression: the adopt phase replays with the variant's own policy.  A vLLM+ chain
    ignores α (reading V8), so every grid entry ties, α* = 0, and the whole tuned run must
    equal the plain vLLM+ live pass -- including the requests after the window."""
    tr, _ = _small()
    v = tg.Variant(tg.MODEL_7B, 4 * tg.GB, 0, 0, 32)
    h, f, info = O.live_tune(tr, v, [0.0, 1.0, 64.0])
    assert info["window"] is not None and info["window"][1] < tr.n_requests
    assert len(set(info["grid_hit_sums"])) == 1 and info["alpha_star"] == 0.0
    o = O.Oracle(tr, v.model, v.capacity_bytes, 0, 0.0, block=32)
    h0, f0, _ = o.run(1, tr.n_requests)
    assert np.array_equal(h, h0) and np.array_equal(f, f0)
