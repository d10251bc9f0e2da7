"""Pins for the oracle's replay against the hand-derived worked examples.

tests/golden/scenarios.json, each citing the paper
passage it illustrates: PAPER:378 (third occurrence / instantaneous reuse),
PAPER:300-301 and PAPER:246 (all-or-nothing vs KV slicing)
(absorption, single-node touch), Eq. 2.
"""
import numpy as np
import pytest

import oracle as O
import scenarios as SC
import tracegen as tg

SPEC = SC.load()


@pytest.mark.parametrize("sc", SPEC["scenarios"], ids=lambda s: s["name"])
def test_scenario_hits(sc):
    tr = SC.scenario_trace(SPEC, sc)
    v = SC.variant(sc)
    for a in sc["alphas"]:
        o = O.Oracle(tr, v.model, v.capacity_bytes, v.capacity_nodes, a)
        hits = []
        prev = 0
        deltas = []
        for r in range(1, tr.n_requests + 1):
            h, f, b = o.step(r)
            hits.append(h)
            assert f == O.prefill_flops(v.model, h)       # FLOPs saved = F(reuse), root-anchored
            tot, _ = o.total()
            deltas.append(tot - prev)
            prev = tot
            if r == 2 and "dump_after_2" in sc:
                d, _ = o.dump()
                got = [[int(x["id"]), int(x["parent_id"]), int(x["d_start"]), int(x["d_end"]),
                        int(x["has_ssm"]), int(x["t_last"])] for x in d]
                assert got == sc["dump_after_2"]
        assert hits == sc["hits"], (a, hits)
        if "delta_bytes" in sc:
            assert deltas == sc["delta_bytes"]
        if "first_eviction" in sc:
            lg = o.log()
            fe = sc["first_eviction"]
            assert (int(lg[0]["req"]), int(lg[0]["node_id"]), int(lg[0]["kind"])) == \
                (fe["req"], fe["node_id"], fe["kind"])
            assert lg[0]["utility"] == fe["utility"]


def test_s6_merged_child_bytes_and_eff():
    """After the α=0 absorption in S6, id2 covers [0,75) with 31,703,040 B (SURVEY c.5 S6)."""
    sc = next(s for s in SPEC["scenarios"] if s["name"] == "S6_absorption_alpha0")
    tr = SC.scenario_trace(SPEC, sc)
    v = SC.variant(sc)
    o = O.Oracle(tr, v.model, v.capacity_bytes, v.capacity_nodes, 0.0)
    for r in (1, 2, 3):
        o.step(r)
    d, _ = o.dump()
    rec = d[d["id"] == 2][0]
    assert (rec["d_start"], rec["d_end"], rec["parent_id"]) == (0, 75, 0)
    s, b, e = O.node_cost(v.model, 0, 75, True)
    assert b == 31_703_040
    assert abs(e - 30969.76800962936) <= 1e-12 * e


@pytest.mark.parametrize("ex", SPEC["eviction_examples"], ids=lambda s: s["name"])
def test_eviction_examples(ex):
    tr, nodes, nid = SC.eviction_example(SPEC, ex)
    snap = np.array(nodes, dtype=[("id", "<u4"), ("parent_id", "<u4"), ("ref_off", "<u8"), ("d_start", "<u4"),
                                  ("d_end", "<u4"), ("t_last", "<u4"), ("has_ssm", "<u4")])
    snap = snap.astype(O.NODE_DTYPE)
    m = SC.MODELS[ex["model"]]
    if "eff" in ex:
        for rec in nodes:
            e = O.node_cost(m, rec[3], rec[4], bool(rec[6]))[2]
            assert abs(e - ex["eff"][str(rec[0])]) <= 1e-12 * e
    for a, want in ex["expect"].items():
        o = O.Oracle(tr, m, tg.UNLIMITED_BYTES, ex["cap_nodes"], float(a))
        o.load(snap, nid)
        o.step(ex["request"])
        lg = o.log()
        assert (int(lg[0]["node_id"]), int(lg[0]["kind"])) == (want["node_id"], want["kind"]), a
        assert abs(lg[0]["utility"] - want["utility"]) <= 1e-15 * max(1.0, want["utility"])
    if "effn_1" in ex:  # α = 1/64 (exact power of two): A's u = effn_A / 64 < B's 0.5
        o = O.Oracle(tr, m, tg.UNLIMITED_BYTES, ex["cap_nodes"], 1.0 / 64)
        o.load(snap, nid)
        o.step(ex["request"])
        lg = o.log()
        assert int(lg[0]["node_id"]) == 1
        assert abs(lg[0]["utility"] * 64 - ex["effn_1"]) <= 1e-15


def test_no_cache_baseline_all_bypass():
    """Vanilla inference: capacity 0 -> every request bypasses, hits stay 0."""
    tr = tg.toy_trace(7, 16)
    o = O.Oracle(tr, tg.MODEL_TOY, 0, 0, 0.0)
    h, f, b = o.run(1, tr.n_requests)
    assert h.sum() == 0 and b.all()
    assert o.total() == (0, 0)


def test_input_validation():
    tr = tg.from_sequences([([1, 2, 3], [4])])
    with pytest.raises(O.OracleError):
        O.Oracle(tr, tg.MODEL_7B, 10 ** 12, 0, -1.0)
    with pytest.raises(O.OracleError):
        O.Oracle(tr, tg.Model(4, 24, 28, bytes_per_param=3), 10 ** 12, 0, 0.0)
    bad = tg.from_sequences([([], [4])])
    with pytest.raises(O.OracleError):
        O.Oracle(bad, tg.MODEL_7B, 10 ** 12, 0, 0.0)
