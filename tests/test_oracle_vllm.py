"""Pins for the oracle's vLLM+ baseline (readings V1-V8).

vLLM+ = vLLM's prefix caching extended to hybrid models: "fine-grained checkpointing
and caches a state for every token block" with block size 32, each block
holding the KVs of its tokens and the SSM states of all prior tokens,
vLLM's LRU caching policy.

Pinned against:
* the brute-force flat-list block model (tests/flatlist.py FlatBlocks) on micro traces:
  hits, bypass flags, eviction log (ids + utility bits) and final cache;
* fig:motivation(b): one 10K-token sequence at block 16 holds 17.4 GB;
* the occurrence rule of §4.1: a purely-input prefix is reused by Marconi
  from its third occurrence, by block checkpointing from its second;
* pure-Transformer collapse: without SSM layers the block cache hits the
  Marconi hit rounded down to a whole block (unlimited capacity);
* structural invariants (block-aligned nodes, parent touched no earlier than child,
  exact byte accounting) and snapshot round trips.
"""
import numpy as np
import pytest

import flatlist as FL
import oracle as O
import tracegen as tg

M7 = tg.MODEL_7B


def _bb(model, x):
    return FL.KVT(model) * x + FL.SSMB(model)


def _run(tr, model, capb, capn, x, with_ctr=False):
    o = O.Oracle(tr, model, capb, capn, 0.0, block=x)
    h, f, b = o.run(1, tr.n_requests)
    lg, (d, nid) = o.log(), o.dump()
    tot = o.total()
    ctr = o.counters()
    o.close()
    return (h, f, b, lg, d, tot, ctr) if with_ctr else (h, f, b, lg, d, tot)


def _cap(seed, model, x):
    bb = _bb(model, x)
    k = seed % 3
    if k == 0:
        return tg.UNLIMITED_BYTES, 2 + seed % 7
    if k == 1:
        return (2 + seed % 5) * bb + seed % 7, 0
    return (3 + seed % 4) * bb, 3 + seed % 5


@pytest.mark.parametrize("part", range(6))
def test_flat_blocks_equivalence(part):
    """300 micro traces x block sizes 1..8: identical hits, logs and final caches."""
    for seed in range(part * 50, part * 50 + 50):
        tr = tg.micro_trace(seed, n_req=20, max_len=64, alphabet=2 + seed % 3)
        model = M7 if seed % 2 else tg.MODEL_TOY
        x = 1 + seed % 8
        capb, capn = _cap(seed, model, x)
        h, f, b, lg, d, _, ctr = _run(tr, model, capb, capn, x, with_ctr=True)
        res, fc = FL.replay_blocks(tr, model, capb, capn, x)
        assert [int(v) for v in h] == [r[0] for r in res], seed
        assert [int(v) for v in f] == [r[1] for r in res], seed
        assert [int(v) for v in b] == [r[2] for r in res], seed
        got = [(int(e["req"]), int(e["node_id"]), int(e["kind"]), float(e["utility"]).hex()) for e in lg]
        assert got == [(r, i, k, u.hex()) for r, i, k, u in fc.log], seed
        dd = [(int(e["id"]), int(e["parent_id"]), int(e["d_start"]), int(e["d_end"]), int(e["has_ssm"]),
               int(e["t_last"])) for e in d]
        assert dd == fc.dump(), seed
        assert [int(v) for v in ctr] == fc.ctr, (seed, ctr, fc.ctr)  # d.3 counters


def test_fig2b_17_4_GB_one_10k_sequence_block16():
    """'for a 7B model, a single sequence of 10K tokens consumes 17.4 GB'
    with a state per 16-token block (fig:motivation(b)); 3.3x a same-size Transformer."""
    tr = tg.from_sequences([(list(range(1, 10_001)), [])])
    h, f, b, lg, d, (tot, cnt) = _run(tr, M7, tg.UNLIMITED_BYTES, 0, 16)
    assert cnt == 625 and len(d) == 625
    assert tot == 17_397_760_000
    assert round(tot / 1e9, 1) == 17.4
    assert int(h[0]) == 0 and int(b[0]) == 0
    tf = tg.Model(32, 0, 32)  # the Transformer of the same size: 32 attention layers, KVs only
    _, _, _, _, _, (tot_tf, _) = _run(tr, tf, tg.UNLIMITED_BYTES, 0, 16)
    assert round(tot / tot_tf, 1) == 3.3


@pytest.mark.parametrize("L", [1, 31, 32, 33, 100, 257])
def test_occurrence_rule(L):
    """purely-input prefixes are reused by Marconi only from the third
    occurrence; block checkpointing reuses whole blocks from the second."""
    P = list(range(7, 7 + L))
    tr = tg.from_sequences([(P, [900 + k, 901 + k]) for k in range(3)])
    hv, *_ = _run(tr, M7, tg.UNLIMITED_BYTES, 0, 32)
    assert [int(v) for v in hv] == [0, (L // 32) * 32, (L // 32) * 32]
    o = O.Oracle(tr, M7, tg.UNLIMITED_BYTES, 0, 1.0)
    hm, _, _ = o.run(1, 3)
    o.close()
    assert [int(v) for v in hm] == [0, 0, L]


@pytest.mark.parametrize("seed", range(20))
def test_pure_transformer_collapse(seed):
    """PAPER:666 'When serving a pure Transformer, the three systems achieve the same
    performance': with n_ssm = 0 and unlimited capacity the block cache hits exactly the
    Marconi hit (longest cached prefix within the input) rounded down to a block."""
    tr = tg.micro_trace(seed, n_req=20, max_len=64, alphabet=2 + seed % 3)
    model = tg.Model(4, 0, 4)
    x = 1 + seed % 8
    hv, *_ = _run(tr, model, tg.UNLIMITED_BYTES, 0, x)
    o = O.Oracle(tr, model, tg.UNLIMITED_BYTES, 0, 0.0)
    hm, _, _ = o.run(1, tr.n_requests)
    o.close()
    assert [int(v) for v in hv] == [(int(v) // x) * x for v in hm]


@pytest.mark.parametrize("seed", range(12))
def test_structure_invariants(seed):
    w = tg.workload(2, R=600)
    model = w.variants[0].model
    x = (16, 32, 64)[seed % 3]
    capb = (40 + 13 * seed) * _bb(model, x)
    o = O.Oracle(w.trace, model, capb, 0, 0.0, block=x)
    for r in range(1, 601, 150):
        o.run(r, 150)
        d, _ = o.dump()
        tot, cnt = o.total()
        assert cnt == len(d) and tot == cnt * _bb(model, x) and tot <= capb
        assert np.all(d["d_end"] - d["d_start"] == x) and np.all(d["d_start"] % x == 0)
        assert np.all(d["has_ssm"] == 1)
        t = {int(e["id"]): int(e["t_last"]) for e in d}
        for e in d:
            if int(e["parent_id"]):
                assert t[int(e["parent_id"])] >= int(e["t_last"])  # the path is touched as a whole
    o.close()


def test_snapshot_round_trip():
    w = tg.workload(2, R=800)
    model = w.variants[0].model
    capb = 60 * _bb(model, 32)
    a = O.Oracle(w.trace, model, capb, 0, 0.0, block=32)
    ha, _, _ = a.run(1, 800)
    b = O.Oracle(w.trace, model, capb, 0, 0.0, block=32)
    b.run(1, 400)
    d, nid = b.dump()
    c = O.Oracle(w.trace, model, capb, 0, 0.0, block=32)
    c.load(d, nid)
    hc, _, _ = c.run(401, 400)
    assert np.array_equal(ha[400:], hc)
    assert np.array_equal(a.dump()[0], c.dump()[0])
    for o in (a, b, c):
        o.close()


def test_bypass_when_path_plus_blocks_exceed_capacity():
    """V7: a sequence whose blocks alone exceed the capacity is not admitted."""
    tr = tg.from_sequences([(list(range(1, 129)), []), (list(range(1, 129)), [5])])
    h, f, b, lg, d, (tot, cnt) = _run(tr, M7, 3 * _bb(M7, 32), 0, 32)
    assert [int(v) for v in b] == [1, 1] and cnt == 0 and [int(v) for v in h] == [0, 0]
