"""Pin the oracle's read-only lookup (steps 1-4 of SURVEY.md c.2: walk, hit, speculative
insertion point, insertion plan) against the
flat-list simulator's brute-force lookup (tests/flatlist.py), request by request on micro
traces, with the hit it predicts checked against the step that follows."""
import numpy as np
import pytest

import flatlist as FL
import oracle as O
import tracegen as tg

FIELDS = ("reuse", "m", "p", "hit_id", "div_id", "div_off", "path_len", "d_nodes", "d_bytes")


@pytest.mark.parametrize("block", range(4))
def test_lookup_equals_flatlist(block):
    for seed in range(block * 40, block * 40 + 40):
        tr = tg.micro_trace(seed, n_req=18, max_len=48, alphabet=2 + seed % 3)
        model = tg.MODEL_7B if seed % 3 else tg.MODEL_TOY
        if seed % 7 == 0:
            model = tg.Model(4, 0, 4)  # pure Transformer: mid-edge hits
        chunk = (0, 0, 4, 8)[seed % 4]
        capb = (3 + seed % 4) * FL.SSMB(tg.MODEL_7B) if seed % 2 else tg.UNLIMITED_BYTES
        capn = 0 if seed % 2 else 3 + seed % 5
        a = tg.ALPHA_GRID16[seed % 16]
        var = tg.Variant(model, capb, capn, chunk)
        o = O.Oracle(tr, model, capb, capn, a, chunk)
        fc = FL.FlatCache(model, capb, capn, a, chunk=chunk)
        for r in range(1, tr.n_requests + 1):
            i = r - 1
            S = tr.seq(r)
            inp, out = S[:int(tr.lin[i])].tolist(), S[int(tr.lin[i]):].tolist()
            got = o.lookup(r)
            ref = fc.lookup(inp, out)
            assert {k: int(got[k]) for k in FIELDS} == ref, (seed, r)
            h, _, _ = o.step(r)
            assert h == ref["reuse"], (seed, r)  # the lookup predicts the step's hit
            fc.step(r, inp, out)
        o.close()


def test_lookup_does_not_mutate():
    tr = tg.micro_trace(11, n_req=20, max_len=64, alphabet=3)
    o = O.Oracle(tr, tg.MODEL_7B, tg.UNLIMITED_BYTES, 5, 1.0)
    o.run(1, 12)
    before = o.dump()
    for r in range(1, 21):
        o.lookup(r)
    after = o.dump()
    assert after[1] == before[1] and np.array_equal(after[0], before[0])
    o.close()
