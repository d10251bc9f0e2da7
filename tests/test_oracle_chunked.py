"""Pins for chunk-aligned prefill checkpoints (NEXT-3; "Obtaining states
during prefill": chunked state passing checkpoints the chunk boundary at or below the
branch point, e.g. 80 -> 64 with chunk 32; SPEC:329 skips aligned values that are 0 or not
beyond the current hit).  Final (decode) checkpoints stay exact."""
import numpy as np
import pytest

import flatlist as FL
import oracle as O
import tracegen as tg


def _paper_example(chunk):
    A = list(range(1, 81))                      # 80 shared input tokens
    reqs = [(A + [500 + j for j in range(20)], []),
            (A + [600 + j for j in range(20)], []),
            (A + [700 + j for j in range(20)], [])]
    tr = tg.from_sequences(reqs)
    o = O.Oracle(tr, tg.MODEL_7B, tg.UNLIMITED_BYTES, 0, 0.0, chunk)
    return [o.step(r)[0] for r in (1, 2, 3)], o


def test_paper_80_to_64():
    hits, o = _paper_example(32)
    assert hits == [0, 0, 64]                   # the state at 80 is checkpointed at 64
    d, _ = o.dump()
    assert any(int(x["d_end"]) == 64 and x["has_ssm"] for x in d)
    hits_exact, _ = _paper_example(0)
    assert hits_exact == [0, 0, 80]             # two-pass prefill: exact


def test_aligned_zero_or_below_hit_is_skipped():
    hits, o = _paper_example(128)               # floor(80 / 128) * 128 = 0 -> no checkpoint
    assert hits == [0, 0, 0]
    d, _ = o.dump()
    assert not any(int(x["d_end"]) == 0 for x in d)


@pytest.mark.parametrize("chunk", [2, 3, 8])
def test_flatlist_equivalence_chunked(chunk):
    for seed in range(150):
        tr = tg.micro_trace(seed, n_req=20, max_len=64, alphabet=2 + seed % 3)
        capn = 2 + seed % 6
        a = tg.ALPHA_GRID16[seed % 16]
        o = O.Oracle(tr, tg.MODEL_7B, tg.UNLIMITED_BYTES, capn, a, chunk)
        h, f, b = o.run(1, tr.n_requests)
        res, fc = FL.replay(tr, tg.MODEL_7B, tg.UNLIMITED_BYTES, capn, a, chunk=chunk)
        assert [int(x) for x in h] == [x[0] for x in res], (chunk, seed)
        assert [int(x) for x in o.counters()] == fc.ctr, (chunk, seed)
        lg = o.log()
        assert [(int(x["req"]), int(x["node_id"]), int(x["kind"])) for x in lg] == \
            [(r, i, k) for r, i, k, _ in fc.log], (chunk, seed)
        d, _ = o.dump()
        assert [(int(x["id"]), int(x["parent_id"]), int(x["d_start"]), int(x["d_end"]), int(x["has_ssm"]),
                 int(x["t_last"])) for x in d] == fc.dump(), (chunk, seed)


def test_chunk_one_is_exact():
    for seed in range(40):
        tr = tg.micro_trace(seed, n_req=20, max_len=64, alphabet=3)
        h1 = O.Oracle(tr, tg.MODEL_7B, tg.UNLIMITED_BYTES, 4, 0.5, 1).run(1, tr.n_requests)[0]
        h0 = O.Oracle(tr, tg.MODEL_7B, tg.UNLIMITED_BYTES, 4, 0.5, 0).run(1, tr.n_requests)[0]
        assert np.array_equal(h1, h0)
