"""GPU: the standalone batched lookup (mc_lookup: steps 1-4 of the replay against a frozen
snapshot, read-only) equals the oracle's lookup (pinned against the flat-list simulator,
tests/test_oracle_lookup.py) field by field -- micro traces with chunked checkpoints,
node/byte caps and n_ssm = 0, and sampled requests against config-3/4 snapshots."""
import numpy as np
import pytest

import oracle as O
import tracegen as tg

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_19379_b200 import marconi as M  # noqa: E402

FIELDS = ("reuse", "m", "p", "hit_id", "div_id", "div_off", "path_len", "d_nodes", "d_bytes")


def _check(tr, var, window, reqs_per_snap=None, max_nodes=8192, rng=None):
    snaps, *_ = O.live_pass(tr, var, window)
    ctx = M.Context([var], max_nodes=max_nodes)
    ctx.upload_trace(tr.tokens, tr.off, tr.lin, tr.lout)
    ctx.set_snapshots(0, snaps)
    R = tr.n_requests
    qr, qs = [], []
    for k in range(len(snaps)):
        rs = np.arange(1, R + 1) if reqs_per_snap is None else rng.choice(np.arange(1, R + 1), reqs_per_snap)
        qr += rs.tolist()
        qs += [k] * len(rs)
    out = ctx.lookup(np.asarray(qr), 0, np.asarray(qs))
    ctx.check()
    got = ctx.lookup_records(out)
    o = O.Oracle(tr, var.model, var.capacity_bytes, var.capacity_nodes, 0.0, getattr(var, "chunk_size", 0))
    loaded = None
    for i, (r, k) in enumerate(zip(qr, qs)):
        if loaded != k:
            o.close()
            o = O.Oracle(tr, var.model, var.capacity_bytes, var.capacity_nodes, 0.0, getattr(var, "chunk_size", 0))
            o.load(*snaps[k])
            loaded = k
        ref = o.lookup(r)
        assert {f: int(got[i][f]) for f in FIELDS} == {f: int(ref[f]) for f in FIELDS}, (r, k)
    o.close()
    return len(qr)


def test_lookup_micro_traces():
    n = 0
    for seed in range(120):
        tr = tg.micro_trace(seed, n_req=20, max_len=64, alphabet=2 + seed % 3)
        model = tg.MODEL_7B if seed % 5 else tg.Model(4, 0, 4)
        chunk = (0, 0, 4, 8)[seed % 4] if model.n_ssm else 0
        capb = (3 + seed % 4) * 27_000_000 if seed % 2 else tg.UNLIMITED_BYTES
        var = tg.Variant(model, capb, 0 if seed % 2 else 3 + seed % 5, chunk)
        n += _check(tr, var, window=5, max_nodes=128)
    assert n > 5000


@pytest.mark.parametrize("cfg", [3, 4])
def test_lookup_config_snapshots(cfg):
    w = tg.workload(cfg, R=6000 if cfg == 3 else 3000)
    rng = np.random.default_rng(cfg)
    _check(w.trace, w.variants[0], w.window * 8, reqs_per_snap=150, rng=rng)


def test_lookup_rejects_bad_queries():
    w = tg.workload(3, R=500)
    ctx = M.Context(w.variants, max_nodes=1024)
    ctx.upload_trace(w.trace.tokens, w.trace.off, w.trace.lin, w.trace.lout)
    ctx.live_pass(100)
    for bad in (dict(req=0), dict(req=501), dict(snapshot=99), dict(variant=1)):
        kw = dict(req=1, variant=0, snapshot=0)
        kw.update(bad)
        with pytest.raises(M.MarconiError):
            ctx.lookup(kw["req"], kw["variant"], kw["snapshot"])
