"""GPU: the end-to-end host-buffer path -- device-side trace check (mc_set_trace_async),
asynchronous snapshot upload and the double-buffered HostPipeline -- gives exactly the
kernel-only run's results, and a rejected trace is reported loudly without any replay."""
import numpy as np
import pytest

import oracle as O
import tracegen as tg

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_19379_b200 import AlphaGrid  # noqa: E402
from paper_2411_19379_b200 import marconi as M  # noqa: E402
from paper_2411_19379_b200.grid import HostPipeline  # noqa: E402


def _pinned_job(g, tr):
    h_tok = torch.from_numpy(np.ascontiguousarray(tr.tokens, np.uint32).view(np.int32)).pin_memory()
    h_req = torch.from_numpy(M.requests_array(tr.off, tr.lin, tr.lout).view(np.int64)).pin_memory()
    snaps = []
    for v in range(len(g.variants)):
        nodes, off, nid = g.ctx.pack_snapshots([g.ctx.get_snapshot(v, k) for k in range(g.ctx.snapshot_count(v))])
        pin = torch.empty(nodes.nbytes, dtype=torch.uint8).pin_memory()
        pn = pin.numpy().view(M.SNAP_DTYPE)
        pn[:] = nodes
        snaps.append((pn, off, nid))
    return h_tok, h_req, snaps, pin


def test_host_pipeline_matches_kernel_run():
    """Config 3 at 6k requests (16 α x 128 segments): 5 pipelined jobs == one kernel-only
    replay, hit by hit; α* equals the oracle's rule on the same sums."""
    w = tg.workload(3, R=6000)
    g = AlphaGrid(w.trace, w.variants, w.alphas, w.n_segments).setup()
    out = g.run()
    g.ctx.check()
    ref_hit = out["hit"].cpu().numpy()
    ref_hs = out["hit_sum"].cpu().numpy()
    h_tok, h_req, snaps, keep = _pinned_job(g, w.trace)
    p = HostPipeline(g)
    tickets = [p.submit(h_tok, h_req, snaps) for _ in range(2)]
    for _ in range(3):
        hit, hs, a_star = p.result(tickets.pop(0))
        assert np.array_equal(hit.numpy(), ref_hit) and np.array_equal(hs, ref_hs)
        assert a_star[0] == O.select_alpha(w.alphas, [int(x) for x in ref_hs[0]])
        tickets.append(p.submit(h_tok, h_req, snaps))
    for t in tickets:
        hit, hs, _ = p.result(t)
        assert np.array_equal(hit.numpy(), ref_hit)


def test_async_trace_check_rejects_loudly():
    """A request with input_len 0 (and one past the pool) passes the synchronous scalar
    checks of mc_set_trace_async; the device check flags it, the replay reads nothing,
    and mc_check names the first bad request."""
    w = tg.workload(3, R=2000)
    g = AlphaGrid(w.trace, w.variants, w.alphas[:2], 4).setup()
    tr = w.trace
    req = M.requests_array(tr.off, tr.lin, tr.lout)
    req["input_len"][6] = 0                       # request 7
    req["tok_off"][40] = tr.tokens.shape[0]       # request 41: outside the pool
    d_tok = torch.from_numpy(np.ascontiguousarray(tr.tokens, np.uint32).view(np.int32)).cuda()
    d_req = torch.from_numpy(req.view(np.int64)).cuda()
    g.ctx.set_trace_async(d_tok, d_req, tr.n_requests)
    out = g.run()
    with pytest.raises(M.MarconiError, match="request 7 "):
        g.ctx.check()
    assert int(out["hit"].abs().sum()) == 0 and int(out["hit_sum"].abs().sum()) == 0
    # the status is cleared by the report: a valid trace replays normally again
    d_req2 = torch.from_numpy(M.requests_array(tr.off, tr.lin, tr.lout).view(np.int64)).cuda()
    g.ctx.set_trace_async(d_tok, d_req2, tr.n_requests)
    out2 = g.run()
    g.ctx.check()
    assert int(out2["hit_sum"].sum()) > 0


def test_async_trace_check_length_limit():
    """F(L) < 2^53 bounds the request length (Appendix A cost model, exact u64 -> f64):
    at the 7B model the longest admissible request is 284,096 tokens (R15)."""
    m = tg.MODEL_7B
    fa = 8 * m.n_attn * m.d_model ** 2 + m.n_ssm * (12 * m.d_model ** 2 + 16 * m.d_model * m.d_state + 10) \
        + 16 * m.n_mlp * m.d_model ** 2
    fb = 4 * m.n_attn * m.d_model
    L = 284_096
    assert fa * L + fb * L * L < 2 ** 53 <= fa * (L + 1) + fb * (L + 1) ** 2
    base = [(list(range(1, 9)), [])]
    for n, ok in ((L, True), (L + 1, False)):
        toks = np.arange(1, n + 1, dtype=np.uint32)
        tr = tg.from_sequences(base + [(toks.tolist(), [])])
        ctx = M.Context([tg.Variant(m, 60 * tg.GB, 0)], max_nodes=64)
        d_tok = torch.from_numpy(np.ascontiguousarray(tr.tokens, np.uint32).view(np.int32)).cuda()
        d_req = torch.from_numpy(M.requests_array(tr.off, tr.lin, tr.lout).view(np.int64)).cuda()
        ctx.set_trace_async(d_tok, d_req, tr.n_requests)
        if ok:
            ctx.check()
        else:
            with pytest.raises(M.MarconiError, match="request 2 "):
                ctx.check()


def test_cost_feedback_order_changes_no_result():
    """Chains ordered by the live pass's window cycles, then re-ordered by the measured
    per-chain cycles of a replay (grid.AlphaGrid.reorder_by_cycles): the same chain set,
    identical per-request hits, FLOPs and hit sums."""
    w = tg.workload(5, R=8000)
    g = AlphaGrid(w.trace, w.variants[:3], w.alphas[:4], w.n_segments).setup()
    wc = g.ctx.live_window_cycles(0)
    assert wc.shape[0] == w.n_segments and int(wc.sum()) > 0
    out = g.run(chain_cycles=True)
    g.ctx.check()
    before = sorted(g.chains.tolist())
    g.reorder_by_cycles(out["cycles"])
    assert sorted(g.chains.tolist()) == before
    cyc = out["cycles"].cpu().numpy()[g.chains.astype(np.int64)]
    assert np.all(cyc[:-1] >= cyc[1:])  # longest first
    out2 = g.run(chain_cycles=True)
    g.ctx.check()
    for k in ("hit", "flops", "bypass", "hit_sum"):
        assert torch.equal(out[k], out2[k]), k


def test_chain_sums_match_outputs():
    """mc_chain_sums: per chain Σ hit, Σ input tokens and Σ FLOPs saved (exact, 128-bit)
    equal the sums of the replay's per-request outputs over the chain's window."""
    w = tg.workload(3, R=5000)
    g = AlphaGrid(w.trace, w.variants, w.alphas, w.n_segments).setup()
    out = g.run()
    g.ctx.check()
    sums = g.ctx.chain_sums(out, len(w.alphas), g.chains)
    hit = out["hit"].cpu().numpy()
    fl = out["flops"].cpu().numpy().astype(np.uint64)
    na, ns = len(w.alphas), len(g.segs)
    for c, (sh, sl, sf) in zip(g.chains.tolist(), sums):
        v, a, s = c // (na * ns), (c // ns) % na, c % ns
        f, n, _ = g.segs[s]
        sl_ref = int(w.trace.lin[f - 1:f - 1 + n].astype(np.int64).sum())
        assert sh == int(hit[v, a, f - 1:f - 1 + n].astype(np.int64).sum())
        assert sl == sl_ref
        assert sf == sum(int(x) for x in fl[v, a, f - 1:f - 1 + n])
