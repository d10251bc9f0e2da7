"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Bar (north_star): bit-exact hit tokens, FLOPs saved, bypass flags, eviction
order (request, node id, kind) and chosen α; utilities compared by bit pattern
(the contractual bound is 1e-12 relative, checked as well).
"""
import numpy as np
import pytest

import gpu_util as GU
import oracle as O
import scenarios as SC
import tracegen as tg

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_19379_b200 import marconi as M  # noqa: E402
from paper_2411_19379_b200 import AlphaGrid  # noqa: E402

DEV = torch.device("cuda", 0)


def _assert_logs_equal(glog, gn, olog, ctx=""):
    assert gn == len(olog), (ctx, gn, len(olog))
    olog = olog[: len(glog)]  # the device log keeps the first log_cap records
    assert np.array_equal(glog["req"], olog["req"]), ctx
    assert np.array_equal(glog["node_id"], olog["node_id"]), ctx
    assert np.array_equal(glog["kind"], olog["kind"]), ctx
    assert np.array_equal(glog["n_live"], olog["n_live"]), ctx
    gu, ou = glog["utility"], olog["utility"]
    assert np.all(np.abs(gu - ou) <= 1e-12 * np.maximum(1.0, np.abs(ou))), ctx
    assert np.array_equal(gu.view(np.uint64), ou.view(np.uint64)), ctx  # bitwise


# ---------------------------------------------------------------- K1
def test_k1_node_cost_bitexact():
    rng = np.random.default_rng(1)
    models = [tg.MODEL_7B, tg.MODEL_TOY, tg.model_ratio(2), tg.model_ratio(4), tg.model_ratio(8),
              tg.Model(4, 0, 4), tg.Model(4, 24, 28, d_state=16), tg.Model(4, 24, 28, bytes_per_param=4)]
    n = 3000
    for m in models:
        ds = rng.integers(0, 32768, n).astype(np.int32)
        ln = rng.integers(1, 32768, n)
        ln[:50] = 1
        de = np.minimum(ds + ln, 65535).astype(np.int32)
        ssm = (rng.random(n) < 0.6).astype(np.uint8)
        if m.n_ssm == 0:
            ssm[:] = 0
        s, b, e = M.node_cost(m, torch.from_numpy(ds).to(DEV), torch.from_numpy(de).to(DEV),
                              torch.from_numpy(ssm).to(DEV))
        s, b, e = s.cpu().numpy(), b.cpu().numpy(), e.cpu().numpy()
        for i in range(0, n, 7):
            os_, ob, oe = O.node_cost(m, int(ds[i]), int(de[i]), bool(ssm[i]))
            assert int(s[i]) == os_ and int(b[i]) == ob
            assert np.float64(e[i]).view(np.uint64) == np.float64(oe).view(np.uint64)


# ---------------------------------------------------------------- K3
def test_k3_score_argmin_segmented():
    rng = np.random.default_rng(2)
    tabs = []
    for k in range(600):
        n = int(rng.integers(0, 3000)) if k % 50 == 0 else int(rng.integers(1, 200))
        t = rng.integers(1, 5000, n).astype(np.uint32)
        if k % 3 == 0 and n:
            t[:] = t[0]                                 # degenerate recency range
        eff = rng.uniform(1e3, 3e5, n)
        if k % 5 == 0 and n > 3:
            eff[1:4] = eff[0]                           # equal eff -> ties on u
            t[1:4] = t[0]                               # ... and on t: id decides
        cand = (rng.random(n) < 0.6).astype(np.uint8)
        ids = (rng.permutation(n) + 1).astype(np.uint32)
        a = float(tg.ALPHA_GRID16[k % 16])
        tabs.append((t, cand, ids, eff, a))
    off = np.zeros(len(tabs) + 1, np.int32)
    off[1:] = np.cumsum([len(x[0]) for x in tabs])
    cat = lambda i, dt: torch.from_numpy(np.concatenate([x[i] for x in tabs]).astype(dt)).to(DEV)
    best, u = M.score_argmin(torch.from_numpy(off).to(DEV), cat(0, np.int32), cat(1, np.uint8), cat(2, np.int32),
                             cat(3, np.float64), torch.tensor([x[4] for x in tabs], dtype=torch.float64, device=DEV))
    best, u = best.cpu().numpy(), u.cpu().numpy()
    for k, (t, cand, ids, eff, a) in enumerate(tabs):
        ob, ou = O.score_argmin(t, cand, ids, eff, a)
        if ob is None:
            assert best[k] == -1
        else:
            assert best[k] == ob, k
            assert np.float64(u[k]).view(np.uint64) == np.float64(ou).view(np.uint64)


# ---------------------------------------------------------------- scenarios
SPEC = SC.load()


@pytest.mark.parametrize("sc", SPEC["scenarios"], ids=lambda s: s["name"])
def test_scenarios_on_gpu(sc):
    tr = SC.scenario_trace(SPEC, sc)
    v = SC.variant(sc)
    g, out = GU.gpu_grid(tr, [v], sc["alphas"], 1, max_nodes=64, log_cap=64)
    hit = out["hit"].cpu().numpy()
    for ai, a in enumerate(sc["alphas"]):
        assert hit[0, ai].tolist() == sc["hits"], (a, hit[0, ai])
        h, f, b, lg = GU.oracle_chain_log(tr, v, a, 1, tr.n_requests, (np.zeros(0, O.NODE_DTYPE), 1))
        assert np.array_equal(out["flops"].cpu().numpy()[0, ai], f.astype(np.int64))
        glog, gn = g.ctx.read_log(out, ai)
        _assert_logs_equal(glog, gn, lg, sc["name"])


@pytest.mark.parametrize("ex", SPEC["eviction_examples"], ids=lambda s: s["name"])
def test_eviction_examples_on_gpu(ex):
    tr, nodes, nid = SC.eviction_example(SPEC, ex)
    snap = np.zeros(len(nodes), M.SNAP_DTYPE)
    for i, (a, b, c, d, e, f, g) in enumerate(nodes):
        snap[i] = (a, b, c, d, e, f, g)
    alphas = [float(a) for a in ex["expect"]]
    ctx = M.Context([tg.Variant(SC.MODELS[ex["model"]], tg.UNLIMITED_BYTES, ex["cap_nodes"])], max_nodes=64)
    ctx.upload_trace(tr.tokens, tr.off, tr.lin, tr.lout)
    ctx.set_snapshots(0, [(snap, nid)])
    ctx.set_segments([(ex["request"], 1, 0)])
    out = ctx.replay(alphas, log_cap=8)
    ctx.check()
    for ai, a in enumerate(alphas):
        glog, gn = ctx.read_log(out, ai)
        want = ex["expect"][str(a) if str(a) in ex["expect"] else repr(a)]
        assert (int(glog[0]["node_id"]), int(glog[0]["kind"])) == (want["node_id"], want["kind"])
        _, _, _, lg = GU.oracle_chain_log(tr, ctx.variants[0], a, ex["request"], 1,
                                          (snap.astype(O.NODE_DTYPE), nid))
        _assert_logs_equal(glog, gn, lg, ex["name"])


# ---------------------------------------------------------------- micro traces
def _micro_variant(seed):
    k = seed % 3
    ssmb = 26_787_840
    kvt = 65_536
    if k == 0:
        return tg.Variant(tg.MODEL_7B, tg.UNLIMITED_BYTES, 2 + seed % 6)
    if k == 1:
        return tg.Variant(tg.MODEL_7B, (2 + seed % 4) * ssmb + (seed % 50) * kvt, 0)
    return tg.Variant(tg.MODEL_7B, (3 + seed % 3) * ssmb, 3 + seed % 5)


def test_micro_traces_full_parity():
    """300 micro traces: live-pass snapshots, every chain's hits/flops/bypass and eviction log."""
    for seed in range(300):
        tr = tg.micro_trace(seed, n_req=20, max_len=64, alphabet=2 + seed % 3)
        v = _micro_variant(seed)
        alphas = [0.0, tg.ALPHA_GRID16[seed % 16], 64.0]
        g, out = GU.gpu_grid(tr, [v], alphas, 2, max_nodes=128, log_cap=256)
        snaps, live, res, segs = GU.oracle_grid(tr, [v], alphas, 2, threads=1)
        # device live pass == oracle live pass (per request and snapshots)
        lh, lf, lb = (x.cpu().numpy()[0] for x in g.live)
        assert np.array_equal(lh, live[0][0]) and np.array_equal(lf, live[0][1].astype(np.int64)), seed
        assert np.array_equal(lb, live[0][2].astype(np.uint8)), seed
        for k in range(len(snaps[0])):
            gs, gn = g.ctx.get_snapshot(0, k)
            on, onid = snaps[0][k]
            assert gn == onid and np.array_equal(GU.canon(gs), GU.canon(on)), (seed, k)
        hit, fl, by = (out[x].cpu().numpy() for x in ("hit", "flops", "bypass"))
        for cid, (h, f, b, ctr) in res.items():
            ai, si = cid // len(segs), cid % len(segs)
            first, n, k = segs[si]
            sl = slice(first - 1, first - 1 + n)
            assert np.array_equal(hit[0, ai, sl], h), (seed, cid)
            assert np.array_equal(fl[0, ai, sl], f.astype(np.int64)), (seed, cid)
            assert np.array_equal(by[0, ai, sl], b.astype(np.uint8)), (seed, cid)
            _, _, _, lg = GU.oracle_chain_log(tr, v, alphas[ai], first, n, snaps[0][k])
            glog, gn = g.ctx.read_log(out, cid)
            _assert_logs_equal(glog, gn, lg, f"seed {seed} chain {cid}")


def test_toy_config_and_family():
    """Config 1 (toy: 16 requests, {4,28,32}, 6-node cache, α in {0,1}) plus 200 seeds of its family."""
    for seed in [1001] + list(range(5000, 5200)):
        w = tg.workload(1) if seed == 1001 else None
        tr = w.trace if w else tg.toy_trace(seed, 16)
        var = tg.Variant(tg.MODEL_TOY, tg.UNLIMITED_BYTES, 6)
        g, out = GU.gpu_grid(tr, [var], (0.0, 1.0), 1, max_nodes=64, log_cap=64)
        a_star = g.select(out)
        sums = []
        for ai, a in enumerate((0.0, 1.0)):
            h, f, b, lg = GU.oracle_chain_log(tr, var, a, 1, tr.n_requests, (np.zeros(0, O.NODE_DTYPE), 1))
            assert np.array_equal(out["hit"].cpu().numpy()[0, ai], h), seed
            glog, gn = g.ctx.read_log(out, ai)
            _assert_logs_equal(glog, gn, lg, f"toy {seed}")
            sums.append(int(h.sum()))
        assert a_star[0] == O.select_alpha((0.0, 1.0), sums)


def _compare_grid(w, R_cap_nodes=8192, log_cap=0, threads=0):
    tr = w.trace
    g, out = GU.gpu_grid(tr, w.variants, w.alphas, w.n_segments, max_nodes=R_cap_nodes, log_cap=log_cap,
                         counters=True)
    snaps, live, res, segs = GU.oracle_grid(tr, w.variants, w.alphas, w.n_segments, threads=threads)
    hit, fl, by = (out[x].cpu().numpy() for x in ("hit", "flops", "bypass"))
    ctr = out["counters"].cpu().numpy()
    na, ns = len(w.alphas), len(segs)
    for v in range(len(w.variants)):
        for k in range(len(snaps[v])):
            gs, gn = g.ctx.get_snapshot(v, k)
            on, onid = snaps[v][k]
            assert gn == onid and np.array_equal(GU.canon(gs), GU.canon(on)), (v, k)
    for cid, (h, f, b, c) in res.items():
        v, ai, si = cid // (na * ns), (cid // ns) % na, cid % ns
        first, n, k = segs[si]
        sl = slice(first - 1, first - 1 + n)
        assert np.array_equal(hit[v, ai, sl], h), cid
        assert np.array_equal(fl[v, ai, sl], f.astype(np.int64)), cid
        assert np.array_equal(by[v, ai, sl], b.astype(np.uint8)), cid
        assert np.array_equal(ctr[cid], c.astype(np.int64)), (cid, ctr[cid], c)
        if log_cap:
            _, _, _, lg = GU.oracle_chain_log(tr, w.variants[v], w.alphas[ai], first, n, snaps[v][k])
            glog, gn = g.ctx.read_log(out, cid)
            _assert_logs_equal(glog, gn, lg, f"chain {cid}")
    # α* per variant
    a_star = g.select(out)
    for v in range(len(w.variants)):
        sums = [sum(int(res[(v * na + ai) * ns + si][0].sum()) for si in range(ns)) for ai in range(na)]
        assert a_star[v] == O.select_alpha(w.alphas, sums)
    return g, out


def test_config3_reduced_full_parity():
    w = tg.workload(3, R=4000)
    w.n_segments = 8
    g, out = _compare_grid(w, log_cap=4096)
    # the same logs through the C ABI call (mc_eviction_log) as through the raw buffers
    na, ns = len(w.alphas), len(g.segs)
    for ai in (0, na // 2, na - 1):
        for si in (0, ns - 1):
            rec, n = g.ctx.eviction_log(out, na, 0, ai, si)
            raw, n2 = g.ctx.read_log(out, ai * ns + si)
            assert n == n2 and np.array_equal(rec.view(np.uint8), raw.view(np.uint8))


def test_config2_reduced():
    w = tg.workload(2, R=2500)
    _compare_grid(w, log_cap=8192)


def test_config4_reduced():
    w = tg.workload(4, R=800)
    w.alphas = (0.0, 1 / 16, 1.0, 64.0)
    w.n_segments = 4
    _compare_grid(w, log_cap=2048)


def test_config5_reduced():
    w = tg.workload(5, R=3000)
    w.alphas = (0.0, 1.0)
    w.n_segments = 2
    _compare_grid(w)


def test_uploaded_snapshots_match_live_pass():
    """mc_set_snapshots with the ORACLE's snapshots gives the same results as the device live pass."""
    w = tg.workload(3, R=3000)
    alphas = (0.0, 0.5, 4.0)
    snaps, live, res, segs = GU.oracle_grid(w.trace, w.variants, alphas, 6)
    g, out = GU.gpu_grid(w.trace, w.variants, alphas, 6, snapshots={0: snaps[0]})
    hit = out["hit"].cpu().numpy()
    for cid, (h, f, b, c) in res.items():
        ai, si = cid // len(segs), cid % len(segs)
        first, n, k = segs[si]
        assert np.array_equal(hit[0, ai, first - 1:first - 1 + n], h)


def test_chain_subsets_and_order_do_not_matter():
    w = tg.workload(3, R=3000)
    alphas = tg.ALPHA_GRID16[::3]
    g, out = GU.gpu_grid(w.trace, w.variants, alphas, 6)
    total = g.n_chains_total
    rng = np.random.default_rng(0)
    perm = rng.permutation(total).astype(np.uint32)
    halves = [perm[: total // 2], perm[total // 2:]]
    o2 = g.ctx.alloc_outputs(len(alphas))
    for h in halves:
        g.ctx.replay(alphas, chains=h, out=o2, n_workers=7)
    g.ctx.check()
    for key in ("hit", "flops", "bypass", "hit_sum"):
        assert torch.equal(out[key], o2[key]), key


def _full_grid_parity(cfg, log_chains=(), layout="stream"):
    """All chains of BASELINE config `cfg` at full size, in the bench launch configuration
    (eviction logs OFF: the branch bench.py times), against the oracle (live-pass snapshots,
    every request of every chain, d.3 counters, hit sums, α*).  Then a second replay call
    with eviction logs on the `log_chains` subset: logs equal the oracle's bitwise and
    turning logs on changes no output."""
    import os
    w = tg.workload(cfg, layout=layout)
    tr = w.trace
    g = AlphaGrid(tr, w.variants, w.alphas, w.n_segments).setup()
    out = g.run(counters=True)
    g.ctx.check()
    hit, fl, by = (out[x].cpu().numpy() for x in ("hit", "flops", "bypass"))
    ctr = out["counters"].cpu().numpy()
    snaps, live, res, segs = GU.oracle_grid(tr, w.variants, w.alphas, w.n_segments, threads=os.cpu_count() or 1)
    na, ns = len(w.alphas), len(segs)
    for v in range(len(w.variants)):
        lh = g.live[0].cpu().numpy()[v]
        assert np.array_equal(lh, live[v][0]), v                      # device live pass == oracle live pass
        for k in range(len(snaps[v])):
            gs, gn = g.ctx.get_snapshot(v, k)
            on, onid = snaps[v][k]
            assert gn == onid and np.array_equal(GU.canon(gs), GU.canon(on)), (v, k)
    for cid, (h, f, b, c) in res.items():
        v, ai, si = cid // (na * ns), (cid // ns) % na, cid % ns
        first, n, k = segs[si]
        sl = slice(first - 1, first - 1 + n)
        assert np.array_equal(hit[v, ai, sl], h), cid
        assert np.array_equal(fl[v, ai, sl], f.astype(np.int64)), cid
        assert np.array_equal(by[v, ai, sl], b.astype(np.uint8)), cid
        assert np.array_equal(ctr[cid], c.astype(np.int64)), cid
    a_star = g.select(out)
    for v in range(len(w.variants)):
        sums = [sum(int(res[(v * na + ai) * ns + si][0].sum()) for si in range(ns)) for ai in range(na)]
        assert [int(x) for x in g.hit_sums[v]] == sums
        assert a_star[v] == O.select_alpha(w.alphas, sums)
    if log_chains:
        out2 = g.ctx.alloc_outputs(na, log_cap=16384, counters=True)
        g.ctx.replay(w.alphas, chains=list(log_chains), out=out2)
        g.ctx.check()
        h2 = out2["hit"].cpu().numpy()
        c2 = out2["counters"].cpu().numpy()
        for cid in log_chains:
            v, ai, si = cid // (na * ns), (cid // ns) % na, cid % ns
            first, n, k = segs[si]
            sl = slice(first - 1, first - 1 + n)
            assert np.array_equal(h2[v, ai, sl], hit[v, ai, sl]), cid
            assert np.array_equal(c2[cid], ctr[cid]), cid
            _, _, _, lg = GU.oracle_chain_log(tr, w.variants[v], w.alphas[ai], first, n, snaps[v][k])
            glog, gn = g.ctx.read_log(out2, cid)
            _assert_logs_equal(glog, gn, lg, f"cfg{cfg} chain {cid}")
    return g, out


def test_full_config2_lmsys():
    """configs[1]: LMSys-shaped 10k requests, one chain at α = 1 over the whole trace."""
    _full_grid_parity(2, log_chains=(0,))


def test_full_config3_sharegpt():
    """configs[2] (the bench workload): 2,048 chains, every request, vs the oracle."""
    _full_grid_parity(3, log_chains=(0, 127, 8 * 128 + 64, 15 * 128 + 127))


def test_full_config4_swebench():
    """configs[3]: SWEBench-shaped, contexts up to 32,768 tokens, 2,048 chains."""
    _full_grid_parity(4, log_chains=(5, 9 * 128 + 77))


def test_full_config4_copy_layout():
    """configs[3] with every request holding its own copy of its sequence (no shared session
    stream, so no compare is skipped): the long-compare path (16-byte loads, funnel-shifted
    edge side) at full size, 2,048 chains, vs the oracle."""
    _full_grid_parity(4, log_chains=(5, 9 * 128 + 77), layout="copy")


def test_full_config3_copy_layout():
    """configs[2] in the copy layout: every walk level compares tokens."""
    _full_grid_parity(3, log_chains=(0, 8 * 128 + 64), layout="copy")


def test_long_compare_alignments():
    """Long shared prefixes (600-3,000 tokens) whose first mismatch falls at every offset
    class around the vector path's 16-byte quads (head, body, last partial quad, exactly at
    the end), with request offsets in all four alignments: hits, snapshots and eviction
    logs equal the oracle's."""
    rng = np.random.default_rng(77)
    for seed in range(24):
        L = int(rng.integers(600, 3000))
        base = (rng.integers(1, 1 << 30, L)).astype(np.uint32)
        reqs = []
        for i in range(14):
            k = int(rng.choice([0, 1, 2, 3, 4, 5, 127, 128, 129, 511, 512, 513, L - 5, L - 1, L,
                                int(rng.integers(0, L))]))
            k = max(0, min(k, L))
            pad = int(rng.integers(0, 4))  # shifts the request's pool offset modulo 4
            seq = base[:k].tolist() + [int(x) for x in rng.integers(1 << 30, (1 << 31) - 1, 3 + pad)]
            cut = int(rng.integers(1, len(seq)))
            reqs.append((seq[:cut], seq[cut:]))
        tr = tg.from_sequences(reqs)
        v = tg.Variant(tg.MODEL_7B, int(rng.choice([2, 4, 8])) * 27_000_000 + 1_000_000_000, 0)
        alphas = [0.0, 1.0]
        g, out = GU.gpu_grid(tr, [v], alphas, 2, max_nodes=256, log_cap=128)
        snaps, live, res, segs = GU.oracle_grid(tr, [v], alphas, 2, threads=1)
        assert np.array_equal(g.live[0].cpu().numpy()[0], live[0][0]), seed
        for k in range(len(snaps[0])):
            gs, gn = g.ctx.get_snapshot(0, k)
            on, onid = snaps[0][k]
            assert gn == onid and np.array_equal(GU.canon(gs), GU.canon(on)), (seed, k)
        hit = out["hit"].cpu().numpy()
        for cid, (h, f, b, ctr) in res.items():
            ai, si = cid // len(segs), cid % len(segs)
            first, n, k = segs[si]
            assert np.array_equal(hit[0, ai, first - 1:first - 1 + n], h), (seed, cid)
            _, _, _, lg = GU.oracle_chain_log(tr, v, alphas[ai], first, n, snaps[0][k])
            glog, gn = g.ctx.read_log(out, cid)
            _assert_logs_equal(glog, gn, lg, f"long-compare seed {seed} chain {cid}")


def test_full_config5_sampled():
    """configs[4]: 200k requests x 15 cache variants (1:2/1:4/1:8 x 60-140 GB) x 16 α x 16
    segments = 3,840 chains on the device (logs off, the bench launch).  Against the oracle:
    live passes and snapshots 0-2 of every variant, and ONE FULL SEGMENT (12,500 requests)
    for all 15 variants x 16 α = 240 chains (hits, FLOPs, bypass, d.3 counters); eviction
    logs of 6 of those chains from a second, logged call.  Every chain: hit <= L_in and
    α = 0 replays == the device live pass.  (All 3,840 chains against the oracle:
    tools/parity_full.py --config 5, summary in profiles/r02_parity_cfg5.json.)"""
    import os
    from concurrent.futures import ThreadPoolExecutor
    w = tg.workload(5)
    tr = w.trace
    nv, na = len(w.variants), len(w.alphas)
    g = AlphaGrid(tr, w.variants, w.alphas, w.n_segments).setup()
    out = g.run(counters=True)
    g.ctx.check()
    hit, fl, by = (out[x].cpu().numpy() for x in ("hit", "flops", "bypass"))
    ctr = out["counters"].cpu().numpy()
    live = g.live[0].cpu().numpy()
    assert (hit <= tr.lin[None, None, :]).all()
    for v in range(nv):
        assert np.array_equal(hit[v, 0], live[v])          # α = 0 segment replays == live pass
    W, ns = g.window, len(g.segs)
    with ThreadPoolExecutor(max_workers=min(nv, os.cpu_count() or 1)) as ex:
        lp = list(ex.map(lambda v: O.live_pass(tr, v, W, upto=2 * W), w.variants))
    for v in range(nv):
        snaps, h_live = lp[v][0], lp[v][1]
        assert np.array_equal(live[v][: 2 * W], h_live), v
        for k in (1, 2):
            gs, gn = g.ctx.get_snapshot(v, k)
            assert gn == snaps[k][1] and np.array_equal(GU.canon(gs), GU.canon(snaps[k][0])), (v, k)
    si = 1
    first, n, k = g.segs[si]
    flat = [lp[v][0][k] for v in range(nv)]
    chains = [(v, w.alphas[ai], first, n, v) for v in range(nv) for ai in range(na)]
    oh, of, ob, _, octr = O.run_chains(tr, w.variants, chains, flat, n_threads=os.cpu_count() or 1)
    sl = slice(first - 1, first - 1 + n)
    for i, (v, alpha, *_rest) in enumerate(chains):
        ai = i % na
        cid = (v * na + ai) * ns + si
        assert np.array_equal(hit[v, ai, sl], oh[i]), (v, ai)
        assert np.array_equal(fl[v, ai, sl], of[i].astype(np.int64)), (v, ai)
        assert np.array_equal(by[v, ai, sl], ob[i].astype(np.uint8)), (v, ai)
        assert np.array_equal(ctr[cid], octr[i].astype(np.int64)), (v, ai)
    logged = [(0, 5), (4, 15), (7, 1), (9, 9), (12, 12), (14, 3)]
    ids = [(v * na + ai) * ns + si for v, ai in logged]
    out2 = g.ctx.alloc_outputs(na, log_cap=1 << 15)
    g.ctx.replay(w.alphas, chains=ids, out=out2)
    g.ctx.check()
    for (v, ai), cid in zip(logged, ids):
        _, _, _, lg = GU.oracle_chain_log(tr, w.variants[v], w.alphas[ai], first, n, flat[v])
        glog, gn = g.ctx.read_log(out2, cid)
        _assert_logs_equal(glog, gn, lg, f"cfg5 v{v} a{ai}")
    a_star = g.select(out)
    assert len(a_star) == 15 and all(a in w.alphas for a in a_star)


def test_errors_are_loud():
    tr = tg.workload(3, R=2000).trace
    v = tg.Variant(tg.MODEL_7B, 60 * tg.GB)
    ctx = M.Context([v], max_nodes=64)   # far too small for this trace
    ctx.upload_trace(tr.tokens, tr.off, tr.lin, tr.lout)
    with pytest.raises(M.MarconiError) as e:
        ctx.live_pass(200)
    assert "MC_EOVERFLOW" in str(e.value)
    ctx2 = M.Context([v], max_nodes=8192)
    ctx2.upload_trace(tr.tokens, tr.off, tr.lin, tr.lout)
    ctx2.live_pass(1000)
    ctx2.set_segments([(1, 1000, 0)])
    with pytest.raises(M.MarconiError):
        ctx2.replay([-1.0])
    with pytest.raises(M.MarconiError):
        M.Context([tg.Variant(tg.Model(0, 4, 4), 10)], max_nodes=64)


# ---------------------------------------------------------------- NEXT-3: chunk-aligned checkpoints
def test_chunked_paper_example_on_gpu():
    """branch at 80, chunk 32 -> the state is checkpointed at 64."""
    A = list(range(1, 81))
    reqs = [(A + [500 + j for j in range(20)], []), (A + [600 + j for j in range(20)], []),
            (A + [700 + j for j in range(20)], [])]
    tr = tg.from_sequences(reqs)
    for chunk, want in ((32, [0, 0, 64]), (0, [0, 0, 80]), (128, [0, 0, 0])):
        v = tg.Variant(tg.MODEL_7B, tg.UNLIMITED_BYTES, 0, chunk)
        g, out = GU.gpu_grid(tr, [v], [0.0], 1, max_nodes=64)
        assert out["hit"].cpu().numpy()[0, 0].tolist() == want, chunk


def test_chunked_micro_traces():
    for chunk in (2, 3, 8):
        for seed in range(60):
            tr = tg.micro_trace(seed, n_req=20, max_len=64, alphabet=2 + seed % 3)
            v = tg.Variant(tg.MODEL_7B, tg.UNLIMITED_BYTES, 2 + seed % 6, chunk)
            alphas = [0.0, tg.ALPHA_GRID16[seed % 16]]
            g, out = GU.gpu_grid(tr, [v], alphas, 2, max_nodes=128, log_cap=256)
            snaps, live, res, segs = GU.oracle_grid(tr, [v], alphas, 2, threads=1)
            for k in range(len(snaps[0])):
                gs, gn = g.ctx.get_snapshot(0, k)
                assert gn == snaps[0][k][1] and np.array_equal(GU.canon(gs), GU.canon(snaps[0][k][0]))
            hit = out["hit"].cpu().numpy()
            for cid, (h, f, b, c) in res.items():
                ai, si = cid // len(segs), cid % len(segs)
                first, n, k = segs[si]
                assert np.array_equal(hit[0, ai, first - 1:first - 1 + n], h), (chunk, seed, cid)
                _, _, _, lg = GU.oracle_chain_log(tr, v, alphas[ai], first, n, snaps[0][k])
                glog, gn = g.ctx.read_log(out, cid)
                _assert_logs_equal(glog, gn, lg, f"chunk {chunk} seed {seed}")


@pytest.mark.parametrize("chunk", [32, 256])
def test_chunked_config3_reduced(chunk):
    w = tg.workload(3, R=6000)
    w.variants = [tg.Variant(tg.MODEL_7B, 60 * tg.GB, 0, chunk)]
    w.n_segments = 12
    _compare_grid(w)


def test_chunked_config4_full():
    w = tg.workload(4)
    w.variants = [tg.Variant(tg.MODEL_7B, 60 * tg.GB, 0, 64)]
    _compare_grid(w)


# ---------------------------------------------------------------- NEXT-4: sweeps on the same kernels
def test_state_dim_sweep():
    """fig:microbenchmark_state_dim axis: N in {16, 32, 64, 128} as 4 cache variants
    of one grid (one context, one launch), every chain vs the oracle."""
    w = tg.workload(3, R=5000)
    w.variants = tg.state_dim_variants()
    w.alphas = (0.0, 1 / 16, 1.0, 16.0)
    w.n_segments = 10
    _compare_grid(w)


@pytest.mark.parametrize("rate,delay", [(0.5, 5.0), (2.0, 5.0), (1.0, 10.0)])
def test_arrival_sweep(rate, delay):
    """fig:micro_arrival axes: session rate 0.5 -> 2 /s, response time 5 -> 10 s."""
    w = tg.arrival_workload(rate, delay, R=6000, n_segments=12, alphas=(0.0, 0.25, 4.0))
    _compare_grid(w)


# ---------------------------------------------------------------- NEXT-2: vLLM+ baseline
def _vllm(model, capb, capn, x):
    return tg.Variant(model, capb, capn, 0, x)


def test_vllm_occurrence_rule_on_gpu():
    """PAPER:378 + PAPER:532: block checkpointing reuses a purely-input prefix from its
    second occurrence, whole blocks only."""
    P = list(range(7, 107))
    tr = tg.from_sequences([(P, [900 + k, 901 + k]) for k in range(3)])
    g, out = GU.gpu_grid(tr, [_vllm(tg.MODEL_7B, tg.UNLIMITED_BYTES, 0, 32)], [0.0], 1, max_nodes=64)
    assert out["hit"].cpu().numpy()[0, 0].tolist() == [0, 96, 96]


def test_vllm_micro_traces():
    """Micro traces x block sizes 1..8 x byte / node capacities, two segments, two α
    (ignored by the policy): snapshots, per-request hits and eviction logs vs the oracle."""
    for seed in range(120):
        tr = tg.micro_trace(seed, n_req=20, max_len=64, alphabet=2 + seed % 3)
        model = tg.MODEL_7B if seed % 2 else tg.MODEL_TOY
        x = 1 + seed % 8
        bb = FL_KVT(model) * x + FL_SSMB(model)
        k = seed % 3
        capb, capn = ((tg.UNLIMITED_BYTES, 2 + seed % 7) if k == 0 else
                      ((2 + seed % 5) * bb + seed % 7, 0) if k == 1 else ((3 + seed % 4) * bb, 3 + seed % 5))
        v = _vllm(model, capb, capn, x)
        alphas = [0.0, 1.0]
        g, out = GU.gpu_grid(tr, [v], alphas, 2, max_nodes=128, log_cap=256, counters=True)
        snaps, live, res, segs = GU.oracle_grid(tr, [v], alphas, 2, threads=1)
        for kk in range(len(snaps[0])):
            gs, gn = g.ctx.get_snapshot(0, kk)
            assert gn == snaps[0][kk][1] and np.array_equal(GU.canon(gs), GU.canon(snaps[0][kk][0])), (seed, kk)
        hit = out["hit"].cpu().numpy()
        ctr = out["counters"].cpu().numpy()
        for cid, (h, f, b, c) in res.items():
            ai, si = cid // len(segs), cid % len(segs)
            first, n, kk = segs[si]
            assert np.array_equal(hit[0, ai, first - 1:first - 1 + n], h), (seed, cid)
            assert np.array_equal(ctr[cid], c.astype(np.int64)), (seed, cid, ctr[cid], c)
            _, _, _, lg = GU.oracle_chain_log(tr, v, alphas[ai], first, n, snaps[0][kk])
            glog, gn = g.ctx.read_log(out, cid)
            _assert_logs_equal(glog, gn, lg, f"vllm seed {seed}")
        assert np.array_equal(hit[0, 0], hit[0, 1])  # α does not enter LRU


def FL_KVT(m):
    return m.n_attn * 2 * m.d_model * m.bytes_per_param


def FL_SSMB(m):
    return m.n_ssm * (m.d_model * m.d_state + m.conv_in * m.conv_kernel) * m.bytes_per_param


@pytest.mark.parametrize("x", [16, 32, 64])
def test_vllm_config3_reduced(x):
    w = tg.workload(3, R=5000)
    w.variants = [_vllm(tg.MODEL_7B, 60 * tg.GB, 0, x)]
    w.alphas = (0.0,)
    w.n_segments = 10
    _compare_grid(w, log_cap=4096)


def test_vllm_and_marconi_in_one_grid():
    """Mixed policies in one context: the replay runs the Marconi chains and the vLLM+
    chains as two launches; both match the oracle; Marconi's hit sum is compared too."""
    w = tg.workload(3, R=4000)
    w.variants = [tg.Variant(tg.MODEL_7B, 60 * tg.GB), _vllm(tg.MODEL_7B, 60 * tg.GB, 0, 32)]
    w.alphas = (0.0, 0.5, 2.0)
    w.n_segments = 8
    _compare_grid(w)


def test_vllm_config2_full():
    w = tg.workload(2)
    w.variants = [_vllm(v.model, v.capacity_bytes, v.capacity_nodes, 32) for v in w.variants]
    w.alphas = (0.0,)
    _compare_grid(w)


def test_vllm_config4_reduced():
    """SWEBench-shaped (32K-token contexts): ~1000 blocks per sequence, ~125 evictions
    per request (the oracle's cost bounds the size: 600 requests, 4 segments)."""
    w = tg.workload(4, R=600)
    w.variants = [_vllm(tg.MODEL_7B, 60 * tg.GB, 0, 32)]
    w.alphas = (0.0,)
    w.n_segments = 4
    _compare_grid(w)


def test_dense_positions_beyond_half_the_node_table():
    """Regression: live counts above max_nodes/2 on concurrent workers (the exact-eff array
    of one worker slice used to overrun into the next slice)."""
    w = tg.workload(3, R=3000)
    w.n_segments = 8
    w.alphas = (0.0, 1.0, 4.0)
    _compare_grid(w, R_cap_nodes=2048)
    w.variants = [_vllm(tg.MODEL_7B, 120 * tg.GB, 0, 16)]
    w.alphas = (0.0,)
    _compare_grid(w)


# ---------------------------------------------------------------- fp32 filter edge cases
def test_adversarial_filter_near_ties():
    """The kernel's fp32 filter-and-verify argmin on built edge
    cases (tests/adversarial.py): Δe32 = 0 and 1 ulp, top-2 exact utilities within 4 ulps,
    α = 64 (up to 1e300) with a tiny Δe, exact (u, t) ties.  Snapshots are uploaded through
    mc_set_snapshots; every eviction of every (case, α) chain -- logs OFF first (the bench
    branch: hits, FLOPs, bypass, counters), then logs ON -- must equal the oracle's,
    utilities bit for bit."""
    import adversarial as A
    n_ev = 0
    for c in A.make_cases(range(240)):
        ctx = M.Context([c.variant], max_nodes=128)
        ctx.upload_trace(c.trace.tokens, c.trace.off, c.trace.lin, c.trace.lout)
        ctx.set_snapshots(0, [c.snapshot])
        ctx.set_segments([(c.first, c.n, 0)])
        o0 = ctx.replay(c.alphas, counters=True)
        o1 = ctx.replay(c.alphas, log_cap=16, counters=True)
        ctx.check()
        sl = slice(c.first - 1, c.first - 1 + c.n)
        for ai, a in enumerate(c.alphas):
            h, f, b, lg = GU.oracle_chain_log(c.trace, c.variant, a, c.first, c.n, c.snapshot)
            for o in (o0, o1):
                assert np.array_equal(o["hit"].cpu().numpy()[0, ai, sl], h), a
                assert np.array_equal(o["flops"].cpu().numpy()[0, ai, sl], f.astype(np.int64)), a
                assert np.array_equal(o["bypass"].cpu().numpy()[0, ai, sl], b.astype(np.uint8)), a
            assert torch.equal(o0["counters"], o1["counters"])
            glog, gn = ctx.read_log(o1, ai)
            _assert_logs_equal(glog, gn, lg, f"case {c.tmode} alpha {a!r}")
            n_ev += gn
        ctx.close()
    assert n_ev > 5000
