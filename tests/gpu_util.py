"""Helpers shared by the GPU parity tests: run the CUDA path and the oracle on the same inputs."""
import numpy as np

import oracle as O
import tracegen as tg


def gpu_grid(trace, variants, alphas, n_segments, max_nodes=8192, log_cap=0, counters=False, snapshots=None,
             chains=None):
    """Device live pass (or uploaded snapshots) + replay of all (or the given) chains."""
    from paper_2411_19379_b200 import AlphaGrid
    g = AlphaGrid(trace, variants, alphas, n_segments, max_nodes=max_nodes)
    g.setup(snapshots=snapshots)
    if chains is not None:
        g.chains = np.asarray(chains, np.uint32)
        g.workspace = g.ctx.alloc_workspace(0, len(alphas), len(g.chains))
    out = g.run(log_cap=log_cap, counters=counters)
    g.ctx.check()
    return g, out


def oracle_grid(trace, variants, alphas, n_segments, threads=0, chains=None):
    """Oracle live pass per variant + oracle replay of every chain.

    Returns (snapshots {v: [(nodes, next_id)]}, live {v: (hit, flops, bypass)},
    per-chain results {chain_id: (hit, flops, bypass, counters)})."""
    R = trace.n_requests
    W = -(-R // n_segments)
    segs = [(k * W + 1, min(W, R - k * W), k) for k in range(n_segments) if k * W < R]
    snaps, live = {}, {}
    for v, var in enumerate(variants):
        s, h, f, b = O.live_pass(trace, var, W)
        snaps[v] = s
        live[v] = (h, f, b)
    ns, na = len(segs), len(alphas)
    res = {}
    for v, var in enumerate(variants):
        ch = []
        ids = []
        for a_i, a in enumerate(alphas):
            for s_i, (first, n, k) in enumerate(segs):
                cid = (v * na + a_i) * ns + s_i
                if chains is not None and cid not in chains:
                    continue
                ch.append((0, a, first, n, k))
                ids.append(cid)
        if not ch:
            continue
        hit, fl, by, hs, ctr = O.run_chains(trace, [var], ch, snaps[v], n_threads=threads)
        for i, cid in enumerate(ids):
            res[cid] = (hit[i], fl[i], by[i], ctr[i])
    return snaps, live, res, segs


def oracle_chain_log(trace, var, alpha, first, n, snap):
    o = O.Oracle(trace, var.model, var.capacity_bytes, var.capacity_nodes, alpha, getattr(var, "chunk_size", 0),
                 getattr(var, "block_size", 0))
    o.load(*snap)
    h, f, b = o.run(first, n)
    lg = o.log()
    o.close()
    return h, f, b, lg


def canon(nodes):
    """Rows (id, parent_id, ref_off, d_start, d_end, t_last, has_ssm) ordered by id."""
    a = np.asarray([tuple(int(x[k]) for k in ("id", "parent_id", "ref_off", "d_start", "d_end", "t_last",
                                               "has_ssm")) for x in nodes], dtype=np.int64).reshape(-1, 7)
    return a[np.argsort(a[:, 0], kind="stable")]
