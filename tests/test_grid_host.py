"""Host logic of the α-grid driver (no GPU): the chain-id layout of the live-pass cost
model, longest-first ordering by measured cycles, and the copy-layout trace transform."""
import numpy as np

import tracegen as tg
from paper_2411_19379_b200.grid import AlphaGrid, chain_costs_live, chain_id, lpt_shard


def test_chain_costs_live_follow_chain_ids():
    segs = [(1, 10, 0), (11, 10, 1), (21, 5, 2)]
    wc = [np.array([7, 3, 9], np.uint64), np.array([1, 8, 2], np.uint64)]  # [variant][segment]
    n_alpha = 4
    c = chain_costs_live(wc, segs, n_alpha)
    assert c.shape == (2 * n_alpha * 3,)
    for v in range(2):
        for a in range(n_alpha):
            for s in range(3):
                assert c[chain_id(v, a, s, n_alpha, 3)] == int(wc[v][s])
    # LPT over these costs: every chain exactly once, longest first on one rank
    order = lpt_shard(c, 3, n_alpha, 1)[0]
    assert sorted(order.tolist()) == list(range(c.shape[0]))
    assert np.all(np.diff(c[order.astype(np.int64)]) <= 0)


def test_reorder_by_cycles_longest_first_same_set():
    g = AlphaGrid.__new__(AlphaGrid)  # host logic only (no context)
    g.chains = np.array([5, 2, 9, 0, 7], np.uint32)
    cyc = np.zeros(10, np.int64)
    cyc[[5, 2, 9, 0, 7]] = [30, 50, 10, 50, 40]
    g.reorder_by_cycles(cyc)
    assert g.chains.tolist() == [0, 2, 7, 5, 9]  # ties (50) by chain id


def test_copy_layout_keeps_every_sequence():
    w = tg.workload(3, R=800)
    c = w.trace.copy_layout()
    assert c.n_requests == w.trace.n_requests
    n = w.trace.lin.astype(np.int64) + w.trace.lout
    assert c.n_tokens == int(n.sum())
    assert np.all(np.diff(c.off.astype(np.int64)) == n[:-1])  # disjoint, back to back
    for r in (1, 2, 400, 800):
        assert np.array_equal(c.seq(r), w.trace.seq(r))
