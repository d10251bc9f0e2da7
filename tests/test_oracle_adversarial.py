"""The adversarial eviction cases (tests/adversarial.py) really reach the fp32 filter's
edge cases, and the oracle's choice on them is the Eq. 2 argmin.

* coverage: Δe32 = 0, Δe32 = 1 ulp, top-2 utilities within 4 fp64 ulps, α >= 64 with a
  relative Δe < 1e-6, exact (u, t) ties (id decides) and exact u ties (t decides) each
  occur in many cases' first evictions;
* pin: the oracle's first victim and its utility bits equal an independent numpy
  evaluation of Eq. 2 + min-max normalisation + the (u, t, id) argmin (reading R4) on
  the snapshot state (a fresh request pins and touches nothing).
"""
import collections

import numpy as np

import adversarial as A
import oracle as O

SEEDS = range(240)


def test_cases_cover_the_filter_edge_cases():
    cnt = collections.Counter()
    for c in A.make_cases(SEEDS):
        cnt.update(A.classify(c))
    for tag in ("de32_zero", "de32_one_ulp", "top2_within_4ulp", "alpha64_tiny_de", "u_t_tie_id_decides",
                "u_tie_t_decides"):
        assert cnt[tag] >= 20, (tag, cnt)


def test_oracle_first_victim_is_the_eq2_argmin():
    n = 0
    for c in A.make_cases(SEEDS):
        nodes, nid = c.snapshot
        t, eff, cand, ids = A.first_eviction_state(c.variant.model, nodes)
        ci = np.nonzero(cand)[0]
        for a in c.alphas:
            o = O.Oracle(c.trace, c.variant.model, c.variant.capacity_bytes, c.variant.capacity_nodes, a)
            o.load(nodes, nid)
            o.run(c.first, 1)
            lg = o.log()
            o.close()
            u = A.utilities(t, eff, a)[ci]
            best = np.lexsort((ids[ci], t[ci], u))[0]
            assert len(lg) == 1 and int(lg[0]["node_id"]) == int(ids[ci][best]), (a, lg)
            assert np.float64(lg[0]["utility"]).view(np.uint64) == np.float64(u[best]).view(np.uint64)
            n += 1
    assert n > 1000
