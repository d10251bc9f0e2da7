"""Adversarial eviction cases for the fp32 filter-and-verify victim selection (test input).

The kernel selects the Eq. 2 argmin with an fp32 filter key and verifies
the survivors with the exact IEEE fp64 recipe.  Random traces
reach its edge cases only by chance, so this module BUILDS them:

  * Δe32 = 0: every node's FLOP efficiency rounds to the same fp32 value while the fp64
    values differ (the kernel must fall back to the exact pass);
  * Δe32 = 1 fp32 ulp;
  * the top-2 exact utilities 1-4 fp64 ulps apart (α placed at the crossing of two
    lower-hull candidates, and its fp64 neighbours);
  * α = 64 (and α up to 1e300) with a tiny relative Δe;
  * exact (u, t) ties, decided by the node id (reading R4).

A case = a tree snapshot (built by the ORACLE from a micro trace with unlimited capacity,
then re-stamped with adversarial t_last values) + a window of fresh requests, each of
which must evict exactly one node (node cap = snapshot size), + an α list.  The first
eviction of every window sees exactly the snapshot's state (a fresh request matches
nothing: no pin, no touch), so `classify` can compute, on the test side, which edge case
it exercises.  Parity itself is GPU log == oracle log, bit for bit.

Models: the 7B hybrid, and KV-only "wide-MLP" models (n_ssm = 0, tiny d_model, tens of
millions of MLP layers) whose FLOP efficiency is dominated by a constant, so that Δe is a
few fp32 ulps or less while F(L) stays < 2^53 for the short sequences used here.
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Tuple

import numpy as np

import oracle as O
import tracegen as tg

# KV-only wide-MLP models: eff = D (4 + 8 nM/nA)/bpp + 2 (d_start + d_end)/bpp (Appendix A
# with n_ssm = 0), i.e. a huge constant plus a tiny depth term.
WIDE = [
    tg.Model(1, 0, 31_250_000, 64, 1, 4, 0, 0),   # eff ~ 4.0e9, fp32 ulp 512, depth term <= 64
    tg.Model(1, 0, 6_250_000, 64, 1, 4, 0, 0),    # eff ~ 8.0e8, ulp 64: often 1 ulp apart
    tg.Model(1, 0, 2_000_000, 64, 1, 4, 0, 0),    # eff ~ 2.6e8, ulp 16-32
    tg.Model(2, 0, 600_000, 32, 1, 2, 0, 0),      # eff ~ 3.8e7, ulp 2-4
    tg.Model(1, 1, 3_000_000, 64, 1, 4, 0, 0),    # hybrid: 256 B of state per checkpoint (2/3 of a token's KVs)
]
MODELS = [tg.MODEL_7B] + WIDE


@dataclasses.dataclass
class Case:
    trace: tg.Trace
    variant: tg.Variant
    snapshot: Tuple[np.ndarray, int]
    first: int
    n: int
    alphas: List[float]
    tmode: str


def _eff_exact(model, ds: int, de: int, ssm: bool) -> float:
    """Eq. 1 with exact integer ΔF and bytes, one correctly rounded division (classification only)."""
    D, N = model.d_model, model.d_state

    def F(L):
        return (model.n_attn * (8 * L * D * D + 4 * L * L * D) + model.n_mlp * 16 * L * D * D
                + model.n_ssm * (12 * L * D * D + 16 * L * D * N + 10 * L))
    kvt = model.n_attn * 2 * D * model.bytes_per_param
    ssmb = model.n_ssm * (D * N + model.conv_in * model.conv_kernel) * model.bytes_per_param
    return float(F(de) - F(ds)) / float(kvt * (de - ds) + (ssmb if ssm else 0))


def first_eviction_state(model, nodes):
    """(t, eff, cand, id) arrays of the snapshot's nodes (candidates: <= 1 child)."""
    ids = nodes["id"].astype(np.int64)
    par = nodes["parent_id"].astype(np.int64)
    nch = {int(i): 0 for i in ids}
    for p in par:
        if p:
            nch[int(p)] += 1
    t = nodes["t_last"].astype(np.int64)
    eff = np.array([_eff_exact(model, int(x["d_start"]), int(x["d_end"]), bool(x["has_ssm"])) for x in nodes])
    cand = np.array([nch[int(i)] <= 1 for i in ids])
    return t, eff, cand, ids


def utilities(t, eff, alpha):
    """Eq. 2 with min-max normalisation, every op rounded separately (numpy fp64 = IEEE)."""
    tmin, tmax, emin, emax = t.min(), t.max(), eff.min(), eff.max()
    rec = np.full(t.shape, 0.5) if tmax == tmin else (t - tmin).astype(np.float64) / float(tmax - tmin)
    effn = np.full(t.shape, 0.5) if emax == emin else (eff - emin) / (emax - emin)
    with np.errstate(over="ignore"):
        return rec + np.float64(alpha) * effn


def crossing_alphas(t, eff, cand, k=3):
    """α values at which two candidates tie for the minimum utility (lower-hull crossings)."""
    tmin, tmax, emin, emax = t.min(), t.max(), eff.min(), eff.max()
    if tmax == tmin or emax == emin:
        return []
    rec = (t - tmin).astype(np.float64) / float(tmax - tmin)
    effn = (eff - emin) / (emax - emin)
    ci = np.nonzero(cand)[0]
    out = []
    for a_i in ci:
        for b_i in ci:
            if effn[a_i] > effn[b_i] and rec[a_i] < rec[b_i]:
                al = (rec[b_i] - rec[a_i]) / (effn[a_i] - effn[b_i])
                if not (0 < al < 1e300):
                    continue
                u = utilities(t, eff, al)[ci]
                two = np.sort(u)[:2]
                if two[1] - two[0] <= 8 * np.spacing(two[0]):
                    out.append(float(al))
    out = sorted(set(out))
    if len(out) > k:
        out = [out[i * len(out) // k] for i in range(k)]
    return out


def classify(case: Case):
    """Edge cases exercised by the FIRST eviction of the case's window, per α."""
    nodes, _ = case.snapshot
    t, eff, cand, ids = first_eviction_state(case.variant.model, nodes)
    lo32, hi32 = np.float32(eff.min()), np.float32(eff.max())
    de32 = float(hi32) - float(lo32)
    tags = set()
    if de32 == 0 and eff.max() != eff.min():
        tags.add("de32_zero")
    if de32 != 0 and np.nextafter(lo32, np.float32(np.inf)) == hi32:
        tags.add("de32_one_ulp")
    rel = (eff.max() - eff.min()) / eff.max()
    ci = np.nonzero(cand)[0]
    for a in case.alphas:
        u = utilities(t, eff, a)[ci]
        order = np.lexsort((ids[ci], t[ci], u))
        if len(order) < 2:
            continue
        u0, u1 = u[order[0]], u[order[1]]
        if a >= 64 and rel < 1e-6:
            tags.add("alpha64_tiny_de")
        if u0 == u1 and t[ci][order[0]] == t[ci][order[1]]:
            tags.add("u_t_tie_id_decides")
        elif u0 == u1:
            tags.add("u_tie_t_decides")
        elif u1 - u0 <= 4 * np.spacing(u0):
            tags.add("top2_within_4ulp")
    return tags


def _fresh(seed: int, k: int, base: int) -> List[Tuple[list, list]]:
    rng = np.random.default_rng(seed)
    out = []
    for j in range(k):
        L = int(rng.integers(2, 12))
        s = [base + 1000 * j + i for i in range(L)]
        lin = int(rng.integers(1, L + 1))
        out.append((s[:lin], s[lin:]))
    return out


def make_case(seed: int) -> Case:
    rng = np.random.default_rng(10_000 + seed)
    model = MODELS[seed % len(MODELS)]
    mt = tg.micro_trace(seed, n_req=int(rng.integers(8, 21)), max_len=48, alphabet=2 + seed % 3)
    hist = []
    for r in range(1, mt.n_requests + 1):
        s = [int(x) for x in mt.seq(r)]
        L = int(mt.lin[r - 1])
        hist.append((s[:L], s[L:]))
    K = 6
    tr = tg.from_sequences(hist + _fresh(seed, K, 1 << 20))
    R1 = len(hist)
    o = O.Oracle(tr, model, tg.UNLIMITED_BYTES, 0, 0.0)
    o.run(1, R1)
    nodes, nid = o.dump()
    o.close()
    # adversarial timestamps (all < the window's request indices)
    tmode = ("ties", "few", "spread", "pairs")[seed % 4]
    n = len(nodes)
    if tmode == "ties":
        nodes["t_last"] = 1 + rng.integers(0, 2, n)
    elif tmode == "few":
        nodes["t_last"] = 1 + rng.integers(0, 4, n)
    elif tmode == "pairs":
        nodes["t_last"] = 1 + (np.arange(n) // 2) % R1
    t, eff, cand, ids = first_eviction_state(model, nodes)
    alphas = {0.0, 1.0, 64.0}
    for a in crossing_alphas(t, eff, cand):
        alphas.update([a, float(np.nextafter(a, 0.0)), float(np.nextafter(a, np.inf))])
    if seed % 5 == 0:
        alphas.update([1e30, 1e300])  # ADVICE: huge α must not overflow the fp32 filter
    v = tg.Variant(model, tg.UNLIMITED_BYTES, n)
    return Case(tr, v, (nodes, nid), R1 + 1, K, sorted(alphas), tmode)


def make_cases(seeds) -> List[Case]:
    return [c for c in (make_case(s) for s in seeds) if len(c.snapshot[0]) >= 2]
