"""CPU oracle for the Marconi α-grid replay -- TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
reference legs may import this package.  The product path
(paper_2411_19379_b200) never imports it and shares no code with it.

`oracle.cpp` is a plain pointer radix tree following SURVEY.md §8(c) c.2 step
by step, citing PAPER.md (§3; §4.1; §4.2 Eq. 1/2
PAPER:395-427; §4.3; Appendix A).  This module is
a thin ctypes wrapper around it.

Parity status of each function:
  cost model (prefill_flops, layer_terms, node_cost)   pinned: closed forms, SPEC goldens
  Oracle.step / run (walk, admission, eviction)          pinned: worked examples S1-S6/E1/E2,
                                                          flat-list brute force, independent LRU,
                                                          OPT bound, invariants
  run_chains (α-grid over segments)                     pinned: α=0 segment replay == live pass
  counters (d.3 algorithmic bytes)                       pinned: the flat-list simulator's own
                                                          counts (tests/flatlist.py) + S1 by hand
  live_pass (segment snapshots)                          pinned: as Oracle.run + dump round-trip
  Oracle.lookup (steps 1-4, read-only)                   pinned: the flat-list simulator's own lookup
                                                          (tests/flatlist.py FlatCache.lookup) and
                                                          the next step's hit
"""
from __future__ import annotations

import ctypes as C
import os
from typing import List, Optional, Sequence, Tuple

import numpy as np

from . import build as _build

_LIB = None


class orc_model(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("n_attn", "n_ssm", "n_mlp", "d_model", "d_state",
                                          "bytes_per_param", "conv_in", "conv_kernel")]


NODE_DTYPE = np.dtype([("id", "<u4"), ("parent_id", "<u4"), ("ref_off", "<u8"), ("d_start", "<u4"),
                       ("d_end", "<u4"), ("t_last", "<u4"), ("has_ssm", "<u4")], align=True)
EVICT_DTYPE = np.dtype([("req", "<u4"), ("node_id", "<u4"), ("kind", "<u4"), ("n_live", "<u4"),
                        ("utility", "<f8")], align=True)
LOOKUP_DTYPE = np.dtype([("reuse", "<u4"), ("m", "<u4"), ("p", "<u4"), ("hit_id", "<u4"), ("div_id", "<u4"),
                         ("div_off", "<u4"), ("path_len", "<u4"), ("d_nodes", "<u4"), ("d_bytes", "<u8")])
assert NODE_DTYPE.itemsize == 32 and EVICT_DTYPE.itemsize == 24 and LOOKUP_DTYPE.itemsize == 40


def lib():
    global _LIB
    if _LIB is None:
        path = _build.build()
        L = C.CDLL(path)
        P, U32, U64, D = C.c_void_p, C.c_uint32, C.c_uint64, C.c_double
        L.orc_last_error.restype = C.c_char_p
        L.orc_create.restype = P
        L.orc_create.argtypes = [P, U64, U32, D, P, U64, P, P, P, U32]
        L.orc_destroy.argtypes = [P]
        L.orc_set_alpha.argtypes = [P, D]
        L.orc_set_chunk.argtypes = [P, U32]
        L.orc_set_block.argtypes = [P, U32]
        L.orc_load.argtypes = [P, P, U32, U32]
        L.orc_step.argtypes = [P, U32, P, P, P]
        L.orc_run.argtypes = [P, U32, U32, P, P, P]
        L.orc_dump.argtypes = [P, P, U64, P, P]
        L.orc_log.argtypes = [P, P, U64, P]
        L.orc_counters.argtypes = [P, P]
        L.orc_lookup_req.argtypes = [P, U32, P]
        L.orc_total.argtypes = [P, P, P]
        L.orc_prefill_flops.argtypes = [P, U64, P]
        L.orc_layer_terms.argtypes = [P, U64, P]
        L.orc_node_cost.argtypes = [P, U64, U64, U32, P, P, P]
        L.orc_score_argmin.argtypes = [U32, P, P, P, P, D, P, P]
        L.orc_run_chains.argtypes = [P, P, P, P, P, P, P, P, P, P, P, P, P, U32, P, U64, P, P, P, U32, P,
                                     P, P, P, P, P, U32]
        _LIB = L
    return _LIB


class OracleError(RuntimeError):
    pass


def _check(rc):
    if rc != 0:
        raise OracleError(lib().orc_last_error().decode())


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _model(m) -> orc_model:
    return orc_model(*m.astuple())


# --------------------------------------------------------------------------
# Cost model (Appendix A, tab:flops_breakdown)
# --------------------------------------------------------------------------
def prefill_flops(model, L: int) -> int:
    out = np.zeros(1, np.uint64)
    mm = _model(model)
    _check(lib().orc_prefill_flops(C.byref(mm), L, _ptr(out)))
    return int(out[0])


def layer_terms(model, L: int) -> dict:
    """Per-layer terms: attention/mlp/ssm FLOPs, kv bytes (per attn layer), ssm/conv state bytes."""
    out = np.zeros(6, np.uint64)
    mm = _model(model)
    _check(lib().orc_layer_terms(C.byref(mm), L, _ptr(out)))
    k = ("attention_flops", "mlp_flops", "ssm_flops", "kv_bytes", "ssm_state_bytes", "conv_state_bytes")
    return {a: int(b) for a, b in zip(k, out)}


def node_cost(model, d_start: int, d_end: int, has_ssm: bool) -> Tuple[int, int, float]:
    """(FLOPs saved relative to parent, bytes, FLOP efficiency) of a node (Eq. 1)."""
    s = np.zeros(1, np.uint64)
    b = np.zeros(1, np.uint64)
    e = np.zeros(1, np.float64)
    mm = _model(model)
    _check(lib().orc_node_cost(C.byref(mm), d_start, d_end, int(bool(has_ssm)), _ptr(s), _ptr(b), _ptr(e)))
    return int(s[0]), int(b[0]), float(e[0])


def score_argmin(t, cand, ids, eff, alpha: float):
    """Eviction choice on an explicit table (Eq. 2 + min-max normalisation + (u, t, id) argmin).
    Returns (row index or None, utility)."""
    t = np.ascontiguousarray(t, np.uint32)
    cand = np.ascontiguousarray(cand, np.uint8)
    ids = np.ascontiguousarray(ids, np.uint32)
    eff = np.ascontiguousarray(eff, np.float64)
    b = np.zeros(1, np.uint32)
    u = np.zeros(1, np.float64)
    _check(lib().orc_score_argmin(t.shape[0], _ptr(t), _ptr(cand), _ptr(ids), _ptr(eff), float(alpha),
                                  _ptr(b), _ptr(u)))
    return (None if b[0] == 0xFFFFFFFF else int(b[0])), float(u[0])


# --------------------------------------------------------------------------
# Replay
# --------------------------------------------------------------------------
class Oracle:
    """One cache (one chain): a radix tree replaying requests of `trace` in order."""

    def __init__(self, trace, model, capacity_bytes: int, capacity_nodes: int = 0, alpha: float = 0.0,
                 chunk: int = 0, block: int = 0):
        self.h = None
        self.trace = trace
        self._keep = (np.ascontiguousarray(trace.tokens, np.uint32), np.ascontiguousarray(trace.off, np.uint64),
                      np.ascontiguousarray(trace.lin, np.uint32), np.ascontiguousarray(trace.lout, np.uint32))
        self._mm = _model(model)
        t, o, li, lo = self._keep
        h = lib().orc_create(C.byref(self._mm), int(capacity_bytes), int(capacity_nodes), float(alpha),
                             _ptr(t), t.shape[0], _ptr(o), _ptr(li), _ptr(lo), o.shape[0])
        if not h:
            raise OracleError(lib().orc_last_error().decode())
        self.h = h
        if chunk:
            _check(lib().orc_set_chunk(self.h, int(chunk)))
        if block:  # vLLM+ baseline (NEXT-2): token blocks of `block`, LRU
            _check(lib().orc_set_block(self.h, int(block)))

    def close(self):
        if self.h:
            lib().orc_destroy(self.h)
            self.h = None

    __del__ = close

    def set_alpha(self, a: float):
        _check(lib().orc_set_alpha(self.h, float(a)))

    def load(self, nodes: np.ndarray, next_id: int):
        nodes = np.ascontiguousarray(nodes, dtype=NODE_DTYPE)
        _check(lib().orc_load(self.h, _ptr(nodes), nodes.shape[0], int(next_id)))

    def step(self, r: int) -> Tuple[int, int, int]:
        h = np.zeros(1, np.uint32)
        f = np.zeros(1, np.uint64)
        b = np.zeros(1, np.uint32)
        _check(lib().orc_step(self.h, r, _ptr(h), _ptr(f), _ptr(b)))
        return int(h[0]), int(f[0]), int(b[0])

    def lookup(self, r: int) -> np.ndarray:
        """Steps 1-4 of c.2 for request r against the current tree, without mutating it:
        one LOOKUP_DTYPE record (reuse, m, p, hit / divergence node, plan)."""
        out = np.zeros(1, LOOKUP_DTYPE)
        _check(lib().orc_lookup_req(self.h, r, _ptr(out)))
        return out[0]

    def run(self, first: int, n: int):
        """Replay requests first..first+n-1 -> (hit u32[n], flops u64[n], bypass u32[n])."""
        h = np.zeros(n, np.uint32)
        f = np.zeros(n, np.uint64)
        b = np.zeros(n, np.uint32)
        _check(lib().orc_run(self.h, first, n, _ptr(h), _ptr(f), _ptr(b)))
        return h, f, b

    def dump(self) -> Tuple[np.ndarray, int]:
        n = np.zeros(1, np.uint64)
        nid = np.zeros(1, np.uint32)
        _check(lib().orc_dump(self.h, None, 0, _ptr(n), _ptr(nid)))
        out = np.zeros(int(n[0]), NODE_DTYPE)
        _check(lib().orc_dump(self.h, _ptr(out), out.shape[0], _ptr(n), _ptr(nid)))
        return out, int(nid[0])

    def log(self) -> np.ndarray:
        n = np.zeros(1, np.uint64)
        _check(lib().orc_log(self.h, None, 0, _ptr(n)))
        out = np.zeros(int(n[0]), EVICT_DTYPE)
        _check(lib().orc_log(self.h, _ptr(out), out.shape[0], _ptr(n)))
        return out

    def counters(self) -> np.ndarray:
        """[Σ compared positions, Σ visited nodes, Σ nodes scanned by evictions, Σ records written]."""
        out = np.zeros(4, np.uint64)
        _check(lib().orc_counters(self.h, _ptr(out)))
        return out

    def total(self) -> Tuple[int, int]:
        t = np.zeros(1, np.uint64)
        c = np.zeros(1, np.uint64)
        _check(lib().orc_total(self.h, _ptr(t), _ptr(c)))
        return int(t[0]), int(c[0])


def _chunk(variant) -> int:
    return int(getattr(variant, "chunk_size", 0) or 0)


def _block(variant) -> int:
    return int(getattr(variant, "block_size", 0) or 0)


def live_pass(trace, variant, window: int, upto: Optional[int] = None):
    """The α = 0 live LRU pass from an empty cache (SURVEY.md §8(c) c.2 "Segment mode").

    Returns (snapshots, hit, flops, bypass) where snapshots[k] = (nodes, next_id) is
    the tree after request k*window (snapshots[0] is the empty tree).  `upto` stops
    after that many requests (default: the whole trace).
    """
    R = trace.n_requests if upto is None else upto
    o = Oracle(trace, variant.model, variant.capacity_bytes, variant.capacity_nodes, 0.0, _chunk(variant), _block(variant))
    snaps = [(np.zeros(0, NODE_DTYPE), 1)]
    hs, fs, bs = [], [], []
    r = 1
    while r <= R:
        n = min(window, R - r + 1)
        h, f, b = o.run(r, n)
        hs.append(h); fs.append(f); bs.append(b)
        r += n
        if n == window and r <= trace.n_requests:
            snaps.append(o.dump())
    o.close()
    return snaps, np.concatenate(hs), np.concatenate(fs), np.concatenate(bs)


def run_chains(trace, variants: Sequence, chains: Sequence[Tuple[int, float, int, int, int]],
               snapshots: Sequence[Tuple[np.ndarray, int]], n_threads: int = 0):
    """Replay independent chains across host threads.

    chains: (variant_idx, alpha, first_req, n_req, snapshot_idx).
    Returns (hit list of arrays, flops list, bypass list, hit_sum u64[n_chains], counters u64[n,4]).
    """
    if n_threads <= 0:
        n_threads = os.cpu_count() or 1
    nc = len(chains)
    models = (orc_model * len(variants))(*[_model(v.model) for v in variants])
    capb = np.asarray([v.capacity_bytes for v in variants], np.uint64)
    capn = np.asarray([v.capacity_nodes for v in variants], np.uint32)
    chk = np.asarray([_chunk(v) for v in variants], np.uint32)
    blk = np.asarray([_block(v) for v in variants], np.uint32)
    var = np.asarray([c[0] for c in chains], np.uint32)
    alp = np.asarray([c[1] for c in chains], np.float64)
    first = np.asarray([c[2] for c in chains], np.uint32)
    nreq = np.asarray([c[3] for c in chains], np.uint32)
    sidx = np.asarray([c[4] for c in chains], np.uint32)
    snodes = np.concatenate([s[0] for s in snapshots]) if snapshots else np.zeros(0, NODE_DTYPE)
    snodes = np.ascontiguousarray(snodes, NODE_DTYPE)
    soff = np.zeros(len(snapshots) + 1, np.uint64)
    soff[1:] = np.cumsum([s[0].shape[0] for s in snapshots])
    snid = np.asarray([s[1] for s in snapshots], np.uint32)
    out_off = np.zeros(nc, np.uint64)
    out_off[1:] = np.cumsum(nreq.astype(np.uint64))[:-1]
    tot = int(nreq.astype(np.uint64).sum())
    hit = np.zeros(tot, np.uint32)
    flops = np.zeros(tot, np.uint64)
    byp = np.zeros(tot, np.uint32)
    hsum = np.zeros(nc, np.uint64)
    ctr = np.zeros((nc, 4), np.uint64)
    t = np.ascontiguousarray(trace.tokens, np.uint32)
    o = np.ascontiguousarray(trace.off, np.uint64)
    li = np.ascontiguousarray(trace.lin, np.uint32)
    lo = np.ascontiguousarray(trace.lout, np.uint32)
    _check(lib().orc_run_chains(models, _ptr(capb), _ptr(capn), _ptr(chk), _ptr(blk), _ptr(var), _ptr(alp), _ptr(first), _ptr(nreq),
                                _ptr(sidx), _ptr(snodes), _ptr(soff), _ptr(snid), nc, _ptr(t), t.shape[0],
                                _ptr(o), _ptr(li), _ptr(lo), o.shape[0], _ptr(out_off), _ptr(hit),
                                _ptr(flops), _ptr(byp), _ptr(hsum), _ptr(ctr), n_threads))
    sl = [slice(int(a), int(a) + int(n)) for a, n in zip(out_off, nreq)]
    return [hit[s] for s in sl], [flops[s] for s in sl], [byp[s] for s in sl], hsum, ctr


def select_alpha(alphas: Sequence[float], hit_sums: Sequence[int]) -> float:
    """α* = argmax of Σ hits, ties to the smallest α (SURVEY c.3 #17)."""
    best = None
    for a, s in sorted(zip(alphas, hit_sums), key=lambda x: x[0]):
        if best is None or s > best[1]:
            best = (a, s)
    return best[0]


def live_tune(trace, variant, alphas: Sequence[float], multiplier: int = 10, n_threads: int = 0):
    """The paper's tuning loop on the oracle, step by step:
    α = 0 until the first request r_F whose admission evicted; snapshot; α = 0 over the
    bootstrap window (r_F, r_F + multiplier*r_F]; grid replay of that window from the
    snapshot; adopt α* for the rest.  Returns (hits, flops, info)."""
    R = trace.n_requests
    o = Oracle(trace, variant.model, variant.capacity_bytes, variant.capacity_nodes, 0.0, _chunk(variant), _block(variant))
    hits = np.zeros(R, np.uint32)
    flops = np.zeros(R, np.uint64)
    r_f = 0
    snap = None
    for r in range(1, R + 1):
        h, f, _ = o.step(r)
        hits[r - 1], flops[r - 1] = h, f
        if r_f == 0 and len(o.log()) > 0:
            r_f = r
            snap = o.dump()
            break
    info = {"r_first_evict": r_f, "alpha_star": 0.0, "window": None, "grid_hit_sums": None}
    if r_f == 0 or r_f >= R:  # never evicted (the loop ran to R) or evicted only at the end
        o.close()
        return hits, flops, info
    b_end = min(r_f + multiplier * r_f, R)
    info["window"] = (r_f + 1, b_end)
    h, f, _ = o.run(r_f + 1, b_end - r_f)           # live α = 0 bootstrap
    hits[r_f:b_end], flops[r_f:b_end] = h, f
    end_snap = o.dump() if b_end < R else None
    o.close()
    chains = [(0, a, r_f + 1, b_end - r_f, 0) for a in alphas]
    _, _, _, hs, _ = run_chains(trace, [variant], chains, [snap], n_threads=n_threads)
    a_star = select_alpha(alphas, [int(x) for x in hs])
    info["alpha_star"] = a_star
    info["grid_hit_sums"] = [int(x) for x in hs]
    if b_end < R:
        o2 = Oracle(trace, variant.model, variant.capacity_bytes, variant.capacity_nodes, a_star, _chunk(variant),
                    _block(variant))
        o2.load(*end_snap)
        h, f, _ = o2.run(b_end + 1, R - b_end)
        hits[b_end:], flops[b_end:] = h, f
        o2.close()
    return hits, flops, info
