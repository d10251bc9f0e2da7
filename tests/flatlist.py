"""Brute-force flat-list cache simulator -- an independent pin for the oracle.

A second, tree-free implementation of the same rules (SURVEY.md §8(c) c.1
"Flat-list simulator").  The cache is an unordered list of entries
(path = full root-to-node token tuple, has_ssm, t_last, id); every relation is
derived by brute force on each query:

  parent(e)   = the entry with the longest path that is a strict prefix of e.path (or root)
  children(e) = the entries whose parent is e
  boundary x  = some entry has path == S[:x]   (x = 0 is the root)
  m           = max over entries of LCP(S, e.path)
  bytes(e)    = KVT * (|e.path| - |parent(e).path|) + has_ssm * SSMB

A split adds an entry; a merge (absorption) just deletes the entry
because the child's path is unchanged.  Lookup = max{|e.path| : has_ssm,
e.path prefix of S, |e.path| <= L_in}.

It shares nothing with oracle/oracle.cpp (pure Python, no tree) and the cost
model is written here from tab:flops_breakdown independently.
Policies: "marconi" (Eq. 2 utility), "lru" (min (t_last, id)),
or a callable victim chooser (used by the OPT search).
"""
from __future__ import annotations

import copy
from typing import Callable, Dict, List, Optional, Tuple


def F(L: int, m) -> int:
    """Prefill FLOPs of L tokens: Σ layers of tab:flops_breakdown row 1."""
    D, N = m.d_model, m.d_state
    return (m.n_attn * (8 * L * D * D + 4 * L * L * D) + m.n_mlp * (16 * L * D * D)
            + m.n_ssm * (12 * L * D * D + 16 * L * D * N + 10 * L))


def KVT(m) -> int:  # KV bytes per token over all attention layers: n_attn * 2 * D * bpp
    return m.n_attn * 2 * m.d_model * m.bytes_per_param


def SSMB(m) -> int:  # one checkpoint: n_ssm * (D*N + conv_in*conv_k) * bpp
    return m.n_ssm * (m.d_model * m.d_state + m.conv_in * m.conv_kernel) * m.bytes_per_param


class Entry:
    __slots__ = ("path", "has_ssm", "t", "id")

    def __init__(self, path, has_ssm, t, id_):
        self.path, self.has_ssm, self.t, self.id = tuple(path), has_ssm, t, id_


def _lcp(a, b) -> int:
    k = 0
    n = min(len(a), len(b))
    while k < n and a[k] == b[k]:
        k += 1
    return k


class FlatCache:
    def __init__(self, model, cap_bytes: int, cap_nodes: int = 0, alpha: float = 0.0,
                 policy="marconi", chunk: int = 0):
        self.chunk = chunk
        self.m = model
        self.cap_bytes = cap_bytes
        self.cap_nodes = cap_nodes
        self.alpha = alpha
        self.policy = policy
        self.E: Dict[int, Entry] = {}
        self.next_id = 1
        self.log: List[Tuple[int, int, int, float]] = []
        # SURVEY.md §8(d) d.3 counters, derived here from the brute-force relations:
        # [Σ c_r = min(m+1, n), Σ v_r = |P| + 1, Σ_j N_j = live entries at eviction j,
        #  Σ w_r = records written (touch 1, split 2, gain 1, leaf 1, timestamp-only 1,
        #  leaf removal 1, absorption 2)]
        self.ctr = [0, 0, 0, 0]

    def clone(self) -> "FlatCache":
        c = copy.copy(self)
        c.E = {k: Entry(e.path, e.has_ssm, e.t, e.id) for k, e in self.E.items()}
        c.log = list(self.log)
        c.ctr = list(self.ctr)
        return c

    # ---- brute-force relations ----
    def parent_len(self, e: Entry) -> int:
        best = 0
        for f in self.E.values():
            if len(f.path) < len(e.path) and e.path[:len(f.path)] == f.path:
                best = max(best, len(f.path))
        return best

    def parent(self, e: Entry) -> Optional[Entry]:
        best = None
        for f in self.E.values():
            if len(f.path) < len(e.path) and e.path[:len(f.path)] == f.path:
                if best is None or len(f.path) > len(best.path):
                    best = f
        return best

    def n_children(self, e: Entry) -> int:
        return sum(1 for f in self.E.values() if f is not e and self.parent(f) is e)

    def bytes(self, e: Entry) -> int:
        return KVT(self.m) * (len(e.path) - self.parent_len(e)) + (SSMB(self.m) if e.has_ssm else 0)

    def total(self) -> int:
        return sum(self.bytes(e) for e in self.E.values())

    def at(self, S, x) -> Optional[Entry]:
        for e in self.E.values():
            if len(e.path) == x and tuple(S[:x]) == e.path:
                return e
        return None

    def eff(self, e: Entry) -> float:  # Eq. 1 relative to the parent
        pl = self.parent_len(e)
        return float(F(len(e.path), self.m) - F(pl, self.m)) / float(self.bytes(e))

    # ---- one request ----
    def lookup(self, inp, out) -> dict:
        """Steps 1-4 by brute force, read-only: m, reuse, the hit entry, the checkpoint p, the
        entry where the match ends (mid-edge: the shortest extension; else the entry at m,
        the root = id 0) with its matched edge length, |P| and the insertion plan."""
        S = tuple(inp) + tuple(out)
        n, L_in = len(S), len(inp)
        m = max([_lcp(S, e.path) for e in self.E.values()] + [0])
        hits = [e for e in self.E.values() if e.has_ssm and len(e.path) <= L_in and S[:len(e.path)] == e.path]
        if self.m.n_ssm == 0:
            reuse = min(m, L_in)
            cont = [e for e in self.E.values() if len(e.path) > reuse - 1 and reuse > 0
                    and e.path[:reuse] == S[:reuse] and self.parent_len(e) < reuse]
            hit = cont[0] if cont else None
        else:
            hit = max(hits, key=lambda e: len(e.path)) if hits else None
            reuse = len(hit.path) if hit else 0
        full = [e for e in self.E.values() if len(e.path) <= m and S[:len(e.path)] == e.path]
        m_mid = m > 0 and self.at(S, m) is None
        partial = None
        if m_mid:
            ext = [e for e in self.E.values() if len(e.path) > m and e.path[:m] == S[:m]]
            partial = min(ext, key=lambda e: len(e.path))
        m_in = min(m, L_in)
        q = 0
        if m_in > 0:
            b = self.at(S, m_in)
            if b is None or not b.has_ssm:
                q = m_in
        p = q
        if q and self.chunk:
            p = (q // self.chunk) * self.chunk
            if p == 0 or p <= reuse:
                p = 0
        p_split = False
        if p:
            b = self.at(S, p)
            if b is None:
                p_split = True
            elif b.has_ssm:
                p = 0
        n_splits = int(p_split) + int(m_mid and m < n and m != p) + int(m_mid and m == n and n != p)
        leaf = m < n
        n_gain = (not m_mid and m == n and n != p and not self.at(S, n).has_ssm)
        ck = (1 if p else 0) + (1 if n != p and (leaf or m_mid or n_gain) else 0)
        div = partial if m_mid else self.at(S, m)
        return {"reuse": reuse, "m": m, "p": p, "hit_id": hit.id if hit else 0,
                "div_id": div.id if div is not None else 0,
                "div_off": (m - self.parent_len(div)) if div is not None else 0,
                "path_len": len(full) + (1 if partial else 0),
                "d_nodes": n_splits + (1 if leaf else 0),
                "d_bytes": KVT(self.m) * (n - m) + SSMB(self.m) * ck}

    def step(self, r: int, inp, out, chooser: Optional[Callable] = None):
        S = tuple(inp) + tuple(out)
        n, L_in = len(S), len(inp)
        m = max([_lcp(S, e.path) for e in self.E.values()] + [0])
        # lookup (all-or-nothing)
        hits = [e for e in self.E.values() if e.has_ssm and len(e.path) <= L_in and S[:len(e.path)] == e.path]
        if self.m.n_ssm == 0:
            reuse = min(m, L_in)
            cont = [e for e in self.E.values() if len(e.path) > reuse - 1 and reuse > 0
                    and e.path[:reuse] == S[:reuse] and self.parent_len(e) < reuse]
            hit = cont[0] if cont else None
        else:
            hit = max(hits, key=lambda e: len(e.path)) if hits else None
            reuse = len(hit.path) if hit else 0
        # pinned path: fully matched entries + the partially matched one
        full = [e for e in self.E.values() if len(e.path) <= m and S[:len(e.path)] == e.path]
        m_mid = m > 0 and self.at(S, m) is None
        partial = None
        if m_mid:
            ext = [e for e in self.E.values() if len(e.path) > m and e.path[:m] == S[:m]]
            partial = min(ext, key=lambda e: len(e.path))
        P = full + ([partial] if partial else [])
        self.ctr[0] += min(m + 1, n)
        self.ctr[1] += len(P) + 1
        # speculative insertion with the c.3 #8/#9 readings
        m_in = min(m, L_in)
        q = 0
        if m_in > 0:
            b = self.at(S, m_in)
            if b is None or not b.has_ssm:
                q = m_in
        # chunked state passing: checkpoint at the chunk boundary <= q
        p = q
        if q and self.chunk:
            p = (q // self.chunk) * self.chunk
            if p == 0 or p <= reuse:
                p = 0
        p_split, p_gain = False, None
        if p:
            b = self.at(S, p)
            if b is None:
                p_split = True
            elif not b.has_ssm:
                p_gain = b
            else:
                p = 0
        splits = []
        if p_split:
            splits.append((p, True))
        if m_mid and m < n and m != p:
            splits.append((m, False))
        if m_mid and m == n and n != p:
            splits.append((n, True))
        splits.sort()
        leaf = m < n
        n_gain = None
        if not m_mid and m == n and n != p:
            b = self.at(S, n)
            if not b.has_ssm:
                n_gain = b
        ck = (1 if p else 0) + (1 if n != p and (leaf or m_mid or n_gain) else 0)
        d_bytes = KVT(self.m) * (n - m) + SSMB(self.m) * ck
        d_nodes = len(splits) + (1 if leaf else 0)
        if hit is not None:
            hit.t = r
            self.ctr[3] += 1
        pinned_bytes = sum(self.bytes(e) for e in P)
        bypass = (pinned_bytes + d_bytes > self.cap_bytes or
                  (self.cap_nodes and len(P) + d_nodes > self.cap_nodes))
        if not bypass:
            pids = {id(e) for e in P}
            while (self.total() + d_bytes > self.cap_bytes or
                   (self.cap_nodes and len(self.E) + d_nodes > self.cap_nodes)):
                cands = [e for e in self.E.values() if id(e) not in pids and self.n_children(e) <= 1]
                assert cands, "no candidate"
                victim, u = self._choose(cands, chooser, r)
                kind = 0 if self.n_children(victim) == 0 else 1
                self.log.append((r, victim.id, kind, u))
                self.ctr[2] += len(self.E)
                self.ctr[3] += 1 + kind
                del self.E[victim.id]
            for x, stateful in splits:
                self.E[self.next_id] = Entry(S[:x], stateful, r, self.next_id)
                self.next_id += 1
                self.ctr[3] += 2  # the new upper entry and the lower one's shortened edge
            if p_gain is not None:
                p_gain.has_ssm, p_gain.t = True, r
                self.ctr[3] += 1
            if n_gain is not None:
                n_gain.has_ssm, n_gain.t = True, r
                self.ctr[3] += 1
            if leaf:
                self.E[self.next_id] = Entry(S, True, r, self.next_id)
                self.next_id += 1
                self.ctr[3] += 1
            else:
                fin = self.at(S, n)
                if not m_mid and n_gain is None and fin is not p_gain:
                    self.ctr[3] += 1  # timestamp-only write of the existing final entry
                fin.t = r
        return reuse, F(reuse, self.m), int(bool(bypass))

    def _choose(self, cands, chooser, r):
        if chooser is not None:
            v = chooser(self, cands, r)
            return v, float("nan")
        if self.policy == "lru":
            v = min(cands, key=lambda e: (e.t, e.id))
            return v, float("nan")
        allv = list(self.E.values())
        ts = [e.t for e in allv]
        es = [self.eff(e) for e in allv]
        tmin, tmax, emin, emax = min(ts), max(ts), min(es), max(es)
        best = None
        for e in cands:
            rec = 0.5 if tmax == tmin else float(e.t - tmin) / float(tmax - tmin)
            effn = 0.5 if emax == emin else (self.eff(e) - emin) / (emax - emin)
            u = rec + self.alpha * effn
            key = (u, e.t, e.id)
            if best is None or key < best[0]:
                best = (key, e)
        return best[1], best[0][0]

    def dump(self):
        """Canonical dump tuples (id, parent_id, d_start, d_end, has_ssm, t_last), by id."""
        out = []
        for e in sorted(self.E.values(), key=lambda e: e.id):
            par = self.parent(e)
            out.append((e.id, par.id if par else 0, self.parent_len(e), len(e.path), int(e.has_ssm), e.t))
        return out


def replay(trace, model, cap_bytes, cap_nodes, alpha, policy="marconi", chunk=0):
    c = FlatCache(model, cap_bytes, cap_nodes, alpha, policy, chunk)
    res = []
    for r in range(1, trace.n_requests + 1):
        s = trace.seq(r)
        L = int(trace.lin[r - 1])
        res.append(c.step(r, [int(x) for x in s[:L]], [int(x) for x in s[L:]]))
    return res, c


def opt_reuse(trace, model, cap_bytes, cap_nodes) -> int:
    """Exhaustive search over the victim choice at every eviction (SURVEY.md c.1 "OPT search").

    Admission, bypass and trigger rules are unchanged; the objective is Σ reuse.
    Exponential -- only for <= 8 requests and cap_nodes <= 4.
    """
    seqs = []
    for r in range(1, trace.n_requests + 1):
        s = trace.seq(r)
        L = int(trace.lin[r - 1])
        seqs.append(([int(x) for x in s[:L]], [int(x) for x in s[L:]]))

    class _Branch(Exception):
        pass

    best = [0]

    def rec(cache: FlatCache, r: int, acc: int, forced: List[int]):
        # replay request r with a victim sequence prefix `forced`; branch at the first free choice
        if r > len(seqs):
            best[0] = max(best[0], acc)
            return
        trial = cache.clone()
        k = [0]
        choice_sets = []

        def chooser(c, cands, rr):
            ids = sorted(e.id for e in cands)
            if k[0] < len(forced):
                vid = forced[k[0]]
            else:
                choice_sets.append(ids)
                raise _Branch()
            k[0] += 1
            return next(e for e in cands if e.id == vid)

        try:
            reuse, _, _ = trial.step(r, *seqs[r - 1], chooser=chooser)
        except _Branch:
            for vid in choice_sets[-1]:
                rec(cache, r, acc, forced + [vid])
            return
        rec(trial, r + 1, acc + reuse, [])

    rec(FlatCache(model, cap_bytes, cap_nodes, 0.0), 1, 0, [])
    return best[0]


# ----------------------------------------------------------------------------
# vLLM+ baseline (readings V1-V8), brute force.
# ----------------------------------------------------------------------------
class FlatBlocks:
    """Block-granular cache as an unordered list of entries (path = the full token
    prefix S[:jx] a block ends, t_last, id); relations by brute force on each query:

      parent(e)  = the entry whose path is e.path minus its last x tokens (or root)
      leaf(e)    = no entry has e as parent
      matched mb = largest k with S[:jx] cached for every j <= k
      block bytes = x tokens of KVs + one set of SSM/conv states

    Lookup hit = min(mb, L_in // x) * x (every block carries a state);
    every matched block and every inserted one gets t_last = r; LRU over leaf blocks
    off the matched path, min (t_last, id) ("vLLM's caching policy").
    Shares nothing with oracle/oracle.cpp (no trie, no maps keyed by content)."""

    def __init__(self, model, cap_bytes: int, cap_nodes: int, x: int):
        self.m, self.cap_bytes, self.cap_nodes, self.x = model, cap_bytes, cap_nodes, x
        self.E: Dict[int, Entry] = {}
        self.next_id = 1
        self.log: List[Tuple[int, int, int, float]] = []
        self.ctr = [0, 0, 0, 0]  # d.3 counters, as FlatCache.ctr at block granularity

    def bb(self) -> int:
        return KVT(self.m) * self.x + SSMB(self.m)

    def cached(self, p) -> Optional[Entry]:
        for e in self.E.values():
            if e.path == tuple(p):
                return e
        return None

    def is_leaf(self, e: Entry) -> bool:
        return not any(len(f.path) == len(e.path) + self.x and f.path[:len(e.path)] == e.path
                       for f in self.E.values())

    def step(self, r: int, inp, out):
        S = tuple(inp) + tuple(out)
        n, L_in, x = len(S), len(inp), self.x
        nb = n // x
        mb = 0
        while mb < nb and self.cached(S[:(mb + 1) * x]) is not None:
            mb += 1
        reuse = min(mb, L_in // x) * x
        path = [self.cached(S[:(j + 1) * x]) for j in range(mb)]
        for e in path:
            e.t = r
        self.ctr[0] += mb * x
        self.ctr[1] += mb + 1
        self.ctr[3] += mb
        bb = self.bb()
        n_new = nb - mb
        bypass = (mb + n_new) * bb > self.cap_bytes or bool(self.cap_nodes and nb > self.cap_nodes)
        if not bypass:
            pids = {id(e) for e in path}
            while (len(self.E) + n_new) * bb > self.cap_bytes or (self.cap_nodes and len(self.E) + n_new > self.cap_nodes):
                ts = [e.t for e in self.E.values()]
                tmin, tmax = min(ts), max(ts)
                cands = [e for e in self.E.values() if id(e) not in pids and self.is_leaf(e)]
                assert cands, "no candidate"
                v = min(cands, key=lambda e: (e.t, e.id))
                u = 0.5 if tmax == tmin else float(v.t - tmin) / float(tmax - tmin)
                self.log.append((r, v.id, 0, u))
                self.ctr[2] += len(self.E)
                self.ctr[3] += 1
                del self.E[v.id]
            for j in range(mb, nb):
                self.E[self.next_id] = Entry(S[:(j + 1) * x], True, r, self.next_id)
                self.next_id += 1
                self.ctr[3] += 1
        return reuse, F(reuse, self.m), int(bool(bypass))

    def dump(self):
        out = []
        for e in sorted(self.E.values(), key=lambda e: e.id):
            par = self.cached(e.path[:-self.x]) if len(e.path) > self.x else None
            out.append((e.id, par.id if par else 0, len(e.path) - self.x, len(e.path), 1, e.t))
        return out


def replay_blocks(trace, model, cap_bytes, cap_nodes, x):
    c = FlatBlocks(model, cap_bytes, cap_nodes, x)
    res = []
    for r in range(1, trace.n_requests + 1):
        s = trace.seq(r)
        L = int(trace.lin[r - 1])
        res.append(c.step(r, [int(t) for t in s[:L]], [int(t) for t in s[L:]]))
    return res, c
