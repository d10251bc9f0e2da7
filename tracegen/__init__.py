"""Seeded synthetic request traces for the Marconi α-grid replay (input generator only).

This module is shared INPUT for both the CUDA path and the CPU oracle.  It holds
none of the method's arithmetic (no FLOP model, no lookup, no eviction): it only
draws token ids and request lengths.  Every random number comes from a
counter-based SplitMix64 keyed by (seed, stream, a, b), so traces are
bit-reproducible and independent of call order.

Trace shape:
  tokens  u32[T]   one contiguous stream per session: prompt ++ u1 o1 u2 o2 ...
  off     u64[R]   request r's sequence is tokens[off[r] : off[r] + lin[r] + lout[r]]
  lin     u32[R]   input length (history + new user turn)
  lout    u32[R]   output length
Requests are numbered 1..R in arrival order; array index = r - 1.

Workload shapes follow PAPER.md §5 "Workloads" (LMSys outputs
"often reaching thousands", ShareGPT "succinct", SWEBench "hundreds to tens of
thousands") and the arrival axes of fig:micro_arrival.  The
exact distributions are this build's proposal; the
recipe is restated in DESIGN.md.
"""
from __future__ import annotations

import dataclasses
import functools
import math
from typing import List, Optional, Sequence

import numpy as np

__all__ = [
    "Model", "Trace", "Variant", "Workload",
    "MODEL_7B", "MODEL_TOY", "model_ratio", "ALPHA_GRID16",
    "splitmix64", "gen_trace", "toy_trace", "micro_trace", "session_params",
    "workload", "from_sequences",
]

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)
_GOLD = np.uint64(0x9E3779B97F4A7C15)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """SplitMix64 finaliser applied elementwise to a u64 array (wrapping arithmetic)."""
    x = np.asarray(x, dtype=np.uint64)
    with np.errstate(over="ignore"):
        z = x + _GOLD
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


@functools.lru_cache(maxsize=4096)
def _key(seed: int, stream: int) -> np.uint64:
    return splitmix64(np.array([(seed & 0xFFFFFFFF) << 16 | (stream & 0xFFFF)], dtype=np.uint64))[0]


def _draw(seed: int, stream: int, a, b=0) -> np.ndarray:
    """u64 random words for counters (a, b) under (seed, stream); a/b broadcast."""
    k = _key(seed, stream)
    a = np.atleast_1d(np.asarray(a, dtype=np.uint64))
    b = np.atleast_1d(np.asarray(b, dtype=np.uint64))
    with np.errstate(over="ignore"):
        return splitmix64(splitmix64(k ^ (a * np.uint64(0xD1B54A32D192ED03))) ^ b)


def _u01(seed, stream, a, b=0) -> np.ndarray:
    """Uniform doubles in (0, 1)."""
    w = _draw(seed, stream, a, b) >> np.uint64(11)
    return (w.astype(np.float64) + 0.5) * (1.0 / 9007199254740992.0)


def _lognormal(seed, stream, a, b, mu, sigma, lo, hi) -> np.ndarray:
    u1 = _u01(seed, stream, a, 2 * np.asarray(b, dtype=np.uint64))
    u2 = _u01(seed, stream, a, 2 * np.asarray(b, dtype=np.uint64) + np.uint64(1))
    z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * math.pi * u2)
    v = np.floor(np.exp(mu + sigma * z))
    return np.clip(v, lo, hi).astype(np.int64)


# ----------------------------------------------------------------------------
# Model / variant / workload descriptors (plain data; the oracle and the CUDA
# path each implement the cost model themselves).
# ----------------------------------------------------------------------------
@dataclasses.dataclass(frozen=True)
class Model:
    """ModelConfig.  Layer counts {Attn, SSM, MLP}, D, N, fp16, conv_1d.

    Defaults are the paper's 7B hybrid {4,24,28}, D=4096, N=128 (PAPER:543,
    PAPER:779) with conv_1d in_channels = 2D+2N, kernel 4.
    """
    n_attn: int = 4
    n_ssm: int = 24
    n_mlp: int = 28
    d_model: int = 4096
    d_state: int = 128
    bytes_per_param: int = 2
    conv_in: int = 2 * 4096 + 2 * 128
    conv_kernel: int = 4

    def astuple(self):
        return (self.n_attn, self.n_ssm, self.n_mlp, self.d_model, self.d_state,
                self.bytes_per_param, self.conv_in, self.conv_kernel)


MODEL_7B = Model()
# Toy: "1 Attn : 7 SSM" (BASELINE.json configs[0]) -> {4, 28, 32}.
MODEL_TOY = Model(4, 28, 32)


def model_ratio(rho: int) -> Model:
    """Attention:SSM ratio 1:rho with nA=4, nS=4*rho, nM=nA+nS."""
    return Model(4, 4 * rho, 4 + 4 * rho)


# 16 dyadic α values, exact in binary.
ALPHA_GRID16 = (0.0, 1 / 64, 1 / 32, 1 / 16, 1 / 8, 1 / 4, 1 / 2, 3 / 4,
                1.0, 1.5, 2.0, 3.0, 4.0, 8.0, 16.0, 64.0)


@dataclasses.dataclass(frozen=True)
class Variant:
    """One cache configuration: model + capacity (bytes, 1e9 = GB) + node cap (0 = none).

    capacity_bytes = 2**64-1 means unlimited bytes; capacity_bytes = 0 is the
    no-cache baseline (every request bypasses admission)."""
    model: Model
    capacity_bytes: int
    capacity_nodes: int = 0
    chunk_size: int = 0  # 0 = exact checkpoints; else chunk-aligned prefill checkpoints (NEXT-3)
    block_size: int = 0  # 0 = Marconi; x > 0 = the vLLM+ baseline with token blocks of x (NEXT-2)


@dataclasses.dataclass
class Trace:
    tokens: np.ndarray   # u32[T]
    off: np.ndarray      # u64[R]
    lin: np.ndarray      # u32[R]
    lout: np.ndarray     # u32[R]
    name: str = ""
    seed: int = 0

    @property
    def n_requests(self) -> int:
        return int(self.off.shape[0])

    @property
    def n_tokens(self) -> int:
        return int(self.tokens.shape[0])

    def seq(self, r: int) -> np.ndarray:
        """Full sequence of request r (1-based)."""
        i = r - 1
        o = int(self.off[i])
        return self.tokens[o:o + int(self.lin[i]) + int(self.lout[i])]

    def copy_layout(self) -> "Trace":
        """The same requests with every full sequence copied into its own pool range (as
        an engine that stores each request's tokens separately would hold them): no two
        requests share pool offsets, so every lookup compares tokens (
        the shared-stream layout lets same-session continuations skip their compares)."""
        n = self.lin.astype(np.int64) + self.lout
        off = np.zeros(self.n_requests, np.uint64)
        off[1:] = np.cumsum(n)[:-1]
        idx = np.concatenate([np.arange(int(o), int(o) + int(k), dtype=np.int64) for o, k in zip(self.off, n)]) \
            if self.n_requests else np.zeros(0, np.int64)
        return Trace(np.ascontiguousarray(self.tokens[idx]), off, self.lin.copy(), self.lout.copy(),
                     self.name + "-copy", self.seed)

    def head(self, n: int) -> "Trace":
        """First n requests (the token pool is shared, unchanged)."""
        return Trace(self.tokens, self.off[:n].copy(), self.lin[:n].copy(),
                     self.lout[:n].copy(), self.name, self.seed)


@dataclasses.dataclass
class Workload:
    """A benchmark configuration: trace + cache variants + α grid + segments."""
    name: str
    trace: Trace
    variants: List[Variant]
    alphas: Sequence[float]
    n_segments: int

    @property
    def window(self) -> int:
        R = self.trace.n_requests
        return -(-R // self.n_segments)

    def segments(self):
        """Windows (kW, min((k+1)W, R)] as (first_req, n_req), first_req 1-based."""
        R, W = self.trace.n_requests, self.window
        out = []
        for k in range(self.n_segments):
            a = k * W
            b = min((k + 1) * W, R)
            if b > a:
                out.append((a + 1, b - a))
        return out

    @property
    def n_chains(self) -> int:
        return len(self.variants) * len(self.alphas) * len(self.segments())


def from_sequences(reqs, name="manual") -> Trace:
    """Build a trace from explicit (input_tokens, output_tokens) pairs.

    Each request gets its own copy of its full sequence in the pool (sharing is
    by token equality, not by offset), which is the layout the oracle and the
    GPU must both handle.  Used for hand-written scenarios and micro traces.
    """
    toks, off, lin, lout = [], [], [], []
    pos = 0
    for inp, out in reqs:
        s = list(inp) + list(out)
        toks.extend(s)
        off.append(pos)
        lin.append(len(inp))
        lout.append(len(out))
        pos += len(s)
    return Trace(np.asarray(toks, dtype=np.uint32), np.asarray(off, dtype=np.uint64),
                 np.asarray(lin, dtype=np.uint32), np.asarray(lout, dtype=np.uint32), name)


# ----------------------------------------------------------------------------
# Session-structured multi-turn generator
# ----------------------------------------------------------------------------
_KINDS = {
    # kind: (p_sys, prompt_pool, prompt_lo, prompt_hi, p_geom, max_rounds,
    #        u_mu, u_sigma, u_lo, u_hi, o_mu, o_sigma, o_lo, o_hi, cap)
    "lmsys": (0.3, 16, 64, 512, 0.35, 12, math.log(80), 1.0, 4, 2048,
              math.log(300), 0.9, 8, 4096, 16384),
    "sharegpt": (0.2, 32, 32, 256, 0.3, 16, math.log(40), 1.0, 2, 1024,
                 math.log(120), 0.8, 4, 1024, 4096),
}
# SWEBench-shaped agent sessions: 2 agent prompts (1536 / 2304 tokens), issue
# LN(ln 800, 0.7) in [100, 4000]; actions LN(ln 90, 0.6) in [10, 600];
# observations LN(ln 500, 1.2) in [10, 8000]; context cap 32,768; <= 60 steps.
_SWE = dict(prompts=(1536, 2304), issue=(math.log(800), 0.7, 100, 4000),
            act=(math.log(90), 0.6, 10, 600), obs=(math.log(500), 1.2, 10, 8000),
            cap=32768, steps=60)

# stream ids (keep stable: they define the traces)
_S_START, _S_KIND, _S_SYS, _S_PID, _S_ROUNDS, _S_U, _S_O, _S_DELAY, _S_TOK, _S_PTOK, _S_PLEN = range(11)


@functools.lru_cache(maxsize=16)
def _zipf_cdf(n: int) -> np.ndarray:
    w = 1.0 / np.arange(1, n + 1)
    return np.cumsum(w) / w.sum()


def _rounds(us, os_, plen, cap, stop_at_cap):
    rounds = []
    ctx = plen
    for u, o in zip(us, os_):
        if ctx + u + o > cap:
            u = cap - ctx - o
            if u >= 1:
                rounds.append((u, o))
            break
        rounds.append((u, o))
        ctx += u + o
        if stop_at_cap and ctx >= cap:
            break
    return rounds


def session_batch(kind: str, seed: int, sids: np.ndarray):
    """Lengths of sessions `sids`: list of (prompt_id, prompt_len, [(u_i, o_i)])."""
    sids = np.asarray(sids, dtype=np.uint64)
    S = sids.shape[0]
    out = []
    if kind == "swebench":
        pid = (_draw(seed, _S_PID, sids) & np.uint64(1)).astype(np.int64)
        steps = _SWE["steps"]
        i = np.arange(steps, dtype=np.uint64)[None, :]
        mu, sg, lo, hi = _SWE["obs"]
        obs = _lognormal(seed, _S_U, sids[:, None], i, mu, sg, lo, hi)
        mu, sg, lo, hi = _SWE["issue"]
        obs[:, 0] = _lognormal(seed, _S_U, sids, np.uint64(1000), mu, sg, lo, hi)
        mu, sg, lo, hi = _SWE["act"]
        act = _lognormal(seed, _S_O, sids[:, None], i, mu, sg, lo, hi)
        obs_l, act_l = obs.tolist(), act.tolist()
        for j in range(S):
            plen = _SWE["prompts"][int(pid[j])]
            out.append((int(pid[j]) + 1000, plen,
                        _rounds(obs_l[j], act_l[j], plen, _SWE["cap"], True)))
        return out
    (p_sys, pool, plo, phi, pg, maxr, umu, usg, ulo, uhi, omu, osg, olo, ohi, cap) = _KINDS[kind]
    base = 0 if kind == "lmsys" else 100
    has_sys = _u01(seed, _S_SYS, sids) < p_sys
    # Zipf(1.0) over the prompt pool
    pid = np.minimum(np.searchsorted(_zipf_cdf(pool), _u01(seed, _S_PID, sids)), pool - 1)
    plen_tab = plo + (_draw(seed, _S_PLEN, np.arange(pool, dtype=np.uint64) + np.uint64(base))
                      % np.uint64(phi - plo + 1)).astype(np.int64)
    g = _u01(seed, _S_ROUNDS, sids)
    nr = np.minimum(1 + np.floor(np.log(g) / math.log(1.0 - pg)).astype(np.int64), maxr)
    i = np.arange(maxr, dtype=np.uint64)[None, :]
    us = _lognormal(seed, _S_U, sids[:, None], i, umu, usg, ulo, uhi).tolist()
    os_ = _lognormal(seed, _S_O, sids[:, None], i, omu, osg, olo, ohi).tolist()
    for j in range(S):
        if has_sys[j]:
            p_, pl = int(pid[j]) + base, int(plen_tab[int(pid[j])])
        else:
            p_, pl = -1, 0
        n = int(nr[j])
        rounds = _rounds(us[j][:n], os_[j][:n], pl, cap, False)
        if not rounds:  # always at least one request per session
            u = max(1, min(int(us[j][0]), cap - pl - 1))
            o = max(0, min(int(os_[j][0]), cap - pl - u))
            rounds.append((u, o))
        out.append((p_, pl, rounds))
    return out


def session_params(kind: str, seed: int, s: int):
    """Lengths of one session: (prompt_id, prompt_len, [(u_i, o_i)])."""
    return session_batch(kind, seed, np.array([s], dtype=np.uint64))[0]


def gen_trace(name: str, R: int, seed: int, rate: float, mix, mean_delay: float = 5.0,
              alphabet: int = 0) -> Trace:
    """Generate R requests from Poisson session arrivals (rate λ_s per second).

    mix: list of (kind, weight).  Requests of a session arrive Exp(mean_delay)
    apart.  The merged stream is ordered by (arrival, session, round) and the
    first R requests are kept.  alphabet > 0 draws token ids mod alphabet.
    """
    kinds = [k for k, _ in mix]
    wts = np.asarray([w for _, w in mix], dtype=np.float64)
    cdf = np.cumsum(wts) / wts.sum()
    S = max(16, int(R / 2))
    while True:
        idx = np.arange(S, dtype=np.uint64)
        gaps = -np.log(_u01(seed, _S_START, idx)) / rate
        starts = np.cumsum(gaps)
        ku = _u01(seed, _S_KIND, idx)
        kid = np.minimum(np.searchsorted(cdf, ku), len(kinds) - 1)
        sess = [None] * S
        for k_i, kind in enumerate(kinds):
            sel = np.nonzero(kid == k_i)[0]
            for s_, v in zip(sel.tolist(), session_batch(kind, seed, sel)):
                sess[s_] = v
        nrs = np.asarray([len(v[2]) for v in sess], dtype=np.int64)
        sid = np.repeat(np.arange(S, dtype=np.int64), nrs)
        first = np.cumsum(nrs) - nrs
        rid = np.arange(sid.shape[0], dtype=np.int64) - first[sid]
        d = -np.log(_u01(seed, _S_DELAY, sid.astype(np.uint64), rid.astype(np.uint64))) * mean_delay
        d[rid == 0] = 0.0
        cs = np.cumsum(d)
        arr = starts[sid] + (cs - (cs - d)[first][sid])
        order = np.lexsort((rid, sid, arr))
        if order.shape[0] >= R and arr[order[R - 1]] <= starts[-1]:
            break
        S *= 2
    keep = order[:R]
    sid_k, rid_k = sid[keep], rid[keep]
    # per session: number of kept rounds (kept rounds are a prefix of the session's rounds)
    last_round = {}
    for s_, r_ in zip(sid_k.tolist(), rid_k.tolist()):
        if r_ > last_round.get(s_, -1):
            last_round[s_] = r_
    # build token pool: one stream per session with >= 1 kept request, in session order
    sess_off = {}
    chunks = []
    pos = 0
    for s_ in sorted(last_round):
        pid, plen, rounds = sess[s_]
        ctx = plen + sum(u + o for u, o in rounds[:last_round[s_] + 1])
        sess_off[s_] = pos
        if plen > 0:
            j = np.arange(plen, dtype=np.uint64)
            pt = _draw(seed, _S_PTOK, pid, j)
            chunks.append(pt)
        j = np.arange(plen, ctx, dtype=np.uint64)
        chunks.append(_draw(seed, _S_TOK, s_, j))
        pos += ctx
    words = np.concatenate(chunks) if chunks else np.zeros(0, dtype=np.uint64)
    if alphabet > 0:
        tokens = (words % np.uint64(alphabet)).astype(np.uint32)
    else:
        tokens = (words & np.uint64(0x7FFFFFFF)).astype(np.uint32)
    off = np.empty(R, dtype=np.uint64)
    lin = np.empty(R, dtype=np.uint32)
    lout = np.empty(R, dtype=np.uint32)
    for i, (s_, r_) in enumerate(zip(sid_k.tolist(), rid_k.tolist())):
        pid, plen, rounds = sess[s_]
        hist = plen + sum(u + o for u, o in rounds[:r_])
        u, o = rounds[r_]
        off[i] = sess_off[s_]
        lin[i] = hist + u
        lout[i] = o
    return Trace(tokens, off, lin, lout, name, seed)


def toy_trace(seed: int = 1001, R: int = 16) -> Trace:
    """Config 1 family: ~6 sessions, 1-4 rounds, alphabet 4, 2 prompts x 12 tokens,
    u, o ~ U[2, 12].  Sequences stay <= 128 tokens."""
    sess = []
    s = 0
    arr_all = []
    while sum(len(x[2]) for x in sess) < R + 8:
        has = _u01(seed, _S_SYS, s)[0] < 0.5
        pid = int(_draw(seed, _S_PID, s)[0] & np.uint64(1)) if has else -1
        plen = 12 if has else 0
        nr = 1 + int(_draw(seed, _S_ROUNDS, s)[0] % np.uint64(4))
        i = np.arange(nr, dtype=np.uint64)
        us = 2 + (_draw(seed, _S_U, s, i) % np.uint64(11)).astype(np.int64)
        os_ = 2 + (_draw(seed, _S_O, s, i) % np.uint64(11)).astype(np.int64)
        rounds = [(int(a), int(b)) for a, b in zip(us, os_)]
        sess.append((pid, plen, rounds))
        start = s * 3.0 + float(_u01(seed, _S_START, s)[0]) * 3.0
        d = np.cumsum(np.r_[0.0, 2.0 + 6.0 * _u01(seed, _S_DELAY, s, np.arange(nr - 1, dtype=np.uint64))])
        for k in range(nr):
            arr_all.append((start + d[k], s, k))
        s += 1
    arr_all.sort()
    keep = arr_all[:R]
    reqs = []
    for _, s_, k in keep:
        pid, plen, rounds = sess[s_]
        ctx = plen + sum(u + o for u, o in rounds[:k + 1])
        j = np.arange(ctx, dtype=np.uint64)
        words = _draw(seed, _S_TOK, s_, j)
        if plen:
            words[:plen] = _draw(seed, _S_PTOK, pid, np.arange(plen, dtype=np.uint64))
        toks = (words % np.uint64(4)).astype(np.uint32)
        hist = plen + sum(u + o for u, o in rounds[:k])
        u, o = rounds[k]
        reqs.append((toks[:hist + u], toks[hist + u:hist + u + o]))
    tr = from_sequences(reqs, name=f"toy{seed}")
    tr.seed = seed
    return tr


def micro_trace(seed: int, n_req: int = 20, max_len: int = 64, alphabet: int = 3) -> Trace:
    """Random micro trace (<= 20 requests, <= 64 tokens, small alphabet).

    Mixes fresh random sequences with continuations/variations of earlier ones so
    that splits, gains, stateless output-region splits and merges all occur.
    """
    reqs = []
    c = 0

    def rnd(n):
        nonlocal c
        w = _draw(seed, _S_TOK, c, np.arange(n, dtype=np.uint64))
        c += 1
        return [int(x) for x in (w % np.uint64(alphabet))]

    def ri(lo, hi):
        nonlocal c
        v = lo + int(_draw(seed, _S_U, c)[0] % np.uint64(hi - lo + 1))
        c += 1
        return v

    for i in range(n_req):
        mode = ri(0, 3) if reqs else 0
        if mode == 0:
            L = ri(1, max_len)
            s = rnd(L)
        elif mode == 1:  # continue a previous full sequence (input+output reuse)
            j = ri(0, len(reqs) - 1)
            base = reqs[j][0] + reqs[j][1]
            s = base + rnd(ri(1, max(1, max_len - len(base))))
            s = s[:max_len]
        elif mode == 2:  # share a prefix of a previous input (purely-input reuse)
            j = ri(0, len(reqs) - 1)
            base = reqs[j][0]
            k = ri(1, len(base))
            s = base[:k] + rnd(ri(1, max(1, max_len - k)))
            s = s[:max_len]
        else:  # exact repeat of a previous input with new output
            j = ri(0, len(reqs) - 1)
            s = list(reqs[j][0]) + rnd(ri(0, max(0, min(8, max_len - len(reqs[j][0])))))
        lin = ri(1, len(s))
        reqs.append((s[:lin], s[lin:]))
    tr = from_sequences(reqs, name=f"micro{seed}")
    tr.seed = seed
    return tr


# ----------------------------------------------------------------------------
# The five BASELINE.json configs.  GB = 1e9 B (c.3 #13).
# ----------------------------------------------------------------------------
GB = 1_000_000_000
UNLIMITED_BYTES = (1 << 64) - 1   # "bytes unlimited" (toy config: node-count capacity only)


def workload(cfg: int, R: Optional[int] = None, problem: int = 0, layout: str = "stream") -> Workload:
    """Build config `cfg` (1..5).  R overrides the request count (for small parity runs).
    problem > 0 draws an independent trace of the same shape (seed offset), used by the
    weak-scaling bench (one α-tuning problem per GPU).  layout = "copy": every request
    holds its own copy of its sequence (Trace.copy_layout)."""
    w = _workload(cfg, R, problem)
    if layout == "copy":
        w.trace = w.trace.copy_layout()
        w.name += "-copy"
    elif layout != "stream":
        raise ValueError(f"unknown layout {layout}")
    return w


def _workload(cfg: int, R: Optional[int], problem: int) -> Workload:
    seed = 1000 + cfg + 7919 * problem
    if cfg == 1:
        tr = toy_trace(seed, R or 16)
        return Workload("toy", tr, [Variant(MODEL_TOY, UNLIMITED_BYTES, 6)], (0.0, 1.0), 1)
    if cfg == 2:
        tr = gen_trace("lmsys", R or 10_000, seed, 1.0, [("lmsys", 1.0)])
        return Workload("lmsys", tr, [Variant(MODEL_7B, 60 * GB)], (1.0,), 1)
    if cfg == 3:
        tr = gen_trace("sharegpt", R or 50_000, seed, 1.0, [("sharegpt", 1.0)])
        return Workload("sharegpt", tr, [Variant(MODEL_7B, 60 * GB)], ALPHA_GRID16, 128)
    if cfg == 4:
        tr = gen_trace("swebench", R or 20_000, seed, 0.5, [("swebench", 1.0)])
        return Workload("swebench", tr, [Variant(MODEL_7B, 60 * GB)], ALPHA_GRID16, 128)
    if cfg == 5:
        tr = gen_trace("synthetic", R or 200_000, seed, 2.0,
                       [("sharegpt", 0.5), ("lmsys", 0.35), ("swebench", 0.15)])
        vs = [Variant(model_ratio(rho), c * GB) for rho in (2, 4, 8)
              for c in (60, 80, 100, 120, 140)]
        return Workload("synthetic", tr, vs, ALPHA_GRID16, 16)
    raise ValueError(f"unknown config {cfg}")


# ----------------------------------------------------------------------------
# NEXT-4 sweeps (same kernels, second workloads): SSM state dimension N
# (fig:microbenchmark_state_dim) and session / request arrival rates
# (fig:micro_arrival).
# ----------------------------------------------------------------------------
def state_dim_variants(capacity_bytes: int = 60 * GB, dims=(16, 32, 64, 128)) -> List[Variant]:
    """7B hybrid {4,24,28} with d_state N in dims (conv_in = 2D + 2N follows N)."""
    return [Variant(Model(4, 24, 28, 4096, n, 2, 2 * 4096 + 2 * n, 4), capacity_bytes) for n in dims]


def arrival_workload(session_rate: float, mean_delay: float, R: int = 20_000, n_segments: int = 32,
                     alphas=ALPHA_GRID16) -> Workload:
    """ShareGPT-shaped trace with the given session arrival rate (sessions/s) and mean
    inter-request delay within a session (s) -- the two axes of fig:micro_arrival."""
    seed = 2000 + int(session_rate * 100) + int(mean_delay * 10)
    tr = gen_trace(f"sharegpt_rate{session_rate}_delay{mean_delay}", R, seed, session_rate,
                   [("sharegpt", 1.0)], mean_delay=mean_delay)
    return Workload(tr.name, tr, [Variant(MODEL_7B, 60 * GB)], tuple(alphas), n_segments)
