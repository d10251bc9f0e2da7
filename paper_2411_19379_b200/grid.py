"""α-grid driver (K6): chain sharding, replay, NCCL all-gather of per-α hit sums, α*.

The paper tunes α by replaying the bootstrap requests from a tree snapshot for
every α in a grid, "parallelized across CPU cores", and adopts the α that
maximises the hit rate (§4.2 "Managing the balance").  Here the
unit of work is a chain (variant, α, segment) replayed by one warp; chains are
sharded across the GPUs of one box (one process per GPU), each GPU reduces its
chains' hits into u64[n_variant, n_alpha], one all_gather_into_tensor over
NCCL (NVLink/NVSwitch) exchanges them, and every rank takes the same argmax
(ties -> smallest α).
"""
from __future__ import annotations

from typing import List, Optional, Sequence

import numpy as np

from . import marconi as M


def chain_id(v: int, a: int, s: int, n_alpha: int, n_segs: int) -> int:
    return (v * n_alpha + a) * n_segs + s


def chain_costs(lens: np.ndarray, segs, n_var: int, n_alpha: int) -> np.ndarray:
    """Estimated cost per chain id: tokens of the window + a per-request constant."""
    cs = np.cumsum(np.r_[0, lens.astype(np.int64)])
    seg_cost = np.asarray([cs[f - 1 + n] - cs[f - 1] + 256 * n for f, n, _ in segs], np.int64)
    return np.tile(seg_cost, n_var * n_alpha)


def chain_costs_live(window_cycles: Sequence[np.ndarray], segs, n_alpha: int) -> np.ndarray:
    """Cost per chain id from the α = 0 live pass: the device cycles it spent on the
    segment's window (mc_live_window_cycles; the same requests from the same tree at α = 0),
    for every α of the segment.  Chains are independent, so only the order changes."""
    per_vs = np.asarray([[int(wc[k]) if k < len(wc) else 0 for (_, _, k) in segs] for wc in window_cycles],
                        np.int64)                                   # [variant, segment]
    return np.repeat(per_vs, n_alpha, axis=0).reshape(-1)           # chain id = (v * n_alpha + a) * ns + s


def lpt_shard(costs: np.ndarray, n_segs: int, n_alpha: int, world: int) -> List[np.ndarray]:
    """Deterministic longest-processing-time assignment of chains to ranks.

    Chains are taken by decreasing cost (ties: variant, segment, α -- so the α
    siblings of a segment stay adjacent and share trace tokens in L2) and each
    goes to the least-loaded rank (ties: lowest rank).  Every rank computes the
    same assignment.  Returns, per rank, its chain ids in execution order.
    """
    ids = np.arange(costs.shape[0], dtype=np.int64)
    s = ids % n_segs
    a = (ids // n_segs) % n_alpha
    v = ids // (n_segs * n_alpha)
    order = np.lexsort((a, s, v, -costs))
    load = np.zeros(world, np.int64)
    out = [[] for _ in range(world)]
    for c in order:
        r = int(np.argmin(load))
        out[r].append(int(c))
        load[r] += int(costs[c])
    return [np.asarray(x, np.uint32) for x in out]


def select_alpha(alphas: Sequence[float], hit_sums: np.ndarray) -> List[float]:
    """Per variant: α* = argmax Σ hits (equal denominators Σ L_in), ties -> smallest α."""
    alphas = np.asarray(alphas, np.float64)
    order = np.argsort(alphas, kind="stable")
    res = []
    for row in np.asarray(hit_sums).reshape(-1, len(alphas)):
        best = None
        for i in order:
            if best is None or row[i] > row[best]:
                best = i
        res.append(float(alphas[best]))
    return res


def gather_hit_sums(hs, world: int, group=None):
    """Sum every rank's partial u64[n_variant, n_alpha] hit sums (one all-gather).

    NCCL (NVLink/NVSwitch): all_gather_into_tensor on the device tensor.  gloo
    (CPU tests): the list form.  Summation is in rank order on every rank, exact
    in int64, so all ranks hold identical totals.
    """
    import torch
    import torch.distributed as dist
    if world == 1:
        return hs
    if dist.get_backend(group) == "nccl":
        g = torch.empty((world,) + tuple(hs.shape), dtype=hs.dtype, device=hs.device)
        dist.all_gather_into_tensor(g, hs.contiguous(), group=group)
        return g.sum(0)
    h = hs.detach().cpu().contiguous()  # gloo: host tensors
    parts = [torch.empty_like(h) for _ in range(world)]
    dist.all_gather(parts, h, group=group)
    tot = torch.zeros_like(h)
    for p in parts:
        tot += p
    return tot.to(hs.device)


class AlphaGrid:
    """One rank's share of an α-grid replay over segment windows.

    setup(): trace -> device, α = 0 live pass on the device producing the
    segment snapshots S_k (tree after request k*W), segments, this rank's chain
    shard and the workspace.  run(): replay the shard (async).  select():
    all-gather the per-α hit sums and return α* per variant.
    """

    def __init__(self, trace, variants, alphas: Sequence[float], n_segments: int, rank: int = 0, world: int = 1,
                 max_nodes: int = 8192, device: int = 0, group=None):
        self.trace = trace
        self.variants = list(variants)
        self.alphas = [float(a) for a in alphas]
        self.n_segments = n_segments
        self.rank, self.world = rank, world
        self.group = group
        self.ctx = M.Context(self.variants, max_nodes=max_nodes, device=device)
        R = trace.n_requests
        self.window = -(-R // n_segments)
        self.segs = []
        for k in range(n_segments):
            a, b = k * self.window, min((k + 1) * self.window, R)
            if b > a:
                self.segs.append((a + 1, b - a, k))

    def setup(self, snapshots=None):
        """snapshots: optional {variant: [(nodes, next_id), ...]} to upload instead of the device live pass."""
        tr = self.trace
        self.d_tokens, self.d_reqs = self.ctx.upload_trace(tr.tokens, tr.off, tr.lin, tr.lout)
        if snapshots is None:
            self.live = self.ctx.live_pass(self.window)
        else:
            for v, snaps in snapshots.items():
                self.ctx.set_snapshots(v, snaps)
            self.live = None
        self.ctx.set_segments(self.segs)
        if self.live is not None:  # longest chains first: the live pass's own window cycles
            costs = chain_costs_live([self.ctx.live_window_cycles(v) for v in range(len(self.variants))],
                                     self.segs, len(self.alphas))
        else:
            lens = tr.lin.astype(np.int64) + tr.lout
            costs = chain_costs(lens, self.segs, len(self.variants), len(self.alphas))
        self.shards = lpt_shard(costs, len(self.segs), len(self.alphas), self.world)
        self.chains = self.shards[self.rank]
        dflt = self.ctx.workspace_size(0, len(self.alphas), len(self.chains))
        one = self.ctx.workspace_size(1, len(self.alphas), len(self.chains))
        per = self.ctx.workspace_size(2, len(self.alphas), len(self.chains)) - one
        workers = min(max(1, len(self.chains)), (dflt - one) // per + 1)
        self.workspace = self.ctx.alloc_workspace(workers, len(self.alphas), len(self.chains))
        return self

    @property
    def n_chains_total(self) -> int:
        return len(self.variants) * len(self.alphas) * len(self.segs)

    def run(self, out=None, **kw):
        return self.ctx.replay(self.alphas, chains=self.chains, workspace=self.workspace, out=out, **kw)

    def metrics(self, out):
        """This rank's per-(variant, α) token hit rate (Σ skipped prefill tokens / Σ input
        tokens) and exact Σ FLOPs saved, from the device per-chain
        sums (mc_chain_sums).  Returns {(v, α): (hit_rate, flops_saved)}."""
        na, ns = len(self.alphas), len(self.segs)
        acc = {}
        for c, (sh, sl, sf) in zip(self.chains.tolist(), self.ctx.chain_sums(out, na, self.chains)):
            key = (c // (na * ns), self.alphas[(c // ns) % na])
            h, l, f = acc.get(key, (0, 0, 0))
            acc[key] = (h + sh, l + sl, f + sf)
        return {k: (h / l if l else 0.0, f) for k, (h, l, f) in acc.items()}

    def reorder_by_cycles(self, cycles) -> None:
        """Cost feedback: order this rank's chains longest-first by the per-chain cycles a
        previous replay of the same chains measured (outputs["cycles"]); the persistent
        queue then packs them LPT.  Results never depend on the order."""
        cyc = np.asarray(cycles.cpu().numpy() if hasattr(cycles, "cpu") else cycles, np.int64)
        ch = self.chains.astype(np.int64)
        self.chains = ch[np.lexsort((ch, -cyc[ch]))].astype(np.uint32)

    def select(self, out, gathered=None) -> List[float]:
        hs = gathered if gathered is not None else gather_hit_sums(out["hit_sum"], self.world, self.group)
        self.hit_sums = hs.cpu().numpy()
        return select_alpha(self.alphas, self.hit_sums)


class LiveTuner:
    """The paper's online α tuning loop on the device (§4.2 "Managing the balance",
    PAPER:426-427), one cache variant:

    1. α = 0 (LRU) from an empty cache until the first request r_F whose
       admission evicted a node; snapshot the tree after r_F;
    2. bootstrap: keep α = 0 for the next multiplier * r_F requests (10x, reading R16);
    3. grid: replay the bootstrap window from the snapshot for every α; α* = argmax of
       hit tokens (ties -> smallest α);
    4. adopt α* for the rest of the trace (replayed from the tree at the end of the
       bootstrap).
    If no eviction ever happens, or the window is empty, α stays 0.
    Every step runs in the CUDA kernels (live pass, replays); this class only sequences them.
    """

    def __init__(self, trace, variant, alphas, multiplier: int = 10, max_nodes: int = 8192, device: int = 0):
        self.trace = trace
        self.variant = variant
        self.alphas = [float(a) for a in alphas]
        self.multiplier = multiplier
        self.ctx = M.Context([variant], max_nodes=max_nodes, device=device)

    def run(self):
        import torch
        tr = self.trace
        R = tr.n_requests
        self.ctx.upload_trace(tr.tokens, tr.off, tr.lin, tr.lout)
        # one live pass: α = 0 outputs for every request plus the snapshots after r_F and
        # after the bootstrap window, taken as the pass reaches them
        h1, f1, _, fe = self.ctx.live_pass_bootstrap(self.multiplier)
        r_f = fe[0]
        hits = h1[0].cpu().numpy().copy()
        flops = f1[0].cpu().numpy().copy()
        info = {"r_first_evict": r_f, "alpha_star": 0.0, "window": None, "grid_hit_sums": None}
        if r_f == 0 or r_f >= R:
            return hits, flops, info
        b_end = min(r_f + self.multiplier * r_f, R)
        info["window"] = (r_f + 1, b_end)
        segs = [(r_f + 1, b_end - r_f, 1)]
        if b_end < R:
            segs.append((b_end + 1, R - b_end, 2))
        self.ctx.set_segments(segs)
        ns, na = len(segs), len(self.alphas)
        out = self.ctx.replay(self.alphas, chains=[a * ns for a in range(na)], log_cap=0)
        self.ctx.check()
        sums = out["hit_sum"].cpu().numpy()[0]
        a_star = select_alpha(self.alphas, sums[None, :])[0]
        info["alpha_star"] = a_star
        info["grid_hit_sums"] = [int(x) for x in sums]
        if b_end < R:
            ai = self.alphas.index(a_star)
            out2 = self.ctx.replay(self.alphas, chains=[ai * ns + 1], log_cap=0)
            self.ctx.check()
            hits[b_end:] = out2["hit"].cpu().numpy()[0, ai, b_end:]
            flops[b_end:] = out2["flops"].cpu().numpy()[0, ai, b_end:]
        return hits, flops, info


class HostPipeline:
    """End-to-end α-grid replay from HOST buffers, double-buffered (the path a serving
    system's tuner takes when each tuning job arrives in host memory).

    Per job: H2D of the trace (tokens + request table) and of the packed segment
    snapshots, the device-side trace check (mc_set_trace_async), the snapshot images,
    the replay of `grid`'s chain shard, D2H of the per-request hits and the per-α hit
    sums, α* on the host.  Two slots (each its own context, device buffers, workspace
    and outputs) alternate: job k+1's copies and image build run on a copy stream while
    job k replays on the compute stream, so the transfers hide under the replay.  Every
    step of the path runs in libmarconi's kernels; this class only sequences streams.

    grid: a set-up AlphaGrid (its segments, chain shard and variants are reused).
    """

    def __init__(self, grid: "AlphaGrid", n_slots: int = 2):
        import torch
        self.torch = torch
        self.g = grid
        self.copy_stream = torch.cuda.Stream()
        self.compute_stream = torch.cuda.Stream()
        self.slots = []
        for _ in range(n_slots):
            ctx = M.Context(grid.variants, max_nodes=grid.ctx.max_nodes, device=grid.ctx.device.index or 0)
            self.slots.append({"ctx": ctx, "ws": ctx.alloc_workspace(0, len(grid.alphas), len(grid.chains)),
                               "d_tok": None, "d_req": None, "out": None, "h_hit": None, "h_hs": None,
                               "done": None})
        self.k = 0

    def submit(self, h_tok, h_req, snapshots):
        """Queue one job.  h_tok: pinned int32 tensor of tokens; h_req: pinned int64 tensor
        holding REQUEST_DTYPE records; snapshots: per variant (nodes SNAP_DTYPE in pinned
        memory, offsets u64, next ids u32) as from Context.pack_snapshots.  Returns a ticket."""
        torch = self.torch
        s = self.slots[self.k % len(self.slots)]
        ctx = s["ctx"]
        n_req = h_req.numel() * 8 // M.REQUEST_DTYPE.itemsize
        if s["d_tok"] is None or s["d_tok"].numel() != h_tok.numel() or s["d_req"].numel() != h_req.numel():
            s["d_tok"] = torch.empty(h_tok.shape, dtype=h_tok.dtype, device=ctx.device)
            s["d_req"] = torch.empty(h_req.shape, dtype=h_req.dtype, device=ctx.device)
        cs, ks = self.copy_stream, self.compute_stream
        if s["done"] is not None:
            cs.wait_event(s["done"])  # the slot's previous job has left its buffers
        with torch.cuda.stream(cs):
            s["d_tok"].copy_(h_tok, non_blocking=True)
            s["d_req"].copy_(h_req, non_blocking=True)
            ctx.set_trace_async(s["d_tok"], s["d_req"], n_req, stream=cs)
            if ctx.segments is None:
                ctx.set_segments(self.g.segs)  # (validated against the request count: once, after the trace)
            for v, (nodes, off, nid) in enumerate(snapshots):
                ctx.set_snapshots_packed(v, nodes, off, nid, stream=cs)
            ready = torch.cuda.Event()
            ready.record(cs)
        if s["out"] is None or s["out"]["hit"].shape[-1] != n_req:
            s["out"] = ctx.alloc_outputs(len(self.g.alphas))
            s["h_hit"] = torch.empty(s["out"]["hit"].shape, dtype=torch.int32).pin_memory()
            s["h_hs"] = torch.empty(s["out"]["hit_sum"].shape, dtype=torch.int64).pin_memory()
        ks.wait_event(ready)
        with torch.cuda.stream(ks):
            s["out"]["hit_sum"].zero_()
            ctx.replay(self.g.alphas, chains=self.g.chains, workspace=s["ws"], out=s["out"], stream=ks)
            s["h_hit"].copy_(s["out"]["hit"], non_blocking=True)
            s["h_hs"].copy_(s["out"]["hit_sum"], non_blocking=True)
            done = torch.cuda.Event()
            done.record(ks)
        s["done"] = done
        t = self.k
        self.k += 1
        return t

    def result(self, ticket):
        """Wait for job `ticket` (the most recent len(slots) jobs stay retrievable);
        returns (hits int32[n_var, n_alpha, R] host tensor, hit sums, α* per variant)."""
        s = self.slots[ticket % len(self.slots)]
        s["done"].synchronize()
        s["ctx"].check(stream=self._idle())  # device status of this slot's context
        hs = s["h_hs"].numpy()
        return s["h_hit"], hs, select_alpha(self.g.alphas, hs)

    def _idle(self):
        if not hasattr(self, "_idle_stream"):
            self._idle_stream = self.torch.cuda.Stream()
        return self._idle_stream
