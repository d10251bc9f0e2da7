"""Per-chain cycles of the same chains replayed with fewer chains in flight (dev tool).

Replays config CFG's full chain list, then subsets of it (every k-th chain), and reports
the per-request cycles of the subset's chains in both runs.  With 148 chains (one warp
per SM) the per-chain L2 footprint of all chains in flight fits in L2 and no warp shares
its SM, so the ratio bounds what a smaller working set could gain.
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import tracegen as tg
from paper_2411_19379_b200 import AlphaGrid

cfg = int(os.environ.get("CFG", "3"))
w = tg.workload(cfg)
g = AlphaGrid(w.trace, w.variants, w.alphas, w.n_segments).setup()
full = g.chains.copy()


def run(chains, reps=3):
    out = g.ctx.alloc_outputs(len(w.alphas), chain_cycles=True)
    ws = g.ctx.alloc_workspace(0, len(w.alphas), len(chains))
    ts = []
    for _ in range(reps):
        out["hit_sum"].zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        g.ctx.replay(g.alphas, chains=chains, workspace=ws, out=out)
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    g.ctx.check()
    return np.median(ts), out["cycles"].cpu().numpy().astype(np.float64) * 1024


ms_full, cyc_full = run(full)
win = np.array([n for _, n, _ in g.segs], np.float64)
nseg = len(g.segs)
print(f"cfg{cfg} all {len(full)} chains: {ms_full:.2f} ms, chain cycles median {np.median(cyc_full[full]) / 1e6:.2f}M "
      f"max {cyc_full[full].max() / 1e6:.2f}M")
for k in (int(x) for x in os.environ.get("STRIDES", "14,4,2").split(",")):
    sub = full[::k]
    ms, cyc = run(sub)
    idx = sub.astype(np.int64)
    per_req_full = cyc_full[idx] / win[idx % nseg]
    per_req_sub = cyc[idx] / win[idx % nseg]
    print(f"  {len(sub):5d} chains ({len(sub) / 148:.1f}/SM): {ms:.2f} ms; same chains per request: "
          f"{np.median(per_req_sub) / 1e3:.1f}k cycles vs {np.median(per_req_full) / 1e3:.1f}k in the full run "
          f"(ratio {np.median(per_req_sub / per_req_full):.3f}); max chain {cyc[idx].max() / 1e6:.2f}M vs "
          f"{cyc_full[idx].max() / 1e6:.2f}M", flush=True)
