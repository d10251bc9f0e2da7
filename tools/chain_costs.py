"""Per-variant chain cycles of one replay of config CFG (dev tool): how uneven the chains
are and how the persistent queue packs them (makespan vs the ideal)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import tracegen as tg
from paper_2411_19379_b200 import AlphaGrid

cfg = int(os.environ.get("CFG", "5"))
w = tg.workload(cfg)
g = AlphaGrid(w.trace, w.variants, w.alphas, w.n_segments).setup()
out = g.ctx.alloc_outputs(len(w.alphas), counters=True, chain_cycles=True)
for _ in range(2):
    out["hit_sum"].zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.run(out=out)
    e1.record()
    torch.cuda.synchronize()
ms = e0.elapsed_time(e1)
cyc = out["cycles"].cpu().numpy().astype(np.float64) * 1024
ctr = out["counters"].cpu().numpy().astype(np.float64)
na, ns = len(w.alphas), len(g.segs)
print(f"cfg{cfg}: {ms:.1f} ms, {len(g.chains)} chains, workers {g.ctx.workspace_size(0) and ''}")
for v, var in enumerate(w.variants):
    ids = np.arange(v * na * ns, (v + 1) * na * ns)
    c = cyc[ids]
    print(f"  variant {v} (d_state {var.model.d_state}, n_ssm {var.model.n_ssm}, {var.capacity_bytes / 1e9:.0f} GB): "
          f"chain Mcycles mean {c.mean() / 1e6:.1f} max {c.max() / 1e6:.1f}; scanned/req {ctr[ids, 2].sum() / (len(ids) * w.window):.0f}")
tot = cyc[g.chains.astype(np.int64)].sum()
print(f"sum of chain cycles / 2368 slots = {tot / 2368 / 1.965e6:.1f} ms at 1965 MHz; longest chain {cyc.max() / 1.965e6:.1f} ms")
print("queue order estimated cost vs measured rank correlation:",
      float(np.corrcoef(np.arange(len(g.chains)), cyc[g.chains.astype(np.int64)])[0, 1]))
if os.environ.get("SAVE"):
    nsnap = np.array([[g.ctx.snapshot_count(v) for v in range(len(w.variants))]])
    sizes = np.zeros((len(w.variants), ns), np.int64)
    import ctypes as C
    from paper_2411_19379_b200 import marconi as M
    for v in range(len(w.variants)):
        for si, (f, n, k) in enumerate(g.segs):
            nn = C.c_uint64(); nid = C.c_uint32()
            M.check(M.lib().mc_get_snapshot(g.ctx.h, v, k, None, 0, C.byref(nn), C.byref(nid)))
            sizes[v, si] = nn.value
    lens = w.trace.lin.astype(np.int64) + w.trace.lout
    np.savez(os.environ["SAVE"], cycles=cyc, counters=ctr, sizes=sizes, lens=lens,
             segs=np.array(g.segs), n_alpha=na, caps=np.array([v.capacity_bytes for v in w.variants]))
    print("saved", os.environ["SAVE"])
