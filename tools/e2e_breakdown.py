"""Wall-clock breakdown of one e2e step (bench.py e2e_measure) by phase (dev tool)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import tracegen as tg
from paper_2411_19379_b200 import AlphaGrid
from paper_2411_19379_b200 import marconi as M

w = tg.workload(3)
g = AlphaGrid(w.trace, w.variants, w.alphas, w.n_segments).setup()
ctx, tr = g.ctx, w.trace
o = ctx.alloc_outputs(len(w.alphas))
h_tok = torch.from_numpy(np.ascontiguousarray(tr.tokens, np.uint32).view(np.int32)).pin_memory()
h_req = torch.from_numpy(M.requests_array(tr.off, tr.lin, tr.lout).view(np.int64)).pin_memory()
nodes, off, nid = ctx.pack_snapshots([ctx.get_snapshot(0, k) for k in range(ctx.snapshot_count(0))])
pin = torch.empty(nodes.nbytes, dtype=torch.uint8).pin_memory()
pn = pin.numpy().view(M.SNAP_DTYPE)
pn[:] = nodes
d_tok = torch.empty_like(h_tok, device="cuda")
d_req = torch.empty_like(h_req, device="cuda")
h_hit = torch.empty(o["hit"].shape, dtype=torch.int32).pin_memory()
ph = {k: [] for k in ("h2d", "set_trace", "set_snapshots", "replay", "d2h+select")}
for it in range(8):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    d_tok.copy_(h_tok, non_blocking=True); d_req.copy_(h_req, non_blocking=True); torch.cuda.synchronize()
    t1 = time.perf_counter()
    ctx.set_trace_device(d_tok, d_req, tr.n_requests); torch.cuda.synchronize()
    t2 = time.perf_counter()
    ctx.set_snapshots_packed(0, pn, off, nid); torch.cuda.synchronize()
    t3 = time.perf_counter()
    o["hit_sum"].zero_(); g.run(out=o); torch.cuda.synchronize()
    t4 = time.perf_counter()
    h_hit.copy_(o["hit"], non_blocking=True); g.select(o); torch.cuda.synchronize()
    t5 = time.perf_counter()
    if it >= 2:
        for k, a, b in zip(ph, (t0, t1, t2, t3, t4), (t1, t2, t3, t4, t5)):
            ph[k].append(1000 * (b - a))
print({k: round(float(np.median(v)), 3) for k, v in ph.items()}, "ms;", "bytes h2d", h_tok.numel() * 4 + h_req.numel() * 8 + pn.nbytes)
