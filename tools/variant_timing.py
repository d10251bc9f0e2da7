"""Time the replay kernel of alternative builds (MARCONI_LIB=<.so>) on one config; dev tool."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import tracegen as tg
from paper_2411_19379_b200 import AlphaGrid

cfg = int(os.environ.get("CFG", "3"))
w = tg.workload(cfg)
g = AlphaGrid(w.trace, w.variants, w.alphas, w.n_segments, max_nodes=int(os.environ.get('MAXN', '8192'))).setup()
out = g.ctx.alloc_outputs(len(w.alphas), counters=True, chain_cycles=True)
ts = []
for it in range(6):
    out["hit_sum"].zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.run(out=out)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
g.ctx.check()
cyc = out["cycles"].cpu().numpy().astype(np.float64) * 1024
ctr = out["counters"].cpu().numpy()
print(f"{os.path.basename(os.environ.get('MARCONI_LIB', 'default'))} cfg{cfg}: replay ms {np.median(ts[1:]):.2f} "
      f"(min {min(ts[1:]):.2f}) chains {len(g.chains)} chain-cycles median {np.median(cyc)/1e6:.2f}M max {cyc.max()/1e6:.2f}M "
      f"hitsum {int(out['hit_sum'].sum())}", flush=True)
if os.environ.get("PHASES"):
    tot = ctr.astype(np.float64).sum(0)
    print("phase cycles share walk/evict/insert/unpin:", np.round(tot / tot.sum(), 3), "per request (M):",
          np.round(tot / (len(g.chains) * w.window) / 1e3, 1), "k-cycles")
if os.environ.get("PHASES3"):
    tot = ctr.astype(np.float64).sum(0)
    nreq = len(g.chains) * w.window
    print("per request k-cycles: pass1 %.1f pass2 %.1f verify %.1f ; fallbacks per request %.4f" %
          (tot[0] / nreq / 1e3, tot[1] / nreq / 1e3, tot[2] / nreq / 1e3, tot[3] / nreq))
if os.environ.get("PHASES3"):
    tot_pass1 = (ctr[:, 2].astype(np.uint64) >> np.uint64(32)).sum()
    print("full bound passes (pass 1) per request: %.3f" % (float(tot_pass1) / (len(g.chains) * w.window)))
