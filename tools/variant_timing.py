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
w = tg.workload(cfg, layout=os.environ.get("LAYOUT", "stream"))
g = AlphaGrid(w.trace, w.variants, w.alphas, w.n_segments, max_nodes=int(os.environ.get('MAXN', '8192'))).setup()
out = g.ctx.alloc_outputs(len(w.alphas), counters=True, chain_cycles=True)
ts = []
for it in range(6):
    out["hit_sum"].zero_()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    kw = {'n_workers': int(os.environ['NW'])} if os.environ.get('NW') else {}
    if os.environ.get('SMEMN'):
        kw['smem_nodes'] = int(os.environ['SMEMN'])
    g.run(out=out, **kw)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
    if it == 0 and os.environ.get("REORDER"):  # cost feedback as bench.py does (longest chains first)
        g.reorder_by_cycles(out["cycles"])
g.ctx.check()
cyc = out["cycles"].cpu().numpy().astype(np.float64) * 1024
ctr = out["counters"].cpu().numpy()
print(f"{os.path.basename(os.environ.get('MARCONI_LIB', 'default'))} NW={os.environ.get('NW', '-')} cfg{cfg} {os.environ.get('LAYOUT', 'stream')}: replay ms {np.median(ts[1:]):.2f} "
      f"(min {min(ts[1:]):.2f}) chains {len(g.chains)} chain-cycles median {np.median(cyc)/1e6:.2f}M max {cyc.max()/1e6:.2f}M "
      f"hitsum {int(out['hit_sum'].sum())}", flush=True)
if os.environ.get("PHASES"):
    tot = ctr.astype(np.float64).sum(0)
    print("phase cycles share walk/evict/insert/unpin:", np.round(tot / tot.sum(), 3), "per request (M):",
          np.round(tot / (len(g.chains) * w.window) / 1e3, 1), "k-cycles")
if os.environ.get("PHASES3"):
    c = ctr.astype(np.uint64)
    nreq = len(g.chains) * w.window
    m40 = np.uint64((1 << 40) - 1)
    sel = c[:, 0].astype(np.float64).sum() / nreq / 1e3
    p2 = (c[:, 1] & m40).astype(np.float64).sum() / nreq / 1e3
    fp = float((c[:, 1] >> np.uint64(40)).sum()) / nreq
    rem = (c[:, 2] & m40).astype(np.float64).sum() / nreq / 1e3
    sl = float((c[:, 2] >> np.uint64(40)).sum()) / nreq
    p1 = float((c[:, 3] >> np.uint64(32)).sum()) / nreq
    fb = float((c[:, 3] & np.uint64(0xFFFF)).sum()) / nreq
    nt = float(((c[:, 3] >> np.uint64(16)) & np.uint64(0xFFFF)).sum()) / nreq
    print("per request k-cycles: select %.1f (pass2 %.1f) removal %.1f ; pass-1 runs/request %.3f fallbacks/request %.4f "
          "near-ties/request %.4f shortlist-decided selections/request %.3f full passes/request %.3f" % (sel, p2, rem, p1, fb, nt, sl, fp))
if os.environ.get("CTR"):
    nreq = len(g.chains) * w.window
    print("per request: compared %.1f visited %.2f scanned %.1f written %.2f" % tuple(ctr.astype(np.float64).sum(0) / nreq))
if os.environ.get("PHASES4"):
    t = ctr.astype(np.float64).sum(0)
    print("pass-2 scans: %.0f, entries/scan %.1f, cycles/scan %.0f, cycles per entry-per-lane %.1f"
          % (t[2], t[1] / t[2], t[0] / t[2], t[0] / (t[1] / 32)))
if os.environ.get("LOADT"):
    c = ctr.astype(np.float64)
    print("snapshot load cycles per chain: median %.0f mean %.0f max %.0f; share of chain cycles %.3f"
          % (np.median(c[:, 0]), c[:, 0].mean(), c[:, 0].max(), c[:, 0].sum() / cyc.sum()))
if os.environ.get("CHAINS"):
    na, ns = len(w.alphas), len(g.segs)
    cy = np.zeros(na * ns)
    cy[g.chains.astype(np.int64)] = cyc[g.chains.astype(np.int64)] if cyc.shape[0] == na * ns else 0
    M = cy.reshape(na, ns) / 1e6
    print("per-alpha mean/max chain Mcycles:", [(a, round(M[i].mean(), 2), round(M[i].max(), 2)) for i, a in enumerate(w.alphas)])
    segm = M.mean(0)
    print("segment mean Mcycles: min %.2f median %.2f max %.2f" % (segm.min(), np.median(segm), segm.max()))
    top = np.argsort(-cy)[:12]
    print("top chains (alpha, seg, Mcyc, seg-mean):", [(w.alphas[c // ns], c % ns, round(cy[c] / 1e6, 2), round(segm[c % ns], 2)) for c in top])
if os.environ.get("PHASES3A"):
    na, ns = len(w.alphas), len(g.segs)
    c = ctr.astype(np.uint64)
    for ai, a in enumerate(w.alphas):
        ids = [ai * ns + s for s in range(ns)]
        sub = c[ids]
        nreq = ns * w.window
        sel = sub[:, 0].astype(np.float64).sum() / nreq / 1e3
        p2 = (sub[:, 1] & np.uint64((1 << 40) - 1)).astype(np.float64).sum() / nreq / 1e3
        fp = float((sub[:, 1] >> np.uint64(40)).sum()) / nreq
        rem = (sub[:, 2] & np.uint64((1 << 40) - 1)).astype(np.float64).sum() / nreq / 1e3
        sl = float((sub[:, 2] >> np.uint64(40)).sum()) / nreq
        p1 = float((sub[:, 3] >> np.uint64(32)).sum()) / nreq
        fb = float((sub[:, 3] & np.uint64(0xFFFF)).sum()) / nreq
        nt = float(((sub[:, 3] >> np.uint64(16)) & np.uint64(0xFFFF)).sum()) / nreq
        print("alpha %-8g select %.1f pass2 %.1f removal %.1f k-cyc/req; pass1 %.3f fallback %.4f near-tie %.4f shortlist %.3f full %.3f per req"
              % (a, sel, p2, rem, p1, fb, nt, sl, fp))
if os.environ.get("DUMP"):
    os.makedirs("gpurun_out", exist_ok=True)
    np.savez(os.environ["DUMP"], cycles=cyc, counters=ctr, chains=g.chains.astype(np.int64),
             est=np.asarray(g.costs if hasattr(g, "costs") else [], np.int64))
