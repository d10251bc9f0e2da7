"""Dev tool: find vLLM+ variants whose device replay fails or disagrees with the oracle."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np

import gpu_util as GU
import oracle as O
import tracegen as tg

R = int(os.environ.get("R", "3000"))
w = tg.workload(3, R=R)
m = w.variants[0].model
for b in (16, 32, 64, 128):
    for c in (30, 60, 90, 120):
        v = tg.Variant(m, c * tg.GB, 0, 0, b)
        try:
            from paper_2411_19379_b200 import AlphaGrid
            g = AlphaGrid(w.trace, [v], [0.0], 8, max_nodes=8192)
            g.setup()
            g.ctx.check()
            live_ok = "live ok"
        except Exception as e:
            print(b, c, "LIVE FAIL", e, flush=True)
            continue
        snaps, h, f, by = O.live_pass(w.trace, v, g.window)
        lh = g.live[0].cpu().numpy()[0]
        bad = np.nonzero(lh != h)[0]
        print(b, c, live_ok, "live mismatches", len(bad), (bad[:3] + 1).tolist(), flush=True)
        try:
            out = g.run()
            g.ctx.check()
            print(b, c, "replay ok", flush=True)
        except Exception as e:
            print(b, c, "REPLAY FAIL", e, flush=True)
