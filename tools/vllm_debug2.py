"""Dev tool: reproduce one failing vLLM+ variant (run under compute-sanitizer)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tracegen as tg
from paper_2411_19379_b200 import AlphaGrid

R = int(os.environ.get("R", "3000"))
b, c = int(os.environ.get("B", "16")), int(os.environ.get("CAP", "120"))
w = tg.workload(3, R=R)
v = tg.Variant(w.variants[0].model, c * tg.GB, 0, 0, b)
g = AlphaGrid(w.trace, [v], [0.0], int(os.environ.get("SEGS", "8")), max_nodes=8192)
g.setup()
g.ctx.check()
print("snapshot sizes", [len(g.ctx.get_snapshot(0, k)[0]) for k in range(g.ctx.snapshot_count(0))], flush=True)
out = g.run(n_workers=int(os.environ.get("NW", "0")))
g.ctx.check()
print("ok", int(out["hit_sum"].sum()))
