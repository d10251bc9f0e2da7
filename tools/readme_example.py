import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import tracegen as tg
from paper_2411_19379_b200 import AlphaGrid, LiveTuner
from paper_2411_19379_b200.grid import HostPipeline

w = tg.workload(3)                      # ShareGPT-shaped trace, 7B hybrid, 60 GB, 16 α x 128 segments
g = AlphaGrid(w.trace, w.variants, w.alphas, w.n_segments).setup()   # H2D + device live pass (snapshots)
out = g.run(chain_cycles=True)          # the α-grid replay (async); out["hit"], out["flops"]: per request
g.ctx.check()                           # device status -> exception on any violated invariant
alpha_star = g.select(out)              # NCCL all-gather of per-α hit sums (N > 1), argmax, ties -> smallest α
rates = g.metrics(out)                  # {(variant, α): (token hit rate, FLOPs saved)}
g.reorder_by_cycles(out["cycles"])      # optional: longest chains first in the next replay

hits, flops, info = LiveTuner(w.trace, w.variants[0], w.alphas).run()   # the paper's online loop (§4.2)
res = g.ctx.lookup(req=[1, 2, 3], variant=0, snapshot=5)              # read-only lookups vs a snapshot

print('alpha*', alpha_star, 'rate', rates[(0, alpha_star[0])][0], 'tuner', info['alpha_star'], 'lookup', g.ctx.lookup_records(res)['reuse'].tolist())
