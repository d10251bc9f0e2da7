"""Multi-rank α-grid on the GPU: the REAL device replay (AlphaGrid over libmarconi.so) at
world sizes 2 and 4, ranks sharing the visible GPU(s) and exchanging the per-(variant, α)
hit sums over gloo (NCCL refuses two ranks on one device; on an 8-GPU box bench.py uses
NCCL, one rank per GPU).  Chains are independent replays, so every request's
hit / FLOPs saved, the hit sums and α* must not depend on the sharding: they are compared
with a world-size-1 run, and every rank must select the same α* (SURVEY.md §4 item 4).
"""
import os
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

import torch.multiprocessing as mp  # noqa: E402

import tracegen as tg  # noqa: E402


def _workload():
    w = tg.workload(3, R=6000)
    w.n_segments = 12
    return w


def _rank(rank, world, port, outdir):
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, root)
    import torch.distributed as dist
    from paper_2411_19379_b200 import AlphaGrid
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    if world > 1:
        dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = rank % torch.cuda.device_count()
    torch.cuda.set_device(dev)
    w = _workload()
    g = AlphaGrid(w.trace, w.variants, w.alphas, w.n_segments, rank=rank, world=world, device=dev).setup()
    out = g.run()
    g.ctx.check()
    a_star = g.select(out)
    np.savez(os.path.join(outdir, f"r{world}_{rank}.npz"), chains=g.chains, hit=out["hit"].cpu().numpy(),
             flops=out["flops"].cpu().numpy(), hit_sums=g.hit_sums, a_star=np.asarray(a_star),
             segs=np.asarray(g.segs))
    if world > 1:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 4])
def test_world_size_does_not_change_results(world):
    with tempfile.TemporaryDirectory() as d:
        port = 29600 + (os.getpid() % 1000)
        mp.spawn(_rank, args=(1, port, d), nprocs=1, join=True)
        mp.spawn(_rank, args=(world, port + 1, d), nprocs=world, join=True)
        ref = np.load(os.path.join(d, "r1_0.npz"))
        parts = [np.load(os.path.join(d, f"r{world}_{k}.npz")) for k in range(world)]
        w = _workload()
        na, segs = len(w.alphas), ref["segs"]
        ns = len(segs)
        seen = np.concatenate([p["chains"] for p in parts])
        assert sorted(seen.tolist()) == list(range(na * ns))            # every chain exactly once
        assert all(len(p["chains"]) > 0 for p in parts)
        for p in parts:
            assert np.array_equal(p["hit_sums"], ref["hit_sums"])         # identical after the all-gather
            assert np.array_equal(p["a_star"], ref["a_star"])             # every rank: the same α*
            for c in p["chains"].tolist():
                ai, si = c // ns, c % ns
                first, n, _ = segs[si]
                sl = slice(first - 1, first - 1 + n)
                assert np.array_equal(p["hit"][0, ai, sl], ref["hit"][0, ai, sl]), c
                assert np.array_equal(p["flops"][0, ai, sl], ref["flops"][0, ai, sl]), c
