"""GPU parity of the online tuning loop (LiveTuner, NEXT-1) against oracle.live_tune:
first-eviction request, bootstrap window, grid hit sums, α*, and every request's hit
tokens / FLOPs saved over the whole trace."""
import os

import numpy as np
import pytest

import oracle as O
import tracegen as tg

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_19379_b200 import LiveTuner  # noqa: E402


def _check(tr, v, alphas, mult=10, max_nodes=8192):
    lt = LiveTuner(tr, v, alphas, multiplier=mult, max_nodes=max_nodes)
    h, f, info = lt.run()
    oh, of, oinfo = O.live_tune(tr, v, alphas, multiplier=mult, n_threads=os.cpu_count() or 1)
    assert info["r_first_evict"] == oinfo["r_first_evict"]
    assert info["window"] == oinfo["window"]
    assert info["grid_hit_sums"] == oinfo["grid_hit_sums"]
    assert info["alpha_star"] == oinfo["alpha_star"]
    assert np.array_equal(h, oh)
    assert np.array_equal(f, of.astype(np.int64))
    return info


@pytest.mark.parametrize("cfg", [2, 3, 4])
def test_live_tuning_full_configs(cfg):
    w = tg.workload(cfg)
    info = _check(w.trace, w.variants[0], tg.ALPHA_GRID16)
    assert info["r_first_evict"] > 0


def test_live_tuning_toy_and_micro():
    w = tg.workload(1)
    _check(w.trace, w.variants[0], (0.0, 1.0), mult=2, max_nodes=64)
    for seed in range(40):
        tr = tg.micro_trace(seed, n_req=20, max_len=64, alphabet=2 + seed % 3)
        v = tg.Variant(tg.MODEL_7B, tg.UNLIMITED_BYTES, 2 + seed % 5)
        _check(tr, v, (0.0, 1 / 16, 1.0, 64.0), mult=2, max_nodes=128)


def test_live_tuning_no_eviction():
    w = tg.workload(3, R=2000)
    info = _check(w.trace, tg.Variant(tg.MODEL_7B, tg.UNLIMITED_BYTES), (0.0, 1.0))
    assert info["r_first_evict"] == 0 and info["alpha_star"] == 0.0
