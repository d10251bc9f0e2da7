"""GPU: the report's per-policy numbers equal the oracle's on the same traces -- vLLM+
(block 32, LRU), SGLang+ (Marconi admission + LRU = the α = 0 live pass) and Marconi's
online tuning loop (oracle.live_tune) -- hit rates exact, TTFT proxies from identical
per-request FLOPs."""
import dataclasses

import numpy as np
import pytest

import oracle as O
import tracegen as tg

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
if not torch.cuda.is_available():
    pytest.skip("needs a CUDA device", allow_module_level=True)

from paper_2411_19379_b200 import report as RP  # noqa: E402


@pytest.mark.parametrize("cfg,R", [(3, 4000), (4, 1500)])
def test_report_matches_oracle(cfg, R):
    w = tg.workload(cfg, R=R)
    v = dataclasses.replace(w.variants[0], capacity_bytes=20 * tg.GB)  # contention at this size
    tfl = 500.0
    res = RP.evaluate(w.trace, v, tg.ALPHA_GRID16, tfl)
    lin = w.trace.lin.astype(np.int64)
    f_in = np.array([O.prefill_flops(v.model, int(x)) for x in lin], np.uint64)
    assert np.array_equal(RP.prefill_flops_device(v.model, w.trace.lin), f_in)
    vl = dataclasses.replace(v, block_size=RP.VLLM_BLOCK)
    for name, var in (("vllm+", vl), ("sglang+", v)):
        _, h, f, _ = O.live_pass(w.trace, var, w.trace.n_requests)
        assert res[name].hit_rate == float(h.astype(np.int64).sum()) / float(lin.sum()), name
        assert res[name].ttft == RP.ttft_proxy(f_in, f.astype(np.uint64), tfl), name
    h, f, info = O.live_tune(w.trace, v, tg.ALPHA_GRID16)
    assert res["marconi"].alpha_star == info["alpha_star"]
    assert res["marconi"].hit_rate == float(h.astype(np.int64).sum()) / float(lin.sum())
    assert res["marconi"].ttft == RP.ttft_proxy(f_in, f.astype(np.uint64), tfl)
