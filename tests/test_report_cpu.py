"""The report's host arithmetic (no GPU): the TTFT proxy's closed forms ("FLOP
saved is a reasonable proxy for compute and latency savings") and the hit-rate rule."""
import numpy as np

import oracle as O
import tracegen as tg
from paper_2411_19379_b200 import report as RP


def test_ttft_proxy_closed_forms():
    m = tg.MODEL_7B
    lin = np.array([100, 1000, 10000], np.int64)
    f_in = np.array([O.prefill_flops(m, int(x)) for x in lin], np.uint64)
    # no hits: the proxy is F(L_in) / throughput and equals the no-cache P95
    p = RP.ttft_proxy(f_in, np.zeros(3, np.uint64), 1000.0)
    assert abs(p["p95_rel_no_cache"] - 1.0) < 1e-12
    assert abs(p["p50_ms"] - float(f_in[1]) / 1e15 * 1e3) < 1e-9
    # full-input hits: nothing left to prefill
    p = RP.ttft_proxy(f_in, f_in.copy(), 1000.0)
    assert p["p95_ms"] == 0.0 and p["p95_rel_no_cache"] == 0.0
    # F(10000) - F(1000) over a 10x faster assumed throughput is 10x smaller
    hit = np.array([0, 0, O.prefill_flops(m, 1000)], np.uint64)
    a, b = RP.ttft_proxy(f_in, hit, 100.0), RP.ttft_proxy(f_in, hit, 1000.0)
    assert abs(a["p95_ms"] / b["p95_ms"] - 10.0) < 1e-9


def test_default_throughput_is_labelled_fraction_of_measured_peak():
    assert 100.0 < RP.default_prefill_tflops() < 2250.0


def test_markdown_tables_cover_every_section():
    row = {"case": "x", "hit_vllm+": 0.1, "hit_sglang+": 0.5, "hit_marconi": 0.6, "alpha_star": 0.25,
           "marconi_vs_vllm+": 6.0, "marconi_vs_sglang+": 1.2,
           "ttft_p95_rel_no_cache": {"vllm+": 0.9, "sglang+": 0.5, "marconi": 0.4},
           "ttft_proxy_ms": {}}
    rep = {"prefill_tflops_assumed": 500.0, "ttft_note": "proxy", "data": "synthetic"}
    for sec in ("main", "state_dim", "arrival", "cache_size", "ratio"):
        rep[sec] = [dict(row, case=sec)]
    md = RP.to_markdown(rep)
    for sec in ("main", "state_dim", "arrival", "cache_size", "ratio"):
        assert f"## {sec}" in md and f"| {sec} | 10.0 % | 50.0 % | 60.0 % (0.25) | 6.00 | 1.20 |" in md
