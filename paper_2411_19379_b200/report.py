"""Report mode: the paper's comparisons re-run on the synthetic
traces with the device replay, plus a labelled FLOP-based TTFT proxy.

  python -m paper_2411_19379_b200.report [--quick] [--json out.json]

Every number comes from the CUDA kernels (live pass, α-grid replay, LiveTuner, the
K1 cost-model kernel); this module only sums and tabulates their outputs.

Policies compared per trace:
  * vLLM+   -- a state per 32-token block, LRU (block_size = 32);
  * SGLang+ -- Marconi's judicious admission with LRU eviction = the α = 0 live pass
               (α = 0 falls back to LRU);
  * Marconi -- the paper's online loop: α = 0 until the first eviction, bootstrap
               replay of 10x those requests, α-grid, adopt α* (LiveTuner).

Metrics: token hit rate = Σ skipped prefill tokens / Σ input tokens.
TTFT proxy (labelled, "FLOP saved is a reasonable proxy for compute and
latency savings because prefill is easily compute-bottlenecked"): per request,
remaining prefill FLOPs F(L_in) - F(hit) (Appendix A cost model, exact, from the K1
kernel and the replay's F(hit) output) divided by an ASSUMED prefill throughput
(--prefill-tflops, default 40 % of the measured dense bf16 B200 GEMM peak).  It is
not a measured latency: no model runs here.  Reported as
P5/P50/P95 in ms and the P95 relative to no prefix caching (fig:ttft_total_distribution).

Sweeps (same kernels, second workloads): SSM state dimension N in {16, 32, 64, 128}
(fig:microbenchmark_state_dim), session rate / response time
(fig:micro_arrival), cache size 60-140 GB (fig:micro_contention,
PAPER:640-643), Attention:SSM ratio 1:2 / 1:4 / 1:8.  The traces are
synthetic shapes of the paper's workloads, so absolute numbers are not the paper's.
"""
from __future__ import annotations

import argparse
import dataclasses
import json
import os
import sys
from typing import Dict, List, Sequence

import numpy as np

from . import marconi as M
from .grid import LiveTuner

VLLM_BLOCK = 32
MAX_NODES = 16384  # node-table size of every report context (vLLM+ at N = 16 holds ~9k blocks)


def _root():
    return os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def default_prefill_tflops() -> float:
    """40 % of the measured sustained dense bf16 GEMM peak (MEASURED_PEAKS.json), else of
    the profiling guide's fallback -- an assumption, stated in every report."""
    p = os.path.join(_root(), "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        peak = float(d.get("bf16_tflops_sustained") or d["bf16_tflops"])
    except (OSError, KeyError, ValueError):
        peak = 1590.0
    return 0.4 * peak


def prefill_flops_device(model, lengths: np.ndarray) -> np.ndarray:
    """F(L) for every L (Appendix A, exact u64) from the K1 kernel (mc_node_cost with
    d_start = 0, d_end = L)."""
    import torch
    n = lengths.shape[0]
    ds = torch.zeros(n, dtype=torch.int32, device="cuda")
    de = torch.from_numpy(lengths.astype(np.int32)).cuda()
    ssm = torch.zeros(n, dtype=torch.uint8, device="cuda")
    saved, _, _ = M.node_cost(model, ds, de, ssm)
    return saved.cpu().numpy().astype(np.uint64)


def ttft_proxy(f_in: np.ndarray, f_hit: np.ndarray, tflops: float) -> Dict[str, float]:
    """Labelled TTFT proxy from per-request prefill FLOPs: with caching F(L_in) - F(hit),
    without caching F(L_in); divided by an assumed prefill throughput (TFLOP/s)."""
    rem = (f_in.astype(np.float64) - f_hit.astype(np.float64)) / (tflops * 1e12) * 1e3
    full = f_in.astype(np.float64) / (tflops * 1e12) * 1e3
    p = {f"p{q}_ms": float(np.percentile(rem, q)) for q in (5, 50, 95)}
    p["p95_no_cache_ms"] = float(np.percentile(full, 95))
    p["p95_rel_no_cache"] = p["p95_ms"] / p["p95_no_cache_ms"] if p["p95_no_cache_ms"] > 0 else 1.0
    return p


@dataclasses.dataclass
class PolicyResult:
    hit_rate: float
    ttft: Dict[str, float]
    alpha_star: float = 0.0


def evaluate(trace, variant, alphas: Sequence[float], tflops: float, multiplier: int = 10) -> Dict[str, PolicyResult]:
    """vLLM+, SGLang+ and Marconi (LiveTuner) on one trace and cache configuration."""
    lin = trace.lin.astype(np.int64)
    denom = float(lin.sum())
    f_in = prefill_flops_device(variant.model, trace.lin)
    out = {}
    # vLLM+ and SGLang+: device live passes (LRU) of one context with both variants
    vl = dataclasses.replace(variant, block_size=VLLM_BLOCK, chunk_size=0)
    sg = dataclasses.replace(variant, block_size=0)
    ctx = M.Context([vl, sg], max_nodes=MAX_NODES)
    ctx.upload_trace(trace.tokens, trace.off, trace.lin, trace.lout)
    hit, fl, _, _ = ctx.live_pass_at([0])
    hit, fl = hit.cpu().numpy(), fl.cpu().numpy().astype(np.uint64)
    for i, name in enumerate(("vllm+", "sglang+")):
        out[name] = PolicyResult(float(hit[i].astype(np.int64).sum()) / denom, ttft_proxy(f_in, fl[i], tflops))
    ctx.close()
    # Marconi: the online tuning loop
    h, f, info = LiveTuner(trace, sg, alphas, multiplier=multiplier, max_nodes=MAX_NODES).run()
    out["marconi"] = PolicyResult(float(h.astype(np.int64).sum()) / denom, ttft_proxy(f_in, f.astype(np.uint64), tflops),
                                  info["alpha_star"])
    return out


def _row(label, res: Dict[str, PolicyResult]) -> dict:
    m, s, v = res["marconi"], res["sglang+"], res["vllm+"]
    return {"case": label, "hit_vllm+": v.hit_rate, "hit_sglang+": s.hit_rate, "hit_marconi": m.hit_rate,
            "alpha_star": m.alpha_star,
            "marconi_vs_vllm+": m.hit_rate / v.hit_rate if v.hit_rate else float("inf"),
            "marconi_vs_sglang+": m.hit_rate / s.hit_rate if s.hit_rate else float("inf"),
            "ttft_p95_rel_no_cache": {k: r.ttft["p95_rel_no_cache"] for k, r in res.items()},
            "ttft_proxy_ms": {k: {q: r.ttft[q] for q in ("p5_ms", "p50_ms", "p95_ms")} for k, r in res.items()}}


def run(quick: bool = False, tflops: float = 0.0) -> dict:
    import tracegen as tg
    tflops = tflops or default_prefill_tflops()
    scale = 0.25 if quick else 1.0
    alphas = tg.ALPHA_GRID16
    rep = {"prefill_tflops_assumed": tflops,
           "ttft_note": "TTFT proxy = remaining prefill FLOPs / assumed throughput; not a measured latency",
           "data": "synthetic traces shaped like the paper's workloads; numbers are not the paper's"}
    main = []
    for cfg, R in ((2, 10_000), (3, 50_000), (4, 20_000)):
        w = tg.workload(cfg, R=int(R * scale))
        main.append(_row(f"config{cfg} {w.name} R={w.trace.n_requests} 60 GB", evaluate(w.trace, w.variants[0], alphas, tflops)))
    rep["main"] = main
    # state dimension N, config-4-shaped trace (long contexts)
    w4 = tg.workload(4, R=int(20_000 * scale))
    rep["state_dim"] = [_row(f"N={v.model.d_state}", evaluate(w4.trace, v, alphas, tflops))
                        for v in tg.state_dim_variants()]
    # arrival patterns
    arr = []
    for rate, delay in ((0.5, 5.0), (1.0, 5.0), (2.0, 5.0), (1.0, 10.0)):
        wa = tg.arrival_workload(rate, delay, R=int(20_000 * scale))
        arr.append(_row(f"sessions/s={rate} response={delay}s", evaluate(wa.trace, wa.variants[0], alphas, tflops)))
    rep["arrival"] = arr
    # cache size and Attention:SSM ratio on the config-5 mixture
    w5 = tg.workload(5, R=int(50_000 * scale))
    rep["cache_size"] = [_row(f"{c} GB (1:4)", evaluate(w5.trace, tg.Variant(tg.model_ratio(4), c * tg.GB), alphas, tflops))
                         for c in (60, 80, 100, 120, 140)]
    rep["ratio"] = [_row(f"1:{rho} (60 GB)", evaluate(w5.trace, tg.Variant(tg.model_ratio(rho), 60 * tg.GB), alphas, tflops))
                    for rho in (2, 4, 8)]
    return rep


def to_markdown(rep: dict) -> str:
    lines = [f"# Marconi replay report (device kernels; {rep['data']})",
             f"TTFT proxy at an assumed {rep['prefill_tflops_assumed']:.0f} TFLOP/s prefill: {rep['ttft_note']}.", ""]
    for sec in ("main", "state_dim", "arrival", "cache_size", "ratio"):
        lines += [f"## {sec}", "",
                  "| case | vLLM+ | SGLang+ | Marconi (α*) | ×vLLM+ | ×SGLang+ | P95 TTFT proxy vs no cache (vLLM+/SGLang+/Marconi) |",
                  "|---|---|---|---|---|---|---|"]
        for r in rep[sec]:
            t = r["ttft_p95_rel_no_cache"]
            lines.append(f"| {r['case']} | {100 * r['hit_vllm+']:.1f} % | {100 * r['hit_sglang+']:.1f} % | "
                         f"{100 * r['hit_marconi']:.1f} % ({r['alpha_star']:g}) | {r['marconi_vs_vllm+']:.2f} | "
                         f"{r['marconi_vs_sglang+']:.2f} | {t['vllm+']:.3f} / {t['sglang+']:.3f} / {t['marconi']:.3f} |")
        lines.append("")
    return "\n".join(lines)


def main(argv=None):
    sys.path.insert(0, _root())
    p = argparse.ArgumentParser()
    p.add_argument("--quick", action="store_true", help="quarter-size traces")
    p.add_argument("--prefill-tflops", type=float, default=0.0, help="assumed prefill throughput (TFLOP/s)")
    p.add_argument("--json", default="")
    a = p.parse_args(argv)
    rep = run(a.quick, a.prefill_tflops)
    if a.json:
        json.dump(rep, open(a.json, "w"), indent=1)
    print(to_markdown(rep))


if __name__ == "__main__":
    main()
