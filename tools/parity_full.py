#!/usr/bin/env python3
"""Full-size GPU-vs-oracle parity of one BASELINE config, every chain (test tooling).

Runs the α-grid exactly as bench.py launches it (device live pass, default workers,
eviction logs OFF -- the benchmarked branch of the kernel), then the CPU oracle over
every chain on all host cores, and compares element by element: segment snapshots,
live-pass hits, every request's hit / FLOPs saved / bypass flag, the d.3 counters of
every chain, the per-α hit sums and α*.  A second replay call with eviction logs on a
chain subset compares the logs bitwise (request, node id, kind, live count, utility
bits) and checks that turning logs on changes no output.

  python tools/parity_full.py --config 5 --out gpurun_out/parity_cfg5.json

The oracle is test infrastructure (oracle/__init__.py header); this script is a test
driver, not a product path.  Output: one JSON summary (committed under profiles/).
"""
from __future__ import annotations

import argparse
import json
import os
import platform
import subprocess
import sys
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))


def cpu_model() -> str:
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for ln in out.splitlines():
            if ln.startswith("Model name:"):
                return ln.split(":", 1)[1].strip()
    except Exception:
        pass
    return platform.processor() or "unknown"


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=5)
    ap.add_argument("--requests", type=int, default=0)
    ap.add_argument("--layout", default="stream", choices=["stream", "copy"])
    ap.add_argument("--policy", default="marconi", choices=["marconi", "vllm"],
                    help="vllm: bench.py's vLLM+ sweep (block sizes x cache sizes as variants, α = 0)")
    ap.add_argument("--blocks", default="16,32,64,128")
    ap.add_argument("--caps-gb", default="30,60,90,120")
    ap.add_argument("--log-chains", type=int, default=24, help="chains replayed a second time with eviction logs")
    ap.add_argument("--out", default="")
    a = ap.parse_args()

    import torch
    import oracle as O
    import tracegen as tg
    import gpu_util as GU
    from paper_2411_19379_b200 import AlphaGrid

    w = tg.workload(a.config, R=a.requests or None, layout=a.layout)
    if a.policy == "vllm":  # the same variant set as bench.py --policy vllm
        m = w.variants[0].model
        w.variants = [tg.Variant(m, int(float(c) * tg.GB), 0, 0, int(b)) for b in a.blocks.split(",")
                      for c in a.caps_gb.split(",")]
        w.alphas = (0.0,)
    tr = w.trace
    nv, na = len(w.variants), len(w.alphas)
    res = {"config": a.config, "policy": a.policy, "workload": w.name, "requests": tr.n_requests, "variants": nv, "alphas": na,
           "segments": w.n_segments, "chains": w.n_chains, "host_cores": os.cpu_count(), "cpu_model": cpu_model(),
           "gpu": torch.cuda.get_device_name(0)}
    t0 = time.perf_counter()
    g = AlphaGrid(tr, w.variants, w.alphas, w.n_segments).setup()
    out = g.run(counters=True)            # logs off: the bench branch
    g.ctx.check()
    torch.cuda.synchronize()
    res["gpu_s"] = round(time.perf_counter() - t0, 2)
    hit, fl, by = (out[x].cpu().numpy() for x in ("hit", "flops", "bypass"))
    ctr = out["counters"].cpu().numpy()
    live = g.live[0].cpu().numpy()
    segs = g.segs
    ns = len(segs)
    W = g.window

    # ---- oracle: live passes (one thread per variant), then every chain on every core
    t1 = time.perf_counter()
    with ThreadPoolExecutor(max_workers=min(nv, os.cpu_count() or 1)) as ex:
        lp = list(ex.map(lambda v: O.live_pass(tr, v, W), w.variants))
    res["oracle_live_s"] = round(time.perf_counter() - t1, 2)
    snaps = [x[0] for x in lp]
    t2 = time.perf_counter()
    flat_snaps, base = [], []
    for v in range(nv):
        base.append(len(flat_snaps))
        flat_snaps.extend(snaps[v])
    chains = [(v, w.alphas[ai], f, n, base[v] + k) for v in range(nv) for ai in range(na) for (f, n, k) in segs]
    oh, of, ob, ohs, octr = O.run_chains(tr, w.variants, chains, flat_snaps, n_threads=os.cpu_count() or 1)
    res["oracle_chains_s"] = round(time.perf_counter() - t2, 2)
    res["oracle_request_replays"] = int(sum(c[3] for c in chains))
    res["oracle_rate_per_s"] = res["oracle_request_replays"] / res["oracle_chains_s"]

    # ---- compare
    bad = []
    n_req_cmp = 0
    for v in range(nv):
        if not np.array_equal(live[v], lp[v][1]):
            bad.append(f"live hits v{v}")
        for k in range(len(snaps[v])):
            gs, gn = g.ctx.get_snapshot(v, k)
            on, onid = snaps[v][k]
            if gn != onid or not np.array_equal(GU.canon(gs), GU.canon(on)):
                bad.append(f"snapshot v{v} k{k}")
    for cid, (v, alpha, first, n, _) in enumerate(chains):
        ai = (cid // ns) % na
        sl = slice(first - 1, first - 1 + n)
        if not np.array_equal(hit[v, ai, sl], oh[cid]):
            bad.append(f"hit chain {cid}")
        if not np.array_equal(fl[v, ai, sl], of[cid].astype(np.int64)):
            bad.append(f"flops chain {cid}")
        if not np.array_equal(by[v, ai, sl], ob[cid].astype(np.uint8)):
            bad.append(f"bypass chain {cid}")
        if not np.array_equal(ctr[cid], octr[cid].astype(np.int64)):
            bad.append(f"counters chain {cid}")
        n_req_cmp += n
    a_star = g.select(out)
    for v in range(nv):
        sums = [int(sum(int(ohs[(v * na + ai) * ns + si]) for si in range(ns))) for ai in range(na)]
        if [int(x) for x in g.hit_sums[v]] != sums:
            bad.append(f"hit sums v{v}")
        if a_star[v] != O.select_alpha(w.alphas, sums):
            bad.append(f"alpha* v{v}")
    res["alpha_star"] = a_star

    # ---- eviction logs on a chain subset (second call, logs on), spread over variants / α / segments
    rng = np.random.default_rng(a.config)
    sub = sorted(set(int(x) for x in rng.choice(len(chains), size=min(a.log_chains, len(chains)), replace=False)))
    out2 = g.ctx.alloc_outputs(na, log_cap=1 << 18, counters=True)
    g.ctx.replay(w.alphas, chains=sub, out=out2)
    g.ctx.check()
    h2 = out2["hit"].cpu().numpy()
    n_ev = 0
    t3 = time.perf_counter()

    def one(cid):
        v, alpha, first, n, k = chains[cid]
        _, _, _, lg = GU.oracle_chain_log(tr, w.variants[v], alpha, first, n, flat_snaps[k])
        return cid, lg

    with ThreadPoolExecutor(max_workers=os.cpu_count() or 1) as ex:
        logs = list(ex.map(one, sub))
    for cid, lg in logs:
        v, alpha, first, n, _ = chains[cid]
        ai = (cid // ns) % na
        sl = slice(first - 1, first - 1 + n)
        if not np.array_equal(h2[v, ai, sl], hit[v, ai, sl]):
            bad.append(f"logged replay changed hits chain {cid}")
        glog, gn = g.ctx.read_log(out2, cid)
        ok = gn == len(lg)  # the device counts every eviction; it keeps the first log_cap records
        lgk = lg[:len(glog)]
        if ok:
            for f in ("req", "node_id", "kind", "n_live"):
                ok &= np.array_equal(glog[f], lgk[f])
            ok &= np.array_equal(glog["utility"].view(np.uint64), lgk["utility"].view(np.uint64))
        if len(glog) < gn:
            res["log_truncated_chains"] = res.get("log_truncated_chains", 0) + 1
        if not ok:
            bad.append(f"eviction log chain {cid}")
        n_ev += len(glog)
    res["log_chains"] = sub
    res["log_evictions_compared"] = n_ev
    res["oracle_log_s"] = round(time.perf_counter() - t3, 2)
    res["requests_compared"] = n_req_cmp
    res["mismatches"] = bad[:50]
    res["n_mismatches"] = len(bad)
    res["parity"] = "green" if not bad else "RED"
    s = json.dumps(res, indent=1)
    print(s)
    if a.out:
        os.makedirs(os.path.dirname(os.path.abspath(a.out)), exist_ok=True)
        open(a.out, "w").write(s + "\n")
    sys.exit(0 if not bad else 1)


if __name__ == "__main__":
    main()
