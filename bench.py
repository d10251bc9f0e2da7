#!/usr/bin/env python3
"""bench.py -- α-grid replay throughput of Marconi's hybrid prefix cache on B200.

Metric (BASELINE.json): "requests replayed/sec × α-candidates at 1/2/4/8 B200;
HBM GB/s vs peak".  Workload: BASELINE.json configs[2] -- the ShareGPT-shaped
50k-request trace, 7B hybrid {4,24,28}, 60 GB cache, 16-value α grid x 128
trace segments = 2,048 chains.  At N GPUs: N independent problems of that shape
(trace seeds k = 0..N-1; weak scaling), the chains of every problem
LPT-sharded across all ranks.  A step = replay of this rank's chains from their
segment snapshots + one NCCL all-gather of per-(problem, α) hit sums + α*
selection.  Why weak by default: a chain is sequential, and
one config-3 problem's 2,048 chains already run concurrently on one B200, so a
fixed chain list of that size cannot get much faster on more GPUs.  `--scaling
strong` shards ONE problem's chain list over the ranks instead (
config 5's 3,840 chains take two waves on one GPU).

  python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference] [--config 3]
                  [--scaling weak|strong]

`--gpus N` without torchrun re-launches itself as N ranks (torch.distributed.run on
127.0.0.1).  If fewer GPUs are visible than ranks, ranks share devices and exchange
over gloo (flagged in the line's config: runnable, not a scaling number).

Setup (untimed, reported): trace generation, H2D, the α = 0 device live pass
that produces the 128 segment snapshots.  L2 is flushed (a 256 MiB write)
between timed steps, outside the per-step CUDA-event window.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "requests replayed/sec×α-candidates at 1/2/4/8 B200; HBM GB/s vs peak"
UNIT = "request-replays/s"
# algorithmic bytes per request-replay:
#   B_r = 8*c_r + 16*v_r + 13*sum_j N_j + 32*w_r + 16
W_CMP, W_VIS, W_SCAN, W_WR, W_OUT = 8, 16, 13, 32, 16


def parse():
    p = argparse.ArgumentParser()
    p.add_argument("--gpus", type=int, default=1)
    p.add_argument("--steps", type=int, default=10)
    p.add_argument("--warmup", type=int, default=3)
    p.add_argument("--impl", default="b200", choices=["b200", "reference"])
    p.add_argument("--config", type=int, default=3)
    p.add_argument("--policy", default="marconi", choices=["marconi", "vllm"],
                   help="vllm: the vLLM+ baseline (NEXT-2) on the same trace -- a sweep of block sizes x "
                        "cache sizes as variants (alpha does not apply to its LRU)")
    p.add_argument("--blocks", default="16,32,64,128", help="vLLM+ block sizes (tokens)")
    p.add_argument("--caps-gb", default="30,60,90,120", help="vLLM+ cache sizes (GB)")
    p.add_argument("--requests", type=int, default=0, help="override R (testing only)")
    p.add_argument("--layout", default="stream", choices=["stream", "copy"],
                   help="copy: every request holds its own copy of its sequence (no shared session stream, "
                        "so every walk level compares tokens; SURVEY.md a2)")
    p.add_argument("--no-e2e", action="store_true")
    p.add_argument("--no-cpu-baseline", action="store_true")
    p.add_argument("--cpu-seconds", type=float, default=15.0, help="target wall time of the oracle sample")
    p.add_argument("--no-traffic", action="store_true",
                   help="skip the ncu DRAM-bytes probe of one replay launch (roofline.traffic)")
    p.add_argument("--traffic-probe", action="store_true", help=argparse.SUPPRESS)  # internal: the probe's child
    p.add_argument("--scaling", default="weak", choices=["weak", "strong"],
                   help="weak: N independent problems at N GPUs (default); strong: ONE problem's chain list "
                        "LPT-sharded over the N ranks (SURVEY.md d.4; the primary mode for config 5)")
    return p.parse_args()


def free_port() -> int:
    import socket
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def respawn(args):
    """`bench.py --gpus N` (N > 1) started without torchrun: re-launch itself as N ranks,
    one process per GPU (torch.distributed.run, rendezvous on 127.0.0.1), and exit with
    the ranks' status.  Rank 0 prints the JSON line."""
    if args.gpus <= 1 or "WORLD_SIZE" in os.environ:
        return
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={free_port()}", os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        d = json.load(open(path))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


class Clocks:
    """nvidia-smi sampler running during the timed region (B200_PROFILING.md clocks line)."""
    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except Exception:
            self.proc = None

    def _read(self):
        for ln in self.proc.stdout:
            self.lines.append(ln.strip())

    def stop(self):
        if not self.proc:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.t.join(timeout=2)
        sm, mx, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 7:
                continue
            try:
                sm.append(float(f[0]))
                mx.append(float(f[1]))
            except ValueError:
                continue
            for nm, val in zip(names, f[3:7]):
                if val.lower() == "active":
                    reasons.add(nm)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": sorted(reasons), "samples": len(sm)}


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def algorithmic_bytes(ctr: np.ndarray, n_req_replayed: int) -> int:
    c = ctr.astype(np.int64).sum(0)
    return int(W_CMP * c[0] + W_VIS * c[1] + W_SCAN * c[2] + W_WR * c[3] + W_OUT * n_req_replayed)


# ----------------------------------------------------------------------------
# CPU oracle arms (the only places bench.py executes oracle/)
# ----------------------------------------------------------------------------
def cpu_model() -> str:
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def oracle_sample(w, target_s: float, cores: int):
    """A bounded sample of the same workload for the oracle: the first k segments x all
    (variant, α) chains, k sized so the sample takes about target_s seconds on `cores`
    threads.  Returns (snapshots, chains, k); chain snapshot index = variant * k + segment."""
    import oracle as O
    tr, v0 = w.trace, w.variants[0]
    W = w.window
    # calibrate: single-thread time per request-replay on one chain of segment 1
    snaps, *_ = O.live_pass(tr, v0, W, upto=W)
    t0 = time.perf_counter()
    O.run_chains(tr, [v0], [(0, w.alphas[-1], W + 1, W, 1)], snaps, n_threads=1) if len(snaps) > 1 else None
    per_req = max((time.perf_counter() - t0) / W, 1e-6)
    oracle_sample.single_thread_rate = 1.0 / per_req
    nchain_per_seg = len(w.alphas) * len(w.variants)
    k = int(max(1, min(len(w.segments()), target_s * cores / (per_req * W * nchain_per_seg))))
    segs = w.segments()[:k]
    all_snaps = []
    for v in w.variants:
        sv, *_ = O.live_pass(tr, v, W, upto=min(k * W, tr.n_requests))
        sv = (sv + [sv[-1]] * k)[:k]  # pad (only segments < k are used)
        all_snaps.extend(sv)
    chains = [(vi, a, f, n, vi * k + i) for vi in range(len(w.variants)) for a in w.alphas
              for i, (f, n) in enumerate(segs)]
    return all_snaps, chains, k


def run_oracle(w, snaps, chains, cores):
    import oracle as O
    t0 = time.perf_counter()
    hit, fl, by, hs, ctr = O.run_chains(w.trace, w.variants, chains, snaps, n_threads=cores)
    dt = time.perf_counter() - t0
    n = sum(c[3] for c in chains)
    return n, dt


def cpu_baseline(w, target_s):
    cores = os.cpu_count() or 1
    snaps, chains, k = oracle_sample(w, target_s, cores)
    n, dt = run_oracle(w, snaps, chains, cores)
    return {"value": n / dt, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
            "single_thread_rate": getattr(oracle_sample, "single_thread_rate", None),
            "sample": f"first {k} of {len(w.segments())} segments x {len(w.variants)} variant(s) x "
                      f"{len(w.alphas)} alphas = {len(chains)} chains, "
                      f"{n} request-replays in {dt:.2f} s (snapshots from the oracle's own live pass, untimed)"}


def reference_arm(args, w, config):
    rank, world, local = dist_env()
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    snaps, chains, k = oracle_sample(w, min(args.cpu_seconds, 8.0), cores)
    for _ in range(args.warmup):
        run_oracle(w, snaps, chains, cores)
    tot_n, tot_t = 0, 0.0
    for _ in range(args.steps):
        n, dt = run_oracle(w, snaps, chains, cores)
        tot_n += n
        tot_t += dt
    v = tot_n / tot_t
    line = {"impl": "reference", "metric": METRIC, "value": v, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1000 * tot_t / args.steps,
            "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "u64+f64",
            "data": "synthetic", "config": config,
            "cpu_baseline": {"value": v, "unit": UNIT, "cores": cores, "kind": "oracle", "cpu_model": cpu_model(),
                             "single_thread_rate": getattr(oracle_sample, "single_thread_rate", None),
                             "sample": f"{len(chains)} chains of the first {k} segments per step"},
            "e2e": {"value": v, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


# ----------------------------------------------------------------------------
# B200 arm
# ----------------------------------------------------------------------------
def main():
    args = parse()
    respawn(args)
    import tracegen as tg
    rank, world, local = dist_env()
    n_prob = max(1, world) if (args.impl == "b200" and args.scaling == "weak") else 1
    t_gen = time.perf_counter()
    ws = [tg.workload(args.config, R=args.requests or None, problem=k, layout=args.layout) for k in range(n_prob)]
    if args.policy == "vllm":  # NEXT-2: the vLLM+ baseline on the same traces, block x cache-size sweep
        blocks = [int(b) for b in args.blocks.split(",")]
        caps = [int(float(c) * tg.GB) for c in args.caps_gb.split(",")]
        for wk in ws:
            m = wk.variants[0].model
            wk.variants = [tg.Variant(m, c, 0, 0, b) for b in blocks for c in caps]
            wk.alphas = (0.0,)
    t_gen = time.perf_counter() - t_gen
    w = ws[0]
    tr = w.trace
    pol = (f"vLLM+ baseline (state per token block, full blocks only as in vLLM, LRU; blocks {args.blocks} x "
           f"caches {args.caps_gb} GB), " if args.policy == "vllm" else "")
    config = {"workload": f"config{args.config} {w.name}-shaped trace, {pol}{tr.n_requests} requests, "
                          f"{len(w.variants)} cache variant(s), {len(w.alphas)} alphas x {len(w.segments())} "
                          f"segments = {w.n_chains} chains" +
                          (f"; x {n_prob} independent problems (one per GPU, weak scaling)" if n_prob > 1 else "") +
                          (f"; one chain list sharded over {world} ranks (strong scaling)"
                           if args.scaling == "strong" and world > 1 else ""),
              "requests": tr.n_requests, "tokens": tr.n_tokens, "layout": args.layout, "alphas": len(w.alphas),
              "segments": len(w.segments()), "chains": w.n_chains * n_prob, "window": w.window,
              "problems": n_prob, "policy": args.policy,
              "model": "7B hybrid {4 attn, 24 ssm, 28 mlp}, D=4096, N=128, fp16" if args.config in (2, 3, 4)
              else "see tracegen.workload", "cache_bytes": [v.capacity_bytes for v in w.variants],
              "l2": "flushed (256 MiB write) between timed steps, outside the event window"}
    if args.impl == "reference":
        return reference_arm(args, w, config)

    import torch
    import torch.distributed as dist
    n_dev = torch.cuda.device_count()
    # one process per GPU; if fewer GPUs are visible than ranks (e.g. a 1-GPU box asked for
    # --gpus 2), ranks share devices round-robin and exchange over gloo (NCCL refuses two
    # ranks on one device) -- a runnable but not a scaling measurement, flagged in config
    shared = world > n_dev
    dev = local % max(1, n_dev)
    torch.cuda.set_device(dev)
    if world > 1:
        if shared:
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", dev))
    if shared:
        config["ranks_share_gpus"] = f"{world} ranks on {n_dev} visible GPU(s): exchange over gloo; not a scaling number"
    from paper_2411_19379_b200 import AlphaGrid
    from paper_2411_19379_b200.grid import gather_hit_sums

    # N problems (weak scaling): the chains of EVERY problem are LPT-sharded across all
    # ranks, so each rank replays ~one problem's worth of chains and the per-(problem, α)
    # hit sums must be all-gathered before any rank can pick α*.
    # NVTX ranges mark the phases (setup, replay, all-gather + α*, e2e) for an nsys timeline
    nvtx = torch.cuda.nvtx
    t_setup = time.perf_counter()
    nvtx.range_push("setup: trace H2D + live pass + snapshot images + shard")
    gs = []
    for k, wk in enumerate(ws):
        g = AlphaGrid(wk.trace, wk.variants, wk.alphas, wk.n_segments, rank=rank, world=world, device=dev)
        g.setup()
        gs.append(g)
    torch.cuda.synchronize()
    nvtx.range_pop()
    t_setup = time.perf_counter() - t_setup
    stream = torch.cuda.current_stream()
    streams = [torch.cuda.Stream() for _ in gs] if len(gs) > 1 else [stream]
    outs = [g.ctx.alloc_outputs(len(w.alphas), counters=True, chain_cycles=True) for g in gs]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    my_reqs = sum(int(sum(g.segs[c % len(g.segs)][1] for c in g.chains)) for g in gs)
    all_reqs = sum(sum(n for _, n, _ in g.segs) * len(w.alphas) * len(w.variants) for g in gs)

    def launch():
        nvtx.range_push("replay: alpha-grid chains")
        ev = torch.cuda.Event()
        ev.record(stream)
        ends = []
        for g, o, s in zip(gs, outs, streams):
            s.wait_event(ev)
            with torch.cuda.stream(s):
                o["hit_sum"].zero_()
                g.run(out=o, stream=s)
                e = torch.cuda.Event()
                e.record(s)
                ends.append(e)
        for e in ends:
            stream.wait_event(e)
        nvtx.range_pop()

    def select():
        nvtx.range_push("select: all-gather of hit sums + alpha*")
        hs = torch.stack([o["hit_sum"] for o in outs])          # [problem, variant, alpha]
        tot = gather_hit_sums(hs, world)                        # one all-gather over NCCL
        res = [g.select(o, gathered=tot[k]) for k, (g, o) in enumerate(zip(gs, outs))]
        nvtx.range_pop()
        return res

    if args.traffic_probe:  # child of traffic_probe(): one warm launch, then the launch ncu measures
        for _ in range(2):
            launch()
            torch.cuda.synchronize()
        return
    # warm-up: the first two replays run in the order of the live pass's per-segment cycles
    # (the first also pays the lazy module load; the second is reported as
    # run.first_replay_ms); their per-chain cycle counters then order the chains
    # longest-first for the rest (cost feedback) -- the order never changes
    # a result
    first_ms = None
    for i in range(args.warmup):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        launch()
        e1.record(stream)
        select()
        if i == min(1, args.warmup - 1):
            torch.cuda.synchronize()
            first_ms = e0.elapsed_time(e1)
            for g, o in zip(gs, outs):
                g.reorder_by_cycles(o["cycles"])
    for g in gs:
        g.ctx.check()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clocks = Clocks(dev)
    clocks.start()
    time.sleep(0.3)
    step_ms, kern_ms = [], []
    for _ in range(args.steps):
        flush.fill_(1)
        torch.cuda.synchronize()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e2 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        launch()                     # replay_kernel per problem, concurrently on their streams
        e1.record(stream)
        a_star = select()            # all-gather + D2H + argmax
        e2.record(stream)
        torch.cuda.synchronize()
        step_ms.append(e0.elapsed_time(e2))
        kern_ms.append(e0.elapsed_time(e1))
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    clk = clocks.stop()
    for g in gs:
        g.ctx.check()
    tot = torch.tensor([sum(step_ms), sum(kern_ms)], dtype=torch.float64, device="cpu" if shared else "cuda")
    if world > 1:
        dist.all_reduce(tot, op=dist.ReduceOp.MAX)   # max over ranks (device-timed per rank)
    T_ms, K_ms = float(tot[0]), float(tot[1])
    value = all_reqs * args.steps / (T_ms / 1000.0)

    # roofline of the dominant kernel (replay_kernel) from the device counters of this rank
    alg_bytes = 0
    for g, o in zip(gs, outs):
        ctr = o["counters"].cpu().numpy()[g.chains.astype(np.int64)]
        alg_bytes += algorithmic_bytes(ctr, int(sum(g.segs[c % len(g.segs)][1] for c in g.chains)))
    kern_avg_s = (sum(kern_ms) / len(kern_ms)) / 1000.0
    peak, peak_kind = peaks()
    achieved = alg_bytes / kern_avg_s / 1e9
    # d.3 split of the algorithmic bytes and per-request facts of the latency-bound kernel
    csum = sum(o["counters"].cpu().numpy()[g.chains.astype(np.int64)].astype(np.int64).sum(0)
               for g, o in zip(gs, outs))
    split = {"compare_8c": int(W_CMP * csum[0]), "visit_16v": int(W_VIS * csum[1]),
             "scan_13N": int(W_SCAN * csum[2]), "write_32w": int(W_WR * csum[3]), "outputs_16": int(W_OUT * my_reqs)}
    cyc = np.concatenate([o["cycles"].cpu().numpy()[g.chains.astype(np.int64)].astype(np.float64) * 1024 /
                          np.array([g.segs[c % len(g.segs)][1] for c in g.chains], np.float64)
                          for g, o in zip(gs, outs)])
    per_request = {"cycles_median": float(np.median(cyc)), "compared_positions": float(csum[0] / my_reqs),
                   "levels_visited": float(csum[1] / my_reqs), "nodes_scanned": float(csum[2] / my_reqs),
                   "records_written": float(csum[3] / my_reqs)}
    traffic, probe = (None, "skipped (--no-traffic)") if args.no_traffic else \
        ((None, "not run at N > 1 (ncu wraps one process)") if world > 1 else traffic_probe(args))

    # e2e through the public API with host buffers (this rank's shards of every problem)
    e2e = None
    if not args.no_e2e:
        nvtx.range_push("e2e: host-buffer pipeline")
        e2e = e2e_measure(gs, ws, args, outs, shared)
        nvtx.range_pop()

    # the paper's metrics at α* (this rank's chains), from the device sums
    met = gs[0].metrics(outs[0])
    hit_rate_at_star = [round(met.get((v, a_star[0][v]), (0.0, 0))[0], 6) for v in range(len(w.variants))]
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(w, args.cpu_seconds)

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": T_ms / args.steps,
            "ms_per_step_median": float(np.median(step_ms)), "higher_is_better": True,
            "scaling": args.scaling, "vs_baseline": None, "dtype": "u64+f64", "data": "synthetic",
            # config: the workload only, identical to the reference arm's; run-specific facts in "run"
            "config": config,
            "run": dict(parallelism=f"chains of every problem LPT-sharded over {world} GPU(s); one "
                                    f"{'gloo' if shared else 'NCCL'} all-gather of per-(problem, alpha) "
                                    f"hit sums per step",
                        alpha_star=[a[0] for a in a_star],
                        token_hit_rate_at_alpha_star=hit_rate_at_star if world == 1 else None,
                        schedule="persistent queue, chains longest-first: the first replay by the live pass's "
                                 "per-segment cycles, later ones by the previous replay's per-chain cycles",
                        first_replay_ms=first_ms,
                        setup_s={"trace_gen": round(t_gen, 2), "upload_live_pass_shard": round(t_setup, 2)}),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "kernel": "replay_kernel<%d>" % (args.policy == "vllm"), "alg_bytes_per_launch": alg_bytes,
                         "launch_ms": kern_avg_s * 1000.0, "d3_split": split,
                         "dram_gbs": (traffic / kern_avg_s / 1e9) if traffic else None,
                         "dram_frac": (traffic / kern_avg_s / 1e9 / peak) if traffic else None,
                         "traffic_probe": probe, "per_request": per_request,
                         "note": ("latency-bound: achieved/frac count SURVEY d.3 algorithmic bytes: the "
                                  f"{split['scan_13N'] / max(1, alg_bytes):.0%} scan term (13 B per live node per "
                                  "eviction) is served from shared memory, and of the "
                                  f"{split['compare_8c'] / max(1, alg_bytes):.0%} compare term (8 B per compared "
                                  "token position) the positions whose edge lies on the query's own trace range "
                                  "are skipped without loads; dram_frac is the measured DRAM traffic of the same "
                                  "launch" +
                                  ("; frac > 1.2 because those bytes never reach HBM, not because HBM is "
                                   "saturated" if achieved / peak > 1.2 else ""))},
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": args.steps * len(gs),  # one replay_kernel launch per problem per step
            "clocks": clk,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


def traffic_probe(args):
    """DRAM bytes of one replay launch of this workload, measured by ncu in a child process
    (`bench.py --traffic-probe`: setup, one warm launch, the measured launch).  Only the
    byte counters are taken from the profiled run, never a time.  Returns (bytes, how)."""
    metrics = "dram__bytes_read.sum,dram__bytes_write.sum"
    cmd = ["ncu", "--metrics", metrics, "--clock-control", "none", "-k", "regex:replay_kernel", "-s", "1", "-c", "1",
           "--csv", sys.executable, os.path.abspath(__file__), "--traffic-probe", "--config", str(args.config),
           "--policy", args.policy, "--blocks", args.blocks, "--caps-gb", args.caps_gb, "--layout", args.layout]
    if args.requests:
        cmd += ["--requests", str(args.requests)]
    try:
        r = subprocess.run(cmd, capture_output=True, text=True, timeout=600)
    except (OSError, subprocess.TimeoutExpired) as e:
        return None, f"ncu probe failed: {type(e).__name__}"
    import csv
    import io
    tot, seen = 0.0, set()
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "KB": 1e3, "MB": 1e6, "GB": 1e9}
    for row in csv.reader(io.StringIO(r.stdout)):
        if len(row) > 3 and row[-3] in metrics.split(","):
            try:
                tot += float(row[-1].replace(",", "")) * scale.get(row[-2], 1)
                seen.add(row[-3])
            except ValueError:
                pass
    if len(seen) != 2:
        return None, "ncu probe gave no DRAM counters (rc %d)" % r.returncode
    return tot, "ncu dram__bytes_read.sum + dram__bytes_write.sum of one replay_kernel launch (child process)"


def e2e_measure(gs, ws, args, outs, shared=False):
    """Same metric end to end through the public API from host buffers (grid.HostPipeline):
    per step and problem, H2D of the trace (tokens + requests, pinned) and of the packed
    segment snapshots, the device-side trace check, the snapshot images, the replay of this
    rank's chains, D2H of the per-request hits and the hit sums, α* on the host.  Two
    slots alternate, so step k+1's transfers run under step k's replay (wall clock over
    the steady state, the pipeline drained at the end)."""
    import torch
    from paper_2411_19379_b200 import marconi as M
    from paper_2411_19379_b200.grid import HostPipeline
    jobs = []
    for g, wk in zip(gs, ws):
        tr = wk.trace
        h_tok = torch.from_numpy(np.ascontiguousarray(tr.tokens, np.uint32).view(np.int32)).pin_memory()
        h_req = torch.from_numpy(M.requests_array(tr.off, tr.lin, tr.lout).view(np.int64)).pin_memory()
        snaps = []
        for v in range(len(wk.variants)):
            nodes, off, nid = g.ctx.pack_snapshots([g.ctx.get_snapshot(v, k) for k in range(g.ctx.snapshot_count(v))])
            pin = torch.empty(nodes.nbytes, dtype=torch.uint8).pin_memory()
            pnodes = pin.numpy().view(M.SNAP_DTYPE)
            pnodes[:] = nodes
            snaps.append((pnodes, off, nid, pin))
        jobs.append((HostPipeline(g), h_tok, h_req, [(a, b, c) for a, b, c, _ in snaps], snaps))
    h2d = sum(j[1].numel() * 4 + j[2].numel() * 8 + sum(a.nbytes + b.nbytes + c.nbytes for a, b, c in j[3])
              for j in jobs)
    d2h = sum(int(np.prod(o["hit"].shape)) * 4 + o["hit_sum"].numel() * 8 for o in outs)
    n_units = sum(sum(n for _, n, _ in g.segs) * len(wk.alphas) * len(wk.variants) for g, wk in zip(gs, ws))
    ref = [o["hit_sum"].cpu().numpy() for o in outs]

    def run(steps):
        pending = []
        for _ in range(steps):
            pending.append([p.submit(ht, hr, sn) for p, ht, hr, sn, _ in jobs])
            if len(pending) > 1:
                for (p, *_), t in zip(jobs, pending.pop(0)):
                    p.result(t)
        res = None
        for tick in pending:
            res = [p.result(t) for (p, *_), t in zip(jobs, tick)]
        return res

    run(2)
    steps = max(3, args.steps // 2)
    t0 = time.perf_counter()
    res = run(steps)
    dt = time.perf_counter() - t0
    # the pipelined result equals the kernel-only run's (same chains, same inputs)
    same = all(np.array_equal(r[1], h) for r, h in zip(res, ref))
    import torch.distributed as dist
    if dist.is_initialized():
        t = torch.tensor([dt], dtype=torch.float64, device="cpu" if shared else "cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        dt = float(t[0])
    return {"value": n_units * steps / dt, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
            "d2h_bytes_per_step": int(d2h), "steps": steps, "hit_sums_match_kernel_run": bool(same),
            "note": "wall clock over pipelined steps (2 slots: step k+1's H2D of trace+requests+packed segment "
                    "snapshots, device trace check and snapshot images run under step k's replay), incl. D2H of "
                    "per-request hits and hit sums and alpha* on the host"}


if __name__ == "__main__":
    main()
