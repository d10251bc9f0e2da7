"""ctypes binding of libmarconi.so (include/marconi.h) -- argument marshalling only.

Every step of the replay runs in the CUDA kernels behind the C ABI; this module
only converts Python/numpy/torch arguments into pointers and checks statuses.
There is no CPU fallback: if the extension is missing or no CUDA device is
present the calls raise.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Optional, Sequence

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MARCONI_LIB") or os.path.join(HERE, "libmarconi.so")

# ---- struct layouts (must match include/marconi.h) ----
REQUEST_DTYPE = np.dtype([("tok_off", "<u8"), ("input_len", "<u4"), ("output_len", "<u4")])
SNAP_DTYPE = np.dtype([("id", "<u4"), ("parent_id", "<u4"), ("ref_off", "<u8"), ("d_start", "<u4"),
                       ("d_end", "<u4"), ("t_last", "<u4"), ("has_ssm", "<u4")], align=True)
SEGMENT_DTYPE = np.dtype([("first_req", "<u4"), ("n_req", "<u4"), ("snapshot", "<u4"), ("reserved", "<u4")])
EVICT_DTYPE = np.dtype([("req", "<u4"), ("node_id", "<u4"), ("kind", "<u4"), ("n_live", "<u4"),
                        ("utility", "<f8")], align=True)
QUERY_DTYPE = np.dtype([("req", "<u4"), ("variant", "<u4"), ("snapshot", "<u4"), ("reserved", "<u4")])
LOOKUP_DTYPE = np.dtype([("reuse", "<u4"), ("m", "<u4"), ("p", "<u4"), ("hit_id", "<u4"), ("div_id", "<u4"),
                         ("div_off", "<u4"), ("path_len", "<u4"), ("d_nodes", "<u4"), ("d_bytes", "<u8")])
assert REQUEST_DTYPE.itemsize == 16 and SNAP_DTYPE.itemsize == 32 and EVICT_DTYPE.itemsize == 24
assert QUERY_DTYPE.itemsize == 16 and LOOKUP_DTYPE.itemsize == 40

EXPORTED = ("mc_create", "mc_destroy", "mc_set_trace", "mc_set_trace_async", "mc_set_snapshots", "mc_live_pass", "mc_live_pass_at", "mc_live_pass_bootstrap",
            "mc_snapshot_count", "mc_live_window_cycles",
            "mc_get_snapshot", "mc_set_segments", "mc_workspace_size", "mc_workspace_workers", "mc_replay",
            "mc_check", "mc_last_error", "mc_node_cost", "mc_score_argmin", "mc_eviction_log", "mc_lookup", "mc_chain_sums")

MC_STATUS = {0: "MC_OK", -1: "MC_EINVAL", -2: "MC_ENOMEM", -3: "MC_ECUDA", -4: "MC_EOVERFLOW",
             -5: "MC_ESTATE", -6: "MC_EDEVICE"}


class mc_model(C.Structure):
    _fields_ = [(n, C.c_uint32) for n in ("n_attn", "n_ssm", "n_mlp", "d_model", "d_state",
                                          "bytes_per_param", "conv_in", "conv_kernel")]


class mc_variant(C.Structure):
    _fields_ = [("model", mc_model), ("capacity_bytes", C.c_uint64), ("capacity_nodes", C.c_uint32),
                ("chunk_size", C.c_uint32), ("block_size", C.c_uint32), ("reserved", C.c_uint32)]


class mc_replay_args(C.Structure):
    _fields_ = [("h_alphas", C.c_void_p), ("n_alpha", C.c_uint32), ("h_chains", C.c_void_p),
                ("n_chains", C.c_uint32), ("d_workspace", C.c_void_p), ("workspace_bytes", C.c_uint64),
                ("d_hit", C.c_void_p), ("d_flops", C.c_void_p), ("d_bypass", C.c_void_p),
                ("d_hit_sum", C.c_void_p), ("d_counters", C.c_void_p), ("d_log", C.c_void_p),
                ("log_cap", C.c_uint32), ("d_log_n", C.c_void_p), ("d_chain_ns", C.c_void_p),
                ("n_workers", C.c_uint32), ("smem_nodes", C.c_uint32)]


class MarconiError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"{MC_STATUS.get(status, status)}: {msg}")
        self.status = status


_LIB = None


def lib():
    """Load the in-tree extension.  Raises loudly if it was not built."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise ImportError(f"{LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = C.CDLL(LIB_PATH)
        P, U32, U64, I = C.c_void_p, C.c_uint32, C.c_uint64, C.c_int
        L.mc_last_error.restype = C.c_char_p
        for name, args in {
            "mc_create": [P, U32, U32, I, P],
            "mc_set_trace": [P, P, U64, P, U32],
            "mc_set_trace_async": [P, P, U64, P, U32, P],
            "mc_set_snapshots": [P, U32, P, P, P, U32, P],
            "mc_live_pass": [P, U32, P, U64, P, P, P, P],
            "mc_live_pass_at": [P, P, U32, P, U64, P, P, P, P, P],
            "mc_live_pass_bootstrap": [P, U32, P, U64, P, P, P, P, P],
            "mc_snapshot_count": [P, U32, P],
            "mc_live_window_cycles": [P, U32, P, U32, P],
            "mc_get_snapshot": [P, U32, U32, P, U64, P, P],
            "mc_set_segments": [P, P, U32],
            "mc_workspace_size": [P, U32, U32, U32, P],
            "mc_workspace_workers": [P, U64, U32, U32, P],
            "mc_replay": [P, P, P],
            "mc_check": [P, P],
            "mc_lookup": [P, P, U32, P, U64, P, P],
            "mc_chain_sums": [P, U32, P, P, P, U32, P, P],
            "mc_eviction_log": [P, P, U32, U32, U32, P, U64, P, P],
            "mc_node_cost": [P, U32, P, P, P, P, P, P, P],
            "mc_score_argmin": [U32, P, P, P, P, P, P, P, P, P],
        }.items():
            f = getattr(L, name)
            f.argtypes = args
            f.restype = C.c_int
        L.mc_destroy.argtypes = [P]
        L.mc_destroy.restype = None
        _LIB = L
    return _LIB


def check(rc: int):
    if rc != 0:
        raise MarconiError(rc, lib().mc_last_error().decode())


def _np_ptr(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _tptr(t) -> Optional[int]:
    """Raw device pointer of a torch tensor (or None)."""
    if t is None:
        return None
    assert t.is_cuda and t.is_contiguous(), "device tensors must be contiguous CUDA tensors"
    return C.c_void_p(t.data_ptr())


def _stream_ptr(stream) -> C.c_void_p:
    import torch
    s = stream if stream is not None else torch.cuda.current_stream()
    return C.c_void_p(s.cuda_stream)


def make_variant(model, capacity_bytes: int, capacity_nodes: int = 0, chunk_size: int = 0,
                 block_size: int = 0) -> mc_variant:
    """block_size > 0 selects the vLLM+ baseline (token blocks of that size, NEXT-2)."""
    return mc_variant(mc_model(*model.astuple()), int(capacity_bytes), int(capacity_nodes), int(chunk_size),
                      int(block_size), 0)


def requests_array(off, lin, lout) -> np.ndarray:
    r = np.zeros(len(off), REQUEST_DTYPE)
    r["tok_off"] = off
    r["input_len"] = lin
    r["output_len"] = lout
    return r


# --------------------------------------------------------------------------
# Context: owns an mc_ctx; device memory comes from torch.
# --------------------------------------------------------------------------
class Context:
    """One replay context (C ABI mc_ctx) on a CUDA device.

    variants: sequence of objects with .model (n_attn..conv_kernel via astuple()),
    .capacity_bytes, .capacity_nodes.
    """

    def __init__(self, variants: Sequence, max_nodes: int = 8192, device: int = 0):
        import torch
        self.torch = torch
        self.device = torch.device("cuda", device)
        self.variants = list(variants)
        arr = (mc_variant * len(self.variants))(*[make_variant(v.model, v.capacity_bytes, v.capacity_nodes,
                                                                getattr(v, "chunk_size", 0),
                                                                getattr(v, "block_size", 0))
                                                   for v in self.variants])
        h = C.c_void_p()
        check(lib().mc_create(arr, len(self.variants), int(max_nodes), int(device), C.byref(h)))
        self.h = h
        self.max_nodes = max_nodes
        self._keep = []
        self.n_req = 0
        self.segments = None

    def close(self):
        if getattr(self, "h", None):
            lib().mc_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ---- trace ----
    def set_trace_device(self, d_tokens, d_reqs, n_reqs: int):
        """d_tokens: int32/uint32 CUDA tensor; d_reqs: CUDA tensor holding REQUEST_DTYPE records."""
        self._keep = [d_tokens, d_reqs]
        check(lib().mc_set_trace(self.h, _tptr(d_tokens), d_tokens.numel(), _tptr(d_reqs), int(n_reqs)))
        self.n_req = int(n_reqs)

    def set_trace_async(self, d_tokens, d_reqs, n_reqs: int, stream=None):
        """As set_trace_device, validated by a device kernel on `stream` (errors at check())."""
        self._keep = [d_tokens, d_reqs]
        check(lib().mc_set_trace_async(self.h, _tptr(d_tokens), d_tokens.numel(), _tptr(d_reqs), int(n_reqs),
                                       _stream_ptr(stream)))
        self.n_req = int(n_reqs)

    def upload_trace(self, tokens: np.ndarray, off, lin, lout, stream=None):
        """Copy a host trace to device tensors (synchronously) and borrow them."""
        torch = self.torch
        t = torch.from_numpy(np.ascontiguousarray(tokens, np.uint32).view(np.int32)).to(self.device)
        r = requests_array(off, lin, lout)
        d_r = torch.from_numpy(r.view(np.int64)).to(self.device)
        torch.cuda.synchronize(self.device)
        self.set_trace_device(t, d_r, len(off))
        return t, d_r

    # ---- snapshots ----
    @staticmethod
    def pack_snapshots(snapshots):
        """list of (nodes, next_id) -> (nodes SNAP_DTYPE[total], offsets u64[k+1], next_id u32[k])."""
        nodes = np.concatenate([np.asarray(s[0]).astype(SNAP_DTYPE) for s in snapshots]) \
            if snapshots else np.zeros(0, SNAP_DTYPE)
        nodes = np.ascontiguousarray(nodes, SNAP_DTYPE)
        off = np.zeros(len(snapshots) + 1, np.uint64)
        off[1:] = np.cumsum([len(s[0]) for s in snapshots])
        nid = np.asarray([s[1] for s in snapshots], np.uint32)
        return nodes, off, nid

    def set_snapshots(self, variant: int, snapshots, stream=None):
        """snapshots: list of (nodes structured array with SNAP_DTYPE fields, next_id)."""
        self.set_snapshots_packed(variant, *self.pack_snapshots(snapshots), stream=stream)

    def set_snapshots_packed(self, variant: int, nodes, off, nid, stream=None):
        """Packed host arrays (see pack_snapshots; nodes may live in pinned memory)."""
        assert nodes.dtype == SNAP_DTYPE and nodes.flags.c_contiguous
        off = np.ascontiguousarray(off, np.uint64)
        nid = np.ascontiguousarray(nid, np.uint32)
        check(lib().mc_set_snapshots(self.h, variant, _np_ptr(nodes), _np_ptr(off), _np_ptr(nid),
                                     len(nid), _stream_ptr(stream)))

    def snapshot_count(self, variant: int) -> int:
        n = C.c_uint32()
        check(lib().mc_snapshot_count(self.h, variant, C.byref(n)))
        return n.value

    def live_window_cycles(self, variant: int) -> np.ndarray:
        """Cycles the last live pass spent per window between its snapshot points (u64)."""
        n = C.c_uint32()
        check(lib().mc_live_window_cycles(self.h, variant, None, 0, C.byref(n)))
        out = np.zeros(n.value, np.uint64)
        check(lib().mc_live_window_cycles(self.h, variant, _np_ptr(out), n.value, C.byref(n)))
        return out

    def get_snapshot(self, variant: int, k: int):
        n = C.c_uint64()
        nid = C.c_uint32()
        check(lib().mc_get_snapshot(self.h, variant, k, None, 0, C.byref(n), C.byref(nid)))
        out = np.zeros(n.value, SNAP_DTYPE)
        check(lib().mc_get_snapshot(self.h, variant, k, _np_ptr(out), out.shape[0], C.byref(n), C.byref(nid)))
        return out, nid.value

    # ---- workspace ----
    def workspace_size(self, n_workers: int = 0, n_alpha: int = 1, n_chains: int = 0) -> int:
        b = C.c_uint64()
        check(lib().mc_workspace_size(self.h, n_workers, n_alpha, n_chains, C.byref(b)))
        return b.value

    def alloc_workspace(self, n_workers: int = 0, n_alpha: int = 1, n_chains: int = 0):
        nbytes = self.workspace_size(n_workers, n_alpha, n_chains)
        # zero-initialised once (include/marconi.h: child-index generation tags start at 0)
        return self.torch.zeros(nbytes, dtype=self.torch.uint8, device=self.device)

    # ---- live pass ----
    def live_pass(self, window: int, workspace=None, stream=None):
        """α = 0 live pass on the device; snapshots stay in the context.  Returns
        (hit int32[n_var, R], flops int64[n_var, R], bypass uint8[n_var, R]) device tensors."""
        torch = self.torch
        nv = len(self.variants)
        ws = workspace if workspace is not None else self.alloc_workspace(n_workers=nv)
        hit = torch.zeros((nv, self.n_req), dtype=torch.int32, device=self.device)
        fl = torch.zeros((nv, self.n_req), dtype=torch.int64, device=self.device)
        by = torch.zeros((nv, self.n_req), dtype=torch.uint8, device=self.device)
        check(lib().mc_live_pass(self.h, int(window), _tptr(ws), ws.numel(), _tptr(hit), _tptr(fl), _tptr(by),
                                 _stream_ptr(stream)))
        self.check(stream)
        return hit, fl, by

    def live_pass_at(self, points, workspace=None, stream=None):
        """α = 0 live pass with snapshot k = tree after request points[k] (points[0] = 0).
        Returns (hit, flops, bypass device tensors [n_var, R], first_evict list per variant)."""
        torch = self.torch
        nv = len(self.variants)
        ws = workspace if workspace is not None else self.alloc_workspace(n_workers=nv)
        hit = torch.zeros((nv, self.n_req), dtype=torch.int32, device=self.device)
        fl = torch.zeros((nv, self.n_req), dtype=torch.int64, device=self.device)
        by = torch.zeros((nv, self.n_req), dtype=torch.uint8, device=self.device)
        pts = np.ascontiguousarray(points, np.uint32)
        fe = np.zeros(nv, np.uint32)
        check(lib().mc_live_pass_at(self.h, _np_ptr(pts), len(pts), _tptr(ws), ws.numel(), _tptr(hit), _tptr(fl),
                                    _tptr(by), _np_ptr(fe), _stream_ptr(stream)))
        self.check(stream)
        return hit, fl, by, [int(x) for x in fe]

    def live_pass_bootstrap(self, multiplier: int = 10, workspace=None, stream=None):
        """One α = 0 live pass that also takes the paper's tuning snapshots:
        snapshot 1 after the first evicting request r_F, 2 after r_F + multiplier*r_F.
        Returns (hit, flops, bypass device tensors [n_var, R], r_F list per variant)."""
        torch = self.torch
        nv = len(self.variants)
        ws = workspace if workspace is not None else self.alloc_workspace(n_workers=nv)
        hit = torch.zeros((nv, self.n_req), dtype=torch.int32, device=self.device)
        fl = torch.zeros((nv, self.n_req), dtype=torch.int64, device=self.device)
        by = torch.zeros((nv, self.n_req), dtype=torch.uint8, device=self.device)
        fe = np.zeros(nv, np.uint32)
        check(lib().mc_live_pass_bootstrap(self.h, int(multiplier), _tptr(ws), ws.numel(), _tptr(hit), _tptr(fl),
                                           _tptr(by), _np_ptr(fe), _stream_ptr(stream)))
        self.check(stream)
        return hit, fl, by, [int(x) for x in fe]

    # ---- segments ----
    def set_segments(self, segs):
        """segs: list of (first_req, n_req, snapshot_idx)."""
        a = np.zeros(len(segs), SEGMENT_DTYPE)
        for i, (f, n, k) in enumerate(segs):
            a[i] = (f, n, k, 0)
        check(lib().mc_set_segments(self.h, _np_ptr(a), len(segs)))
        self.segments = list(segs)

    # ---- replay ----
    def replay(self, alphas, chains=None, workspace=None, out=None, log_cap: int = 0, counters: bool = False,
               chain_cycles: bool = False, n_workers: int = 0, smem_nodes: int = 0, stream=None):
        """Launch the α-grid replay (asynchronous).  Returns a dict of device tensors:
        hit int32[n_var, n_alpha, R], flops int64[...], bypass uint8[...], hit_sum int64[n_var, n_alpha]
        (+ counters int64[n_chains_total, 4], log, log_n, cycles when requested)."""
        torch = self.torch
        nv, na, ns = len(self.variants), len(alphas), len(self.segments)
        total = nv * na * ns
        if out is None:
            out = self.alloc_outputs(na, log_cap, counters, chain_cycles)
        alph = np.ascontiguousarray(alphas, np.float64)
        ch = None if chains is None else np.ascontiguousarray(chains, np.uint32)
        ws = workspace if workspace is not None else self.alloc_workspace(
            n_workers, na, 0 if ch is None else len(ch))
        args = mc_replay_args()
        args.h_alphas = _np_ptr(alph)
        args.n_alpha = na
        args.h_chains = None if ch is None else _np_ptr(ch)
        args.n_chains = 0 if ch is None else len(ch)
        args.d_workspace = ws.data_ptr()
        args.workspace_bytes = ws.numel()
        args.d_hit = out["hit"].data_ptr()
        args.d_flops = out["flops"].data_ptr()
        args.d_bypass = out["bypass"].data_ptr()
        args.d_hit_sum = out["hit_sum"].data_ptr()
        args.d_counters = out["counters"].data_ptr() if out.get("counters") is not None else None
        args.d_log = out["log"].data_ptr() if out.get("log") is not None else None
        args.log_cap = out.get("log_cap", 0)
        args.d_log_n = out["log_n"].data_ptr() if out.get("log_n") is not None else None
        args.d_chain_ns = out["cycles"].data_ptr() if out.get("cycles") is not None else None
        args.n_workers = n_workers
        args.smem_nodes = smem_nodes
        self._last_args = (alph, ch, ws, args)
        check(lib().mc_replay(self.h, C.byref(args), _stream_ptr(stream)))
        return out

    def lookup(self, req, variant=0, snapshot=0, workspace=None, stream=None):
        """Batched read-only lookup (mc_lookup) of requests `req` (1-based, array) against
        snapshot `snapshot` of `variant` (scalars or arrays).  Returns a device uint8 tensor
        viewable as LOOKUP_DTYPE records (see lookup_records)."""
        torch = self.torch
        req = np.atleast_1d(np.asarray(req, np.uint32))
        q = np.zeros(req.shape[0], QUERY_DTYPE)
        q["req"] = req
        q["variant"] = variant
        q["snapshot"] = snapshot
        n = q.shape[0]
        n_groups = len(set(zip(q["variant"].tolist(), q["snapshot"].tolist())))
        if workspace is None:
            workspace = self.alloc_workspace(min(n_groups, 4 * 148), 1, 0)
            workspace = torch.cat([workspace, torch.zeros(64 * n + 4096, dtype=torch.uint8, device=self.device)])
        out = torch.zeros(n * LOOKUP_DTYPE.itemsize, dtype=torch.uint8, device=self.device)
        check(lib().mc_lookup(self.h, _np_ptr(q), n, _tptr(workspace), workspace.numel(), _tptr(out),
                              _stream_ptr(stream)))
        self._last_lookup = (q, workspace)
        return out

    def chain_sums(self, out, n_alpha: int, chains, stream=None):
        """Per chain (device replay outputs, mc_chain_sums): list of (Σ hit, Σ input tokens,
        Σ FLOPs saved as an exact Python int)."""
        torch = self.torch
        ch = torch.from_numpy(np.ascontiguousarray(chains, np.uint32).view(np.int32)).to(self.device)
        res = torch.zeros((ch.numel(), 4), dtype=torch.int64, device=self.device)
        check(lib().mc_chain_sums(self.h, n_alpha, _tptr(out["hit"]), _tptr(out["flops"]), _tptr(ch), ch.numel(),
                                  _tptr(res), _stream_ptr(stream)))
        r = res.cpu().numpy().view(np.uint64)
        return [(int(a), int(b), int(c) | (int(d) << 64)) for a, b, c, d in r]

    @staticmethod
    def lookup_records(out) -> np.ndarray:
        return out.cpu().numpy().view(LOOKUP_DTYPE).copy()

    def alloc_outputs(self, n_alpha: int, log_cap: int = 0, counters: bool = False, chain_cycles: bool = False):
        torch = self.torch
        nv, ns = len(self.variants), len(self.segments)
        total = nv * n_alpha * ns
        d = self.device
        out = {
            "hit": torch.zeros((nv, n_alpha, self.n_req), dtype=torch.int32, device=d),
            "flops": torch.zeros((nv, n_alpha, self.n_req), dtype=torch.int64, device=d),
            "bypass": torch.zeros((nv, n_alpha, self.n_req), dtype=torch.uint8, device=d),
            "hit_sum": torch.zeros((nv, n_alpha), dtype=torch.int64, device=d),
            "counters": torch.zeros((total, 4), dtype=torch.int64, device=d) if counters else None,
            "log": torch.zeros((total, max(log_cap, 1) * EVICT_DTYPE.itemsize), dtype=torch.uint8, device=d)
            if log_cap else None,
            "log_n": torch.zeros(total, dtype=torch.int32, device=d) if log_cap else None,
            "log_cap": int(log_cap),
            "cycles": torch.zeros(total, dtype=torch.int32, device=d) if chain_cycles else None,
        }
        return out

    def check(self, stream=None):
        check(lib().mc_check(self.h, _stream_ptr(stream)))

    def eviction_log(self, out, n_alpha: int, variant: int, alpha_idx: int, seg: int, stream=None):
        """One chain's eviction log through the C ABI (mc_eviction_log): (records, n_evictions)."""
        a = mc_replay_args()
        a.n_alpha = n_alpha
        a.d_log = out["log"].data_ptr()
        a.d_log_n = out["log_n"].data_ptr()
        a.log_cap = out["log_cap"]
        n = C.c_uint64()
        check(lib().mc_eviction_log(self.h, C.byref(a), variant, alpha_idx, seg, None, 0, C.byref(n),
                                    _stream_ptr(stream)))
        k = min(n.value, out["log_cap"])
        rec = np.zeros(k, EVICT_DTYPE)
        check(lib().mc_eviction_log(self.h, C.byref(a), variant, alpha_idx, seg, _np_ptr(rec), k, C.byref(n),
                                    _stream_ptr(stream)))
        return rec, n.value

    @staticmethod
    def read_log(out, chain: int) -> np.ndarray:
        n = int(out["log_n"][chain].item())
        cap = out["log_cap"]
        raw = out["log"][chain].cpu().numpy()
        recs = raw.view(EVICT_DTYPE)
        return recs[:min(n, cap)].copy(), n


# --------------------------------------------------------------------------
# Unit-level kernels (K1, K3)
# --------------------------------------------------------------------------
def node_cost(model, d_start, d_end, has_ssm, stream=None):
    """Batched K1 on device tensors (int32 d_start/d_end, uint8 has_ssm) -> (saved, bytes, eff)."""
    import torch
    n = d_start.numel()
    saved = torch.empty(n, dtype=torch.int64, device=d_start.device)
    by = torch.empty(n, dtype=torch.int64, device=d_start.device)
    eff = torch.empty(n, dtype=torch.float64, device=d_start.device)
    mm = mc_model(*model.astuple())
    check(lib().mc_node_cost(C.byref(mm), n, _tptr(d_start), _tptr(d_end), _tptr(has_ssm), _tptr(saved),
                             _tptr(by), _tptr(eff), _stream_ptr(stream)))
    return saved, by, eff


def score_argmin(off, t, cand, ids, eff, alpha, stream=None):
    """Segmented K3 on device tensors -> (best row per table int32 (-1 = none), utility f64)."""
    import torch
    nt = off.numel() - 1
    best = torch.empty(nt, dtype=torch.int32, device=off.device)
    u = torch.empty(nt, dtype=torch.float64, device=off.device)
    check(lib().mc_score_argmin(nt, _tptr(off), _tptr(t), _tptr(cand), _tptr(ids), _tptr(eff), _tptr(alpha),
                                _tptr(best), _tptr(u), _stream_ptr(stream)))
    return best, u
