// replay.cuh -- device code of the Marconi α-grid replay (sm_100a).
//
// One WARP owns one chain (variant, α, segment): a private flattened radix
// tree in a global-memory workspace slice, replayed request by request.
// Warp-cooperative stages:
//   K2 walk      -- child lookup = 32-wide linear-probe window of an
//                   open-addressing hash keyed by (parent slot, first token);
//                   edge compare = 128 tokens per step, coalesced loads +
//                   __ballot_sync/__ffs for the first mismatch (PAPER:246,
//                   PAPER:300-301; speculative insertion PAPER:365 fused in);
//   K3 scan      -- one pass over the dense live-node list for the min/max
//                   normalisation bounds, one pass for the lexicographic
//                   (u, t_last, id) argmin of Eq. 2, both
//                   reduced with warp shuffles;
//   snapshot load / dump -- 32 nodes per step.
// Scalar tree mutations (K4: split, leaf, gain, leaf removal, absorption --
// PAPER:362-365) run on lane 0 with the chain's scalar state
// broadcast afterwards.  K1 (Eq. 1 cost model, Appendix A) is inlined at
// every node create/split/merge/gain.
//
// Bit-exactness: integer FLOPs/bytes are exact u64; eff = one IEEE division;
// the utility uses __dsub_rn/__ddiv_rn/__dmul_rn/__dadd_rn (no FMA).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "marconi.h"

namespace mcd {

constexpr uint32_t NIL = 0xFFFFFFFFu;
constexpr unsigned long long EMPTY = ~0ull;
constexpr uint32_t NOTC = 0x80000000u;  // dense record: not an eviction candidate
constexpr uint32_t F_SSM = 1u, F_PIN = 2u;
constexpr unsigned FULL = 0xFFFFFFFFu;

// device status word bits (mc_check)
enum : uint32_t {
  ST_OVERFLOW = 1u,   // node table full
  ST_INVARIANT = 2u,  // capacity exceeded after admission / hit > input / bad snapshot
  ST_NOCAND = 4u,     // eviction needed but no candidate (cannot happen after the precheck)
  ST_SNAPOVF = 8u,    // snapshot store too small
};

// Cost model constants (Appendix A tab:flops_breakdown PAPER:771-772),
// computed exactly on the host: F(L) = fa*L + fb*L^2 over all layers.
struct DevModel {
  uint64_t fa, fb;  // fa = 8 nA D^2 + nS (12 D^2 + 16 D N + 10) + 16 nM D^2 ; fb = 4 nA D
  uint64_t kvt;     // KV bytes per token over all attention layers = nA * 2 * D * bpp
  uint64_t ssmb;    // one checkpoint = nS * (D*N + conv_in*conv_k) * bpp
  uint32_t n_ssm, pad;
};
struct DevVariant {
  DevModel m;
  uint64_t cap_bytes;
  uint32_t cap_nodes, pad;
};
struct DevSnapStore {
  const mc_snap_node* nodes;
  const uint32_t* pidx;  // parent position within the same snapshot, NIL = root
  const uint64_t* off;
  const uint32_t* n;
  const uint32_t* nid;
  uint32_t count, pad;
};
// Writable view used by the live pass.
struct DevSnapOut {
  mc_snap_node* nodes;
  uint32_t* pidx;
  uint64_t* off;
  uint32_t* n;
  uint32_t* nid;
  uint64_t stride;  // records per snapshot slot
  uint32_t count, pad;
};

struct __align__(16) DenseRec {
  uint32_t tc;  // t_last | NOTC
  uint32_t id;
  double eff;
};

struct KParams {
  const uint32_t* tok;
  uint64_t n_tok;
  const mc_request* req;
  uint32_t n_req, n_var;
  const DevVariant* var;
  const DevSnapStore* snap;
  const mc_segment* segs;
  uint32_t n_segs, n_alpha;
  const double* alphas;
  const uint32_t* chains;
  uint32_t n_chains, ncap, hcap, n_workers;
  unsigned* queue;
  char* ws;
  uint64_t ws_stride;
  uint32_t* hit;
  unsigned long long* flops;
  uint8_t* bypass;
  unsigned long long* hit_sum;
  unsigned long long* counters;
  mc_evict_rec* log;
  uint32_t log_cap;
  uint32_t* log_n;
  uint32_t* chain_cycles;
  uint32_t* status;
  // live pass
  DevSnapOut* live_out;
  uint32_t window;
};

// Per-worker workspace slice (SoA node table + dense live list + hash).  Only the
// base pointer and sizes live in registers; array addresses are recomputed.
__host__ __device__ inline uint64_t ws_bytes_per_worker(uint32_t ncap, uint32_t hcap) {
  uint64_t b = 14ull * 4 * ncap  // 13 u32 node arrays (+1 spare)
               + 8ull * ncap     // roff
               + 16ull * ncap    // dense
               + 12ull * hcap;   // hkey + hval
  return (b + 255) & ~255ull;
}

struct WS {
  char* b;
  uint32_t n, h;
  __device__ __forceinline__ DenseRec* dense() const { return (DenseRec*)b; }
  __device__ __forceinline__ uint64_t* roff() const { return (uint64_t*)(b + 16ull * n); }
  __device__ __forceinline__ unsigned long long* hkey() const { return (unsigned long long*)(b + 24ull * n); }
  __device__ __forceinline__ uint32_t* a32(uint32_t k) const { return (uint32_t*)(b + 24ull * n + 8ull * h + 4ull * k * n); }
  __device__ __forceinline__ uint32_t* id() const { return a32(0); }
  __device__ __forceinline__ uint32_t* parent() const { return a32(1); }
  __device__ __forceinline__ uint32_t* ds() const { return a32(2); }
  __device__ __forceinline__ uint32_t* de() const { return a32(3); }
  __device__ __forceinline__ uint32_t* t() const { return a32(4); }
  __device__ __forceinline__ uint32_t* nchild() const { return a32(5); }
  __device__ __forceinline__ uint32_t* cxor() const { return a32(6); }
  __device__ __forceinline__ uint32_t* ftok() const { return a32(7); }
  __device__ __forceinline__ uint32_t* flags() const { return a32(8); }
  __device__ __forceinline__ uint32_t* dpos() const { return a32(9); }
  __device__ __forceinline__ uint32_t* dslot() const { return a32(10); }
  __device__ __forceinline__ uint32_t* path() const { return a32(11); }
  __device__ __forceinline__ uint32_t* freel() const { return a32(12); }
  __device__ __forceinline__ uint32_t* hval() const { return (uint32_t*)(b + 24ull * n + 8ull * h + 52ull * n); }
};

__device__ inline WS ws_slice(char* base, uint32_t ncap, uint32_t hcap) {
  WS w;
  w.b = base;
  w.n = ncap;
  w.h = hcap;
  return w;
}

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }

// ---------------------------------------------------------------------------
// K1: cost model (Eq. 1 with Appendix A), bit-exact with the host definition.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t prefill_F(const DevModel& m, uint64_t L) {
  return m.fa * L + m.fb * L * L;
}
__device__ __forceinline__ uint64_t node_bytes(const DevModel& m, uint32_t ds, uint32_t de, bool ssm) {
  return m.kvt * (uint64_t)(de - ds) + (ssm ? m.ssmb : 0ull);
}
__device__ __forceinline__ double node_eff(const DevModel& m, uint32_t ds, uint32_t de, bool ssm) {
  uint64_t saved = prefill_F(m, de) - prefill_F(m, ds);  // relative to the parent
  return __ddiv_rn((double)saved, (double)node_bytes(m, ds, de, ssm));
}

// ---------------------------------------------------------------------------
// K3 helpers: normalisation bounds and lexicographic argmin (Eq. 2).
// ---------------------------------------------------------------------------
struct Bounds {
  uint32_t tmin, tmax;
  double emin, emax;
};
__device__ __forceinline__ void bounds_init(Bounds& b) {
  b.tmin = 0xFFFFFFFFu;
  b.tmax = 0;
  b.emin = __longlong_as_double(0x7FF0000000000000ll);   // +inf
  b.emax = __longlong_as_double((long long)0xFFF0000000000000ull);  // -inf
}
__device__ __forceinline__ void bounds_add(Bounds& b, uint32_t t, double e) {
  b.tmin = min(b.tmin, t);
  b.tmax = max(b.tmax, t);
  b.emin = fmin(b.emin, e);
  b.emax = fmax(b.emax, e);
}
__device__ __forceinline__ void bounds_reduce(Bounds& b) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    b.tmin = min(b.tmin, __shfl_xor_sync(FULL, b.tmin, o));
    b.tmax = max(b.tmax, __shfl_xor_sync(FULL, b.tmax, o));
    b.emin = fmin(b.emin, __shfl_xor_sync(FULL, b.emin, o));
    b.emax = fmax(b.emax, __shfl_xor_sync(FULL, b.emax, o));
  }
}
// u = rec + α·effn, each operation rounded (no FMA); degenerate range -> 0.5 (R2).
__device__ __forceinline__ double utility(const Bounds& b, uint32_t t, double e, double alpha) {
  double rec = (b.tmax == b.tmin) ? 0.5 : __ddiv_rn((double)(t - b.tmin), (double)(b.tmax - b.tmin));
  double effn = (b.emax == b.emin) ? 0.5 : __ddiv_rn(__dsub_rn(e, b.emin), __dsub_rn(b.emax, b.emin));
  return __dadd_rn(rec, __dmul_rn(alpha, effn));
}
struct Best {
  double u;
  uint32_t t, id, i;
};
__device__ __forceinline__ bool better(double u, uint32_t t, uint32_t id, const Best& b) {
  return u < b.u || (u == b.u && (t < b.t || (t == b.t && id < b.id)));
}
__device__ __forceinline__ void best_init(Best& b) {
  b.u = __longlong_as_double(0x7FF0000000000000ll);
  b.t = 0xFFFFFFFFu;
  b.id = 0xFFFFFFFFu;
  b.i = NIL;
}
__device__ __forceinline__ void best_reduce(Best& b) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    double u = __shfl_xor_sync(FULL, b.u, o);
    uint32_t t = __shfl_xor_sync(FULL, b.t, o);
    uint32_t id = __shfl_xor_sync(FULL, b.id, o);
    uint32_t i = __shfl_xor_sync(FULL, b.i, o);
    if (i != NIL && (b.i == NIL || better(u, t, id, b))) {
      b.u = u; b.t = t; b.id = id; b.i = i;
    }
  }
}

// ---------------------------------------------------------------------------
// Chain state (per warp; scalars are warp-uniform, lane 0 is the writer)
// ---------------------------------------------------------------------------
struct Chain {
  WS w;
  uint32_t ncap, hmask;
  uint32_t count;     // live non-root nodes (= dense list length)
  uint64_t total;     // bytes of all live nodes
  uint32_t next_id, hwm, nfree;
  DevModel m;
  uint64_t capb;
  uint32_t capn;
  double alpha;
  uint64_t c_cmp, c_vis, c_scan, c_wr;
  bool failed;
};

__device__ __forceinline__ void sync_state(Chain& C) {
  __syncwarp();
  C.count = __shfl_sync(FULL, C.count, 0);
  C.total = __shfl_sync(FULL, (unsigned long long)C.total, 0);
  C.next_id = __shfl_sync(FULL, C.next_id, 0);
  C.hwm = __shfl_sync(FULL, C.hwm, 0);
  C.nfree = __shfl_sync(FULL, C.nfree, 0);
  C.c_wr = __shfl_sync(FULL, (unsigned long long)C.c_wr, 0);
  C.failed = __shfl_sync(FULL, (int)C.failed, 0);
}

__device__ __forceinline__ uint32_t hslot(unsigned long long key, uint32_t mask) {
  key ^= key >> 33;
  key *= 0xff51afd7ed558ccdull;
  key ^= key >> 33;
  key *= 0xc4ceb9fe1a85ec53ull;
  key ^= key >> 33;
  return (uint32_t)key & mask;
}
__device__ __forceinline__ unsigned long long hkey_of(uint32_t parent, uint32_t tok) {
  return ((unsigned long long)parent << 32) | tok;
}

// Warp-cooperative lookup of child(parent, tok): 32 probe positions per step.
__device__ __forceinline__ uint32_t hash_find_warp(const Chain& C, uint32_t parent, uint32_t tok) {
  const unsigned long long key = hkey_of(parent, tok);
  const uint32_t h = hslot(key, C.hmask);
  const uint32_t lane = lane_id();
  for (uint32_t base = 0; base <= C.hmask; base += 32) {
    const uint32_t idx = (h + base + lane) & C.hmask;
    const unsigned long long k = C.w.hkey()[idx];
    const unsigned mm = __ballot_sync(FULL, k == key);
    const unsigned me = __ballot_sync(FULL, k == EMPTY);
    if (mm) {
      const int fm = __ffs(mm) - 1;
      if (!me || fm < __ffs(me) - 1) return C.w.hval()[(h + base + fm) & C.hmask];
      return NIL;
    }
    if (me) return NIL;
  }
  return NIL;
}

// ---- single-thread (lane 0) hash mutations: linear probing, backward-shift delete ----
__device__ __forceinline__ uint32_t hash_index_1(const Chain& C, unsigned long long key) {
  uint32_t i = hslot(key, C.hmask);
  for (;;) {
    unsigned long long k = C.w.hkey()[i];
    if (k == key) return i;
    if (k == EMPTY) return NIL;
    i = (i + 1) & C.hmask;
  }
}
__device__ __forceinline__ void hash_insert_1(Chain& C, unsigned long long key, uint32_t val) {
  uint32_t i = hslot(key, C.hmask);
  while (C.w.hkey()[i] != EMPTY) i = (i + 1) & C.hmask;
  C.w.hkey()[i] = key;
  C.w.hval()[i] = val;
}
__device__ __forceinline__ void hash_erase_at_1(Chain& C, uint32_t i) {
  uint32_t j = i;
  for (;;) {
    j = (j + 1) & C.hmask;
    unsigned long long k = C.w.hkey()[j];
    if (k == EMPTY) break;
    uint32_t home = hslot(k, C.hmask);
    bool stays = (i <= j) ? (i < home && home <= j) : (i < home || home <= j);
    if (!stays) {
      C.w.hkey()[i] = k;
      C.w.hval()[i] = C.w.hval()[j];
      i = j;
    }
  }
  C.w.hkey()[i] = EMPTY;
}

// ---- dense live list (lane 0) ----
__device__ __forceinline__ void dense_refresh_1(Chain& C, uint32_t s) {
  const bool cand = C.w.nchild()[s] <= 1 && !(C.w.flags()[s] & F_PIN);
  C.w.dense()[C.w.dpos()[s]].tc = C.w.t()[s] | (cand ? 0u : NOTC);
}
__device__ __forceinline__ void dense_set_eff_1(Chain& C, uint32_t s) {
  C.w.dense()[C.w.dpos()[s]].eff = node_eff(C.m, C.w.ds()[s], C.w.de()[s], C.w.flags()[s] & F_SSM);
}
__device__ __forceinline__ void dense_add_1(Chain& C, uint32_t s) {
  const uint32_t i = C.count++;
  C.w.dpos()[s] = i;
  C.w.dslot()[i] = s;
  DenseRec d;
  d.tc = 0;
  d.id = C.w.id()[s];
  d.eff = node_eff(C.m, C.w.ds()[s], C.w.de()[s], C.w.flags()[s] & F_SSM);
  C.w.dense()[i] = d;
  dense_refresh_1(C, s);
}
__device__ __forceinline__ void dense_remove_1(Chain& C, uint32_t s) {
  const uint32_t i = C.w.dpos()[s];
  const uint32_t last = --C.count;
  if (i != last) {
    C.w.dense()[i] = C.w.dense()[last];
    const uint32_t s2 = C.w.dslot()[last];
    C.w.dslot()[i] = s2;
    C.w.dpos()[s2] = i;
  }
}
__device__ __forceinline__ uint32_t alloc_1(Chain& C, uint32_t* status) {
  if (C.nfree) return C.w.freel()[--C.nfree];
  if (C.hwm >= C.ncap) {
    atomicOr(status, ST_OVERFLOW);
    C.failed = true;
    return NIL;
  }
  return C.hwm++;
}

// ---------------------------------------------------------------------------
// Snapshot load (warp-cooperative).  Slot 0 = root, snapshot record i -> slot i+1.
// ---------------------------------------------------------------------------
__device__ void load_snapshot(Chain& C, const KParams& P, const DevSnapStore* st, uint32_t k) {
  const uint32_t lane = lane_id();
  uint32_t n = 0, nid = 1;
  const mc_snap_node* nodes = nullptr;
  const uint32_t* pidx = nullptr;
  if (st) {
    n = st->n[k];
    nid = st->nid[k];
    nodes = st->nodes + st->off[k];
    pidx = st->pidx + st->off[k];
  }
  if (n + 1 > C.ncap) {
    if (lane == 0) atomicOr(P.status, ST_OVERFLOW);
    C.failed = true;
    return;
  }
  for (uint32_t i = lane; i <= C.hmask; i += 32) C.w.hkey()[i] = EMPTY;
  for (uint32_t i = lane; i <= n; i += 32) {
    C.w.nchild()[i] = 0;
    C.w.cxor()[i] = 0;
  }
  if (lane == 0) {
    C.w.id()[0] = 0; C.w.parent()[0] = NIL; C.w.ds()[0] = 0; C.w.de()[0] = 0; C.w.t()[0] = 0;
    C.w.flags()[0] = 0; C.w.roff()[0] = 0; C.w.ftok()[0] = 0;
  }
  __syncwarp();
  uint64_t bytes = 0;
  bool bad = false;
  for (uint32_t i = lane; i < n; i += 32) {
    const mc_snap_node r = nodes[i];
    const uint32_t s = i + 1;
    const uint32_t pi = pidx[i];
    const uint32_t ps = (pi == NIL) ? 0u : pi + 1;
    bad |= (r.d_end <= r.d_start) || (r.ref_off + r.d_end > P.n_tok) || (pi != NIL && pi >= n);
    C.w.id()[s] = r.id;
    C.w.parent()[s] = ps;
    C.w.ds()[s] = r.d_start;
    C.w.de()[s] = r.d_end;
    C.w.t()[s] = r.t_last;
    C.w.roff()[s] = r.ref_off;
    C.w.flags()[s] = r.has_ssm ? F_SSM : 0u;
    const uint32_t ft = P.tok[r.ref_off + r.d_start];
    C.w.ftok()[s] = ft;
    C.w.dpos()[s] = i;
    C.w.dslot()[i] = s;
    atomicAdd(&C.w.nchild()[ps], 1u);
    atomicXor(&C.w.cxor()[ps], s);
    const unsigned long long key = hkey_of(ps, ft);
    uint32_t j = hslot(key, C.hmask);
    while (atomicCAS(&C.w.hkey()[j], EMPTY, key) != EMPTY) j = (j + 1) & C.hmask;
    C.w.hval()[j] = s;
    bytes += node_bytes(C.m, r.d_start, r.d_end, r.has_ssm);
  }
  __syncwarp();
  for (uint32_t i = lane; i < n; i += 32) {
    const uint32_t s = i + 1;
    DenseRec d;
    d.tc = C.w.t()[s] | (C.w.nchild()[s] <= 1 ? 0u : NOTC);
    d.id = C.w.id()[s];
    d.eff = node_eff(C.m, C.w.ds()[s], C.w.de()[s], C.w.flags()[s] & F_SSM);
    C.w.dense()[i] = d;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) bytes += __shfl_xor_sync(FULL, (unsigned long long)bytes, o);
  if (__any_sync(FULL, bad)) {
    if (lane == 0) atomicOr(P.status, ST_INVARIANT);
    C.failed = true;
  }
  C.total = bytes;
  C.count = n;
  C.next_id = nid;
  C.hwm = n + 1;
  C.nfree = 0;
  __syncwarp();
}

// Live pass: write the current tree as snapshot k (dense order, parent positions).
__device__ void dump_snapshot(Chain& C, const KParams& P, DevSnapOut* out, uint32_t k) {
  const uint32_t lane = lane_id();
  if (k >= out->count || C.count > out->stride) {
    if (lane == 0) atomicOr(P.status, ST_SNAPOVF);
    C.failed = true;
    return;
  }
  mc_snap_node* dst = out->nodes + (uint64_t)k * out->stride;
  uint32_t* pdst = out->pidx + (uint64_t)k * out->stride;
  for (uint32_t i = lane; i < C.count; i += 32) {
    const uint32_t s = C.w.dslot()[i];
    const uint32_t p = C.w.parent()[s];
    mc_snap_node r;
    r.id = C.w.id()[s];
    r.parent_id = (p == 0) ? 0u : C.w.id()[p];
    r.ref_off = C.w.roff()[s];
    r.d_start = C.w.ds()[s];
    r.d_end = C.w.de()[s];
    r.t_last = C.w.t()[s];
    r.has_ssm = (C.w.flags()[s] & F_SSM) ? 1u : 0u;
    dst[i] = r;
    pdst[i] = (p == 0) ? NIL : C.w.dpos()[p];
  }
  if (lane == 0) {
    out->off[k] = (uint64_t)k * out->stride;
    out->n[k] = C.count;
    out->nid[k] = C.next_id;
  }
  __syncwarp();
}

// Warp-cooperative first mismatch of tok[a..a+cmp) vs tok[b..b+cmp).
__device__ __forceinline__ uint32_t match_len(const uint32_t* __restrict__ tok, uint64_t a, uint64_t b,
                                              uint32_t cmp) {
  if (a == b) return cmp;  // same pool range: identical tokens
  const uint32_t lane = lane_id();
  for (uint32_t base = 0; base < cmp; base += 128) {
    unsigned mis[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const uint32_t j = base + 32 * q + lane;
      bool bad = false;
      if (j < cmp) bad = __ldg(tok + a + j) != __ldg(tok + b + j);
      mis[q] = __ballot_sync(FULL, bad);
    }
#pragma unroll
    for (int q = 0; q < 4; q++)
      if (mis[q]) return base + 32 * q + (__ffs(mis[q]) - 1);
  }
  return cmp;
}

// ---------------------------------------------------------------------------
// K3 + K4: one eviction
// ---------------------------------------------------------------------------
// Exact victim selection over the dense live list (Eq. 2).
//   α = 0: u = rec exactly and rec is strictly monotone in t, so the victim is
//          the candidate with the smallest (t_last, id) -- one pass (LRU,
//          PAPER:424); only the victim's u is computed.
//   α > 0: filter and verify.  Pass 1: bounds.  Pass 2: a division-free
//          approximate key k' = (t - tmin) * RN(1/Δt) + (e - emin) * RN(α/Δe)
//          with |k' - u| <= 10 (1+α) 2^-53; each lane keeps its best two keys.
//          Only entries with k' <= min k' + δ, δ = (1+α) 2^-45, can be the exact
//          argmin; their exact u (the IEEE recipe) decides.  If any lane has
//          two entries within δ (near-ties), fall back to the exact full pass.
#ifndef MC_UNROLL
#define MC_UNROLL 2
#endif
constexpr int kUnroll = MC_UNROLL;

__device__ __forceinline__ Best select_victim(const Chain& C, uint32_t cnt, Bounds& b) {
  const uint32_t lane = lane_id();
  const DenseRec* __restrict__ dn = C.w.dense();
  Best best;
  best_init(best);
  bounds_init(b);
  if (C.alpha == 0.0) {
    for (uint32_t base = 0; base < cnt; base += 32 * kUnroll) {
      DenseRec d[kUnroll];
#pragma unroll
      for (int q = 0; q < kUnroll; q++) {
        const uint32_t i = base + 32 * q + lane;
        if (i < cnt) d[q] = dn[i];
      }
#pragma unroll
      for (int q = 0; q < kUnroll; q++) {
        const uint32_t i = base + 32 * q + lane;
        if (i >= cnt) continue;
        const uint32_t t = d[q].tc & ~NOTC;
        b.tmin = min(b.tmin, t);
        b.tmax = max(b.tmax, t);
        if (!(d[q].tc & NOTC) && (t < best.t || (t == best.t && d[q].id < best.id))) {
          best.t = t; best.id = d[q].id; best.i = i;
        }
      }
    }
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      b.tmin = min(b.tmin, __shfl_xor_sync(FULL, b.tmin, o));
      b.tmax = max(b.tmax, __shfl_xor_sync(FULL, b.tmax, o));
      const uint32_t t = __shfl_xor_sync(FULL, best.t, o);
      const uint32_t id = __shfl_xor_sync(FULL, best.id, o);
      const uint32_t i = __shfl_xor_sync(FULL, best.i, o);
      if (i != NIL && (best.i == NIL || t < best.t || (t == best.t && id < best.id))) {
        best.t = t; best.id = id; best.i = i;
      }
    }
    if (best.i != NIL) {
      const double rec = (b.tmax == b.tmin) ? 0.5 : __ddiv_rn((double)(best.t - b.tmin), (double)(b.tmax - b.tmin));
      best.u = __dadd_rn(rec, __dmul_rn(0.0, 0.5));  // = rec (α·effn = +0)
    }
    return best;
  }
  // pass 1: bounds over ALL non-root nodes (R1)
  for (uint32_t base = 0; base < cnt; base += 32 * kUnroll) {
    DenseRec d[kUnroll];
#pragma unroll
    for (int q = 0; q < kUnroll; q++) {
      const uint32_t i = base + 32 * q + lane;
      if (i < cnt) d[q] = dn[i];
    }
#pragma unroll
    for (int q = 0; q < kUnroll; q++)
      if (base + 32 * q + lane < cnt) bounds_add(b, d[q].tc & ~NOTC, d[q].eff);
  }
  bounds_reduce(b);
  // pass 2: approximate keys, best two per lane
  const bool dt0 = b.tmax == b.tmin, de0 = b.emax == b.emin;
  const double idt = dt0 ? 0.0 : __drcp_rn((double)(b.tmax - b.tmin));
  const double aide = de0 ? 0.0 : __ddiv_rn(C.alpha, __dsub_rn(b.emax, b.emin));
  const double kconst = __dadd_rn(dt0 ? 0.5 : 0.0, de0 ? __dmul_rn(C.alpha, 0.5) : 0.0);
  const double INF = __longlong_as_double(0x7FF0000000000000ll);
  double k1 = INF, k2 = INF;
  uint32_t i1 = NIL;
  for (uint32_t base = 0; base < cnt; base += 32 * kUnroll) {
    DenseRec d[kUnroll];
#pragma unroll
    for (int q = 0; q < kUnroll; q++) {
      const uint32_t i = base + 32 * q + lane;
      if (i < cnt) d[q] = dn[i];
    }
#pragma unroll
    for (int q = 0; q < kUnroll; q++) {
      const uint32_t i = base + 32 * q + lane;
      if (i >= cnt || (d[q].tc & NOTC)) continue;
      const double k = __dadd_rn(__dadd_rn(__dmul_rn((double)(d[q].tc - b.tmin), idt),
                                           __dmul_rn(__dsub_rn(d[q].eff, b.emin), aide)), kconst);
      if (k < k1) { k2 = k1; k1 = k; i1 = i; }
      else if (k < k2) { k2 = k; }
    }
  }
  double kmin = k1;
#pragma unroll
  for (int o = 16; o; o >>= 1) kmin = fmin(kmin, __shfl_xor_sync(FULL, kmin, o));
  if (kmin == INF) return best;  // no candidate
  const double delta = __dmul_rn(__dadd_rn(1.0, C.alpha), 2.842170943040401e-14);  // (1+α) 2^-45
  const double lim = __dadd_rn(kmin, delta);
  if (!__any_sync(FULL, k2 <= lim)) {
    if (k1 <= lim) {
      const DenseRec d = dn[i1];
      best.u = utility(b, d.tc, d.eff, C.alpha);
      best.t = d.tc;
      best.id = d.id;
      best.i = i1;
    }
    best_reduce(best);
    return best;
  }
  // near-ties: exact full pass
  for (uint32_t i = lane; i < cnt; i += 32) {
    const DenseRec d = dn[i];
    if (d.tc & NOTC) continue;
    const double u = utility(b, d.tc, d.eff, C.alpha);
    if (best.i == NIL || better(u, d.tc, d.id, best)) {
      best.u = u; best.t = d.tc; best.id = d.id; best.i = i;
    }
  }
  best_reduce(best);
  return best;
}

__device__ void evict_one(Chain& C, const KParams& P, uint32_t r, mc_evict_rec* log, uint32_t* log_n) {
  const uint32_t lane = lane_id();
  const uint32_t cnt = C.count;
  Bounds b;
  const Best best = select_victim(C, cnt, b);
  C.c_scan += cnt;
  if (best.i == NIL) {
    if (lane == 0) atomicOr(P.status, ST_NOCAND);
    C.failed = true;
    return;
  }
  if (lane == 0) {
    const uint32_t x = C.w.dslot()[best.i];
    const uint32_t p = C.w.parent()[x];
    const uint32_t xf = C.w.flags()[x];
    uint32_t kind;
    if (C.w.nchild()[x] == 0) {  // leaf: free KVs + state
      kind = 0;
      C.total -= node_bytes(C.m, C.w.ds()[x], C.w.de()[x], xf & F_SSM);
      hash_erase_at_1(C, hash_index_1(C, hkey_of(p, C.w.ftok()[x])));
      C.w.nchild()[p] -= 1;
      C.w.cxor()[p] ^= x;
      if (p != 0) dense_refresh_1(C, p);
      C.c_wr += 1;
    } else {  // one child: release the state, the child absorbs the KVs
      kind = 1;
      const uint32_t c = C.w.cxor()[x];
      if (xf & F_SSM) C.total -= C.m.ssmb;
      hash_erase_at_1(C, hash_index_1(C, hkey_of(x, C.w.ftok()[c])));
      C.w.hval()[hash_index_1(C, hkey_of(p, C.w.ftok()[x]))] = c;
      C.w.ds()[c] = C.w.ds()[x];
      C.w.ftok()[c] = C.w.ftok()[x];
      C.w.parent()[c] = p;
      C.w.cxor()[p] ^= x ^ c;
      dense_set_eff_1(C, c);
      C.c_wr += 2;
    }
    if (log) {
      const uint32_t li = *log_n;
      if (li < P.log_cap) {
        mc_evict_rec e;
        e.req = r; e.node_id = best.id; e.kind = kind; e.n_live = cnt; e.utility = best.u;
        log[li] = e;
      }
      *log_n = li + 1;
    }
    dense_remove_1(C, x);
    C.w.flags()[x] = 0;
    C.w.freel()[C.nfree++] = x;
  }
  sync_state(C);
}

// Split node y at absolute depth x: new upper node [ds, x) takes a new id, y keeps
// its id and becomes [x, de) (R4).  Lane 0 only.
__device__ __forceinline__ uint32_t split_1(Chain& C, const KParams& P, uint32_t y, uint32_t x, bool stateful,
                                            uint32_t r) {
  const uint32_t u = alloc_1(C, P.status);
  if (u == NIL) return NIL;
  const uint32_t p = C.w.parent()[y];
  const uint32_t ods = C.w.ds()[y];
  C.w.id()[u] = C.next_id++;
  C.w.parent()[u] = p;
  C.w.ds()[u] = ods;
  C.w.de()[u] = x;
  C.w.roff()[u] = C.w.roff()[y];
  C.w.ftok()[u] = C.w.ftok()[y];
  C.w.flags()[u] = stateful ? F_SSM : 0u;
  C.w.t()[u] = r;
  C.w.nchild()[u] = 1;
  C.w.cxor()[u] = y;
  C.w.hval()[hash_index_1(C, hkey_of(p, C.w.ftok()[u]))] = u;  // same key, new child
  C.w.ds()[y] = x;
  const uint32_t ft = P.tok[C.w.roff()[y] + x];
  C.w.ftok()[y] = ft;
  C.w.parent()[y] = u;
  hash_insert_1(C, hkey_of(u, ft), y);
  C.w.cxor()[p] ^= y ^ u;
  dense_add_1(C, u);
  dense_set_eff_1(C, y);
  C.c_wr += 2;
  return u;
}

__device__ __forceinline__ void gain_1(Chain& C, uint32_t x, uint32_t r) {
  C.w.flags()[x] |= F_SSM;
  C.w.t()[x] = r;
  dense_set_eff_1(C, x);
  dense_refresh_1(C, x);
  C.c_wr += 1;
}

// ---------------------------------------------------------------------------
// One request: SURVEY.md §8(c) c.2 steps 1-9.
// ---------------------------------------------------------------------------
struct ReqOut {
  uint32_t reuse;
  uint64_t flops;
  bool bypass;
};

__device__ ReqOut process_request(Chain& C, const KParams& P, uint32_t r, mc_evict_rec* log, uint32_t* log_n) {
  const uint32_t lane = lane_id();
  const mc_request q = P.req[r - 1];
  const uint64_t off = q.tok_off;
  const uint32_t L_in = q.input_len;
  const uint32_t n = q.input_len + q.output_len;

  // Step 1: walk = lookup + speculative insertion bookkeeping.
  uint32_t v = 0, pos = 0, npath = 0, m = 0;
  uint32_t partial = NIL, hit = NIL, reuse = 0;
  uint32_t lin_node = NIL;   // node whose edge strictly contains L_in (when m >= L_in)
  uint32_t lin_bnd = NIL;    // fully matched node ending exactly at L_in
  uint64_t pinned_bytes = 0;
  for (;;) {
    if (pos == n) { m = n; break; }
    const uint32_t tk = __ldg(P.tok + off + pos);
    const uint32_t c = hash_find_warp(C, v, tk);
    if (c == NIL) { m = pos; break; }
    const uint32_t ds = C.w.ds()[c], de = C.w.de()[c], fl = C.w.flags()[c];
    const uint64_t ro = C.w.roff()[c];
    const uint32_t len = de - ds;
    const uint32_t cmp = min(len, n - pos);
    const uint32_t k = match_len(P.tok, ro + ds, off + pos, cmp);
    if (lane == 0) {
      C.w.path()[npath] = c;
      C.w.flags()[c] = fl | F_PIN;   // pin the path (R12)
      C.w.dense()[C.w.dpos()[c]].tc |= NOTC;
    }
    npath++;
    pinned_bytes += node_bytes(C.m, ds, de, fl & F_SSM);
    if (pos < L_in && L_in < pos + len && L_in <= pos + k) lin_node = c;
    if (k == len) {
      v = c;
      pos += len;
      if (de == L_in) lin_bnd = c;
      if ((fl & F_SSM) && de <= L_in) { hit = c; reuse = de; }  // all-or-nothing hit (R6, R7)
    } else {
      m = pos + k;
      partial = c;
      break;
    }
  }
  __syncwarp();
  C.c_cmp += min(m + 1, n);
  C.c_vis += npath + 1;

  // Step 2: pure Transformer (n_ssm = 0): KVs can be sliced mid-edge.
  if (C.m.n_ssm == 0) {
    reuse = min(m, L_in);
    hit = NIL;
    for (uint32_t i = 0; i < npath; i++) {
      const uint32_t x = C.w.path()[i];
      if (C.w.ds()[x] < reuse) hit = x;
    }
  }

  // Step 3: speculative insertion of the input (R8, R9).
  const uint32_t m_in = min(m, L_in);
  uint32_t p = 0, p_split = NIL, p_gain = NIL;
  if (m_in > 0) {
    if (m >= L_in) {
      if (lin_bnd != NIL) {
        if (!(C.w.flags()[lin_bnd] & F_SSM)) { p = m_in; p_gain = lin_bnd; }
      } else {
        p = m_in;
        p_split = lin_node;
      }
    } else if (partial != NIL) {
      p = m_in;
      p_split = partial;
    } else if (!(C.w.flags()[v] & F_SSM)) {
      p = m_in;
      p_gain = v;
    }
  }
  // Step 4: plan -- checkpoints {p, n}, at most two.
  const bool leaf = m < n;
  const bool split_m = partial != NIL && m < n && m != p;   // stateless output-region split (R10)
  const bool split_n = partial != NIL && m == n && n != p;  // sequence ends inside an edge
  uint32_t n_gain = NIL;
  if (partial == NIL && m == n && n != p && !(C.w.flags()[v] & F_SSM)) n_gain = v;
  uint32_t n_ck = p ? 1u : 0u;
  if (n != p && (leaf || split_n || n_gain != NIL)) n_ck++;
  const uint64_t d_bytes = C.m.kvt * (uint64_t)(n - m) + C.m.ssmb * n_ck;
  const uint32_t d_nodes = (p_split != NIL ? 1u : 0u) + (split_m ? 1u : 0u) + (split_n ? 1u : 0u) + (leaf ? 1u : 0u);

  // Step 5: touch only the hit node.
  if (hit != NIL) {
    if (lane == 0) {
      C.w.t()[hit] = r;
      dense_refresh_1(C, hit);
    }
    C.c_wr += 1;
  }
  __syncwarp();

  // Step 6: admission precheck (R12).
  const bool bypass = (pinned_bytes + d_bytes > C.capb) || (C.capn && npath + d_nodes > C.capn);
  if (!bypass) {
    // Step 7: evict the argmin utility until the request fits.
    while (!C.failed && (C.total + d_bytes > C.capb || (C.capn && C.count + d_nodes > C.capn)))
      evict_one(C, P, r, log, log_n);
    // Step 8: insert.
    if (lane == 0 && !C.failed) {
      uint32_t attach = v;  // node at depth m after the splits
      if (p_split != NIL) {
        const uint32_t u = split_1(C, P, p_split, p, true, r);
        if (p == m) attach = u;
      }
      if (split_m && !C.failed) attach = split_1(C, P, partial, m, false, r);
      if (split_n && !C.failed) split_1(C, P, partial, n, true, r);
      if (p_gain != NIL) gain_1(C, p_gain, r);
      if (n_gain != NIL) gain_1(C, n_gain, r);
      if (leaf && !C.failed) {
        const uint32_t w = alloc_1(C, P.status);
        if (w != NIL) {
          C.w.id()[w] = C.next_id++;
          C.w.parent()[w] = attach;
          C.w.ds()[w] = m;
          C.w.de()[w] = n;
          C.w.roff()[w] = off;
          const uint32_t ft = P.tok[off + m];
          C.w.ftok()[w] = ft;
          C.w.flags()[w] = F_SSM;
          C.w.t()[w] = r;
          C.w.nchild()[w] = 0;
          C.w.cxor()[w] = 0;
          hash_insert_1(C, hkey_of(attach, ft), w);
          C.w.nchild()[attach] += 1;
          C.w.cxor()[attach] ^= w;
          if (attach != 0) dense_refresh_1(C, attach);
          dense_add_1(C, w);
          C.c_wr += 1;
        }
      } else if (partial == NIL) {
        // final node at n already exists: timestamp it (R5)
        C.w.t()[v] = r;
        dense_refresh_1(C, v);
        if (n_gain == NIL && p_gain != v) C.c_wr += 1;
      }
      C.total += d_bytes;
      if (C.total > C.capb || (C.capn && C.count > C.capn)) {
        atomicOr(P.status, ST_INVARIANT);
        C.failed = true;
      }
    }
    sync_state(C);
  }
  // Step 9: unpin, outputs.
  if (lane == 0) {
    for (uint32_t i = 0; i < npath; i++) {
      const uint32_t x = C.w.path()[i];
      C.w.flags()[x] &= ~F_PIN;
      dense_refresh_1(C, x);
    }
    if (reuse > L_in) {
      atomicOr(P.status, ST_INVARIANT);
      C.failed = true;
    }
  }
  sync_state(C);
  ReqOut o;
  o.reuse = reuse;
  o.flops = prefill_F(C.m, reuse);
  o.bypass = bypass;
  return o;
}

__device__ __forceinline__ void chain_init(Chain& C, const KParams& P, uint32_t worker, const DevVariant& V,
                                           double alpha) {
  C.w = ws_slice(P.ws + (uint64_t)worker * P.ws_stride, P.ncap, P.hcap);
  C.ncap = P.ncap;
  C.hmask = P.hcap - 1;
  C.m = V.m;
  C.capb = V.cap_bytes;
  C.capn = V.cap_nodes;
  C.alpha = alpha;
  C.c_cmp = C.c_vis = C.c_scan = C.c_wr = 0;
  C.failed = false;
}

}  // namespace mcd
