// replay.cuh -- device code of the Marconi α-grid replay (sm_100a).
//
// One WARP owns one chain (variant, α, segment): a private flattened radix
// tree replayed request by request.
//
// Data layout per chain:
//   shared memory  dense list by node slot: t_last|pin|multi (u32) and RN32(FLOP
//                  efficiency) (f32) for slots < S -- the data every eviction scans --
//                  then the counters, constants and the snapshot-copy mbarrier;
//   global (L2)    32-byte node records {parent, own child-index position, d_start,
//                  d_end, pool offset, child xor, nchild|flags, id}; a 16-byte-entry
//                  open-addressing child index keyed by (parent, first token) whose
//                  entries carry the child's slot, depth, state flag and pool offset
//                  plus a generation tag (no table clear between chains); the dense
//                  tail (slots >= S).  The exact fp64 eff is recomputed from a record
//                  when a cold path needs it.
// Warp-cooperative stages:
//   K2 walk      -- child lookup = one 128 B line of the index per probe step; edge
//                   compare = 8 x 32 tokens per round trip with __ballot_sync/__ffs,
//                   long compares prefetched into L2 by cp.async.bulk.prefetch
//                   (speculative insertion PAPER:365 fused in);
//   K3 scan      -- normalisation bounds + filter-and-verify argmin of Eq. 2
//                   (PAPER:414-419), warp-shuffle reductions;
//   snapshot image load -- dense list by one cp.async.bulk (TMA) into shared memory;
//   lookup       -- mc_lookup's read-only steps 1-4 (lookup_request).
// Scalar tree mutations (K4: split, leaf, gain, leaf removal, absorption --
// PAPER:362-365) run on lane 0; the chain scalars are then
// broadcast.  K1 (Eq. 1 cost model, Appendix A) is inlined wherever a node's
// range or state changes.
//
// Bit-exactness: integer FLOPs/bytes are exact u64; eff = one IEEE division;
// the utility uses __dsub_rn/__ddiv_rn/__dmul_rn/__dadd_rn (no FMA).
#pragma once
#include <cstdint>
#include <cuda_runtime.h>
#include "marconi.h"

namespace mcd {

constexpr uint32_t NIL = 0xFFFFFFFFu;
// dense word tc = t_last (bits 0..29) | D_PIN | D_MULTI; a node is an eviction
// candidate iff neither flag is set (<= 1 child and not on the current path)
constexpr uint32_t D_PIN = 0x80000000u;    // on the current request's path (pinned, R12)
constexpr uint32_t D_MULTI = 0x40000000u;  // >= 2 children
constexpr uint32_t D_FLAGS = D_PIN | D_MULTI;
constexpr uint32_t T_MASK = 0x3FFFFFFFu;
// Dense position = node slot.  A free slot (and slot 0, the root) holds a hole: both
// flags set (never a candidate), t = T_MASK (never the t minimum) and e32 = NaN (fminf /
// fmaxf ignore it); bound passes skip holes for the t maximum explicitly.
constexpr uint32_t HOLE_TC = 0xFFFFFFFFu;
constexpr uint32_t HOLE_E32 = 0x7FC00000u;
constexpr uint32_t F_SSM = 1u;  // node flag (bits 24.. of NodeRec::nf)
constexpr uint32_t NCH_MASK = 0x00FFFFFFu;
// child-index entry (16 B): {first token, gen<<28 | parent slot<<14 | child slot,
// d_end | has_ssm<<31, pool offset}.  An entry is live iff its generation is the
// chain's (the previous chain's entries are stale without clearing the table); it
// carries everything the walk needs about the child, so the walk reads no records.
constexpr uint32_t GEN_MAX = 15, SLOT14 = 0x3FFFu;
struct __align__(16) HEnt {
  uint32_t tok, key, de, roff;
};
constexpr unsigned FULL = 0xFFFFFFFFu;

// device status word bits (mc_check)
enum : uint32_t {
  ST_OVERFLOW = 1u,   // node table full
  ST_INVARIANT = 2u,  // capacity exceeded after admission / hit > input / bad snapshot
  ST_NOCAND = 4u,     // eviction needed but no candidate (cannot happen after the precheck)
  ST_SNAPOVF = 8u,    // snapshot store too small
  ST_BADTRACE = 16u,  // the device-side trace check (mc_set_trace_async) rejected a request
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
  uint32_t cap_nodes, chunk;  // chunk = 0: exact checkpoints; else chunk-aligned prefill checkpoints
  uint32_t block, pad;        // block > 0: the vLLM+ baseline with token blocks of `block` (NEXT-2)
};
// Per-chain read-only constants, kept in the warp's shared memory (64 B) so that the
// replay loop does not hold them in registers (the kernel runs at the 128-register cap).
struct ChainConst {
  DevModel m;
  uint64_t capb;
  uint32_t capn, chunk;
  double alpha;
};
static_assert(sizeof(ChainConst) == 64, "ChainConst is carved from 8 dense slots");
// Per-chain algorithmic counters, lane 0 accumulates them in shared
// memory (read once, at the end of the chain).
struct ChainCtr {
  uint64_t cmp, vis, scan, wr;
};
static_assert(sizeof(ChainCtr) == 32, "ChainCtr is carved from 4 dense slots");
// dense slots per warp above its S dense positions: ChainCtr (4), ChainConst (8), the
// snapshot-copy mbarrier and its phase word (2)
constexpr uint32_t kSmemReserved = 14;
struct DevSnapStore {
  const mc_snap_node* nodes;
  const uint32_t* pidx;  // parent position within the same snapshot, NIL = root
  const uint64_t* off;
  const uint32_t* n;
  const uint32_t* nid;
  const char* img;         // loadable images of the snapshots (see ImgHdr), built at setup
  const uint64_t* img_off; // byte offset of snapshot k's image
  uint32_t count, pad;
};

// Snapshot image: a chain's workspace state right after loading the snapshot, built once
// per snapshot at setup (image_kernel) so the 16+ chains that start from the same
// snapshot copy it (coalesced, no child-index CAS, no Eq. 1 divisions) instead of
// rebuilding it.  Byte layout from the image base (n = nodes):
//   ImgHdr 64 | records 32(n+1) | dense 8(n+1) | child-index positions 4n |
//   child-index entries 16n      (regions 16 B aligned)
// (records carry the node ids; dense is indexed by slot; slot 0, the root, is a hole)
struct ImgHdr {
  unsigned long long total;
  uint32_t n, nid, tmin, tmax;
  float lo32, hi32;
  double elo, ehi;
  uint32_t bc_valid, pad0, pad1, pad2;
};
__host__ __device__ inline uint64_t img_al16(uint64_t x) { return (x + 15) & ~15ull; }
__host__ __device__ inline uint64_t img_off_dense(uint32_t n) { return 64 + 32ull * (n + 1); }
__host__ __device__ inline uint64_t img_off_tpos(uint32_t n) { return img_off_dense(n) + img_al16(8ull * (n + 1)); }
__host__ __device__ inline uint64_t img_off_tent(uint32_t n) { return img_off_tpos(n) + img_al16(4ull * n); }
__host__ __device__ inline uint64_t img_bytes(uint32_t n) { return img_off_tent(n) + 16ull * n; }
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

struct __align__(8) DenseRec {  // one dense position: the scanned key pair
  uint32_t tc;  // t_last | D_PIN | D_MULTI
  float e32;    // RN32(eff) -- filter and bounds; the exact eff is recomputed from the record
};

struct __align__(16) NodeRec {
  uint32_t parent, hidx, ds, de;  // hidx = position of the node's own entry in the child index
  uint32_t roff, cxor, nf, id;    // roff = pool offset of the node's request; nf = nchild | flags << 24;
                                  // id = creation ordinal (R4)
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
  const uint32_t* live_points;  // snapshot k = tree after request live_points[k] (ascending, [0] = 0)
  uint32_t n_points;
  uint32_t* first_evict;        // [n_var] first request whose admission evicted (0 = none)
  uint32_t live_mult;           // > 0: bootstrap points instead (snapshot 1 after r_F, 2 after r_F + mult r_F)
  unsigned long long* live_cyc; // [n_var][n_points] SM cycles the live pass spent on window k (static points)
  uint32_t smem_nodes;  // dense positions held in shared memory per warp
};

// Per-worker workspace slice.  The caller zero-initialises the workspace once
// (header word 0 = child-index generation, word 1 = layout signature).
// Slice layout (byte offsets from the slice base; n = ncap, h = hcap):
//   header 256 | records 32n | scratch 4n | path 4n | freel 4n | child index 16h |
//   dense tail 8n
// (n is a power of two >= 64, so every region stays 16 B aligned).  ws_bytes_per_worker
// is the end of the last region, so the accessors below and the stride cannot disagree.
// Node ids live in the records and the exact fp64 eff is recomputed from a record when a
// cold path needs it (one IEEE division, bit-identical to the value the dense list's
// RN32 came from), so neither is a per-slot array a chain must copy or keep in L2.
__host__ __device__ inline uint64_t ws_off_tab(uint32_t n) { return 256 + 44ull * n; }
__host__ __device__ inline uint64_t ws_off_tail(uint32_t n, uint32_t h) { return ws_off_tab(n) + 16ull * h; }
__host__ __device__ inline uint64_t ws_bytes_per_worker(uint32_t ncap, uint32_t hcap) {
  const uint64_t b = ws_off_tail(ncap, hcap) + 8ull * ncap;
  return (b + 255) & ~255ull;
}

struct WS {
  char* b;
  uint32_t n, h;
  __device__ __forceinline__ uint32_t* hdr() const { return (uint32_t*)b; }
  __device__ __forceinline__ NodeRec* rec() const { return (NodeRec*)(b + 256); }
  __device__ __forceinline__ uint32_t* scratch() const { return (uint32_t*)(b + 256 + 32ull * n); }  // dump map
  __device__ __forceinline__ uint32_t* path() const { return (uint32_t*)(b + 256 + 36ull * n); }
  __device__ __forceinline__ uint32_t* freel() const { return (uint32_t*)(b + 256 + 40ull * n); }
  __device__ __forceinline__ HEnt* tab() const { return (HEnt*)(b + ws_off_tab(n)); }
  __device__ __forceinline__ DenseRec* tail() const { return (DenseRec*)(b + ws_off_tail(n, h)); }
};

__device__ __forceinline__ uint32_t lane_id() { return threadIdx.x & 31u; }
#define CTR_ADD(C, f, v)                      \
  do {                                        \
    if (lane_id() == 0) (C).X->f += (v);      \
  } while (0)

// ---------------------------------------------------------------------------
// K1: cost model (Eq. 1 with Appendix A), bit-exact with the host definition.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t prefill_F(const DevModel& m, uint64_t L) {
  return m.fa * L + m.fb * L * L;
}
__device__ __forceinline__ uint64_t node_bytes(const DevModel& m, uint32_t ds, uint32_t de, bool ssm) {
  return m.kvt * (uint64_t)(de - ds) + (ssm ? m.ssmb : 0ull);
}
// out of line: the IEEE division sequence is long and the call sites are cold (I-cache)
__device__ __forceinline__ double node_eff(DevModel m, uint32_t ds, uint32_t de, bool ssm) {
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
  b.emin = e < b.emin ? e : b.emin;  // eff is finite and positive: no NaN handling needed
  b.emax = e > b.emax ? e : b.emax;
}
__device__ __forceinline__ void bounds_reduce(Bounds& b) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    b.tmin = min(b.tmin, __shfl_xor_sync(FULL, b.tmin, o));
    b.tmax = max(b.tmax, __shfl_xor_sync(FULL, b.tmax, o));
    const double lo = __shfl_xor_sync(FULL, b.emin, o), hi = __shfl_xor_sync(FULL, b.emax, o);
    b.emin = lo < b.emin ? lo : b.emin;
    b.emax = hi > b.emax ? hi : b.emax;
  }
}
// u = rec + α·effn, each operation rounded (no FMA); degenerate range -> 0.5 (R2).
__device__ __forceinline__ double utility(Bounds b, uint32_t t, double e, double alpha) {
  double rec = (b.tmax == b.tmin) ? 0.5 : __ddiv_rn((double)(t - b.tmin), (double)(b.tmax - b.tmin));
  double effn = (b.emax == b.emin) ? 0.5 : __ddiv_rn(__dsub_rn(e, b.emin), __dsub_rn(b.emax, b.emin));
  return __dadd_rn(rec, __dmul_rn(alpha, effn));
}
struct Best {
  double u;
  uint32_t t, id, i, slot;  // i = slot = the node's dense position
};
__device__ __forceinline__ bool better(double u, uint32_t t, uint32_t id, const Best& b) {
  return u < b.u || (u == b.u && (t < b.t || (t == b.t && id < b.id)));
}
__device__ __forceinline__ void best_init(Best& b) {
  b.u = __longlong_as_double(0x7FF0000000000000ll);
  b.t = 0xFFFFFFFFu;
  b.id = 0xFFFFFFFFu;
  b.i = NIL;
  b.slot = NIL;
}
__device__ __forceinline__ void best_reduce(Best& b) {
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    double u = __shfl_xor_sync(FULL, b.u, o);
    uint32_t t = __shfl_xor_sync(FULL, b.t, o);
    uint32_t id = __shfl_xor_sync(FULL, b.id, o);
    uint32_t i = __shfl_xor_sync(FULL, b.i, o);
    uint32_t sl = __shfl_xor_sync(FULL, b.slot, o);
    if (i != NIL && (b.i == NIL || better(u, t, id, b))) {
      b.u = u; b.t = t; b.id = id; b.i = i; b.slot = sl;
    }
  }
}

// ---------------------------------------------------------------------------
// Chain state (per warp; scalars are warp-uniform, lane 0 is the writer)
// ---------------------------------------------------------------------------
struct Chain {
  WS w;
  DenseRec* sd;     // SMEM: dense {t_last|D_PIN|D_MULTI, RN32(eff)} for positions < S
  uint32_t S;       // SMEM-resident dense positions (the tail lives in global)
  uint32_t ncap, hmask, gen;
  uint32_t count;     // live non-root nodes (the dense list spans slots [0, hwm), holes included)
  uint64_t total;     // bytes of all live nodes
  uint32_t next_id, hwm, nfree;
  const ChainConst* K;  // the chain's read-only constants, in shared memory (not registers)
  uint32_t block;  // > 0: vLLM+ baseline (token blocks of `block`), else Marconi
  uint32_t mthr;   // D_MULTI threshold: children that make a node a non-candidate (2 Marconi, 1 vLLM+)
  ChainCtr* X;  // counters (shared memory, lane 0 writes)
  uint32_t n_evict;   // evictions so far (uniform)
  // cached normalisation bounds (bc_valid bit 0: t and fp32 eff bounds exact; bits 1 / 2:
  // bc_elo / bc_ehi also exact -- recovered lazily, only a logged or near-tied victim
  // needs them): adds extend them, removing or
  // changing a node that holds an extreme invalidates them (pass 1 then recomputes)
  // (bc_elo/bc_ehi: the exact fp64 extremes; bc_lo/bc_hi = their RN32 images, which are
  // the fp32 extremes because RN is monotone)
  uint32_t bc_valid, bc_tmin, bc_tmax;
  float bc_lo, bc_hi;
  double bc_elo, bc_ehi;
#if defined(MC_PHASE_TIMERS) || defined(MC_PHASE_TIMERS3)
  unsigned long long t_walk, t_evict, t_insert, t_unpin;
#endif
  bool failed;
};

__device__ __forceinline__ void sync_state(Chain& C) {
  __syncwarp();
  C.count = __shfl_sync(FULL, C.count, 0);
  C.total = __shfl_sync(FULL, (unsigned long long)C.total, 0);
  C.next_id = __shfl_sync(FULL, C.next_id, 0);
  C.hwm = __shfl_sync(FULL, C.hwm, 0);
  C.nfree = __shfl_sync(FULL, C.nfree, 0);
  C.failed = __shfl_sync(FULL, (int)C.failed, 0);
  C.bc_valid = __shfl_sync(FULL, C.bc_valid, 0);
  C.bc_tmin = __shfl_sync(FULL, C.bc_tmin, 0);
  C.bc_tmax = __shfl_sync(FULL, C.bc_tmax, 0);
  C.bc_lo = __shfl_sync(FULL, C.bc_lo, 0);
  C.bc_hi = __shfl_sync(FULL, C.bc_hi, 0);
  C.bc_elo = __shfl_sync(FULL, C.bc_elo, 0);
  C.bc_ehi = __shfl_sync(FULL, C.bc_ehi, 0);
}

__device__ __forceinline__ uint32_t hslot(uint32_t parent, uint32_t tok, uint32_t mask) {
  uint32_t h = tok * 0x9E3779B1u ^ parent * 0x85EBCA77u;
  h ^= h >> 15;
  h *= 0x2C1B3C6Du;
  h ^= h >> 13;
  return h & mask;
}
__device__ __forceinline__ bool hvalid(const Chain& C, uint32_t key) { return (key >> 28) == C.gen; }
__device__ __forceinline__ uint32_t hkey(const Chain& C, uint32_t parent, uint32_t slot) {
  return (C.gen << 28) | (parent << 14) | slot;
}
__device__ __forceinline__ HEnt hmake(const Chain& C, uint32_t parent, uint32_t tok, uint32_t slot, uint32_t de,
                                      bool ssm, uint32_t roff) {
  HEnt e;
  e.tok = tok;
  e.key = hkey(C, parent, slot);
  e.de = de | (ssm ? 0x80000000u : 0u);
  e.roff = roff;
  return e;
}
__device__ __forceinline__ bool hmatch(const HEnt& e, uint32_t parent, uint32_t tok) {
  return e.tok == tok && ((e.key >> 14) & SLOT14) == parent;
}
__device__ __forceinline__ uint32_t hhome(const Chain& C, const HEnt& e) {
  return hslot((e.key >> 14) & SLOT14, e.tok, C.hmask);
}

// Warp-cooperative lookup of child(parent, tok).  Linear probing from the home
// position h, one 128 B line (8 entries) per step: the first step covers h .. end of
// h's line, later steps whole lines, so a typical lookup (hit or miss at h) touches
// one or two 32 B sectors instead of a 512 B window.  Returns the entry (key == 0
// when absent).  hcap is a multiple of 8, so a line never wraps.
__device__ __forceinline__ HEnt hash_find_warp(const Chain& C, uint32_t parent, uint32_t tok) {
  const uint32_t lane = lane_id();
  const HEnt* __restrict__ tab = C.w.tab();
  HEnt none;
  none.tok = 0; none.key = 0; none.de = 0; none.roff = 0;
  uint32_t i0 = hslot(parent, tok, C.hmask);
  for (uint32_t seen = 0; seen <= C.hmask;) {
    const uint32_t lim = (i0 | 7u) - i0 + 1;  // entries from i0 to the end of its line
    const bool act = lane < lim;
    HEnt e = none;
    if (act) e = tab[i0 + lane];
    const bool valid = act && hvalid(C, e.key);
    const unsigned mm = __ballot_sync(FULL, valid && hmatch(e, parent, tok));
    const unsigned me = __ballot_sync(FULL, act && !valid);
    if (mm) {
      const int fm = __ffs(mm) - 1;
      HEnt r;
      r.tok = tok;
      r.key = __shfl_sync(FULL, e.key, fm);
      r.de = __shfl_sync(FULL, e.de, fm);
      r.roff = __shfl_sync(FULL, e.roff, fm);
      if (!me || fm < __ffs(me) - 1) return r;
      return none;
    }
    if (me) return none;
    seen += lim;
    i0 = (i0 + lim) & C.hmask;
  }
  return none;
}

// ---- single-thread (lane 0) child-index mutations: linear probing, backward-shift delete ----
__device__ __forceinline__ uint32_t hash_index_1(const Chain& C, uint32_t parent, uint32_t tok) {
  uint32_t i = hslot(parent, tok, C.hmask);
  for (;;) {
    const HEnt e = C.w.tab()[i];
    if (!hvalid(C, e.key)) return NIL;
    if (hmatch(e, parent, tok)) return i;
    i = (i + 1) & C.hmask;
  }
}
__device__ __forceinline__ uint32_t hash_insert_1(Chain& C, const HEnt& ne, uint32_t parent) {
  uint32_t i = hslot(parent, ne.tok, C.hmask);
  while (hvalid(C, C.w.tab()[i].key)) i = (i + 1) & C.hmask;
  C.w.tab()[i] = ne;
  return i;
}
__device__ __forceinline__ void hash_erase_at_1(Chain& C, uint32_t i) {
  uint32_t j = i;
  for (;;) {
    j = (j + 1) & C.hmask;
    const HEnt e = C.w.tab()[j];
    if (!hvalid(C, e.key)) break;
    const uint32_t home = hhome(C, e);
    const bool stays = (i <= j) ? (i < home && home <= j) : (i < home || home <= j);
    if (!stays) {
      C.w.tab()[i] = e;
      C.w.rec()[e.key & SLOT14].hidx = i;  // the moved entry's node keeps knowing its position
      i = j;
    }
  }
  C.w.tab()[i].key = 0;
}

// ---- dense live list: positions < S in shared memory, the tail in global ----
__device__ __forceinline__ DenseRec* d_ptr(const Chain& C, uint32_t i) { return i < C.S ? C.sd + i : C.w.tail() + i; }
__device__ __forceinline__ uint32_t d_tc(const Chain& C, uint32_t i) { return d_ptr(C, i)->tc; }
__device__ __forceinline__ double rec_eff(const DevModel& m, const NodeRec& R) {
  return node_eff(m, R.ds, R.de, (R.nf >> 24) & F_SSM);
}
// out of line: the IEEE division sequence is long and the callers (a logged or near-tied
// victim's exact utility) are cold
__device__ __noinline__ double slot_eff(const NodeRec* rec, const DevModel m, uint32_t i) { return rec_eff(m, rec[i]); }
__device__ __forceinline__ double d_eff(const Chain& C, uint32_t i) { return slot_eff(C.w.rec(), C.K->m, i); }
__device__ __forceinline__ uint32_t d_id(const Chain& C, uint32_t i) { return C.w.rec()[i].id; }
__device__ __forceinline__ void d_hole(Chain& C, uint32_t i) {
  DenseRec h;
  h.tc = HOLE_TC;
  h.e32 = __uint_as_float(HOLE_E32);
  *d_ptr(C, i) = h;
}
__device__ __forceinline__ void d_set_tc(Chain& C, uint32_t i, uint32_t v) { d_ptr(C, i)->tc = v; }
// bound-cache hooks (lane 0, or uniform)
// RN32 is monotone, so e32 < lo32 implies e64 is below every live value: the new exact
// minimum is known even when the old one was not (likewise for the maximum).
__device__ __forceinline__ void bc_extend_e(Chain& C, float e32, double e64) {
  if (e32 < C.bc_lo) { C.bc_lo = e32; C.bc_elo = e64; C.bc_valid |= 2u; }
  else if (e32 == C.bc_lo && e64 < C.bc_elo) C.bc_elo = e64;
  if (e32 > C.bc_hi) { C.bc_hi = e32; C.bc_ehi = e64; C.bc_valid |= 4u; }
  else if (e32 == C.bc_hi && e64 > C.bc_ehi) C.bc_ehi = e64;
}
__device__ __forceinline__ void bc_add(Chain& C, uint32_t t, float e32, double e64) {
  C.bc_tmin = min(C.bc_tmin, t);
  C.bc_tmax = max(C.bc_tmax, t);
  bc_extend_e(C, e32, e64);
}
__device__ __forceinline__ void bc_change_e(Chain& C, float old_e, float new_e32, double new_e64) {
  if (old_e == C.bc_lo || old_e == C.bc_hi) C.bc_valid = 0;
  bc_extend_e(C, new_e32, new_e64);
}
__device__ __forceinline__ void bc_change_t(Chain& C, uint32_t old_t, uint32_t new_t) {
  if (old_t == C.bc_tmin) C.bc_valid = 0;
  C.bc_tmax = max(C.bc_tmax, new_t);
}
__device__ __forceinline__ void bc_remove(Chain& C, uint32_t t, float e) {
  if (t == C.bc_tmin || t == C.bc_tmax || e == C.bc_lo || e == C.bc_hi) C.bc_valid = 0;
}
// eff of an EXISTING dense position changes
__device__ __forceinline__ void d_set_eff(Chain& C, uint32_t i, double v) {
  DenseRec* d = d_ptr(C, i);
  const float e = __double2float_rn(v);
  bc_change_e(C, d->e32, e, v);
  d->e32 = e;
}
// (re)stamp dense position i with timestamp t, keeping its flags (lane 0)
__device__ __forceinline__ void d_stamp(Chain& C, uint32_t i, uint32_t t) {
  DenseRec* d = d_ptr(C, i);
  bc_change_t(C, d->tc & T_MASK, t);
  d->tc = t | (d->tc & D_FLAGS);
}
__device__ __forceinline__ void d_multi(Chain& C, uint32_t i, uint32_t nchild) {
  DenseRec* d = d_ptr(C, i);
  d->tc = (d->tc & ~D_MULTI) | (nchild >= C.mthr ? D_MULTI : 0u);
}
__device__ __forceinline__ void dense_add_1(Chain& C, uint32_t s, uint32_t t) {
  const uint32_t i = s;
  C.count++;
  const NodeRec& R = C.w.rec()[s];
  const double v = node_eff(C.K->m, R.ds, R.de, (R.nf >> 24) & F_SSM);
  DenseRec* d = d_ptr(C, i);
  d->e32 = __double2float_rn(v);
  d->tc = t | ((R.nf & NCH_MASK) >= C.mthr ? D_MULTI : 0u);
  bc_add(C, t, d->e32, v);
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

// ---- vLLM+ block keys: content hash of a token block (sum of position-mixed tokens,
// so one lane or a whole warp computes the same value); equal hashes are always
// verified against the tokens, so collisions cost time, never correctness ----
__device__ __forceinline__ uint32_t tok_mix(uint32_t t, uint32_t j) {
  uint32_t h = t ^ (j * 0x9E3779B9u);
  h ^= h >> 16;
  h *= 0x85EBCA6Bu;
  h ^= h >> 13;
  h *= 0xC2B2AE35u;
  h ^= h >> 16;
  return h;
}
__device__ __forceinline__ uint32_t block_hash_1(const uint32_t* __restrict__ p, uint32_t x) {
  uint32_t h0 = 0, h1 = 0, h2 = 0, h3 = 0;
  uint32_t j = 0;
  for (; j + 4 <= x; j += 4) {
    h0 += tok_mix(__ldg(p + j), j);
    h1 += tok_mix(__ldg(p + j + 1), j + 1);
    h2 += tok_mix(__ldg(p + j + 2), j + 2);
    h3 += tok_mix(__ldg(p + j + 3), j + 3);
  }
  for (; j < x; j++) h0 += tok_mix(__ldg(p + j), j);
  return (h0 + h1) + (h2 + h3);
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
  // child-index generation: entries of earlier chains on this worker become stale
  uint32_t g = 0;
  bool clear = false;
  if (lane == 0) {
    uint32_t* hd = C.w.hdr();
    g = hd[0] + 1;
    if (g > GEN_MAX || hd[1] != C.ncap) {
      clear = true;
      g = 1;
      hd[1] = C.ncap;
    }
    hd[0] = g;
  }
  g = __shfl_sync(FULL, g, 0);
  clear = __shfl_sync(FULL, (int)clear, 0);
  if (clear)
    for (uint32_t i = lane; i <= C.hmask; i += 32) C.w.tab()[i].key = 0;
  C.gen = g;
  __syncwarp();
  if (lane == 0) {
    NodeRec z;
    z.parent = NIL; z.hidx = NIL; z.ds = 0; z.de = 0; z.roff = 0; z.cxor = 0; z.nf = 0; z.id = 0;
    C.w.rec()[0] = z;
    d_hole(C, 0);  // the root is never a candidate and not in the bounds
  }
  uint64_t bytes = 0;
  bool bad = false;
  for (uint32_t i = lane; i < n; i += 32) {
    const mc_snap_node r = nodes[i];
    const uint32_t s = i + 1;
    const uint32_t pi = pidx[i];
    bad |= (r.d_end <= r.d_start) || (r.ref_off + r.d_end > P.n_tok) || (pi != NIL && pi >= n);
    if (C.block) bad |= (r.d_end - r.d_start != C.block) || (r.d_start % C.block) || !r.has_ssm;
    NodeRec R;
    R.parent = (pi == NIL) ? 0u : pi + 1;
    R.hidx = NIL;
    R.ds = r.d_start;
    R.de = r.d_end;
    R.roff = (uint32_t)r.ref_off;
    R.cxor = 0;
    R.nf = (r.has_ssm ? F_SSM : 0u) << 24;
    R.id = r.id;
    C.w.rec()[s] = R;
    bytes += node_bytes(C.K->m, r.d_start, r.d_end, r.has_ssm);
  }
  __syncwarp();
  for (uint32_t i = lane; i < n; i += 32) {
    const uint32_t s = i + 1;
    const NodeRec& R = C.w.rec()[s];
    const uint32_t ps = R.parent;
    // child-index key token: the edge's first token (Marconi) or the block's content hash (vLLM+)
    const uint32_t ft = C.block ? block_hash_1(P.tok + R.roff + R.ds, C.block) : P.tok[(uint64_t)R.roff + R.ds];
    atomicAdd(&C.w.rec()[ps].nf, 1u);
    atomicXor(&C.w.rec()[ps].cxor, s);
    uint32_t j = hslot(ps, ft, C.hmask);
    const uint32_t nk = hkey(C, ps, s);
    for (;;) {
      const uint32_t k = atomicAdd(&C.w.tab()[j].key, 0u);  // coherent read (lanes insert concurrently)
      if (hvalid(C, k)) { j = (j + 1) & C.hmask; continue; }
      if (atomicCAS(&C.w.tab()[j].key, k, nk) == k) break;
    }
    C.w.rec()[s].hidx = j;
    HEnt& E = C.w.tab()[j];
    E.tok = ft;
    E.de = R.de | (((R.nf >> 24) & F_SSM) ? 0x80000000u : 0u);
    E.roff = R.roff;
  }
  __syncwarp();
  bool bad_t = false;
  for (uint32_t i = lane; i < n; i += 32) {
    const uint32_t s = i + 1;
    const NodeRec R = C.w.rec()[s];
    const double v = node_eff(C.K->m, R.ds, R.de, (R.nf >> 24) & F_SSM);
    DenseRec* d = d_ptr(C, s);
    d->tc = nodes[i].t_last | ((R.nf & NCH_MASK) >= C.mthr ? D_MULTI : 0u);
    // vLLM+ keeps the node id in the second dense word (LRU key (t, id)); Marconi RN32(eff)
    d->e32 = C.block ? __uint_as_float(nodes[i].id) : __double2float_rn(v);
    // vLLM+ trees keep t_last(parent) >= t_last(child) (whole paths are touched); the
    // batched LRU eviction relies on it, so a snapshot violating it is rejected
    if (C.block && pidx[i] != NIL && nodes[pidx[i]].t_last < nodes[i].t_last) bad_t = true;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) bytes += __shfl_xor_sync(FULL, (unsigned long long)bytes, o);
  if (__any_sync(FULL, bad || bad_t)) {
    if (lane == 0) atomicOr(P.status, ST_INVARIANT);
    C.failed = true;
  }
  C.total = bytes;
  C.count = n;
  C.next_id = nid;
  C.hwm = n + 1;
  C.nfree = 0;
  C.bc_valid = 0;
  __syncwarp();
}

// Live pass: write the current tree as snapshot k (dense order, parent positions).
// Write the state load_snapshot just built (with S = 0: the whole dense list in the
// global tail) as a snapshot image at dst, including the exact normalisation bounds a
// first victim selection would compute (so chains start with the bound cache valid).
__device__ void export_image(Chain& C, char* dst) {
  const uint32_t lane = lane_id();
  const uint32_t n = C.count;
  uint32_t tmn = 0xFFFFFFFFu, tmx = 0;
  float lo = __int_as_float(0x7F800000), hi = 0.0f;
  double elo = __longlong_as_double(0x7FF0000000000000ll), ehi = 0.0;
  const DenseRec* dense = C.w.tail();
  for (uint32_t i = lane + 1; i <= n; i += 32) {  // slots 1..n (slot 0 = root hole)
    const DenseRec d = dense[i];
    const uint32_t t = d.tc & T_MASK;
    tmn = min(tmn, t);
    tmx = max(tmx, t);
    lo = fminf(lo, d.e32);
    hi = fmaxf(hi, d.e32);
    const double e = d_eff(C, i);
    elo = e < elo ? e : elo;
    ehi = e > ehi ? e : ehi;
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    tmn = min(tmn, __shfl_xor_sync(FULL, tmn, o));
    tmx = max(tmx, __shfl_xor_sync(FULL, tmx, o));
    lo = fminf(lo, __shfl_xor_sync(FULL, lo, o));
    hi = fmaxf(hi, __shfl_xor_sync(FULL, hi, o));
    const double a = __shfl_xor_sync(FULL, elo, o), b = __shfl_xor_sync(FULL, ehi, o);
    elo = a < elo ? a : elo;
    ehi = b > ehi ? b : ehi;
  }
  // records (with ids) and dense, by slot
  NodeRec* rec = (NodeRec*)(dst + 64);
  DenseRec* dn = (DenseRec*)(dst + img_off_dense(n));
  for (uint32_t i = lane; i <= n; i += 32) {
    rec[i] = C.w.rec()[i];
    dn[i] = dense[i];
  }
  // occupied child-index slots of this generation, compacted in slot order
  uint32_t* tpos = (uint32_t*)(dst + img_off_tpos(n));
  HEnt* tent = (HEnt*)(dst + img_off_tent(n));
  uint32_t w = 0;
  for (uint32_t base = 0; base <= C.hmask; base += 128) {  // 4 loads in flight per lane
    HEnt e[4];
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const uint32_t j = base + 32 * q + lane;
      if (j <= C.hmask) e[q] = C.w.tab()[j]; else e[q].key = 0;
    }
#pragma unroll
    for (int q = 0; q < 4; q++) {
      const uint32_t j = base + 32 * q + lane;
      const bool occ = hvalid(C, e[q].key);
      const unsigned b = __ballot_sync(FULL, occ);
      if (occ) {
        const uint32_t k = w + __popc(b & ((1u << lane) - 1u));
        tpos[k] = j;
        tent[k] = e[q];
      }
      w += __popc(b);
    }
  }
  if (lane == 0) {
    ImgHdr h;
    h.total = C.total;
    h.n = n;
    h.nid = C.next_id;
    h.tmin = tmn; h.tmax = tmx;
    h.lo32 = lo; h.hi32 = hi;
    h.elo = elo; h.ehi = ehi;
    h.bc_valid = (n > 0 && w == n && !C.failed) ? 1u : 0u;
    h.pad0 = w; h.pad1 = 0; h.pad2 = (C.failed || w != n) ? 1u : 0u;  // pad2: unusable image
    *(ImgHdr*)dst = h;
  }
  __syncwarp();
}

// ---- TMA bulk copy (global -> shared) completing on an mbarrier: the dense list of a
// chain's snapshot image lands in shared memory without passing through registers ----
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// one lane: arm the barrier with the byte count and start the copy (16 B aligned, size % 16 == 0)
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // order earlier generic accesses first
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_addr(dst)),
               "l"(src), "r"(bytes), "r"(smem_addr(bar))
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t phase) {
  uint32_t ok = 0;
  do {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(ok)
        : "r"(smem_addr(bar)), "r"(phase)
        : "memory");
  } while (!ok);
}

#ifndef MC_COPY_UNROLL
#define MC_COPY_UNROLL 1
#endif
constexpr int kCopyU = MC_COPY_UNROLL;  // loads in flight per lane in the image copies
// Warp copy of n 16-byte words with kCopyU loads in flight per lane (latency-bound otherwise).
__device__ __forceinline__ void warp_copy16(uint4* __restrict__ d, const uint4* __restrict__ s, uint32_t n) {
  const uint32_t lane = lane_id();
  for (uint32_t b = 0; b < n; b += 32 * kCopyU) {
    uint4 v[kCopyU];
#pragma unroll
    for (int q = 0; q < kCopyU; q++) {
      const uint32_t i = b + 32 * q + lane;
      if (i < n) v[q] = __ldcs(s + i);
    }
#pragma unroll
    for (int q = 0; q < kCopyU; q++) {
      const uint32_t i = b + 32 * q + lane;
      if (i < n) d[i] = v[q];
    }
  }
}

// The copies of load_image, out of line: its unrolled loads need registers the replay
// loop's allocation should not pay for (plain arguments, so the Chain stays in registers).
__device__ __forceinline__ void copy_image(const WS w, DenseRec* sd, uint32_t S, const char* __restrict__ src,
                                        uint32_t n, uint32_t g) {
  const uint32_t lane = lane_id();
  warp_copy16((uint4*)w.rec(), (const uint4*)(src + 64), 2 * (n + 1));
  // dense list: the shared-memory part [0, ns) by one bulk copy on the TMA engine (its
  // 16-byte multiple; an odd last entry by lane 0) while the warp copies the rest; the
  // copy completes on the warp's mbarrier (at sd + S + 12, its phase word beside it)
  const uint32_t m = n + 1, ns = min(m, S);  // slots 0..n
  const DenseRec* dn = (const DenseRec*)(src + img_off_dense(n));
  const uint32_t nb = (ns * 8u) & ~15u;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sd + S + 12);
  uint32_t* phase = reinterpret_cast<uint32_t*>(sd + S + 13);
  uint32_t ph = 0;
  if (lane == 0) {
    ph = *phase;
    if (nb) {
      bulk_g2s(sd, dn, nb, bar);
      *phase = ph ^ 1u;
    }
    if (nb / 8 < ns) sd[ns - 1] = dn[ns - 1];
  }
  for (uint32_t i = ns + lane; i < m; i += 32) w.tail()[i] = dn[i];
  {
    const uint32_t* tpos = (const uint32_t*)(src + img_off_tpos(n));
    const HEnt* tent = (const HEnt*)(src + img_off_tent(n));
    for (uint32_t b = 0; b < n; b += 32 * kCopyU) {
      HEnt e[kCopyU];
      uint32_t tp[kCopyU];
#pragma unroll
      for (int q = 0; q < kCopyU; q++) {
        const uint32_t i = b + 32 * q + lane;
        if (i < n) { e[q] = tent[i]; tp[q] = tpos[i]; }
      }
#pragma unroll
      for (int q = 0; q < kCopyU; q++) {
        const uint32_t i = b + 32 * q + lane;
        if (i < n) {
          e[q].key = (e[q].key & 0x0FFFFFFFu) | (g << 28);
          w.tab()[tp[q]] = e[q];
        }
      }
    }
  }
  ph = __shfl_sync(FULL, ph, 0);
  if (nb) {
    mbar_wait(bar, ph);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // async-proxy writes before generic reads
  }
}

// A chain's initial state from a snapshot image (replaces load_snapshot on the replay
// path): bump the child-index generation, copy the image, re-tag the copied entries.
__device__ void load_image(Chain& C, const KParams& P, const char* src) {
  const uint32_t lane = lane_id();
  const ImgHdr h = *(const ImgHdr*)src;
  const uint32_t n = h.n;
  if (n + 1 > C.ncap || h.pad2) {
    if (lane == 0) atomicOr(P.status, h.pad2 ? ST_INVARIANT : ST_OVERFLOW);
    C.failed = true;
    return;
  }
  uint32_t g = 0;
  bool clear = false;
  if (lane == 0) {
    uint32_t* hd = C.w.hdr();
    g = hd[0] + 1;
    if (g > GEN_MAX || hd[1] != C.ncap) {
      clear = true;
      g = 1;
      hd[1] = C.ncap;
    }
    hd[0] = g;
  }
  g = __shfl_sync(FULL, g, 0);
  clear = __shfl_sync(FULL, (int)clear, 0);
  if (clear)
    for (uint32_t i = lane; i <= C.hmask; i += 32) C.w.tab()[i].key = 0;
  C.gen = g;
  __syncwarp();
  copy_image(C.w, C.sd, C.S, src, n, g);
  C.total = h.total;
  C.count = n;
  C.next_id = h.nid;
  C.hwm = n + 1;
  C.nfree = 0;
  C.bc_valid = h.bc_valid ? 7u : 0u;  // the image carries exact fp64 extremes
  C.bc_tmin = h.tmin; C.bc_tmax = h.tmax;
  C.bc_lo = h.lo32; C.bc_hi = h.hi32;
  C.bc_elo = h.elo; C.bc_ehi = h.ehi;
  __syncwarp();
}

__device__ void dump_snapshot(Chain& C, const KParams& P, DevSnapOut* out, uint32_t k) {
  const uint32_t lane = lane_id();
  if (k >= out->count || C.count > out->stride) {
    if (lane == 0) atomicOr(P.status, ST_SNAPOVF);
    C.failed = true;
    return;
  }
  mc_snap_node* dst = out->nodes + (uint64_t)k * out->stride;
  uint32_t* pdst = out->pidx + (uint64_t)k * out->stride;
  // output index of every live slot (slot order), kept in the scratch map
  uint32_t* map = C.w.scratch();
  uint32_t w = 0;
  for (uint32_t b = 0; b < C.hwm; b += 32) {
    const uint32_t s = b + lane;
    const bool live = s < C.hwm && d_tc(C, s) != HOLE_TC;
    const unsigned bl = __ballot_sync(FULL, live);
    if (live) map[s] = w + __popc(bl & ((1u << lane) - 1u));
    w += __popc(bl);
  }
  __syncwarp();
  for (uint32_t s = lane; s < C.hwm; s += 32) {
    if (d_tc(C, s) == HOLE_TC) continue;
    const uint32_t i = map[s];
    const NodeRec R = C.w.rec()[s];
    const uint32_t p = R.parent;
    mc_snap_node r;
    r.id = R.id;
    r.parent_id = (p == 0) ? 0u : C.w.rec()[p].id;
    r.ref_off = R.roff;
    r.d_start = R.ds;
    r.d_end = R.de;
    r.t_last = d_tc(C, s) & T_MASK;
    r.has_ssm = ((R.nf >> 24) & F_SSM) ? 1u : 0u;
    dst[i] = r;
    pdst[i] = (p == 0) ? NIL : map[p];
  }
  if (lane == 0) {
    out->off[k] = (uint64_t)k * out->stride;
    out->n[k] = C.count;
    out->nid[k] = C.next_id;
  }
  __syncwarp();
}

// Long compares (up to 32k-token contexts): beyond the
// first round trip's 32 * kB tokens, lane 0 asks the TMA engine to prefetch the rest of
// both ranges into L2 (cp.async.bulk.prefetch.L2: one instruction per range, any size),
// so the following round trips hit L2 instead of DRAM.
__device__ __forceinline__ void bulk_prefetch_l2(const uint32_t* tok, uint64_t t0, uint64_t t1, uint64_t n_tok) {
  t0 &= ~3ull;                                   // 16-byte aligned start
  t1 = min((t1 + 3) & ~3ull, n_tok & ~3ull);     // 16-byte multiple, inside the pool
  if (t1 > t0)
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(tok + t0), "r"((uint32_t)(4 * (t1 - t0)))
                 : "memory");
}

// Warp-cooperative first mismatch of tok[a..a+cmp) vs tok[b..b+cmp) (n_tok: pool size).
__device__ __forceinline__ uint32_t match_len(const uint32_t* __restrict__ tok, uint64_t a, uint64_t b,
                                              uint32_t cmp, uint64_t n_tok) {
  if (a == b) return cmp;  // same pool range: identical tokens
  const uint32_t lane = lane_id();
#ifndef MC_MATCH_BLOCKS
#define MC_MATCH_BLOCKS 8
#endif
  constexpr int kB = MC_MATCH_BLOCKS;  // 32-token blocks compared per round trip
  if (cmp > 32 * kB && lane == 0) {
    bulk_prefetch_l2(tok, a + 32 * kB, a + cmp, n_tok);
    bulk_prefetch_l2(tok, b + 32 * kB, b + cmp, n_tok);
  }
  for (uint32_t base = 0; base < cmp; base += 32 * kB) {
    unsigned mis[kB];
#pragma unroll
    for (int q = 0; q < kB; q++) {
      const uint32_t j = base + 32 * q + lane;
      bool bad = false;
      if (j < cmp) bad = __ldg(tok + a + j) != __ldg(tok + b + j);
      mis[q] = __ballot_sync(FULL, bad);
    }
#pragma unroll
    for (int q = 0; q < kB; q++)
      if (mis[q]) return base + 32 * q + (__ffs(mis[q]) - 1);
  }
  return cmp;
}

#ifndef MC_UNROLL
#define MC_UNROLL 4
#endif
constexpr int kUnroll = MC_UNROLL;

// Development build (-DMC_PHASE_TIMERS): the 4 per-chain counters record clock64
// cycles spent in walk / plan+evict / insert / unpin+outputs instead.
#ifdef MC_PHASE_TIMERS
#define PHASE_T0() long long _pt = clock64()
#define PHASE_MARK(ctr) do { long long _n = clock64(); ctr += (unsigned long long)(_n - _pt); _pt = _n; } while (0)
#else
#define PHASE_T0() do {} while (0)
#define PHASE_MARK(ctr) do {} while (0)
#endif

// Visit every dense position i < cnt as f(q, i, tc, e32), q = unroll slot (so callers can
// keep kUnroll independent accumulator sets): shared-memory part first, then the global
// tail.  Full blocks of 32*kUnroll positions run without bounds checks.
template <class F>
__device__ __forceinline__ void scan_block(const DenseRec* __restrict__ d, uint32_t lo, uint32_t hi, F&& f) {
  const uint32_t lane = lane_id();
  uint32_t base = lo;
  for (; base + 32 * kUnroll <= hi; base += 32 * kUnroll) {
    DenseRec r[kUnroll];
#pragma unroll
    for (int q = 0; q < kUnroll; q++) r[q] = d[base + 32 * q + lane];
#pragma unroll
    for (int q = 0; q < kUnroll; q++) f(q, base + 32 * q + lane, r[q].tc, r[q].e32);
  }
  for (; base < hi; base += 32) {
    const uint32_t i = base + lane;
    if (i < hi) {
      const DenseRec r = d[i];
      f(0, i, r.tc, r.e32);
    }
  }
}
// Visit every dense position i < cnt as f(q, i, tc, e32), q = unroll slot (callers keep
// kUnroll independent accumulator sets): shared-memory part first, then the global tail.
template <class F>
__device__ __forceinline__ void scan_dense(const Chain& C, uint32_t cnt, F&& f) {
  const uint32_t ns = min(cnt, C.S);
  scan_block(C.sd, 0, ns, f);
  if (cnt > ns) scan_block(C.w.tail(), ns, cnt, f);
}

// Cold paths of the victim selection, kept out of line (instruction cache).
// (rec, m: the exact eff of a slot is recomputed from its record, rec_eff)
__device__ __noinline__ double2 recover_extremes(const DenseRec* sd, const DenseRec* tail, const NodeRec* rec,
                                                 const DevModel m, uint32_t cnt, uint32_t S, float lo32, float hi32) {
  const uint32_t lane = lane_id();
  double elo = __longlong_as_double(0x7FF0000000000000ll), ehi = 0.0;
  for (uint32_t i = lane; i < cnt; i += 32) {
    const float e = (i < S ? sd[i] : tail[i]).e32;
    if (e == lo32 || e == hi32) {
      const double x = rec_eff(m, rec[i]);
      if (e == lo32) elo = fmin(elo, x);
      if (e == hi32) ehi = fmax(ehi, x);
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    const double xl = __shfl_xor_sync(FULL, elo, o), xh = __shfl_xor_sync(FULL, ehi, o);
    elo = xl < elo ? xl : elo;
    ehi = xh > ehi ? xh : ehi;
  }
  return make_double2(elo, ehi);
}
__device__ __noinline__ Best exact_select(const DenseRec* sd, const DenseRec* tail, const NodeRec* rec,
                                          const DevModel m, uint32_t cnt, uint32_t S, Bounds b, double alpha) {
  const uint32_t lane = lane_id();
  Best best;
  best_init(best);
  for (uint32_t i = lane; i < cnt; i += 32) {
    const uint32_t tc = (i < S ? sd[i] : tail[i]).tc;
    if (tc & D_FLAGS) continue;
    const NodeRec R = rec[i];
    const double u = utility(b, tc, rec_eff(m, R), alpha);
    const uint32_t id = R.id;
    if (best.i == NIL || better(u, tc, id, best)) {
      best.u = u; best.t = tc; best.id = id; best.i = i;
    }
  }
  best_reduce(best);
  return best;
}

// Pass 1 of the α > 0 selection (cold: only when the bound cache was invalidated, ~7 % of
// requests), out of line to keep it out of the hot loop's instruction footprint: exact t
// bounds and fp32 eff bounds over every non-root node (R1; holes excluded).
struct Bounds32 {
  uint32_t tmin, tmax;
  float lo, hi;
};
__device__ __noinline__ Bounds32 bounds_pass(const DenseRec* sd, const DenseRec* tail, uint32_t cnt, uint32_t S) {
  uint32_t tmn[kUnroll], tmx[kUnroll];
  float lo[kUnroll], hi[kUnroll];
#pragma unroll
  for (int q = 0; q < kUnroll; q++) {
    tmn[q] = 0xFFFFFFFFu; tmx[q] = 0; lo[q] = __int_as_float(0x7F800000); hi[q] = 0.0f;
  }
  auto f = [&](int q, uint32_t, uint32_t tc, float e) {
    const uint32_t t = tc & T_MASK;
    tmn[q] = min(tmn[q], t);
    tmx[q] = max(tmx[q], tc == HOLE_TC ? 0u : t);
    lo[q] = fminf(lo[q], e);
    hi[q] = fmaxf(hi[q], e);
  };
  const uint32_t ns = min(cnt, S);
  scan_block(sd, 0, ns, f);
  if (cnt > ns) scan_block(tail, ns, cnt, f);
  Bounds32 r;
  r.tmin = tmn[0]; r.tmax = tmx[0]; r.lo = lo[0]; r.hi = hi[0];
#pragma unroll
  for (int q = 1; q < kUnroll; q++) {
    r.tmin = min(r.tmin, tmn[q]); r.tmax = max(r.tmax, tmx[q]); r.lo = fminf(r.lo, lo[q]); r.hi = fmaxf(r.hi, hi[q]);
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    r.tmin = min(r.tmin, __shfl_xor_sync(FULL, r.tmin, o));
    r.tmax = max(r.tmax, __shfl_xor_sync(FULL, r.tmax, o));
    r.lo = fminf(r.lo, __shfl_xor_sync(FULL, r.lo, o));
    r.hi = fmaxf(r.hi, __shfl_xor_sync(FULL, r.hi, o));
  }
  return r;
}

// α = 0 with the oldest t shared by several candidates: the one with the smallest id.
__device__ __noinline__ uint32_t lru_tiebreak(const DenseRec* sd, const DenseRec* tail, const NodeRec* rec,
                                              uint32_t cnt, uint32_t S, uint32_t t) {
  const uint32_t lane = lane_id();
  uint32_t bid = 0xFFFFFFFFu, bi = NIL;
  for (uint32_t i = lane; i < cnt; i += 32) {
    const uint32_t tc = (i < S ? sd[i] : tail[i]).tc;
    if (!(tc & D_FLAGS) && tc == t) {
      const uint32_t id = rec[i].id;
      if (id < bid) { bid = id; bi = i; }
    }
  }
  uint32_t m = bid;
#pragma unroll
  for (int o = 16; o; o >>= 1) m = min(m, __shfl_xor_sync(FULL, m, o));
  const unsigned w = __ballot_sync(FULL, bid == m && bi != NIL);
  return __shfl_sync(FULL, bi, __ffs(w) - 1);
}

// Exact victim selection over the dense live list (Eq. 2).
//   α = 0: u = rec exactly and rec is strictly monotone in t, so the victim is the
//          candidate with the smallest (t_last, id) -- one integer pass (LRU).
//   α > 0: pass 1 -- exact t bounds and fp32 eff bounds (RN32 is monotone, so the exact
//          fp64 extremes are among the entries whose fp32 value equals the fp32 extreme;
//          pass 2 reads only those fp64 values).  Pass 2 -- fp32 filter key per candidate,
//          best two per lane.  Verify -- exact IEEE utility of the entries within δ of
//          the minimum key; near-ties -> exact full pass.
__device__ __forceinline__ Best select_victim(const Chain& C, uint32_t cnt, Bounds& b, bool need_u) {
  const uint32_t lane = lane_id();
  Best best;
  best_init(best);
  bounds_init(b);
  if (C.K->alpha == 0.0) {
    // One branch-free pass: per unroll slot the smallest candidate t, its slot and whether
    // another candidate shares that t; ids are read only when the minimum t is tied.
    uint32_t bt[kUnroll], bi[kUnroll], tmn[kUnroll], tmx[kUnroll];
    bool tie[kUnroll];
#pragma unroll
    for (int q = 0; q < kUnroll; q++) {
      bt[q] = 0xFFFFFFFFu; bi[q] = NIL; tmn[q] = 0xFFFFFFFFu; tmx[q] = 0; tie[q] = false;
    }
    scan_dense(C, cnt, [&](int q, uint32_t i, uint32_t tc, float) {
      const uint32_t t = tc & T_MASK;
      tmn[q] = min(tmn[q], t);
      tmx[q] = max(tmx[q], tc == HOLE_TC ? 0u : t);
      const uint32_t k = (tc & D_FLAGS) ? 0xFFFFFFFFu : t;  // non-candidates never win
      const bool lt = k < bt[q];
      tie[q] = lt ? false : (tie[q] | (k == bt[q]));
      bi[q] = lt ? i : bi[q];
      bt[q] = lt ? k : bt[q];
    });
    uint32_t t1 = bt[0], i1 = bi[0];
    bool tied1 = tie[0];
    b.tmin = tmn[0];
    b.tmax = tmx[0];
#pragma unroll
    for (int q = 1; q < kUnroll; q++) {
      b.tmin = min(b.tmin, tmn[q]);
      b.tmax = max(b.tmax, tmx[q]);
      if (bt[q] < t1) { t1 = bt[q]; i1 = bi[q]; tied1 = tie[q]; }
      else if (bt[q] == t1) tied1 = true;
    }
    uint32_t tbest = t1;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      b.tmin = min(b.tmin, __shfl_xor_sync(FULL, b.tmin, o));
      b.tmax = max(b.tmax, __shfl_xor_sync(FULL, b.tmax, o));
      tbest = min(tbest, __shfl_xor_sync(FULL, tbest, o));
    }
    if (tbest == 0xFFFFFFFFu) return best;  // no candidate
    const unsigned at = __ballot_sync(FULL, t1 == tbest);
    const bool unique = __popc(at) == 1 && !__shfl_sync(FULL, (int)tied1, __ffs(at) - 1);
    best.t = tbest;
    if (unique) {
      best.i = __shfl_sync(FULL, i1, __ffs(at) - 1);
    } else {  // several candidates share the oldest t: smallest id (R4), cold path
      best.i = lru_tiebreak(C.sd, C.w.tail(), C.w.rec(), cnt, C.S, tbest);
    }
    best.slot = best.i;
    const double rec = (b.tmax == b.tmin) ? 0.5 : __ddiv_rn((double)(best.t - b.tmin), (double)(b.tmax - b.tmin));
    best.u = __dadd_rn(rec, __dmul_rn(0.0, 0.5));  // = rec (α·effn = +0)
    return best;
  }
#ifdef MC_PHASE_TIMERS3
  Chain& CC = const_cast<Chain&>(C);
  long long _t3 = clock64();
#define T3(ctr) do { long long _n3 = clock64(); CC.ctr += (unsigned long long)(_n3 - _t3); _t3 = _n3; } while (0)
#else
#define T3(ctr) do {} while (0)
#endif
  // pass 1: exact t bounds, fp32 eff bounds over ALL non-root nodes (R1) -- skipped when
  // the cached bounds are known exact
  uint32_t tmin, tmax;
  float lo32, hi32;
  Chain& Cw = const_cast<Chain&>(C);
  if (C.bc_valid & 1u) {
    tmin = C.bc_tmin; tmax = C.bc_tmax; lo32 = C.bc_lo; hi32 = C.bc_hi;
  } else {
    const Bounds32 bp = bounds_pass(C.sd, C.w.tail(), cnt, C.S);
    tmin = bp.tmin; tmax = bp.tmax; lo32 = bp.lo; hi32 = bp.hi;
    // the exact fp64 extremes are recovered only when a victim's exact utility is needed
    Cw.bc_valid = 1; Cw.bc_tmin = tmin; Cw.bc_tmax = tmax; Cw.bc_lo = lo32; Cw.bc_hi = hi32;
#ifdef MC_PHASE_TIMERS3
    CC.t_unpin += 1ull << 32;  // count full bound passes (high half)
#endif
  }
  b.tmin = tmin;
  b.tmax = tmax;
#ifdef MC_PHASE_TIMERS3
  _t3 = clock64();
#endif
  // pass 2: fp32 filter keys, best two per lane (branch-free), exact fp64 extremes
  const bool dt0 = tmax == tmin;
  const double de32 = (double)hi32 - (double)lo32;  // exact in fp64
  const float idt = dt0 ? 0.0f : __frcp_rn((float)(tmax - tmin));
  const float aide = (de32 == 0.0) ? 0.0f : __double2float_rn(__ddiv_rn(C.K->alpha, de32));
  const float INF = __int_as_float(0x7F800000);
  float a1[kUnroll], a2[kUnroll];
  uint32_t ai[kUnroll];
#pragma unroll
  for (int q = 0; q < kUnroll; q++) { a1[q] = INF; a2[q] = INF; ai[q] = NIL; }
  // Keys two at a time on the packed fp32x2 pipe (FADD2 / FMUL2 / FFMA2: per key the
  // same three roundings as the scalar recipe, so the filter bound is unchanged); best
  // two per lane by min/max instead of nested selects (fewer register moves in the
  // unrolled loop).  config 3: 5.06 -> 4.92 ms in A/B (profiles/r02o_pass2_ab.txt).
  static_assert(kUnroll % 2 == 0, "pass 2 pairs the unrolled loads");
  {
    const unsigned long long lo2 = ((unsigned long long)__float_as_uint(lo32) << 32) | __float_as_uint(lo32);
    const unsigned long long ae2 = ((unsigned long long)__float_as_uint(aide) << 32) | __float_as_uint(aide);
    const unsigned long long it2 = ((unsigned long long)__float_as_uint(idt) << 32) | __float_as_uint(idt);
    auto pair = [&](int q, uint32_t i0, const DenseRec r0, const DenseRec r1) {
      unsigned long long e2 = ((unsigned long long)__float_as_uint(r1.e32) << 32) | __float_as_uint(r0.e32);
      unsigned long long t2 = ((unsigned long long)__float_as_uint(__uint2float_rn(r1.tc - tmin)) << 32) |
                              __float_as_uint(__uint2float_rn(r0.tc - tmin));
      unsigned long long k2;
      asm("sub.rn.f32x2 %0, %0, %1;" : "+l"(e2) : "l"(lo2));
      asm("mul.rn.f32x2 %0, %0, %1;" : "+l"(t2) : "l"(it2));
      asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(k2) : "l"(e2), "l"(ae2), "l"(t2));
      const float k0 = (r0.tc & D_FLAGS) ? INF : __uint_as_float((uint32_t)k2);
      const float k1 = (r1.tc & D_FLAGS) ? INF : __uint_as_float((uint32_t)(k2 >> 32));
      a2[q] = fminf(a2[q], fmaxf(a1[q], k0));
      ai[q] = k0 < a1[q] ? i0 : ai[q];
      a1[q] = fminf(a1[q], k0);
      a2[q + 1] = fminf(a2[q + 1], fmaxf(a1[q + 1], k1));
      ai[q + 1] = k1 < a1[q + 1] ? i0 + 32 : ai[q + 1];
      a1[q + 1] = fminf(a1[q + 1], k1);
    };
    auto one = [&](int q, uint32_t i, uint32_t tc, float e) {
      const float k = (tc & D_FLAGS) ? INF : __fmaf_rn(__fsub_rn(e, lo32), aide, __fmul_rn(__uint2float_rn(tc - tmin), idt));
      a2[q] = fminf(a2[q], fmaxf(a1[q], k));
      ai[q] = k < a1[q] ? i : ai[q];
      a1[q] = fminf(a1[q], k);
    };
    auto blk = [&](const DenseRec* __restrict__ d, uint32_t lo, uint32_t hi) {
      uint32_t base = lo;
      for (; base + 32 * kUnroll <= hi; base += 32 * kUnroll) {
        DenseRec r[kUnroll];
#pragma unroll
        for (int q = 0; q < kUnroll; q++) r[q] = d[base + 32 * q + lane];
#pragma unroll
        for (int q = 0; q < kUnroll; q += 2) pair(q, base + 32 * q + lane, r[q], r[q + 1]);
      }
      for (; base < hi; base += 32) {
        const uint32_t i = base + lane;
        if (i < hi) { const DenseRec r = d[i]; one(0, i, r.tc, r.e32); }
      }
    };
    const uint32_t ns = min(cnt, C.S);
    blk(C.sd, 0, ns);
    if (cnt > ns) blk(C.w.tail(), ns, cnt);
  }

  // merge the per-slot best-two lists
  float k1 = a1[0], k2 = a2[0];
  uint32_t i1 = ai[0];
#pragma unroll
  for (int q = 1; q < kUnroll; q++) {
    if (a1[q] < k1) { k2 = fminf(k1, a2[q]); k1 = a1[q]; i1 = ai[q]; }
    else { k2 = fminf(k2, a1[q]); }
  }
  float kmin = k1;
#pragma unroll
  for (int o = 16; o; o >>= 1) kmin = fminf(kmin, __shfl_xor_sync(FULL, kmin, o));
  T3(t_evict);
  // exact fp64 extremes (lazily, the fp64 values of the entries holding the fp32 extremes)
#define ENSURE_EXTREMES()                                                                  \
  do {                                                                                     \
    if ((C.bc_valid & 6u) != 6u) {                                                         \
      const double2 ex = recover_extremes(C.sd, C.w.tail(), C.w.rec(), C.K->m, cnt, C.S, lo32, hi32); \
      Cw.bc_elo = ex.x; Cw.bc_ehi = ex.y; Cw.bc_valid |= 6u;                               \
    }                                                                                      \
    b.emin = C.bc_elo; b.emax = C.bc_ehi;                                                  \
  } while (0)
  // No finite filter key: either no candidate at all (exact_select then reports none) or
  // an α so large that α/Δe32 or the key overflows fp32 (0 * inf = NaN keys never win the
  // comparisons): the exact fp64 pass decides, as the oracle does for any finite α.
  if (!(kmin < INF)) {
    ENSURE_EXTREMES();
    return exact_select(C.sd, C.w.tail(), C.w.rec(), C.K->m, cnt, C.S, b, C.K->alpha);
  }
  // δ = 2^-19 (1 + α (1 + 4 emax/Δe32)); a zero fp32 range cannot resolve eff -> exact pass
  if (de32 == 0.0) ENSURE_EXTREMES();
  const bool exact_only = (de32 == 0.0) && (b.emax != b.emin);
  const double ratio = (de32 == 0.0) ? 0.0 : __ddiv_rn((double)hi32, de32);
  const double delta = 1.9073486328125e-06 * (1.0 + C.K->alpha * (1.0 + 4.0 * ratio));
  const double lim = (double)kmin + delta;
  if (!exact_only && !__any_sync(FULL, (double)k2 <= lim)) {
    const bool mine = (double)k1 <= lim;
    const unsigned who = __ballot_sync(FULL, mine);
    if (__popc(who) == 1) {  // the common case: one candidate survives the filter
      const int src = __ffs(who) - 1;
      best.i = __shfl_sync(FULL, i1, src);
      best.slot = best.i;
      best.id = NIL;
      if (need_u) {  // the exact utility is only logged (no global read otherwise)
        ENSURE_EXTREMES();
        if (mine) best.u = utility(b, d_tc(C, i1), d_eff(C, i1), C.K->alpha);
        best.u = __shfl_sync(FULL, best.u, src);
      }
      return best;
    }
#ifdef MC_PHASE_TIMERS3
    CC.t_unpin += 1ull << 16;  // near-tie verifications (bits 16..31)
#endif
    ENSURE_EXTREMES();
    if (mine) {  // near-ties: exact utilities, ids for exact ties
      best.t = d_tc(C, i1);
      best.u = utility(b, best.t, d_eff(C, i1), C.K->alpha);
      best.i = i1;
      best.slot = i1;
      best.id = d_id(C, i1);
    }
    best_reduce(best);
    return best;
  }
#ifdef MC_PHASE_TIMERS3
  CC.t_unpin += 1;  // number of exact fallback passes
#endif
  // near-ties / unresolvable fp32 range: exact full pass (cold path)
  ENSURE_EXTREMES();
#undef ENSURE_EXTREMES
  return exact_select(C.sd, C.w.tail(), C.w.rec(), C.K->m, cnt, C.S, b, C.K->alpha);
}

__device__ void evict_one(Chain& C, const KParams& P, uint32_t r, mc_evict_rec* log, uint32_t* log_n) {
  const uint32_t lane = lane_id();
  const uint32_t cnt = C.count;
  Bounds b;
#ifdef MC_PHASE_TIMERS3
  long long _e3 = clock64();
#endif
  const Best best = select_victim(C, C.hwm, b, log != nullptr);
#ifdef MC_PHASE_TIMERS3
  { long long _n = clock64(); C.t_walk += (unsigned long long)(_n - _e3); _e3 = _n; }
#endif
  CTR_ADD(C, scan, cnt);
  C.n_evict++;
  if (best.i == NIL) {
    if (lane == 0) atomicOr(P.status, ST_NOCAND);
    C.failed = true;
    return;
  }
  if (lane == 0) {
    // Loads first (independent ones back to back), then the stores: every store
    // below targets fields no later load in this block reads.
    const uint32_t x = best.i;  // slot = dense position
    const NodeRec X = C.w.rec()[x];
    const uint32_t p = X.parent;
    const uint32_t xf = X.nf >> 24;
    const NodeRec Rp = C.w.rec()[p];
    const uint32_t xid = X.id;
    const DenseRec dv = *d_ptr(C, x);
    uint32_t kind;
    if ((X.nf & NCH_MASK) == 0) {  // leaf: free KVs + state
      kind = 0;
      C.total -= node_bytes(C.K->m, X.ds, X.de, xf & F_SSM);
      hash_erase_at_1(C, X.hidx);
      NodeRec& Wp = C.w.rec()[p];
      Wp.nf = Rp.nf - 1;
      Wp.cxor = Rp.cxor ^ x;
      if (p != 0) d_multi(C, p, (Rp.nf & NCH_MASK) - 1);
      CTR_ADD(C, wr, 1);
    } else {  // one child: release the state, the child absorbs the KVs
      kind = 1;
      const uint32_t c = X.cxor;
      const NodeRec Rc = C.w.rec()[c];
      const uint32_t hc = Rc.hidx;   // entry of c under x (erased)
      const uint32_t hx = X.hidx;    // entry of x under p (becomes c's: same key)
      const uint32_t xtok = C.w.tab()[hx].tok;
      if (xf & F_SSM) C.total -= C.K->m.ssmb;
      NodeRec& Wc = C.w.rec()[c];
      Wc.ds = X.ds;
      Wc.parent = p;
      Wc.hidx = hx;
      C.w.tab()[hx] = hmake(C, p, xtok, c, Rc.de, (Rc.nf >> 24) & F_SSM, Rc.roff);
      hash_erase_at_1(C, hc);
      C.w.rec()[p].cxor = Rp.cxor ^ x ^ c;
      const double ec = node_eff(C.K->m, X.ds, Rc.de, (Rc.nf >> 24) & F_SSM);
      d_set_eff(C, c, ec);
      CTR_ADD(C, wr, 2);
    }
    if (log) {
      const uint32_t li = *log_n;
      if (li < P.log_cap) {
        mc_evict_rec e;
        e.req = r; e.node_id = xid; e.kind = kind; e.n_live = cnt; e.utility = best.u;
        log[li] = e;
      }
      *log_n = li + 1;
    }
    // the victim's slot becomes a hole (no dense entry moves)
    bc_remove(C, dv.tc & T_MASK, dv.e32);
    d_hole(C, x);
    C.count = cnt - 1;
    C.w.rec()[x].nf = 0;
    C.w.freel()[C.nfree++] = x;
  }
  sync_state(C);
#ifdef MC_PHASE_TIMERS3
  C.t_insert += (unsigned long long)(clock64() - _e3);
#endif
}

// Split node y at absolute depth x: new upper node [ds, x) takes a new id, y keeps
// its id and becomes [x, de) (R4).  Lane 0 only.
__device__ __forceinline__ uint32_t split_1(Chain& C, const KParams& P, uint32_t y, uint32_t x, bool stateful,
                                            uint32_t r) {
  const uint32_t u = alloc_1(C, P.status);
  if (u == NIL) return NIL;
  const NodeRec Y = C.w.rec()[y];
  const uint32_t cx = C.w.rec()[Y.parent].cxor;
  const uint32_t ft = P.tok[(uint64_t)Y.roff + x];
  const uint32_t hi = Y.hidx;                  // entry of y under its parent
  const uint32_t ytok = C.w.tab()[hi].tok;
  NodeRec U;
  U.parent = Y.parent; U.hidx = hi; U.ds = Y.ds; U.de = x;
  U.roff = Y.roff; U.cxor = y; U.nf = 1u | ((stateful ? F_SSM : 0u) << 24); U.id = C.next_id++;
  C.w.rec()[u] = U;
  C.w.tab()[hi] = hmake(C, Y.parent, ytok, u, x, stateful, Y.roff);  // same key, new child
  NodeRec& Ry = C.w.rec()[y];
  Ry.parent = u;
  Ry.ds = x;
  Ry.hidx = hash_insert_1(C, hmake(C, u, ft, y, Y.de, (Y.nf >> 24) & F_SSM, Y.roff), u);
  C.w.rec()[Y.parent].cxor = cx ^ y ^ u;
  dense_add_1(C, u, r);
  d_set_eff(C, y, node_eff(C.K->m, x, Y.de, (Y.nf >> 24) & F_SSM));
  CTR_ADD(C, wr, 2);
  return u;
}

__device__ __forceinline__ void gain_1(Chain& C, uint32_t x, uint32_t r) {
  NodeRec& R = C.w.rec()[x];
  const uint32_t nf = R.nf, dp = x, ds = R.ds, de = R.de, hi = R.hidx;
  R.nf = nf | (F_SSM << 24);
  C.w.tab()[hi].de = de | 0x80000000u;  // the child index carries the state flag for the walk
  d_set_eff(C, dp, node_eff(C.K->m, ds, de, true));
  d_stamp(C, dp, r);
  CTR_ADD(C, wr, 1);
}

// ---------------------------------------------------------------------------
// One request: SURVEY.md §8(c) c.2 steps 1-9.
// The path P is held lane-distributed: lane i keeps path node i (i < 32), deeper
// nodes spill to the workspace path array.
// ---------------------------------------------------------------------------
struct ReqOut {
  uint32_t reuse;
  uint64_t flops;
  bool bypass;
};

__device__ __forceinline__ uint32_t path_at(const Chain& C, uint32_t my_path, uint32_t i) {
  return i < 32 ? __shfl_sync(FULL, my_path, i) : C.w.path()[i];
}

// Software pipelining across requests: the caller passes request r's header and
// first token (loaded during request r-1); this request loads request r+1's header
// at its start, its first token after the walk, and prefetches the child-index line
// of its root lookup into L2 -- three dependent round trips off the critical path.
struct ReqHdr {
  uint32_t off, lin, lout;
};
struct Prefetched {
  ReqHdr q;
  uint32_t tk0;
};
__device__ __forceinline__ ReqHdr load_req(const KParams& P, uint32_t r) {
  const mc_request m = P.req[r - 1];
  ReqHdr h;
  h.off = (uint32_t)m.tok_off;
  h.lin = m.input_len;
  h.lout = m.output_len;
  return h;
}
__device__ __forceinline__ Prefetched fetch_request(const KParams& P, uint32_t r) {
  Prefetched f;
  f.q = load_req(P, r);
  f.tk0 = __ldg(P.tok + f.q.off);
  return f;
}

// kGen = false: the lean instantiation for chains without eviction logs, chunked
// checkpoints or n_ssm = 0 (the benchmarked grid) -- those paths compiled out, so the hot
// loop is smaller (instruction cache) and holds fewer live values.  kGen = true handles
// every chain.
template <bool kGen>
__device__ ReqOut process_request(Chain& C, const KParams& P, uint32_t r, const Prefetched cur, Prefetched& nxt,
                                  bool has_next, mc_evict_rec* log, uint32_t* log_n) {
  if (!kGen) log = nullptr;
  const uint32_t lane = lane_id();
  const ReqHdr q = cur.q;
  const uint32_t off = q.off;
  const uint32_t L_in = q.lin;
  const uint32_t n = q.lin + q.lout;
  if (has_next) nxt.q = load_req(P, r + 1);  // request r+1

  PHASE_T0();
  // Step 1: walk = lookup + speculative insertion bookkeeping.
  uint32_t v = 0, pos = 0, npath = 0, m = 0, my_path = NIL, my_ds = 0, my_de = 0, my_fl = 0, my_dp = NIL;
  uint32_t partial = NIL, hit = NIL, reuse = 0, hit_idx = NIL;
  uint32_t lin_node = NIL;   // node whose edge strictly contains L_in (when m >= L_in)
  uint32_t lin_bnd = NIL;    // fully matched node ending exactly at L_in
  uint32_t v_flags = 0, lin_bnd_flags = 0;
  uint64_t pinned_bytes = 0;
  uint32_t tk = cur.tk0;
  for (;;) {
    if (pos == n) { m = n; break; }
    const HEnt E = hash_find_warp(C, v, tk);  // one round trip per level: no record reads
    if (E.key == 0) { m = pos; break; }
    const uint32_t c = E.key & SLOT14;
    const uint32_t de = E.de & 0x7FFFFFFFu;
    const uint32_t fl = E.de >> 31;             // has_ssm
    const uint32_t len = de - pos;              // the child's edge starts at the parent's depth
    // prefetch the query token the next level will look up
    const uint32_t nt = (de < n) ? __ldg(P.tok + off + de) : 0u;
    const uint32_t cmp = min(len, n - pos);
    const uint32_t k = match_len(P.tok, (uint64_t)E.roff + pos, off + pos, cmp, P.n_tok);
    if (lane == 0 && npath >= 32) C.w.path()[npath] = c;
    if (lane == npath) {
      my_path = c; my_ds = pos; my_de = de; my_fl = fl;
      my_dp = c;  // dense position = slot
    }
    npath++;
    pinned_bytes += node_bytes(C.K->m, pos, de, fl & F_SSM);
    if (pos < L_in && L_in < pos + len && L_in <= pos + k) lin_node = c;
    if (k == len) {
      v = c;
      v_flags = fl;
      pos += len;
      tk = nt;
      if (de == L_in) { lin_bnd = c; lin_bnd_flags = fl; }
      if ((fl & F_SSM) && de <= L_in) { hit = c; reuse = de; hit_idx = npath - 1; }  // all-or-nothing (R6, R7)
    } else {
      m = pos + k;
      partial = c;
      break;
    }
  }
  __syncwarp();
  CTR_ADD(C, cmp, min(m + 1, n));
  CTR_ADD(C, vis, npath + 1);
  if (has_next) {
    nxt.tk0 = __ldg(P.tok + nxt.q.off);
    if (lane == 0) {
      const HEnt* line = C.w.tab() + hslot(0, nxt.tk0, C.hmask);
      asm volatile("prefetch.global.L2 [%0];" ::"l"(line));
    }
  }

  // Step 2: pure Transformer (n_ssm = 0): KVs can be sliced mid-edge.
  if (kGen && C.K->m.n_ssm == 0) {
    reuse = min(m, L_in);
    hit = NIL;
    hit_idx = NIL;
    for (uint32_t i = 0; i < npath; i++) {
      const uint32_t x = path_at(C, my_path, i);
      if (C.w.rec()[x].ds < reuse) { hit = x; hit_idx = i; }
    }
  }

  // Pin the path (R12) and touch only the hit node (step 5): every path
  // lane reads its node's dense position and updates its dense word in parallel.
  uint32_t old_t = 0;
  if (lane < min(npath, 32u)) {
    DenseRec* d = d_ptr(C, my_dp);
    const uint32_t tc = d->tc;
    if (lane == hit_idx) old_t = tc & T_MASK;
    d->tc = (lane == hit_idx ? (r | (tc & D_MULTI)) : tc) | D_PIN;
  }
  if (lane == 0)
    for (uint32_t i = 32; i < npath; i++) {
      DenseRec* d = d_ptr(C, C.w.path()[i]);
      if (i == hit_idx) old_t = d->tc & T_MASK;
      d->tc = (i == hit_idx ? (r | (d->tc & D_MULTI)) : d->tc) | D_PIN;
    }
  if (hit != NIL) {
    CTR_ADD(C, wr, 1);
    old_t = __shfl_sync(FULL, old_t, hit_idx < 32 ? hit_idx : 0);
    bc_change_t(C, old_t, r);  // uniform: every lane updates its copy of the bound cache
  }
  __syncwarp();

  // Step 3: speculative insertion of the input (R8, R9).
  const uint32_t m_in = min(m, L_in);
  uint32_t p = 0, p_split = NIL, p_gain = NIL;
  if (m_in > 0) {
    if (m >= L_in) {
      if (lin_bnd != NIL) {
        if (!(lin_bnd_flags & F_SSM)) { p = m_in; p_gain = lin_bnd; }
      } else {
        p = m_in;
        p_split = lin_node;
      }
    } else if (partial != NIL) {
      p = m_in;
      p_split = partial;
    } else if (!(v_flags & F_SSM)) {
      p = m_in;
      p_gain = v;
    }
  }
  // Chunked state passing (NEXT-3): the prefill checkpoint moves down to the
  // chunk boundary at or below the branch point; skipped if that is 0 or not beyond the hit.
  if (kGen && C.K->chunk && p) {
    uint32_t pa = (p / C.K->chunk) * C.K->chunk;
    if (pa == 0 || pa <= reuse) pa = 0;
    p_split = NIL;
    p_gain = NIL;
    if (pa) {
      const bool mine = lane < min(npath, 32u);
      const unsigned bnd = __ballot_sync(FULL, mine && my_de == pa && my_path != partial);
      const unsigned ins = __ballot_sync(FULL, mine && my_ds < pa && pa < my_de);
      if (bnd) {
        const int src = __ffs(bnd) - 1;
        const uint32_t x = __shfl_sync(FULL, my_path, src);
        if (__shfl_sync(FULL, my_fl, src) & F_SSM) pa = 0; else p_gain = x;
      } else if (ins) {
        p_split = __shfl_sync(FULL, my_path, __ffs(ins) - 1);
      } else {  // deeper than 32 levels: scan the spilled part of the path
        uint32_t kind = 0, x = NIL;
        if (lane == 0)
          for (uint32_t i = 32; i < npath; i++) {
            const uint32_t y = C.w.path()[i];
            const NodeRec Ry = C.w.rec()[y];
            if (y != partial && Ry.de == pa) { kind = ((Ry.nf >> 24) & F_SSM) ? 3 : 1; x = y; break; }
            if (Ry.ds < pa && pa < Ry.de) { kind = 2; x = y; break; }
          }
        kind = __shfl_sync(FULL, kind, 0);
        x = __shfl_sync(FULL, x, 0);
        if (kind == 1) p_gain = x;
        else if (kind == 2) p_split = x;
        else pa = 0;
      }
    }
    p = pa;
  }
  // Step 4: plan -- checkpoints {p, n}, at most two.
  const bool leaf = m < n;
  const bool split_m = partial != NIL && m < n && m != p;   // stateless output-region split (R10)
  const bool split_n = partial != NIL && m == n && n != p;  // sequence ends inside an edge
  uint32_t n_gain = NIL;
  if (partial == NIL && m == n && n != p && !(v_flags & F_SSM)) n_gain = v;
  uint32_t n_ck = p ? 1u : 0u;
  if (n != p && (leaf || split_n || n_gain != NIL)) n_ck++;
  const uint64_t d_bytes = C.K->m.kvt * (uint64_t)(n - m) + C.K->m.ssmb * n_ck;
  const uint32_t d_nodes = (p_split != NIL ? 1u : 0u) + (split_m ? 1u : 0u) + (split_n ? 1u : 0u) + (leaf ? 1u : 0u);

  PHASE_MARK(C.t_walk);

  // Step 6: admission precheck (R12).
  const bool bypass = (pinned_bytes + d_bytes > C.K->capb) || (C.K->capn && npath + d_nodes > C.K->capn);
  if (!bypass) {
    // Step 7: evict the argmin utility until the request fits.
    while (!C.failed && (C.total + d_bytes > C.K->capb || (C.K->capn && C.count + d_nodes > C.K->capn))) {
      evict_one(C, P, r, log, log_n);
    }
    PHASE_MARK(C.t_evict);
    // Step 8: insert.
    if (lane == 0 && !C.failed) {
      uint32_t attach = v;  // node at depth m after the splits
      // splits in depth order: p_split at p (stateful), partial at m (stateless), partial
      // at n (stateful); one loop keeps a single inlined copy of split_1 (code size)
      unsigned todo = (p_split != NIL ? 1u : 0u) | (split_m ? 2u : 0u) | (split_n ? 4u : 0u);
      while (todo) {
        const int k = __ffs(todo) - 1;
        todo &= todo - 1;
        const uint32_t x = k == 0 ? p : (k == 1 ? m : n);
        const uint32_t u = split_1(C, P, k == 0 ? p_split : partial, x, k != 1, r);
        if (k < 2 && x == m) attach = u;
        if (C.failed) break;
      }
      unsigned gains = (p_gain != NIL ? 1u : 0u) | (n_gain != NIL ? 2u : 0u);
      while (gains) {
        const uint32_t g = (gains & 1u) ? p_gain : n_gain;
        gains &= gains - 1;
        gain_1(C, g, r);
      }
      if (leaf && !C.failed) {
        const uint32_t w = alloc_1(C, P.status);
        if (w != NIL) {
          const uint32_t ft = P.tok[off + m];
          const NodeRec Ra = C.w.rec()[attach];
          NodeRec W;
          W.parent = attach; W.hidx = NIL; W.ds = m; W.de = n;
          W.roff = (uint32_t)off; W.cxor = 0; W.nf = F_SSM << 24; W.id = C.next_id++;
          C.w.rec()[w] = W;
          C.w.rec()[w].hidx = hash_insert_1(C, hmake(C, attach, ft, w, n, true, (uint32_t)off), attach);
          NodeRec& Wa = C.w.rec()[attach];
          Wa.nf = Ra.nf + 1;
          Wa.cxor = Ra.cxor ^ w;
          if (attach != 0) d_multi(C, attach, (Ra.nf & NCH_MASK) + 1);
          dense_add_1(C, w, r);
          CTR_ADD(C, wr, 1);
        }
      } else if (partial == NIL) {
        // final node at n already exists: timestamp it (R5)
        d_stamp(C, v, r);
        if (n_gain == NIL && p_gain != v) CTR_ADD(C, wr, 1);
      }
      C.total += d_bytes;
      if (C.total > C.K->capb || (C.K->capn && C.count > C.K->capn)) {
        atomicOr(P.status, ST_INVARIANT);
        C.failed = true;
      }
    }
    sync_state(C);
  }
  PHASE_MARK(C.t_insert);
  // Step 9: unpin (every path lane clears its node's pin bit in parallel), outputs.
  if (lane < min(npath, 32u)) {
    DenseRec* d = d_ptr(C, my_dp);
    d->tc &= ~D_PIN;
  }
  if (lane == 0) {
    for (uint32_t i = 32; i < npath; i++) {
      DenseRec* d = d_ptr(C, C.w.path()[i]);
      d->tc &= ~D_PIN;
    }
    if (reuse > L_in) {
      atomicOr(P.status, ST_INVARIANT);
      C.failed = true;
    }
  }
  sync_state(C);
  PHASE_MARK(C.t_unpin);
  ReqOut o;
  o.reuse = reuse;
  o.flops = prefill_F(C.K->m, reuse);
  o.bypass = bypass;
  return o;
}

// ---------------------------------------------------------------------------
// vLLM+ baseline (readings V1-V8): a state per
// token block, vLLM's LRU policy.  Every full block of a
// sequence is one node; its child-index key is (parent, content hash) and every
// hash match is verified against the tokens.  Same workspace, dense list, victim
// selection (α = 0 LRU pass over leaf blocks) and removal as the Marconi path.
// ---------------------------------------------------------------------------

// Child of `parent` whose block equals tokens[b0, b0 + x) (hash h), or NIL.  Walks
// the probe sequence line by line; every (parent, h) match is verified with a token
// compare (collisions are skipped, so the result is exact).
__device__ __forceinline__ uint32_t child_block(const Chain& C, const KParams& P, uint32_t parent, uint32_t h,
                                                uint64_t b0, uint32_t kx) {
  const uint32_t lane = lane_id();
  const HEnt* __restrict__ tab = C.w.tab();
  const uint32_t x = C.block;
  uint32_t i0 = hslot(parent, h, C.hmask);
  for (uint32_t seen = 0; seen <= C.hmask;) {
    const uint32_t lim = (i0 | 7u) - i0 + 1;
    const bool act = lane < lim;
    HEnt e;
    e.tok = 0; e.key = 0; e.de = 0; e.roff = 0;
    if (act) e = tab[i0 + lane];
    const bool valid = act && hvalid(C, e.key);
    const unsigned me = __ballot_sync(FULL, act && !valid);
    unsigned mm = __ballot_sync(FULL, valid && hmatch(e, parent, h));
    if (me) mm &= (1u << (__ffs(me) - 1)) - 1u;  // only entries before the first empty slot
    while (mm) {
      const int fm = __ffs(mm) - 1;
      mm &= mm - 1;
      const uint32_t roff = __shfl_sync(FULL, e.roff, fm);
      const uint32_t key = __shfl_sync(FULL, e.key, fm);
      if (match_len(P.tok, (uint64_t)roff + kx, b0, x, P.n_tok) == x) return key & SLOT14;
    }
    if (me) return NIL;
    seen += lim;
    i0 = (i0 + lim) & C.hmask;
  }
  return NIL;
}

// vLLM+ LRU eviction of `need` leaf blocks (V6), batched: one scan keeps each lane's
// K smallest candidate keys (t_last << 32 | id) and W = a lower bound of every key not
// kept; victims are then extracted in exact (t, id) order while the smallest kept key is
// below W.  A removal can expose the parent as a new candidate (its last child gone):
// it joins the kept keys (or is covered by W).  Because whole paths are touched, t(parent)
// >= t(child) and the global t minimum is always the victim's, so the logged utility
// (Eq. 2 at α = 0) is 0, or 0.5 when every node shares t.  Same victims, order, log and
// counters as one full scan per eviction.
__device__ void evict_lru_blocks(Chain& C, const KParams& P, uint32_t r, uint32_t need, mc_evict_rec* log,
                                 uint32_t* log_n) {
  constexpr int K = 4;
  const uint64_t INF64 = ~0ull;
  const uint32_t lane = lane_id();
  while (need && !C.failed) {
    uint64_t key[K];
    uint32_t pos[K];
#pragma unroll
    for (int q = 0; q < K; q++) { key[q] = INF64; pos[q] = NIL; }
    uint64_t wl = INF64;
    uint32_t tmax = 0;
    scan_dense(C, C.hwm, [&](int, uint32_t i, uint32_t tc, float e) {
      tmax = max(tmax, tc == HOLE_TC ? 0u : (tc & T_MASK));
      if (tc & D_FLAGS) return;
      const uint64_t k = ((uint64_t)(tc & T_MASK) << 32) | __float_as_uint(e);
      if (k < key[K - 1]) {
        wl = min(wl, key[K - 1]);  // the dropped key (INF64 while the list is not full)
        key[K - 1] = k;
        pos[K - 1] = i;
#pragma unroll
        for (int q = K - 1; q > 0; q--) {
          if (key[q] < key[q - 1]) {
            const uint64_t tk = key[q]; key[q] = key[q - 1]; key[q - 1] = tk;
            const uint32_t tp = pos[q]; pos[q] = pos[q - 1]; pos[q - 1] = tp;
          }
        }
      } else {
        wl = min(wl, k);
      }
    });
    uint64_t W = wl;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      W = min(W, (uint64_t)__shfl_xor_sync(FULL, (unsigned long long)W, o));
      tmax = max(tmax, __shfl_xor_sync(FULL, tmax, o));
    }
    bool progressed = false;
    while (need) {
      uint64_t m = key[0];
#pragma unroll
      for (int o = 16; o; o >>= 1) m = min(m, (uint64_t)__shfl_xor_sync(FULL, (unsigned long long)m, o));
      if (m == INF64 || m >= W) break;  // the next victim may be unlisted: rescan
      const int src = __ffs(__ballot_sync(FULL, key[0] == m)) - 1;
      const uint32_t vpos = __shfl_sync(FULL, pos[0], src);
      if (lane == src) {
#pragma unroll
        for (int q = 0; q < K - 1; q++) { key[q] = key[q + 1]; pos[q] = pos[q + 1]; }
        key[K - 1] = INF64;
        pos[K - 1] = NIL;
      }
      const uint32_t cnt = C.count, last = cnt - 1;
      const uint32_t t_v = (uint32_t)(m >> 32);
      uint32_t e_pos = NIL;
      uint64_t e_key = INF64;
      if (lane == 0) {
        const uint32_t x = vpos;  // slot = dense position
        const NodeRec X = C.w.rec()[x];
        const uint32_t p = X.parent;
        const NodeRec Rp = C.w.rec()[p];
        C.total -= node_bytes(C.K->m, X.ds, X.de, (X.nf >> 24) & F_SSM);
        hash_erase_at_1(C, X.hidx);
        NodeRec& Wp = C.w.rec()[p];
        Wp.nf = Rp.nf - 1;
        Wp.cxor = Rp.cxor ^ x;
        if (p != 0) d_multi(C, p, (Rp.nf & NCH_MASK) - 1);
        if (log) {
          const uint32_t li = *log_n;
          if (li < P.log_cap) {
            mc_evict_rec e;
            e.req = r; e.node_id = (uint32_t)m; e.kind = 0; e.n_live = cnt;
            e.utility = (t_v == tmax) ? 0.5 : 0.0;  // (t - tmin)/(tmax - tmin) with tmin = t_v
            log[li] = e;
          }
          *log_n = li + 1;
        }
        d_hole(C, vpos);
        C.count = last;
        C.w.rec()[x].nf = 0;
        C.w.freel()[C.nfree++] = x;
        CTR_ADD(C, wr, 1);
        if (p != 0 && (Rp.nf & NCH_MASK) == 1) {  // the parent lost its last child
          const uint32_t pp = p;
          const DenseRec dp = *d_ptr(C, pp);
          if (!(dp.tc & D_FLAGS)) {
            e_pos = pp;
            e_key = ((uint64_t)(dp.tc & T_MASK) << 32) | __float_as_uint(dp.e32);
          }
        }
      }
      sync_state(C);
      CTR_ADD(C, scan, cnt);
      C.n_evict++;
      need--;
      progressed = true;
      e_pos = __shfl_sync(FULL, e_pos, 0);
      e_key = __shfl_sync(FULL, (unsigned long long)e_key, 0);
      if (e_pos != NIL && e_key < W) {  // keep the exposed parent (else W covers it)
        if (lane == (e_pos & 31u)) {
          const uint64_t dropped = key[K - 1];
          key[K - 1] = e_key;
          pos[K - 1] = e_pos;
#pragma unroll
          for (int q = K - 1; q > 0; q--) {
            if (key[q] < key[q - 1]) {
              const uint64_t tk = key[q]; key[q] = key[q - 1]; key[q - 1] = tk;
              const uint32_t tp = pos[q]; pos[q] = pos[q - 1]; pos[q - 1] = tp;
            }
          }
          wl = dropped;
        }
        const uint64_t d = __shfl_sync(FULL, (unsigned long long)wl, e_pos & 31u);
        W = min(W, d);
      }
    }
    if (!progressed && need) {  // no candidate at all
      if (lane == 0) atomicOr(P.status, ST_NOCAND);
      C.failed = true;
    }
  }
}

__device__ ReqOut process_request_vllm(Chain& C, const KParams& P, uint32_t r, const Prefetched cur,
                                       Prefetched& nxt, bool has_next, mc_evict_rec* log, uint32_t* log_n) {
  const uint32_t lane = lane_id();
  const ReqHdr q = cur.q;
  const uint32_t off = q.off;
  const uint32_t L_in = q.lin;
  const uint32_t n = q.lin + q.lout;
  const uint32_t x = C.block;
  const uint32_t nb = n / x;  // full blocks; a trailing partial block is not cached (V2)
  if (has_next) nxt.q = load_req(P, r + 1);
  uint32_t* __restrict__ path = C.w.path();

  // Step 1: walk block by block (V1).  Block hashes are computed 32 at a time, one
  // block per lane, ahead of the dependent child-index probes.
  uint32_t v = 0, mb = 0;
  if (nb > C.ncap) {  // the sequence's blocks cannot all be held: the path array bounds the walk
    if (lane == 0) atomicOr(P.status, ST_OVERFLOW);
    C.failed = true;
    ReqOut o;
    o.reuse = 0; o.flops = 0; o.bypass = true;
    return o;
  }
  for (uint32_t k0 = 0; k0 < nb && mb == k0; k0 += 32) {
    const uint32_t kl = k0 + lane;
    const uint32_t my_h = (kl < nb) ? block_hash_1(P.tok + off + (uint64_t)kl * x, x) : 0u;
    const uint32_t kend = min(nb, k0 + 32);
    for (uint32_t k = k0; k < kend; k++) {
      const uint32_t h = __shfl_sync(FULL, my_h, k - k0);
      const uint32_t c = child_block(C, P, v, h, off + (uint64_t)k * x, k * x);
      if (c == NIL) break;
      if (lane == 0) path[k] = c;
      v = c;
      mb++;
    }
  }
  __syncwarp();
  CTR_ADD(C, cmp, (uint64_t)mb * x);
  CTR_ADD(C, vis, mb + 1);
  if (has_next) nxt.tk0 = __ldg(P.tok + nxt.q.off);

  // Step 2: hit = the deepest matched block end <= L_in (V4).
  const uint32_t reuse = min(mb, L_in / x) * x;

#ifdef MC_DEBUG
  for (uint32_t i = lane; i < mb; i += 32) {
    const uint32_t sl = path[i];
    if (sl >= C.hwm || d_tc(C, sl) == HOLE_TC)
      printf("vllm walk: r %u k %u/%u slot %u hwm %u count %u nb %u S %u\n", r, i, mb, sl, C.hwm, C.count, nb, C.S);
  }
#endif
  // Step 3: touch (t_last = r) and pin every matched block (V5, V7), in parallel.
  for (uint32_t i = lane; i < mb; i += 32) {
    DenseRec* d = d_ptr(C, path[i]);
    d->tc = r | (d->tc & D_MULTI) | D_PIN;
  }
  CTR_ADD(C, wr, mb);
  __syncwarp();

  // Step 4: admission (V7): bypass when the matched path plus the new blocks exceed the capacity.
  const uint64_t bb = node_bytes(C.K->m, 0, x, true);
  const uint32_t n_new = nb - mb;
  const uint64_t d_bytes = bb * n_new;
  const bool bypass = (bb * mb + d_bytes > C.K->capb) || (C.K->capn && nb > C.K->capn);
  if (!bypass) {
    // Step 5: LRU leaf eviction (V6) until the new blocks fit; every block has the same
    // size, so the number of victims is known up front.
    uint64_t need = 0;
    if (C.total + d_bytes > C.K->capb) need = (C.total + d_bytes - C.K->capb + bb - 1) / bb;
    if (C.K->capn && C.count + n_new > C.K->capn) need = max(need, (uint64_t)(C.count + n_new - C.K->capn));
    if (need) evict_lru_blocks(C, P, r, (uint32_t)need, log, log_n);
    // Step 6: insert blocks mb .. nb-1 under v, in parallel (one block per lane).
    if (n_new && !C.failed) {
      const uint32_t take = min(C.nfree, n_new);
      if (C.hwm + (n_new - take) > C.ncap) {
        if (lane == 0) atomicOr(P.status, ST_OVERFLOW);
        C.failed = true;
      } else {
        for (uint32_t j = lane; j < n_new; j += 32)
          path[mb + j] = (j < take) ? C.w.freel()[C.nfree - 1 - j] : C.hwm + (j - take);
        __syncwarp();
        const uint32_t cnt0 = C.count, id0 = C.next_id;
        for (uint32_t j = lane; j < n_new; j += 32) {
          const uint32_t k = mb + j;
          const uint32_t s = path[k];
          const uint32_t par = (j == 0) ? v : path[k - 1];
          const bool inner = j + 1 < n_new;
          NodeRec R;
          R.parent = par;
          R.ds = k * x;
          R.de = (k + 1) * x;
          R.roff = (uint32_t)off;
          R.cxor = inner ? path[k + 1] : 0u;
          R.nf = (F_SSM << 24) | (inner ? 1u : 0u);
          R.id = id0 + j;
          const uint32_t h = block_hash_1(P.tok + off + (uint64_t)k * x, x);
          uint32_t hi = hslot(par, h, C.hmask);
          const uint32_t nk = hkey(C, par, s);
          for (;;) {  // lanes insert concurrently: claim an empty slot by CAS on its key word
            const uint32_t kw = atomicAdd(&C.w.tab()[hi].key, 0u);
            if (hvalid(C, kw)) { hi = (hi + 1) & C.hmask; continue; }
            if (atomicCAS(&C.w.tab()[hi].key, kw, nk) == kw) break;
          }
          HEnt& E = C.w.tab()[hi];
          E.tok = h;
          E.de = R.de | 0x80000000u;
          E.roff = R.roff;
          R.hidx = hi;
          C.w.rec()[s] = R;
          DenseRec* d = d_ptr(C, s);
          d->tc = r | (inner ? D_MULTI : 0u);
          d->e32 = __uint_as_float(id0 + j);  // vLLM+: the id, so (t, id) LRU keys need no global read
        }
        if (lane == 0) {
          NodeRec& Rv = C.w.rec()[v];
          const uint32_t nf0 = Rv.nf;
          Rv.nf = nf0 + 1;
          Rv.cxor ^= path[mb];
          if (v != 0 && (nf0 & NCH_MASK) + 1 >= C.mthr) {
            DenseRec* d = d_ptr(C, v);
            d->tc |= D_MULTI;
          }
          C.nfree -= take;
          C.hwm += n_new - take;
          C.count = cnt0 + n_new;
          C.next_id = id0 + n_new;
          C.total += d_bytes;
          CTR_ADD(C, wr, n_new);
          if (C.total > C.K->capb || (C.K->capn && C.count > C.K->capn)) {
            atomicOr(P.status, ST_INVARIANT);
            C.failed = true;
          }
        }
      }
    }
    sync_state(C);
  }
  // Unpin the matched path (evictions may have moved dense entries: positions re-read).
  for (uint32_t i = lane; i < mb; i += 32) {
    DenseRec* d = d_ptr(C, path[i]);
    d->tc &= ~D_PIN;
  }
  __syncwarp();
  ReqOut o;
  o.reuse = reuse;
  o.flops = prefill_F(C.K->m, reuse);
  o.bypass = bypass;
  return o;
}

// ---------------------------------------------------------------------------
// Standalone lookup (mc_lookup): steps 1-4 of SURVEY.md §8(c) c.2 for request r against
// the chain's current tree, read-only -- the walk (K2: child-index probe + warp compare,
// PAPER:246, 300-301), the hit (all-or-nothing, or mid-edge KV reuse when n_ssm = 0), the
// speculative-insertion checkpoint (chunk-aligned PAPER:371-373) and the
// insertion plan.  Same rules as process_request steps 1-4.
// ---------------------------------------------------------------------------
__device__ void lookup_request(const Chain& C, const KParams& P, uint32_t r, mc_lookup_result* out) {
  const uint32_t lane = lane_id();
  const ReqHdr q = load_req(P, r);
  const uint32_t off = q.off, L_in = q.lin, n = q.lin + q.lout;
  uint32_t v = 0, v_ds = 0, pos = 0, npath = 0, m = 0, my_path = NIL, my_ds = 0, my_de = 0, my_fl = 0;
  uint32_t partial = NIL, partial_ds = 0, hit = NIL, reuse = 0;
  uint32_t lin_node = NIL, lin_bnd = NIL, v_flags = 0, lin_bnd_flags = 0;
  uint32_t tk = __ldg(P.tok + off);
  for (;;) {
    if (pos == n) { m = n; break; }
    const HEnt E = hash_find_warp(C, v, tk);
    if (E.key == 0) { m = pos; break; }
    const uint32_t c = E.key & SLOT14;
    const uint32_t de = E.de & 0x7FFFFFFFu;
    const uint32_t fl = E.de >> 31;
    const uint32_t len = de - pos;
    const uint32_t nt = (de < n) ? __ldg(P.tok + off + de) : 0u;
    const uint32_t k = match_len(P.tok, (uint64_t)E.roff + pos, (uint64_t)off + pos, min(len, n - pos), P.n_tok);
    if (lane == npath) { my_path = c; my_ds = pos; my_de = de; my_fl = fl; }
    npath++;
    if (pos < L_in && L_in < pos + len && L_in <= pos + k) lin_node = c;
    if (k == len) {
      v = c; v_ds = pos; v_flags = fl;
      pos += len;
      tk = nt;
      if (de == L_in) { lin_bnd = c; lin_bnd_flags = fl; }
      if ((fl & F_SSM) && de <= L_in) { hit = c; reuse = de; }
    } else {
      m = pos + k;
      partial = c;
      partial_ds = pos;
      break;
    }
  }
  // (the lanes hold the first 32 path nodes; deeper ones are reached by a parent walk)
  if (C.K->m.n_ssm == 0) {  // pure Transformer: KVs sliced mid-edge
    reuse = min(m, L_in);
    hit = NIL;
    uint32_t hi = NIL;
    const bool mine = lane < min(npath, 32u) && my_ds < reuse;
    const unsigned b = __ballot_sync(FULL, mine);
    if (b) { hi = 31 - __clz(b); hit = __shfl_sync(FULL, my_path, hi); }
    if (npath > 32) {  // deeper path nodes: walk the tree from the partial/last node upwards
      uint32_t x = partial != NIL ? partial : v;
      while (x != 0 && x != NIL) {
        const NodeRec R = C.w.rec()[x];
        if (R.ds < reuse) { hit = x; break; }
        x = R.parent;
      }
    }
  }
  // step 3: speculative insertion of the input (R8, R9), chunk alignment (R11)
  const uint32_t m_in = min(m, L_in);
  uint32_t p = 0;
  if (m_in > 0) {
    if (m >= L_in) {
      if (lin_bnd != NIL) { if (!(lin_bnd_flags & F_SSM)) p = m_in; }
      else p = m_in;
    } else if (partial != NIL) {
      p = m_in;
    } else if (!(v_flags & F_SSM)) {
      p = m_in;
    }
  }
  bool p_split = (p != 0) && ((m >= L_in) ? (lin_bnd == NIL) : (partial != NIL));
  if (C.K->chunk && p) {
    uint32_t pa = (p / C.K->chunk) * C.K->chunk;
    if (pa == 0 || pa <= reuse) pa = 0;
    p_split = false;
    if (pa) {
      // the node at or containing pa on the path: lanes < 32, deeper ones by a parent walk
      const bool mine = lane < min(npath, 32u);
      const unsigned bnd = __ballot_sync(FULL, mine && my_de == pa && my_path != partial);
      const unsigned ins = __ballot_sync(FULL, mine && my_ds < pa && pa < my_de);
      if (bnd) {
        if (__shfl_sync(FULL, my_fl, __ffs(bnd) - 1) & F_SSM) pa = 0;
      } else if (ins) {
        p_split = true;
      } else {
        uint32_t kind = 0;
        uint32_t x = partial != NIL ? partial : v;
        while (x != 0 && x != NIL) {
          const NodeRec R = C.w.rec()[x];
          if (x != partial && R.de == pa) { kind = ((R.nf >> 24) & F_SSM) ? 3 : 1; break; }
          if (R.ds < pa && pa < R.de) { kind = 2; break; }
          x = R.parent;
        }
        if (kind == 2) p_split = true;
        else if (kind != 1) pa = 0;
      }
    }
    p = pa;
  }
  // step 4: plan
  const bool leaf = m < n;
  const bool split_m = partial != NIL && m < n && m != p;
  const bool split_n = partial != NIL && m == n && n != p;
  const bool n_gain = partial == NIL && m == n && n != p && !(v_flags & F_SSM);
  uint32_t n_ck = p ? 1u : 0u;
  if (n != p && (leaf || split_n || n_gain)) n_ck++;
  if (lane == 0) {
    mc_lookup_result o;
    o.reuse = reuse;
    o.m = m;
    o.p = p;
    o.hit_id = hit == NIL ? 0u : C.w.rec()[hit].id;
    const uint32_t dv = partial != NIL ? partial : v;
    o.div_id = dv == 0 ? 0u : C.w.rec()[dv].id;
    o.div_off = m - (partial != NIL ? partial_ds : v_ds);
    o.path_len = npath;
    o.d_nodes = (p_split ? 1u : 0u) + (split_m ? 1u : 0u) + (split_n ? 1u : 0u) + (leaf ? 1u : 0u);
    o.d_bytes = C.K->m.kvt * (uint64_t)(n - m) + C.K->m.ssmb * n_ck;
    *out = o;
  }
  __syncwarp();
}

// kc / kx: shared memory for the chain's constants and counters (written by lane 0 here).
__device__ __forceinline__ void chain_init(Chain& C, const KParams& P, uint32_t worker, const DevVariant& V,
                                           double alpha, char* smem_warp, uint32_t S, ChainConst* kc, ChainCtr* kx) {
  C.w.b = P.ws + (uint64_t)worker * P.ws_stride;
  C.w.n = P.ncap;
  C.w.h = P.hcap;
  C.sd = (DenseRec*)smem_warp;
  C.S = S;
  C.ncap = P.ncap;
  C.hmask = P.hcap - 1;
  C.gen = 0;
  if (lane_id() == 0) {
    kc->m = V.m;
    kc->capb = V.cap_bytes;
    kc->capn = V.cap_nodes;
    kc->chunk = V.chunk;
    kc->alpha = V.block ? 0.0 : alpha;  // vLLM+ is LRU: α does not apply
    kx->cmp = kx->vis = kx->scan = kx->wr = 0;
  }
  __syncwarp();
  C.K = kc;
  C.X = kx;
  C.block = V.block;
  C.mthr = V.block ? 1u : 2u;  // vLLM+ evicts leaf blocks only (V6)
  C.n_evict = 0;
  C.bc_valid = 0;
  C.bc_tmin = 0; C.bc_tmax = 0; C.bc_lo = 0.0f; C.bc_hi = 0.0f; C.bc_elo = 0.0; C.bc_ehi = 0.0;
#if defined(MC_PHASE_TIMERS) || defined(MC_PHASE_TIMERS3)
  C.t_walk = C.t_evict = C.t_insert = C.t_unpin = 0;
#endif
  C.failed = false;
}

}  // namespace mcd
