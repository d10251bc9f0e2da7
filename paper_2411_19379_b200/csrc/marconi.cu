// marconi.cu -- kernels and C ABI of libmarconi.so (see include/marconi.h).
//
// Kernels (all sm_100a, hand-written, no tensor cores -- nothing on the path is
// a dense contraction):
//   replay_kernel     K5: persistent; each warp pops chains (variant, α, segment)
//                     from a device queue, loads the segment snapshot and
//                     replays the window (K1-K4 inlined, see replay.cuh); a lean
//                     Marconi instantiation (no log / chunk / n_ssm = 0 paths), a
//                     general one, and the vLLM+ one.
//   live_kernel       the α = 0 live LRU pass per variant, dumping snapshot k
//                     after every `window` requests (segment mode, R19) or at the
//                     bootstrap points, with per-window cycle counts.
//   image_kernel      loadable snapshot images.
//   lookup_kernel     mc_lookup: read-only lookups against frozen snapshots.
//   chain_sums_kernel mc_chain_sums: per-chain Σ hit / Σ L_in / 128-bit Σ FLOPs.
//   trace_check_kernel  mc_set_trace_async: the trace rules on the device.
//   snap_link_kernel  resolves parent ids of uploaded canonical snapshots.
//   node_cost_kernel  K1 batched (unit parity).
//   score_argmin_kernel  K3 segmented, one warp per table (unit parity).
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <string>
#include <vector>

#include "marconi.h"
#include "replay.cuh"

using namespace mcd;

namespace {
thread_local std::string g_err;

mc_status fail(mc_status s, const std::string& m) {
  g_err = m;
  return s;
}
#define CU(x)                                                                               \
  do {                                                                                      \
    cudaError_t e_ = (x);                                                                   \
    if (e_ != cudaSuccess) return fail(MC_ECUDA, std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

#ifndef MC_MINBLOCKS
#define MC_MINBLOCKS 16
#endif
#ifndef MC_WARPS_PER_CTA
#define MC_WARPS_PER_CTA 1
#endif
constexpr int kWarpsPerCta = MC_WARPS_PER_CTA;
}  // namespace

// ---------------------------------------------------------------------------
// Kernels
// ---------------------------------------------------------------------------
// kPolicy 0 = Marconi chains, 1 = vLLM+ chains (block_size > 0): one instantiation per
// policy so the Marconi kernel carries no vLLM+ code (registers, instruction cache).
// kGen (Marconi chains): false = the lean instantiation (no eviction log, no chunked
// checkpoints, n_ssm > 0), chosen by mc_replay whenever the call allows it.
template <int kPolicy, bool kGen>
#ifdef MC_MAXNREG  // explicit register budget (sizes the resident warps per SM instead of MC_MINBLOCKS)
__global__ void __maxnreg__(MC_MAXNREG) replay_kernel(KParams P) {
#else
__global__ void __launch_bounds__(32 * kWarpsPerCta, MC_MINBLOCKS) replay_kernel(KParams P) {
#endif
  extern __shared__ __align__(16) char smem[];
  const uint32_t lane = lane_id();
  const uint32_t worker = blockIdx.x * kWarpsPerCta + (threadIdx.x >> 5);
  if (worker >= P.n_workers) return;
  {  // the warp's snapshot-copy mbarrier and phase word (dense slots S + 12, S + 13)
    char* sw = smem + (threadIdx.x >> 5) * 8ull * P.smem_nodes;
    const uint32_t S = P.smem_nodes - kSmemReserved;
    if (lane == 0) {
      mbar_init(reinterpret_cast<uint64_t*>(sw + 8ull * (S + 12)));
      *reinterpret_cast<uint32_t*>(sw + 8ull * (S + 13)) = 0;
    }
    __syncwarp();
  }
  for (;;) {
    uint32_t qi = 0;
    if (lane == 0) qi = atomicAdd(P.queue, 1u);
    qi = __shfl_sync(FULL, qi, 0);
    if (qi >= P.n_chains) return;
    if (*(volatile uint32_t*)P.status & ST_BADTRACE) return;  // rejected trace: read nothing
    const long long t0 = clock64();
    const uint32_t c = P.chains[qi];
    const uint32_t s = c % P.n_segs;
    const uint32_t a = (c / P.n_segs) % P.n_alpha;
    const uint32_t v = c / (P.n_segs * P.n_alpha);
    const DevVariant V = P.var[v];
    const mc_segment seg = P.segs[s];
    Chain C;
    // the warp's shared memory: dense slots [0, S), the counters (32 B), the chain
    // constants (64 B), the snapshot-copy mbarrier and its phase word
    char* sw = smem + (threadIdx.x >> 5) * 8ull * P.smem_nodes;
    const uint32_t S = P.smem_nodes - kSmemReserved;
    chain_init(C, P, worker, V, P.alphas[a], sw, S, reinterpret_cast<ChainConst*>(sw + 8ull * (S + 4)),
               reinterpret_cast<ChainCtr*>(sw + 8ull * S));
    // the policy is a compile-time constant in each instantiation (vLLM+ chains have
    // block > 0, so chain_init already set their α to 0)
    if (kPolicy == 0) { C.block = 0; C.mthr = 2; } else { C.mthr = 1; }
#ifdef MC_LOAD_TIMER
    const long long _l0 = clock64();
#endif
    load_image(C, P, P.snap[v].img + P.snap[v].img_off[seg.snapshot]);
#ifdef MC_LOAD_TIMER
    const long long _l1 = clock64();
#endif
    mc_evict_rec* log = P.log ? P.log + (uint64_t)c * P.log_cap : nullptr;
    uint32_t* log_n = P.log ? P.log_n + c : nullptr;
    if (lane == 0 && log_n) *log_n = 0;
    unsigned long long sum = 0;
    const uint64_t obase = ((uint64_t)v * P.n_alpha + a) * P.n_req;
    Prefetched cur = fetch_request(P, seg.first_req), nxt = cur;
    for (uint32_t i = 0; i < seg.n_req && !C.failed; i++) {
      const uint32_t r = seg.first_req + i;
      const ReqOut o = kPolicy ? process_request_vllm(C, P, r, cur, nxt, i + 1 < seg.n_req, log, log_n)
                               : process_request<kGen>(C, P, r, cur, nxt, i + 1 < seg.n_req, log, log_n);
      cur = nxt;
      if (lane == 0) {
        P.hit[obase + r - 1] = o.reuse;
        P.flops[obase + r - 1] = o.flops;
        if (P.bypass) P.bypass[obase + r - 1] = o.bypass ? 1 : 0;
      }
      sum += o.reuse;
    }
    if (lane == 0) {
      atomicAdd(P.hit_sum + (uint64_t)v * P.n_alpha + a, sum);
      if (P.counters) {
#if defined(MC_PHASE_TIMERS) || defined(MC_PHASE_TIMERS3)
        P.counters[4ull * c + 0] = C.t_walk;
        P.counters[4ull * c + 1] = C.t_evict;
        P.counters[4ull * c + 2] = C.t_insert;
        P.counters[4ull * c + 3] = C.t_unpin;
#else
        P.counters[4ull * c + 0] = C.X->cmp;
        P.counters[4ull * c + 1] = C.X->vis;
        P.counters[4ull * c + 2] = C.X->scan;
        P.counters[4ull * c + 3] = C.X->wr;
#ifdef MC_LOAD_TIMER
        P.counters[4ull * c + 0] = (unsigned long long)(_l1 - _l0);
#endif
#endif
      }
#ifdef MC_CHAIN_SMID  // dev builds: SM id in the top 8 bits, cycles >> 10 below
      if (P.chain_cycles) {
        uint32_t sm;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(sm));
        P.chain_cycles[c] = (sm << 24) | (uint32_t)min((long long)0xFFFFFF, (clock64() - t0) >> 10);
      }
#else
      if (P.chain_cycles) P.chain_cycles[c] = (uint32_t)min((long long)0xFFFFFFFF, (clock64() - t0) >> 10);
#endif
    }
    __syncwarp();
  }
}

// Snapshot images (setup): warp w builds the images of snapshots w, w + n_workers, ...
// of variant `v` by running load_snapshot on its scratch slice (whole dense list in the
// global tail) and exporting the result.
__global__ void __launch_bounds__(32) image_kernel(KParams P, uint32_t v, char* img, const uint64_t* img_off) {
  const uint32_t w = blockIdx.x;
  const DevSnapStore& st = P.snap[v];
  for (uint32_t k = w; k < st.count; k += P.n_workers) {
    Chain C;
    __shared__ ChainConst kc;
    __shared__ ChainCtr kx;
    chain_init(C, P, w, P.var[v], 0.0, nullptr, 0, &kc, &kx);
    load_snapshot(C, P, &st, k);
    export_image(C, img + img_off[k]);
  }
}

__global__ void __launch_bounds__(32) live_kernel(KParams P) {
  extern __shared__ __align__(16) char smem[];
  const uint32_t lane = lane_id();
  const uint32_t v = blockIdx.x;
  if (v >= P.n_var) return;
  if (*(volatile uint32_t*)P.status & ST_BADTRACE) return;  // rejected trace: read nothing
  Chain C;
  const uint32_t S = P.smem_nodes - kSmemReserved;
  chain_init(C, P, v, P.var[v], 0.0, smem, S, reinterpret_cast<ChainConst*>(smem + 8ull * (S + 4)),
             reinterpret_cast<ChainCtr*>(smem + 8ull * S));
  load_snapshot(C, P, nullptr, 0);  // empty tree
  DevSnapOut* out = P.live_out + v;
  dump_snapshot(C, P, out, 0);
  uint32_t next = 1, first = 0, boot_end = 0;
  long long tw = clock64();  // start of the current window (chain-cost feedback for the α-grid)
  Prefetched cur = fetch_request(P, 1), nxt = cur;
  for (uint32_t r = 1; r <= P.n_req && !C.failed; r++) {
    const uint32_t ev0 = C.n_evict;
    const ReqOut o = C.block ? process_request_vllm(C, P, r, cur, nxt, r < P.n_req, nullptr, nullptr)
                             : process_request<true>(C, P, r, cur, nxt, r < P.n_req, nullptr, nullptr);
    cur = nxt;
    if (first == 0 && C.n_evict != ev0) {  // the paper's "first eviction"
      first = r;
      if (P.live_mult) {  // bootstrap mode: the tuning snapshot and the end of the bootstrap window
        dump_snapshot(C, P, out, 1);
        boot_end = r + P.live_mult * r;
      }
    }
    if (lane == 0) {
      const uint64_t k = (uint64_t)v * P.n_req + r - 1;
      if (P.hit) P.hit[k] = o.reuse;
      if (P.flops) P.flops[k] = o.flops;
      if (P.bypass) P.bypass[k] = o.bypass ? 1 : 0;
    }
    if (P.live_mult) {
      if (r == boot_end && r < P.n_req) dump_snapshot(C, P, out, 2);
    } else {
      while (next < P.n_points && P.live_points[next] == r) {
        if (lane == 0 && P.live_cyc) {
          const long long now = clock64();
          P.live_cyc[(uint64_t)v * P.n_points + next - 1] = (unsigned long long)(now - tw);
          tw = now;
        }
        dump_snapshot(C, P, out, next);
        next++;
      }
    }
  }
  if (lane == 0 && P.first_evict) P.first_evict[v] = first;
  if (lane == 0 && P.live_cyc && !P.live_mult)  // the last window (after the last point)
    P.live_cyc[(uint64_t)v * P.n_points + P.n_points - 1] = (unsigned long long)(clock64() - tw);
}

// Batched lookup (mc_lookup): warp w answers query groups w, w + n_workers, ...; a group
// = the queries against one (variant, snapshot): its image is loaded into the warp's
// workspace slice (private mode, dense list in the global tail) and every query walks it
// read-only (lookup_request).  groups: {variant, snapshot, first, count} over perm.
__global__ void __launch_bounds__(32) lookup_kernel(KParams P, const uint4* groups, uint32_t n_groups,
                                                   const uint32_t* perm, const mc_lookup_query* q,
                                                   mc_lookup_result* out) {
  __shared__ __align__(16) DenseRec hdr[kSmemReserved];  // counters, constants, copy mbarrier (S = 0)
  const uint32_t w = blockIdx.x;
  if (*(volatile uint32_t*)P.status & ST_BADTRACE) return;
  if (lane_id() == 0) {
    mbar_init(reinterpret_cast<uint64_t*>(hdr + 12));
    *reinterpret_cast<uint32_t*>(hdr + 13) = 0;
  }
  __syncwarp();
  for (uint32_t gi = w; gi < n_groups; gi += P.n_workers) {
    const uint4 g = groups[gi];
    Chain C;
    chain_init(C, P, w, P.var[g.x], 0.0, reinterpret_cast<char*>(hdr), 0, reinterpret_cast<ChainConst*>(hdr + 4),
               reinterpret_cast<ChainCtr*>(hdr));
    load_image(C, P, P.snap[g.x].img + P.snap[g.x].img_off[g.y]);
    if (C.failed) continue;
    for (uint32_t k = 0; k < g.w; k++) {
      const uint32_t qi = perm[g.z + k];
      lookup_request(C, P, q[qi].req, out + qi);
    }
  }
}

// Per-chain sums of a replay's outputs (mc_chain_sums; PAPER:537-538 metrics): one warp
// per chain (variant, α, segment) reduces its window's hits, input tokens and FLOPs saved;
// FLOPs in 128-bit (a window's sum can pass 2^64).  out[i] = {Σhit, ΣL_in, Σflops lo, hi}.
__global__ void chain_sums_kernel(const mc_request* req, const mc_segment* segs, uint32_t n_segs, uint32_t n_alpha,
                                  uint32_t n_var, uint32_t n_req, const uint32_t* chains, uint32_t n_chains,
                                  const uint32_t* hit, const unsigned long long* flops, unsigned long long* out,
                                  uint32_t* status) {
  const uint32_t lane = lane_id();
  const uint32_t i = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (i >= n_chains) return;
  const uint32_t c = chains[i];
  if ((uint64_t)c >= (uint64_t)n_var * n_alpha * n_segs) {  // not a chain id of this context
    if (lane == 0) atomicOr(status, ST_INVARIANT);
    return;
  }
  const uint32_t s = c % n_segs, a = (c / n_segs) % n_alpha, v = c / (n_segs * n_alpha);
  const mc_segment seg = segs[s];
  const uint64_t base = ((uint64_t)v * n_alpha + a) * n_req;
  unsigned long long sh = 0, sl = 0;
  unsigned __int128 sf = 0;
  for (uint32_t k = lane; k < seg.n_req; k += 32) {
    const uint32_t r = seg.first_req + k;
    sh += hit[base + r - 1];
    sl += req[r - 1].input_len;
    sf += flops[base + r - 1];
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    sh += __shfl_xor_sync(FULL, sh, o);
    sl += __shfl_xor_sync(FULL, sl, o);
    const unsigned long long lo = __shfl_xor_sync(FULL, (unsigned long long)sf, o);
    const unsigned long long hi = __shfl_xor_sync(FULL, (unsigned long long)(sf >> 64), o);
    sf += ((unsigned __int128)hi << 64) | lo;
  }
  if (lane == 0) {
    out[4ull * i + 0] = sh;
    out[4ull * i + 1] = sl;
    out[4ull * i + 2] = (unsigned long long)sf;
    out[4ull * i + 3] = (unsigned long long)(sf >> 64);
  }
}

// Device-side trace check (mc_set_trace_async): the same rules as mc_set_trace's host
// pass; a violation sets ST_BADTRACE and records the first bad request (1-based) in
// status[1], so no request table ever travels back to the host.
__global__ void trace_check_kernel(const mc_request* req, uint32_t n_reqs, uint64_t n_tok, uint32_t lmax,
                                   uint32_t* status) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_reqs; i += gridDim.x * blockDim.x) {
    const mc_request q = req[i];
    const uint64_t n = (uint64_t)q.input_len + q.output_len;
    if (q.input_len == 0 || n > lmax || q.tok_off + n > n_tok) {
      atomicOr(status, ST_BADTRACE);
      atomicMin(status + 1, i + 1);
    }
  }
}

// parent_idx of uploaded canonical records (sorted by id within each snapshot).
__global__ void snap_link_kernel(const mc_snap_node* nodes, const uint64_t* off, uint32_t n_snap, uint32_t* pidx,
                                 uint32_t* status) {
  const uint32_t k = blockIdx.y;
  if (k >= n_snap) return;
  const uint64_t a = off[k], b = off[k + 1];
  const uint32_t n = (uint32_t)(b - a);
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t pid = nodes[a + i].parent_id;
    uint32_t res = NIL;
    if (pid != 0) {
      uint32_t lo = 0, hi = n;
      while (lo < hi) {
        const uint32_t mid = (lo + hi) >> 1;
        if (nodes[a + mid].id < pid) lo = mid + 1; else hi = mid;
      }
      if (lo < n && nodes[a + lo].id == pid) res = lo;
      else atomicOr(status, ST_INVARIANT);
    }
    pidx[a + i] = res;
  }
}

__global__ void node_cost_kernel(DevModel m, uint32_t n, const uint32_t* ds, const uint32_t* de, const uint8_t* ssm,
                                 unsigned long long* saved, unsigned long long* bytes, double* eff) {
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) {
    const uint32_t a = ds[i], b = de[i];
    const bool s = ssm[i] != 0;
    saved[i] = prefill_F(m, b) - prefill_F(m, a);
    bytes[i] = node_bytes(m, a, b, s);
    eff[i] = node_eff(m, a, b, s);
  }
}

__global__ void score_argmin_kernel(uint32_t n_tables, const uint32_t* off, const uint32_t* t, const uint8_t* cand,
                                    const uint32_t* id, const double* eff, const double* alpha, uint32_t* best_out,
                                    double* u_out) {
  const uint32_t lane = lane_id();
  const uint32_t s = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (s >= n_tables) return;
  const uint32_t a = off[s], b = off[s + 1];
  Bounds bd;
  bounds_init(bd);
  for (uint32_t i = a + lane; i < b; i += 32) bounds_add(bd, t[i], eff[i]);
  bounds_reduce(bd);
  Best best;
  best_init(best);
  const double al = alpha[s];
  for (uint32_t i = a + lane; i < b; i += 32) {
    if (!cand[i]) continue;
    const double u = utility(bd, t[i], eff[i], al);
    if (best.i == NIL || better(u, t[i], id[i], best)) {
      best.u = u; best.t = t[i]; best.id = id[i]; best.i = i - a;
    }
  }
  best_reduce(best);
  if (lane == 0) {
    best_out[s] = best.i;
    u_out[s] = best.i == NIL ? 0.0 : best.u;
  }
}

// ---------------------------------------------------------------------------
// Host side
// ---------------------------------------------------------------------------
struct SnapStore {
  mc_snap_node* nodes = nullptr;
  uint32_t* pidx = nullptr;
  uint64_t* off = nullptr;
  uint32_t* n = nullptr;
  uint32_t* nid = nullptr;
  uint32_t count = 0;
  uint64_t cap = 0;
  char* img = nullptr;          // snapshot images (ImgHdr layout), rebuilt whenever the store changes
  uint64_t* img_off = nullptr;
  uint64_t img_cap = 0;         // allocated bytes of img / entries of img_off (reused when large enough)
  uint32_t img_off_cap = 0;
  void release() {
    cudaFree(nodes); cudaFree(pidx); cudaFree(off); cudaFree(n); cudaFree(nid);
    cudaFree(img); cudaFree(img_off);
    *this = SnapStore();
  }
};

struct mc_ctx {
  int device = 0;
  int n_sm = 0;
  int blocks_per_sm = 1;
  uint32_t smem_nodes = 0;       // default dense positions per warp in shared memory (replay)
  uint32_t smem_nodes_live = 0;  // same for the 1-warp live-pass CTAs
  uint64_t smem_optin = 0;
  uint32_t ncap = 0, hcap = 0;
  std::vector<mc_variant> hv;
  std::vector<DevVariant> dvh;
  DevVariant* d_var = nullptr;
  const uint32_t* tok = nullptr;
  uint64_t n_tok = 0;
  const mc_request* req = nullptr;
  uint32_t n_req = 0;
  std::vector<SnapStore> snaps;
  DevSnapStore* d_stores = nullptr;
  std::vector<mc_segment> segs;
  mc_segment* d_segs = nullptr;
  uint32_t* d_status = nullptr;
  uint32_t* d_points = nullptr;  // live-pass snapshot points + first-eviction outputs
  unsigned long long* d_live_cyc = nullptr;  // [n_var][points] cycles per live-pass window
  uint32_t live_points = 0;
  uint32_t alpha_cap = 0;        // α values per mc_replay call (they travel in the workspace header)
  char* img_scratch = nullptr;   // image_kernel workspace slices (zeroed once, reused: generation tags)
  uint64_t img_scratch_bytes = 0;
};

namespace {
// Workspace layout: control header (kCtrl bytes: queue counters at 0 and 64, this call's
// α grid at kAlphaOff, live-pass snapshot views at 256) | worker slices at the FIXED offset
// kCtrl (so a workspace reused with a different chain count keeps every slice -- and its
// child-index generation header -- in place) | the call's chain ids at the end.
constexpr uint64_t kCtrl = 4096;
constexpr uint64_t kAlphaOff = 2048;  // up to 256 doubles
uint64_t ids_bytes(uint64_t n_chains) { return (4ull * n_chains + 255) & ~255ull; }

DevModel make_model(const mc_model& m) {
  // Appendix A tab:flops_breakdown summed over layers, and PAPER:814.
  const unsigned __int128 D = m.d_model, N = m.d_state;
  unsigned __int128 fa = 8 * (unsigned __int128)m.n_attn * D * D +
                         (unsigned __int128)m.n_ssm * (12 * D * D + 16 * D * N + 10) +
                         16 * (unsigned __int128)m.n_mlp * D * D;
  unsigned __int128 fb = 4 * (unsigned __int128)m.n_attn * D;
  DevModel d;
  d.fa = (uint64_t)fa;
  d.fb = (uint64_t)fb;
  d.kvt = (uint64_t)m.n_attn * 2ull * m.d_model * m.bytes_per_param;
  d.ssmb = (uint64_t)m.n_ssm *
           ((uint64_t)m.d_model * m.d_state + (uint64_t)m.conv_in * m.conv_kernel) * m.bytes_per_param;
  d.n_ssm = m.n_ssm;
  d.pad = 0;
  return d;
}

// (asynchronous on st: the staging of the pageable host array completes before return)
mc_status upload_stores(mc_ctx* c, cudaStream_t st = nullptr) {
  std::vector<DevSnapStore> h(c->snaps.size());
  for (size_t v = 0; v < c->snaps.size(); v++) {
    h[v].nodes = c->snaps[v].nodes;
    h[v].pidx = c->snaps[v].pidx;
    h[v].off = c->snaps[v].off;
    h[v].n = c->snaps[v].n;
    h[v].nid = c->snaps[v].nid;
    h[v].img = c->snaps[v].img;
    h[v].img_off = c->snaps[v].img_off;
    h[v].count = c->snaps[v].count;
    h[v].pad = 0;
  }
  CU(cudaMemcpyAsync(c->d_stores, h.data(), sizeof(DevSnapStore) * h.size(), cudaMemcpyHostToDevice, st));
  return MC_OK;
}

uint32_t default_workers(const mc_ctx* c) { return (uint32_t)(c->n_sm * c->blocks_per_sm * kWarpsPerCta); }

// (Re)build the loadable images of variant v's snapshots (setup-time; allocates).
// host_n: the snapshot sizes when the caller knows them (else read back from the store).
// Buffers are kept across calls and grown only when too small (no allocation on the
// steady-state upload path).
mc_status build_images(mc_ctx* c, uint32_t v, cudaStream_t st, const uint32_t* host_n = nullptr) {
  SnapStore& s = c->snaps[v];
  if (s.count == 0) {
    cudaFree(s.img);
    cudaFree(s.img_off);
    s.img = nullptr;
    s.img_off = nullptr;
    s.img_cap = 0;
    s.img_off_cap = 0;
    return upload_stores(c, st);
  }
  std::vector<uint32_t> n(s.count);
  if (host_n) {
    std::copy(host_n, host_n + s.count, n.begin());
  } else {
    CU(cudaMemcpyAsync(n.data(), s.n, sizeof(uint32_t) * s.count, cudaMemcpyDeviceToHost, st));
    CU(cudaStreamSynchronize(st));
  }
  std::vector<uint64_t> off(s.count + 1, 0);
  for (uint32_t k = 0; k < s.count; k++) {
    if (n[k] + 1 > c->ncap) return fail(MC_EOVERFLOW, "snapshot larger than max_nodes");
    off[k + 1] = off[k] + ((img_bytes(n[k]) + 255) & ~255ull);
  }
  if (s.img_cap < off[s.count] || s.img_off_cap < s.count + 1) {
    CU(cudaStreamSynchronize(st));  // the old images may still be read by queued work
    cudaFree(s.img);
    cudaFree(s.img_off);
    s.img = nullptr;
    s.img_off = nullptr;
    s.img_cap = 0;
    s.img_off_cap = 0;
    if (cudaMalloc(&s.img, off[s.count]) != cudaSuccess ||
        cudaMalloc(&s.img_off, sizeof(uint64_t) * (s.count + 1)) != cudaSuccess)
      return fail(MC_ENOMEM, "snapshot image allocation failed");
    s.img_cap = off[s.count];
    s.img_off_cap = s.count + 1;
  }
  CU(cudaMemcpyAsync(s.img_off, off.data(), sizeof(uint64_t) * (s.count + 1), cudaMemcpyHostToDevice, st));
  mc_status rc = upload_stores(c, st);
  if (rc != MC_OK) return rc;
  const uint32_t nb = std::min<uint32_t>(s.count, 4u * (uint32_t)c->n_sm);
  const uint64_t per = ws_bytes_per_worker(c->ncap, c->hcap);
  if (c->img_scratch_bytes < per * nb) {
    CU(cudaStreamSynchronize(st));
    cudaFree(c->img_scratch);
    c->img_scratch = nullptr;
    c->img_scratch_bytes = 0;
    if (cudaMalloc(&c->img_scratch, per * nb) != cudaSuccess) return fail(MC_ENOMEM, "image scratch allocation failed");
    c->img_scratch_bytes = per * nb;
    CU(cudaMemsetAsync(c->img_scratch, 0, per * nb, st));  // slices start zeroed (generation header)
  }
  char* scratch = c->img_scratch;
  KParams P;
  memset(&P, 0, sizeof(P));
  P.tok = c->tok;
  P.n_tok = c->n_tok;
  P.req = c->req;
  P.n_req = c->n_req;
  P.n_var = (uint32_t)c->hv.size();
  P.var = c->d_var;
  P.snap = c->d_stores;
  P.ncap = c->ncap;
  P.hcap = c->hcap;
  P.n_workers = nb;
  P.ws = scratch;
  P.ws_stride = per;
  P.status = c->d_status;
  image_kernel<<<nb, 32, 0, st>>>(P, v, s.img, s.img_off);
  const cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) return fail(MC_ECUDA, std::string("image_kernel: ") + cudaGetErrorString(e));
  return MC_OK;
}
}  // namespace

extern "C" {

const char* mc_last_error(void) { return g_err.c_str(); }

mc_status mc_create(const mc_variant* hv, uint32_t n_var, uint32_t max_nodes, int device, mc_ctx** out) {
  if (!out || !hv || n_var == 0) return fail(MC_EINVAL, "mc_create: null argument or no variants");
  *out = nullptr;
  if (max_nodes < 64 || max_nodes > (1u << 14) || (max_nodes & (max_nodes - 1)))
    return fail(MC_EINVAL, "max_nodes must be a power of two in [64, 16384] (14-bit slots in the child index)");
  for (uint32_t v = 0; v < n_var; v++) {
    const mc_model& m = hv[v].model;
    if (m.bytes_per_param != 1 && m.bytes_per_param != 2 && m.bytes_per_param != 4)
      return fail(MC_EINVAL, "bytes_per_param must be 1, 2 or 4 (SPEC:36)");
    if (m.n_attn == 0) return fail(MC_EINVAL, "n_attn = 0 would allow zero-byte nodes (SPEC:136)");
    if (m.d_model == 0) return fail(MC_EINVAL, "d_model must be >= 1");
    if (hv[v].block_size && hv[v].chunk_size)
      return fail(MC_EINVAL, "block_size (vLLM+) and chunk_size (Marconi chunked prefill) are exclusive");
    if (hv[v].block_size > (1u << 20)) return fail(MC_EINVAL, "block_size must be <= 2^20");
    if (hv[v].reserved) return fail(MC_EINVAL, "mc_variant.reserved must be 0");
    // F(L) must stay exact in fp64 (< 2^53) for L up to 2^20 tokens handled below per trace
  }
  CU(cudaSetDevice(device));
  mc_ctx* c = new mc_ctx();
  c->device = device;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) {
    delete c;
    return fail(MC_ECUDA, "cudaGetDeviceProperties failed");
  }
  c->n_sm = prop.multiProcessorCount;
  // Shared memory: fill each SM with MC_MINBLOCKS CTAs of kWarpsPerCta warps; each
  // warp keeps the first S dense positions (12 B each) of its chain on chip.
  int smem_sm = 0, smem_optin = 0;
  cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, device);
  cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, device);
  c->smem_optin = (uint64_t)smem_optin;
  {
    const int64_t per_cta = std::min<int64_t>(smem_optin, smem_sm / MC_MINBLOCKS - 1024);
    const int64_t per_warp = per_cta / kWarpsPerCta;
    c->smem_nodes = (uint32_t)std::max<int64_t>(0, (per_warp / 8) & ~31ll);
    c->smem_nodes = std::min<uint32_t>(c->smem_nodes, max_nodes);
    c->smem_nodes_live = std::min<uint32_t>((uint32_t)((smem_optin / 8) & ~31), max_nodes);
  }
  cudaFuncSetAttribute(replay_kernel<0, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin);
  cudaFuncSetAttribute(replay_kernel<0, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin);
  cudaFuncSetAttribute(replay_kernel<1, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin);
  cudaFuncSetAttribute(live_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_optin);
  int bps = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, replay_kernel<0, true>, 32 * kWarpsPerCta,
                                                kWarpsPerCta * 8ull * c->smem_nodes);
  c->blocks_per_sm = std::max(1, bps);
  c->ncap = max_nodes;
#ifndef MC_HASH_SHIFT
#define MC_HASH_SHIFT 1
#endif
  c->hcap = max_nodes << MC_HASH_SHIFT;  // child-index entries (load factor <= 2^-MC_HASH_SHIFT)
  c->hv.assign(hv, hv + n_var);
  for (uint32_t v = 0; v < n_var; v++) {
    DevVariant d;
    d.m = make_model(hv[v].model);
    d.cap_bytes = hv[v].capacity_bytes;
    d.cap_nodes = hv[v].capacity_nodes;
    d.chunk = hv[v].chunk_size;
    d.block = hv[v].block_size;
    d.pad = 0;
    c->dvh.push_back(d);
  }
  c->snaps.resize(n_var);
  c->alpha_cap = (uint32_t)((kCtrl - kAlphaOff) / sizeof(double));  // 256
  if (cudaMalloc(&c->d_var, sizeof(DevVariant) * n_var) != cudaSuccess ||
      cudaMalloc(&c->d_stores, sizeof(DevSnapStore) * n_var) != cudaSuccess ||
      cudaMalloc(&c->d_status, 2 * sizeof(uint32_t)) != cudaSuccess) {
    mc_destroy(c);
    return fail(MC_ENOMEM, "mc_create: device allocation failed");
  }
  cudaMemcpy(c->d_var, c->dvh.data(), sizeof(DevVariant) * n_var, cudaMemcpyHostToDevice);
  cudaMemset(c->d_status, 0, sizeof(uint32_t));
  cudaMemset(c->d_status + 1, 0xFF, sizeof(uint32_t));  // first rejected request: none
  if (upload_stores(c) != MC_OK) {
    mc_destroy(c);
    return MC_ECUDA;
  }
  *out = c;
  return MC_OK;
}

void mc_destroy(mc_ctx* c) {
  if (!c) return;
  for (auto& s : c->snaps) s.release();
  cudaFree(c->img_scratch);
  cudaFree(c->d_var);
  cudaFree(c->d_stores);
  cudaFree(c->d_segs);
  cudaFree(c->d_status);
  cudaFree(c->d_points);
  cudaFree(c->d_live_cyc);
  delete c;
}

mc_status mc_set_trace(mc_ctx* c, const uint32_t* d_tokens, uint64_t n_tokens, const mc_request* d_reqs,
                       uint32_t n_reqs) {
  if (!c || !d_tokens || !d_reqs || n_reqs == 0) return fail(MC_EINVAL, "mc_set_trace: null/empty argument");
  if (n_reqs >= (1u << 30)) return fail(MC_EINVAL, "too many requests (timestamps must stay < 2^30)");
  if (n_tokens > 0xFFFFFFFFull) return fail(MC_EINVAL, "token pool must hold < 2^32 tokens (u32 node offsets)");
  std::vector<mc_request> h(n_reqs);
  CU(cudaMemcpy(h.data(), d_reqs, sizeof(mc_request) * n_reqs, cudaMemcpyDeviceToHost));
  for (uint32_t i = 0; i < n_reqs; i++) {
    const mc_request& q = h[i];
    if (q.input_len == 0) return fail(MC_EINVAL, "request " + std::to_string(i + 1) + ": input_len == 0");
    const uint64_t n = (uint64_t)q.input_len + q.output_len;
    if (n > (1u << 20)) return fail(MC_EINVAL, "request longer than 2^20 tokens");
    if (q.tok_off + n > n_tokens) return fail(MC_EINVAL, "request " + std::to_string(i + 1) + ": range outside pool");
  }
  for (const auto& d : c->dvh) {  // F(L) exact in u64 and < 2^53 (exact fp64 conversion) for the longest request
    uint64_t Lmax = 0;
    for (const auto& q : h) Lmax = std::max<uint64_t>(Lmax, (uint64_t)q.input_len + q.output_len);
    unsigned __int128 F = (unsigned __int128)d.m.fa * Lmax + (unsigned __int128)d.m.fb * Lmax * Lmax;
    if (F >= ((unsigned __int128)1 << 53)) return fail(MC_EINVAL, "F(L) exceeds 2^53 for the longest request");
  }
  c->tok = d_tokens;
  c->n_tok = n_tokens;
  c->req = d_reqs;
  c->n_req = n_reqs;
  return MC_OK;
}

mc_status mc_set_trace_async(mc_ctx* c, const uint32_t* d_tokens, uint64_t n_tokens, const mc_request* d_reqs,
                             uint32_t n_reqs, void* stream) {
  if (!c || !d_tokens || !d_reqs || n_reqs == 0) return fail(MC_EINVAL, "mc_set_trace_async: null/empty argument");
  if (n_reqs >= (1u << 30)) return fail(MC_EINVAL, "too many requests (timestamps must stay < 2^30)");
  if (n_tokens > 0xFFFFFFFFull) return fail(MC_EINVAL, "token pool must hold < 2^32 tokens (u32 node offsets)");
  // longest admissible request: <= 2^20 tokens and F(L) < 2^53 for every variant
  uint32_t lmax = 1u << 20;
  for (const auto& d : c->dvh) {
    const auto F = [&](uint64_t L) { return (unsigned __int128)d.m.fa * L + (unsigned __int128)d.m.fb * L * L; };
    uint32_t lo = 0, hi = lmax;  // largest L <= lmax with F(L) < 2^53 (F is increasing)
    while (lo < hi) {
      const uint32_t mid = lo + (hi - lo + 1) / 2;
      if (F(mid) < ((unsigned __int128)1 << 53)) lo = mid; else hi = mid - 1;
    }
    lmax = lo;
  }
  cudaStream_t st = (cudaStream_t)stream;
  const int blocks = (int)std::min<uint32_t>((n_reqs + 255) / 256, 148 * 4);
  trace_check_kernel<<<blocks, 256, 0, st>>>(d_reqs, n_reqs, n_tokens, lmax, c->d_status);
  CU(cudaGetLastError());
  c->tok = d_tokens;
  c->n_tok = n_tokens;
  c->req = d_reqs;
  c->n_req = n_reqs;
  return MC_OK;
}

mc_status mc_set_snapshots(mc_ctx* c, uint32_t variant, const mc_snap_node* h_nodes, const uint64_t* h_off,
                           const uint32_t* h_nid, uint32_t n_snap, void* stream) {
  if (!c || variant >= c->hv.size() || !h_off || !h_nid || n_snap == 0)
    return fail(MC_EINVAL, "mc_set_snapshots: bad argument");
  if (!c->tok) return fail(MC_ESTATE, "mc_set_snapshots before mc_set_trace");
  const uint64_t total = h_off[n_snap];
  if (h_off[0] != 0) return fail(MC_EINVAL, "h_offsets[0] must be 0");
  // Records must be sorted by id within each snapshot for the device-side parent
  // resolution; sort a copy only when the caller's order is not already sorted.
  bool is_sorted = true;
  for (uint32_t k = 0; k < n_snap; k++) {
    if (h_off[k + 1] < h_off[k]) return fail(MC_EINVAL, "offsets must be non-decreasing");
    if (h_off[k + 1] - h_off[k] + 1 > c->ncap) return fail(MC_EOVERFLOW, "snapshot larger than max_nodes");
    for (uint64_t i = h_off[k] + 1; i < h_off[k + 1]; i++)
      if (h_nodes[i - 1].id >= h_nodes[i].id) is_sorted = false;
  }
  std::vector<mc_snap_node> sorted;
  const mc_snap_node* src = h_nodes;
  if (!is_sorted) {
    sorted.assign(h_nodes, h_nodes + total);
    for (uint32_t k = 0; k < n_snap; k++)
      std::sort(sorted.begin() + h_off[k], sorted.begin() + h_off[k + 1],
                [](const mc_snap_node& a, const mc_snap_node& b) { return a.id < b.id; });
    src = sorted.data();
  }
  for (uint32_t k = 0; k < n_snap; k++) {
    for (uint64_t i = h_off[k]; i < h_off[k + 1]; i++) {
      const mc_snap_node& r = src[i];
      if (r.id == 0 || (i > h_off[k] && src[i - 1].id == r.id)) return fail(MC_EINVAL, "bad/duplicate node id");
      if (r.d_end <= r.d_start || r.ref_off + r.d_end > c->n_tok) return fail(MC_EINVAL, "bad node range");
    }
  }
  SnapStore& s = c->snaps[variant];
  const uint64_t nn = std::max<uint64_t>(total, 1);
  if (s.cap < nn || s.count < n_snap || !s.nodes) {  // reuse the store when it is large enough
    s.release();
    if (cudaMalloc(&s.nodes, sizeof(mc_snap_node) * nn) != cudaSuccess ||
        cudaMalloc(&s.pidx, sizeof(uint32_t) * nn) != cudaSuccess ||
        cudaMalloc(&s.off, sizeof(uint64_t) * (n_snap + 1)) != cudaSuccess ||
        cudaMalloc(&s.n, sizeof(uint32_t) * n_snap) != cudaSuccess ||
        cudaMalloc(&s.nid, sizeof(uint32_t) * n_snap) != cudaSuccess) {
      s.release();
      return fail(MC_ENOMEM, "snapshot store allocation failed");
    }
    s.cap = nn;
  }
  std::vector<uint32_t> cnt(n_snap);
  for (uint32_t k = 0; k < n_snap; k++) cnt[k] = (uint32_t)(h_off[k + 1] - h_off[k]);
  cudaStream_t st = (cudaStream_t)stream;
  CU(cudaMemcpyAsync(s.nodes, src, sizeof(mc_snap_node) * total, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(s.off, h_off, sizeof(uint64_t) * (n_snap + 1), cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(s.n, cnt.data(), sizeof(uint32_t) * n_snap, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(s.nid, h_nid, sizeof(uint32_t) * n_snap, cudaMemcpyHostToDevice, st));
  dim3 grid(8, n_snap);
  snap_link_kernel<<<grid, 256, 0, st>>>(s.nodes, s.off, n_snap, s.pidx, c->d_status);
  CU(cudaGetLastError());
  s.count = n_snap;
  mc_status rc = upload_stores(c, st);
  if (rc != MC_OK) return rc;
  return build_images(c, variant, st, cnt.data());
}

mc_status mc_workspace_size(const mc_ctx* c, uint32_t n_workers, uint32_t n_alpha, uint32_t n_chains,
                            uint64_t* bytes) {
  if (!c || !bytes) return fail(MC_EINVAL, "mc_workspace_size: null argument");
  if (n_workers == 0) n_workers = default_workers(c);
  if (n_chains == 0) n_chains = (uint32_t)(c->hv.size() * std::max(1u, n_alpha) * std::max<size_t>(1, c->segs.size()));
  *bytes = kCtrl + (uint64_t)n_workers * ws_bytes_per_worker(c->ncap, c->hcap) + ids_bytes(n_chains);
  return MC_OK;
}

mc_status mc_workspace_workers(const mc_ctx* c, uint64_t bytes, uint32_t n_alpha, uint32_t n_chains,
                               uint32_t* n_workers) {
  if (!c || !n_workers) return fail(MC_EINVAL, "mc_workspace_workers: null argument");
  if (n_chains == 0) n_chains = (uint32_t)(c->hv.size() * std::max(1u, n_alpha) * std::max<size_t>(1, c->segs.size()));
  const uint64_t fixed = kCtrl + ids_bytes(n_chains);
  *n_workers = bytes <= fixed ? 0 : (uint32_t)((bytes - fixed) / ws_bytes_per_worker(c->ncap, c->hcap));
  return MC_OK;
}

namespace {
// The live pass proper: static snapshot points (mult = 0) or the bootstrap points
// {0, r_F, r_F + mult r_F} found during the pass (n_points = 3; an undumped snapshot
// stays empty).
mc_status live_pass_impl(mc_ctx* c, const uint32_t* h_points, uint32_t n_points, uint32_t mult, void* d_ws,
                         uint64_t ws_bytes, uint32_t* d_hit, uint64_t* d_flops, uint8_t* d_bypass,
                         uint32_t* h_first_evict, void* stream) {
  const uint32_t nv = (uint32_t)c->hv.size();
  const uint64_t per = ws_bytes_per_worker(c->ncap, c->hcap);
  if (ws_bytes < kCtrl + per * nv) return fail(MC_ENOMEM, "workspace too small for the live pass");
  const uint32_t K = n_points;
  std::vector<DevSnapOut> outs(nv);
  for (uint32_t v = 0; v < nv; v++) {
    SnapStore& s = c->snaps[v];
    s.release();
    const uint64_t cap = (uint64_t)K * c->ncap;
    if (cudaMalloc(&s.nodes, sizeof(mc_snap_node) * cap) != cudaSuccess ||
        cudaMalloc(&s.pidx, sizeof(uint32_t) * cap) != cudaSuccess ||
        cudaMalloc(&s.off, sizeof(uint64_t) * (K + 1)) != cudaSuccess ||
        cudaMalloc(&s.n, sizeof(uint32_t) * K) != cudaSuccess ||
        cudaMalloc(&s.nid, sizeof(uint32_t) * K) != cudaSuccess) {
      s.release();
      return fail(MC_ENOMEM, "snapshot store allocation failed");
    }
    s.count = K;
    s.cap = cap;
    outs[v].nodes = s.nodes;
    outs[v].pidx = s.pidx;
    outs[v].off = s.off;
    outs[v].n = s.n;
    outs[v].nid = s.nid;
    outs[v].stride = c->ncap;
    outs[v].count = K;
    outs[v].pad = 0;
  }
  cudaFree(c->d_points);
  c->d_points = nullptr;
  cudaFree(c->d_live_cyc);
  c->d_live_cyc = nullptr;
  CU(cudaMalloc(&c->d_points, sizeof(uint32_t) * (K + nv)));
  CU(cudaMalloc(&c->d_live_cyc, sizeof(unsigned long long) * K * nv));
  CU(cudaMemsetAsync(c->d_live_cyc, 0, sizeof(unsigned long long) * K * nv, (cudaStream_t)stream));
  c->live_points = K;
  cudaStream_t st = (cudaStream_t)stream;
  DevSnapOut* d_outs = (DevSnapOut*)((char*)d_ws + 256);
  if (sizeof(DevSnapOut) * nv + 256 > kCtrl) return fail(MC_EINVAL, "too many variants for the live pass");
  CU(cudaMemcpyAsync(d_outs, outs.data(), sizeof(DevSnapOut) * nv, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(c->d_points, h_points, sizeof(uint32_t) * K, cudaMemcpyHostToDevice, st));
  {  // every snapshot starts empty (a bootstrap point the pass never reaches stays so)
    std::vector<uint64_t> off0(K);
    std::vector<uint32_t> nid0(K, 1);
    for (uint32_t k = 0; k < K; k++) off0[k] = (uint64_t)k * c->ncap;
    for (uint32_t v = 0; v < nv; v++) {
      CU(cudaMemsetAsync(c->snaps[v].n, 0, sizeof(uint32_t) * K, st));
      CU(cudaMemcpyAsync(c->snaps[v].off, off0.data(), sizeof(uint64_t) * K, cudaMemcpyHostToDevice, st));
      CU(cudaMemcpyAsync(c->snaps[v].nid, nid0.data(), sizeof(uint32_t) * K, cudaMemcpyHostToDevice, st));
    }
  }
  KParams P;
  memset(&P, 0, sizeof(P));
  P.tok = c->tok;
  P.n_tok = c->n_tok;
  P.req = c->req;
  P.n_req = c->n_req;
  P.n_var = nv;
  P.var = c->d_var;
  P.ncap = c->ncap;
  P.hcap = c->hcap;
  P.n_workers = nv;
  P.ws = (char*)d_ws + kCtrl;
  P.ws_stride = per;
  P.hit = d_hit;
  P.flops = (unsigned long long*)d_flops;
  P.bypass = d_bypass;
  P.status = c->d_status;
  P.live_out = d_outs;
  P.live_points = c->d_points;
  P.n_points = K;
  P.first_evict = c->d_points + K;
  P.live_mult = mult;
  P.live_cyc = c->d_live_cyc;
  P.smem_nodes = c->smem_nodes_live;
  live_kernel<<<nv, 32, 8ull * c->smem_nodes_live, st>>>(P);
  CU(cudaGetLastError());
  // the last snapshot offset entry (K) for completeness
  std::vector<uint64_t> offK(1, (uint64_t)K * c->ncap);
  for (uint32_t v = 0; v < nv; v++)
    CU(cudaMemcpyAsync(c->snaps[v].off + K, offK.data(), sizeof(uint64_t), cudaMemcpyHostToDevice, st));
  if (h_first_evict)
    CU(cudaMemcpyAsync(h_first_evict, c->d_points + K, sizeof(uint32_t) * nv, cudaMemcpyDeviceToHost, st));
  CU(cudaStreamSynchronize(st));
  mc_status rc = upload_stores(c);
  for (uint32_t v = 0; v < nv && rc == MC_OK; v++) rc = build_images(c, v, st);
  return rc;
}
}  // namespace

mc_status mc_live_pass_at(mc_ctx* c, const uint32_t* h_points, uint32_t n_points, void* d_ws, uint64_t ws_bytes,
                          uint32_t* d_hit, uint64_t* d_flops, uint8_t* d_bypass, uint32_t* h_first_evict,
                          void* stream) {
  if (!c || !d_ws || !h_points || n_points == 0) return fail(MC_EINVAL, "mc_live_pass_at: bad argument");
  if (!c->tok) return fail(MC_ESTATE, "mc_live_pass before mc_set_trace");
  if (h_points[0] != 0) return fail(MC_EINVAL, "snapshot point 0 must be 0 (the empty tree)");
  for (uint32_t k = 1; k < n_points; k++)
    if (h_points[k] <= h_points[k - 1] || h_points[k] > c->n_req)
      return fail(MC_EINVAL, "snapshot points must be strictly increasing request indices <= n_reqs");
  return live_pass_impl(c, h_points, n_points, 0, d_ws, ws_bytes, d_hit, d_flops, d_bypass, h_first_evict, stream);
}

mc_status mc_live_pass_bootstrap(mc_ctx* c, uint32_t multiplier, void* d_ws, uint64_t ws_bytes, uint32_t* d_hit,
                                 uint64_t* d_flops, uint8_t* d_bypass, uint32_t* h_first_evict, void* stream) {
  if (!c || !d_ws || multiplier == 0) return fail(MC_EINVAL, "mc_live_pass_bootstrap: bad argument");
  if (!c->tok) return fail(MC_ESTATE, "mc_live_pass before mc_set_trace");
  const uint32_t pts[3] = {0, 0, 0};  // (dynamic: found during the pass)
  return live_pass_impl(c, pts, 3, multiplier, d_ws, ws_bytes, d_hit, d_flops, d_bypass, h_first_evict, stream);
}

mc_status mc_live_pass(mc_ctx* c, uint32_t window, void* d_ws, uint64_t ws_bytes, uint32_t* d_hit,
                       uint64_t* d_flops, uint8_t* d_bypass, void* stream) {
  if (!c || window == 0) return fail(MC_EINVAL, "mc_live_pass: bad argument");
  if (!c->tok) return fail(MC_ESTATE, "mc_live_pass before mc_set_trace");
  std::vector<uint32_t> pts;
  for (uint64_t r = 0; r < c->n_req; r += window) pts.push_back((uint32_t)r);
  return mc_live_pass_at(c, pts.data(), (uint32_t)pts.size(), d_ws, ws_bytes, d_hit, d_flops, d_bypass, nullptr,
                         stream);
}

mc_status mc_snapshot_count(const mc_ctx* c, uint32_t variant, uint32_t* n_out) {
  if (!c || !n_out || variant >= c->hv.size()) return fail(MC_EINVAL, "mc_snapshot_count: bad argument");
  *n_out = c->snaps[variant].count;
  return MC_OK;
}

mc_status mc_live_window_cycles(mc_ctx* c, uint32_t variant, uint64_t* h_out, uint32_t cap, uint32_t* n_out) {
  if (!c || !n_out || variant >= c->hv.size()) return fail(MC_EINVAL, "mc_live_window_cycles: bad argument");
  if (!c->d_live_cyc) return fail(MC_ESTATE, "mc_live_window_cycles before a live pass");
  *n_out = c->live_points;
  if (!h_out) return MC_OK;
  if (cap < c->live_points) return fail(MC_EINVAL, "output buffer too small");
  CU(cudaDeviceSynchronize());
  CU(cudaMemcpy(h_out, c->d_live_cyc + (uint64_t)variant * c->live_points, sizeof(uint64_t) * c->live_points,
                cudaMemcpyDeviceToHost));
  return MC_OK;
}

mc_status mc_get_snapshot(mc_ctx* c, uint32_t variant, uint32_t k, mc_snap_node* h_out, uint64_t cap,
                          uint64_t* n_out, uint32_t* next_id) {
  if (!c || !n_out || variant >= c->hv.size()) return fail(MC_EINVAL, "mc_get_snapshot: bad argument");
  const SnapStore& s = c->snaps[variant];
  if (k >= s.count) return fail(MC_EINVAL, "snapshot index out of range");
  CU(cudaDeviceSynchronize());
  uint64_t off = 0;
  uint32_t n = 0, nid = 0;
  CU(cudaMemcpy(&off, s.off + k, sizeof(uint64_t), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(&n, s.n + k, sizeof(uint32_t), cudaMemcpyDeviceToHost));
  CU(cudaMemcpy(&nid, s.nid + k, sizeof(uint32_t), cudaMemcpyDeviceToHost));
  *n_out = n;
  if (next_id) *next_id = nid;
  if (!h_out) return MC_OK;
  if (cap < n) return fail(MC_EINVAL, "output buffer too small");
  CU(cudaMemcpy(h_out, s.nodes + off, sizeof(mc_snap_node) * n, cudaMemcpyDeviceToHost));
  std::sort(h_out, h_out + n, [](const mc_snap_node& a, const mc_snap_node& b) { return a.id < b.id; });
  return MC_OK;
}

mc_status mc_set_segments(mc_ctx* c, const mc_segment* h_segs, uint32_t n_segs) {
  if (!c || !h_segs || n_segs == 0) return fail(MC_EINVAL, "mc_set_segments: bad argument");
  if (!c->tok) return fail(MC_ESTATE, "mc_set_segments before mc_set_trace");
  for (uint32_t i = 0; i < n_segs; i++) {
    const mc_segment& s = h_segs[i];
    if (s.n_req == 0) return fail(MC_EINVAL, "segment " + std::to_string(i) + ": empty window (n_req == 0)");
    if (s.first_req < 1 || (uint64_t)s.first_req + s.n_req - 1 > c->n_req)
      return fail(MC_EINVAL, "segment " + std::to_string(i) + " outside the trace");
  }
  cudaFree(c->d_segs);
  c->d_segs = nullptr;
  CU(cudaMalloc(&c->d_segs, sizeof(mc_segment) * n_segs));
  CU(cudaMemcpy(c->d_segs, h_segs, sizeof(mc_segment) * n_segs, cudaMemcpyHostToDevice));
  c->segs.assign(h_segs, h_segs + n_segs);
  return MC_OK;
}

mc_status mc_replay(mc_ctx* c, const mc_replay_args* A, void* stream) {
  if (!c || !A) return fail(MC_EINVAL, "mc_replay: null argument");
  if (!c->tok || c->segs.empty()) return fail(MC_ESTATE, "mc_replay before mc_set_trace/mc_set_segments");
  if (!A->h_alphas || A->n_alpha == 0 || A->n_alpha > c->alpha_cap) return fail(MC_EINVAL, "bad alpha grid");
  for (uint32_t i = 0; i < A->n_alpha; i++)
    if (!(A->h_alphas[i] >= 0.0) || A->h_alphas[i] == __builtin_inf())
      return fail(MC_EINVAL, "alpha must be finite and >= 0 (SPEC:308)");
  if (!A->d_workspace || !A->d_hit || !A->d_flops || !A->d_hit_sum) return fail(MC_EINVAL, "null output buffer");
  const uint32_t nv = (uint32_t)c->hv.size(), ns = (uint32_t)c->segs.size();
  const uint64_t total_chains = (uint64_t)nv * A->n_alpha * ns;
  if (total_chains >= (1ull << 32)) return fail(MC_EINVAL, "too many chains");
  for (uint32_t v = 0; v < nv; v++)
    for (const auto& s : c->segs)
      if (s.snapshot >= c->snaps[v].count)
        return fail(MC_ESTATE, "segment snapshot index missing for variant " + std::to_string(v));
  const uint32_t n_chains = A->h_chains ? A->n_chains : (uint32_t)total_chains;
  if (n_chains == 0) return MC_OK;
  // chain ids, Marconi chains first, then vLLM+ chains (each group keeps the caller's order)
  std::vector<uint32_t> ids;
  ids.reserve(n_chains);
  uint32_t n_marconi = 0;
  for (int pass = 0; pass < 2; pass++)
    for (uint32_t i = 0; i < n_chains; i++) {
      const uint32_t id = A->h_chains ? A->h_chains[i] : i;
      if (id >= total_chains) return fail(MC_EINVAL, "chain id out of range");
      const bool vl = c->hv[id / (ns * A->n_alpha)].block_size != 0;
      if (vl == (pass == 1)) ids.push_back(id);
      if (pass == 0 && !vl) n_marconi++;
    }
  const uint64_t fixed = kCtrl + ids_bytes(n_chains);
  const uint64_t per = ws_bytes_per_worker(c->ncap, c->hcap);
  if (A->workspace_bytes < fixed + per) return fail(MC_ENOMEM, "workspace too small");
  uint32_t workers = (uint32_t)((A->workspace_bytes - fixed) / per);
  if (A->n_workers) workers = std::min(workers, A->n_workers);
  workers = std::min(workers, n_chains);
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = (char*)A->d_workspace;
  char* ids_at = ws + (A->workspace_bytes - ids_bytes(n_chains)) / 256 * 256;
  // the α grid travels with the call (in its workspace), so concurrent calls on other
  // streams with other workspaces never see each other's grid
  CU(cudaMemsetAsync(ws, 0, 256, st));
  CU(cudaMemcpyAsync(ws + kAlphaOff, A->h_alphas, sizeof(double) * A->n_alpha, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(ids_at, ids.data(), 4ull * n_chains, cudaMemcpyHostToDevice, st));
  KParams P;
  memset(&P, 0, sizeof(P));
  P.tok = c->tok;
  P.n_tok = c->n_tok;
  P.req = c->req;
  P.n_req = c->n_req;
  P.n_var = nv;
  P.var = c->d_var;
  P.snap = c->d_stores;
  P.segs = c->d_segs;
  P.n_segs = ns;
  P.n_alpha = A->n_alpha;
  P.alphas = (const double*)(ws + kAlphaOff);
  P.chains = (const uint32_t*)ids_at;
  P.n_chains = n_chains;
  P.ncap = c->ncap;
  P.hcap = c->hcap;
  P.n_workers = workers;
  P.queue = (unsigned*)ws;
  P.ws = ws + kCtrl;
  P.ws_stride = per;
  P.hit = A->d_hit;
  P.flops = (unsigned long long*)A->d_flops;
  P.bypass = A->d_bypass;
  P.hit_sum = (unsigned long long*)A->d_hit_sum;
  P.counters = (unsigned long long*)A->d_counters;
  P.log = A->d_log;
  P.log_cap = A->log_cap;
  P.log_n = A->d_log_n;
  P.chain_cycles = A->d_chain_ns;
  P.status = c->d_status;
  uint32_t S = A->smem_nodes ? A->smem_nodes : c->smem_nodes;
  S = std::min<uint32_t>(S, c->ncap) & ~31u;
  if (kWarpsPerCta * 8ull * S > c->smem_optin) return fail(MC_EINVAL, "smem_nodes exceeds shared memory");
  if (S < 32) return fail(MC_EINVAL, "smem_nodes must be >= 32 (14 slots hold the chain counters, constants and the copy mbarrier)");
  P.smem_nodes = S;
  // the lean Marconi instantiation unless this call logs evictions or a Marconi variant
  // uses chunked checkpoints or has no SSM layers
  bool lean = A->d_log == nullptr;
  for (const auto& v : c->hv)
    if (v.block_size == 0 && (v.chunk_size != 0 || v.model.n_ssm == 0)) lean = false;
  // one launch per policy group, back to back on `st` (they share the worker slices);
  // each launch has its own queue word
  const uint32_t groups[2] = {n_marconi, n_chains - n_marconi};
  uint32_t first = 0;
  for (int g = 0; g < 2; g++) {
    if (groups[g] == 0) continue;
    P.chains = (const uint32_t*)ids_at + first;
    P.n_chains = groups[g];
    P.queue = (unsigned*)ws + 16 * g;
    P.n_workers = std::min(workers, groups[g]);
    const uint32_t ctas = (P.n_workers + kWarpsPerCta - 1) / kWarpsPerCta;
    if (g == 0 && lean)
      replay_kernel<0, false><<<ctas, 32 * kWarpsPerCta, kWarpsPerCta * 8ull * S, st>>>(P);
    else if (g == 0)
      replay_kernel<0, true><<<ctas, 32 * kWarpsPerCta, kWarpsPerCta * 8ull * S, st>>>(P);
    else
      replay_kernel<1, true><<<ctas, 32 * kWarpsPerCta, kWarpsPerCta * 8ull * S, st>>>(P);
    CU(cudaGetLastError());
    first += groups[g];
  }
  return MC_OK;
}

mc_status mc_eviction_log(mc_ctx* c, const mc_replay_args* A, uint32_t v, uint32_t a, uint32_t s,
                          mc_evict_rec* h_out, uint64_t cap, uint64_t* n_out, void* stream) {
  if (!c || !A || !n_out) return fail(MC_EINVAL, "mc_eviction_log: null argument");
  if (!A->d_log || !A->d_log_n) return fail(MC_EINVAL, "mc_eviction_log: the replay call had no log buffers");
  const uint32_t nv = (uint32_t)c->hv.size(), ns = (uint32_t)c->segs.size();
  if (v >= nv || a >= A->n_alpha || s >= ns) return fail(MC_EINVAL, "mc_eviction_log: chain out of range");
  const uint64_t chain = ((uint64_t)v * A->n_alpha + a) * ns + s;
  CU(cudaStreamSynchronize((cudaStream_t)stream));
  uint32_t n = 0;
  CU(cudaMemcpy(&n, A->d_log_n + chain, sizeof(uint32_t), cudaMemcpyDeviceToHost));
  *n_out = n;
  if (h_out) {
    const uint64_t k = std::min<uint64_t>(std::min<uint64_t>(n, A->log_cap), cap);
    if (k) CU(cudaMemcpy(h_out, A->d_log + chain * A->log_cap, k * sizeof(mc_evict_rec), cudaMemcpyDeviceToHost));
  }
  return MC_OK;
}

mc_status mc_chain_sums(mc_ctx* c, uint32_t n_alpha, const uint32_t* d_hit, const uint64_t* d_flops,
                        const uint32_t* d_chains, uint32_t n_chains, uint64_t* d_out, void* stream) {
  if (!c || !d_hit || !d_flops || (n_chains && (!d_chains || !d_out)) || n_alpha == 0)
    return fail(MC_EINVAL, "mc_chain_sums: bad argument");
  if (!c->tok || c->segs.empty()) return fail(MC_ESTATE, "mc_chain_sums before mc_set_trace/mc_set_segments");
  if (n_chains == 0) return MC_OK;
  const uint32_t ns = (uint32_t)c->segs.size();
  chain_sums_kernel<<<(n_chains + 7) / 8, 256, 0, (cudaStream_t)stream>>>(
      c->req, c->d_segs, ns, n_alpha, (uint32_t)c->hv.size(), c->n_req, d_chains, n_chains, d_hit,
      (const unsigned long long*)d_flops, (unsigned long long*)d_out, c->d_status);
  CU(cudaGetLastError());
  return MC_OK;
}

mc_status mc_lookup(mc_ctx* c, const mc_lookup_query* h_q, uint32_t n, void* d_ws, uint64_t ws_bytes,
                    mc_lookup_result* d_out, void* stream) {
  if (!c || (n && (!h_q || !d_ws || !d_out))) return fail(MC_EINVAL, "mc_lookup: null argument");
  if (!c->tok) return fail(MC_ESTATE, "mc_lookup before mc_set_trace");
  if (n == 0) return MC_OK;
  const uint32_t nv = (uint32_t)c->hv.size();
  std::vector<uint32_t> perm(n);
  for (uint32_t i = 0; i < n; i++) {
    const mc_lookup_query& q = h_q[i];
    if (q.reserved) return fail(MC_EINVAL, "mc_lookup_query.reserved must be 0");
    if (q.variant >= nv) return fail(MC_EINVAL, "query " + std::to_string(i) + ": variant out of range");
    if (c->hv[q.variant].block_size) return fail(MC_EINVAL, "mc_lookup: vLLM+ variants (block_size > 0) have no lookup");
    if (q.snapshot >= c->snaps[q.variant].count) return fail(MC_ESTATE, "query " + std::to_string(i) + ": no such snapshot");
    if (q.req < 1 || q.req > c->n_req) return fail(MC_EINVAL, "query " + std::to_string(i) + ": request out of range");
    perm[i] = i;
  }
  std::stable_sort(perm.begin(), perm.end(), [&](uint32_t a, uint32_t b) {
    return h_q[a].variant != h_q[b].variant ? h_q[a].variant < h_q[b].variant : h_q[a].snapshot < h_q[b].snapshot;
  });
  std::vector<uint32_t> groups;  // {variant, snapshot, first, count} per group
  for (uint32_t i = 0; i < n; i++) {
    const mc_lookup_query& q = h_q[perm[i]];
    const size_t G = groups.size();
    if (G && groups[G - 4] == q.variant && groups[G - 3] == q.snapshot) groups[G - 1]++;
    else { groups.push_back(q.variant); groups.push_back(q.snapshot); groups.push_back(i); groups.push_back(1); }
  }
  const uint32_t n_groups = (uint32_t)(groups.size() / 4);
  // workspace: control header | worker slices | perm | groups | queries
  const uint64_t tail = ((4ull * n + 15) & ~15ull) + 16ull * n_groups + sizeof(mc_lookup_query) * n;
  const uint64_t per = ws_bytes_per_worker(c->ncap, c->hcap);
  if (ws_bytes < kCtrl + per + tail) return fail(MC_ENOMEM, "workspace too small for mc_lookup");
  const uint32_t workers = (uint32_t)std::min<uint64_t>((ws_bytes - kCtrl - tail) / per, n_groups);
  cudaStream_t st = (cudaStream_t)stream;
  char* ws = (char*)d_ws;
  char* at = ws + kCtrl + (uint64_t)workers * per;
  uint32_t* d_perm = (uint32_t*)at;
  uint4* d_groups = (uint4*)(at + ((4ull * n + 15) & ~15ull));
  mc_lookup_query* d_q = (mc_lookup_query*)((char*)d_groups + 16ull * n_groups);
  CU(cudaMemcpyAsync(d_perm, perm.data(), 4ull * n, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(d_groups, groups.data(), 16ull * n_groups, cudaMemcpyHostToDevice, st));
  CU(cudaMemcpyAsync(d_q, h_q, sizeof(mc_lookup_query) * n, cudaMemcpyHostToDevice, st));
  KParams P;
  memset(&P, 0, sizeof(P));
  P.tok = c->tok;
  P.n_tok = c->n_tok;
  P.req = c->req;
  P.n_req = c->n_req;
  P.n_var = nv;
  P.var = c->d_var;
  P.snap = c->d_stores;
  P.ncap = c->ncap;
  P.hcap = c->hcap;
  P.n_workers = workers;
  P.ws = ws + kCtrl;
  P.ws_stride = per;
  P.status = c->d_status;
  lookup_kernel<<<workers, 32, 0, st>>>(P, d_groups, n_groups, d_perm, d_q, d_out);
  CU(cudaGetLastError());
  return MC_OK;
}

mc_status mc_check(mc_ctx* c, void* stream) {
  if (!c) return fail(MC_EINVAL, "mc_check: null context");
  CU(cudaStreamSynchronize((cudaStream_t)stream));
  uint32_t sw[2] = {0, 0};
  CU(cudaMemcpy(sw, c->d_status, 2 * sizeof(uint32_t), cudaMemcpyDeviceToHost));
  const uint32_t st = sw[0];
  if (st) {
    cudaMemset(c->d_status, 0, sizeof(uint32_t));
    cudaMemset(c->d_status + 1, 0xFF, sizeof(uint32_t));
    if (st & ST_BADTRACE)
      return fail(MC_EINVAL, "trace rejected by the device check: request " + std::to_string(sw[1]) +
                                 " has input_len == 0, a range outside the pool, or is too long (2^20 tokens / "
                                 "F(L) < 2^53)");
    std::string m = "device status:";
    if (st & ST_OVERFLOW) m += " node-table overflow (raise max_nodes);";
    if (st & ST_INVARIANT) m += " invariant violated (capacity / hit <= input / snapshot);";
    if (st & ST_NOCAND) m += " no eviction candidate;";
    if (st & ST_SNAPOVF) m += " snapshot store overflow;";
    return fail((st & (ST_OVERFLOW | ST_SNAPOVF)) ? MC_EOVERFLOW : MC_EDEVICE, m);
  }
  return MC_OK;
}

mc_status mc_node_cost(const mc_model* m, uint32_t n, const uint32_t* ds, const uint32_t* de, const uint8_t* ssm,
                       uint64_t* saved, uint64_t* bytes, double* eff, void* stream) {
  if (!m || (n && (!ds || !de || !ssm || !saved || !bytes || !eff))) return fail(MC_EINVAL, "mc_node_cost: null");
  if (n == 0) return MC_OK;
  const int blocks = (int)std::min<uint32_t>((n + 255) / 256, 148 * 8);
  node_cost_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(make_model(*m), n, ds, de, ssm,
                                                             (unsigned long long*)saved, (unsigned long long*)bytes,
                                                             eff);
  CU(cudaGetLastError());
  return MC_OK;
}

mc_status mc_score_argmin(uint32_t n_tables, const uint32_t* off, const uint32_t* t, const uint8_t* cand,
                          const uint32_t* id, const double* eff, const double* alpha, uint32_t* best, double* u,
                          void* stream) {
  if (n_tables == 0) return MC_OK;
  if (!off || !t || !cand || !id || !eff || !alpha || !best || !u) return fail(MC_EINVAL, "mc_score_argmin: null");
  const int wpb = 4;
  score_argmin_kernel<<<(n_tables + wpb - 1) / wpb, 32 * wpb, 0, (cudaStream_t)stream>>>(n_tables, off, t, cand, id,
                                                                                         eff, alpha, best, u);
  CU(cudaGetLastError());
  return MC_OK;
}

}  // extern "C"
