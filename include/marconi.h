/*
 * marconi.h -- C ABI of libmarconi.so: B200 (sm_100a) α-grid trace replay of
 * Marconi's hybrid-model radix-tree prefix cache (arXiv 2411.19379).
 *
 * The method:
 *   - hybrid "all-or-nothing" longest-prefix lookup: a hit needs the KVs of every
 *     prefix token and one SSM state that matches the prefix exactly
 *     (§3; §2.2);
 *   - judicious admission by speculative insertion: checkpoint the SSM state at a
 *     branch point found by a dry-run insertion of the input, and at the last
 *     decoded token (§4.1, fig:spec_insertion);
 *   - FLOP-aware eviction: utility S(n) = recency(n) + α·flop_efficiency(n)
 *     (Eq. 2), both min-max normalised over all nodes,
 *     flop_efficiency = FLOPs saved / bytes of all states (Eq. 1, PAPER:395-397,
 *     Appendix A tab:flops_breakdown PAPER:771-772, conv_1d PAPER:814), the
 *     argmin evicted until the request fits; candidates are nodes
 *     with <= 1 child, an evicted 1-child node is absorbed by its child, a hit
 *     touches only the accessed node (§4.3);
 *   - α tuning: replay the bootstrap requests from a tree snapshot for a grid of
 *     α and adopt the α with the best token hit rate (§4.2).
 * The readings where the paper is silent are listed in DESIGN.md ("Readings").
 *
 * Conventions
 *   - Every function returns an mc_status (negative = error) and never throws.
 *     mc_last_error() returns a thread-local message for the last failure.
 *   - d_* arguments are DEVICE pointers (CUDA global memory, e.g. torch tensors),
 *     h_* arguments are HOST pointers.  The caller owns every buffer it passes;
 *     device buffers passed to mc_set_trace are BORROWED for the context's
 *     lifetime.  Snapshot stores are owned by the context (allocated by the
 *     setup calls mc_set_snapshots / mc_live_pass, freed by mc_destroy).
 *     Nothing is allocated on the replay path.
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *     Compute calls are asynchronous on it; argument errors are returned
 *     synchronously; device-side failures (node-table overflow, an invariant
 *     such as "hit <= input length" or "capacity respected" broken) set a device
 *     status word that mc_check() reads.
 *   - Requests are numbered 1..n_reqs in trace order; request r's logical
 *     timestamp is r (reading R3).
 *   - Results never depend on the stream, the chain order, the chain subset
 *     passed to one call, or the launch configuration.
 */
#ifndef MARCONI_H_
#define MARCONI_H_

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  MC_OK = 0,
  MC_EINVAL = -1,     /* invalid argument (returned synchronously)                 */
  MC_ENOMEM = -2,     /* device allocation failed / workspace too small            */
  MC_ECUDA = -3,      /* CUDA runtime error                                        */
  MC_EOVERFLOW = -4,  /* node table (max_nodes) or snapshot store overflow         */
  MC_ESTATE = -5,     /* call order (e.g. replay before set_trace)                 */
  MC_EDEVICE = -6     /* device status word: an invariant was violated on device   */
} mc_status;

/* ModelConfig: layer counts {Attention, SSM, MLP}, D = d_model,
 * N = d_state, bytes per parameter (1, 2 or 4; fp16 = 2) and the
 * conv_1d state shape. */
typedef struct {
  uint32_t n_attn, n_ssm, n_mlp, d_model, d_state, bytes_per_param, conv_in, conv_kernel;
} mc_model;

/* One cache configuration.  capacity_bytes = UINT64_MAX means unlimited bytes,
 * 0 = no cache (every request bypasses admission).  capacity_nodes
 * caps the number of non-root nodes (0 = no node cap; the toy config uses 6).
 * chunk_size = 0: exact checkpoint positions (two-pass prefill);
 * chunk_size = c > 0: chunked state passing -- the prefill (branch) checkpoint is
 * placed at the multiple of c at or below the branch point and skipped if that is 0
 * or not beyond the hit; decode checkpoints stay exact.
 * block_size = 0: the Marconi policy above.  block_size = x > 0: the vLLM+
 * baseline instead: "fine-grained checkpointing ... a state
 * for every token block" of x tokens (PAPER:302, PAPER:532 uses x = 32) with vLLM's
 * LRU policy -- every full block of a sequence is a cache node holding its KVs and
 * the SSM states at its end; a hit is the deepest cached block boundary <= the
 * input length; the matched blocks are touched; LRU evicts leaf blocks (min
 * (t_last, id)); the readings are DESIGN.md V1-V8.  α is ignored (chains of a
 * vLLM+ variant replay identically for every α).  chunk_size must be 0 then.
 * reserved must be 0. */
typedef struct {
  mc_model model;
  uint64_t capacity_bytes;
  uint32_t capacity_nodes;
  uint32_t chunk_size;
  uint32_t block_size;
  uint32_t reserved;
} mc_variant;

/* Request r (1-based, at index r-1): sequence = tokens[tok_off, tok_off + input_len
 * + output_len), input = the first input_len tokens. */
typedef struct {
  uint64_t tok_off;
  uint32_t input_len, output_len;
} mc_request;

/* Canonical snapshot record (one radix node).  id 0 is the root (never listed);
 * parent_id 0 = child of the root.  The node's edge is tokens[ref_off + d_start,
 * ref_off + d_end); its SSM state (if has_ssm) represents depth d_end.  For a
 * vLLM+ variant every record is one block: d_end - d_start = block_size,
 * d_start a multiple of it, has_ssm = 1. */
typedef struct {
  uint32_t id, parent_id;
  uint64_t ref_off;
  uint32_t d_start, d_end, t_last, has_ssm;
} mc_snap_node;

/* Replay window: requests first_req .. first_req + n_req - 1 from snapshot
 * `snapshot` of the chain's variant (SURVEY.md §8(c) c.2 "Grid"). */
typedef struct {
  uint32_t first_req, n_req, snapshot, reserved;
} mc_segment;

/* One eviction: request, victim node id, kind (0 leaf removal, 1 absorption
 * into the single child), live non-root nodes scanned, utility S (Eq. 2). */
typedef struct {
  uint32_t req, node_id, kind, n_live;
  double utility;
} mc_evict_rec;

typedef struct mc_ctx mc_ctx;

/* Create a context for n_variants cache variants.  max_nodes (power of two,
 * 64 .. 16384) sizes each chain's node table; exceeding it is MC_EOVERFLOW.
 * Validation: bytes_per_param in {1,2,4}; n_attn >= 1 (a node without KVs and
 * without state would be zero bytes); d_model >= 1. */
mc_status mc_create(const mc_variant* h_variants, uint32_t n_variants, uint32_t max_nodes, int device,
                    mc_ctx** out);
void mc_destroy(mc_ctx* ctx);

/* Borrow the trace (device pointers).  Validated synchronously (input_len >= 1,
 * ranges inside the pool, n_reqs < 2^30, n_tokens < 2^32). */
mc_status mc_set_trace(mc_ctx* ctx, const uint32_t* d_tokens, uint64_t n_tokens, const mc_request* d_reqs,
                       uint32_t n_reqs);

/* The same, validated on the device instead (no request table travels back to the
 * host): a check kernel on `stream` applies the rules above plus the longest
 * admissible request (2^20 tokens and F(L) < 2^53, Appendix A); a violation makes
 * the replay and live kernels on that stream read nothing and the next mc_check
 * return MC_EINVAL naming the first bad request.  Scalar arguments are validated
 * synchronously.  The end-to-end path of bench.py uses it. */
mc_status mc_set_trace_async(mc_ctx* ctx, const uint32_t* d_tokens, uint64_t n_tokens, const mc_request* d_reqs,
                             uint32_t n_reqs, void* stream);

/* Upload n_snapshots canonical snapshots for `variant` from host memory:
 * snapshot k is h_nodes[h_offsets[k] .. h_offsets[k+1]) with next node id
 * h_next_id[k].  Records may be in any order; parent links are resolved on the
 * device.  Replaces the variant's snapshot store.  Asynchronous on `stream`:
 * records are validated on the host before return, parent links on the device
 * (mc_check reports a broken link); pageable host arrays may be reused on return,
 * page-locked h_nodes must stay unchanged until the stream has passed the call.
 * Work on other streams must not replay this context while the upload runs. */
mc_status mc_set_snapshots(mc_ctx* ctx, uint32_t variant, const mc_snap_node* h_nodes, const uint64_t* h_offsets,
                           const uint32_t* h_next_id, uint32_t n_snapshots, void* stream);

/* The α = 0 live LRU pass (α = 0 falls back to LRU) over the whole
 * trace from an empty cache, for every variant at once, on the device.  Stores
 * snapshot k = the tree after request k*window (k = 0 .. ceil(R/window)-1;
 * snapshot 0 is empty) in each variant's snapshot store, and writes the live
 * per-request outputs d_hit/d_flops/d_bypass [n_variants][n_reqs] (nullable).
 * Needs a workspace of mc_workspace_size(ctx, n_variants) bytes. */
mc_status mc_live_pass(mc_ctx* ctx, uint32_t window, void* d_workspace, uint64_t workspace_bytes,
                       uint32_t* d_hit, uint64_t* d_flops, uint8_t* d_bypass, void* stream);

/* General form: snapshot k = the tree after request h_points[k] (h_points[0] = 0,
 * strictly increasing, <= n_reqs).  h_first_evict (host, nullable) receives per
 * variant the first request whose admission evicted a node (0 = none) -- the point
 * where the paper takes its tuning snapshot (§4.2 "Managing the balance"). */
mc_status mc_live_pass_at(mc_ctx* ctx, const uint32_t* h_points, uint32_t n_points, void* d_workspace,
                          uint64_t workspace_bytes, uint32_t* d_hit, uint64_t* d_flops, uint8_t* d_bypass,
                          uint32_t* h_first_evict, void* stream);

/* The paper's tuning pass in ONE live pass (§4.2 "Managing the balance"):
 * α = 0 from the empty cache; the first request r_F whose admission evicts is found on
 * the fly; snapshot 1 = the tree after r_F, snapshot 2 = the tree after
 * r_F + multiplier * r_F (when that is < n_reqs), snapshot 0 = empty; a snapshot the
 * pass never reaches stays empty.  h_first_evict receives r_F per variant (0 = no
 * eviction).  Per-request outputs and workspace as mc_live_pass_at; multiplier >= 1. */
mc_status mc_live_pass_bootstrap(mc_ctx* ctx, uint32_t multiplier, void* d_workspace, uint64_t workspace_bytes,
                                 uint32_t* d_hit, uint64_t* d_flops, uint8_t* d_bypass, uint32_t* h_first_evict,
                                 void* stream);

/* SM cycles the last live pass (mc_live_pass / mc_live_pass_at) spent on each window
 * between consecutive snapshot points of `variant` (window k = requests after point k
 * up to point k+1, the last one to the end of the trace) -- the α = 0 cost of segment k,
 * which grid.AlphaGrid uses to order chains longest-first.  h_out (host, nullable) gets
 * *n_out = number of points values. */
mc_status mc_live_window_cycles(mc_ctx* ctx, uint32_t variant, uint64_t* h_out, uint32_t cap, uint32_t* n_out);

/* Number of snapshots held for a variant and copy one back as canonical
 * records sorted by id (host).  *n_out receives the record count; h_out may be
 * NULL to query it. */
mc_status mc_snapshot_count(const mc_ctx* ctx, uint32_t variant, uint32_t* n_out);
mc_status mc_get_snapshot(mc_ctx* ctx, uint32_t variant, uint32_t k, mc_snap_node* h_out, uint64_t cap,
                          uint64_t* n_out, uint32_t* next_id);

/* Replay windows.  Chain c = ((variant * n_alpha) + alpha_idx) * n_segs + seg.
 * Each window must hold >= 1 request inside the trace (MC_EINVAL otherwise). */
mc_status mc_set_segments(mc_ctx* ctx, const mc_segment* h_segs, uint32_t n_segs);

/* Workspaces (d_workspace of mc_replay / mc_live_pass) must be ZERO-INITIALISED
 * by the caller when first allocated; they may then be reused across calls of
 * the same context without clearing (the per-worker slices sit at a fixed offset,
 * whatever the chain count of a call).  One workspace serves one call at a time;
 * calls that may overlap (other streams) need their own workspaces -- each call's
 * α grid and chain list travel in its workspace.
 * Workspace bytes for `n_workers` concurrent chains (one warp each; 0 = the
 * default: every SM filled at the kernel's occupancy) and up to n_chains chain
 * ids per mc_replay call (0 = every chain of n_alpha α values). */
mc_status mc_workspace_size(const mc_ctx* ctx, uint32_t n_workers, uint32_t n_alpha, uint32_t n_chains,
                            uint64_t* bytes);
/* Worker count a workspace of `bytes` supports (the replay uses min(this, chains)). */
mc_status mc_workspace_workers(const mc_ctx* ctx, uint64_t bytes, uint32_t n_alpha, uint32_t n_chains,
                               uint32_t* n_workers);

typedef struct {
  const double* h_alphas;   /* [n_alpha], each >= 0 and not NaN            */
  uint32_t n_alpha;
  const uint32_t* h_chains; /* chain ids to run on this call (this rank's shard), in  */
  uint32_t n_chains;        /* the order warps take them (longest first packs best);
                               NULL = all chains in id order                          */
  void* d_workspace;
  uint64_t workspace_bytes;
  uint32_t* d_hit;          /* [n_variants][n_alpha][n_reqs]  hit tokens per request   */
  uint64_t* d_flops;        /* [n_variants][n_alpha][n_reqs]  FLOPs saved = F(hit)     */
  uint8_t* d_bypass;        /* [n_variants][n_alpha][n_reqs]  nullable                 */
  uint64_t* d_hit_sum;      /* [n_variants][n_alpha]  += Σ hits of the chains run      */
  uint64_t* d_counters;     /* [n_chains_total][4] nullable: Σ compared token positions,
                               Σ visited nodes, Σ nodes scanned by evictions,
                               Σ node records written                                 */
  mc_evict_rec* d_log;      /* [n_chains_total][log_cap] nullable: eviction log        */
  uint32_t log_cap;
  uint32_t* d_log_n;        /* [n_chains_total] records produced (may exceed log_cap)  */
  uint32_t* d_chain_ns;     /* [n_chains_total] nullable: per-chain SM cycles / 1024    */
  uint32_t n_workers;       /* 0 = default (derived from the workspace size)          */
  uint32_t smem_nodes;      /* dense live-list positions per chain held in shared
                               memory (0 = auto: fill the SM at the target occupancy) */
} mc_replay_args;

/* The α-grid replay (§4.2 "Managing the balance": replay the
 * bootstrap requests from the tree snapshot for every α of the grid; here one chain =
 * (variant, α, segment)).  Asynchronous on `stream`.  Each chain loads its segment's
 * snapshot and replays its window request by request -- hybrid lookup + speculative
 * insertion, admission, Eq. 2 eviction
 * until the request fits -- writing d_hit / d_flops / d_bypass
 * per request and adding its Σ hits to d_hit_sum[variant][alpha].  Argument errors
 * (NaN / negative / infinite α, bad chain ids, workspace too small, missing
 * snapshots) return synchronously; device-side failures go to mc_check. */
mc_status mc_replay(mc_ctx* ctx, const mc_replay_args* args, void* stream);

/* Copy one chain's eviction log of an mc_replay call to the host (SURVEY.md §8(b)
 * mc_eviction_log).  `args` = the arguments of that call (d_log, d_log_n, log_cap and
 * n_alpha are used); chain = ((variant * n_alpha) + alpha_idx) * n_segs + seg.
 * Synchronises `stream` first.  *n_out = evictions the chain made in that call (may
 * exceed log_cap: only the first log_cap were recorded); h_out (nullable) receives
 * min(*n_out, log_cap, cap) records in eviction order.  MC_EINVAL if the call had no log. */
mc_status mc_eviction_log(mc_ctx* ctx, const mc_replay_args* args, uint32_t variant, uint32_t alpha_idx,
                          uint32_t seg, mc_evict_rec* h_out, uint64_t cap, uint64_t* n_out, void* stream);

/* Per-chain sums of a replay's outputs (token hit rate = skipped prefill
 * tokens / input tokens; FLOPs saved): for each chain id d_chains[i] (device, as passed to
 * mc_replay), d_out[4i .. 4i+3] = {Σ hit, Σ input_len, Σ FLOPs saved low 64 bits, high 64
 * bits} over the chain's segment window, read from the replay's d_hit / d_flops
 * ([n_variants][n_alpha][n_reqs]).  One warp per chain, async on `stream`; a chain id
 * outside [0, n_variants * n_alpha * n_segments) is skipped and flagged for mc_check. */
mc_status mc_chain_sums(mc_ctx* ctx, uint32_t n_alpha, const uint32_t* d_hit, const uint64_t* d_flops,
                        const uint32_t* d_chains, uint32_t n_chains, uint64_t* d_out, void* stream);

/* Standalone batched lookup (SURVEY.md §8(a) a2-a3 as a query; PAPER:246, 300-301,
 * 356-365, 371-373, 380): for each query, request `req` (1-based) of the trace is looked
 * up against snapshot `snapshot` of `variant` (a frozen tree from mc_live_pass* or
 * mc_set_snapshots) without changing it -- steps 1-4 of the replay: the walk, the hit,
 * the speculative-insertion checkpoint and the insertion plan.  Marconi variants only
 * (block_size = 0).  Queries are grouped by (variant, snapshot) on the host; one warp loads
 * a snapshot image into its workspace slice and answers that group.  d_out[i] answers
 * h_queries[i].  Workspace: mc_workspace_size(ctx, n_workers, 1, n_queries).  Async on
 * `stream`; argument errors synchronous. */
typedef struct {
  uint32_t req, variant, snapshot, reserved;  /* reserved must be 0 */
} mc_lookup_query;
typedef struct {
  uint32_t reuse;     /* skipped prefill tokens (the hit)                        */
  uint32_t m;         /* matched length of the full sequence                                 */
  uint32_t p;         /* speculative-insertion checkpoint position (0 = none)                */
  uint32_t hit_id;    /* node whose state is reused (0 = none)                               */
  uint32_t div_id;    /* node where the match ends: mid-edge node, else last full match (0 = root) */
  uint32_t div_off;   /* m - d_start(div node)                                               */
  uint32_t path_len;  /* fully matched nodes + the partially matched one                     */
  uint32_t d_nodes;   /* nodes the insertion would create                                    */
  uint64_t d_bytes;   /* bytes the insertion would add                                       */
} mc_lookup_result;
mc_status mc_lookup(mc_ctx* ctx, const mc_lookup_query* h_queries, uint32_t n_queries, void* d_workspace,
                    uint64_t workspace_bytes, mc_lookup_result* d_out, void* stream);

/* Synchronise `stream` and map the device status word to an mc_status. */
mc_status mc_check(mc_ctx* ctx, void* stream);

const char* mc_last_error(void);

/* ---- unit-level kernels (same device code as the replay), for parity tests ---- */

/* K1 flop_byte_model, batched: per node, saved = F(d_end) - F(d_start) with
 * F(L) = Σ_layers tab:flops_breakdown row 1 (exact u64), bytes = KVs of the edge
 * + has_ssm * (SSM + conv states), eff = saved / bytes (IEEE fp64, Eq. 1). */
mc_status mc_node_cost(const mc_model* h_model, uint32_t n, const uint32_t* d_d_start, const uint32_t* d_d_end,
                       const uint8_t* d_has_ssm, uint64_t* d_saved, uint64_t* d_bytes, double* d_eff, void* stream);

/* K3 score_argmin, segmented: table s is rows [d_off[s], d_off[s+1]) of
 * (t_last, candidate, id, eff); bounds over ALL rows of the table, utility
 * u = rec + α_s * effn (Eq. 2, degenerate range -> 0.5) for candidate rows,
 * victim = lexicographic min (u, t_last, id).  d_best[s] = row index (or
 * 0xFFFFFFFF if no candidate), d_u[s] = its utility. */
mc_status mc_score_argmin(uint32_t n_tables, const uint32_t* d_off, const uint32_t* d_t, const uint8_t* d_cand,
                          const uint32_t* d_id, const double* d_eff, const double* d_alpha, uint32_t* d_best,
                          double* d_u, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* MARCONI_H_ */
