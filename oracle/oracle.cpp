// oracle.cpp -- CPU ORACLE FOR TESTS ONLY.
//
// Test infrastructure, not product code.  Only tests/, __graft_entry__.smoke()
// and bench.py's cpu_baseline / --impl reference legs may load this library.
// It shares no code, header, table or constant with the CUDA path under
// paper_2411_19379_b200/csrc/ (and includes none of it).
//
// What it is: a deliberately plain, slow, step-by-step simulation of Marconi's
// prefix cache (arXiv 2411.19379) -- a pointer radix tree with COPIED edge
// token vectors and std::map children; every derived quantity used by
// eviction (depths, per-node bytes, FLOP efficiency, min/max normalisation,
// total bytes) is recomputed from scratch by a full tree walk at each
// eviction step.  It follows SURVEY.md §8(c) c.2, which restates:
//   * lookup: PAPER.md §3 "all or nothing", §2.2
//   * admission / speculative insertion: §4.1
//   * FLOP efficiency, Eq. 1 with Appendix A
//     tab:flops_breakdown and the conv_1d note
//   * utility, Eq. 2, min-max normalisation,
//     iterative argmin eviction
//   * candidates / absorption / single-node touch: §4.3
// The readings where the paper is silent are SURVEY.md §8(c) c.3 #1-#21 and
// DESIGN.md "Readings"; each is marked [c.3 #k] where it is applied.
//
// Pins: tests/test_oracle_*.py (closed forms, worked examples, brute-force
// flat-list simulator, independent LRU, OPT bound, invariants).
//
// Build: g++ -std=c++17 -O2 -ffp-contract=off -fPIC -shared (see build.py).
#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <map>
#include <stdexcept>
#include <string>
#include <thread>
#include <atomic>
#include <vector>

typedef uint64_t u64;
typedef uint32_t u32;
typedef unsigned __int128 u128;

extern "C" {
struct orc_model {
  u32 n_attn, n_ssm, n_mlp, d_model, d_state, bytes_per_param, conv_in, conv_kernel;
};
// Canonical dump record (SURVEY.md §8(c) c.1 "Canonical dump").
struct orc_node {
  u32 id, parent_id;  // root has id 0
  u64 ref_off;        // pool offset of a request whose sequence has this node's root path as prefix
  u32 d_start, d_end; // token depth range of the node's edge
  u32 t_last;
  u32 has_ssm;
};
// Read-only lookup of one request against the current tree (SURVEY.md §8(a) a2/a3 as a
// standalone query, VERDICT r1 "mc_lookup"): steps 1-4 of c.2 without any mutation.
struct orc_lookup {
  u32 reuse;     // skipped prefill tokens (step 2)
  u32 m;         // matched length of the full sequence (step 1)
  u32 p;         // speculative-insertion checkpoint position after chunk alignment, 0 = none (step 3)
  u32 hit_id;    // node whose state is reused (0 = none)
  u32 div_id;    // node where the walk stopped: the mid-edge node, else the last full match (0 = root)
  u32 div_off;   // m - d_start(div node): tokens of its edge that matched
  u32 path_len;  // |P|: fully matched nodes + the partially matched one
  u32 d_nodes;   // nodes the insertion would create (step 4)
  u64 d_bytes;   // bytes the insertion would add (step 4)
};
struct orc_evict {
  u32 req, node_id, kind;  // kind 0 = leaf removal, 1 = merge (absorption)
  u32 n_live;              // live non-root nodes when this victim was chosen
  double utility;
};
}

static thread_local std::string g_err;

// ---------------------------------------------------------------------------
// Cost model: Appendix A, tab:flops_breakdown.
// All exact in unsigned 64-bit integers; overflow is an error.
// ---------------------------------------------------------------------------
static u64 chk(u128 v) {
  if (v >> 64) throw std::overflow_error("cost model overflow");
  return (u64)v;
}
// FLOPs per Attention layer: 8 L D^2 + 4 L^2 D
static u64 attention_flops(u64 L, const orc_model& m) {
  u128 D = m.d_model;
  return chk(8 * (u128)L * D * D + 4 * (u128)L * L * D);
}
// FLOPs per MLP layer: 16 L D^2
static u64 mlp_flops(u64 L, const orc_model& m) {
  u128 D = m.d_model;
  return chk(16 * (u128)L * D * D);
}
// FLOPs per SSM layer: 12 L D^2 + 16 L D N + 10 L
static u64 ssm_flops(u64 L, const orc_model& m) {
  u128 D = m.d_model, N = m.d_state;
  return chk(12 * (u128)L * D * D + 16 * (u128)L * D * N + 10 * (u128)L);
}
// Total prefill FLOPs of L tokens across all layers (Eq. 1 numerator).
static u64 prefill_flops(u64 L, const orc_model& m) {
  return chk((u128)m.n_attn * attention_flops(L, m) + (u128)m.n_ssm * ssm_flops(L, m) +
             (u128)m.n_mlp * mlp_flops(L, m));
}
// KV bytes of one Attention layer for L tokens: 2 (K,V) * L * D * bytes/param
static u64 kv_bytes_layer(u64 L, const orc_model& m) {
  return chk((u128)2 * L * m.d_model * m.bytes_per_param);
}
// SSM state bytes of one SSM layer: D * N * bytes/param
static u64 ssm_state_bytes_layer(const orc_model& m) {
  return chk((u128)m.d_model * m.d_state * m.bytes_per_param);
}
// conv_1d state bytes of one SSM layer: in_channels * conv_kernel * bytes/param
static u64 conv_state_bytes_layer(const orc_model& m) {
  return chk((u128)m.conv_in * m.conv_kernel * m.bytes_per_param);
}
// Bytes of one node: KVs of its edge tokens over all Attention layers, plus, if
// it holds an SSM checkpoint, the SSM + conv states of all SSM layers [c.3 #14].
static u64 node_bytes(u64 edge_len, bool has_ssm, const orc_model& m) {
  u64 b = chk((u128)m.n_attn * kv_bytes_layer(edge_len, m));
  if (has_ssm) b = chk((u128)b + (u128)m.n_ssm * (ssm_state_bytes_layer(m) + conv_state_bytes_layer(m)));
  return b;
}
// FLOP efficiency, Eq. 1: FLOPs saved by this node relative
// to its parent ("child nodes' FLOP savings are calculated relative
// to parents' savings") divided by the bytes of all its states.
static double flop_efficiency(u64 d_start, u64 d_end, bool has_ssm, const orc_model& m) {
  u64 saved = prefill_flops(d_end, m) - prefill_flops(d_start, m);
  u64 bytes = node_bytes(d_end - d_start, has_ssm, m);
  if (bytes == 0) throw std::invalid_argument("zero-byte node (SPEC:136)");
  return (double)saved / (double)bytes;
}

// ---------------------------------------------------------------------------
// Pointer radix tree.  Edge tokens are copied.
// ---------------------------------------------------------------------------
struct Node {
  u32 id = 0;
  Node* parent = nullptr;
  std::map<u32, Node*> children;  // keyed by first token of the child's edge
  // vLLM+ mode (block trie): children keyed by the child's full block content
  std::map<std::vector<u32>, Node*> bkids;
  std::vector<u32> edge;
  bool has_ssm = false;
  u32 t_last = 0;
  u64 ref_off = 0;
};

static u64 depth_of(const Node* n) {  // recomputed by walking to the root
  u64 d = 0;
  for (const Node* x = n; x->parent; x = x->parent) d += x->edge.size();
  return d;
}

static void collect(Node* n, std::vector<Node*>& out) {  // all non-root nodes, DFS
  for (auto& kv : n->children) {
    out.push_back(kv.second);
    collect(kv.second, out);
  }
  for (auto& kv : n->bkids) {
    out.push_back(kv.second);
    collect(kv.second, out);
  }
}

static void free_subtree(Node* n) {
  for (auto& kv : n->children) free_subtree(kv.second);
  for (auto& kv : n->bkids) free_subtree(kv.second);
  delete n;
}

struct Oracle {
  orc_model model;
  u64 cap_bytes;
  u32 cap_nodes;  // 0 = no node cap
  u32 chunk = 0;  // 0 = exact checkpoint positions; else chunk-aligned prefill checkpoints (NEXT-3)
  double alpha;
  const u32* tokens;
  u64 n_tokens;
  const u64* off;
  const u32* lin;
  const u32* lout;
  u32 n_req;

  Node root;
  u32 next_id = 1;
  u64 total_incremental = 0;
  std::vector<orc_evict> log;
  u64 ctr_compared = 0, ctr_visited = 0, ctr_scanned = 0, ctr_written = 0;

  u32 block = 0;  // 0 = Marconi; x > 0 = vLLM+ baseline with token blocks of x (NEXT-2)

  ~Oracle() {
    for (auto& kv : root.children) free_subtree(kv.second);
    for (auto& kv : root.bkids) free_subtree(kv.second);
  }

  std::vector<u32> seq(u32 r) const {  // full sequence of request r (1-based)
    u64 o = off[r - 1];
    u64 n = (u64)lin[r - 1] + lout[r - 1];
    return std::vector<u32>(tokens + o, tokens + o + n);
  }

  // total bytes by a full walk
  u64 total_bytes() {
    std::vector<Node*> all;
    collect(&root, all);
    u64 t = 0;
    for (Node* x : all) t += node_bytes(x->edge.size(), x->has_ssm, model);
    return t;
  }
  u64 count_nodes() {
    std::vector<Node*> all;
    collect(&root, all);
    return all.size();
  }

  void fail(const char* what) { throw std::runtime_error(what); }

  // ---- One request: SURVEY.md §8(c) c.2 steps 1-9 ----
  void step(u32 r, u32* hit_out, u64* flops_out, u32* bypass_out) {
    if (r < 1 || r > n_req) fail("request index out of range");
    if (block) return vstep(r, hit_out, flops_out, bypass_out);
    const std::vector<u32> S = seq(r);
    const u64 n = S.size();
    const u64 L_in = lin[r - 1];
    if (L_in == 0) fail("input_len == 0 [c.3 #21]");

    // Step 1: walk.
    std::vector<Node*> path;  // fully matched nodes, then the partially matched one
    Node* v = &root;
    u64 pos = 0, m = 0;
    Node* partial = nullptr;  // node in which the walk stopped mid-edge
    Node* hit = nullptr;
    u64 reuse = 0;
    for (;;) {
      if (pos == n) { m = n; break; }
      auto it = v->children.find(S[pos]);
      if (it == v->children.end()) { m = pos; break; }
      Node* c = it->second;
      u64 k = 0;
      while (k < c->edge.size() && pos + k < n && c->edge[k] == S[pos + k]) k++;
      path.push_back(c);
      if (k == c->edge.size()) {
        v = c;
        pos += k;
        // hit candidate: holds an SSM state and depth <= L_in [c.3 #6, #7]
        if (c->has_ssm && depth_of(c) <= L_in) { hit = c; reuse = depth_of(c); }
      } else {
        m = pos + k;
        partial = c;
        break;
      }
    }
    ctr_compared += std::min(m + 1, n);
    ctr_visited += path.size() + 1;

    // Step 2: hit.  Pure Transformer (n_ssm = 0): KVs can be sliced mid-edge.
    if (model.n_ssm == 0) {
      reuse = std::min(m, L_in);
      hit = nullptr;
      for (Node* x : path)
        if (depth_of(x) - x->edge.size() < reuse) hit = x;  // node containing token reuse-1
    }

    // Step 3: speculative insertion of the input (fig:spec_insertion) [c.3 #8, #9].
    const u64 m_in = std::min(m, L_in);
    u64 q = 0;                 // branch position found by the dry-run insertion, 0 = none
    if (m_in > 0) {
      for (Node* x : path) {
        u64 de = depth_of(x), ds = de - x->edge.size();
        if (x != partial && de == m_in) {
          if (!x->has_ssm) q = m_in;
          break;
        }
        if (ds < m_in && m_in < de) { q = m_in; break; }
      }
    }
    // Chunked state passing (NEXT-3): the prefill checkpoint moves down to
    // the chunk boundary at or below q; skipped if that is 0 or not beyond the hit.
    u64 p = q;
    if (q && chunk) {
      p = (q / chunk) * chunk;
      if (p == 0 || p <= reuse) p = 0;
    }
    Node* p_split = nullptr;   // node whose edge strictly contains p
    Node* p_gain = nullptr;    // existing node ending at p that lacks SSM
    if (p) {
      for (Node* x : path) {
        u64 de = depth_of(x), ds = de - x->edge.size();
        if (x != partial && de == p) {
          if (!x->has_ssm) p_gain = x;
          else p = 0;  // the state already exists
          break;
        }
        if (ds < p && p < de) { p_split = x; break; }
      }
    }

    // Step 4: plan -- at most two checkpoints {p, n}.
    struct Split { u64 pos; bool stateful; };
    std::vector<Split> splits;
    if (p_split) splits.push_back({p, true});
    if (partial && m < n && m != p) splits.push_back({m, false});   // output-region branch [c.3 #10]
    if (partial && m == n && n != p) splits.push_back({n, true});    // sequence ends inside an edge
    std::sort(splits.begin(), splits.end(), [](const Split& a, const Split& b) { return a.pos < b.pos; });
    const bool leaf = m < n;
    Node* n_gain = nullptr;  // existing boundary node at n lacking SSM
    if (!partial && m == n && !v->has_ssm && n != p) n_gain = v;
    u64 n_ckpt_new = 0;
    if (p) n_ckpt_new++;
    if (n != p) {
      if (leaf) n_ckpt_new++;
      else if (partial) n_ckpt_new++;
      else if (n_gain) n_ckpt_new++;
    }
    const u64 ssmb = node_bytes(0, true, model);   // SSM+conv bytes of one checkpoint
    const u64 kvt = node_bytes(1, false, model);   // KV bytes per token
    const u64 d_bytes = kvt * (n - m) + ssmb * n_ckpt_new;
    const u64 d_nodes = splits.size() + (leaf ? 1 : 0);

    // Step 5: pin P; touch only the hit node [c.3 #5].
    if (hit) { hit->t_last = (u32)r; ctr_written++; }

    // Step 6: admission precheck [c.3 #12].
    u64 pinned_bytes = 0;
    for (Node* x : path) pinned_bytes += node_bytes(x->edge.size(), x->has_ssm, model);
    bool bypass = (u128)pinned_bytes + d_bytes > cap_bytes ||
                  (cap_nodes && path.size() + d_nodes > cap_nodes);

    if (!bypass) {
      // Step 7: evict the argmin utility until the request fits.
      for (;;) {
        u64 total = total_bytes();
        if (total != total_incremental) fail("byte conservation violated");
        u64 cnt = count_nodes();
        if (!((u128)total + d_bytes > cap_bytes || (cap_nodes && cnt + d_nodes > cap_nodes))) break;
        evict_one(r, path);
      }
      // Step 8: insert.
      for (const Split& s : splits) split_at(S, s.pos, s.stateful, r);
      if (p_gain) { p_gain->has_ssm = true; p_gain->t_last = (u32)r; ctr_written++; }
      if (n_gain) { n_gain->has_ssm = true; n_gain->t_last = (u32)r; ctr_written++; }
      if (leaf) {
        Node* at = node_at_boundary(S, m);
        Node* x = new Node();
        x->id = next_id++;
        x->parent = at;
        x->edge.assign(S.begin() + m, S.end());
        x->has_ssm = true;
        x->t_last = (u32)r;
        x->ref_off = off[r - 1];
        at->children[x->edge[0]] = x;
        ctr_written++;
      } else {
        // final node at n: created by a split, or existing -> timestamp [c.3 #5]
        Node* fin = node_at_boundary(S, n);
        fin->t_last = (u32)r;
        if (!partial && !n_gain && fin != p_gain) ctr_written++;  // timestamp-only write
      }
      total_incremental += d_bytes;
      if (total_bytes() != total_incremental) fail("byte conservation violated after insert");
      if (total_incremental > cap_bytes) fail("capacity exceeded");
      if (cap_nodes && count_nodes() > cap_nodes) fail("node capacity exceeded");
    }

    // Step 9: outputs.
    if (reuse > L_in) fail("hit exceeds input length");
    *hit_out = (u32)reuse;
    *flops_out = prefill_flops(reuse, model);
    *bypass_out = bypass ? 1u : 0u;
  }

  // ---- Lookup of request r (steps 1-4 of c.2, read-only) ----
  void lookup(u32 r, orc_lookup* out) {
    if (r < 1 || r > n_req) fail("request index out of range");
    if (block) fail("lookup is defined for Marconi variants (block_size = 0)");
    const std::vector<u32> S = seq(r);
    const u64 n = S.size();
    const u64 L_in = lin[r - 1];
    if (L_in == 0) fail("input_len == 0 [c.3 #21]");
    // Step 1: walk
    std::vector<Node*> path;
    Node* v = &root;
    u64 pos = 0, m = 0;
    Node* partial = nullptr;
    Node* hit = nullptr;
    u64 reuse = 0;
    for (;;) {
      if (pos == n) { m = n; break; }
      auto it = v->children.find(S[pos]);
      if (it == v->children.end()) { m = pos; break; }
      Node* c = it->second;
      u64 k = 0;
      while (k < c->edge.size() && pos + k < n && c->edge[k] == S[pos + k]) k++;
      path.push_back(c);
      if (k == c->edge.size()) {
        v = c;
        pos += k;
        if (c->has_ssm && depth_of(c) <= L_in) { hit = c; reuse = depth_of(c); }
      } else {
        m = pos + k;
        partial = c;
        break;
      }
    }
    // Step 2: hit (n_ssm = 0: KVs sliced mid-edge)
    if (model.n_ssm == 0) {
      reuse = std::min(m, L_in);
      hit = nullptr;
      for (Node* x : path)
        if (depth_of(x) - x->edge.size() < reuse) hit = x;
    }
    // Step 3: speculative insertion [c.3 #8, #9], chunked
    const u64 m_in = std::min(m, L_in);
    u64 q = 0;
    if (m_in > 0) {
      for (Node* x : path) {
        u64 de = depth_of(x), ds = de - x->edge.size();
        if (x != partial && de == m_in) {
          if (!x->has_ssm) q = m_in;
          break;
        }
        if (ds < m_in && m_in < de) { q = m_in; break; }
      }
    }
    u64 p = q;
    if (q && chunk) {
      p = (q / chunk) * chunk;
      if (p == 0 || p <= reuse) p = 0;
    }
    bool p_split = false;
    if (p) {
      for (Node* x : path) {
        u64 de = depth_of(x), ds = de - x->edge.size();
        if (x != partial && de == p) {
          if (x->has_ssm) p = 0;  // the state already exists
          break;
        }
        if (ds < p && p < de) { p_split = true; break; }
      }
    }
    // Step 4: plan
    u64 n_splits = (p_split ? 1 : 0) + ((partial && m < n && m != p) ? 1 : 0) + ((partial && m == n && n != p) ? 1 : 0);
    const bool leaf = m < n;
    const bool n_gain = !partial && m == n && !v->has_ssm && n != p;
    u64 n_ckpt_new = (p ? 1 : 0) + ((n != p && (leaf || partial || n_gain)) ? 1 : 0);
    const u64 ssmb = node_bytes(0, true, model), kvt = node_bytes(1, false, model);
    Node* div = partial ? partial : v;
    out->reuse = (u32)reuse;
    out->m = (u32)m;
    out->p = (u32)p;
    out->hit_id = hit ? hit->id : 0;
    out->div_id = div->id;
    out->div_off = (u32)(m - (div == &root ? 0 : depth_of(div) - div->edge.size()));
    out->path_len = (u32)path.size();
    out->d_nodes = (u32)(n_splits + (leaf ? 1 : 0));
    out->d_bytes = kvt * (n - m) + ssmb * n_ckpt_new;
  }

  // Node whose edge ends exactly at depth x along S (x must be a boundary).
  Node* node_at_boundary(const std::vector<u32>& S, u64 x) {
    Node* v = &root;
    u64 pos = 0;
    while (pos < x) {
      auto it = v->children.find(S[pos]);
      if (it == v->children.end()) fail("boundary walk fell off the tree");
      v = it->second;
      pos += v->edge.size();
    }
    if (pos != x) fail("not a node boundary");
    return v;
  }

  // Split the edge containing depth x (strictly inside) along S.  The new upper
  // node takes next_id; the lower part keeps its id [c.3 #4].
  void split_at(const std::vector<u32>& S, u64 x, bool stateful, u32 r) {
    Node* v = &root;
    u64 pos = 0;
    for (;;) {
      auto it = v->children.find(S[pos]);
      if (it == v->children.end()) fail("split walk fell off the tree");
      Node* c = it->second;
      if (pos + c->edge.size() <= x) {
        v = c;
        pos += c->edge.size();
        if (pos == x) fail("split position is already a boundary");
        continue;
      }
      u64 j = x - pos;
      Node* up = new Node();
      up->id = next_id++;
      up->parent = v;
      up->edge.assign(c->edge.begin(), c->edge.begin() + j);
      up->has_ssm = stateful;
      up->t_last = r;
      up->ref_off = c->ref_off;
      c->edge.erase(c->edge.begin(), c->edge.begin() + j);
      c->parent = up;
      up->children[c->edge[0]] = c;
      v->children[up->edge[0]] = up;
      ctr_written += 2;
      return;
    }
  }

  // One eviction step, everything recomputed.
  void evict_one(u32 r, const std::vector<Node*>& pinned) {
    std::vector<Node*> all;
    collect(&root, all);
    if (all.empty()) fail("nothing to evict");
    ctr_scanned += all.size();
    // normalisation bounds over ALL non-root nodes [c.3 #1]
    u32 tmin = all[0]->t_last, tmax = all[0]->t_last;
    std::vector<double> eff(all.size());
    for (size_t i = 0; i < all.size(); i++) {
      Node* x = all[i];
      tmin = std::min(tmin, x->t_last);
      tmax = std::max(tmax, x->t_last);
      u64 de = depth_of(x);
      eff[i] = flop_efficiency(de - x->edge.size(), de, x->has_ssm, model);
    }
    double emin = eff[0], emax = eff[0];
    for (double e : eff) { emin = std::min(emin, e); emax = std::max(emax, e); }

    Node* best = nullptr;
    double best_u = 0;
    for (size_t i = 0; i < all.size(); i++) {
      Node* x = all[i];
      if (std::find(pinned.begin(), pinned.end(), x) != pinned.end()) continue;
      if (x->children.size() > 1) continue;  // candidates: <= 1 child
      // [c.3 #2] degenerate range -> 0.5; [c.3 #15] each op rounded, no FMA
      double rec = (tmax == tmin) ? 0.5 : (double)(x->t_last - tmin) / (double)(tmax - tmin);
      double effn = (emax == emin) ? 0.5 : (eff[i] - emin) / (emax - emin);
      double u = rec + alpha * effn;  // Eq. 2
      // victim = lexicographic min of (u, t_last, id) [c.3 #4]
      if (!best || u < best_u || (u == best_u && (x->t_last < best->t_last ||
                                                  (x->t_last == best->t_last && x->id < best->id)))) {
        best = x;
        best_u = u;
      }
    }
    if (!best) fail("no eviction candidate");
    Node* par = best->parent;
    orc_evict rec{r, best->id, 0, (u32)all.size(), best_u};
    if (best->children.empty()) {
      // leaf: free its KVs and state
      total_incremental -= node_bytes(best->edge.size(), best->has_ssm, model);
      par->children.erase(best->edge[0]);
      ctr_written += 1;
    } else {
      // one child: release the SSM state, the child absorbs the KVs
      Node* c = best->children.begin()->second;
      total_incremental -= best->has_ssm ? node_bytes(0, true, model) : 0;
      std::vector<u32> e = best->edge;
      e.insert(e.end(), c->edge.begin(), c->edge.end());
      c->edge = e;
      c->parent = par;
      par->children.erase(best->edge[0]);
      par->children[c->edge[0]] = c;
      rec.kind = 1;
      ctr_written += 2;
    }
    delete best;
    log.push_back(rec);
  }

  // ---- vLLM+ baseline (readings V1-V8) ----
  // "fine-grained checkpointing and caches a state for every token block" with
  // block size x = 32; each block holds the KVs of its x tokens and the
  // SSM states that represent all prior tokens, vLLM's caching policy
  // (LRU) extended to hybrid models.  Step by step:
  //   1. walk the block trie from the root, block k = S[kx, (k+1)x) matched by its
  //      whole content; only full blocks exist [V1, V2];
  //   2. hit = the deepest matched block end <= L_in (every block carries a state;
  //      all-or-nothing) [V4];
  //   3. every matched block is touched (t_last = r) [V5];
  //   4. admission of the missing full blocks; bypass when the matched path plus the
  //      new blocks exceed the capacity [V7];
  //   5. evict LRU leaf blocks (min (t_last, id)) not on the matched path until the
  //      new blocks fit [V6];
  //   6. insert the new blocks, t_last = r.
  // A block charges node_bytes(x, state) = x tokens of KVs + one set of SSM/conv
  // states (Appendix A) [V3].
  void vstep(u32 r, u32* hit_out, u64* flops_out, u32* bypass_out) {
    const std::vector<u32> S = seq(r);
    const u64 n = S.size();
    const u64 L_in = lin[r - 1];
    if (L_in == 0) fail("input_len == 0 [c.3 #21]");
    const u64 x = block;
    const u64 nb = n / x;  // full blocks of the sequence [V2]
    // Step 1: walk, block content compared token by token.
    std::vector<Node*> path;
    Node* v = &root;
    for (u64 k = 0; k < nb; k++) {
      std::vector<u32> blk(S.begin() + k * x, S.begin() + (k + 1) * x);
      auto it = v->bkids.find(blk);
      if (it == v->bkids.end()) break;
      v = it->second;
      path.push_back(v);
    }
    const u64 mb = path.size();
    ctr_compared += mb * x;
    ctr_visited += mb + 1;
    // Step 2: hit [V4].
    const u64 reuse = std::min<u64>(mb, L_in / x) * x;
    // Step 3: touch the matched path [V5].
    for (Node* c : path) c->t_last = r;
    ctr_written += mb;
    // Step 4: admission [V7].
    const u64 bb = node_bytes(x, true, model);
    const u64 n_new = nb - mb;
    const u64 d_bytes = bb * n_new;
    const u64 pinned_bytes = bb * mb;
    const bool bypass = (pinned_bytes + d_bytes > cap_bytes) || (cap_nodes && mb + n_new > cap_nodes);
    if (!bypass) {
      // Step 5: LRU leaf eviction [V6].
      while (total_incremental + d_bytes > cap_bytes || (cap_nodes && count_nodes() + n_new > cap_nodes))
        vevict_one(r, path);
      // Step 6: insert the missing blocks under the deepest matched one.
      for (u64 k = mb; k < nb; k++) {
        Node* c = new Node();
        c->id = next_id++;
        c->parent = v;
        c->edge.assign(S.begin() + k * x, S.begin() + (k + 1) * x);
        c->has_ssm = true;
        c->t_last = r;
        c->ref_off = off[r - 1];
        v->bkids[c->edge] = c;
        v = c;
        ctr_written += 1;
      }
      total_incremental += d_bytes;
      if (total_bytes() != total_incremental) fail("byte accounting mismatch");
      if (total_incremental > cap_bytes) fail("capacity exceeded");
      if (cap_nodes && count_nodes() > cap_nodes) fail("node capacity exceeded");
    }
    if (reuse > L_in) fail("hit exceeds input length");
    *hit_out = (u32)reuse;
    *flops_out = prefill_flops(reuse, model);
    *bypass_out = bypass ? 1u : 0u;
  }

  // One LRU eviction among the leaf blocks off the pinned path [V6]; the logged
  // utility is Eq. 2 at alpha = 0 (the recency term) for the log format.
  void vevict_one(u32 r, const std::vector<Node*>& pinned) {
    std::vector<Node*> all;
    collect(&root, all);
    if (all.empty()) fail("nothing to evict");
    ctr_scanned += all.size();
    u32 tmin = all[0]->t_last, tmax = all[0]->t_last;
    for (Node* x : all) { tmin = std::min(tmin, x->t_last); tmax = std::max(tmax, x->t_last); }
    Node* best = nullptr;
    for (Node* x : all) {
      if (!x->bkids.empty()) continue;  // only leaf blocks: an inner block's descendants need it
      if (std::find(pinned.begin(), pinned.end(), x) != pinned.end()) continue;
      if (!best || x->t_last < best->t_last || (x->t_last == best->t_last && x->id < best->id)) best = x;
    }
    if (!best) fail("no eviction candidate");
    const double u = (tmax == tmin) ? 0.5 : (double)(best->t_last - tmin) / (double)(tmax - tmin);
    log.push_back(orc_evict{r, best->id, 0, (u32)all.size(), u});
    total_incremental -= node_bytes(best->edge.size(), best->has_ssm, model);
    best->parent->bkids.erase(best->edge);
    delete best;
    ctr_written += 1;
  }

  // ---- snapshots (canonical dump) ----
  std::vector<orc_node> dump() {
    std::vector<Node*> all;
    collect(&root, all);
    std::vector<orc_node> out;
    for (Node* x : all) {
      u64 de = depth_of(x);
      orc_node o;
      o.id = x->id;
      o.parent_id = x->parent->id;
      o.ref_off = x->ref_off;
      o.d_start = (u32)(de - x->edge.size());
      o.d_end = (u32)de;
      o.t_last = x->t_last;
      o.has_ssm = x->has_ssm ? 1 : 0;
      out.push_back(o);
    }
    std::sort(out.begin(), out.end(), [](const orc_node& a, const orc_node& b) { return a.id < b.id; });
    return out;
  }

  void load(const orc_node* nodes, u32 n, u32 nid) {
    for (auto& kv : root.children) free_subtree(kv.second);
    for (auto& kv : root.bkids) free_subtree(kv.second);
    root.children.clear();
    root.bkids.clear();
    std::map<u32, Node*> by_id;
    by_id[0] = &root;
    for (u32 i = 0; i < n; i++) {
      const orc_node& o = nodes[i];
      if (o.id == 0 || by_id.count(o.id)) fail("bad snapshot id");
      if (o.d_end <= o.d_start || o.ref_off + o.d_end > n_tokens) fail("bad snapshot range");
      Node* x = new Node();
      x->id = o.id;
      x->edge.assign(tokens + o.ref_off + o.d_start, tokens + o.ref_off + o.d_end);
      x->has_ssm = o.has_ssm != 0;
      x->t_last = o.t_last;
      x->ref_off = o.ref_off;
      by_id[o.id] = x;
    }
    for (u32 i = 0; i < n; i++) {
      auto it = by_id.find(nodes[i].parent_id);
      if (it == by_id.end()) fail("snapshot parent missing");
      Node* x = by_id[nodes[i].id];
      x->parent = it->second;
      if (block) {
        if (x->edge.size() != block || nodes[i].d_start % block) fail("snapshot record is not one block");
        if (it->second->bkids.count(x->edge)) fail("snapshot block trie property violated");
        it->second->bkids[x->edge] = x;
        continue;
      }
      if (it->second->children.count(x->edge[0])) fail("snapshot radix property violated");
      it->second->children[x->edge[0]] = x;
    }
    for (u32 i = 0; i < n; i++) {
      Node* x = by_id[nodes[i].id];
      if (depth_of(x) != nodes[i].d_end) fail("snapshot depth mismatch");
    }
    next_id = nid;
    total_incremental = total_bytes();
  }
};

// ---------------------------------------------------------------------------
// C ABI for the Python test wrapper (oracle/__init__.py).
// All functions return 0 on success, -1 on error (message via orc_last_error).
// ---------------------------------------------------------------------------
#define ORC_TRY(body)            \
  try {                          \
    body;                        \
    return 0;                    \
  } catch (const std::exception& e) { \
    g_err = e.what();            \
    return -1;                   \
  }

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

int orc_prefill_flops(const orc_model* m, u64 L, u64* out) { ORC_TRY(*out = prefill_flops(L, *m)) }
int orc_layer_terms(const orc_model* m, u64 L, u64* out6) {
  ORC_TRY(out6[0] = attention_flops(L, *m); out6[1] = mlp_flops(L, *m); out6[2] = ssm_flops(L, *m);
          out6[3] = kv_bytes_layer(L, *m); out6[4] = ssm_state_bytes_layer(*m);
          out6[5] = conv_state_bytes_layer(*m))
}
int orc_node_cost(const orc_model* m, u64 d_start, u64 d_end, u32 has_ssm, u64* saved, u64* bytes,
                  double* eff) {
  ORC_TRY(if (d_end < d_start) throw std::invalid_argument("d_end < d_start");
          *saved = prefill_flops(d_end, *m) - prefill_flops(d_start, *m);
          *bytes = node_bytes(d_end - d_start, has_ssm != 0, *m);
          *eff = flop_efficiency(d_start, d_end, has_ssm != 0, *m))
}

// Eviction scoring on an explicit node table:
// bounds over ALL rows, utility for candidate rows, lexicographic (u, t, id) min.
// *best = row index or 0xFFFFFFFF when no row is a candidate.
int orc_score_argmin(u32 n, const u32* t, const uint8_t* cand, const u32* id, const double* eff, double alpha,
                     u32* best, double* u_out) {
  *best = 0xFFFFFFFFu;
  *u_out = 0;
  if (n == 0) return 0;
  u32 tmin = t[0], tmax = t[0];
  double emin = eff[0], emax = eff[0];
  for (u32 i = 0; i < n; i++) {
    tmin = std::min(tmin, t[i]);
    tmax = std::max(tmax, t[i]);
    emin = std::min(emin, eff[i]);
    emax = std::max(emax, eff[i]);
  }
  double bu = 0;
  for (u32 i = 0; i < n; i++) {
    if (!cand[i]) continue;
    double rec = (tmax == tmin) ? 0.5 : (double)(t[i] - tmin) / (double)(tmax - tmin);
    double effn = (emax == emin) ? 0.5 : (eff[i] - emin) / (emax - emin);
    double u = rec + alpha * effn;
    if (*best == 0xFFFFFFFFu || u < bu ||
        (u == bu && (t[i] < t[*best] || (t[i] == t[*best] && id[i] < id[*best])))) {
      *best = i;
      bu = u;
    }
  }
  *u_out = bu;
  return 0;
}

void* orc_create(const orc_model* m, u64 cap_bytes, u32 cap_nodes, double alpha, const u32* tokens,
                 u64 n_tokens, const u64* off, const u32* lin, const u32* lout, u32 n_req) {
  try {
    if (!(alpha >= 0)) throw std::invalid_argument("alpha must be >= 0 (SPEC:308)");
    if (m->bytes_per_param != 1 && m->bytes_per_param != 2 && m->bytes_per_param != 4)
      throw std::invalid_argument("bytes_per_param must be 1, 2 or 4");
    if (m->n_attn == 0) throw std::invalid_argument("n_attn = 0 would allow zero-byte nodes");
    for (u32 i = 0; i < n_req; i++)
      if (lin[i] == 0 || off[i] + (u64)lin[i] + lout[i] > n_tokens)
        throw std::invalid_argument("bad request");
    Oracle* o = new Oracle();
    o->model = *m;
    o->cap_bytes = cap_bytes;
    o->cap_nodes = cap_nodes;
    o->alpha = alpha;
    o->tokens = tokens;
    o->n_tokens = n_tokens;
    o->off = off;
    o->lin = lin;
    o->lout = lout;
    o->n_req = n_req;
    return o;
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}
void orc_destroy(void* h) { delete (Oracle*)h; }
int orc_set_chunk(void* h, u32 chunk) { ORC_TRY(((Oracle*)h)->chunk = chunk) }
// vLLM+ baseline with token blocks of `block` (0 = Marconi); set before any step/load.
int orc_set_block(void* h, u32 block) { ORC_TRY(((Oracle*)h)->block = block) }
int orc_set_alpha(void* h, double a) {
  ORC_TRY(if (!(a >= 0)) throw std::invalid_argument("alpha < 0"); ((Oracle*)h)->alpha = a)
}
int orc_load(void* h, const orc_node* nodes, u32 n, u32 next_id) {
  ORC_TRY(((Oracle*)h)->load(nodes, n, next_id))
}
int orc_step(void* h, u32 r, u32* hit, u64* flops, u32* bypass) {
  ORC_TRY(((Oracle*)h)->step(r, hit, flops, bypass))
}
// Replay requests first..first+n-1; optional snapshot after every `every` requests
// counted from request index 0 (i.e. after requests every, 2*every, ...).
int orc_run(void* h, u32 first, u32 n, u32* hit, u64* flops, u32* bypass) {
  ORC_TRY(Oracle* o = (Oracle*)h;
          for (u32 i = 0; i < n; i++) o->step(first + i, hit + i, flops + i, bypass + i))
}
int orc_dump(void* h, orc_node* out, u64 cap, u64* n_out, u32* next_id) {
  ORC_TRY(Oracle* o = (Oracle*)h; std::vector<orc_node> d = o->dump(); *n_out = d.size();
          *next_id = o->next_id;
          if (out) {
            if (d.size() > cap) throw std::length_error("dump buffer too small");
            std::copy(d.begin(), d.end(), out);
          })
}
int orc_log(void* h, orc_evict* out, u64 cap, u64* n_out) {
  ORC_TRY(Oracle* o = (Oracle*)h; *n_out = o->log.size();
          if (out) {
            if (o->log.size() > cap) throw std::length_error("log buffer too small");
            std::copy(o->log.begin(), o->log.end(), out);
          })
}
int orc_lookup_req(void* h, u32 r, orc_lookup* out) { ORC_TRY(((Oracle*)h)->lookup(r, out)) }
int orc_counters(void* h, u64* out4) {
  ORC_TRY(Oracle* o = (Oracle*)h; out4[0] = o->ctr_compared; out4[1] = o->ctr_visited;
          out4[2] = o->ctr_scanned; out4[3] = o->ctr_written)
}
int orc_total(void* h, u64* total, u64* count) {
  ORC_TRY(Oracle* o = (Oracle*)h; *total = o->total_bytes(); *count = o->count_nodes())
}

// Independent chains across host threads (the paper's "grid search is
// parallelized across CPU cores").  Chain c replays requests
// first[c] .. first[c]+n[c]-1 at alpha[c] from snapshot
// snap_nodes[snap_off[s] .. snap_off[s+1]) with s = snap_idx[c]; outputs are
// written at hit[out_off[c] + i].  hit_sum[c] = sum of hits.
int orc_run_chains(const orc_model* models, const u64* cap_bytes, const u32* cap_nodes, const u32* chunks,
                   const u32* blocks,
                   const u32* variant, const double* alpha, const u32* first, const u32* n,
                   const u32* snap_idx, const orc_node* snap_nodes, const u64* snap_off,
                   const u32* snap_next_id, u32 n_chains, const u32* tokens, u64 n_tokens,
                   const u64* off, const u32* lin, const u32* lout, u32 n_req, const u64* out_off,
                   u32* hit, u64* flops, u32* bypass, u64* hit_sum, u64* counters4, u32 n_threads) {
  std::atomic<u32> next{0};
  std::atomic<int> err{0};
  std::string err_msg;
  std::vector<std::thread> pool;
  if (n_threads == 0) n_threads = 1;
  for (u32 t = 0; t < n_threads; t++) {
    pool.emplace_back([&]() {
      for (;;) {
        u32 c = next.fetch_add(1);
        if (c >= n_chains || err.load()) return;
        try {
          u32 v = variant[c];
          Oracle* o = (Oracle*)orc_create(&models[v], cap_bytes[v], cap_nodes[v], alpha[c], tokens,
                                          n_tokens, off, lin, lout, n_req);
          if (!o) throw std::runtime_error(g_err);
          o->chunk = chunks ? chunks[v] : 0;
          o->block = blocks ? blocks[v] : 0;
          u32 s = snap_idx[c];
          o->load(snap_nodes + snap_off[s], (u32)(snap_off[s + 1] - snap_off[s]), snap_next_id[s]);
          u64 sum = 0;
          for (u32 i = 0; i < n[c]; i++) {
            u64 k = out_off[c] + i;
            o->step(first[c] + i, hit + k, flops + k, bypass + k);
            sum += hit[k];
          }
          hit_sum[c] = sum;
          if (counters4) {
            counters4[4 * c + 0] = o->ctr_compared;
            counters4[4 * c + 1] = o->ctr_visited;
            counters4[4 * c + 2] = o->ctr_scanned;
            counters4[4 * c + 3] = o->ctr_written;
          }
          delete o;
        } catch (const std::exception& e) {
          if (!err.exchange(1)) err_msg = e.what();
          return;
        }
      }
    });
  }
  for (auto& th : pool) th.join();
  if (err.load()) {
    g_err = err_msg;
    return -1;
  }
  return 0;
}

}  // extern "C"
