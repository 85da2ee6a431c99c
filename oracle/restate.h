/* TEST INFRASTRUCTURE ONLY — plain-C restatement of the reference's
 * token-tree verification path, used by tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg as the CHECKER. The product never links it.
 *
 * Every function cites the reference file:line it restates (paths relative
 * to /root/reference). Pinned against the reference itself: the fixtures in tests/golden
 * are produced by oracle/gen_golden.py from oracle/_ref (the unmodified
 * reference compiled from its own sources) and tests/test_oracle_golden.py
 * checks this restatement against them.
 *
 * Status codes: 0 = ok, otherwise 1 + spectree::Errc
 * (proj/include/spectree/error.hpp:8-25). */
#ifndef SPECTREE_ORACLE_RESTATE_H
#define SPECTREE_ORACLE_RESTATE_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* TokenTree::merge_sequences — proj/src/token_tree.cpp:42-102. */
int or_merge(const int32_t* flat, const int32_t* lens, int nseq, int max_nodes, int32_t* tok,
             int32_t* parent, int32_t* depth, int cap, int* n_out);

/* verify — proj/src/token_tree.cpp:153-175. Also returns the accepted node
 * ids (root first, one per matched node): ids[0..*n_verified-1). */
int or_verify(const int32_t* tok, const int32_t* parent, int n, const int32_t* outputs,
              int n_outputs, int32_t* verified, int32_t* ids, int* n_verified);

/* argmax_token — proj/src/transformer.cpp:116-122 (strict '>', lowest id wins). */
int or_argmax_f64(const double* x, int n);
int or_argmax_f32(const float* x, int n);

/* Ancestor bitmask: mask[u] = mask[parent(u)] | bit(u) in preorder
 * (proj/src/token_tree.cpp:130-139 gives the same node set). W = words/node. */
void or_ancestor_masks(const int32_t* parent, int n, int W, uint64_t* mask);

/* UniformStream — proj/include/spectree/rng.hpp:13-44. */
void or_uniform_stream(uint64_t seed, int64_t n, double lo, double hi, double* out);

/* Masked tree attention (the arithmetic of proj/src/transformer.cpp:270-299,
 * restated for one masked pass over all tree rows). Layout = the device layout
 * (DESIGN.md §3):
 *   q     [B][T][H][D]
 *   kc,vc [B][Hkv][Lmax][D]   committed rows [0,P[b]) + tree rows [P[b],P[b]+n[b])
 *   mask  [B][T][W] u64       bit v of mask[b][u] -> tree row v visible to node u
 *   o     [B][T][H][D]        rows u >= n[b] are left untouched
 *   lse   [B][H][T] (optional, natural log)
 * Accumulation in f64. */
void or_tree_attention(const double* q, const double* kc, const double* vc, const uint64_t* mask,
                       const int32_t* P, const int32_t* n_nodes, int B, int T, int H, int Hkv,
                       int D, int Lmax, int W, double scale, double* o, double* lse);

/* Greedy verify for one request: per-node argmax over fp32 logits [n][V]
 * (transformer.cpp:116-122) then the Alg.-2 walk (token_tree.cpp:153-175). */
int or_greedy_verify(const float* logits, int V, const int32_t* tok, const int32_t* parent, int n,
                     int32_t* out_tokens, int32_t* verified, int32_t* ids, int* n_verified);

/* Multi-step speculative sampling (MSS) for one request — NOT in the
 * reference: the contract of SURVEY.md Appendix B, defined
 * in DESIGN.md §5 (parity unpinned against the reference; this oracle is the
 * pin for K4). logits [n][V] f32; q [n][V] f32 = draft distribution of the
 * SSM that proposed node v (row v, root row unused); uniforms consumed in
 * order. Reductions use the fixed blocked order of DESIGN.md §5. */
int or_mss_verify(const float* logits, const float* q, int V, const int32_t* tok,
                  const int32_t* parent, int n, float temperature, const float* uniforms,
                  int n_uniforms, int32_t* verified, int32_t* ids, int* n_verified);

#ifdef __cplusplus
}
#endif
#endif
