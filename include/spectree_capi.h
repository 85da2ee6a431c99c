/* spectree_capi.h — the C-ABI of the B200-native token-tree verification path.
 *
 * This is the drop-in boundary: plain pointers and sizes,
 * no torch or C++ types. The C++ headers in include/spectree/ (same
 * declarations as the reference's proj/include/spectree headers) sit on top of
 * it, and so do the Python ctypes bindings (paper_2305_09781_b200/_capi.py).
 *
 * Conventions
 *   - Status: 0 = ok, otherwise 1 + spectree::Errc
 *     (reference proj/include/spectree/error.hpp:8-25); st_last_error_message()
 *     returns a thread-local description of the last failure.
 *   - All tensor pointers are DEVICE pointers, caller-owned; no allocation
 *     happens inside a launch (workspaces are caller-provided). Launches are
 *     ordered on the given cudaStream_t (passed as void*; NULL = legacy stream).
 *   - No CPU fallback: on a machine without a CUDA device every compute entry
 *     point fails with ST_ERR_NO_DEVICE.
 *   - Layouts:
 *       q, o        [B][T][H][D]          tree-node queries / outputs
 *       k/v cache   [B][Hkv][Lmax][D]     per layer; rows [0,P[b]) committed,
 *                                         rows [P[b], P[b]+n[b]) = tree scratch
 *                                         indexed by preorder node id
 *       mask        [B][T][W] uint64      bit v of mask[b][u]: tree row v is an
 *                                         ancestor-or-self of node u
 *       logits      [B][T][V] float32
 *       parent,tok  [B][T] int32          preorder (parent[u] < u, root = 0)
 */
#ifndef SPECTREE_CAPI_H
#define SPECTREE_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define ST_ABI_VERSION 5

typedef int st_status;

/* 1 + spectree::Errc (reference error.hpp:8-25), plus ABI-only codes >= 100. */
enum {
    ST_OK = 0,
    ST_ERR_EMPTY_INPUT = 1,
    ST_ERR_ROOT_MISMATCH = 2,
    ST_ERR_UNKNOWN_NODE = 3,
    ST_ERR_MISSING_OUTPUT = 4,
    ST_ERR_TREE_TOO_LARGE = 5,
    ST_ERR_TREE_TOO_DEEP = 6,
    ST_ERR_SHAPE_MISMATCH = 7,
    ST_ERR_PROMPT_TOO_LONG = 8,
    ST_ERR_CACHE_GAP = 9,
    ST_ERR_CHAIN_NOT_LINKED = 10,
    ST_ERR_EMPTY_CONTEXT = 11,
    ST_ERR_INVALID_ARGUMENT = 16,
    ST_ERR_NO_DEVICE = 100,
    ST_ERR_CUDA = 101,
    ST_ERR_UNSUPPORTED = 102,
};

typedef enum { ST_F16 = 0, ST_BF16 = 1, ST_F32 = 2, ST_F64 = 3 } st_dtype;

int st_abi_version(void);
const char* st_last_error_message(void);
/* Number of visible CUDA devices (0 on a CPU-only host; never fails). */
int st_device_count(void);

/* ------------------------------------------------------------------ K1 ---
 * Tree attention: for every (request b, head h, node u < n[b]):
 *   o[b][u][h] = softmax_{r in R(b,u)} (q[b][u][h] . k[b][h/G][r] * scale) . v[b][h/G][r]
 *   R(b,u) = [0, P[b]) U { P[b]+v : bit v of mask[b][u] }
 * Replaces the per-chain loop of reference transformer.cpp:394-446 over
 * chain_attention_step_impl's attention core (transformer.cpp:270-299) with
 * one masked pass. Masked rows contribute exactly +0 (transformer.hpp:13-16).
 * Rows u >= n[b] of o are not written. lse (optional) = natural-log
 * log-sum-exp [B][H][T] in float32. */
typedef struct {
    st_dtype dtype;           /* q/k/v/o element type */
    int B, T, H, Hkv, D;      /* T = max nodes per request (row stride of q/o/mask) */
    int W;                    /* mask words per node, >= ceil(T/64) */
    int64_t Lmax;             /* cache rows per (b, kv head) */
    const void* q;
    const void* k_cache;
    const void* v_cache;
    const uint64_t* mask;
    const int32_t* prefix_len; /* [B] committed rows P[b] (device) */
    const int32_t* n_nodes;    /* [B] tree nodes n[b] <= T (device) */
    void* o;
    float* lse;                /* optional, NULL allowed */
    double scale;              /* usually 1/sqrt(D) */
    void* workspace;           /* st_tree_attention_workspace_size() bytes, zeroed once */
    size_t workspace_bytes;
    int force_path;            /* 0 auto, 1 CUDA-core, 2 tcgen05 tensor-core */
    /* Optional: the tree nodes' own K/V rows, [B][T][Hkv][D] (the step's new
     * rows, e.g. from the QKV projection). When set, tree row v of request b
     * is read from here instead of cache row P[b]+v — K1 then needs no
     * st_kv_append before it, and st_verify_greedy_compact copies the
     * accepted rows from the same tensors into the cache. NULL: the tree rows
     * are in the cache at [P[b], P[b]+n[b]). */
    const void* k_tree;
    const void* v_tree;
    /* Optional promise (0 = off): the kernel launched right before K1 on the
     * stream writes neither prefix_len / n_nodes nor the committed cache rows
     * [0, P[b]). K1 (tcgen05 path, programmatic dependent launch) then builds
     * its schedule and starts streaming those rows while that kernel drains,
     * before griddepcontrol.wait; Q, the masks and tree rows are still read
     * after the wait. The promise is transitive: no kernel still running when
     * K1 starts may write those rows either. Programmatic launches chain, so
     * the kernel before K1 must not release its dependents (launch_dependents)
     * before its OWN griddepcontrol.wait has returned — st_build_masks_early
     * and st_tree_prepare follow this rule, which makes "previous step's
     * commit -> masks -> early_kv K1" safe while P advances every step. */
    int early_kv;
    /* Optional (0 = off; ABI 5): q, o and lse hold only q_rows rows per
     * request — tree nodes [q_node0, q_node0 + q_rows), e.g. one level of a
     * draft tree grown level by level — while the mask rows and the tree rows
     * (k_tree; required on the tcgen05 path) stay indexed by node id over T and n_nodes counts
     * every node so far. q/o row stride q_rows, lse [B][H][q_rows]. */
    int q_rows;
    int q_node0;
} st_attn_args;

size_t st_tree_attention_workspace_size(const st_attn_args* a);
st_status st_tree_attention(const st_attn_args* a, void* stream);
/* Which kernel `auto` picks for these args: 1 CUDA-core, 2 tcgen05. */
int st_tree_attention_path(const st_attn_args* a);

/* ------------------------------------------------------------------ K2 ---
 * Append: write the tree nodes' K/V rows into the cache scratch region
 *   cache[b][h][P[b] + u] = new[b][u][h]     for u < n[b]
 * (the reference writes chain rows straight into cache positions,
 * transformer.cpp:265-268). k_new/v_new: [B][T][Hkv][D]. */
st_status st_kv_append(st_dtype dtype, int B, int T, int Hkv, int D, int64_t Lmax,
                       const void* k_new, const void* v_new, const int32_t* prefix_len,
                       const int32_t* n_nodes, void* k_cache, void* v_cache, void* stream);

/* st_kv_append and st_build_masks in one launch (the two independent steps
 * that precede K1): same effects as the two calls. */
st_status st_tree_prepare(st_dtype dtype, int B, int T, int Hkv, int D, int64_t Lmax,
                          const void* k_new, const void* v_new, const int32_t* prefix_len,
                          const int32_t* n_nodes, void* k_cache, void* v_cache,
                          const int32_t* parent, int W, uint64_t* mask, void* stream);

/* Compact: keep the accepted root-to-node path, in place, for n_layers layers
 * (cache pointer of layer l = base + l * layer_stride elements):
 *   cache[b][h][P[b] + k] = cache[b][h][P[b] + ids[b][k]]   for k < n_keep[b]
 * then (if new_prefix_len != NULL) new_prefix_len[b] = P[b] + n_keep[b].
 * Replaces the post-verify re-decode of reference engine.cpp:123-129. ids is
 * [B][ids_stride], strictly increasing with ids[b][0] == 0 (the root). */
st_status st_kv_compact(st_dtype dtype, int B, int Hkv, int D, int64_t Lmax, int n_layers,
                        int64_t layer_stride, const int32_t* ids, int ids_stride,
                        const int32_t* n_keep, const int32_t* prefix_len,
                        int32_t* new_prefix_len, void* k_cache, void* v_cache, void* stream);

/* The same commit from the tree's own K/V (K1's k_tree mode: no append
 * preceded it): cache[l][b][h][P + k] = tree[l][b][ids[k]][h] for k in
 * [0, n_keep[b]); tree layer l at k_tree + l * tree_layer_stride elements,
 * [B][T][Hkv][D] each. */
st_status st_kv_commit_tree(st_dtype dtype, int B, int T, int Hkv, int D, int64_t Lmax,
                            int n_layers, int64_t layer_stride, const int32_t* ids,
                            int ids_stride, const int32_t* n_keep, const int32_t* prefix_len,
                            int32_t* new_prefix_len, const void* k_tree, const void* v_tree,
                            int64_t tree_layer_stride, void* k_cache, void* v_cache,
                            void* stream);

/* Head-sharded attention (C4): reorder an all-gathered
 * [world][B][T][Hl][D] (rank r's K1 output for heads r*Hl..r*Hl+Hl-1) into
 * [B][T][world*Hl][D]. */
st_status st_heads_gather_layout(st_dtype dtype, int world, int B, int T, int Hl, int D,
                                 const void* gathered, void* out, void* stream);

/* ------------------------------------------------------------------ K3 ---
 * Greedy verification: per-node argmax over logits (lowest id wins ties,
 * reference transformer.cpp:116-122) then the Alg.-2 walk (reference
 * token_tree.cpp:153-175). Outputs per request b:
 *   argmax[b][u]            greedy LLM output of node u            (optional)
 *   verified[b][0..len)     accepted tokens + bonus token
 *   ids[b][0..len)          accepted node ids, root first (input to st_kv_compact)
 *   len[b]
 * Optional engine step semantics (reference engine.cpp:110-121): if budget
 * != NULL, truncate to budget[b] tokens; then cut after the first `eos`
 * (eos < 0 disables). The truncated length is what st_kv_compact keeps.
 * verified/ids have row stride T+1. workspace: st_verify_workspace_size(). */
size_t st_verify_workspace_size(int B, int T);
st_status st_verify_greedy(const float* logits, int B, int T, int V, const int32_t* tokens,
                           const int32_t* parent, const int32_t* n_nodes,
                           const int32_t* budget, int32_t eos, int32_t* argmax,
                           int32_t* verified, int32_t* ids, int32_t* len, void* workspace,
                           void* stream);

/* st_verify_greedy followed by st_kv_compact of the accepted rows
 * (n_keep = len) over n_layers layers, in two launches instead of three: the
 * walk is fused into the compaction kernel (every block of a request repeats
 * the request's walk in shared memory, then moves its share of the KV heads).
 * Same outputs as the two calls; requires T <= 1024, D * sizeof(dtype) a
 * multiple of 16 and new_prefix_len (optional) not aliasing prefix_len.
 * k_tree/v_tree (optional, [B][T][Hkv][D] per layer, layer l at
 * + l * tree_layer_stride elements): take the accepted rows from the tree's
 * own K/V (the st_attn_args.k_tree mode: nothing was appended to the cache)
 *   cache[b][h][P + k] = tree[b][ids[k]][h]   for k < len[b]. */
st_status st_verify_greedy_compact(const float* logits, int B, int T, int V, const int32_t* tokens,
                                   const int32_t* parent, const int32_t* n_nodes,
                                   const int32_t* budget, int32_t eos, int32_t* argmax,
                                   int32_t* verified, int32_t* ids, int32_t* len, void* workspace,
                                   st_dtype dtype, int Hkv, int D, int64_t Lmax, int n_layers,
                                   int64_t layer_stride, const int32_t* prefix_len,
                                   int32_t* new_prefix_len, const void* k_tree,
                                   const void* v_tree, int64_t tree_layer_stride, void* k_cache,
                                   void* v_cache, void* stream);

/* The walk alone, given per-node LLM outputs [B][T] (what the reference's
 * verify() consumes, token_tree.cpp:153-175); same outputs as st_verify_greedy. */
st_status st_verify_outputs(const int32_t* outputs, int B, int T, const int32_t* tokens,
                            const int32_t* parent, const int32_t* n_nodes,
                            const int32_t* budget, int32_t eos, int32_t* verified,
                            int32_t* ids, int32_t* len, void* stream);

/* ------------------------------------------------------------------ K4 ---
 * Stochastic multi-step speculative sampling (SpecInfer MSS; NOT in the
 * reference — contract in DESIGN.md §5). q[b][v][:] is the draft
 * distribution of the SSM that proposed node v (row 0 unused). uniforms
 * [B][n_uniforms] in [0,1), consumed strictly in order. */
st_status st_verify_mss(const float* logits, const float* q, int B, int T, int V,
                        const int32_t* tokens, const int32_t* parent, const int32_t* n_nodes,
                        float temperature, const float* uniforms, int n_uniforms,
                        int32_t* verified, int32_t* ids, int32_t* len, void* stream);

/* ---------------------------------------- head-sharded K1 (C4, §8(e)) ---
 * K1 over this rank's H heads (heads [rank*H, (rank+1)*H) of world*H) with
 * the all-gather fused into the epilogue: every output row (b, u, local head
 * h) is stored straight into each rank's full-head buffer out[k]
 * ([B][T][world*H][D], k = 0..world-1, peer-mapped device pointers such as
 * symmetric-memory buffers) at head rank*H + h — over NVLink, overlapped with
 * the attention kernel — instead of an NCCL all-gather + relayout afterwards.
 * a->o is ignored; a->lse (local heads) is still written when non-NULL.
 * Completion is published with st_peer_signal and consumed with
 * st_peer_wait. Needs the tcgen05 path. */
typedef struct {
    int world, rank;
    void* const* out;   /* DEVICE array [world] of device pointers */
} st_peer_out;
st_status st_tree_attention_allgather(const st_attn_args* a, const st_peer_out* po, void* stream);

/* Stream-ordered after this rank's peer writes: a system-scope release store
 * of `epoch` into slot `rank` of every rank's signal array (signals: DEVICE
 * array [world] of peer-mapped uint32_t[world]). */
st_status st_peer_signal(uint32_t* const* signals, int world, int rank, uint32_t epoch,
                         void* stream);
/* Holds the stream until every slot of this rank's signal array has reached
 * `epoch` (wrap-around compare); traps after ~10 s instead of hanging. */
st_status st_peer_wait(const uint32_t* my_signals, int world, uint32_t epoch, void* stream);

/* ------------------------------------------------------------ host tree ---
 * TokenTree::merge_sequences of the host C++ library (drop-in for reference
 * token_tree.cpp:42-102): sequences given flattened (flat, lens[nseq]);
 * writes preorder tok/parent/depth (cap entries) and *n_out. Host-only: needs
 * no GPU. Returns tree_too_large / root_mismatch / empty_input like the
 * reference; ST_ERR_INVALID_ARGUMENT if cap is too small. */
st_status st_tree_merge(const int32_t* flat, const int32_t* lens, int nseq, int max_nodes,
                        int32_t* tok, int32_t* parent, int32_t* depth, int cap, int* n_out);

/* Batched host tree pipeline: merge_sequences for B
 * requests on a persistent host thread pool (n_threads <= 0: all hardware
 * threads), packed into padded [B][T] tok / parent / depth (depth may be
 * NULL) and n_nodes[B]; rows past a tree's size are filled with token 0,
 * parent -1, depth 0. Request b's sequences are the next nseq[b] entries of
 * lens[], their tokens the next sum(lens) entries of flat[]. Per-request
 * status (same codes as st_tree_merge) into status[B] when non-NULL; returns
 * the first non-OK status. A failed request gets n_nodes = 0. Host-only. */
st_status st_tree_merge_batch(int B, const int32_t* flat, const int32_t* lens,
                              const int32_t* nseq, int max_nodes, int T, int32_t* tok,
                              int32_t* parent, int32_t* depth, int32_t* n_nodes,
                              int32_t* status, int n_threads);

/* ------------------------------------------------- device decoder model ---
 * The reference's pre-LN decoder (proj/include/spectree/transformer.hpp:18-57)
 * resident on the device in f16/bf16 for the full-stack path (C3): weights are
 * generated on the GPU from UniformStream(seed) in the serialized order of
 * init_random_weights (reference transformer.cpp:71-114). st_model_tree_forward
 * runs every tree row of a batch through all layers (GEMMs over B*T rows; K2
 * append + K1 tree attention per layer) and writes f32 logits [B][T][V].
 * KV caches: [num_layers][B][H][Lmax][D]; row u of request b is written at
 * P[b]+u and sees rows [0,P[b]) plus its mask. */
typedef struct st_model st_model;
typedef struct {
    int num_layers, num_heads, d_model, vocab_size, max_positions, ffn_mult;
} st_model_config;
st_status st_model_create(const st_model_config* cfg, uint64_t seed, st_dtype dtype,
                          st_model** out);
void st_model_destroy(st_model* m);
size_t st_model_param_count(const st_model* m);
size_t st_model_workspace_size(const st_model* m, int B, int T);
st_status st_model_tree_forward(st_model* m, int B, int T, const int32_t* tokens,
                                const int32_t* positions, const uint64_t* mask, int W,
                                const int32_t* prefix_len, const int32_t* n_nodes, void* k_cache,
                                void* v_cache, int64_t Lmax, float* logits, void* workspace,
                                size_t workspace_bytes, void* stream);
/* The same pass in K1's k_tree mode: every layer's Q|K|V projection is written
 * to tree_qkv [num_layers][3][B*T][d_model] and K1 reads the tree rows from
 * there — no per-layer K2 append into the caches (rows [P, P+n) untouched).
 * After verification, st_kv_commit_tree(ids, len, ..., k_tree = tree_qkv +
 * B*T*d, v_tree = tree_qkv + 2*B*T*d, tree_layer_stride = 3*B*T*d) commits the
 * accepted rows of every layer. */
st_status st_model_tree_forward_kt(st_model* m, int B, int T, const int32_t* tokens,
                                   const int32_t* positions, const uint64_t* mask, int W,
                                   const int32_t* prefix_len, const int32_t* n_nodes,
                                   void* k_cache, void* v_cache, int64_t Lmax, void* tree_qkv,
                                   float* logits, void* workspace, size_t workspace_bytes,
                                   void* stream);
/* The k_tree pass over a SLICE of the tree: only nodes [u0, u0 + nf) of every
 * request (e.g. one level of a tree grown level by level) go through the
 * model — B*nf rows — attending to the committed rows and to every tree node
 * whose K/V is already in tree_qkv (earlier slices); the slice's own K/V rows
 * are written there (rows b*T + u), so after the last slice tree_qkv holds
 * the whole tree as st_model_tree_forward_kt leaves it. tokens / positions /
 * mask are the full-tree arrays ([B][T]); n_nodes counts the nodes so far.
 * logits (optional) [B][nf][V]; workspace st_model_workspace_size(m, B, nf). */
st_status st_model_tree_forward_slice(st_model* m, int B, int T, int u0, int nf,
                                      const int32_t* tokens, const int32_t* positions,
                                      const uint64_t* mask, int W, const int32_t* prefix_len,
                                      const int32_t* n_nodes, void* k_cache, void* v_cache,
                                      int64_t Lmax, void* tree_qkv, float* logits, void* workspace,
                                      size_t workspace_bytes, void* stream);

/* ------------------------------------------------- verification step plan ---
 * One verification step of a batch as a prepared object:
 * ancestor masks -> K1 -> K3 argmax -> K3 walk + K2 commit, from the tree's
 * own K/V rows (attn.k_tree/v_tree) or, with k_tree == NULL, after a K2 append
 * of k_new/v_new into the cache. st_verify_plan_run issues the four launches
 * with programmatic dependent launch, so back-to-back steps chain without a
 * boundary; K1's tensor maps are encoded once at creation. attn.mask is the
 * plan's mask buffer [B][T][W] (written by every run); attn.early_kv may be
 * set (the masks / append kernel before K1 honours the transitivity rule).
 * All pointers stay fixed for the plan's lifetime (their contents may change). */
typedef struct st_verify_plan st_verify_plan;
typedef struct {
    st_attn_args attn;
    const int32_t* tokens;       /* [B][T] */
    const int32_t* parent;       /* [B][T] */
    const float* logits;         /* [B][T][V] */
    int V;
    const int32_t* budget;       /* optional [B] */
    int32_t eos;                 /* < 0: none */
    int32_t* verified;           /* [B][T+1] */
    int32_t* ids;                /* [B][T+1] */
    int32_t* len;                /* [B] */
    void* verify_workspace;      /* st_verify_workspace_size(B, T) bytes, zeroed once */
    int32_t* new_prefix_len;     /* optional [B]: P + len */
    const void* k_new;           /* cache mode only: [B][T][Hkv][D] rows to append */
    const void* v_new;
} st_verify_step_desc;
st_status st_verify_plan_create(const st_verify_step_desc* d, st_verify_plan** out);
st_status st_verify_plan_run(st_verify_plan* p, void* stream);
void st_verify_plan_destroy(st_verify_plan* p);

/* ------------------------------------------------------- around-path GEMM ---
 * The device decoder's projections: C[z] (op)= A · W[z] on
 * the tcgen05 tensor cores, fp32 accumulate, the decoder's elementwise work
 * fused into the epilogue. A [M][lda] row-major, W [Z][K][ldw] row-major (the
 * stored weight layout), C [Z][M][ldc] (c_stride_z elements apart); f16/bf16
 * in; C f16/bf16, or f32 for ST_GEMM_STORE_F32. lda, ldw multiples of 8. */
enum { ST_GEMM_STORE = 0, ST_GEMM_GELU = 1, ST_GEMM_ADD_TO = 2, ST_GEMM_STORE_F32 = 3 };
st_status st_gemm(st_dtype dtype, int M, int N, int K, int Z, const void* A, int lda,
                  const void* W, int ldw, void* C, int ldc, int64_t c_stride_z, int epilogue,
                  void* stream);

/* The model's configuration and element type. */
void st_model_get_config(const st_model* m, st_model_config* out);
st_dtype st_model_get_dtype(const st_model* m);

/* ------------------------------------------------ device-resident engine ---
 * The reference's speculative loop (run_speculative, proj/src/engine.cpp:64-141)
 * for a batch of requests, resident on the device in f16/bf16 (SURVEY.md §8(f)
 * 3 and 4). Each st_engine_step (no host sync; capturable in a CUDA graph):
 * the draft model grows every live request's expansion tree <e_1..e_depth>
 * on the GPU (a masked tree pass per level + a top-e kernel), the LLM verifies
 * all trees in one tree pass, K3 walks them with budget truncation and the EOS
 * cut on the device, K2 commits the accepted rows of both caches, and the
 * accepted tokens are appended to the device sequences. ssm = NULL drafts with
 * the LLM itself; depth = 0 decodes one token per step (incremental greedy).
 * Trees are stored level by level (parent[u] < u). */
typedef struct st_engine st_engine;
typedef struct {
    int max_batch;       /* requests */
    int max_prompt;      /* longest prompt */
    int depth;           /* draft levels d (0..16) */
    int expansion[16];   /* e_1..e_d in [1, 8]: children kept per frontier node */
    int32_t eos;         /* < 0: none */
} st_engine_config;
st_status st_engine_create(st_model* llm, st_model* ssm, const st_engine_config* cfg,
                           st_engine** out);
void st_engine_destroy(st_engine* e);
int st_engine_tree_nodes(const st_engine* e);
/* host prompts (flattened), lengths and token budgets; prefills both models */
st_status st_engine_start(st_engine* e, int B, const int32_t* prompts, const int32_t* prompt_lens,
                          const int32_t* budgets, void* stream);
st_status st_engine_step(st_engine* e, void* stream);
/* the last step's accepted tokens [B][T+1], lengths [B], done flags [B] (host; syncs) */
st_status st_engine_read(st_engine* e, int32_t* verified, int32_t* len, int32_t* done,
                         void* stream);
/* request b's sequence (prompt + generated) into host out[cap] (syncs) */
st_status st_engine_sequence(st_engine* e, int b, int32_t* out, int cap, int* n_out,
                             void* stream);

/* ----------------------------------------------------- NCCL (DP exchange) ---
 * The data-parallel exchange of the verification step:
 * requests are partitioned over the ranks, and after each step every rank
 * all-gathers its requests' accepted tokens + lengths. NCCL is loaded at run
 * time (libnccl.so.2), so single-GPU users need none. One rank calls
 * st_comm_get_unique_id and shares the id out of band. */
typedef struct st_comm st_comm;
#define ST_COMM_ID_BYTES 128
st_status st_comm_get_unique_id(uint8_t* id);
st_status st_comm_init(int nranks, int rank, const uint8_t* id, st_comm** out);
st_status st_comm_allgather(st_comm* c, const void* send, void* recv, size_t bytes_per_rank,
                            void* stream);
/* pack verified [B][T+1] + len [B] into pack [B*(T+2)], all-gather into
 * gathered [nranks][B*(T+2)] */
st_status st_comm_gather_accepted(st_comm* c, const int32_t* verified, const int32_t* len, int B,
                                  int T, int32_t* pack, int32_t* gathered, void* stream);
int st_comm_size(const st_comm* c);
int st_comm_rank(const st_comm* c);
void st_comm_destroy(st_comm* c);

/* --------------------------------------------------------- tree packing ---
 * Device-side ancestor bitmask build: mask[b][u] = mask[b][parent[u]] | bit(u)
 * (reference TokenTree::ancestors, token_tree.cpp:130-139, as a bitset). */
st_status st_build_masks(const int32_t* parent, const int32_t* n_nodes, int B, int T, int W,
                         uint64_t* mask, void* stream);
/* Same masks, under the caller's promise that the kernel launched right
 * before it on the stream neither writes parent / n_nodes nor reads or writes
 * mask (e.g. the previous verification step's commit): the masks are built
 * while that kernel drains (programmatic dependent launch). */
st_status st_build_masks_early(const int32_t* parent, const int32_t* n_nodes, int B, int T, int W,
                               uint64_t* mask, void* stream);

#ifdef __cplusplus
}
#endif
#endif /* SPECTREE_CAPI_H */
