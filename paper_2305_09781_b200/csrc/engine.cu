// Device-resident speculative engine (SURVEY.md §8(f)3 + (f)4): the reference's
// run_speculative loop (proj/src/engine.cpp:64-141) for a BATCH of requests in
// f16/bf16 on the B200, with draft generation on the GPU.
//
// One step (st_engine_step, no host synchronisation, CUDA-graph capturable):
//   draft  : the SSM (or the LLM itself) grows each request's expansion tree
//            <e_1..e_d> level by level — one pass of the draft model over the
//            frontier level ONLY (st_model_tree_forward_slice: the earlier
//            levels' K/V stay in the draft tree buffer, so each node goes
//            through the draft model once per step, not once per level), then
//            the e_i most likely next tokens of every frontier node become its
//            children (top-e kernel below); one more slice pass over the last
//            level completes the tree's draft K/V, committed to the draft
//            model's cache with the accepted ids after verification
//   verify : one tree pass of the LLM over every request's tree -> K3 greedy
//            walk with the engine's budget truncation and EOS cut applied on
//            the device (engine.cpp:110-121), fused with the K2 commit of the
//            accepted rows; the draft model's cache is compacted with the same
//            accepted ids
//   commit : accepted tokens appended to the device sequences, budgets,
//            occupancies and done flags updated on the device
// Only the accepted tokens cross to the host (st_engine_read). Trees are laid
// out level by level (BFS): parent[u] < u, children of a node have distinct
// tokens — what the mask builder, K1 and the K3 walk need (preorder is not).
// Positions: node u sits at P[b] + depth(u), where P[b] = committed rows =
// sequence length - 1 (the root, the last accepted token, is recomputed in
// each step's tree pass, as the reference's root recompute,
// transformer.cpp:415-423). Depth is clamped so positions stay below
// max_positions (engine.cpp:95-103).
#include <algorithm>
#include <vector>

#include "common.cuh"
#include "tree_masks.cuh"

struct st_engine {
    st_model* llm = nullptr;
    st_model* ssm = nullptr;       // == llm when self-drafting
    st_engine_config cfg{};
    st_model_config mc{}, sc{};
    st_dtype dtype{};
    int B = 0, T = 0, W = 0, Tpf = 0, Lmax = 0, Lseq = 0;
    std::vector<int> lvl_end;      // nodes after level i (host constants)
    // device state
    void* buf = nullptr;
    int32_t *tok, *par, *pos, *n, *P, *Pnext, *seq, *seqlen, *remaining, *done, *ver, *ids, *len;
    uint64_t* mask;
    float *logits_llm, *logits_ssm;
    void *llm_k, *llm_v, *ssm_k, *ssm_v;
    void* tree_draft = nullptr;    // [ssm layers][3][B*T][d]: the draft tree's Q|K|V (slice passes)
    void *ws_model, *ws_ssm, *ws_ver;
    size_t ws_model_bytes = 0, ws_ssm_bytes = 0;
    int32_t* host = nullptr;       // pinned: [B][T+1] verified | [B] len | [B] done
};

namespace st {
namespace {

constexpr int kTopThreads = 256;
constexpr int kMaxE = 8;

__device__ __forceinline__ unsigned long long top_key(float v, int i) {
    // larger value first, then lower index (NaN never wins)
    if (v != v) v = -INFINITY;
    uint32_t u = v == 0.0f ? 0u : __float_as_uint(v);
    u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    return ((unsigned long long)u << 32) | (uint32_t)(~(uint32_t)i);
}

// Root of every live request's tree: the last accepted token at position P.
__global__ void tree_init_kernel(const int32_t* __restrict__ seq, const int32_t* __restrict__ seqlen,
                                 const int32_t* __restrict__ P, const int32_t* __restrict__ done,
                                 int Lseq, int T, int32_t* tok, int32_t* par, int32_t* pos,
                                 int32_t* n) {
    const int b = blockIdx.x;
    for (int u = threadIdx.x; u < T; u += blockDim.x) {
        tok[(int64_t)b * T + u] = 0;  // valid ids / positions for the rows past n
        par[(int64_t)b * T + u] = u > 0 ? u - 1 : -1;
        pos[(int64_t)b * T + u] = 0;
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const bool live = !done[b];
        n[b] = live ? 1 : 0;
        tok[(int64_t)b * T] = live ? seq[(int64_t)b * Lseq + seqlen[b] - 1] : 0;
        par[(int64_t)b * T] = -1;
        pos[(int64_t)b * T] = live ? P[b] : 0;
    }
}

// Level i of the expansion: frontier nodes [f0, f1) each keep their e most
// likely next tokens (draft logits row of the node) as children, written at
// f1 + k*e + j for frontier node f0 + k (BFS order). Block (k, b).
__global__ void __launch_bounds__(kTopThreads)
expand_kernel(const float* __restrict__ logits, int T, int V, int f0, int f1, int e, int depth,
              int max_positions, const int32_t* __restrict__ P, const int32_t* __restrict__ done,
              int32_t* tok, int32_t* par, int32_t* pos, int32_t* n) {
    const int k = blockIdx.x, b = blockIdx.y, u = f0 + k;
    const bool allowed = !done[b] && P[b] + depth + 1 <= max_positions - 1;
    if (!allowed || u >= f1) return;
    // the slice pass's logits: [B][f1 - f0][V], row k of request b = node f0 + k
    const float* row = logits + ((int64_t)b * (f1 - f0) + k) * V;
    // per-thread top-e (sorted, largest key first), then e block-wide rounds
    unsigned long long mine[kMaxE];
#pragma unroll
    for (int j = 0; j < kMaxE; ++j) mine[j] = 0;
    for (int t = threadIdx.x; t < V; t += kTopThreads) {
        unsigned long long key = top_key(row[t], t);
#pragma unroll
        for (int j = 0; j < kMaxE; ++j) {
            if (j < e && key > mine[j]) {
                const unsigned long long x = mine[j];
                mine[j] = key;
                key = x;
            }
        }
    }
    __shared__ unsigned long long red[kTopThreads / 32];
    __shared__ unsigned long long win;
    int head = 0;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (int j = 0; j < e; ++j) {
        unsigned long long best = head < e ? mine[head] : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (lane == 0) red[warp] = best;
        __syncthreads();
        if (threadIdx.x == 0) {
            unsigned long long m = red[0];
            for (int w = 1; w < kTopThreads / 32; ++w) m = max(m, red[w]);
            win = m;
            const int child = f1 + k * e + j;
            const int t = (int)(~(uint32_t)(m & 0xffffffffu));
            tok[(int64_t)b * T + child] = t;
            par[(int64_t)b * T + child] = u;
            pos[(int64_t)b * T + child] = P[b] + depth + 1;
        }
        __syncthreads();
        if (head < e && mine[head] == win) ++head;  // keys are unique (index in the low word)
        __syncthreads();
    }
    if (k == 0 && threadIdx.x == 0) n[b] = f1 + (f1 - f0) * e;
}

// After the verification: append the accepted tokens, budgets / done flags,
// occupancy P <- P + len (engine.cpp:110-133 on the device).
__global__ void commit_rows_kernel(const int32_t* __restrict__ ver, const int32_t* __restrict__ len,
                                   const int32_t* __restrict__ Pnext, int B, int T, int Lseq,
                                   int32_t eos, int32_t* seq, int32_t* seqlen, int32_t* remaining,
                                   int32_t* done, int32_t* P) {
    const int b = blockIdx.x * blockDim.x + threadIdx.x;
    if (b >= B || done[b]) return;
    const int L = len[b];
    const int at = seqlen[b];
    bool hit = false;
    for (int k = 0; k < L && at + k < Lseq; ++k) {
        const int32_t t = ver[(int64_t)b * (T + 1) + k];
        seq[(int64_t)b * Lseq + at + k] = t;
        hit |= eos >= 0 && t == eos;
    }
    seqlen[b] = at + L;
    remaining[b] -= L;
    P[b] = Pnext[b];
    if (hit || remaining[b] <= 0) done[b] = 1;
}

template <class X>
X* carve(char*& at, size_t count) {
    X* p = reinterpret_cast<X*>(at);
    at += (count * sizeof(X) + 255) & ~size_t(255);
    return p;
}

}  // namespace
}  // namespace st

extern "C" {

st_status st_engine_create(st_model* llm, st_model* ssm, const st_engine_config* cfg,
                           st_engine** out) {
    if (st_status e = st::require_device()) return e;
    ST_CHECK_ARG(llm && cfg && out, ST_ERR_INVALID_ARGUMENT, "null pointer");
    const st_engine_config c = *cfg;
    ST_CHECK_ARG(c.max_batch >= 1 && c.max_prompt >= 1 && c.depth >= 0 && c.depth <= 16,
                 ST_ERR_INVALID_ARGUMENT, "bad engine config");
    int nodes = 1, level = 1;
    std::vector<int> lvl_end{1};
    for (int i = 0; i < c.depth; ++i) {
        ST_CHECK_ARG(c.expansion[i] >= 1 && c.expansion[i] <= st::kMaxE, ST_ERR_INVALID_ARGUMENT,
                     "expansion e_i must be in [1, 8]");
        level *= c.expansion[i];
        nodes += level;
        lvl_end.push_back(nodes);
    }
    ST_CHECK_ARG(nodes <= 1024, ST_ERR_TREE_TOO_LARGE, "expansion tree > 1024 nodes");
    auto* e = new st_engine;
    e->llm = llm;
    e->ssm = ssm ? ssm : llm;
    e->cfg = c;
    e->lvl_end = lvl_end;
    st_model_get_config(llm, &e->mc);
    st_model_get_config(e->ssm, &e->sc);
    e->dtype = st_model_get_dtype(llm);
    if (e->mc.vocab_size != e->sc.vocab_size || e->mc.max_positions != e->sc.max_positions ||
        st_model_get_dtype(e->ssm) != e->dtype) {
        delete e;
        st::set_error("st_engine_create: LLM and SSM must share vocab, max_positions and dtype");
        return ST_ERR_SHAPE_MISMATCH;
    }
    e->B = c.max_batch;
    e->T = nodes;
    e->W = (std::max(nodes, c.max_prompt) + 63) / 64;
    e->Tpf = c.max_prompt;
    e->Lmax = e->mc.max_positions + std::max(nodes, c.max_prompt);  // + tree scratch rows
    e->Lseq = e->mc.max_positions;
    const int B = e->B, T = e->T, Tall = std::max(T, e->Tpf), V = e->mc.vocab_size;
    auto cache_elems = [&](const st_model_config& m) {
        return (size_t)m.num_layers * B * m.num_heads * e->Lmax * (m.d_model / m.num_heads);
    };
    const size_t es = st::dtype_size(e->dtype);
    e->ws_model_bytes = st_model_workspace_size(llm, B, Tall);
    e->ws_ssm_bytes = ssm && ssm != llm ? st_model_workspace_size(ssm, B, Tall) : 0;
    size_t bytes = 0;
    const size_t i32 = (size_t)B * Tall * 4 + 256;
    bytes += 3 * i32 + 10 * ((size_t)B * 4 + 256) + (size_t)B * e->Lseq * 4 + 256;
    bytes += 2 * ((size_t)B * (T + 1) * 4 + 256);
    bytes += (size_t)B * Tall * e->W * 8 + 256;
    bytes += (size_t)B * Tall * V * 4 + 256;                       // LLM logits
    bytes += (c.depth > 0 ? (size_t)B * T * V * 4 : 0) + 256;        // draft logits
    bytes += 2 * (cache_elems(e->mc) * es + 256);
    if (e->ssm != e->llm) bytes += 2 * (cache_elems(e->sc) * es + 256);
    const size_t tree_draft_bytes =
        c.depth > 0 ? (size_t)e->sc.num_layers * 3 * B * T * e->sc.d_model * es : 0;
    bytes += tree_draft_bytes + 256;
    bytes += e->ws_model_bytes + e->ws_ssm_bytes + st_verify_workspace_size(B, T) + 3 * 256;
    if (cudaMalloc(&e->buf, bytes) != cudaSuccess) {
        cudaGetLastError();
        delete e;
        st::set_error("st_engine_create: out of device memory");
        return ST_ERR_CUDA;
    }
    cudaMemset(e->buf, 0, bytes);
    char* at = static_cast<char*>(e->buf);
    e->tok = st::carve<int32_t>(at, (size_t)B * Tall);
    e->par = st::carve<int32_t>(at, (size_t)B * Tall);
    e->pos = st::carve<int32_t>(at, (size_t)B * Tall);
    e->n = st::carve<int32_t>(at, B);
    e->P = st::carve<int32_t>(at, B);
    e->Pnext = st::carve<int32_t>(at, B);
    e->seqlen = st::carve<int32_t>(at, B);
    e->remaining = st::carve<int32_t>(at, B);
    e->done = st::carve<int32_t>(at, B);
    e->len = st::carve<int32_t>(at, B);
    e->seq = st::carve<int32_t>(at, (size_t)B * e->Lseq);
    e->ver = st::carve<int32_t>(at, (size_t)B * (T + 1));
    e->ids = st::carve<int32_t>(at, (size_t)B * (T + 1));
    e->mask = st::carve<uint64_t>(at, (size_t)B * Tall * e->W);
    e->logits_llm = st::carve<float>(at, (size_t)B * Tall * V);
    e->logits_ssm = c.depth > 0 ? st::carve<float>(at, (size_t)B * T * V) : nullptr;
    e->llm_k = st::carve<char>(at, cache_elems(e->mc) * es);
    e->llm_v = st::carve<char>(at, cache_elems(e->mc) * es);
    if (e->ssm != e->llm) {
        e->ssm_k = st::carve<char>(at, cache_elems(e->sc) * es);
        e->ssm_v = st::carve<char>(at, cache_elems(e->sc) * es);
    } else {
        e->ssm_k = e->llm_k;  // self-drafting: the draft passes use the LLM's own cache
        e->ssm_v = e->llm_v;
    }
    e->tree_draft = tree_draft_bytes ? st::carve<char>(at, tree_draft_bytes) : nullptr;
    e->ws_model = st::carve<char>(at, e->ws_model_bytes);
    e->ws_ssm = e->ws_ssm_bytes ? st::carve<char>(at, e->ws_ssm_bytes) : e->ws_model;
    if (!e->ws_ssm_bytes) e->ws_ssm_bytes = e->ws_model_bytes;
    e->ws_ver = st::carve<char>(at, st_verify_workspace_size(B, T));
    if (cudaMallocHost(&e->host, ((size_t)B * (T + 1) + 2 * B) * 4) != cudaSuccess) {
        cudaGetLastError();
        cudaFree(e->buf);
        delete e;
        st::set_error("st_engine_create: out of pinned host memory");
        return ST_ERR_CUDA;
    }
    *out = e;
    return ST_OK;
}

void st_engine_destroy(st_engine* e) {
    if (!e) return;
    if (e->buf) cudaFree(e->buf);
    if (e->host) cudaFreeHost(e->host);
    delete e;
}

int st_engine_tree_nodes(const st_engine* e) { return e ? e->T : 0; }

st_status st_engine_start(st_engine* e, int B, const int32_t* prompts, const int32_t* prompt_lens,
                          const int32_t* budgets, void* stream) {
    if (st_status s = st::require_device()) return s;
    ST_CHECK_ARG(e && prompts && prompt_lens && budgets && B >= 1 && B <= e->B,
                 ST_ERR_INVALID_ARGUMENT, "bad arguments");
    cudaStream_t s = st::as_stream(stream);
    const int Tpf = e->Tpf, Tall = std::max(e->T, e->Tpf);
    std::vector<int32_t> tok((size_t)e->B * Tpf, 0), par((size_t)e->B * Tpf), pos((size_t)e->B * Tpf, 0);
    std::vector<int32_t> n(e->B, 0), zero(e->B, 0), seqlen(e->B, 0), rem(e->B, 0), done(e->B, 1);
    std::vector<int32_t> seq((size_t)e->B * e->Lseq, 0);
    size_t at = 0;
    for (int b = 0; b < e->B; ++b) {
        for (int u = 0; u < Tpf; ++u) par[(size_t)b * Tpf + u] = u - 1;
        if (b >= B) continue;
        const int L = prompt_lens[b];
        ST_CHECK_ARG(L >= 1, ST_ERR_EMPTY_INPUT, "empty prompt");
        ST_CHECK_ARG(L <= Tpf, ST_ERR_PROMPT_TOO_LONG, "prompt longer than max_prompt");
        ST_CHECK_ARG(budgets[b] >= 1 && L + budgets[b] <= e->mc.max_positions, ST_ERR_PROMPT_TOO_LONG,
                     "prompt + budget exceeds max_positions");
        for (int u = 0; u < L; ++u) {
            tok[(size_t)b * Tpf + u] = prompts[at + u];
            pos[(size_t)b * Tpf + u] = u;
            seq[(size_t)b * e->Lseq + u] = prompts[at + u];
        }
        at += L;
        n[b] = L;
        seqlen[b] = L;
        rem[b] = budgets[b];
        done[b] = 0;
    }
    // prefill: every prompt as a chain (causal masks) through the LLM and the SSM
    ST_CUDA_TRY(cudaMemcpyAsync(e->tok, tok.data(), tok.size() * 4, cudaMemcpyHostToDevice, s));
    ST_CUDA_TRY(cudaMemcpyAsync(e->par, par.data(), par.size() * 4, cudaMemcpyHostToDevice, s));
    ST_CUDA_TRY(cudaMemcpyAsync(e->pos, pos.data(), pos.size() * 4, cudaMemcpyHostToDevice, s));
    ST_CUDA_TRY(cudaMemcpyAsync(e->n, n.data(), e->B * 4, cudaMemcpyHostToDevice, s));
    ST_CUDA_TRY(cudaMemcpyAsync(e->P, zero.data(), e->B * 4, cudaMemcpyHostToDevice, s));
    ST_CUDA_TRY(cudaMemcpyAsync(e->seq, seq.data(), seq.size() * 4, cudaMemcpyHostToDevice, s));
    ST_CUDA_TRY(cudaMemcpyAsync(e->seqlen, seqlen.data(), e->B * 4, cudaMemcpyHostToDevice, s));
    ST_CUDA_TRY(cudaMemcpyAsync(e->remaining, rem.data(), e->B * 4, cudaMemcpyHostToDevice, s));
    ST_CUDA_TRY(cudaMemcpyAsync(e->done, done.data(), e->B * 4, cudaMemcpyHostToDevice, s));
    const int Wp = (Tpf + 63) / 64;
    if (st_status r = st_build_masks(e->par, e->n, e->B, Tpf, Wp, e->mask, stream)) return r;
    if (st_status r = st_model_tree_forward(e->llm, e->B, Tpf, e->tok, e->pos, e->mask, Wp, e->P,
                                            e->n, e->llm_k, e->llm_v, e->Lmax, e->logits_llm,
                                            e->ws_model, e->ws_model_bytes, stream))
        return r;
    if (e->ssm != e->llm && e->cfg.depth > 0) {
        if (st_status r = st_model_tree_forward(e->ssm, e->B, Tpf, e->tok, e->pos, e->mask, Wp,
                                                e->P, e->n, e->ssm_k, e->ssm_v, e->Lmax,
                                                e->logits_llm, e->ws_ssm, e->ws_ssm_bytes, stream))
            return r;
    }
    // committed rows: the prompt minus its last token (recomputed as each tree's root)
    std::vector<int32_t> P0(e->B, 0);
    for (int b = 0; b < B; ++b) P0[b] = prompt_lens[b] - 1;
    ST_CUDA_TRY(cudaMemcpyAsync(e->P, P0.data(), e->B * 4, cudaMemcpyHostToDevice, s));
    (void)Tall;
    return ST_OK;
}

st_status st_engine_step(st_engine* e, void* stream) {
    ST_CHECK_ARG(e != nullptr, ST_ERR_INVALID_ARGUMENT, "null engine");
    cudaStream_t s = st::as_stream(stream);
    const int B = e->B, T = e->T, W = (T + 63) / 64, V = e->mc.vocab_size;
    st::tree_init_kernel<<<B, 128, 0, s>>>(e->seq, e->seqlen, e->P, e->done, e->Lseq, T, e->tok,
                                           e->par, e->pos, e->n);
    ST_LAUNCH_CHECK();
    const int d = e->cfg.depth;
    for (int i = 0; i < d; ++i) {   // draft: grow level i+1 from level i
        const int f0 = i == 0 ? 0 : e->lvl_end[i - 1], f1 = e->lvl_end[i];
        if (st_status r = st_build_masks(e->par, e->n, B, T, W, e->mask, stream)) return r;
        // the frontier level through the draft model (earlier levels' K/V
        // are in tree_draft from the previous slices)
        if (st_status r = st_model_tree_forward_slice(e->ssm, B, T, f0, f1 - f0, e->tok, e->pos,
                                                      e->mask, W, e->P, e->n, e->ssm_k, e->ssm_v,
                                                      e->Lmax, e->tree_draft, e->logits_ssm,
                                                      e->ws_ssm, e->ws_ssm_bytes, stream))
            return r;
        st::expand_kernel<<<dim3(f1 - f0, B), st::kTopThreads, 0, s>>>(
            e->logits_ssm, T, V, f0, f1, e->cfg.expansion[i], i, e->mc.max_positions, e->P, e->done,
            e->tok, e->par, e->pos, e->n);
        ST_LAUNCH_CHECK();
    }
    if (st_status r = st_build_masks(e->par, e->n, B, T, W, e->mask, stream)) return r;
    if (d > 0 && e->ssm != e->llm) {  // draft-model K/V of the last level (no logits needed)
        const int f0 = e->lvl_end[d - 1], f1 = e->lvl_end[d];
        if (st_status r = st_model_tree_forward_slice(e->ssm, B, T, f0, f1 - f0, e->tok, e->pos,
                                                      e->mask, W, e->P, e->n, e->ssm_k, e->ssm_v,
                                                      e->Lmax, e->tree_draft, nullptr, e->ws_ssm,
                                                      e->ws_ssm_bytes, stream))
            return r;
    }
    // verify: the LLM over every tree, greedy walk + budget/EOS + K2 commit
    if (st_status r = st_model_tree_forward(e->llm, B, T, e->tok, e->pos, e->mask, W, e->P, e->n,
                                            e->llm_k, e->llm_v, e->Lmax, e->logits_llm,
                                            e->ws_model, e->ws_model_bytes, stream))
        return r;
    const int Dh = e->mc.d_model / e->mc.num_heads;
    const int64_t layer = (int64_t)B * e->mc.num_heads * e->Lmax * Dh;
    if (st_status r = st_verify_greedy_compact(
            e->logits_llm, B, T, V, e->tok, e->par, e->n, e->remaining, e->cfg.eos, nullptr,
            e->ver, e->ids, e->len, e->ws_ver, e->dtype, e->mc.num_heads, Dh, e->Lmax,
            e->mc.num_layers, layer, e->P, e->Pnext, nullptr, nullptr, 0, e->llm_k, e->llm_v,
            stream))
        return r;
    if (d > 0 && e->ssm != e->llm) {  // the accepted rows' draft K/V into the draft cache
        const int sDh = e->sc.d_model / e->sc.num_heads;
        const size_t tl = (size_t)B * T * e->sc.d_model;  // one [B*T][d] slot of tree_draft
        const size_t es = st::dtype_size(e->dtype);
        if (st_status r = st_kv_commit_tree(
                e->dtype, B, T, e->sc.num_heads, sDh, e->Lmax, e->sc.num_layers,
                (int64_t)B * e->sc.num_heads * e->Lmax * sDh, e->ids, T + 1, e->len, e->P, nullptr,
                static_cast<char*>(e->tree_draft) + tl * es, static_cast<char*>(e->tree_draft) + 2 * tl * es,
                (int64_t)(3 * tl), e->ssm_k, e->ssm_v, stream))
            return r;
    }
    st::commit_rows_kernel<<<(B + 127) / 128, 128, 0, s>>>(e->ver, e->len, e->Pnext, B, T, e->Lseq,
                                                          e->cfg.eos, e->seq, e->seqlen,
                                                          e->remaining, e->done, e->P);
    ST_LAUNCH_CHECK();
    return ST_OK;
}

st_status st_engine_read(st_engine* e, int32_t* verified, int32_t* len, int32_t* done,
                         void* stream) {
    ST_CHECK_ARG(e != nullptr, ST_ERR_INVALID_ARGUMENT, "null engine");
    cudaStream_t s = st::as_stream(stream);
    const int B = e->B, T = e->T;
    int32_t* h = e->host;
    ST_CUDA_TRY(cudaMemcpyAsync(h, e->ver, (size_t)B * (T + 1) * 4, cudaMemcpyDeviceToHost, s));
    ST_CUDA_TRY(cudaMemcpyAsync(h + (size_t)B * (T + 1), e->len, (size_t)B * 4,
                                cudaMemcpyDeviceToHost, s));
    ST_CUDA_TRY(cudaMemcpyAsync(h + (size_t)B * (T + 2), e->done, (size_t)B * 4,
                                cudaMemcpyDeviceToHost, s));
    ST_CUDA_TRY(cudaStreamSynchronize(s));
    if (verified) std::copy(h, h + (size_t)B * (T + 1), verified);
    if (len) std::copy(h + (size_t)B * (T + 1), h + (size_t)B * (T + 2), len);
    if (done) std::copy(h + (size_t)B * (T + 2), h + (size_t)B * (T + 3), done);
    return ST_OK;
}

st_status st_engine_sequence(st_engine* e, int b, int32_t* out, int cap, int* n_out,
                             void* stream) {
    ST_CHECK_ARG(e && out && n_out && b >= 0 && b < e->B, ST_ERR_INVALID_ARGUMENT, "bad arguments");
    cudaStream_t s = st::as_stream(stream);
    int32_t L = 0;
    ST_CUDA_TRY(cudaMemcpyAsync(&L, e->seqlen + b, 4, cudaMemcpyDeviceToHost, s));
    ST_CUDA_TRY(cudaStreamSynchronize(s));
    *n_out = L;
    ST_CHECK_ARG(L <= cap, ST_ERR_INVALID_ARGUMENT, "output buffer too small");
    ST_CUDA_TRY(cudaMemcpyAsync(out, e->seq + (size_t)b * e->Lseq, (size_t)L * 4,
                                cudaMemcpyDeviceToHost, s));
    ST_CUDA_TRY(cudaStreamSynchronize(s));
    return ST_OK;
}

}  // extern "C"
