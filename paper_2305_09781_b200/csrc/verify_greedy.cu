// K3: greedy verification — per-node vocabulary argmax fused with the
// accepted-path walk — and the device-side ancestor-bitmask builder.
//
// Reference semantics:
//   * argmax_token (proj/src/transformer.cpp:116-122): best starts at 0 and
//     index i replaces it only if logits[i] > logits[best] — lowest id wins
//     ties; a NaN never wins, and a NaN at index 0 is never replaced.
//   * verify (proj/src/token_tree.cpp:153-175): from the root, follow the child
//     whose token equals the node's output, then append the last node's output
//     (the bonus token).
//   * engine step (proj/src/engine.cpp:110-121): budget truncation, then the
//     EOS cut.
//
// Work split: kSplit 256-thread blocks per (request, node) stream slices of
// that node's logits row once (HBM-bound: 4*V bytes per node, float4 loads)
// and fold their best (value, lowest index) into one 64-bit order-preserving
// key with atomicMax (order-independent, hence deterministic); a second,
// PDL-launched kernel (one warp per request) resolves the keys and walks:
// children of u are the ids v > u with parent[v] == u, scanned 32 at a time
// with a ballot.
#include <algorithm>
#include <cfloat>

#include "common.cuh"
#include "kv_move.cuh"
#include "tree_masks.cuh"

namespace st {
namespace {

constexpr int kThreads = 256;

// Alg.-2 walk (reference token_tree.cpp:153-175) + engine truncation
// (engine.cpp:110-121) for request b, executed by one full warp.
// `outs` holds the per-node LLM outputs [B][T] (read through L2 when written by
// other CTAs). The tree is staged in shared memory and every node's matching
// child is found in parallel first (children have unique tokens, so at most one
// matches), which turns the walk into a short pointer chase in smem instead of
// a chain of dependent global loads per level.
constexpr int kWalkMax = 1024;   // nodes staged in smem; larger trees walk from global

__device__ void walk_warp(const int32_t* outs, const int32_t* __restrict__ tokens,
                          const int32_t* __restrict__ parent, int n, int T, int b,
                          const int32_t* __restrict__ budget, int32_t eos,
                          int32_t* __restrict__ verified, int32_t* __restrict__ ids,
                          int32_t* __restrict__ len, int lane, bool coherent, int* s_out,
                          int* s_next) {
    const int32_t* tok = tokens + (int64_t)b * T;
    const int32_t* par = parent + (int64_t)b * T;
    const int32_t* am = outs + (int64_t)b * T;
    int32_t* vrow = verified + (int64_t)b * (T + 1);
    int32_t* irow = ids + (int64_t)b * (T + 1);
    int m = 0, cur = 0;
    if (n <= 0) {  // no tree: nothing accepted
        if (lane == 0) len[b] = 0;
        return;
    }
    if (n <= kWalkMax) {
        for (int v = lane; v < n; v += 32) {
            s_out[v] = coherent ? __ldcg(am + v) : am[v];
            s_next[v] = -1;
        }
        __syncwarp();
        for (int v = 1 + lane; v < n; v += 32) {
            const int u = par[v];
            if (tok[v] == s_out[u]) s_next[u] = v;
        }
        __syncwarp();
        if (lane == 0) {
            irow[0] = 0;
            for (int nx = s_next[0]; nx >= 0; nx = s_next[cur]) {
                vrow[m] = s_out[cur];
                irow[m + 1] = nx;
                cur = nx;
                ++m;
            }
            vrow[m] = s_out[cur];  // bonus token
        }
    } else {
        if (lane == 0) irow[0] = 0;
        for (;;) {
            const int32_t want = coherent ? __ldcg(am + cur) : am[cur];
            int next = -1;
            for (int v0 = cur + 1; v0 < n && next < 0; v0 += 32) {
                const int v = v0 + lane;
                const bool hit = v < n && par[v] == cur && tok[v] == want;
                const unsigned bal = __ballot_sync(0xffffffffu, hit);
                if (bal) next = v0 + __ffs(bal) - 1;
            }
            if (next < 0) break;
            cur = next;
            if (lane == 0) {
                vrow[m] = want;
                irow[m + 1] = cur;
            }
            ++m;
        }
        if (lane == 0) vrow[m] = coherent ? __ldcg(am + cur) : am[cur];  // bonus token
    }
    if (lane == 0) {
        int L = m + 1;
        if (budget && L > budget[b]) L = budget[b] > 0 ? budget[b] : 0;
        if (eos >= 0) {
            for (int k = 0; k < L; ++k)
                if (vrow[k] == eos) { L = k + 1; break; }
        }
        len[b] = L;
    }
}

__global__ void walk_kernel(const int32_t* __restrict__ outs, int T,
                            const int32_t* __restrict__ tokens, const int32_t* __restrict__ parent,
                            const int32_t* __restrict__ n_nodes, const int32_t* __restrict__ budget,
                            int32_t eos, int32_t* __restrict__ verified, int32_t* __restrict__ ids,
                            int32_t* __restrict__ len) {
    __shared__ int s_out[kWalkMax], s_next[kWalkMax];
    const int b = blockIdx.x;
    walk_warp(outs, tokens, parent, n_nodes[b], T, b, budget, eos, verified, ids, len,
              threadIdx.x & 31, false, s_out, s_next);
}

// Order-preserving 64-bit key: high word = orderable float bits, low word =
// ~index, so an unsigned max picks the largest value and, among equal values,
// the LOWEST index (reference tie rule). NaN maps to -inf (never wins); a NaN
// at index 0 gets the maximal key (the reference never replaces index 0).
// -0.0 and +0.0 compare equal under the reference's '>', so both map to the
// same key and the lower index wins between them too.
__device__ __forceinline__ unsigned long long arg_key(float v, int i) {
    if (v != v) {
        if (i == 0) return ~0ull;
        v = -INFINITY;
    }
    uint32_t u = v == 0.0f ? 0u : __float_as_uint(v);  // canonicalise -0.0
    u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    return ((unsigned long long)u << 32) | (uint32_t)(~(uint32_t)i);
}
__device__ __forceinline__ int key_index(unsigned long long k) {
    return k == ~0ull ? 0 : (int)(~(uint32_t)(k & 0xffffffffu));
}

constexpr int kSplit = 8;   // blocks per logits row (tools/argmax_bench.cu: 8 x 4 loads beat 4 x 8)
constexpr int kUnroll = 4;  // float4 loads in flight per thread (a 4000-float slice in one batch)

// Block-level walk of request b (blockDim.x threads, n <= kWalkMax):
// greedy outputs from the slice keys, every node's matching child found in
// parallel (children have distinct tokens: at most one matches), the pointer
// chase from the root, then the engine's budget truncation and EOS cut
// (engine.cpp:110-121). Results in shared memory: s_ids/s_ver [0, *s_full)
// and the truncated length *s_len. `lead`: also write argmax_out, the
// verified/ids rows and len to global memory.
struct WalkSmem {
    int out[kWalkMax], next[kWalkMax], ver[kWalkMax + 1], ids[kWalkMax + 1];
    int len, full;
};

__device__ unsigned long long resolve_max(const unsigned long long* keys, int64_t row);

__device__ void walk_block(WalkSmem& w, const unsigned long long* keys, int T, int b, int n,
                           const int32_t* __restrict__ tokens, const int32_t* __restrict__ parent,
                           const int32_t* __restrict__ budget, int32_t eos, bool lead,
                           int32_t* __restrict__ argmax_out, int32_t* __restrict__ verified,
                           int32_t* __restrict__ ids, int32_t* __restrict__ len) {
    const int32_t* tok = tokens + (int64_t)b * T;
    const int32_t* par = parent + (int64_t)b * T;
    for (int v = threadIdx.x; v < n; v += blockDim.x) {
        const int a = key_index(resolve_max(keys, (int64_t)b * T + v));
        w.out[v] = a;
        w.next[v] = -1;
        if (lead && argmax_out) argmax_out[(int64_t)b * T + v] = a;
    }
    __syncthreads();
    for (int v = 1 + threadIdx.x; v < n; v += blockDim.x) {
        const int u = par[v];
        if (tok[v] == w.out[u]) w.next[u] = v;  // one writer per u
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        int m = 0, cur = 0;
        w.ids[0] = 0;
        for (int nx = n > 0 ? w.next[0] : -1; nx >= 0; nx = w.next[cur]) {
            w.ver[m] = w.out[cur];
            w.ids[m + 1] = nx;
            cur = nx;
            ++m;
        }
        w.ver[m] = n > 0 ? w.out[cur] : 0;  // bonus token
        w.full = n > 0 ? m + 1 : 0;
        int L = w.full;
        if (budget && L > budget[b]) L = budget[b] > 0 ? budget[b] : 0;
        if (eos >= 0) {
            for (int k = 0; k < L; ++k)
                if (w.ver[k] == eos) { L = k + 1; break; }
        }
        w.len = L;
    }
    __syncthreads();
    if (lead) {
        // the whole walk (path + bonus); len carries the budget / EOS truncation
        int32_t* vrow = verified + (int64_t)b * (T + 1);
        int32_t* irow = ids + (int64_t)b * (T + 1);
        for (int k = threadIdx.x; k < w.full; k += blockDim.x) {
            vrow[k] = w.ver[k];
            irow[k] = w.ids[k];
        }
        if (threadIdx.x == 0) len[b] = w.len;
    }
}

// Phase 1: stream every live node's logits once; kSplit blocks per row each
// reduce their slice to one order-preserving key, written to its own slot
// keys[b][u][part] (no atomics, nothing to reset; the consumer takes the max
// of the kSplit keys — order-independent, hence deterministic).
//
// Fused walk (`counters` != NULL, T <= kWalkMax): after publishing its key a
// block counts itself in (threadfence + atomicAdd, the classic last-block
// pattern — no block ever waits for another); the block that completes
// request b's n*kSplit keys runs the walk for b and re-arms the counter. One
// launch instead of argmax + a dependent walk kernel.
struct WalkArgs {
    unsigned* counters;  // [B], zero between calls
    const int32_t* tokens;
    const int32_t* parent;
    const int32_t* budget;
    int32_t eos;
    int32_t* argmax_out;
    int32_t* verified;
    int32_t* ids;
    int32_t* len;
};

__global__ void __launch_bounds__(kThreads)
greedy_argmax_kernel(const float* __restrict__ logits, int T, int V,
                     const int32_t* __restrict__ n_nodes, unsigned long long* keys,
                     const WalkArgs wa, int early) {
    // early (the step plan): the kernel before this one writes neither the
    // logits nor the node counts, so the rows stream while it drains and only
    // the key store waits for it (every block's completion still implies the
    // previous kernel's, as the launches after this one rely on)
    if (!early) pdl_wait();
    pdl_trigger();  // let the next kernel get scheduled while the rows stream
    const int part = blockIdx.x, u = blockIdx.y, b = blockIdx.z;
    const int n = n_nodes[b];
    if (u >= n) {
        if (early) pdl_wait();
        if (wa.counters && n <= 0 && u == 0 && part == 0 && threadIdx.x == 0) wa.len[b] = 0;
        return;
    }
    const float* row = logits + ((int64_t)b * T + u) * V;
    const bool vec = ((reinterpret_cast<uintptr_t>(row) & 15) == 0) && (V % 4 == 0);
    unsigned long long best = 0;
    if (vec) {
        const int nv = V >> 2;
        const int per = (nv + kSplit - 1) / kSplit;
        const int lo = part * per, hi = min(nv, lo + per);
        const float4* r4 = reinterpret_cast<const float4*>(row);
        // this thread's elements in increasing index order with the reference's
        // strict '>' (NaN never wins, ties keep the lower index); the 64-bit key
        // is formed once per thread. Starts at the thread's first index so an
        // all -inf/NaN slice reports its lowest index, as arg_key would.
        float bv = -INFINITY;
        int bi = lo + (int)threadIdx.x < hi ? (lo + (int)threadIdx.x) * 4 : -1;
        for (int base = lo + threadIdx.x; base < hi; base += kThreads * kUnroll) {
            float4 x[kUnroll];
#pragma unroll
            for (int k = 0; k < kUnroll; ++k) {
                const int j = base + k * kThreads;
                x[k] = j < hi ? __ldcs(r4 + j) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
            }
#pragma unroll
            for (int k = 0; k < kUnroll; ++k) {
                const int j = (base + k * kThreads) * 4;
                if (x[k].x > bv) { bv = x[k].x; bi = j; }
                if (x[k].y > bv) { bv = x[k].y; bi = j + 1; }
                if (x[k].z > bv) { bv = x[k].z; bi = j + 2; }
                if (x[k].w > bv) { bv = x[k].w; bi = j + 3; }
            }
        }
        if (bi >= 0) best = arg_key(bv, bi);
        if (lo == 0 && threadIdx.x == 0 && row[0] != row[0]) best = ~0ull;  // NaN at index 0
    } else {
        const int per = (V + kSplit - 1) / kSplit;
        const int lo = part * per, hi = min(V, lo + per);
        for (int j = lo + threadIdx.x; j < hi; j += kThreads) best = max(best, arg_key(row[j], j));
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    __shared__ unsigned long long red[kThreads / 32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[warp] = best;
    __syncthreads();
    __shared__ bool s_last;
    if (threadIdx.x == 0) {
        for (int w = 1; w < kThreads / 32; ++w) best = max(best, red[w]);
        if (early) pdl_wait();
        keys[((int64_t)b * T + u) * kSplit + part] = best;
        if (wa.counters) {
            __threadfence();  // the key before the count
            s_last = atomicAdd(wa.counters + b, 1u) == (unsigned)(n * kSplit) - 1u;
        }
    }
    if (!wa.counters) return;
    __syncthreads();
    if (!s_last) return;
    __threadfence();  // every other block's key is visible (they fenced before counting)
    __shared__ WalkSmem w;
    walk_block(w, keys, T, b, n, wa.tokens, wa.parent, wa.budget, wa.eos, true, wa.argmax_out,
               wa.verified, wa.ids, wa.len);
    if (threadIdx.x == 0) wa.counters[b] = 0u;  // re-armed for the next call
}

// Greedy output of node v: the best of its kSplit slice keys.
__device__ unsigned long long resolve_max(const unsigned long long* keys, int64_t row) {
    unsigned long long k = 0;
#pragma unroll
    for (int j = 0; j < kSplit; ++j) k = max(k, __ldcg(keys + row * kSplit + j));
    return k;
}
__device__ __forceinline__ int resolve_key(const unsigned long long* keys, int64_t row) {
    return key_index(resolve_max(keys, row));
}

// Phase 2 (launched with programmatic dependent launch): one warp per request
// resolves the argmax keys, then walks.
__global__ void __launch_bounds__(32)
greedy_walk_kernel(int T, const int32_t* __restrict__ tokens, const int32_t* __restrict__ parent,
                   const int32_t* __restrict__ n_nodes, const int32_t* __restrict__ budget,
                   int32_t eos, int32_t* __restrict__ argmax_out, const unsigned long long* keys,
                   int32_t* argmax_ws, int32_t* __restrict__ verified, int32_t* __restrict__ ids,
                   int32_t* __restrict__ len) {
    pdl_wait();
    pdl_trigger();
    __shared__ int s_out[kWalkMax], s_next[kWalkMax];
    const int b = blockIdx.x, lane = threadIdx.x;
    const int n = n_nodes[b];
    int32_t* am = argmax_ws + (int64_t)b * T;
    for (int v = lane; v < n; v += 32) {
        const int a = resolve_key(keys, (int64_t)b * T + v);
        am[v] = a;
        if (argmax_out) argmax_out[(int64_t)b * T + v] = a;
    }
    __syncwarp();
    walk_warp(argmax_ws, tokens, parent, n, T, b, budget, eos, verified, ids, len, lane, false,
              s_out, s_next);
}

// ------------------------------------------------ K3 walk fused with K2 ---
// Walk + compaction in one launch (st_verify_greedy_compact): block (b, y)
// resolves request b's greedy outputs, walks its tree in shared memory (every
// block of the request repeats this tiny walk, so no grid-wide dependency is
// needed), then moves the accepted rows of its `hpb` KV heads of one layer:
//   cache[b][h][P + k] = cache[b][h][P + ids[k]],  k = 1 .. len-1.
// ids are strictly increasing with ids[k] >= k, so a destination row k is
// never a source of a later k; within a chunk of rows every source is loaded
// before any destination is stored (one barrier), and chunks go in increasing
// k — no sequential per-row chain. Block (b, 0) writes the walk's outputs.
constexpr int kWcThreads = 256;

template <class V>
__global__ void __launch_bounds__(kWcThreads)
walk_compact_kernel(int T, const int32_t* __restrict__ tokens, const int32_t* __restrict__ parent,
                    const int32_t* __restrict__ n_nodes, const int32_t* __restrict__ budget,
                    int32_t eos, int32_t* __restrict__ argmax_out, const unsigned long long* keys,
                    int32_t* __restrict__ verified, int32_t* __restrict__ ids,
                    int32_t* __restrict__ len, char* k_cache, char* v_cache, int Hkv,
                    int row_vecs, int64_t Lmax, int nhc, int hpb, int64_t layer_stride_bytes,
                    const int32_t* __restrict__ prefix_len, int32_t* __restrict__ new_prefix_len,
                    const char* __restrict__ k_tree, const char* __restrict__ v_tree,
                    int64_t tree_layer_stride_bytes, int walk_done) {
    pdl_wait();
    pdl_trigger();
    __shared__ WalkSmem w;
    const int b = blockIdx.x, layer = blockIdx.y / nhc, hc = blockIdx.y % nhc;
    const int n = n_nodes[b];
    const bool lead = blockIdx.y == 0;
    if (walk_done) {  // the argmax kernel already walked: accepted ids and len from global
        const int L0 = len[b];
        for (int k = threadIdx.x; k < L0; k += kWcThreads) w.ids[k] = ids[(int64_t)b * (T + 1) + k];
        if (threadIdx.x == 0) w.len = L0;
        __syncthreads();
    } else {
        walk_block(w, keys, T, b, n, tokens, parent, budget, eos, lead, argmax_out, verified, ids,
                   len);
    }
    const int* s_ids = w.ids;
    const int L = w.len;
    const int64_t P = prefix_len[b];
    if (lead && threadIdx.x == 0 && new_prefix_len) new_prefix_len[b] = (int32_t)(P + L);
    // ---- compaction of rows k0..L-1 for heads [hc*hpb, hc*hpb + hpb) of this layer ----
    // (in place: rows 1.. from cache row P + ids[k]; k_tree mode: rows 0.. from
    // the tree's own K/V, tree[b][ids[k]][h])
    const int h0 = hc * hpb, nh = min(hpb, Hkv - h0);
    const int kfirst = k_tree ? 0 : 1;
    if (L <= kfirst || nh <= 0) return;
    char* kl = k_cache + layer * layer_stride_bytes;
    char* vl = v_cache + layer * layer_stride_bytes;
    const char* ktl = k_tree ? k_tree + layer * tree_layer_stride_bytes : nullptr;
    const char* vtl = v_tree ? v_tree + layer * tree_layer_stride_bytes : nullptr;
    move_rows_block<V>(s_ids, L, kfirst, b, h0, nh, Hkv, row_vecs, Lmax, P, kl, vl, ktl, vtl, T);
}

// One thread per (request, node): tree_masks.cuh.
// early: the caller promises the previous kernel on the stream neither writes
// parent / n_nodes nor touches mask, so the masks are built while it drains.
// The dependents' launch is released only AFTER this kernel's own wait: an
// early_kv K1 that follows streams the committed rows [0, P) before ITS wait,
// so it must not start while the kernel before this one (e.g. the previous
// step's commit, which writes rows [P_prev, P)) may still run.
__global__ void build_masks_kernel(const int32_t* __restrict__ parent,
                                   const int32_t* __restrict__ n_nodes, int T, int W,
                                   uint64_t* __restrict__ mask, int early) {
    extern __shared__ int s_par[];
    if (!early) {
        pdl_wait();
        pdl_trigger();
    }
    build_masks_block(parent, n_nodes, T, W, mask, blockIdx.x, blockIdx.y, s_par);
    if (early) {
        pdl_wait();
        pdl_trigger();
    }
}

}  // namespace
}  // namespace st

extern "C" {

size_t st_verify_workspace_size(int B, int T) {
    // slice keys [B][T][kSplit] u64 | argmax scratch [B][T] | walk counters [B]
    // (zeroed once by the caller; every call leaves the counters zero)
    return (size_t)B * T * st::kSplit * 8 + (size_t)B * T * sizeof(int32_t) +
           (size_t)B * sizeof(unsigned) + 512;
}

st_status st_verify_greedy(const float* logits, int B, int T, int V, const int32_t* tokens,
                           const int32_t* parent, const int32_t* n_nodes, const int32_t* budget,
                           int32_t eos, int32_t* argmax, int32_t* verified, int32_t* ids,
                           int32_t* len, void* workspace, void* stream) {
    if (st_status e = st::require_device()) return e;
    ST_CHECK_ARG(B >= 0 && T >= 1 && V >= 1, ST_ERR_SHAPE_MISMATCH, "bad shape");
    if (B == 0) return ST_OK;
    ST_CHECK_ARG(logits && tokens && parent && n_nodes && verified && ids && len && workspace,
                 ST_ERR_INVALID_ARGUMENT, "null pointer");
    ST_CHECK_ARG(B <= 65535 && T <= 2147483647, ST_ERR_SHAPE_MISMATCH, "too many requests");
    ST_CHECK_ARG((reinterpret_cast<uintptr_t>(workspace) & 7) == 0, ST_ERR_INVALID_ARGUMENT,
                 "workspace must be 8-byte aligned");
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(workspace);
    int32_t* scratch = reinterpret_cast<int32_t*>(keys + (size_t)B * T * st::kSplit);
    unsigned* counters = reinterpret_cast<unsigned*>(scratch + (size_t)B * T);
    const dim3 grid(st::kSplit, T, B);
    auto strm = st::as_stream(stream);
    if (T <= st::kWalkMax) {  // one launch: the last argmax block of each request walks it
        const st::WalkArgs wa{counters, tokens, parent, budget, eos, argmax, verified, ids, len};
        ST_CUDA_TRY(st::launch_pdl(st::greedy_argmax_kernel, grid, dim3(st::kThreads), 0, strm,
                                   logits, T, V, n_nodes, keys, wa, 0));
        ST_LAUNCH_CHECK();
        return ST_OK;
    }
    const st::WalkArgs none{};
    ST_CUDA_TRY(st::launch_pdl(st::greedy_argmax_kernel, grid, dim3(st::kThreads), 0, strm, logits,
                               T, V, n_nodes, keys, none, 0));
    ST_LAUNCH_CHECK();
    ST_CUDA_TRY(st::launch_pdl(st::greedy_walk_kernel, dim3(B), dim3(32), 0, strm, T, tokens,
                               parent, n_nodes, budget, eos, argmax, keys, scratch, verified, ids,
                               len));
    ST_LAUNCH_CHECK();
    return ST_OK;
}

static st_status verify_greedy_compact_impl(const float* logits, int B, int T, int V, const int32_t*
                                            tokens,
                                   const int32_t* parent, const int32_t* n_nodes,
                                   const int32_t* budget, int32_t eos, int32_t* argmax,
                                   int32_t* verified, int32_t* ids, int32_t* len, void* workspace,
                                   st_dtype dtype, int Hkv, int D, int64_t Lmax, int n_layers,
                                   int64_t layer_stride, const int32_t* prefix_len,
                                   int32_t* new_prefix_len, const void* k_tree,
                                   const void* v_tree, int64_t tree_layer_stride, void* k_cache,
                                   void* v_cache, void* stream, int early) {
    if (st_status e = st::require_device()) return e;
    ST_CHECK_ARG(B >= 0 && T >= 1 && V >= 1 && Hkv >= 1 && D >= 1 && n_layers >= 1,
                 ST_ERR_SHAPE_MISMATCH, "bad shape");
    ST_CHECK_ARG(st::dtype_size(dtype) != 0, ST_ERR_INVALID_ARGUMENT, "bad dtype");
    if (B == 0) return ST_OK;
    ST_CHECK_ARG(logits && tokens && parent && n_nodes && verified && ids && len && workspace &&
                     prefix_len && k_cache && v_cache,
                 ST_ERR_INVALID_ARGUMENT, "null pointer");
    ST_CHECK_ARG(new_prefix_len != prefix_len, ST_ERR_INVALID_ARGUMENT,
                 "new_prefix_len must not alias prefix_len");
    ST_CHECK_ARG((k_tree == nullptr) == (v_tree == nullptr), ST_ERR_INVALID_ARGUMENT,
                 "k_tree and v_tree must be both set or both NULL");
    ST_CHECK_ARG(B <= 65535 && T <= st::kWalkMax, ST_ERR_SHAPE_MISMATCH,
                 "B <= 65535 and T <= 1024 (use st_verify_greedy + st_kv_compact)");
    ST_CHECK_ARG((reinterpret_cast<uintptr_t>(workspace) & 7) == 0, ST_ERR_INVALID_ARGUMENT,
                 "workspace must be 8-byte aligned");
    const int64_t row_bytes = (int64_t)D * st::dtype_size(dtype);
    ST_CHECK_ARG(row_bytes % 16 == 0, ST_ERR_SHAPE_MISMATCH, "D * sizeof(dtype) must be a multiple of 16");
    unsigned long long* keys = reinterpret_cast<unsigned long long*>(workspace);
    auto strm = st::as_stream(stream);
    // argmax, then the compaction kernel, every block of which repeats its
    // request's walk (measured: fusing the walk into the argmax kernel's last
    // block instead costs 1.8 us per C2 step here — the compaction has to
    // follow as a kernel anyway, so it only lengthens the argmax tail)
    const st::WalkArgs none{};
    ST_CUDA_TRY(st::launch_pdl(st::greedy_argmax_kernel, dim3(st::kSplit, T, B), dim3(st::kThreads), 0,
                               strm, logits, T, V, n_nodes, keys, none, early));
    ST_LAUNCH_CHECK();
    // heads per block: about 2 KB of K+V per accepted row per block
    const int row_vecs = (int)(row_bytes / 16);
    const int hpb = std::max(1, std::min(Hkv, 64 / row_vecs));
    const int nhc = (Hkv + hpb - 1) / hpb;
    ST_CHECK_ARG((int64_t)n_layers * nhc <= 65535, ST_ERR_SHAPE_MISMATCH, "too many layers x heads");
    const int64_t es = (int64_t)st::dtype_size(dtype);
    ST_CUDA_TRY(st::launch_pdl(st::walk_compact_kernel<int4>, dim3(B, n_layers * nhc),
                               dim3(st::kWcThreads), 0, strm, T, tokens, parent, n_nodes, budget,
                               eos, argmax, (const unsigned long long*)keys, verified, ids, len,
                               (char*)k_cache, (char*)v_cache, Hkv, row_vecs, Lmax, nhc, hpb,
                               layer_stride * es, prefix_len, new_prefix_len,
                               (const char*)k_tree, (const char*)v_tree, tree_layer_stride * es, 0));
    ST_LAUNCH_CHECK();
    return ST_OK;
}

st_status st_verify_greedy_compact(const float* logits, int B, int T, int V, const int32_t* tokens,
                                   const int32_t* parent, const int32_t* n_nodes,
                                   const int32_t* budget, int32_t eos, int32_t* argmax,
                                   int32_t* verified, int32_t* ids, int32_t* len, void* workspace,
                                   st_dtype dtype, int Hkv, int D, int64_t Lmax, int n_layers,
                                   int64_t layer_stride, const int32_t* prefix_len,
                                   int32_t* new_prefix_len, const void* k_tree,
                                   const void* v_tree, int64_t tree_layer_stride, void* k_cache,
                                   void* v_cache, void* stream) {
    return verify_greedy_compact_impl(logits, B, T, V, tokens, parent, n_nodes, budget, eos, argmax,
                                      verified, ids, len, workspace, dtype, Hkv, D, Lmax, n_layers,
                                      layer_stride, prefix_len, new_prefix_len, k_tree, v_tree,
                                      tree_layer_stride, k_cache, v_cache, stream, 0);
}

st_status st_verify_outputs(const int32_t* outputs, int B, int T, const int32_t* tokens,
                            const int32_t* parent, const int32_t* n_nodes, const int32_t* budget,
                            int32_t eos, int32_t* verified, int32_t* ids, int32_t* len,
                            void* stream) {
    if (st_status e = st::require_device()) return e;
    ST_CHECK_ARG(B >= 0 && T >= 1, ST_ERR_SHAPE_MISMATCH, "bad shape");
    if (B == 0) return ST_OK;
    ST_CHECK_ARG(outputs && tokens && parent && n_nodes && verified && ids && len,
                 ST_ERR_INVALID_ARGUMENT, "null pointer");
    st::walk_kernel<<<B, 32, 0, st::as_stream(stream)>>>(outputs, T, tokens, parent, n_nodes,
                                                         budget, eos, verified, ids, len);
    ST_LAUNCH_CHECK();
    return ST_OK;
}

static st_status build_masks(const int32_t* parent, const int32_t* n_nodes, int B, int T, int W,
                             uint64_t* mask, int early, void* stream) {
    if (st_status e = st::require_device()) return e;
    ST_CHECK_ARG(B >= 0 && T >= 1 && W >= (T + 63) / 64 && W <= 32, ST_ERR_SHAPE_MISMATCH,
                 "bad shape (need ceil(T/64) <= W <= 32)");
    if (B == 0) return ST_OK;
    ST_CHECK_ARG(parent && n_nodes && mask, ST_ERR_INVALID_ARGUMENT, "null pointer");
    const dim3 grid((T + 127) / 128, B);
    const size_t smem = (size_t)std::min(T, 128 * (int)grid.x) * sizeof(int32_t);
    ST_CUDA_TRY(st::launch_pdl(st::build_masks_kernel, grid, dim3(128), smem, st::as_stream(stream),
                               parent, n_nodes, T, W, mask, early));
    ST_LAUNCH_CHECK();
    return ST_OK;
}

st_status st_build_masks(const int32_t* parent, const int32_t* n_nodes, int B, int T, int W,
                         uint64_t* mask, void* stream) {
    return build_masks(parent, n_nodes, B, T, W, mask, 0, stream);
}

st_status st_build_masks_early(const int32_t* parent, const int32_t* n_nodes, int B, int T, int W,
                               uint64_t* mask, void* stream) {
    return build_masks(parent, n_nodes, B, T, W, mask, 1, stream);
}

}  // extern "C"

namespace st {
st_status verify_greedy_compact_early(const float* logits, int B, int T, int V, const int32_t* tokens,
                                   const int32_t* parent, const int32_t* n_nodes,
                                   const int32_t* budget, int32_t eos, int32_t* argmax,
                                   int32_t* verified, int32_t* ids, int32_t* len, void* workspace,
                                   st_dtype dtype, int Hkv, int D, int64_t Lmax, int n_layers,
                                   int64_t layer_stride, const int32_t* prefix_len,
                                   int32_t* new_prefix_len, const void* k_tree,
                                   const void* v_tree, int64_t tree_layer_stride, void* k_cache,
                                   void* v_cache, void* stream) {
    return verify_greedy_compact_impl(logits, B, T, V, tokens, parent, n_nodes, budget, eos, argmax,
                                      verified, ids, len, workspace, dtype, Hkv, D, Lmax, n_layers,
                                      layer_stride, prefix_len, new_prefix_len, k_tree, v_tree,
                                      tree_layer_stride, k_cache, v_cache, stream, 1);
}
}  // namespace st
