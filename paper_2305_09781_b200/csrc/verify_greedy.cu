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
__device__ __forceinline__ unsigned long long arg_key(float v, int i) {
    if (v != v) {
        if (i == 0) return ~0ull;
        v = -INFINITY;
    }
    uint32_t u = __float_as_uint(v);
    u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    return ((unsigned long long)u << 32) | (uint32_t)(~(uint32_t)i);
}
__device__ __forceinline__ int key_index(unsigned long long k) {
    return k == ~0ull ? 0 : (int)(~(uint32_t)(k & 0xffffffffu));
}

constexpr int kSplit = 4;   // blocks per logits row
constexpr int kUnroll = 8;  // float4 loads in flight per thread (a 4000-float slice in one batch)

// Phase 1: stream every live node's logits once; kSplit blocks per row each
// reduce their slice to one order-preserving key and fold it in with
// atomicMax (order-independent -> deterministic). No fences or tickets.
__global__ void __launch_bounds__(kThreads)
greedy_argmax_kernel(const float* __restrict__ logits, int T, int V,
                     const int32_t* __restrict__ n_nodes, unsigned long long* keys) {
    pdl_wait();
    pdl_trigger();  // let the walk kernel get scheduled while the rows stream
    const int part = blockIdx.x, u = blockIdx.y, b = blockIdx.z;
    if (u >= n_nodes[b]) return;
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
    if (threadIdx.x == 0) {
        for (int w = 1; w < kThreads / 32; ++w) best = max(best, red[w]);
        atomicMax(keys + (int64_t)b * T + u, best);
    }
}

// Phase 2 (launched with programmatic dependent launch): one warp per request
// resolves the argmax keys (resetting them for the next call), then walks.
__global__ void __launch_bounds__(32)
greedy_walk_kernel(int T, const int32_t* __restrict__ tokens, const int32_t* __restrict__ parent,
                   const int32_t* __restrict__ n_nodes, const int32_t* __restrict__ budget,
                   int32_t eos, int32_t* __restrict__ argmax_out, unsigned long long* keys,
                   int32_t* argmax_ws, int32_t* __restrict__ verified, int32_t* __restrict__ ids,
                   int32_t* __restrict__ len) {
    pdl_wait();
    pdl_trigger();
    __shared__ int s_out[kWalkMax], s_next[kWalkMax];
    const int b = blockIdx.x, lane = threadIdx.x;
    const int n = n_nodes[b];
    int32_t* am = argmax_ws + (int64_t)b * T;
    for (int v = lane; v < n; v += 32) {
        unsigned long long* kp = keys + (int64_t)b * T + v;
        const int a = key_index(*kp);
        *kp = 0ull;  // reset for the next call
        am[v] = a;
        if (argmax_out) argmax_out[(int64_t)b * T + v] = a;
    }
    __syncwarp();
    walk_warp(argmax_ws, tokens, parent, n, T, b, budget, eos, verified, ids, len, lane, false,
              s_out, s_next);
}

// One thread per (request, node). The request's parent row is staged in
// shared memory first; the walk up the parent chain (ids strictly decrease)
// then emits the ancestor-or-self bits word by word, high word first, so no
// per-thread word array is needed (nothing spills to local memory).
__global__ void build_masks_kernel(const int32_t* __restrict__ parent,
                                   const int32_t* __restrict__ n_nodes, int T, int W,
                                   uint64_t* __restrict__ mask) {
    extern __shared__ int s_par[];
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.y;
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    const int n = n_nodes[b];
    const int upto = min(n, (int)((blockIdx.x + 1) * blockDim.x));  // nodes this block needs
    const int32_t* par = parent + (int64_t)b * T;
    for (int v = threadIdx.x; v < upto; v += blockDim.x) s_par[v] = par[v];
    __syncthreads();
    if (u >= T) return;
    uint64_t* mu = mask + ((int64_t)b * T + u) * W;
    int wi = W - 1;
    if (u < n) {
        uint64_t acc = 0;
        for (int v = u; v >= 0;) {
            const int vw = v >> 6;
            while (wi > vw) {
                mu[wi] = acc;
                acc = 0;
                --wi;
            }
            acc |= 1ull << (v & 63);
            const int pv = s_par[v];
            v = pv < v ? pv : -1;  // preorder: parent id < child id (stop on malformed input)
        }
        mu[wi] = acc;
        --wi;
    }
    for (; wi >= 0; --wi) mu[wi] = 0;
}

}  // namespace
}  // namespace st

extern "C" {

size_t st_verify_workspace_size(int B, int T) {
    // keys [B][T] u64 | tickets [B] | argmax scratch [B][T]   (zeroed once by the caller)
    return (size_t)B * T * 8 + (size_t)B * sizeof(unsigned) + (size_t)B * T * sizeof(int32_t) + 512;
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
    unsigned* tickets = reinterpret_cast<unsigned*>(keys + (size_t)B * T);
    int32_t* scratch = reinterpret_cast<int32_t*>(
        (reinterpret_cast<uintptr_t>(tickets + B) + 15) & ~uintptr_t(15));
    const dim3 grid(st::kSplit, T, B);
    auto strm = st::as_stream(stream);
    ST_CUDA_TRY(st::launch_pdl(st::greedy_argmax_kernel, grid, dim3(st::kThreads), 0, strm, logits,
                               T, V, n_nodes, keys));
    ST_LAUNCH_CHECK();
    ST_CUDA_TRY(st::launch_pdl(st::greedy_walk_kernel, dim3(B), dim3(32), 0, strm, T, tokens,
                               parent, n_nodes, budget, eos, argmax, keys, scratch, verified, ids,
                               len));
    ST_LAUNCH_CHECK();
    return ST_OK;
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

st_status st_build_masks(const int32_t* parent, const int32_t* n_nodes, int B, int T, int W,
                         uint64_t* mask, void* stream) {
    if (st_status e = st::require_device()) return e;
    ST_CHECK_ARG(B >= 0 && T >= 1 && W >= (T + 63) / 64 && W <= 32, ST_ERR_SHAPE_MISMATCH,
                 "bad shape (need ceil(T/64) <= W <= 32)");
    if (B == 0) return ST_OK;
    ST_CHECK_ARG(parent && n_nodes && mask, ST_ERR_INVALID_ARGUMENT, "null pointer");
    const dim3 grid((T + 127) / 128, B);
    const size_t smem = (size_t)std::min(T, 128 * (int)grid.x) * sizeof(int32_t);
    ST_CUDA_TRY(st::launch_pdl(st::build_masks_kernel, grid, dim3(128), smem, st::as_stream(stream),
                               parent, n_nodes, T, W, mask));
    ST_LAUNCH_CHECK();
    return ST_OK;
}

}  // extern "C"
