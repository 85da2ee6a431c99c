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
// Work split: one 256-thread block per (request, node) streams that node's
// logits row once (HBM-bound: 4*V bytes per node, float4 loads, 8 in flight
// per thread); the last block of a request to finish (atomic ticket, reset by
// the walker so the workspace is reusable) runs the walk with one warp:
// children of u are the ids v > u with parent[v] == u, scanned 32 at a time
// with a ballot.
#include <cfloat>

#include "common.cuh"

namespace st {
namespace {

constexpr int kThreads = 256;

struct ArgBest {
    float v;
    int i;
};

// a "beats" b under first-index-of-max ordering (NaN already mapped to -inf).
__device__ __forceinline__ bool beats(float av, int ai, float bv, int bi) {
    return av > bv || (av == bv && ai < bi);
}

__device__ __forceinline__ float sanitize(float x) { return x != x ? -INFINITY : x; }

// Alg.-2 walk (reference token_tree.cpp:153-175) + engine truncation
// (engine.cpp:110-121) for request b, executed by one full warp. `outs` holds
// the per-node LLM outputs [B][T]; read through L2 when written by other CTAs.
__device__ void walk_warp(const int32_t* outs, const int32_t* __restrict__ tokens,
                          const int32_t* __restrict__ parent, int n, int T, int b,
                          const int32_t* __restrict__ budget, int32_t eos,
                          int32_t* __restrict__ verified, int32_t* __restrict__ ids,
                          int32_t* __restrict__ len, int lane, bool coherent) {
    const int32_t* tok = tokens + (int64_t)b * T;
    const int32_t* par = parent + (int64_t)b * T;
    const int32_t* am = outs + (int64_t)b * T;
    int32_t* vrow = verified + (int64_t)b * (T + 1);
    int32_t* irow = ids + (int64_t)b * (T + 1);
    int cur = 0, m = 0;
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
    if (lane == 0) {
        vrow[m] = coherent ? __ldcg(am + cur) : am[cur];  // bonus token
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
    const int b = blockIdx.x;
    walk_warp(outs, tokens, parent, n_nodes[b], T, b, budget, eos, verified, ids, len,
              threadIdx.x & 31, false);
}

__global__ void __launch_bounds__(kThreads)
greedy_verify_kernel(const float* __restrict__ logits, int T, int V,
                     const int32_t* __restrict__ tokens, const int32_t* __restrict__ parent,
                     const int32_t* __restrict__ n_nodes, const int32_t* __restrict__ budget,
                     int32_t eos, int32_t* __restrict__ argmax_out, int32_t* argmax_ws,
                     int32_t* __restrict__ verified, int32_t* __restrict__ ids,
                     int32_t* __restrict__ len, unsigned* tickets) {
    const int u = blockIdx.x, b = blockIdx.y;
    const int n = n_nodes[b];
    if (u >= n) return;
    const float* row = logits + ((int64_t)b * T + u) * V;

    // ---- argmax over the row (first index of the maximum) ----
    float bv = -INFINITY;
    int bi = 0x7fffffff;
    const bool aligned = ((reinterpret_cast<uintptr_t>(row) & 15) == 0);
    int i0 = 0;
    if (aligned) {
        const int nv = V >> 2;
        const float4* r4 = reinterpret_cast<const float4*>(row);
        constexpr int U = 8;
        for (int base = threadIdx.x; base < nv; base += kThreads * U) {
            float4 x[U];
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int j = base + k * kThreads;
                x[k] = j < nv ? __ldg(r4 + j) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
            }
#pragma unroll
            for (int k = 0; k < U; ++k) {
                const int j = (base + k * kThreads) * 4;
                if (j < V) {
                    const float e0 = sanitize(x[k].x), e1 = sanitize(x[k].y), e2 = sanitize(x[k].z),
                                e3 = sanitize(x[k].w);
                    if (beats(e0, j, bv, bi)) { bv = e0; bi = j; }
                    if (beats(e1, j + 1, bv, bi)) { bv = e1; bi = j + 1; }
                    if (beats(e2, j + 2, bv, bi)) { bv = e2; bi = j + 2; }
                    if (beats(e3, j + 3, bv, bi)) { bv = e3; bi = j + 3; }
                }
            }
        }
        i0 = nv * 4;
    }
    for (int j = i0 + threadIdx.x; j < V; j += kThreads) {
        const float e = sanitize(row[j]);
        if (beats(e, j, bv, bi)) { bv = e; bi = j; }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const float ov = __shfl_xor_sync(0xffffffffu, bv, o);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
        if (beats(ov, oi, bv, bi)) { bv = ov; bi = oi; }
    }
    __shared__ ArgBest red[kThreads / 32];
    __shared__ bool is_last;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[warp] = {bv, bi};
    __syncthreads();
    if (threadIdx.x == 0) {
        ArgBest best = red[0];
        for (int w = 1; w < kThreads / 32; ++w)
            if (beats(red[w].v, red[w].i, best.v, best.i)) best = red[w];
        // reference rule: a NaN at index 0 is never replaced.
        const float x0 = row[0];
        int arg = (x0 != x0) ? 0 : best.i;
        if (arg == 0x7fffffff) arg = 0;  // all entries NaN-mapped: index 0
        argmax_ws[(int64_t)b * T + u] = arg;
        if (argmax_out) argmax_out[(int64_t)b * T + u] = arg;
        __threadfence();
        const unsigned t = atomicAdd(&tickets[b], 1u);
        is_last = (t == (unsigned)n - 1);
    }
    __syncthreads();
    if (!is_last || warp != 0) return;

    // ---- Alg.-2 walk by the last block of request b (one warp) ----
    __threadfence();
    walk_warp(argmax_ws, tokens, parent, n, T, b, budget, eos, verified, ids, len, lane, true);
    if (lane == 0) tickets[b] = 0;  // reusable workspace
}

// One thread per (request, node): walk the parent chain (depth <= T) and set
// the ancestor-or-self bits; no inter-thread dependency, one launch per batch.
__global__ void build_masks_kernel(const int32_t* __restrict__ parent,
                                   const int32_t* __restrict__ n_nodes, int T, int W,
                                   uint64_t* __restrict__ mask) {
    const int b = blockIdx.y;
    const int u = blockIdx.x * blockDim.x + threadIdx.x;
    if (u >= T) return;
    const int n = n_nodes[b];
    const int32_t* par = parent + (int64_t)b * T;
    uint64_t* mu = mask + ((int64_t)b * T + u) * W;
    uint64_t w[32];
#pragma unroll
    for (int i = 0; i < 32; ++i) w[i] = 0;
    if (u < n) {
        for (int v = u; v >= 0; v = par[v]) w[v >> 6] |= 1ull << (v & 63);
    }
#pragma unroll
    for (int i = 0; i < 32; ++i)
        if (i < W) mu[i] = w[i];
}

}  // namespace
}  // namespace st

extern "C" {

size_t st_verify_workspace_size(int B, int T) {
    // tickets [B] + argmax scratch [B][T]
    return (size_t)B * sizeof(unsigned) + (size_t)B * T * sizeof(int32_t) + 256;
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
    unsigned* tickets = reinterpret_cast<unsigned*>(workspace);
    int32_t* scratch = reinterpret_cast<int32_t*>(
        (reinterpret_cast<uintptr_t>(tickets + B) + 15) & ~uintptr_t(15));
    const dim3 grid(T, B);
    st::greedy_verify_kernel<<<grid, st::kThreads, 0, st::as_stream(stream)>>>(
        logits, T, V, tokens, parent, n_nodes, budget, eos, argmax, scratch, verified, ids, len,
        tickets);
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
    st::build_masks_kernel<<<grid, 128, 0, st::as_stream(stream)>>>(parent, n_nodes, T, W, mask);
    ST_LAUNCH_CHECK();
    return ST_OK;
}

}  // extern "C"
