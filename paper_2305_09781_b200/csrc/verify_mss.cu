// K4: stochastic multi-step speculative sampling (MSS) — SpecInfer's
// stochastic verification, which the reference does NOT implement
// (SPEC.md:8, :100). Contract: DESIGN.md §5 / SURVEY.md Appendix B; the fp32
// CPU oracle oracle/restate_mss.c fixes every rounding step, and this kernel
// reproduces it bit for bit given the same host-supplied uniforms:
//
//   u = root
//   loop: p = softmax(z[u] / tau)
//         for each child v of u (ascending id): r = U[k++]
//             accept if r * q_v[t_v] <= p[t_v]      -> emit t_v, u = v, continue loop
//             else p = norm(max(p - q_v, 0))        (residual renormalisation)
//         emit inverse-CDF sample of p with r = U[k++]; stop
//
// One 1024-thread block per request keeps the working distribution p[V] in
// shared memory. Every vocabulary reduction uses the fixed order of the
// contract: chunk owner t (threads 0..255) sums the contiguous chunk
// [t*CH, (t+1)*CH) sequentially, warps 0..7 combine their 32 chunk sums with an
// xor butterfly and the 8 warp sums are added in order; the exponential is the
// contract's exp_spec (fma Horner polynomial + exact power-of-two scaling); all
// fp32 operations use explicit _rn intrinsics so nothing is contracted.
// Element-wise passes (exp, normalisation, max) use all 1024 threads, and
// every global read is batched (16-32 independent loads in flight per thread)
// so a vocabulary pass costs a few memory round trips, not one per element.
#include <cfloat>

#include "common.cuh"

namespace st {
namespace {

constexpr int NT = 256;       // reduction lanes of the contract (chunk owners)
constexpr int NTHR = 1024;    // threads per block
constexpr int kBatch = 16;    // independent global loads in flight per thread

__device__ __forceinline__ float exp_spec(float x) {
    if (!(x > -104.0f)) return 0.0f;
    const float t = __fmul_rn(x, 1.44269504f);
    const float nf = rintf(t);
    const float f = __fsub_rn(t, nf);
    float p = 1.54035304e-4f;
    p = __fmaf_rn(p, f, 1.33335581e-3f);
    p = __fmaf_rn(p, f, 9.61812911e-3f);
    p = __fmaf_rn(p, f, 5.55041087e-2f);
    p = __fmaf_rn(p, f, 2.40226507e-1f);
    p = __fmaf_rn(p, f, 6.93147182e-1f);
    p = __fmaf_rn(p, f, 1.0f);
    const int n = (int)nf;
    if (n >= -126) return __fmul_rn(p, __uint_as_float((uint32_t)(n + 127) << 23));
    return __fmul_rn(__fmul_rn(p, __uint_as_float((uint32_t)(n + 227) << 23)),
                     __uint_as_float((uint32_t)27 << 23));
}

// Combine the chunk owners' partials (threads 0..255; other threads pass
// anything) in the contract order; result broadcast to all threads.
__device__ float combine_spec(float part, float* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) part = __fadd_rn(part, __shfl_xor_sync(0xffffffffu, part, o));
    __syncthreads();
    if (lane == 0 && warp < NT / 32) red[warp] = part;
    __syncthreads();
    float tot = red[0];
#pragma unroll
    for (int w = 1; w < NT / 32; ++w) tot = __fadd_rn(tot, red[w]);
    return tot;
}

// max over all threads (exact and order-independent)
__device__ float block_max(float v, float* red) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    __syncthreads();
    if (lane == 0) red[warp] = v;
    __syncthreads();
    float m = red[0];
#pragma unroll 4
    for (int w = 1; w < NTHR / 32; ++w) m = fmaxf(m, red[w]);
    return m;
}

// Chunk owner's sequential sum of f(p[i], g[i]) over [c0, c1), the global row g
// read kBatch elements at a time (all loads of a batch in flight).
constexpr int kChunkBatch = 32;
template <class F>
__device__ __forceinline__ float chunk_sum_g(const float* p, const float* __restrict__ g, int c0, int c1,
                                             F f) {
    float a = 0.0f;
    for (int i0 = c0; i0 < c1; i0 += kChunkBatch) {
        float x[kChunkBatch];
#pragma unroll
        for (int j = 0; j < kChunkBatch; ++j) x[j] = i0 + j < c1 ? __ldg(g + i0 + j) : 0.0f;
#pragma unroll
        for (int j = 0; j < kChunkBatch; ++j)
            if (i0 + j < c1) a = __fadd_rn(a, f(p[i0 + j], x[j]));
    }
    return a;
}

__global__ void __launch_bounds__(NTHR)
mss_kernel(const float* __restrict__ logits, const float* __restrict__ q, int T, int V,
           const int32_t* __restrict__ tokens, const int32_t* __restrict__ parent,
           const int32_t* __restrict__ n_nodes, float temperature,
           const float* __restrict__ uniforms, int n_uniforms, int32_t* __restrict__ verified,
           int32_t* __restrict__ ids, int32_t* __restrict__ len) {
    extern __shared__ float p[];  // [V], then the request's parent / token rows
    __shared__ float red[NTHR / 32];
    __shared__ float cum[NT], csum[NT];
    __shared__ int sh_pick;
    const int b = blockIdx.x, tid = threadIdx.x;
    const int n = n_nodes[b];
    const int CH = (V + NT - 1) / NT;
    const bool owner = tid < NT;  // chunk owner of the contract's reductions
    const int c0 = owner ? tid * CH : 0, c1 = owner ? min(V, c0 + CH) : 0;
    // the tree staged once: the child scan below reads it for every visited
    // node (from global memory it was one dependent round trip per node id)
    int32_t* par = reinterpret_cast<int32_t*>(p + V);
    int32_t* tok = par + T;
    for (int v = tid; v < n; v += NTHR) {
        par[v] = parent[(int64_t)b * T + v];
        tok[v] = tokens[(int64_t)b * T + v];
    }
    const float* U = uniforms + (int64_t)b * n_uniforms;
    int32_t* vrow = verified + (int64_t)b * (T + 1);
    int32_t* irow = ids + (int64_t)b * (T + 1);
    const float inv_tau = __fdiv_rn(1.0f, temperature);
    int u = 0, k = 0, m = 0;
    if (tid == 0) irow[0] = 0;

    for (;;) {
        __syncthreads();  // every reader of the previous p is done
        // ---- p = softmax(z[u] / tau) in the contract's arithmetic ----
        const float* z = logits + ((int64_t)b * T + u) * V;
        float mx = -INFINITY;
        for (int i0 = tid; i0 < V; i0 += NTHR * kBatch) {
            float x[kBatch];
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                const int i = i0 + j * NTHR;
                x[j] = i < V ? __ldg(z + i) : -INFINITY;
            }
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                const int i = i0 + j * NTHR;
                if (i < V) {
                    p[i] = x[j];
                    mx = fmaxf(mx, x[j]);
                }
            }
        }
        mx = block_max(mx, red);
        for (int i = tid; i < V; i += NTHR) p[i] = exp_spec(__fmul_rn(__fsub_rn(p[i], mx), inv_tau));
        __syncthreads();
        float a = 0.0f;
        for (int i = c0; i < c1; ++i) a = __fadd_rn(a, p[i]);
        const float S = combine_spec(a, red);
        for (int i = tid; i < V; i += NTHR) p[i] = __fdiv_rn(p[i], S);
        __syncthreads();

        // ---- children of u in ascending id order ----
        int next = -1;
        for (int v = u + 1; v < n; ++v) {
            if (par[v] != u) continue;
            const float r = U[k++];
            const int32_t t = tok[v];
            const float* qv = q + ((int64_t)b * T + v) * V;
            if (__fmul_rn(r, qv[t]) <= p[t]) {
                next = v;
                break;
            }
            const float s2 = chunk_sum_g(p, qv, c0, c1,
                                         [](float pi, float qi) { return fmaxf(__fsub_rn(pi, qi), 0.0f); });
            const float S2 = combine_spec(s2, red);
            if (S2 > 0.0f) {  // element-wise: every thread, q read kBatch at a time
                for (int i0 = tid; i0 < V; i0 += NTHR * kBatch) {
                    float x[kBatch];
#pragma unroll
                    for (int j = 0; j < kBatch; ++j) {
                        const int i = i0 + j * NTHR;
                        x[j] = i < V ? __ldg(qv + i) : 0.0f;
                    }
#pragma unroll
                    for (int j = 0; j < kBatch; ++j) {
                        const int i = i0 + j * NTHR;
                        if (i < V) p[i] = __fdiv_rn(fmaxf(__fsub_rn(p[i], x[j]), 0.0f), S2);
                    }
                }
            }
            __syncthreads();
        }
        if (next >= 0) {
            if (tid == 0) {
                vrow[m] = tok[next];
                irow[m + 1] = next;
            }
            ++m;
            u = next;
            continue;
        }

        // ---- inverse-CDF sample of p ----
        const float r = U[k++];
        float c = 0.0f;
        for (int i = c0; i < c1; ++i) c = __fadd_rn(c, p[i]);
        if (owner) csum[tid] = c;
        __syncthreads();
        if (tid == 0) {
            float run = 0.0f;
            for (int t = 0; t < NT; ++t) {
                run = __fadd_rn(run, csum[t]);
                cum[t] = run;
            }
            const float target = __fmul_rn(r, cum[NT - 1]);
            int tc = -1;
            for (int t = 0; t < NT; ++t)
                if (cum[t] > target) { tc = t; break; }
            if (tc < 0)
                for (int t = NT - 1; t >= 0; --t)
                    if (csum[t] > 0.0f) { tc = t; break; }
            int pick = 0;
            if (tc >= 0) {
                float acc = tc > 0 ? cum[tc - 1] : 0.0f;
                int last_pos = -1;
                pick = -1;
                for (int i = tc * CH; i < min(V, (tc + 1) * CH); ++i) {
                    acc = __fadd_rn(acc, p[i]);
                    if (p[i] > 0.0f) last_pos = i;
                    if (acc > target) { pick = i; break; }
                }
                if (pick < 0) pick = last_pos >= 0 ? last_pos : tc * CH;
            }
            sh_pick = pick;
        }
        __syncthreads();
        if (tid == 0) {
            vrow[m] = sh_pick;
            len[b] = m + 1;
        }
        break;
    }
}

}  // namespace
}  // namespace st

extern "C" st_status st_verify_mss(const float* logits, const float* q, int B, int T, int V,
                                   const int32_t* tokens, const int32_t* parent,
                                   const int32_t* n_nodes, float temperature,
                                   const float* uniforms, int n_uniforms, int32_t* verified,
                                   int32_t* ids, int32_t* len, void* stream) {
    if (st_status e = st::require_device()) return e;
    ST_CHECK_ARG(B >= 0 && T >= 1 && V >= 1, ST_ERR_SHAPE_MISMATCH, "bad shape");
    ST_CHECK_ARG(temperature > 0.0f, ST_ERR_INVALID_ARGUMENT, "temperature must be > 0");
    ST_CHECK_ARG(n_uniforms >= T + 1, ST_ERR_INVALID_ARGUMENT,
                 "need n_uniforms >= T + 1 (one per visited child plus the final sample)");
    if (B == 0) return ST_OK;
    ST_CHECK_ARG(logits && q && tokens && parent && n_nodes && uniforms && verified && ids && len,
                 ST_ERR_INVALID_ARGUMENT, "null pointer");
    const size_t smem = (size_t)V * sizeof(float) + 2 * (size_t)T * sizeof(int32_t);
    ST_CHECK_ARG(smem <= 200 * 1024, ST_ERR_UNSUPPORTED,
                 "vocabulary too large for K4 (V * 4 + T * 8 <= 200 KB)");
    static size_t attr_set = 0;
    if (smem > 48 * 1024 && smem > attr_set) {
        ST_CUDA_TRY(cudaFuncSetAttribute(st::mss_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)smem));
        attr_set = smem;
    }
    st::mss_kernel<<<B, st::NTHR, smem, st::as_stream(stream)>>>(logits, q, T, V, tokens, parent,
                                                               n_nodes, temperature, uniforms,
                                                               n_uniforms, verified, ids, len);
    ST_LAUNCH_CHECK();
    return ST_OK;
}
