// K1, CUDA-core instantiation: masked one-pass tree attention for any element
// type (f64 / f32 / f16 / bf16) with f64 accumulation for f64 and f32
// accumulation otherwise.
//
// This is the parity kernel (f64 reproduces the reference's <=1e-9 logits,
// reference proj/tests/transformer_test.cpp:335-399) and the small-tree path
// (T x G too small for tensor cores to pay). One warp owns one
// (request b, head h, node u): lanes split the visible rows 32 at a time for
// the scores, an online softmax keeps (m, l) per warp, and lanes split the
// head dimension for the P.V accumulation. Masked rows are skipped, so they
// contribute exactly +0 (reference transformer.hpp:13-16), and the reduction
// order depends only on (P, n, D) — outputs are bitwise reproducible and
// independent of non-ancestor rows (reference transformer_test.cpp:401-423).
#include <cfloat>
#include <cmath>

#include "common.cuh"
#include "tree_attn.h"

namespace st {
namespace {

template <class A> __device__ __forceinline__ A neg_inf();
template <> __device__ __forceinline__ float neg_inf<float>() { return -INFINITY; }
template <> __device__ __forceinline__ double neg_inf<double>() { return -INFINITY; }

__device__ __forceinline__ float exp_acc(float x) { return expf(x); }
__device__ __forceinline__ double exp_acc(double x) { return exp(x); }
__device__ __forceinline__ float log_acc(float x) { return logf(x); }
__device__ __forceinline__ double log_acc(double x) { return log(x); }

template <class A> __device__ __forceinline__ A warp_max(A v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}
template <class A> __device__ __forceinline__ A warp_sum(A v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}

constexpr int kWarps = 4;

template <class T, int DPL>
__global__ void __launch_bounds__(32 * kWarps)
tree_attn_cc_kernel(const T* __restrict__ q, const T* __restrict__ kc, const T* __restrict__ vc,
                    const uint64_t* __restrict__ mask, const int32_t* __restrict__ prefix_len,
                    const int32_t* __restrict__ n_nodes, T* __restrict__ o, float* __restrict__ lse,
                    int B, int T_, int H, int Hkv, int D, int W, int64_t Lmax, double scale_d,
                    const T* __restrict__ kt, const T* __restrict__ vt, int Tq, int u0) {
    using A = typename acc_of<T>::type;
    __shared__ A qs[kWarps][32 * DPL];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int64_t item = (int64_t)blockIdx.x * kWarps + warp;
    if (item >= (int64_t)B * Tq * H) return;
    // Q row r of the Tq-row slice is tree node u = u0 + r (u0 = 0, Tq = T: all nodes)
    const int h = (int)(item % H);
    const int r = (int)((item / H) % Tq);
    const int u = u0 + r;
    const int b = (int)(item / ((int64_t)H * Tq));
    const int n = n_nodes[b];
    if (u >= n) return;
    const int P = prefix_len[b];
    const int hk = h / (H / Hkv);
    const A scale = (A)scale_d;

    const T* qrow = q + (((int64_t)b * Tq + r) * H + h) * D;
    for (int d = lane; d < 32 * DPL; d += 32) qs[warp][d] = d < D ? to_acc<A>(qrow[d]) : (A)0;
    __syncwarp();

    const uint64_t* mu = mask + ((int64_t)b * T_ + u) * W;
    const T* kb = kc + ((int64_t)b * Hkv + hk) * Lmax * D;
    const T* vb = vc + ((int64_t)b * Hkv + hk) * Lmax * D;
    const int rows = P + n;
    // kv row r: cache row r, or (k_tree mode) tree node r - P of [B][T][Hkv][D]
    auto row_of = [&](const T* cache, const T* tree, int r) -> const T* {
        if (tree && r >= P) return tree + (((int64_t)b * T_ + (r - P)) * Hkv + hk) * D;
        return cache + (int64_t)r * D;
    };

    A m = neg_inf<A>(), l = (A)0;
    A acc[DPL];
#pragma unroll
    for (int i = 0; i < DPL; ++i) acc[i] = (A)0;

    for (int r0 = 0; r0 < rows; r0 += 32) {
        const int r = r0 + lane;
        bool vis = r < rows;
        if (vis && r >= P) {
            const int v = r - P;
            vis = (mu[v >> 6] >> (v & 63)) & 1ull;
        }
        A s = neg_inf<A>();
        if (vis) {
            const T* kr = row_of(kb, kt, r);
            A dot = (A)0;
            for (int d = 0; d < D; ++d) dot += qs[warp][d] * to_acc<A>(kr[d]);
            s = dot * scale;
        }
        const A mx = warp_max(s);
        const A m_new = fmax(m, mx);
        if (m_new == neg_inf<A>()) continue;  // nothing visible yet (warp-uniform)
        const A alpha = (m == neg_inf<A>()) ? (A)0 : exp_acc(m - m_new);
        const A p = vis ? exp_acc(s - m_new) : (A)0;
        l = l * alpha + warp_sum(p);
#pragma unroll
        for (int i = 0; i < DPL; ++i) acc[i] *= alpha;
        unsigned live = __ballot_sync(0xffffffffu, p != (A)0);
        while (live) {
            const int j = __ffs(live) - 1;
            live &= live - 1;
            const A pj = __shfl_sync(0xffffffffu, p, j);
            const T* vr = row_of(vb, vt, r0 + j);
#pragma unroll
            for (int i = 0; i < DPL; ++i) {
                const int d = lane + 32 * i;
                if (d < D) acc[i] += pj * to_acc<A>(vr[d]);
            }
        }
        m = m_new;
    }

    T* orow = o + (((int64_t)b * Tq + r) * H + h) * D;
    const A inv = (A)1 / l;
#pragma unroll
    for (int i = 0; i < DPL; ++i) {
        const int d = lane + 32 * i;
        if (d < D) {
            if constexpr (sizeof(A) == 8) orow[d] = from_acc_d<T>(acc[i] * inv);
            else orow[d] = from_acc<T>(acc[i] * inv);
        }
    }
    if (lse && lane == 0) lse[((int64_t)b * H + h) * Tq + r] = (float)(m + log_acc(l));
}

template <class T>
st_status launch_cc(const st_attn_args* a, cudaStream_t s) {
    const int Tq = a->q_rows > 0 ? a->q_rows : a->T, u0 = a->q_rows > 0 ? a->q_node0 : 0;
    const int64_t items = (int64_t)a->B * Tq * a->H;
    const unsigned grid = (unsigned)((items + kWarps - 1) / kWarps);
    if (grid == 0) return ST_OK;
    const int dpl = (a->D + 31) / 32;
#define ST_CC_LAUNCH(N)                                                                       \
    tree_attn_cc_kernel<T, N><<<grid, 32 * kWarps, 0, s>>>(                                  \
        (const T*)a->q, (const T*)a->k_cache, (const T*)a->v_cache, a->mask, a->prefix_len, \
        a->n_nodes, (T*)a->o, a->lse, a->B, a->T, a->H, a->Hkv, a->D, a->W, a->Lmax, a->scale, \
        (const T*)a->k_tree, (const T*)a->v_tree, Tq, u0)
    if (dpl <= 1) ST_CC_LAUNCH(1);
    else if (dpl <= 2) ST_CC_LAUNCH(2);
    else if (dpl <= 4) ST_CC_LAUNCH(4);
    else if (dpl <= 8) ST_CC_LAUNCH(8);
    else if (dpl <= 16) ST_CC_LAUNCH(16);
    else if (dpl <= 32) ST_CC_LAUNCH(32);
    else {
        set_error("st_tree_attention: head dim > 1024 unsupported");
        return ST_ERR_UNSUPPORTED;
    }
#undef ST_CC_LAUNCH
    ST_LAUNCH_CHECK();
    return ST_OK;
}

}  // namespace

st_status tree_attention_cc(const st_attn_args* a, cudaStream_t s) {
    ST_DISPATCH_DTYPE(a->dtype, T, return launch_cc<T>(a, s));
    return ST_OK;
}

}  // namespace st
