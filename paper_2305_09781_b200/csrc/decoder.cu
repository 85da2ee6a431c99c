// Around-path decoder kernels (not among K1-K4; needed to run the reference's
// pre-LN transformer end to end for C1 and for the drop-in C++ API):
//   embedding (token + learned absolute position), LayerNorm (eps 1e-5,
//   two-pass mean/variance), row-major GEMM out(+)= A * W with a FIXED
//   ascending-k accumulation per output element (results independent of how
//   many rows are batched — the bitwise non-ancestor property needs that),
//   GELU(erf), and a row argmax for f64 logits.
// Reference recipe: proj/src/transformer.cpp:48-67 (layer_norm, gelu),
// :244-250 (embeddings), :262-319 (per-node matvecs, batched here over rows).
#include <cmath>

#include "common.cuh"
#include "decoder.h"

namespace st {
namespace {

template <class T>
__global__ void embed_kernel(const T* __restrict__ tok_emb, const T* __restrict__ pos_emb,
                             const int32_t* __restrict__ tokens, const int32_t* __restrict__ pos,
                             int d, T* __restrict__ x) {
    const int i = blockIdx.x;
    const T* te = tok_emb + (int64_t)tokens[i] * d;
    const T* pe = pos_emb + (int64_t)pos[i] * d;
    for (int c = threadIdx.x; c < d; c += blockDim.x) x[(int64_t)i * d + c] = te[c] + pe[c];
}

template <class T>
__device__ T block_sum(T v, T* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    T s = 0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[k];
    return s;
}

template <class T>
__global__ void layernorm_kernel(const T* __restrict__ x, const T* __restrict__ g,
                                 const T* __restrict__ b, int d, T* __restrict__ out) {
    __shared__ T red[32];
    const T* xr = x + (int64_t)blockIdx.x * d;
    T* orow = out + (int64_t)blockIdx.x * d;
    T s = 0;
    for (int c = threadIdx.x; c < d; c += blockDim.x) s += xr[c];
    const T mean = block_sum(s, red) / (T)d;
    T v = 0;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        const T z = xr[c] - mean;
        v += z * z;
    }
    const T var = block_sum(v, red) / (T)d;
    const T inv = (T)1 / sqrt(var + (T)1e-5);
    for (int c = threadIdx.x; c < d; c += blockDim.x) orow[c] = g[c] * (xr[c] - mean) * inv + b[c];
}

// C[M][N] (+)= A[M][K] * W[K][N]; 64x64 tile, 256 threads x 16 outputs, K
// accumulated in ascending order for every element.
template <class T, bool ACCUM>
__global__ void __launch_bounds__(256)
gemm_kernel(const T* __restrict__ A, const T* __restrict__ W, T* __restrict__ C, int M, int N,
            int K) {
    constexpr int TM = 64, TN = 64, TK = 16;
    __shared__ T As[TK][TM + 1];
    __shared__ T Ws[TK][TN];
    const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
    const int m0 = blockIdx.y * TM, n0 = blockIdx.x * TN;
    T acc[4][4];
#pragma unroll
    for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) acc[i][j] = 0;
    for (int k0 = 0; k0 < K; k0 += TK) {
        for (int e = threadIdx.x; e < TM * TK; e += 256) {
            const int mm = e / TK, kk = e % TK;
            const int gm = m0 + mm, gk = k0 + kk;
            As[kk][mm] = (gm < M && gk < K) ? A[(int64_t)gm * K + gk] : (T)0;
        }
        for (int e = threadIdx.x; e < TK * TN; e += 256) {
            const int kk = e / TN, nn = e % TN;
            const int gk = k0 + kk, gn = n0 + nn;
            Ws[kk][nn] = (gk < K && gn < N) ? W[(int64_t)gk * N + gn] : (T)0;
        }
        __syncthreads();
#pragma unroll
        for (int kk = 0; kk < TK; ++kk) {
            T a[4], w[4];
#pragma unroll
            for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
            for (int j = 0; j < 4; ++j) w[j] = Ws[kk][tx * 4 + j];
#pragma unroll
            for (int i = 0; i < 4; ++i)
#pragma unroll
                for (int j = 0; j < 4; ++j) acc[i][j] = fma(a[i], w[j], acc[i][j]);
        }
        __syncthreads();
    }
#pragma unroll
    for (int i = 0; i < 4; ++i) {
        const int gm = m0 + ty * 4 + i;
        if (gm >= M) continue;
#pragma unroll
        for (int j = 0; j < 4; ++j) {
            const int gn = n0 + tx * 4 + j;
            if (gn >= N) continue;
            T* c = C + (int64_t)gm * N + gn;
            if (ACCUM) *c += acc[i][j];
            else *c = acc[i][j];
        }
    }
}

template <class T>
__global__ void gelu_kernel(T* __restrict__ x, int64_t n) {
    const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    if (i < n) {
        const T v = x[i];
        x[i] = (T)0.5 * v * ((T)1 + erf(v * (T)0.7071067811865476));
    }
}

// First index of the row maximum, NaN never wins, NaN at 0 is kept
// (reference argmax_token, transformer.cpp:116-122).
template <class T>
__global__ void argmax_rows_kernel(const T* __restrict__ x, int V, int32_t* __restrict__ out) {
    const T* row = x + (int64_t)blockIdx.x * V;
    T bv = -INFINITY;
    int bi = 0x7fffffff;
    for (int i = threadIdx.x; i < V; i += blockDim.x) {
        T v = row[i];
        if (v != v) v = -INFINITY;
        if (v > bv || (v == bv && i < bi)) { bv = v; bi = i; }
    }
    __shared__ T sv[256];
    __shared__ int si[256];
    sv[threadIdx.x] = bv;
    si[threadIdx.x] = bi;
    __syncthreads();
    for (int s = blockDim.x / 2; s > 0; s >>= 1) {
        if (threadIdx.x < s) {
            const T ov = sv[threadIdx.x + s];
            const int oi = si[threadIdx.x + s];
            if (ov > sv[threadIdx.x] || (ov == sv[threadIdx.x] && oi < si[threadIdx.x])) {
                sv[threadIdx.x] = ov;
                si[threadIdx.x] = oi;
            }
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        const T x0 = row[0];
        out[blockIdx.x] = (x0 != x0 || si[0] == 0x7fffffff) ? 0 : si[0];
    }
}

}  // namespace

template <class T>
st_status embed(const T* tok_emb, const T* pos_emb, const int32_t* tokens, const int32_t* pos,
                int n, int d, T* x, cudaStream_t s) {
    if (n == 0) return ST_OK;
    embed_kernel<T><<<n, 128, 0, s>>>(tok_emb, pos_emb, tokens, pos, d, x);
    ST_LAUNCH_CHECK();
    return ST_OK;
}

template <class T>
st_status layernorm(const T* x, const T* g, const T* b, int n, int d, T* out, cudaStream_t s) {
    if (n == 0) return ST_OK;
    layernorm_kernel<T><<<n, 128, 0, s>>>(x, g, b, d, out);
    ST_LAUNCH_CHECK();
    return ST_OK;
}

template <class T>
st_status gemm(const T* A, const T* W, T* C, int M, int N, int K, bool accumulate, cudaStream_t s) {
    if (M == 0 || N == 0) return ST_OK;
    const dim3 grid((N + 63) / 64, (M + 63) / 64);
    if (accumulate) gemm_kernel<T, true><<<grid, 256, 0, s>>>(A, W, C, M, N, K);
    else gemm_kernel<T, false><<<grid, 256, 0, s>>>(A, W, C, M, N, K);
    ST_LAUNCH_CHECK();
    return ST_OK;
}

template <class T>
st_status gelu(T* x, int64_t n, cudaStream_t s) {
    if (n == 0) return ST_OK;
    gelu_kernel<T><<<(unsigned)((n + 255) / 256), 256, 0, s>>>(x, n);
    ST_LAUNCH_CHECK();
    return ST_OK;
}

template <class T>
st_status argmax_rows(const T* x, int rows, int V, int32_t* out, cudaStream_t s) {
    if (rows == 0) return ST_OK;
    argmax_rows_kernel<T><<<rows, 256, 0, s>>>(x, V, out);
    ST_LAUNCH_CHECK();
    return ST_OK;
}

#define ST_DECODER_INST(T)                                                                      \
    template st_status embed<T>(const T*, const T*, const int32_t*, const int32_t*, int, int, T*, \
                                cudaStream_t);                                                  \
    template st_status layernorm<T>(const T*, const T*, const T*, int, int, T*, cudaStream_t);  \
    template st_status gemm<T>(const T*, const T*, T*, int, int, int, bool, cudaStream_t);      \
    template st_status gelu<T>(T*, int64_t, cudaStream_t);                                      \
    template st_status argmax_rows<T>(const T*, int, int, int32_t*, cudaStream_t);
ST_DECODER_INST(double)
ST_DECODER_INST(float)

}  // namespace st
