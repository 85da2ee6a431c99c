// Device-resident half-precision decoder (the reference recipe at LLaMA
// shapes: "batched around-path GEMMs" for the C3 full
// stack). The reference runs one f64 matvec per tree node per matrix
// (proj/src/transformer.cpp:262-319); here every projection is ONE GEMM over
// all B*T tree rows of the batch (cuBLAS — plain library GEMMs, fp32
// accumulate), and the verification hot path in between is ours: K2 append of
// the rows' K/V into the per-layer cache, K1 masked tree attention.
//
// Weights follow init_random_weights exactly (proj/src/transformer.cpp:71-114):
// every tensor is drawn from ONE UniformStream(seed) in the serialized order
// (tok, pos, per layer [ln1 g,b, wq, wk, wv, wo, ln2 g,b, w1, w2], lnf g,b,
// W_out), U(-0.08, 0.08) — generated on the device (value i is a pure function
// of (seed, i)) and rounded to the model dtype.
#include <cublas_v2.h>

#include <cmath>
#include <vector>

#include "common.cuh"

struct st_model {
    st_model_config cfg;
    st_dtype dtype;
    void* buf = nullptr;
    size_t elems = 0;
    cublasHandle_t blas = nullptr;
    void* blas_ws = nullptr;  // cuBLAS workspace: lets the heuristics pick split-K / stream-K kernels
    // element offsets into buf
    size_t tok, pos, lnf_g, lnf_b, wout;
    struct Layer {
        size_t ln1_g, ln1_b, wq, wk, wv, wo, ln2_g, ln2_b, w1, w2;
    };
    std::vector<Layer> layers;
};

namespace st {
namespace {

__device__ __forceinline__ uint64_t mix64(uint64_t z) {
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
    return z ^ (z >> 31);
}

// UniformStream(seed) value number `index` (0-based): reference rng.hpp:17-28.
__device__ __forceinline__ double uniform_at(uint64_t seed, uint64_t index, double lo, double hi) {
    const uint64_t z = mix64(seed + (index + 1) * 0x9e3779b97f4a7c15ULL);
    return lo + (hi - lo) * ((double)(z >> 11) * 0x1.0p-53);
}

template <class T>
__global__ void gen_weights_kernel(T* dst, int64_t n, uint64_t seed, uint64_t stream_offset) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x)
        dst[i] = from_acc<T>((float)uniform_at(seed, stream_offset + i, -0.08, 0.08));
}

template <class T>
__global__ void embed_kernel(const T* __restrict__ tok_emb, const T* __restrict__ pos_emb,
                             const int32_t* __restrict__ tokens, const int32_t* __restrict__ pos,
                             int d, T* __restrict__ x) {
    const int i = blockIdx.x;
    const T* te = tok_emb + (int64_t)tokens[i] * d;
    const T* pe = pos_emb + (int64_t)pos[i] * d;
    for (int c = threadIdx.x; c < d; c += blockDim.x)
        x[(int64_t)i * d + c] = from_acc<T>(to_acc<float>(te[c]) + to_acc<float>(pe[c]));
}

__device__ float block_sum(float v, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
    __syncthreads();
    if (l == 0) red[w] = v;
    __syncthreads();
    float s = 0.f;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) s += red[k];
    return s;
}

// LayerNorm (eps 1e-5, two-pass mean/variance; reference transformer.cpp:48-65), fp32 math.
template <class T>
__global__ void layernorm_kernel(const T* __restrict__ x, const T* __restrict__ g,
                                 const T* __restrict__ b, int d, T* __restrict__ out) {
    __shared__ float red[32];
    const T* xr = x + (int64_t)blockIdx.x * d;
    T* orow = out + (int64_t)blockIdx.x * d;
    float s = 0.f;
    for (int c = threadIdx.x; c < d; c += blockDim.x) s += to_acc<float>(xr[c]);
    const float mean = block_sum(s, red) / d;
    float v = 0.f;
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        const float z = to_acc<float>(xr[c]) - mean;
        v += z * z;
    }
    const float inv = rsqrtf(block_sum(v, red) / d + 1e-5f);
    for (int c = threadIdx.x; c < d; c += blockDim.x)
        orow[c] = from_acc<T>(to_acc<float>(g[c]) * (to_acc<float>(xr[c]) - mean) * inv +
                              to_acc<float>(b[c]));
}

template <class T>
__global__ void gelu_kernel(T* __restrict__ x, int64_t n) {
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const float v = to_acc<float>(x[i]);
        x[i] = from_acc<T>(0.5f * v * (1.f + erff(v * 0.70710678118654752f)));
    }
}

// 8 half-precision values <-> one 16-byte vector
template <class T> __device__ __forceinline__ void unpack8(const uint4& u, float (&f)[8]) {
    const T* h = reinterpret_cast<const T*>(&u);
#pragma unroll
    for (int k = 0; k < 8; ++k) f[k] = to_acc<float>(h[k]);
}
template <class T> __device__ __forceinline__ uint4 pack8(const float (&f)[8]) {
    uint4 u;
    T* h = reinterpret_cast<T*>(&u);
#pragma unroll
    for (int k = 0; k < 8; ++k) h[k] = from_acc<T>(f[k]);
    return u;
}

// LayerNorm with the row held in registers: 128 threads per row, 16-byte
// accesses, the reference's two passes (mean, then variance of x - mean) as
// two 4-warp reductions over registers (d % 8 == 0, d <= 8 * 128 * LN_MAXC).
constexpr int LN_THREADS = 128, LN_MAXC = 8;
__device__ __forceinline__ float ln_block_sum(float v, float* red) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    const int w = threadIdx.x >> 5;
    __syncthreads();  // red[] reuse across the two passes
    if ((threadIdx.x & 31) == 0) red[w] = v;
    __syncthreads();
    return (red[0] + red[1]) + (red[2] + red[3]);
}
template <class T, int NC>
__global__ void __launch_bounds__(LN_THREADS)
layernorm_vec_kernel(const T* __restrict__ x, const T* __restrict__ g, const T* __restrict__ b,
                     int d, T* __restrict__ out) {
    __shared__ float red[LN_THREADS / 32];
    const int nv = d >> 3;
    const uint4* xr = reinterpret_cast<const uint4*>(x + (int64_t)blockIdx.x * d);
    float v[NC][8];
    uint4 gq[NC], bq[NC];   // gamma / beta chunks, loaded with the row (no extra round trip)
    const uint4* gr = reinterpret_cast<const uint4*>(g);
    const uint4* br = reinterpret_cast<const uint4*>(b);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const int j = c * LN_THREADS + threadIdx.x;
        if (j < nv) {
            gq[c] = __ldg(gr + j);
            bq[c] = __ldg(br + j);
        }
    }
    float s = 0.f;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const int j = c * LN_THREADS + threadIdx.x;
        if (j < nv) {
            unpack8<T>(xr[j], v[c]);
#pragma unroll
            for (int k = 0; k < 8; ++k) s += v[c][k];
        }
    }
    const float mean = ln_block_sum(s, red) / d;
    float q = 0.f;
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        if (c * LN_THREADS + (int)threadIdx.x < nv) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const float z = v[c][k] - mean;
                q += z * z;
            }
        }
    }
    const float inv = rsqrtf(ln_block_sum(q, red) / d + 1e-5f);
    uint4* orow = reinterpret_cast<uint4*>(out + (int64_t)blockIdx.x * d);
#pragma unroll
    for (int c = 0; c < NC; ++c) {
        const int j = c * LN_THREADS + threadIdx.x;
        if (j < nv) {
            float gg[8], bb[8], o[8];
            unpack8<T>(gq[c], gg);
            unpack8<T>(bq[c], bb);
#pragma unroll
            for (int k = 0; k < 8; ++k) o[k] = gg[k] * (v[c][k] - mean) * inv + bb[k];
            orow[j] = pack8<T>(o);
        }
    }
}

// GELU (erf form, reference transformer.cpp:67): 0.5 v (1 + erf(v / sqrt 2)).
// 1 + erf(x) via Abramowitz & Stegun 7.1.26 (|erf error| <= 1.5e-7, far below
// the f16/bf16 output resolution), evaluated as erfc(|x|) = poly(t) e^{-x^2}
// for x < 0 so the small values of the negative tail keep their relative
// accuracy (no 1 - erf cancellation). Branch-free: 2 MUFU ops (approximate
// reciprocal and exp2, each ~2 ulp) + 7 FMAs instead of erff's branchy
// evaluation.
__device__ __forceinline__ float gelu_f(float v) {
    const float x = v * 0.70710678118654752f;
    const float a = fabsf(x);
    const float t = __fdividef(1.f, fmaf(0.3275911f, a, 1.f));  // MUFU.RCP: ~1 ulp, no Newton step
    float y = fmaf(1.061405429f, t, -1.453152027f);
    y = fmaf(y, t, 1.421413741f);
    y = fmaf(y, t, -0.284496736f);
    y = fmaf(y, t, 0.254829592f);
    y *= t * __expf(-a * a);          // erfc(|x|)
    const float one_plus_erf = x >= 0.f ? 2.f - y : y;
    return 0.5f * v * one_plus_erf;
}

// GELU in place, 8 values per 16-byte access; each thread keeps GELU_ILP
// independent loads in flight before its stores (in place, so the compiler
// cannot hoist the next load over the previous store by itself).
constexpr int GELU_ILP = 4;
template <class T>
__global__ void gelu_vec_kernel(uint4* __restrict__ x, int64_t n8) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i0 = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i0 < n8;
         i0 += stride * GELU_ILP) {
        uint4 u[GELU_ILP];
#pragma unroll
        for (int r = 0; r < GELU_ILP; ++r)
            if (i0 + r * stride < n8) u[r] = x[i0 + r * stride];
#pragma unroll
        for (int r = 0; r < GELU_ILP; ++r) {
            if (i0 + r * stride < n8) {
                float f[8];
                unpack8<T>(u[r], f);
#pragma unroll
                for (int k = 0; k < 8; ++k) f[k] = gelu_f(f[k]);
                x[i0 + r * stride] = pack8<T>(f);
            }
        }
    }
}

cudaDataType_t cuda_type(st_dtype t) { return t == ST_F16 ? CUDA_R_16F : CUDA_R_16BF; }

// Row-major C[M][N] (+)= A[M][K] * W[K][N]  (column-major view: C^T = W^T A^T)
st_status gemm(st_model* m, const void* A, size_t w_off, void* C, cudaDataType_t ctype, int M, int N,
               int K, bool accumulate, cudaStream_t s) {
    const float alpha = 1.f, beta = accumulate ? 1.f : 0.f;
    const size_t es = dtype_size(m->dtype);
    const void* W = static_cast<const char*>(m->buf) + w_off * es;
    cublasSetStream(m->blas, s);
    const cublasStatus_t st =
        cublasGemmEx(m->blas, CUBLAS_OP_N, CUBLAS_OP_N, N, M, K, &alpha, W, cuda_type(m->dtype), N,
                     A, cuda_type(m->dtype), K, &beta, C, ctype, N, CUBLAS_COMPUTE_32F,
                     CUBLAS_GEMM_DEFAULT);
    if (st != CUBLAS_STATUS_SUCCESS) {
        set_error("cublasGemmEx failed: status " + std::to_string((int)st));
        return ST_ERR_CUDA;
    }
    return ST_OK;
}

// `batch` GEMMs sharing the activation A: C_i = A W_i, W_i at w_off + i*w_stride
// elements, C_i at C + i*c_stride elements (one launch for Q/K/V).
st_status gemm_shared_a(st_model* m, const void* A, size_t w_off, size_t w_stride, void* C,
                        long long c_stride, int batch, int M, int N, int K, cudaStream_t s) {
    const float alpha = 1.f, beta = 0.f;
    const size_t es = dtype_size(m->dtype);
    const void* W = static_cast<const char*>(m->buf) + w_off * es;
    cublasSetStream(m->blas, s);
    const cublasStatus_t st = cublasGemmStridedBatchedEx(
        m->blas, CUBLAS_OP_N, CUBLAS_OP_N, N, M, K, &alpha, W, cuda_type(m->dtype), N,
        (long long)w_stride, A, cuda_type(m->dtype), K, 0, &beta, C, cuda_type(m->dtype), N,
        c_stride, batch, CUBLAS_COMPUTE_32F, CUBLAS_GEMM_DEFAULT);
    if (st != CUBLAS_STATUS_SUCCESS) {
        set_error("cublasGemmStridedBatchedEx failed: status " + std::to_string((int)st));
        return ST_ERR_CUDA;
    }
    return ST_OK;
}

template <class T>
const T* wptr(const st_model* m, size_t off) {
    return static_cast<const T*>(m->buf) + off;
}

}  // namespace
}  // namespace st

extern "C" {

st_status st_model_create(const st_model_config* cfg, uint64_t seed, st_dtype dtype,
                          st_model** out) {
    if (st_status e = st::require_device()) return e;
    ST_CHECK_ARG(cfg && out, ST_ERR_INVALID_ARGUMENT, "null pointer");
    ST_CHECK_ARG(dtype == ST_F16 || dtype == ST_BF16, ST_ERR_UNSUPPORTED,
                 "device model supports f16/bf16 (the f64 parity model is the C++ API)");
    const auto& c = *cfg;
    ST_CHECK_ARG(c.num_layers >= 1 && c.num_heads >= 1 && c.d_model >= 1 && c.vocab_size >= 2 &&
                     c.max_positions >= 1 && c.ffn_mult >= 1 && c.d_model % c.num_heads == 0,
                 ST_ERR_SHAPE_MISMATCH, "bad model config");
    auto* m = new st_model;
    m->cfg = c;
    m->dtype = dtype;
    const size_t d = c.d_model, F = (size_t)c.ffn_mult * d, V = c.vocab_size;
    size_t at = 0;
    auto take = [&](size_t n) {
        const size_t o = at;
        at += n;
        return o;
    };
    m->tok = take(V * d);
    m->pos = take((size_t)c.max_positions * d);
    for (int l = 0; l < c.num_layers; ++l) {
        st_model::Layer L;
        L.ln1_g = take(d);
        L.ln1_b = take(d);
        L.wq = take(d * d);
        L.wk = take(d * d);
        L.wv = take(d * d);
        L.wo = take(d * d);
        L.ln2_g = take(d);
        L.ln2_b = take(d);
        L.w1 = take(d * F);
        L.w2 = take(F * d);
        m->layers.push_back(L);
    }
    m->lnf_g = take(d);
    m->lnf_b = take(d);
    m->wout = take(d * V);
    m->elems = at;
    if (cudaMalloc(&m->buf, at * st::dtype_size(dtype)) != cudaSuccess) {
        cudaGetLastError();
        delete m;
        st::set_error("st_model_create: out of device memory");
        return ST_ERR_CUDA;
    }
    // the whole parameter vector IS the stream: element i = UniformStream(seed) value i
    const unsigned blocks = 148 * 8;
    if (dtype == ST_F16)
        st::gen_weights_kernel<__half><<<blocks, 256>>>((__half*)m->buf, (int64_t)at, seed, 0);
    else
        st::gen_weights_kernel<__nv_bfloat16><<<blocks, 256>>>((__nv_bfloat16*)m->buf, (int64_t)at,
                                                               seed, 0);
    constexpr size_t kBlasWs = 64ull << 20;
    if (cudaDeviceSynchronize() != cudaSuccess || cublasCreate(&m->blas) != CUBLAS_STATUS_SUCCESS ||
        cudaMalloc(&m->blas_ws, kBlasWs) != cudaSuccess ||
        cublasSetWorkspace(m->blas, m->blas_ws, kBlasWs) != CUBLAS_STATUS_SUCCESS) {
        cudaGetLastError();
        cudaFree(m->buf);
        delete m;
        st::set_error("st_model_create: init failed");
        return ST_ERR_CUDA;
    }
    *out = m;
    return ST_OK;
}

void st_model_destroy(st_model* m) {
    if (!m) return;
    if (m->blas) cublasDestroy(m->blas);
    if (m->blas_ws) cudaFree(m->blas_ws);
    if (m->buf) cudaFree(m->buf);
    delete m;
}

size_t st_model_param_count(const st_model* m) { return m ? m->elems : 0; }

void st_model_get_config(const st_model* m, st_model_config* out) {
    if (m && out) *out = m->cfg;
}

st_dtype st_model_get_dtype(const st_model* m) { return m ? m->dtype : ST_F16; }

size_t st_model_workspace_size(const st_model* m, int B, int T) {
    if (!m) return 0;
    const size_t rows = (size_t)B * T, d = m->cfg.d_model, F = (size_t)m->cfg.ffn_mult * d;
    st_attn_args a{};
    a.dtype = m->dtype;
    a.B = B;
    a.T = T;
    a.H = m->cfg.num_heads;
    a.Hkv = m->cfg.num_heads;
    a.D = (int)(d / m->cfg.num_heads);
    a.W = (T + 63) / 64;
    a.Lmax = T;
    const size_t es = st::dtype_size(m->dtype);
    return rows * (6 * d + F) * es + st_tree_attention_workspace_size(&a) + 8 * 256;
}

st_status st_model_tree_forward(st_model* m, int B, int T, const int32_t* tokens,
                                const int32_t* positions, const uint64_t* mask, int W,
                                const int32_t* prefix_len, const int32_t* n_nodes, void* k_cache,
                                void* v_cache, int64_t Lmax, float* logits, void* workspace,
                                size_t workspace_bytes, void* stream) {
    if (st_status e = st::require_device()) return e;
    ST_CHECK_ARG(m && tokens && positions && mask && prefix_len && n_nodes && k_cache && v_cache &&
                     logits && workspace,
                 ST_ERR_INVALID_ARGUMENT, "null pointer");
    ST_CHECK_ARG(B >= 1 && T >= 1 && W * 64 >= T && Lmax >= T, ST_ERR_SHAPE_MISMATCH, "bad shape");
    ST_CHECK_ARG(workspace_bytes >= st_model_workspace_size(m, B, T), ST_ERR_INVALID_ARGUMENT,
                 "workspace too small");
    const auto& c = m->cfg;
    const int rows = B * T, d = c.d_model, H = c.num_heads, Dh = d / H, F = c.ffn_mult * d;
    const size_t es = st::dtype_size(m->dtype);
    cudaStream_t s = st::as_stream(stream);
    char* ws = static_cast<char*>(workspace);
    auto take = [&](size_t bytes) {
        char* p = ws;
        ws += (bytes + 255) & ~size_t(255);
        return (void*)p;
    };
    void* x = take((size_t)rows * d * es);
    void* h = take((size_t)rows * d * es);
    void* q = take((size_t)rows * d * es);
    void* kn = take((size_t)rows * d * es);
    void* vn = take((size_t)rows * d * es);
    void* o = take((size_t)rows * d * es);
    void* f = take((size_t)rows * F * es);
    st_attn_args a{};
    a.dtype = m->dtype;
    a.B = B;
    a.T = T;
    a.H = H;
    a.Hkv = H;
    a.D = Dh;
    a.W = W;
    a.Lmax = Lmax;
    a.mask = mask;
    a.prefix_len = prefix_len;
    a.n_nodes = n_nodes;
    a.scale = 1.0 / std::sqrt((double)Dh);
    a.workspace = ws;
    a.workspace_bytes = st_tree_attention_workspace_size(&a);
    // K1's predecessor is the layer's K2 append (tree rows [P, P+n) only): the
    // committed rows and the lengths are stable, so K1 may stream them early
    a.early_kv = 1;
    const size_t layer_elems = (size_t)B * H * Lmax * Dh;
    const cudaDataType_t ht = st::cuda_type(m->dtype);

#define ST_M_DISPATCH(...)                                                   \
    if (m->dtype == ST_F16) {                                                \
        using T = __half;                                                    \
        __VA_ARGS__;                                                         \
    } else {                                                                 \
        using T = __nv_bfloat16;                                             \
        __VA_ARGS__;                                                         \
    }
    ST_M_DISPATCH(st::embed_kernel<T><<<rows, 256, 0, s>>>(st::wptr<T>(m, m->tok),
                                                           st::wptr<T>(m, m->pos), tokens,
                                                           positions, d, (T*)x));
    ST_LAUNCH_CHECK();
    auto aligned16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
    // LayerNorm of x into h: register-resident vector kernel when the shapes allow
    auto layernorm = [&](size_t g_off, size_t b_off) -> st_status {
        ST_M_DISPATCH(
            const T* gp = st::wptr<T>(m, g_off); const T* bp = st::wptr<T>(m, b_off);
            if (d % 8 == 0 && d <= 8 * st::LN_THREADS * st::LN_MAXC && aligned16(gp) &&
                aligned16(bp) && aligned16(x) && aligned16(h)) {
                const int nc = (d / 8 + st::LN_THREADS - 1) / st::LN_THREADS;
                auto* kern = nc <= 1 ? st::layernorm_vec_kernel<T, 1>
                             : nc <= 2 ? st::layernorm_vec_kernel<T, 2>
                             : nc <= 4 ? st::layernorm_vec_kernel<T, 4>
                                       : st::layernorm_vec_kernel<T, 8>;
                kern<<<rows, st::LN_THREADS, 0, s>>>((const T*)x, gp, bp, d, (T*)h);
            } else {
                st::layernorm_kernel<T><<<rows, 256, 0, s>>>((const T*)x, gp, bp, d, (T*)h);
            });
        ST_LAUNCH_CHECK();
        return ST_OK;
    };
    for (int l = 0; l < c.num_layers; ++l) {
        const auto& L = m->layers[l];
        void* kc = static_cast<char*>(k_cache) + (size_t)l * layer_elems * es;
        void* vc = static_cast<char*>(v_cache) + (size_t)l * layer_elems * es;
        if (st_status e = layernorm(L.ln1_g, L.ln1_b)) return e;
        const size_t dd = (size_t)d * d;
        const long long qkv_stride = (static_cast<char*>(kn) - static_cast<char*>(q)) / (long long)es;
        if (L.wk == L.wq + dd && L.wv == L.wk + dd &&
            static_cast<char*>(vn) - static_cast<char*>(kn) == qkv_stride * (long long)es) {
            // wq|wk|wv are consecutive in the serialized order: one batched launch
            if (st_status e = st::gemm_shared_a(m, h, L.wq, dd, q, qkv_stride, 3, rows, d, d, s))
                return e;
        } else {
            if (st_status e = st::gemm(m, h, L.wq, q, ht, rows, d, d, false, s)) return e;
            if (st_status e = st::gemm(m, h, L.wk, kn, ht, rows, d, d, false, s)) return e;
            if (st_status e = st::gemm(m, h, L.wv, vn, ht, rows, d, d, false, s)) return e;
        }
        if (st_status e = st_kv_append(m->dtype, B, T, H, Dh, Lmax, kn, vn, prefix_len, n_nodes, kc,
                                       vc, stream))
            return e;
        a.q = q;
        a.k_cache = kc;
        a.v_cache = vc;
        a.o = o;
        if (st_status e = st_tree_attention(&a, stream)) return e;
        if (st_status e = st::gemm(m, o, L.wo, x, ht, rows, d, d, true, s)) return e;
        if (st_status e = layernorm(L.ln2_g, L.ln2_b)) return e;
        if (st_status e = st::gemm(m, h, L.w1, f, ht, rows, F, d, false, s)) return e;
        const int64_t nf = (int64_t)rows * F;
        if (nf % 8 == 0 && aligned16(f)) {
            ST_M_DISPATCH(st::gelu_vec_kernel<T><<<148 * 8, 256, 0, s>>>((uint4*)f, nf / 8));
        } else {
            ST_M_DISPATCH(st::gelu_kernel<T><<<148 * 8, 256, 0, s>>>((T*)f, nf));
        }
        ST_LAUNCH_CHECK();
        if (st_status e = st::gemm(m, f, L.w2, x, ht, rows, d, F, true, s)) return e;
    }
    if (st_status e = layernorm(m->lnf_g, m->lnf_b)) return e;
#undef ST_M_DISPATCH
    return st::gemm(m, h, m->wout, logits, CUDA_R_32F, rows, c.vocab_size, d, false, s);
}

}  // extern "C"
