// Device-resident half-precision decoder (the reference recipe at LLaMA
// shapes: "batched around-path GEMMs" for the C3 full
// stack). The reference runs one f64 matvec per tree node per matrix
// (proj/src/transformer.cpp:262-319); here every projection is ONE GEMM over
// all B*T tree rows of the batch — the hand-written tcgen05 GEMM of gemm.cu,
// fp32 accumulate, with GELU (FFN-1) and the residual adds (WO, FFN-2) fused
// into its epilogue — and the verification hot path in between is ours: K2
// append of the rows' K/V into the per-layer cache, K1 masked tree attention.
//
// Weights follow init_random_weights exactly (proj/src/transformer.cpp:71-114):
// every tensor is drawn from ONE UniformStream(seed) in the serialized order
// (tok, pos, per layer [ln1 g,b, wq, wk, wv, wo, ln2 g,b, w1, w2], lnf g,b,
// W_out), U(-0.08, 0.08) — generated on the device (value i is a pure function
// of (seed, i)) and rounded to the model dtype.
#include <cmath>
#include <vector>

#include "common.cuh"
#include "gemm.h"

struct st_model {
    st_model_config cfg;
    st_dtype dtype;
    void* buf = nullptr;
    size_t elems = 0;
    void* wout_pad = nullptr;  // W_out with its row stride padded to a multiple of 8 (TMA)
    int ldw_out = 0;
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

// The embedding rows of a tree slice: row j = b * nf + r is node u0 + r of
// request b (full-tree token / position arrays [B][T]).
template <class T>
__global__ void embed_slice_kernel(const T* __restrict__ tok_emb, const T* __restrict__ pos_emb,
                                   const int32_t* __restrict__ tokens, const int32_t* __restrict__ pos,
                                   int Ttree, int u0, int nf, int d, T* __restrict__ x) {
    const int j = blockIdx.x, b = j / nf, u = u0 + (j - b * nf);
    const int32_t t = tokens[(int64_t)b * Ttree + u], p = pos[(int64_t)b * Ttree + u];
    const T* te = tok_emb + (int64_t)t * d;
    const T* pe = pos_emb + (int64_t)p * d;
    for (int c = threadIdx.x; c < d; c += blockDim.x)
        x[(int64_t)j * d + c] = from_acc<T>(to_acc<float>(te[c]) + to_acc<float>(pe[c]));
}

// Compact slice rows [B*nf][d] -> full-tree rows (b*T + u0 + r) of dst, for
// K and V at once (16-byte vectors; d % 8 == 0).
__global__ void scatter_slice_kernel(const uint4* __restrict__ k_src, const uint4* __restrict__ v_src,
                                     uint4* __restrict__ k_dst, uint4* __restrict__ v_dst, int Ttree,
                                     int u0, int nf, int row_vecs) {
    const int j = blockIdx.x, b = j / nf, u = u0 + (j - b * nf);
    const int64_t src = (int64_t)j * row_vecs, dst = ((int64_t)b * Ttree + u) * row_vecs;
    for (int c = threadIdx.x; c < row_vecs; c += blockDim.x) {
        k_dst[dst + c] = k_src[src + c];
        v_dst[dst + c] = v_src[src + c];
    }
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

// LayerNorm with one WARP per row (d = 256 * NPL): a lane holds NPL 16-byte
// chunks of its row in registers, both passes (mean, then the variance of
// x - mean, as the reference) reduce with warp shuffles only — no block
// barriers or shared memory on the row's dependency chain — and gamma / beta
// are read next to the store (L1-resident after the first rows). C3's
// d = 4096 rows (NPL = 16): 12.1 -> 9.0 us per LayerNorm over 2048 rows
// (torch.profiler, tools/c3_profile.py).
constexpr int LNW_WARPS = 8;  // rows per 256-thread block
// an opaque copy: each pass unpacks the row's halves afresh instead of the
// compiler keeping all 8 * NPL floats of the first pass live (254 registers)
__device__ __forceinline__ uint4 opaque(uint4 v) {
    asm volatile("" : "+r"(v.x), "+r"(v.y), "+r"(v.z), "+r"(v.w));
    return v;
}
__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
template <class T, int NPL>
__global__ void __launch_bounds__(LNW_WARPS * 32)
layernorm_warp_kernel(const T* __restrict__ x, const T* __restrict__ g, const T* __restrict__ b, int rows,
                      T* __restrict__ out) {
    constexpr int d = 256 * NPL;
    const int lane = threadIdx.x & 31;
    const int row = blockIdx.x * LNW_WARPS + (threadIdx.x >> 5);
    if (row >= rows) return;
    const uint4* xr = reinterpret_cast<const uint4*>(x + (int64_t)row * d);
    uint4 xv[NPL];
#pragma unroll
    for (int i = 0; i < NPL; ++i) xv[i] = __ldg(xr + lane + 32 * i);
    float s = 0.f;
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
        float f[8];
        unpack8<T>(xv[i], f);
#pragma unroll
        for (int k = 0; k < 8; ++k) s += f[k];
    }
    const float mean = warp_sum(s) / d;
    float q = 0.f;
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
        float f[8];
        unpack8<T>(opaque(xv[i]), f);
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const float z = f[k] - mean;
            q += z * z;
        }
    }
    const float inv = rsqrtf(warp_sum(q) / d + 1e-5f);
    const uint4* gr = reinterpret_cast<const uint4*>(g);
    const uint4* br = reinterpret_cast<const uint4*>(b);
    uint4* orow = reinterpret_cast<uint4*>(out + (int64_t)row * d);
#pragma unroll
    for (int i = 0; i < NPL; ++i) {
        const int j = lane + 32 * i;
        float f[8], gg[8], bb[8], o[8];
        unpack8<T>(opaque(xv[i]), f);
        unpack8<T>(__ldg(gr + j), gg);
        unpack8<T>(__ldg(br + j), bb);
#pragma unroll
        for (int k = 0; k < 8; ++k) o[k] = gg[k] * (f[k] - mean) * inv + bb[k];
        orow[j] = pack8<T>(o);
    }
}

// Row-major C[z] (op)= A W[z] on the tcgen05 GEMM (gemm.cu).
// fp32 scratch lent to the GEMM for split-K partials (small-M projections:
// the engine's drafting passes and small batches)
constexpr size_t kSplitScratch = 64ull << 20;

st_status gemm(st_model* m, const void* A, const void* W, int ldw, void* C, int ldc, int M, int N,
               int K, int Z, long long c_stride_z, int epi, cudaStream_t s, float* work) {
    GemmArgs g{m->dtype, A, K, W, ldw, C, c_stride_z, ldc, M, N, K, Z, epi};
    g.work = work;
    g.work_bytes = work ? kSplitScratch : 0;
    return gemm_sm100(g, s);
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
    ST_CHECK_ARG(c.d_model % 8 == 0, ST_ERR_UNSUPPORTED,
                 "device model needs d_model % 8 == 0 (16-byte rows for the TMA-fed GEMMs)");
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
    // the LM head's W_out [d][V]: TMA needs 16-byte row strides, so a vocabulary
    // that is not a multiple of 8 gets a copy with padded rows (zeros past V)
    m->ldw_out = (int)((V + 7) / 8 * 8);
    bool ok = cudaDeviceSynchronize() == cudaSuccess;
    if (ok && (size_t)m->ldw_out != V) {
        const size_t es = st::dtype_size(dtype);
        ok = cudaMalloc(&m->wout_pad, d * m->ldw_out * es) == cudaSuccess &&
             cudaMemset(m->wout_pad, 0, d * m->ldw_out * es) == cudaSuccess &&
             cudaMemcpy2D(m->wout_pad, m->ldw_out * es, static_cast<char*>(m->buf) + m->wout * es,
                          V * es, V * es, d, cudaMemcpyDeviceToDevice) == cudaSuccess;
    }
    if (!ok) {
        cudaGetLastError();
        if (m->wout_pad) cudaFree(m->wout_pad);
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
    if (m->wout_pad) cudaFree(m->wout_pad);
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
    return rows * (6 * d + F) * es + st_tree_attention_workspace_size(&a) + st::kSplitScratch + 9 * 256;
}

// nf > 0: the slice pass (st_model_tree_forward_slice) — only nodes
// [u0, u0 + nf) of every request go through the model (rows = B * nf), their
// K/V scattered into tree_qkv's full-tree rows before each layer's K1, which
// reads Q for the slice and the tree rows from tree_qkv (q_rows / q_node0).
static st_status tree_forward(st_model* m, int B, int T, const int32_t* tokens,
                              const int32_t* positions, const uint64_t* mask, int W,
                              const int32_t* prefix_len, const int32_t* n_nodes, void* k_cache,
                              void* v_cache, int64_t Lmax, void* tree_qkv, float* logits,
                              void* workspace, size_t workspace_bytes, void* stream, int u0 = 0,
                              int nf = 0) {
    if (st_status e = st::require_device()) return e;
    const bool slice = nf > 0;
    ST_CHECK_ARG(m && tokens && positions && mask && prefix_len && n_nodes && k_cache && v_cache &&
                     (logits || slice) && workspace && (tree_qkv || !slice),
                 ST_ERR_INVALID_ARGUMENT, "null pointer");
    ST_CHECK_ARG(B >= 1 && T >= 1 && W * 64 >= T && Lmax >= T, ST_ERR_SHAPE_MISMATCH, "bad shape");
    ST_CHECK_ARG(!slice || (u0 >= 0 && u0 + nf <= T), ST_ERR_SHAPE_MISMATCH, "bad tree slice");
    const int Tr = slice ? nf : T;   // model rows per request
    const auto& c = m->cfg;
    const int rows = B * Tr, d = c.d_model, H = c.num_heads, Dh = d / H, F = c.ffn_mult * d;
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
    if (slice) {
        a.q_rows = nf;
        a.q_node0 = u0;
    }
    a.workspace = ws;
    a.k_tree = a.v_tree = tree_qkv;  // (the path, hence the size, depends on k_tree being set)
    a.workspace_bytes = st_tree_attention_workspace_size(&a);
    ws += (a.workspace_bytes + 255) & ~size_t(255);
    float* splitk = reinterpret_cast<float*>(take(st::kSplitScratch));
    // exact need of this pass (a slice's K1 spans T nodes with q_rows = nf;
    // st_model_workspace_size(m, B, T) always covers it)
    ST_CHECK_ARG((size_t)(ws - static_cast<char*>(workspace)) <= workspace_bytes,
                 ST_ERR_INVALID_ARGUMENT, "workspace too small");
    // K1's predecessor is the layer's K2 append (tree rows [P, P+n) only) or,
    // in k_tree mode, the QKV GEMM: the committed rows and the lengths are
    // stable, so K1 may stream them early
    a.early_kv = 1;
    const size_t layer_elems = (size_t)B * H * Lmax * Dh;
    auto Wp = [&](size_t off) -> const void* { return static_cast<const char*>(m->buf) + off * es; };

#define ST_M_DISPATCH(...)                                                   \
    if (m->dtype == ST_F16) {                                                \
        using T = __half;                                                    \
        __VA_ARGS__;                                                         \
    } else {                                                                 \
        using T = __nv_bfloat16;                                             \
        __VA_ARGS__;                                                         \
    }
    const int Ttree = T;  // (the dispatch macro binds T to the element type)
    if (slice) {
        ST_M_DISPATCH(st::embed_slice_kernel<T><<<rows, 256, 0, s>>>(
            st::wptr<T>(m, m->tok), st::wptr<T>(m, m->pos), tokens, positions, Ttree, u0, nf, d, (T*)x));
    } else {
        ST_M_DISPATCH(st::embed_kernel<T><<<rows, 256, 0, s>>>(st::wptr<T>(m, m->tok),
                                                               st::wptr<T>(m, m->pos), tokens,
                                                               positions, d, (T*)x));
    }
    ST_LAUNCH_CHECK();
    auto aligned16 = [](const void* ptr) { return (reinterpret_cast<uintptr_t>(ptr) & 15) == 0; };
    // LayerNorm of x into h: register-resident vector kernel when the shapes allow
    auto layernorm = [&](size_t g_off, size_t b_off) -> st_status {
        ST_M_DISPATCH(
            const T* gp = st::wptr<T>(m, g_off); const T* bp = st::wptr<T>(m, b_off);
            const bool al = aligned16(gp) && aligned16(bp) && aligned16(x) && aligned16(h);
            const int npl = d % 256 == 0 ? d / 256 : 0;
            if (al && (npl == 1 || npl == 2 || npl == 4 || npl == 8 || npl == 16)) {
                auto* kern = npl == 1 ? st::layernorm_warp_kernel<T, 1>
                             : npl == 2 ? st::layernorm_warp_kernel<T, 2>
                             : npl == 4 ? st::layernorm_warp_kernel<T, 4>
                             : npl == 8 ? st::layernorm_warp_kernel<T, 8>
                                        : st::layernorm_warp_kernel<T, 16>;
                kern<<<(rows + st::LNW_WARPS - 1) / st::LNW_WARPS, st::LNW_WARPS * 32, 0, s>>>(
                    (const T*)x, gp, bp, rows, (T*)h);
            } else if (d % 8 == 0 && d <= 8 * st::LN_THREADS * st::LN_MAXC && al) {
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
        // tree_qkv layer l: [3][B*T][d] (Q | K | V of every tree node)
        char* tq_l = tree_qkv ? static_cast<char*>(tree_qkv) + (size_t)l * 3 * B * T * d * es : nullptr;
        char* tk_l = tq_l ? tq_l + (size_t)B * T * d * es : nullptr;
        char* tv_l = tq_l ? tk_l + (size_t)B * T * d * es : nullptr;
        if (tree_qkv && !slice) {  // k_tree mode: this layer's Q|K|V stay in the caller's buffer
            q = tq_l;
            kn = tk_l;
            vn = tv_l;
        }
        const long long qkv_stride = (static_cast<char*>(kn) - static_cast<char*>(q)) / (long long)es;
        if (L.wk == L.wq + dd && L.wv == L.wk + dd &&
            static_cast<char*>(vn) - static_cast<char*>(kn) == qkv_stride * (long long)es) {
            // wq|wk|wv are consecutive in the serialized order: one batched launch
            if (st_status e = st::gemm(m, h, Wp(L.wq), d, q, d, rows, d, d, 3, qkv_stride,
                                       st::kGemmStore, s, splitk))
                return e;
        } else {
            if (st_status e = st::gemm(m, h, Wp(L.wq), d, q, d, rows, d, d, 1, 0, st::kGemmStore, s, splitk))
                return e;
            if (st_status e = st::gemm(m, h, Wp(L.wk), d, kn, d, rows, d, d, 1, 0, st::kGemmStore, s, splitk))
                return e;
            if (st_status e = st::gemm(m, h, Wp(L.wv), d, vn, d, rows, d, d, 1, 0, st::kGemmStore, s, splitk))
                return e;
        }
        if (!tree_qkv) {
            if (st_status e = st_kv_append(m->dtype, B, T, H, Dh, Lmax, kn, vn, prefix_len, n_nodes,
                                           kc, vc, stream))
                return e;
        }
        if (slice) {  // the slice's K/V rows into the full-tree rows b*T + u0 + r
            st::scatter_slice_kernel<<<rows, 128, 0, s>>>(
                static_cast<const uint4*>(kn), static_cast<const uint4*>(vn), reinterpret_cast<uint4*>(tk_l),
                reinterpret_cast<uint4*>(tv_l), T, u0, nf, (int)((size_t)d * es / 16));
            ST_LAUNCH_CHECK();
        }
        a.q = q;
        a.k_cache = kc;
        a.v_cache = vc;
        a.o = o;
        a.k_tree = tree_qkv ? tk_l : nullptr;
        a.v_tree = tree_qkv ? tv_l : nullptr;
        if (st_status e = st_tree_attention(&a, stream)) return e;
        // x += o W_o (residual add in the epilogue)
        if (st_status e = st::gemm(m, o, Wp(L.wo), d, x, d, rows, d, d, 1, 0, st::kGemmAddTo, s, splitk))
            return e;
        if (st_status e = layernorm(L.ln2_g, L.ln2_b)) return e;
        // f = gelu(h W_1) (GELU in the epilogue), then x += f W_2
        if (st_status e = st::gemm(m, h, Wp(L.w1), F, f, F, rows, F, d, 1, 0, st::kGemmGelu, s, splitk))
            return e;
        if (st_status e = st::gemm(m, f, Wp(L.w2), d, x, d, rows, d, F, 1, 0, st::kGemmAddTo, s, splitk))
            return e;
    }
    if (!logits) return ST_OK;  // (slice pass for the tree's K/V only)
    if (st_status e = layernorm(m->lnf_g, m->lnf_b)) return e;
#undef ST_M_DISPATCH
    const void* wout = m->wout_pad ? m->wout_pad : Wp(m->wout);
    return st::gemm(m, h, wout, m->ldw_out, logits, c.vocab_size, rows, c.vocab_size, d, 1, 0,
                    st::kGemmStoreF32, s, splitk);
}

st_status st_model_tree_forward(st_model* m, int B, int T, const int32_t* tokens,
                                const int32_t* positions, const uint64_t* mask, int W,
                                const int32_t* prefix_len, const int32_t* n_nodes, void* k_cache,
                                void* v_cache, int64_t Lmax, float* logits, void* workspace,
                                size_t workspace_bytes, void* stream) {
    return tree_forward(m, B, T, tokens, positions, mask, W, prefix_len, n_nodes, k_cache, v_cache,
                        Lmax, nullptr, logits, workspace, workspace_bytes, stream);
}

st_status st_model_tree_forward_kt(st_model* m, int B, int T, const int32_t* tokens,
                                   const int32_t* positions, const uint64_t* mask, int W,
                                   const int32_t* prefix_len, const int32_t* n_nodes,
                                   void* k_cache, void* v_cache, int64_t Lmax, void* tree_qkv,
                                   float* logits, void* workspace, size_t workspace_bytes,
                                   void* stream) {
    ST_CHECK_ARG(tree_qkv != nullptr, ST_ERR_INVALID_ARGUMENT, "null tree_qkv");
    return tree_forward(m, B, T, tokens, positions, mask, W, prefix_len, n_nodes, k_cache, v_cache,
                        Lmax, tree_qkv, logits, workspace, workspace_bytes, stream);
}

}  // extern "C"

st_status st_model_tree_forward_slice(st_model* m, int B, int T, int u0, int nf,
                                      const int32_t* tokens, const int32_t* positions,
                                      const uint64_t* mask, int W, const int32_t* prefix_len,
                                      const int32_t* n_nodes, void* k_cache, void* v_cache,
                                      int64_t Lmax, void* tree_qkv, float* logits, void* workspace,
                                      size_t workspace_bytes, void* stream) {
    ST_CHECK_ARG(tree_qkv != nullptr && nf >= 1, ST_ERR_INVALID_ARGUMENT, "null tree_qkv or empty slice");
    ST_CHECK_ARG(m && m->cfg.d_model % 8 == 0, ST_ERR_UNSUPPORTED, "slice pass needs d_model % 8 == 0");
    return tree_forward(m, B, T, tokens, positions, mask, W, prefix_len, n_nodes, k_cache, v_cache,
                        Lmax, tree_qkv, logits, workspace, workspace_bytes, stream, u0, nf);
}
