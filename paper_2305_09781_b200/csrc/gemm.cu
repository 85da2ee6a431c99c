// Around-path projections of the device decoder: a
// hand-written sm_100a GEMM, C[z] (op)= A · W[z], on the 5th-gen tensor cores
// with the decoder's elementwise work fused into the epilogue — the reference
// runs one f64 matvec per tree node per matrix (proj/src/transformer.cpp:
// 262-319); here every projection is one GEMM over all B·T tree rows.
//
//   A [M][K] row-major f16/bf16 (activations; K-major UMMA operand)
//   W [Z][K][N] row-major f16/bf16 (weights as stored: MN-major UMMA operand)
//   C [Z][M][N] (ldc, c_stride_z) f16/bf16 or f32
//   epilogue: store | GELU (erf form, transformer.cpp:67) | add-to (residual:
//   C += A·W, the pre-LN blocks' x + ...) | store f32 (LM-head logits)
//
// Design: persistent, one CTA per SM over 128 x 256 output tiles (m fastest, so
// the CTAs working at one time share each W tile through L2); warp roles:
// a TMA producer (A box 64x128, W as four 64x64 boxes per 64-deep K block,
// SWIZZLE_128B, 4-stage ring of 48 KB), an MMA issuer (tcgen05.mma kind::f16
// M=128 N=256 K=16, fp32 accumulators double-buffered in TMEM: 2 x 256
// columns, so one tile's epilogue overlaps the next tile's MMAs), and four
// epilogue warps (tcgen05.ld 32 columns at a time -> epilogue op -> 16-byte
// global stores).
#include <cuda.h>
#include <cudaTypedefs.h>

#include <mutex>
#include <type_traits>

#include "common.cuh"
#include "gemm.h"
#include "sm100.cuh"

namespace st {
namespace {

using namespace sm100;

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr uint32_t A_BYTES = BM * BK * 2;            // 16 KB
constexpr uint32_t B_ATOM = BK * 128;                // 64 K rows x 128 B (64 N elements)
constexpr uint32_t B_BYTES = 4 * B_ATOM;             // 32 KB
constexpr uint32_t STAGE_BYTES = A_BYTES + B_BYTES;  // 48 KB
constexpr uint32_t OFF_BAR = STAGES * STAGE_BYTES;
constexpr uint32_t SMEM_BYTES = OFF_BAR + 256;
constexpr int THREADS = 6 * 32;  // producer, MMA, 4 epilogue warps

struct GemmParams {
    void* C;
    long long c_stride_z;  // elements
    int ldc;
    int M, N, K, Z;
    int nm, nn, nk;        // tile counts
    int vec;               // 16-byte stores allowed (aligned C rows)
    // schedule: tiles [0, dp_tiles) whole (tile t on CTA t % G), then the
    // remaining sk_tiles split into G equal ranges of (tile, k-block) units
    int dp_tiles, sk_tiles;
    float* partial;        // [G][BM*BN] fp32 split-tile pieces (stream-K)
    unsigned* flags;       // [G] piece published (re-armed by the consumer)
};

// One unit of a CTA's work: tile t, k-blocks [kb0, kb1).
struct Work {
    int t, kb0, kb1;
};

__device__ __forceinline__ long long sk_start(const GemmParams& p, int c) {
    return (long long)p.sk_tiles * p.nk * c / gridDim.x;
}

// The i-th work item of this CTA (false when done): its whole tiles first,
// then the segments of its stream-K range.
__device__ __forceinline__ bool work_at(const GemmParams& p, int i, Work& w, long long& u) {
    const int G = gridDim.x;
    const int ndp = (p.dp_tiles - (int)blockIdx.x + G - 1) / G;
    if (i < ndp) {
        w.t = blockIdx.x + i * G;
        w.kb0 = 0;
        w.kb1 = p.nk;
        return true;
    }
    if (i == ndp) u = sk_start(p, blockIdx.x);
    const long long u1 = sk_start(p, blockIdx.x + 1);
    if (u >= u1) return false;
    const int ts = (int)(u / p.nk);
    w.t = p.dp_tiles + ts;
    w.kb0 = (int)(u - (long long)ts * p.nk);
    const long long tile_end = (long long)(ts + 1) * p.nk;
    w.kb1 = (int)((tile_end < u1 ? tile_end : u1) - (long long)ts * p.nk);
    u += w.kb1 - w.kb0;
    return true;
}

template <class T> struct pk;
template <> struct pk<__half> {
    static __device__ __forceinline__ uint32_t two(float a, float b) {
        __half2 h = __floats2half2_rn(a, b);
        return *reinterpret_cast<uint32_t*>(&h);
    }
    static __device__ __forceinline__ float lo(uint32_t w) {
        return __half2float(__ushort_as_half((unsigned short)(w & 0xffffu)));
    }
    static __device__ __forceinline__ float hi(uint32_t w) {
        return __half2float(__ushort_as_half((unsigned short)(w >> 16)));
    }
    static __device__ __forceinline__ __half one(float a) { return __float2half_rn(a); }
    static __device__ __forceinline__ float get(__half x) { return __half2float(x); }
};
template <> struct pk<__nv_bfloat16> {
    static __device__ __forceinline__ uint32_t two(float a, float b) {
        __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
        return *reinterpret_cast<uint32_t*>(&h);
    }
    static __device__ __forceinline__ float lo(uint32_t w) { return __uint_as_float(w << 16); }
    static __device__ __forceinline__ float hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }
    static __device__ __forceinline__ __nv_bfloat16 one(float a) { return __float2bfloat16_rn(a); }
    static __device__ __forceinline__ float get(__nv_bfloat16 x) { return __bfloat162float(x); }
};

// Apply the epilogue to one row's 32 accumulator columns [col0, col0+32) and
// store them.
template <class T, int EPI>
__device__ __forceinline__ void epilogue_chunk(const GemmParams& p, int z, int row, int col0,
                                               float (&v)[32]) {
    if (row >= p.M) return;
    if constexpr (EPI == kGemmGelu) {
#pragma unroll
        for (int k = 0; k < 32; ++k) v[k] = gelu_erf(v[k]);
    }
    const bool full = col0 + 32 <= p.N;
    if constexpr (EPI == kGemmStoreF32) {
        float* c = reinterpret_cast<float*>(p.C) + z * p.c_stride_z + (long long)row * p.ldc + col0;
        if (full && p.vec) {
#pragma unroll
            for (int k = 0; k < 8; ++k)
                reinterpret_cast<float4*>(c)[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
        } else {
#pragma unroll
            for (int k = 0; k < 32; ++k)
                if (col0 + k < p.N) c[k] = v[k];
        }
    } else {
        T* c = reinterpret_cast<T*>(p.C) + z * p.c_stride_z + (long long)row * p.ldc + col0;
        if (full && p.vec) {
            uint4* c4 = reinterpret_cast<uint4*>(c);
            if constexpr (EPI == kGemmAddTo) {
                uint4 old[4];
#pragma unroll
                for (int q = 0; q < 4; ++q) old[q] = c4[q];
#pragma unroll
                for (int q = 0; q < 4; ++q) {
                    const uint32_t w[4] = {old[q].x, old[q].y, old[q].z, old[q].w};
#pragma unroll
                    for (int e = 0; e < 4; ++e) {
                        v[q * 8 + 2 * e] += pk<T>::lo(w[e]);
                        v[q * 8 + 2 * e + 1] += pk<T>::hi(w[e]);
                    }
                }
            }
#pragma unroll
            for (int q = 0; q < 4; ++q)
                c4[q] = make_uint4(pk<T>::two(v[q * 8], v[q * 8 + 1]), pk<T>::two(v[q * 8 + 2], v[q * 8 + 3]),
                                   pk<T>::two(v[q * 8 + 4], v[q * 8 + 5]), pk<T>::two(v[q * 8 + 6], v[q * 8 + 7]));
        } else {
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                if (col0 + k < p.N) {
                    float x = v[k];
                    if constexpr (EPI == kGemmAddTo) x += pk<T>::get(c[k]);
                    c[k] = pk<T>::one(x);
                }
            }
        }
    }
}

template <class T, int EPI>
__global__ void __launch_bounds__(THREADS, 1)
gemm_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
            const GemmParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + OFF_BAR);
    uint64_t* empty = full + STAGES;
    uint64_t* acc_full = empty + STAGES;   // [2]
    uint64_t* acc_empty = acc_full + 2;    // [2]
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        if (smem_u32(smem) & 1023u) __trap();
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(acc_full + i, 1);
            mbar_init(acc_empty + i, 4 * 32);
        }
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tm_a);
        prefetch_tmap(&tm_b);
    }
    if (warp == 1) tmem_alloc<512>(tmem_slot);
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();       // A (and C for add-to) come from the previous kernel
    pdl_trigger();
    if (warp == 0) {
        // ============================ TMA producer ============================
        if (lane == 0) {
            uint32_t kc = 0;
            Work w;
            long long u = 0;
            for (int i = 0; work_at(p, i, w, u); ++i) {
                const int t = w.t;
                const int mb = t % p.nm, rest = t / p.nm, nb = rest % p.nn, z = rest / p.nn;
                for (int kb = w.kb0; kb < w.kb1; ++kb, ++kc) {
                    const uint32_t s = kc % STAGES;
                    mbar_wait(empty + s, ((kc / STAGES) & 1) ^ 1);
                    mbar_arrive_expect_tx(full + s, STAGE_BYTES);
                    uint8_t* a = smem + s * STAGE_BYTES;
                    tma_load_2d(a, &tm_a, full + s, kb * BK, mb * BM);
#pragma unroll
                    for (int j = 0; j < 4; ++j)
                        tma_load_3d(a + A_BYTES + j * B_ATOM, &tm_b, full + s, nb * BN + j * 64,
                                    kb * BK, z);
                }
            }
        }
    } else if (warp == 1) {
        // ============================= MMA issuer =============================
        constexpr uint32_t fmt = std::is_same<T, __half>::value ? 0u : 1u;
        constexpr uint32_t idesc = idesc_f16(fmt, BM, BN, 0, 1);  // A K-major, W MN-major
        uint32_t kc = 0, ac = 0;
        Work w;
        long long u = 0;
        for (int i = 0; work_at(p, i, w, u); ++i, ++ac) {
            const uint32_t acc = ac & 1;
            mbar_wait(acc_empty + acc, ((ac >> 1) & 1) ^ 1);
            tc_fence_after();
            const uint32_t d = tmem + acc * BN;
            for (int kb = w.kb0; kb < w.kb1; ++kb, ++kc) {
                const uint32_t s = kc % STAGES;
                mbar_wait(full + s, (kc / STAGES) & 1);
                tc_fence_after();
                const uint32_t a_base = smem_u32(smem + s * STAGE_BYTES);
                const uint64_t ad = smem_desc(a_base, 16, 1024);
                const uint64_t bd = smem_desc(a_base + A_BYTES, B_ATOM, 1024);
#pragma unroll
                for (int kk = 0; kk < BK / 16; ++kk)
                    umma_f16_ss_warp(d, ad + ((kk * 32) >> 4), bd + ((kk * 2048) >> 4), idesc,
                                     (kb > w.kb0 || kk) ? 1u : 0u);
                umma_commit_warp(empty + s);
            }
            umma_commit_warp(acc_full + acc);
        }
    } else {
        // ============================== epilogue ==============================
        const int q = warp & 3;  // TMEM lane quadrant this warp may access
        const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
        uint32_t ac = 0;
        Work w;
        long long u = 0;
        const int r = q * 32 + lane;  // this thread's row of the tile
        for (int i = 0; work_at(p, i, w, u); ++i, ++ac) {
            const int t = w.t;
            const int mb = t % p.nm, rest = t / p.nm, nb = rest % p.nn, z = rest / p.nn;
            const uint32_t acc = ac & 1;
            // stream-K: a segment that starts past k-block 0 is a PIECE (first
            // segment of this CTA's range) and leaves its fp32 partial for the
            // tile's owner; the segment holding k-block 0 of a split tile is
            // its OWNER (last segment of the owner's range) and adds the
            // pieces of the following CTAs, in CTA order (deterministic)
            const bool piece = w.kb0 > 0;
            const bool owner = !piece && w.kb1 < p.nk;
            int np = 0, first = 0;
            if (owner) {
                const long long tile_end = (long long)(t - p.dp_tiles + 1) * p.nk;
                first = blockIdx.x + 1;
                while (first + np < (int)gridDim.x && sk_start(p, first + np) < tile_end) ++np;
                for (int j = 0; j < np; ++j) wait_flag_gpu(p.flags + first + j);
            }
            mbar_wait(acc_full + acc, (ac >> 1) & 1);
            tc_fence_after();
            const int row = mb * BM + r;
            float4* mine = reinterpret_cast<float4*>(p.partial + (long long)blockIdx.x * BM * BN);
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                const int col0 = nb * BN + c * 32;
                if (!piece && col0 >= p.N) break;
                uint32_t raw[32];
                tmem_ld_32x32b_x32(lane_base + acc * BN + c * 32, raw);
                tmem_ld_wait();
                float v[32];
#pragma unroll
                for (int k = 0; k < 32; ++k) v[k] = __uint_as_float(raw[k]);
                if (piece) {  // float4 (r, 4j..4j+3) of chunk c at (c*8 + j)*BM + r: coalesced
#pragma unroll
                    for (int j = 0; j < 8; ++j)
                        mine[(c * 8 + j) * BM + r] = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
                    continue;
                }
                for (int pc = 0; pc < np; ++pc) {
                    const float4* other =
                        reinterpret_cast<const float4*>(p.partial + (long long)(first + pc) * BM * BN);
#pragma unroll
                    for (int j = 0; j < 8; ++j) {
                        const float4 x = __ldcg(other + (c * 8 + j) * BM + r);
                        v[4 * j] += x.x;
                        v[4 * j + 1] += x.y;
                        v[4 * j + 2] += x.z;
                        v[4 * j + 3] += x.w;
                    }
                }
                epilogue_chunk<T, EPI>(p, z, row, col0, v);
            }
            tc_fence_before();
            mbar_arrive(acc_empty + acc);
            if (piece) {  // every epilogue thread's stores, then one gpu-scope release
                named_bar_sync(1, 4 * 32);
                if (threadIdx.x == 2 * 32) st_release_gpu(p.flags + blockIdx.x, 1u);
            }
            if (owner) {  // re-arm the pieces' flags for the next launch (all reads done)
                named_bar_sync(1, 4 * 32);
                if (threadIdx.x == 2 * 32)
                    for (int j = 0; j < np; ++j) p.flags[first + j] = 0u;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc<512>(tmem);
}

PFN_cuTensorMapEncodeTiled_v12000 encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
                cudaSuccess && q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

int sm_count() {
    static int n = 0;
    if (!n) {
        int dev = 0;
        cudaGetDevice(&dev);
        cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev);
    }
    return n;
}

template <class T, int EPI>
st_status launch(const GemmArgs& g, const CUtensorMap& ta, const CUtensorMap& tb,
                 const GemmParams& p, cudaStream_t s) {
    static bool attr = false;
    if (!attr) {
        ST_CUDA_TRY(cudaFuncSetAttribute(gemm_kernel<T, EPI>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, SMEM_BYTES));
        attr = true;
    }
    const int tiles = p.nm * p.nn * p.Z;
    const int grid = tiles < sm_count() ? tiles : sm_count();
    // stream-K owners wait for pieces of other CTAs: cooperative launch
    // guarantees they are all resident (one CTA per SM either way)
    ST_CUDA_TRY(launch_pdl_ex(gemm_kernel<T, EPI>, dim3(grid), dim3(THREADS), SMEM_BYTES, s,
                              p.sk_tiles > 0, ta, tb, p));
    (void)g;
    return ST_OK;
}

}  // namespace

size_t gemm_workspace_size() {
    return (size_t)sm_count() * BM * BN * sizeof(float) + (size_t)sm_count() * sizeof(unsigned) + 256;
}

bool gemm_supported(const GemmArgs& g) {
    auto al = [](const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15) == 0; };
    return (g.dtype == ST_F16 || g.dtype == ST_BF16) && g.M >= 1 && g.N >= 1 && g.K >= 1 &&
           g.Z >= 1 && g.ldw >= g.N && g.ldw % 8 == 0 && g.lda >= g.K && g.lda % 8 == 0 &&
           al(g.A) && al(g.W);
}

st_status gemm_sm100(const GemmArgs& g, cudaStream_t s) {
    ST_CHECK_ARG(gemm_supported(g), ST_ERR_UNSUPPORTED,
                 "gemm: f16/bf16, lda and ldw multiples of 8, 16-byte aligned A / W");
    auto enc = encoder();
    ST_CHECK_ARG(enc != nullptr, ST_ERR_CUDA, "cuTensorMapEncodeTiled unavailable");
    const CUtensorMapDataType dt =
        g.dtype == ST_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    CUtensorMap ta, tb;
    const uint32_t es[3] = {1, 1, 1};
    {
        const uint64_t dims[2] = {(uint64_t)g.K, (uint64_t)g.M};
        const uint64_t strides[1] = {(uint64_t)g.lda * 2};
        const uint32_t box[2] = {BK, BM};
        if (enc(&ta, dt, 2, const_cast<void*>(g.A), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            set_error("gemm: cuTensorMapEncodeTiled(A) failed");
            return ST_ERR_CUDA;
        }
    }
    {
        const uint64_t dims[3] = {(uint64_t)g.N, (uint64_t)g.K, (uint64_t)g.Z};
        const uint64_t strides[2] = {(uint64_t)g.ldw * 2, (uint64_t)g.ldw * g.K * 2};
        const uint32_t box[3] = {64, BK, 1};
        if (enc(&tb, dt, 3, const_cast<void*>(g.W), dims, strides, box, es,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            set_error("gemm: cuTensorMapEncodeTiled(W) failed");
            return ST_ERR_CUDA;
        }
    }
    GemmParams p;
    p.C = g.C;
    p.c_stride_z = g.c_stride_z;
    p.ldc = g.ldc;
    p.M = g.M;
    p.N = g.N;
    p.K = g.K;
    p.Z = g.Z;
    p.nm = (g.M + BM - 1) / BM;
    p.nn = (g.N + BN - 1) / BN;
    p.nk = (g.K + BK - 1) / BK;
    // Schedule: whole tiles in full waves, the last (partial) wave plus one full
    // wave spread over all CTAs as equal (tile, k-block) ranges (stream-K), so
    // no SM idles through a fractional last wave. Needs the workspace (fp32
    // pieces + flags, zeroed once) and at least two k-blocks per CTA.
    const int tiles = p.nm * p.nn * p.Z;
    const int G = tiles < sm_count() ? tiles : sm_count();
    p.dp_tiles = tiles;
    p.sk_tiles = 0;
    p.partial = nullptr;
    p.flags = nullptr;
    if (g.workspace && g.workspace_bytes >= gemm_workspace_size() && tiles % G != 0 && tiles > G) {
        const int waves = tiles / G;
        const int sk = tiles - (waves - 1) * G;
        if ((long long)sk * p.nk >= 2LL * G) {
            p.dp_tiles = tiles - sk;
            p.sk_tiles = sk;
            p.partial = reinterpret_cast<float*>(g.workspace);
            p.flags = reinterpret_cast<unsigned*>(static_cast<char*>(g.workspace) +
                                                  (size_t)sm_count() * BM * BN * sizeof(float));
        }
    }
    const size_t cbytes = g.epi == kGemmStoreF32 ? 4 : 2;
    p.vec = (reinterpret_cast<uintptr_t>(g.C) % 16 == 0) && ((size_t)g.ldc * cbytes) % 16 == 0 &&
            ((size_t)g.c_stride_z * cbytes) % 16 == 0;
#define ST_GEMM_EPI(TT)                                                              \
    switch (g.epi) {                                                                 \
        case kGemmStore: return launch<TT, kGemmStore>(g, ta, tb, p, s);             \
        case kGemmGelu: return launch<TT, kGemmGelu>(g, ta, tb, p, s);               \
        case kGemmAddTo: return launch<TT, kGemmAddTo>(g, ta, tb, p, s);             \
        case kGemmStoreF32: return launch<TT, kGemmStoreF32>(g, ta, tb, p, s);       \
    }
    if (g.dtype == ST_F16) {
        ST_GEMM_EPI(__half)
    } else {
        ST_GEMM_EPI(__nv_bfloat16)
    }
#undef ST_GEMM_EPI
    set_error("gemm: bad epilogue");
    return ST_ERR_INVALID_ARGUMENT;
}

}  // namespace st

extern "C" size_t st_gemm_workspace_size(void) { return st::gemm_workspace_size(); }

extern "C" st_status st_gemm(st_dtype dtype, int M, int N, int K, int Z, const void* A, int lda,
                             const void* W, int ldw, void* C, int ldc, int64_t c_stride_z,
                             int epilogue, void* workspace, size_t workspace_bytes, void* stream) {
    if (st_status e = st::require_device()) return e;
    ST_CHECK_ARG(A && W && C, ST_ERR_INVALID_ARGUMENT, "null pointer");
    st::GemmArgs g{dtype, A, lda, W, ldw, C, c_stride_z, ldc, M, N, K, Z, epilogue, workspace,
                   workspace_bytes};
    if (st_status e = st::gemm_sm100(g, st::as_stream(stream))) return e;
    ST_LAUNCH_CHECK();
    return ST_OK;
}
