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

#include <cstdlib>
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
    int wmerge;            // N % 64 == 0: the W map views N as (64, N/64), one box per K block
    // split-K (ks > 1, GEMMs with fewer output tiles than CTAs): work unit u is
    // split u % ks of tile u / ks over K blocks [split * nkb, +nkb); each unit
    // stores its fp32 partial tile to part[split][z][M][N], and a second kernel
    // sums the ks partials in split order and applies the epilogue
    int ks, nkb;
    float* part;
};

// The work unit's tile coordinates and K-block range.
struct Unit {
    int mb, nb, z, split, kb0, kb1;
};
__device__ __forceinline__ Unit unit_of(const GemmParams& p, int u, int nm) {
    Unit w;
    const int t = u / p.ks;
    w.split = u - t * p.ks;
    w.mb = t % nm;
    const int rest = t / nm;
    w.nb = rest % p.nn;
    w.z = rest / p.nn;
    w.kb0 = w.split * p.nkb;
    w.kb1 = min(p.nk, w.kb0 + p.nkb);
    return w;
}

// Split-K: this unit's fp32 partial of one row's 32 columns [col0, col0+32).
__device__ __forceinline__ void partial_chunk(const GemmParams& p, const Unit& w, int row, int col0,
                                              const float (&v)[32]) {
    if (row >= p.M) return;
    float* c = p.part + (((long long)w.split * p.Z + w.z) * p.M + row) * p.N + col0;
    if (col0 + 32 <= p.N && (p.N & 3) == 0) {
#pragma unroll
        for (int k = 0; k < 8; ++k)
            reinterpret_cast<float4*>(c)[k] = make_float4(v[4 * k], v[4 * k + 1], v[4 * k + 2], v[4 * k + 3]);
    } else {
#pragma unroll
        for (int k = 0; k < 32; ++k)
            if (col0 + k < p.N) c[k] = v[k];
    }
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

// Split-K reduction: C = epi(sum over splits of part[split], in split order —
// deterministic), 32 columns of one row per thread.
template <class T, int EPI>
__global__ void __launch_bounds__(256)
splitk_reduce_kernel(const GemmParams p) {
    pdl_wait();
    pdl_trigger();
    const int cpr = (p.N + 31) / 32;  // 32-column chunks per row
    const long long chunks = (long long)p.Z * p.M * cpr;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < chunks;
         i += (long long)gridDim.x * blockDim.x) {
        const int c = (int)(i % cpr);
        const long long zr = i / cpr;
        const int row = (int)(zr % p.M), z = (int)(zr / p.M);
        const int col0 = c * 32;
        float v[32];
#pragma unroll
        for (int k = 0; k < 32; ++k) v[k] = 0.f;
        const bool vec = col0 + 32 <= p.N && (p.N & 3) == 0;
        for (int sp = 0; sp < p.ks; ++sp) {
            const float* src = p.part + (((long long)sp * p.Z + z) * p.M + row) * p.N + col0;
            if (vec) {
#pragma unroll
                for (int k = 0; k < 8; ++k) {
                    const float4 x = __ldcs(reinterpret_cast<const float4*>(src) + k);
                    v[4 * k] += x.x;
                    v[4 * k + 1] += x.y;
                    v[4 * k + 2] += x.z;
                    v[4 * k + 3] += x.w;
                }
            } else {
#pragma unroll
                for (int k = 0; k < 32; ++k)
                    if (col0 + k < p.N) v[k] += src[k];
            }
        }
        epilogue_chunk<T, EPI>(p, z, row, col0, v);
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
    const int units = p.nm * p.nn * p.Z * p.ks;

    if (warp == 0) {
        // ============================ TMA producer ============================
        if (lane == 0) {
            uint32_t kc = 0;
            for (int u = blockIdx.x; u < units; u += gridDim.x) {
                const Unit w = unit_of(p, u, p.nm);
                const int mb = w.mb, nb = w.nb, z = w.z;
                for (int kb = w.kb0; kb < w.kb1; ++kb, ++kc) {
                    const uint32_t s = kc % STAGES;
                    mbar_wait(empty + s, ((kc / STAGES) & 1) ^ 1);
                    mbar_arrive_expect_tx(full + s, STAGE_BYTES);
                    uint8_t* a = smem + s * STAGE_BYTES;
                    tma_load_2d(a, &tm_a, full + s, kb * BK, mb * BM);
                    if (p.wmerge) {  // the four 64-column W atoms in one box
                        tma_load_4d(a + A_BYTES, &tm_b, full + s, 0, kb * BK, nb * (BN / 64), z);
                    } else {
#pragma unroll
                        for (int j = 0; j < 4; ++j)
                            tma_load_3d(a + A_BYTES + j * B_ATOM, &tm_b, full + s, nb * BN + j * 64,
                                        kb * BK, z);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ============================= MMA issuer =============================
        constexpr uint32_t fmt = std::is_same<T, __half>::value ? 0u : 1u;
        constexpr uint32_t idesc = idesc_f16(fmt, BM, BN, 0, 1);  // A K-major, W MN-major
        uint32_t kc = 0, ac = 0;
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++ac) {
            const Unit w = unit_of(p, u, p.nm);
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
        for (int u = blockIdx.x; u < units; u += gridDim.x, ++ac) {
            const Unit w = unit_of(p, u, p.nm);
            const int mb = w.mb, nb = w.nb, z = w.z;
            const uint32_t acc = ac & 1;
            mbar_wait(acc_full + acc, (ac >> 1) & 1);
            tc_fence_after();
            const int row = mb * BM + q * 32 + lane;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                const int col0 = nb * BN + c * 32;
                if (col0 >= p.N) break;
                uint32_t raw[32];
                tmem_ld_32x32b_x32(lane_base + acc * BN + c * 32, raw);
                tmem_ld_wait();
                float v[32];
#pragma unroll
                for (int k = 0; k < 32; ++k) v[k] = __uint_as_float(raw[k]);
                if (p.ks > 1) partial_chunk(p, w, row, col0, v);
                else epilogue_chunk<T, EPI>(p, z, row, col0, v);
            }
            tc_fence_before();
            mbar_arrive(acc_empty + acc);
        }
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 1) tmem_dealloc<512>(tmem);
}

// ---------------------------------------------------------- CTA-pair GEMM ---
// The same GEMM on 256 x 256 output tiles computed by a CTA PAIR (cluster of
// 2) with tcgen05.mma.cta_group::2 (M=256, N=256, K=16): CTA r of the pair
// loads rows [128r, 128r+128) of the A tile and columns [128r, 128r+128) of the
// W tile (32 KB per 64-deep K block instead of 48 KB per CTA: the pair reads
// each A and W byte once), the leader (rank 0) issues the MMAs over both CTAs'
// shared memory, each CTA's TMEM holds its 128 rows of the 256-column
// accumulator, and each CTA's four epilogue warps store their own rows.
constexpr int P_STAGES = 6;
constexpr uint32_t PA_BYTES = 128 * BK * 2;             // 16 KB: this CTA's A half
constexpr uint32_t PB_BYTES = 2 * B_ATOM;               // 16 KB: this CTA's W half (128 N)
constexpr uint32_t P_STAGE = PA_BYTES + PB_BYTES;       // 32 KB
constexpr uint32_t P_OFF_BAR = P_STAGES * P_STAGE;
constexpr uint32_t P_SMEM = P_OFF_BAR + 256;

// the leader CTA's copy of a barrier (shared::cluster address with the peer bit cleared)
__device__ __forceinline__ uint32_t leader_addr(const void* p) { return smem_u32(p) & 0xFEFFFFFFu; }
__device__ __forceinline__ void tma2_load_2d(void* dst, const CUtensorMap* m, uint32_t bar, int c0, int c1) {
    asm volatile(
        "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ void tma2_load_3d(void* dst, const CUtensorMap* m, uint32_t bar, int c0, int c1,
                                             int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}
__device__ __forceinline__ void tma2_load_4d(void* dst, const CUtensorMap* m, uint32_t bar, int c0, int c1,
                                             int c2, int c3) {
    asm volatile(
        "cp.async.bulk.tensor.4d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(bar), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
        : "memory");
}
__device__ __forceinline__ void umma2_warp(uint32_t d_tmem, uint64_t a_desc, uint64_t b_desc,
                                           uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p, e;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(d_tmem),
        "l"(a_desc), "l"(b_desc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// commit: arrive on the barrier at this offset in BOTH CTAs of the pair
__device__ __forceinline__ void umma2_commit_both(uint64_t* bar) {
    asm volatile(
        "{\n\t.reg .pred e;\n\t"
        "elect.sync _|e, 0xffffffff;\n\t"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n\t}"
        ::"r"(smem_u32(bar)), "h"((unsigned short)3)
        : "memory");
}

template <class T, int EPI>
__global__ void __launch_bounds__(THREADS, 1)
gemm2_kernel(const __grid_constant__ CUtensorMap tm_a, const __grid_constant__ CUtensorMap tm_b,
             const GemmParams p) {
    extern __shared__ __align__(1024) uint8_t smem[];
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + P_OFF_BAR);
    uint64_t* empty = full + P_STAGES;
    uint64_t* acc_full = empty + P_STAGES;   // [2]
    uint64_t* acc_empty = acc_full + 2;      // [2] (leader: both CTAs' epilogue warps arrive)
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(acc_empty + 2);
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const uint32_t rank = cluster_rank();
    if (threadIdx.x == 0) {
        if (smem_u32(smem) & 1023u) __trap();
        for (int i = 0; i < P_STAGES; ++i) {
            mbar_init(full + i, 1);
            mbar_init(empty + i, 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(acc_full + i, 1);
            mbar_init(acc_empty + i, 2 * 4);   // lane 0 of 4 epilogue warps x 2 CTAs
        }
        fence_barrier_init();
    }
    if (warp == 0 && lane == 0) {
        prefetch_tmap(&tm_a);
        prefetch_tmap(&tm_b);
    }
    if (warp == 1) {
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         smem_u32(tmem_slot))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    cluster_sync();       // both CTAs' barriers initialised, TMEM allocated
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    pdl_wait();
    pdl_trigger();
    const int nm2 = (p.M + 255) / 256;
    const int units = nm2 * p.nn * p.Z * p.ks;
    const int cid = blockIdx.x >> 1, ncl = gridDim.x >> 1;

    if (warp == 0) {
        // ========================= TMA producer (both CTAs) ======================
        if (lane == 0) {
            uint32_t kc = 0;
            for (int u = cid; u < units; u += ncl) {
                const Unit w = unit_of(p, u, nm2);
                const int mb = w.mb, nb = w.nb, z = w.z;
                for (int kb = w.kb0; kb < w.kb1; ++kb, ++kc) {
                    const uint32_t s = kc % P_STAGES;
                    mbar_wait(empty + s, ((kc / P_STAGES) & 1) ^ 1);
                    // the leader's full barrier counts both CTAs' bytes
                    if (rank == 0) mbar_arrive_expect_tx(full + s, 2 * P_STAGE);
                    const uint32_t fb = leader_addr(full + s);
                    uint8_t* a = smem + s * P_STAGE;
                    tma2_load_2d(a, &tm_a, fb, kb * BK, mb * 256 + (int)rank * 128);
                    if (p.wmerge) {  // this CTA's two 64-column W atoms in one box
                        tma2_load_4d(a + PA_BYTES, &tm_b, fb, 0, kb * BK, (nb * BN + (int)rank * 128) / 64, z);
                    } else {
#pragma unroll
                        for (int j = 0; j < 2; ++j)
                            tma2_load_3d(a + PA_BYTES + j * B_ATOM, &tm_b, fb,
                                         nb * BN + (int)rank * 128 + j * 64, kb * BK, z);
                    }
                }
            }
        }
    } else if (warp == 1) {
        // ===================== MMA issuer (leader CTA only) ======================
        if (rank == 0) {
            constexpr uint32_t fmt = std::is_same<T, __half>::value ? 0u : 1u;
            constexpr uint32_t idesc = idesc_f16(fmt, 256, BN, 0, 1);
            uint32_t kc = 0, ac = 0;
            for (int u = cid; u < units; u += ncl, ++ac) {
                const Unit w = unit_of(p, u, nm2);
                const uint32_t acc = ac & 1;
                mbar_wait(acc_empty + acc, ((ac >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t d = tmem + acc * BN;
                for (int kb = w.kb0; kb < w.kb1; ++kb, ++kc) {
                    const uint32_t s = kc % P_STAGES;
                    mbar_wait(full + s, (kc / P_STAGES) & 1);
                    tc_fence_after();
                    const uint32_t a_base = smem_u32(smem + s * P_STAGE);
                    const uint64_t ad = smem_desc(a_base, 16, 1024);
                    const uint64_t bd = smem_desc(a_base + PA_BYTES, B_ATOM, 1024);
#pragma unroll
                    for (int kk = 0; kk < BK / 16; ++kk)
                        umma2_warp(d, ad + ((kk * 32) >> 4), bd + ((kk * 2048) >> 4), idesc,
                                   (kb > w.kb0 || kk) ? 1u : 0u);
                    umma2_commit_both(empty + s);
                }
                umma2_commit_both(acc_full + acc);
            }
        }
    } else {
        // ======================= epilogue (both CTAs) ============================
        const int q = warp & 3;
        const uint32_t lane_base = tmem + ((uint32_t)(q * 32) << 16);
        const uint32_t ae0 = leader_addr(acc_empty), ae1 = leader_addr(acc_empty + 1);
        uint32_t ac = 0;
        for (int u = cid; u < units; u += ncl, ++ac) {
            const Unit w = unit_of(p, u, nm2);
            const int mb = w.mb, nb = w.nb, z = w.z;
            const uint32_t acc = ac & 1;
            mbar_wait(acc_full + acc, (ac >> 1) & 1);
            tc_fence_after();
            const int row = mb * 256 + (int)rank * 128 + q * 32 + lane;
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                const int col0 = nb * BN + c * 32;
                if (col0 >= p.N) break;
                uint32_t raw[32];
                tmem_ld_32x32b_x32(lane_base + acc * BN + c * 32, raw);
                tmem_ld_wait();
                float v[32];
#pragma unroll
                for (int k = 0; k < 32; ++k) v[k] = __uint_as_float(raw[k]);
                if (p.ks > 1) partial_chunk(p, w, row, col0, v);
                else epilogue_chunk<T, EPI>(p, z, row, col0, v);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive_cluster(acc ? ae1 : ae0);
        }
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync();       // no CTA leaves while its peer may still use its memory
    tc_fence_after();
    if (warp == 1)
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
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
    const int units = p.nm * p.nn * p.Z * p.ks;
    const int grid = units < sm_count() ? units : sm_count();
    ST_CUDA_TRY(launch_pdl(gemm_kernel<T, EPI>, dim3(grid), dim3(THREADS), SMEM_BYTES, s, ta, tb, p));
    (void)g;
    return ST_OK;
}

// Split-K: the reduction + epilogue pass after the partial GEMM (PDL-chained).
template <class T, int EPI>
st_status launch_reduce(const GemmParams& p, cudaStream_t s) {
    const long long chunks = (long long)p.Z * p.M * ((p.N + 31) / 32);
    const long long blocks = (chunks + 255) / 256;
    const int grid = (int)(blocks < 8 * sm_count() ? blocks : 8 * sm_count());
    ST_CUDA_TRY(launch_pdl(splitk_reduce_kernel<T, EPI>, dim3(grid), dim3(256), 0, s, p));
    return ST_OK;
}

template <class T, int EPI>
st_status launch_pair(const CUtensorMap& ta, const CUtensorMap& tb, const GemmParams& p,
                      cudaStream_t s) {
    static int max_clusters = 0;
    if (!max_clusters) {
        ST_CUDA_TRY(cudaFuncSetAttribute(gemm2_kernel<T, EPI>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, P_SMEM));
        ST_CUDA_TRY(cudaFuncSetAttribute(gemm2_kernel<T, EPI>,
                                         cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(2 * sm_count());
        cfg.blockDim = dim3(THREADS);
        cfg.dynamicSmemBytes = P_SMEM;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        ST_CUDA_TRY(cudaOccupancyMaxActiveClusters(&max_clusters, gemm2_kernel<T, EPI>, &cfg));
        if (max_clusters < 1) max_clusters = 1;
    }
    const int units = ((p.M + 255) / 256) * p.nn * p.Z * p.ks;
    const int clusters = units < max_clusters ? units : max_clusters;
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(2 * clusters);
    cfg.blockDim = dim3(THREADS);
    cfg.dynamicSmemBytes = P_SMEM;
    cfg.stream = s;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 2;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    at[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[1].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 2;
    ST_CUDA_TRY(cudaLaunchKernelEx(&cfg, gemm2_kernel<T, EPI>, ta, tb, p));
    return ST_OK;
}

}  // namespace

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
    static const bool pair_env = !(getenv("ST_GEMM_PAIR") && atoi(getenv("ST_GEMM_PAIR")) == 0);
    const bool pair = pair_env && g.M >= 256;
    // N % 64 == 0: W viewed as (64, K, N/64, Z) — the 64-column block index a
    // dimension of stride 128 B outside K — so a CTA's 2 (pair) or 4 W atoms
    // of a K block are one box (one TMA issue instead of 2 / 4)
    const bool wmerge = g.N % 64 == 0;
    if (wmerge) {
        const uint64_t dims[4] = {64, (uint64_t)g.K, (uint64_t)g.N / 64, (uint64_t)g.Z};
        const uint64_t strides[3] = {(uint64_t)g.ldw * 2, 128, (uint64_t)g.ldw * g.K * 2};
        const uint32_t box[4] = {64, BK, pair ? 2u : 4u, 1};
        const uint32_t es4[4] = {1, 1, 1, 1};
        if (enc(&tb, dt, 4, const_cast<void*>(g.W), dims, strides, box, es4,
                CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
            set_error("gemm: cuTensorMapEncodeTiled(W, merged) failed");
            return ST_ERR_CUDA;
        }
    } else {
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
    const size_t cbytes = g.epi == kGemmStoreF32 ? 4 : 2;
    p.vec = (reinterpret_cast<uintptr_t>(g.C) % 16 == 0) && ((size_t)g.ldc * cbytes) % 16 == 0 &&
            ((size_t)g.c_stride_z * cbytes) % 16 == 0;
    p.wmerge = wmerge ? 1 : 0;
    // Split-K for GEMMs with fewer output tiles than CTA slots (the engine's
    // drafting passes, small batches), when the caller lends fp32 scratch:
    // pick ks minimising (waves of units) x (K blocks per unit) x (per-block
    // time: the larger of the MMA time and the per-SM load time) + the
    // partials' extra HBM traffic and the reduction launch.
    p.ks = 1;
    p.nkb = p.nk;
    p.part = nullptr;
    static const bool splitk_env = !(getenv("ST_GEMM_SPLITK") && atoi(getenv("ST_GEMM_SPLITK")) == 0);
    {
        const int slots = pair ? sm_count() / 2 : sm_count();
        const long long tiles = (long long)(pair ? (g.M + 255) / 256 : p.nm) * p.nn * p.Z;
        const double tau = pair ? 0.44 : 0.64;  // us per K block per CTA (pair: MMA; single: 48 KB loads)
        const double out_bytes = 4.0 * g.Z * (double)g.M * g.N;
        auto cost = [&](int ks) {
            const long long units = tiles * ks;
            const long long waves = (units + slots - 1) / slots;
            const int nkb = (p.nk + ks - 1) / ks;
            return waves * nkb * tau + (ks > 1 ? (ks + 1) * out_bytes / 6.0e6 + 2.0 : 0.0);
        };
        if (splitk_env && g.work && tiles < slots) {
            double best = cost(1);
            for (int ks = 2; ks <= 16 && p.nk / ks >= 4; ++ks) {
                if ((double)ks * out_bytes > (double)g.work_bytes) break;
                const double c = cost(ks);
                if (c < best * 0.9) {
                    best = c;
                    p.ks = ks;
                }
            }
        }
        if (p.ks > 1) {
            p.nkb = (p.nk + p.ks - 1) / p.ks;
            p.ks = (p.nk + p.nkb - 1) / p.nkb;  // no empty splits
            p.part = g.work;
        }
    }
#define ST_GEMM_RUN(TT, E)                                                          \
    {                                                                               \
        const st_status r_ = pair ? launch_pair<TT, E>(ta, tb, p, s) : launch<TT, E>(g, ta, tb, p, s); \
        if (r_ != ST_OK || p.ks == 1) return r_;                                    \
        return launch_reduce<TT, E>(p, s);                                          \
    }
#define ST_GEMM_EPI(TT)                                                              \
    switch (g.epi) {                                                                 \
        case kGemmStore: ST_GEMM_RUN(TT, kGemmStore)                                 \
        case kGemmGelu: ST_GEMM_RUN(TT, kGemmGelu)                                   \
        case kGemmAddTo: ST_GEMM_RUN(TT, kGemmAddTo)                                 \
        case kGemmStoreF32: ST_GEMM_RUN(TT, kGemmStoreF32)                           \
    }
    if (g.dtype == ST_F16) {
        ST_GEMM_EPI(__half)
    } else {
        ST_GEMM_EPI(__nv_bfloat16)
    }
#undef ST_GEMM_EPI
#undef ST_GEMM_RUN
    set_error("gemm: bad epilogue");
    return ST_ERR_INVALID_ARGUMENT;
}

}  // namespace st

extern "C" st_status st_gemm(st_dtype dtype, int M, int N, int K, int Z, const void* A, int lda,
                             const void* W, int ldw, void* C, int ldc, int64_t c_stride_z,
                             int epilogue, void* stream) {
    if (st_status e = st::require_device()) return e;
    ST_CHECK_ARG(A && W && C, ST_ERR_INVALID_ARGUMENT, "null pointer");
    st::GemmArgs g{dtype, A, lda, W, ldw, C, c_stride_z, ldc, M, N, K, Z, epilogue};
    if (st_status e = st::gemm_sm100(g, st::as_stream(stream))) return e;
    ST_LAUNCH_CHECK();
    return ST_OK;
}
