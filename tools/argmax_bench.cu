// Diagnostic microbenchmark: the K3 logits-streaming argmax (verify_greedy.cu)
// at the C2 shape (B=8, T=64, V=32000 fp32 = 65.5 MB) for several
// (blocks per row, float4 loads in flight per thread, threads per block)
// configurations, cycling over 3 logits buffers (196 MB > L2).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/argmax_bench tools/argmax_bench.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ unsigned long long arg_key(float v, int i) {
    if (v != v) {
        if (i == 0) return ~0ull;
        v = -INFINITY;
    }
    uint32_t u = __float_as_uint(v);
    u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    return ((unsigned long long)u << 32) | (uint32_t)(~(uint32_t)i);
}

// LD: 0 __ldcs (ld.global.cs), 1 ld.global.nc.L1::no_allocate.L2::256B,
// 2 ld.global.L1::no_allocate.L2::256B, 3 __ldg
template <int LD>
__device__ __forceinline__ float4 ld4(const float4* p) {
    if constexpr (LD == 0) return __ldcs(p);
    if constexpr (LD == 3) return __ldg(p);
    float4 v;
    if constexpr (LD == 1)
        asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    else
        asm volatile("ld.global.L1::no_allocate.L2::256B.v4.f32 {%0,%1,%2,%3}, [%4];"
                     : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}

template <int SPLIT, int UNROLL, int NT, int LD = 0>
__global__ void __launch_bounds__(NT) argmax_kernel(const float* __restrict__ logits, int T, int V,
                                                    unsigned long long* keys) {
    const int part = blockIdx.x, u = blockIdx.y, b = blockIdx.z;
    const float* row = logits + ((int64_t)b * T + u) * V;
    const int nv = V >> 2;
    const int per = (nv + SPLIT - 1) / SPLIT;
    const int lo = part * per, hi = min(nv, lo + per);
    const float4* r4 = reinterpret_cast<const float4*>(row);
    float bv = -INFINITY;
    int bi = lo + (int)threadIdx.x < hi ? (lo + (int)threadIdx.x) * 4 : -1;
    for (int base = lo + threadIdx.x; base < hi; base += NT * UNROLL) {
        float4 x[UNROLL];
#pragma unroll
        for (int k = 0; k < UNROLL; ++k) {
            const int j = base + k * NT;
            x[k] = j < hi ? ld4<LD>(r4 + j) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        }
#pragma unroll
        for (int k = 0; k < UNROLL; ++k) {
            const int j = (base + k * NT) * 4;
            if (x[k].x > bv) { bv = x[k].x; bi = j; }
            if (x[k].y > bv) { bv = x[k].y; bi = j + 1; }
            if (x[k].z > bv) { bv = x[k].z; bi = j + 2; }
            if (x[k].w > bv) { bv = x[k].w; bi = j + 3; }
        }
    }
    unsigned long long best = bi >= 0 ? arg_key(bv, bi) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    __shared__ unsigned long long red[NT / 32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[warp] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < NT / 32; ++w) best = max(best, red[w]);
        keys[((int64_t)b * T + u) * SPLIT + part] = best;
    }
}

// Persistent variant: G blocks loop over the B*T*SPLIT slices (grid-stride),
// the next slice's loads issued before the current slice is reduced.
template <int SPLIT, int UNROLL, int NT>
__global__ void __launch_bounds__(NT) argmax_persist(const float* __restrict__ logits, int T, int V,
                                                     unsigned long long* keys, int nslices) {
    const int nv = V >> 2;
    const int per = (nv + SPLIT - 1) / SPLIT;
    __shared__ unsigned long long red[2][NT / 32];
    int sl = blockIdx.x;
    float4 x[UNROLL];
    auto load = [&](int s_, float4 (&dst)[UNROLL]) {
        const int part = s_ % SPLIT, row = s_ / SPLIT;
        const float4* r4 = reinterpret_cast<const float4*>(logits + (int64_t)row * V);
        const int lo = part * per, hi = min(nv, lo + per);
#pragma unroll
        for (int k = 0; k < UNROLL; ++k) {
            const int j = lo + threadIdx.x + k * NT;
            dst[k] = j < hi ? __ldcs(r4 + j) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        }
    };
    if (sl < nslices) load(sl, x);
    int it = 0;
    for (; sl < nslices; sl += gridDim.x, ++it) {
        float4 y[UNROLL];
        const int nx = sl + gridDim.x;
        if (nx < nslices) load(nx, y);
        const int part = sl % SPLIT;
        const int lo = part * per;
        float bv = -INFINITY;
        int bi = (lo + (int)threadIdx.x) * 4;
#pragma unroll
        for (int k = 0; k < UNROLL; ++k) {
            const int j = (lo + threadIdx.x + k * NT) * 4;
            if (x[k].x > bv) { bv = x[k].x; bi = j; }
            if (x[k].y > bv) { bv = x[k].y; bi = j + 1; }
            if (x[k].z > bv) { bv = x[k].z; bi = j + 2; }
            if (x[k].w > bv) { bv = x[k].w; bi = j + 3; }
        }
        unsigned long long best = arg_key(bv, bi);
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
        const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
        if (lane == 0) red[it & 1][warp] = best;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < NT / 32; ++w) best = max(best, red[it & 1][w]);
            keys[sl] = best;
        }
#pragma unroll
        for (int k = 0; k < UNROLL; ++k) x[k] = y[k];
    }
}

template <int SPLIT, int UNROLL, int NT>
void run_p(float* const* bufs, unsigned long long* keys, int B, int T, int V, int blocks) {
    const int ns = B * T * SPLIT;
    for (int i = 0; i < 6; ++i) argmax_persist<SPLIT, UNROLL, NT><<<blocks, NT>>>(bufs[i % 3], T, V, keys, ns);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 60;
    cudaEventRecord(e0);
    for (int i = 0; i < iters; ++i) argmax_persist<SPLIT, UNROLL, NT><<<blocks, NT>>>(bufs[i % 3], T, V, keys, ns);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / iters;
    printf("persistent split %d unroll %2d threads %4d blocks %4d: %7.2f us  %6.0f GB/s\n", SPLIT, UNROLL, NT,
           blocks, us, 4.0 * B * T * V / us / 1e3);
}

// TMA variant: the block's slice arrives in shared memory through one (or a
// few) cp.async.bulk copies completing on an mbarrier, then the threads scan it.
template <int SPLIT, int NT>
__global__ void __launch_bounds__(NT) argmax_bulk(const float* __restrict__ logits, int T, int V,
                                                  unsigned long long* keys) {
    extern __shared__ __align__(128) float sl[];
    __shared__ __align__(8) unsigned long long bar;
    __shared__ unsigned long long red[NT / 32];
    const int part = blockIdx.x, u = blockIdx.y, b = blockIdx.z;
    const float* row = logits + ((int64_t)b * T + u) * V;
    const int per = (V + SPLIT - 1) / SPLIT;
    const int lo = part * per, hi = min(V, lo + per), cnt = hi - lo;
    const uint32_t bar_a = (uint32_t)__cvta_generic_to_shared(&bar);
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(bar_a));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        const uint32_t bytes = (uint32_t)cnt * 4;  // multiple of 16 when per % 4 == 0
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(bar_a), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                     ::"r"((uint32_t)__cvta_generic_to_shared(sl)), "l"(row + lo), "r"(bytes), "r"(bar_a)
                     : "memory");
    }
    uint32_t done = 0;
    while (!done)
        asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared.b64 p, [%1], 0; selp.u32 %0, 1, 0, p; }"
                     : "=r"(done) : "r"(bar_a) : "memory");
    float bv = -INFINITY;
    int bi = threadIdx.x < cnt ? lo + threadIdx.x : -1;
    for (int i = threadIdx.x; i < cnt; i += NT) {
        const float x = sl[i];
        if (x > bv) { bv = x; bi = lo + i; }
    }
    unsigned long long best = bi >= 0 ? arg_key(bv, bi) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (lane == 0) red[warp] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < NT / 32; ++w) best = max(best, red[w]);
        keys[((int64_t)b * T + u) * SPLIT + part] = best;
    }
}

template <int SPLIT, int NT>
void run_b(float* const* bufs, unsigned long long* keys, int B, int T, int V) {
    dim3 grid(SPLIT, T, B);
    const size_t smem = (size_t)((V + SPLIT - 1) / SPLIT) * 4;
    cudaFuncSetAttribute(argmax_bulk<SPLIT, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    for (int i = 0; i < 6; ++i) argmax_bulk<SPLIT, NT><<<grid, NT, smem>>>(bufs[i % 3], T, V, keys);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 60;
    cudaEventRecord(e0);
    for (int i = 0; i < iters; ++i) argmax_bulk<SPLIT, NT><<<grid, NT, smem>>>(bufs[i % 3], T, V, keys);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / iters;
    printf("bulk split %d threads %4d: %7.2f us  %6.0f GB/s  (%s)\n", SPLIT, NT, us,
           4.0 * B * T * V / us / 1e3, cudaGetErrorString(cudaGetLastError()));
}

template <int SPLIT, int UNROLL, int NT, int LD = 0>
void run(float* const* bufs, unsigned long long* keys, int B, int T, int V) {
    dim3 grid(SPLIT, T, B);
    for (int i = 0; i < 6; ++i) argmax_kernel<SPLIT, UNROLL, NT, LD><<<grid, NT>>>(bufs[i % 3], T, V, keys);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int iters = 60;
    cudaEventRecord(e0);
    for (int i = 0; i < iters; ++i) argmax_kernel<SPLIT, UNROLL, NT, LD><<<grid, NT>>>(bufs[i % 3], T, V, keys);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    const double us = ms * 1e3 / iters;
    const double bytes = 4.0 * B * T * V;
    printf("split %d unroll %2d threads %4d ld %d: %7.2f us  %6.0f GB/s\n", SPLIT, UNROLL, NT, LD, us, bytes / us / 1e3);
}

int main() {
    const int B = 8, T = 64, V = 32000;
    float* bufs[3];
    for (auto& p : bufs) {
        cudaMalloc(&p, (size_t)B * T * V * 4);
        cudaMemset(p, 0, (size_t)B * T * V * 4);
    }
    unsigned long long* keys;
    cudaMalloc(&keys, (size_t)B * T * 16 * 8);
    for (int rep = 0; rep < 2; ++rep) {
        run<8, 4, 256>(bufs, keys, B, T, V);
        run<8, 4, 256, 1>(bufs, keys, B, T, V);
        run<8, 4, 256, 2>(bufs, keys, B, T, V);
        run<8, 4, 256, 3>(bufs, keys, B, T, V);
        run<4, 8, 256, 1>(bufs, keys, B, T, V);
        run<8, 4, 512, 1>(bufs, keys, B, T, V);
        run<16, 2, 256, 1>(bufs, keys, B, T, V);
        run<7, 5, 256>(bufs, keys, B, T, V);
        run<9, 4, 256>(bufs, keys, B, T, V);
        run<10, 4, 256>(bufs, keys, B, T, V);
        run<6, 6, 256>(bufs, keys, B, T, V);
        run<12, 3, 256>(bufs, keys, B, T, V);
        run<14, 3, 256>(bufs, keys, B, T, V);
        run<16, 2, 256>(bufs, keys, B, T, V);
    }
    return 0;
}
