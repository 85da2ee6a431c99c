// Diagnostic microbenchmark: K3 logits argmax as a persistent TMA-bulk ring
// (one block per SM, a producer warp streams 32 KB row slices into a
// STAGES-deep shared-memory ring with cp.async.bulk; consumer warps scan each
// slice and fold it to one key) vs the current grid kernel, at the C2 shape
// (B=8, T=64, V=32000 fp32 = 65.5 MB), cycling over 3 buffers (> L2).
//   nvcc -std=c++17 -gencode arch=compute_100a,code=sm_100a -O3 -I paper_2305_09781_b200/csrc \
//        -o /tmp/argmax_ring tools/argmax_ring.cu
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

#include "sm100.cuh"

using namespace st::sm100;

__device__ __forceinline__ unsigned long long arg_key(float v, int i) {
    if (v != v) {
        if (i == 0) return ~0ull;
        v = -INFINITY;
    }
    uint32_t u = v == 0.0f ? 0u : __float_as_uint(v);
    u = (u & 0x80000000u) ? ~u : (u | 0x80000000u);
    return ((unsigned long long)u << 32) | (uint32_t)(~(uint32_t)i);
}

// current production kernel shape: <SPLIT=8, UNROLL=4, 256 threads>, grid (8, T, B)
__global__ void __launch_bounds__(256) argmax_grid(const float* __restrict__ logits, int T, int V,
                                                   unsigned long long* keys) {
    const int part = blockIdx.x, u = blockIdx.y, b = blockIdx.z;
    const float* row = logits + ((int64_t)b * T + u) * V;
    const int nv = V >> 2, per = (nv + 7) / 8;
    const int lo = part * per, hi = min(nv, lo + per);
    const float4* r4 = reinterpret_cast<const float4*>(row);
    float bv = -INFINITY;
    int bi = lo + (int)threadIdx.x < hi ? (lo + (int)threadIdx.x) * 4 : -1;
    for (int base = lo + threadIdx.x; base < hi; base += 256 * 4) {
        float4 x[4];
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int j = base + k * 256;
            x[k] = j < hi ? __ldcs(r4 + j) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
        }
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const int j = (base + k * 256) * 4;
            if (x[k].x > bv) { bv = x[k].x; bi = j; }
            if (x[k].y > bv) { bv = x[k].y; bi = j + 1; }
            if (x[k].z > bv) { bv = x[k].z; bi = j + 2; }
            if (x[k].w > bv) { bv = x[k].w; bi = j + 3; }
        }
    }
    unsigned long long best = bi >= 0 ? arg_key(bv, bi) : 0;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
    __shared__ unsigned long long red[8];
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = best;
    __syncthreads();
    if (threadIdx.x == 0) {
        for (int w = 1; w < 8; ++w) best = max(best, red[w]);
        keys[((int64_t)b * T + u) * 8 + part] = best;
    }
}

// Persistent ring: NT consumer threads + one producer warp. Chunk k = slice
// (k % nsl) of row (k / nsl), `per` floats (multiple of 4). Block c takes the
// contiguous chunks [c*total/G, (c+1)*total/G).
template <int NT, int STAGES>
__global__ void __launch_bounds__(NT + 32) argmax_ring(const float* __restrict__ logits, int rows,
                                                       int V, int nsl, int per,
                                                       unsigned long long* keys) {
    extern __shared__ __align__(128) uint8_t smem[];
    float* buf = reinterpret_cast<float*>(smem);
    __shared__ __align__(8) uint64_t full[STAGES], empty[STAGES];
    __shared__ unsigned long long skey[STAGES];
    const int total = rows * nsl;
    const int c0 = (int)((long long)blockIdx.x * total / gridDim.x);
    const int c1 = (int)((long long)(blockIdx.x + 1) * total / gridDim.x);
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s) {
            mbar_init(full + s, 1);
            mbar_init(empty + s, 1);
            skey[s] = 0;
        }
        fence_barrier_init();
    }
    __syncthreads();
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == NT / 32) {  // producer
        if (lane == 0) {
            for (int k = c0, i = 0; k < c1; ++k, ++i) {
                const int st = i % STAGES;
                mbar_wait(empty + st, ((i / STAGES) & 1) ^ 1);
                const int row = k / nsl, part = k - row * nsl;
                const int lo = part * per, cnt = min(per, V - lo);
                mbar_arrive_expect_tx(full + st, (uint32_t)cnt * 4);
                bulk_load(buf + (size_t)st * per, logits + (int64_t)row * V + lo, (uint32_t)cnt * 4,
                          full + st);
            }
        }
        return;
    }
    for (int k = c0, i = 0; k < c1; ++k, ++i) {
        const int st = i % STAGES;
        const int row = k / nsl, part = k - row * nsl;
        const int lo = part * per, cnt = min(per, V - lo), nv = cnt >> 2;
        mbar_wait(full + st, (i / STAGES) & 1);
        const float4* s4 = reinterpret_cast<const float4*>(buf + (size_t)st * per);
        float bv = -INFINITY;
        int bi = (int)threadIdx.x < nv ? lo + (int)threadIdx.x * 4 : -1;
        for (int j = threadIdx.x; j < nv; j += NT) {
            const float4 x = s4[j];
            const int e = lo + j * 4;
            if (x.x > bv) { bv = x.x; bi = e; }
            if (x.y > bv) { bv = x.y; bi = e + 1; }
            if (x.z > bv) { bv = x.z; bi = e + 2; }
            if (x.w > bv) { bv = x.w; bi = e + 3; }
        }
        unsigned long long best = bi >= 0 ? arg_key(bv, bi) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (lane == 0) atomicMax(skey + st, best);
        named_bar_sync(1, NT);
        if (threadIdx.x == 0) {
            keys[(int64_t)row * 8 + part] = skey[st];
            skey[st] = 0;
            mbar_arrive(empty + st);
        }
    }
}


// Equal-share single wave: G blocks (resident all at once), block c scans the
// contiguous float4 range [c*N/G, (c+1)*N/G) of the flattened [rows][V/4]
// logits; a range spans a few rows, and the block writes one key per row
// piece into keys[row][slot], slot = c - first block touching the row.
template <int NT, int UNR>
__global__ void __launch_bounds__(NT) argmax_share(const float* __restrict__ logits, int rows, int V,
                                                   unsigned long long* keys) {
    const int nv = V >> 2;
    const long long N = (long long)rows * nv;
    const long long lo = (long long)blockIdx.x * N / gridDim.x;
    const long long hi = (long long)(blockIdx.x + 1) * N / gridDim.x;
    const float4* r4 = reinterpret_cast<const float4*>(logits);
    __shared__ unsigned long long red[NT / 32];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    for (long long a = lo; a < hi;) {
        const int row = (int)(a / nv);
        const long long rend = min(hi, (long long)(row + 1) * nv);
        float bv = -INFINITY;
        int bi = -1;
        for (long long base = a + threadIdx.x; base < rend; base += (long long)NT * UNR) {
            float4 x[UNR];
#pragma unroll
            for (int k = 0; k < UNR; ++k) {
                const long long j = base + (long long)k * NT;
                x[k] = j < rend ? __ldcs(r4 + j) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
            }
#pragma unroll
            for (int k = 0; k < UNR; ++k) {
                const long long j = base + (long long)k * NT;
                if (j >= rend) continue;
                const int e = (int)(j - (long long)row * nv) * 4;
                if (bi < 0) { bv = x[k].x; bi = e; }
                else if (x[k].x > bv) { bv = x[k].x; bi = e; }
                if (x[k].y > bv) { bv = x[k].y; bi = e + 1; }
                if (x[k].z > bv) { bv = x[k].z; bi = e + 2; }
                if (x[k].w > bv) { bv = x[k].w; bi = e + 3; }
            }
        }
        unsigned long long best = bi >= 0 ? arg_key(bv, bi) : 0;
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) best = max(best, __shfl_xor_sync(0xffffffffu, best, o));
        if (lane == 0) red[warp] = best;
        __syncthreads();
        if (threadIdx.x == 0) {
            for (int w = 1; w < NT / 32; ++w) best = max(best, red[w]);
            const long long first = ((long long)row * nv * gridDim.x) / N;  // first block touching row
            keys[(long long)row * 8 + (blockIdx.x - first)] = best;
        }
        __syncthreads();
        a = rend;
    }
}

template <class F>
double timeit(F&& launch, int iters = 60) {
    for (int i = 0; i < 6; ++i) launch(i);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    for (int i = 0; i < iters; ++i) launch(i);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms * 1e3 / iters;
}

template <int NT, int STAGES>
void ring(float* const* bufs, unsigned long long* keys, unsigned long long* ref, int rows, int V,
          int nsl, int blocks_per_sm, int nsm) {
    const int per = ((V + nsl - 1) / nsl + 3) / 4 * 4;
    const size_t smem = (size_t)STAGES * per * 4;
    cudaFuncSetAttribute(argmax_ring<NT, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int G = nsm * blocks_per_sm;
    const double us = timeit([&](int i) {
        argmax_ring<NT, STAGES><<<G, NT + 32, smem>>>(bufs[i % 3], rows, V, nsl, per, keys);
    });
    // check against the grid kernel's keys (max over slices per row)
    cudaMemset(keys, 0, (size_t)rows * 8 * 8);
    argmax_ring<NT, STAGES><<<G, NT + 32, smem>>>(bufs[0], rows, V, nsl, per, keys);
    static unsigned long long h[8 * 64 * 8], r[8 * 64 * 8];
    cudaMemcpy(h, keys, sizeof h, cudaMemcpyDeviceToHost);
    cudaMemcpy(r, ref, sizeof r, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int row = 0; row < rows; ++row) {
        unsigned long long a = 0, b = 0;
        for (int j = 0; j < 8; ++j) {
            a = a > h[row * 8 + j] ? a : h[row * 8 + j];
            b = b > r[row * 8 + j] ? b : r[row * 8 + j];
        }
        bad += a != b;
    }
    printf("ring NT %3d stages %d slices %d blocks/SM %d smem %6zu: %7.2f us  %6.0f GB/s  bad %d  (%s)\n",
           NT, STAGES, nsl, blocks_per_sm, smem, us, 4.0 * rows * V / us / 1e3, bad,
           cudaGetErrorString(cudaGetLastError()));
}

template <int NT, int UNR>
void share(float* const* bufs, unsigned long long* keys, unsigned long long* ref, int rows, int V, int G) {
    const double us = timeit([&](int i) { argmax_share<NT, UNR><<<G, NT>>>(bufs[i % 3], rows, V, keys); });
    cudaMemset(keys, 0, (size_t)rows * 8 * 8);
    argmax_share<NT, UNR><<<G, NT>>>(bufs[0], rows, V, keys);
    static unsigned long long h[8 * 64 * 8], r[8 * 64 * 8];
    cudaMemcpy(h, keys, sizeof h, cudaMemcpyDeviceToHost);
    cudaMemcpy(r, ref, sizeof r, cudaMemcpyDeviceToHost);
    int bad = 0;
    for (int row = 0; row < rows; ++row) {
        unsigned long long a = 0, b = 0;
        for (int j = 0; j < 8; ++j) {
            a = a > h[row * 8 + j] ? a : h[row * 8 + j];
            b = b > r[row * 8 + j] ? b : r[row * 8 + j];
        }
        bad += a != b;
    }
    printf("share NT %3d unroll %d blocks %5d: %7.2f us  %6.0f GB/s  bad %d  (%s)\n", NT, UNR, G, us,
           4.0 * rows * V / us / 1e3, bad, cudaGetErrorString(cudaGetLastError()));
}

__global__ void fill(float* p, size_t n, unsigned seed) {
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x) {
        unsigned x = (unsigned)i * 2654435761u ^ seed;
        x ^= x >> 13;
        x *= 0x5bd1e995u;
        x ^= x >> 15;
        p[i] = (float)(x & 0xffffff) / 16777216.0f;
    }
}

int main() {
    const int B = 8, T = 64, V = 32000, rows = B * T;
    int nsm = 0;
    cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, 0);
    float* bufs[3];
    for (int i = 0; i < 3; ++i) {
        cudaMalloc(&bufs[i], (size_t)rows * V * 4);
        fill<<<1024, 256>>>(bufs[i], (size_t)rows * V, 17u + i);
    }
    unsigned long long *keys, *ref;
    cudaMalloc(&keys, (size_t)rows * 8 * 8);
    cudaMalloc(&ref, (size_t)rows * 8 * 8);
    for (int rep = 0; rep < 2; ++rep) {
        const double us = timeit([&](int i) { argmax_grid<<<dim3(8, T, B), 256>>>(bufs[i % 3], T, V, ref); });
        printf("grid (8 x T x B) x 256: %7.2f us  %6.0f GB/s\n", us, 4.0 * rows * V / us / 1e3);
        argmax_grid<<<dim3(8, T, B), 256>>>(bufs[0], T, V, ref);
        share<256, 4>(bufs, keys, ref, rows, V, nsm * 8);
        share<256, 8>(bufs, keys, ref, rows, V, nsm * 8);
        share<512, 4>(bufs, keys, ref, rows, V, nsm * 4);
        share<256, 4>(bufs, keys, ref, rows, V, nsm * 16);
        share<128, 8>(bufs, keys, ref, rows, V, nsm * 16);
        share<256, 2>(bufs, keys, ref, rows, V, nsm * 8);
        ring<256, 4>(bufs, keys, ref, rows, V, 4, 1, nsm);
        ring<256, 6>(bufs, keys, ref, rows, V, 4, 1, nsm);
        ring<512, 6>(bufs, keys, ref, rows, V, 4, 1, nsm);
        ring<256, 3>(bufs, keys, ref, rows, V, 4, 2, nsm);
        ring<256, 6>(bufs, keys, ref, rows, V, 8, 2, nsm);
        ring<128, 6>(bufs, keys, ref, rows, V, 8, 2, nsm);
        ring<256, 8>(bufs, keys, ref, rows, V, 8, 1, nsm);
        ring<512, 12>(bufs, keys, ref, rows, V, 8, 1, nsm);
    }
    return 0;
}
