// Diagnostic (not product): is the per-CTA duration spread of K1 (equal tile
// counts, end times 36-44 us at C2) a property of the SM? One CTA per SM
// streams an equal share of a 268 MB buffer (the C2 KV layout) through a
// 4-stage TMA ring of 32 KB tiles and records (smid, ns from its first load
// to its last tile landed). Several passes; prints per-SM rates and the
// correlation of each pass with the first.
//   nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2305_09781_b200/csrc \
//        -I include tools/sm_rate.cu -o build/sm_rate -lcuda
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "sm100.cuh"

using namespace st::sm100;

constexpr int STAGES = 4, ROWS = 128;

__global__ void __launch_bounds__(64, 1)
rate_kernel(const __grid_constant__ CUtensorMap tm, int n_seq, int tiles_per_seq,
            unsigned long long* out) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr uint32_t BOX = ROWS * 128;
    constexpr uint32_t STAGE_BYTES = 2 * BOX;
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
        fence_barrier_init();
    }
    __syncthreads();
    const long long total = (long long)n_seq * tiles_per_seq;
    const long long t0 = blockIdx.x * total / gridDim.x, t1 = (blockIdx.x + 1) * total / gridDim.x;
    unsigned long long g0 = 0, g1 = 0;
    if (threadIdx.x == 0) {
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g0));
        uint32_t c = 0;
        for (long long t = t0; t < t1; ++t, ++c) {
            const uint32_t s = c % STAGES;
            mbar_wait(empty + s, ((c / STAGES) & 1) ^ 1);
            mbar_arrive_expect_tx(full + s, STAGE_BYTES);
            const int seq = (int)(t / tiles_per_seq), row = (int)(t % tiles_per_seq) * ROWS;
            tma_load_3d(smem + s * STAGE_BYTES, &tm, full + s, 0, row, seq);
            tma_load_3d(smem + s * STAGE_BYTES + BOX, &tm, full + s, 64, row, seq);
        }
    } else if (threadIdx.x == 32) {
        uint32_t c = 0;
        unsigned long long acc = 0;
        for (long long t = t0; t < t1; ++t, ++c) {
            const uint32_t s = c % STAGES;
            mbar_wait(full + s, (c / STAGES) & 1);
            acc += smem[s * STAGE_BYTES + (c & 127)];
            mbar_arrive(empty + s);
        }
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(g1));
        unsigned smid;
        asm volatile("mov.u32 %0, %%smid;" : "=r"(smid));
        out[3 * blockIdx.x] = smid;
        out[3 * blockIdx.x + 2] = g1 + (acc == 0xdeadbeef);
    }
    __syncthreads();
    if (threadIdx.x == 0) out[3 * blockIdx.x + 1] = g0;
}

int main(int argc, char** argv) {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    if (argc > 1) sms = atoi(argv[1]);  // CTAs (one per SM)
    const int n_seq = 2 * 8 * 32, L = 2048;
    void* buf;
    cudaMalloc(&buf, (size_t)n_seq * L * 256);
    cudaMemset(buf, 1, (size_t)n_seq * L * 256);
    unsigned long long* out;
    cudaMalloc(&out, sms * 3 * 8);
    CUtensorMap tm;
    const uint64_t dims[3] = {128, (uint64_t)L, (uint64_t)n_seq};
    const uint64_t strides[2] = {256, (uint64_t)L * 256};
    const uint32_t box[3] = {64, ROWS, 1}, es[3] = {1, 1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const size_t smem = STAGES * 2 * ROWS * 128 + 1024 + 256;
    cudaFuncSetAttribute(rate_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int passes = 6;
    std::vector<std::vector<double>> dur(passes, std::vector<double>(sms, 0));
    std::vector<unsigned long long> h(sms * 3);
    for (int w = 0; w < 3; ++w) rate_kernel<<<sms, 64, smem>>>(tm, n_seq, L / ROWS, out);
    for (int p = 0; p < passes; ++p) {
        rate_kernel<<<sms, 64, smem>>>(tm, n_seq, L / ROWS, out);
        cudaMemcpy(h.data(), out, h.size() * 8, cudaMemcpyDeviceToHost);
        unsigned long long gmin = ~0ull, gmax = 0;
        for (int c = 0; c < sms; ++c) {
            const int smid = (int)h[3 * c];
            dur[p][smid % sms] = (h[3 * c + 2] - h[3 * c + 1]) / 1e3;
            gmin = std::min(gmin, h[3 * c + 1]);
            gmax = std::max(gmax, h[3 * c + 2]);
        }
        auto d = dur[p];
        std::sort(d.begin(), d.end());
        printf("pass %d: first load -> last tile (us) min %.1f median %.1f max %.1f; kernel span %.1f us\n", p,
               d[0], d[sms / 2], d[sms - 1], (gmax - gmin) / 1e3);
    }
    auto corr = [&](const std::vector<double>& a, const std::vector<double>& b) {
        double ma = 0, mb = 0;
        for (int i = 0; i < sms; ++i) { ma += a[i]; mb += b[i]; }
        ma /= sms; mb /= sms;
        double sab = 0, saa = 0, sbb = 0;
        for (int i = 0; i < sms; ++i) {
            sab += (a[i] - ma) * (b[i] - mb);
            saa += (a[i] - ma) * (a[i] - ma);
            sbb += (b[i] - mb) * (b[i] - mb);
        }
        return sab / std::sqrt(saa * sbb);
    };
    for (int p = 1; p < passes; ++p) printf("corr(pass 0, pass %d) by smid = %.3f\n", p, corr(dur[0], dur[p]));
    printf("per-SM mean duration (us), smid order:\n");
    for (int s = 0; s < sms; ++s) {
        double m = 0;
        for (int p = 0; p < passes; ++p) m += dur[p][s];
        printf("%5.1f%c", m / passes, (s % 16 == 15) ? '\n' : ' ');
    }
    printf("\n");
    return 0;
}
