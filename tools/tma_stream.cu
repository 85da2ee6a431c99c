// Microbenchmark (diagnostic, not product): how fast can one CTA per SM stream
// the K1 KV layout [B*H][L][128] fp16 through TMA with S stages of R-row boxes
// (64 x R elements, SWIZZLE_128B), consumer = one thread that just releases
// slots. Also an LDG.128 streaming baseline. Prints GB/s per configuration.
//   nvcc -std=c++20 -O3 -gencode arch=compute_100a,code=sm_100a -I paper_2305_09781_b200/csrc \
//        -I include tools/tma_stream.cu -o build/tma_stream
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <cstdio>
#include <vector>

#include "sm100.cuh"

using namespace st::sm100;

template <int STAGES, int ROWS>
__global__ void __launch_bounds__(64, 1)
stream_kernel(const __grid_constant__ CUtensorMap tm, int n_seq, int tiles_per_seq,
              unsigned long long* sink) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
    constexpr uint32_t BOX = ROWS * 128;            // one 64-elem x ROWS box
    constexpr uint32_t STAGE_BYTES = 2 * BOX;       // both halves of the 128-wide rows
    uint64_t* full = reinterpret_cast<uint64_t*>(smem + STAGES * STAGE_BYTES);
    uint64_t* empty = full + STAGES;
    if (threadIdx.x == 0) {
        for (int i = 0; i < STAGES; ++i) { mbar_init(full + i, 1); mbar_init(empty + i, 1); }
        fence_barrier_init();
    }
    __syncthreads();
    const long long total = (long long)n_seq * tiles_per_seq;
    const long long t0 = blockIdx.x * total / gridDim.x, t1 = (blockIdx.x + 1) * total / gridDim.x;
    if (threadIdx.x == 0) {
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
        if (acc == 0xdeadbeef) *sink = acc;
    }
}

__global__ void ldg_kernel(const int4* __restrict__ p, long long n, unsigned long long* sink) {
    int4 acc = make_int4(0, 0, 0, 0);
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
        int4 v = __ldcs(p + i);
        acc.x ^= v.x; acc.y ^= v.y; acc.z ^= v.z; acc.w ^= v.w;
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345) *sink = 1;
}

template <int STAGES, int ROWS>
void run(PFN_cuTensorMapEncodeTiled_v12000 enc, void* buf, int n_seq, int L, unsigned long long* sink, int sms) {
    CUtensorMap tm;
    const uint64_t dims[3] = {128, (uint64_t)L, (uint64_t)n_seq};
    const uint64_t strides[2] = {256, (uint64_t)L * 256};
    const uint32_t box[3] = {64, ROWS, 1}, es[3] = {1, 1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, 3, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    const size_t smem = STAGES * 2 * ROWS * 128 + 1024 + 256;
    cudaFuncSetAttribute(stream_kernel<STAGES, ROWS>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    const int tiles = L / ROWS;
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) stream_kernel<STAGES, ROWS><<<sms, 64, smem>>>(tm, n_seq, tiles, sink);
    cudaEventRecord(a);
    const int reps = 10;
    for (int r = 0; r < reps; ++r) stream_kernel<STAGES, ROWS><<<sms, 64, smem>>>(tm, n_seq, tiles, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    const double bytes = (double)n_seq * L * 256;
    printf("TMA stages=%d rows=%3d (%3d KB in flight max): %7.1f GB/s  (%.1f us/pass) %s\n", STAGES, ROWS,
           STAGES * ROWS * 256 / 1024, bytes * reps / (ms * 1e-3) / 1e9, ms * 1e3 / reps,
           cudaGetErrorString(cudaGetLastError()));
}

int main() {
    cudaDriverEntryPointQueryResult q;
    void* f = nullptr;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q);
    auto enc = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const int n_seq = 2 * 8 * 32, L = 2048;  // K and V of C2 = 512 sequences x 2048 rows x 256 B = 268 MB
    void* buf;
    cudaMalloc(&buf, (size_t)n_seq * L * 256);
    cudaMemset(buf, 1, (size_t)n_seq * L * 256);
    unsigned long long* sink;
    cudaMalloc(&sink, 8);
    run<2, 128>(enc, buf, n_seq, L, sink, sms);
    run<3, 128>(enc, buf, n_seq, L, sink, sms);
    run<4, 128>(enc, buf, n_seq, L, sink, sms);
    run<5, 128>(enc, buf, n_seq, L, sink, sms);
    run<6, 128>(enc, buf, n_seq, L, sink, sms);
    run<4, 64>(enc, buf, n_seq, L, sink, sms);
    run<6, 64>(enc, buf, n_seq, L, sink, sms);
    run<8, 64>(enc, buf, n_seq, L, sink, sms);
    run<12, 64>(enc, buf, n_seq, L, sink, sms);
    run<8, 32>(enc, buf, n_seq, L, sink, sms);
    run<16, 32>(enc, buf, n_seq, L, sink, sms);
    {
        const long long n = (long long)n_seq * L * 256 / 16;
        cudaEvent_t a, b;
        cudaEventCreate(&a);
        cudaEventCreate(&b);
        for (int blocks : {sms * 4, sms * 8, sms * 16}) {
            for (int w = 0; w < 3; ++w) ldg_kernel<<<blocks, 512>>>((const int4*)buf, n, sink);
            cudaEventRecord(a);
            for (int r = 0; r < 10; ++r) ldg_kernel<<<blocks, 512>>>((const int4*)buf, n, sink);
            cudaEventRecord(b);
            cudaEventSynchronize(b);
            float ms;
            cudaEventElapsedTime(&ms, a, b);
            printf("LDG.128 grid=%5d x 512: %7.1f GB/s\n", blocks, (double)n * 16 * 10 / (ms * 1e-3) / 1e9);
        }
    }
    return 0;
}
