// Diagnostic: kernel-parameter (constant bank) load latency, first touch vs hit.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/cbank tools/cbank_latency.cu
#include <cstdint>
struct P { uint32_t w[256]; unsigned long long* out; };
__device__ __forceinline__ unsigned long long clk_after(uint32_t v) {
    unsigned long long t;
    asm volatile("{ .reg .pred q; setp.eq.u32 q, %1, 0x7fff1234; @q trap; mov.u64 %0, %%clock64; }" : "=l"(t) : "r"(v) : "memory");
    return t;
}
__device__ __forceinline__ uint32_t ldp(const uint32_t* a) {
    uint32_t v; asm volatile("ld.param.u32 %0, [%1];" : "=r"(v) : "l"(a) : "memory"); return v;
}
__global__ void k(const __grid_constant__ P p, int o1, int o2, int o3) {
    if (threadIdx.x) return;
    unsigned long long t0 = clk_after(0);
    uint32_t a = ldp(&p.w[3]);      unsigned long long t1 = clk_after(a);
    uint32_t b = ldp(&p.w[4]);      unsigned long long t2 = clk_after(b);
    uint32_t c = ldp(&p.w[o1]);     unsigned long long t3 = clk_after(c);
    uint32_t d = ldp(&p.w[o2]);     unsigned long long t4 = clk_after(d);
    uint32_t e = ldp(&p.w[o3]);     unsigned long long t5 = clk_after(e);
    if (blockIdx.x == 7) { p.out[0] = t1 - t0; p.out[1] = t2 - t1; p.out[2] = t3 - t2; p.out[3] = t4 - t3; p.out[4] = t5 - t4; }
}
int main() {
    P p{};
    cudaMalloc(&p.out, 64);
    for (int i = 0; i < 4; ++i) {
        k<<<148, 32>>>(p, 200, 120, 60);
        unsigned long long h[5];
        cudaMemcpy(h, p.out, 40, cudaMemcpyDeviceToHost);
        printf("launch %d: first %llu | same 64B line %llu | w[200] %llu | w[120] %llu | w[60] %llu cycles\n", i, h[0], h[1], h[2], h[3], h[4]);
    }
}
