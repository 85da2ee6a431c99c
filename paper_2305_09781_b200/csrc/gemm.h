// Around-path GEMM of the device decoder (gemm.cu) and its fused epilogues.
#pragma once
#include <cuda_runtime.h>

#include "spectree_capi.h"

namespace st {

enum GemmEpilogue : int {
    kGemmStore = ST_GEMM_STORE,        // C = A W            (f16/bf16)
    kGemmGelu = ST_GEMM_GELU,          // C = gelu(A W)
    kGemmAddTo = ST_GEMM_ADD_TO,       // C += A W           (residual)
    kGemmStoreF32 = ST_GEMM_STORE_F32  // C = A W            (f32, e.g. logits)
};

struct GemmArgs {
    st_dtype dtype;
    const void* A;
    int lda;                // elements
    const void* W;          // [Z][K][ldw] (row stride ldw >= N, multiple of 8)
    int ldw;
    void* C;
    long long c_stride_z;   // elements between the Z outputs
    int ldc;                // elements
    int M, N, K, Z;
    int epi;
    float* work = nullptr;  // optional fp32 scratch for split-K partials (none: no split)
    size_t work_bytes = 0;
};

bool gemm_supported(const GemmArgs& g);
st_status gemm_sm100(const GemmArgs& g, cudaStream_t s);

// GELU, erf form (reference transformer.cpp:67): 0.5 v (1 + erf(v / sqrt 2)).
// 1 + erf(x) via Abramowitz & Stegun 7.1.26 (|erf error| <= 1.5e-7, far below
// the f16/bf16 output resolution), evaluated as erfc(|x|) = poly(t) e^{-x^2}
// for x < 0 so the small values of the negative tail keep their relative
// accuracy (no 1 - erf cancellation). Branch-free: 2 MUFU ops + 7 FMAs.
__device__ __forceinline__ float gelu_erf(float v) {
    const float x = v * 0.70710678118654752f;
    const float a = fabsf(x);
    const float t = __fdividef(1.f, fmaf(0.3275911f, a, 1.f));
    float y = fmaf(1.061405429f, t, -1.453152027f);
    y = fmaf(y, t, 1.421413741f);
    y = fmaf(y, t, -0.284496736f);
    y = fmaf(y, t, 0.254829592f);
    y *= t * __expf(-a * a);  // erfc(|x|)
    const float one_plus_erf = x >= 0.f ? 2.f - y : y;
    return 0.5f * v * one_plus_erf;
}

}  // namespace st
