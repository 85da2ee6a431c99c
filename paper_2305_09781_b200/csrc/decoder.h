// Internal around-path decoder kernels (csrc/decoder.cu).
#pragma once
#include <cuda_runtime.h>

#include <cstdint>

#include "spectree_capi.h"

namespace st {
template <class T>
st_status embed(const T* tok_emb, const T* pos_emb, const int32_t* tokens, const int32_t* pos,
                int n, int d, T* x, cudaStream_t s);
template <class T>
st_status layernorm(const T* x, const T* g, const T* b, int n, int d, T* out, cudaStream_t s);
template <class T>
st_status gemm(const T* A, const T* W, T* C, int M, int N, int K, bool accumulate, cudaStream_t s);
template <class T>
st_status gelu(T* x, int64_t n, cudaStream_t s);
template <class T>
st_status argmax_rows(const T* x, int rows, int V, int32_t* out, cudaStream_t s);
}  // namespace st
