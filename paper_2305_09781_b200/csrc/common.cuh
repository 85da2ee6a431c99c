// Shared helpers for the sm_100a kernels and the C-ABI layer.
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <string>
#include <utility>

#include "spectree_capi.h"

namespace st {

// Thread-local last error (st_last_error_message).
void set_error(const std::string& msg);
const std::string& last_error();

// Returns ST_ERR_NO_DEVICE when no CUDA device is visible (no CPU fallback).
st_status require_device();

inline cudaStream_t as_stream(void* s) { return reinterpret_cast<cudaStream_t>(s); }

#define ST_CHECK_ARG(cond, code, msg)                      \
    do {                                                   \
        if (!(cond)) {                                     \
            ::st::set_error(std::string(__func__) + ": " + (msg)); \
            return (code);                                 \
        }                                                  \
    } while (0)

#define ST_CUDA_TRY(expr)                                                            \
    do {                                                                             \
        cudaError_t _e = (expr);                                                     \
        if (_e != cudaSuccess) {                                                     \
            ::st::set_error(std::string(__func__) + ": " #expr ": " + cudaGetErrorString(_e)); \
            return ST_ERR_CUDA;                                                      \
        }                                                                            \
    } while (0)

#define ST_LAUNCH_CHECK() ST_CUDA_TRY(cudaGetLastError())

inline size_t dtype_size(st_dtype t) {
    switch (t) {
        case ST_F16: return 2;
        case ST_BF16: return 2;
        case ST_F32: return 4;
        case ST_F64: return 8;
    }
    return 0;
}

// ------------------------------------------- programmatic dependent launch ---
// Every path kernel is launched with programmatic stream serialization: its
// grid may be scheduled while the previous kernel on the stream drains, runs
// its prologue (barrier init, TMEM alloc, tensor-map prefetch — nothing that
// reads another kernel's output) and then blocks in pdl_wait() until that
// kernel has completed and its writes are visible. Because every kernel waits
// before it exits, completion stays transitive along the stream.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() {
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}

// cooperative: the grid is launched as a cooperative kernel — the runtime
// guarantees every CTA is co-resident (or fails the launch), which a
// persistent grid whose CTAs wait on each other's flags relies on (K1's split
// pairs) when other work (NCCL kernels, MPS clients) shares the device.
template <typename... KArgs, typename... Args>
cudaError_t launch_pdl_ex(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                          cudaStream_t stream, bool cooperative, int cluster_x, Args&&... args) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = stream;
    cudaLaunchAttribute attr[3];
    int n = 0;
    attr[n].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[n++].val.programmaticStreamSerializationAllowed = 1;
    if (cooperative) {
        attr[n].id = cudaLaunchAttributeCooperative;
        attr[n++].val.cooperative = 1;
    }
    if (cluster_x > 1) {
        attr[n].id = cudaLaunchAttributeClusterDimension;
        attr[n].val.clusterDim.x = (unsigned)cluster_x;
        attr[n].val.clusterDim.y = 1;
        attr[n++].val.clusterDim.z = 1;
    }
    cfg.attrs = attr;
    cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, kernel, std::forward<Args>(args)...);
}

template <typename... KArgs, typename... Args>
cudaError_t launch_pdl(void (*kernel)(KArgs...), dim3 grid, dim3 block, size_t smem,
                       cudaStream_t stream, Args&&... args) {
    return launch_pdl_ex(kernel, grid, block, smem, stream, false, 1, std::forward<Args>(args)...);
}

// ----------------------------------------------------------- conversions ---
template <class T> struct acc_of { using type = float; };
template <> struct acc_of<double> { using type = double; };

template <class A> __device__ __forceinline__ A to_acc(__half x) { return (A)__half2float(x); }
template <class A> __device__ __forceinline__ A to_acc(__nv_bfloat16 x) { return (A)__bfloat162float(x); }
template <class A> __device__ __forceinline__ A to_acc(float x) { return (A)x; }
template <class A> __device__ __forceinline__ A to_acc(double x) { return (A)x; }

template <class T> __device__ __forceinline__ T from_acc(float x);
template <> __device__ __forceinline__ __half from_acc<__half>(float x) { return __float2half_rn(x); }
template <> __device__ __forceinline__ __nv_bfloat16 from_acc<__nv_bfloat16>(float x) { return __float2bfloat16_rn(x); }
template <> __device__ __forceinline__ float from_acc<float>(float x) { return x; }
template <> __device__ __forceinline__ double from_acc<double>(float x) { return (double)x; }
template <class T> __device__ __forceinline__ T from_acc_d(double x);
template <> __device__ __forceinline__ double from_acc_d<double>(double x) { return x; }

}  // namespace st

// Dispatch an st_dtype onto a C++ element type.
#define ST_DISPATCH_DTYPE(DT, T, ...)                      \
    switch (DT) {                                          \
        case ST_F16: { using T = __half; __VA_ARGS__; break; }        \
        case ST_BF16: { using T = __nv_bfloat16; __VA_ARGS__; break; } \
        case ST_F32: { using T = float; __VA_ARGS__; break; }         \
        case ST_F64: { using T = double; __VA_ARGS__; break; }        \
        default: ::st::set_error("unknown dtype"); return ST_ERR_INVALID_ARGUMENT; \
    }
