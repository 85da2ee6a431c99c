// Internal glue between the drop-in transformer layer and the engine.
#pragma once

#include <cuda_runtime.h>

#include <cstdint>
#include <mutex>
#include <vector>

#include "spectree/transformer.hpp"

namespace spectree::detail {

// Device mirror of a KVCache: [layer][head][Lmax][head_dim] f64.
struct DeviceKV {
    double* k = nullptr;
    double* v = nullptr;
    int layers = 0, H = 0, Lmax = 0, Dh = 0;
    // true while the device rows are the source of truth (engine-private
    // caches): passes then skip the host<->device row traffic entirely.
    bool authoritative = false;
    size_t layer_elems() const { return (size_t)H * Lmax * Dh; }
    void release() {
        if (k) cudaFree(k);
        if (v) cudaFree(v);
        k = v = nullptr;
    }
    ~DeviceKV() { release(); }
};

std::recursive_mutex& compat_mutex();
cudaStream_t compat_stream();

// Engine-private caches keep their rows on the device only. Turning it on
// first sizes the device mirror for max_positions + scratch_rows rows: a tree
// pass writes node u at row P + u (rows are indexed by node id, positions by
// depth), so a branching tree near the position limit needs up to
// max_tree_nodes rows past P while its positions stay below max_positions.
void set_device_authoritative(KVCache& cache, bool on, int scratch_rows = 0);

// One batched pass in device-authoritative mode; returns the per-row greedy
// outputs and (via argmax_dev) their device copy, valid until the next pass.
std::vector<TokenId> device_pass(const ModelWeights& w, KVCache& cache,
                                 const std::vector<TokenId>& tokens,
                                 const std::vector<int32_t>& positions, int P,
                                 const std::vector<uint64_t>& masks, int W,
                                 int32_t** argmax_dev);

}  // namespace spectree::detail
