// Ancestor-or-self bitmasks of preorder token trees (K1's tree mask), as a
// block-level device function shared by st_build_masks and the fused
// append + masks launch (st_tree_prepare).
//
// mask[b][u][w] bit j: tree node 64*w + j is an ancestor-or-self of node u —
// the per-node path S_u of the reference's TokenTree::ancestors
// (proj/src/token_tree.cpp:130-139) as a bitmask. One thread per (request,
// node); the request's parent row is staged in shared memory first, then the
// walk up the parent chain (ids strictly decrease) emits the words high word
// first, so no per-thread word array is needed.
#pragma once

#include <cstdint>

namespace st {

// Block `bx` of request `b` (blockDim.x threads, nodes bx*blockDim.x + tid);
// s_par holds at least min(T, (bx+1)*blockDim.x) ints.
__device__ __forceinline__ void build_masks_block(const int32_t* __restrict__ parent,
                                                  const int32_t* __restrict__ n_nodes, int T, int W,
                                                  uint64_t* __restrict__ mask, int bx, int b,
                                                  int* s_par) {
    const int u = bx * blockDim.x + threadIdx.x;
    const int n = n_nodes[b];
    const int upto = min(n, (int)((bx + 1) * blockDim.x));  // nodes this block needs
    const int32_t* par = parent + (int64_t)b * T;
    for (int v = threadIdx.x; v < upto; v += blockDim.x) s_par[v] = par[v];
    __syncthreads();
    if (u >= T) return;
    uint64_t* mu = mask + ((int64_t)b * T + u) * W;
    int wi = W - 1;
    if (u < n) {
        uint64_t acc = 0;
        for (int v = u; v >= 0;) {
            const int vw = v >> 6;
            while (wi > vw) {
                mu[wi] = acc;
                acc = 0;
                --wi;
            }
            acc |= 1ull << (v & 63);
            const int pv = s_par[v];
            v = pv < v ? pv : -1;  // preorder: parent id < child id (stop on malformed input)
        }
        mu[wi] = acc;
        --wi;
    }
    for (; wi >= 0; --wi) mu[wi] = 0;
}

}  // namespace st
