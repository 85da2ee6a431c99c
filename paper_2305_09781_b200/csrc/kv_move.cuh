// K2 commit of a request's accepted rows, block-level (shared by st_kv_compact
// and st_verify_greedy_compact):
//   cache[b][h][P + k] = src row ids[k]      k = kfirst .. L-1, h in [h0, h0+nh)
// src = the cache itself (in place: cache row P + ids[k]; kfirst = 1, the root
// is already at P) or the tree's own K/V (tree[b][ids[k]][h], [B][T][Hkv][D];
// kfirst = 0). In place is safe without a per-row chain: ids are strictly
// increasing with ids[k] >= k, so a destination row k is never a source of a
// later k; within a chunk of rows every source is loaded before any
// destination is stored (one barrier), and chunks go in increasing k.
// Replaces the reference's post-verify re-decode of every accepted token
// (proj/src/engine.cpp:123-129).
#pragma once

#include <cstdint>

namespace st {

constexpr int kMoveVecs = 4;  // vectors in flight per thread per chunk

template <class V>
__device__ void move_rows_block(const int* ids, int L, int kfirst, int b, int h0, int nh, int Hkv,
                                int row_vecs, int64_t Lmax, int64_t P, char* kl, char* vl,
                                const char* ktl, const char* vtl, int T) {
    const int per_row = nh * row_vecs;  // vectors of one row, all of this block's heads
    const int cap = (int)blockDim.x * kMoveVecs;   // vectors one pass of the block moves
    // Rows wider than one pass (e.g. f64 rows of a long head dim on the byte
    // path) move one row at a time in slices of `cap` vectors: the source row
    // ids[k] > k is never a destination of an earlier row, and a later row's
    // destination is written only after this row is read completely.
    const int rows_chunk = per_row > cap ? 1 : max(1, cap / (2 * per_row));
    const int slice = min(per_row, cap);
    for (int k0 = kfirst, s0 = 0; k0 < L;) {
        const int k1 = min(L, k0 + rows_chunk);
        const int total = per_row > cap ? min(slice, per_row - s0) : (k1 - k0) * per_row;
        V kx[kMoveVecs], vx[kMoveVecs];
        int64_t dst[kMoveVecs];
#pragma unroll
        for (int r = 0; r < kMoveVecs; ++r) {
            const int i = threadIdx.x + r * blockDim.x;
            dst[r] = -1;
            if (i < total) {
                const int kk = k0 + i / per_row, rem = i % per_row + s0;
                const int h = h0 + rem / row_vecs, e = rem % row_vecs;
                const int src = ids[kk];
                const int64_t base = ((int64_t)b * Hkv + h) * Lmax + P;
                if (ktl) {
                    const int64_t so = (((int64_t)b * T + src) * Hkv + h) * row_vecs + e;
                    dst[r] = (base + kk) * row_vecs + e;
                    kx[r] = reinterpret_cast<const V*>(ktl)[so];
                    vx[r] = reinterpret_cast<const V*>(vtl)[so];
                } else if (src != kk) {
                    const int64_t so = (base + src) * row_vecs + e;
                    dst[r] = (base + kk) * row_vecs + e;
                    kx[r] = reinterpret_cast<const V*>(kl)[so];
                    vx[r] = reinterpret_cast<const V*>(vl)[so];
                }
            }
        }
        __syncthreads();  // every source of this chunk read before any store
#pragma unroll
        for (int r = 0; r < kMoveVecs; ++r) {
            if (dst[r] >= 0) {
                reinterpret_cast<V*>(kl)[dst[r]] = kx[r];
                reinterpret_cast<V*>(vl)[dst[r]] = vx[r];
            }
        }
        __syncthreads();
        if (per_row > cap && (s0 += slice) < per_row) continue;  // next slice of row k0
        s0 = 0;
        k0 = k1;
    }
}

}  // namespace st
