// K2: KV-cache append of the tree nodes' K/V and in-place compaction of the
// accepted root-to-node path.
//
// Reference behaviour being replaced:
//   * chain rows are written straight into cache positions base+i
//     (proj/src/transformer.cpp:265-268), siblings overwriting each other;
//   * after verify, run_speculative re-decodes every accepted token one at a
//     time to repair the cache (proj/src/engine.cpp:123-129).
// Here the tree's rows live at [P, P+n) indexed by preorder node id, and after
// verification the accepted rows (root + matched path) are moved to
// [P, P+n_keep) — one pass over 2*(n_keep)*Hkv*D elements per layer instead of
// n_keep full forward passes.
//
// In-place safety: ids are strictly increasing with
// ids[k] >= k, so copying row ids[k] -> k in increasing k never overwrites a
// source that a LATER copy still needs; the kernel therefore walks k
// sequentially (one barrier per row) while all threads of the block copy the
// row's Hkv*D elements in parallel with 16-byte vectors.
#include <algorithm>

#include "common.cuh"
#include "kv_move.cuh"
#include "tree_masks.cuh"

namespace st {
namespace {

// One block per (b, u) tree row: copies Hkv rows of D elements for K and V.
// The node's Hkv*D source elements are contiguous; each thread keeps kUnroll
// K and V vectors in flight before storing them (the copy is latency-bound
// otherwise: one 16 B load per thread per round trip).
constexpr int kAppendThreads = 128;
constexpr int kAppendUnroll = 4;

template <class V>
__device__ __forceinline__ void kv_append_row(const char* __restrict__ k_new, const char* __restrict__ v_new,
                                              const int32_t* __restrict__ prefix_len,
                                              const int32_t* __restrict__ n_nodes,
                                              char* __restrict__ k_cache, char* __restrict__ v_cache,
                                              int T, int Hkv, int row_vecs, int64_t Lmax, int b, int u) {
    if (u >= n_nodes[b]) return;
    const int64_t P = prefix_len[b];
    const int total = Hkv * row_vecs;
    const V* ks = reinterpret_cast<const V*>(k_new) + ((int64_t)b * T + u) * total;
    const V* vs = reinterpret_cast<const V*>(v_new) + ((int64_t)b * T + u) * total;
    V* kd = reinterpret_cast<V*>(k_cache) + ((int64_t)b * Hkv * Lmax + P + u) * row_vecs;
    V* vd = reinterpret_cast<V*>(v_cache) + ((int64_t)b * Hkv * Lmax + P + u) * row_vecs;
    const int64_t head_stride = Lmax * row_vecs;  // vectors between heads in the cache
    for (int i0 = threadIdx.x; i0 < total; i0 += kAppendThreads * kAppendUnroll) {
        V kx[kAppendUnroll], vx[kAppendUnroll];
#pragma unroll
        for (int r = 0; r < kAppendUnroll; ++r) {
            const int i = i0 + r * kAppendThreads;
            if (i < total) {
                kx[r] = ks[i];
                vx[r] = vs[i];
            }
        }
#pragma unroll
        for (int r = 0; r < kAppendUnroll; ++r) {
            const int i = i0 + r * kAppendThreads;
            if (i < total) {
                const int h = i / row_vecs, e = i - h * row_vecs;
                kd[h * head_stride + e] = kx[r];
                vd[h * head_stride + e] = vx[r];
            }
        }
    }
}

template <class V>
__global__ void __launch_bounds__(kAppendThreads)
kv_append_kernel(const char* __restrict__ k_new, const char* __restrict__ v_new,
                 const int32_t* __restrict__ prefix_len, const int32_t* __restrict__ n_nodes,
                 char* __restrict__ k_cache, char* __restrict__ v_cache, int T, int Hkv,
                 int row_vecs, int64_t Lmax) {
    pdl_wait();
    pdl_trigger();
    kv_append_row<V>(k_new, v_new, prefix_len, n_nodes, k_cache, v_cache, T, Hkv, row_vecs, Lmax,
                     blockIdx.y, blockIdx.x);
}

// st_tree_prepare: blocks x < T append tree row x of request y; the remaining
// ceil(T / kAppendThreads) blocks build request y's masks.
template <class V>
__global__ void __launch_bounds__(kAppendThreads)
tree_prepare_kernel(const char* __restrict__ k_new, const char* __restrict__ v_new,
                    const int32_t* __restrict__ prefix_len, const int32_t* __restrict__ n_nodes,
                    char* __restrict__ k_cache, char* __restrict__ v_cache, int T, int Hkv,
                    int row_vecs, int64_t Lmax, const int32_t* __restrict__ parent, int W,
                    uint64_t* __restrict__ mask) {
    extern __shared__ int s_par[];  // T ints (mask blocks stage the parent row)
    pdl_wait();
    pdl_trigger();
    if ((int)blockIdx.x < T)
        kv_append_row<V>(k_new, v_new, prefix_len, n_nodes, k_cache, v_cache, T, Hkv, row_vecs, Lmax,
                         blockIdx.y, blockIdx.x);
    else
        build_masks_block(parent, n_nodes, T, W, mask, blockIdx.x - T, blockIdx.y, s_par);
}

// st_kv_compact / st_kv_commit_tree: block (b, layer * nhc + hc) moves the
// accepted rows of its hpb KV heads of one layer (kv_move.cuh: chunked, no
// per-row barrier chain) — in place (rows 1.. from cache row P + ids[k]), or
// from the tree's own K/V (k_tree != NULL: rows 0.. from tree[b][ids[k]][h]).
template <class V>
__global__ void __launch_bounds__(256)
kv_compact_kernel(const int32_t* __restrict__ ids, int ids_stride, const int32_t* __restrict__ n_keep,
                  const int32_t* __restrict__ prefix_len, int32_t* __restrict__ new_prefix_len,
                  char* k_cache, char* v_cache, int Hkv, int row_vecs, int64_t Lmax,
                  int64_t layer_stride_bytes, int nhc, int hpb, const char* k_tree,
                  const char* v_tree, int64_t tree_layer_stride_bytes, int T) {
    extern __shared__ int s_ids[];  // ids_stride ints
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.x, layer = blockIdx.y / nhc, hc = blockIdx.y % nhc;
    const int keep = min(n_keep[b], ids_stride);
    const int64_t P = prefix_len[b];
    for (int k = threadIdx.x; k < keep; k += blockDim.x) s_ids[k] = ids[(int64_t)b * ids_stride + k];
    __syncthreads();
    if (new_prefix_len && blockIdx.y == 0 && threadIdx.x == 0) new_prefix_len[b] = (int32_t)(P + keep);
    const int h0 = hc * hpb, nh = min(hpb, Hkv - h0);
    const int kfirst = k_tree ? 0 : 1;
    if (keep <= kfirst || nh <= 0) return;
    move_rows_block<V>(s_ids, keep, kfirst, b, h0, nh, Hkv, row_vecs, Lmax, P,
                       k_cache + layer * layer_stride_bytes, v_cache + layer * layer_stride_bytes,
                       k_tree ? k_tree + layer * tree_layer_stride_bytes : nullptr,
                       v_tree ? v_tree + layer * tree_layer_stride_bytes : nullptr, T);
}

}  // namespace
}  // namespace st

extern "C" {

st_status st_kv_append(st_dtype dtype, int B, int T, int Hkv, int D, int64_t Lmax,
                       const void* k_new, const void* v_new, const int32_t* prefix_len,
                       const int32_t* n_nodes, void* k_cache, void* v_cache, void* stream) {
    if (st_status e = st::require_device()) return e;
    ST_CHECK_ARG(B >= 0 && T >= 1 && Hkv >= 1 && D >= 1 && Lmax >= T, ST_ERR_SHAPE_MISMATCH,
                 "bad shape");
    ST_CHECK_ARG(st::dtype_size(dtype) != 0, ST_ERR_INVALID_ARGUMENT, "bad dtype");
    if (B == 0) return ST_OK;
    ST_CHECK_ARG(k_new && v_new && prefix_len && n_nodes && k_cache && v_cache,
                 ST_ERR_INVALID_ARGUMENT, "null pointer");
    const int64_t row_bytes = (int64_t)D * st::dtype_size(dtype);
    const dim3 grid(T, B);
    auto s = st::as_stream(stream);
    const bool vec = row_bytes % 16 == 0;
    ST_CUDA_TRY(st::launch_pdl(vec ? st::kv_append_kernel<int4> : st::kv_append_kernel<char>, grid,
                               dim3(st::kAppendThreads), 0, s, (const char*)k_new,
                               (const char*)v_new, prefix_len, n_nodes, (char*)k_cache,
                               (char*)v_cache, T, Hkv, (int)(vec ? row_bytes / 16 : row_bytes),
                               Lmax));
    ST_LAUNCH_CHECK();
    return ST_OK;
}

st_status st_tree_prepare(st_dtype dtype, int B, int T, int Hkv, int D, int64_t Lmax,
                          const void* k_new, const void* v_new, const int32_t* prefix_len,
                          const int32_t* n_nodes, void* k_cache, void* v_cache,
                          const int32_t* parent, int W, uint64_t* mask, void* stream) {
    if (st_status e = st::require_device()) return e;
    ST_CHECK_ARG(B >= 0 && T >= 1 && Hkv >= 1 && D >= 1 && Lmax >= T, ST_ERR_SHAPE_MISMATCH,
                 "bad shape");
    ST_CHECK_ARG(W >= (T + 63) / 64 && W <= 32, ST_ERR_SHAPE_MISMATCH,
                 "bad shape (need ceil(T/64) <= W <= 32)");
    ST_CHECK_ARG(st::dtype_size(dtype) != 0, ST_ERR_INVALID_ARGUMENT, "bad dtype");
    if (B == 0) return ST_OK;
    ST_CHECK_ARG(k_new && v_new && prefix_len && n_nodes && k_cache && v_cache && parent && mask,
                 ST_ERR_INVALID_ARGUMENT, "null pointer");
    ST_CHECK_ARG(B <= 65535 && T <= 12288, ST_ERR_SHAPE_MISMATCH, "too many requests or nodes");
    const int64_t row_bytes = (int64_t)D * st::dtype_size(dtype);
    const dim3 grid(T + (T + st::kAppendThreads - 1) / st::kAppendThreads, B);
    const size_t smem = (size_t)T * sizeof(int32_t);
    const bool vec = row_bytes % 16 == 0;
    ST_CUDA_TRY(st::launch_pdl(vec ? st::tree_prepare_kernel<int4> : st::tree_prepare_kernel<char>,
                               grid, dim3(st::kAppendThreads), smem, st::as_stream(stream),
                               (const char*)k_new, (const char*)v_new, prefix_len, n_nodes,
                               (char*)k_cache, (char*)v_cache, T, Hkv,
                               (int)(vec ? row_bytes / 16 : row_bytes), Lmax, parent, W, mask));
    ST_LAUNCH_CHECK();
    return ST_OK;
}

static st_status kv_commit(st_dtype dtype, int B, int Hkv, int D, int64_t Lmax, int n_layers,
                           int64_t layer_stride, const int32_t* ids, int ids_stride,
                           const int32_t* n_keep, const int32_t* prefix_len,
                           int32_t* new_prefix_len, const void* k_tree, const void* v_tree, int T,
                           int64_t tree_layer_stride, void* k_cache, void* v_cache, void* stream) {
    if (st_status e = st::require_device()) return e;
    ST_CHECK_ARG(B >= 0 && Hkv >= 1 && D >= 1 && n_layers >= 1 && ids_stride >= 1,
                 ST_ERR_SHAPE_MISMATCH, "bad shape");
    ST_CHECK_ARG(st::dtype_size(dtype) != 0, ST_ERR_INVALID_ARGUMENT, "bad dtype");
    if (B == 0) return ST_OK;
    ST_CHECK_ARG(ids && n_keep && prefix_len && k_cache && v_cache, ST_ERR_INVALID_ARGUMENT,
                 "null pointer");
    ST_CHECK_ARG(ids_stride <= 16384, ST_ERR_SHAPE_MISMATCH, "ids_stride > 16384");
    const int64_t es = (int64_t)st::dtype_size(dtype);
    const int64_t row_bytes = (int64_t)D * es;
    const bool vec = row_bytes % 16 == 0;
    const int row_vecs = (int)(vec ? row_bytes / 16 : row_bytes);
    // heads per block: about 2 KB of K+V per accepted row per block
    const int hpb = std::max(1, std::min(Hkv, (vec ? 64 : 1024) / std::max(1, row_vecs)));
    const int nhc = (Hkv + hpb - 1) / hpb;
    ST_CHECK_ARG(B <= 2147483647 && (int64_t)n_layers * nhc <= 65535, ST_ERR_SHAPE_MISMATCH,
                 "too many layers x heads");
    auto s = st::as_stream(stream);
    ST_CUDA_TRY(st::launch_pdl(vec ? st::kv_compact_kernel<int4> : st::kv_compact_kernel<char>,
                               dim3(B, n_layers * nhc), dim3(256), (size_t)ids_stride * sizeof(int), s,
                               ids, ids_stride, n_keep, prefix_len, new_prefix_len, (char*)k_cache,
                               (char*)v_cache, Hkv, row_vecs, Lmax, layer_stride * es, nhc, hpb,
                               (const char*)k_tree, (const char*)v_tree, tree_layer_stride * es, T));
    ST_LAUNCH_CHECK();
    return ST_OK;
}

st_status st_kv_compact(st_dtype dtype, int B, int Hkv, int D, int64_t Lmax, int n_layers,
                        int64_t layer_stride, const int32_t* ids, int ids_stride,
                        const int32_t* n_keep, const int32_t* prefix_len,
                        int32_t* new_prefix_len, void* k_cache, void* v_cache, void* stream) {
    return kv_commit(dtype, B, Hkv, D, Lmax, n_layers, layer_stride, ids, ids_stride, n_keep,
                     prefix_len, new_prefix_len, nullptr, nullptr, 0, 0, k_cache, v_cache, stream);
}

st_status st_kv_commit_tree(st_dtype dtype, int B, int T, int Hkv, int D, int64_t Lmax,
                            int n_layers, int64_t layer_stride, const int32_t* ids,
                            int ids_stride, const int32_t* n_keep, const int32_t* prefix_len,
                            int32_t* new_prefix_len, const void* k_tree, const void* v_tree,
                            int64_t tree_layer_stride, void* k_cache, void* v_cache,
                            void* stream) {
    ST_CHECK_ARG(k_tree && v_tree && T >= 1, ST_ERR_INVALID_ARGUMENT, "k_tree / v_tree / T");
    return kv_commit(dtype, B, Hkv, D, Lmax, n_layers, layer_stride, ids, ids_stride, n_keep,
                     prefix_len, new_prefix_len, k_tree, v_tree, T, tree_layer_stride, k_cache,
                     v_cache, stream);
}

}  // extern "C"

// ------------------------------------------------------------------------
// Head-sharded attention (C4): every rank computes K1 for its Hl heads and the
// ranks all-gather their [B][T][Hl][D] outputs (NCCL, contiguous per rank);
// this reorders the gathered [world][B][T][Hl][D] into [B][T][world*Hl][D]
// (the row layout the output projection consumes). 16-byte vector copies.
namespace st {
namespace {
__global__ void heads_layout_kernel(const int4* __restrict__ src, int4* __restrict__ dst,
                                    int world, int BT, int row_vecs /* Hl*D*s/16 */) {
    const int64_t total = (int64_t)world * BT * row_vecs;
    for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < total;
         i += (int64_t)gridDim.x * blockDim.x) {
        const int e = (int)(i % row_vecs);
        const int64_t rest = i / row_vecs;
        const int bt = (int)(rest % BT);
        const int r = (int)(rest / BT);
        dst[((int64_t)bt * world + r) * row_vecs + e] = src[i];
    }
}
}  // namespace
}  // namespace st

extern "C" st_status st_heads_gather_layout(st_dtype dtype, int world, int B, int T, int Hl, int D,
                                            const void* gathered, void* out, void* stream) {
    if (st_status e = st::require_device()) return e;
    ST_CHECK_ARG(world >= 1 && B >= 0 && T >= 1 && Hl >= 1 && D >= 1, ST_ERR_SHAPE_MISMATCH,
                 "bad shape");
    const int64_t row_bytes = (int64_t)Hl * D * st::dtype_size(dtype);
    ST_CHECK_ARG(row_bytes % 16 == 0 && st::dtype_size(dtype) != 0, ST_ERR_SHAPE_MISMATCH,
                 "Hl*D*sizeof(dtype) must be a multiple of 16 bytes");
    if (B == 0) return ST_OK;
    ST_CHECK_ARG(gathered && out && gathered != out, ST_ERR_INVALID_ARGUMENT,
                 "null or aliased pointer");
    const int row_vecs = (int)(row_bytes / 16);
    const int64_t total = (int64_t)world * B * T * row_vecs;
    const unsigned blocks = (unsigned)std::min<int64_t>((total + 255) / 256, 148 * 16);
    st::heads_layout_kernel<<<blocks, 256, 0, st::as_stream(stream)>>>(
        (const int4*)gathered, (int4*)out, world, B * T, row_vecs);
    ST_LAUNCH_CHECK();
    return ST_OK;
}
