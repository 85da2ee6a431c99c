// K1 dispatcher: st_tree_attention (C-ABI) -> CUDA-core or tcgen05 kernel.
//
// Dispatch rule: half-precision inputs with D == 128 go to the tcgen05
// kernel; f32/f64 (the reference-parity runs) and other head dims to the
// CUDA-core kernel. Small trees (G*T < 16) used to go to the CUDA-core kernel
// because their MMAs are mostly zero rows (north star: tensor cores "only where
// GQA head-grouping x tree width makes them dense enough to pay"), but what
// pays at ANY tree size is the tiling: the tcgen05 kernel streams each KV tile
// once for all of a pair's rows, the CUDA-core kernel once per (node, head) —
// 300-700x apart on the GQA sweep (profiles/gqa_sweep.json) — and an
// M=64 tile with a few live rows skips the softmax of its empty warps.
#include "common.cuh"
#include "tree_attn.h"

namespace {

st_status validate(const st_attn_args* a) {
    ST_CHECK_ARG(a != nullptr, ST_ERR_INVALID_ARGUMENT, "null args");
    ST_CHECK_ARG(a->B >= 0 && a->T >= 1 && a->H >= 1 && a->Hkv >= 1 && a->D >= 1,
                 ST_ERR_SHAPE_MISMATCH, "bad shape");
    ST_CHECK_ARG(a->H % a->Hkv == 0, ST_ERR_SHAPE_MISMATCH, "H must be a multiple of Hkv");
    ST_CHECK_ARG(a->W * 64 >= a->T, ST_ERR_SHAPE_MISMATCH, "mask words W < ceil(T/64)");
    ST_CHECK_ARG(a->Lmax >= a->T, ST_ERR_SHAPE_MISMATCH, "cache rows Lmax < T");
    ST_CHECK_ARG((a->k_tree == nullptr) == (a->v_tree == nullptr), ST_ERR_INVALID_ARGUMENT,
                 "k_tree and v_tree must be both set or both NULL");
    return ST_OK;
}

st_status validate_ptrs(const st_attn_args* a) {
    ST_CHECK_ARG(a->B == 0 || (a->q && a->k_cache && a->v_cache && a->mask && a->prefix_len &&
                               a->n_nodes && a->o),
                 ST_ERR_INVALID_ARGUMENT, "null tensor pointer");
    return ST_OK;
}

int choose_path(const st_attn_args* a) {
    if (a->force_path == 1 || a->force_path == 2) return a->force_path;
    return st::tree_attention_tc_supported(a) ? 2 : 1;
}

}  // namespace

extern "C" {

int st_tree_attention_path(const st_attn_args* a) {
    if (validate(a) != ST_OK) return 0;
    return choose_path(a);
}

size_t st_tree_attention_workspace_size(const st_attn_args* a) {
    if (validate(a) != ST_OK) return 0;
    return choose_path(a) == 2 ? st::tree_attention_tc_workspace(a) : 0;
}

st_status st_tree_attention(const st_attn_args* a, void* stream) {
    if (st_status e = st::require_device()) return e;
    if (st_status e = validate(a)) return e;
    if (st_status e = validate_ptrs(a)) return e;
    if (a->B == 0) return ST_OK;
    const int path = choose_path(a);
    ST_CHECK_ARG(a->q_rows <= 0 || (a->q_node0 >= 0 && (int64_t)a->q_node0 + a->q_rows <= a->T),
                 ST_ERR_INVALID_ARGUMENT,
                 "st_tree_attention: q_rows slice [q_node0, q_node0 + q_rows) outside [0, T)");
    if (path == 2) {
        if (!st::tree_attention_tc_supported(a)) {
            st::set_error("st_tree_attention: tcgen05 path needs f16/bf16, D == 128, G*T <= 128");
            return ST_ERR_UNSUPPORTED;
        }
        const size_t need = st::tree_attention_tc_workspace(a);
        if (a->workspace_bytes < need || (need && !a->workspace)) {
            st::set_error("st_tree_attention: workspace too small");
            return ST_ERR_INVALID_ARGUMENT;
        }
        return st::tree_attention_tc(a, st::as_stream(stream));
    }
    return st::tree_attention_cc(a, st::as_stream(stream));
}

st_status st_tree_attention_allgather(const st_attn_args* a, const st_peer_out* po,
                                      void* stream) {
    if (st_status e = st::require_device()) return e;
    if (st_status e = validate(a)) return e;
    ST_CHECK_ARG(po && po->out && po->world >= 1 && po->rank >= 0 && po->rank < po->world,
                 ST_ERR_INVALID_ARGUMENT, "bad st_peer_out");
    ST_CHECK_ARG(a->B == 0 || (a->q && a->k_cache && a->v_cache && a->mask && a->prefix_len &&
                               a->n_nodes),
                 ST_ERR_INVALID_ARGUMENT, "null tensor pointer");
    if (a->B == 0) return ST_OK;
    if (choose_path(a) != 2 || !st::tree_attention_tc_supported(a)) {
        st::set_error("st_tree_attention_allgather: needs the tcgen05 path (f16/bf16, D == 128, "
                      "(H/Hkv)*T <= 128)");
        return ST_ERR_UNSUPPORTED;
    }
    const size_t need = st::tree_attention_tc_workspace(a);
    if (a->workspace_bytes < need || (need && !a->workspace)) {
        st::set_error("st_tree_attention_allgather: workspace too small");
        return ST_ERR_INVALID_ARGUMENT;
    }
    return st::tree_attention_tc(a, st::as_stream(stream), po);
}

}  // extern "C"
