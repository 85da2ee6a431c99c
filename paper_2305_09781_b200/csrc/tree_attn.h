// Internal K1 entry points (the C-ABI dispatcher lives in tree_attn.cu).
#pragma once
#include <cuda_runtime.h>

#include <cuda.h>

#include "spectree_capi.h"

namespace st {
// Parameter block of the tcgen05 kernel (tree_attn_tc.cu).
struct TcParams {
    const int32_t* prefix_len;
    const int32_t* n_nodes;
    const uint64_t* mask;
    void* o;
    float* lse;
    float* partial;      // [gridDim.x][SLOT_FLOATS]: the piece a CTA's first segment leaves
    unsigned* flags;     // [gridDim.x]: 1 while that piece is published and not yet merged
    int B, T, H, W;      // H: KV heads (one (b, h) pair per request and KV head)
    int Tq, u0;          // Q / o / lse rows per request and the node id of Q row 0
                         // (st_attn_args.q_rows / q_node0; Tq = T, u0 = 0 when unset)
    int G, Hq;           // query heads per KV head (GQA group), query heads = G * H
    int R;               // row blocks per pair: G*T <= 128 -> 1; <= 256 -> 2 (CTAs 2s, 2s+1
                         // take the two 128-row blocks of schedule slot s)
    int tree_src;        // tree rows come from k_tree/v_tree: ceil(n/BN) tiles after ceil(P/BN)
    int early_kv;        // st_attn_args.early_kv: stream committed KV before griddepcontrol.wait
    float c_log2;        // scale * log2(e)
    float scale;
    unsigned long long* trace;  // optional pipeline trace of CTA 0 (ST_K1_TRACE)
    int aligned_slack;          // whole-pair schedule allowed within this many tiles of stream-K
    int head_extra;             // split schedule: extra tiles for each pair's head piece
    int trace_cta;              // CTA whose per-tile pipeline is traced (ST_K1_TRACE_CTA)
    unsigned long long g_magic; // floor(2^64 / G) + 1, G = schedule slots: exact floor(x / G)
                                // for x < 2^40 as one 64-bit high multiply
    int o_tma;                  // `to` is valid: whole-pair last segments store o with one TMA store
    int pre_cap;                // producer fast start: tiles per ring before the CTA barrier (0: the ring)
    int most_aligned;           // whole pairs when 4G/5 <= pairs <= G (ST_K1_MOST=0: off)
    int cluster2;               // launched as 2-CTA clusters: split pairs of two pieces merge
                                // over DSMEM (the piece's (O, m, l) copied into the head's
                                // drained K ring) instead of the global publish / flag path
    // head-sharded output (st_tree_attention_allgather): rows go to every rank's
    // [B][T][H_out][D] buffer at head head_offset + h; null -> o with H_out = H
    void* const* o_peers;
    int world, head_offset, H_out;
};
// A prepared tcgen05 launch: tensor maps encoded once (a plan re-launches it).
struct TcLaunch {
    CUtensorMap tq, tk, tv, tkt, tvt;  // one box = both d halves of a tile
    CUtensorMap tk1, tv1, tkt1, tvt1;  // one d half (multicast two-row-block loads)
    CUtensorMap to;                    // o, same view as tq (TMA-store epilogue)
    TcParams prm;
    int grid;
    bool coop, m64, mw4, f16;
};
st_status tree_attention_cc(const st_attn_args* a, cudaStream_t s);
// tcgen05 path: fp16/bf16, D == 128, G*T <= 128.
bool tree_attention_tc_supported(const st_attn_args* a);
size_t tree_attention_tc_workspace(const st_attn_args* a);
// po: head-sharded output (fused all-gather), or null for a->o.
st_status tree_attention_tc(const st_attn_args* a, cudaStream_t s, const st_peer_out* po = nullptr);
st_status tree_attention_tc_prepare(const st_attn_args* a, const st_peer_out* po, TcLaunch* out);
st_status tree_attention_tc_launch(const TcLaunch& l, cudaStream_t s);
// st_verify_greedy_compact for the step plan: the argmax streams the logits
// before the previous kernel (K1) completes — it writes neither the logits
// nor the node counts — and only its key stores wait (griddepcontrol)
st_status verify_greedy_compact_early(const float* logits, int B, int T, int V, const int32_t*
                                      tokens,
                                   const int32_t* parent, const int32_t* n_nodes,
                                   const int32_t* budget, int32_t eos, int32_t* argmax,
                                   int32_t* verified, int32_t* ids, int32_t* len, void* workspace,
                                   st_dtype dtype, int Hkv, int D, int64_t Lmax, int n_layers,
                                   int64_t layer_stride, const int32_t* prefix_len,
                                   int32_t* new_prefix_len, const void* k_tree,
                                   const void* v_tree, int64_t tree_layer_stride, void* k_cache,
                                   void* v_cache, void* stream);
}  // namespace st
