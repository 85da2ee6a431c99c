// Verification-step plan: the batch's whole step —
// ancestor masks -> K1 -> K3 argmax -> K3 walk fused with the K2 commit — as
// one prepared object. st_verify_plan_run issues the four launches with
// programmatic dependent launch, so consecutive steps chain with no boundary
// between them (a CUDA graph per step pays one: graph replays do not overlap),
// and K1's tensor maps and schedule parameters are encoded once, not per call.
#include <cstdlib>

#include "common.cuh"
#include "tree_attn.h"

struct st_verify_plan {
    st_verify_step_desc d;
    bool tc = false;
    st::TcLaunch k1;
};

extern "C" {

st_status st_verify_plan_create(const st_verify_step_desc* d, st_verify_plan** out) {
    if (st_status e = st::require_device()) return e;
    ST_CHECK_ARG(d && out, ST_ERR_INVALID_ARGUMENT, "null pointer");
    const st_attn_args& a = d->attn;
    ST_CHECK_ARG(d->tokens && d->parent && d->logits && d->verified && d->ids && d->len &&
                     d->verify_workspace && a.mask && a.prefix_len && a.n_nodes && a.o &&
                     a.k_cache && a.v_cache && a.q,
                 ST_ERR_INVALID_ARGUMENT, "null pointer");
    ST_CHECK_ARG(a.k_tree || (d->k_new && d->v_new), ST_ERR_INVALID_ARGUMENT,
                 "cache mode (k_tree == NULL) needs k_new / v_new to append");
    ST_CHECK_ARG(d->V >= 1 && a.B >= 1 && a.T >= 1, ST_ERR_SHAPE_MISMATCH, "bad shape");
    auto* p = new st_verify_plan;
    p->d = *d;
    p->tc = st_tree_attention_path(&a) == 2;
    if (p->tc) {
        if (a.workspace_bytes < st_tree_attention_workspace_size(&a) || !a.workspace) {
            delete p;
            st::set_error("st_verify_plan_create: K1 workspace too small");
            return ST_ERR_INVALID_ARGUMENT;
        }
        if (st_status e = st::tree_attention_tc_prepare(&a, nullptr, &p->k1)) {
            delete p;
            return e;
        }
    }
    *out = p;
    return ST_OK;
}

st_status st_verify_plan_run(st_verify_plan* p, void* stream) {
    ST_CHECK_ARG(p != nullptr, ST_ERR_INVALID_ARGUMENT, "null plan");
    const st_verify_step_desc& d = p->d;
    const st_attn_args& a = d.attn;
    uint64_t* mask = const_cast<uint64_t*>(a.mask);
    if (a.k_tree) {  // the tree rows stay in their own tensors: masks only
        if (st_status e = st_build_masks_early(d.parent, a.n_nodes, a.B, a.T, a.W, mask, stream))
            return e;
    } else {         // the reference's cache discipline: K2 append + masks
        if (st_status e = st_tree_prepare(a.dtype, a.B, a.T, a.Hkv, a.D, a.Lmax, d.k_new, d.v_new,
                                          a.prefix_len, a.n_nodes, const_cast<void*>(a.k_cache),
                                          const_cast<void*>(a.v_cache), d.parent, a.W, mask,
                                          stream))
            return e;
    }
    if (p->tc) {
        if (st_status e = st::tree_attention_tc_launch(p->k1, st::as_stream(stream))) return e;
    } else {
        if (st_status e = st_tree_attention(&a, stream)) return e;
    }
    const int64_t layer = (int64_t)a.B * a.Hkv * a.Lmax * a.D;
    // K1 releases its dependents once past its own griddepcontrol.wait and
    // nothing it writes is read by the argmax (logits, node counts are step
    // inputs): the argmax blocks stream the logits on the SMs K1's tail frees
    // (ST_K3_EARLY=0: wait for K1 first)
    static const bool early = !(getenv("ST_K3_EARLY") && atoi(getenv("ST_K3_EARLY")) == 0);
    auto* compact = early && p->tc ? st::verify_greedy_compact_early : st_verify_greedy_compact;
    return compact(d.logits, a.B, a.T, d.V, d.tokens, d.parent, a.n_nodes,
                                    d.budget, d.eos, nullptr, d.verified, d.ids, d.len,
                                    d.verify_workspace, a.dtype, a.Hkv, a.D, a.Lmax, 1, layer,
                                    a.prefix_len, d.new_prefix_len, a.k_tree, a.v_tree, 0,
                                    const_cast<void*>(a.k_cache), const_cast<void*>(a.v_cache),
                                    stream);
}

void st_verify_plan_destroy(st_verify_plan* p) { delete p; }

}  // extern "C"
