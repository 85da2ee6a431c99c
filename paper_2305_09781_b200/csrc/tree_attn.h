// Internal K1 entry points (the C-ABI dispatcher lives in tree_attn.cu).
#pragma once
#include <cuda_runtime.h>

#include "spectree_capi.h"

namespace st {
st_status tree_attention_cc(const st_attn_args* a, cudaStream_t s);
// tcgen05 path: fp16/bf16, D == 128, G*T <= 128.
bool tree_attention_tc_supported(const st_attn_args* a);
size_t tree_attention_tc_workspace(const st_attn_args* a);
// po: head-sharded output (fused all-gather), or null for a->o.
st_status tree_attention_tc(const st_attn_args* a, cudaStream_t s, const st_peer_out* po = nullptr);
}  // namespace st
