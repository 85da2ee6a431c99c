// K1 tcgen05 path — placeholder until the tensor-core kernel lands.
#include "common.cuh"
#include "tree_attn.h"

namespace st {
bool tree_attention_tc_supported(const st_attn_args*) { return false; }
size_t tree_attention_tc_workspace(const st_attn_args*) { return 0; }
st_status tree_attention_tc(const st_attn_args*, cudaStream_t) {
    set_error("tcgen05 path not built");
    return ST_ERR_UNSUPPORTED;
}
}  // namespace st
