// K4 placeholder (multi-step speculative sampling lands in a later commit).
#include "common.cuh"

extern "C" st_status st_verify_mss(const float*, const float*, int, int, int, const int32_t*,
                                   const int32_t*, const int32_t*, float, const float*, int,
                                   int32_t*, int32_t*, int32_t*, void*) {
    if (st_status e = st::require_device()) return e;
    st::set_error("st_verify_mss: not built yet");
    return ST_ERR_UNSUPPORTED;
}
