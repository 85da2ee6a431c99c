// C-ABI housekeeping: version, last-error, device probe.
#include "common.cuh"

namespace st {

static thread_local std::string g_last_error;

void set_error(const std::string& msg) { g_last_error = msg; }
const std::string& last_error() { return g_last_error; }

st_status require_device() {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
        cudaGetLastError();  // clear the sticky "no device" error
        set_error("no CUDA device visible: the spectree B200 path has no CPU fallback");
        return ST_ERR_NO_DEVICE;
    }
    return ST_OK;
}

}  // namespace st

extern "C" {

int st_abi_version(void) { return ST_ABI_VERSION; }

const char* st_last_error_message(void) { return st::last_error().c_str(); }

int st_device_count(void) {
    int n = 0;
    if (cudaGetDeviceCount(&n) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    return n;
}

}  // extern "C"
