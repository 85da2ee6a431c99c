// Completion signalling for the fused head-sharded all-gather (C4): after a
// rank's K1 has stored its rows into every peer's buffer, one release store
// per peer publishes an epoch; a consumer holds its stream until all ranks'
// epochs have arrived. This replaces the NCCL all-gather's synchronisation;
// the data itself already moved inside K1's epilogue.
#include "common.cuh"

namespace st {
namespace {

__global__ void peer_signal_kernel(uint32_t* const* signals, int world, int rank, uint32_t epoch) {
    pdl_wait();  // K1 has completed: its peer stores are performed
    const int k = threadIdx.x;
    if (k < world) {
        __threadfence_system();
        uint32_t* slot = signals[k] + rank;
        asm volatile("st.release.sys.global.u32 [%0], %1;" ::"l"(slot), "r"(epoch) : "memory");
    }
}

__global__ void peer_wait_kernel(const uint32_t* sig, int world, uint32_t epoch) {
    pdl_wait();
    const int k = threadIdx.x;
    if (k < world) {
        unsigned long long t0;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t0));
        for (;;) {
            uint32_t v;
            asm volatile("ld.acquire.sys.global.u32 %0, [%1];" : "=r"(v) : "l"(sig + k) : "memory");
            if ((int32_t)(v - epoch) >= 0) break;
            unsigned long long t;
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
            if (t - t0 > 10000000000ull) __trap();  // a peer never signalled: fail, don't hang
            __nanosleep(64);
        }
    }
    __syncthreads();
    pdl_trigger();
}

}  // namespace
}  // namespace st

extern "C" {

st_status st_peer_signal(uint32_t* const* signals, int world, int rank, uint32_t epoch,
                         void* stream) {
    if (st_status e = st::require_device()) return e;
    ST_CHECK_ARG(signals && world >= 1 && world <= 1024 && rank >= 0 && rank < world,
                 ST_ERR_INVALID_ARGUMENT, "bad signal arguments");
    ST_CUDA_TRY(st::launch_pdl(st::peer_signal_kernel, dim3(1), dim3((world + 31) / 32 * 32), 0,
                               st::as_stream(stream), signals, world, rank, epoch));
    return ST_OK;
}

st_status st_peer_wait(const uint32_t* my_signals, int world, uint32_t epoch, void* stream) {
    if (st_status e = st::require_device()) return e;
    ST_CHECK_ARG(my_signals && world >= 1 && world <= 1024, ST_ERR_INVALID_ARGUMENT,
                 "bad signal arguments");
    ST_CUDA_TRY(st::launch_pdl(st::peer_wait_kernel, dim3(1), dim3((world + 31) / 32 * 32), 0,
                               st::as_stream(stream), my_signals, world, epoch));
    return ST_OK;
}

}  // extern "C"
