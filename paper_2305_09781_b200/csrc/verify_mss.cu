// K4: stochastic multi-step speculative sampling (MSS) — SpecInfer's
// stochastic verification, which the reference does NOT implement
// (SPEC.md:8, :100). Contract: DESIGN.md §5 / SURVEY.md Appendix B; the fp32
// CPU oracle oracle/restate_mss.c fixes every rounding step, and this kernel
// reproduces it bit for bit given the same host-supplied uniforms:
//
//   u = root
//   loop: p = softmax(z[u] / tau)
//         for each child v of u (ascending id): r = U[k++]
//             accept if r * q_v[t_v] <= p[t_v]      -> emit t_v, u = v, continue loop
//             else p = norm(max(p - q_v, 0))        (residual renormalisation)
//         emit inverse-CDF sample of p with r = U[k++]; stop
//
// One thread-block cluster of 4 CTAs (1024 threads each) per request keeps the
// working distribution p[V] in the cluster's shared memory, a quarter per CTA.
// Every vocabulary reduction uses the fixed order of the contract: chunk owner
// t (of 256) sums the contiguous chunk [t*CH, (t+1)*CH) sequentially, the 8
// warps of chunk owners combine their 32 chunk sums with an xor butterfly and
// the 8 warp sums are added in order (exchanged over DSMEM); the exponential is
// the contract's exp_spec (fma Horner polynomial + exact power-of-two
// scaling); all fp32 operations use explicit _rn intrinsics so nothing is
// contracted. Element-wise passes (exp, normalisation, residual) use all 4096
// threads, every global read is batched, and each rejected child's q row is
// staged in shared memory once (read by the residual sum and the
// renormalisation).
#include <cfloat>

#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace st {
namespace {

constexpr int NT = 256;       // reduction lanes of the contract (chunk owners)
constexpr int kBatch = 16;    // independent global loads in flight per thread

// Asynchronous global -> shared copies (the next child's q slice is fetched
// while the current child is tested and its residual computed).
__device__ __forceinline__ void cp_async4(float* dst, const float* src) {
    asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
    asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

__device__ __forceinline__ float exp_spec(float x) {
    if (!(x > -104.0f)) return 0.0f;
    const float t = __fmul_rn(x, 1.44269504f);
    const float nf = rintf(t);
    const float f = __fsub_rn(t, nf);
    float p = 1.54035304e-4f;
    p = __fmaf_rn(p, f, 1.33335581e-3f);
    p = __fmaf_rn(p, f, 9.61812911e-3f);
    p = __fmaf_rn(p, f, 5.55041087e-2f);
    p = __fmaf_rn(p, f, 2.40226507e-1f);
    p = __fmaf_rn(p, f, 6.93147182e-1f);
    p = __fmaf_rn(p, f, 1.0f);
    const int n = (int)nf;
    if (n >= -126) return __fmul_rn(p, __uint_as_float((uint32_t)(n + 127) << 23));
    return __fmul_rn(__fmul_rn(p, __uint_as_float((uint32_t)(n + 227) << 23)),
                     __uint_as_float((uint32_t)27 << 23));
}

// ------------------------------------------------------------------------
// Cluster version: one thread-block cluster of CN CTAs per request. CTA k of
// the cluster owns the contract's chunks [k*OWN, (k+1)*OWN) — vocabulary
// elements [k*OWN*CH, (k+1)*OWN*CH) — in its shared memory, so every
// element-wise pass and every global read is spread over CN SMs. The fixed-
// order reductions are unchanged: chunk owners sum their chunks
// sequentially, the 8 warp butterflies of the contract are warps 0..1 of
// each CTA (global warp 2k+w), and the warp sums are broadcast into every
// CTA's shared memory over DSMEM (double-buffered slots, one cluster barrier
// per reduction) and added in the contract's order — bit-identical to the
// single-CTA kernel and to the oracle. Remote p[t] reads (accept test,
// inverse-CDF scan) go through DSMEM as well.
constexpr int CN = 4;              // CTAs per request (measured: 2 -> 147 us, 4 -> 132, 8 -> 189 at C3)
constexpr int NTC = 1024;          // threads per CTA
constexpr int OWN = NT / CN;       // chunk owners per CTA (2 warps)
static_assert(OWN % 32 == 0, "chunk owners fill whole warps");

struct MssCluster {
    float red[NTC / 32];           // CTA-local max
    float xsum[2][NT / 32];        // contract warp sums, every CTA's copy (double-buffered)
    float xmax[2][CN];             // per-CTA maxima
    float csum[NT];                // all chunk sums (inverse CDF; leader)
    float cum[NT];
    float pt, qt;                  // p[t], q_v[t] of the current accept test
    int pick;
};

__device__ __forceinline__ float cluster_max(float v, MssCluster& sh, int slot, cg::cluster_group& cl) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    if (lane == 0) sh.red[warp] = v;
    __syncthreads();
    if (threadIdx.x < CN) {  // thread j sends this CTA's max to CTA j
        float m = sh.red[0];
        for (int w = 1; w < NTC / 32; ++w) m = fmaxf(m, sh.red[w]);
        MssCluster* dst = cl.map_shared_rank(&sh, threadIdx.x);
        dst->xmax[slot][cl.block_rank()] = m;
    }
    cl.sync();
    float m = sh.xmax[slot][0];
#pragma unroll
    for (int j = 1; j < CN; ++j) m = fmaxf(m, sh.xmax[slot][j]);
    return m;
}

// the contract's combine: owners' chunk partials, butterfly per (global) warp,
// the 8 warp sums added in order
__device__ __forceinline__ float cluster_combine(float part, MssCluster& sh, int slot, cg::cluster_group& cl) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (warp < OWN / 32) {
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) part = __fadd_rn(part, __shfl_xor_sync(0xffffffffu, part, o));
        if (lane < CN) {  // lane j sends this warp's sum to CTA j
            MssCluster* dst = cl.map_shared_rank(&sh, lane);
            dst->xsum[slot][cl.block_rank() * (OWN / 32) + warp] = part;
        }
    }
    cl.sync();
    float tot = sh.xsum[slot][0];
#pragma unroll
    for (int w = 1; w < NT / 32; ++w) tot = __fadd_rn(tot, sh.xsum[slot][w]);
    return tot;
}

__global__ void __cluster_dims__(CN, 1, 1) __launch_bounds__(NTC)
mss_cluster_kernel(const float* __restrict__ logits, const float* __restrict__ q, int T, int V,
                   const int32_t* __restrict__ tokens, const int32_t* __restrict__ parent,
                   const int32_t* __restrict__ n_nodes, float temperature,
                   const float* __restrict__ uniforms, int n_uniforms, int32_t* __restrict__ verified,
                   int32_t* __restrict__ ids, int32_t* __restrict__ len) {
    cg::cluster_group cl = cg::this_cluster();
    extern __shared__ float p[];  // this CTA's elements [e0, e1), then the tree
    __shared__ MssCluster sh;
    const int kr = (int)cl.block_rank();
    const int b = blockIdx.x / CN, tid = threadIdx.x;
    const int n = n_nodes[b];
    const int CH = (V + NT - 1) / NT;
    const int SPAN = OWN * CH;                       // elements per CTA (last may be short)
    const int e0 = min(V, kr * SPAN), e1 = min(V, e0 + SPAN), ne = e1 - e0;
    const bool owner = tid < OWN;
    const int gc = kr * OWN + tid;                   // global chunk of an owner
    const int c0 = owner ? min(V, gc * CH) - e0 : 0, c1 = owner ? min(V, (gc + 1) * CH) - e0 : 0;
    float* qbuf = p + SPAN;  // two q slices: the current child's and the next child's (prefetch)
    int32_t* par = reinterpret_cast<int32_t*>(qbuf + 2 * SPAN);
    int32_t* tok = par + T;
    int32_t* kids = tok + T;  // children of the current node, ascending id
    // this CTA's slice of child v's draft row, copied asynchronously into buffer `slot`
    auto prefetch_q = [&](int v, int slot) {
        const float* qe = q + ((int64_t)b * T + v) * V + e0;
        float* dst = qbuf + slot * SPAN;
        for (int i = tid; i < ne; i += NTC) cp_async4(dst + i, qe + i);
        cp_async_commit();
    };
    for (int v = tid; v < n; v += NTC) {
        par[v] = parent[(int64_t)b * T + v];
        tok[v] = tokens[(int64_t)b * T + v];
    }
    const float* U = uniforms + (int64_t)b * n_uniforms;
    int32_t* vrow = verified + (int64_t)b * (T + 1);
    int32_t* irow = ids + (int64_t)b * (T + 1);
    const bool lead = kr == 0;
    const float inv_tau = __fdiv_rn(1.0f, temperature);
    int u = 0, k = 0, m = 0, rc = 0;  // rc: reduction counter (slot parity), identical in all CTAs
    if (lead && tid == 0) irow[0] = 0;

    for (;;) {
        cl.sync();  // every remote reader of the previous p is done
        // children of u (ascending id); the first one's q slice starts loading now,
        // behind the softmax
        __shared__ int nkids;
        if (tid == 0) {
            int c = 0;
            for (int v = u + 1; v < n; ++v)
                if (par[v] == u) kids[c++] = v;
            nkids = c;
        }
        __syncthreads();
        const int nk = nkids;
        if (nk > 0) prefetch_q(kids[0], 0);
        // ---- p = softmax(z[u] / tau) in the contract's arithmetic ----
        const float* z = logits + ((int64_t)b * T + u) * V + e0;
        float mx = -INFINITY;
        for (int i0 = tid; i0 < ne; i0 += NTC * kBatch) {
            float x[kBatch];
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                const int i = i0 + j * NTC;
                x[j] = i < ne ? __ldg(z + i) : -INFINITY;
            }
#pragma unroll
            for (int j = 0; j < kBatch; ++j) {
                const int i = i0 + j * NTC;
                if (i < ne) {
                    p[i] = x[j];
                    mx = fmaxf(mx, x[j]);
                }
            }
        }
        mx = cluster_max(mx, sh, (rc++) & 1, cl);
        for (int i = tid; i < ne; i += NTC) p[i] = exp_spec(__fmul_rn(__fsub_rn(p[i], mx), inv_tau));
        __syncthreads();
        float a = 0.0f;
        for (int i = c0; i < c1; ++i) a = __fadd_rn(a, p[i]);
        const float S = cluster_combine(a, sh, (rc++) & 1, cl);
        for (int i = tid; i < ne; i += NTC) p[i] = __fdiv_rn(p[i], S);
        cl.sync();  // p final in every CTA before any remote p[t] read

        // ---- children of u in ascending id order ----
        int next = -1;
        for (int ci = 0; ci < nk; ++ci) {
            const int v = kids[ci];
            const float* qs = qbuf + (ci & 1) * SPAN;
            // the next child's slice loads while this child is tested
            // (buffer (ci+1)&1 was last read before the previous cluster barrier)
            if (ci + 1 < nk) prefetch_q(kids[ci + 1], (ci + 1) & 1);
            const float r = U[k++];
            const int32_t t = tok[v];
            const float* qv = q + ((int64_t)b * T + v) * V;
            if (tid == 0) {  // p[t] (DSMEM) and q_v[t] for the test
                const int kt = t / SPAN;
                sh.pt = cl.map_shared_rank(p, kt)[t - kt * SPAN];
                sh.qt = __ldg(qv + t);
            }
            if (ci + 1 < nk) cp_async_wait<1>(); else cp_async_wait<0>();  // this child's slice
            __syncthreads();
            if (__fmul_rn(r, sh.qt) <= sh.pt) {
                cp_async_wait<0>();  // drain the prefetch before the buffers are reused
                next = v;
                break;
            }
            float s2 = 0.0f;
            for (int i = c0; i < c1; ++i) s2 = __fadd_rn(s2, fmaxf(__fsub_rn(p[i], qs[i]), 0.0f));
            const float S2 = cluster_combine(s2, sh, (rc++) & 1, cl);
            if (S2 > 0.0f)
                for (int i = tid; i < ne; i += NTC) p[i] = __fdiv_rn(fmaxf(__fsub_rn(p[i], qs[i]), 0.0f), S2);
            cl.sync();  // renormalised p everywhere before the next remote read
        }
        if (next >= 0) {
            if (lead && tid == 0) {
                vrow[m] = tok[next];
                irow[m + 1] = next;
            }
            ++m;
            u = next;
            continue;
        }

        // ---- inverse-CDF sample of p (the leader scans; p read over DSMEM) ----
        const float r = U[k++];
        float c = 0.0f;
        for (int i = c0; i < c1; ++i) c = __fadd_rn(c, p[i]);
        if (owner) cl.map_shared_rank(&sh, 0)->csum[gc] = c;
        cl.sync();
        if (lead && tid < 32) {  // warp 0 of the leader
            __shared__ float target_s;
            __shared__ int tc_s;
            if (tid == 0) {
                float run = 0.0f;
                for (int t = 0; t < NT; ++t) {
                    run = __fadd_rn(run, sh.csum[t]);
                    sh.cum[t] = run;
                }
                const float target = __fmul_rn(r, sh.cum[NT - 1]);
                int tc = -1;
                for (int t = 0; t < NT; ++t)
                    if (sh.cum[t] > target) { tc = t; break; }
                if (tc < 0)
                    for (int t = NT - 1; t >= 0; --t)
                        if (sh.csum[t] > 0.0f) { tc = t; break; }
                target_s = target;
                tc_s = tc;
            }
            __syncwarp();
            const int tc = tc_s;
            int pick = 0;
            if (tc >= 0) {
                // the chosen chunk, fetched over DSMEM by the whole warp (independent
                // loads) into local scratch, then scanned sequentially in the
                // contract's order by lane 0
                const int lo = tc * CH, hi = min(V, (tc + 1) * CH);
                const int kt = lo / SPAN;
                const float* pr = cl.map_shared_rank(p, kt) - kt * SPAN;  // global element index
                float* loc = qbuf;  // the q slices are free here
                for (int i = lo + tid; i < hi; i += 32) loc[i - lo] = pr[i];
                __syncwarp();
                if (tid == 0) {
                    const float target = target_s;
                    float acc = tc > 0 ? sh.cum[tc - 1] : 0.0f;
                    int last_pos = -1;
                    pick = -1;
                    for (int i = lo; i < hi; ++i) {
                        const float pi = loc[i - lo];
                        acc = __fadd_rn(acc, pi);
                        if (pi > 0.0f) last_pos = i;
                        if (acc > target) { pick = i; break; }
                    }
                    if (pick < 0) pick = last_pos >= 0 ? last_pos : lo;
                }
            }
            if (tid == 0) {
                vrow[m] = pick;
                len[b] = m + 1;
            }
        }
        cl.sync();  // the leader's remote reads are done before any CTA exits
        break;
    }
}

}  // namespace
}  // namespace st

extern "C" st_status st_verify_mss(const float* logits, const float* q, int B, int T, int V,
                                   const int32_t* tokens, const int32_t* parent,
                                   const int32_t* n_nodes, float temperature,
                                   const float* uniforms, int n_uniforms, int32_t* verified,
                                   int32_t* ids, int32_t* len, void* stream) {
    if (st_status e = st::require_device()) return e;
    ST_CHECK_ARG(B >= 0 && T >= 1 && V >= 1, ST_ERR_SHAPE_MISMATCH, "bad shape");
    ST_CHECK_ARG(temperature > 0.0f, ST_ERR_INVALID_ARGUMENT, "temperature must be > 0");
    ST_CHECK_ARG(n_uniforms >= T + 1, ST_ERR_INVALID_ARGUMENT,
                 "need n_uniforms >= T + 1 (one per visited child plus the final sample)");
    if (B == 0) return ST_OK;
    ST_CHECK_ARG(logits && q && tokens && parent && n_nodes && uniforms && verified && ids && len,
                 ST_ERR_INVALID_ARGUMENT, "null pointer");
    // one cluster of CN CTAs per request; each CTA holds its OWN chunks of p
    // and two q slices (current child + prefetched next child)
    const int CH = (V + st::NT - 1) / st::NT;
    const size_t smem = 3 * (size_t)st::OWN * CH * sizeof(float) + 3 * (size_t)T * sizeof(int32_t);
    ST_CHECK_ARG(smem <= 200 * 1024, ST_ERR_UNSUPPORTED,
                 "vocabulary / tree too large for K4 (3 * V/4 * 4 + T * 12 <= 200 KB)");
    ST_CHECK_ARG((int64_t)B * st::CN <= 2147483647, ST_ERR_SHAPE_MISMATCH, "too many requests");
    static size_t attr_set = 0;
    if (smem > 48 * 1024 && smem > attr_set) {
        ST_CUDA_TRY(cudaFuncSetAttribute(st::mss_cluster_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_set = smem;
    }
    st::mss_cluster_kernel<<<B * st::CN, st::NTC, smem, st::as_stream(stream)>>>(
        logits, q, T, V, tokens, parent, n_nodes, temperature, uniforms, n_uniforms, verified, ids,
        len);
    ST_LAUNCH_CHECK();
    return ST_OK;
}
