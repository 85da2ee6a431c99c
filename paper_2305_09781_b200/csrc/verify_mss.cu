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
// contracted.
//
// Latency, not bandwidth, bounds it (a chain of dependent steps per visited
// node), so the chain is kept short: the accept test of a child needs one
// element of p, which every CTA recomputes from prefetched scalars (z_u[t],
// q_j[t]) with the element-wise passes' own operations — no barrier, DSMEM
// read or global round trip before a test; p is materialised lazily (p_0 =
// e / S only when a child is rejected or the node samples), fused with the
// residual of the rejected child into one pass, so a rejection costs one
// element-wise pass and one cluster reduction; children are found by a
// ballot compaction; the candidate children's logits slices are prefetched
// into L2 behind the softmax. Element-wise passes use all 4096 threads and
// each rejected child's q slice is copied into shared memory asynchronously
// while the previous child is processed.
#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <string>

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
    if (warp == 0) {  // lane j < CN sends this CTA's max to CTA j
        float m = sh.red[lane];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (lane < CN) {
            MssCluster* dst = cl.map_shared_rank(&sh, lane);
            dst->xmax[slot][cl.block_rank()] = m;
        }
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

// Per-node test scalars of the first kPre children (shared memory): the
// accept test of child k needs p_k[t_k] only, which every CTA recomputes from
// z_u[t_k], the node's (max, sum) and q_j[t_k] / S_j of the children rejected
// before it — the contract's own element-wise operations applied to one
// element, hence the same bits — so no child waits for a materialised p, a
// DSMEM read or a cluster barrier before its test.
constexpr int kPre = 32;
struct MssNode {
    float zt[kPre];              // z_u[t_k]
    float qtt[kPre][kPre];       // q_{kids[j]}[t_k] at [j][k], j <= k
    float ztk;                   // z_u[t_k], k >= kPre
    int acc;
};

__device__ __forceinline__ void cp_async16(float* dst, const float* src) {
    asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                     (uint32_t)__cvta_generic_to_shared(dst)),
                 "l"(src)
                 : "memory");
}

__global__ void __cluster_dims__(CN, 1, 1) __launch_bounds__(NTC)
mss_cluster_kernel(const float* __restrict__ logits, const float* __restrict__ q, int T, int V,
                   const int32_t* __restrict__ tokens, const int32_t* __restrict__ parent,
                   const int32_t* __restrict__ n_nodes, float temperature,
                   const float* __restrict__ uniforms, int n_uniforms, int32_t* __restrict__ verified,
                   int32_t* __restrict__ ids, int32_t* __restrict__ len, int vec,
                   unsigned long long* trace, int trace_req) {
    cg::cluster_group cl = cg::this_cluster();
    // this CTA's elements [e0, e1) of p and of the residual d, two q slices, then the tree
    extern __shared__ __align__(16) float p[];
    __shared__ MssCluster sh;
    __shared__ MssNode nd;
    const int kr = (int)cl.block_rank();
    const int b = blockIdx.x / CN, tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int n = n_nodes[b];
    const int CH = (V + NT - 1) / NT;
    const int SPAN = OWN * CH;                       // elements per CTA (last may be short)
    const int e0 = min(V, kr * SPAN), e1 = min(V, e0 + SPAN), ne = e1 - e0;
    const bool owner = tid < OWN;
    const int gc = kr * OWN + tid;                   // global chunk of an owner
    const int c0 = owner ? min(V, gc * CH) - e0 : 0, c1 = owner ? min(V, (gc + 1) * CH) - e0 : 0;
    float* d = p + SPAN;        // residual max(p_k - q_k, 0) of the last rejected child
    float* qbuf = d + SPAN;     // two q slices: the current child's and the next child's (prefetch)
    int32_t* par = reinterpret_cast<int32_t*>(qbuf + 2 * SPAN);
    int32_t* tok = par + T;
    int32_t* kall = tok + T;    // children of every node, grouped by parent, ascending id
    int32_t* koff = kall + T;   // [T + 1]: node u's children are kall[koff[u] .. koff[u+1])
    int32_t* fill = koff + T + 1;
    float* Sh = reinterpret_cast<float*>(fill + T);  // residual sums of the rejected children
    float* qcol = Sh + T;       // test scalars of child k >= kPre
    // element-wise passes: element i = tid mod NTC (consecutive lanes, no bank
    // conflicts); the slice copies land in float4 granules, so a pass reads q
    // only after a barrier that follows every thread's wait
    auto for_each = [&](auto&& fn) {
        for (int i = tid; i < ne; i += NTC) fn(i);
    };
    // this CTA's slice of child v's draft row, copied asynchronously into buffer `slot`
    auto prefetch_q = [&](int v, int slot) {
        const float* qe = q + ((int64_t)b * T + v) * V + e0;
        float* dst = qbuf + slot * SPAN;
        if (vec) {
            for (int j = tid; j < (ne >> 2); j += NTC) cp_async16(dst + 4 * j, qe + 4 * j);
        } else {
            for (int i = tid; i < ne; i += NTC) cp_async4(dst + i, qe + i);
        }
        cp_async_commit();
    };
    // the contract's chunk partial of this owner, x(i) summed in index order
    auto owner_sum = [&](const float* x) {
        float a = 0.0f;
#pragma unroll 8
        for (int i = c0; i < c1; ++i) a = __fadd_rn(a, x[i]);
        return a;
    };
    for (int v = tid; v < n; v += NTC) {
        par[v] = parent[(int64_t)b * T + v];
        tok[v] = tokens[(int64_t)b * T + v];
    }
    for (int v = tid; v < T; v += NTC) fill[v] = 0;
    __syncthreads();
    // children lists of every node, once (the tree is fixed): warp 0 walks the
    // nodes 32 at a time in id order; lanes with the same parent (match_any)
    // take consecutive slots, so each list is in ascending id order. Only
    // children with a larger id count (parent-before-child order, as the
    // contract's scan from u + 1).
    if (warp == 0) {
        for (int c = 0; c < n; c += 32) {  // counts
            const int v = c + lane;
            const int pu = v < n && v > 0 && par[v] >= 0 && par[v] < v ? par[v] : -1 - lane;
            const unsigned peers = __match_any_sync(0xffffffffu, pu);
            if (pu >= 0 && lane == __ffs(peers) - 1) fill[pu] += __popc(peers);
            __syncwarp();
        }
        int carry = 0;  // exclusive prefix over the counts
        for (int c = 0; c < n; c += 32) {
            const int u = c + lane;
            const int x = u < n ? fill[u] : 0;
            int inc = x;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, inc, o);
                if (lane >= o) inc += y;
            }
            if (u < n) koff[u] = fill[u] = carry + inc - x;
            carry += __shfl_sync(0xffffffffu, inc, 31);
        }
        if (lane == 0) koff[n] = carry;
        __syncwarp();
        for (int c = 0; c < n; c += 32) {  // placement
            const int v = c + lane;
            const int pu = v < n && v > 0 && par[v] >= 0 && par[v] < v ? par[v] : -1 - lane;
            const unsigned peers = __match_any_sync(0xffffffffu, pu);
            const int base = pu >= 0 ? fill[pu] : 0;
            __syncwarp();
            if (pu >= 0) {
                kall[base + __popc(peers & ((1u << lane) - 1u))] = v;
                if (lane == __ffs(peers) - 1) fill[pu] = base + __popc(peers);
            }
            __syncwarp();
        }
    }
    // (a cluster barrier, not only a CTA one: no CTA writes a peer's shared
    // memory before every CTA of the cluster has started)
    cl.sync();
    const float* U = uniforms + (int64_t)b * n_uniforms;
    int32_t* vrow = verified + (int64_t)b * (T + 1);
    int32_t* irow = ids + (int64_t)b * (T + 1);
    const bool lead = kr == 0;
    const float inv_tau = __fdiv_rn(1.0f, temperature);
    int u = 0, k = 0, m = 0, rc = 0;  // rc: reduction counter (slot parity), identical in all CTAs
    if (lead && tid == 0) irow[0] = 0;
    // ST_K4_TRACE (diagnostic): (phase, clock64) events of one request's leader thread
    int tn = 0;
#define K4T(code)                                                                  \
    do {                                                                           \
        if (trace && b == trace_req && kr == 0 && tid == 0 && tn < 1024) {         \
            trace[2 * tn] = (code);                                                \
            trace[2 * tn + 1] = clock64();                                         \
            ++tn;                                                                  \
        }                                                                          \
    } while (0)
    K4T(0);

    for (;;) {
        // (no barrier here: every shared read of the previous node — the test
        // scalars, p, d, the slices — precedes a barrier the children loop or
        // the reductions already passed)
        K4T(1);
        const int32_t* kids = kall + koff[u];
        const int nk = koff[u + 1] - koff[u];
        K4T(2);
        if (nk > 0) prefetch_q(kids[0], 0);
        const float* zrow = logits + ((int64_t)b * T + u) * V;
        const int npre = min(nk, kPre);
        for (int x = tid; x < npre * npre + npre; x += NTC) {
            if (x < npre * npre) {
                const int j = x / npre, kk = x - j * npre;
                if (j <= kk) cp_async4(&nd.qtt[j][kk], q + ((int64_t)b * T + kids[j]) * V + tok[kids[kk]]);
            } else {
                const int kk = x - npre * npre;
                cp_async4(&nd.zt[kk], zrow + tok[kids[kk]]);
            }
        }
        cp_async_commit();
        if (vec) {  // one bulk L2 prefetch per candidate child's slice
            if (tid < npre)
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(logits + ((int64_t)b * T + kids[tid]) * V + e0),
                             "r"((uint32_t)ne * 4u)
                             : "memory");
        } else {
            const int lines = (ne + 31) >> 5;  // 128-byte lines of this CTA's slice
            for (int x = tid; x < npre * lines; x += NTC) {
                const int kk = x / lines, l = x - kk * lines;
                asm volatile("prefetch.global.L2 [%0];" ::"l"(logits + ((int64_t)b * T + kids[kk]) * V + e0 + 32 * l));
            }
        }
        // ---- softmax(z[u] / tau): e in p, its sum S (p_0 = e / S, materialised lazily) ----
        const float* z = zrow + e0;
        float mx = -INFINITY;
        if (vec) {
            const float4* z4 = reinterpret_cast<const float4*>(z);
            float4* p4 = reinterpret_cast<float4*>(p);
            for (int j0 = tid; j0 < (ne >> 2); j0 += NTC * 4) {
                float4 x[4];
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int i = j0 + j * NTC;
                    x[j] = i < (ne >> 2) ? __ldg(z4 + i) : make_float4(-INFINITY, -INFINITY, -INFINITY, -INFINITY);
                }
#pragma unroll
                for (int j = 0; j < 4; ++j) {
                    const int i = j0 + j * NTC;
                    if (i < (ne >> 2)) {
                        p4[i] = x[j];
                        mx = fmaxf(mx, fmaxf(fmaxf(x[j].x, x[j].y), fmaxf(x[j].z, x[j].w)));
                    }
                }
            }
        } else
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
        K4T(3);
        mx = cluster_max(mx, sh, (rc++) & 1, cl);
        K4T(4);
        for_each([&](int i) { p[i] = exp_spec(__fmul_rn(__fsub_rn(p[i], mx), inv_tau)); });
        __syncthreads();
        K4T(5);
        const float S = cluster_combine(owner_sum(p), sh, (rc++) & 1, cl);
        K4T(7);
        cp_async_wait<0>();  // this thread's test scalars (and child 0's slice)
        __syncthreads();
        K4T(8);

        // ---- children of u in ascending id order ----
        int next = -1;
        float S_last = S;  // sum of the last rejected child's residual (every thread's copy)
        for (int ci = 0; ci < nk; ++ci) {
            const int v = kids[ci];
            const float r = U[k++];
            // child ci's slice (issued a step earlier) landed — this thread's
            // copies; the test's barrier publishes everyone's — and the next
            // child's slice starts loading (buffer (ci+1)&1 was last read by
            // the pass before the previous barrier)
            cp_async_wait<0>();
            if (ci + 1 < nk) prefetch_q(kids[ci + 1], (ci + 1) & 1);
            if (ci >= kPre) {  // test scalars not prefetched
                for (int j = tid; j <= ci; j += NTC) qcol[j] = __ldg(q + ((int64_t)b * T + kids[j]) * V + tok[v]);
                if (tid == 0) nd.ztk = __ldg(zrow + tok[v]);
                __syncthreads();
            }
            if (tid == 0) {
                // p_ci[t]: p_0[t] = e[t] / S, then the residual step of every
                // rejected earlier child — the element-wise passes' arithmetic
                const float zt = ci < kPre ? nd.zt[ci] : nd.ztk;
                float x = __fdiv_rn(exp_spec(__fmul_rn(__fsub_rn(zt, mx), inv_tau)), S);
                for (int j = 0; j < ci; ++j) {
                    const float Sj = Sh[j];
                    if (Sj > 0.0f) {
                        const float qj = ci < kPre ? nd.qtt[j][ci] : qcol[j];
                        x = __fdiv_rn(fmaxf(__fsub_rn(x, qj), 0.0f), Sj);
                    }
                }
                const float qk = ci < kPre ? nd.qtt[ci][ci] : qcol[ci];
                nd.acc = __fmul_rn(r, qk) <= x;
            }
            __syncthreads();
            K4T(9);
            if (nd.acc) {
                next = v;
                break;
            }
            // rejected: p_ci materialised (from e / S, or the previous residual
            // over its sum unless that was 0) and its residual against q_ci
            const float* qs = qbuf + (ci & 1) * SPAN;
            const bool div = ci == 0 || S_last > 0.0f;
            const float Sp = S_last;
            const float* src = ci == 0 ? p : d;
            K4T(10);
            for_each([&](int i) {
                const float pk = div ? __fdiv_rn(src[i], Sp) : p[i];
                p[i] = pk;
                d[i] = fmaxf(__fsub_rn(pk, qs[i]), 0.0f);
            });
            __syncthreads();
            K4T(11);
            S_last = cluster_combine(owner_sum(d), sh, (rc++) & 1, cl);
            K4T(12);
            if (tid == 0) Sh[ci] = S_last;  // (thread 0's test recursion)
        }
        if (next >= 0) {
            cp_async_wait<0>();  // a prefetched slice must land before its buffer is reused
            if (lead && tid == 0) {
                vrow[m] = tok[next];
                irow[m + 1] = next;
            }
            ++m;
            u = next;
            continue;
        }

        // ---- inverse-CDF sample of the final p (the leader scans; p read over DSMEM) ----
        {
            const float* src = nk == 0 ? p : d;
            if (nk == 0 || S_last > 0.0f) for_each([&](int i) { p[i] = __fdiv_rn(src[i], S_last); });
        }
        __syncthreads();
        const float r = U[k++];
        const float c = owner_sum(p);
        if (owner) cl.map_shared_rank(&sh, 0)->csum[gc] = c;
        K4T(13);
        cl.sync();
        K4T(14);
        if (lead && tid < 32) {  // warp 0 of the leader
            __shared__ float target_s;
            if (tid == 0) {  // C_t in the contract's sequential order, 32 loads in flight at a time
                float run = 0.0f;
                for (int t0 = 0; t0 < NT; t0 += 32) {
                    float v[32];
#pragma unroll
                    for (int j = 0; j < 32; ++j) v[j] = sh.csum[t0 + j];
#pragma unroll
                    for (int j = 0; j < 32; ++j) {
                        run = __fadd_rn(run, v[j]);
                        sh.cum[t0 + j] = run;
                    }
                }
                target_s = __fmul_rn(r, run);
            }
            __syncwarp();
            const float target = target_s;
            // the first chunk with C_t > target, else the last with a positive sum (ballots)
            int tc = -1;
            for (int t0 = 0; t0 < NT && tc < 0; t0 += 32) {
                const unsigned bal = __ballot_sync(0xffffffffu, sh.cum[t0 + lane] > target);
                if (bal) tc = t0 + __ffs(bal) - 1;
            }
            for (int t0 = NT - 32; t0 >= 0 && tc < 0; t0 -= 32) {
                const unsigned bal = __ballot_sync(0xffffffffu, sh.csum[t0 + lane] > 0.0f);
                if (bal) tc = t0 + 31 - __clz(bal);
            }
            K4T(15);
            int pick = 0;
            if (tc >= 0) {
                // the chosen chunk, fetched over DSMEM by the whole warp (independent
                // loads) into local scratch, then scanned sequentially in the
                // contract's order by lane 0, 16 values loaded at a time
                const int lo = tc * CH, hi = min(V, (tc + 1) * CH);
                const int kt = lo / SPAN;
                const float* pr = cl.map_shared_rank(p, kt) - kt * SPAN;  // global element index
                float* loc = qbuf;  // the q slices are free here
                for (int i = lo + tid; i < hi; i += 32) loc[i - lo] = pr[i];
                __syncwarp();
                if (tid == 0) {
                    float acc = tc > 0 ? sh.cum[tc - 1] : 0.0f;
                    int last_pos = -1;
                    pick = -1;
                    for (int i0 = lo; i0 < hi && pick < 0; i0 += 16) {
                        float v[16];
#pragma unroll
                        for (int j = 0; j < 16; ++j) v[j] = i0 + j < hi ? loc[i0 + j - lo] : 0.0f;
#pragma unroll
                        for (int j = 0; j < 16; ++j) {
                            if (pick < 0 && i0 + j < hi) {
                                acc = __fadd_rn(acc, v[j]);
                                if (v[j] > 0.0f) last_pos = i0 + j;
                                if (acc > target) pick = i0 + j;
                            }
                        }
                    }
                    if (pick < 0) pick = last_pos >= 0 ? last_pos : lo;
                }
            }
            if (tid == 0) {
                vrow[m] = pick;
                len[b] = m + 1;
            }
        }
        K4T(16);
        cl.sync();  // the leader's remote reads are done before any CTA exits
        K4T(17);
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
    const size_t smem = 4 * (size_t)st::OWN * CH * sizeof(float) + (7 * (size_t)T + 1) * sizeof(int32_t);
    ST_CHECK_ARG(smem <= 212 * 1024, ST_ERR_UNSUPPORTED,
                 "vocabulary / tree too large for K4 (4 * 4 * V/4 + 28 * T bytes <= 212 KB)");
    ST_CHECK_ARG((int64_t)B * st::CN <= 2147483647, ST_ERR_SHAPE_MISMATCH, "too many requests");
    static size_t attr_set = 0;
    if (smem > 48 * 1024 && smem > attr_set) {
        ST_CUDA_TRY(cudaFuncSetAttribute(st::mss_cluster_kernel,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr_set = smem;
    }
    static unsigned long long* trace = nullptr;  // ST_K4_TRACE=path[:request] (diagnostic)
    static const char* trace_env = getenv("ST_K4_TRACE");
    static const int trace_req = trace_env && strchr(trace_env, ':') ? atoi(strchr(trace_env, ':') + 1) : 0;
    if (trace_env && !trace) ST_CUDA_TRY(cudaMalloc(&trace, 2048 * sizeof(unsigned long long)));
    if (trace) ST_CUDA_TRY(cudaMemsetAsync(trace, 0, 2048 * sizeof(unsigned long long), st::as_stream(stream)));
    st::mss_cluster_kernel<<<B * st::CN, st::NTC, smem, st::as_stream(stream)>>>(
        logits, q, T, V, tokens, parent, n_nodes, temperature, uniforms, n_uniforms, verified, ids,
        len,
        (V % 4 == 0 && ((reinterpret_cast<uintptr_t>(q) | reinterpret_cast<uintptr_t>(logits)) & 15) == 0) ? 1 : 0,
        trace, trace_req);
    ST_LAUNCH_CHECK();
    if (trace) {
        unsigned long long h[2048];
        ST_CUDA_TRY(cudaStreamSynchronize(st::as_stream(stream)));
        ST_CUDA_TRY(cudaMemcpy(h, trace, sizeof(h), cudaMemcpyDeviceToHost));
        std::string path(trace_env);
        path = path.substr(0, path.find(':'));
        if (FILE* f = fopen(path.c_str(), "w")) {
            for (int i = 0; i < 1024 && h[2 * i + 1]; ++i) fprintf(f, "%llu %llu\n", h[2 * i], h[2 * i + 1]);
            fclose(f);
        }
    }
    return ST_OK;
}
