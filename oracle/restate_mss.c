/* TEST INFRASTRUCTURE ONLY — CPU oracle for K4, multi-step speculative
 * sampling (MSS).
 *
 * PARITY UNPINNED AGAINST THE REFERENCE: the reference has no stochastic
 * verification (PAPER.md:181-190 is greedy only), so
 * there is nothing of the reference's to check against. This file IS the pin:
 * it states the contract of DESIGN.md §5 (SpecInfer's
 * published MSS) with every floating-point operation fixed, and K4 must match
 * it bit for bit given the same host-supplied uniforms.
 *
 * Fixed arithmetic (all fp32, round-to-nearest, no contraction; built with
 * -ffp-contract=off):
 *   NT = 256 reduction lanes; chunk t = [t*CH, min(V,(t+1)*CH)), CH = ceil(V/NT)
 *   sum_spec(x): chunk partials summed sequentially in index order from 0.0f;
 *                per warp of 32 chunks an xor-butterfly (16,8,4,2,1), lane 0;
 *                the 8 warp values added sequentially w0+w1+...+w7.
 *   exp_spec(x): 0 for x <= -104; t = x*log2e; n = rint(t); f = t-n;
 *                2^f by a degree-6 Horner polynomial with fmaf; times 2^n
 *                (exact power-of-two multiplies).
 *   softmax:     m = max z; e_i = exp_spec((z_i - m) * (1/tau)); p_i = e_i / S.
 *   accept v:    r*q_v[t_v] <= p[t_v]  (r = next uniform)
 *   reject v:    S' = sum_spec(max(p - q_v, 0)); if S' > 0: p = max(p - q_v, 0)/S'
 *   sample:      r = next uniform; chunk cumulative C_t (sequential over t);
 *                target = r*C_last; first chunk with C_t > target; inside it a
 *                running sum from C_{t-1}; first i with acc > target, else the
 *                last i of that chunk with p_i > 0.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "restate.h"

#define NT 256

static float exp_spec(float x) {
    if (!(x > -104.0f)) return 0.0f;
    const float t = x * 1.44269504f;
    const float nf = rintf(t);
    const float f = t - nf;
    float p = 1.54035304e-4f;
    p = fmaf(p, f, 1.33335581e-3f);
    p = fmaf(p, f, 9.61812911e-3f);
    p = fmaf(p, f, 5.55041087e-2f);
    p = fmaf(p, f, 2.40226507e-1f);
    p = fmaf(p, f, 6.93147182e-1f);
    p = fmaf(p, f, 1.0f);
    const int n = (int)nf;
    if (n >= -126) {
        union { uint32_t u; float f; } s;
        s.u = (uint32_t)(n + 127) << 23;
        return p * s.f;
    }
    union { uint32_t u; float f; } s1, s2;
    s1.u = (uint32_t)(n + 100 + 127) << 23;
    s2.u = (uint32_t)(-100 + 127) << 23;
    return (p * s1.f) * s2.f;
}

static int chunk_size(int V) { return (V + NT - 1) / NT; }

/* chunk partial sums of values produced by f(i) */
static float combine_spec(const float* part) {
    float warp_val[NT / 32];
    for (int w = 0; w < NT / 32; ++w) {
        float s[32], t[32];
        for (int l = 0; l < 32; ++l) s[l] = part[32 * w + l];
        for (int o = 16; o > 0; o >>= 1) {
            for (int l = 0; l < 32; ++l) t[l] = s[l] + s[l ^ o];
            memcpy(s, t, sizeof s);
        }
        warp_val[w] = s[0];
    }
    float tot = warp_val[0];
    for (int w = 1; w < NT / 32; ++w) tot = tot + warp_val[w];
    return tot;
}

static float sum_spec(const float* x, int V) {
    const int CH = chunk_size(V);
    float part[NT];
    for (int t = 0; t < NT; ++t) {
        float a = 0.0f;
        for (int i = t * CH; i < (t + 1) * CH && i < V; ++i) a = a + x[i];
        part[t] = a;
    }
    return combine_spec(part);
}

static float residual_sum_spec(const float* p, const float* q, int V) {
    const int CH = chunk_size(V);
    float part[NT];
    for (int t = 0; t < NT; ++t) {
        float a = 0.0f;
        for (int i = t * CH; i < (t + 1) * CH && i < V; ++i) a = a + fmaxf(p[i] - q[i], 0.0f);
        part[t] = a;
    }
    return combine_spec(part);
}

static int sample_spec(const float* p, int V, float r) {
    const int CH = chunk_size(V);
    float c[NT], C[NT];
    for (int t = 0; t < NT; ++t) {
        float a = 0.0f;
        for (int i = t * CH; i < (t + 1) * CH && i < V; ++i) a = a + p[i];
        c[t] = a;
    }
    float run = 0.0f;
    for (int t = 0; t < NT; ++t) { run = run + c[t]; C[t] = run; }
    const float target = r * C[NT - 1];
    int tc = -1;
    for (int t = 0; t < NT; ++t)
        if (C[t] > target) { tc = t; break; }
    if (tc < 0)
        for (int t = NT - 1; t >= 0; --t)
            if (c[t] > 0.0f) { tc = t; break; }
    if (tc < 0) return 0;
    float acc = tc > 0 ? C[tc - 1] : 0.0f;
    int last_pos = -1;
    for (int i = tc * CH; i < (tc + 1) * CH && i < V; ++i) {
        acc = acc + p[i];
        if (p[i] > 0.0f) last_pos = i;
        if (acc > target) return i;
    }
    return last_pos >= 0 ? last_pos : tc * CH;
}

int or_mss_verify(const float* logits, const float* q, int V, const int32_t* tok,
                  const int32_t* parent, int n, float temperature, const float* uniforms,
                  int n_uniforms, int32_t* verified, int32_t* ids, int* n_verified) {
    if (n < 1 || V < 1 || !(temperature > 0.0f) || n_uniforms < n + 1) return 1 + 15;
    float* p = (float*)malloc(sizeof(float) * (size_t)V);
    const float inv_tau = 1.0f / temperature;
    int u = 0, k = 0, m = 0;
    ids[0] = 0;
    for (;;) {
        const float* z = logits + (size_t)u * V;
        float mx = -INFINITY;
        for (int i = 0; i < V; ++i) mx = fmaxf(mx, z[i]);
        for (int i = 0; i < V; ++i) p[i] = exp_spec((z[i] - mx) * inv_tau);
        const float S = sum_spec(p, V);
        for (int i = 0; i < V; ++i) p[i] = p[i] / S;
        int next = -1;
        for (int v = u + 1; v < n && next < 0; ++v) {
            if (parent[v] != u) continue;
            const float r = uniforms[k++];
            const int32_t t = tok[v];
            const float* qv = q + (size_t)v * V;
            if (r * qv[t] <= p[t]) {
                next = v;
            } else {
                const float S2 = residual_sum_spec(p, qv, V);
                if (S2 > 0.0f)
                    for (int i = 0; i < V; ++i) p[i] = fmaxf(p[i] - qv[i], 0.0f) / S2;
            }
        }
        if (next >= 0) {
            verified[m++] = tok[next];
            ids[m] = next;
            u = next;
            continue;
        }
        const float r = uniforms[k++];
        verified[m++] = sample_spec(p, V, r);
        break;
    }
    *n_verified = m;
    free(p);
    return 0;
}
