/* TEST INFRASTRUCTURE ONLY — see restate.h for the contract and provenance.
 * Plain C, scalar, single-threaded: the checker for the CUDA path, never the
 * thing measured or shipped. */
#include "restate.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* spectree::Errc numeric values (proj/include/spectree/error.hpp:8-25) + 1. */
enum {
    ST_OK = 0,
    ST_EMPTY_INPUT = 1 + 0,
    ST_ROOT_MISMATCH = 1 + 1,
    ST_UNKNOWN_NODE = 1 + 2,
    ST_MISSING_OUTPUT = 1 + 3,
    ST_TREE_TOO_LARGE = 1 + 4,
    ST_INVALID_ARGUMENT = 1 + 15,
};

/* ---------------------------------------------------------------- merge --- */
/* Trie with per-node child lists kept sorted by token (the std::map of
 * token_tree.cpp:35-38), then a preorder flatten visiting children in
 * ascending token order (token_tree.cpp:77-100). */
typedef struct {
    int32_t token;
    int nkids, capkids;
    int* kids; /* trie indices, sorted by token */
} trie_node;

static int trie_find(const trie_node* tr, int at, int32_t token, int* pos) {
    const trie_node* n = &tr[at];
    int lo = 0, hi = n->nkids;
    while (lo < hi) {
        int mid = (lo + hi) / 2;
        if (tr[n->kids[mid]].token < token) lo = mid + 1;
        else hi = mid;
    }
    *pos = lo;
    return (lo < n->nkids && tr[n->kids[lo]].token == token) ? n->kids[lo] : -1;
}

int or_merge(const int32_t* flat, const int32_t* lens, int nseq, int max_nodes, int32_t* tok,
             int32_t* parent, int32_t* depth, int cap, int* n_out) {
    /* token_tree.cpp:44-48: no sequences / empty sequence -> empty_input */
    if (nseq <= 0) return ST_EMPTY_INPUT;
    for (int i = 0; i < nseq; ++i)
        if (lens[i] <= 0) return ST_EMPTY_INPUT;
    /* token_tree.cpp:50-55: every sequence must share the first token */
    const int32_t root = flat[0];
    long at = 0;
    for (int i = 0; i < nseq; ++i) {
        if (flat[at] != root) return ST_ROOT_MISMATCH;
        at += lens[i];
    }
    long total = 0;
    for (int i = 0; i < nseq; ++i) total += lens[i];
    int trcap = (int)(total + 1);
    trie_node* tr = (trie_node*)calloc((size_t)trcap, sizeof(trie_node));
    int ntr = 1;
    tr[0].token = root;
    int status = ST_OK;
    at = 0;
    for (int i = 0; i < nseq && status == ST_OK; ++i) {
        int cur = 0;
        for (int j = 1; j < lens[i]; ++j) {
            int pos;
            int nxt = trie_find(tr, cur, flat[at + j], &pos);
            if (nxt < 0) {
                /* token_tree.cpp:64-66: refuse to grow past max_nodes */
                if (ntr >= max_nodes) { status = ST_TREE_TOO_LARGE; break; }
                nxt = ntr++;
                tr[nxt].token = flat[at + j];
                trie_node* p = &tr[cur];
                if (p->nkids == p->capkids) {
                    p->capkids = p->capkids ? 2 * p->capkids : 4;
                    p->kids = (int*)realloc(p->kids, sizeof(int) * (size_t)p->capkids);
                }
                memmove(p->kids + pos + 1, p->kids + pos, sizeof(int) * (size_t)(p->nkids - pos));
                p->kids[pos] = nxt;
                p->nkids++;
            }
            cur = nxt;
        }
        at += lens[i];
    }
    if (status == ST_OK) {
        *n_out = ntr;
        if (ntr > cap) {
            status = -1;
        } else {
            /* explicit-stack preorder; push children in descending order */
            int* st_node = (int*)malloc(sizeof(int) * (size_t)ntr);
            int* st_par = (int*)malloc(sizeof(int) * (size_t)ntr);
            int* st_dep = (int*)malloc(sizeof(int) * (size_t)ntr);
            int sp = 0, id = 0;
            st_node[sp] = 0; st_par[sp] = -1; st_dep[sp] = 0; ++sp;
            while (sp > 0) {
                --sp;
                int tn = st_node[sp], pa = st_par[sp], de = st_dep[sp];
                tok[id] = tr[tn].token;
                parent[id] = pa;
                depth[id] = de;
                for (int k = tr[tn].nkids - 1; k >= 0; --k) {
                    st_node[sp] = tr[tn].kids[k]; st_par[sp] = id; st_dep[sp] = de + 1; ++sp;
                }
                ++id;
            }
            free(st_node); free(st_par); free(st_dep);
        }
    }
    for (int i = 0; i < ntr; ++i) free(tr[i].kids);
    free(tr);
    return status;
}

/* --------------------------------------------------------------- verify --- */
int or_verify(const int32_t* tok, const int32_t* parent, int n, const int32_t* outputs,
              int n_outputs, int32_t* verified, int32_t* ids, int* n_verified) {
    /* token_tree.cpp:154-156 */
    if (n_outputs != n) return ST_MISSING_OUTPUT;
    int u = 0, m = 0;
    ids[0] = 0;
    for (;;) {
        const int32_t want = outputs[u];
        int next = -1;
        /* children of u in ascending id order = ascending token (preorder) */
        for (int v = u + 1; v < n; ++v)
            if (parent[v] == u && tok[v] == want) { next = v; break; }
        if (next < 0) break;
        u = next;
        verified[m++] = want;
        ids[m] = u;
    }
    verified[m++] = outputs[u]; /* bonus token, token_tree.cpp:173 */
    *n_verified = m;
    return ST_OK;
}

/* --------------------------------------------------------------- argmax --- */
int or_argmax_f64(const double* x, int n) {
    int best = 0;
    for (int i = 1; i < n; ++i)
        if (x[i] > x[best]) best = i;
    return best;
}

int or_argmax_f32(const float* x, int n) {
    int best = 0;
    for (int i = 1; i < n; ++i)
        if (x[i] > x[best]) best = i;
    return best;
}

/* ---------------------------------------------------------------- masks --- */
void or_ancestor_masks(const int32_t* parent, int n, int W, uint64_t* mask) {
    for (int u = 0; u < n; ++u) {
        uint64_t* mu = mask + (size_t)u * W;
        if (parent[u] >= 0) memcpy(mu, mask + (size_t)parent[u] * W, sizeof(uint64_t) * (size_t)W);
        else memset(mu, 0, sizeof(uint64_t) * (size_t)W);
        mu[u / 64] |= (uint64_t)1 << (u % 64);
    }
}

/* ---------------------------------------------------------------- rng ----- */
void or_uniform_stream(uint64_t seed, int64_t n, double lo, double hi, double* out) {
    uint64_t state = seed;
    for (int64_t i = 0; i < n; ++i) {
        state += 0x9e3779b97f4a7c15ULL;
        uint64_t z = state;
        z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ULL;
        z = (z ^ (z >> 27)) * 0x94d049bb133111ebULL;
        z = z ^ (z >> 31);
        const double u = (double)(z >> 11) * 0x1.0p-53;
        out[i] = lo + (hi - lo) * u;
    }
}

/* ------------------------------------------------------ tree attention ---- */
/* For node u of request b and head h: softmax over committed rows [0,P) and
 * the tree rows v with bit v of mask[u] set, of q.k * scale, times V —
 * scores/softmax/PV as transformer.cpp:276-298 with the -1e30 mask realised as
 * exclusion (masked weights are exactly 0 there, transformer.hpp:13-16). */
void or_tree_attention(const double* q, const double* kc, const double* vc, const uint64_t* mask,
                       const int32_t* P, const int32_t* n_nodes, int B, int T, int H, int Hkv,
                       int D, int Lmax, int W, double scale, double* o, double* lse) {
    const int group = H / Hkv;
    double* s = (double*)malloc(sizeof(double) * (size_t)(Lmax + 1));
    for (int b = 0; b < B; ++b) {
        const int Pb = P[b];
        for (int u = 0; u < n_nodes[b]; ++u) {
            const uint64_t* mu = mask + ((size_t)b * T + u) * W;
            for (int h = 0; h < H; ++h) {
                const int hk = h / group;
                const double* qr = q + (((size_t)b * T + u) * H + h) * D;
                const double* kb = kc + ((size_t)b * Hkv + hk) * (size_t)Lmax * D;
                const double* vb = vc + ((size_t)b * Hkv + hk) * (size_t)Lmax * D;
                const int rows = Pb + n_nodes[b];
                double mx = -INFINITY;
                for (int p = 0; p < rows; ++p) {
                    int vis = 1;
                    if (p >= Pb) {
                        int v = p - Pb;
                        vis = (int)((mu[v / 64] >> (v % 64)) & 1u);
                    }
                    if (!vis) { s[p] = -INFINITY; continue; }
                    double acc = 0.0;
                    for (int t = 0; t < D; ++t) acc += qr[t] * kb[(size_t)p * D + t];
                    s[p] = acc * scale;
                    if (s[p] > mx) mx = s[p];
                }
                double denom = 0.0;
                for (int p = 0; p < rows; ++p) {
                    s[p] = (s[p] == -INFINITY) ? 0.0 : exp(s[p] - mx);
                    denom += s[p];
                }
                double* orow = o + (((size_t)b * T + u) * H + h) * D;
                for (int t = 0; t < D; ++t) orow[t] = 0.0;
                for (int p = 0; p < rows; ++p) {
                    if (s[p] == 0.0) continue;
                    const double w = s[p] / denom;
                    for (int t = 0; t < D; ++t) orow[t] += w * vb[(size_t)p * D + t];
                }
                if (lse) lse[((size_t)b * H + h) * T + u] = mx + log(denom);
            }
        }
    }
    free(s);
}

/* -------------------------------------------------------- greedy verify --- */
int or_greedy_verify(const float* logits, int V, const int32_t* tok, const int32_t* parent, int n,
                     int32_t* out_tokens, int32_t* verified, int32_t* ids, int* n_verified) {
    for (int u = 0; u < n; ++u) out_tokens[u] = or_argmax_f32(logits + (size_t)u * V, V);
    return or_verify(tok, parent, n, out_tokens, n, verified, ids, n_verified);
}

/* ------------------------------------------------------------------ MSS --- */
/* Defined in restate_mss.c. */
