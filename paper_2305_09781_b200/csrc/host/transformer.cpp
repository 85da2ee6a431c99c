// Drop-in C++ transformer API (include/spectree/transformer.hpp) over the
// sm_100a kernels. Reference: proj/src/transformer.cpp (same observable
// behaviour and error codes; different machinery).
//
// Every forward pass — prefill, decode_incremental, chain_attention_step,
// final_hidden, attention() and tree_parallel_decode — is one batched GPU pass
// over all its rows: embeddings -> per layer [LN1, QKV GEMM, K2 append of the
// rows' K/V into the device cache, K1 masked attention, WO GEMM + residual,
// LN2, FFN GEMMs + GELU + residual] -> LN_f -> LM-head GEMM -> device argmax.
// The reference instead loops over DFS chains and does one matvec per node
// (transformer.cpp:220-326, 394-446). Arithmetic is f64 so the reference's
// own <=1e-9 tests hold.
//
// Host state mirrors the reference exactly: KVCache keeps host f64 rows (the
// API hands out double* rows), uploaded before and written back after each
// pass; tree decoding reproduces the reference's DFS-overwrite cache contents
// and hook timing (transformer.hpp:157-172, transformer_test.cpp:425-452).
#include "spectree/transformer.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstring>
#include <list>
#include <mutex>
#include <string>

#include "../decoder.h"
#include "internal.h"
#include "spectree/rng.hpp"
#include "spectree_capi.h"

namespace spectree {

// ---------------------------------------------------------------- host API --
void matvec(std::span<const double> x, const Matrix& w, std::span<double> out) {
    std::fill(out.begin(), out.end(), 0.0);
    for (int i = 0; i < w.rows; ++i) {
        const double xi = x[i];
        const double* wr = w.row(i);
        for (int j = 0; j < w.cols; ++j) out[j] += xi * wr[j];
    }
}

void ModelConfig::validate() const {
    if (num_layers < 1 || num_heads < 1 || d_model < 1 || vocab_size < 2 || max_positions < 1 ||
        ffn_mult < 1)
        fail(Errc::shape_mismatch, "model config: all dims must be >= 1 (vocab >= 2)");
    if (d_model % num_heads != 0)
        fail(Errc::shape_mismatch, "model config: d_model " + std::to_string(d_model) +
                                       " not divisible by " + std::to_string(num_heads) + " heads");
}

std::size_t ModelConfig::parameter_count() const {
    const std::size_t d = d_model, f = ffn_dim(), L = num_layers;
    return (std::size_t)vocab_size * d * 2 + (std::size_t)max_positions * d +
           L * (4 * d * d + 2 * d * f + 4 * d) + 2 * d;
}

ModelWeights init_random_weights(const ModelConfig& cfg, std::uint64_t seed) {
    cfg.validate();
    constexpr double lo = -0.08, hi = 0.08;
    ModelWeights w;
    w.config = cfg;
    UniformStream rng(seed);
    const int d = cfg.d_model, f = cfg.ffn_dim();
    w.token_embedding = Matrix(cfg.vocab_size, d);
    rng.fill(w.token_embedding, lo, hi);
    w.position_embedding = Matrix(cfg.max_positions, d);
    rng.fill(w.position_embedding, lo, hi);
    w.layers.resize(cfg.num_layers);
    for (auto& L : w.layers) {
        for (auto* v : {&L.ln1_gamma, &L.ln1_beta}) {
            v->resize(d);
            rng.fill(*v, lo, hi);
        }
        for (auto* m : {&L.wq, &L.wk, &L.wv, &L.wo}) {
            *m = Matrix(d, d);
            rng.fill(*m, lo, hi);
        }
        for (auto* v : {&L.ln2_gamma, &L.ln2_beta}) {
            v->resize(d);
            rng.fill(*v, lo, hi);
        }
        L.w_ff1 = Matrix(d, f);
        rng.fill(L.w_ff1, lo, hi);
        L.w_ff2 = Matrix(f, d);
        rng.fill(L.w_ff2, lo, hi);
    }
    w.lnf_gamma.resize(d);
    w.lnf_beta.resize(d);
    rng.fill(w.lnf_gamma, lo, hi);
    rng.fill(w.lnf_beta, lo, hi);
    w.output_projection = Matrix(d, cfg.vocab_size);
    rng.fill(w.output_projection, lo, hi);
    return w;
}

TokenId argmax_token(std::span<const double> logits) {
    int best = 0;
    for (int i = 1; i < static_cast<int>(logits.size()); ++i)
        if (logits[i] > logits[best]) best = i;
    return best;
}

Matrix causal_mask(int rows) {
    Matrix m(rows, rows);
    for (int j = 0; j < rows; ++j)
        for (int k = j + 1; k < rows; ++k) m.at(j, k) = kMaskNegInf;
    return m;
}

// ------------------------------------------------------------ device side --
namespace {

std::recursive_mutex g_mu;

[[noreturn]] void throw_status(st_status st, const std::string& what) {
    const int e = st - 1;
    if (e >= 0 && e < 16) throw Error(static_cast<Errc>(e), what + ": " + st_last_error_message());
    throw std::runtime_error(what + ": " + st_last_error_message() + " (status " +
                             std::to_string(st) + ")");
}

void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) {
        cudaGetLastError();
        int n = 0;
        if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
            cudaGetLastError();
            throw std::runtime_error(std::string(what) +
                                     ": no CUDA device (the B200 path has no CPU fallback)");
        }
        throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
    }
}

void st_ok(st_status st, const char* what) {
    if (st != ST_OK) throw_status(st, what);
}

cudaStream_t stream() {
    static cudaStream_t s = [] {
        cudaStream_t x = nullptr;
        cuda_ok(cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking), "cudaStreamCreate");
        return x;
    }();
    return s;
}

// Grow-only device scratch.
struct Arena {
    char* base = nullptr;
    size_t cap = 0, used = 0;
    void reset(size_t need) {
        if (need > cap) {
            if (base) cudaFree(base);
            cap = std::max(need, cap * 2);
            cuda_ok(cudaMalloc(&base, cap), "cudaMalloc(arena)");
        }
        used = 0;
    }
    template <class T>
    T* take(size_t n) {
        used = (used + 255) & ~size_t(255);
        T* p = reinterpret_cast<T*>(base + used);
        used += n * sizeof(T);
        return p;
    }
};
Arena g_arena;

// Device copy of a ModelWeights, cached by address + content fingerprint.
struct DeviceModel {
    ModelConfig cfg;
    const void* key = nullptr;
    uint64_t fp = 0;
    double* buf = nullptr;
    const double *tok = nullptr, *pos = nullptr, *lnf_g = nullptr, *lnf_b = nullptr,
                 *wout = nullptr;
    struct Layer {
        const double *ln1_g, *ln1_b, *wq, *wk, *wv, *wo, *ln2_g, *ln2_b, *w1, *w2;
    };
    std::vector<Layer> layers;
    ~DeviceModel() {
        if (buf) cudaFree(buf);
    }
};

// Hash of EVERY weight (an in-place edit anywhere must re-upload; a sampled
// hash missed edits between samples). Four independent multiply-xor lanes keep
// it at memory speed — far below the reference's own per-node weight traffic.
uint64_t fingerprint(const ModelWeights& w) {
    uint64_t h = 1469598103934665603ull;
    auto mixv = [&](const std::vector<double>& v) {
        uint64_t a[4] = {h, h ^ 0x9e3779b97f4a7c15ull, h ^ 0xbf58476d1ce4e5b9ull,
                         h ^ 0x94d049bb133111ebull};
        const size_t n = v.size(), n4 = n & ~size_t(3);
        const auto* p = reinterpret_cast<const unsigned char*>(v.data());
        for (size_t i = 0; i < n4; i += 4)
            for (int j = 0; j < 4; ++j) {
                uint64_t b;
                std::memcpy(&b, p + (i + j) * 8, 8);
                a[j] = (a[j] ^ b) * 0x100000001b3ull;
            }
        for (size_t i = n4; i < n; ++i) {
            uint64_t b;
            std::memcpy(&b, p + i * 8, 8);
            a[0] = (a[0] ^ b) * 0x100000001b3ull;
        }
        for (int j = 0; j < 4; ++j) h = (h ^ a[j]) * 1099511628211ull;
        h = (h ^ n) * 1099511628211ull;
    };
    const auto& c = w.config;
    for (int x : {c.num_layers, c.num_heads, c.d_model, c.vocab_size, c.max_positions, c.ffn_mult})
        h = (h ^ (uint64_t)x) * 1099511628211ull;
    mixv(w.token_embedding.data);
    mixv(w.position_embedding.data);
    for (const auto& L : w.layers)
        for (const auto* v : {&L.ln1_gamma, &L.ln1_beta, &L.wq.data, &L.wk.data, &L.wv.data,
                              &L.wo.data, &L.ln2_gamma, &L.ln2_beta, &L.w_ff1.data, &L.w_ff2.data})
            mixv(*v);
    mixv(w.lnf_gamma);
    mixv(w.lnf_beta);
    mixv(w.output_projection.data);
    return h;
}

DeviceModel& device_model(const ModelWeights& w) {
    static std::list<DeviceModel> cache;  // most recent first
    const uint64_t fp = fingerprint(w);
    for (auto it = cache.begin(); it != cache.end(); ++it)
        if (it->key == &w && it->fp == fp) {
            cache.splice(cache.begin(), cache, it);
            return cache.front();
        }
    while (cache.size() >= 4) cache.pop_back();
    cache.emplace_front();
    DeviceModel& m = cache.front();
    m.cfg = w.config;
    m.key = &w;
    m.fp = fp;
    std::vector<double> host;
    host.reserve(w.config.parameter_count());
    std::vector<size_t> off;
    auto put = [&](const std::vector<double>& v) {
        off.push_back(host.size());
        host.insert(host.end(), v.begin(), v.end());
    };
    put(w.token_embedding.data);
    put(w.position_embedding.data);
    for (const auto& L : w.layers)
        for (const auto* v : {&L.ln1_gamma, &L.ln1_beta, &L.wq.data, &L.wk.data, &L.wv.data,
                              &L.wo.data, &L.ln2_gamma, &L.ln2_beta, &L.w_ff1.data, &L.w_ff2.data})
            put(*v);
    put(w.lnf_gamma);
    put(w.lnf_beta);
    put(w.output_projection.data);
    cuda_ok(cudaMalloc(&m.buf, host.size() * sizeof(double)), "cudaMalloc(weights)");
    cuda_ok(cudaMemcpy(m.buf, host.data(), host.size() * sizeof(double), cudaMemcpyHostToDevice),
            "upload weights");
    size_t k = 0;
    m.tok = m.buf + off[k++];
    m.pos = m.buf + off[k++];
    m.layers.resize(w.layers.size());
    for (auto& L : m.layers) {
        const double** f[] = {&L.ln1_g, &L.ln1_b, &L.wq, &L.wk, &L.wv,
                              &L.wo,    &L.ln2_g, &L.ln2_b, &L.w1, &L.w2};
        for (auto* p : f) *p = m.buf + off[k++];
    }
    m.lnf_g = m.buf + off[k++];
    m.lnf_b = m.buf + off[k++];
    m.wout = m.buf + off[k++];
    return m;
}

}  // namespace

namespace detail {

// Make room for rows [0, rows) in the device mirror (tree scratch may extend
// past max_positions: node rows are indexed by id, positions by depth).
void ensure_rows(DeviceKV& dk, int rows) {
    if (rows <= dk.Lmax && dk.k) return;
    if (dk.authoritative && dk.k)
        throw std::runtime_error("device KV cache cannot grow while authoritative");
    dk.release();
    dk.Lmax = std::max(rows, dk.Lmax);
    const size_t bytes = (size_t)dk.layers * dk.layer_elems() * sizeof(double);
    cuda_ok(cudaMalloc(&dk.k, bytes), "cudaMalloc(kv)");
    cuda_ok(cudaMalloc(&dk.v, bytes), "cudaMalloc(kv)");
    cuda_ok(cudaMemset(dk.k, 0, bytes), "memset kv");
    cuda_ok(cudaMemset(dk.v, 0, bytes), "memset kv");
}

}  // namespace detail

namespace {

struct PassResult {
    std::vector<LogitRow> logits;
    std::vector<TokenId> argmax;
    std::vector<std::vector<double>> hidden;
    std::vector<double> k_rows, v_rows;  // [layer][n][d_model] of the pass's rows
    int32_t* argmax_dev = nullptr;        // valid until the next pass
};

// Upload host cache rows [0, P) of every layer into the device mirror.
void upload_prefix(const KVCache& cache, detail::DeviceKV& dk, int P) {
    const int d = cache.config().d_model;
    for (int l = 0; l < dk.layers; ++l)
        for (int h = 0; h < dk.H; ++h) {
            if (P == 0) continue;
            const size_t dst = (size_t)l * dk.layer_elems() + (size_t)h * dk.Lmax * dk.Dh;
            cuda_ok(cudaMemcpy2DAsync(dk.k + dst, dk.Dh * 8, cache.key_row(l, 0) + h * dk.Dh, d * 8,
                                      dk.Dh * 8, P, cudaMemcpyHostToDevice, stream()),
                    "upload K");
            cuda_ok(cudaMemcpy2DAsync(dk.v + dst, dk.Dh * 8, cache.value_row(l, 0) + h * dk.Dh,
                                      d * 8, dk.Dh * 8, P, cudaMemcpyHostToDevice, stream()),
                    "upload V");
        }
}

// One batched forward pass of n rows: rows see cache rows [0, P) plus the
// rows whose bit is set in their mask; row i's K/V land in device rows P+i.
PassResult forward_pass(const ModelWeights& w, KVCache& cache, const std::vector<TokenId>& tokens,
                        const std::vector<int32_t>& positions, int P,
                        const std::vector<uint64_t>& masks, int W, bool want_hidden) {
    const ModelConfig& c = w.config;
    const int n = static_cast<int>(tokens.size());
    const int d = c.d_model, H = c.num_heads, Dh = c.head_dim(), F = c.ffn_dim(),
              V = c.vocab_size;
    DeviceModel& m = device_model(w);
    detail::DeviceKV& dk = cache.device();
    detail::ensure_rows(dk, P + n);
    cudaStream_t s = stream();
    const bool host_rows = !dk.authoritative;
    if (host_rows) upload_prefix(cache, dk, P);

    g_arena.reset(sizeof(double) * ((size_t)n * (6 * d + F + V + d) + 4096) +
                  sizeof(int32_t) * (4 * n + 8) + sizeof(uint64_t) * (size_t)n * W + 16 * 256);
    double* x = g_arena.take<double>((size_t)n * d);
    double* hbuf = g_arena.take<double>((size_t)n * d);
    double* q = g_arena.take<double>((size_t)n * d);
    double* kn = g_arena.take<double>((size_t)n * d);
    double* vn = g_arena.take<double>((size_t)n * d);
    double* att = g_arena.take<double>((size_t)n * d);
    double* ff = g_arena.take<double>((size_t)n * F);
    double* logits = g_arena.take<double>((size_t)n * V);
    int32_t* dtok = g_arena.take<int32_t>(n);
    int32_t* dpos = g_arena.take<int32_t>(n);
    int32_t* dam = g_arena.take<int32_t>(n);
    int32_t* dPn = g_arena.take<int32_t>(2);
    uint64_t* dmask = g_arena.take<uint64_t>((size_t)n * W);

    std::vector<int32_t> pn{P, n};
    cuda_ok(cudaMemcpyAsync(dtok, tokens.data(), n * 4, cudaMemcpyHostToDevice, s), "h2d tokens");
    cuda_ok(cudaMemcpyAsync(dpos, positions.data(), n * 4, cudaMemcpyHostToDevice, s), "h2d pos");
    cuda_ok(cudaMemcpyAsync(dPn, pn.data(), 8, cudaMemcpyHostToDevice, s), "h2d P");
    cuda_ok(cudaMemcpyAsync(dmask, masks.data(), (size_t)n * W * 8, cudaMemcpyHostToDevice, s),
            "h2d mask");

    st_ok(st::embed<double>(m.tok, m.pos, dtok, dpos, n, d, x, s), "embed");
    for (int l = 0; l < c.num_layers; ++l) {
        const auto& L = m.layers[l];
        double* kc = dk.k + (size_t)l * dk.layer_elems();
        double* vc = dk.v + (size_t)l * dk.layer_elems();
        st_ok(st::layernorm<double>(x, L.ln1_g, L.ln1_b, n, d, hbuf, s), "ln1");
        st_ok(st::gemm<double>(hbuf, L.wq, q, n, d, d, false, s), "wq");
        st_ok(st::gemm<double>(hbuf, L.wk, kn, n, d, d, false, s), "wk");
        st_ok(st::gemm<double>(hbuf, L.wv, vn, n, d, d, false, s), "wv");
        st_ok(st_kv_append(ST_F64, 1, n, H, Dh, dk.Lmax, kn, vn, dPn, dPn + 1, kc, vc, s),
              "kv_append");
        st_attn_args a{};
        a.dtype = ST_F64;
        a.B = 1;
        a.T = n;
        a.H = H;
        a.Hkv = H;
        a.D = Dh;
        a.W = W;
        a.Lmax = dk.Lmax;
        a.q = q;
        a.k_cache = kc;
        a.v_cache = vc;
        a.mask = dmask;
        a.prefix_len = dPn;
        a.n_nodes = dPn + 1;
        a.o = att;
        a.scale = 1.0 / std::sqrt(static_cast<double>(Dh));
        a.force_path = 1;
        st_ok(st_tree_attention(&a, s), "tree_attention");
        st_ok(st::gemm<double>(att, L.wo, x, n, d, d, true, s), "wo");
        st_ok(st::layernorm<double>(x, L.ln2_g, L.ln2_b, n, d, hbuf, s), "ln2");
        st_ok(st::gemm<double>(hbuf, L.w1, ff, n, F, d, false, s), "w1");
        st_ok(st::gelu<double>(ff, (int64_t)n * F, s), "gelu");
        st_ok(st::gemm<double>(ff, L.w2, x, n, d, F, true, s), "w2");
    }
    st_ok(st::layernorm<double>(x, m.lnf_g, m.lnf_b, n, d, hbuf, s), "lnf");
    st_ok(st::gemm<double>(hbuf, m.wout, logits, n, V, d, false, s), "lm_head");
    st_ok(st::argmax_rows<double>(logits, n, V, dam, s), "argmax");

    PassResult r;
    r.argmax_dev = dam;
    r.argmax.resize(n);
    cuda_ok(cudaMemcpyAsync(r.argmax.data(), dam, n * 4, cudaMemcpyDeviceToHost, s), "d2h argmax");
    if (!host_rows) {  // device-authoritative (engine): only the greedy tokens come back
        std::vector<double> hh;
        if (want_hidden) {
            hh.resize((size_t)n * d);
            cuda_ok(cudaMemcpyAsync(hh.data(), hbuf, hh.size() * 8, cudaMemcpyDeviceToHost, s),
                    "d2h hidden");
        }
        cuda_ok(cudaStreamSynchronize(s), "forward pass");
        if (want_hidden) {
            r.hidden.resize(n);
            for (int i = 0; i < n; ++i)
                r.hidden[i].assign(hh.begin() + (size_t)i * d, hh.begin() + (size_t)(i + 1) * d);
        }
        return r;
    }
    std::vector<double> hl((size_t)n * V);
    cuda_ok(cudaMemcpyAsync(hl.data(), logits, hl.size() * 8, cudaMemcpyDeviceToHost, s),
            "d2h logits");
    std::vector<double> hh;
    if (want_hidden) {
        hh.resize((size_t)n * d);
        cuda_ok(cudaMemcpyAsync(hh.data(), hbuf, hh.size() * 8, cudaMemcpyDeviceToHost, s),
                "d2h hidden");
    }
    // the pass's K/V rows back to host layout [layer][n][d_model]
    r.k_rows.resize((size_t)c.num_layers * n * d);
    r.v_rows.resize((size_t)c.num_layers * n * d);
    for (int l = 0; l < c.num_layers; ++l)
        for (int h = 0; h < H; ++h) {
            const size_t src = (size_t)l * dk.layer_elems() + ((size_t)h * dk.Lmax + P) * Dh;
            cuda_ok(cudaMemcpy2DAsync(r.k_rows.data() + (size_t)l * n * d + h * Dh, d * 8,
                                      dk.k + src, Dh * 8, Dh * 8, n, cudaMemcpyDeviceToHost, s),
                    "d2h K rows");
            cuda_ok(cudaMemcpy2DAsync(r.v_rows.data() + (size_t)l * n * d + h * Dh, d * 8,
                                      dk.v + src, Dh * 8, Dh * 8, n, cudaMemcpyDeviceToHost, s),
                    "d2h V rows");
        }
    cuda_ok(cudaStreamSynchronize(s), "forward pass");
    r.logits.resize(n);
    for (int i = 0; i < n; ++i)
        r.logits[i].assign(hl.begin() + (size_t)i * V, hl.begin() + (size_t)(i + 1) * V);
    if (want_hidden) {
        r.hidden.resize(n);
        for (int i = 0; i < n; ++i)
            r.hidden[i].assign(hh.begin() + (size_t)i * d, hh.begin() + (size_t)(i + 1) * d);
    }
    return r;
}

// host cache row <- row i of a pass (no-op while the device is authoritative)
void put_row(KVCache& cache, const PassResult& r, int n, int i, int position) {
    if (r.k_rows.empty()) return;
    const auto& c = cache.config();
    const int d = c.d_model;
    for (int l = 0; l < c.num_layers; ++l) {
        std::memcpy(cache.key_row(l, position), r.k_rows.data() + ((size_t)l * n + i) * d, d * 8);
        std::memcpy(cache.value_row(l, position), r.v_rows.data() + ((size_t)l * n + i) * d, d * 8);
    }
}

void validate_chain(const TokenTree& tree, std::span<const int> chain) {
    if (chain.empty()) fail(Errc::empty_input, "chain_attention_step: empty chain");
    for (size_t i = 1; i < chain.size(); ++i)
        if (tree.parent(chain[i]) != chain[i - 1])
            fail(Errc::chain_not_linked, "chain element " + std::to_string(chain[i]) +
                                             " is not a child of its predecessor " +
                                             std::to_string(chain[i - 1]));
}

}  // namespace

// -------------------------------------------------------------- KVCache ----
KVCache::KVCache(const ModelConfig& config) : config_(config) {
    config.validate();
    const size_t per_layer = (size_t)config.max_positions * config.d_model;
    keys_.assign(config.num_layers, std::vector<double>(per_layer, 0.0));
    values_.assign(config.num_layers, std::vector<double>(per_layer, 0.0));
    tokens_.assign(config.max_positions, kNoEosToken);
}
KVCache::KVCache(const KVCache& o)
    : config_(o.config_), occupancy_(o.occupancy_), keys_(o.keys_), values_(o.values_),
      tokens_(o.tokens_) {}
KVCache& KVCache::operator=(const KVCache& o) {
    if (this != &o) {
        config_ = o.config_;
        occupancy_ = o.occupancy_;
        keys_ = o.keys_;
        values_ = o.values_;
        tokens_ = o.tokens_;
        dev_.reset();
    }
    return *this;
}
KVCache::KVCache(KVCache&&) noexcept = default;
KVCache& KVCache::operator=(KVCache&&) noexcept = default;
KVCache::~KVCache() = default;

void KVCache::rollback(int new_occupancy) {
    if (new_occupancy < 0 || new_occupancy > occupancy_)
        fail(Errc::invalid_argument, "rollback: bad occupancy " + std::to_string(new_occupancy));
    occupancy_ = new_occupancy;
}

double* KVCache::key_row(int layer, int position) {
    return keys_[layer].data() + (size_t)position * config_.d_model;
}
double* KVCache::value_row(int layer, int position) {
    return values_[layer].data() + (size_t)position * config_.d_model;
}
const double* KVCache::key_row(int layer, int position) const {
    return keys_[layer].data() + (size_t)position * config_.d_model;
}
const double* KVCache::value_row(int layer, int position) const {
    return values_[layer].data() + (size_t)position * config_.d_model;
}

detail::DeviceKV& KVCache::device() const {
    if (!dev_) {
        auto dk = std::make_unique<detail::DeviceKV>();
        dk->layers = config_.num_layers;
        dk->H = config_.num_heads;
        dk->Dh = config_.head_dim();
        dk->Lmax = config_.max_positions;
        const size_t bytes = (size_t)dk->layers * dk->layer_elems() * sizeof(double);
        cuda_ok(cudaMalloc(&dk->k, bytes), "cudaMalloc(kv)");
        cuda_ok(cudaMalloc(&dk->v, bytes), "cudaMalloc(kv)");
        cuda_ok(cudaMemset(dk->k, 0, bytes), "memset kv");
        cuda_ok(cudaMemset(dk->v, 0, bytes), "memset kv");
        dev_ = std::move(dk);
    }
    return *dev_;
}

// ------------------------------------------------------------ attention() --
Matrix attention(const Matrix& x, const Matrix& wq, const Matrix& wk, const Matrix& wv,
                 const Matrix& wo, int num_heads, const Matrix& mask) {
    const int l = x.rows, d = x.cols;
    if (d == 0 || num_heads < 1 || d % num_heads != 0)
        fail(Errc::shape_mismatch, "attention: bad head split");
    for (const Matrix* m : {&wq, &wk, &wv, &wo})
        if (m->rows != d || m->cols != d) fail(Errc::shape_mismatch, "attention: weight shape mismatch");
    if (mask.rows != l || mask.cols != l) fail(Errc::shape_mismatch, "attention: mask must be l x l");
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    const int Dh = d / num_heads, W = (l + 63) / 64;
    cudaStream_t s = stream();
    g_arena.reset(sizeof(double) * ((size_t)10 * l * d + 4 * (size_t)d * d + 4096) +
                  sizeof(uint64_t) * (size_t)l * W + 4096);
    double* dx = g_arena.take<double>((size_t)l * d);
    double* dw[4];
    for (auto& p : dw) p = g_arena.take<double>((size_t)d * d);
    double* q = g_arena.take<double>((size_t)l * d);
    double* k = g_arena.take<double>((size_t)l * d);
    double* v = g_arena.take<double>((size_t)l * d);
    double* kc = g_arena.take<double>((size_t)l * d);
    double* vc = g_arena.take<double>((size_t)l * d);
    double* heads = g_arena.take<double>((size_t)l * d);
    double* out = g_arena.take<double>((size_t)l * d);
    int32_t* dPn = g_arena.take<int32_t>(2);
    uint64_t* dmask = g_arena.take<uint64_t>((size_t)l * W);
    std::vector<uint64_t> bits((size_t)l * W, 0);
    for (int j = 0; j < l; ++j)
        for (int c = 0; c < l; ++c)
            if (mask.at(j, c) == 0.0) bits[(size_t)j * W + c / 64] |= 1ull << (c % 64);
    const int32_t pn[2] = {0, l};
    cuda_ok(cudaMemcpyAsync(dx, x.data.data(), (size_t)l * d * 8, cudaMemcpyHostToDevice, s), "h2d");
    const Matrix* ws[4] = {&wq, &wk, &wv, &wo};
    for (int i = 0; i < 4; ++i)
        cuda_ok(cudaMemcpyAsync(dw[i], ws[i]->data.data(), (size_t)d * d * 8, cudaMemcpyHostToDevice, s),
                "h2d");
    cuda_ok(cudaMemcpyAsync(dPn, pn, 8, cudaMemcpyHostToDevice, s), "h2d");
    cuda_ok(cudaMemcpyAsync(dmask, bits.data(), bits.size() * 8, cudaMemcpyHostToDevice, s), "h2d");
    st_ok(st::gemm<double>(dx, dw[0], q, l, d, d, false, s), "wq");
    st_ok(st::gemm<double>(dx, dw[1], k, l, d, d, false, s), "wk");
    st_ok(st::gemm<double>(dx, dw[2], v, l, d, d, false, s), "wv");
    st_ok(st_kv_append(ST_F64, 1, l, num_heads, Dh, l, k, v, dPn, dPn + 1, kc, vc, s), "append");
    st_attn_args a{};
    a.dtype = ST_F64;
    a.B = 1;
    a.T = l;
    a.H = num_heads;
    a.Hkv = num_heads;
    a.D = Dh;
    a.W = W;
    a.Lmax = l;
    a.q = q;
    a.k_cache = kc;
    a.v_cache = vc;
    a.mask = dmask;
    a.prefix_len = dPn;
    a.n_nodes = dPn + 1;
    a.o = heads;
    a.scale = 1.0 / std::sqrt(static_cast<double>(Dh));
    a.force_path = 1;
    st_ok(st_tree_attention(&a, s), "attention");
    st_ok(st::gemm<double>(heads, dw[3], out, l, d, d, false, s), "wo");
    Matrix o(l, d);
    cuda_ok(cudaMemcpyAsync(o.data.data(), out, (size_t)l * d * 8, cudaMemcpyDeviceToHost, s), "d2h");
    cuda_ok(cudaStreamSynchronize(s), "attention");
    return o;
}

// ----------------------------------------------------------- chain decode --
namespace detail {

std::vector<LogitRow> chain_attention_step_impl(const ModelWeights& w,
                                                std::span<const TokenId> chain_tokens,
                                                int base_position, KVCache& cache,
                                                bool apply_causal_fix,
                                                std::vector<std::vector<double>>* hidden_rows) {
    const ModelConfig& cfg = w.config;
    const int len = static_cast<int>(chain_tokens.size());
    if (len == 0) fail(Errc::empty_input, "chain_attention_step: empty chain");
    if (base_position < 0 || base_position + len > cfg.max_positions)
        fail(Errc::tree_too_deep, "chain_attention_step: positions " + std::to_string(base_position) +
                                      ".." + std::to_string(base_position + len - 1) +
                                      " exceed max " + std::to_string(cfg.max_positions));
    for (TokenId t : chain_tokens)
        if (t < 0 || t >= cfg.vocab_size)
            fail(Errc::invalid_argument, "chain_attention_step: token out of vocab");
    std::lock_guard<std::recursive_mutex> lock(g_mu);
    const int W = (len + 63) / 64;
    std::vector<uint64_t> masks((size_t)len * W, 0);
    std::vector<int32_t> pos(len);
    for (int i = 0; i < len; ++i) {
        pos[i] = base_position + i;
        const int upto = apply_causal_fix ? i : len - 1;
        for (int j = 0; j <= upto; ++j) masks[(size_t)i * W + j / 64] |= 1ull << (j % 64);
    }
    std::vector<TokenId> toks(chain_tokens.begin(), chain_tokens.end());
    PassResult r = forward_pass(w, cache, toks, pos, base_position, masks, W, hidden_rows != nullptr);
    for (int i = 0; i < len; ++i) {
        put_row(cache, r, len, i, base_position + i);
        cache.record_token(base_position + i, chain_tokens[i]);
    }
    if (base_position <= cache.occupancy()) cache.set_occupancy(base_position + len);
    if (hidden_rows) *hidden_rows = std::move(r.hidden);
    return std::move(r.logits);
}

}  // namespace detail

std::vector<LogitRow> chain_attention_step(const ModelWeights& w,
                                           std::span<const TokenId> chain_tokens,
                                           int base_position, KVCache& cache) {
    return detail::chain_attention_step_impl(w, chain_tokens, base_position, cache, true);
}

std::vector<LogitRow> chain_attention_step(const ModelWeights& w, const TokenTree& tree,
                                           std::span<const int> chain, int prefix_len,
                                           KVCache& cache) {
    validate_chain(tree, chain);
    std::vector<TokenId> toks;
    for (int node : chain) toks.push_back(tree.token(node));
    return detail::chain_attention_step_impl(w, toks, prefix_len - 1 + tree.depth(chain.front()),
                                             cache, true);
}

LogitRow prefill(const ModelWeights& w, std::span<const TokenId> prompt, KVCache& cache) {
    if (prompt.empty()) fail(Errc::empty_input, "prefill: empty prompt");
    if (static_cast<int>(prompt.size()) > w.config.max_positions)
        fail(Errc::prompt_too_long, "prefill: prompt length " + std::to_string(prompt.size()) +
                                        " exceeds max positions " +
                                        std::to_string(w.config.max_positions));
    cache.rollback(0);
    auto rows = detail::chain_attention_step_impl(w, prompt, 0, cache, true);
    return std::move(rows.back());
}

LogitRow decode_incremental(const ModelWeights& w, TokenId token, int position, KVCache& cache) {
    if (position < 0 || position > cache.occupancy())
        fail(Errc::cache_gap, "decode_incremental: position " + std::to_string(position) +
                                  " beyond occupancy " + std::to_string(cache.occupancy()));
    const TokenId one[1] = {token};
    auto rows = detail::chain_attention_step_impl(w, one, position, cache, true);
    return std::move(rows.front());
}

std::vector<double> final_hidden(const ModelWeights& w, KVCache& cache) {
    const int occ = cache.occupancy();
    if (occ == 0) fail(Errc::empty_context, "final_hidden: no decoded positions");
    const TokenId one[1] = {cache.token_at(occ - 1)};
    std::vector<std::vector<double>> hidden;
    detail::chain_attention_step_impl(w, one, occ - 1, cache, true, &hidden);
    return std::move(hidden.front());
}

// ------------------------------------------------------------ tree decode --
TreeDecodeResult tree_parallel_decode(const ModelWeights& w, const TokenTree& tree,
                                      int prefix_len, KVCache& cache,
                                      const TreeDecodeHooks* hooks) {
    const ModelConfig& cfg = w.config;
    if (prefix_len < 1 || cache.occupancy() != prefix_len)
        fail(Errc::cache_gap, "tree_parallel_decode: cache occupancy " +
                                  std::to_string(cache.occupancy()) + " != prefix length " +
                                  std::to_string(prefix_len));
    if (prefix_len + tree.max_depth() > cfg.max_positions)
        fail(Errc::tree_too_deep, "tree_parallel_decode: prefix " + std::to_string(prefix_len) +
                                      " + depth " + std::to_string(tree.max_depth()) +
                                      " exceeds max positions " + std::to_string(cfg.max_positions));
    if (cache.token_at(prefix_len - 1) != tree.token(tree.root()))
        fail(Errc::root_mismatch,
             "tree_parallel_decode: root token does not match the cached last verified token");
    const int n = tree.size();
    for (int u = 0; u < n; ++u)
        if (tree.token(u) < 0 || tree.token(u) >= cfg.vocab_size)
            fail(Errc::invalid_argument, "tree_parallel_decode: token out of vocab");
    const bool fix = hooks == nullptr || hooks->apply_chain_causal_fix;
    std::lock_guard<std::recursive_mutex> lock(g_mu);

    const int P = prefix_len - 1;
    const int W = (n + 63) / 64;
    std::vector<uint64_t> masks((size_t)n * W, 0);
    std::vector<int32_t> pos(n);
    std::vector<TokenId> toks(n);
    for (int u = 0; u < n; ++u) {
        toks[u] = tree.token(u);
        pos[u] = P + tree.depth(u);
        uint64_t* mu = &masks[(size_t)u * W];
        if (u > 0) std::memcpy(mu, &masks[(size_t)tree.parent(u) * W], W * 8);
        mu[u / 64] |= 1ull << (u % 64);
    }
    if (!fix) {
        // negative control: inside each DFS chain every row sees the whole
        // chain (the reference without its intra-chain re-mask, :281-285)
        for (const auto& chain : tree.dfs_chains()) {
            std::vector<uint64_t> all(W, 0);
            for (int v : chain) all[v / 64] |= 1ull << (v % 64);
            for (int v : chain)
                for (int k = 0; k < W; ++k) masks[(size_t)v * W + k] |= all[k];
        }
    }
    PassResult r = forward_pass(w, cache, toks, pos, P, masks, W, false);

    TreeDecodeResult out;
    out.tokens = r.argmax;
    out.logits = std::move(r.logits);
    // DFS-overwrite cache state + hook timing: visiting nodes in preorder,
    // node u's K/V and token land at position P + depth(u)
    for (int u = 0; u < n; ++u) {
        const int position = P + tree.depth(u);
        put_row(cache, r, n, u, position);
        cache.record_token(position, tree.token(u));
        if (hooks && hooks->on_node) hooks->on_node(u, position, cache);
    }
    cache.rollback(prefix_len);
    return out;
}

}  // namespace spectree

// ------------------------------------------------------ engine interface ---
namespace spectree::detail {

std::recursive_mutex& compat_mutex() { return g_mu; }
cudaStream_t compat_stream() { return stream(); }

void set_device_authoritative(KVCache& cache, bool on, int scratch_rows) {
    DeviceKV& dk = cache.device();
    if (on && !dk.authoritative)
        ensure_rows(dk, cache.config().max_positions + std::max(scratch_rows, 0));
    dk.authoritative = on;
}

std::vector<TokenId> device_pass(const ModelWeights& w, KVCache& cache,
                                 const std::vector<TokenId>& tokens,
                                 const std::vector<int32_t>& positions, int P,
                                 const std::vector<uint64_t>& masks, int W,
                                 int32_t** argmax_dev) {
    PassResult r = forward_pass(w, cache, tokens, positions, P, masks, W, false);
    if (argmax_dev) *argmax_dev = r.argmax_dev;
    return r.argmax;
}

}  // namespace spectree::detail
