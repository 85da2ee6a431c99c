// TEST INFRASTRUCTURE ONLY — a C shim over the UNMODIFIED reference library
// (/root/reference/proj, compiled by oracle/Makefile into oracle/_ref/).
//
// Purpose: let the Python test suite, the golden-vector generator
// (oracle/gen_golden.py) and bench.py's `cpu_baseline` / `--impl reference`
// arm drive the reference's own public API (proj/include/spectree/*.hpp)
// through ctypes. Nothing in the product links this file.
//
// Status convention: 0 = ok, otherwise 1 + (int)spectree::Errc
// (proj/include/spectree/error.hpp:8-25), -1 = buffer too small / other.

#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstring>
#include <map>
#include <memory>
#include <mutex>
#include <thread>
#include <tuple>
#include <vector>

#include "spectree/engine.hpp"
#include "spectree/rng.hpp"
#include "spectree/speculator.hpp"
#include "spectree/token_tree.hpp"
#include "spectree/transformer.hpp"

using namespace spectree;

namespace {

thread_local std::string g_last_error;

ModelConfig make_cfg(int layers, int heads, int d_model, int vocab, int max_pos, int ffn_mult) {
    ModelConfig c;
    c.num_layers = layers;
    c.num_heads = heads;
    c.d_model = d_model;
    c.vocab_size = vocab;
    c.max_positions = max_pos;
    c.ffn_mult = ffn_mult;
    return c;
}

// Weights are expensive at LLaMA shapes; keep one copy per (config, seed).
std::shared_ptr<const ModelWeights> cached_weights(const ModelConfig& c, uint64_t seed) {
    static std::mutex mu;
    static std::map<std::tuple<int, int, int, int, int, int, uint64_t>,
                    std::shared_ptr<const ModelWeights>> cache;
    std::lock_guard<std::mutex> lock(mu);
    auto key = std::make_tuple(c.num_layers, c.num_heads, c.d_model, c.vocab_size,
                               c.max_positions, c.ffn_mult, seed);
    auto it = cache.find(key);
    if (it != cache.end()) return it->second;
    if (cache.size() > 4) cache.clear();
    auto w = std::make_shared<const ModelWeights>(init_random_weights(c, seed));
    cache.emplace(key, w);
    return w;
}

std::vector<std::vector<TokenId>> unflatten(const int32_t* flat, const int32_t* lens, int nseq) {
    std::vector<std::vector<TokenId>> seqs(nseq);
    size_t at = 0;
    for (int i = 0; i < nseq; ++i) {
        seqs[i].assign(flat + at, flat + at + lens[i]);
        at += lens[i];
    }
    return seqs;
}

template <class F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const Error& e) {
        g_last_error = e.what();
        return 1 + static_cast<int>(e.code());
    } catch (const std::exception& e) {
        g_last_error = e.what();
        return -1;
    }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

// TokenTree::merge_sequences (proj/src/token_tree.cpp:42-102) flattened to
// preorder arrays.
int ref_merge(const int32_t* flat, const int32_t* lens, int nseq, int max_nodes, int32_t* tok,
              int32_t* parent, int32_t* depth, int cap, int* n_out) {
    return guarded([&] {
        const TokenTree t = TokenTree::merge_sequences(unflatten(flat, lens, nseq), max_nodes);
        *n_out = t.size();
        if (t.size() > cap) return -1;
        for (int n = 0; n < t.size(); ++n) {
            tok[n] = t.token(n);
            parent[n] = t.parent(n);
            depth[n] = t.depth(n);
        }
        return 0;
    });
}

// TokenTree::dfs_chains (proj/src/token_tree.cpp:141-151): chain ids flattened,
// chain lengths in chain_lens.
int ref_dfs_chains(const int32_t* flat, const int32_t* lens, int nseq, int max_nodes,
                   int32_t* ids, int32_t* chain_lens, int cap, int* n_chains) {
    return guarded([&] {
        const TokenTree t = TokenTree::merge_sequences(unflatten(flat, lens, nseq), max_nodes);
        const auto chains = t.dfs_chains();
        *n_chains = static_cast<int>(chains.size());
        int at = 0;
        for (size_t c = 0; c < chains.size(); ++c) {
            chain_lens[c] = static_cast<int>(chains[c].size());
            for (int id : chains[c]) {
                if (at >= cap) return -1;
                ids[at++] = id;
            }
        }
        return 0;
    });
}

// verify (proj/src/token_tree.cpp:153-175) over the merge of the given sequences.
int ref_verify(const int32_t* flat, const int32_t* lens, int nseq, int max_nodes,
               const int32_t* outputs, int n_outputs, int32_t* verified, int cap,
               int* n_verified) {
    return guarded([&] {
        const TokenTree t = TokenTree::merge_sequences(unflatten(flat, lens, nseq), max_nodes);
        const auto v = verify(t, std::span<const TokenId>(outputs, n_outputs));
        *n_verified = static_cast<int>(v.size());
        if (static_cast<int>(v.size()) > cap) return -1;
        std::copy(v.begin(), v.end(), verified);
        return 0;
    });
}

// attention() (proj/src/transformer.cpp:160-216): explicit Eq.-2 multi-head
// attention on X [l][d] with an explicit additive mask [l][l]. out: [l][d].
int ref_attention(const double* x, const double* wq, const double* wk, const double* wv,
                  const double* wo, int l, int d, int heads, const double* mask, double* out) {
    return guarded([&] {
        auto mk = [](const double* src, int r, int c) {
            Matrix m(r, c);
            std::copy(src, src + (size_t)r * c, m.data.begin());
            return m;
        };
        const Matrix o = attention(mk(x, l, d), mk(wq, d, d), mk(wk, d, d), mk(wv, d, d),
                                   mk(wo, d, d), heads, mk(mask, l, l));
        std::copy(o.data.begin(), o.data.end(), out);
        return 0;
    });
}

int ref_argmax(const double* logits, int n) {
    return argmax_token(std::span<const double>(logits, n));
}

// init_random_weights (proj/src/transformer.cpp:71-114) in serialized order.
int64_t ref_param_count(int layers, int heads, int d_model, int vocab, int max_pos,
                        int ffn_mult) {
    return static_cast<int64_t>(make_cfg(layers, heads, d_model, vocab, max_pos, ffn_mult)
                                    .parameter_count());
}

int ref_init_weights(int layers, int heads, int d_model, int vocab, int max_pos, int ffn_mult,
                     uint64_t seed, double* out, int64_t n) {
    return guarded([&] {
        const ModelConfig c = make_cfg(layers, heads, d_model, vocab, max_pos, ffn_mult);
        const ModelWeights w = init_random_weights(c, seed);
        int64_t at = 0;
        auto put = [&](const std::vector<double>& v) {
            for (double x : v) {
                if (at >= n) throw std::runtime_error("ref_init_weights: buffer too small");
                out[at++] = x;
            }
        };
        put(w.token_embedding.data);
        put(w.position_embedding.data);
        for (const auto& l : w.layers) {
            put(l.ln1_gamma); put(l.ln1_beta);
            put(l.wq.data); put(l.wk.data); put(l.wv.data); put(l.wo.data);
            put(l.ln2_gamma); put(l.ln2_beta);
            put(l.w_ff1.data); put(l.w_ff2.data);
        }
        put(w.lnf_gamma); put(w.lnf_beta);
        put(w.output_projection.data);
        return 0;
    });
}

// prefill(prompt) then tree_parallel_decode (proj/src/transformer.cpp:394-446).
// logits: [T][vocab] f64, tokens: [T].
int ref_tree_decode(int layers, int heads, int d_model, int vocab, int max_pos, int ffn_mult,
                    uint64_t seed, const int32_t* prompt, int prompt_len, const int32_t* flat,
                    const int32_t* lens, int nseq, int max_nodes, int apply_fix, double* logits,
                    int32_t* tokens, int cap_nodes, int* n_nodes) {
    return guarded([&] {
        const ModelConfig c = make_cfg(layers, heads, d_model, vocab, max_pos, ffn_mult);
        auto w = cached_weights(c, seed);
        const TokenTree t = TokenTree::merge_sequences(unflatten(flat, lens, nseq), max_nodes);
        *n_nodes = t.size();
        if (t.size() > cap_nodes) return -1;
        KVCache cache(c);
        prefill(*w, std::span<const TokenId>(prompt, prompt_len), cache);
        TreeDecodeHooks hooks;
        hooks.apply_chain_causal_fix = apply_fix != 0;
        const auto r = tree_parallel_decode(*w, t, prompt_len, cache, &hooks);
        for (int n = 0; n < t.size(); ++n) {
            tokens[n] = r.tokens[n];
            std::copy(r.logits[n].begin(), r.logits[n].end(), logits + (size_t)n * vocab);
        }
        return 0;
    });
}

// Per-path incremental oracle (proj/tests/transformer_test.cpp:31-43): the
// logits after prefill(prompt) + decode_incremental along `path_below_root`.
int ref_per_path_logits(int layers, int heads, int d_model, int vocab, int max_pos, int ffn_mult,
                        uint64_t seed, const int32_t* prompt, int prompt_len, const int32_t* path,
                        int path_len, double* logits) {
    return guarded([&] {
        const ModelConfig c = make_cfg(layers, heads, d_model, vocab, max_pos, ffn_mult);
        auto w = cached_weights(c, seed);
        KVCache cache(c);
        LogitRow l = prefill(*w, std::span<const TokenId>(prompt, prompt_len), cache);
        int pos = prompt_len;
        for (int i = 0; i < path_len; ++i) l = decode_incremental(*w, path[i], pos++, cache);
        std::copy(l.begin(), l.end(), logits);
        return 0;
    });
}

// Alg.-1 greedy loop (proj/src/engine.cpp:39-62).
int ref_run_incremental(int layers, int heads, int d_model, int vocab, int max_pos, int ffn_mult,
                        uint64_t seed, const int32_t* prompt, int prompt_len, int max_new,
                        int32_t eos, int32_t* seq_out, int cap, int* n_out, int64_t* llm_steps) {
    return guarded([&] {
        const ModelConfig c = make_cfg(layers, heads, d_model, vocab, max_pos, ffn_mult);
        auto w = cached_weights(c, seed);
        GenerationRequest req{{prompt, prompt + prompt_len}, max_new, eos};
        const auto r = run_incremental(*w, req);
        *n_out = static_cast<int>(r.sequence.size());
        *llm_steps = r.metrics.llm_steps;
        if (*n_out > cap) return -1;
        std::copy(r.sequence.begin(), r.sequence.end(), seq_out);
        return 0;
    });
}

// Alg.-2 loop (proj/src/engine.cpp:64-141) with the LLM as its own perfect
// speculator (proj/tests/acceptance_test.cpp:219-237).
int ref_run_speculative_self(int layers, int heads, int d_model, int vocab, int max_pos,
                             int ffn_mult, uint64_t seed, const int32_t* prompt, int prompt_len,
                             int max_new, int32_t eos, int beam_width, int beam_depth,
                             int max_tree_nodes, int32_t* seq_out, int cap, int* n_out,
                             int64_t* llm_steps) {
    return guarded([&] {
        const ModelConfig c = make_cfg(layers, heads, d_model, vocab, max_pos, ffn_mult);
        auto w = cached_weights(c, seed);
        std::vector<std::shared_ptr<Ssm>> pool{std::make_shared<TransformerSsm>(0, w)};
        GenerationRequest req{{prompt, prompt + prompt_len}, max_new, eos};
        SpeculativeOptions opts;
        opts.max_tree_nodes = max_tree_nodes;
        const auto r = run_speculative(*w, pool, SpecConfig{beam_width, beam_depth}, req, opts);
        *n_out = static_cast<int>(r.sequence.size());
        *llm_steps = r.metrics.llm_steps;
        if (*n_out > cap) return -1;
        std::copy(r.sequence.begin(), r.sequence.end(), seq_out);
        return 0;
    });
}

// CPU baseline: the reference tree_parallel_decode through its
// public API with prefill skipped — every request gets its own KVCache whose
// rows [0, prefix_len) are injected from a UniformStream (key_row / value_row /
// record_token / set_occupancy) — one request per std::thread over shared
// const ModelWeights. Returns wall seconds for the
// `n_requests` tree decodes (all threads), or a negative status.
double ref_bench_tree_decode(int layers, int heads, int d_model, int vocab, int max_pos,
                             int ffn_mult, uint64_t seed, int n_requests, int prefix_len,
                             const int32_t* flat, const int32_t* lens, int nseq, int max_nodes,
                             int n_threads) {
    double secs = -1.0;
    int st = guarded([&] {
        const ModelConfig c = make_cfg(layers, heads, d_model, vocab, max_pos, ffn_mult);
        auto w = cached_weights(c, seed);
        const TokenTree t = TokenTree::merge_sequences(unflatten(flat, lens, nseq), max_nodes);
        std::vector<std::unique_ptr<KVCache>> caches;
        for (int r = 0; r < n_requests; ++r) {
            auto cache = std::make_unique<KVCache>(c);
            UniformStream u(seed * 7919 + r);
            for (int l = 0; l < c.num_layers; ++l)
                for (int p = 0; p < prefix_len; ++p) {
                    double* k = cache->key_row(l, p);
                    double* v = cache->value_row(l, p);
                    for (int i = 0; i < c.d_model; ++i) k[i] = u.next(-1.0, 1.0);
                    for (int i = 0; i < c.d_model; ++i) v[i] = u.next(-1.0, 1.0);
                }
            for (int p = 0; p < prefix_len - 1; ++p) cache->record_token(p, p % c.vocab_size);
            cache->record_token(prefix_len - 1, t.token(0));
            cache->set_occupancy(prefix_len);
            caches.push_back(std::move(cache));
        }
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        const int nt = std::max(1, std::min(n_threads, n_requests));
        for (int th = 0; th < nt; ++th)
            pool.emplace_back([&, th] {
                for (int r = th; r < n_requests; r += nt)
                    (void)tree_parallel_decode(*w, t, prefix_len, *caches[r]);
            });
        for (auto& th : pool) th.join();
        secs = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        return 0;
    });
    return st == 0 ? secs : -static_cast<double>(st < 0 ? 1000 : st);
}

// beam_speculate (proj/src/speculator.cpp:97-169) with a TransformerSsm over
// init_random_weights(cfg, seed): the sequences flattened (lens[i] tokens each).
int ref_beam_speculate(int layers, int heads, int d_model, int vocab, int max_pos, int ffn_mult,
                       uint64_t seed, const int32_t* prefix, int prefix_len, int width, int depth,
                       int32_t eos, int32_t* flat, int32_t* lens, int cap, int* nseq) {
    return guarded([&] {
        const ModelConfig c = make_cfg(layers, heads, d_model, vocab, max_pos, ffn_mult);
        TransformerSsm ssm(0, cached_weights(c, seed));
        const auto seqs = beam_speculate(ssm, std::span<const TokenId>(prefix, prefix_len),
                                         SpecConfig{width, depth}, eos);
        int at = 0;
        for (size_t i = 0; i < seqs.size(); ++i) {
            if (at + (int)seqs[i].size() > cap) return -1;
            std::copy(seqs[i].begin(), seqs[i].end(), flat + at);
            lens[i] = (int32_t)seqs[i].size();
            at += (int)seqs[i].size();
        }
        *nseq = (int)seqs.size();
        return 0;
    });
}

// TransformerSsm::next_log_probs (proj/src/speculator.cpp:85-95).
int ref_next_log_probs(int layers, int heads, int d_model, int vocab, int max_pos, int ffn_mult,
                       uint64_t seed, const int32_t* ctx, int n, double* out) {
    return guarded([&] {
        const ModelConfig c = make_cfg(layers, heads, d_model, vocab, max_pos, ffn_mult);
        TransformerSsm ssm(0, cached_weights(c, seed));
        const auto lp = ssm.next_log_probs(std::span<const TokenId>(ctx, n));
        std::copy(lp.begin(), lp.end(), out);
        return 0;
    });
}

}  // extern "C"
