// Serving loop (drop-in for reference proj/src/engine.cpp's public surface).
//
// B200-native step of run_speculative, with the request's KV cache resident
// on the device for the whole generation:
//   1. speculate_tree (host C++): draft sequences merged into a TokenTree;
//   2. ONE tree pass (all nodes, every layer: K2 append + K1 masked attention);
//   3. K3 walk on device over the pass's greedy outputs, with the engine's
//      budget truncation then EOS cut (engine.cpp:110-121) applied on device;
//   4. K2 in-place compaction of the accepted root-to-node rows.
// Only the accepted tokens cross back to the host. The reference instead
// re-decodes every accepted token one forward pass at a time
// (engine.cpp:123-129).
#include "spectree/engine.hpp"

#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <string>

#include "internal.h"
#include "spectree_capi.h"

namespace spectree {

namespace {

using Clock = std::chrono::steady_clock;

double ms_since(Clock::time_point t0) {
    return std::chrono::duration<double, std::milli>(Clock::now() - t0).count();
}

void check_request(const ModelWeights& llm, const GenerationRequest& req) {
    if (req.prompt.empty()) fail(Errc::empty_input, "generation request: empty prompt");
    if (req.max_new_tokens < 1)
        fail(Errc::invalid_argument, "generation request: max_new_tokens must be >= 1");
    if (static_cast<int>(req.prompt.size()) + req.max_new_tokens > llm.config.max_positions)
        fail(Errc::prompt_too_long, "generation request: prompt + budget exceeds max positions " +
                                        std::to_string(llm.config.max_positions));
}

void ck(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

void ck(st_status s, const char* what) {
    if (s != ST_OK)
        throw std::runtime_error(std::string(what) + ": " + st_last_error_message());
}

// prompt rows [0, len): causal masks
std::vector<TokenId> prefill_device(const ModelWeights& w, KVCache& cache,
                                    const std::vector<TokenId>& prompt) {
    const int n = static_cast<int>(prompt.size());
    const int W = (n + 63) / 64;
    std::vector<uint64_t> masks((size_t)n * W, 0);
    std::vector<int32_t> pos(n);
    for (int i = 0; i < n; ++i) {
        pos[i] = i;
        for (int j = 0; j <= i; ++j) masks[(size_t)i * W + j / 64] |= 1ull << (j % 64);
    }
    auto am = detail::device_pass(w, cache, prompt, pos, 0, masks, W, nullptr);
    for (int i = 0; i < n; ++i) cache.record_token(i, prompt[i]);
    cache.set_occupancy(n);
    return am;
}

void finish(RunMetrics& m, Clock::time_point t0) {
    m.wall_ms = ms_since(t0);
    m.verified_per_step =
        m.llm_steps > 0 ? static_cast<double>(m.tokens_generated) / static_cast<double>(m.llm_steps)
                        : 0.0;
}

}  // namespace

void RunMetrics::accumulate(const RunMetrics& o) {
    llm_steps += o.llm_steps;
    ssm_runs += o.ssm_runs;
    tokens_generated += o.tokens_generated;
    wall_ms += o.wall_ms;
    verified_per_step =
        llm_steps > 0 ? static_cast<double>(tokens_generated) / static_cast<double>(llm_steps) : 0.0;
}

GenerationResult run_incremental(const ModelWeights& llm, const GenerationRequest& req) {
    check_request(llm, req);
    const auto t0 = Clock::now();
    std::lock_guard<std::recursive_mutex> lock(detail::compat_mutex());
    GenerationResult res;
    res.sequence = req.prompt;
    KVCache cache(llm.config);
    detail::set_device_authoritative(cache, true);
    TokenId next = prefill_device(llm, cache, req.prompt).back();
    const std::vector<uint64_t> self{1ull};
    for (int produced = 0; produced < req.max_new_tokens; ++produced) {
        res.sequence.push_back(next);
        res.metrics.llm_steps += 1;
        res.metrics.tokens_generated += 1;
        if (next == req.eos || produced + 1 == req.max_new_tokens) break;
        const int position = static_cast<int>(res.sequence.size()) - 1;
        next = detail::device_pass(llm, cache, {next}, {position}, position, self, 1, nullptr)[0];
        cache.record_token(position, res.sequence.back());
        cache.set_occupancy(position + 1);
    }
    finish(res.metrics, t0);
    return res;
}

GenerationResult run_speculative(const ModelWeights& llm,
                                 std::span<const std::shared_ptr<Ssm>> pool,
                                 ConfigSelector& selector, const GenerationRequest& req,
                                 const SpeculativeOptions& opts) {
    check_request(llm, req);
    if (pool.empty()) fail(Errc::empty_input, "run_speculative: empty pool");
    const auto t0 = Clock::now();
    GenerationResult res;
    res.sequence = req.prompt;
    auto& seq = res.sequence;
    auto& met = res.metrics;
    const ModelConfig& c = llm.config;

    KVCache cache(llm.config);
    {
        std::lock_guard<std::recursive_mutex> lock(detail::compat_mutex());
        // tree scratch rows past max_positions: node u of a tree lands at row P + u
        detail::set_device_authoritative(cache, true, std::max(opts.max_tree_nodes, 1));
        prefill_device(llm, cache, req.prompt);  // the first tree pass recomputes the root row
    }
    // device staging for the walk: tok | parent | n | budget, outputs: verified | ids | len
    const int cap = std::max(opts.max_tree_nodes, 1) + 1;
    int32_t* dbuf = nullptr;
    ck(cudaMalloc(&dbuf, sizeof(int32_t) * (size_t)(2 * cap + 2 + 2 * (cap + 1) + 1 + 2)),
       "cudaMalloc(engine)");
    int32_t *dtok = dbuf, *dpar = dbuf + cap, *dn = dpar + cap, *dbudget = dn + 1;
    int32_t *dver = dbudget + 1, *dids = dver + (cap + 1), *dlen = dids + (cap + 1),
            *dP = dlen + 1;

    const int budget = req.max_new_tokens;
    int produced = 0;
    try {
        while (produced < budget) {
            SpecConfig cfg;
            if (selector.wants_hidden()) {
                std::vector<double> hidden;
                {
                    std::lock_guard<std::recursive_mutex> lock(detail::compat_mutex());
                    hidden = final_hidden(llm, cache);
                }
                cfg = selector.choose(seq, hidden);
            } else {
                cfg = selector.choose(seq, {});
            }
            if (cfg.beam_width < 1 || cfg.beam_depth < 1)
                fail(Errc::invalid_argument, "run_speculative: selector returned invalid config");
            cfg.beam_depth = std::min(cfg.beam_depth, c.max_positions - static_cast<int>(seq.size()) - 1);
            met.ssm_runs += static_cast<std::int64_t>(pool.size()) * std::max(cfg.beam_depth, 0);
            TokenTree tree = cfg.beam_depth >= 1
                                 ? speculate_tree(pool, seq, cfg, opts.max_tree_nodes, req.eos)
                                 : TokenTree::merge_sequences({{seq.back()}}, opts.max_tree_nodes);

            std::lock_guard<std::recursive_mutex> lock(detail::compat_mutex());
            cudaStream_t s = detail::compat_stream();
            const int n = tree.size();
            const int P = static_cast<int>(seq.size()) - 1;
            if (cache.token_at(P) != tree.token(0))
                fail(Errc::root_mismatch, "run_speculative: tree root is not the last token");
            const int W = (n + 63) / 64;
            std::vector<uint64_t> masks((size_t)n * W, 0);
            std::vector<int32_t> pos(n), host_in(2 * cap + 3, 0);
            std::vector<TokenId> toks(n);
            for (int u = 0; u < n; ++u) {
                toks[u] = tree.token(u);
                pos[u] = P + tree.depth(u);
                if (u > 0) std::memcpy(&masks[(size_t)u * W], &masks[(size_t)tree.parent(u) * W], W * 8);
                masks[(size_t)u * W + u / 64] |= 1ull << (u % 64);
                host_in[u] = toks[u];
                host_in[cap + u] = tree.parent(u);
            }
            host_in[2 * cap] = n;
            host_in[2 * cap + 1] = budget - produced;
            int32_t* argmax_dev = nullptr;
            detail::device_pass(llm, cache, toks, pos, P, masks, W, &argmax_dev);
            met.llm_steps += 1;
            ck(cudaMemcpyAsync(dtok, host_in.data(), sizeof(int32_t) * (2 * cap + 2),
                               cudaMemcpyHostToDevice, s), "h2d tree");
            ck(cudaMemcpyAsync(dP, &P, sizeof(int32_t), cudaMemcpyHostToDevice, s), "h2d P");
            ck(st_verify_outputs(argmax_dev, 1, n, dtok, dpar, dn, dbudget, req.eos, dver, dids,
                                 dlen, s), "verify");
            const detail::DeviceKV& dk = cache.device();
            ck(st_kv_compact(ST_F64, 1, dk.H, dk.Dh, dk.Lmax, dk.layers, (int64_t)dk.layer_elems(),
                             dids, cap + 1, dlen, dP, nullptr, dk.k, dk.v, s), "compact");
            std::vector<int32_t> out(cap + 2);
            ck(cudaMemcpyAsync(out.data(), dver, sizeof(int32_t) * (cap + 1), cudaMemcpyDeviceToHost, s),
               "d2h verified");
            ck(cudaMemcpyAsync(out.data() + cap + 1, dlen, sizeof(int32_t), cudaMemcpyDeviceToHost, s),
               "d2h len");
            ck(cudaStreamSynchronize(s), "engine step");
            const int len = out[cap + 1];
            bool hit_eos = false;
            for (int k = 0; k < len; ++k) {
                seq.push_back(out[k]);
                cache.record_token(static_cast<int>(seq.size()) - 1, out[k]);
                if (req.eos != kNoEosToken && out[k] == req.eos) hit_eos = true;
            }
            cache.set_occupancy(static_cast<int>(seq.size()));
            produced += len;
            met.tokens_generated += len;
            if (hit_eos) break;
        }
    } catch (...) {
        cudaFree(dbuf);
        throw;
    }
    cudaFree(dbuf);
    finish(met, t0);
    return res;
}

ComparisonReport compare_equivalence(const ModelWeights& llm,
                                     std::span<const std::shared_ptr<Ssm>> pool,
                                     ConfigSelector& selector,
                                     std::span<const GenerationRequest> corpus,
                                     const SpeculativeOptions& opts, const CompareHooks* hooks) {
    ComparisonReport rep;
    for (const GenerationRequest& req : corpus) {
        GenerationResult inc = run_incremental(llm, req);
        GenerationResult spec = run_speculative(llm, pool, selector, req, opts);
        if (hooks && hooks->perturb_speculative) hooks->perturb_speculative(spec.sequence);
        ComparisonReport::PromptOutcome o;
        o.incremental = inc.metrics;
        o.speculative = spec.metrics;
        o.match = inc.sequence == spec.sequence;
        if (!o.match) {
            const size_t lim = std::min(inc.sequence.size(), spec.sequence.size());
            size_t i = 0;
            while (i < lim && inc.sequence[i] == spec.sequence[i]) ++i;
            o.first_mismatch = static_cast<int>(i);
            rep.mismatches += 1;
        }
        rep.incremental_total.accumulate(inc.metrics);
        rep.speculative_total.accumulate(spec.metrics);
        rep.prompts.push_back(std::move(o));
    }
    return rep;
}

}  // namespace spectree
