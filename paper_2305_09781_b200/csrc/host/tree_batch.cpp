// Host tree pipeline: TokenTree::merge_sequences for
// every request of a batch on a persistent host thread pool, packed straight
// into the padded [B][T] arrays the device kernels consume (ideally pinned
// host memory, so one H2D copy follows). The reference merges one tree per
// engine step on the calling thread (speculator.cpp:204 -> token_tree.cpp:
// 42-102, ~6.7 us for a 61-node tree); at B requests per step this is the
// host work that has to overlap the GPU.
//
// The pool is created on first use and lives for the process: N-1 workers
// plus the calling thread pull request indices from an atomic counter, so a
// call costs one wake-up, not thread creation.
#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cstdint>
#include <functional>
#include <mutex>
#include <thread>
#include <vector>

#include "spectree/token_tree.hpp"
#include "spectree_capi.h"

namespace {

class MergePool {
  public:
    static MergePool& get() {
        static MergePool pool;
        return pool;
    }

    // Runs fn(i) for i in [0, n) on up to `threads` threads (caller included).
    void parallel_for(int n, int threads, const std::function<void(int)>& fn) {
        std::lock_guard<std::mutex> call(call_mu_);  // one batch at a time
        const int helpers = std::max(0, std::min({threads, n, (int)workers_.size() + 1}) - 1);
        {
            std::lock_guard<std::mutex> lk(mu_);
            fn_ = &fn;
            n_ = n;
            next_.store(0);
            participants_ = helpers;
            remaining_ = helpers;
            ++generation_;
        }
        cv_.notify_all();
        run();
        std::unique_lock<std::mutex> lk(mu_);
        done_cv_.wait(lk, [&] { return remaining_ == 0; });
        fn_ = nullptr;
    }

  private:
    MergePool() {
        const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
        const unsigned n = std::min(hw, 32u) - 1;
        for (unsigned i = 0; i < n; ++i) workers_.emplace_back([this, i] { loop(i); });
    }
    ~MergePool() {
        {
            std::lock_guard<std::mutex> lk(mu_);
            stop_ = true;
        }
        cv_.notify_all();
        for (auto& t : workers_) t.join();
    }

    void run() {
        for (int i = next_.fetch_add(1); i < n_; i = next_.fetch_add(1)) (*fn_)(i);
    }

    void loop(unsigned id) {
        uint64_t seen = 0;
        for (;;) {
            {
                std::unique_lock<std::mutex> lk(mu_);
                // only the first `participants_` workers of a generation take part
                cv_.wait(lk, [&] {
                    return stop_ || (generation_ != seen && id < (unsigned)participants_);
                });
                if (stop_) return;
                seen = generation_;
            }
            run();
            {
                std::lock_guard<std::mutex> lk(mu_);
                --remaining_;
            }
            done_cv_.notify_one();
        }
    }

    std::vector<std::thread> workers_;
    std::mutex call_mu_, mu_;
    std::condition_variable cv_, done_cv_;
    const std::function<void(int)>* fn_ = nullptr;
    std::atomic<int> next_{0};
    int n_ = 0, participants_ = 0, remaining_ = 0;
    uint64_t generation_ = 0;
    bool stop_ = false;
};

}  // namespace

extern "C" st_status st_tree_merge_batch(int B, const int32_t* flat, const int32_t* lens,
                                         const int32_t* nseq, int max_nodes, int T, int32_t* tok,
                                         int32_t* parent, int32_t* depth, int32_t* n_nodes,
                                         int32_t* status, int n_threads) {
    if (B < 0 || T < 1 || !nseq || !tok || !parent || !n_nodes) return ST_ERR_INVALID_ARGUMENT;
    if (B == 0) return ST_OK;
    // per-request offsets into lens (sequences) and flat (tokens)
    std::vector<int64_t> seq0(B + 1, 0), tok0(B + 1, 0);
    for (int b = 0; b < B; ++b) {
        if (nseq[b] < 0) return ST_ERR_INVALID_ARGUMENT;
        seq0[b + 1] = seq0[b] + nseq[b];
    }
    for (int b = 0; b < B; ++b) {
        int64_t n = 0;
        for (int64_t i = seq0[b]; i < seq0[b + 1]; ++i) {
            if (lens[i] < 0) return ST_ERR_INVALID_ARGUMENT;
            n += lens[i];
        }
        tok0[b + 1] = tok0[b] + n;
    }
    std::vector<st_status> st(B, ST_OK);
    auto merge_one = [&](int b) {
        int32_t* tk = tok + (int64_t)b * T;
        int32_t* pr = parent + (int64_t)b * T;
        int32_t* dp = depth ? depth + (int64_t)b * T : nullptr;
        int n = 0;
        try {
            std::vector<std::vector<spectree::TokenId>> seqs(nseq[b]);
            const int32_t* f = flat + tok0[b];
            for (int i = 0; i < nseq[b]; ++i) {
                const int len = lens[seq0[b] + i];
                seqs[i].assign(f, f + len);
                f += len;
            }
            const auto t = spectree::TokenTree::merge_sequences(seqs, max_nodes);
            if (t.size() > T) {
                st[b] = ST_ERR_INVALID_ARGUMENT;  // batch row too short for this tree
            } else {
                n = t.size();
                for (int u = 0; u < n; ++u) {
                    tk[u] = t.token(u);
                    pr[u] = t.parent(u);
                    if (dp) dp[u] = t.depth(u);
                }
            }
        } catch (const spectree::Error& e) {
            st[b] = 1 + static_cast<int>(e.code());
        } catch (...) {
            st[b] = ST_ERR_INVALID_ARGUMENT;
        }
        for (int u = n; u < T; ++u) {  // padding: rows the kernels never read
            tk[u] = 0;
            pr[u] = spectree::kRootParent;
            if (dp) dp[u] = 0;
        }
        n_nodes[b] = n;
    };
    const int threads = n_threads > 0 ? n_threads : (int)std::thread::hardware_concurrency();
    if (threads <= 1 || B == 1)
        for (int b = 0; b < B; ++b) merge_one(b);
    else
        MergePool::get().parallel_for(B, threads, merge_one);
    st_status first = ST_OK;
    for (int b = 0; b < B; ++b) {
        if (status) status[b] = st[b];
        if (first == ST_OK) first = st[b];
    }
    return first;
}
