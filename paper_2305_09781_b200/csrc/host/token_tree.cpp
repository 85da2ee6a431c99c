// Host C++ token-tree library (drop-in for reference proj/src/token_tree.cpp's
// public surface; independent implementation).
//
// Construction by sorting instead of a trie: lexicographically sorted
// sequences enumerate the distinct prefixes in exactly the DFS preorder with
// ascending-token children that the reference's trie flatten produces
// (token_tree.cpp:77-100). Each sequence only adds the nodes past its longest
// common prefix with its sorted predecessor, so the whole merge is one sort
// plus one linear scan and allocation happens once.
//
// verify() is not computed here: it uploads the outputs and runs the K3 walk
// on the GPU (no CPU fallback, per the north star).
#include <algorithm>
#include <cstring>
#include <numeric>
#include <string>

#include <cuda_runtime.h>

#include "spectree/token_tree.hpp"
#include "spectree_capi.h"

namespace spectree {

const char* errc_name(Errc code) {
    static const char* const names[] = {
        "empty_input",   "root_mismatch",     "unknown_node",  "missing_output",
        "tree_too_large", "tree_too_deep",    "shape_mismatch", "prompt_too_long",
        "cache_gap",     "chain_not_linked",  "empty_context", "incomplete_profile",
        "bad_magic",     "crc_mismatch",      "io_error",      "invalid_argument"};
    const int i = static_cast<int>(code);
    return (i >= 0 && i < 16) ? names[i] : "unknown";
}

TokenTree TokenTree::merge_sequences(const std::vector<std::vector<TokenId>>& sequences,
                                     int max_nodes) {
    // validation order mirrors the reference: emptiness, then root agreement
    if (sequences.empty()) fail(Errc::empty_input, "merge_sequences: no sequences");
    for (const auto& s : sequences)
        if (s.empty()) fail(Errc::empty_input, "merge_sequences: empty sequence");
    const TokenId root = sequences.front().front();
    for (const auto& s : sequences)
        if (s.front() != root)
            fail(Errc::root_mismatch, "merge_sequences: first tokens differ (" +
                                          std::to_string(root) + " vs " +
                                          std::to_string(s.front()) + ")");

    std::vector<int> order(sequences.size());
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(), [&](int a, int b) {
        return std::lexicographical_compare(sequences[a].begin(), sequences[a].end(),
                                            sequences[b].begin(), sequences[b].end());
    });

    TokenTree tree;
    tree.nodes_.push_back({root, kRootParent, 0});
    std::vector<int> path{0};  // path[i] = node id of the length-(i+1) prefix of `prev`
    const std::vector<TokenId>* prev = &sequences[order[0]];
    const int cap = std::max(max_nodes, 1);
    for (size_t k = 0; k < order.size(); ++k) {
        const auto& s = sequences[order[k]];
        size_t lcp = 1;
        if (k > 0) {
            const size_t lim = std::min(prev->size(), s.size());
            while (lcp < lim && (*prev)[lcp] == s[lcp]) ++lcp;
        }
        path.resize(lcp);
        for (size_t i = lcp; i < s.size(); ++i) {
            if (static_cast<int>(tree.nodes_.size()) >= cap)
                fail(Errc::tree_too_large,
                     "merge_sequences: tree exceeds " + std::to_string(max_nodes) + " nodes");
            const int id = static_cast<int>(tree.nodes_.size());
            tree.nodes_.push_back({s[i], path.back(), static_cast<int>(i)});
            path.push_back(id);
            tree.max_depth_ = std::max(tree.max_depth_, static_cast<int>(i));
        }
        prev = &s;
    }
    tree.children_.assign(tree.nodes_.size(), {});
    for (int v = 1; v < tree.size(); ++v) tree.children_[tree.nodes_[v].parent].push_back(v);
    return tree;
}

void TokenTree::check_node(int node) const {
    if (node < 0 || node >= size())
        fail(Errc::unknown_node,
             "node " + std::to_string(node) + " not in tree of size " + std::to_string(size()));
}

TokenId TokenTree::token(int node) const { check_node(node); return nodes_[node].token; }
int TokenTree::parent(int node) const { check_node(node); return nodes_[node].parent; }
int TokenTree::depth(int node) const { check_node(node); return nodes_[node].depth; }

const std::vector<int>& TokenTree::children(int node) const {
    check_node(node);
    return children_[node];
}

std::vector<TokenId> TokenTree::ancestors(int node) const {
    check_node(node);
    std::vector<TokenId> path(nodes_[node].depth + 1);
    for (int at = node, i = nodes_[node].depth; at != kRootParent; at = nodes_[at].parent, --i)
        path[i] = nodes_[at].token;
    return path;
}

std::vector<std::vector<int>> TokenTree::dfs_chains() const {
    std::vector<std::vector<int>> chains;
    for (int v = 1; v < size(); ++v) {
        if (chains.empty() || nodes_[v].parent != v - 1) chains.emplace_back();
        chains.back().push_back(v);
    }
    return chains;
}

void TokenTree::ancestor_mask(int node, std::span<std::uint64_t> words) const {
    check_node(node);
    std::fill(words.begin(), words.end(), 0ull);
    for (int at = node; at != kRootParent; at = nodes_[at].parent) {
        if (static_cast<size_t>(at >> 6) >= words.size())
            fail(Errc::invalid_argument, "ancestor_mask: too few words");
        words[at >> 6] |= 1ull << (at & 63);
    }
}

TokenTreeBatch pack_trees(std::span<const TokenTree> trees, int T) {
    TokenTreeBatch b;
    b.B = static_cast<int>(trees.size());
    int tmax = 1;
    for (const auto& t : trees) tmax = std::max(tmax, t.size());
    if (T == 0) T = tmax;
    if (T < tmax) fail(Errc::tree_too_large, "pack_trees: tree larger than T");
    b.T = T;
    b.W = (T + 63) / 64;
    b.tokens.assign((size_t)b.B * T, 0);
    b.parent.assign((size_t)b.B * T, -1);
    b.depth.assign((size_t)b.B * T, 0);
    b.n_nodes.assign(b.B, 0);
    b.mask.assign((size_t)b.B * T * b.W, 0ull);
    for (int i = 0; i < b.B; ++i) {
        const TokenTree& t = trees[i];
        b.n_nodes[i] = t.size();
        for (int u = 0; u < t.size(); ++u) {
            const size_t at = (size_t)i * T + u;
            b.tokens[at] = t.token(u);
            b.parent[at] = t.parent(u);
            b.depth[at] = t.depth(u);
            std::uint64_t* m = &b.mask[at * b.W];
            if (u > 0) std::memcpy(m, &b.mask[((size_t)i * T + t.parent(u)) * b.W], 8 * b.W);
            m[u >> 6] |= 1ull << (u & 63);
        }
    }
    return b;
}

namespace {

[[noreturn]] void throw_status(st_status st, const char* what) {
    const int errc = st - 1;
    if (errc >= 0 && errc < 16)
        throw Error(static_cast<Errc>(errc), std::string(what) + ": " + st_last_error_message());
    throw std::runtime_error(std::string(what) + ": " + st_last_error_message());
}

}  // namespace

std::vector<TokenId> verify(const TokenTree& tree, std::span<const TokenId> llm_outputs) {
    if (static_cast<int>(llm_outputs.size()) != tree.size())
        fail(Errc::missing_output, "verify: got " + std::to_string(llm_outputs.size()) +
                                       " outputs for " + std::to_string(tree.size()) + " nodes");
    const int T = tree.size();
    std::vector<int32_t> host(4 * T + 1);
    for (int u = 0; u < T; ++u) {
        host[u] = llm_outputs[u];
        host[T + u] = tree.token(u);
        host[2 * T + u] = tree.parent(u);
    }
    host[4 * T] = T;
    // device staging: outputs | tokens | parent | (unused) | n ; results: verified | ids | len
    int32_t* d = nullptr;
    const size_t in_bytes = host.size() * sizeof(int32_t);
    const size_t out_elems = 2 * (size_t)(T + 1) + 1;
    cudaStream_t s = nullptr;
    if (cudaMallocAsync(reinterpret_cast<void**>(&d), in_bytes + out_elems * sizeof(int32_t), s) !=
        cudaSuccess) {
        cudaGetLastError();
        throw_status(st_device_count() == 0 ? ST_ERR_NO_DEVICE : ST_ERR_CUDA, "verify");
    }
    std::vector<int32_t> out(out_elems);
    st_status st = ST_OK;
    if (cudaMemcpyAsync(d, host.data(), in_bytes, cudaMemcpyHostToDevice, s) != cudaSuccess)
        st = ST_ERR_CUDA;
    int32_t* res = d + host.size();
    if (st == ST_OK)
        st = st_verify_outputs(d, 1, T, d + T, d + 2 * T, d + 4 * T, nullptr, -1, res,
                               res + (T + 1), res + 2 * (T + 1), s);
    if (st == ST_OK &&
        cudaMemcpyAsync(out.data(), res, out_elems * sizeof(int32_t), cudaMemcpyDeviceToHost, s) !=
            cudaSuccess)
        st = ST_ERR_CUDA;
    cudaFreeAsync(d, s);
    if (cudaStreamSynchronize(s) != cudaSuccess && st == ST_OK) st = ST_ERR_CUDA;
    if (st != ST_OK) throw_status(st, "verify");
    const int len = out[2 * (T + 1)];
    return std::vector<TokenId>(out.begin(), out.begin() + len);
}

}  // namespace spectree

// ----------------------------------------------------------- C-ABI (host) --
extern "C" st_status st_tree_merge(const int32_t* flat, const int32_t* lens, int nseq,
                                   int max_nodes, int32_t* tok, int32_t* parent, int32_t* depth,
                                   int cap, int* n_out) {
    try {
        std::vector<std::vector<spectree::TokenId>> seqs(nseq > 0 ? nseq : 0);
        size_t at = 0;
        for (int i = 0; i < nseq; ++i) {
            if (lens[i] < 0) return ST_ERR_INVALID_ARGUMENT;
            seqs[i].assign(flat + at, flat + at + lens[i]);
            at += lens[i];
        }
        const auto t = spectree::TokenTree::merge_sequences(seqs, max_nodes);
        if (n_out) *n_out = t.size();
        if (t.size() > cap) return ST_ERR_INVALID_ARGUMENT;
        for (int u = 0; u < t.size(); ++u) {
            tok[u] = t.token(u);
            parent[u] = t.parent(u);
            if (depth) depth[u] = t.depth(u);
        }
        return ST_OK;
    } catch (const spectree::Error& e) {
        return 1 + static_cast<int>(e.code());
    } catch (...) {
        return ST_ERR_INVALID_ARGUMENT;
    }
}
