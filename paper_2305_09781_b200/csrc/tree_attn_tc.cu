// K1, tcgen05 instantiation: masked one-pass tree attention on the sm_100a
// 5th-gen tensor cores (f16 / bf16 in, fp32 accumulate), head dim 128.
//
// What it computes is exactly K1 of the C-ABI (include/spectree_capi.h): for
// every (request b, head h, tree node u) a softmax over the committed KV rows
// [0, P[b]) plus the tree rows P[b]+v whose bit v is set in mask[b][u] — the
// reference's per-chain loop (proj/src/transformer.cpp:394-446 over the
// attention core :270-299) collapsed into one masked pass.
//
// Design:
//   * Persistent, one CTA per SM, over the pair-major sequence of every
//     (b, KV head) pair's 128-row KV tiles. Ranges are whole pairs, equal
//     single-segment pieces of every pair (small uniform batches), or
//     stream-K (equal tile counts per CTA). A pair cut by range boundaries
//     leaves pieces (O, m, l) that the pair's head owner merges in-kernel, in
//     CTA order (deterministic, no atomics in any reduction), after staging
//     them into its drained K ring with TMA. On 2-CTA clusters a pair of two
//     pieces (the split schedule) merges over DSMEM instead: the piece
//     bulk-copies its (O, m, l) into the head's first freed K stage while the
//     head runs its last tile (M=128: the two CTAs exchange d halves).
//   * GQA: the G query heads of a KV head share one M-row Q tile (row r =
//     node r/G of head r%G). k_tree mode: the tree rows come from their own
//     [B][T][Hkv][D] tensors as one extra tile after the prefix tiles.
//   * Warp roles: SW softmax/epilogue warps (4 for M=64, 8 for M=128), then a
//     TMA producer for Q and K, a TMA producer for V and the MMA issuer (the
//     whole warp runs its loop; one elected lane issues inside the asm).
//   * TMA (SWIZZLE_128B) streams K and V tiles [128 rows x 128 d] through
//     3-stage rings, one box per tile (the maps view d as (64, half)); Q
//     (rows >= T zero-filled by TMA) double-buffered for M=64 so the next
//     pair's Q is in smem before its first S.
//   * S = Q K^T (SS MMA) and O += P V (TS MMA: P read from TMEM) on tcgen05
//     (kind::f16, fp32 accumulate). M=64 (T <= 64): every product is split into
//     two N=64 MMAs whose accumulators land in TMEM lanes 0-15 and 16-31 of
//     each subpartition, so all 32 lanes of a softmax warp hold data (half a
//     row each); the two halves share (m, l) and O. M=128 (T <= 128, "DUAL"):
//     warps w and w+4 read the same TMEM lanes and own one column half each,
//     with their own running (m, l) and their own O accumulator (O_a += P_a
//     V[0:64], O_b += P_b V[64:128]) — no cross-warp traffic per tile; the
//     halves merge once per segment in the epilogue.
//   * Softmax: tcgen05.ld of S (double-buffered in TMEM), the tree mask applied
//     only on tiles that reach the tree rows (one 32-bit visibility word per 32
//     columns), ex2 with lazy rescaling (the running max moves only when it
//     grows by > 2^8; O is then rescaled in TMEM), P written (f16/bf16) back
//     into TMEM over the tile's own S columns; V read MN-major by the P.V MMA.
//   * Masked rows are exact zeros in P, so they contribute +0 (reference
//     transformer.hpp:13-16) and outputs do not depend on non-ancestor rows.
#include <cuda.h>
#include <cudaTypedefs.h>

#include <cfloat>
#include <cstdio>
#include <cstdlib>
#include <mutex>
#include <type_traits>
#include <unordered_map>

#include "common.cuh"
#include "sm100.cuh"
#include "tree_attn.h"

namespace st {
namespace {

using namespace sm100;

constexpr int BN = 128;            // KV rows per tile
constexpr int HD = 128;            // head dim
constexpr uint32_t KV_ATOM = 128 * 128;             // 128 rows x 64 elems x 2 B
constexpr uint32_t TILE_BYTES = 2 * KV_ATOM;        // 32 KB K or V tile
constexpr int SLOT_FLOATS = 128 * HD + 2 * 128;      // partial O rows + m + l
constexpr float kLazyThreshLog2 = 8.0f;
// Batches of up to kTabB requests get their cumulative tile counts staged in
// shared memory once per CTA (one parallel round of global loads); larger
// batches walk the lengths in global memory.
constexpr int kTabB = 128;
// Pieces a split pair may leave beyond its head: at most gridDim.x - 1 (the
// host launches at most kMaxPieces + 1 CTAs).
constexpr int kMaxPieces = 255;

// Per-M configuration: M = 64 query rows (T <= 64) or 128 (T <= 128).
template <int M> struct Cfg {
    // M=64: 4 softmax warps, the two column halves of a row in lanes l / l+16
    // sharing one (m, l, O). M=128 ("DUAL"): 8 softmax warps, warps w and w+4
    // read the same TMEM lanes and take one column half each, with their own
    // running (m, l) and their own O accumulator, merged once per segment.
    static constexpr bool DUAL = M == 128;
    static constexpr int SW = M == 64 ? 4 : 8;              // softmax warps
    // + K-TMA, V-TMA, MMA warps; M=128: + one idle warp, so the three form a
    // whole warpgroup that hands registers to the two softmax warpgroups
    // (setmaxnreg: 168 at launch -> 56 / 224; at 168 the M=128 softmax spilled)
    static constexpr int THREADS = (SW + (M == 128 ? 4 : 3)) * 32;
    static constexpr uint32_t REG_LOW = 56, REG_HIGH = 224;
    static constexpr int SPLIT = M == 64 ? 2 : 1;           // threads per query row in a warp
    static constexpr uint32_t A_ATOM = M * 128;             // M rows x 64 elems x 2 B
    static constexpr uint32_t A_BYTES = 2 * A_ATOM;         // Q or one P buffer
    static constexpr int QSTAGES = M == 64 ? 2 : 1;          // next pair's Q prefetched
    static constexpr int KSTAGES = 3;
    static constexpr int VSTAGES = 3;
    static constexpr uint32_t S_COLS = BN / SPLIT;          // TMEM columns per S buffer
    static constexpr uint32_t O_COL = 2 * S_COLS;           // O accumulator column (DUAL: O_a)
    static constexpr uint32_t OB_COL = O_COL + HD;          // DUAL: O_b
    static constexpr uint32_t TMEM_COLS = M == 64 ? 256 : 512;
    static constexpr uint32_t OFF_Q = 0;
    static constexpr uint32_t OFF_K = OFF_Q + QSTAGES * A_BYTES;
    static constexpr uint32_t OFF_V = OFF_K + KSTAGES * TILE_BYTES;
    static constexpr uint32_t OFF_BAR = OFF_V + VSTAGES * TILE_BYTES;
    // A split pair's head owner stages the pair's other pieces into the drained
    // K ring: the (m, l) block (1 KB), then the piece's O, stored column-block
    // major — float4 (r, 4j..4j+3) at j*M + r — so the publishing warps' stores
    // coalesce (a warp writes 512 contiguous bytes per instruction), one bulk
    // copy stages it, and the row-per-thread reads are bank-conflict-free.
    static constexpr uint32_t PIECE_BOX = M * 128;
    static constexpr uint32_t PIECE_SMEM = 1024 + 4 * PIECE_BOX;
    static constexpr int STAGED_PIECES = (KSTAGES * TILE_BYTES) / PIECE_SMEM;
    static constexpr uint32_t OFF_TAB = OFF_BAR + 256;     // per-request tile table
    // DUAL: (m, l) of both column halves of every row, exchanged per segment
    static constexpr uint32_t OFF_XCHG = OFF_TAB + (kTabB + 4) * 4;
    static constexpr uint32_t SMEM_BYTES = OFF_XCHG + (DUAL ? 2 * 128 * 2 * 4 : 0);
    // the head owner's piece list sits at the end of the drained K ring
    static constexpr uint32_t OFF_PIECES = OFF_K + KSTAGES * TILE_BYTES - (kMaxPieces + 1) * 4;
    static_assert(STAGED_PIECES * PIECE_SMEM <= KSTAGES * TILE_BYTES - (kMaxPieces + 1) * 4,
                  "piece list overlaps the staged pieces");
    static_assert(SMEM_BYTES <= 232448, "shared memory budget");
};

// TcParams: tree_attn.h

constexpr int kTraceCta = 12;   // per-CTA globaltimer/clock slots of the ST_K1_TRACE dump
constexpr int kTraceRows = 16;  // per-tile (rows 0-11) and per-segment (12-15) clock rows

#define K1_GT(k)                                                                  \
    do {                                                                          \
        if (p.trace) {                                                            \
            unsigned long long gt_;                                               \
            asm volatile("mov.u64 %0, %globaltimer;" : "=l"(gt_));               \
            p.trace[kTraceRows * 64 + kTraceCta * blockIdx.x + (k)] = gt_;                        \
        }                                                                         \
    } while (0)

#define K1_TRACE(slot, idx)                                                       \
    do {                                                                          \
        if (p.trace && blockIdx.x == p.trace_cta && (idx) < 64)                   \
            p.trace[(slot) * 64 + (idx)] = clock64();                             \
    } while (0)

// Tile indices over the pair-major sequence are 32-bit (the host rejects
// launches with 2^31 or more tiles): 64-bit integer division is a ~70
// instruction subroutine, and the schedule arithmetic sits on every CTA's
// path to its first load.
struct Seg {
    int b, h, lo, hi, ntiles;
    uint32_t pair_start;
};

__device__ __forceinline__ int ntiles_of(const TcParams& p, int b) {
    // both loads issued together (one round trip on the startup path)
    const int n = __ldg(p.n_nodes + b);
    const int P = __ldg(p.prefix_len + b);
    if (n <= 0) return 0;
    // k_tree mode: the prefix tiles, then ceil(n/BN) tiles of the tree rows
    return p.tree_src ? (P + BN - 1) / BN + (n + BN - 1) / BN : (P + n + BN - 1) / BN;
}

// k_tree mode: the segment's last tree_tiles tiles are the tree's own rows
__device__ __forceinline__ int tree_tiles(const TcParams& p, const Seg& s) {
    return s.ntiles - (__ldg(p.prefix_len + s.b) + BN - 1) / BN;
}

// Segment starting at global tile t (t < t_end) of this CTA's range. `cum`
// (shared memory, or null): cum[b] = tiles of requests < b, cum[kTabB+1..3] =
// requests with tiles, min and max tiles per request.
__device__ Seg find_seg(const TcParams& p, const int* cum, uint32_t t, uint32_t t_end) {
    Seg s{};
    const uint32_t H = (uint32_t)p.H;
    if (cum) {
        int lo = 0, hi = p.B;  // largest b with H*cum[b] <= t (skips empty requests)
        while (hi - lo > 1) {
            const int mid = (lo + hi) >> 1;
            if (H * (uint32_t)cum[mid] <= t) lo = mid; else hi = mid;
        }
        const uint32_t nt = (uint32_t)(cum[lo + 1] - cum[lo]);
        const uint32_t base = H * (uint32_t)cum[lo];
        const uint32_t off = t - base;
        const uint32_t hh = off / nt;
        s.b = lo;
        s.h = (int)hh;
        s.lo = (int)(off - hh * nt);
        s.ntiles = (int)nt;
        s.pair_start = base + hh * nt;
        const uint32_t h2 = (uint32_t)s.lo + (t_end - t);
        s.hi = (int)(h2 < nt ? h2 : nt);
        return s;
    }
    uint32_t base = 0;
    for (int b = 0; b < p.B; ++b) {
        const uint32_t nt = (uint32_t)ntiles_of(p, b);
        const uint32_t span = H * nt;
        if (t < base + span) {
            const uint32_t off = t - base;
            const uint32_t hh = off / nt;
            s.b = b;
            s.h = (int)hh;
            s.lo = (int)(off - hh * nt);
            s.ntiles = (int)nt;
            s.pair_start = base + hh * nt;
            const uint32_t h2 = (uint32_t)s.lo + (t_end - t);
            s.hi = (int)(h2 < nt ? h2 : nt);
            return s;
        }
        base += span;
    }
    s.b = -1;
    return s;
}

// CTA work ranges over the pair-major tile sequence. Stream-K (equal tile
// counts; pairs may be split, leaving pieces that the pair's head owner merges
// in-kernel) unless every pair has the same tile count and a static shape is
// within aligned_slack tiles of perfect balance (or 4G/5 <= Np <= G):
//   * aligned: CTA c takes pairs [c*Np/G, (c+1)*Np/G), no pair is split;
//   * split (Np <= G/2): every pair is cut into S = G/Np equal pieces, one
//     per CTA (CTAs past Np*S idle) — each CTA has a single segment, so no
//     CTA pays a second epilogue or a piece publish between two segments,
//     which is what small batches (C4's 64 pairs x 17 tiles) lose to.
constexpr int kAlignedSlack = 3;
// Split schedule: extra tiles given to each pair's head piece (ST_K1_HEADX overrides)
constexpr int kHeadExtra = 1;

enum : int { kStreamK = 0, kAligned = 1, kSplit = 2 };

struct Sched {
    uint32_t total;
    uint32_t np;    // pairs with tiles
    int nt;         // tiles per pair when uniform
    int mode;       // kStreamK / kAligned / kSplit
    uint32_t S;     // kSplit: pieces per pair
    uint64_t magic; // TcParams::g_magic
    uint32_t hx;    // kSplit: extra tiles of a pair's head piece
};

// floor(x / G) for x < 2^40, G <= 256, m = floor(2^64 / G) + 1 (host): x*m/2^64
// exceeds x/G by less than x/2^64 < 2^-24 < 1/G, which cannot carry the
// quotient past the next integer. One IMAD.WIDE chain — the schedule sits on
// every CTA's path to its first load (the double-precision form it replaces
// cost ~1.5k cycles there with its reciprocal subroutine).
__device__ __forceinline__ uint32_t div_g(uint64_t x, uint64_t m) {
    return (uint32_t)__umul64hi(x, m);
}

__device__ __forceinline__ void sched_finish(const TcParams& p, Sched& s, int lo, int hi, uint32_t G);

__device__ Sched make_sched(const TcParams& p, const int* cum, uint32_t G) {
    Sched s{0, 0, 0, kStreamK, 1, p.g_magic, 0};
    int lo = 1 << 30, hi = 0;
    if (cum) {
        s.total = (uint32_t)p.H * (uint32_t)cum[p.B];
        s.np = (uint32_t)p.H * (uint32_t)cum[kTabB + 1];
        lo = cum[kTabB + 2];
        hi = cum[kTabB + 3];
    }
    for (int b = 0; b < (cum ? 0 : p.B); ++b) {
        const int nt = ntiles_of(p, b);
        if (nt > 0) {
            lo = min(lo, nt);
            hi = max(hi, nt);
            s.np += p.H;
        }
        s.total += (uint32_t)p.H * (uint32_t)nt;
    }
    sched_finish(p, s, lo, hi, G);
    return s;
}

// Mode choice once the totals are known (every path into make_sched*).
__device__ __forceinline__ void sched_finish(const TcParams& p, Sched& s, int lo, int hi, uint32_t G) {
    if (s.np > 0 && lo == hi) {
        s.nt = lo;
        const long long aligned_span = (long long)div_g(s.np + G - 1, s.magic) * (uint32_t)s.nt;
        const long long streamk_span = div_g((uint64_t)s.total + G - 1, s.magic);
        const uint32_t S = s.np <= G ? min(G / s.np, (uint32_t)s.nt) : 0;
        const long long split_span = S >= 2 ? (s.nt + S - 1) / S : 1ll << 40;
        // whole pairs also when there are no more pairs than CTAs but at least
        // 4/5 as many: the ~15% of SMs left idle are not needed to saturate HBM
        // (the busy ones get their bandwidth share), and no CTA pays a piece
        // publish or a merge (GQA 128 pairs x 33 tiles: 54.6 -> 52.9 us,
        // tools/k1_sched_ab.py)
        const bool most = p.most_aligned && s.np <= G && 5 * s.np >= 4 * G && p.aligned_slack >= 0;
        if (aligned_span <= streamk_span + p.aligned_slack || most) {
            s.mode = kAligned;
        } else if (split_span <= streamk_span + p.aligned_slack) {
            s.mode = kSplit;
            s.S = S;
            // the symmetric DSMEM exchange (M=128 pairs of two pieces on
            // 2-CTA clusters) wants equal halves; otherwise the head piece
            // takes extra tiles, so the other pieces are in by its last P.V
            const bool sym = p.cluster2 && S == 2 && p.R == 1 && p.G * p.Tq > 64;
            s.hx = sym ? 0u : min((uint32_t)p.head_extra, (uint32_t)s.nt - S);
        }
    }
}

__device__ __forceinline__ uint32_t range_start(uint32_t c, const Sched& s, uint32_t G) {
    if (s.mode == kAligned) return div_g((uint64_t)c * s.np, s.magic) * (uint32_t)s.nt;
    if (s.mode == kSplit) {
        if (c >= s.np * s.S) return s.total;
        const uint32_t pr = c / s.S, k = c - pr * s.S;
        // the head piece gets hx extra tiles: the later pieces (all running
        // beside it) are published by the time it reaches its merge
        return pr * (uint32_t)s.nt + (k == 0 ? 0u : s.hx + (k * ((uint32_t)s.nt - s.hx)) / s.S);
    }
    return div_g((uint64_t)c * s.total, s.magic);
}

// Register-only schedule of this CTA's first segment, computed by a whole warp
// when B <= 32 (lane b holds request b): the two TMA producer warps run it
// right after the barrier setup, so their first loads go out without waiting
// for warp 0's shared-memory table, the CTA barrier after it and the binary
// search of find_seg — a dependent chain of ~3k cycles on the path to the
// first tile (tools/k1_trace.py). Same inputs and arithmetic as make_sched /
// range_start / find_seg, so the ranges agree with what the other warps
// compute from the table.
struct First {
    uint32_t t_begin, t_end;
    Seg s;
    int P;  // prefix_len of s.b
};

__device__ __forceinline__ First warp_first_seg(const TcParams& p, uint32_t G, uint32_t slot, int lane) {
    int x = 0, Pl = 0;
    if (lane < p.B) {
        x = ntiles_of(p, lane);
        Pl = __ldg(p.prefix_len + lane);
    }
    if (p.trace) {  // (stamp once every lane's loads have landed)
        const bool all = __all_sync(0xffffffffu, x >= 0 && Pl >= 0);
        if (lane == 0 && all) K1_TRACE(13, 56);
    }
    int inc = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
        const int y = __shfl_up_sync(0xffffffffu, inc, o);
        if (lane >= o) inc += y;
    }
    const int excl = inc - x;
    const uint32_t H = (uint32_t)p.H;
    Sched sc{0, 0, 0, kStreamK, 1, p.g_magic, 0};
    sc.total = H * (uint32_t)__shfl_sync(0xffffffffu, inc, 31);
    sc.np = H * (uint32_t)__popc(__ballot_sync(0xffffffffu, x > 0));
    const int lo = __reduce_min_sync(0xffffffffu, x > 0 ? x : 1 << 30);
    const int hi = __reduce_max_sync(0xffffffffu, x);
    if (lane == 0) K1_TRACE(13, 57);
    sched_finish(p, sc, lo, hi, G);
    if (lane == 0) K1_TRACE(13, 58);
    First f{};
    f.t_begin = range_start(slot, sc, G);
    f.t_end = range_start(slot + 1, sc, G);
    if (lane == 0) K1_TRACE(13, 59);
    if (f.t_begin < f.t_end) {
        // largest b with H * cum[b] <= t (skips empty requests), as find_seg
        const uint32_t bal = __ballot_sync(0xffffffffu, lane < p.B && H * (uint32_t)excl <= f.t_begin);
        const int b = 31 - __clz(bal);
        const uint32_t nt = (uint32_t)__shfl_sync(0xffffffffu, x, b);
        const uint32_t base = H * (uint32_t)__shfl_sync(0xffffffffu, excl, b);
        const uint32_t off = f.t_begin - base;
        const uint32_t hh = off / nt;
        f.s.b = b;
        f.s.h = (int)hh;
        f.s.lo = (int)(off - hh * nt);
        f.s.ntiles = (int)nt;
        f.s.pair_start = base + hh * nt;
        const uint32_t h2 = (uint32_t)f.s.lo + (f.t_end - f.t_begin);
        f.s.hi = (int)(h2 < nt ? h2 : nt);
        f.P = __shfl_sync(0xffffffffu, Pl, b);
    }
    return f;
}

template <class T> struct pk2;
template <> struct pk2<__half> {
    static __device__ __forceinline__ uint32_t pack(float a, float b) {
        __half2 h = __floats2half2_rn(a, b);
        return *reinterpret_cast<uint32_t*>(&h);
    }
};
template <> struct pk2<__nv_bfloat16> {
    static __device__ __forceinline__ uint32_t pack(float a, float b) {
        __nv_bfloat162 h = __floats2bfloat162_rn(a, b);
        return *reinterpret_cast<uint32_t*>(&h);
    }
};

// A thread's NCOL output values of one row (scaled, rounded to T). Rows of a
// warp are a head's stride apart, so every store is its own request: 32-byte
// (sector) stores halve the request count when the row is 32-byte aligned.
template <class T, int NCOL>
__device__ __forceinline__ void store_row(T* dst_row, const float* v, float scale) {
    if ((reinterpret_cast<uintptr_t>(dst_row) & 31) == 0) {
#pragma unroll
        for (int ch = 0; ch < NCOL / 16; ++ch) {
            uint32_t w8[8];
#pragma unroll
            for (int k = 0; k < 8; ++k)
                w8[k] = pk2<T>::pack(v[ch * 16 + 2 * k] * scale, v[ch * 16 + 2 * k + 1] * scale);
            asm volatile("st.global.v8.b32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};" ::"l"(dst_row + ch * 16),
                         "r"(w8[0]), "r"(w8[1]), "r"(w8[2]), "r"(w8[3]), "r"(w8[4]), "r"(w8[5]), "r"(w8[6]),
                         "r"(w8[7])
                         : "memory");
        }
        return;
    }
    uint4* dst = reinterpret_cast<uint4*>(dst_row);
#pragma unroll
    for (int ch = 0; ch < NCOL / 8; ++ch) {
        uint32_t w4[4];
#pragma unroll
        for (int k = 0; k < 4; ++k)
            w4[k] = pk2<T>::pack(v[ch * 8 + 2 * k] * scale, v[ch * 8 + 2 * k + 1] * scale);
        dst[ch] = make_uint4(w4[0], w4[1], w4[2], w4[3]);
    }
}

// One 128-row K or V tile into `dst` as two 64-column SWIZZLE_128B atoms
// [d half][128 rows][64] — ONE TMA: the maps view D = 128 as (64, half) with
// the half dimension (stride 128 B) outside the rows — from the cache
// ([B*Hkv][Lmax][D], rows from `row`; map dims (64, Lmax, 2, B*Hkv)) or,
// `tree`, from the tree's own rows ([B][T][Hkv][D]; (64, Hkv, T, 2, B)).
// mc (two row blocks per pair on a 2-CTA cluster; maps with a one-half box):
// this CTA loads only d half `rank` and multicasts it into both CTAs' rings,
// so each tile is read from L2 once and every ring still gets the whole tile
// (each CTA's barrier expects the full tile bytes).
__device__ __forceinline__ void load_kv_tile(uint8_t* dst, uint64_t* bar, const CUtensorMap* cache_map,
                                             const CUtensorMap* tree_map, bool tree, int row, int h, int b,
                                             int bh, uint64_t pol, bool mc, int rank) {
    if (mc) {
        uint8_t* d = dst + rank * KV_ATOM;
        if (tree) tma_load_5d_mc(d, tree_map, bar, 0, h, row, rank, b, 0x3);
        else tma_load_4d_mc_hint(d, cache_map, bar, 0, row, rank, bh, 0x3, pol);
    } else if (tree) {
        tma_load_5d(dst, tree_map, bar, 0, h, row, 0, b);
    } else {
        tma_load_4d_hint(dst, cache_map, bar, 0, row, 0, bh, pol);
    }
}

// MW: ancestor-mask words held per row (2: T <= 128; 4: T <= 256, the
// two-row-block instantiation — kept separate so the common case keeps its
// registers).
template <class T, int M, int MW>
__global__ void __launch_bounds__(Cfg<M>::THREADS, 1)
tree_attn_tc_kernel(const __grid_constant__ CUtensorMap tm_q, const __grid_constant__ CUtensorMap tm_k,
                    const __grid_constant__ CUtensorMap tm_v,
                    const __grid_constant__ CUtensorMap tm_kt, const __grid_constant__ CUtensorMap tm_vt,
                    const __grid_constant__ CUtensorMap tm_o, const __grid_constant__ TcParams p) {
    using C = Cfg<M>;
    constexpr int KS = C::KSTAGES, VS = C::VSTAGES, QS = C::QSTAGES;
    constexpr int SPLIT = C::SPLIT;          // threads per query row in a warp (2 for M=64)
    constexpr bool DUAL = C::DUAL;
    constexpr int SW = C::SW;                // softmax warps; then K-TMA, V-TMA, MMA
    constexpr int COLS = BN / 2;             // S columns per thread per tile (one half)
    constexpr int DCOLS = HD / 2;            // output d columns per thread
    // SWIZZLE_128B tiles need 1024-byte alignment: the dynamic window starts
    // after the 1 KB the hardware reserves per CTA (checked below)
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t* smem = smem_raw;
    uint8_t* sm_q = smem + C::OFF_Q;
    uint8_t* sm_k = smem + C::OFF_K;
    uint8_t* sm_v = smem + C::OFF_V;
    uint64_t* bars = reinterpret_cast<uint64_t*>(smem + C::OFF_BAR);
    uint64_t* q_full = bars;             // [QS]
    uint64_t* q_empty = q_full + QS;     // [QS]
    uint64_t* k_full = q_empty + QS;     // [KS]
    uint64_t* k_empty = k_full + KS;     // [KS]
    uint64_t* v_full = k_empty + KS;     // [VS]
    uint64_t* v_empty = v_full + VS;     // [VS]
    uint64_t* s_full = v_empty + VS;     // [2]
    uint64_t* p_full = s_full + 2;       // [2]
    uint64_t* pv_done = p_full + 2;      // [2]
    uint64_t* o_empty = pv_done + 2;
    uint64_t* merge_full = o_empty + 1;  // staged pieces landed (head owner only)
    uint64_t* peer_ready = merge_full + 1;  // DSMEM exchange: the peer's K ring is drained
    uint64_t* xchg_full = peer_ready + 1;   // DSMEM exchange: the peer's (m, l) + O half landed
    uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(xchg_full + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) K1_GT(8);
    // startup stamps of the traced CTA (clock64): row 15, columns 56-63
    if (threadIdx.x == 0) K1_TRACE(15, 56);

    if (threadIdx.x == 0) {
        if (smem_u32(smem) & 1023u) __trap();  // misaligned dynamic shared memory
        for (int i = 0; i < QS; ++i) { mbar_init(q_full + i, 1); mbar_init(q_empty + i, 1); }
        // mc: a stage is free once BOTH CTAs' MMAs have read it (the MMA
        // warps commit to the empty barriers of the whole cluster)
        const uint32_t ne = M == 128 && p.R == 2 && p.cluster2 ? 2u : 1u;
        for (int i = 0; i < KS; ++i) { mbar_init(k_full + i, 1); mbar_init(k_empty + i, ne); }
        for (int i = 0; i < VS; ++i) { mbar_init(v_full + i, 1); mbar_init(v_empty + i, ne); }
        for (int i = 0; i < 2; ++i) {
            mbar_init(s_full + i, 1);
            mbar_init(p_full + i, SW * 32);
            mbar_init(pv_done + i, 1);
        }
        mbar_init(o_empty, SW * 32);
        mbar_init(merge_full, 1);
        mbar_init(peer_ready, 1);
        mbar_init(xchg_full, DUAL ? 128 : 1);  // DUAL: one sending thread per row in the peer
        fence_barrier_init();
    }
    if (warp == SW && lane == 0) {
        prefetch_tmap(&tm_q);
        prefetch_tmap(&tm_k);
        if (p.tree_src) prefetch_tmap(&tm_kt);
    }
    if (warp == SW + 1 && lane == 0) {
        prefetch_tmap(&tm_v);
        if (p.tree_src) prefetch_tmap(&tm_vt);
    }
    if (warp == SW + 2) tmem_alloc<C::TMEM_COLS>(tmem_slot);
    // two row blocks per pair on a 2-CTA cluster: the slot's CTAs multicast
    // K/V tiles into each other's rings, so both must have initialised their
    // barriers before either issues a load
    const bool mc = M == 128 && p.R == 2 && p.cluster2;  // (M=64 pairs never take two row blocks)
    tc_fence_before();
    if (mc) cluster_sync();
    else __syncthreads();
    tc_fence_after();
    const uint32_t tmem = *tmem_slot;
    if (threadIdx.x == 0) K1_TRACE(15, 57);
    // Everything above touches no other kernel's output; from here on the
    // lengths, masks, Q and the KV cache are read. early_kv: the caller
    // guarantees the previous kernel writes neither the lengths nor the
    // committed KV rows [0, P), so the schedule and the first prefix tiles of
    // each ring go ahead of griddepcontrol.wait; every warp that reads Q, the
    // masks, tree rows or another CTA's output waits first.
    if (!p.early_kv) pdl_wait();

    // Schedule slots: with R = 2 row blocks per pair, CTAs 2s and 2s+1 take
    // slot s's tile range for Q rows [0, 128) and [128, 256) of each pair, so
    // both stream the same KV tiles at the same time (the second read is an L2
    // hit) and each runs the M=128 pipeline unchanged.
    const uint32_t G = gridDim.x / (uint32_t)p.R;
    const uint32_t slot = blockIdx.x / (uint32_t)p.R;
    const int rblk = (int)(blockIdx.x - slot * (uint32_t)p.R);

    // Producer fast start (B <= 32): each TMA producer warp schedules its
    // first segment in registers (warp_first_seg) and its lane 0 issues the
    // segment's first ring-full of tiles (and, unless early_kv, its Q) before
    // the lengths table below exists; the loops further down resume after the
    // pre-issued tiles. early_kv: only committed-prefix tiles, as in the loops.
    // (Scheduling before the CTA barrier, overlapping the TMEM allocation,
    // measured no earlier first load and a slower C2 K1.)
    const bool fast = p.B <= 32;
    First f0{};
    uint32_t pre_n = 0;   // first-segment tiles this producer already issued
    bool pre_q = false;   // K producer: the first segment's Q already issued
    if (fast && (warp == SW || warp == SW + 1)) {
        if (lane == 0) K1_TRACE(15, 60);
        f0 = warp_first_seg(p, G, slot, lane);
        if (lane == 0) K1_TRACE(15, 61);
        if (lane == 0 && f0.t_begin < f0.t_end) {
            const Seg& s0 = f0.s;
            const bool kside = warp == SW;
            const uint64_t pol = p.R == 1 || mc ? l2_policy_evict_first() : l2_policy_evict_normal();
            const int jt0 = p.tree_src ? (f0.P + BN - 1) / BN : 1 << 30;  // first tree tile
            const int bh0 = s0.b * p.H + s0.h;
            if (kside) K1_TRACE(13, 48);
            if (kside && !p.early_kv) {
                mbar_arrive_expect_tx(q_full, C::A_BYTES);
                const int node0 = rblk * (M / p.G);
                tma_load_5d(sm_q, &tm_q, q_full, 0, s0.h * p.G, node0, 0, s0.b);  // both d halves
                pre_q = true;
                K1_TRACE(13, 49);
            }
            uint64_t* full = kside ? k_full : v_full;
            uint8_t* ring = kside ? sm_k : sm_v;
            const CUtensorMap* mcache = kside ? &tm_k : &tm_v;
            const CUtensorMap* mt = kside ? &tm_kt : &tm_vt;
            const uint32_t stages = kside ? (uint32_t)KS : (uint32_t)VS;
            const uint32_t cap = p.pre_cap > 0 && (uint32_t)p.pre_cap < stages ? (uint32_t)p.pre_cap : stages;
            for (int j = s0.lo; j < s0.hi && pre_n < cap &&
                                (!p.early_kv || (p.tree_src ? j < jt0 : j * BN + BN <= f0.P));
                 ++j, ++pre_n) {
                // first use of each stage: nothing to wait for
                mbar_arrive_expect_tx(full + pre_n, TILE_BYTES);
                const bool tr = j >= jt0;
                load_kv_tile(ring + pre_n * TILE_BYTES, full + pre_n, mcache, mt, tr, (tr ? j - jt0 : j) * BN,
                             s0.h, s0.b, bh0, pol, mc, rblk);
                if (kside) K1_TRACE(13, 50 + pre_n);
            }
            if (kside) K1_TRACE(15, 62);
            if (kside && pre_n > 0) K1_GT(5);
        }
    }

    int* cum = p.B <= kTabB ? reinterpret_cast<int*>(smem + C::OFF_TAB) : nullptr;
    if (cum && warp == 0) {
        int v[kTabB / 32];
#pragma unroll
        for (int c = 0; c < kTabB / 32; ++c) {  // all loads in flight together
            const int b = c * 32 + lane;
            v[c] = b < p.B ? ntiles_of(p, b) : 0;
        }
        int carry = 0, cnt = 0, mn = 1 << 30, mx = 0;
#pragma unroll
        for (int c = 0; c < kTabB / 32; ++c) {
            int x = v[c];
            cnt += __popc(__ballot_sync(0xffffffffu, x > 0));
            mn = min(mn, x > 0 ? x : 1 << 30);
            mx = max(mx, x);
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int y = __shfl_up_sync(0xffffffffu, x, o);
                if (lane >= o) x += y;
            }
            cum[c * 32 + lane + 1] = carry + x;
            carry += __shfl_sync(0xffffffffu, x, 31);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) {
            mn = min(mn, __shfl_xor_sync(0xffffffffu, mn, o));
            mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
        }
        if (lane == 0) {
            cum[0] = 0;
            cum[kTabB + 1] = cnt;
            cum[kTabB + 2] = mn;
            cum[kTabB + 3] = mx;
        }
    }
    __syncthreads();
    if (threadIdx.x == 0) K1_GT(9);
    if (threadIdx.x == 0) K1_TRACE(15, 58);

    const Sched sched = make_sched(p, cum, G);
    const uint32_t t_begin = range_start(slot, sched, G);
    const uint32_t t_end = range_start(slot + 1, sched, G);
    // DSMEM merge (uniform over the grid): 2-CTA clusters and a split schedule
    // of two pieces per pair — pair k's head is CTA 2k (cluster rank 0), its
    // piece CTA 2k+1 (rank 1), so the piece's (O, m, l) goes straight into the
    // head's drained K ring with one shared::cluster bulk copy completing on
    // the head's merge_full barrier: no global publish, no gpu-scope release,
    // no flag polling, no staging copy back out of L2.
    const bool dsm = p.cluster2 && sched.mode == kSplit && sched.S == 2 && p.R == 1;
    if (p.trace && threadIdx.x == 0) {
        unsigned long long gt;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(gt));
        p.trace[kTraceRows * 64 + kTraceCta * blockIdx.x] = gt;
        p.trace[kTraceRows * 64 + kTraceCta * blockIdx.x + 2] = (unsigned long long)(t_end - t_begin);
        p.trace[kTraceRows * 64 + kTraceCta * blockIdx.x + 6] = clock64();
    }
    if (threadIdx.x == 0) K1_TRACE(15, 59);

    if (warp >= SW) {
        // producer / MMA warpgroup (M=128: with the idle warp): registers handed
        // to the softmax warpgroups, each role's code allocated under its limit
        if constexpr (DUAL) reg_dealloc<C::REG_LOW>();
        if (warp == SW) {
            // ======================= TMA producer: Q and K =========================
            if (lane == 0) {
                // the KV stream is read once (R = 1): evict_first keeps Q, masks and
                // pieces in L2. With two row blocks (R = 2) both CTAs of a slot read
                // every tile: normal priority, so the second read finds it in L2.
                const uint64_t pol = p.R == 1 || mc ? l2_policy_evict_first() : l2_policy_evict_normal();
                uint32_t qc = 0, kc = 0;
                bool waited = !p.early_kv;
                for (uint32_t t = t_begin; t < t_end;) {
                    const bool first = t == t_begin;
                    const Seg s = fast && first ? f0.s : find_seg(p, cum, t, t_end);
                    int j = s.lo;
                    const int jt0 = p.tree_src ? s.ntiles - tree_tiles(p, s) : 1 << 30;  // first tree tile
                    if (first) {  // resume after the fast start's tiles
                        j += (int)pre_n;
                        kc = pre_n;
                    }
                    if (!waited) {  // early_kv: up to KS committed-prefix K tiles before the wait
                        const int P0 = __ldg(p.prefix_len + s.b);
                        const int bh0 = s.b * p.H + s.h;
                        for (; j < s.hi && kc < (uint32_t)KS &&
                               (p.tree_src ? j < jt0 : j * BN + BN <= P0);
                             ++j, ++kc) {
                            const uint32_t st = kc;  // first use of each stage: nothing to wait for
                            mbar_arrive_expect_tx(k_full + st, TILE_BYTES);
                            load_kv_tile(sm_k + st * TILE_BYTES, k_full + st, &tm_k, &tm_kt, false, j * BN, s.h,
                                         s.b, bh0, pol, mc, rblk);
                        }
                        pdl_wait();
                        waited = true;
                    }
                    if (!(first && pre_q)) {
                        const uint32_t qb = qc % QS;
                        mbar_wait(q_empty + qb, ((qc / QS) & 1) ^ 1);
                        mbar_arrive_expect_tx(q_full + qb, C::A_BYTES);
                        // box {64 d, G heads, M/G nodes}: smem row = node * G + head;
                        // row block rblk starts at node rblk * M / G
                        const int node0 = rblk * (M / p.G);
                        tma_load_5d(sm_q + qb * C::A_BYTES, &tm_q, q_full + qb, 0, s.h * p.G, node0, 0, s.b);
                    }
                    ++qc;
                    const int bh = s.b * p.H + s.h;
                    for (; j < s.hi; ++j, ++kc) {
                        const uint32_t st = kc % KS, ph = (kc / KS) & 1;
                        mbar_wait(k_empty + st, ph ^ 1);
                        K1_TRACE(0, kc);
                        if (kc == 0) K1_GT(5);
                        mbar_arrive_expect_tx(k_full + st, TILE_BYTES);
                        // (tree tiles: the tree's own rows [B][T][Hkv][D], 128 nodes per tile)
                        const bool tr = j >= jt0;
                        load_kv_tile(sm_k + st * TILE_BYTES, k_full + st, &tm_k, &tm_kt, tr, (tr ? j - jt0 : j) * BN,
                                     s.h, s.b, bh, pol, mc, rblk);
                    }
                    t += s.hi - s.lo;
                }
            }
            // If this range ends with a pair's head, stage the pair's other pieces
            // (published by the following CTAs early in their ranges) into the K
            // ring as soon as the last S MMA has drained it, so the softmax warps'
            // merge reads shared memory instead of making L2 round trips.
            if (t_end > t_begin && dsm) {
                // DSMEM merge of a pair's two pieces on one 2-CTA cluster.
                //   M=64: the head (rank 0, one tile more) receives the piece's O
                //   in the first K stage its last tiles free — stage kc % KS once
                //   S of tile kc - KS is done (or the never-used stage kc) — so the
                //   piece pushes it while the head still runs its last tile.
                //   DUAL: both CTAs receive the other's half once the whole ring
                //   has drained (symmetric exchange).
                if (lane == 0) {
                    const uint32_t kc = (uint32_t)(t_end - t_begin);
                    if constexpr (!DUAL) {
                        if ((blockIdx.x & 1u) == 0) {
                            if (kc >= (uint32_t)KS) mbar_wait(k_empty + kc % KS, ((kc - KS) / KS) & 1);
                            mbar_arrive_expect_tx(xchg_full, 4u * C::PIECE_BOX + 8u * M);
                            K1_GT(11);
                            mbar_arrive_cluster(mapa_rank(peer_ready, 1));
                        }
                    } else {
                        for (uint32_t st = 0; st < (uint32_t)KS && st < kc; ++st) {
                            const uint32_t k = kc - 1 - ((kc - 1 - st) % KS);  // last use of stage st
                            mbar_wait(k_empty + st, (k / KS) & 1);
                        }
                        K1_GT(11);
                        mbar_arrive_cluster(mapa_rank(peer_ready, (blockIdx.x & 1u) ^ 1u));
                    }
                }
            } else if (t_end > t_begin) {
                const Seg ls = find_seg(p, cum, t_end - 1, t_end);
                const uint32_t pend = ls.pair_start + (uint32_t)ls.ntiles;
                if (ls.pair_start >= t_begin && pend > t_end) {
                    const uint32_t kc = (uint32_t)(t_end - t_begin);  // K tiles this CTA loaded
                    if (lane == 0) {
                        // piece list for the softmax warps; every piece's flag is
                        // awaited (and re-armed for the next launch) before its
                        // copy is issued into the drained K ring (the first
                        // STAGED_PIECES pieces) or, beyond those, before the final
                        // arrival that releases the softmax warps to read it from L2
                        // the list and the staged pieces live in the K ring: drain it
                        for (uint32_t st = 0; st < (uint32_t)KS && st < kc; ++st) {
                            const uint32_t k = kc - 1 - ((kc - 1 - st) % KS);  // last use of stage st
                            mbar_wait(k_empty + st, (k / KS) & 1);
                        }
                        int* pieces = reinterpret_cast<int*>(smem + C::OFF_PIECES);
                        int np = 0;
                        for (uint32_t c2 = slot + 1; c2 < G && np < kMaxPieces; ++c2) {
                            const uint32_t rs = range_start(c2, sched, G);
                            if (rs >= pend) break;
                            if (range_start(c2 + 1, sched, G) == rs) continue;  // empty range
                            pieces[1 + np++] = (int)(c2 * (uint32_t)p.R) + rblk;  // same row block
                        }
                        pieces[0] = np;
                        const int ns = np < C::STAGED_PIECES ? np : C::STAGED_PIECES;
                        mbar_expect_tx(merge_full, (uint32_t)ns * (1024u + 4u * C::PIECE_BOX));
                        K1_GT(11);
                        for (int i = 0; i < np; ++i) {
                            const int c2 = pieces[1 + i];
                            wait_flag_gpu(p.flags + c2);
                            p.flags[c2] = 0u;
                            if (i < ns) {
                                fence_proxy_async_global();
                                uint8_t* dst = sm_k + i * C::PIECE_SMEM;
                                bulk_load(dst, p.partial + (long long)c2 * SLOT_FLOATS + 128 * HD, 1024, merge_full);
                                bulk_load(dst + 1024, p.partial + (long long)c2 * SLOT_FLOATS, 4 * C::PIECE_BOX, merge_full);
                            }
                        }
                        mbar_arrive(merge_full);
                    }
                }
            }
        } else if (warp == SW + 1) {
            // =========================== TMA producer: V ============================
            if (lane == 0) {
                const uint64_t pol = p.R == 1 || mc ? l2_policy_evict_first() : l2_policy_evict_normal();
                uint32_t vc = 0;
                bool waited = !p.early_kv;
                for (uint32_t t = t_begin; t < t_end;) {
                    const bool first = t == t_begin;
                    const Seg s = fast && first ? f0.s : find_seg(p, cum, t, t_end);
                    const int bh = s.b * p.H + s.h;
                    int j = s.lo;
                    const int jt0 = p.tree_src ? s.ntiles - tree_tiles(p, s) : 1 << 30;  // first tree tile
                    if (first) {  // resume after the fast start's tiles
                        j += (int)pre_n;
                        vc = pre_n;
                    }
                    if (!waited) {  // early_kv: up to VS committed-prefix V tiles before the wait
                        const int P0 = __ldg(p.prefix_len + s.b);
                        for (; j < s.hi && vc < (uint32_t)VS &&
                               (p.tree_src ? j < jt0 : j * BN + BN <= P0);
                             ++j, ++vc) {
                            const uint32_t st = vc;
                            mbar_arrive_expect_tx(v_full + st, TILE_BYTES);
                            load_kv_tile(sm_v + st * TILE_BYTES, v_full + st, &tm_v, &tm_vt, false, j * BN, s.h,
                                         s.b, bh, pol, mc, rblk);
                        }
                        pdl_wait();
                        waited = true;
                    }
                    for (; j < s.hi; ++j, ++vc) {
                        const uint32_t st = vc % VS, ph = (vc / VS) & 1;
                        mbar_wait(v_empty + st, ph ^ 1);
                        K1_TRACE(1, vc);
                        mbar_arrive_expect_tx(v_full + st, TILE_BYTES);
                        const bool tr = j >= jt0;
                        load_kv_tile(sm_v + st * TILE_BYTES, v_full + st, &tm_v, &tm_vt, tr, (tr ? j - jt0 : j) * BN,
                                     s.h, s.b, bh, pol, mc, rblk);
                    }
                    t += s.hi - s.lo;
                }
            }
        } else if (warp == SW + 2) {
            // ============================ MMA issuer ==============================
            // M=128: S = Q K^T (N=128); O_a += P[:, 0:64] V[0:64] and
            //        O_b += P[:, 64:128] V[64:128] (N=128, K=64 each), one
            //        accumulator per column half of the softmax.
            // M=64 : every product is split into two N=64 MMAs whose accumulators
            //        land in TMEM lanes 0-15 and 16-31 of each subpartition (the
            //        interleaved M=64 layout), so all 32 softmax lanes hold data:
            //        S kv-rows 0-63 | 64-127 and O d 0-63 | 64-127.
            // The whole warp runs this loop (uniform control flow); MMAs and
            // commits are issued by one elected lane inside the asm.
            constexpr uint32_t fmt = std::is_same<T, __half>::value ? 0u : 1u;
            constexpr uint32_t NS = BN / SPLIT, NO = HD / SPLIT;
            constexpr uint32_t idS = idesc_f16(fmt, M, NS, 0, 0);   // Q K^T: both K-major
            constexpr uint32_t idPV = idesc_f16(fmt, M, NO, 0, 1);  // P V: V is MN-major
            constexpr uint32_t HI_LANES = 16u << 16;                // lane offset of the 2nd half
            const uint32_t q_base0 = smem_u32(sm_q), k_base = smem_u32(sm_k);
            const uint32_t v_base = smem_u32(sm_v);
            uint32_t qc = 0, kc = 0, vc = 0, sc = 0, pc = 0, segc = 0;
            auto issue_pv = [&](int i_local) {
                const uint32_t pb = pc & 1;
                mbar_wait(p_full + pb, (pc >> 1) & 1);
                const uint32_t st = vc % VS;
                mbar_wait(v_full + st, (vc / VS) & 1);
                K1_TRACE(7, vc);
                if (i_local == 0) mbar_wait(o_empty, (segc & 1) ^ 1);
                tc_fence_after();
                const uint32_t vb = v_base + st * TILE_BYTES;
                const uint64_t vd = smem_desc(vb, KV_ATOM, 1024);
                // P of this tile sits in TMEM over its S buffer (K-major, 2 elements
                // per column: K=16 per MMA = 8 columns). For M=64 each half-lane
                // group holds the full P rows, matching its O accumulator's lanes.
                const uint32_t pt = tmem + pb * C::S_COLS;
    #pragma unroll
                for (int kk = 0; kk < BN / 16; ++kk) {
                    const uint32_t acc = (i_local > 0 || (kk & 3) > 0) ? 1u : 0u;
                    if constexpr (DUAL) {  // half h's P sits at S columns [64h, 64h+32)
                        const uint32_t h = kk >> 2;
                        umma_f16_ts_warp(tmem + (h ? C::OB_COL : C::O_COL), pt + h * 64 + (kk & 3) * 8,
                                         vd + ((kk * 2048) >> 4), idPV, acc);
                    } else {
                        const uint32_t acc = (i_local > 0 || kk > 0) ? 1u : 0u;
                        umma_f16_ts_warp(tmem + C::O_COL, pt + kk * 8, vd + ((kk * 2048) >> 4), idPV, acc);
                        umma_f16_ts_warp(tmem + HI_LANES + C::O_COL, pt + HI_LANES + kk * 8,
                                         vd + ((KV_ATOM + kk * 2048) >> 4), idPV, acc);
                    }
                }
                K1_TRACE(3, pc);
                umma_commit_warp(pv_done + pb);
                if (mc) umma_commit_warp_mc(v_empty + st, 0x3);
                else umma_commit_warp(v_empty + st);
                ++vc;
                ++pc;
            };
            for (uint32_t t = t_begin; t < t_end;) {
                const Seg s = find_seg(p, cum, t, t_end);
                const int ntl = s.hi - s.lo;
                const uint32_t qb = qc % QS;
                mbar_wait(q_full + qb, (qc / QS) & 1);
                ++qc;
                const uint32_t q_base = q_base0 + qb * C::A_BYTES;
                for (int i = 0; i < ntl; ++i) {
                    const uint32_t st = kc % KS;
                    mbar_wait(k_full + st, (kc / KS) & 1);
                    K1_TRACE(6, kc);
                    // S buffer sb last held P of tile sc-2, read by the P.V MMA
                    // issued before this one: tcgen05 MMAs of one thread execute in
                    // issue order, so no barrier is needed before overwriting it.
                    const uint32_t sb = sc & 1;
                    tc_fence_after();
                    const uint32_t kb = k_base + st * TILE_BYTES;
                    const uint32_t scol = sb * C::S_COLS;
                    const uint64_t qd = smem_desc(q_base, 16, 1024), kd = smem_desc(kb, 16, 1024);
    #pragma unroll
                    for (int kk = 0; kk < HD / 16; ++kk) {
                        const uint32_t off = (kk >> 2) * C::A_ATOM + (kk & 3) * 32;
                        const uint32_t koff = (kk >> 2) * KV_ATOM + (kk & 3) * 32;
                        const uint64_t a = qd + (off >> 4);
                        const uint32_t acc = kk > 0 ? 1u : 0u;
                        if constexpr (SPLIT == 1) {
                            umma_f16_ss_warp(tmem + scol, a, kd + (koff >> 4), idS, acc);
                        } else {  // kv rows 0-63 -> lanes 0-15, kv rows 64-127 -> lanes 16-31
                            umma_f16_ss_warp(tmem + scol, a, kd + (koff >> 4), idS, acc);
                            umma_f16_ss_warp(tmem + HI_LANES + scol, a,
                                             kd + ((koff + 64 * 128) >> 4), idS, acc);
                        }
                    }
                    K1_TRACE(2, sc);
                    umma_commit_warp(s_full + sb);
                    if (mc) umma_commit_warp_mc(k_empty + st, 0x3);
                    else umma_commit_warp(k_empty + st);
                    if (i == ntl - 1) umma_commit_warp(q_empty + qb);
                    ++kc;
                    ++sc;
                    if (i > 0) issue_pv(i - 1);
                }
                issue_pv(ntl - 1);
                ++segc;
                t += ntl;
            }
        }  // (warp SW + 3, M=128: idle — it completes the producers' warpgroup)
    } else {
        if constexpr (DUAL) reg_alloc<C::REG_HIGH>();
        // ===================== softmax + epilogue (warps 0..SW-1) ==================
        // Thread (warp w, lane t) reads TMEM lane 32(w%4)+t and owns column half
        // `half` of its row's kv tile (S) and of d (output). M=64: row
        // 16w+(t&15), half t>>4; the two halves of a row exchange max / sum with
        // one shuffle and share O. M=128 (DUAL): row 32(w%4)+t, half w/4; each
        // half keeps its own (m, l) and O accumulator, merged in the epilogue.
        const int half = DUAL ? (warp >> 2) : (lane >> 4);
        const int r = DUAL ? (warp & 3) * 32 + lane : warp * 16 + (lane & 15);
        // Q/S/O row r holds tree node u_r of query head g_r of the pair's
        // KV-head group (the Q box lays rows out node-major, head-minor)
        const int rr = rblk * M + r;  // row within the pair's G*T rows
        // Q row qr of request b is tree node u_r (q_rows / q_node0: a slice)
        const int qr = rr / p.G, g_r = rr - qr * p.G;
        const int u_r = p.u0 + qr;
        const uint32_t lane_addr = tmem + ((uint32_t)((warp & 3) * 32) << 16);
        const uint32_t s_half = DUAL ? half * COLS : 0;          // this half's S columns
        const uint32_t o_own = DUAL ? (half ? C::OB_COL : C::O_COL) : C::O_COL;
        constexpr int OWN_COLS = DUAL ? HD : DCOLS;              // O columns this thread rescales
        const float c = p.c_log2;
        const float thresh_raw = kLazyThreshLog2 / c;
        uint32_t sc = 0, pc = 0;
        // A segment's metadata (node count, prefix length, this row's mask
        // words) is loaded by the previous segment's epilogue — all four loads
        // independent, in flight while that epilogue runs — so a segment
        // transition costs no global round trip on the softmax path.
        struct Meta {
            int n, P;
            uint64_t mw[MW];   // this row's ancestor words
        };
        auto load_meta = [&](const Seg& sg) {
            Meta mt;
            mt.n = __ldg(p.n_nodes + sg.b);
            mt.P = __ldg(p.prefix_len + sg.b);
#pragma unroll
            for (int w = 0; w < MW; ++w) mt.mw[w] = 0;
            if (qr < p.Tq && u_r < p.T) {
                const uint64_t* mr = p.mask + ((long long)sg.b * p.T + u_r) * p.W;
#pragma unroll
                for (int w = 0; w < MW; ++w)
                    if (w < p.W) mt.mw[w] = __ldg(mr + w);
            }
            return mt;
        };
        Seg s_next{};
        Meta m_next{};
        if (p.early_kv) pdl_wait();  // masks and lengths below; outputs written later
        // past this CTA's own wait (either branch above): the next kernel may be
        // scheduled — it waits for this grid before reading anything K1 writes
        // (the step plan's argmax streams its logits on the SMs K1's tail frees)
        pdl_trigger();
        if (t_begin < t_end) {
            s_next = find_seg(p, cum, t_begin, t_end);
            m_next = load_meta(s_next);
        }
        uint32_t segn = 0;  // segments done (trace index)
        for (uint32_t t = t_begin; t < t_end;) {
            const Seg s = s_next;
            const int ntl = s.hi - s.lo;
            const int n = m_next.n;
            const int P = m_next.P;
            // first kv row index of the tree rows: P, or (k_tree mode) the
            // start of the extra tree tile after the ceil(P/BN) prefix tiles
            const int Pt = p.tree_src ? (s.ntiles - (n + BN - 1) / BN) * BN : P;
            const bool valid = qr < p.Tq && u_r < n;
            const bool warp_live = __any_sync(0xffffffffu, valid);
            uint64_t mw[MW];
#pragma unroll
            for (int w = 0; w < MW; ++w) mw[w] = valid ? m_next.mw[w] : 0;
            float m = -INFINITY, l = 0.f;   // l: this thread's share of the row sum
            for (int i = 0; i < ntl; ++i) {
                const int j = s.lo + i;
                const uint32_t sb = sc & 1;
                const uint32_t pb = pc & 1;
                mbar_wait(s_full + sb, (sc >> 1) & 1);
                if (warp_live) {
                    float sv[COLS];
                    tc_fence_after();
                    if (threadIdx.x == 0) K1_TRACE(4, sc);
#pragma unroll
                    for (int ch = 0; ch < COLS / 32; ++ch) {
                        uint32_t raw[32];
                        tmem_ld_32x32b_x32(lane_addr + sb * C::S_COLS + s_half + ch * 32, raw);
                        tmem_ld_wait();
#pragma unroll
                        for (int k = 0; k < 32; ++k) sv[ch * 32 + k] = __uint_as_float(raw[k]);
                    }
                    if (threadIdx.x == 0) K1_TRACE(8, sc);
                    // ---- tree mask: one visibility word per 32 columns ----
                    if (j * BN + BN > P) {
#pragma unroll
                        for (int wd = 0; wd < COLS / 32; ++wd) {
                            const int a = j * BN + half * COLS + wd * 32;  // first kv row of the word
                            const int pre = P - a;
                            uint32_t vis = pre >= 32 ? 0xffffffffu : (pre <= 0 ? 0u : ((1u << pre) - 1u));
                            const int o = a - Pt;                         // tree index of bit 0
                            if (o > -32 && o < n) {
                                // bits [o, o + 32) of the row's 256-bit ancestor mask
                                uint32_t win;
                                if (o < 0) {
                                    win = (uint32_t)(mw[0] << (-o));
                                } else {
                                    const int wd0 = o >> 6, sh = o & 63;
                                    uint64_t lo = 0, hi = 0;
#pragma unroll
                                    for (int w = 0; w < MW; ++w) {
                                        if (w == wd0) lo = mw[w];
                                        if (w == wd0 + 1) hi = mw[w];
                                    }
                                    win = (uint32_t)(sh ? (lo >> sh) | (hi << (64 - sh)) : lo);
                                }
                                vis |= win;
                            }
#pragma unroll
                            for (int k = 0; k < 32; ++k)
                                if (!((vis >> k) & 1u)) sv[wd * 32 + k] = -INFINITY;
                        }
                    }
                    // row max: two chains of three-input maxes (FMNMX3)
                    float mq0 = -INFINITY, mq1 = -INFINITY;
#pragma unroll
                    for (int k = 0; k < COLS; k += 4) {
                        mq0 = fmax3(mq0, sv[k], sv[k + 1]);
                        mq1 = fmax3(mq1, sv[k + 2], sv[k + 3]);
                    }
                    float mx = fmaxf(mq0, mq1);
                    if constexpr (!DUAL) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, 16));
                    const float m_new = fmaxf(m, mx);
                    if (threadIdx.x == 0) K1_TRACE(9, sc);

                    float alpha = 1.f;
                    bool rescale = false;
                    if (m == -INFINITY) {
                        m = m_new;  // nothing with nonzero weight accumulated yet
                    } else if (m_new - m > thresh_raw) {
                        alpha = ex2((m - m_new) * c);
                        l *= alpha;
                        m = m_new;
                        rescale = true;
                    }
                    if (__any_sync(0xffffffffu, rescale && valid)) {
                        // O must be stable: wait for P.V number pc-1 (this segment, i > 0)
                        const uint32_t q1 = pc - 1;
                        mbar_wait(pv_done + (q1 & 1), (q1 >> 1) & 1);
                        tc_fence_after();
#pragma unroll
                        for (int ch = 0; ch < OWN_COLS / 32; ++ch) {
                            uint32_t raw[32];
                            tmem_ld_32x32b_x32(lane_addr + o_own + ch * 32, raw);
                            tmem_ld_wait();
#pragma unroll
                            for (int k = 0; k < 32; ++k)
                                raw[k] = __float_as_uint(__uint_as_float(raw[k]) * alpha);
                            tmem_st_32x32b_x32(lane_addr + o_own + ch * 32, raw);
                        }
                        tmem_st_wait();
                    }
                    if (threadIdx.x == 0) K1_TRACE(11, sc);
                    const float base = (m == -INFINITY) ? 0.f : m * c;
                    // exponentials two columns per issue slot: s*c - base as
                    // one FFMA2, the running sums as FADD2 (four partial sums)
                    float ls[4] = {0.f, 0.f, 0.f, 0.f};
                    uint32_t pk[COLS / 2];
#pragma unroll
                    for (int k = 0; k < COLS / 2; ++k) {
                        float x0, x1;
                        ffma2_bcast(sv[2 * k], sv[2 * k + 1], c, -base, x0, x1);
                        const float p0 = ex2(x0);
                        const float p1 = ex2(x1);
                        fadd2_acc(ls[2 * (k & 1)], ls[2 * (k & 1) + 1], p0, p1);
                        pk[k] = pk2<T>::pack(p0, p1);
                    }
                    // P (f16/bf16, 2 per column) into TMEM over this tile's S
                    // columns. M=64: the two lanes of a row swap halves so both
                    // hold the full row (64 columns; the P.V MMA of each half-lane
                    // group reads A from its own lanes). DUAL: each half writes its
                    // 32 columns at the start of its own S columns.
                    const uint32_t pt = lane_addr + sb * C::S_COLS + s_half;
                    if constexpr (DUAL) {
                        tmem_st_32x32b_x32(pt, pk);
                    } else {
                        uint32_t lo[32], hi[32];
#pragma unroll
                        for (int k = 0; k < 32; ++k) {
                            const uint32_t o = __shfl_xor_sync(0xffffffffu, pk[k], 16);
                            lo[k] = half ? o : pk[k];
                            hi[k] = half ? pk[k] : o;
                        }
                        tmem_st_32x32b_x32(pt, lo);
                        tmem_st_32x32b_x32(pt + 32, hi);
                    }
                    tmem_st_wait();
                    if (threadIdx.x == 0) K1_TRACE(10, sc);
                    l += (ls[0] + ls[1]) + (ls[2] + ls[3]);
                    tc_fence_before();
                }
                // (rows all padding: no TMEM traffic or math, only the arrival)
                ++sc;
                if (threadIdx.x == 0) K1_TRACE(5, pc);
                mbar_arrive(p_full + pb);
                ++pc;
            }

            // ---- segment epilogue: this thread's O columns from TMEM ----
            // A segment is a whole pair (written out), a pair's head (lo == 0,
            // the last segment of this range: this CTA merges the pair's other
            // pieces into it and writes it out) or a later piece (lo > 0, the
            // first segment of this range: published as (O, m, l) for the
            // pair's head owner). The pieces were computed at the START of the
            // following CTAs' ranges, so the head owner — at the END of its
            // range — normally finds them ready.
            if (t + ntl < t_end) {
                s_next = find_seg(p, cum, t + ntl, t_end);
                m_next = load_meta(s_next);
            }
            const bool full = (s.lo == 0 && s.hi == s.ntiles);
            const bool head = (s.lo == 0 && !full);
            const int d0 = half * DCOLS;
            const long long orow =
                (((long long)s.b * p.Tq + qr) * p.H_out + p.head_offset + s.h * p.G + g_r) * HD + d0;
            const uint32_t q1 = pc - 1;
            mbar_wait(pv_done + (q1 & 1), (q1 >> 1) & 1);
            if (threadIdx.x == 0) K1_GT(3);
            if (threadIdx.x == 0) K1_TRACE(12, segn);
            float l_row = l;
            // DUAL: weights of the two halves' accumulators under the merged max
            float wa = 1.f, wb = 0.f;
            if constexpr (!DUAL) {
                l_row += __shfl_xor_sync(0xffffffffu, l, 16);
            } else {
                // exchange (m, l) with the other half's thread of this row
                // through shared memory (bar.sync orders it in the CTA)
                float2* xc = reinterpret_cast<float2*>(smem + C::OFF_XCHG);
                xc[half * 128 + r] = make_float2(m, l);
                named_bar_sync(1, SW * 32);
                const float2 o2 = xc[(1 - half) * 128 + r];
                const float m_o = o2.x, l_o = o2.y;
                named_bar_sync(1, SW * 32);  // reads done before the next segment's writes
                if (threadIdx.x == 0) K1_TRACE(13, segn);
                const float ma = half ? m_o : m, mb = half ? m : m_o;
                const float la = half ? l_o : l, lb = half ? l : l_o;
                const float mm = fmaxf(ma, mb);
                wa = ma == -INFINITY ? 0.f : ex2((ma - mm) * c);
                wb = mb == -INFINITY ? 0.f : ex2((mb - mm) * c);
                l_row = la * wa + lb * wb;
                m = mm;
            }
            if (dsm && !DUAL) {
                // ==== DSMEM merge, M=64: the pair's head (rank 0) and piece ====
                // (rank 1) sit in one 2-CTA cluster. The piece stages its O,
                // float4 (r, 4q..4q+3) at q * M + r, and its (m, l) in its own
                // drained K ring and bulk-copies them (cluster shared memory,
                // completing on the head's xchg_full) into the head's first
                // freed K stage and its idle second Q buffer (one segment per
                // CTA in this schedule) while the head still runs its last
                // tile; the head merges and writes the rows out. (Per-thread
                // st.shared::cluster stores + a release arrive measured
                // slower: the release waits for every remote store.)
                const uint32_t rank = blockIdx.x & 1u;
                float ov[DCOLS];
                if (warp_live) {
                    tc_fence_after();
#pragma unroll
                    for (int ch = 0; ch < DCOLS / 32; ++ch) {
                        uint32_t raw[32];
                        tmem_ld_32x32b_x32(lane_addr + C::O_COL + ch * 32, raw);
                        tmem_ld_wait();
#pragma unroll
                        for (int k = 0; k < 32; ++k) ov[ch * 32 + k] = __uint_as_float(raw[k]);
                    }
                    tc_fence_before();
                }
                const uint32_t khead = rank ? (uint32_t)s.lo : (uint32_t)ntl;  // the head's K tiles
                uint8_t* rx = sm_k + (khead >= (uint32_t)KS ? khead % KS : khead) * TILE_BYTES;
                float* mlb = reinterpret_cast<float*>(sm_q + C::A_BYTES);
                const bool stamp = threadIdx.x == 0;
                if (stamp) K1_TRACE(14, 40 + 4 * rank);
                if (rank) {
                    // O and (m, l) into this CTA's own drained K ring, then two
                    // bulk copies into the head's, completing on its xchg_full
                    float* lo_o = reinterpret_cast<float*>(sm_k);
                    float* lo_ml = reinterpret_cast<float*>(sm_k + 4 * C::PIECE_BOX);
                    if (half == 0) reinterpret_cast<float2*>(lo_ml)[r] = make_float2(m, l_row);
                    if (warp_live) {
                        float4* po = reinterpret_cast<float4*>(lo_o) + half * (DCOLS / 4) * M + r;
#pragma unroll
                        for (int q = 0; q < DCOLS / 4; ++q)
                            po[q * M] = make_float4(ov[4 * q], ov[4 * q + 1], ov[4 * q + 2], ov[4 * q + 3]);
                    }
                    fence_proxy_async_smem();
                    named_bar_sync(2, SW * 32);
                    if (stamp) K1_TRACE(14, 46);
                    if (threadIdx.x == 0) {
                        mbar_wait_cluster(peer_ready, 0);
                        K1_TRACE(14, 45);
                        bulk_s2s_cluster(mapa_rank(rx, 0), lo_o, 4u * C::PIECE_BOX, mapa_rank(xchg_full, 0));
                        bulk_s2s_cluster(mapa_rank(mlb, 0), lo_ml, 8u * M, mapa_rank(xchg_full, 0));
                        K1_TRACE(14, 47);
                    }
                } else {
                    mbar_wait_cluster(xchg_full, 0);
                    if (threadIdx.x == 0) K1_GT(10);
                    if (stamp) K1_TRACE(14, 41);
                    const float2 ml = reinterpret_cast<const float2*>(mlb)[r];
                    const float mf = fmaxf(m, ml.x);
                    const float w_self = m == -INFINITY ? 0.f : ex2((m - mf) * c);
                    const float wp = ml.x == -INFINITY ? 0.f : ex2((ml.x - mf) * c);
                    const float lf = l_row * w_self + ml.y * wp;
                    if (valid) {
                        const float4* pp = reinterpret_cast<const float4*>(rx) + half * (DCOLS / 4) * M + r;
#pragma unroll
                        for (int q = 0; q < DCOLS / 4; ++q) {
                            const float4 x = pp[q * M];
                            ov[4 * q] = fmaf(x.x, wp, ov[4 * q] * w_self);
                            ov[4 * q + 1] = fmaf(x.y, wp, ov[4 * q + 1] * w_self);
                            ov[4 * q + 2] = fmaf(x.z, wp, ov[4 * q + 2] * w_self);
                            ov[4 * q + 3] = fmaf(x.w, wp, ov[4 * q + 3] * w_self);
                        }
                        if (stamp) K1_TRACE(14, 43);
                        const float inv = 1.f / lf;
                        if (p.o_peers) {  // fused all-gather: this row into every rank's buffer
                            for (int k = 0; k < p.world; ++k)
                                store_row<T, DCOLS>(reinterpret_cast<T*>(p.o_peers[k]) + orow, ov, inv);
                        } else {
                            store_row<T, DCOLS>(reinterpret_cast<T*>(p.o) + orow, ov, inv);
                        }
                        if (p.lse && half == 0)
                            p.lse[((long long)s.b * p.Hq + s.h * p.G + g_r) * p.Tq + qr] = mf * p.scale + __logf(lf);
                    }
                    if (stamp) K1_TRACE(14, 42);
                }
                mbar_arrive(o_empty);
            } else if (dsm) {
                // ==== DSMEM exchange, DUAL: the pair's two pieces sit in one 2-CTA ====
                // cluster (piece index = cluster rank) and finish together. CTA
                // `rank` finalises d columns [64 rank, 64 rank + 64): the threads
                // holding the other d half (one per row) store their (m, l) and
                // O columns into the peer's drained K ring and arrive on its
                // xchg_full; the threads holding this CTA's half wait for the
                // peer's, merge in piece order and write the rows out.
                const uint32_t rank = blockIdx.x & 1u;
                const bool sender = (uint32_t)half != rank;
                // this thread's d half of O, 32 columns at a time (DUAL: both
                // accumulators, weighted). M=64: a row's two d halves sit in
                // one warp, one sending, one receiving, so both chunks are read
                // (warp-collective) before any lane waits; DUAL: the halves
                // are whole warps and read chunk by chunk.
                float ov[DUAL ? 1 : DCOLS];
                auto chunk = [&](int ch, float (&cv)[32]) {
                    if constexpr (DUAL) {
                        uint32_t raw[32];
                        tmem_ld_32x32b_x32(lane_addr + C::O_COL + half * DCOLS + ch * 32, raw);
                        tmem_ld_wait();
#pragma unroll
                        for (int k = 0; k < 32; ++k) cv[k] = __uint_as_float(raw[k]) * wa;
                        tmem_ld_32x32b_x32(lane_addr + C::OB_COL + half * DCOLS + ch * 32, raw);
                        tmem_ld_wait();
#pragma unroll
                        for (int k = 0; k < 32; ++k) cv[k] += __uint_as_float(raw[k]) * wb;
                    } else {
#pragma unroll
                        for (int k = 0; k < 32; ++k) cv[k] = ov[ch * 32 + k];
                    }
                };
                if (warp_live) tc_fence_after();
                if constexpr (!DUAL) {
                    if (warp_live) {
#pragma unroll
                        for (int ch = 0; ch < DCOLS / 32; ++ch) {
                            uint32_t raw[32];
                            tmem_ld_32x32b_x32(lane_addr + C::O_COL + ch * 32, raw);
                            tmem_ld_wait();
#pragma unroll
                            for (int k = 0; k < 32; ++k) ov[ch * 32 + k] = __uint_as_float(raw[k]);
                        }
                    }
                }
                // receive area in the drained K ring: (m, l) as float2[M], then
                // the O half as float4 (r, 4q..4q+3) at q * M + r
                float* xb = reinterpret_cast<float*>(sm_k);
                // trace stamps (row 14, columns 40-47): thread 0 and the first
                // thread of the other d half (lane 16 for M=64, warp 4 DUAL)
                const bool stamp = threadIdx.x == 0 || threadIdx.x == (DUAL ? 128 : 16);
                if (stamp) K1_TRACE(14, 40 + (sender ? 4 : 0));
                if (sender) {
                    const uint32_t peer = rank ^ 1u;
                    mbar_wait_cluster(peer_ready, 0);
                    if (stamp) K1_TRACE(14, 45);
                    st_cluster_v2(mapa_rank(xb + 2 * r, peer), m, l_row);
                    if (warp_live) {
                        const uint32_t ob = mapa_rank(xb + 2 * 128, peer) + 16u * (uint32_t)r;
#pragma unroll
                        for (int ch = 0; ch < DCOLS / 32; ++ch) {
                            float cv[32];
                            chunk(ch, cv);
#pragma unroll
                            for (int q = 0; q < 8; ++q)
                                st_cluster_v4(ob + 16u * (uint32_t)((ch * 8 + q) * M), cv[4 * q], cv[4 * q + 1],
                                              cv[4 * q + 2], cv[4 * q + 3]);
                        }
                    }
                    if (stamp) K1_TRACE(14, 46);
                    mbar_arrive_cluster(mapa_rank(xchg_full, peer));
                    if (stamp) K1_TRACE(14, 47);
                } else {
                    mbar_wait_cluster(xchg_full, 0);
                    if (threadIdx.x == 0) K1_GT(10);
                    if (stamp) K1_TRACE(14, 41);
                    const float2 ml = reinterpret_cast<const float2*>(xb)[r];
                    // piece order (rank 0 first), whichever CTA finalises the half
                    const float m0 = rank ? ml.x : m, l0 = rank ? ml.y : l_row;
                    const float m1 = rank ? m : ml.x, l1 = rank ? l_row : ml.y;
                    const float mf = fmaxf(m0, m1);
                    const float w0 = m0 == -INFINITY ? 0.f : ex2((m0 - mf) * c);
                    const float w1 = m1 == -INFINITY ? 0.f : ex2((m1 - mf) * c);
                    const float lf = l0 * w0 + l1 * w1;
                    const float inv = 1.f / lf;
                    if (warp_live) {
                        const float4* pp = reinterpret_cast<const float4*>(xb + 2 * 128) + r;
#pragma unroll
                        for (int ch = 0; ch < DCOLS / 32; ++ch) {
                            float cv[32];
                            chunk(ch, cv);
                            if (!valid) continue;
#pragma unroll
                            for (int q = 0; q < 8; ++q) {
                                const float4 x = pp[(ch * 8 + q) * M];
                                const float xs[4] = {x.x, x.y, x.z, x.w};
#pragma unroll
                                for (int k = 0; k < 4; ++k) {
                                    const float a0 = rank ? xs[k] : cv[4 * q + k];
                                    const float a1 = rank ? cv[4 * q + k] : xs[k];
                                    cv[4 * q + k] = fmaf(a1, w1, a0 * w0);
                                }
                            }
                            if (p.o_peers) {  // fused all-gather: this row into every rank's buffer
                                for (int k = 0; k < p.world; ++k)
                                    store_row<T, 32>(reinterpret_cast<T*>(p.o_peers[k]) + orow + ch * 32, cv, inv);
                            } else {
                                store_row<T, 32>(reinterpret_cast<T*>(p.o) + orow + ch * 32, cv, inv);
                            }
                        }
                        if (valid && p.lse && rank == 0)
                            p.lse[((long long)s.b * p.Hq + s.h * p.G + g_r) * p.Tq + qr] = mf * p.scale + __logf(lf);
                    }
                    if (stamp) K1_TRACE(14, 42);
                }
                if (warp_live) tc_fence_before();
                mbar_arrive(o_empty);
            } else {
                // head: final (m, l) over this segment and the pieces of CTAs
                // blockIdx.x+1, ... whose ranges start inside the pair (CTA order:
                // deterministic); pass 2 below adds their O chunk by chunk
                // (the first STAGED_PIECES pieces were staged into the drained K
                // ring by the K producer warp; any further ones are read from L2)
                float m_fin = m, l_fin = l_row;
                const int* pieces = reinterpret_cast<const int*>(smem + C::OFF_PIECES);
                int np = 0;
                if (head) {
                    mbar_wait(merge_full, 0);
                    if (threadIdx.x == 0) K1_GT(10);
                    if (threadIdx.x == 0) K1_TRACE(13, 40);
                    np = pieces[0];
                }
                if (head && valid) {
                    for (int i = 0; i < np; ++i) {
                        float mp, lp;
                        if (i < C::STAGED_PIECES) {
                            const float* ml = reinterpret_cast<const float*>(sm_k + i * C::PIECE_SMEM);
                            mp = ml[r];
                            lp = ml[128 + r];
                        } else {
                            const float* piece = p.partial + (long long)pieces[1 + i] * SLOT_FLOATS;
                            mp = __ldcg(piece + 128 * HD + r);
                            lp = __ldcg(piece + 128 * HD + 128 + r);
                        }
                        const float mm = fmaxf(m_fin, mp);
                        if (mm != -INFINITY) {
                            l_fin = (m_fin == -INFINITY ? 0.f : l_fin * ex2((m_fin - mm) * c)) +
                                    (mp == -INFINITY ? 0.f : lp * ex2((mp - mm) * c));
                            m_fin = mm;
                        }
                    }
                }
                if (threadIdx.x == 0) K1_TRACE(13, 41);
                const bool publish = !full && !head;
                const float w_self = (m == -INFINITY) ? 0.f : ex2((m - m_fin) * c);
                const float inv = 1.f / l_fin;
                float* sp = p.partial + (long long)blockIdx.x * SLOT_FLOATS;
                // TMA-store epilogue: a whole pair that is this CTA's last
                // segment, every row of its Q box a live node — the rows are
                // staged (normalised, as the 128-byte-swizzled rows of the Q box
                // layout) in this segment's Q buffer, free once its last P.V is
                // done and reloaded by no later segment, and leave with one
                // tensor store instead of a warp's 32 row-strided stores
                const int node0 = rblk * (M / p.G);
                // (M=128 only: measured, GQA T=16 at 4K 52.66 -> 52.30 us; M=64's
                // two lanes per row already write 256 contiguous bytes, and the
                // staging barrier cost it 0.3 us at GQA T=8)
                const bool tma_out = DUAL && p.o_tma && full && t + ntl >= t_end &&
                                     p.u0 + min(node0 + M / p.G, p.Tq) <= n;
                uint8_t* stage = sm_q + (segn % QS) * C::A_BYTES;
                if (warp_live) {
                    tc_fence_after();
    #pragma unroll 1
                    for (int ch = 0; ch < DCOLS / 32; ++ch) {
                        float ov[32];
                        uint32_t raw[32];
                        // M=64: this lane's d half of the shared O. DUAL: d half
                        // `half` of both accumulators, weighted.
                        tmem_ld_32x32b_x32(lane_addr + C::O_COL + (DUAL ? half * DCOLS : 0) + ch * 32, raw);
                        if constexpr (DUAL) {  // both accumulators' loads in flight, one wait
                            uint32_t rawb[32];
                            tmem_ld_32x32b_x32(lane_addr + C::OB_COL + half * DCOLS + ch * 32, rawb);
                            tmem_ld_wait();
    #pragma unroll
                            for (int k = 0; k < 32; ++k)
                                ov[k] = fmaf(__uint_as_float(rawb[k]), wb, __uint_as_float(raw[k]) * wa);
                        } else {
                            tmem_ld_wait();
    #pragma unroll
                            for (int k = 0; k < 32; ++k) ov[k] = __uint_as_float(raw[k]) * wa;
                        }
                        if (!valid) continue;
                        const int dc = d0 + ch * 32;
                        if (publish) {  // later piece of a pair: unnormalised O for the head owner
                            float4* po = reinterpret_cast<float4*>(sp) + (dc >> 2) * M + r;
    #pragma unroll
                            for (int k = 0; k < 8; ++k)
                                po[k * M] = make_float4(ov[4 * k], ov[4 * k + 1], ov[4 * k + 2], ov[4 * k + 3]);
                            continue;
                        }
                        if (head) {
    #pragma unroll
                            for (int k = 0; k < 32; ++k) ov[k] *= w_self;
                            for (int i = 0; i < np; ++i) {
                                const bool staged = i < C::STAGED_PIECES;
                                const float* piece = staged
                                    ? reinterpret_cast<const float*>(sm_k + i * C::PIECE_SMEM)
                                    : p.partial + (long long)pieces[1 + i] * SLOT_FLOATS;
                                const float mp = staged ? piece[r] : __ldcg(piece + 128 * HD + r);
                                if (mp == -INFINITY) continue;
                                const float wp = ex2((mp - m_fin) * c);
                                // float4 (r, dc + 4k) at (dc/4 + k) * M + r of the piece's O
                                const float4* pp =
                                    reinterpret_cast<const float4*>(staged ? reinterpret_cast<const uint8_t*>(piece) + 1024
                                                                           : reinterpret_cast<const uint8_t*>(piece)) +
                                    (dc >> 2) * M + r;
    #pragma unroll
                                for (int k = 0; k < 8; ++k) {
                                    const float4 x = staged ? pp[k * M] : __ldcg(pp + k * M);
                                    ov[4 * k] = fmaf(x.x, wp, ov[4 * k]);
                                    ov[4 * k + 1] = fmaf(x.y, wp, ov[4 * k + 1]);
                                    ov[4 * k + 2] = fmaf(x.z, wp, ov[4 * k + 2]);
                                    ov[4 * k + 3] = fmaf(x.w, wp, ov[4 * k + 3]);
                                }
                            }
                        }
                        if (threadIdx.x == 0) K1_TRACE(13, 42 + 2 * ch);
                        if (tma_out) {
                            uint8_t* rowp = stage + (half * M + r) * 128;
#pragma unroll
                            for (int j = 0; j < 4; ++j) {
                                uint32_t w4[4];
#pragma unroll
                                for (int e = 0; e < 4; ++e)
                                    w4[e] = pk2<T>::pack(ov[8 * j + 2 * e] * inv, ov[8 * j + 2 * e + 1] * inv);
                                const int cx = ch * 4 + j;  // 16-byte chunk of the row, swizzled
                                *reinterpret_cast<uint4*>(rowp + ((cx ^ (r & 7)) << 4)) =
                                    make_uint4(w4[0], w4[1], w4[2], w4[3]);
                            }
                        } else if (p.o_peers) {  // fused all-gather: this row into every rank's buffer
                            for (int k = 0; k < p.world; ++k)
                                store_row<T, 32>(reinterpret_cast<T*>(p.o_peers[k]) + orow + ch * 32, ov, inv);
                        } else {
                            store_row<T, 32>(reinterpret_cast<T*>(p.o) + orow + ch * 32, ov, inv);
                        }
                        if (threadIdx.x == 0) K1_TRACE(13, 43 + 2 * ch);
                    }
                    tc_fence_before();
                }
                if (tma_out) {
                    fence_proxy_async_smem();  // the staged rows, visible to the tensor store
                    named_bar_sync(1, SW * 32);
                    if (threadIdx.x == 0) {
                        tma_store_5d(&tm_o, stage, 0, s.h * p.G, node0, 0, s.b);
                        bulk_commit_group();
                        bulk_wait_group_read0();  // (the CTA's shared memory outlives the read)
                    }
                }
                if (threadIdx.x == 0) K1_TRACE(14, segn);
                mbar_arrive(o_empty);
                if (publish) {
                    if (valid && half == 0) {
                        sp[128 * HD + r] = m;
                        sp[128 * HD + 128 + r] = l_row;
                    }
                    // bar.sync orders every thread's stores before thread 0's
                    // gpu-scope release (release is cumulative)
                    named_bar_sync(2, SW * 32);
                    if (threadIdx.x == 0) st_release_gpu(p.flags + blockIdx.x, 1u);
                } else {
                    if (valid && p.lse && half == 0)
                        p.lse[((long long)s.b * p.Hq + s.h * p.G + g_r) * p.Tq + qr] = m_fin * p.scale + __logf(l_fin);
                }
            }
            if (threadIdx.x == 0) K1_GT(4);
            if (threadIdx.x == 0) K1_TRACE(15, segn);
            ++segn;
            t += ntl;
        }
    }

    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    // DSMEM merge: no CTA leaves while its peer may still copy out of / into it
    // (mc: no CTA leaves while its peer may still multicast into it or
    // commit to its barriers)
    if (dsm || mc) cluster_sync();
    if (p.trace && threadIdx.x == 0) {
        unsigned long long gt;
        asm volatile("mov.u64 %0, %globaltimer;" : "=l"(gt));
        p.trace[kTraceRows * 64 + kTraceCta * blockIdx.x + 1] = gt;
        p.trace[kTraceRows * 64 + kTraceCta * blockIdx.x + 7] = clock64();
    }
    if (warp == SW + 2) tmem_dealloc<C::TMEM_COLS>(tmem);
}

// ------------------------------------------------------------------ host --
PFN_cuTensorMapEncodeTiled_v12000 get_encode() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    static std::once_flag once;
    std::call_once(once, [] {
        cudaDriverEntryPointQueryResult q;
        void* f = nullptr;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &f, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(f);
    });
    return fn;
}

int num_sms() {
    static int cache[64] = {0};
    int dev = 0;
    cudaGetDevice(&dev);
    if (dev < 0 || dev >= 64) return 148;
    if (!cache[dev]) cudaDeviceGetAttribute(&cache[dev], cudaDevAttrMultiProcessorCount, dev);
    return cache[dev];
}

bool encode(CUtensorMap* m, CUtensorMapDataType dt, int rank, const void* ptr, const uint64_t* dims,
            const uint64_t* strides_bytes, const uint32_t* box) {
    auto fn = get_encode();
    if (!fn) return false;
    uint32_t es[5] = {1, 1, 1, 1, 1};  // element strides, up to rank 5
    return fn(m, dt, rank, const_cast<void*>(ptr), dims, strides_bytes, box, es,
              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

size_t align_up(size_t x, size_t a) { return (x + a - 1) / a * a; }

}  // namespace

bool tree_attention_tc_supported(const st_attn_args* a) {
    auto al = [](const void* q) { return (reinterpret_cast<uintptr_t>(q) & 15) == 0; };
    // GQA: G = H/Hkv query heads share a KV head; a pair's Q rows are its G*T
    // (node, head) rows in M-row blocks (M = 64 or 128; G*T > 128: two blocks
    // of 128 on a CTA pair), so G must divide M and G*T <= 256
    const int G = a->Hkv > 0 && a->H % a->Hkv == 0 ? a->H / a->Hkv : 0;
    const int Tq = a->q_rows > 0 ? a->q_rows : a->T;
    const int M = (int64_t)G * Tq <= 64 ? 64 : 128;
    const bool slice_ok = a->q_rows <= 0 ||
                          (a->k_tree && a->q_node0 >= 0 && (int64_t)a->q_node0 + a->q_rows <= a->T);
    return (a->dtype == ST_F16 || a->dtype == ST_BF16) && a->D == HD && G >= 1 && M % G == 0 &&
           slice_ok && (int64_t)G * Tq <= 256 && a->W <= 4 && a->Lmax < (1ll << 31) && al(a->q) && al(a->k_cache) &&
           al(a->v_cache) && al(a->o) && al(a->k_tree) && al(a->v_tree) &&
           (int64_t)a->B * a->Hkv * ((a->Lmax + BN - 1) / BN) < (1ll << 31);  // 32-bit tile indices
}


// Workspace: per CTA one piece slot and one piece flag (zero on first use;
// every launch leaves the flags zero).
size_t tree_attention_tc_workspace(const st_attn_args* a) {
    return align_up((size_t)num_sms() * SLOT_FLOATS * sizeof(float), 256) +
           (size_t)num_sms() * sizeof(unsigned);
}

namespace {

// K1 is launched with programmatic dependent launch (common.cuh): its prologue
// overlaps the previous kernel's tail. Split pairs are merged inside K1: a
// pair's head CTA waits for flags the piece CTAs release, so the grid (one CTA
// per SM) is launched cooperatively — co-residency guaranteed by the runtime,
// not assumed (ST_K1_COOP=0 turns it off for A/B runs).
template <class TT, int MM, int MW>
st_status launch_tc(const TcLaunch& L, cudaStream_t stream) {
    static bool attr = false;
    static int max_pairs = 0;  // co-resident 2-CTA clusters
    if (!attr) {
        ST_CUDA_TRY(cudaFuncSetAttribute(tree_attn_tc_kernel<TT, MM, MW>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         Cfg<MM>::SMEM_BYTES));
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(L.grid);
        cfg.blockDim = dim3(Cfg<MM>::THREADS);
        cfg.dynamicSmemBytes = Cfg<MM>::SMEM_BYTES;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        if (cudaOccupancyMaxActiveClusters(&max_pairs, tree_attn_tc_kernel<TT, MM, MW>, &cfg) != cudaSuccess) {
            (void)cudaGetLastError();
            max_pairs = 0;
        }
        attr = true;
    }
    // 2-CTA clusters (the DSMEM merge of two-piece split pairs) whenever every
    // pair of the grid fits at once; ST_K1_CLUSTER=0 keeps the global path
    static const bool allow = !(getenv("ST_K1_CLUSTER") && atoi(getenv("ST_K1_CLUSTER")) == 0);
    const bool clus = allow && L.grid % 2 == 0 && 2 * max_pairs >= L.grid;
    TcParams prm = L.prm;
    prm.cluster2 = clus ? 1 : 0;
    // two row blocks per pair on clusters: each CTA multicasts one d half
    // (the kernel's `mc`), so it gets the one-half maps
    const bool mc = MM == 128 && L.prm.R == 2 && clus;
    ST_CUDA_TRY(launch_pdl_ex(tree_attn_tc_kernel<TT, MM, MW>, dim3(L.grid), dim3(Cfg<MM>::THREADS),
                              Cfg<MM>::SMEM_BYTES, stream, L.coop, clus ? 2 : 1, L.tq, mc ? L.tk1 : L.tk,
                              mc ? L.tv1 : L.tv, mc ? L.tkt1 : L.tkt, mc ? L.tvt1 : L.tvt, L.to, prm));
    return ST_OK;
}

}  // namespace

st_status tree_attention_tc_prepare(const st_attn_args* a, const st_peer_out* po, TcLaunch* L) {
    const CUtensorMapDataType dt =
        a->dtype == ST_F16 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT16 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16;
    {
        // D = 128 as (64, half): dims (64, H, T, 2, B), the half (stride 128 B)
        // outside the nodes, so one box lands as the two K-major atoms
        const uint64_t Tq = a->q_rows > 0 ? (uint64_t)a->q_rows : (uint64_t)a->T;
        const uint64_t dims[5] = {64, (uint64_t)a->H, Tq, 2, (uint64_t)a->B};
        const uint64_t strides[4] = {HD * 2ull, (uint64_t)a->H * HD * 2, 128, Tq * a->H * HD * 2};
        const int G = a->H / a->Hkv;
        const uint32_t M = (int64_t)G * Tq <= 64 ? 64 : 128;
        const uint32_t box[5] = {64, (uint32_t)G, M / G, 2, 1};
        if (!encode(&L->tq, dt, 5, a->q, dims, strides, box)) {
            set_error("st_tree_attention: cuTensorMapEncodeTiled(q) failed");
            return ST_ERR_CUDA;
        }
        // o has q's layout (no head-sharded peer output): the same view, so a
        // staged tile leaves with one TMA store (ST_K1_OTMA=0: per-thread stores)
        static const bool otma = !(getenv("ST_K1_OTMA") && atoi(getenv("ST_K1_OTMA")) == 0);
        L->prm.o_tma = otma && !po && a->o && (reinterpret_cast<uintptr_t>(a->o) & 15) == 0 &&
                       encode(&L->to, dt, 5, a->o, dims, strides, box) ? 1 : 0;
        if (!L->prm.o_tma) L->to = L->tq;
    }
    {
        // (64, Lmax, 2, B*Hkv): one box = both d halves of a 128-row tile;
        // the one-half maps feed the multicast two-row-block loads
        const uint64_t dims[4] = {64, (uint64_t)a->Lmax, 2, (uint64_t)a->B * a->Hkv};
        const uint64_t strides[3] = {HD * 2ull, 128, (uint64_t)a->Lmax * HD * 2};
        const uint32_t box[4] = {64, BN, 2, 1}, box1[4] = {64, BN, 1, 1};
        if (!encode(&L->tk, dt, 4, a->k_cache, dims, strides, box) ||
            !encode(&L->tv, dt, 4, a->v_cache, dims, strides, box) ||
            !encode(&L->tk1, dt, 4, a->k_cache, dims, strides, box1) ||
            !encode(&L->tv1, dt, 4, a->v_cache, dims, strides, box1)) {
            set_error("st_tree_attention: cuTensorMapEncodeTiled(kv) failed");
            return ST_ERR_CUDA;
        }
    }
    L->tkt = L->tk;  // k_tree mode: the tree's rows, [B][T][Hkv][D], 128-node boxes
    L->tvt = L->tv;
    L->tkt1 = L->tk1;
    L->tvt1 = L->tv1;
    if (a->k_tree) {
        const uint64_t dims[5] = {64, (uint64_t)a->Hkv, (uint64_t)a->T, 2, (uint64_t)a->B};
        const uint64_t strides[4] = {HD * 2ull, (uint64_t)a->Hkv * HD * 2, 128,
                                     (uint64_t)a->T * a->Hkv * HD * 2};
        const uint32_t box[5] = {64, 1, BN, 2, 1}, box1[5] = {64, 1, BN, 1, 1};
        if (!encode(&L->tkt, dt, 5, a->k_tree, dims, strides, box) ||
            !encode(&L->tvt, dt, 5, a->v_tree, dims, strides, box) ||
            !encode(&L->tkt1, dt, 5, a->k_tree, dims, strides, box1) ||
            !encode(&L->tvt1, dt, 5, a->v_tree, dims, strides, box1)) {
            set_error("st_tree_attention: cuTensorMapEncodeTiled(k_tree/v_tree) failed");
            return ST_ERR_CUDA;
        }
    }
    const int Tq = a->q_rows > 0 ? a->q_rows : a->T;                 // Q rows per request
    const int R = (int64_t)(a->H / a->Hkv) * Tq <= 128 ? 1 : 2;      // row blocks per pair
    // ST_K1_GRID (diagnostic): fewer CTAs than SMs, e.g. to measure the HBM
    // rate K1 keeps on a subset of the SMs
    static const int grid_env = getenv("ST_K1_GRID") ? atoi(getenv("ST_K1_GRID")) : 0;
    const int sms = grid_env > 0 && grid_env < num_sms() ? grid_env : num_sms();
    const int G = (sms < kMaxPieces + 1 ? sms : kMaxPieces + 1) / R * R;
    TcParams& prm = L->prm;
    prm.prefix_len = a->prefix_len;
    prm.n_nodes = a->n_nodes;
    prm.mask = a->mask;
    prm.o = a->o;
    prm.lse = a->lse;
    prm.partial = reinterpret_cast<float*>(a->workspace);
    prm.flags = reinterpret_cast<unsigned*>(reinterpret_cast<uint8_t*>(a->workspace) +
                                            align_up((size_t)G * SLOT_FLOATS * sizeof(float), 256));
    prm.B = a->B;
    prm.T = a->T;
    prm.Tq = Tq;
    prm.u0 = a->q_rows > 0 ? a->q_node0 : 0;
    prm.H = a->Hkv;
    prm.G = a->H / a->Hkv;
    prm.Hq = a->H;
    prm.R = R;
    prm.tree_src = a->k_tree != nullptr;
    prm.early_kv = a->early_kv != 0;
    prm.W = a->W;
    prm.scale = (float)a->scale;
    prm.c_log2 = (float)(a->scale * 1.4426950408889634);
    prm.o_peers = po ? po->out : nullptr;
    prm.world = po ? po->world : 1;
    prm.head_offset = po ? po->rank * a->H : 0;
    prm.H_out = po ? po->world * a->H : a->H;
    prm.trace = nullptr;
    // diagnostic override of the whole-pair schedule threshold (ST_K1_SLACK=-1: always stream-K)
    static const int slack_env = getenv("ST_K1_SLACK") ? atoi(getenv("ST_K1_SLACK")) : (int)kAlignedSlack;
    prm.aligned_slack = slack_env;
    static const int hx_env = getenv("ST_K1_HEADX") ? atoi(getenv("ST_K1_HEADX")) : (int)kHeadExtra;
    prm.head_extra = hx_env < 0 ? 0 : hx_env;
    prm.trace_cta = getenv("ST_K1_TRACE_CTA") ? atoi(getenv("ST_K1_TRACE_CTA")) : 0;
    prm.g_magic = ~0ull / (unsigned long long)(G / R) + 1ull;  // floor(2^64 / slots) + 1
    prm.cluster2 = 0;  // set per launch (launch_tc)
    // fast start: two tiles per ring before the CTA barrier, not the whole
    // ring — every CTA's first burst queues less in front of the metadata and
    // the later issues (measured: 0.2-0.5 % on every K1 shape of
    // tools/k1_sched_ab.py, three same-box repetitions; ST_K1_PRE=0: the ring)
    static const int pre_env = getenv("ST_K1_PRE") ? atoi(getenv("ST_K1_PRE")) : 2;
    prm.pre_cap = pre_env;
    static const int most_env = getenv("ST_K1_MOST") ? atoi(getenv("ST_K1_MOST")) : 1;
    prm.most_aligned = most_env;
    static const bool coop = !(getenv("ST_K1_COOP") && atoi(getenv("ST_K1_COOP")) == 0);
    L->coop = coop;
    L->grid = G;
    L->m64 = (int64_t)prm.G * Tq <= 64;
    L->mw4 = a->W > 2;   // T > 128
    L->f16 = a->dtype == ST_F16;
    return ST_OK;
}

st_status tree_attention_tc_launch(const TcLaunch& L, cudaStream_t stream) {
    st_status r;
    if (L.f16) {
        r = L.m64 ? launch_tc<__half, 64, 2>(L, stream)
            : !L.mw4 ? launch_tc<__half, 128, 2>(L, stream) : launch_tc<__half, 128, 4>(L, stream);
    } else {
        r = L.m64 ? launch_tc<__nv_bfloat16, 64, 2>(L, stream)
            : !L.mw4 ? launch_tc<__nv_bfloat16, 128, 2>(L, stream)
                     : launch_tc<__nv_bfloat16, 128, 4>(L, stream);
    }
    if (r != ST_OK) return r;
    ST_LAUNCH_CHECK();
    return ST_OK;
}

st_status tree_attention_tc(const st_attn_args* a, cudaStream_t stream, const st_peer_out* po) {
    TcLaunch L;
    if (st_status e = tree_attention_tc_prepare(a, po, &L)) return e;
    static unsigned long long* trace_buf = nullptr;
    const int G = L.grid;
    if (getenv("ST_K1_TRACE")) {
        if (!trace_buf) cudaMalloc(&trace_buf, (kTraceRows * 64 + kTraceCta * 1024) * sizeof(unsigned long long));
        cudaMemsetAsync(trace_buf, 0, (kTraceRows * 64 + kTraceCta * 1024) * sizeof(unsigned long long), stream);
        L.prm.trace = trace_buf;
    }
    if (st_status e = tree_attention_tc_launch(L, stream)) return e;
    if (L.prm.trace) {  // diagnostic only: dump CTA 0's pipeline timestamps
        static unsigned long long h[kTraceRows * 64 + kTraceCta * 1024];
        cudaMemcpyAsync(h, L.prm.trace, sizeof h, cudaMemcpyDeviceToHost, stream);
        cudaStreamSynchronize(stream);
        if (FILE* f = fopen(getenv("ST_K1_TRACE"), "a")) {
            for (int r = 0; r < kTraceRows; ++r) {
                for (int i = 0; i < 64; ++i) fprintf(f, "%llu ", h[r * 64 + i]);
                fprintf(f, "\n");
            }
            for (int i = 0; i < kTraceCta * G; ++i) fprintf(f, "%llu ", h[kTraceRows * 64 + i]);
            fprintf(f, "\n");
            fclose(f);
        }
    }
    return ST_OK;
}

}  // namespace st
