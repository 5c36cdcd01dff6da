// Exact maximum-weight perfect matching of a square integer weight matrix by
// multilevel, dual-warm-started successive shortest paths on the GPU.
//
// Replaces the reference's O(n^3) Kuhn-Munkres (`_solve_min_assignment`,
// /root/reference/pkg/src/muxsim/matching.py:45-101) for the square case
// N == M of `max_weight_matching` (matching.py:148-208).  The reference's
// Hungarian is itself a successive-shortest-path method: one Dijkstra over the
// reduced costs per row, dual update, augment.  On predictor weights started
// from zero duals every row explores ~n/3 columns (n^3 work); here two things
// change:
//
//  * Warm duals.  Rows and columns are ordered by a scalar key (the online /
//    offline SM demand for the table predictor, row / column sums otherwise),
//    and a stratified 1-in-f subsample of both is solved first, recursively.
//    Its optimal row profits pi^c are carried to the finer level by the
//    c-transform p_j = max_k (a_kj - pi^c_k) over the coarse rows: the largest
//    column prices the coarse optimum supports.  Measured on the 10k x 10k
//    predictor round, a Dijkstra from these prices scans ~1.7 columns per
//    augmentation instead of ~3,000.
//
//  * Sparse candidates with an exactness horizon.  Each row keeps its KC best
//    columns by value a_ij - p_j and tau_i, an upper bound on the value of
//    every other column.  Prices only rise, so tau_i stays valid, and a column
//    outside the list is at reduced distance >= h_i = d_i + pi_i - tau_i from
//    the search root.  The Dijkstra pops only while the next distance is
//    <= min h_i; past the horizon the row is re-scanned densely (its next KC
//    columns by distance join the search).  Every dual update therefore keeps
//    pi_i + p_j >= a_ij on ALL n^2 edges: the result is exactly optimal for
//    the dense matrix, with exact integer duals.
//
// Parallelism: one Dijkstra per warp, many warps at once.  A search locks a
// column (atomicCAS) when it pops it; prices read earlier without the lock are
// re-validated after locking (a raised price only lengthens the entry, which
// is then re-queued).  Nothing global is written before the augmenting path is
// found, so a search that meets a column locked by another simply releases
// its locks and is retried later.  Searches that grow past the warp's shared
// memory table or step budget are deferred to an exclusive single-CTA pass
// with global-memory tables (the few long augmenting paths of a level).
//
// Values: benefits a_ij are the quantised weights (int32, qbits <= 30);
// prices and distances are int64.  Sort keys pack a distance (< 2^39) above a
// 24-bit index, so n < 2^24.
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <numeric>
#include <vector>

#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace mux {
// One source, two solvers: int32 weights (qbits <= 30; ssp.cu) and int64
// weights (qbits <= 44, n < 65,000; ssp_w64.cu includes this file with
// MUX_SSP_W64).  Sort keys pack a value above an index field of kSH bits
// (the top one a "column is matched" flag): 24 bits for int32 problems, 17
// for int64 ones, whose values need the extra range.
#ifndef MUX_SSP_W64
namespace ssp {
using wt_t = int32_t;
constexpr int kSH = 24;
constexpr int64_t kDistLim = 1ll << 39;
#else
namespace ssp64 {
using wt_t = int64_t;
constexpr int kSH = 17;
constexpr int64_t kDistLim = 1ll << 46;
#endif
constexpr uint32_t kFreeBit = 1u << (kSH - 1);          // set = matched column (free columns sort first)
constexpr uint32_t kIdxMask = kFreeBit - 1u;             // column / entry index
constexpr uint64_t kLowMask = (1ull << kSH) - 1ull;      // flag + index

constexpr int KC = 32;                 // candidates per row record (one per lane)
constexpr int TC = 256;                // touched columns per warp table (parallel mode)
constexpr int HSZ = 512;               // hash slots per warp table
constexpr int PWARPS = 8;              // warps per CTA in parallel mode
constexpr int STEP_BUDGET_DEFAULT = 48;   // Dijkstra pops before a search is deferred
constexpr int DEEP_BUDGET_DEFAULT = 4;    // dense row re-scans before a search is deferred
constexpr int MAX_TRIES = 16;          // lock-conflict retries before deferral
constexpr int64_t kInf = INT64_MAX / 4;
constexpr uint64_t kNoKey = ~0ull;

enum : uint32_t {
    kErrDist = 1u << 0,      // a distance / price left the packed key range
    kErrNoPath = 1u << 1,    // a search ran out of columns (cannot happen on a complete graph)
    kErrOpenCap = 1u << 2,   // exclusive-mode open list overflow
};

struct Cnt {
    int32_t qhead;
    int32_t nretry;
    int32_t ndefer;
    uint32_t errors;
    unsigned long long steps, deep, aborts, augs, xsteps, xdeep, refresh, overflow;
    long long xcyc[4];   // exclusive kernel: pop, horizon re-scans, scan steps, augment
    unsigned long long xpfhits;   // register-key kernel: pops whose row slice was prefetched into smem
    unsigned long long xwalk, xwalkcyc, xsearch, xsynccyc;   // timing mode: augmenting-path walk steps / cycles, searches
    unsigned long long xrounds;   // register-key kernel: exchange steps (pops minus batched ties)
    unsigned long long xt[5];     // timing mode: load+relax cycles / steps of prefetch-hit steps, of tie steps; push-to-arrival cycles
};

struct Lvl {
    const wt_t* A;   // [nreal][lda] benefits; rows >= nreal are zero (the reference's square padding)
    int64_t lda;
    int32_t m;
    int32_t nreal;
    const wt_t* zrow;   // m zeros
    int64_t* p;         // [m] column prices
    int32_t* cor;       // [m] column of row (-1 free)
    int32_t* roc;       // [m] row of column (-1 free)
    int32_t* lock;      // [m] 0 or owner warp id + 1
    int32_t* cj;        // [m][KC] candidate columns (-1 empty)
    wt_t* ca;           // [m][KC] their benefits
    int64_t* tau;       // [m] bound on every non-candidate value
    const int32_t* in;  // rows to process this pass
    int32_t nin;
    int32_t* retry;     // rows to retry next pass
    int32_t* defer;     // rows for the exclusive pass
    int32_t* tries;     // [m]
    Cnt* cnt;
    int32_t step_budget;
    int32_t deep_budget;
    // exclusive-mode scratch (global, direct-indexed by column)
    int64_t* xdist;
    int32_t* xpred;
    int32_t* xstamp;    // flags (uint8) when the tables live in global memory
    int32_t* xscol;     // scanned columns of the current search
    int32_t* xgap;      // global fallback: horizon gaps
    // rank-neighbour L2 prefetch of the long-path kernel (level 0): a long search pops
    // the rows of a contiguous key-rank window, so rows rpf ranks either side of the
    // popped row are fetched into L2 a few steps ahead (rpf = 0: off)
    const int32_t* rankof;   // [m] key rank of each row
    const int32_t* rowat;    // [m] row of each key rank
    int32_t rpf;
};

__device__ __forceinline__ const wt_t* rowp(const Lvl& L, int32_t i) {
    return i < L.nreal ? L.A + (int64_t)i * L.lda : L.zrow;
}

__device__ __forceinline__ int64_t ldv64(const int64_t* p) { return *reinterpret_cast<const volatile int64_t*>(p); }
__device__ __forceinline__ int32_t ldv32(const int32_t* p) { return *reinterpret_cast<const volatile int32_t*>(p); }
__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// 64-bit warp minimum as two 32-bit redux.sync reductions (high word, then
// the low word among the lanes holding the minimal high word): two dependent
// REDUX ops instead of five shuffle pairs on the search's critical path.
__device__ __forceinline__ uint64_t wmin64(uint64_t v) {
    const uint32_t hi = (uint32_t)(v >> 32), lo = (uint32_t)v;
    const uint32_t mh = __reduce_min_sync(0xffffffffu, hi);
    const uint32_t ml = __reduce_min_sync(0xffffffffu, hi == mh ? lo : 0xffffffffu);
    return ((uint64_t)mh << 32) | ml;
}
__device__ __forceinline__ int64_t wmax64s(int64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const int64_t w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w > v ? w : v;
    }
    return v;
}
__device__ __forceinline__ int64_t wmin64s(int64_t v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const int64_t w = __shfl_xor_sync(0xffffffffu, v, o);
        v = w < v ? w : v;
    }
    return v;
}

// key = (value + 2^39) << kSH | j : ascending key = ascending value, lowest j on ties
__device__ __forceinline__ uint64_t mkkey(int64_t v, int32_t j, uint32_t* err) {
    if (v <= -kDistLim || v >= kDistLim) { atomicOr(err, kErrDist); v = v < 0 ? -kDistLim + 1 : kDistLim - 1; }
    return ((uint64_t)(v + kDistLim) << kSH) | (uint64_t)(uint32_t)j;
}
__device__ __forceinline__ int64_t key_val(uint64_t k) { return (int64_t)(k >> kSH) - kDistLim; }
__device__ __forceinline__ int32_t key_idx(uint64_t k) { return (int32_t)(k & kLowMask); }

// Warp-wide selection of the 32 smallest keys produced by keyf(j), j in [0, m)
// (kNoKey = skip).  Lane r receives the r-th smallest (kNoKey when fewer);
// `bound` is a key <= every key not returned.  Per lane: a sorted top-8 in
// registers plus the smallest key it discarded; then 32 warp-min rounds.
template <class F>
__device__ __forceinline__ void warp_top32(int32_t m, F keyf, uint64_t& mine, uint64_t& bound) {
    uint64_t L[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) L[k] = kNoKey;
    uint64_t disc = kNoKey;
    // 8 keys per lane per trip: their loads are issued back to back
    constexpr int U = 8;
    for (int32_t j0 = 0; j0 < m; j0 += 32 * U) {
        uint64_t keys[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t j = j0 + u * 32 + lane_id();
            keys[u] = j < m ? keyf(j) : kNoKey;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const uint64_t key = keys[u];
            if (key < L[7]) {
                disc = L[7] < disc ? L[7] : disc;
                L[7] = key;
#pragma unroll
                for (int k = 7; k > 0; --k)
                    if (L[k] < L[k - 1]) { const uint64_t t = L[k]; L[k] = L[k - 1]; L[k - 1] = t; }
            } else {
                disc = key < disc ? key : disc;
            }
        }
    }
    mine = kNoKey;
#pragma unroll 1
    for (int r = 0; r < 32; ++r) {
        const uint64_t mn = wmin64(L[0]);
        if (mn == kNoKey) break;
        if (lane_id() == r) mine = mn;
        if (L[0] == mn) {
#pragma unroll
            for (int k = 0; k < 7; ++k) L[k] = L[k + 1];
            L[7] = kNoKey;
        }
    }
    const uint64_t b1 = wmin64(L[0]), b2 = wmin64(disc);
    bound = b1 < b2 ? b1 : b2;
}

// Rebuild row i's candidate record: its KC best columns by value a_ij - p_j
// and tau_i >= the value of every other column (prices only rise afterwards).
__device__ void refresh_row(const Lvl& L, int32_t i) {
    const wt_t* Ar = rowp(L, i);
    uint64_t mine, bound;
    // plain L2 loads (pipelined): a price read late is still a price the column
    // had, and prices only rise, so tau stays an upper bound
    warp_top32(L.m, [&](int32_t j) { return mkkey(__ldcg(L.p + j) - (int64_t)__ldg(Ar + j), j, &L.cnt->errors); },
               mine, bound);
    const int32_t j = mine == kNoKey ? -1 : key_idx(mine);
    L.cj[(int64_t)i * KC + lane_id()] = j;
    L.ca[(int64_t)i * KC + lane_id()] = j >= 0 ? __ldg(Ar + j) : 0;
    if (lane_id() == 0) L.tau[i] = bound == kNoKey ? -kInf : -key_val(bound);
    __syncwarp();
}

// One warp per row: initial candidate records of a level.
// Padding rows [plo, phi) are all-zero rows, so they share one record: only
// row plo is built here and pad_copy_kernel replicates it.
#ifndef CAND_MINB
#define CAND_MINB 5   // 48 registers: more resident warps for this latency-bound scan (level-0 setup 0.69 -> 0.63 ms)
#endif
__global__ void __launch_bounds__(256, CAND_MINB) cand_kernel(Lvl L, int32_t plo, int32_t phi) {
    const int32_t wid = (int32_t)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    const int32_t nw = (int32_t)((gridDim.x * (int64_t)blockDim.x) >> 5);
    for (int32_t i = wid; i < L.m; i += nw)
        if (i <= plo || i >= phi) refresh_row(L, i);
}

__global__ void pad_copy_kernel(Lvl L, int32_t plo, int32_t phi) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t rows = (int64_t)(phi - plo - 1);
    if (t >= rows * KC) return;
    const int32_t i = plo + 1 + (int32_t)(t / KC);
    const int32_t k = (int32_t)(t % KC);
    L.cj[(int64_t)i * KC + k] = L.cj[(int64_t)plo * KC + k];
    L.ca[(int64_t)i * KC + k] = L.ca[(int64_t)plo * KC + k];
    if (k == 0) L.tau[i] = L.tau[plo];
}

// ---------------------------------------------------------------------------
// parallel mode: one Dijkstra per warp, shared-memory table, column locks
// ---------------------------------------------------------------------------

enum : uint8_t { kScanned = 1, kLocked = 2, kFreeHint = 4 };

struct WTab {
    int64_t dist[TC];
    int64_t snap[TC];    // price the distance was computed with
    int64_t hor[TC];     // scanned entries: horizon of their row
    int32_t col[TC];
    int32_t pred[TC];    // predecessor row
    int32_t row[TC];     // scanned entries: the column's matched row
    uint8_t st[TC];
    int32_t hash[HSZ];   // entry + 1, 0 = empty
};

__device__ __forceinline__ uint32_t hslot(int32_t c) { return ((uint32_t)c * 2654435761u) >> (32 - 9); }

__device__ __forceinline__ int32_t hfind(const WTab& T, int32_t c) {
    uint32_t h = hslot(c);
    while (true) {
        const int32_t e = T.hash[h];
        if (e == 0) return -1;
        if (T.col[e - 1] == c) return e - 1;
        h = (h + 1) & (HSZ - 1);
    }
}

// Relax one candidate per lane (c < 0: none) at distance nd with price pc.
// Returns false when the table is full.
__device__ __forceinline__ bool tab_relax(WTab& T, int32_t& nt, const Lvl& L, int32_t c, int64_t nd, int64_t pc,
                                          int32_t i) {
    int32_t e = c >= 0 ? hfind(T, c) : -1;
    if (c >= 0 && e >= 0 && !(T.st[e] & kScanned)) {
        // compare both paths at today's price: the entry's distance was
        // computed with the price it saw then (snap), which may have risen
        const int64_t cur = T.dist[e] + (pc - T.snap[e]);
        if (nd < cur) {
            T.dist[e] = nd;
            T.pred[e] = i;
        } else {
            T.dist[e] = cur;
        }
        T.snap[e] = pc;
    }
    const bool need = c >= 0 && e < 0;
    const unsigned bal = __ballot_sync(0xffffffffu, need);
    const int cntn = __popc(bal);
    if (nt + cntn > TC) return false;
    if (need) {
        e = nt + __popc(bal & ((1u << lane_id()) - 1u));
        T.col[e] = c;
        T.dist[e] = nd;
        T.snap[e] = pc;
        T.pred[e] = i;
        T.st[e] = ldv32(L.roc + c) < 0 ? kFreeHint : 0;
    }
    __syncwarp();
    if (need) {
        uint32_t h = hslot(c);
        while (atomicCAS(&T.hash[h], 0, e + 1) != 0) h = (h + 1) & (HSZ - 1);
    }
    __syncwarp();
    nt += cntn;
    return true;
}

__device__ __forceinline__ void tab_clear(WTab& T) {
    for (int k = lane_id(); k < HSZ; k += 32) T.hash[k] = 0;
    __syncwarp();
}

__device__ __forceinline__ void release_locks(WTab& T, int32_t nt, const Lvl& L) {
    // every lane publishes its own writes (prices, path) before any lock drops
    __threadfence();
    __syncwarp();
    for (int e = lane_id(); e < nt; e += 32)
        if (T.st[e] & kLocked) atomicExch(L.lock + T.col[e], 0);
    __syncwarp();
}

// Dense re-scan of row r at base distance db (= d_r + pi_r): its 32 nearest
// columns not yet scanned join the search; returns the row's new horizon.
__device__ int64_t deep_relax(WTab& T, int32_t& nt, const Lvl& L, int32_t r, int64_t db, bool& ok) {
    const wt_t* Ar = rowp(L, r);
    uint64_t mine, bound;
    warp_top32(L.m, [&](int32_t j) -> uint64_t {
        const int32_t e = hfind(T, j);
        if (e >= 0 && (T.st[e] & kScanned)) return kNoKey;
        return mkkey(db + __ldcg(L.p + j) - (int64_t)__ldg(Ar + j), j, &L.cnt->errors);
    }, mine, bound);
    const int32_t c = mine == kNoKey ? -1 : key_idx(mine);
    int64_t pc = 0, nd = 0;
    if (c >= 0) {
        pc = ldv64(L.p + c);
        nd = db + pc - (int64_t)__ldg(Ar + c);
    }
    ok = tab_relax(T, nt, L, c, nd, pc, r);
    return bound == kNoKey ? kInf : key_val(bound);
}

// Outcome of one search.
enum { kDone = 0, kConflict = 1, kTooBig = 2 };

__device__ int search(WTab& T, const Lvl& L, int32_t s, int32_t me, unsigned long long& steps_out,
                      unsigned long long& deep_out) {
    const int lane = lane_id();
    tab_clear(T);
    int32_t nt = 0;
    // source profit from its record; re-scan when the record no longer bounds the row
    int32_t c = __ldcg(L.cj + (int64_t)s * KC + lane);
    int64_t a = __ldcg(L.ca + (int64_t)s * KC + lane);
    int64_t pc = c >= 0 ? ldv64(L.p + c) : 0;
    int64_t pis = wmax64s(c >= 0 ? a - pc : -kInf);
    int64_t taus = __ldcg(L.tau + s);
    if (pis < taus) {
        refresh_row(L, s);
        atomicAdd(&L.cnt->refresh, 1ull);
        c = __ldcg(L.cj + (int64_t)s * KC + lane);
        a = __ldcg(L.ca + (int64_t)s * KC + lane);
        pc = c >= 0 ? ldv64(L.p + c) : 0;
        pis = wmax64s(c >= 0 ? a - pc : -kInf);
        taus = __ldcg(L.tau + s);
    }
    tab_relax(T, nt, L, c, pis + pc - a, pc, s);
    int64_t hsrc = pis - taus;
    int64_t H = hsrc;
    int steps = 0, deeps = 0;
    int result = kTooBig;
    int32_t jf = -1, ef = -1;
    int64_t D = 0;
    while (true) {
        // pop the nearest open entry (free columns first on ties)
        uint64_t best = kNoKey;
        for (int e = lane; e < nt; e += 32) {
            const uint8_t f = T.st[e];
            if (f & kScanned) continue;
            const int64_t d = T.dist[e];
            const uint64_t k = ((uint64_t)(d < kDistLim ? d : kDistLim - 1) << kSH) | ((f & kFreeHint) ? 0u : kFreeBit) | (uint32_t)e;
            best = k < best ? k : best;
        }
        best = wmin64(best);
        const int64_t dmin = best == kNoKey ? kInf : (int64_t)(best >> kSH);
        if (dmin > H) {
            // horizon: re-scan every tree row whose bound is below dmin
            bool ok = true;
            if (hsrc < dmin) {
                if (++deeps > L.deep_budget) { result = kTooBig; break; }
                hsrc = deep_relax(T, nt, L, s, pis, ok);
            }
            int64_t nh = hsrc;
            for (int e0 = 0; e0 < nt && ok; e0 += 32) {
                const int e = e0 + lane;
                const bool cand = e < nt && (T.st[e] & kScanned) && T.hor[e] < dmin;
                unsigned bal = __ballot_sync(0xffffffffu, cand);
                while (bal && ok) {
                    const int src = __ffs(bal) - 1;
                    bal &= bal - 1;
                    if (++deeps > L.deep_budget) { ok = false; break; }
                    const int ee = e0 + src;
                    const int32_t r = T.row[ee];
                    const int64_t pir = (int64_t)__ldg(rowp(L, r) + T.col[ee]) - T.snap[ee];
                    const int64_t h = deep_relax(T, nt, L, r, T.dist[ee] + pir, ok);
                    if (lane == 0) T.hor[ee] = h;
                    __syncwarp();
                }
            }
            if (!ok) { result = kTooBig; break; }
            for (int e = lane; e < nt; e += 32)
                if ((T.st[e] & kScanned) && T.hor[e] < nh) nh = T.hor[e];
            H = wmin64s(nh);
            if (best == kNoKey && H >= kInf) {
                // no open entry and nothing left to re-scan: cannot happen on a complete graph
                atomicOr(&L.cnt->errors, kErrNoPath);
                result = kTooBig;
                break;
            }
            continue;
        }
        const int32_t e = (int32_t)(best & kIdxMask);
        const int32_t cc = T.col[e];
        // lock the column (validated price, current owner)
        int32_t ok = 1;
        int64_t pnow = 0;
        int32_t own = -1;
        if (lane == 0) {
            if (!(T.st[e] & kLocked)) {
                if (atomicCAS(L.lock + cc, 0, me) != 0) ok = 0;
                else { T.st[e] |= kLocked; __threadfence(); }
            }
            if (ok) { pnow = ldv64(L.p + cc); own = ldv32(L.roc + cc); }
        }
        ok = __shfl_sync(0xffffffffu, ok, 0);
        if (!ok) { result = kConflict; break; }
        pnow = __shfl_sync(0xffffffffu, pnow, 0);
        own = __shfl_sync(0xffffffffu, own, 0);
        __syncwarp();
        if (pnow != T.snap[e]) {
            // raised since it was relaxed: re-queue at its true distance
            if (lane == 0) { T.dist[e] += pnow - T.snap[e]; T.snap[e] = pnow; }
            __syncwarp();
            continue;
        }
        if (own < 0) { jf = cc; ef = e; D = dmin; result = kDone; break; }
        if (++steps > L.step_budget) { result = kTooBig; break; }
        const int64_t pir = (int64_t)__ldg(rowp(L, own) + cc) - pnow;
        if (lane == 0) { T.st[e] |= kScanned; T.row[e] = own; }
        __syncwarp();
        const int32_t c2 = __ldcg(L.cj + (int64_t)own * KC + lane);
        const int64_t a2 = __ldcg(L.ca + (int64_t)own * KC + lane);
        const int64_t p2 = c2 >= 0 ? ldv64(L.p + c2) : 0;
        if (!tab_relax(T, nt, L, c2, dmin + pir + p2 - a2, p2, own)) { result = kTooBig; break; }
        const int64_t h = dmin + pir - __ldcg(L.tau + own);
        if (lane == 0) T.hor[e] = h;
        __syncwarp();
        H = h < H ? h : H;
    }
    steps_out += (unsigned long long)steps;
    deep_out += (unsigned long long)deeps;
    if (result != kDone) {
        release_locks(T, nt, L);
        return result;
    }
    // dual update on the scanned (locked) columns, then the path
    for (int k = lane; k < nt; k += 32)
        if ((T.st[k] & kScanned)) L.p[T.col[k]] = T.snap[k] + (D - T.dist[k]);
    __syncwarp();
    if (lane == 0) {
        int32_t j = jf, ej = ef;
        while (true) {
            const int32_t i = T.pred[ej];
            // cor[i] was written by whichever search last moved row i (any SM):
            // read it past the non-coherent L1
            const int32_t jn = (i == s) ? -1 : ldv32(L.cor + i);
            L.roc[j] = i;
            L.cor[i] = j;
            if (i == s) break;
            j = jn;
            ej = hfind(T, j);
        }
    }
    __syncwarp();
    release_locks(T, nt, L);
    return kDone;
}

__global__ void __launch_bounds__(PWARPS * 32) ssp_parallel_kernel(Lvl L, int32_t serial) {
    extern __shared__ __align__(16) unsigned char smem[];
    if (serial && (blockIdx.x > 0 || threadIdx.x >= 32)) return;   // debugging: one search at a time
    WTab& T = reinterpret_cast<WTab*>(smem)[threadIdx.x >> 5];
    const int32_t me = (int32_t)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5) + 1;
    unsigned long long steps = 0, deep = 0, aborts = 0, augs = 0, over = 0;
    while (true) {
        int32_t k = 0;
        if (lane_id() == 0) k = atomicAdd(&L.cnt->qhead, 1);
        k = __shfl_sync(0xffffffffu, k, 0);
        if (k >= L.nin) break;
        const int32_t s = L.in[k];
        const int r = search(T, L, s, me, steps, deep);
        if (r == kDone) { ++augs; continue; }
        if (lane_id() == 0) {
            if (r == kConflict && ++L.tries[s] <= MAX_TRIES) {
                L.retry[atomicAdd(&L.cnt->nretry, 1)] = s;
                ++aborts;
            } else {
                L.defer[atomicAdd(&L.cnt->ndefer, 1)] = s;
                ++over;
            }
        }
        __syncwarp();
    }
    if (lane_id() == 0) {
        atomicAdd(&L.cnt->steps, steps);
        atomicAdd(&L.cnt->deep, deep);
        atomicAdd(&L.cnt->aborts, aborts);
        atomicAdd(&L.cnt->augs, augs);
        atomicAdd(&L.cnt->overflow, over);
    }
}

// ---------------------------------------------------------------------------
// exclusive mode: one warp, one search at a time, tables indexed by column
// (shared memory when they fit, else global scratch)
// ---------------------------------------------------------------------------

enum : uint8_t { kXTouched = 1, kXScanned = 2, kXFree = 4 };

// Per-column tables (shared memory when 17 m bytes + the open list fit):
// dist, pred, flag, and for scanned columns the horizon gap of their row
// (h = dist + gap, clamped to int32; INT32_MAX = beyond any distance).
struct XTab {
    int32_t* ocol;    // open list
    int32_t ocap;
    int64_t* dist;
    int32_t* pred;
    int32_t* gap;
    uint8_t* flag;
    int32_t nopen;
};

// finite gaps saturate at INT32_MAX - 1 (a lower horizon only re-scans earlier);
// INT32_MAX means "no column outside the record"
__device__ __forceinline__ int32_t clamp_gap(int64_t g) {
    if (g >= kInf / 2) return INT32_MAX;
    return g >= INT32_MAX - 1 ? INT32_MAX - 1 : (int32_t)(g < 0 ? 0 : g);
}

__device__ __forceinline__ bool x_relax(XTab& X, const Lvl& L, int32_t c, int64_t nd, int32_t i) {
    bool need = false;
    if (c >= 0) {
        const uint8_t f = X.flag[c];
        if (f & kXTouched) {
            if (!(f & kXScanned) && nd < X.dist[c]) { X.dist[c] = nd; X.pred[c] = i; }
        } else {
            need = true;
        }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, need);
    const int cnt = __popc(bal);
    if (X.nopen + cnt > X.ocap) { if (lane_id() == 0) atomicOr(&L.cnt->errors, kErrOpenCap); return false; }
    if (need) {
        const int pos = X.nopen + __popc(bal & ((1u << lane_id()) - 1u));
        X.ocol[pos] = c;
        X.dist[c] = nd;
        X.pred[c] = i;
        X.flag[c] = kXTouched | (__ldcg(L.roc + c) < 0 ? kXFree : 0);
    }
    X.nopen += cnt;
    __syncwarp();
    return true;
}

// Dense re-scan of row r at base db (excluding scanned columns): every column
// nearer than `thr` joins the search; the row's new horizon is thr.  Callers
// double the row's reach on each re-scan, so a row is re-scanned O(log) times.
__device__ int64_t x_deep(XTab& X, const Lvl& L, int32_t r, int64_t db, int64_t thr, bool& ok) {
    const wt_t* Ar = rowp(L, r);
    constexpr int U = 8;
    for (int32_t j0 = 0; j0 < L.m && ok; j0 += 32 * U) {
        int64_t nd[U];
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t j = j0 + u * 32 + lane_id();
            nd[u] = j < L.m ? db + __ldcg(L.p + j) - (int64_t)__ldg(Ar + j) : kInf;
        }
#pragma unroll
        for (int u = 0; u < U; ++u) {
            const int32_t j = j0 + u * 32 + lane_id();
            const bool take = nd[u] < thr && !(X.flag[j < L.m ? j : 0] & kXScanned) && j < L.m;
            if (__any_sync(0xffffffffu, take)) ok = x_relax(X, L, take ? j : -1, nd[u], r) && ok;
        }
    }
    return thr;
}

__global__ void __launch_bounds__(32, 1) ssp_exclusive_kernel(Lvl L, int32_t ndef, int32_t use_smem, int32_t ocap) {
    extern __shared__ __align__(16) unsigned char smem[];
    const int lane = lane_id();
    const int32_t m = L.m;
    XTab X;
    if (use_smem) {
        X.dist = reinterpret_cast<int64_t*>(smem);
        X.pred = reinterpret_cast<int32_t*>(X.dist + m);
        X.gap = X.pred + m;
        X.ocol = X.gap + m;
        X.flag = reinterpret_cast<uint8_t*>(X.ocol + ocap);
    } else {
        X.dist = L.xdist;
        X.pred = L.xpred;
        X.gap = L.xgap;
        X.ocol = L.xscol;
        X.flag = reinterpret_cast<uint8_t*>(L.xstamp);
    }
    X.ocap = ocap;
    for (int32_t j = lane; j < m; j += 32) X.flag[j] = 0;
    __syncwarp();
    unsigned long long steps = 0, deeps = 0;
    long long cyc[4] = {0, 0, 0, 0};
    for (int32_t q = 0; q < ndef; ++q) {
        const int32_t s = L.defer[q];
        X.nopen = 0;
        int32_t c = __ldcg(L.cj + (int64_t)s * KC + lane);
        int64_t pis = wmax64s(c >= 0 ? (int64_t)__ldcg(L.ca + (int64_t)s * KC + lane) - __ldcg(L.p + c) : -kInf);
        if (pis < __ldcg(L.tau + s)) {
            refresh_row(L, s);
            c = __ldcg(L.cj + (int64_t)s * KC + lane);
            pis = wmax64s(c >= 0 ? (int64_t)__ldcg(L.ca + (int64_t)s * KC + lane) - __ldcg(L.p + c) : -kInf);
        }
        bool ok = x_relax(X, L, c, c >= 0 ? pis + __ldcg(L.p + c) - __ldcg(L.ca + (int64_t)s * KC + lane) : 0, s);
        int64_t hsrc = pis - __ldcg(L.tau + s);
        int64_t H = hsrc;
        int32_t jf = -1;
        int64_t D = 0;
        while (ok) {
            long long c0 = clock64();
            uint64_t best = kNoKey;
            for (int k = lane; k < X.nopen; k += 32) {
                const int32_t cc = X.ocol[k];
                const int64_t d = X.dist[cc];
                const uint64_t key = ((uint64_t)(d < kDistLim ? d : kDistLim - 1) << kSH) |
                                     ((X.flag[cc] & kXFree) ? 0u : kFreeBit) | (uint32_t)k;
                best = key < best ? key : best;
            }
            best = wmin64(best);
            const int64_t dmin = best == kNoKey ? kInf : (int64_t)(best >> kSH);
            { const long long c1 = clock64(); cyc[0] += c1 - c0; c0 = c1; }
            if (dmin > H) {
                // horizon: re-scan the source and every tree row whose bound is below dmin
                ++deeps;
                // new reach: double the distance already covered (everything when nothing is open)
                const int64_t reach_src = dmin >= kInf ? kInf : dmin + (dmin > 0 ? dmin : 1);
                if (hsrc < dmin) hsrc = x_deep(X, L, s, pis, reach_src, ok);
                int64_t nh = hsrc;
                for (int32_t j0 = 0; j0 < m && ok; j0 += 32) {
                    const int32_t j = j0 + lane;
                    bool cand = false;
                    int64_t h = kInf;
                    if (j < m && (X.flag[j] & kXScanned)) {
                        const int32_t g = X.gap[j];
                        h = g == INT32_MAX ? kInf : X.dist[j] + g;
                        cand = h < dmin;
                    }
                    unsigned bal = __ballot_sync(0xffffffffu, cand);
                    while (bal && ok) {
                        const int32_t col = j0 + __ffs(bal) - 1;
                        bal &= bal - 1;
                        const int32_t r = __ldcg(L.roc + col);
                        const int64_t dc = X.dist[col];
                        const int64_t pir = (int64_t)__ldg(rowp(L, r) + col) - __ldcg(L.p + col);
                        int64_t hn = x_deep(X, L, r, dc + pir, dmin >= kInf ? kInf : dmin + (dmin - dc > 0 ? dmin - dc : 1), ok);
                        if (lane == 0) X.gap[col] = hn >= kInf ? INT32_MAX : clamp_gap(hn - dc);
                        if (hn < kInf) hn = dc + (int64_t)X.gap[col];   // the stored (possibly saturated) bound
                        __syncwarp();
                        if (lane == col - j0) h = hn;
                    }
                    nh = h < nh ? h : nh;
                }
                H = wmin64s(nh);
                if (best == kNoKey && X.nopen == 0) { if (lane == 0) atomicOr(&L.cnt->errors, kErrNoPath); ok = false; }
                cyc[1] += clock64() - c0;
                continue;
            }
            const int32_t k = (int32_t)(best & kIdxMask);
            const int32_t cc = X.ocol[k];
            __syncwarp();
            if (lane == 0) {
                X.ocol[k] = X.ocol[X.nopen - 1];
                X.flag[cc] |= kXScanned;
            }
            X.nopen -= 1;
            __syncwarp();
            const int32_t own = __ldcg(L.roc + cc);
            if (own < 0) { jf = cc; D = dmin; break; }
            ++steps;
            const int64_t pir = (int64_t)__ldg(rowp(L, own) + cc) - __ldcg(L.p + cc);
            const int32_t c2 = __ldcg(L.cj + (int64_t)own * KC + lane);
            ok = x_relax(X, L, c2, c2 >= 0 ? dmin + pir + __ldcg(L.p + c2) - __ldcg(L.ca + (int64_t)own * KC + lane) : 0, own);
            const int64_t tg = pir - __ldcg(L.tau + own);
            if (lane == 0) X.gap[cc] = clamp_gap(tg);
            const int64_t h = tg >= kInf / 2 ? kInf : dmin + (tg >= INT32_MAX - 1 ? (int64_t)INT32_MAX - 1 : tg);
            H = h < H ? h : H;
            __syncwarp();
            cyc[2] += clock64() - c0;
        }
        if (!ok) break;
        const long long ca0 = clock64();
        // dual update on the scanned columns, augment, clear the flags
        for (int32_t j = lane; j < m; j += 32) {
            const uint8_t f = X.flag[j];
            if ((f & kXScanned) && j != jf) L.p[j] = __ldcg(L.p + j) + (D - X.dist[j]);
        }
        __syncwarp();
        if (lane == 0) {
            int32_t j = jf;
            while (true) {
                const int32_t i = X.pred[j];
                const int32_t jn = (i == s) ? -1 : __ldcg(L.cor + i);
                L.roc[j] = i;
                L.cor[i] = j;
                if (i == s) break;
                j = jn;
            }
        }
        __syncwarp();
        for (int32_t j = lane; j < m; j += 32) X.flag[j] = 0;
        __syncwarp();
        cyc[3] += clock64() - ca0;
    }
    if (lane == 0) {
        atomicAdd(&L.cnt->xsteps, steps);
        atomicAdd(&L.cnt->xdeep, deeps);
        for (int k = 0; k < 4; ++k) atomicAdd((unsigned long long*)&L.cnt->xcyc[k], (unsigned long long)cyc[k]);
    }
}

// ---------------------------------------------------------------------------
// dense exclusive mode: the long searches, one CTA of 1024 threads, a classic
// dense Dijkstra (every scanned row relaxes all m columns once).  Prices are
// constant during a search and live in shared memory with the distances,
// predecessors and flags (21 bytes per column); relax and argmin are fused
// into one pass per step.
// ---------------------------------------------------------------------------

constexpr int DTHREADS = 1024;
constexpr int DCOLS = 11;            // columns per thread: m <= 11264 (21 bytes of shared memory each)

// block-wide min; red holds two 33-entry buffers used alternately, so a
// step needs only the two barriers inside
__device__ __forceinline__ uint64_t block_min64(uint64_t v, uint64_t* red, int& par) {
    v = wmin64(v);
    uint64_t* R = red + par * 33;
    par ^= 1;
    const int w = threadIdx.x >> 5;
    if (lane_id() == 0) R[w] = v;
    __syncthreads();
    if (w == 0) {
        uint64_t x = lane_id() < (DTHREADS / 32) ? R[lane_id()] : kNoKey;
        x = wmin64(x);
        if (lane_id() == 0) R[32] = x;
    }
    __syncthreads();
    return R[32];
}

__global__ void __launch_bounds__(DTHREADS, 1) ssp_dense_kernel(Lvl L, int32_t ndef) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint64_t red[66];
    const int32_t m = L.m;
    int64_t* d = reinterpret_cast<int64_t*>(smem);
    int64_t* ps = d + m;
    int16_t* pred = reinterpret_cast<int16_t*>(ps + m);
    int16_t* rocs = pred + m;
    uint8_t* fl = reinterpret_cast<uint8_t*>(rocs + m);   // bit0 scanned, bit1 free
    const int tid = threadIdx.x;
    int par = 0;
    unsigned long long steps = 0;
    for (int32_t q = 0; q < ndef; ++q) {
        const int32_t s = L.defer[q];
        const wt_t* As = rowp(L, s);
        uint64_t vmin = kNoKey;   // max value as the min of (2^39 - value)
#pragma unroll
        for (int u = 0; u < DCOLS; ++u) {
            const int32_t j = tid + u * DTHREADS;
            if (j < m) {
                const int64_t pj = __ldcg(L.p + j);
                const int32_t r = __ldcg(L.roc + j);
                ps[j] = pj;
                rocs[j] = (int16_t)r;
                fl[j] = r < 0 ? 2 : 0;
                const uint64_t k = (uint64_t)(kDistLim - ((int64_t)__ldg(As + j) - pj));
                vmin = k < vmin ? k : vmin;
            }
        }
        const int64_t pis = kDistLim - (int64_t)block_min64(vmin, red, par);
        uint64_t best = kNoKey;
#pragma unroll
        for (int u = 0; u < DCOLS; ++u) {
            const int32_t j = tid + u * DTHREADS;
            if (j < m) {
                const int64_t nd = pis + ps[j] - (int64_t)__ldg(As + j);
                d[j] = nd;
                pred[j] = (int16_t)s;
                const uint64_t k = ((uint64_t)nd << kSH) | ((fl[j] & 2) ? 0u : kFreeBit) | (uint32_t)j;
                best = k < best ? k : best;
            }
        }
        best = block_min64(best, red, par);
        int32_t jf;
        int64_t D;
        while (true) {
            const int32_t jm = (int32_t)(best & kIdxMask);
            const int64_t dmin = (int64_t)(best >> kSH);
            if (fl[jm] & 2) { jf = jm; D = dmin; break; }
            const int32_t i = rocs[jm];
            if ((jm & (DTHREADS - 1)) == tid) fl[jm] |= 1;   // only the column's owner thread reads its flag
            const wt_t* Ai = rowp(L, i);
            // the whole row slice and a_i,jm in one batch of loads
            int32_t av[DCOLS];
#pragma unroll
            for (int u = 0; u < DCOLS; ++u) {
                const int32_t j = tid + u * DTHREADS;
                av[u] = j < m ? __ldg(Ai + j) : 0;
            }
            const int64_t base = dmin + (int64_t)__ldg(Ai + jm) - ps[jm];
            best = kNoKey;
#pragma unroll
            for (int u = 0; u < DCOLS; ++u) {
                const int32_t j = tid + u * DTHREADS;
                if (j < m) {
                    const uint8_t f = fl[j];
                    if (!(f & 1)) {
                        int64_t dj = d[j];
                        const int64_t nd = base + ps[j] - (int64_t)av[u];
                        if (nd < dj) { dj = nd; d[j] = nd; pred[j] = (int16_t)i; }
                        const uint64_t k = ((uint64_t)dj << kSH) | ((f & 2) ? 0u : kFreeBit) | (uint32_t)j;
                        best = k < best ? k : best;
                    }
                }
            }
            best = block_min64(best, red, par);
            ++steps;
        }
        // dual update on the scanned columns, then the path (thread 0)
#pragma unroll
        for (int u = 0; u < DCOLS; ++u) {
            const int32_t j = tid + u * DTHREADS;
            if (j < m && (fl[j] & 1)) L.p[j] = ps[j] + (D - d[j]);
        }
        if (tid == 0) {
            int32_t j = jf;
            while (true) {
                const int32_t i = pred[j];
                const int32_t jn = (i == s) ? -1 : __ldcg(L.cor + i);
                L.roc[j] = i;
                L.cor[i] = j;
                if (i == s) break;
                j = jn;
            }
        }
        __threadfence();
        __syncthreads();
    }
    if (tid == 0) atomicAdd(&L.cnt->xsteps, steps);
}

// ---------------------------------------------------------------------------
// cluster modes for the long searches: the dense Dijkstra spread over a
// thread-block cluster of CL CTAs (CL SMs), CTA r owning columns
// [r*mc, (r+1)*mc).  Two exchanges of the per-step minimum:
//  * push (ssp_rkey_kernel, m <= CL * 2048): prices and owners are replicated
//    in every CTA; lanes 0..CL-1 of every warp push the warp's minimum with
//    st.async into slot [rank*32 + warp] of each CTA, completing bytes on
//    that CTA's mbarrier; warp 0 of each CTA waits, reduces, re-arms.
//  * barrier (ssp_slice_kernel, larger m): each CTA keeps only its slice;
//    warps publish minima in their CTA's slots, one barrier.cluster, warp 0
//    of every CTA reads the CL*32 slots through DSMEM and fetches the
//    winner's owner / price from the CTA that holds it.
// ---------------------------------------------------------------------------

constexpr int CL = 8;
constexpr int CTHREADS = 1024;
constexpr int CCOLS = 8;            // local columns per thread: m <= CL * CTHREADS * CCOLS = 65536
constexpr int CBYTES = 25;          // shared bytes per local column: d, p (int64), pred, owner (int32), flag

struct CShared {
    uint64_t slots[2][32];   // per-warp minima, double-buffered by step parity
    uint64_t bkey[2];        // cluster-wide minimum
    int32_t bown[2];         // its column's owner row (-1 = free column)
    int64_t bprice[2];       // its column's price
};

// Barrier exchange: cluster-wide minimum key; warp 0 also reads the winning
// column's owner row and price from the CTA that holds it (DSMEM) before the
// CTA barrier, so every thread gets them without another round trip.
template <int CLS>
__device__ __forceinline__ uint64_t cluster_min_fetch(uint64_t v, CShared& S, int& par, cg::cluster_group& cluster,
                                                      int32_t mc, int32_t* rocs, int64_t* ps, int32_t& own, int64_t& pw) {
    v = wmin64(v);
    const int w = threadIdx.x >> 5;
    if (lane_id() == 0) S.slots[par][w] = v;
    cluster.sync();
    if (w == 0) {
        uint64_t x = kNoKey;
#pragma unroll
        for (int r = 0; r < CLS; ++r) {
            const uint64_t* rs = cluster.map_shared_rank(&S.slots[par][0], r);
            const uint64_t y = rs[lane_id()];
            x = y < x ? y : x;
        }
        x = wmin64(x);
        if (lane_id() == 0) {
            S.bkey[par] = x;
            if (x != kNoKey) {
                const int32_t j = (int32_t)(x & kIdxMask);
                const int owner = j / mc;
                S.bown[par] = cluster.map_shared_rank(rocs, owner)[j - owner * mc];
                S.bprice[par] = cluster.map_shared_rank(ps, owner)[j - owner * mc];
            }
        }
    }
    __syncthreads();
    const uint64_t r = S.bkey[par];
    own = S.bown[par];
    pw = S.bprice[par];
    par ^= 1;
    return r;
}

// Push exchange buffers: per-warp minima from every CTA, double-buffered by
// step parity.  A CTA can only push step k+2 into a buffer after receiving
// every CTA's step k+1, which each CTA sends only after it has consumed step
// k from that buffer, so no slot is overwritten early.
template <int CLS>
struct CPush {
    uint64_t slots[2][CLS * 32];
    uint64_t bar[2];
};

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int CLS, int NW>
__device__ __forceinline__ void cpush_init(CPush<CLS>& P) {
    if (threadIdx.x == 0) {
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const uint32_t a = smem_u32(&P.bar[b]);
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(a) : "memory");
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
        for (int b = 0; b < 2; ++b) {
            const uint32_t a = smem_u32(&P.bar[b]);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(a), "r"(CLS * NW * 8) : "memory");
        }
    }
}

// Push exchange: cluster-wide minimum key.  cand2 (warp 0's lanes): per lane
// the best key of its slot column other than the winner -- its warp minimum
// is the runner-up, whose row the caller prefetches.
template <int CLS, int NW>
__device__ __forceinline__ uint64_t cluster_min_push(uint64_t v, CShared& S, CPush<CLS>& P, int& par, uint32_t& ph, int rank,
                                                     uint64_t& cand2) {
    v = wmin64(v);
    const int w = threadIdx.x >> 5, ln = lane_id();
    const uint32_t lb = smem_u32(&P.bar[par]);
    if (ln < CLS) {
        const uint32_t la = smem_u32(&P.slots[par][rank * 32 + w]);
        uint32_t ra, rb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(ln));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(lb), "r"(ln));
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(ra), "l"(v), "r"(rb)
                     : "memory");
    }
    if (w == 0) {
        const uint32_t parity = (ph >> par) & 1u;
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(lb), "r"(parity)
                : "memory");
        }
        uint64_t x = kNoKey, x2 = kNoKey;   // this lane's smallest and second smallest of its CLS slots
#pragma unroll
        for (int r = 0; r < CLS; ++r) {
            const uint64_t y = ln < NW ? P.slots[par][r * 32 + ln] : kNoKey;
            x2 = y < x2 ? y : x2;
            if (y < x) { x2 = x; x = y; }
        }
        const uint64_t xl = x;
        x = wmin64(x);
        cand2 = xl == x ? x2 : xl;
        if (ln == 0) {
            S.bkey[par] = x;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(lb), "r"(CLS * NW * 8) : "memory");
        }
    }
    ph ^= 1u << par;
    __syncthreads();
    const uint64_t r = S.bkey[par];
    par ^= 1;
    return r;
}

// Tie batching (the register-key kernel): warp minima at the winner's
// distance are popped in the same step -- Dijkstra may settle columns of equal
// distance in any order, and a relaxation from one of them cannot take another
// below that distance.  Only matched winners batch (a free winner ends the
// search; free columns sort first, so none ties with a matched winner).
#ifndef MUX_TIE_MAX
#define MUX_TIE_MAX 2
#endif
constexpr int kTieMax = MUX_TIE_MAX;
struct CTies {
    uint64_t key[2][kTieMax];
    int32_t n[2];
};

// cluster_min_push that also returns up to kTieMax further warp minima at the
// winner's distance (tk[0..nt)); cand2 skips every key at that distance.
template <int CLS, int NW>
__device__ __forceinline__ uint64_t cluster_min_push_ties(uint64_t v, CShared& S, CPush<CLS>& P, CTies& T, int& par,
                                                          uint32_t& ph, int rank, uint64_t& cand2, uint64_t (&tk)[kTieMax],
                                                          int& nt, bool ties, unsigned long long* tw = nullptr) {
    const long long tw0 = tw ? clock64() : 0;
    v = wmin64(v);
    const int w = threadIdx.x >> 5, ln = lane_id();
    const uint32_t lb = smem_u32(&P.bar[par]);
    if (ln < CLS) {
        const uint32_t la = smem_u32(&P.slots[par][rank * 32 + w]);
        uint32_t ra, rb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(ln));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(lb), "r"(ln));
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.b64 [%0], %1, [%2];" ::"r"(ra), "l"(v), "r"(rb)
                     : "memory");
    }
    if (w == 0) {
        const uint32_t parity = (ph >> par) & 1u;
        uint32_t done = 0;
        while (!done) {
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(lb), "r"(parity)
                : "memory");
        }
        if (tw) *tw += clock64() - tw0;
        // the CLS x NW warp minima spread over all 32 lanes (KPL each): short
        // dependency chains for the minimum and the tie list
        constexpr int TOT = CLS * NW, KPL = (TOT + 31) / 32;
        uint64_t ys[KPL];
        uint64_t x = kNoKey;
#pragma unroll
        for (int k = 0; k < KPL; ++k) {
            const int e = ln + 32 * k;
            ys[k] = e < TOT ? P.slots[par][(e / NW) * 32 + (e % NW)] : kNoKey;
            x = ys[k] < x ? ys[k] : x;
        }
        x = wmin64(x);
        const uint64_t dhi = x >> kSH;
        const bool batch = ties && (x & kFreeBit) != 0 && x != kNoKey;
        const unsigned lt = (1u << ln) - 1u;
        uint64_t c2 = kNoKey;
        int cnt = 0;
#pragma unroll
        for (int k = 0; k < KPL; ++k) {
            const uint64_t y = ys[k];
            const bool same = (y >> kSH) == dhi;
            const bool tie = batch && same && y != x;
            const unsigned msk = __ballot_sync(~0u, tie);
            if (tie) {
                const int pos = cnt + __popc(msk & lt);
                if (pos < kTieMax) T.key[par][pos] = y;
            }
            cnt += __popc(msk);
            if (ties ? !same : y != x) c2 = y < c2 ? y : c2;
        }
        cand2 = c2;
        if (ln == 0) {
            S.bkey[par] = x;
            T.n[par] = cnt < kTieMax ? cnt : kTieMax;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(lb), "r"(CLS * NW * 8) : "memory");
        }
    }
    ph ^= 1u << par;
    __syncthreads();
    const uint64_t r = S.bkey[par];
    nt = ties ? T.n[par] : 0;
    uint64_t raw[kTieMax];
#pragma unroll
    for (int t = 0; t < kTieMax; ++t) raw[t] = T.key[par][t];   // independent of nt: loads in parallel
#pragma unroll
    for (int t = 0; t < kTieMax; ++t) tk[t] = t < nt ? raw[t] : kNoKey;
    par ^= 1;
    return r;
}

// Sliced long-path kernel (m too large to replicate prices and owners in
// every CTA: the 10k x 40k rounds).  Per local column: distance, price,
// predecessor, owner, scanned flag in shared memory (25 bytes).
template <int CC, int CLS>
__global__ void __cluster_dims__(CLS, 1, 1) __launch_bounds__(CTHREADS, 1)
ssp_slice_kernel(Lvl L, int32_t ndef, int32_t pop_limit) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ CShared S;
    cg::cluster_group cluster = cg::this_cluster();
    constexpr int NT = CTHREADS;
    const int32_t m = L.m;
    const int32_t mc = (m + CLS - 1) / CLS;
    const int rank = (int)cluster.block_rank();
    const int32_t c0 = rank * mc;
    const int32_t nloc = max(0, min(mc, m - c0));
    int64_t* d = reinterpret_cast<int64_t*>(smem);
    int64_t* ps = d + mc;
    int32_t* pred = reinterpret_cast<int32_t*>(ps + mc);
    int32_t* rocs = pred + mc;
    uint8_t* fl = reinterpret_cast<uint8_t*>(rocs + mc);       // bit0 scanned
    const int tid = threadIdx.x;
    int par = 0;
    unsigned long long steps = 0;
    if (tid < 64) S.slots[tid >> 5][tid & 31] = kNoKey;
    __syncthreads();
    for (int32_t q = 0; q < ndef; ++q) {
        const int32_t s = L.defer[q];
        const wt_t* As = rowp(L, s);
        // one reduction finds both the source's profit (the largest a_sj - p_j)
        // and the first pop (that column, at distance 0; free columns first)
        uint64_t vmin = kNoKey;
#pragma unroll
        for (int u = 0; u < CC; ++u) {
            const int32_t jj = tid + u * NT;
            if (jj < nloc) {
                const int64_t pj = __ldcg(L.p + c0 + jj);
                const int32_t r = __ldcg(L.roc + c0 + jj);
                ps[jj] = pj;
                rocs[jj] = r;
                fl[jj] = 0;
                const int64_t v = pj - (int64_t)__ldg(As + c0 + jj);   // = -(a_sj - p_j)
                const uint64_t k = ((uint64_t)(v + kDistLim) << kSH) | (r < 0 ? 0u : kFreeBit) | (uint32_t)(c0 + jj);
                vmin = k < vmin ? k : vmin;
            }
        }
        int32_t i;
        int64_t pjm;
        const uint64_t k0 = cluster_min_fetch<CLS>(vmin, S, par, cluster, mc, rocs, ps, i, pjm);
        const int64_t pis = -((int64_t)(k0 >> kSH) - kDistLim);
        uint64_t best = k0 & kLowMask;   // distance 0, same column and free bit
#pragma unroll
        for (int u = 0; u < CC; ++u) {
            const int32_t jj = tid + u * NT;
            if (jj < nloc) {
                d[jj] = pis + ps[jj] - (int64_t)__ldg(As + c0 + jj);
                pred[jj] = s;
            }
        }
        int32_t jf;
        int64_t D;
        int32_t pops = 0;
        bool abandon = false;
        while (true) {
            const int32_t jm = (int32_t)(best & kIdxMask);
            const int64_t dmin = (int64_t)(best >> kSH);
            if (i < 0) { jf = jm; D = dmin; break; }
            // coarse levels: a search past the pop limit is abandoned (row stays free)
            if (pop_limit > 0 && ++pops > pop_limit) { abandon = true; jf = -1; D = 0; break; }
            if (jm >= c0 && jm < c0 + nloc && ((jm - c0) & (NT - 1)) == tid) fl[jm - c0] |= 1;
            const wt_t* Ai = rowp(L, i);
            wt_t av[CC];
#pragma unroll
            for (int u = 0; u < CC; ++u) {
                const int32_t jj = tid + u * NT;
                av[u] = jj < nloc ? __ldg(Ai + c0 + jj) : 0;
            }
            const int64_t base = dmin + (int64_t)__ldg(Ai + jm) - pjm;
            best = kNoKey;
#pragma unroll
            for (int u = 0; u < CC; ++u) {
                const int32_t jj = tid + u * NT;
                if (jj < nloc && !(fl[jj] & 1)) {
                    int64_t dj = d[jj];
                    const int64_t nd = base + ps[jj] - (int64_t)av[u];
                    if (nd < dj) { dj = nd; d[jj] = nd; pred[jj] = i; }
                    const uint64_t k = ((uint64_t)dj << kSH) | (rocs[jj] < 0 ? 0u : kFreeBit) | (uint32_t)(c0 + jj);
                    best = k < best ? k : best;
                }
            }
            best = cluster_min_fetch<CLS>(best, S, par, cluster, mc, rocs, ps, i, pjm);
            ++steps;
        }
        if (abandon) { cluster.sync(); continue; }
        // dual update on the local scanned columns
#pragma unroll
        for (int u = 0; u < CC; ++u) {
            const int32_t jj = tid + u * NT;
            if (jj < nloc && (fl[jj] & 1)) L.p[c0 + jj] = ps[jj] + (D - d[jj]);
        }
        // the path: predecessors live in their owners' shared memory
        if (rank == 0 && tid == 0) {
            int32_t j = jf;
            while (true) {
                const int owner = j / mc;
                const int32_t ii = cluster.map_shared_rank(pred, owner)[j - owner * mc];
                const int32_t jn = (ii == s) ? -1 : __ldcg(L.cor + ii);
                L.roc[j] = ii;
                L.cor[ii] = j;
                if (ii == s) break;
                j = jn;
            }
        }
        __threadfence();
        cluster.sync();
    }
    if (rank == 0 && tid == 0) atomicAdd(&L.cnt->xsteps, steps);
}

// ---------------------------------------------------------------------------
// register-key long-path kernel (the default for m <= CL * 512 * 4): the same
// cluster Dijkstra as ssp_cluster_kernel's replicated push mode, with each
// thread's tentative distances held in REGISTERS as ready-made sort keys.
//
// Thread t of CTA r owns columns c0 + t + u * NT (u < CC) for the whole
// search, so their state never needs shared memory:
//   kd[u] = (d_j << kSH) | low_j           tentative distance as a sort key
//   pk[u] = (p_j << kSH) | low_j           price (constant during a search)
//   low_j = (owned ? 1 << 23 : 0) | j     free columns first on ties, then lowest j
// and relaxing row i at base distance b is one 64-bit add-subtract-compare:
//   nk = (b << kSH) + pk[u] - (a_ij << kSH) = ((b + p_j - a_ij) << kSH) | low_j.
// A popped column gets bit 63 in both words: its nk then carries bit 63 and is
// never below kd (nd >= the popped distance), and it drops out of the minimum.
// Only the predecessor row stays in shared memory (the augmenting-path walk
// reads it across the cluster).
// ---------------------------------------------------------------------------

constexpr uint64_t kTop = 1ull << 63;
#ifndef RPF_LANES
#define RPF_LANES 2   // lanes of the rank-neighbour prefetch (two per distance: up and down)
#endif

template <int CC, int CLS, int NT>
__global__ void __cluster_dims__(CLS, 1, 1) __launch_bounds__(NT, 1)
ssp_rkey_kernel(Lvl L, int32_t ndef, int32_t pop_limit, int32_t push) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ CShared S;
    __shared__ __align__(16) CPush<CLS> P;
    __shared__ CTies TS;
    cg::cluster_group cluster = cg::this_cluster();
    const int32_t m = L.m;
    const int32_t mc = (m + CLS - 1) / CLS;
    const int rank = (int)cluster.block_rank();
    const int32_t c0 = rank * mc;
    const int32_t nloc = max(0, min(mc, m - c0));
    int64_t* psr = reinterpret_cast<int64_t*>(smem);                          // [m] prices (replicated)
    int32_t* rocr = reinterpret_cast<int32_t*>(psr + m);                      // [m] owners (replicated)
    // CTA 0: colof[i] = the column whose pop brought row i into the tree (its
    // matched column), so the augmenting-path walk stays in shared memory
    int32_t* colof = rocr + ((m + 1) & ~1);                                  // [m] (CTA 0)
    int32_t* pred = colof + ((m + 1) & ~1);                                  // [mc] predecessor rows (local)
    // two row-slice buffers for the runner-up prefetch (TMA bulk copies)
    const int32_t slot_words = ((mc + 8 + 3) & ~3);
    wt_t* rowbuf = reinterpret_cast<wt_t*>((reinterpret_cast<uintptr_t>(pred + mc) + 127) & ~(uintptr_t)127);
    __shared__ __align__(8) uint64_t pfbar[2];
    __shared__ int32_t pfrow[2], pfshift[2];
    __shared__ uint32_t pfpar[2];
    const bool pf = (push & 4) != 0;
    const bool l2pf = (push & 32) != 0;
    const bool ties = (push & 64) != 0;
    uint32_t pfcount[2] = {0, 0};   // tid 0: copies issued per slot
    int cur = 0;
    const int tid = threadIdx.x;
    int par = 0;
    uint32_t ph = 0;
    uint64_t cand2 = kNoKey;
    unsigned long long steps = 0, pfhits = 0, rounds = 0, walk = 0;
    long long wcyc = 0;
    uint64_t tk[kTieMax];
    int nt = 0;
    int32_t rpf_rank = -1, rpf_row = -1;   // rank-neighbour prefetch pipeline (two lanes)
    const bool tm = (push & 16) != 0;
    long long tcyc[3] = {0, 0, 0};
    unsigned long long txt[5] = {0, 0, 0, 0, 0};
    if (tid < 64) S.slots[tid >> 5][tid & 31] = kNoKey;
    if (tid < 2) {
        pfrow[tid] = -1;
        pfshift[tid] = 0;
        pfpar[tid] = 0;
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&pfbar[tid])) : "memory");
    }
    if (tid == 0) asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncthreads();
    cpush_init<CLS, NT / 32>(P);
    cluster.sync();
    for (int32_t q = 0; q < ndef; ++q) {
        const int32_t s = L.defer[q];
        const wt_t* As = rowp(L, s);
        for (int32_t j = tid; j < m; j += NT) {
            psr[j] = __ldcg(L.p + j);
            rocr[j] = __ldcg(L.roc + j);
        }
        __syncthreads();
        uint64_t kd[CC], pk[CC];
        wt_t as[CC];
        // one reduction finds the source's profit (the largest a_sj - p_j) and
        // the first pop (that column at distance 0; free columns first)
        uint64_t vmin = kNoKey;
#pragma unroll
        for (int u = 0; u < CC; ++u) {
            const int32_t jj = tid + u * NT;
            as[u] = jj < nloc ? __ldg(As + c0 + jj) : 0;
        }
#pragma unroll
        for (int u = 0; u < CC; ++u) {
            const int32_t jj = tid + u * NT;
            if (jj < nloc) {
                const int32_t j = c0 + jj;
                const int64_t pj = psr[j];
                if (pj < 0 || pj >= kDistLim) atomicOr(&L.cnt->errors, kErrDist);
                const uint64_t low = (rocr[j] < 0 ? 0u : kFreeBit) | (uint32_t)j;
                pk[u] = ((uint64_t)pj << kSH) | low;
                const uint64_t k = ((uint64_t)(pj - (int64_t)as[u] + kDistLim) << kSH) | low;
                vmin = k < vmin ? k : vmin;
                pred[jj] = s;
            } else {
                pk[u] = kTop;
            }
        }
        const uint64_t k0 = cluster_min_push_ties<CLS, NT / 32>(vmin, S, P, TS, par, ph, rank, cand2, tk, nt, ties);
        const int64_t pis = -((int64_t)(k0 >> kSH) - kDistLim);
#pragma unroll
        for (int u = 0; u < CC; ++u) {
            const int32_t jj = tid + u * NT;
            kd[u] = jj < nloc ? (((uint64_t)pis << kSH) + pk[u] - ((uint64_t)as[u] << kSH)) : kNoKey;
        }
        uint64_t best = k0 & kLowMask;   // distance 0, same column and free bit
#pragma unroll
        for (int t = 0; t < kTieMax; ++t) tk[t] &= kLowMask;   // ties at distance 0
        int32_t jf;
        int64_t D;
        int32_t pops = 0;
        bool abandon = false;
        while (true) {
            const int32_t jm = (int32_t)(best & kIdxMask);
            const int64_t dmin = (int64_t)(best >> kSH);
            const int32_t i = rocr[jm];
            // this step's row loads go out first (a free winner, i < 0, ends the search
            // below; its loads read the zero row); the bookkeeping follows them
            const long long tA = tm ? clock64() : 0;
            const wt_t* Ai = i >= 0 ? rowp(L, i) : L.zrow;
            const int64_t aim = (int64_t)__ldg(Ai + jm);
            wt_t av[CC];
            // the runner-up of the previous step has its slice (being) copied into smem;
            // its barrier is waited on only after every global load of this step is issued
            const bool hit = pf && i >= 0 && pfrow[cur] == i;
            if (!hit) {
#pragma unroll
                for (int u = 0; u < CC; ++u) {
                    const int32_t jj = tid + u * NT;
                    av[u] = jj < nloc ? __ldg(Ai + c0 + jj) : 0;
                }
            }
            // the tied columns' rows (matched: a tie never carries the free flag); their
            // bases are formed at the relaxation so no load result is waited on here
            wt_t avt[kTieMax][CC];
            wt_t aimt[kTieMax];
            int32_t it[kTieMax];
#pragma unroll
            for (int t = 0; t < kTieMax; ++t) {
                if (t < nt) {
                    const int32_t jt = (int32_t)(tk[t] & kIdxMask);
                    it[t] = rocr[jt];
                    const wt_t* At = rowp(L, it[t]);
                    aimt[t] = __ldg(At + jt);
#pragma unroll
                    for (int u = 0; u < CC; ++u) {
                        const int32_t jj = tid + u * NT;
                        avt[t][u] = jj < nloc ? __ldg(At + c0 + jj) : 0;
                    }
                }
            }
            asm volatile("" ::: "memory");
            if (i < 0) { jf = jm; D = dmin; break; }
            if (pop_limit > 0 && (pops += 1 + nt) > pop_limit) { abandon = true; jf = -1; D = 0; break; }
            if (L.rpf > 0 && tid >= NT - RPF_LANES) {
                // two lanes of the last warp, one step per stage: prefetch the row found
                // last step, look up the row rpf ranks away from last step's rank, load
                // this step's rank (each load is consumed a step later, off the critical path)
                if (rpf_row >= 0 && nloc > 0) {
                    const wt_t* src = rowp(L, rpf_row) + c0;
                    const uintptr_t a0 = reinterpret_cast<uintptr_t>(src) & ~(uintptr_t)15;
                    const uintptr_t a1 = (reinterpret_cast<uintptr_t>(src + nloc) + 15) & ~(uintptr_t)15;
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0)) : "memory");
                }
                // lane NT-1-k: distance (k / 2 + 1) * rpf / (RPF_LANES / 2), up for even k, down for odd
                const int kq = NT - 1 - tid;
                const int32_t dist = (int32_t)(((kq >> 1) + 1) * L.rpf / (RPF_LANES / 2));
                const int32_t rr = rpf_rank < 0 ? -1 : rpf_rank + ((kq & 1) ? -dist : dist);
                if (L.rankof) {   // level 0: rows in the caller's order
                    rpf_row = rr >= 0 && rr < m ? __ldcg(L.rowat + rr) : -1;
                    rpf_rank = __ldcg(L.rankof + i);
                } else {          // coarse levels index their rows in key order
                    rpf_row = rr >= 0 && rr < m ? rr : -1;
                    rpf_rank = i;
                }
            }
            if (rank == 0 && tid == 0) {
                colof[i] = jm;
#pragma unroll
                for (int t = 0; t < kTieMax; ++t)
                    if (t < nt) colof[it[t]] = (int32_t)(tk[t] & kIdxMask);
            }
            // runner-up prefetch: warp 0 copies this CTA's slice of the row owning the
            // runner-up column (often the next pop) into the other buffer by TMA
            if (pf && tid < 32) {
                const uint64_t k2 = wmin64(cand2);
                const int nb = cur ^ 1;
                if (tid == 0 && k2 != kNoKey && nloc > 0) {
                    const int32_t i2 = rocr[k2 & kIdxMask];
                    if (i2 >= 0 && i2 != pfrow[nb]) {
                        const uint32_t bar = smem_u32(&pfbar[nb]);
                        if (pfcount[nb] > 0) {
                            // the buffer's previous copy must have landed before it is rewritten
                            const uint32_t parity = (pfcount[nb] - 1) & 1u;
                            uint32_t done = 0;
                            while (!done)
                                asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                                             : "=r"(done) : "r"(bar), "r"(parity) : "memory");
                        }
                        const wt_t* src = rowp(L, i2) + c0;
                        const uintptr_t a0 = reinterpret_cast<uintptr_t>(src) & ~(uintptr_t)15;
                        const uintptr_t a1 = (reinterpret_cast<uintptr_t>(src + nloc) + 15) & ~(uintptr_t)15;
                        const uint32_t bytes = (uint32_t)(a1 - a0);
                        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
                        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
                        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                                     ::"r"(smem_u32(rowbuf + nb * slot_words)), "l"(a0), "r"(bytes), "r"(bar) : "memory");
                        pfpar[nb] = pfcount[nb] & 1u;
                        ++pfcount[nb];
                        pfrow[nb] = i2;
                        pfshift[nb] = (int32_t)((reinterpret_cast<uintptr_t>(src) - a0) / sizeof(wt_t));
                    }
                }
            }
            // L2 prefetch: every lane's candidate (its warp-index minimum other than the
            // winner, one of the next few pops) gets this CTA's slice of its row pulled
            // from HBM into L2
            if (l2pf && tid < NT / 32 && cand2 != kNoKey && nloc > 0) {
                const int32_t i2 = rocr[cand2 & kIdxMask];
                if (i2 >= 0) {
                    const wt_t* src = rowp(L, i2) + c0;
                    const uintptr_t a0 = reinterpret_cast<uintptr_t>(src) & ~(uintptr_t)15;
                    const uintptr_t a1 = (reinterpret_cast<uintptr_t>(src + nloc) + 15) & ~(uintptr_t)15;
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0)) : "memory");
                }
            }
            // pop jm and the ties: their owner threads mark them scanned
            if (jm >= c0 && jm < c0 + nloc) {
#pragma unroll
                for (int u = 0; u < CC; ++u)
                    if (jm - c0 == tid + u * NT) { kd[u] |= kTop; pk[u] |= kTop; }
            }
#pragma unroll
            for (int t = 0; t < kTieMax; ++t) {
                const int32_t jt = (int32_t)(tk[t] & kIdxMask) - c0;   // tk = kNoKey past nt: out of range
                if (t < nt && jt >= 0 && jt < nloc) {
#pragma unroll
                    for (int u = 0; u < CC; ++u)
                        if (jt == tid + u * NT) { kd[u] |= kTop; pk[u] |= kTop; }
                }
            }
            if (hit) {
                const uint32_t bar = smem_u32(&pfbar[cur]), parity = pfpar[cur];
                uint32_t done = 0;
                while (!done)
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
                const wt_t* rb = rowbuf + cur * slot_words + pfshift[cur];
#pragma unroll
                for (int u = 0; u < CC; ++u) {
                    const int32_t jj = tid + u * NT;
                    av[u] = jj < nloc ? rb[jj] : 0;
                }
                ++pfhits;
            }
            const uint64_t base = (uint64_t)(dmin + aim - psr[jm]) << kSH;
            best = kNoKey;
#pragma unroll
            for (int u = 0; u < CC; ++u) {
                const uint64_t nk = base + pk[u] - ((uint64_t)av[u] << kSH);
                if (tid + u * NT < nloc && nk < kd[u]) { kd[u] = nk; pred[tid + u * NT] = i; }
            }
#pragma unroll
            for (int t = 0; t < kTieMax; ++t) {
                if (t < nt) {
                    const int32_t jt = (int32_t)(tk[t] & kIdxMask);
                    const uint64_t b = (uint64_t)(dmin + (int64_t)aimt[t] - psr[jt]) << kSH;
#pragma unroll
                    for (int u = 0; u < CC; ++u) {
                        const uint64_t nk = b + pk[u] - ((uint64_t)avt[t][u] << kSH);
                        if (tid + u * NT < nloc && nk < kd[u]) { kd[u] = nk; pred[tid + u * NT] = it[t]; }
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < CC; ++u) best = kd[u] < best ? kd[u] : best;
            steps += nt;
            ++rounds;
            const int nt_step = nt;
            const long long tB = tm ? clock64() : 0;
            best = cluster_min_push_ties<CLS, NT / 32>(best, S, P, TS, par, ph, rank, cand2, tk, nt, ties, tm && tid == 0 ? &txt[4] : nullptr);
            if (tm) {
                const long long tC = clock64();
                tcyc[0] += tB - tA;
                tcyc[1] += tC - tB;
                tcyc[2] += 1;
                if (hit) { txt[0] += tB - tA; txt[1] += 1; }
                if (nt_step > 0) { txt[2] += tB - tA; txt[3] += 1; }
            }
            cur ^= 1;
            ++steps;
        }
        if (!abandon) {
            // dual update on the local scanned columns: p_j += D - d_j
#pragma unroll
            for (int u = 0; u < CC; ++u) {
                const int32_t jj = tid + u * NT;
                if (jj < nloc && (kd[u] & kTop)) {
                    const int64_t pj = (int64_t)((pk[u] & ~kTop) >> kSH), dj = (int64_t)((kd[u] & ~kTop) >> kSH);
                    L.p[c0 + jj] = pj + (D - dj);
                }
            }
            // the path walk reads every column's predecessor: gather them into CTA 0
            // first (into its price table, unused until the next search reloads it),
            // so each hop is a local shared-memory read instead of a DSMEM round trip
            int32_t* predall = reinterpret_cast<int32_t*>(psr);
            int32_t* dst = cluster.map_shared_rank(predall, 0);
            for (int32_t jj = tid; jj < nloc; jj += NT) dst[c0 + jj] = pred[jj];
            cluster.sync();
            if (rank == 0 && tid == 0) {
                const long long tw = tm ? clock64() : 0;
                int32_t j = jf;
                while (true) {
                    const int32_t ii = predall[j];
                    const int32_t jn = (ii == s) ? -1 : colof[ii];
                    L.roc[j] = ii;
                    L.cor[ii] = j;
                    ++walk;
                    if (ii == s) break;
                    j = jn;
                }
                if (tm) wcyc += clock64() - tw;
            }
        }
        __threadfence();
        cluster.sync();
    }
    // no bulk copy may still be writing this CTA's shared memory at exit
    if (tid == 0)
        for (int b = 0; b < 2; ++b)
            if (pfcount[b] > 0) {
                const uint32_t bar = smem_u32(&pfbar[b]), parity = (pfcount[b] - 1) & 1u;
                uint32_t done = 0;
                while (!done)
                    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
            }
    if (rank == 0 && tid == 0) {
        atomicAdd(&L.cnt->xsteps, steps);
        atomicAdd(&L.cnt->xpfhits, pfhits);
        atomicAdd(&L.cnt->xrounds, rounds);
    }
    if (tm && rank == 0 && tid == 0)
        for (int k = 0; k < 3; ++k) atomicAdd((unsigned long long*)&L.cnt->xcyc[k], (unsigned long long)tcyc[k]);
    if (tm && rank == 0 && tid == 0) {
        for (int k = 0; k < 5; ++k) atomicAdd(&L.cnt->xt[k], txt[k]);
        atomicAdd(&L.cnt->xwalk, walk);
        atomicAdd(&L.cnt->xwalkcyc, (unsigned long long)wcyc);
        atomicAdd(&L.cnt->xsearch, (unsigned long long)ndef);
    }
}

// Register-key kernel for levels too large to replicate prices and owners
// in every CTA (m > CL * 2048: the 10k x 40k rounds of config 5).  Each
// thread keeps its columns' keys, prices and owners in registers; a warp's
// minimum travels with its column's owner row and price packed into a second
// word (price << kSH | owner + 1), pushed as one 16-byte st.async, so the
// winner's row and price arrive with the key -- no replicated tables, no
// DSMEM fetch after the exchange.
template <int CLS, int NW>
struct CPush2 {
    ulonglong2 slots[2][CLS * 32];
    uint64_t bar[2];
};

template <int CLS, int NW>
__device__ __forceinline__ void cpush2_init(CPush2<CLS, NW>& P) {
    if (threadIdx.x == 0) {
#pragma unroll
        for (int b = 0; b < 2; ++b)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&P.bar[b])) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
#pragma unroll
        for (int b = 0; b < 2; ++b)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&P.bar[b])), "r"(CLS * NW * 16)
                         : "memory");
    }
}

// cluster-wide minimum of (key, payload) pairs by key
template <int CLS, int NW>
__device__ __forceinline__ ulonglong2 cluster_min_push2(uint64_t v, uint64_t pay, ulonglong2* bres, CPush2<CLS, NW>& P,
                                                        int& par, uint32_t& ph, int rank) {
    const uint64_t wv = wmin64(v);
    const unsigned who = __ballot_sync(0xffffffffu, v == wv);
    pay = __shfl_sync(0xffffffffu, pay, __ffs(who) - 1);
    const int w = threadIdx.x >> 5, ln = lane_id();
    const uint32_t lb = smem_u32(&P.bar[par]);
    if (ln < CLS) {
        const uint32_t la = smem_u32(&P.slots[par][rank * 32 + w]);
        uint32_t ra, rb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(ln));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(lb), "r"(ln));
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(ra),
                     "l"(wv), "l"(pay), "r"(rb)
                     : "memory");
    }
    if (w == 0) {
        const uint32_t parity = (ph >> par) & 1u;
        uint32_t done = 0;
        while (!done)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(lb), "r"(parity)
                : "memory");
        ulonglong2 x = make_ulonglong2(kNoKey, 0ull);
#pragma unroll
        for (int r = 0; r < CLS; ++r) {
            const ulonglong2 y = ln < NW ? P.slots[par][r * 32 + ln] : make_ulonglong2(kNoKey, 0ull);
            if (y.x < x.x) x = y;
        }
        const uint64_t m2 = wmin64(x.x);
        const unsigned h = __ballot_sync(0xffffffffu, x.x == m2);
        const uint64_t p2 = __shfl_sync(0xffffffffu, x.y, __ffs(h) - 1);
        if (ln == 0) {
            bres[par] = make_ulonglong2(m2, p2);
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(lb), "r"(CLS * NW * 16) : "memory");
        }
    }
    ph ^= 1u << par;
    __syncthreads();
    const ulonglong2 r = bres[par];
    par ^= 1;
    return r;
}

// cluster_min_push2 with tie batching (as cluster_min_push_ties): up to TM
// further (key, payload) warp minima at the winner's distance, the CLS x NW
// slots spread over all 32 lanes.
template <int TM>
struct CTies2 {
    ulonglong2 e[2][TM];
    int32_t n[2];
};

template <int CLS, int NW, int TM>
__device__ __forceinline__ ulonglong2 cluster_min_push2_ties(uint64_t v, uint64_t pay, ulonglong2* bres, CPush2<CLS, NW>& P,
                                                             CTies2<TM>& T, int& par, uint32_t& ph, int rank,
                                                             ulonglong2 (&te)[TM], int& nt, bool ties) {
    const uint64_t wv = wmin64(v);
    const unsigned who = __ballot_sync(0xffffffffu, v == wv);
    pay = __shfl_sync(0xffffffffu, pay, __ffs(who) - 1);
    const int w = threadIdx.x >> 5, ln = lane_id();
    const uint32_t lb = smem_u32(&P.bar[par]);
    if (ln < CLS) {
        const uint32_t la = smem_u32(&P.slots[par][rank * 32 + w]);
        uint32_t ra, rb;
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(ln));
        asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(rb) : "r"(lb), "r"(ln));
        asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v2.b64 [%0], {%1, %2}, [%3];" ::"r"(ra),
                     "l"(wv), "l"(pay), "r"(rb)
                     : "memory");
    }
    if (w == 0) {
        const uint32_t parity = (ph >> par) & 1u;
        uint32_t done = 0;
        while (!done)
            asm volatile(
                "{ .reg .pred p; mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                : "=r"(done)
                : "r"(lb), "r"(parity)
                : "memory");
        constexpr int TOT = CLS * NW, KPL = (TOT + 31) / 32;
        ulonglong2 ys[KPL];
        ulonglong2 x = make_ulonglong2(kNoKey, 0ull);
#pragma unroll
        for (int k = 0; k < KPL; ++k) {
            const int e = ln + 32 * k;
            ys[k] = e < TOT ? P.slots[par][(e / NW) * 32 + (e % NW)] : make_ulonglong2(kNoKey, 0ull);
            if (ys[k].x < x.x) x = ys[k];
        }
        const uint64_t m2 = wmin64(x.x);
        const unsigned h = __ballot_sync(0xffffffffu, x.x == m2);
        const uint64_t p2 = __shfl_sync(0xffffffffu, x.y, __ffs(h) - 1);
        const bool batch = ties && (m2 & kFreeBit) != 0 && m2 != kNoKey;
        const uint64_t dhi = m2 >> kSH;
        const unsigned lt = (1u << ln) - 1u;
        int cnt = 0;
#pragma unroll
        for (int k = 0; k < KPL; ++k) {
            const bool tie = batch && (ys[k].x >> kSH) == dhi && ys[k].x != m2;
            const unsigned msk = __ballot_sync(~0u, tie);
            if (tie) {
                const int pos = cnt + __popc(msk & lt);
                if (pos < TM) T.e[par][pos] = ys[k];
            }
            cnt += __popc(msk);
        }
        if (ln == 0) {
            bres[par] = make_ulonglong2(m2, p2);
            T.n[par] = cnt < TM ? cnt : TM;
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(lb), "r"(CLS * NW * 16) : "memory");
        }
    }
    ph ^= 1u << par;
    __syncthreads();
    const ulonglong2 r = bres[par];
    nt = ties ? T.n[par] : 0;
    ulonglong2 raw[TM];
#pragma unroll
    for (int t = 0; t < TM; ++t) raw[t] = T.e[par][t];
#pragma unroll
    for (int t = 0; t < TM; ++t) te[t] = t < nt ? raw[t] : make_ulonglong2(kNoKey, 0ull);
    par ^= 1;
    return r;
}

constexpr int kTieMaxSlice = 1;   // the slice kernel's register budget (512 threads, up to 16 columns each)

template <int CC, int CLS, int NT>
__global__ void __cluster_dims__(CLS, 1, 1) __launch_bounds__(NT, 1)
ssp_rkey_slice_kernel(Lvl L, int32_t ndef, int32_t pop_limit, int32_t flags) {
    constexpr int NW = NT / 32;
    unsigned long long walk = 0;
    long long wcyc = 0, scyc = 0;
    __shared__ __align__(16) CPush2<CLS, NW> P;
    __shared__ __align__(16) ulonglong2 bres[2];
    __shared__ __align__(16) CTies2<kTieMaxSlice> TS;
    constexpr int TM = kTieMaxSlice;
    ulonglong2 te[TM];
    int nt = 0;
    int32_t rpf_rank = -1, rpf_row = -1;   // rank-neighbour prefetch pipeline (two lanes)
    extern __shared__ __align__(16) unsigned char smem[];
    int32_t* pred = reinterpret_cast<int32_t*>(smem);   // [mc] predecessor rows (local)
    cg::cluster_group cluster = cg::this_cluster();
    const int32_t m = L.m;
    const int32_t mc = (m + CLS - 1) / CLS;
    const int rank = (int)cluster.block_rank();
    const int32_t c0 = rank * mc;
    const int32_t nloc = max(0, min(mc, m - c0));
    const int tid = threadIdx.x;
    int par = 0;
    uint32_t ph = 0;
    unsigned long long steps = 0, rounds = 0;
    const bool tm = (flags & 16) != 0;
    const bool ties = (flags & 64) != 0;
    long long tcyc[3] = {0, 0, 0};
    cpush2_init<CLS, NW>(P);
    cluster.sync();
    for (int32_t q = 0; q < ndef; ++q) {
        const int32_t s = L.defer[q];
        const wt_t* As = rowp(L, s);
        uint64_t kd[CC], pk[CC];
        int32_t own[CC], as[CC];
#pragma unroll
        for (int u = 0; u < CC; ++u) {
            const int32_t jj = tid + u * NT;
            as[u] = jj < nloc ? __ldg(As + c0 + jj) : 0;
            own[u] = jj < nloc ? __ldcg(L.roc + c0 + jj) : -1;
        }
        uint64_t vmin = kNoKey, vpay = 0;
#pragma unroll
        for (int u = 0; u < CC; ++u) {
            const int32_t jj = tid + u * NT;
            if (jj < nloc) {
                const int32_t j = c0 + jj;
                const int64_t pj = __ldcg(L.p + j);
                if (pj < 0 || pj >= kDistLim) atomicOr(&L.cnt->errors, kErrDist);
                const uint64_t low = (own[u] < 0 ? 0u : kFreeBit) | (uint32_t)j;
                pk[u] = ((uint64_t)pj << kSH) | low;
                const uint64_t k = ((uint64_t)(pj - (int64_t)as[u] + kDistLim) << kSH) | low;
                if (k < vmin) { vmin = k; vpay = ((uint64_t)pj << kSH) | (uint32_t)(own[u] + 1); }
                pred[jj] = s;
            } else {
                pk[u] = kTop;
            }
        }
        const ulonglong2 r0 = cluster_min_push2_ties<CLS, NW, TM>(vmin, vpay, bres, P, TS, par, ph, rank, te, nt, ties);
#pragma unroll
        for (int t = 0; t < TM; ++t) te[t].x &= kLowMask;   // ties at distance 0
        const int64_t pis = -((int64_t)(r0.x >> kSH) - kDistLim);
#pragma unroll
        for (int u = 0; u < CC; ++u) {
            const int32_t jj = tid + u * NT;
            kd[u] = jj < nloc ? (((uint64_t)pis << kSH) + pk[u] - ((uint64_t)as[u] << kSH)) : kNoKey;
        }
        uint64_t best = r0.x & kLowMask;
        uint64_t bpay = r0.y;
        int32_t jf;
        int64_t D;
        int32_t pops = 0;
        bool abandon = false;
        while (true) {
            const int32_t jm = (int32_t)(best & kIdxMask);
            const int64_t dmin = (int64_t)(best >> kSH);
            const int32_t i = (int32_t)(bpay & kLowMask) - 1;
            const int64_t pjm = (int64_t)(bpay >> kSH);
            if (i < 0) { jf = jm; D = dmin; break; }
            if (pop_limit > 0 && (pops += 1 + nt) > pop_limit) { abandon = true; jf = -1; D = 0; break; }
            const long long tA = tm ? clock64() : 0;
            const wt_t* Ai = rowp(L, i);
            wt_t av[CC];
#pragma unroll
            for (int u = 0; u < CC; ++u) {
                const int32_t jj = tid + u * NT;
                av[u] = jj < nloc ? __ldg(Ai + c0 + jj) : 0;
            }
            const int64_t aim = (int64_t)__ldg(Ai + jm);
            // tied columns (matched): owner row and price travel in the payload
            wt_t avt[TM][CC];
            wt_t aimt[TM];
#pragma unroll
            for (int t = 0; t < TM; ++t) {
                if (t < nt) {
                    const int32_t it = (int32_t)(te[t].y & kLowMask) - 1;
                    const wt_t* At = rowp(L, it);
                    aimt[t] = __ldg(At + (int32_t)(te[t].x & kIdxMask));
#pragma unroll
                    for (int u = 0; u < CC; ++u) {
                        const int32_t jj = tid + u * NT;
                        avt[t][u] = jj < nloc ? __ldg(At + c0 + jj) : 0;
                    }
                }
            }
            if (L.rpf > 0 && tid >= NT - RPF_LANES) {
                // rank-neighbour L2 prefetch pipeline (as in ssp_rkey_kernel)
                if (rpf_row >= 0 && nloc > 0) {
                    const wt_t* src = rowp(L, rpf_row) + c0;
                    const uintptr_t a0 = reinterpret_cast<uintptr_t>(src) & ~(uintptr_t)15;
                    const uintptr_t a1 = (reinterpret_cast<uintptr_t>(src + nloc) + 15) & ~(uintptr_t)15;
                    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(a0), "r"((uint32_t)(a1 - a0)) : "memory");
                }
                // lane NT-1-k: distance (k / 2 + 1) * rpf / (RPF_LANES / 2), up for even k, down for odd
                const int kq = NT - 1 - tid;
                const int32_t dist = (int32_t)(((kq >> 1) + 1) * L.rpf / (RPF_LANES / 2));
                const int32_t rr = rpf_rank < 0 ? -1 : rpf_rank + ((kq & 1) ? -dist : dist);
                if (L.rankof) {
                    rpf_row = rr >= 0 && rr < m ? __ldcg(L.rowat + rr) : -1;
                    rpf_rank = __ldcg(L.rankof + i);
                } else {
                    rpf_row = rr >= 0 && rr < m ? rr : -1;
                    rpf_rank = i;
                }
            }
            if (jm >= c0 && jm < c0 + nloc) {
#pragma unroll
                for (int u = 0; u < CC; ++u)
                    if (jm - c0 == tid + u * NT) { kd[u] |= kTop; pk[u] |= kTop; }
            }
#pragma unroll
            for (int t = 0; t < TM; ++t) {
                const int32_t jt = (int32_t)(te[t].x & kIdxMask) - c0;
                if (t < nt && jt >= 0 && jt < nloc) {
#pragma unroll
                    for (int u = 0; u < CC; ++u)
                        if (jt == tid + u * NT) { kd[u] |= kTop; pk[u] |= kTop; }
                }
            }
            const uint64_t base = (uint64_t)(dmin + aim - pjm) << kSH;
            best = kNoKey;
            uint64_t pay = 0;
#pragma unroll
            for (int u = 0; u < CC; ++u) {
                const uint64_t nk = base + pk[u] - ((uint64_t)av[u] << kSH);
                if (tid + u * NT < nloc && nk < kd[u]) { kd[u] = nk; pred[tid + u * NT] = i; }
            }
#pragma unroll
            for (int t = 0; t < TM; ++t) {
                if (t < nt) {
                    const int32_t it = (int32_t)(te[t].y & kLowMask) - 1;
                    const uint64_t b = (uint64_t)(dmin + (int64_t)aimt[t] - (int64_t)(te[t].y >> kSH)) << kSH;
#pragma unroll
                    for (int u = 0; u < CC; ++u) {
                        const uint64_t nk = b + pk[u] - ((uint64_t)avt[t][u] << kSH);
                        if (tid + u * NT < nloc && nk < kd[u]) { kd[u] = nk; pred[tid + u * NT] = it; }
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < CC; ++u)
                if (kd[u] < best) { best = kd[u]; pay = ((pk[u] & ~kTop) & ~kLowMask) | (uint32_t)(own[u] + 1); }
            steps += nt;
            ++rounds;
            const long long tB = tm ? clock64() : 0;
            const ulonglong2 r = cluster_min_push2_ties<CLS, NW, TM>(best, pay, bres, P, TS, par, ph, rank, te, nt, ties);
            best = r.x;
            bpay = r.y;
            if (tm) {
                const long long tC = clock64();
                tcyc[0] += tB - tA;
                tcyc[1] += tC - tB;
                tcyc[2] += 1;
            }
            ++steps;
        }
        if (!abandon) {
#pragma unroll
            for (int u = 0; u < CC; ++u) {
                const int32_t jj = tid + u * NT;
                if (jj < nloc && (kd[u] & kTop)) {
                    const int64_t pj = (int64_t)((pk[u] & ~kTop) >> kSH), dj = (int64_t)((kd[u] & ~kTop) >> kSH);
                    L.p[c0 + jj] = pj + (D - dj);
                }
            }
            if (flags & 128) {
                // local walk: every column's (predecessor, predecessor's old column) pair,
                // 16 bits each, gathered into CTA 0 (launched with 4 m more bytes) in one
                // parallel pass, so a hop is a shared-memory read instead of a DSMEM read
                // plus a global one
                uint32_t* ps = reinterpret_cast<uint32_t*>(smem + 4 * (size_t)mc + 64);
                uint32_t* dst = cluster.map_shared_rank(ps, 0);
                for (int32_t jj = tid; jj < nloc; jj += NT) {
                    const int32_t ii = pred[jj];
                    const int32_t jo = ii == s ? 0xFFFF : __ldcg(L.cor + ii);
                    dst[c0 + jj] = ((uint32_t)ii << 16) | (uint32_t)(jo & 0xFFFF);
                }
                cluster.sync();
                if (rank == 0 && tid == 0) {
                    const long long tw = tm ? clock64() : 0;
                    int32_t j = jf;
                    while (true) {
                        const uint32_t v = ps[j];
                        const int32_t ii = (int32_t)(v >> 16);
                        L.roc[j] = ii;
                        L.cor[ii] = j;
                        ++walk;
                        if (ii == s) break;
                        j = (int32_t)(v & 0xFFFF);
                    }
                    if (tm) wcyc += clock64() - tw;
                }
            } else if (rank == 0 && tid == 0) {
                const long long tw = tm ? clock64() : 0;
                int32_t j = jf;
                while (true) {
                    const int owner = j / mc;
                    const int32_t ii = cluster.map_shared_rank(pred, owner)[j - owner * mc];
                    const int32_t jn = (ii == s) ? -1 : __ldcg(L.cor + ii);
                    L.roc[j] = ii;
                    L.cor[ii] = j;
                    ++walk;
                    if (ii == s) break;
                    j = jn;
                }
                if (tm) wcyc += clock64() - tw;
            }
        }
        const long long ts = tm ? clock64() : 0;
        __threadfence();
        cluster.sync();
        if (tm) scyc += clock64() - ts;
    }
    if (rank == 0 && tid == 0) {
        atomicAdd(&L.cnt->xsteps, steps);
        atomicAdd(&L.cnt->xrounds, rounds);
    }
    if (tm && rank == 0 && tid == 0) {
        for (int k = 0; k < 3; ++k) atomicAdd((unsigned long long*)&L.cnt->xcyc[k], (unsigned long long)tcyc[k]);
        atomicAdd(&L.cnt->xwalk, walk);
        atomicAdd(&L.cnt->xwalkcyc, (unsigned long long)wcyc);
        atomicAdd(&L.cnt->xsearch, (unsigned long long)ndef);
        atomicAdd(&L.cnt->xsynccyc, (unsigned long long)scyc);
    }
}

// Single-CTA register-key kernel for levels small enough for one SM
// (m <= 1024 * CC): the same register-resident keys, the whole row slice on
// one SM, and a block-wide minimum with ONE barrier per pop -- every warp
// writes its minimum to a parity-double-buffered slot array, and after the
// barrier every warp reduces the 32 slots itself.  No DSMEM round trip.
template <int CC, int NT>
__global__ void __launch_bounds__(NT, 1) ssp_rkey1_kernel(Lvl L, int32_t ndef, int32_t pop_limit, int32_t flags) {
    extern __shared__ __align__(16) unsigned char smem[];
    __shared__ uint64_t slots[2][32];   // per-warp minima (slots past NT / 32 stay kNoKey)
    const int32_t m = L.m;
    int64_t* psr = reinterpret_cast<int64_t*>(smem);                          // [m] prices
    int32_t* rocr = reinterpret_cast<int32_t*>(psr + m);                      // [m] owners
    int32_t* colof = rocr + ((m + 1) & ~1);                                  // [m] matched column of each tree row
    int32_t* pred = colof + ((m + 1) & ~1);                                  // [m] predecessor rows
    const int tid = threadIdx.x, w = tid >> 5;
    int par = 0;
    unsigned long long steps = 0;
    const bool tm = (flags & 16) != 0;
    const bool ties = (flags & 64) != 0;
    long long tcyc[3] = {0, 0, 0};
    unsigned long long rounds = 0;
    uint64_t tk[kTieMax];
    int nt = 0;
    // block minimum; with tie batching, also up to kTieMax further warp minima
    // at the winner's distance (every warp derives the same list from the slots)
    auto block_min = [&](uint64_t v) -> uint64_t {
        v = wmin64(v);
        if (lane_id() == 0) slots[par][w] = v;
        __syncthreads();
        const uint64_t y = slots[par][lane_id()];
        const uint64_t x = wmin64(y);
        const bool batch = ties && (x & kFreeBit) != 0 && x != kNoKey;
        unsigned msk = __ballot_sync(~0u, batch && (y >> kSH) == (x >> kSH) && y != x);
        nt = min(__popc(msk), kTieMax);
#pragma unroll
        for (int t = 0; t < kTieMax; ++t) {
            const int l = __ffs(msk) - 1;
            const uint64_t yt = __shfl_sync(~0u, y, l < 0 ? 0 : l);
            tk[t] = t < nt ? yt : kNoKey;
            msk &= msk - 1;
        }
        par ^= 1;
        return x;
    };
    if (tid < 64) slots[tid >> 5][tid & 31] = kNoKey;
    __syncthreads();
    for (int32_t q = 0; q < ndef; ++q) {
        const int32_t s = L.defer[q];
        const wt_t* As = rowp(L, s);
        for (int32_t j = tid; j < m; j += NT) {
            psr[j] = __ldcg(L.p + j);
            rocr[j] = __ldcg(L.roc + j);
        }
        __syncthreads();
        uint64_t kd[CC], pk[CC];
        wt_t as[CC];
        uint64_t vmin = kNoKey;
#pragma unroll
        for (int u = 0; u < CC; ++u) {
            const int32_t j = tid + u * NT;
            as[u] = j < m ? __ldg(As + j) : 0;
        }
#pragma unroll
        for (int u = 0; u < CC; ++u) {
            const int32_t j = tid + u * NT;
            if (j < m) {
                const int64_t pj = psr[j];
                if (pj < 0 || pj >= kDistLim) atomicOr(&L.cnt->errors, kErrDist);
                const uint64_t low = (rocr[j] < 0 ? 0u : kFreeBit) | (uint32_t)j;
                pk[u] = ((uint64_t)pj << kSH) | low;
                const uint64_t k = ((uint64_t)(pj - (int64_t)as[u] + kDistLim) << kSH) | low;
                vmin = k < vmin ? k : vmin;
                pred[j] = s;
            } else {
                pk[u] = kTop;
            }
        }
        const uint64_t k0 = block_min(vmin);
        const int64_t pis = -((int64_t)(k0 >> kSH) - kDistLim);
#pragma unroll
        for (int u = 0; u < CC; ++u) {
            const int32_t j = tid + u * NT;
            kd[u] = j < m ? (((uint64_t)pis << kSH) + pk[u] - ((uint64_t)as[u] << kSH)) : kNoKey;
        }
        uint64_t best = k0 & kLowMask;
#pragma unroll
        for (int t = 0; t < kTieMax; ++t) tk[t] &= kLowMask;   // ties at distance 0
        int32_t jf;
        int64_t D;
        int32_t pops = 0;
        bool abandon = false;
        while (true) {
            const int32_t jm = (int32_t)(best & kIdxMask);
            const int64_t dmin = (int64_t)(best >> kSH);
            const int32_t i = rocr[jm];
            // this step's loads first (a free winner ends the search below; its
            // loads read the zero row), the bookkeeping after them
            const long long tA = tm ? clock64() : 0;
            const wt_t* Ai = i >= 0 ? rowp(L, i) : L.zrow;
            wt_t av[CC];
#pragma unroll
            for (int u = 0; u < CC; ++u) {
                const int32_t j = tid + u * NT;
                av[u] = j < m ? __ldg(Ai + j) : 0;
            }
            const int64_t aim = (int64_t)__ldg(Ai + jm);
            wt_t avt[kTieMax][CC];
            wt_t aimt[kTieMax];
            int32_t it[kTieMax];
#pragma unroll
            for (int t = 0; t < kTieMax; ++t) {
                if (t < nt) {
                    const int32_t jt = (int32_t)(tk[t] & kIdxMask);
                    it[t] = rocr[jt];
                    const wt_t* At = rowp(L, it[t]);
                    aimt[t] = __ldg(At + jt);
#pragma unroll
                    for (int u = 0; u < CC; ++u) {
                        const int32_t j = tid + u * NT;
                        avt[t][u] = j < m ? __ldg(At + j) : 0;
                    }
                }
            }
            asm volatile("" ::: "memory");
            if (i < 0) { jf = jm; D = dmin; break; }
            if (pop_limit > 0 && (pops += 1 + nt) > pop_limit) { abandon = true; jf = -1; D = 0; break; }
            if (tid == 0) {
                colof[i] = jm;
#pragma unroll
                for (int t = 0; t < kTieMax; ++t)
                    if (t < nt) colof[it[t]] = (int32_t)(tk[t] & kIdxMask);
            }
#pragma unroll
            for (int u = 0; u < CC; ++u)
                if (jm == tid + u * NT) { kd[u] |= kTop; pk[u] |= kTop; }
#pragma unroll
            for (int t = 0; t < kTieMax; ++t) {
                const int32_t jt = (int32_t)(tk[t] & kIdxMask);
                if (t < nt) {
#pragma unroll
                    for (int u = 0; u < CC; ++u)
                        if (jt == tid + u * NT) { kd[u] |= kTop; pk[u] |= kTop; }
                }
            }
            const uint64_t base = (uint64_t)(dmin + aim - psr[jm]) << kSH;
            best = kNoKey;
#pragma unroll
            for (int u = 0; u < CC; ++u) {
                const uint64_t nk = base + pk[u] - ((uint64_t)av[u] << kSH);
                if (tid + u * NT < m && nk < kd[u]) { kd[u] = nk; pred[tid + u * NT] = i; }
            }
#pragma unroll
            for (int t = 0; t < kTieMax; ++t) {
                if (t < nt) {
                    const int32_t jt = (int32_t)(tk[t] & kIdxMask);
                    const uint64_t b = (uint64_t)(dmin + (int64_t)aimt[t] - psr[jt]) << kSH;
#pragma unroll
                    for (int u = 0; u < CC; ++u) {
                        const uint64_t nk = b + pk[u] - ((uint64_t)avt[t][u] << kSH);
                        if (tid + u * NT < m && nk < kd[u]) { kd[u] = nk; pred[tid + u * NT] = it[t]; }
                    }
                }
            }
#pragma unroll
            for (int u = 0; u < CC; ++u) best = kd[u] < best ? kd[u] : best;
            steps += nt;
            ++rounds;
            const long long tB = tm ? clock64() : 0;
            best = block_min(best);
            if (tm) {
                const long long tC = clock64();
                tcyc[0] += tB - tA;
                tcyc[1] += tC - tB;
                tcyc[2] += 1;
            }
            ++steps;
        }
        if (!abandon) {
#pragma unroll
            for (int u = 0; u < CC; ++u) {
                const int32_t j = tid + u * NT;
                if (j < m && (kd[u] & kTop)) {
                    const int64_t pj = (int64_t)((pk[u] & ~kTop) >> kSH), dj = (int64_t)((kd[u] & ~kTop) >> kSH);
                    L.p[j] = pj + (D - dj);
                }
            }
            __syncthreads();   // pred complete
            if (tid == 0) {
                int32_t j = jf;
                while (true) {
                    const int32_t ii = pred[j];
                    const int32_t jn = (ii == s) ? -1 : colof[ii];
                    L.roc[j] = ii;
                    L.cor[ii] = j;
                    if (ii == s) break;
                    j = jn;
                }
            }
        }
        __threadfence();
        __syncthreads();
    }
    if (tid == 0) {
        atomicAdd(&L.cnt->xsteps, steps);
        atomicAdd(&L.cnt->xrounds, rounds);
    }
    if (tm && tid == 0)
        for (int k = 0; k < 3; ++k) atomicAdd((unsigned long long*)&L.cnt->xcyc[k], (unsigned long long)tcyc[k]);
}

// ---------------------------------------------------------------------------
// level setup kernels
// ---------------------------------------------------------------------------

// A_l[r][c] = W[rows[r]][cols[c]] (rows >= N are the zero padding rows)
__global__ void gather_kernel(const wt_t* W, int64_t ldw, int32_t N, const int32_t* rows, const int32_t* cols,
                              int32_t m, wt_t* out) {
    for (int32_t r = blockIdx.x; r < m; r += gridDim.x) {
        const int32_t ri = rows[r];
        if (ri >= N) {
            for (int32_t c = threadIdx.x; c < m; c += blockDim.x) out[(int64_t)r * m + c] = 0;
            continue;
        }
        const wt_t* Wr = W + (int64_t)ri * ldw;
        for (int32_t c = threadIdx.x; c < m; c += blockDim.x) out[(int64_t)r * m + c] = __ldg(Wr + cols[c]);
    }
}

// base level: p_j = max_i a_ij (rows >= nreal are zero)
__global__ void colmax_kernel(const wt_t* A, int64_t lda, int32_t nreal, int32_t m, int64_t* p) {
    const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    int64_t b = nreal < m ? 0 : INT64_MIN;
    for (int32_t i = 0; i < nreal && i < m; ++i) {
        const int64_t v = A[(int64_t)i * lda + j];
        b = v > b ? v : b;
    }
    p[j] = b;
}

// ---------------------------------------------------------------------------
// warm start across rounds (config-5 replays): the previous round's optimal
// column prices (INT64_MIN = a column it did not have) and its assignment
// mapped to this round's indices.  Any prices with row profits taken as the
// c-transform pi_i = max_j (a_ij - p_j) are dual feasible; every previous
// pair that is still tight under them stays matched, and only the rest of
// the rows (those whose features changed, new columns' takers) are searched.
//  1. pi_i over the carried columns (warp per real row)
//  2. new columns priced at max(max_i (a_ij - pi_i), p_min): feasible for
//     every real row and for the zero padding rows (pi_pad = -p_min)
//  3. tight previous pairs kept; padding rows take free columns at p_min
// ---------------------------------------------------------------------------

// block-wide minimum of the carried prices into *pmin (pre-set to INT64_MAX)
__global__ void warm_pmin_kernel(const int64_t* pin, int32_t m, unsigned long long* pmin) {
    int64_t b = INT64_MAX;
    for (int32_t j = blockIdx.x * blockDim.x + threadIdx.x; j < m; j += gridDim.x * blockDim.x)
        if (pin[j] != INT64_MIN) b = pin[j] < b ? pin[j] : b;
    b = wmin64s(b);
    if (lane_id() == 0 && b != INT64_MAX) atomicMin(reinterpret_cast<long long*>(pmin), (long long)b);
}

__global__ void warm_profit_kernel(const wt_t* A, int64_t lda, int32_t nreal, int32_t m, const int64_t* pin,
                                   int64_t* pi) {
    const int32_t k = (int32_t)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    if (k >= nreal) return;
    int64_t b = -kInf;
    for (int32_t c = lane_id(); c < m; c += 32) {
        const int64_t pc = pin[c];
        if (pc != INT64_MIN) {
            const int64_t v = (int64_t)A[(int64_t)k * lda + c] - pc;
            b = v > b ? v : b;
        }
    }
    b = wmax64s(b);
    if (lane_id() == 0) pi[k] = b;
}

__global__ void warm_price_kernel(const wt_t* A, int64_t lda, int32_t nreal, int32_t m, const int64_t* pin,
                                  const int64_t* pi, const unsigned long long* pminp, int64_t* p) {
    const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const int64_t c = pin[j];
    if (c != INT64_MIN) { p[j] = c; return; }
    int64_t b = nreal < m ? (int64_t)*pminp : INT64_MIN;   // padding rows: 0 - pi_pad = p_min
    for (int32_t i = 0; i < nreal; ++i) {
        const int64_t v = (int64_t)A[(int64_t)i * lda + j] - pi[i];
        b = v > b ? v : b;
    }
    p[j] = b;
}

// keep the previous pairs that are still tight; the unmatched rows form the
// search list (cnt->qhead counts them)
__global__ void warm_match_kernel(const wt_t* A, int64_t lda, int32_t nreal, int32_t m, const int32_t* wcol,
                                  const int64_t* pi, const int64_t* p, int32_t* cor, int32_t* roc) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i >= nreal) return;
    const int32_t c = wcol ? wcol[i] : -1;
    if (c >= 0 && c < m && (int64_t)A[(int64_t)i * lda + c] - p[c] == pi[i]) {
        cor[i] = c;
        roc[c] = i;
    }
}

// padding rows [plo, phi) take the free columns priced p_min (tight for them:
// their profit is -p_min); padding rows are interchangeable
__global__ void warm_pad_kernel(int32_t plo, int32_t phi, int32_t m, const int64_t* p, const unsigned long long* pminp,
                                int32_t* cor, int32_t* roc, int32_t* counter) {
    const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m || roc[j] >= 0 || p[j] != (int64_t)*pminp) return;
    const int32_t k = atomicAdd(counter, 1);
    if (plo + k < phi) {
        roc[j] = plo + k;
        cor[plo + k] = j;
    }
}

// unmatched rows among [lo, hi) -> in[]
__global__ void warm_list_kernel(int32_t lo, int32_t hi, const int32_t* cor, int32_t* in, int32_t* counter) {
    const int32_t i = lo + blockIdx.x * blockDim.x + threadIdx.x;
    if (i < hi && cor[i] < 0) in[atomicAdd(counter, 1)] = i;
}

// split a row list into real rows and padding rows [plo, phi)
__global__ void split_rows_kernel(int32_t n, const int32_t* in, int32_t plo, int32_t phi, int32_t* real, int32_t* counter) {
    const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    const int32_t r = in[k];
    if (r < plo || r >= phi) real[atomicAdd(counter, 1)] = r;
}

// pi_k of a solved level: a_k,cor(k) - p_cor(k) for matched rows; rows a
// coarse level left unmatched (its long searches are skipped) take the
// dual-feasible max_j (a_kj - p_j).  One warp per row.
__global__ void profit_kernel(const wt_t* A, int64_t lda, int32_t m, const int32_t* cor, const int64_t* p,
                              int64_t* pi) {
    const int32_t k = (int32_t)((blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5);
    if (k >= m) return;
    const int32_t j = cor[k];
    if (j >= 0) {
        if (lane_id() == 0) pi[k] = (int64_t)A[(int64_t)k * lda + j] - p[j];
        return;
    }
    int64_t b = -kInf;
    for (int32_t c = lane_id(); c < m; c += 32) {
        const int64_t v = (int64_t)A[(int64_t)k * lda + c] - p[c];
        b = v > b ? v : b;
    }
    b = wmax64s(b);
    if (lane_id() == 0) pi[k] = b;
}

// c-transform: p_j = max_k (A[sub[k]][j] - pi_k) over the coarse rows k.
// blockIdx.y takes one chunk of the coarse rows; partial maxima meet in an
// atomicMax (p pre-filled with INT64_MIN).
__global__ void ctransform_kernel(const wt_t* A, int64_t lda, int32_t nreal, const wt_t* zrow, int32_t m,
                                  const int32_t* sub, const int64_t* pi, int32_t mc, int32_t chunk, int64_t* p) {
    const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= m) return;
    const int32_t k0 = blockIdx.y * chunk, k1 = min(mc, k0 + chunk);
    int64_t b = INT64_MIN;
    int32_t k = k0;
    for (; k + 4 <= k1; k += 4) {
        int64_t v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
            const int32_t r = __ldg(sub + k + u);
            const wt_t* Ar = r < nreal ? A + (int64_t)r * lda : zrow;
            v[u] = (int64_t)__ldg(Ar + j) - __ldg(pi + k + u);
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) b = v[u] > b ? v[u] : b;
    }
    for (; k < k1; ++k) {
        const int32_t r = __ldg(sub + k);
        const wt_t* Ar = r < nreal ? A + (int64_t)r * lda : zrow;
        const int64_t v = (int64_t)__ldg(Ar + j) - __ldg(pi + k);
        b = v > b ? v : b;
    }
    if (b != INT64_MIN) atomicMax(reinterpret_cast<long long*>(p + j), (long long)b);
}

__global__ void fill_i64_kernel(int64_t* p, int32_t m, int64_t v) {
    const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < m) p[j] = v;
}

__global__ void init_level_kernel(int32_t m, int32_t* cor, int32_t* roc, int32_t* lock, int32_t* tries,
                                  int32_t* in, int32_t stride) {
    const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= m) return;
    cor[k] = -1;
    roc[k] = -1;
    lock[k] = 0;
    tries[k] = 0;
    in[k] = (int32_t)(((int64_t)k * stride) % m);
}

// finished level 0: col_out (original indexing) and the total
__global__ void finish_kernel(const wt_t* W, int64_t ldw, int32_t n, const int32_t* cor, int32_t* col_out,
                              unsigned long long* total) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    long long q = 0;
    if (i < n) {
        const int32_t j = cor[i];
        q = j >= 0 ? (long long)W[(int64_t)i * ldw + j] : 0;
        col_out[i] = (j >= 0 && q > 0) ? j : -1;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    if ((threadIdx.x & 31) == 0 && q) atomicAdd(total, (unsigned long long)q);
}

// dense certificate (tests / MUX_SSP_CHECK): bad[0] unmatched rows, bad[1]
// row/column inconsistency, bad[2] dual violations pi_i + p_j < a_ij,
// bad[3] = first violating (i << 32 | j)
__global__ void check_kernel(const wt_t* A, int64_t lda, int32_t nreal, const wt_t* zrow, int32_t m,
                             const int32_t* cor, const int32_t* roc, const int64_t* p, unsigned long long* bad) {
    const int32_t i = blockIdx.x;
    if (i >= m) return;
    const wt_t* Ai = i < nreal ? A + (int64_t)i * lda : zrow;
    const int32_t j0 = cor[i];
    if (j0 < 0) { if (threadIdx.x == 0) atomicAdd(bad, 1ull); return; }
    if (threadIdx.x == 0 && roc[j0] != i) atomicAdd(bad + 1, 1ull);
    const int64_t pi = (int64_t)Ai[j0] - p[j0];
    unsigned long long b = 0;
    for (int32_t j = threadIdx.x; j < m; j += blockDim.x)
        if ((int64_t)Ai[j] - p[j] > pi) {
            ++b;
            atomicCAS(bad + 3, 0ull, ((unsigned long long)i << 32) | (unsigned)j);
        }
    if (b) atomicAdd(bad + 2, b);
}

// row / column sums: generic ordering keys when the caller has none
__global__ void rowsum_kernel(const wt_t* W, int64_t ldw, int32_t M, double* rs, double* cs) {
    const int32_t i = blockIdx.x;
    double s = 0;
    for (int32_t j = threadIdx.x; j < M; j += blockDim.x) {
        const double v = (double)W[(int64_t)i * ldw + j];
        s += v;
        atomicAdd(cs + j, v);
    }
    for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if ((threadIdx.x & 31) == 0) atomicAdd(rs + i, s);
}

}  // namespace ssp / ssp64
}  // namespace mux

using namespace mux;
#ifndef MUX_SSP_W64
using namespace mux::ssp;
#define MUX_SSP_IMPL mux_ssp_impl
#else
using namespace mux::ssp64;
#define MUX_SSP_IMPL mux_ssp_impl64
#endif

static size_t al256(size_t b) { return (b + 255) & ~(size_t)255; }

// Indices 0..n-1 in ascending key order, equal keys in index order: the order
// std::stable_sort gives with `<`, by an LSD radix sort on the keys' ordered
// bit patterns (8 passes of 8 bits; -0.0 is folded into +0.0 first, keys
// are never NaN).
static void key_order(const std::vector<double>& key, std::vector<int32_t>& idx) {
    const size_t n = key.size();
    std::vector<uint64_t> k(n), k2(n);
    std::vector<int32_t> i2(n);
    for (size_t t = 0; t < n; ++t) {
        const double v = key[t] == 0.0 ? 0.0 : key[t];
        uint64_t b;
        memcpy(&b, &v, 8);
        k[t] = (b >> 63) ? ~b : (b | (1ull << 63));
        idx[t] = (int32_t)t;
    }
    for (int sh = 0; sh < 64; sh += 8) {
        size_t cnt[257] = {0};
        for (size_t t = 0; t < n; ++t) ++cnt[((k[t] >> sh) & 255) + 1];
        if (cnt[((k[0] >> sh) & 255) + 1] == n) continue;   // one bucket: the pass keeps the order
        for (int b = 0; b < 256; ++b) cnt[b + 1] += cnt[b];
        for (size_t t = 0; t < n; ++t) {
            const size_t d = cnt[(k[t] >> sh) & 255]++;
            k2[d] = k[t];
            i2[d] = idx[t];
        }
        k.swap(k2);
        idx.swap(i2);
    }
}

// Multilevel exact solve of the square int32 problem W [n][ldw].
// rowkey / colkey: host ordering keys (may be null: row / column sums).
// price_out (device int64 [n], optional): optimal column prices (max form).
// Solves the reference's square problem of size n = M: rows N..M-1 are the
// zero padding rows (N <= M).
int MUX_SSP_IMPL(mux_ctx_t* ctx, const wt_t* W, int64_t ldw, int32_t N, int32_t M, const double* rowkey,
                 const double* colkey, int32_t* col_out, int64_t* total_q, int64_t* price_out,
                 int32_t* cor_out, int32_t* roc_out, mux_stats_t* stats, cudaStream_t st, const int64_t* price_in,
                 const int32_t* warm_col) {
    const int32_t n = M;
    if (n <= 0 || N <= 0) { if (total_q) *total_q = 0; return MUX_OK; }
    if (N > M) { set_error("ssp: needs N <= M"); return MUX_EINVAL; }
    if (n >= (int32_t)kIdxMask - 128) { set_error("ssp: problem too large for its key format"); return MUX_EINVAL; }
    const Tuning& T = tuning();
    const bool verbose = T.verbose;
    const int fct = T.ssp_f;
    const int base = T.ssp_base;
    const bool check = T.ssp_check;
    const int32_t serial = T.ssp_serial ? 1 : 0;
    const int32_t step_budget = T.ssp_steps;
    const int32_t deep_budget = T.ssp_deep;
    // pop limit of the long searches at coarse levels (0 = exact coarse levels)
    const int32_t coarse_pops = T.ssp_coarse_pops;
    const bool coarse_exact = coarse_pops == 0;
    auto t0 = std::chrono::steady_clock::now();

    // ordering keys -> sorted index lists
    // padding rows sort first (key -inf): the stratified levels keep their share
    std::vector<double> rk(n, -1e300), ck(n);
    if (rowkey && colkey) {
        std::copy(rowkey, rowkey + N, rk.begin());
        std::copy(colkey, colkey + M, ck.begin());
    } else {
        MUX_TRY(ctx->ssp.ensure(16ull * n + 256));
        double* d = ctx->ssp.as<double>();
        MUX_CUDA_TRY(cudaMemsetAsync(d, 0, 16ull * n, st));
        rowsum_kernel<<<N, 256, 0, st>>>(W, ldw, M, d, d + n);
        MUX_CUDA_TRY(cudaMemcpyAsync(rk.data(), d, 8ull * N, cudaMemcpyDeviceToHost, st));
        MUX_CUDA_TRY(cudaMemcpyAsync(ck.data(), d + n, 8ull * M, cudaMemcpyDeviceToHost, st));
        MUX_CUDA_TRY(cudaStreamSynchronize(st));
    }
    std::vector<int32_t> ro(n), co(n);
    std::iota(ro.begin(), ro.end(), 0);
    std::iota(co.begin(), co.end(), 0);
    key_order(rk, ro);
    key_order(ck, co);

    // level hierarchy: level 0 = all (original order); level l+1 = every f-th of level l's sorted order
    struct LInfo { int32_t m; std::vector<int32_t> rows, cols, sub; int32_t plo = 0, phi = 0; };
    std::vector<LInfo> lv;
    lv.push_back({n, {}, {}, {}});
    std::vector<int32_t> cur_r = ro, cur_c = co;   // sorted original ids of the current level
    // warm start (price_in: the previous round's optimal column prices): one level
    while (lv.back().m > base && price_in == nullptr) {
        const int32_t m = lv.back().m;
        std::vector<int32_t> nr, nc, sub;
        auto take_k = [&](int32_t k) {
            nr.push_back(cur_r[k]);
            nc.push_back(cur_c[k]);
            // coarse row index within the finer level's row indexing
            sub.push_back(lv.size() == 1 ? cur_r[k] : k);
        };
        if (T.ssp_fx > 0) {   // fractional factor fx / 100: evenly spaced strata
            const int32_t mc = std::max<int32_t>(1, (int32_t)((int64_t)m * 100 / T.ssp_fx));
            for (int32_t i = 0; i < mc; ++i) take_k((int32_t)(((int64_t)(2 * i + 1) * m) / (2 * (int64_t)mc)));
        } else {
            for (int32_t k = fct / 2; k < m; k += fct) take_k(k);
        }
        lv.back().sub = sub;
        LInfo L;
        L.m = (int32_t)nr.size();
        L.rows = nr;
        L.cols = nc;
        if (T.ssp_cperm && nc.size() > 64) {
            // store the level's columns in a golden-ratio stride order: columns next to
            // each other in key order (equal scores, often) then sit in different warps
            // and CTAs of the long-path kernels, whose tie batching sees only warp minima
            const int64_t mm = (int64_t)nc.size();
            int64_t S = ((int64_t)(mm * 0.6180339887) | 1);
            while (std::gcd(S, mm) != 1) S += 2;
            for (int64_t k = 0; k < mm; ++k) L.cols[(size_t)((k * S) % mm)] = nc[(size_t)k];
        }
        lv.push_back(L);
        cur_r = nr;
        cur_c = nc;
    }
    const int nl = (int)lv.size();
    // padding rows of each level (the reference's zero rows when N < M): the
    // original rows N..M-1 at level 0; at coarse levels they sort first
    for (int l = 0; l < nl; ++l) {
        if (N >= M) continue;
        if (l == 0) { lv[l].plo = N; lv[l].phi = M; continue; }
        int32_t np = 0;
        for (int32_t r : lv[l].rows) np += r >= N;
        lv[l].plo = 0;
        lv[l].phi = np;
    }

    // workspace
    size_t off = 0;
    auto take = [&](size_t b) { size_t o = off; off += al256(b); return o; };
    const size_t o_cnt = take(sizeof(Cnt));
    const size_t o_tot = take(32);
    const size_t o_zero = take(sizeof(wt_t) * n + 64);
    std::vector<size_t> o_A(nl), o_p(nl), o_cor(nl), o_roc(nl), o_lock(nl), o_cj(nl), o_ca(nl), o_tau(nl), o_in(nl),
        o_re(nl), o_de(nl), o_tr(nl), o_pi(nl), o_sub(nl), o_rows(nl), o_cols(nl), o_rl(nl);
    for (int l = 0; l < nl; ++l) {
        const size_t m = (size_t)lv[l].m;
        o_A[l] = l ? take(sizeof(wt_t) * m * m) : 0;
        o_p[l] = take(8 * m); o_cor[l] = take(4 * m); o_roc[l] = take(4 * m); o_lock[l] = take(4 * m);
        o_cj[l] = take(4 * m * KC); o_ca[l] = take(sizeof(wt_t) * m * KC); o_tau[l] = take(8 * m);
        o_in[l] = take(4 * m); o_re[l] = take(4 * m); o_de[l] = take(4 * m); o_tr[l] = take(4 * m);
        o_pi[l] = take(8 * m);
        o_sub[l] = take(4 * (lv[l].sub.size() + 1));
        o_rows[l] = take(4 * m); o_cols[l] = take(4 * m);
        o_rl[l] = take(4 * m + 64);
    }
    const size_t o_xd = take(8ull * n), o_xp = take(4ull * n), o_xs = take(4ull * n), o_xc = take(4ull * n + 256),
                 o_xh = take(4ull * n), o_rank = take(4ull * n), o_rowat = take(4ull * n);
    MUX_TRY(ctx->ssp.ensure(off));
    char* B = ctx->ssp.as<char>();
    Cnt* cnt = reinterpret_cast<Cnt*>(B + o_cnt);
    MUX_CUDA_TRY(cudaMemsetAsync(cnt, 0, sizeof(Cnt), st));
    MUX_CUDA_TRY(cudaMemsetAsync(B + o_tot, 0, 8, st));
    MUX_CUDA_TRY(cudaMemsetAsync(B + o_zero, 0, sizeof(wt_t) * n + 64, st));
    const wt_t* zrow = reinterpret_cast<const wt_t*>(B + o_zero);

    // upload index lists and gather the coarse matrices
    for (int l = 1; l < nl; ++l) {
        MUX_CUDA_TRY(cudaMemcpyAsync(B + o_rows[l], lv[l].rows.data(), 4ull * lv[l].m, cudaMemcpyHostToDevice, st));
        MUX_CUDA_TRY(cudaMemcpyAsync(B + o_cols[l], lv[l].cols.data(), 4ull * lv[l].m, cudaMemcpyHostToDevice, st));
        gather_kernel<<<std::min<int32_t>(lv[l].m, 4096), 256, 0, st>>>(
            W, ldw, N, reinterpret_cast<int32_t*>(B + o_rows[l]), reinterpret_cast<int32_t*>(B + o_cols[l]), lv[l].m,
            reinterpret_cast<wt_t*>(B + o_A[l]));
    }
    for (int l = 0; l + 1 < nl; ++l)
        MUX_CUDA_TRY(cudaMemcpyAsync(B + o_sub[l], lv[l].sub.data(), 4ull * lv[l].sub.size(), cudaMemcpyHostToDevice, st));
    std::vector<int32_t> rank0;
    if (T.ssp_rpf > 0) {   // level 0's key ranks for the rank-neighbour prefetch
        rank0.assign(n, 0);
        for (int32_t k = 0; k < n; ++k) rank0[ro[k]] = k;
        MUX_CUDA_TRY(cudaMemcpyAsync(B + o_rank, rank0.data(), 4ull * n, cudaMemcpyHostToDevice, st));
        MUX_CUDA_TRY(cudaMemcpyAsync(B + o_rowat, ro.data(), 4ull * n, cudaMemcpyHostToDevice, st));
    }

    const size_t psmem = sizeof(WTab) * PWARPS;
    // exclusive pass: per-column tables in shared memory when they fit
    int smem_optin = 0;
    MUX_CUDA_TRY(cudaDeviceGetAttribute(&smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, ctx->device));
    const size_t xs_budget = (size_t)smem_optin - 256;
    const size_t xsmem = xs_budget;
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_parallel_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)psmem));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_exclusive_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xsmem));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_dense_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024)));
    // the register-key kernel carries the push-exchange buffers in static shared memory
    const size_t push_b8 = sizeof(CPush<CL>);
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_kernel<1, CL, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024 - push_b8)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_kernel<2, CL, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024 - push_b8)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_kernel<3, CL, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024 - push_b8)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_kernel<4, CL, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024 - push_b8)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_kernel<2, CL, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024 - push_b8)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_kernel<4, CL, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024 - push_b8)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_kernel<6, CL, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024 - push_b8)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_kernel<8, CL, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024 - push_b8)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_kernel<4, CL, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024 - push_b8)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_kernel<8, CL, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024 - push_b8)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_kernel<12, CL, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024 - push_b8)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_kernel<16, CL, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024 - push_b8)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_kernel<1, CL, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024 - push_b8)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_kernel<2, CL, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024 - push_b8)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_slice_kernel<4, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_slice_kernel<6, CL, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_slice_kernel<3, CL, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_slice_kernel<10, CL, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_slice_kernel<16, CL, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey1_kernel<1, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey1_kernel<2, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey1_kernel<3, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey1_kernel<4, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey1_kernel<6, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey1_kernel<1, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey1_kernel<2, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey1_kernel<3, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey1_kernel<5, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey1_kernel<8, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey1_kernel<10, 1024>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024)));
    MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_slice_kernel<CCOLS, CL>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)(xs_budget - 1024)));
    // 16-CTA clusters for the slice kernel when the device can co-schedule them
    bool wide_ok = false;
    static int wide_cache = -1;   // the occupancy query is answered once per process
    if (T.ssp_wide && wide_cache >= 0) {
        wide_ok = wide_cache == 1;
    } else if (T.ssp_wide) {
        MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_slice_kernel<3, 16, 512>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_slice_kernel<6, 16, 512>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_slice_kernel<10, 16, 512>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
        MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_slice_kernel<3, 16, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_slice_kernel<6, 16, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        MUX_CUDA_TRY(cudaFuncSetAttribute(ssp_rkey_slice_kernel<10, 16, 512>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 16;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(16);
        cfg.blockDim = dim3(512);
        cfg.dynamicSmemBytes = 200 * 1024;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int nclusters = 0;
        wide_ok = cudaOccupancyMaxActiveClusters(&nclusters, ssp_rkey_slice_kernel<10, 16, 512>, &cfg) == cudaSuccess &&
                  nclusters >= 1;
        cudaGetLastError();   // a refused query only disables the wide clusters
        wide_cache = wide_ok ? 1 : 0;
    }
    // register-key kernel flags: 4 = runner-up row prefetch into shared memory, 16 = per-pop cycle timing
    const int32_t cpush = (T.ssp_pf ? 4 : 0) | (T.ssp_time ? 16 : 0) | (T.ssp_l2pf ? 32 : 0) | (T.ssp_ties ? 64 : 0);
    const bool use_cluster = T.ssp_cluster;
    int per_sm = 0;
    MUX_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, ssp_parallel_kernel, PWARPS * 32, psmem));
    if (per_sm < 1) { set_error("ssp kernel cannot be resident"); return MUX_ECUDA; }
    int64_t launches = 0;
    Cnt hc{};
    // events are destroyed on every exit path
    struct Events {
        cudaEvent_t e[4] = {nullptr, nullptr, nullptr, nullptr};
        ~Events() { for (auto& x : e) if (x) cudaEventDestroy(x); }
    } evs;
    cudaEvent_t* ev = evs.e;
    for (int k = 0; k < 4; ++k) MUX_CUDA_TRY(cudaEventCreate(&ev[k]));
    double ms_dense = 0, ms_par = 0, dense_bytes = 0;
    int64_t dense_searches = 0, dense_launches = 0;
    unsigned long long xsteps_prev = 0;
    double ms_levels[64] = {0};
    for (int l = nl - 1; l >= 0; --l) {
        auto tl = std::chrono::steady_clock::now();
        const int32_t m = lv[l].m;
        Lvl L{};
        L.A = l ? reinterpret_cast<const wt_t*>(B + o_A[l]) : W;
        L.lda = l ? m : ldw;
        L.m = m;
        L.nreal = l ? m : N;
        L.zrow = zrow;
        L.p = reinterpret_cast<int64_t*>(B + o_p[l]);
        L.cor = reinterpret_cast<int32_t*>(B + o_cor[l]);
        L.roc = reinterpret_cast<int32_t*>(B + o_roc[l]);
        L.lock = reinterpret_cast<int32_t*>(B + o_lock[l]);
        L.cj = reinterpret_cast<int32_t*>(B + o_cj[l]);
        L.ca = reinterpret_cast<wt_t*>(B + o_ca[l]);
        L.tau = reinterpret_cast<int64_t*>(B + o_tau[l]);
        L.retry = reinterpret_cast<int32_t*>(B + o_re[l]);
        L.defer = reinterpret_cast<int32_t*>(B + o_de[l]);
        L.tries = reinterpret_cast<int32_t*>(B + o_tr[l]);
        L.cnt = cnt;
        L.step_budget = step_budget;
        L.deep_budget = deep_budget;
        L.xdist = reinterpret_cast<int64_t*>(B + o_xd);
        L.xpred = reinterpret_cast<int32_t*>(B + o_xp);
        L.xstamp = reinterpret_cast<int32_t*>(B + o_xs);
        L.xscol = reinterpret_cast<int32_t*>(B + o_xc);
        L.xgap = reinterpret_cast<int32_t*>(B + o_xh);
        L.rankof = l == 0 ? reinterpret_cast<const int32_t*>(B + o_rank) : nullptr;
        L.rowat = l == 0 ? reinterpret_cast<const int32_t*>(B + o_rowat) : nullptr;
        L.rpf = (T.ssp_rpf > 0 && sizeof(wt_t) * m * m > ((size_t)T.ssp_rpf_mb << 20)) ? T.ssp_rpf : 0;
        // queue order: a stride permutation spreads concurrent searches over the level
        int32_t stride = 7919;
        while (std::gcd(stride, m) != 1) stride += 2;
        const unsigned g1 = (unsigned)((m + 255) / 256);
        int32_t* in0 = reinterpret_cast<int32_t*>(B + o_in[l]);
        init_level_kernel<<<g1, 256, 0, st>>>(m, L.cor, L.roc, L.lock, L.tries, in0, stride);
        int32_t nwarm = m;   // rows to search (warm start: the unmatched ones)
        // prices
        if (l == nl - 1 && price_in) {
            int64_t* pi = reinterpret_cast<int64_t*>(B + o_pi[l]);
            unsigned long long* pmin = reinterpret_cast<unsigned long long*>(B + o_tot);
            int32_t* wcount = reinterpret_cast<int32_t*>(B + o_tot + 8);
            const unsigned long long big = (unsigned long long)INT64_MAX;
            MUX_CUDA_TRY(cudaMemcpyAsync(pmin, &big, 8, cudaMemcpyHostToDevice, st));
            MUX_CUDA_TRY(cudaMemsetAsync(wcount, 0, 8, st));
            warm_pmin_kernel<<<std::min<unsigned>(g1, 256u), 256, 0, st>>>(price_in, m, pmin);
            warm_profit_kernel<<<(unsigned)(((int64_t)L.nreal * 32 + 255) / 256), 256, 0, st>>>(L.A, L.lda, L.nreal, m,
                                                                                              price_in, pi);
            warm_price_kernel<<<g1, 256, 0, st>>>(L.A, L.lda, L.nreal, m, price_in, pi, pmin, L.p);
            warm_match_kernel<<<(unsigned)((L.nreal + 255) / 256), 256, 0, st>>>(L.A, L.lda, L.nreal, m, warm_col, pi,
                                                                                  L.p, L.cor, L.roc);
            if (L.nreal < m) warm_pad_kernel<<<g1, 256, 0, st>>>(L.nreal, m, m, L.p, pmin, L.cor, L.roc, wcount);
            warm_list_kernel<<<g1, 256, 0, st>>>(0, m, L.cor, in0, wcount + 1);
            MUX_CUDA_TRY(cudaMemcpyAsync(&nwarm, wcount + 1, 4, cudaMemcpyDeviceToHost, st));
            MUX_CUDA_TRY(cudaStreamSynchronize(st));
            launches += 6;
        } else if (l == nl - 1) {
            colmax_kernel<<<g1, 256, 0, st>>>(L.A, L.lda, L.nreal, m, L.p);
        } else {
            const int32_t mc = lv[l + 1].m;
            int64_t* pic = reinterpret_cast<int64_t*>(B + o_pi[l + 1]);
            profit_kernel<<<(unsigned)(((int64_t)mc * 32 + 255) / 256), 256, 0, st>>>(
                reinterpret_cast<const wt_t*>(B + o_A[l + 1]), mc, mc, reinterpret_cast<int32_t*>(B + o_cor[l + 1]),
                reinterpret_cast<int64_t*>(B + o_p[l + 1]), pic);
            fill_i64_kernel<<<g1, 256, 0, st>>>(L.p, m, INT64_MIN);
            const int32_t ksplit = (int32_t)std::max<int64_t>(1, std::min<int64_t>((int64_t)ctx->num_sms * 8 / g1, mc / 64));
            const int32_t chunk = (mc + ksplit - 1) / ksplit;
            ctransform_kernel<<<dim3(g1, (unsigned)((mc + chunk - 1) / chunk)), 256, 0, st>>>(
                L.A, L.lda, L.nreal, L.zrow, m, reinterpret_cast<int32_t*>(B + o_sub[l]), pic, mc, chunk, L.p);
            launches += 3;
        }
        {
            // padding rows share one record (built once, then copied)
            const int32_t cplo = lv[l].phi > lv[l].plo ? lv[l].plo : m, cphi = lv[l].phi > lv[l].plo ? lv[l].phi : m;
            const int64_t built = (int64_t)m - std::max<int32_t>(0, cphi - cplo - 1);
            cand_kernel<<<(unsigned)std::min<int64_t>((built * 32 + 255) / 256, (int64_t)ctx->num_sms * 16), 256, 0, st>>>(
                L, cplo, cphi);
            if (cphi - cplo > 1) {
                const int64_t tot = (int64_t)(cphi - cplo - 1) * KC;
                pad_copy_kernel<<<(unsigned)((tot + 255) / 256), 256, 0, st>>>(L, cplo, cphi);
                ++launches;
            }
        }
        launches += 3;
        double ms_setup = 0;
        if (verbose) {
            MUX_CUDA_TRY(cudaStreamSynchronize(st));
            ms_setup = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tl).count();
        }
        // parallel passes over a row list, then the long paths of the deferred rows
        int32_t* bufs[2] = {L.retry, reinterpret_cast<int32_t*>(B + o_pi[l])};   // pi scratch doubles as 2nd retry list
        int32_t ndef_level = 0, passes_level = 0;
        double ms_par_wall = 0;
        auto solve_rows = [&](const int32_t* list, int32_t nlist) -> int {
        int pass = 0;
        int32_t ndef_total = 0;
        const auto tl2 = std::chrono::steady_clock::now();
        MUX_CUDA_TRY(cudaEventRecord(ev[0], st));
        if (m <= T.ssp_seq && nlist > 0) {
            // tiny level: every row goes straight to the sequential long-path kernel
            // (warps would mostly abort each other on a few dozen columns)
            MUX_CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<int32_t*>(B + o_de[l]), list, 4ull * nlist, cudaMemcpyDeviceToDevice, st));
            ndef_total = nlist;
            nlist = 0;
        }
        while (nlist > 0) {
            if (pass > 0 && nlist <= T.ssp_taildef) {
                // a handful of retried rows: straight to the long-path kernel, which pops
                // as fast as a lone warp and never throws a budget-capped search away
                MUX_CUDA_TRY(cudaMemcpyAsync(reinterpret_cast<int32_t*>(B + o_de[l]) + ndef_total, list, 4ull * nlist,
                                             cudaMemcpyDeviceToDevice, st));
                ndef_total += nlist;
                break;
            }
            L.in = list;
            L.nin = nlist;
            L.retry = bufs[pass & 1];
            L.defer = reinterpret_cast<int32_t*>(B + o_de[l]) + ndef_total;
            MUX_CUDA_TRY(cudaMemsetAsync(cnt, 0, 3 * sizeof(int32_t), st));
            const unsigned grid = (unsigned)std::min<int64_t>((int64_t)ctx->num_sms * per_sm,
                                                              ((int64_t)nlist + PWARPS - 1) / PWARPS);
            const auto tp = std::chrono::steady_clock::now();
            // a handful of rows left: one warp, so they cannot keep aborting each other
            ssp_parallel_kernel<<<grid, PWARPS * 32, psmem, st>>>(L, serial || nlist <= 4);
            ++launches;
            MUX_CUDA_TRY(cudaMemcpyAsync(&hc, cnt, sizeof(Cnt), cudaMemcpyDeviceToHost, st));
            MUX_CUDA_TRY(cudaStreamSynchronize(st));
            if (verbose && l <= 1)
                fprintf(stderr, "[ssp]   pass %d: %d rows, grid %u, %.3f ms -> retry %d defer %d\n", pass, nlist, grid,
                        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tp).count(),
                        hc.nretry, hc.ndefer);
            ndef_total += hc.ndefer;
            list = L.retry;
            nlist = hc.nretry;
            ++pass;
            if (pass > 256) { set_error("ssp: retry passes exceeded"); return MUX_ELIMIT; }
        }
        MUX_CUDA_TRY(cudaEventRecord(ev[1], st));
        ms_par_wall += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tl2).count();
        MUX_CUDA_TRY(cudaEventRecord(ev[2], st));
        // coarse levels only supply warm duals: their long searches are skipped
        // (the partial assignment with its duals is feasible and near-optimal)
        if (ndef_total > 0) {
            L.defer = reinterpret_cast<int32_t*>(B + o_de[l]);
            const size_t dense_bytes = 21ull * m + 64;
            const int32_t mcl = (m + CL - 1) / CL;
            const size_t cl_bytes = (size_t)CBYTES * mcl + 64;
            const int32_t pl = l == 0 ? 0 : coarse_pops;
            if (T.ssp_dorder && ndef_total > 1) {
                // long searches in row-key order (default ascending): in these near-monotone
                // assignments each search shifts a chain of rows toward a free column, and
                // taking the insertions in key order keeps later chains from re-shifting
                // earlier ones (10k rounds: 31k -> 26k pops; 4k: 16.5k -> 10.1k)
                std::vector<int32_t> hd(ndef_total);
                MUX_CUDA_TRY(cudaMemcpyAsync(hd.data(), L.defer, 4ull * ndef_total, cudaMemcpyDeviceToHost, st));
                MUX_CUDA_TRY(cudaStreamSynchronize(st));
                auto key = [&](int32_t r) { return l == 0 ? rk[r] : (double)r; };   // levels >= 1 index rows in key order
                std::stable_sort(hd.begin(), hd.end(), [&](int32_t a, int32_t b) {
                    return T.ssp_dorder == 1 ? key(a) < key(b) : key(a) > key(b);
                });
                MUX_CUDA_TRY(cudaMemcpyAsync(L.defer, hd.data(), 4ull * ndef_total, cudaMemcpyHostToDevice, st));
            }
            if (T.ssp_dump) {
                // analysis dump: header {m, nreal, ndef, level}, A rows [nreal][m], p, roc, cor, defer
                static int seq = 0;
                MUX_CUDA_TRY(cudaStreamSynchronize(st));
                std::vector<wt_t> a((size_t)L.nreal * m);
                MUX_CUDA_TRY(cudaMemcpy2D(a.data(), sizeof(wt_t) * m, L.A, sizeof(wt_t) * L.lda, sizeof(wt_t) * m, L.nreal,
                                          cudaMemcpyDeviceToHost));
                std::vector<int64_t> hp(m);
                std::vector<int32_t> hroc(m), hcor(m), hdef(ndef_total);
                MUX_CUDA_TRY(cudaMemcpy(hp.data(), L.p, 8ull * m, cudaMemcpyDeviceToHost));
                MUX_CUDA_TRY(cudaMemcpy(hroc.data(), L.roc, 4ull * m, cudaMemcpyDeviceToHost));
                MUX_CUDA_TRY(cudaMemcpy(hcor.data(), L.cor, 4ull * m, cudaMemcpyDeviceToHost));
                MUX_CUDA_TRY(cudaMemcpy(hdef.data(), L.defer, 4ull * ndef_total, cudaMemcpyDeviceToHost));
                const std::string path = std::string(T.ssp_dump) + "/lvl" + std::to_string(l) + "_" + std::to_string(seq++) + ".bin";
                if (FILE* f = fopen(path.c_str(), "wb")) {
                    const int32_t hdr[5] = {m, L.nreal, ndef_total, l, (int32_t)sizeof(wt_t)};
                    fwrite(hdr, 4, 5, f);
                    fwrite(a.data(), sizeof(wt_t), a.size(), f);
                    fwrite(hp.data(), 8, m, f);
                    fwrite(hroc.data(), 4, m, f);
                    fwrite(hcor.data(), 4, m, f);
                    fwrite(hdef.data(), 4, ndef_total, f);
                    fclose(f);
                }
            }
            // register-key kernel: 12 m replicated + 4 bytes per local column + two row-slice buffers
            const size_t rk_bytes = 16ull * m + 16 + 4ull * mcl + 128 + 2ull * sizeof(wt_t) * ((mcl + 8 + 3) & ~3) + 64;
            const bool rkey_ok = use_cluster && mcl <= 512 * 4 && rk_bytes <= xs_budget - 2048 - push_b8 && T.ssp_rslice != 2;
            const bool slice_ok = use_cluster && m <= CL * CTHREADS * CCOLS && cl_bytes <= xs_budget - 2048;
            // single SM for levels up to T.ssp_one columns: one barrier per pop, no DSMEM
            const size_t r1_bytes = 20ull * m + 24;
            const bool rkey1_ok = m <= T.ssp_one && m <= 1024 * 10 && r1_bytes <= xs_budget - 2048;
            if (rkey1_ok) {
                // 512 threads (128 registers: the tie rows stay in registers) up to 3072 columns
                if (T.ssp_ct1 == 512 && m <= 512) ssp_rkey1_kernel<1, 512><<<1, 512, r1_bytes, st>>>(L, ndef_total, pl, cpush);
                else if (T.ssp_ct1 == 512 && m <= 1024) ssp_rkey1_kernel<2, 512><<<1, 512, r1_bytes, st>>>(L, ndef_total, pl, cpush);
                else if (T.ssp_ct1 == 512 && m <= 1536) ssp_rkey1_kernel<3, 512><<<1, 512, r1_bytes, st>>>(L, ndef_total, pl, cpush);
                else if (T.ssp_ct1 == 512 && m <= 2048) ssp_rkey1_kernel<4, 512><<<1, 512, r1_bytes, st>>>(L, ndef_total, pl, cpush);
                else if (T.ssp_ct1 == 512 && m <= 3072) ssp_rkey1_kernel<6, 512><<<1, 512, r1_bytes, st>>>(L, ndef_total, pl, cpush);
                else if (m <= 1024) ssp_rkey1_kernel<1, 1024><<<1, 1024, r1_bytes, st>>>(L, ndef_total, pl, cpush);
                else if (m <= 2048) ssp_rkey1_kernel<2, 1024><<<1, 1024, r1_bytes, st>>>(L, ndef_total, pl, cpush);
                else if (m <= 3072) ssp_rkey1_kernel<3, 1024><<<1, 1024, r1_bytes, st>>>(L, ndef_total, pl, cpush);
                else if (m <= 5120) ssp_rkey1_kernel<5, 1024><<<1, 1024, r1_bytes, st>>>(L, ndef_total, pl, cpush);
                else if (m <= 8192) ssp_rkey1_kernel<8, 1024><<<1, 1024, r1_bytes, st>>>(L, ndef_total, pl, cpush);
                else ssp_rkey1_kernel<10, 1024><<<1, 1024, r1_bytes, st>>>(L, ndef_total, pl, cpush);
            } else if (rkey_ok) {
                // 256 threads per CTA (default): fewer warps per barrier, 1.16 -> 1.08 us/pop at 10k
                // against 512; 128 / 512 / 1024 stay selectable (MUX_SSP_CT) for A/B runs
                if (T.ssp_ct == 256) {
                    if (mcl <= 512) ssp_rkey_kernel<2, CL, 256><<<CL, 256, rk_bytes, st>>>(L, ndef_total, pl, cpush);
                    else if (mcl <= 1024) ssp_rkey_kernel<4, CL, 256><<<CL, 256, rk_bytes, st>>>(L, ndef_total, pl, cpush);
                    else if (mcl <= 1536) ssp_rkey_kernel<6, CL, 256><<<CL, 256, rk_bytes, st>>>(L, ndef_total, pl, cpush);
                    else ssp_rkey_kernel<8, CL, 256><<<CL, 256, rk_bytes, st>>>(L, ndef_total, pl, cpush);
                } else if (T.ssp_ct == 128) {
                    if (mcl <= 512) ssp_rkey_kernel<4, CL, 128><<<CL, 128, rk_bytes, st>>>(L, ndef_total, pl, cpush);
                    else if (mcl <= 1024) ssp_rkey_kernel<8, CL, 128><<<CL, 128, rk_bytes, st>>>(L, ndef_total, pl, cpush);
                    else if (mcl <= 1536) ssp_rkey_kernel<12, CL, 128><<<CL, 128, rk_bytes, st>>>(L, ndef_total, pl, cpush);
                    else ssp_rkey_kernel<16, CL, 128><<<CL, 128, rk_bytes, st>>>(L, ndef_total, pl, cpush);
                } else if (T.ssp_ct == 1024) {
                    if (mcl <= 1024) ssp_rkey_kernel<1, CL, 1024><<<CL, 1024, rk_bytes, st>>>(L, ndef_total, pl, cpush);
                    else ssp_rkey_kernel<2, CL, 1024><<<CL, 1024, rk_bytes, st>>>(L, ndef_total, pl, cpush);
                } else if (mcl <= 512) ssp_rkey_kernel<1, CL, 512><<<CL, 512, rk_bytes, st>>>(L, ndef_total, pl, cpush);
                else if (mcl <= 1024) ssp_rkey_kernel<2, CL, 512><<<CL, 512, rk_bytes, st>>>(L, ndef_total, pl, cpush);
                else if (mcl <= 1536) ssp_rkey_kernel<3, CL, 512><<<CL, 512, rk_bytes, st>>>(L, ndef_total, pl, cpush);
                else ssp_rkey_kernel<4, CL, 512><<<CL, 512, rk_bytes, st>>>(L, ndef_total, pl, cpush);
            } else if (use_cluster && T.ssp_rslice > 0 && mcl <= 512 * 16) {
                // register keys with (key, owner | price) pushes: no replicated tables
                const size_t rs_bytes = 4ull * mcl + 64;
                const int32_t m16 = (m + 15) / 16;
                // local path walk (flag 128) when 16-bit indices and 4 m more bytes per CTA fit
                const bool lw = n <= 65535 && T.ssp_lwalk;
                if (wide_ok && m16 <= 512 * 10) {
                    // 16-CTA clusters (non-portable size): half the columns per CTA
                    // (10k x 40k: 156 -> 143 ms of long paths, profiles/r03/cluster16_slice.log)
                    size_t rs16 = 4ull * m16 + 64;
                    int32_t f16 = cpush;
                    if (lw && rs16 + 4ull * m + 64 <= 200ull * 1024) { rs16 += 4ull * m + 64; f16 |= 128; }
                    if (m16 <= 512 * 3) ssp_rkey_slice_kernel<3, 16, 512><<<16, 512, rs16, st>>>(L, ndef_total, pl, f16);
                    else if (m16 <= 512 * 6) ssp_rkey_slice_kernel<6, 16, 512><<<16, 512, rs16, st>>>(L, ndef_total, pl, f16);
                    else ssp_rkey_slice_kernel<10, 16, 512><<<16, 512, rs16, st>>>(L, ndef_total, pl, f16);
                } else {
                    size_t rsb = rs_bytes;
                    int32_t f8 = cpush;
                    if (lw && rsb + 4ull * m + 64 <= 200ull * 1024) { rsb += 4ull * m + 64; f8 |= 128; }
                    if (mcl <= 512 * 3) ssp_rkey_slice_kernel<3, CL, 512><<<CL, 512, rsb, st>>>(L, ndef_total, pl, f8);
                    else if (mcl <= 512 * 6) ssp_rkey_slice_kernel<6, CL, 512><<<CL, 512, rsb, st>>>(L, ndef_total, pl, f8);
                    else if (mcl <= 512 * 10) ssp_rkey_slice_kernel<10, CL, 512><<<CL, 512, rsb, st>>>(L, ndef_total, pl, f8);
                    else ssp_rkey_slice_kernel<16, CL, 512><<<CL, 512, rsb, st>>>(L, ndef_total, pl, f8);
                }
            } else if (slice_ok) {
                if (m <= CL * CTHREADS * 4) ssp_slice_kernel<4, CL><<<CL, CTHREADS, cl_bytes, st>>>(L, ndef_total, pl);
                else ssp_slice_kernel<CCOLS, CL><<<CL, CTHREADS, cl_bytes, st>>>(L, ndef_total, pl);
            } else if (m <= DTHREADS * DCOLS && dense_bytes <= xs_budget - 1024 && !T.ssp_sparsex) {
                // long searches: dense Dijkstra on one CTA, tables in shared memory
                ssp_dense_kernel<<<1, DTHREADS, dense_bytes, st>>>(L, ndef_total);
            } else {
                const size_t per_col = 17ull * m;
                const bool xs_fit = per_col + 4ull * 1024 <= xs_budget;
                const int32_t ocap = xs_fit ? (int32_t)std::min<size_t>((xs_budget - per_col) / 4 - 16, (size_t)m + 64)
                                            : m + 64;
                ssp_exclusive_kernel<<<1, 32, xs_fit ? xsmem : 0, st>>>(L, ndef_total, xs_fit ? 1 : 0, ocap);
            }
            ++launches;
        }
        MUX_CUDA_TRY(cudaEventRecord(ev[3], st));
        MUX_CUDA_TRY(cudaGetLastError());
        MUX_CUDA_TRY(cudaMemcpyAsync(&hc, cnt, sizeof(Cnt), cudaMemcpyDeviceToHost, st));
        MUX_CUDA_TRY(cudaStreamSynchronize(st));
        {
            float a = 0, b = 0;
            cudaEventElapsedTime(&a, ev[0], ev[1]);
            cudaEventElapsedTime(&b, ev[2], ev[3]);
            ms_par += a;
            ms_dense += b;
            dense_bytes += 4.0 * (double)m * (double)(hc.xsteps - xsteps_prev);
            xsteps_prev = hc.xsteps;
            dense_searches += ndef_total;
            dense_launches += ndef_total > 0 ? 1 : 0;
        }
        ndef_level += ndef_total;
        passes_level += pass;
        return MUX_OK;
        };
        const int32_t plo = lv[l].plo, phi = lv[l].phi;
        if (phi <= plo || price_in) {
            MUX_TRY(solve_rows(in0, nwarm));
        } else {
            // real rows first (their searches never meet padding rows, which are
            // all still free), then the interchangeable padding rows: in bulk on
            // the free columns at the minimum price (tight for them), the rest
            // by search.  Row order never changes the optimum.
            int32_t* real = reinterpret_cast<int32_t*>(B + o_rl[l]);
            int32_t* cnts = reinterpret_cast<int32_t*>(B + o_tot + 8);
            unsigned long long* pmin = reinterpret_cast<unsigned long long*>(B + o_tot);
            MUX_CUDA_TRY(cudaMemsetAsync(cnts, 0, 16, st));
            split_rows_kernel<<<g1, 256, 0, st>>>(m, in0, plo, phi, real, cnts);
            int32_t nr = 0;
            MUX_CUDA_TRY(cudaMemcpyAsync(&nr, cnts, 4, cudaMemcpyDeviceToHost, st));
            MUX_CUDA_TRY(cudaStreamSynchronize(st));
            MUX_TRY(solve_rows(real, nr));
            const unsigned long long big = (unsigned long long)INT64_MAX;
            MUX_CUDA_TRY(cudaMemcpyAsync(pmin, &big, 8, cudaMemcpyHostToDevice, st));
            warm_pmin_kernel<<<std::min<unsigned>(g1, 256u), 256, 0, st>>>(L.p, m, pmin);
            warm_pad_kernel<<<g1, 256, 0, st>>>(plo, phi, m, L.p, pmin, L.cor, L.roc, cnts + 1);
            warm_list_kernel<<<(unsigned)((phi - plo + 255) / 256), 256, 0, st>>>(plo, phi, L.cor, real, cnts + 2);
            int32_t np = 0;
            MUX_CUDA_TRY(cudaMemcpyAsync(&np, cnts + 2, 4, cudaMemcpyDeviceToHost, st));
            MUX_CUDA_TRY(cudaStreamSynchronize(st));
            launches += 4;
            if (np > 0) MUX_TRY(solve_rows(real, np));
        }
        const int32_t ndef_total = ndef_level;
        const int pass = passes_level;

        if (hc.errors) {
            set_error(std::string("ssp: device error flags ") + std::to_string(hc.errors));
            return MUX_ELIMIT;
        }
        if (check && (l == 0 || coarse_exact)) {
            unsigned long long* bad = reinterpret_cast<unsigned long long*>(B + o_tot);
            MUX_CUDA_TRY(cudaMemsetAsync(bad, 0, 32, st));
            check_kernel<<<m, 256, 0, st>>>(L.A, L.lda, L.nreal, L.zrow, m, L.cor, L.roc, L.p, bad);
            unsigned long long hb[4] = {0, 0, 0, 0};
            MUX_CUDA_TRY(cudaMemcpyAsync(hb, bad, 32, cudaMemcpyDeviceToHost, st));
            MUX_CUDA_TRY(cudaStreamSynchronize(st));
            if (hb[0] || hb[1] || hb[2]) {
                set_error("ssp: dual certificate failed at level " + std::to_string(l) + ": unmatched " + std::to_string(hb[0]) +
                          ", inconsistent " + std::to_string(hb[1]) + ", dual violations " + std::to_string(hb[2]) +
                          " (first row " + std::to_string(hb[3] >> 32) + " col " + std::to_string(hb[3] & 0xffffffffu) +
                          "; deferred rows " + std::to_string(ndef_total) + ")");
                return MUX_ELIMIT;
            }
        }
        ms_levels[l] = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - tl).count();
        if (verbose)
            fprintf(stderr, "[ssp] level %d m %d: %.3f ms (setup %.3f parallel %.3f) passes %d deferred %d | steps %llu deep %llu aborts %llu "
                            "augs %llu xsteps %llu xrounds %llu xdeep %llu refresh %llu | xcyc pop %.2e deep %.2e step %.2e aug %.2e\n",
                    l, m, ms_levels[l], ms_setup, ms_par_wall, pass, ndef_total, hc.steps, hc.deep, hc.aborts, hc.augs, hc.xsteps, hc.xrounds, hc.xdeep,
                    hc.refresh, (double)hc.xcyc[0], (double)hc.xcyc[1], (double)hc.xcyc[2], (double)hc.xcyc[3]);
    }
    // level 0 result
    const int32_t* cor0 = reinterpret_cast<int32_t*>(B + o_cor[0]);
    unsigned long long* tot = reinterpret_cast<unsigned long long*>(B + o_tot);
    MUX_CUDA_TRY(cudaMemsetAsync(tot, 0, 8, st));
    finish_kernel<<<(unsigned)((N + 255) / 256), 256, 0, st>>>(W, ldw, N, cor0, col_out, tot);
    ++launches;
    if (price_out) MUX_CUDA_TRY(cudaMemcpyAsync(price_out, B + o_p[0], 8ull * n, cudaMemcpyDeviceToDevice, st));
    if (cor_out) MUX_CUDA_TRY(cudaMemcpyAsync(cor_out, B + o_cor[0], 4ull * n, cudaMemcpyDeviceToDevice, st));
    if (roc_out) MUX_CUDA_TRY(cudaMemcpyAsync(roc_out, B + o_roc[0], 4ull * n, cudaMemcpyDeviceToDevice, st));
    unsigned long long ht = 0;
    MUX_CUDA_TRY(cudaMemcpyAsync(&ht, tot, 8, cudaMemcpyDeviceToHost, st));
    MUX_CUDA_TRY(cudaStreamSynchronize(st));
    if (total_q) *total_q = (int64_t)ht;
    const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
    if (stats) {
        stats->n_rows = N; stats->n_cols = M; stats->n_square = n;
        stats->phases = nl;
        stats->rounds = (int64_t)hc.xrounds;
        stats->bids = (int64_t)(hc.steps + hc.xsteps);
        stats->row_scans = (int64_t)(hc.deep + hc.xdeep + hc.refresh);
        stats->tail_bids = (int64_t)hc.xsteps;
        stats->total_q = (int64_t)ht;
        stats->ms_match = ms;
        stats->ms_kernel = ms;
        stats->launches += launches;
        stats->levels = nl;
        stats->par_steps = (int64_t)hc.steps;
        stats->dense_steps = (int64_t)hc.xsteps;
        stats->dense_searches = dense_searches;
        stats->ms_dense = ms_dense;
        stats->ms_parallel = ms_par;
        stats->dense_bytes = dense_bytes;
        stats->dense_launches = dense_launches;
    }
    if (verbose) fprintf(stderr, "[ssp] n %d levels %d total %.3f ms (host wall), dense %.3f ms, parallel %.3f ms\n", n, nl, ms,
                         ms_dense, ms_par);
    if (cpush & 16) {
        const double k = hc.xcyc[2] > 0 ? (double)hc.xcyc[2] : 1.0;
        fprintf(stderr, "[ssp-time] pops %lld cycles/pop (CTA 0 warp 0): load+relax %.0f exchange %.0f | prefetch hits %.3f"
                        " | searches %llu walk steps %llu (%.0f cycles each) end-of-search sync %.0f cycles each\n",
                (long long)hc.xcyc[2], hc.xcyc[0] / k, hc.xcyc[1] / k, (double)hc.xpfhits / (double)std::max(1ull, hc.xsteps),
                hc.xsearch, hc.xwalk, (double)hc.xwalkcyc / (double)std::max(1ull, hc.xwalk),
                (double)hc.xsynccyc / (double)std::max(1ull, hc.xsearch));
        fprintf(stderr, "[ssp-time] register-key steps %llu: push-to-arrival %.0f cycles | prefetch-hit %llu (load+relax %.0f cycles), "
                        "tie steps %llu (load+relax %.0f)\n",
                hc.xrounds, (double)hc.xt[4] / (double)std::max(1ull, hc.xrounds), hc.xt[1],
                (double)hc.xt[0] / (double)std::max(1ull, hc.xt[1]), hc.xt[3], (double)hc.xt[2] / (double)std::max(1ull, hc.xt[3]));
    }
    return MUX_OK;
}
