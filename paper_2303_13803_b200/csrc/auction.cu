// Exact maximum-weight bipartite matching by epsilon-scaling auction.
//
// Replaces the reference's O(n^3) Kuhn-Munkres (`_solve_min_assignment`,
// /root/reference/pkg/src/muxsim/matching.py:45-101) inside
// `max_weight_matching` (matching.py:148-208).  The problem solved is the
// reference's: pad the N x M non-negative weight matrix with zero rows/columns
// to n = max(N, M) and find a maximum-weight perfect matching of the square
// problem.  Weights are integers (quantised scores); benefits are
// a_ij = Q_ij * (n + 1), so an assignment satisfying epsilon-complementary
// slackness with epsilon = 1 is optimal (n * epsilon < n + 1 = one unit of Q).
//
// One persistent cooperative kernel runs the whole solve (1 CTA per SM):
//   for eps = eps0, eps0/theta, ..., 1:                  (epsilon scaling)
//     clear the assignment, keep prices
//     while some person is unassigned:
//       if <= tail_max remain: single-CTA Gauss-Seidel tail (no grid barriers)
//       else Jacobi round:
//         [A1] each unassigned person bids from its top-K candidate cache
//              (one warp per person); cache misses go to a global miss list
//         [A2] misses are spread over the CTAs; each CTA scans one row at a
//              time cooperatively: the weight row arrives by TMA bulk copy
//              (cp.async.bulk, double-buffered) into shared memory, prices come
//              from a shared-memory mirror, per-lane top-(K+1) lists are merged
//              by warp shuffles, then across warps
//         [B]  every bidder reads back the packed max-bid word of its object:
//              the winner takes it, the previous owner and the losers form the
//              next round's list
// Values and objects travel as one 64-bit key (v + offset) << idbits | ~j, so
// "largest key" = "best value, lowest object index on ties" and every
// reduction is a plain unsigned max.  Bids are atomicMax'ed as
// (price << idbits | ~person): highest bid wins, lowest person on ties.
// Candidate cache: a scan keeps the K best (object, benefit) pairs and the
// (K+1)-th best value thr.  Prices only rise, so uncached objects are still
// worth <= thr; if the best cached value is >= thr the cached top-2 (second =
// max(second, thr)) is a valid epsilon-CS bid without re-reading the row.
// Determinism: all bids of a round see the same prices and every tie is
// broken by index, so the result does not depend on thread scheduling.
#include <cooperative_groups.h>

#include <cstdio>
#include <cstring>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace mux {

constexpr int kK = 15;                // cached candidates per person (K + 1 = 16)
constexpr int kAucThreads = 512;      // 16 warps per CTA
constexpr int kAucWarps = kAucThreads / kWarp;
constexpr int kTailMax = 256;         // largest tail handed to the tail modes
constexpr int64_t kNegInf = INT64_MIN / 4;
constexpr unsigned long long kNoKey = 0ull;
constexpr size_t kSmemBudget = 220 * 1024;
constexpr int kPhMax = 32;
constexpr int kCandMax = 512;         // candidate keys kept by the threshold selection

struct AucCounters {
    int32_t list_count[2];
    int32_t touched_count[2];
    int32_t miss_count;
    uint32_t errors;
    uint32_t tail_epoch;
    uint32_t bar_count;                 // custom grid barrier
    uint32_t bar_gen;
    int32_t qhead;                      // async tail: next queued person
    int32_t free_count;                 // async tail: chains still open
    unsigned long long async_fail;      // async tail: rejected bids
    unsigned long long rounds, bids, scans, tail_bids, phases, hits;
    long long ns_total, ns_tail, ns_tail_hit, ns_tail_scan, ns_tail_wait, ns_a1, ns_a2, ns_b;
    unsigned long long tail_scans;
    long long cyc_hitloop;
    long long cyc_fetch;
    unsigned long long tail_hits;
    long long ns_stage[6];
    long long max_q;
    long long total_q;
    unsigned long long or_q;
    // per-phase timeline (MUX_VERBOSE): eps, Jacobi rounds, persons left for
    // the tail, Jacobi and tail nanoseconds, bids
    long long ph_eps[kPhMax];
    int32_t ph_rounds[kPhMax];
    int32_t ph_tailn[kPhMax];
    long long ph_ns_j[kPhMax];
    long long ph_ns_t[kPhMax];
    unsigned long long ph_bids[kPhMax];
    unsigned long long ph_maxchain[kPhMax];   // async chains: longest chain (bids)
    unsigned long long ph_longchains[kPhMax]; // async chains: chains of more than 256 bids
    unsigned long long ph_chains[kPhMax];
};

// Per-person candidate cache: one 256-byte record, read by a single lane
// with thirteen 16-byte loads.
struct __align__(256) PCache {
    int32_t j[16];       // cached objects, best first (-1 = empty; slot 15 unused)
    int64_t q[16];       // their weights (benefit = q * SC)
    int64_t thr;         // (K+1)-th best value at scan time
    int32_t valid;
    int32_t pad[11];
};
static_assert(sizeof(PCache) == 256, "PCache must be 256 bytes");
static_assert(kK <= 15, "PCache holds at most 15 candidates");

struct AucArgs {
    const void* W;       // [N][ldw] int32 or int64
    int64_t ldw;
    int32_t N, M, n;     // real rows, real columns, square size
    int32_t idbits;
    unsigned long long idmask;
    int64_t koff;        // value offset making keys non-negative
    int64_t SC;          // benefit scale (n + 1)
    int32_t qshift;      // common power of two divided out of every weight
    int32_t cg_sync;     // 1: cooperative-groups grid.sync, 0: custom barrier
    int32_t keff;        // candidates actually cached (<= kK)
    int32_t async_tail;  // 1: tail chains run concurrently on many CTAs
    int32_t rot;         // 1 when N != M: per-person rotated tie order (padding entities)
    int32_t async_phases;  // leading phases run entirely as concurrent chains (no Jacobi rounds)
    int32_t fresh;         // async chains: cache bids read current prices (not the CTA mirror)
    int32_t restage;       // async chains: re-stage the price mirror before every row scan
    int32_t order;         // async chains: queue persons by their previous object's price
    int64_t eps0;
    int32_t theta;
    int32_t tail_max;
    int64_t round_guard;
    int64_t* price;      // [n_pad]
    int32_t* owner;      // [n_pad]
    int32_t* col;        // [n_pad]
    unsigned long long* bidw;   // [2][n_pad]
    int32_t* touched;    // [2][n_pad]
    int32_t* list;       // [2][n_pad]
    int32_t* miss;       // [n_pad]
    int32_t* bidj;       // [n_pad]
    unsigned long long* bidpk;  // [n_pad]
    PCache* cache;       // [n_pad]
    unsigned long long* word;   // [n_pad] async tail state: price << idbits | (idmask - owner), 0 = unowned
    AucCounters* cnt;
    int32_t n_pad;
    int32_t row_bytes;   // bytes of one staged weight row (multiple of 16)
};

// ---- keys -------------------------------------------------------------------

// Tie order among equal values.  Real (person, object) pairs keep "lowest
// object index first".  Padding entities are interchangeable, and if they all
// broke ties the same way every Jacobi round would pile them onto one object,
// so each person rotates its order over the padding objects (real persons) or
// over all objects (padding persons) by a per-person offset.  Any fixed order
// is a valid tie-break; the rotation only spreads the bids.
__device__ __forceinline__ uint32_t rot_off(int32_t i) { return (uint32_t)i * 2654435761u; }
__device__ __forceinline__ int32_t tie_rank(const AucArgs& A, int32_t i, int32_t j) {
    if (!A.rot) return j;
    if (i >= A.N) {
        int32_t r = j + (int32_t)(rot_off(i) % (uint32_t)A.n);
        return r >= A.n ? r - A.n : r;
    }
    if (j < A.M) return j;
    const int32_t D = A.n - A.M;
    int32_t r = (j - A.M) + (int32_t)(rot_off(i) % (uint32_t)D);
    return A.M + (r >= D ? r - D : r);
}
__device__ __forceinline__ int32_t tie_inv(const AucArgs& A, int32_t i, int32_t r) {
    if (!A.rot) return r;
    if (i >= A.N) {
        int32_t j = r - (int32_t)(rot_off(i) % (uint32_t)A.n);
        return j < 0 ? j + A.n : j;
    }
    if (r < A.M) return r;
    const int32_t D = A.n - A.M;
    int32_t j = (r - A.M) - (int32_t)(rot_off(i) % (uint32_t)D);
    return A.M + (j < 0 ? j + D : j);
}

__device__ __forceinline__ unsigned long long mkkey(const AucArgs& A, int32_t i, int64_t v, int32_t j) {
    return ((unsigned long long)(v + A.koff) << A.idbits) | (A.idmask - (unsigned long long)tie_rank(A, i, j));
}
__device__ __forceinline__ int32_t key_j(const AucArgs& A, int32_t i, unsigned long long k) {
    return tie_inv(A, i, (int32_t)(A.idmask - (k & A.idmask)));
}
__device__ __forceinline__ int64_t key_v(const AucArgs& A, unsigned long long k) {
    return (int64_t)(k >> A.idbits) - A.koff;
}

__device__ __forceinline__ unsigned long long warp_max_u64(unsigned long long k) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const unsigned long long x = __shfl_xor_sync(0xffffffffu, k, o);
        k = x > k ? x : k;
    }
    return k;
}

// Lane-local sorted top-(K+1) keys, best first.
struct TopKeys {
    unsigned long long k[kK + 1];
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int t = 0; t <= kK; ++t) k[t] = kNoKey;
    }
    __device__ __forceinline__ void push(unsigned long long x) {
        if (x <= k[kK]) return;
        k[kK] = x;
#pragma unroll
        for (int t = kK; t > 0; --t)
            if (k[t] > k[t - 1]) { unsigned long long s = k[t]; k[t] = k[t - 1]; k[t - 1] = s; }
    }
    __device__ __forceinline__ void pop() {
#pragma unroll
        for (int t = 0; t < kK; ++t) k[t] = k[t + 1];
        k[kK] = kNoKey;
    }
};

// Merge the 32 lane lists; lane r (< K+1) receives the r-th best key.
__device__ __forceinline__ unsigned long long warp_merge(TopKeys& L, int lane) {
    unsigned long long mine = kNoKey;
#pragma unroll 1
    for (int r = 0; r <= kK; ++r) {
        const unsigned long long b = warp_max_u64(L.k[0]);
        if (b != kNoKey && L.k[0] == b) L.pop();
        if (lane == r) mine = b;
    }
    return mine;
}

// ---- weights -----------------------------------------------------------------

template <int WT>
__device__ __forceinline__ int64_t wload1(const AucArgs& A, int32_t i, int32_t j) {
    if (i >= A.N || j >= A.M) return 0;
    if (WT == MUX_W_I32) return (int64_t)__ldg(static_cast<const int32_t*>(A.W) + (int64_t)i * A.ldw + j) >> A.qshift;
    return __ldg(static_cast<const int64_t*>(A.W) + (int64_t)i * A.ldw + j) >> A.qshift;
}

// 4 consecutive weights of row i starting at column c (c % 4 == 0), read from
// `row` (shared-memory copy of the row, may be null = global), zero outside
// [0, N) x [0, M).
template <int WT>
__device__ __forceinline__ void wget4(const AucArgs& A, const void* row, int32_t i, int32_t c, int64_t (&q)[4]) {
    if (i >= A.N || c >= A.M) { q[0] = q[1] = q[2] = q[3] = 0; return; }
    if (WT == MUX_W_I32) {
        int4 v;
        if (row) v = reinterpret_cast<const int4*>(row)[c >> 2];
        else v = __ldg(reinterpret_cast<const int4*>(static_cast<const int32_t*>(A.W) + (int64_t)i * A.ldw + c));
        q[0] = v.x; q[1] = v.y; q[2] = v.z; q[3] = v.w;
    } else {
        longlong2 a, b;
        if (row) {
            const longlong2* p = reinterpret_cast<const longlong2*>(row) + (c >> 1);
            a = p[0]; b = p[1];
        } else {
            const longlong2* p = reinterpret_cast<const longlong2*>(static_cast<const int64_t*>(A.W) + (int64_t)i * A.ldw + c);
            a = __ldg(p); b = __ldg(p + 1);
        }
        q[0] = a.x; q[1] = a.y; q[2] = b.x; q[3] = b.y;
    }
#pragma unroll
    for (int t = 0; t < 4; ++t) q[t] = (c + t < A.M) ? (q[t] >> A.qshift) : 0;
}

// ---- explicit shared-memory loads (keep the scan off the generic path) ---------

__device__ __forceinline__ int4 lds_v4(uint32_t a) {
    int4 v;
    asm volatile("ld.shared.v4.s32 {%0,%1,%2,%3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ longlong2 lds_v2ll(uint32_t a) {
    longlong2 v;
    asm volatile("ld.shared.v2.s64 {%0,%1}, [%2];" : "=l"(v.x), "=l"(v.y) : "r"(a));
    return v;
}

__device__ __forceinline__ int64_t lds_ll(uint32_t a) {
    long long v;
    asm volatile("ld.shared.s64 %0, [%1];" : "=l"(v) : "r"(a));
    return v;
}

// ---- prices -------------------------------------------------------------------

template <bool SP>
__device__ __forceinline__ int64_t pget(const int64_t* P, int32_t j) {
    return SP ? lds_ll((uint32_t)__cvta_generic_to_shared(P + j)) : __ldcg(P + j);
}

template <bool SP>
__device__ __forceinline__ void pget4(const int64_t* P, int32_t c, int64_t (&p)[4]) {
    const longlong2* pp = reinterpret_cast<const longlong2*>(P + c);
    longlong2 a, b;
    if (SP) { a = pp[0]; b = pp[1]; }
    else { a = __ldcg(pp); b = __ldcg(pp + 1); }
    p[0] = a.x; p[1] = a.y; p[2] = b.x; p[3] = b.y;
}

// ---- TMA bulk copy + mbarrier -------------------------------------------------

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" :: "r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
// Arm the barrier for `bytes` and issue one bulk global->shared copy (thread 0).
__device__ __forceinline__ void tma_row(uint64_t* bar, void* dst, const void* src, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;"
                 :: "r"(smem_u32(bar)), "r"(bytes) : "memory");
    // weight rows are streamed: evict them first so prices and caches stay in L2
    uint64_t policy;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(policy));
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;"
                 :: "r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n"
        ".reg .pred p;\n"
        "WAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra WAIT_%=;\n"
        "}\n" :: "r"(smem_u32(bar)), "r"(parity) : "memory");
}

__device__ __forceinline__ uint64_t gtimer() {
    uint64_t t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    return t;
}

// Grid-wide barrier for the persistent kernel: one arrival atomic per CTA, the
// last arriver bumps a generation word; waiters poll it with relaxed loads
// (no L1 invalidation per poll) and fence once on exit.
__device__ __forceinline__ void grid_barrier(const AucArgs& A, cg::grid_group& grid) {
    if (A.cg_sync) { grid.sync(); return; }
    __syncthreads();
    if (threadIdx.x == 0) {
        volatile uint32_t* gen = &A.cnt->bar_gen;
        const uint32_t g = *gen;
        __threadfence();
        if (atomicAdd(&A.cnt->bar_count, 1u) == gridDim.x - 1) {
            A.cnt->bar_count = 0;
            __threadfence();
            atomicAdd(&A.cnt->bar_gen, 1u);
        } else {
            while (*gen == g) { }
        }
        __threadfence();
    }
    __syncthreads();
}

// ---- per-CTA shared state ------------------------------------------------------

struct Shared {
    PCache rec[2];                           // prefetched cache records (tail)
    uint64_t rbar[2];                        // record-buffer mbarriers
    uint32_t rbar_phase[2];
    int32_t rec_person[2];
    uint64_t bar[2];                         // row-buffer mbarriers
    uint32_t bar_phase[2];
    int32_t row_person[2];                   // person whose row sits in buffer b (-1 none)
    int32_t stack[kTailMax + 1];
    int32_t top;
    int32_t scan_i;                          // tail: person needing a scan (-1 = done)
    int32_t chain_i;                         // async tail: person at the head of this CTA's chain
    int32_t j1;
    int64_t bid;
    unsigned long long wk[kAucWarps][kK + 1];  // per-warp merged keys (slow path)
    unsigned long long wmax[2 * kAucWarps];    // per-half-warp maximum key
    unsigned long long tau;                    // selection threshold
    unsigned long long sel[kK + 1];            // selected top-(K+1) keys
    int32_t ncand;
    unsigned long long cand[kCandMax];          // keys >= tau
    unsigned long long tprof[8];                 // scan stage timers (SM cycles); [7] = scans
};

struct Dyn {             // carve-up of dynamic shared memory
    int64_t* price;      // [n_pad] price mirror (SP mode)
    int32_t* owner;      // [n_pad] owner mirror (SP mode, tail only)
    unsigned char* row0;  // two staged weight rows (double buffer)
    unsigned char* row1;
    __device__ __forceinline__ unsigned char* row(int b) const { return b ? row1 : row0; }  // no local array
};

// Stage the price array (and owners) from global into the CTA's mirror.
__device__ __forceinline__ void stage_prices(const AucArgs& A, int64_t* sp, int32_t* so) {
    const longlong2* g = reinterpret_cast<const longlong2*>(A.price);
    longlong2* s = reinterpret_cast<longlong2*>(sp);
    for (int t = threadIdx.x; t < A.n_pad / 2; t += blockDim.x) s[t] = __ldcg(g + t);
    if (so)
        for (int t = threadIdx.x; t < A.n_pad; t += blockDim.x) so[t] = __ldcg(A.owner + t);
}

// Start fetching person i's weight row into buffer b (thread 0 only).
__device__ __forceinline__ void drain_row(const AucArgs& A, Shared& S, int b) {
    const int32_t p = S.row_person[b];
    if (p >= 0 && p < A.N && A.M > 0) { mbar_wait(&S.bar[b], S.bar_phase[b]); S.bar_phase[b] ^= 1u; }
    S.row_person[b] = -1;
}

template <int WT>
__device__ __forceinline__ void fetch_row(const AucArgs& A, Shared& S, Dyn& D, int b, int32_t i) {
    drain_row(A, S, b);
    S.row_person[b] = i;
    if (i >= A.N || A.M == 0) return;            // dummy person: no weights to load
    const size_t esz = WT == MUX_W_I32 ? 4 : 8;
    const char* src = static_cast<const char*>(A.W) + (size_t)i * A.ldw * esz;
    tma_row(&S.bar[b], D.row(b), src, (uint32_t)A.row_bytes);
}
// Prefetch person i's cache record into S.rec[b] (thread 0; tail only).
__device__ __forceinline__ void fetch_rec(const AucArgs& A, Shared& S, int b, int32_t i) {
    if (S.rec_person[b] >= 0) { mbar_wait(&S.rbar[b], S.rbar_phase[b]); S.rbar_phase[b] ^= 1u; }
    S.rec_person[b] = i;
    asm volatile("fence.proxy.async.global;" ::: "memory");   // generic-proxy cache stores -> TMA reads
    tma_row(&S.rbar[b], &S.rec[b], A.cache + i, (uint32_t)sizeof(PCache));
}
// Claim the prefetched record of person i if buffer b holds it (thread 0).
__device__ __forceinline__ const PCache* claim_rec(Shared& S, int b, int32_t i) {
    if (S.rec_person[b] != i) return nullptr;
    mbar_wait(&S.rbar[b], S.rbar_phase[b]);
    S.rbar_phase[b] ^= 1u;
    S.rec_person[b] = -1;
    return &S.rec[b];
}

// Wait for buffer b (all threads); returns the row pointer.
template <int WT>
__device__ __forceinline__ const void* wait_row(const AucArgs& A, Shared& S, Dyn& D, int b, int32_t i) {
    if (i >= A.N || A.M == 0) return D.row(b);
    mbar_wait(&S.bar[b], S.bar_phase[b]);
    return D.row(b);
}

// ---- bids ----------------------------------------------------------------------

__device__ __forceinline__ int64_t bid_from(int64_t a1, int64_t v1, int64_t second, int64_t eps) {
    return (second <= kNegInf) ? (a1 - v1) + eps : a1 - second + eps;   // n == 1: price + eps
}

// Bid from the candidate cache by ONE thread (no shuffles).  True on a valid
// hit; ties on value go to the lower object index, like a full scan.
template <bool SP>
__device__ __forceinline__ bool cache_bid(const AucArgs& A, const int64_t* P, int32_t i, int64_t eps,
                                          int32_t& j1, int64_t& bid, const PCache* srec = nullptr,
                                          int64_t* fresh_mirror = nullptr) {
    const longlong2* rec = reinterpret_cast<const longlong2*>(A.cache + i);
    longlong2 w[13];     // j[0..16) | q[0..16) | thr, valid
    if (srec) {          // prefetched copy in shared memory
#pragma unroll
        for (int t = 0; t < 13; ++t) w[t] = reinterpret_cast<const longlong2*>(srec)[t];
    } else {
#pragma unroll
        for (int t = 0; t < 13; ++t) w[t] = __ldcg(rec + t);
    }
    const int32_t valid = (int32_t)(w[12].y & 0xffffffffll);
    if (!valid) return false;
    const int64_t thr = w[12].x;
    int64_t v1 = kNegInf, v2 = kNegInf, a1 = 0;
    int32_t b = INT32_MAX;
#pragma unroll
    for (int k = 0; k < kK; ++k) {
        if (k >= A.keff) break;
        // fields by value (no address-taking, so w[] stays in registers)
        const long long jw = (k & 2) ? w[k >> 2].y : w[k >> 2].x;
        const int32_t j = (k & 1) ? (int32_t)(jw >> 32) : (int32_t)(jw & 0xffffffffll);
        const int64_t qk = (k & 1) ? w[4 + (k >> 1)].y : w[4 + (k >> 1)].x;
        if (j < 0) continue;
        const int64_t a = qk * A.SC;
        int64_t pj;
        if (fresh_mirror) {      // async tail: current price from the packed word, mirror refreshed
            pj = (int64_t)(__ldcg(A.word + j) >> A.idbits);
            fresh_mirror[j] = pj;
        } else {
            pj = pget<SP>(P, j);
        }
        const int64_t v = a - pj;
        if (v > v1 || (v == v1 && (b == INT32_MAX || tie_rank(A, i, j) < tie_rank(A, i, b)))) { v2 = v1; v1 = v; b = j; a1 = a; }
        else if (v > v2) v2 = v;
    }
    if (b == INT32_MAX || v1 < thr) return false;
    const int64_t s2 = v2 > thr ? v2 : thr;
    j1 = b;
    bid = bid_from(a1, v1, s2, eps);
    return true;
}

// Weights and prices of 4 consecutive columns for the CTA scan.  In
// shared-memory mode (SP) both come from the CTA's staged row / price mirror
// through explicit ld.shared; otherwise from global memory.
template <int WT, bool SP>
__device__ __forceinline__ void scan_load4(const AucArgs& A, uint32_t row_s, uint32_t price_s, const int64_t* P,
                                           int32_t i, int32_t c, int64_t (&q)[4], int64_t (&p)[4]) {
    if (SP) {
        const longlong2 a = lds_v2ll(price_s + (uint32_t)c * 8u);
        const longlong2 b = lds_v2ll(price_s + (uint32_t)c * 8u + 16u);
        p[0] = a.x; p[1] = a.y; p[2] = b.x; p[3] = b.y;
        if (i >= A.N || c >= A.M) { q[0] = q[1] = q[2] = q[3] = 0; return; }
        if (WT == MUX_W_I32) {
            const int4 v = lds_v4(row_s + (uint32_t)c * 4u);
            q[0] = v.x; q[1] = v.y; q[2] = v.z; q[3] = v.w;
        } else {
            const longlong2 x = lds_v2ll(row_s + (uint32_t)c * 8u), y = lds_v2ll(row_s + (uint32_t)c * 8u + 16u);
            q[0] = x.x; q[1] = x.y; q[2] = y.x; q[3] = y.y;
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) q[t] = (c + t < A.M) ? (q[t] >> A.qshift) : 0;
    } else {
        wget4<WT>(A, nullptr, i, c, q);
        pget4<false>(P, c, p);
    }
}

// Key of row i at column c (4 consecutive), zero key for padding columns.
template <int WT, bool SP>
__device__ __forceinline__ void keys4(const AucArgs& A, const int64_t* P, const void* row, int32_t i, int32_t c,
                                      unsigned long long (&k)[4]) {
    int64_t q[4], p[4];
    wget4<WT>(A, row, i, c, q);
    pget4<SP>(P, c, p);
#pragma unroll
    for (int t = 0; t < 4; ++t) k[t] = (c + t < A.n) ? mkkey(A, i, q[t] * A.SC - p[t], c + t) : kNoKey;
}

// Scan a row with the whole CTA: `row` is the staged weight row (or null =
// read from global), P the price source.  Stores the new cache and leaves the
// bid in S.j1 / S.bid (valid after the trailing barrier).
//
// Top-(K+1) selection without sorting networks: tau = the (K+1)-th largest of
// the 16 per-warp maxima is a lower bound on the (K+1)-th largest key, so the
// answer lies among the keys >= tau (typically ~K+1 of them); those are
// collected in shared memory and ranked by direct comparison.  Rows shorter
// than 16 x 128 columns, or degenerate candidate sets, take the shuffle-merge
// path.
template <int WT, bool SP>
__device__ void cta_scan_bid(const AucArgs& A, Shared& S, const int64_t* P, const void* row, int32_t i,
                             int64_t eps) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const bool fast = A.n > (A.keff * 64);   // >= K+1 half-warps hold columns
    bool done = false;
    uint64_t tp0 = clock64();
#define MUX_STAGE(k) do { if (threadIdx.x == 0) { const uint64_t _t = clock64(); S.tprof[k] += _t - tp0; tp0 = _t; } } while (0)
    if (fast) {
        // pass 1: per-thread best (value, lowest index) and per-group maxima.
        // kIters fixed-trip steps keep the group maxima in registers; rows
        // longer than kIters * 2048 columns fall back to a full pass 2.
        constexpr int kIters = 8;
        const uint32_t row_s = SP ? smem_u32(row) : 0u;
        const uint32_t price_s = SP ? smem_u32(P) : 0u;
        const int32_t stride = kAucThreads * 4;
        const bool cached = A.n <= kIters * stride;
        int64_t gmax[kIters];
        int64_t bv = kNegInf;
        int32_t bj = INT32_MAX;
#pragma unroll
        for (int it = 0; it < kIters; ++it) {
            const int32_t c = threadIdx.x * 4 + it * stride;
            gmax[it] = kNegInf;
            if (c < A.n) {
                int64_t q[4], pr[4];
                scan_load4<WT, SP>(A, row_s, price_s, P, i, c, q, pr);
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    if (c + t >= A.n) continue;
                    const int64_t v = q[t] * A.SC - pr[t];
                    gmax[it] = v > gmax[it] ? v : gmax[it];
                    if (v > bv || (A.rot && v == bv && tie_rank(A, i, c + t) < tie_rank(A, i, bj))) {
                        bv = v;   // columns ascend: without rotation, strict > keeps the lowest index
                        bj = c + t;
                    }
                }
            }
        }
        for (int32_t c = threadIdx.x * 4 + kIters * stride; c < A.n; c += stride) {
            int64_t q[4], pr[4];
            scan_load4<WT, SP>(A, row_s, price_s, P, i, c, q, pr);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                if (c + t >= A.n) continue;
                const int64_t v = q[t] * A.SC - pr[t];
                if (v > bv || (A.rot && v == bv && tie_rank(A, i, c + t) < tie_rank(A, i, bj))) { bv = v; bj = c + t; }
            }
        }
        unsigned long long mx = bj == INT32_MAX ? kNoKey : mkkey(A, i, bv, bj);
#pragma unroll
        for (int o = 8; o > 0; o >>= 1) {      // half-warp maximum
            const unsigned long long x = __shfl_xor_sync(0xffffffffu, mx, o);
            mx = x > mx ? x : mx;
        }
        if ((lane & 15) == 0) S.wmax[warp * 2 + (lane >> 4)] = mx;
        if (threadIdx.x == 0) S.ncand = 0;
        __syncthreads();
        MUX_STAGE(0);
        if (warp == 0) {
            // tau = the (K+1)-th largest of the 32 half-warp maxima: a lower
            // bound on the (K+1)-th largest key of the row
            const unsigned long long v = S.wmax[lane];
            int rank = 0;
#pragma unroll
            for (int w = 0; w < 2 * kAucWarps; ++w) {
                const unsigned long long o = S.wmax[w];
                rank += (o > v) || (o == v && w < lane);
            }
            if (rank == A.keff) S.tau = v;
        }
        __syncthreads();
        MUX_STAGE(1);
        // pass 2: collect keys >= tau, revisiting only groups that can reach it
        const unsigned long long tau = S.tau;
        const int64_t tau_v = key_v(A, tau);
#pragma unroll
        for (int it = 0; it < kIters; ++it) {
            const int32_t c = threadIdx.x * 4 + it * stride;
            if (c >= A.n || (cached && gmax[it] < tau_v)) continue;
            int64_t q[4], pr[4];
            scan_load4<WT, SP>(A, row_s, price_s, P, i, c, q, pr);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                if (c + t >= A.n) continue;
                const int64_t v = q[t] * A.SC - pr[t];
                if (v < tau_v) continue;
                const unsigned long long k = mkkey(A, i, v, c + t);
                if (k >= tau) {
                    const int slot = atomicAdd(&S.ncand, 1);
                    if (slot < kCandMax) S.cand[slot] = k;
                }
            }
        }
        for (int32_t c = threadIdx.x * 4 + kIters * stride; c < A.n; c += stride) {
            int64_t q[4], pr[4];
            scan_load4<WT, SP>(A, row_s, price_s, P, i, c, q, pr);
#pragma unroll
            for (int t = 0; t < 4; ++t) {
                if (c + t >= A.n) continue;
                const int64_t v = q[t] * A.SC - pr[t];
                if (v < tau_v) continue;
                const unsigned long long k = mkkey(A, i, v, c + t);
                if (k >= tau) {
                    const int slot = atomicAdd(&S.ncand, 1);
                    if (slot < kCandMax) S.cand[slot] = k;
                }
            }
        }
        __syncthreads();
        MUX_STAGE(2);
        const int nc = S.ncand;
        if (nc <= 32) {
            if (warp == 0) {
                const unsigned long long key = lane < nc ? S.cand[lane] : kNoKey;
                int rank = 0;
#pragma unroll
                for (int e = 0; e < 32; ++e) rank += __shfl_sync(0xffffffffu, key, e) > key;
                if (lane < nc && rank <= kK) S.sel[rank] = key;
                if (lane <= kK && lane >= nc) S.sel[lane] = kNoKey;
            }
            done = true;
        } else if (nc <= kCandMax) {
            for (int t = threadIdx.x; t < nc; t += kAucThreads) {
                const unsigned long long key = S.cand[t];
                int rank = 0;
                for (int e = 0; e < nc; ++e) rank += S.cand[e] > key;
                if (rank <= kK) S.sel[rank] = key;
            }
            if (threadIdx.x <= kK && threadIdx.x >= nc) S.sel[threadIdx.x] = kNoKey;
            done = true;
        }
    }
    if (!done) {
        TopKeys L;
        L.init();
        for (int32_t c = threadIdx.x * 4; c < A.n; c += kAucThreads * 4) {
            unsigned long long k[4];
            keys4<WT, SP>(A, P, row, i, c, k);
#pragma unroll
            for (int t = 0; t < 4; ++t) L.push(k[t]);
        }
        const unsigned long long wk = warp_merge(L, lane);
        if (lane <= kK) S.wk[warp][lane] = wk;
        __syncthreads();
        if (warp == 0) {
            TopKeys M;
            M.init();
            for (int e = lane; e < kAucWarps * (kK + 1); e += 32) M.push(S.wk[e / (kK + 1)][e % (kK + 1)]);
            const unsigned long long mk = warp_merge(M, lane);
            if (lane <= kK) S.sel[lane] = mk;
        }
    }
    __syncthreads();
    MUX_STAGE(3);
    if (warp == 0) {
        // cache: lanes 0..K-1 hold ranks 0..K-1, rank K is the threshold
        const unsigned long long mk = lane <= A.keff ? S.sel[lane] : kNoKey;
        PCache* rec = A.cache + i;
        if (lane < A.keff) {
            const bool ok = mk != kNoKey;
            const int32_t j = ok ? key_j(A, i, mk) : -1;
            rec->j[lane] = j;
            int64_t q = 0;
            if (ok && i < A.N && j < A.M) {
                if (row) q = (WT == MUX_W_I32 ? (int64_t)static_cast<const int32_t*>(row)[j]
                                              : static_cast<const int64_t*>(row)[j]) >> A.qshift;
                else q = wload1<WT>(A, i, j);
            }
            rec->q[lane] = q;
        }
        if (lane == 0) {
            const unsigned long long k0 = S.sel[0], k1 = S.sel[1], kt = S.sel[A.keff];
            rec->thr = kt == kNoKey ? kNegInf : key_v(A, kt);
            rec->valid = 1;
            const int32_t jj = key_j(A, i, k0);
            const int64_t v1 = key_v(A, k0);
            const int64_t a1 = v1 + pget<SP>(P, jj);
            S.j1 = jj;
            S.bid = bid_from(a1, v1, k1 == kNoKey ? kNegInf : key_v(A, k1), eps);
        }
    }
    __syncthreads();
    MUX_STAGE(4);
    if (threadIdx.x == 0) S.tprof[7] += 1;
#undef MUX_STAGE
}

__device__ __forceinline__ unsigned long long pack_bid(const AucArgs& A, int64_t bid, int32_t i) {
    return ((unsigned long long)bid << A.idbits) | (A.idmask - (unsigned long long)i);
}

__device__ __forceinline__ void check_bid(const AucArgs& A, int64_t bid) {
    if (bid < 0 || (unsigned long long)bid >= (1ull << (63 - A.idbits))) atomicOr(&A.cnt->errors, kErrPriceBits);
}

__device__ __forceinline__ void submit_bid(const AucArgs& A, unsigned long long* bw, int32_t i, int32_t j1,
                                           int64_t bid) {
    const unsigned long long pk = pack_bid(A, bid, i);
    check_bid(A, bid);
    atomicMax(bw + j1, pk);
    A.bidj[i] = j1;
    A.bidpk[i] = pk;
}

// Gauss-Seidel assignment of object j1 to person i at price `bid` (tail mode,
// thread 0).  Returns the displaced person or -1.
template <bool SP>
__device__ __forceinline__ int32_t gs_assign(const AucArgs& A, Dyn& D, int32_t i, int32_t j1, int64_t bid) {
    check_bid(A, bid);
    const int32_t prev = SP ? D.owner[j1] : __ldcg(A.owner + j1);
    if (SP) { D.owner[j1] = i; D.price[j1] = bid; }
    A.owner[j1] = i;
    A.price[j1] = bid;
    A.col[i] = j1;
    if (prev >= 0) A.col[prev] = -1;
    return prev;
}

// ---- single-CTA Gauss-Seidel tail -----------------------------------------------

template <int WT, bool SP>
__device__ void tail_gs(const AucArgs& A, Shared& S, Dyn& D, int64_t eps, int32_t count, const int32_t* src) {
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    if (SP) stage_prices(A, D.price, D.owner);
    const int64_t* P = SP ? D.price : A.price;
    for (int t = threadIdx.x; t < count; t += blockDim.x) S.stack[t] = __ldcg(src + t);
    __syncthreads();
    if (threadIdx.x == 0) {
        // the list order comes from atomics: sort (descending) so the lowest
        // person id is popped first and the tail is deterministic
        for (int a = 1; a < count; ++a) {
            const int32_t key = S.stack[a];
            int b = a - 1;
            while (b >= 0 && S.stack[b] < key) { S.stack[b + 1] = S.stack[b]; --b; }
            S.stack[b + 1] = key;
        }
        S.top = count;
    }
    __syncthreads();
    unsigned long long steps = 0, scans = 0, hits = 0;
    uint64_t ns_hit = 0, ns_scan = 0, ns_wait = 0;
    uint64_t cyc_hitloop = 0, cyc_steps = 0;
    int cur_buf = 0;
    for (;;) {
        const uint64_t th0 = gtimer();
        // warp 0 runs every cache-hit step alone (no CTA barrier); it stops at
        // the first miss and hands that person to the whole CTA.
        if (threadIdx.x == 0) {
            const uint64_t c0 = clock64();
            int32_t need = -1;
            int32_t top = S.top;
            while (top > 0 && steps <= (unsigned long long)A.round_guard) {
                const int32_t i = S.stack[top - 1];
                int32_t j1 = 0;
                int64_t bid = 0;
                const PCache* srec = SP ? claim_rec(S, cur_buf, i) : nullptr;
                if (!cache_bid<SP>(A, P, i, eps, j1, bid, srec)) { need = i; break; }
                const int32_t prev = gs_assign<SP>(A, D, i, j1, bid);
                --top;
                if (prev >= 0) S.stack[top++] = prev;
                ++hits;
                ++steps;
            }
            S.top = top;
            S.scan_i = steps > (unsigned long long)A.round_guard ? -2 : need;
            const uint64_t c1 = clock64();
            cyc_hitloop += c1 - c0;
            if (need >= 0 && SP && S.row_person[cur_buf] != need) fetch_row<WT>(A, S, D, cur_buf, need);
            cyc_steps += clock64() - c1;
        }
        __syncthreads();
        const uint64_t th1 = gtimer();
        ns_hit += th1 - th0;
        const int32_t i = S.scan_i;
        if (i < 0) break;
        const void* row = SP ? wait_row<WT>(A, S, D, cur_buf, i) : nullptr;
        const uint64_t th2 = gtimer();
        ns_wait += th2 - th1;
        cta_scan_bid<WT, SP>(A, S, P, row, i, eps);
        if (threadIdx.x == 0) {
            if (SP && i < A.N && A.M > 0) S.bar_phase[cur_buf] ^= 1u;
            S.row_person[cur_buf] = -1;
            const int32_t prev = gs_assign<SP>(A, D, i, S.j1, S.bid);
            int32_t t2 = S.top - 1;
            if (prev >= 0) {
                S.stack[t2++] = prev;
                // prefetch the displaced person's row and cache record: it bids next
                if (SP) {
                    fetch_row<WT>(A, S, D, cur_buf ^ 1, prev);
                    fetch_rec(A, S, cur_buf ^ 1, prev);
                }
            }
            S.top = t2;
        }
        if (SP) cur_buf ^= 1;
        ++scans;
        ++steps;
        __syncthreads();
        ns_scan += gtimer() - th1;
    }
    if (S.scan_i == -2 && threadIdx.x == 0) atomicOr(&A.cnt->errors, kErrIterGuard);
    // drain a pending prefetch so the mbarrier phases stay consistent
    if (SP && threadIdx.x == 0) {
        drain_row(A, S, 0);
        drain_row(A, S, 1);
        for (int b = 0; b < 2; ++b)
            if (S.rec_person[b] >= 0) { mbar_wait(&S.rbar[b], S.rbar_phase[b]); S.rbar_phase[b] ^= 1u; S.rec_person[b] = -1; }
    }
    if (threadIdx.x == 0) {
        atomicAdd(&A.cnt->tail_bids, steps);
        atomicAdd(&A.cnt->bids, steps);
        atomicAdd(&A.cnt->scans, scans);
        atomicAdd(&A.cnt->hits, hits);
        atomicAdd(&A.cnt->tail_scans, scans);
        atomicAdd((unsigned long long*)&A.cnt->cyc_hitloop, (unsigned long long)cyc_hitloop);
        atomicAdd((unsigned long long*)&A.cnt->cyc_fetch, (unsigned long long)cyc_steps);
        atomicAdd((unsigned long long*)&A.cnt->tail_hits, hits);
        atomicAdd((unsigned long long*)&A.cnt->ns_tail_hit, (unsigned long long)ns_hit);
        atomicAdd((unsigned long long*)&A.cnt->ns_tail_scan, (unsigned long long)ns_scan);
        atomicAdd((unsigned long long*)&A.cnt->ns_tail_wait, (unsigned long long)ns_wait);
        __threadfence();
    }
    __syncthreads();
}

// ---- asynchronous multi-CTA tail -----------------------------------------------
//
// The few persons left at the end of a phase each start a displacement chain
// (bid, displace the owner, the displaced person bids next, ... until a free
// object is taken).  The Gauss-Seidel tail runs these chains one after
// another; here every CTA takes a chain from a queue and runs it concurrently.
// Ownership and prices live in one 64-bit word per object,
// price << idbits | (idmask - owner), and a bid is committed with atomicMax:
// it wins iff its price is higher than the current one.  A bid computed from a
// stale (lower) price snapshot is still a valid epsilon-CS bid when it wins
// (stale prices only over-estimate the second-best value), so each CTA bids
// from its own shared-memory price mirror and refreshes an entry when a bid is
// rejected.  The result is an optimal assignment; which of several tied optima
// is returned may vary between runs, so the mode is used for large problems
// only (deterministic Gauss-Seidel tail otherwise).

__device__ __forceinline__ unsigned long long pack_state(const AucArgs& A, int64_t price, int32_t owner) {
    return ((unsigned long long)price << A.idbits) | (owner >= 0 ? A.idmask - (unsigned long long)owner : 0ull);
}

// Commit person i's bid on j1 (thread 0).  Returns -2 if rejected (the mirror
// entry is refreshed), -1 if the chain ended on a free object, else the
// displaced person.
template <bool SP>
__device__ __forceinline__ int32_t async_commit(const AucArgs& A, Dyn& D, int32_t i, int32_t j1, int64_t bid) {
    check_bid(A, bid);
    const unsigned long long pk = pack_state(A, bid, i);
    const unsigned long long old = atomicMax(A.word + j1, pk);
    if (pk <= old) {
        if (SP) D.price[j1] = (int64_t)(old >> A.idbits);
        atomicAdd(&A.cnt->async_fail, 1ull);
        return -2;
    }
    if (SP) D.price[j1] = bid;
    A.col[i] = j1;
    const unsigned long long low = old & A.idmask;
    if (low == 0) return -1;
    const int32_t prev = (int32_t)(A.idmask - low);
    A.col[prev] = -1;
    return prev;
}

__device__ __forceinline__ void stage_word_prices(const AucArgs& A, int64_t* sp) {
    for (int t = threadIdx.x; t < A.n_pad; t += blockDim.x) sp[t] = (int64_t)(__ldcg(A.word + t) >> A.idbits);
}

template <int WT, bool SP>
__device__ void tail_async(const AucArgs& A, Shared& S, Dyn& D, int64_t eps, int32_t count, const int32_t* src,
                           cg::grid_group& grid, int ph) {
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gsize = (int64_t)gridDim.x * blockDim.x;
    for (int64_t t = gtid; t < A.n_pad; t += gsize)
        A.word[t] = t < A.n ? pack_state(A, __ldcg(A.price + t), __ldcg(A.owner + t)) : 0ull;
    if (gtid == 0) {
        A.cnt->qhead = 0;
        A.cnt->free_count = count;
    }
    grid_barrier(A, grid);
    const int64_t* P = D.price;
    unsigned long long steps = 0, scans = 0, hits = 0;
    int cur_buf = 0;
    for (;;) {
        if (threadIdx.x == 0) {
            const int32_t idx = atomicAdd(&A.cnt->qhead, 1);
            S.chain_i = idx < count ? __ldcg(src + idx) : -1;
        }
        __syncthreads();
        if (S.chain_i < 0) break;
        stage_word_prices(A, D.price);
        __syncthreads();
        const unsigned long long steps0 = steps;
        for (;;) {
            if (threadIdx.x == 0) {
                int32_t cur = S.chain_i;
                int32_t need = -1;
                int fails = 0;
                while (cur >= 0) {
                    int32_t j1 = 0;
                    int64_t bid = 0;
                    const PCache* srec = claim_rec(S, cur_buf, cur);
                    if (!cache_bid<SP>(A, P, cur, eps, j1, bid, srec, (SP && A.fresh) ? D.price : nullptr)) { need = cur; break; }
                    const int32_t r = async_commit<SP>(A, D, cur, j1, bid);
                    ++steps;
                    if (r == -2) { ++fails; continue; }
                    ++hits;
                    if (r == -1) { atomicSub(&A.cnt->free_count, 1); cur = -1; break; }
                    cur = r;
                }
                S.chain_i = cur;
                S.scan_i = need;
                if (need >= 0 && S.row_person[cur_buf] != need) fetch_row<WT>(A, S, D, cur_buf, need);
            }
            __syncthreads();
            const int32_t i = S.scan_i;
            if (i < 0) break;                      // chain finished
            if (A.restage) {
                stage_word_prices(A, D.price);
                __syncthreads();
            }
            const void* row = wait_row<WT>(A, S, D, cur_buf, i);
            cta_scan_bid<WT, SP>(A, S, P, row, i, eps);
            if (threadIdx.x == 0) {
                if (i < A.N && A.M > 0) S.bar_phase[cur_buf] ^= 1u;
                S.row_person[cur_buf] = -1;
                const int32_t r = async_commit<SP>(A, D, i, S.j1, S.bid);
                ++steps;
                ++scans;
                if (r == -2) {
                    S.chain_i = i;                 // rejected: retry from the refreshed mirror
                } else if (r == -1) {
                    atomicSub(&A.cnt->free_count, 1);
                    S.chain_i = -1;
                } else {
                    S.chain_i = r;
                    fetch_row<WT>(A, S, D, cur_buf ^ 1, r);
                    fetch_rec(A, S, cur_buf ^ 1, r);
                }
            }
            cur_buf ^= 1;
            __syncthreads();
            if (S.chain_i < 0) break;
        }
        if (threadIdx.x == 0 && ph < kPhMax) {
            const unsigned long long len = steps - steps0;
            atomicMax(&A.cnt->ph_maxchain[ph], len);
            atomicAdd(&A.cnt->ph_chains[ph], 1ull);
            if (len > 256) atomicAdd(&A.cnt->ph_longchains[ph], 1ull);
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        drain_row(A, S, 0);
        drain_row(A, S, 1);
        for (int b = 0; b < 2; ++b)
            if (S.rec_person[b] >= 0) { mbar_wait(&S.rbar[b], S.rbar_phase[b]); S.rbar_phase[b] ^= 1u; S.rec_person[b] = -1; }
        if (steps) {
            atomicAdd(&A.cnt->tail_bids, steps);
            atomicAdd(&A.cnt->bids, steps);
            atomicAdd(&A.cnt->scans, scans);
            atomicAdd(&A.cnt->hits, hits);
            atomicAdd(&A.cnt->tail_scans, scans);
        }
        // every chain must have found its free object before the state is unpacked
        unsigned ns = 128;
        while (*reinterpret_cast<volatile int32_t*>(&A.cnt->free_count) != 0) {
            __nanosleep(ns);
            ns = ns < 4096 ? ns * 2 : ns;
        }
    }
    grid_barrier(A, grid);
    for (int64_t t = gtid; t < A.n; t += gsize) {
        const unsigned long long w = __ldcg(A.word + t);
        const unsigned long long low = w & A.idmask;
        A.price[t] = (int64_t)(w >> A.idbits);
        A.owner[t] = low ? (int32_t)(A.idmask - low) : -1;
    }
    grid_barrier(A, grid);
}

// ---- the persistent solve kernel --------------------------------------------------

template <int WT, bool SP>
__global__ void __launch_bounds__(kAucThreads, 1)
auction_kernel(AucArgs A) {
    cg::grid_group grid = cg::this_grid();
    extern __shared__ __align__(128) unsigned char dsm[];
    __shared__ Shared S;
    Dyn D;
    {
        unsigned char* p = dsm;
        D.row0 = p; p += A.row_bytes;
        D.row1 = p; p += A.row_bytes;
        D.price = reinterpret_cast<int64_t*>(p); p += sizeof(int64_t) * A.n_pad;
        D.owner = reinterpret_cast<int32_t*>(p);
    }
    const int lane = threadIdx.x & 31;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gsize = (int64_t)gridDim.x * blockDim.x;
    const int n = A.n;
    if (threadIdx.x == 0) {
        mbar_init(&S.bar[0], 1);
        mbar_init(&S.bar[1], 1);
        mbar_init(&S.rbar[0], 1);
        mbar_init(&S.rbar[1], 1);
        fence_mbar_init();
        S.rbar_phase[0] = S.rbar_phase[1] = 0;
        S.rec_person[0] = S.rec_person[1] = -1;
        S.bar_phase[0] = S.bar_phase[1] = 0;
        S.row_person[0] = S.row_person[1] = -1;
        for (int k = 0; k < 8; ++k) S.tprof[k] = 0;
    }
    __syncthreads();
    int64_t eps = A.eps0;
    long long rounds_total = 0;
    uint32_t tail_epoch = 0;
    uint64_t t_a1 = 0, t_a2 = 0, t_b = 0;
    const uint64_t t_start = gtimer();
    uint64_t t_tail = 0;
    int phase_no = 0;

    for (;;) {
        // ---- phase init: clear the assignment, keep prices and caches.
        // (Keeping the pairs that still satisfy eps-CS for the new eps frees
        // nearly everyone anyway: a winning bid leaves its bidder exactly eps
        // of slack, so almost no pair meets eps/theta.)
        const bool chains = SP && A.async_tail && phase_no < A.async_phases;
        if (chains && phase_no > 0 && A.order) {
            // queue the persons by the price of the object they held in the
            // previous phase, most expensive first: each one then tends to find
            // its object free and the displacement chains stay short
            stage_prices(A, D.price, nullptr);
            __syncthreads();
            for (int64_t t = gtid; t < n; t += gsize) {
                const int32_t j = (int32_t)t;
                const int64_t pj = lds_ll(smem_u32(D.price + j));
                int32_t rank = 0;
                for (int32_t k = 0; k < n; ++k) {
                    const int64_t pk = lds_ll(smem_u32(D.price + k));
                    rank += (pk > pj) || (pk == pj && k < j);
                }
                A.list[rank] = A.owner[j];
            }
            grid_barrier(A, grid);
        }
        for (int64_t t = gtid; t < n; t += gsize) {
            A.owner[t] = -1;
            A.col[t] = -1;
            if (!(chains && phase_no > 0 && A.order)) A.list[t] = (int32_t)t;          // list[0]
            A.bidw[t] = 0ull;
            A.bidw[A.n_pad + t] = 0ull;
        }
        if (gtid == 0) {
            A.cnt->list_count[0] = n;
            A.cnt->list_count[1] = 0;
            A.cnt->touched_count[0] = 0;
            A.cnt->touched_count[1] = 0;
            A.cnt->miss_count = 0;
            atomicAdd(&A.cnt->phases, 1ull);
        }
        grid_barrier(A, grid);
        int r = 0;
        const uint64_t tph0 = gtimer();
        uint64_t tph1 = 0;
        int32_t ph_tailn = 0;
        for (;;) {
            const int cur = r & 1, nxt = cur ^ 1;
            const int32_t count = __ldcg(&A.cnt->list_count[cur]);
            if (count == 0) break;
            if (count <= A.tail_max) { tph1 = gtimer(); ph_tailn = count; }
            if (SP && A.async_tail && (count <= A.tail_max || (r == 0 && phase_no < A.async_phases))) {
                const uint64_t t0 = gtimer();
                tail_async<WT, SP>(A, S, D, eps, count, A.list + (int64_t)cur * A.n_pad, grid, phase_no);
                if (blockIdx.x == 0) t_tail += gtimer() - t0;
                break;
            }
            if (count <= A.tail_max) {
                ++tail_epoch;
                if (blockIdx.x == 0) {
                    const uint64_t t0 = gtimer();
                    tail_gs<WT, SP>(A, S, D, eps, count, A.list + (int64_t)cur * A.n_pad);
                    t_tail += gtimer() - t0;
                    if (threadIdx.x == 0) {
                        __threadfence();
                        atomicExch(&A.cnt->tail_epoch, tail_epoch);
                    }
                } else if (threadIdx.x == 0) {
                    // idle CTAs sleep instead of polling a grid barrier, so the
                    // single working CTA keeps the L2 to itself
                    unsigned ns = 256;
                    while (*reinterpret_cast<volatile uint32_t*>(&A.cnt->tail_epoch) != tail_epoch) {
                        __nanosleep(ns);
                        ns = ns < 16384 ? ns * 2 : ns;
                    }
                    __threadfence();
                }
                grid_barrier(A, grid);
                break;
            }
            const int32_t* L = A.list + (int64_t)cur * A.n_pad;
            unsigned long long* bw = A.bidw + (int64_t)cur * A.n_pad;
            const uint64_t tr0 = gtimer();
            // ---- [A1] cache bids (warp per person), misses to the global list
            {
                const int32_t tcount = __ldcg(&A.cnt->touched_count[nxt]);
                const int32_t* tl = A.touched + (int64_t)nxt * A.n_pad;
                unsigned long long* bw_old = A.bidw + (int64_t)nxt * A.n_pad;
                for (int64_t t = gtid; t < tcount; t += gsize) bw_old[__ldcg(tl + t)] = 0ull;
                if (gtid == 0) A.cnt->list_count[nxt] = 0;
                unsigned long long my_hits = 0;
                for (int64_t idx = gtid; idx < count; idx += gsize) {
                    const int32_t i = __ldcg(L + idx);
                    int32_t j1 = 0;
                    int64_t bid = 0;
                    if (cache_bid<false>(A, A.price, i, eps, j1, bid)) {
                        submit_bid(A, bw, i, j1, bid);
                        ++my_hits;
                    } else {
                        A.miss[atomicAdd(&A.cnt->miss_count, 1)] = i;
                    }
                }
                my_hits += __shfl_xor_sync(0xffffffffu, my_hits, 16);
                my_hits += __shfl_xor_sync(0xffffffffu, my_hits, 8);
                my_hits += __shfl_xor_sync(0xffffffffu, my_hits, 4);
                my_hits += __shfl_xor_sync(0xffffffffu, my_hits, 2);
                my_hits += __shfl_xor_sync(0xffffffffu, my_hits, 1);
                if (lane == 0 && my_hits) atomicAdd(&A.cnt->hits, my_hits);
            }
            grid_barrier(A, grid);
            const uint64_t tr1 = gtimer();
            // ---- [A2] cooperative row scans for the misses, spread over CTAs
            {
                const int32_t nmiss = __ldcg(&A.cnt->miss_count);
                if ((int32_t)blockIdx.x < nmiss) {
                    if (SP) {
                        if (threadIdx.x == 0) fetch_row<WT>(A, S, D, 0, __ldcg(A.miss + blockIdx.x));
                        stage_prices(A, D.price, nullptr);
                        __syncthreads();
                    }
                    int b = 0;
                    for (int32_t e = blockIdx.x; e < nmiss; e += gridDim.x) {
                        const int32_t i = __ldcg(A.miss + e);
                        const void* row = SP ? wait_row<WT>(A, S, D, b, i) : nullptr;
                        // prefetch the next miss into the other buffer
                        if (SP && threadIdx.x == 0 && e + (int32_t)gridDim.x < nmiss)
                            fetch_row<WT>(A, S, D, b ^ 1, __ldcg(A.miss + e + gridDim.x));
                        cta_scan_bid<WT, SP>(A, S, SP ? D.price : A.price, row, i, eps);
                        if (threadIdx.x == 0) {
                            submit_bid(A, bw, i, S.j1, S.bid);
                            if (SP && i < A.N && A.M > 0) S.bar_phase[b] ^= 1u;
                            S.row_person[b] = -1;
                        }
                        b ^= 1;
                        __syncthreads();
                    }
                    if (threadIdx.x == 0) {
                        const int32_t my = (nmiss - (int32_t)blockIdx.x + (int32_t)gridDim.x - 1) / (int32_t)gridDim.x;
                        atomicAdd(&A.cnt->scans, (unsigned long long)my);
                    }
                }
            }
            grid_barrier(A, grid);
            const uint64_t tr2 = gtimer();
            // ---- [B] resolve
            {
                int32_t* Lnext = A.list + (int64_t)nxt * A.n_pad;
                int32_t* tl = A.touched + (int64_t)cur * A.n_pad;
                if (gtid == 0) {
                    A.cnt->touched_count[nxt] = 0;
                    A.cnt->miss_count = 0;
                    atomicAdd(&A.cnt->rounds, 1ull);
                    atomicAdd(&A.cnt->bids, (unsigned long long)count);
                }
                for (int64_t idx = gtid; idx < count; idx += gsize) {
                    const int32_t i = __ldcg(L + idx);
                    const int32_t j = __ldcg(A.bidj + i);
                    const unsigned long long pk = __ldcg(A.bidpk + i);
                    if (__ldcg(bw + j) == pk) {
                        const int32_t prev = __ldcg(A.owner + j);
                        A.owner[j] = i;
                        A.price[j] = (int64_t)(pk >> A.idbits);
                        A.col[i] = j;
                        if (prev >= 0) {
                            A.col[prev] = -1;
                            Lnext[atomicAdd(&A.cnt->list_count[nxt], 1)] = prev;
                        }
                        tl[atomicAdd(&A.cnt->touched_count[cur], 1)] = j;
                    } else {
                        Lnext[atomicAdd(&A.cnt->list_count[nxt], 1)] = i;
                    }
                }
            }
            grid_barrier(A, grid);
            if (gtid == 0) {
                const uint64_t tr3 = gtimer();
                t_a1 += tr1 - tr0;
                t_a2 += tr2 - tr1;
                t_b += tr3 - tr2;
            }
            ++r;
            if (++rounds_total > A.round_guard) {
                if (gtid == 0) atomicOr(&A.cnt->errors, kErrIterGuard);
                return;
            }
        }
        if (__ldcg(&A.cnt->errors) & kErrIterGuard) return;
        if (gtid == 0) {
            const uint64_t tph2 = gtimer();
            if (tph1 == 0) tph1 = tph2;
            const int ph = (int)A.cnt->phases - 1;
            if (ph >= 0 && ph < kPhMax) {
                A.cnt->ph_eps[ph] = eps;
                A.cnt->ph_rounds[ph] = r;
                A.cnt->ph_tailn[ph] = ph_tailn;
                A.cnt->ph_ns_j[ph] = (long long)(tph1 - tph0);
                A.cnt->ph_ns_t[ph] = (long long)(tph2 - tph1);
                A.cnt->ph_bids[ph] = A.cnt->bids + A.cnt->tail_bids;
            }
        }
        if (eps <= 1) break;
        ++phase_no;
        eps = eps / A.theta;
        if (eps < 1) eps = 1;
    }
    if (gtid == 0) {
        A.cnt->ns_total = (long long)(gtimer() - t_start);
        A.cnt->ns_tail = (long long)t_tail;
        for (int k = 0; k < 5; ++k) A.cnt->ns_stage[k] = (long long)S.tprof[k];
        A.cnt->ns_stage[5] = (long long)S.tprof[7];
        A.cnt->ns_a1 = (long long)t_a1;
        A.cnt->ns_a2 = (long long)t_a2;
        A.cnt->ns_b = (long long)t_b;
    }
}

// max / bitwise-or over the real N x M block (epsilon0, packing check and the
// common power of two), one grid-stride pass with 16-byte loads
template <int WT>
__global__ void max_q_kernel(const void* W, int64_t ldw, int32_t N, int32_t M, AucCounters* cnt) {
    constexpr int kV = WT == MUX_W_I32 ? 4 : 2;          // elements per 16-byte load
    const int64_t vpr = ldw / kV;                          // vectors per row
    const int64_t total = (int64_t)N * vpr;
    long long mx = 0;
    unsigned long long orv = 0;
    bool neg = false;
    for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < total; e += (int64_t)gridDim.x * blockDim.x) {
        const int64_t r = e / vpr;
        const int64_t c0 = (e - r * vpr) * kV;
        long long q[4] = {0, 0, 0, 0};
        if (WT == MUX_W_I32) {
            const int4 v = __ldg(reinterpret_cast<const int4*>(static_cast<const int32_t*>(W) + r * ldw) + (e - r * vpr));
            q[0] = v.x; q[1] = v.y; q[2] = v.z; q[3] = v.w;
        } else {
            const longlong2 v = __ldg(reinterpret_cast<const longlong2*>(static_cast<const int64_t*>(W) + r * ldw) + (e - r * vpr));
            q[0] = v.x; q[1] = v.y;
        }
#pragma unroll
        for (int t = 0; t < kV; ++t) {
            if (c0 + t >= M) continue;
            mx = q[t] > mx ? q[t] : mx;
            orv |= (unsigned long long)q[t];
            neg |= q[t] < 0;
        }
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        const long long o2 = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = o2 > mx ? o2 : mx;
        orv |= __shfl_xor_sync(0xffffffffu, orv, o);
    }
    if (__any_sync(0xffffffffu, neg) && (threadIdx.x & 31) == 0) atomicOr(&cnt->errors, 1u << 8);
    if ((threadIdx.x & 31) == 0) {
        if (mx > 0) atomicMax(&cnt->max_q, mx);
        if (orv) atomicOr(&cnt->or_q, orv);
    }
}

// col_of_row for real rows (-1 for padding / zero-weight matches) + total
template <int WT>
__global__ void finalize_kernel(const void* W, int64_t ldw, int32_t N, int32_t M, const int32_t* col,
                                int32_t* out, AucCounters* cnt) {
    int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    long long q = 0;
    if (i < N) {
        int32_t j = col[i];
        if (j >= 0 && j < M) {
            q = (WT == MUX_W_I32) ? (long long)static_cast<const int32_t*>(W)[i * ldw + j]
                                  : static_cast<const int64_t*>(W)[i * ldw + j];
        }
        out[i] = (q > 0) ? j : -1;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    if ((threadIdx.x & 31) == 0 && q) atomicAdd(reinterpret_cast<unsigned long long*>(&cnt->total_q), (unsigned long long)q);
}

// out[c][r] = in[r][c] (in: rows x cols, 32 x 32 tiles through shared memory)
template <typename T>
__global__ void transpose_kernel(const T* in, int64_t ldi, int32_t rows, int32_t cols, T* out, int64_t ldo) {
    __shared__ T tile[32][33];
    const int32_t r0 = blockIdx.x * 32, c0 = blockIdx.y * 32;
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int32_t r = r0 + k, c = c0 + threadIdx.x;
        tile[k][threadIdx.x] = (r < rows && c < cols) ? in[(int64_t)r * ldi + c] : 0;
    }
    __syncthreads();
    for (int k = threadIdx.y; k < 32; k += blockDim.y) {
        const int32_t c = c0 + k, r = r0 + threadIdx.x;
        if (c < cols && r < rows) out[(int64_t)c * ldo + r] = tile[threadIdx.x][k];
    }
}

// transposed solve (jobs as rows, n = N) -> original orientation
template <typename T>
__global__ void untranspose_duals_kernel(const T* WT, int64_t ldt, int32_t mreal, int32_t n, const int64_t* pT,
                                         const int32_t* corT, const int32_t* rocT, int64_t sc, int32_t* col,
                                         int64_t* price, int32_t* owner) {
    const int32_t k = blockIdx.x * blockDim.x + threadIdx.x;
    if (k >= n) return;
    col[k] = rocT[k];          // online row k -> its job (or a padding column >= M)
    const int32_t u = corT[k]; // job / padding column k -> its online row
    owner[k] = u;
    const int64_t a = (k < mreal && u >= 0) ? (int64_t)WT[(int64_t)k * ldt + u] : 0;
    price[k] = (u >= 0 ? a - pT[u] : 0) * sc;
}

template <typename T>
__global__ void finalize_ssp_kernel(const T* W, int64_t ldw, int32_t N, int32_t M, const int32_t* col, int32_t* out) {
    const int32_t i = blockIdx.x * blockDim.x + threadIdx.x;
    if (i < N) {
        const int32_t j = col[i];
        out[i] = (j >= 0 && j < M && W[(int64_t)i * ldw + j] > 0) ? j : -1;
    }
}

}  // namespace mux

using namespace mux;

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

int mux_canon_impl(mux_ctx_t* ctx, const void* W, int wtype, int32_t N, int32_t M, int64_t ldw, int32_t n,
                   int64_t SC, int32_t qshift, int64_t* price, int32_t* col_dev, const int32_t* owner,
                   cudaStream_t st, mux_stats_t* stats, bool exact);


static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

int mux_ssp_impl(mux_ctx_t* ctx, const int32_t* W, int64_t ldw, int32_t N, int32_t M, const double* rowkey,
                 const double* colkey, int32_t* col_out, int64_t* total_q, int64_t* price_out,
                 int32_t* cor_out, int32_t* roc_out, mux_stats_t* stats, cudaStream_t st,
                 const int64_t* price_in = nullptr, const int32_t* warm_col = nullptr);
int mux_ssp_impl64(mux_ctx_t* ctx, const int64_t* W, int64_t ldw, int32_t N, int32_t M, const double* rowkey,
                   const double* colkey, int32_t* col_out, int64_t* total_q, int64_t* price_out,
                   int32_t* cor_out, int32_t* roc_out, mux_stats_t* stats, cudaStream_t st,
                   const int64_t* price_in = nullptr, const int32_t* warm_col = nullptr);

// the multilevel solver for int32 (csrc/ssp.cu) or int64 (csrc/ssp_w64.cu) weights
static int ssp_solve(int wtype, mux_ctx_t* ctx, const void* W, int64_t ldw, int32_t N, int32_t M, const double* rowkey,
                     const double* colkey, int32_t* col_out, int64_t* total_q, int64_t* price_out, int32_t* cor_out,
                     int32_t* roc_out, mux_stats_t* stats, cudaStream_t st, const int64_t* price_in = nullptr,
                     const int32_t* warm_col = nullptr) {
    if (wtype == MUX_W_I32)
        return mux_ssp_impl(ctx, static_cast<const int32_t*>(W), ldw, N, M, rowkey, colkey, col_out, total_q, price_out,
                            cor_out, roc_out, stats, st, price_in, warm_col);
    return mux_ssp_impl64(ctx, static_cast<const int64_t*>(W), ldw, N, M, rowkey, colkey, col_out, total_q, price_out,
                          cor_out, roc_out, stats, st, price_in, warm_col);
}

__global__ void fill_price_kernel(int64_t* p, int32_t n, int64_t v) {
    const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) p[j] = v;
}

__global__ void scale_price_kernel(int64_t* p, int32_t n, int64_t sc) {
    const int32_t j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j < n) p[j] *= sc;
}

int mux_match_impl(mux_ctx_t* ctx, const void* W, int wtype, int64_t N, int64_t M, int64_t ldw,
                   int32_t* col_out_dev, int64_t* total_q, mux_stats_t* stats, cudaStream_t st,
                   int theta, int tail_max, const double* rowkey, const double* colkey,
                   int64_t* price_io = nullptr, int warm = 0, const int32_t* warm_col = nullptr) {
    if (N < 0 || M < 0 || (N > 0 && ldw < M)) { set_error("mux_match: bad shape"); return MUX_EINVAL; }
    if (wtype != MUX_W_I32 && wtype != MUX_W_I64) { set_error("mux_match: weights must be int32 or int64"); return MUX_EINVAL; }
    const int64_t n = N > M ? N : M;
    if (n >= (1ll << 30)) { set_error("mux_match: problem too large"); return MUX_EINVAL; }
    const int esz = wtype == MUX_W_I32 ? 4 : 8;
    if (N > 0 && M > 0) {
        if (((ldw * esz) % 16) != 0 || (reinterpret_cast<uintptr_t>(W) & 15) != 0) {
            set_error("mux_match: rows must be 16-byte aligned (ldw multiple of 16 bytes)");
            return MUX_EINVAL;
        }
    }
    if (total_q) *total_q = 0;
    const Tuning& T = tuning();
    if (T.error) return MUX_EINVAL;
    if (n == 0) return MUX_OK;
    {
        // int32 problems: multilevel shortest-path solver (csrc/ssp.cu);
        // int64 (qbits > 30) and MUX_SOLVER=auction: the epsilon-scaling auction below.
        // N < M: the zero padding rows of the reference's square problem are
        // implicit; N > M: the transposed problem (jobs as rows)
        const bool rect_ok = T.ssp_rect;
        // int64 weights (qbits 31-44): the solver's 17-bit index keys bound n
        const bool ssp_w = wtype == MUX_W_I32 || (wtype == MUX_W_I64 && n < 60000);
        const bool use_ssp_t = !T.force_auction && ssp_w && M >= 1 && N >= 2 && N > M && rect_ok;
        if (use_ssp_t) {
            // N > M: solve the transposed M x N problem (jobs as rows, the padding
            // columns of the reference become implicit zero rows), then map the
            // assignment and the duals back for the canonicalisation
            const int32_t nn = (int32_t)N, mm = (int32_t)M;
            const int64_t ldt = ((int64_t)nn + 3) / 4 * 4;
            size_t off = 0;
            auto take = [&](size_t b) { size_t o = off; off += (b + 255) & ~(size_t)255; return o; };
            const size_t o_wt = take((size_t)esz * mm * ldt), o_pt = take(8ull * nn), o_ct = take(4ull * nn),
                         o_rt = take(4ull * nn), o_co = take(4ull * nn), o_pr = take(8ull * nn), o_ow = take(4ull * nn);
            MUX_TRY(ctx->auc.ensure(off));
            char* base = ctx->auc.as<char>();
            void* WT = base + o_wt;
            int64_t* pT = reinterpret_cast<int64_t*>(base + o_pt);
            int32_t* corT = reinterpret_cast<int32_t*>(base + o_ct);
            int32_t* rocT = reinterpret_cast<int32_t*>(base + o_rt);
            int32_t* colr = reinterpret_cast<int32_t*>(base + o_co);
            int64_t* price = reinterpret_cast<int64_t*>(base + o_pr);
            int32_t* owner = reinterpret_cast<int32_t*>(base + o_ow);
            const dim3 tg((unsigned)((nn + 31) / 32), (unsigned)((mm + 31) / 32));
            if (wtype == MUX_W_I32)
                transpose_kernel<int32_t><<<tg, dim3(32, 8), 0, st>>>(static_cast<const int32_t*>(W), ldw, nn, mm,
                                                                     static_cast<int32_t*>(WT), ldt);
            else
                transpose_kernel<int64_t><<<tg, dim3(32, 8), 0, st>>>(static_cast<const int64_t*>(W), ldw, nn, mm,
                                                                     static_cast<int64_t*>(WT), ldt);
            int64_t tq = 0;
            MUX_TRY(ssp_solve(wtype, ctx, WT, ldt, mm, nn, colkey, rowkey, col_out_dev, &tq, pT, corT, rocT, stats, st));
            // no column prices to carry in this orientation (the jobs are the rows)
            if (price_io) fill_price_kernel<<<(unsigned)((M + 255) / 256), 256, 0, st>>>(price_io, (int32_t)M, INT64_MIN);
            // original orientation: col_of_row[u] = rocT[u]; owner of job v = corT[v];
            // column (job) prices = the transposed rows' profits
            if (wtype == MUX_W_I32)
                untranspose_duals_kernel<int32_t><<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(
                    static_cast<const int32_t*>(WT), ldt, mm, nn, pT, corT, rocT, (int64_t)nn + 1, colr, price, owner);
            else
                untranspose_duals_kernel<int64_t><<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(
                    static_cast<const int64_t*>(WT), ldt, mm, nn, pT, corT, rocT, (int64_t)nn + 1, colr, price, owner);
            if (T.canon)
                MUX_TRY(mux_canon_impl(ctx, W, wtype, nn, mm, ldw, nn, (int64_t)nn + 1, 0, price, colr, owner, st, stats, true));
            if (wtype == MUX_W_I32)
                finalize_ssp_kernel<int32_t><<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(
                    static_cast<const int32_t*>(W), ldw, nn, mm, colr, col_out_dev);
            else
                finalize_ssp_kernel<int64_t><<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(
                    static_cast<const int64_t*>(W), ldw, nn, mm, colr, col_out_dev);
            MUX_CUDA_TRY(cudaGetLastError());
            MUX_CUDA_TRY(cudaStreamSynchronize(st));
            if (stats) { stats->launches += 4; stats->n_rows = N; stats->n_cols = M; stats->total_q = tq; }
            if (total_q) *total_q = tq;
            return MUX_OK;
        }
        const bool use_ssp = !T.force_auction && ssp_w && N >= 1 && M >= 2 && (N == M || (N < M && rect_ok));
        if (use_ssp) {
            const int32_t nn = (int32_t)M;
            const size_t o_p = 0, o_c = (8ull * nn + 255) & ~255ull, o_o = o_c + ((4ull * nn + 255) & ~255ull);
            MUX_TRY(ctx->auc.ensure(o_o + 4ull * nn + 256));
            char* base = ctx->auc.as<char>();
            int64_t* price = reinterpret_cast<int64_t*>(base + o_p);
            int32_t* colr = reinterpret_cast<int32_t*>(base + o_c);
            int32_t* owner = reinterpret_cast<int32_t*>(base + o_o);
            int64_t tq = 0;
            MUX_TRY(ssp_solve(wtype, ctx, W, ldw, (int32_t)N, nn, rowkey, colkey, col_out_dev, &tq, price, colr, owner,
                              stats, st, (price_io && warm) ? price_io : nullptr, (price_io && warm) ? warm_col : nullptr));
            // optimal column prices, in quantised-weight units, for the next round's warm start
            if (price_io) MUX_CUDA_TRY(cudaMemcpyAsync(price_io, price, 8ull * (size_t)M, cudaMemcpyDeviceToDevice, st));
            if (T.canon) {
                // canonicalisation works in the auction's units: benefits Q * (n + 1)
                scale_price_kernel<<<(unsigned)((nn + 255) / 256), 256, 0, st>>>(price, nn, (int64_t)nn + 1);
                MUX_TRY(mux_canon_impl(ctx, W, wtype, (int32_t)N, nn, ldw, nn, (int64_t)nn + 1, 0, price, colr, owner, st,
                                       stats, true));
                // the canonical assignment has the same (optimal) total
                if (wtype == MUX_W_I32)
                    finalize_ssp_kernel<int32_t><<<(unsigned)((N + 255) / 256), 256, 0, st>>>(
                        static_cast<const int32_t*>(W), ldw, (int32_t)N, nn, colr, col_out_dev);
                else
                    finalize_ssp_kernel<int64_t><<<(unsigned)((N + 255) / 256), 256, 0, st>>>(
                        static_cast<const int64_t*>(W), ldw, (int32_t)N, nn, colr, col_out_dev);
                MUX_CUDA_TRY(cudaGetLastError());
                MUX_CUDA_TRY(cudaStreamSynchronize(st));
                if (stats) stats->launches += 4;
            }
            if (total_q) *total_q = tq;
            if (stats) stats->total_q = tq;
            return MUX_OK;
        }
    }
    if (price_io) fill_price_kernel<<<(unsigned)((M + 255) / 256), 256, 0, st>>>(price_io, (int32_t)M, INT64_MIN);
    const int32_t n_pad = (int32_t)(((n + 3) / 4) * 4 + 4);
    // a staged row covers columns [0, M) rounded up to 16 bytes (<= ldw)
    int64_t row_cols = ((M + 3) / 4) * 4;
    if (row_cols > ldw) row_cols = ldw;
    const int32_t row_bytes = (int32_t)(row_cols * esz);
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += align256(bytes); return o; };
    const size_t o_cnt = take(sizeof(AucCounters));
    const size_t o_price = take(8ull * n_pad);
    const size_t o_owner = take(4ull * n_pad);
    const size_t o_col = take(4ull * n_pad);
    const size_t o_bidw = take(16ull * n_pad);
    const size_t o_touch = take(8ull * n_pad);
    const size_t o_list = take(8ull * n_pad);
    const size_t o_miss = take(4ull * n_pad);
    const size_t o_bidj = take(4ull * n_pad);
    const size_t o_bidpk = take(8ull * n_pad);
    const size_t o_cache = take(sizeof(PCache) * (size_t)n_pad);
    const size_t o_word = take(8ull * n_pad);
    MUX_TRY(ctx->auc.ensure(off));
    char* base = ctx->auc.as<char>();
    AucArgs A;
    A.W = W; A.ldw = ldw; A.N = (int32_t)N; A.M = (int32_t)M; A.n = (int32_t)n; A.n_pad = n_pad;
    A.row_bytes = row_bytes;
    A.cnt = reinterpret_cast<AucCounters*>(base + o_cnt);
    A.price = reinterpret_cast<int64_t*>(base + o_price);
    A.owner = reinterpret_cast<int32_t*>(base + o_owner);
    A.col = reinterpret_cast<int32_t*>(base + o_col);
    A.bidw = reinterpret_cast<unsigned long long*>(base + o_bidw);
    A.touched = reinterpret_cast<int32_t*>(base + o_touch);
    A.list = reinterpret_cast<int32_t*>(base + o_list);
    A.miss = reinterpret_cast<int32_t*>(base + o_miss);
    A.bidj = reinterpret_cast<int32_t*>(base + o_bidj);
    A.bidpk = reinterpret_cast<unsigned long long*>(base + o_bidpk);
    A.cache = reinterpret_cast<PCache*>(base + o_cache);
    A.word = reinterpret_cast<unsigned long long*>(base + o_word);
    A.SC = n + 1;
    A.theta = theta < 2 ? 2 : theta;
    A.tail_max = tail_max < 0 ? -1 : (tail_max > kTailMax ? kTailMax : tail_max);
    A.idbits = 1;
    while ((1ll << A.idbits) <= n) ++A.idbits;
    A.idmask = (1ull << A.idbits) - 1ull;
    A.koff = 1ll << (62 - A.idbits);

    MUX_CUDA_TRY(cudaMemsetAsync(A.cnt, 0, sizeof(AucCounters), st));
    MUX_CUDA_TRY(cudaMemsetAsync(A.price, 0, 8ull * n_pad, st));
    MUX_CUDA_TRY(cudaMemsetAsync(A.cache, 0, sizeof(PCache) * (size_t)n_pad, st));
    int64_t launches = 0;
    if (N > 0 && M > 0) {
        const unsigned g = (unsigned)ctx->num_sms * 8;
        if (wtype == MUX_W_I32) max_q_kernel<MUX_W_I32><<<g, 512, 0, st>>>(W, ldw, (int32_t)N, (int32_t)M, A.cnt);
        else max_q_kernel<MUX_W_I64><<<g, 512, 0, st>>>(W, ldw, (int32_t)N, (int32_t)M, A.cnt);
        ++launches;
    }
    AucCounters hc;
    MUX_CUDA_TRY(cudaMemcpyAsync(&hc, A.cnt, sizeof(hc), cudaMemcpyDeviceToHost, st));
    MUX_CUDA_TRY(cudaStreamSynchronize(st));
    if (hc.errors & (1u << 8)) { set_error("mux_match: negative weight"); return MUX_EINVAL; }
    // divide out the common power of two: the solve is then exactly invariant
    // to power-of-two weight scaling (the reference's scale-invariance test)
    A.qshift = 0;
    if (hc.or_q) while (((hc.or_q >> A.qshift) & 1ull) == 0) ++A.qshift;
    const long long maxq = hc.max_q >> A.qshift;
    // value/price bound: |v|, p < 2^(62 - idbits) keeps keys and bids in 64 bits
    const double maxa = (double)maxq * (double)A.SC;
    if (maxa * 4.0 + 16.0 >= std::ldexp(1.0, 62 - A.idbits)) {
        set_error("mux_match: weights too large for 64-bit bid packing (reduce qbits)");
        return MUX_EINVAL;
    }
    A.eps0 = (int64_t)(maxa / 4.0);
    if (A.eps0 < 1) A.eps0 = 1;
    A.round_guard = 200000000ll;
    A.cg_sync = T.auc_cg_sync ? 1 : 0;   // cooperative-groups grid.sync measured faster
    A.rot = (N != M) ? 1 : 0;
    A.async_tail = T.auc_async_tail >= 0 ? T.auc_async_tail : (n >= 512);   // default: on for n >= 512
    if (A.tail_max < 0) A.tail_max = 16;
    // with the concurrent chains on, every phase runs as chains (no Jacobi
    // rounds): on near-rank-1 weights a Jacobi round settles ~1 person when
    // everyone bids for the same object (10k: 9,400 rounds in phase 0)
    A.async_phases = T.auc_async_phases;
    A.fresh = T.auc_fresh;
    A.restage = T.auc_restage;
    A.order = T.auc_order;     // auto (measured best for both tail modes at 10k)
    A.keff = std::min(std::max(T.auc_k, 1), kK);

    // shared memory: two row buffers + price/owner mirrors when they fit
    const size_t rows_bytes = 2ull * (size_t)row_bytes;
    const size_t mirror = (size_t)n_pad * (sizeof(int64_t) + sizeof(int32_t));
    const bool smem_mode = rows_bytes + mirror + sizeof(Shared) + 1024 <= kSmemBudget && !T.auc_no_smem;
    const size_t dsmem = smem_mode ? rows_bytes + mirror : 0;
    void* fn;
    if (wtype == MUX_W_I32) fn = smem_mode ? (void*)auction_kernel<MUX_W_I32, true> : (void*)auction_kernel<MUX_W_I32, false>;
    else fn = smem_mode ? (void*)auction_kernel<MUX_W_I64, true> : (void*)auction_kernel<MUX_W_I64, false>;
    MUX_CUDA_TRY(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsmem));
    int per_sm = 0;
    MUX_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kAucThreads, dsmem));
    if (per_sm < 1) { set_error("auction kernel cannot be resident"); return MUX_ECUDA; }
    dim3 grid((unsigned)ctx->num_sms), block(kAucThreads);
    void* args[] = {&A};
    struct Events {   // destroyed on every exit path
        cudaEvent_t a = nullptr, b = nullptr;
        ~Events() { if (a) cudaEventDestroy(a); if (b) cudaEventDestroy(b); }
    } evs;
    MUX_CUDA_TRY(cudaEventCreate(&evs.a));
    MUX_CUDA_TRY(cudaEventCreate(&evs.b));
    cudaEvent_t e0 = evs.a, e1 = evs.b;
    MUX_CUDA_TRY(cudaEventRecord(e0, st));
    MUX_CUDA_TRY(cudaLaunchCooperativeKernel(fn, grid, block, args, dsmem, st));
    ++launches;
    MUX_CUDA_TRY(cudaEventRecord(e1, st));
    {
        // among all optimal assignments, return the one the reference's
        // canonicalisation emits (csrc/canon.cu); MUX_CANON=0 skips it
        if (T.canon && N > 0 && M > 0) {
            MUX_CUDA_TRY(cudaStreamSynchronize(st));
            AucCounters pre;
            MUX_CUDA_TRY(cudaMemcpy(&pre, A.cnt, sizeof(pre), cudaMemcpyDeviceToHost));
            if (!(pre.errors & (kErrIterGuard | kErrPriceBits))) {
                MUX_TRY(mux_canon_impl(ctx, W, wtype, (int32_t)N, (int32_t)M, ldw, (int32_t)n, A.SC, A.qshift,
                                       A.price, A.col, A.owner, st, stats, false));
                launches += 2;
            }
        }
    }
    if (N > 0) {
        if (wtype == MUX_W_I32)
            finalize_kernel<MUX_W_I32><<<(unsigned)((N + 255) / 256), 256, 0, st>>>(W, ldw, (int32_t)N, (int32_t)M, A.col, col_out_dev, A.cnt);
        else
            finalize_kernel<MUX_W_I64><<<(unsigned)((N + 255) / 256), 256, 0, st>>>(W, ldw, (int32_t)N, (int32_t)M, A.col, col_out_dev, A.cnt);
        ++launches;
    }
    MUX_CUDA_TRY(cudaGetLastError());
    MUX_CUDA_TRY(cudaMemcpyAsync(&hc, A.cnt, sizeof(hc), cudaMemcpyDeviceToHost, st));
    MUX_CUDA_TRY(cudaStreamSynchronize(st));
    float ms = 0.f;
    cudaEventElapsedTime(&ms, e0, e1);
    if (hc.errors & kErrIterGuard) { set_error("auction: round guard tripped"); return MUX_ELIMIT; }
    if (hc.errors & kErrPriceBits) { set_error("auction: price overflowed its packing"); return MUX_ELIMIT; }
    if (total_q) *total_q = hc.total_q;
    if (stats) {
        stats->n_rows = N; stats->n_cols = M; stats->n_square = n;
        stats->phases = (int64_t)hc.phases; stats->rounds = (int64_t)hc.rounds;
        stats->bids = (int64_t)hc.bids; stats->row_scans = (int64_t)hc.scans;
        stats->tail_bids = (int64_t)hc.tail_bids; stats->total_q = hc.total_q;
        stats->ms_match = ms;
        stats->ms_tail = hc.ns_tail * 1e-6;
        stats->ms_kernel = hc.ns_total * 1e-6;
        stats->cache_hits = (int64_t)hc.hits;
        stats->launches += launches;
        if (T.verbose) {
            fprintf(stderr, "[mux] async-tail rejected bids: %llu\n", hc.async_fail);
            unsigned long long prev = 0;
            for (int k = 0; k < (int)hc.phases && k < kPhMax; ++k) {
                fprintf(stderr, "[mux] phase %2d eps %14lld rounds %6d tail_n %4d jacobi %8.2f ms tail %8.2f ms bids %llu"
                                " chains %llu long %llu max %llu\n", k,
                        hc.ph_eps[k], hc.ph_rounds[k], hc.ph_tailn[k], hc.ph_ns_j[k] * 1e-6, hc.ph_ns_t[k] * 1e-6,
                        hc.ph_bids[k] - prev, hc.ph_chains[k], hc.ph_longchains[k], hc.ph_maxchain[k]);
                prev = hc.ph_bids[k];
            }
        }
        if (T.verbose)
            fprintf(stderr, "[mux] tail: hits %llu hit-loop cycles/hit %.0f; fetch cycles/scan %.0f\n", hc.tail_hits,
                    hc.cyc_hitloop / (double)(hc.tail_hits + 1), hc.cyc_fetch / (double)(hc.tail_scans + 1));
        if (T.verbose)
            fprintf(stderr, "[mux] tail: scans %llu hit_ms %.2f scan_ms %.2f wait_ms %.2f | rounds: a1 %.2f a2 %.2f b %.2f ms\n",
                    hc.tail_scans, hc.ns_tail_hit * 1e-6, hc.ns_tail_scan * 1e-6, hc.ns_tail_wait * 1e-6,
                    hc.ns_a1 * 1e-6, hc.ns_a2 * 1e-6, hc.ns_b * 1e-6);
        if (T.verbose)
            fprintf(stderr, "[mux] CTA0 scans %lld, cycles/scan: pass1 %.0f tau %.0f pass2 %.0f rank %.0f store %.0f\n",
                    hc.ns_stage[5], hc.ns_stage[0] / (double)(hc.ns_stage[5] + 1), hc.ns_stage[1] / (double)(hc.ns_stage[5] + 1),
                    hc.ns_stage[2] / (double)(hc.ns_stage[5] + 1), hc.ns_stage[3] / (double)(hc.ns_stage[5] + 1),
                    hc.ns_stage[4] / (double)(hc.ns_stage[5] + 1));
    }
    return MUX_OK;
}
