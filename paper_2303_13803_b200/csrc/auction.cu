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
// Algorithm (one persistent cooperative kernel for the whole solve):
//   for eps = eps0, eps0/theta, ..., 1:                  (epsilon scaling)
//     clear the assignment, keep prices
//     while some person is unassigned:
//       if few remain: single-CTA Gauss-Seidel tail (no grid barriers)
//       else Jacobi round:
//         [A] every unassigned person computes its bid -- best object j1,
//             best value v1, second value v2 (v = a - p), bid = p_j1 + v1 - v2 + eps
//             -- from its top-K candidate cache when still valid, else from a
//             full row scan (coalesced 16-byte loads of W and prices,
//             per-lane top-(K+1) lists, warp-shuffle merge); the bid is
//             atomicMax'ed into a packed 64-bit word (price << idbits | ~person)
//         grid barrier
//         [B] each bidder reads back the word: the winner takes the object,
//             the previous owner and the losers form the next round's list
//         grid barrier
// Candidate cache: a full scan keeps the K best (object, benefit) pairs and the
// (K+1)-th best value thr.  Prices only rise, so any uncached object's value
// is still <= thr; if the best cached value is >= thr the cached top-2 (with
// second = max(second, thr)) gives a valid epsilon-CS bid without re-reading
// the row.  The cache stays valid across phases.
// Determinism: every bid in a round sees the same prices and ties break to
// the lowest object index / lowest person index, so results do not depend on
// thread scheduling.
#include <cooperative_groups.h>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace mux {

constexpr int kK = 8;                 // cached candidates per person
constexpr int kAucThreads = 512;      // 16 warps per CTA
constexpr int kAucWarps = kAucThreads / kWarp;
constexpr int kTailMax = 32;          // persons left when the single-CTA tail takes over
constexpr int64_t kNegInf = INT64_MIN / 4;

struct AucCounters {
    int32_t list_count[2];
    int32_t touched_count[2];
    uint32_t errors;
    int32_t _pad;
    unsigned long long rounds, bids, scans, tail_bids, phases;
    long long max_q;
    long long total_q;
};

struct AucArgs {
    const void* W;       // [N][ldw] int32 or int64
    int64_t ldw;
    int32_t N, M, n;     // real rows, real columns, square size
    int32_t idbits;
    int64_t SC;          // benefit scale (n + 1)
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
    int32_t* bidj;       // [n_pad]
    unsigned long long* bidpk;  // [n_pad]
    int32_t* cj;         // [n_pad][K]
    int64_t* ca;         // [n_pad][K]
    int64_t* cthr;       // [n_pad]
    int32_t* cvalid;     // [n_pad]
    AucCounters* cnt;
    int32_t n_pad;
};

// ---- small helpers --------------------------------------------------------

__device__ __forceinline__ bool better(int64_t v, int32_t j, int64_t bv, int32_t bj) {
    return v > bv || (v == bv && j < bj);
}

template <int WT>
__device__ __forceinline__ int64_t wload1(const AucArgs& A, int32_t i, int32_t j) {
    if (i >= A.N || j >= A.M) return 0;
    if (WT == MUX_W_I32) return (int64_t)__ldg(static_cast<const int32_t*>(A.W) + (int64_t)i * A.ldw + j);
    return __ldg(static_cast<const int64_t*>(A.W) + (int64_t)i * A.ldw + j);
}

// Load 4 consecutive weights W[i][c..c+3] (c % 4 == 0), zero outside [0,N)x[0,M).
template <int WT>
__device__ __forceinline__ void wload4(const AucArgs& A, int32_t i, int32_t c, int64_t (&q)[4]) {
    if (i >= A.N || c >= A.M) { q[0] = q[1] = q[2] = q[3] = 0; return; }
    if (WT == MUX_W_I32) {
        const int4 v = __ldg(reinterpret_cast<const int4*>(static_cast<const int32_t*>(A.W) + (int64_t)i * A.ldw + c));
        q[0] = v.x; q[1] = v.y; q[2] = v.z; q[3] = v.w;
    } else {
        const longlong2* p = reinterpret_cast<const longlong2*>(static_cast<const int64_t*>(A.W) + (int64_t)i * A.ldw + c);
        const longlong2 a = __ldg(p), b = __ldg(p + 1);
        q[0] = a.x; q[1] = a.y; q[2] = b.x; q[3] = b.y;
    }
    if (c + 4 > A.M) {
#pragma unroll
        for (int t = 0; t < 4; ++t) if (c + t >= A.M) q[t] = 0;
    }
}

// Lane-local sorted top-(K+1) list, best first; equal values keep the earlier
// (lower-index) object first because a lane visits its columns in ascending order.
struct TopList {
    int64_t v[kK + 1];
    int32_t j[kK + 1];
    __device__ __forceinline__ void init() {
#pragma unroll
        for (int k = 0; k <= kK; ++k) { v[k] = kNegInf; j[k] = INT32_MAX; }
    }
    __device__ __forceinline__ void push(int64_t nv, int32_t nj) {
        if (!(nv > v[kK])) return;
        v[kK] = nv; j[kK] = nj;
#pragma unroll
        for (int k = kK; k > 0; --k) {
            if (v[k] > v[k - 1]) {
                int64_t tv = v[k]; v[k] = v[k - 1]; v[k - 1] = tv;
                int32_t tj = j[k]; j[k] = j[k - 1]; j[k - 1] = tj;
            }
        }
    }
    __device__ __forceinline__ void pop() {
#pragma unroll
        for (int k = 0; k < kK; ++k) { v[k] = v[k + 1]; j[k] = j[k + 1]; }
        v[kK] = kNegInf; j[kK] = INT32_MAX;
    }
};

// Warp argmax of (v, j) with ties to the lower j; result broadcast to all lanes.
__device__ __forceinline__ void warp_argmax(int64_t& v, int32_t& j) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        int64_t ov = __shfl_xor_sync(0xffffffffu, v, o);
        int32_t oj = __shfl_xor_sync(0xffffffffu, j, o);
        if (better(ov, oj, v, j)) { v = ov; j = oj; }
    }
}

// Merge the 32 lane lists into the warp's top-(K+1).  Lane r (< K+1) ends up
// holding the r-th best in (mv, mj).
__device__ __forceinline__ void warp_merge(TopList& L, int lane, int64_t& mv, int32_t& mj) {
    mv = kNegInf; mj = INT32_MAX;
#pragma unroll 1
    for (int r = 0; r <= kK; ++r) {
        int64_t bv = L.v[0];
        int32_t bj = L.j[0];
        warp_argmax(bv, bj);
        if (L.j[0] == bj && L.v[0] == bv && bj != INT32_MAX) L.pop();
        if (lane == r) { mv = bv; mj = bj; }
    }
}

// Scan the person's full row over objects [c_begin, n) with stride `stride`
// columns per step (each lane handles 4 consecutive objects per step).
template <int WT>
__device__ __forceinline__ void scan_row(const AucArgs& A, int32_t i, int32_t c_begin, int32_t stride,
                                         TopList& L) {
    for (int32_t c = c_begin; c < A.n; c += stride) {
        int64_t q[4];
        wload4<WT>(A, i, c, q);
        const longlong2* pp = reinterpret_cast<const longlong2*>(A.price + c);
        const longlong2 p01 = __ldcg(pp), p23 = __ldcg(pp + 1);
        const int64_t p[4] = {p01.x, p01.y, p23.x, p23.y};
#pragma unroll
        for (int t = 0; t < 4; ++t)
            if (c + t < A.n) L.push(q[t] * A.SC - p[t], c + t);
    }
}

// Store a fresh cache for person i from lane-held ranks (lane r holds rank r).
template <int WT>
__device__ __forceinline__ void store_cache(const AucArgs& A, int32_t i, int lane, int64_t mv, int32_t mj) {
    if (lane < kK) {
        const bool ok = mj != INT32_MAX;
        A.cj[(int64_t)i * kK + lane] = ok ? mj : -1;
        A.ca[(int64_t)i * kK + lane] = ok ? wload1<WT>(A, i, mj) * A.SC : 0;
    }
    const int64_t thr = __shfl_sync(0xffffffffu, mv, kK);
    if (lane == 0) {
        A.cthr[i] = thr;   // kNegInf when fewer than K+1 objects exist
        A.cvalid[i] = 1;
    }
}

// Bid from the candidate cache.  Returns true (and j1, bid) on a valid hit.
__device__ __forceinline__ bool cache_bid(const AucArgs& A, int32_t i, int lane, int64_t eps,
                                          int32_t& j1, int64_t& bid) {
    if (!__ldcg(A.cvalid + i)) return false;
    int64_t v = kNegInf, a = 0;
    int32_t j = INT32_MAX;
    if (lane < kK) {
        const int32_t cj = __ldcg(A.cj + (int64_t)i * kK + lane);
        if (cj >= 0) {
            a = __ldcg(A.ca + (int64_t)i * kK + lane);
            v = a - __ldcg(A.price + cj);
            j = cj;
        }
    }
    int64_t bv = v;
    int32_t bj = j;
    warp_argmax(bv, bj);
    // second best: max over the other lanes
    int64_t sv = (j == bj) ? kNegInf : v;
    int32_t sj = (j == bj) ? INT32_MAX : j;
    warp_argmax(sv, sj);
    const int64_t thr = __ldcg(A.cthr + i);
    if (bj == INT32_MAX || bv < thr) return false;
    const int64_t second = sv > thr ? sv : thr;
    const int64_t a1 = __shfl_sync(0xffffffffu, a, __ffs(__ballot_sync(0xffffffffu, j == bj)) - 1);
    j1 = bj;
    // a single object (n == 1): bid price + eps
    bid = (second <= kNegInf) ? (a1 - bv) + eps : a1 - second + eps;
    return true;
}

// Full-row bid by one warp (bulk rounds).
template <int WT>
__device__ __forceinline__ void warp_scan_bid(const AucArgs& A, int32_t i, int lane, int64_t eps,
                                              int32_t& j1, int64_t& bid) {
    TopList L;
    L.init();
    scan_row<WT>(A, i, lane * 4, 32 * 4, L);
    int64_t mv;
    int32_t mj;
    warp_merge(L, lane, mv, mj);
    store_cache<WT>(A, i, lane, mv, mj);
    const int64_t v1 = __shfl_sync(0xffffffffu, mv, 0);
    const int32_t jj = __shfl_sync(0xffffffffu, mj, 0);
    const int64_t v2 = __shfl_sync(0xffffffffu, mv, 1);
    const int64_t a1 = wload1<WT>(A, i, jj) * A.SC;
    j1 = jj;
    bid = (v2 <= kNegInf) ? (a1 - v1) + eps : a1 - v2 + eps;
}

__device__ __forceinline__ unsigned long long pack_bid(const AucArgs& A, int64_t bid, int32_t i) {
    const unsigned long long idmask = (1ull << A.idbits) - 1ull;
    return ((unsigned long long)bid << A.idbits) | (idmask - (unsigned long long)i);
}

// ---- single-CTA Gauss-Seidel tail -----------------------------------------

template <int WT>
__device__ void tail_gs(const AucArgs& A, int64_t eps, int32_t count, const int32_t* src_list) {
    __shared__ int32_t stack[kTailMax + 1];
    __shared__ int32_t s_top;
    __shared__ int64_t s_mv[kAucWarps][kK + 1];
    __shared__ int32_t s_mj[kAucWarps][kK + 1];
    __shared__ int32_t s_j1;
    __shared__ int64_t s_bid;
    __shared__ int32_t s_hit;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    for (int t = threadIdx.x; t < count; t += blockDim.x) stack[t] = __ldcg(src_list + t);
    __syncthreads();
    if (threadIdx.x == 0) {
        // the list order comes from atomics; sort (descending, so the lowest
        // person id is popped first) to keep the tail deterministic
        for (int a = 1; a < count; ++a) {
            const int32_t key = stack[a];
            int b = a - 1;
            while (b >= 0 && stack[b] < key) { stack[b + 1] = stack[b]; --b; }
            stack[b + 1] = key;
        }
        s_top = count;
    }
    __syncthreads();
    unsigned long long steps = 0, scans = 0;
    while (s_top > 0) {
        const int32_t i = stack[s_top - 1];
        if (warp == 0) {
            int32_t j1;
            int64_t bid;
            const bool hit = cache_bid(A, i, lane, eps, j1, bid);
            if (lane == 0) { s_hit = hit; s_j1 = j1; s_bid = bid; }
        }
        __syncthreads();
        if (!s_hit) {
            TopList L;
            L.init();
            scan_row<WT>(A, i, (warp * 32 + lane) * 4, kAucThreads * 4, L);
            int64_t mv;
            int32_t mj;
            warp_merge(L, lane, mv, mj);
            if (lane <= kK) { s_mv[warp][lane] = mv; s_mj[warp][lane] = mj; }
            __syncthreads();
            if (warp == 0) {
                TopList M;
                M.init();
                // lane l takes candidates l, l+32, ... of the kAucWarps*(K+1) pool,
                // pushed in ascending object order per lane is not guaranteed, so
                // use the full (v, j) order explicitly.
                for (int e = lane; e < kAucWarps * (kK + 1); e += 32) {
                    const int64_t v = s_mv[e / (kK + 1)][e % (kK + 1)];
                    const int32_t j = s_mj[e / (kK + 1)][e % (kK + 1)];
                    if (j == INT32_MAX) continue;
                    // insertion honouring ties by lower j
                    if (better(v, j, M.v[kK], M.j[kK])) {
                        M.v[kK] = v; M.j[kK] = j;
#pragma unroll
                        for (int k = kK; k > 0; --k)
                            if (better(M.v[k], M.j[k], M.v[k - 1], M.j[k - 1])) {
                                int64_t tv = M.v[k]; M.v[k] = M.v[k - 1]; M.v[k - 1] = tv;
                                int32_t tj = M.j[k]; M.j[k] = M.j[k - 1]; M.j[k - 1] = tj;
                            }
                    }
                }
                warp_merge(M, lane, mv, mj);
                store_cache<WT>(A, i, lane, mv, mj);
                const int64_t v1 = __shfl_sync(0xffffffffu, mv, 0);
                const int32_t jj = __shfl_sync(0xffffffffu, mj, 0);
                const int64_t v2 = __shfl_sync(0xffffffffu, mv, 1);
                if (lane == 0) {
                    const int64_t a1 = wload1<WT>(A, i, jj) * A.SC;
                    s_j1 = jj;
                    s_bid = (v2 <= kNegInf) ? (a1 - v1) + eps : a1 - v2 + eps;
                }
            }
            ++scans;
        }
        __syncthreads();
        if (threadIdx.x == 0) {
            const int32_t j = s_j1;
            const int64_t bid = s_bid;
            const int32_t prev = A.owner[j];
            A.owner[j] = i;
            A.price[j] = bid;
            A.col[i] = j;
            --s_top;
            if (prev >= 0) {
                A.col[prev] = -1;
                stack[s_top++] = prev;
            }
            __threadfence_block();
        }
        ++steps;
        __syncthreads();
        if (steps > (unsigned long long)A.round_guard) {
            if (threadIdx.x == 0) atomicOr(&A.cnt->errors, kErrIterGuard);
            break;
        }
    }
    if (threadIdx.x == 0) {
        atomicAdd(&A.cnt->tail_bids, steps);
        atomicAdd(&A.cnt->bids, steps);
        atomicAdd(&A.cnt->scans, scans);
        __threadfence();
    }
}

// ---- the persistent solve kernel ------------------------------------------

template <int WT>
__global__ void __launch_bounds__(kAucThreads)
auction_kernel(AucArgs A) {
    cg::grid_group grid = cg::this_grid();
    const int lane = threadIdx.x & 31;
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gsize = (int64_t)gridDim.x * blockDim.x;
    const int64_t gwarp = gtid >> 5;
    const int64_t nwarps = gsize >> 5;
    const int n = A.n;
    int64_t eps = A.eps0;
    long long rounds_total = 0;

    for (;;) {
        // ---- phase init: clear the assignment, keep prices and caches
        for (int64_t t = gtid; t < n; t += gsize) {
            A.owner[t] = -1;
            A.col[t] = -1;
            A.list[t] = (int32_t)t;          // list[0]
            A.bidw[t] = 0ull;
            A.bidw[A.n_pad + t] = 0ull;
        }
        if (gtid == 0) {
            A.cnt->list_count[0] = n;
            A.cnt->list_count[1] = 0;
            A.cnt->touched_count[0] = 0;
            A.cnt->touched_count[1] = 0;
            atomicAdd(&A.cnt->phases, 1ull);
        }
        grid.sync();
        int r = 0;
        for (;;) {
            const int cur = r & 1, nxt = cur ^ 1;
            const int32_t count = __ldcg(&A.cnt->list_count[cur]);
            if (count == 0) break;
            if (count <= A.tail_max) {
                if (blockIdx.x == 0) {
                    if (WT == MUX_W_I32) tail_gs<MUX_W_I32>(A, eps, count, A.list + (int64_t)cur * A.n_pad);
                    else tail_gs<MUX_W_I64>(A, eps, count, A.list + (int64_t)cur * A.n_pad);
                }
                grid.sync();
                break;
            }
            // ---- [A] bids
            {
                const int32_t tcount = __ldcg(&A.cnt->touched_count[nxt]);
                const int32_t* tl = A.touched + (int64_t)nxt * A.n_pad;
                unsigned long long* bw_old = A.bidw + (int64_t)nxt * A.n_pad;
                for (int64_t t = gtid; t < tcount; t += gsize) bw_old[__ldcg(tl + t)] = 0ull;
                if (gtid == 0) A.cnt->list_count[nxt] = 0;
            }
            unsigned long long my_scans = 0;
            {
                const int32_t* L = A.list + (int64_t)cur * A.n_pad;
                unsigned long long* bw = A.bidw + (int64_t)cur * A.n_pad;
                for (int64_t idx = gwarp; idx < count; idx += nwarps) {
                    const int32_t i = __ldcg(L + idx);
                    int32_t j1;
                    int64_t bid;
                    if (!cache_bid(A, i, lane, eps, j1, bid)) {
                        warp_scan_bid<WT>(A, i, lane, eps, j1, bid);
                        ++my_scans;
                    }
                    if (lane == 0) {
                        const unsigned long long pk = pack_bid(A, bid, i);
                        if (bid < 0 || (unsigned long long)bid >= (1ull << (63 - A.idbits)))
                            atomicOr(&A.cnt->errors, kErrPriceBits);
                        atomicMax(bw + j1, pk);
                        A.bidj[i] = j1;
                        A.bidpk[i] = pk;
                    }
                }
            }
            if (lane == 0 && my_scans) atomicAdd(&A.cnt->scans, my_scans);
            grid.sync();
            // ---- [B] resolve
            {
                const int32_t* L = A.list + (int64_t)cur * A.n_pad;
                int32_t* Lnext = A.list + (int64_t)nxt * A.n_pad;
                const unsigned long long* bw = A.bidw + (int64_t)cur * A.n_pad;
                int32_t* tl = A.touched + (int64_t)cur * A.n_pad;
                if (gtid == 0) {
                    A.cnt->touched_count[nxt] = 0;
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
            grid.sync();
            ++r;
            if (++rounds_total > A.round_guard) {
                if (gtid == 0) atomicOr(&A.cnt->errors, kErrIterGuard);
                return;
            }
        }
        if (__ldcg(&A.cnt->errors) & kErrIterGuard) return;
        if (eps <= 1) break;
        eps = eps / A.theta;
        if (eps < 1) eps = 1;
    }
}

// max over the real N x M block (for epsilon0 and overflow checks)
template <int WT>
__global__ void max_q_kernel(const void* W, int64_t ldw, int32_t N, int32_t M, AucCounters* cnt) {
    long long mx = 0;
    for (int64_t r = blockIdx.y; r < N; r += gridDim.y)
        for (int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; c < M; c += (int64_t)gridDim.x * blockDim.x) {
            long long q = (WT == MUX_W_I32) ? (long long)static_cast<const int32_t*>(W)[r * ldw + c]
                                            : static_cast<const int64_t*>(W)[r * ldw + c];
            mx = q > mx ? q : mx;
            if (q < 0) atomicOr(&cnt->errors, 1u << 8);
        }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
        long long o2 = __shfl_xor_sync(0xffffffffu, mx, o);
        mx = o2 > mx ? o2 : mx;
    }
    if ((threadIdx.x & 31) == 0 && mx > 0) atomicMax(&cnt->max_q, mx);
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

}  // namespace mux

using namespace mux;

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

static size_t align256(size_t b) { return (b + 255) & ~(size_t)255; }

int mux_match_impl(mux_ctx_t* ctx, const void* W, int wtype, int64_t N, int64_t M, int64_t ldw,
                   int32_t* col_out_dev, int64_t* total_q, mux_stats_t* stats, cudaStream_t st,
                   int theta, int tail_max) {
    if (N < 0 || M < 0 || (N > 0 && ldw < M)) { set_error("mux_match: bad shape"); return MUX_EINVAL; }
    if (wtype != MUX_W_I32 && wtype != MUX_W_I64) { set_error("mux_match: weights must be int32 or int64"); return MUX_EINVAL; }
    const int64_t n = N > M ? N : M;
    if (n >= (1ll << 30)) { set_error("mux_match: problem too large"); return MUX_EINVAL; }
    if (N > 0 && M > 0) {
        const int vec = wtype == MUX_W_I32 ? 4 : 2;
        if ((ldw % vec) != 0 || (reinterpret_cast<uintptr_t>(W) & 15) != 0) {
            set_error("mux_match: rows must be 16-byte aligned (ldw multiple of 16 bytes)");
            return MUX_EINVAL;
        }
    }
    if (total_q) *total_q = 0;
    if (n == 0) return MUX_OK;
    const int32_t n_pad = (int32_t)(((n + 3) / 4) * 4 + 4);
    // workspace layout
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += align256(bytes); return o; };
    const size_t o_cnt = take(sizeof(AucCounters));
    const size_t o_price = take(8ull * n_pad);
    const size_t o_owner = take(4ull * n_pad);
    const size_t o_col = take(4ull * n_pad);
    const size_t o_bidw = take(16ull * n_pad);
    const size_t o_touch = take(8ull * n_pad);
    const size_t o_list = take(8ull * n_pad);
    const size_t o_bidj = take(4ull * n_pad);
    const size_t o_bidpk = take(8ull * n_pad);
    const size_t o_cj = take(4ull * kK * n_pad);
    const size_t o_ca = take(8ull * kK * n_pad);
    const size_t o_cthr = take(8ull * n_pad);
    const size_t o_cvalid = take(4ull * n_pad);
    MUX_TRY(ctx->auc.ensure(off));
    char* base = ctx->auc.as<char>();
    AucArgs A;
    A.W = W; A.ldw = ldw; A.N = (int32_t)N; A.M = (int32_t)M; A.n = (int32_t)n; A.n_pad = n_pad;
    A.cnt = reinterpret_cast<AucCounters*>(base + o_cnt);
    A.price = reinterpret_cast<int64_t*>(base + o_price);
    A.owner = reinterpret_cast<int32_t*>(base + o_owner);
    A.col = reinterpret_cast<int32_t*>(base + o_col);
    A.bidw = reinterpret_cast<unsigned long long*>(base + o_bidw);
    A.touched = reinterpret_cast<int32_t*>(base + o_touch);
    A.list = reinterpret_cast<int32_t*>(base + o_list);
    A.bidj = reinterpret_cast<int32_t*>(base + o_bidj);
    A.bidpk = reinterpret_cast<unsigned long long*>(base + o_bidpk);
    A.cj = reinterpret_cast<int32_t*>(base + o_cj);
    A.ca = reinterpret_cast<int64_t*>(base + o_ca);
    A.cthr = reinterpret_cast<int64_t*>(base + o_cthr);
    A.cvalid = reinterpret_cast<int32_t*>(base + o_cvalid);
    A.SC = n + 1;
    A.theta = theta < 2 ? 2 : theta;
    A.tail_max = tail_max < 0 ? 0 : (tail_max > kTailMax ? kTailMax : tail_max);
    A.idbits = 1;
    while ((1ll << A.idbits) <= n) ++A.idbits;

    MUX_CUDA_TRY(cudaMemsetAsync(A.cnt, 0, sizeof(AucCounters), st));
    MUX_CUDA_TRY(cudaMemsetAsync(A.price, 0, 8ull * n_pad, st));
    MUX_CUDA_TRY(cudaMemsetAsync(A.cvalid, 0, 4ull * n_pad, st));
    int64_t launches = 0;
    if (N > 0 && M > 0) {
        dim3 g((unsigned)std::min<int64_t>((M + 255) / 256, 64), (unsigned)std::min<int64_t>(N, 4096));
        if (wtype == MUX_W_I32) max_q_kernel<MUX_W_I32><<<g, 256, 0, st>>>(W, ldw, (int32_t)N, (int32_t)M, A.cnt);
        else max_q_kernel<MUX_W_I64><<<g, 256, 0, st>>>(W, ldw, (int32_t)N, (int32_t)M, A.cnt);
        ++launches;
    }
    AucCounters hc;
    MUX_CUDA_TRY(cudaMemcpyAsync(&hc, A.cnt, sizeof(hc), cudaMemcpyDeviceToHost, st));
    MUX_CUDA_TRY(cudaStreamSynchronize(st));
    if (hc.errors & (1u << 8)) { set_error("mux_match: negative weight"); return MUX_EINVAL; }
    const long long maxq = hc.max_q;
    // price bound: prices stay below max benefit + n * eps0 <= 2^(63 - idbits)
    const double maxa = (double)maxq * (double)A.SC;
    if (maxa * 4.0 + 16.0 >= std::ldexp(1.0, 62 - A.idbits)) {
        set_error("mux_match: weights too large for 64-bit bid packing (reduce qbits)");
        return MUX_EINVAL;
    }
    A.eps0 = (int64_t)(maxa / 4.0);
    if (A.eps0 < 1) A.eps0 = 1;
    A.round_guard = 200000000ll;

    int dev;
    MUX_CUDA_TRY(cudaGetDevice(&dev));
    int per_sm = 0;
    void* fn = wtype == MUX_W_I32 ? (void*)auction_kernel<MUX_W_I32> : (void*)auction_kernel<MUX_W_I64>;
    MUX_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kAucThreads, 0));
    if (per_sm < 1) { set_error("auction kernel cannot be resident"); return MUX_ECUDA; }
    per_sm = per_sm > 2 ? 2 : per_sm;
    dim3 grid((unsigned)(ctx->num_sms * per_sm)), block(kAucThreads);
    void* args[] = {&A};
    cudaEvent_t e0, e1;
    MUX_CUDA_TRY(cudaEventCreate(&e0));
    MUX_CUDA_TRY(cudaEventCreate(&e1));
    MUX_CUDA_TRY(cudaEventRecord(e0, st));
    MUX_CUDA_TRY(cudaLaunchCooperativeKernel(fn, grid, block, args, 0, st));
    ++launches;
    MUX_CUDA_TRY(cudaEventRecord(e1, st));
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
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    if (hc.errors & kErrIterGuard) { set_error("auction: round guard tripped"); return MUX_ELIMIT; }
    if (hc.errors & kErrPriceBits) { set_error("auction: price overflowed its packing"); return MUX_ELIMIT; }
    if (total_q) *total_q = hc.total_q;
    if (stats) {
        stats->n_rows = N; stats->n_cols = M; stats->n_square = n;
        stats->phases = (int64_t)hc.phases; stats->rounds = (int64_t)hc.rounds;
        stats->bids = (int64_t)hc.bids; stats->row_scans = (int64_t)hc.scans;
        stats->tail_bids = (int64_t)hc.tail_bids; stats->total_q = hc.total_q;
        stats->ms_match = ms;
        stats->launches += launches;
    }
    return MUX_OK;
}
