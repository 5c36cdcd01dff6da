// Tie canonicalisation of the optimal assignment: the reference returns, among
// all optimal matchings, the one its row-by-row "repair" pass settles on
// (matching.py:173-199 with _repair_path, matching.py:104-145).  Three steps:
//
//  1. dual_repair_kernel (GPU, cooperative): the auction ends with prices that
//     satisfy 1-complementary slackness on weights scaled by (n + 1).  Exact
//     dual feasibility, a_ij - p_j <= a_i,sigma(i) - p_sigma(i) for every
//     (i, j), is restored by Bellman-Ford relaxation: p_j <- max(p_j,
//     max_i (a_ij - u_i)) over the rows whose profit u_i changed, until no
//     price moves.  The assignment is optimal, so there is no positive cycle
//     and the sweeps terminate.  The prices are then optimal duals.
//  2. tight_kernel (GPU): the tight edges a_ij - p_j == u_i of every real row,
//     written as a CSR in column order.  The tight subgraph under ANY optimal
//     dual contains exactly the optimal matchings, so step 3 reaches the same
//     matchings as the reference working on its own Hungarian duals.
//  3. canonicalise (host, native): the reference's sequential loop over rows
//     on the sparse tight graph.  Padding rows / columns (the reference's zero
//     square padding) are tight to one shared column set each, handled
//     implicitly instead of as dense rows.
//
// Result: for every row that ends with a positive-weight pair the choice is
// the lowest column any optimal matching consistent with the earlier rows
// allows, which is what the reference emits independently of which optimal
// duals its Hungarian produced.  A row left on a zero-weight REAL column keeps
// whichever such column the search history leaves it on, as in the reference;
// that column can differ from the reference's (its history differs), which
// only matters when weights contain real zeros (never in a scheduling round:
// every admissible pair has a positive predicted rate).
#include <cooperative_groups.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "common.cuh"

namespace cg = cooperative_groups;

namespace mux {

struct CanonCounters {
    int32_t act[2];
    int32_t nchanged;
    uint32_t errors;
    unsigned long long sweeps;
    unsigned long long row_scans;
    unsigned long long tight_total;
};

struct CanonArgs {
    const void* W;
    int64_t ldw;
    int32_t N, M, n;
    int32_t qshift;
    int64_t SC;
    int64_t* price;        // [n] auction prices, repaired in place
    const int32_t* col;    // [n]
    const int32_t* owner;  // [n]
    int64_t* u;            // [n] row profits
    int32_t* flag;         // [n] column raised in the current sweep
    int32_t* list;         // [2][n] active rows
    int32_t* changed;      // [n] columns raised in the current sweep
    CanonCounters* cnt;
    int64_t sweep_guard;
    // tight CSR
    int32_t* row_cnt;      // [N]
    int64_t* row_off;      // [N]
    int32_t* ent;          // [cap] column | bit 31 when the weight is zero
    int64_t cap;
};

constexpr uint32_t kCanonErrGuard = 1u << 0;
constexpr uint32_t kCanonErrCap = 1u << 1;
constexpr uint32_t kCanonErrDual = 1u << 2;   // a real pair above its row's profit: the duals are not feasible
constexpr int kCanonThreads = 512;

template <int WT>
__device__ __forceinline__ int64_t cq(const CanonArgs& C, int32_t i, int32_t j) {
    if (i >= C.N || j >= C.M) return 0;
    if (WT == MUX_W_I32) return (int64_t)__ldg(static_cast<const int32_t*>(C.W) + (int64_t)i * C.ldw + j) >> C.qshift;
    return __ldg(static_cast<const int64_t*>(C.W) + (int64_t)i * C.ldw + j) >> C.qshift;
}

// four weights of row i < N from column c (zero at j >= M), no read past M
template <int WT>
__device__ __forceinline__ void cq4(const CanonArgs& C, int32_t i, int32_t c, int64_t (&q)[4]) {
    if (c + 4 <= C.M) {
        if (WT == MUX_W_I32) {
            const int4 v = __ldg(reinterpret_cast<const int4*>(static_cast<const int32_t*>(C.W) + (int64_t)i * C.ldw + c));
            q[0] = v.x; q[1] = v.y; q[2] = v.z; q[3] = v.w;
        } else {
            const longlong2* p = reinterpret_cast<const longlong2*>(static_cast<const int64_t*>(C.W) + (int64_t)i * C.ldw + c);
            const longlong2 a = __ldg(p), b = __ldg(p + 1);
            q[0] = a.x; q[1] = a.y; q[2] = b.x; q[3] = b.y;
        }
#pragma unroll
        for (int t = 0; t < 4; ++t) q[t] >>= C.qshift;
    } else {
#pragma unroll
        for (int t = 0; t < 4; ++t) q[t] = cq<WT>(C, i, c + t);
    }
}

__device__ __forceinline__ void raise_price(const CanonArgs& C, int32_t j, int64_t cand) {
    if (cand <= __ldcg(C.price + j)) return;
    const long long old = atomicMax(reinterpret_cast<long long*>(C.price + j), (long long)cand);
    if (cand > old && atomicExch(C.flag + j, 1) == 0) C.changed[atomicAdd(&C.cnt->nchanged, 1)] = j;
}

template <int WT>
__global__ void __launch_bounds__(kCanonThreads, 1) dual_repair_kernel(CanonArgs C) {
    cg::grid_group grid = cg::this_grid();
    const int64_t gtid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
    const int64_t gsize = (int64_t)gridDim.x * blockDim.x;
    const int lane = threadIdx.x & 31;
    const int64_t gw = gtid >> 5, nw = gsize >> 5;
    const int32_t n = C.n;
    for (int64_t t = gtid; t < n; t += gsize) {
        const int32_t i = (int32_t)t;
        const int32_t j = C.col[i];
        C.u[i] = cq<WT>(C, i, j) * C.SC - C.price[j];
        C.list[i] = i;
        C.flag[i] = 0;
    }
    if (gtid == 0) { C.cnt->act[0] = n; C.cnt->act[1] = 0; C.cnt->nchanged = 0; }
    grid.sync();
    int cur = 0;
    for (int64_t sweep = 0;; ++sweep) {
        const int32_t count = *reinterpret_cast<volatile int32_t*>(&C.cnt->act[cur]);
        if (count == 0) break;
        if (sweep > C.sweep_guard) {
            if (gtid == 0) atomicOr(&C.cnt->errors, kCanonErrGuard);
            return;
        }
        const int nxt = cur ^ 1;
        for (int64_t idx = gw; idx < count; idx += nw) {
            const int32_t i = C.list[(int64_t)cur * n + idx];
            const int64_t ui = __ldcg(C.u + i);
            if (i >= C.N) {                       // padding row: every weight is zero
                for (int32_t j = lane; j < n; j += 32) raise_price(C, j, -ui);
                continue;
            }
            for (int32_t c = lane * 4; c < n; c += 128) {
                int64_t q[4];
                if (c < C.M) cq4<WT>(C, i, c, q);
                else q[0] = q[1] = q[2] = q[3] = 0;
#pragma unroll
                for (int t = 0; t < 4; ++t)
                    if (c + t < n) raise_price(C, c + t, q[t] * C.SC - ui);
            }
        }
        if (gtid == 0) atomicAdd(&C.cnt->row_scans, (unsigned long long)count);
        grid.sync();
        const int32_t nch = *reinterpret_cast<volatile int32_t*>(&C.cnt->nchanged);
        for (int64_t k = gtid; k < nch; k += gsize) {
            const int32_t j = C.changed[k];
            C.flag[j] = 0;
            const int32_t i = C.owner[j];
            C.u[i] = cq<WT>(C, i, j) * C.SC - __ldcg(C.price + j);
            C.list[(int64_t)nxt * n + atomicAdd(&C.cnt->act[nxt], 1)] = i;
        }
        grid.sync();
        if (gtid == 0) { C.cnt->act[cur] = 0; C.cnt->nchanged = 0; C.cnt->sweeps += 1; }
        grid.sync();
        cur = nxt;
    }
}

// Row profits u_i = a_i,col(i) * SC - p_col(i) of duals that are already
// exact (the SSP solver's): the repair sweeps are skipped and the tight
// kernel's count pass checks feasibility instead.
template <int WT>
__global__ void profit_kernel(CanonArgs C) {
    for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < C.n; i += gridDim.x * blockDim.x) {
        const int32_t j = C.col[i];
        C.u[i] = cq<WT>(C, i, j) * C.SC - C.price[j];
    }
}

// Tight edges of every real row, in column order: count, reserve, write.
// The count pass also flags any pair above its row's profit (kCanonErrDual).
template <int WT>
__global__ void __launch_bounds__(256) tight_kernel(CanonArgs C) {
    // one read of each row: its tight entries are gathered in column order in
    // shared memory (kTightBuf per warp) and written out once the row's offset
    // is known; a row with more tight entries reads itself a second time
    constexpr int kTightBuf = 256;
    __shared__ int32_t sbuf[8][kTightBuf];
    int32_t* buf = sbuf[threadIdx.x >> 5];
    const int lane = threadIdx.x & 31;
    const int64_t gw = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
    const int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
    for (int64_t row = gw; row < C.N; row += nw) {
        const int32_t i = (int32_t)row;
        const int64_t ui = C.u[i];
        int32_t base = 0;
        bool above = false;
        for (int32_t c0 = 0; c0 < C.M; c0 += 128) {
            const int32_t c = c0 + lane * 4;
            int64_t q[4] = {0, 0, 0, 0};
            bool tq[4] = {false, false, false, false};
            int32_t mine = 0;
            if (c < C.M) {
                cq4<WT>(C, i, c, q);
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    const int64_t v = c + t < C.M ? q[t] * C.SC - __ldcg(C.price + c + t) : INT64_MIN;
                    tq[t] = v == ui;
                    above |= v > ui;
                    mine += tq[t];
                }
            }
            if (__ballot_sync(0xffffffffu, mine > 0) == 0u) continue;
            int32_t incl = mine;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            int32_t pos = base + incl - mine;
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (tq[t]) {
                    if (pos < kTightBuf) buf[pos] = (c + t) | (q[t] == 0 ? (int32_t)0x80000000 : 0);
                    ++pos;
                }
            base += __shfl_sync(0xffffffffu, incl, 31);
        }
        if (above) atomicOr(&C.cnt->errors, kCanonErrDual);
        const int32_t cnt = base;
        long long off = 0;
        if (lane == 0) off = (long long)atomicAdd(&C.cnt->tight_total, (unsigned long long)cnt);
        off = __shfl_sync(0xffffffffu, off, 0);
        if (lane == 0) { C.row_cnt[i] = cnt; C.row_off[i] = off; }
        __syncwarp();
        if (off + cnt > C.cap) {
            if (lane == 0) atomicOr(&C.cnt->errors, kCanonErrCap);
            continue;
        }
        if (cnt <= kTightBuf) {
            for (int32_t t = lane; t < cnt; t += 32) C.ent[off + t] = buf[t];
            __syncwarp();
            continue;
        }
        // many equal scores: a second read of the row writes its entries directly
        int32_t b2 = 0;
        for (int32_t c0 = 0; c0 < C.M; c0 += 128) {
            const int32_t c = c0 + lane * 4;
            int64_t q[4] = {0, 0, 0, 0};
            bool tq[4] = {false, false, false, false};
            int32_t mine = 0;
            if (c < C.M) {
                cq4<WT>(C, i, c, q);
#pragma unroll
                for (int t = 0; t < 4; ++t) {
                    tq[t] = c + t < C.M && q[t] * C.SC - __ldcg(C.price + c + t) == ui;
                    mine += tq[t];
                }
            }
            int32_t incl = mine;
#pragma unroll
            for (int o = 1; o < 32; o <<= 1) {
                const int32_t y = __shfl_up_sync(0xffffffffu, incl, o);
                if (lane >= o) incl += y;
            }
            int32_t pos = b2 + incl - mine;
#pragma unroll
            for (int t = 0; t < 4; ++t)
                if (tq[t]) C.ent[off + pos++] = (c + t) | (q[t] == 0 ? (int32_t)0x80000000 : 0);
            b2 += __shfl_sync(0xffffffffu, incl, 31);
        }
    }
}

}  // namespace mux

#include "canon_host.h"


using namespace mux;
using mux::canon_host::Canon;
using mux::canon_host::TightGraph;

int mux_canon_impl(mux_ctx_t* ctx, const void* W, int wtype, int32_t N, int32_t M, int64_t ldw, int32_t n,
                   int64_t SC, int32_t qshift, int64_t* price, int32_t* col_dev, const int32_t* owner,
                   cudaStream_t st, mux_stats_t* stats, bool exact) {
    if (N <= 0 || M <= 0 || n <= 0) return MUX_OK;
    const auto h0 = std::chrono::steady_clock::now();
    // default tight-edge buffer: ~4 n edges in a predictor round; a round with
    // more (many equal scores) is re-run at its exact count below
    int64_t cap = std::min<int64_t>((int64_t)N * (int64_t)M, 64ll * n + 1024);
    if (cap < 16) cap = 16;
    size_t off = 0;
    auto take = [&](size_t bytes) { size_t o = off; off += (bytes + 255) & ~(size_t)255; return o; };
    const size_t o_cnt = take(sizeof(CanonCounters));
    const size_t o_u = take(8ull * n);
    const size_t o_flag = take(4ull * n);
    const size_t o_list = take(8ull * n);
    const size_t o_chg = take(4ull * n);
    const size_t o_rcnt = take(4ull * N);
    const size_t o_roff = take(8ull * N);
    const size_t o_ent = take(4ull * (size_t)cap);
    MUX_TRY(ctx->canon.ensure(off));
    char* base = ctx->canon.as<char>();
    CanonArgs C;
    C.W = W; C.ldw = ldw; C.N = N; C.M = M; C.n = n; C.qshift = qshift; C.SC = SC;
    C.price = price; C.col = col_dev; C.owner = owner;
    C.cnt = reinterpret_cast<CanonCounters*>(base + o_cnt);
    C.u = reinterpret_cast<int64_t*>(base + o_u);
    C.flag = reinterpret_cast<int32_t*>(base + o_flag);
    C.list = reinterpret_cast<int32_t*>(base + o_list);
    C.changed = reinterpret_cast<int32_t*>(base + o_chg);
    C.row_cnt = reinterpret_cast<int32_t*>(base + o_rcnt);
    C.row_off = reinterpret_cast<int64_t*>(base + o_roff);
    C.ent = reinterpret_cast<int32_t*>(base + o_ent);
    C.cap = cap;
    C.sweep_guard = 4ll * n + 16;

    const unsigned tg = (unsigned)std::min<int64_t>(((int64_t)N * 32 + 255) / 256, (int64_t)ctx->num_sms * 8);
    auto repair_and_tight = [&](bool repair) -> int {
        if (repair) {
            void* fn = wtype == MUX_W_I32 ? (void*)dual_repair_kernel<MUX_W_I32> : (void*)dual_repair_kernel<MUX_W_I64>;
            int per_sm = 0;
            MUX_CUDA_TRY(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kCanonThreads, 0));
            if (per_sm < 1) { set_error("dual repair kernel cannot be resident"); return MUX_ECUDA; }
            void* args[] = {&C};
            MUX_CUDA_TRY(cudaLaunchCooperativeKernel(fn, dim3((unsigned)ctx->num_sms), dim3(kCanonThreads), args, 0, st));
        } else {
            const unsigned pg = (unsigned)std::min<int64_t>((n + 255) / 256, (int64_t)ctx->num_sms * 4);
            if (wtype == MUX_W_I32) profit_kernel<MUX_W_I32><<<pg, 256, 0, st>>>(C);
            else profit_kernel<MUX_W_I64><<<pg, 256, 0, st>>>(C);
        }
        if (wtype == MUX_W_I32) tight_kernel<MUX_W_I32><<<tg, 256, 0, st>>>(C);
        else tight_kernel<MUX_W_I64><<<tg, 256, 0, st>>>(C);
        MUX_CUDA_TRY(cudaGetLastError());
        return MUX_OK;
    };
    CanonCounters hc;
    std::vector<int32_t> col(n), rcnt(N), ent;
    std::vector<int64_t> p(n), u(n), roff(N);
    // GPU part: profits (+ repair sweeps), tight CSR, copies to the host
    auto gpu_phase = [&](bool repair) -> int {
        MUX_CUDA_TRY(cudaMemsetAsync(C.cnt, 0, sizeof(CanonCounters), st));
        MUX_TRY(repair_and_tight(repair));
        MUX_CUDA_TRY(cudaMemcpyAsync(&hc, C.cnt, sizeof(hc), cudaMemcpyDeviceToHost, st));
        MUX_CUDA_TRY(cudaStreamSynchronize(st));
        if (hc.errors & kCanonErrGuard) { set_error("canonicalisation: dual repair did not converge"); return MUX_ELIMIT; }
        if (hc.errors & kCanonErrDual) return MUX_OK;   // caller decides (exact duals that were not)
        if (hc.errors & kCanonErrCap) {
            // more tight edges than the default buffer holds (many equal scores):
            // the count pass already has the exact total -- size for it and rerun
            const int64_t need = (int64_t)hc.tight_total;
            if (need > (int64_t)N * (int64_t)M) { set_error("canonicalisation: tight-edge count out of range"); return MUX_ELIMIT; }
            MUX_TRY(ctx->canon_ent.ensure(4ull * (size_t)need + 256));
            C.ent = ctx->canon_ent.as<int32_t>();
            C.cap = need;
            MUX_CUDA_TRY(cudaMemsetAsync(&C.cnt->tight_total, 0, sizeof(unsigned long long), st));
            MUX_CUDA_TRY(cudaMemsetAsync(&C.cnt->errors, 0, sizeof(uint32_t), st));
            if (wtype == MUX_W_I32) tight_kernel<MUX_W_I32><<<tg, 256, 0, st>>>(C);
            else tight_kernel<MUX_W_I64><<<tg, 256, 0, st>>>(C);
            MUX_CUDA_TRY(cudaGetLastError());
            MUX_CUDA_TRY(cudaMemcpyAsync(&hc, C.cnt, sizeof(hc), cudaMemcpyDeviceToHost, st));
            MUX_CUDA_TRY(cudaStreamSynchronize(st));
            if (hc.errors & kCanonErrCap) { set_error("canonicalisation: tight-edge graph exceeds its buffer"); return MUX_ELIMIT; }
        }
        ent.resize((size_t)hc.tight_total);
        MUX_CUDA_TRY(cudaMemcpyAsync(col.data(), col_dev, 4ull * n, cudaMemcpyDeviceToHost, st));
        MUX_CUDA_TRY(cudaMemcpyAsync(p.data(), price, 8ull * n, cudaMemcpyDeviceToHost, st));
        MUX_CUDA_TRY(cudaMemcpyAsync(u.data(), C.u, 8ull * n, cudaMemcpyDeviceToHost, st));
        MUX_CUDA_TRY(cudaMemcpyAsync(rcnt.data(), C.row_cnt, 4ull * N, cudaMemcpyDeviceToHost, st));
        MUX_CUDA_TRY(cudaMemcpyAsync(roff.data(), C.row_off, 8ull * N, cudaMemcpyDeviceToHost, st));
        if (hc.tight_total)
            MUX_CUDA_TRY(cudaMemcpyAsync(ent.data(), C.ent, 4ull * hc.tight_total, cudaMemcpyDeviceToHost, st));
        MUX_CUDA_TRY(cudaStreamSynchronize(st));
        return MUX_OK;
    };
    // padding rows / columns are implicit in the tight kernel: their feasibility
    // (a padding row's column has the minimum price; no real row profits below a
    // padding column's -p) is checked here for duals taken as exact
    auto padding_feasible = [&]() -> bool {
        if (N < n) {
            const int64_t pmin = *std::min_element(p.begin(), p.end());
            for (int32_t i = N; i < n; ++i)
                if (p[col[i]] != pmin) return false;
        }
        if (M < n) {
            const int64_t pmin = *std::min_element(p.begin() + M, p.end());
            for (int32_t i = 0; i < N; ++i)
                if (u[i] < -pmin) return false;
        }
        return true;
    };
    // exact duals (the SSP solver's): profits + tight edges only; the repair
    // sweeps run only if a feasibility check fails
    MUX_TRY(gpu_phase(!exact));
    if (exact && ((hc.errors & kCanonErrDual) || !padding_feasible())) MUX_TRY(gpu_phase(true));
    if (hc.errors & kCanonErrDual) { set_error("canonicalisation: duals infeasible after repair"); return MUX_ELIMIT; }
    const auto h1 = std::chrono::steady_clock::now();

    const auto h2 = std::chrono::steady_clock::now();
    TightGraph G;
    G.N = N; G.M = M; G.n = n;
    G.ent = &ent; G.cnt = &rcnt; G.off = &roff;
    if (N < n) {                 // padding rows: tight exactly to the cheapest columns
        const int64_t pmin = *std::min_element(p.begin(), p.end());
        for (int32_t j = 0; j < n; ++j)
            if (p[j] == pmin) G.Z.push_back(j);
    }
    if (M < n) {                 // padding columns: tight to row i iff -p_c == u_i
        const int64_t pmin = *std::min_element(p.begin() + M, p.end());
        for (int32_t j = M; j < n; ++j)
            if (p[j] == pmin) G.Zpad.push_back(j);
        G.padrow_tight.assign(N, 0);
        for (int32_t i = 0; i < N; ++i) G.padrow_tight[i] = (-u[i] == pmin);
    }
    std::vector<int32_t> col_in;
    if (tuning().canon_dump) col_in = col;
    Canon K(G, col);
    K.run();
    const auto h3 = std::chrono::steady_clock::now();
    if (tuning().canon_dump) {
        // analysis dump for tools/canon_host_bench.cpp: the host loop's inputs and output
        if (FILE* f = fopen(tuning().canon_dump, "wb")) {
            const int32_t hdr[7] = {N, M, n, (int32_t)ent.size(), (int32_t)G.Z.size(), (int32_t)G.Zpad.size(),
                                    (int32_t)G.padrow_tight.size()};
            fwrite(hdr, 4, 7, f);
            fwrite(col_in.data(), 4, n, f);
            fwrite(rcnt.data(), 4, N, f);
            fwrite(roff.data(), 8, N, f);
            fwrite(ent.data(), 4, ent.size(), f);
            fwrite(G.Z.data(), 4, G.Z.size(), f);
            fwrite(G.Zpad.data(), 4, G.Zpad.size(), f);
            fwrite(G.padrow_tight.data(), 1, G.padrow_tight.size(), f);
            fwrite(col.data(), 4, n, f);
            fclose(f);
        }
    }
    if (tuning().verbose) {
        auto ms = [](std::chrono::steady_clock::time_point a, std::chrono::steady_clock::time_point b) {
            return std::chrono::duration<double, std::milli>(b - a).count();
        };
        fprintf(stderr, "[mux] canon: GPU (profits / repair, tight CSR) + D2H %.2f ms (%llu sweeps, %llu row scans), setup %.2f ms, "
                        "host %.2f ms (%lld searches, %llu tight edges)\n",
                ms(h0, h1), hc.sweeps, hc.row_scans, ms(h1, h2), ms(h2, h3), K.searches, hc.tight_total);
    }
    MUX_CUDA_TRY(cudaMemcpyAsync(col_dev, col.data(), 4ull * n, cudaMemcpyHostToDevice, st));
    MUX_CUDA_TRY(cudaStreamSynchronize(st));
    if (stats) {
        stats->ms_canon = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
        stats->canon_searches = K.searches;
        stats->tight_edges = (int64_t)hc.tight_total;
        stats->dual_sweeps = (int64_t)hc.sweeps;
    }
    return MUX_OK;
}
