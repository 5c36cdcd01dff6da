// Pair scoring: the N x M predictor evaluation of one scheduling round.
//
// Replaces the reference's per-pair Python loop
//   for u in eligible: for v in candidates: w = predict(table, peak_u, v, share_u)
// (/root/reference/pkg/src/muxsim/scheduler.py:172-180) whose body is trilinear
// interpolation over a dense grid (predictor.py:74-118).
//
// Two arithmetic modes:
//  * EXACT (default): float64 with the reference's operation order and no FMA
//    contraction (__dmul_rn / __dadd_rn), so every score is bit-identical to
//    predict_point(): corners visited i-major, j, k-minor; each term is
//    ((wi*wj)*wk)*v; zero-weight corners contribute +0.0 to a non-negative
//    accumulator, which equals the reference's "skip" exactly.
//  * FAST: the exact rank-J factorisation W = (1-f_v)*A[u,j0_v] + f_v*A[u,j0_v+1]
//     in float32 -- 3 flops/pair, HBM-write bound.
// Quantised outputs apply the reference edge rule first: w < 1e-6 -> 0
// (matching.py:19, 159-162; scheduler.py:177 drops w <= 0), then
// q = rint(w * 2^qbits) (round-half-even, exact power-of-two scaling).
//
// Layout: out is row-major [n][ldo]; each thread produces 4 consecutive
// columns of one row (one 16-byte store for 32-bit outputs, two for 64-bit),
// a CTA covers 1024 columns x kRowsPerCta rows.  Padding columns [m, ldo) of
// quantised outputs are written as 0 so row scans can read whole vectors.
#include <algorithm>

#include "common.cuh"

namespace mux {

struct RowFeat {          // per online row: online_sm and sm_pct brackets
    int32_t i0, i1, k0, k1;
    double wi0, wi1, wk0, wk1;
};
struct ColFeat {          // per offline column: offline_sm bracket
    int32_t j0, j1;
    double wj0, wj1;
};

struct DevTable {
    int32_t ni, nj, nk;
    const double* ax_i;
    const double* ax_j;
    const double* ax_k;
    const double* values;   // [ni][nj][nk]
};

// predictor.py:74-82 `_locate` on device: exact comparisons and one IEEE
// division, identical to the reference's bisect_right-based bracket.
__device__ __forceinline__ void locate(const double* knots, int nkn, double x,
                                       int32_t& lo, int32_t& hi, double& w_lo, double& w_hi) {
    if (nkn == 1 || x <= knots[0]) { lo = 0; hi = 0; w_lo = 1.0; w_hi = 0.0; return; }
    if (x >= knots[nkn - 1]) { lo = nkn - 2; hi = nkn - 1; w_lo = 0.0; w_hi = 1.0; return; }
    int i = 0;
    while (i + 1 < nkn && knots[i + 1] <= x) ++i;   // bisect_right(knots, x) - 1
    double f = __ddiv_rn(__dsub_rn(x, knots[i]), __dsub_rn(knots[i + 1], knots[i]));
    lo = i; hi = i + 1; w_lo = __dsub_rn(1.0, f); w_hi = f;
}

__device__ __forceinline__ bool in_unit(double v) { return v >= 0.0 && v <= 1.0; }

__global__ void row_features_kernel(DevTable t, const double* __restrict__ x,
                                    const double* __restrict__ s, int64_t n,
                                    RowFeat* __restrict__ rf, uint32_t* flags) {
    int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (u >= n) return;
    double xv = x[u], sv = s[u];
    if (!in_unit(xv) || !in_unit(sv)) atomicOr(flags, kErrQueryRange);   // NaN fails too
    RowFeat r;
    locate(t.ax_i, t.ni, xv, r.i0, r.i1, r.wi0, r.wi1);
    locate(t.ax_k, t.nk, sv, r.k0, r.k1, r.wk0, r.wk1);
    rf[u] = r;
}

__global__ void col_features_kernel(DevTable t, const double* __restrict__ y, int64_t m,
                                    ColFeat* __restrict__ cf, uint32_t* flags) {
    int64_t v = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (v >= m) return;
    double yv = y[v];
    if (!in_unit(yv)) atomicOr(flags, kErrQueryRange);
    ColFeat c;
    locate(t.ax_j, t.nj, yv, c.j0, c.j1, c.wj0, c.wj1);
    cf[v] = c;
}

constexpr int kScoreThreads = 256;
constexpr int kColsPerThread = 4;
constexpr int kColsPerCta = kScoreThreads * kColsPerThread;   // 1024
constexpr int kRowsPerCta = 16;
constexpr int kMaxSmemTable = 4096;   // doubles staged in shared memory

template <int WT>
__device__ __forceinline__ void store4(void* out, int64_t ldo, int64_t row, int64_t col,
                                       const double (&w)[4], bool quant, double qscale) {
    if (WT == MUX_W_I32) {
        int4 q;
        int* qq = reinterpret_cast<int*>(&q);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
            double wc = w[c] < 1e-6 ? 0.0 : w[c];
            qq[c] = (int)__double2ll_rn(__dmul_rn(wc, qscale));
        }
        *reinterpret_cast<int4*>(static_cast<int32_t*>(out) + row * ldo + col) = q;
    } else if (WT == MUX_W_I64) {
        longlong2 a, b;
        double wc[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) wc[c] = w[c] < 1e-6 ? 0.0 : w[c];
        a.x = __double2ll_rn(__dmul_rn(wc[0], qscale));
        a.y = __double2ll_rn(__dmul_rn(wc[1], qscale));
        b.x = __double2ll_rn(__dmul_rn(wc[2], qscale));
        b.y = __double2ll_rn(__dmul_rn(wc[3], qscale));
        longlong2* p = reinterpret_cast<longlong2*>(static_cast<int64_t*>(out) + row * ldo + col);
        p[0] = a;
        p[1] = b;
    } else if (WT == MUX_W_F32) {
        float4 f = make_float4((float)w[0], (float)w[1], (float)w[2], (float)w[3]);
        *reinterpret_cast<float4*>(static_cast<float*>(out) + row * ldo + col) = f;
    } else {
        double2* p = reinterpret_cast<double2*>(static_cast<double*>(out) + row * ldo + col);
        p[0] = make_double2(w[0], w[1]);
        p[1] = make_double2(w[2], w[3]);
    }
    (void)quant;
}

// Scalar tail store for the last partial vector of a row (col + 4 > ldo).
template <int WT>
__device__ __forceinline__ void store1(void* out, int64_t ldo, int64_t row, int64_t col,
                                      double w, double qscale) {
    double wc = w < 1e-6 ? 0.0 : w;
    if (WT == MUX_W_I32) static_cast<int32_t*>(out)[row * ldo + col] = (int)__double2ll_rn(__dmul_rn(wc, qscale));
    else if (WT == MUX_W_I64) static_cast<int64_t*>(out)[row * ldo + col] = __double2ll_rn(__dmul_rn(wc, qscale));
    else if (WT == MUX_W_F32) static_cast<float*>(out)[row * ldo + col] = (float)w;
    else static_cast<double*>(out)[row * ldo + col] = w;
}

// EXACT mode: bit-identical float64 trilinear interpolation per pair.
template <int WT>
__global__ void __launch_bounds__(kScoreThreads)
score_exact_kernel(DevTable t, const RowFeat* __restrict__ rf, const ColFeat* __restrict__ cf,
                   int64_t n, int64_t m, void* __restrict__ out, int64_t ldo, double qscale) {
    __shared__ double sV[kMaxSmemTable];
    const int nv = t.ni * t.nj * t.nk;
    const bool smem_table = nv <= kMaxSmemTable;
    if (smem_table)
        for (int e = threadIdx.x; e < nv; e += blockDim.x) sV[e] = t.values[e];
    __syncthreads();
    const double* V = smem_table ? sV : t.values;
    const int nj = t.nj, nk = t.nk;

    const int64_t col0 = (int64_t)blockIdx.x * kColsPerCta + threadIdx.x * kColsPerThread;
    if (col0 >= ldo) return;
    ColFeat c[4];
    bool live[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        live[q] = col0 + q < m;
        if (live[q]) c[q] = cf[col0 + q];
        else { c[q].j0 = 0; c[q].j1 = 0; c[q].wj0 = 0.0; c[q].wj1 = 0.0; }
    }
    // Table offsets split into a column part (j * nk, fixed per thread) and a
    // row part (i * nj * nk + k, four per row) so the inner loop does one
    // 32-bit add per corner; the float64 operation order is unchanged.
    int32_t cj[4][2];
#pragma unroll
    for (int q = 0; q < 4; ++q) { cj[q][0] = c[q].j0 * nk; cj[q][1] = c[q].j1 * nk; }
    const int32_t njk = nj * nk;
    // grid-stride over row blocks: grid.y is capped at 65535
    for (int64_t rb = blockIdx.y; rb * kRowsPerCta < n; rb += gridDim.y) {
    const int64_t row_begin = rb * kRowsPerCta;
    const int64_t row_end = min(n, row_begin + kRowsPerCta);
    for (int64_t row = row_begin; row < row_end; ++row) {
        const RowFeat r = rf[row];
        const int32_t ri[2][2] = {{r.i0 * njk + r.k0, r.i0 * njk + r.k1},
                                  {r.i1 * njk + r.k0, r.i1 * njk + r.k1}};
        const double wi[2] = {r.wi0, r.wi1};
        const double wk[2] = {r.wk0, r.wk1};
        double w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            const double wj[2] = {c[q].wj0, c[q].wj1};
            double acc = 0.0;
#pragma unroll
            for (int a = 0; a < 2; ++a)
#pragma unroll
                for (int b = 0; b < 2; ++b) {
                    const double wij = __dmul_rn(wi[a], wj[b]);
#pragma unroll
                    for (int g = 0; g < 2; ++g)
                        acc = __dadd_rn(acc, __dmul_rn(__dmul_rn(wij, wk[g]), V[ri[a][g] + cj[q][b]]));
                }
            acc = fmin(1.0, fmax(0.0, acc));
            w[q] = live[q] ? acc : 0.0;
        }
        if (col0 + 4 <= ldo) store4<WT>(out, ldo, row, col0, w, true, qscale);
        else
            for (int q = 0; q < 4 && col0 + q < ldo; ++q) store1<WT>(out, ldo, row, col0 + q, w[q], qscale);
    }
    }
}

// FAST mode, step 1: per-row collapse of the table to A[u, 0..nj) (float64
// accumulate, stored float32).
__global__ void row_collapse_kernel(DevTable t, const RowFeat* __restrict__ rf, int64_t n,
                                    float* __restrict__ A) {
    int64_t u = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    if (u >= n) return;
    const RowFeat r = rf[u];
    const int nj = t.nj, nk = t.nk;
    for (int j = 0; j < nj; ++j) {
        double acc = 0.0;
        acc += r.wi0 * r.wk0 * t.values[((int64_t)r.i0 * nj + j) * nk + r.k0];
        acc += r.wi0 * r.wk1 * t.values[((int64_t)r.i0 * nj + j) * nk + r.k1];
        acc += r.wi1 * r.wk0 * t.values[((int64_t)r.i1 * nj + j) * nk + r.k0];
        acc += r.wi1 * r.wk1 * t.values[((int64_t)r.i1 * nj + j) * nk + r.k1];
        A[u * nj + j] = (float)acc;
    }
}

// FAST mode, step 2: W = (1-f) A[j0] + f A[j1], clamp, optional quantise.
template <int WT>
__global__ void __launch_bounds__(kScoreThreads)
score_fast_kernel(const float* __restrict__ A, int nj, const ColFeat* __restrict__ cf,
                  int64_t n, int64_t m, void* __restrict__ out, int64_t ldo, double qscale) {
    const int64_t col0 = (int64_t)blockIdx.x * kColsPerCta + threadIdx.x * kColsPerThread;
    if (col0 >= ldo) return;
    int32_t j0[4], j1[4];
    float f0[4], f1[4];
    bool live[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
        live[q] = col0 + q < m;
        ColFeat c = live[q] ? cf[col0 + q] : ColFeat{0, 0, 0.0, 0.0};
        j0[q] = c.j0; j1[q] = c.j1; f0[q] = (float)c.wj0; f1[q] = (float)c.wj1;
    }
    for (int64_t rb = blockIdx.y; rb * kRowsPerCta < n; rb += gridDim.y) {
    const int64_t row_begin = rb * kRowsPerCta;
    const int64_t row_end = min(n, row_begin + kRowsPerCta);
    for (int64_t row = row_begin; row < row_end; ++row) {
        const float* a = A + row * nj;
        double w[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
            float v = f0[q] * __ldg(a + j0[q]) + f1[q] * __ldg(a + j1[q]);
            v = fminf(1.0f, fmaxf(0.0f, v));
            w[q] = live[q] ? (double)v : 0.0;
        }
        if (col0 + 4 <= ldo) store4<WT>(out, ldo, row, col0, w, true, qscale);
        else
            for (int q = 0; q < 4 && col0 + q < ldo; ++q) store1<WT>(out, ldo, row, col0 + q, w[q], qscale);
    }
    }
}

}  // namespace mux

using namespace mux;

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------

static int upload_table(mux_ctx_t* ctx, const mux_table_t* tb, DevTable* dt, cudaStream_t st) {
    const size_t ni = tb->n_online_sm, nj = tb->n_offline_sm, nk = tb->n_sm_pct;
    const size_t nvals = ni * nj * nk;
    const size_t total = ni + nj + nk + nvals;
    MUX_TRY(ctx->table.ensure(total * sizeof(double)));
    double* d = ctx->table.as<double>();
    MUX_CUDA_TRY(cudaMemcpyAsync(d, tb->online_sm, ni * 8, cudaMemcpyHostToDevice, st));
    MUX_CUDA_TRY(cudaMemcpyAsync(d + ni, tb->offline_sm, nj * 8, cudaMemcpyHostToDevice, st));
    MUX_CUDA_TRY(cudaMemcpyAsync(d + ni + nj, tb->sm_pct, nk * 8, cudaMemcpyHostToDevice, st));
    MUX_CUDA_TRY(cudaMemcpyAsync(d + ni + nj + nk, tb->values, nvals * 8, cudaMemcpyHostToDevice, st));
    dt->ni = (int32_t)ni; dt->nj = (int32_t)nj; dt->nk = (int32_t)nk;
    dt->ax_i = d; dt->ax_j = d + ni; dt->ax_k = d + ni + nj; dt->values = d + ni + nj + nk;
    return MUX_OK;
}

template <int WT>
static void launch_score(int mode, DevTable dt, const RowFeat* rf, const ColFeat* cf, const float* A,
                         int64_t n, int64_t m, void* out, int64_t ldo, double qscale, cudaStream_t st) {
    dim3 grid((unsigned)((ldo + kColsPerCta - 1) / kColsPerCta),
              (unsigned)std::min<int64_t>((n + kRowsPerCta - 1) / kRowsPerCta, 65535));
    if (mode == MUX_SCORE_EXACT)
        score_exact_kernel<WT><<<grid, kScoreThreads, 0, st>>>(dt, rf, cf, n, m, out, ldo, qscale);
    else
        score_fast_kernel<WT><<<grid, kScoreThreads, 0, st>>>(A, dt.nj, cf, n, m, out, ldo, qscale);
}

// Internal entry used by mux_score_table and mux_round.  Leaves a possible
// range error in ctx->flags (checked by the caller after a sync).
int mux_score_table_impl(mux_ctx_t* ctx, const mux_table_t* tb, const double* x, const double* s,
                         int64_t n, const double* y, int64_t m, int mode, int wtype, int qbits,
                         void* out, int64_t ldo, cudaStream_t st, int64_t* launches) {
    DevTable dt;
    MUX_TRY(upload_table(ctx, tb, &dt, st));
    const size_t rf_bytes = sizeof(RowFeat) * (size_t)(n > 0 ? n : 1);
    const size_t a_bytes = sizeof(float) * (size_t)(n > 0 ? n : 1) * (size_t)dt.nj;
    MUX_TRY(ctx->rowfeat.ensure(rf_bytes + (mode == MUX_SCORE_FAST ? a_bytes + 256 : 0)));
    MUX_TRY(ctx->colfeat.ensure(sizeof(ColFeat) * (size_t)(m > 0 ? m : 1)));
    RowFeat* rf = ctx->rowfeat.as<RowFeat>();
    float* A = reinterpret_cast<float*>(reinterpret_cast<char*>(ctx->rowfeat.ptr) + ((rf_bytes + 255) / 256) * 256);
    ColFeat* cf = ctx->colfeat.as<ColFeat>();
    uint32_t* flags = ctx->flags.as<uint32_t>();
    int64_t nl = 0;
    if (n > 0) { row_features_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(dt, x, s, n, rf, flags); ++nl; }
    if (m > 0) { col_features_kernel<<<(unsigned)((m + 255) / 256), 256, 0, st>>>(dt, y, m, cf, flags); ++nl; }
    if (mode == MUX_SCORE_FAST && n > 0) {
        row_collapse_kernel<<<(unsigned)((n + 255) / 256), 256, 0, st>>>(dt, rf, n, A);
        ++nl;
    }
    if (n > 0 && ldo > 0) {
        const double qscale = ldexp(1.0, qbits);
        switch (wtype) {
            case MUX_W_I32: launch_score<MUX_W_I32>(mode, dt, rf, cf, A, n, m, out, ldo, qscale, st); break;
            case MUX_W_I64: launch_score<MUX_W_I64>(mode, dt, rf, cf, A, n, m, out, ldo, qscale, st); break;
            case MUX_W_F32: launch_score<MUX_W_F32>(mode, dt, rf, cf, A, n, m, out, ldo, qscale, st); break;
            default:        launch_score<MUX_W_F64>(mode, dt, rf, cf, A, n, m, out, ldo, qscale, st); break;
        }
        ++nl;
    }
    MUX_CUDA_TRY(cudaGetLastError());
    if (launches) *launches += nl;
    return MUX_OK;
}
