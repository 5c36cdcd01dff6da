// C ABI entry points (include/muxflow.h).  Host-side argument checking,
// context / workspace management, and the fused per-round path.
#include <cmath>
#include <cstring>
#include <string>
#include <vector>

#include "common.cuh"

int mux_score_table_impl(mux_ctx_t* ctx, const mux_table_t* tb, const double* x, const double* s,
                         int64_t n, const double* y, int64_t m, int mode, int wtype, int qbits,
                         void* out, int64_t ldo, cudaStream_t st, int64_t* launches);
int mux_score_mlp_impl(mux_ctx_t* ctx, const mux_mlp_t* w, const double* on, const double* share, int64_t n,
                       const double* off, int64_t m, int wtype, int qbits, void* out, int64_t ldo,
                       cudaStream_t st, int64_t* launches);
int mux_match_impl(mux_ctx_t* ctx, const void* W, int wtype, int64_t N, int64_t M, int64_t ldw,
                   int32_t* col_out_dev, int64_t* total_q, mux_stats_t* stats, cudaStream_t st,
                   int theta, int tail_max, const double* rowkey, const double* colkey,
                   int64_t* price_io = nullptr, int warm = 0, const int32_t* warm_col = nullptr);

namespace mux {
static thread_local std::string g_last_error;
void set_error(const std::string& msg) { g_last_error = msg; }

namespace {
// Integer knob in [lo, hi]; a malformed or out-of-range value sets the error.
int knob(const char* name, int dflt, long lo, long hi, std::string& err) {
    const char* v = getenv(name);
    if (!v || !*v) return dflt;
    char* end = nullptr;
    const long x = strtol(v, &end, 10);
    if (*end != '\0' || x < lo || x > hi) {
        if (err.empty()) err = std::string(name) + "=" + v + " outside [" + std::to_string(lo) + ", " + std::to_string(hi) + "]";
        return dflt;
    }
    return (int)x;
}
}  // namespace

const Tuning& tuning() {
    static thread_local Tuning t;
    t = Tuning{};
    std::string err;
    t.verbose = getenv("MUX_VERBOSE") != nullptr;
    t.ssp_check = knob("MUX_SSP_CHECK", 0, 0, 1, err) == 1;
    t.ssp_time = knob("MUX_SSP_TIME", 0, 0, 1, err) == 1;
    if (knob("MUX_TUNING", 0, 0, 1, err) == 1) {
        const char* sv = getenv("MUX_SOLVER");
        if (sv && *sv) {
            if (strcmp(sv, "auction") == 0) t.force_auction = true;
            else if (strcmp(sv, "ssp") != 0 && err.empty()) err = std::string("MUX_SOLVER=") + sv + " (auction | ssp)";
        }
        t.canon = knob("MUX_CANON", 1, 0, 1, err) == 1;
        t.ssp_rect = knob("MUX_SSP_RECT", 1, 0, 1, err) == 1;
        t.ssp_f = knob("MUX_SSP_F", t.ssp_f, 2, 16, err);
        t.ssp_fx = getenv("MUX_SSP_FX") ? knob("MUX_SSP_FX", 0, 110, 1600, err) : 0;
        t.ssp_base = knob("MUX_SSP_BASE", t.ssp_base, 8, 4096, err);
        t.ssp_steps = knob("MUX_SSP_STEPS", t.ssp_steps, 1, 100000, err);
        t.ssp_deep = knob("MUX_SSP_DEEP", t.ssp_deep, 0, 1000, err);
        t.ssp_coarse_pops = knob("MUX_SSP_COARSE_POPS", 0, 0, 1000000000, err);
        t.ssp_serial = knob("MUX_SSP_SERIAL", 0, 0, 1, err) == 1;
        t.ssp_pf = knob("MUX_SSP_PF", t.ssp_pf ? 1 : 0, 0, 1, err) == 1;
        t.ssp_l2pf = knob("MUX_SSP_L2PF", t.ssp_l2pf ? 1 : 0, 0, 1, err) == 1;
        t.ssp_ties = knob("MUX_SSP_TIES", t.ssp_ties ? 1 : 0, 0, 1, err) == 1;
        t.ssp_cluster = knob("MUX_SSP_CLUSTER", 1, 0, 1, err) == 1;
        t.ssp_sparsex = knob("MUX_SSP_SPARSEX", 0, 0, 1, err) == 1;
        t.ssp_one = knob("MUX_SSP_ONE", t.ssp_one, 0, 10240, err);
        t.ssp_ct = knob("MUX_SSP_CT", t.ssp_ct, 128, 1024, err);
        if (t.ssp_ct != 128 && t.ssp_ct != 256 && t.ssp_ct != 512 && t.ssp_ct != 1024 && err.empty()) err = "MUX_SSP_CT must be 128, 256, 512 or 1024";
        t.ssp_rslice = knob("MUX_SSP_RSLICE", 1, 0, 2, err);
        t.ssp_ct1 = knob("MUX_SSP_CT1", t.ssp_ct1, 512, 1024, err);
        if (t.ssp_ct1 != 512 && t.ssp_ct1 != 1024 && err.empty()) err = "MUX_SSP_CT1 must be 512 or 1024";
        t.ssp_dump = getenv("MUX_SSP_DUMP");
        t.canon_dump = getenv("MUX_CANON_DUMP");
        t.ssp_seq = knob("MUX_SSP_SEQ", t.ssp_seq, 0, 4096, err);
        t.ssp_rpf = knob("MUX_SSP_RPF", t.ssp_rpf, 0, 64, err);
        t.ssp_rpf_mb = knob("MUX_SSP_RPF_MB", t.ssp_rpf_mb, 0, 65536, err);
        t.ssp_lwalk = knob("MUX_SSP_LWALK", t.ssp_lwalk ? 1 : 0, 0, 1, err) == 1;
        t.ssp_cperm = knob("MUX_SSP_CPERM", t.ssp_cperm ? 1 : 0, 0, 1, err) == 1;
        t.ssp_wide = knob("MUX_SSP_WIDE", t.ssp_wide ? 1 : 0, 0, 1, err) == 1;
        t.ssp_taildef = knob("MUX_SSP_TAILDEF", t.ssp_taildef, 0, 4096, err);
        t.ssp_dorder = knob("MUX_SSP_DORDER", t.ssp_dorder, 0, 2, err);
        t.auc_theta = knob("MUX_THETA", t.auc_theta, 2, 64, err);
        t.auc_tail = knob("MUX_TAIL", t.auc_tail, -1, 1 << 20, err);   // clamped to the tail buffer inside
        t.auc_k = knob("MUX_K", t.auc_k, 1, 15, err);
        t.auc_cg_sync = knob("MUX_CG_SYNC", 1, 0, 1, err) == 1;
        t.auc_async_tail = knob("MUX_ASYNC_TAIL", -1, -1, 1, err);
        t.auc_async_phases = knob("MUX_ASYNC_PHASES", t.auc_async_phases, 0, 1 << 20, err);
        t.auc_fresh = knob("MUX_FRESH", 1, 0, 2, err);
        t.auc_restage = knob("MUX_RESTAGE", 0, 0, 2, err);
        t.auc_order = knob("MUX_ORDER", 1, 0, 2, err);
        t.auc_no_smem = knob("MUX_NO_SMEM", 0, 0, 1, err) == 1;
        t.mlp_prefetch = knob("MUX_MLP_PREFETCH", t.mlp_prefetch ? 1 : 0, 0, 1, err) == 1;
    }
    t.error = !err.empty();
    if (t.error) set_error("bad tuning knob: " + err);
    return t;
}

// Read back and clear the device error flags; maps a range error to EINVAL.
static int check_flags(mux_ctx_t* ctx, cudaStream_t st) {
    uint32_t f = 0;
    MUX_CUDA_TRY(cudaMemcpyAsync(&f, ctx->flags.ptr, sizeof(f), cudaMemcpyDeviceToHost, st));
    MUX_CUDA_TRY(cudaStreamSynchronize(st));
    if (f) MUX_CUDA_TRY(cudaMemsetAsync(ctx->flags.ptr, 0, sizeof(uint32_t), st));
    if (f & kErrQueryRange) { set_error("query coordinate outside [0, 1]"); return MUX_EINVAL; }
    return MUX_OK;
}

static int pinned_ensure(mux_ctx_t* ctx, size_t bytes) {
    if (bytes <= ctx->pinned_bytes) return MUX_OK;
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    ctx->pinned = nullptr;
    ctx->pinned_bytes = 0;
    size_t cap = bytes + bytes / 4 + 4096;
    MUX_CUDA_TRY(cudaMallocHost(&ctx->pinned, cap));
    ctx->pinned_bytes = cap;
    return MUX_OK;
}
struct EventPair {
    cudaEvent_t e[2] = {nullptr, nullptr};
    ~EventPair() { for (auto& x : e) if (x) cudaEventDestroy(x); }
};

// Scoring + matching of one round on device-resident features.  wq_dev may be
// null (the context's buffer is used); rowkey/colkey are HOST copies of x / y.
static int round_device(mux_ctx_t* ctx, const mux_table_t* table, const double* x, const double* s, int64_t n,
                        const double* y, int64_t m, int qbits, void* wq_dev, int64_t ldw, const double* rowkey,
                        const double* colkey, int32_t* col_dev, int64_t* total_q, mux_stats_t* stats,
                        cudaStream_t st, int64_t* price_io = nullptr, int warm = 0,
                        const int32_t* warm_col = nullptr) {
    // weights are int32 up to 30 bits, int64 beyond (the exact-parity mode)
    const int wt = qbits > 30 ? MUX_W_I64 : MUX_W_I32;
    const int64_t esz = wt == MUX_W_I64 ? 8 : 4, vec = 16 / esz;
    const int64_t ldw_min = ((m + vec - 1) / vec) * vec;
    void* W = wq_dev;
    if (W == nullptr) {
        ldw = ldw_min;
        MUX_TRY(ctx->wq.ensure((size_t)esz * (size_t)n * (size_t)(ldw > 0 ? ldw : vec)));
        W = ctx->wq.ptr;
    } else if (ldw < ldw_min || (ldw % vec) != 0 || (reinterpret_cast<uintptr_t>(W) & 15)) {
        set_error("round: weight buffer rows must hold m entries, 16-byte aligned");
        return MUX_EINVAL;
    }
    EventPair ev;
    MUX_CUDA_TRY(cudaEventCreate(&ev.e[0]));
    MUX_CUDA_TRY(cudaEventCreate(&ev.e[1]));
    MUX_CUDA_TRY(cudaEventRecord(ev.e[0], st));
    int64_t launches = 0;
    if (m > 0)
        MUX_TRY(mux_score_table_impl(ctx, table, x, s, n, y, m, MUX_SCORE_EXACT, wt, qbits, W, ldw, st, &launches));
    MUX_CUDA_TRY(cudaEventRecord(ev.e[1], st));
    MUX_TRY(check_flags(ctx, st));
    float ms_score = 0.f;
    cudaEventElapsedTime(&ms_score, ev.e[0], ev.e[1]);
    MUX_TRY(mux_match_impl(ctx, W, wt, n, m, ldw, col_dev, total_q, stats, st, tuning().auc_theta,
                           tuning().auc_tail, rowkey, colkey, price_io, warm, warm_col));
    if (stats) {
        stats->ms_score = ms_score;
        stats->launches += launches;
    }
    return MUX_OK;
}
}  // namespace mux

using namespace mux;

extern "C" {

const char* mux_version(void) { return "muxflow-b200 0.1 (sm_100a)"; }
const char* mux_last_error(void) { return g_last_error.c_str(); }

int mux_ctx_create(int device, mux_ctx_t** out) {
    if (!out) { set_error("mux_ctx_create: null out"); return MUX_EINVAL; }
    *out = nullptr;
    int ndev = 0;
    MUX_CUDA_TRY(cudaGetDeviceCount(&ndev));
    if (device < 0 || device >= ndev) { set_error("mux_ctx_create: bad device"); return MUX_EINVAL; }
    MUX_CUDA_TRY(cudaSetDevice(device));
    cudaDeviceProp prop;
    MUX_CUDA_TRY(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) {
        set_error("muxflow is built for sm_100a (B200); device is sm_" + std::to_string(prop.major * 10 + prop.minor));
        return MUX_ECUDA;
    }
    mux_ctx_t* c = new mux_ctx();
    c->device = device;
    c->num_sms = prop.multiProcessorCount;
    int rc = c->flags.ensure(256);
    if (rc != MUX_OK) { delete c; return rc; }
    if (cudaMemset(c->flags.ptr, 0, 256) != cudaSuccess) { delete c; set_error("memset"); return MUX_ECUDA; }
    *out = c;
    return MUX_OK;
}

int mux_ctx_destroy(mux_ctx_t* ctx) {
    if (!ctx) return MUX_OK;
    cudaSetDevice(ctx->device);
    if (ctx->ipc_in) cudaIpcCloseMemHandle(ctx->ipc_in);
    for (DevBuf* b : {&ctx->table, &ctx->rowfeat, &ctx->colfeat, &ctx->flags, &ctx->ipc_out, &ctx->feat_in, &ctx->wq,
                      &ctx->colout, &ctx->auc, &ctx->ssp, &ctx->canon, &ctx->canon_ent, &ctx->mlp})
        b->release();
    if (ctx->pinned) cudaFreeHost(ctx->pinned);
    delete ctx;
    return MUX_OK;
}

// predictor.py:29-37 (_check_axis) and 56-71 (PredictionTable.__post_init__).
int mux_table_validate(const mux_table_t* t) {
    if (!t) { set_error("null table"); return MUX_EINVAL; }
    const int32_t dims[3] = {t->n_online_sm, t->n_offline_sm, t->n_sm_pct};
    const double* axes[3] = {t->online_sm, t->offline_sm, t->sm_pct};
    const char* names[3] = {"online_sm", "offline_sm", "sm_pct"};
    for (int a = 0; a < 3; ++a) {
        if (dims[a] <= 0 || !axes[a]) { set_error(std::string("axis ") + names[a] + " is empty"); return MUX_EINVAL; }
        for (int k = 0; k < dims[a]; ++k) {
            const double v = axes[a][k];
            if (!(v >= 0.0 && v <= 1.0)) { set_error(std::string("axis ") + names[a] + " knot outside [0, 1]"); return MUX_EINVAL; }
            if (k > 0 && !(axes[a][k - 1] < v)) { set_error(std::string("axis ") + names[a] + " knots not strictly increasing"); return MUX_EINVAL; }
        }
    }
    if (!t->values) { set_error("table values missing"); return MUX_EINVAL; }
    const int64_t nv = (int64_t)dims[0] * dims[1] * dims[2];
    // table offsets are int32 on the device (csrc/score.cu)
    if (nv > (int64_t)INT32_MAX) { set_error("table has more than 2^31 - 1 values"); return MUX_EINVAL; }
    double lo = INFINITY, hi = -INFINITY;
    for (int64_t e = 0; e < nv; ++e) {
        const double v = t->values[e];
        if (!std::isfinite(v)) { set_error("table contains non-finite values"); return MUX_EINVAL; }
        lo = v < lo ? v : lo;
        hi = v > hi ? v : hi;
    }
    if (lo < 0.0 || hi > 1.0) { set_error("table values outside [0, 1]"); return MUX_EINVAL; }
    if (dims[2] > 1) {
        double dmin = INFINITY;
        for (int64_t e = 0; e < nv; e += dims[2])
            for (int k = 1; k < dims[2]; ++k) {
                const double d = t->values[e + k] - t->values[e + k - 1];
                dmin = d < dmin ? d : dmin;
            }
        if (dmin < -1e-12) { set_error("values decrease along the sm_pct axis"); return MUX_EINVAL; }
    }
    return MUX_OK;
}

int mux_score_table(mux_ctx_t* ctx, const mux_table_t* table, const double* x_dev, const double* share_dev,
                    int64_t n, const double* y_dev, int64_t m, int mode, int wtype, int qbits, void* out_dev,
                    int64_t ldo, void* stream) {
    if (!ctx) { set_error("null context"); return MUX_EINVAL; }
    MUX_TRY(mux_table_validate(table));
    if (n < 0 || m < 0 || ldo < m) { set_error("mux_score_table: bad shape"); return MUX_EINVAL; }
    if (mode != MUX_SCORE_EXACT && mode != MUX_SCORE_FAST) { set_error("bad mode"); return MUX_EINVAL; }
    if (wtype < MUX_W_F64 || wtype > MUX_W_I64) { set_error("bad wtype"); return MUX_EINVAL; }
    const int maxbits = wtype == MUX_W_I32 ? 30 : 52;
    if ((wtype == MUX_W_I32 || wtype == MUX_W_I64) && (qbits < 0 || qbits > maxbits)) {
        set_error("qbits out of range for the output type");
        return MUX_EINVAL;
    }
    const int vec = (wtype == MUX_W_I32 || wtype == MUX_W_F32) ? 4 : 2;
    if (n > 0 && ((ldo % vec) != 0 || (reinterpret_cast<uintptr_t>(out_dev) & 15))) {
        set_error("mux_score_table: output rows must be 16-byte aligned");
        return MUX_EINVAL;
    }
    MUX_CUDA_TRY(cudaSetDevice(ctx->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int64_t launches = 0;
    MUX_TRY(mux_score_table_impl(ctx, table, x_dev, share_dev, n, y_dev, m, mode, wtype, qbits, out_dev, ldo, st, &launches));
    return check_flags(ctx, st);
}

int mux_score_mlp(mux_ctx_t* ctx, const mux_mlp_t* mlp, const double* on_dev, const double* share_dev,
                  int64_t n, const double* off_dev, int64_t m, int wtype, int qbits, void* out_dev, int64_t ldo,
                  void* stream) {
    if (!ctx || !mlp) { set_error("null argument"); return MUX_EINVAL; }
    if (n < 0 || m < 0 || ldo < m || (ldo % 4) != 0) { set_error("mux_score_mlp: bad shape"); return MUX_EINVAL; }
    if (wtype != MUX_W_F32 && wtype != MUX_W_I32) { set_error("mux_score_mlp: output must be f32 or i32"); return MUX_EINVAL; }
    if (wtype == MUX_W_I32 && (qbits < 0 || qbits > 30)) { set_error("qbits out of range"); return MUX_EINVAL; }
    const float* ps[] = {mlp->W1, mlp->b1, mlp->W2, mlp->b2, mlp->W3, mlp->b3, mlp->w4, mlp->shift, mlp->scale};
    for (const float* q : ps) if (!q) { set_error("mux_score_mlp: missing parameter"); return MUX_EINVAL; }
    MUX_CUDA_TRY(cudaSetDevice(ctx->device));
    int64_t launches = 0;
    return mux_score_mlp_impl(ctx, mlp, on_dev, share_dev, n, off_dev, m, wtype, qbits, out_dev, ldo,
                              static_cast<cudaStream_t>(stream), &launches);
}

int mux_match(mux_ctx_t* ctx, const void* Wq_dev, int wtype, int64_t n, int64_t m, int64_t ldw,
              int32_t* col_of_row_out, int out_on_host, int64_t* total_q, mux_stats_t* stats, void* stream) {
    if (!ctx) { set_error("null context"); return MUX_EINVAL; }
    MUX_CUDA_TRY(cudaSetDevice(ctx->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int32_t* col_dev = col_of_row_out;
    if (out_on_host) {
        MUX_TRY(ctx->colout.ensure(sizeof(int32_t) * (size_t)(n > 0 ? n : 1)));
        col_dev = ctx->colout.as<int32_t>();
    }
    if (stats) memset(stats, 0, sizeof(*stats));
    MUX_TRY(mux_match_impl(ctx, Wq_dev, wtype, n, m, ldw, col_dev, total_q, stats, st,
                           tuning().auc_theta, tuning().auc_tail, nullptr, nullptr));
    if (out_on_host && n > 0) {
        MUX_CUDA_TRY(cudaMemcpyAsync(col_of_row_out, col_dev, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
        MUX_CUDA_TRY(cudaStreamSynchronize(st));
    }
    return MUX_OK;
}

int mux_match_keyed(mux_ctx_t* ctx, const void* Wq_dev, int wtype, int64_t n, int64_t m, int64_t ldw,
                    const double* rowkey_dev, const double* colkey_dev, int32_t* col_of_row_out, int out_on_host,
                    int64_t* total_q, mux_stats_t* stats, void* stream) {
    if (!ctx) { set_error("null context"); return MUX_EINVAL; }
    if ((rowkey_dev == nullptr) != (colkey_dev == nullptr)) { set_error("mux_match_keyed: give both keys or neither"); return MUX_EINVAL; }
    MUX_CUDA_TRY(cudaSetDevice(ctx->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    std::vector<double> rk, ck;
    if (rowkey_dev && n > 0 && m > 0) {
        rk.resize(n);
        ck.resize(m);
        MUX_CUDA_TRY(cudaMemcpyAsync(rk.data(), rowkey_dev, 8ull * n, cudaMemcpyDeviceToHost, st));
        MUX_CUDA_TRY(cudaMemcpyAsync(ck.data(), colkey_dev, 8ull * m, cudaMemcpyDeviceToHost, st));
        MUX_CUDA_TRY(cudaStreamSynchronize(st));
    }
    int32_t* col_dev = col_of_row_out;
    if (out_on_host) {
        MUX_TRY(ctx->colout.ensure(sizeof(int32_t) * (size_t)(n > 0 ? n : 1)));
        col_dev = ctx->colout.as<int32_t>();
    }
    if (stats) memset(stats, 0, sizeof(*stats));
    MUX_TRY(mux_match_impl(ctx, Wq_dev, wtype, n, m, ldw, col_dev, total_q, stats, st,
                           tuning().auc_theta, tuning().auc_tail,
                           rk.empty() ? nullptr : rk.data(), ck.empty() ? nullptr : ck.data()));
    if (out_on_host && n > 0) {
        MUX_CUDA_TRY(cudaMemcpyAsync(col_of_row_out, col_dev, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
        MUX_CUDA_TRY(cudaStreamSynchronize(st));
    }
    return MUX_OK;
}

int mux_round(mux_ctx_t* ctx, const mux_table_t* table, const double* x_host, const double* share_host,
              int64_t n, const double* y_host, int64_t m, int qbits, int32_t* col_of_row_host,
              int64_t* total_q, mux_stats_t* stats, void* stream) {
    if (!ctx) { set_error("null context"); return MUX_EINVAL; }
    MUX_TRY(mux_table_validate(table));
    if (n < 0 || m < 0) { set_error("mux_round: bad shape"); return MUX_EINVAL; }
    if (qbits < 1 || qbits > 52) { set_error("mux_round: qbits must be in [1, 52]"); return MUX_EINVAL; }
    MUX_CUDA_TRY(cudaSetDevice(ctx->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (stats) memset(stats, 0, sizeof(*stats));
    if (total_q) *total_q = 0;
    if (n == 0) return MUX_OK;
    // H2D of the feature arrays through pinned staging (2n + m doubles)
    const size_t fbytes = sizeof(double) * (size_t)(2 * n + m);
    MUX_TRY(pinned_ensure(ctx, fbytes));
    double* hp = static_cast<double*>(ctx->pinned);
    memcpy(hp, x_host, sizeof(double) * n);
    memcpy(hp + n, share_host, sizeof(double) * n);
    if (m) memcpy(hp + 2 * n, y_host, sizeof(double) * m);
    MUX_TRY(ctx->feat_in.ensure(fbytes));
    double* dfeat = ctx->feat_in.as<double>();
    MUX_CUDA_TRY(cudaMemcpyAsync(dfeat, hp, fbytes, cudaMemcpyHostToDevice, st));
    MUX_TRY(ctx->colout.ensure(sizeof(int32_t) * (size_t)n));
    int32_t* col_dev = ctx->colout.as<int32_t>();
    MUX_TRY(round_device(ctx, table, dfeat, dfeat + n, n, dfeat + 2 * n, m, qbits, nullptr, 0, x_host, y_host,
                         col_dev, total_q, stats, st));
    MUX_CUDA_TRY(cudaMemcpyAsync(col_of_row_host, col_dev, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
    MUX_CUDA_TRY(cudaStreamSynchronize(st));
    return MUX_OK;
}

int mux_round_dev(mux_ctx_t* ctx, const mux_table_t* table, const double* x_dev, const double* share_dev,
                  int64_t n, const double* y_dev, int64_t m, int qbits, void* wq_dev, int64_t ldw,
                  int32_t* col_of_row_dev, int64_t* prices_dev, const int32_t* warm_col_dev, int warm,
                  int64_t* total_q, mux_stats_t* stats, void* stream) {
    if (!ctx) { set_error("null context"); return MUX_EINVAL; }
    MUX_TRY(mux_table_validate(table));
    if (n < 0 || m < 0) { set_error("mux_round_dev: bad shape"); return MUX_EINVAL; }
    if (qbits < 1 || qbits > 52) { set_error("mux_round_dev: qbits must be in [1, 52]"); return MUX_EINVAL; }
    MUX_CUDA_TRY(cudaSetDevice(ctx->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (stats) memset(stats, 0, sizeof(*stats));
    if (total_q) *total_q = 0;
    if (n == 0) return MUX_OK;
    // host copies of the ordering keys (the solver sorts them on the host)
    std::vector<double> rk(n), ck(m > 0 ? m : 1);
    MUX_CUDA_TRY(cudaMemcpyAsync(rk.data(), x_dev, 8ull * n, cudaMemcpyDeviceToHost, st));
    if (m) MUX_CUDA_TRY(cudaMemcpyAsync(ck.data(), y_dev, 8ull * m, cudaMemcpyDeviceToHost, st));
    MUX_CUDA_TRY(cudaStreamSynchronize(st));
    if (warm && !prices_dev) { set_error("mux_round_dev: warm start needs prices_dev"); return MUX_EINVAL; }
    return round_device(ctx, table, x_dev, share_dev, n, y_dev, m, qbits, wq_dev, ldw, rk.data(), ck.data(),
                        col_of_row_dev, total_q, stats, st, prices_dev, warm, warm_col_dev);
}

int mux_round_mlp(mux_ctx_t* ctx, const mux_mlp_t* mlp, const double* on_host, const double* share_host, int64_t n,
                  const double* off_host, int64_t m, int qbits, int32_t* col_of_row_host, int64_t* total_q,
                  mux_stats_t* stats, void* stream) {
    if (!ctx || !mlp) { set_error("null argument"); return MUX_EINVAL; }
    if (n < 0 || m < 0) { set_error("mux_round_mlp: bad shape"); return MUX_EINVAL; }
    if (qbits < 1 || qbits > 30) { set_error("mux_round_mlp: qbits must be in [1, 30]"); return MUX_EINVAL; }
    MUX_CUDA_TRY(cudaSetDevice(ctx->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    if (stats) memset(stats, 0, sizeof(*stats));
    if (total_q) *total_q = 0;
    if (n == 0) return MUX_OK;
    const size_t fbytes = sizeof(double) * (size_t)(5 * n + 4 * m);
    MUX_TRY(pinned_ensure(ctx, fbytes));
    double* hp = static_cast<double*>(ctx->pinned);
    memcpy(hp, on_host, sizeof(double) * 4 * n);
    memcpy(hp + 4 * n, share_host, sizeof(double) * n);
    if (m) memcpy(hp + 5 * n, off_host, sizeof(double) * 4 * m);
    MUX_TRY(ctx->feat_in.ensure(fbytes));
    double* df = ctx->feat_in.as<double>();
    MUX_CUDA_TRY(cudaMemcpyAsync(df, hp, fbytes, cudaMemcpyHostToDevice, st));
    const int64_t ldw = ((m + 3) / 4) * 4;
    MUX_TRY(ctx->wq.ensure(4ull * (size_t)n * (size_t)(ldw > 0 ? ldw : 4)));
    MUX_TRY(ctx->colout.ensure(sizeof(int32_t) * (size_t)n));
    int32_t* col_dev = ctx->colout.as<int32_t>();
    EventPair ev;
    MUX_CUDA_TRY(cudaEventCreate(&ev.e[0]));
    MUX_CUDA_TRY(cudaEventCreate(&ev.e[1]));
    MUX_CUDA_TRY(cudaEventRecord(ev.e[0], st));
    int64_t launches = 0;
    if (m > 0)
        MUX_TRY(mux_score_mlp_impl(ctx, mlp, df, df + 4 * n, n, df + 5 * n, m, MUX_W_I32, qbits, ctx->wq.ptr, ldw, st,
                                   &launches));
    MUX_CUDA_TRY(cudaEventRecord(ev.e[1], st));
    // generic ordering keys for the multilevel warm start: row / column sums
    MUX_TRY(mux_match_impl(ctx, ctx->wq.ptr, MUX_W_I32, n, m, ldw, col_dev, total_q, stats, st, tuning().auc_theta,
                           tuning().auc_tail, nullptr, nullptr));
    MUX_CUDA_TRY(cudaMemcpyAsync(col_of_row_host, col_dev, sizeof(int32_t) * n, cudaMemcpyDeviceToHost, st));
    MUX_CUDA_TRY(cudaStreamSynchronize(st));
    if (stats) {
        float ms = 0.f;
        cudaEventElapsedTime(&ms, ev.e[0], ev.e[1]);
        stats->ms_score = ms;
        stats->launches += launches;
    }
    return MUX_OK;
}

int mux_ipc_export(mux_ctx_t* ctx, int64_t bytes, void** dev_ptr, void* handle_out) {
    if (!ctx || !dev_ptr || !handle_out || bytes <= 0) { set_error("mux_ipc_export: bad argument"); return MUX_EINVAL; }
    MUX_CUDA_TRY(cudaSetDevice(ctx->device));
    MUX_TRY(ctx->ipc_out.ensure((size_t)bytes));
    cudaIpcMemHandle_t h;
    MUX_CUDA_TRY(cudaIpcGetMemHandle(&h, ctx->ipc_out.ptr));
    memcpy(handle_out, &h, sizeof(h));
    *dev_ptr = ctx->ipc_out.ptr;
    return MUX_OK;
}

int mux_ipc_import(mux_ctx_t* ctx, const void* handle, void** dev_ptr) {
    if (!ctx || !handle || !dev_ptr) { set_error("mux_ipc_import: bad argument"); return MUX_EINVAL; }
    MUX_CUDA_TRY(cudaSetDevice(ctx->device));
    if (ctx->ipc_in) { cudaIpcCloseMemHandle(ctx->ipc_in); ctx->ipc_in = nullptr; }
    cudaIpcMemHandle_t h;
    memcpy(&h, handle, sizeof(h));
    MUX_CUDA_TRY(cudaIpcOpenMemHandle(&ctx->ipc_in, h, cudaIpcMemLazyEnablePeerAccess));
    *dev_ptr = ctx->ipc_in;
    return MUX_OK;
}

}  // extern "C"
