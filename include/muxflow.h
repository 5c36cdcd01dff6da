/*
 * muxflow.h -- C ABI of the B200-native MuxFlow scheduling round.
 *
 * The reference (/root/reference/pkg/src/muxsim) is pure Python; its hot
 * path is `scheduler.schedule` -> `predict` for every (online, offline) pair
 * -> `max_weight_matching` (SURVEY.md §3 stack A).  Each entry point below
 * replaces one piece of that path; the Python host mirror in
 * `paper_2303_13803_b200/` binds them with ctypes (see INTEGRATION.md for the
 * binding a reference maintainer would add).
 *
 * Conventions
 *   - Plain pointers and sizes only; no torch types.  "_dev" pointers are CUDA
 *     device pointers, "_host" pointers are host memory (pinned or pageable).
 *   - `stream` is a cudaStream_t passed as void* (NULL = legacy default stream).
 *   - Every function returns a status (MUX_OK = 0).  The Python layer maps
 *     MUX_EINVAL -> ValueError/TableError and MUX_ECUDA/MUX_ENOMEM ->
 *     SchedulingAborted, mirroring the reference's error types
 *     (predictor.py:25-26, scheduler.py:32-33).  `mux_last_error()` returns a
 *     thread-local message for the last failure.
 *   - All calls are re-entrant per context; a context owns its device
 *     workspace and must not be used from two host threads at once.
 */
#ifndef MUXFLOW_H
#define MUXFLOW_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define MUX_OK      0
#define MUX_EINVAL  1   /* bad argument / table / out-of-range query  */
#define MUX_ECUDA   2   /* CUDA runtime or kernel failure             */
#define MUX_ENOMEM  3   /* device or host allocation failure          */
#define MUX_ELIMIT  4   /* solver iteration guard tripped (never expected) */

/* Weight element types for mux_score_* outputs and mux_match inputs. */
#define MUX_W_F64   0   /* float64 weights in [0, 1] (exact predictor values) */
#define MUX_W_F32   1   /* float32 weights in [0, 1]                          */
#define MUX_W_I32   2   /* int32 quantised weights rint(w * 2^qbits), qbits <= 30 */
#define MUX_W_I64   3   /* int64 quantised weights, qbits <= 44                   */

/* Scoring arithmetic. */
#define MUX_SCORE_EXACT 0  /* float64, bit-identical to predictor.predict_point */
#define MUX_SCORE_FAST  1  /* float32 rank-J contraction     */

/* Dense prediction table: predictor.py:40-71 (PredictionTable).  values is
 * C-order [n_online_sm][n_offline_sm][n_sm_pct], online_sm outermost.      */
typedef struct {
    int32_t n_online_sm;
    int32_t n_offline_sm;
    int32_t n_sm_pct;
    int32_t _pad;
    const double* online_sm;   /* host pointers */
    const double* offline_sm;
    const double* sm_pct;
    const double* values;
} mux_table_t;

/* MLP speed-predictor plugin weights (paper's predictor; no
 * reference counterpart).  Network in(9) -> 64 -> 64 -> 64 -> 1 with ReLU,
 * output clamped to [0, 1]; features are scaled (x - shift) * scale and
 * ordered [online(4), offline(4), share], each workload contributing
 * (gpu_utilization, sm_activity, sm_occupancy, iter_time_separate).
 * Weight matrices are row-major [out][in].  Host pointers. */
typedef struct {
    const float* W1;     /* [64][9]  */
    const float* b1;     /* [64]     */
    const float* W2;     /* [64][64] */
    const float* b2;     /* [64]     */
    const float* W3;     /* [64][64] */
    const float* b3;     /* [64]     */
    const float* w4;     /* [64]     */
    const float* shift;  /* [9]      */
    const float* scale;  /* [9]      */
    float b4;
    int32_t hidden;      /* must be 64 */
} mux_mlp_t;

/* Per-solve statistics (filled by mux_match / mux_round when non-NULL). */
typedef struct {
    int64_t n_rows;          /* N (real online rows)                      */
    int64_t n_cols;          /* M (real offline columns)                  */
    int64_t n_square;        /* max(N, M): the padded square size          */
    int64_t phases;          /* epsilon-scaling phases run                 */
    int64_t rounds;          /* auction: bidding rounds (grid barriers); ssp: long-path exchange steps */
    int64_t bids;            /* accepted + rejected bids                   */
    int64_t row_scans;       /* full weight-row reads                      */
    int64_t tail_bids;       /* bids made in single-CTA tail mode          */
    int64_t total_q;         /* optimal total, in quantised units          */
    double  ms_score;        /* device time of the scoring kernel(s)       */
    double  ms_match;        /* wall time of the matching (solve + canonicalisation) */
    int64_t launches;        /* kernel launches issued by the call         */
    double  ms_tail;         /* device time in single-CTA tail mode        */
    double  ms_kernel;       /* solver time (multilevel solver: as ms_match; auction: kernel time) */
    int64_t cache_hits;      /* bids served from the candidate cache       */
    double  ms_canon;        /* host time of the tie canonicalisation (incl. its kernels) */
    int64_t canon_searches;  /* alternating-path searches it ran           */
    int64_t tight_edges;     /* tight edges of the real rows               */
    int64_t dual_sweeps;     /* Bellman-Ford sweeps of the exact-dual repair */
    /* multilevel shortest-path solver (csrc/ssp.cu) */
    int64_t levels;          /* coarse-to-fine levels solved               */
    int64_t par_steps;       /* Dijkstra pops of the parallel warp searches */
    int64_t dense_steps;     /* pops of the single-CTA dense searches       */
    int64_t dense_searches;  /* searches handed to the dense kernel         */
    double  ms_dense;        /* device time of the dense kernel (events)    */
    double  ms_parallel;     /* device time of the parallel passes (events) */
    double  dense_bytes;     /* weight-row bytes the dense kernel read (4 m per pop) */
    int64_t dense_launches;  /* launches of the long-path kernel              */
} mux_stats_t;

typedef struct mux_ctx mux_ctx_t;

/* Library identity / version. */
const char* mux_version(void);
/* Thread-local message describing the last non-OK status. */
const char* mux_last_error(void);

/* Create a context bound to CUDA device `device` (workspace grows on demand). */
int mux_ctx_create(int device, mux_ctx_t** out);
int mux_ctx_destroy(mux_ctx_t* ctx);

/* Validate a table exactly like PredictionTable.__post_init__
 * (predictor.py:29-71): axes non-empty, in [0,1], strictly increasing;
 * values finite, in [0,1], non-decreasing along sm_pct within 1e-12. */
int mux_table_validate(const mux_table_t* table);

/*
 * Pair scoring (replaces the N x M predict() loop, scheduler.py:172-180, and
 * predictor.py:85-118).  x_dev / share_dev: float64 [n] (online peak SM
 * activity, granted share), y_dev: float64 [m] (offline SM demand) -- DEVICE
 * pointers.  Output out_dev is row-major [n][ldo] of type wtype; quantised
 * outputs apply the reference edge rule first (w < 1e-6 -> 0,
 * matching.py:19, 159-162).  Coordinates outside [0,1] -> MUX_EINVAL
 * (predictor.py:93-96), checked on the device.
 */
int mux_score_table(mux_ctx_t* ctx, const mux_table_t* table,
                    const double* x_dev, const double* share_dev, int64_t n,
                    const double* y_dev, int64_t m,
                    int mode, int wtype, int qbits,
                    void* out_dev, int64_t ldo, void* stream);

/*
 * MLP pair scoring: the batched N x M evaluation of the MLP plugin, layers
 * 2-3 as tcgen05 fp16 GEMMs over split (hi + lo) activations with fp32 TMEM
 * accumulation and fused ReLU/dot epilogues; W2, b2, W3, b3 must be fp16
 * values (MUX_EINVAL otherwise).  on_dev: float64 [n][4], share_dev: float64 [n],
 * off_dev: float64 [m][4] (DEVICE).  out_dev: [n][ldo] of MUX_W_F32 (scores)
 * or MUX_W_I32 (rint(w * 2^qbits) after the 1e-6 edge floor), ldo % 4 == 0.
 */
int mux_score_mlp(mux_ctx_t* ctx, const mux_mlp_t* mlp,
                  const double* on_dev, const double* share_dev, int64_t n,
                  const double* off_dev, int64_t m, int wtype, int qbits,
                  void* out_dev, int64_t ldo, void* stream);

/*
 * Maximum-weight bipartite matching on non-negative integer weights
 * (replaces max_weight_matching, matching.py:148-208, including its tie
 * canonicalisation, matching.py:173-199).  Wq_dev: row-major [n][ldw] of wtype MUX_W_I32 or
 * MUX_W_I64 (0 = missing edge).  Solves the reference's zero-padded square
 * problem exactly: the multilevel successive-shortest-path solver (csrc/ssp.cu;
 * int64 weights up to 44 bits with max(n, m) < 60,000, csrc/ssp_w64.cu), the
 * epsilon-scaling auction beyond that or under MUX_TUNING=1 MUX_SOLVER=auction.
 * col_of_row_out: int32 [n], -1 when the row is unmatched or
 * matched through a zero-weight / padding edge (the reference never emits
 * those, matching.py:201-208); may be a host or device pointer
 * (`out_on_host`).  *total_q receives the optimal total in quantised units.
 */
int mux_match(mux_ctx_t* ctx, const void* Wq_dev, int wtype,
              int64_t n, int64_t m, int64_t ldw,
              int32_t* col_of_row_out, int out_on_host,
              int64_t* total_q, mux_stats_t* stats, void* stream);

/*
 * mux_match with ordering keys for the multilevel solver: rowkey_dev[n] and
 * colkey_dev[m] (float64, DEVICE) order rows and columns by similarity -- for
 * the table predictor the online and offline SM demands.  NULL keys fall back
 * to row / column sums of the weights.  Same results as mux_match (the keys
 * only steer the warm start, never the optimum).
 */
int mux_match_keyed(mux_ctx_t* ctx, const void* Wq_dev, int wtype,
                    int64_t n, int64_t m, int64_t ldw,
                    const double* rowkey_dev, const double* colkey_dev,
                    int32_t* col_of_row_out, int out_on_host,
                    int64_t* total_q, mux_stats_t* stats, void* stream);

/*
 * One fused scheduling round from HOST feature arrays (the call the
 * reference's `_matching_policy_schedule` makes per round, scheduler.py:143-194):
 * H2D copy of (x, share, y), exact scoring into quantised weights, the solve,
 * D2H copy of col_of_row.  Rows with share <= 0 must already be filtered by
 * the caller (scheduler.py:164-165), as must inadmissible columns
 * (scheduler.py:138-140).  qbits in [1, 52]: weights rint(w * 2^qbits) are
 * int32 up to 30 bits and int64 above (the exact-parity mode that schedule()
 * uses for rounds up to 6,144: 40 bits); the int64 solver's keys bound qbits
 * by 44, the auction's bid packing by about 60 - 2 log2(max(n, m)).
 */
int mux_round(mux_ctx_t* ctx, const mux_table_t* table,
              const double* x_host, const double* share_host, int64_t n,
              const double* y_host, int64_t m, int qbits,
              int32_t* col_of_row_host, int64_t* total_q,
              mux_stats_t* stats, void* stream);

/*
 * mux_round on DEVICE-resident features (x_dev, share_dev [n], y_dev [m]):
 * the same scoring + matching with the weights written to wq_dev ([n][ldw],
 * int32 for qbits <= 30 else int64, rows 16-byte aligned; NULL = the
 * context's own buffer) and col_of_row_dev (int32 [n], device).  Used when
 * the features already live in HBM (a resident cluster snapshot).
 *
 * Warm start across rounds (config 5 replays): prices_dev (int64 [m],
 * device, or NULL) receives the optimal column prices in quantised-weight
 * units (INT64_MIN where the solve has none to give: n > m rounds, int64
 * weights).  With warm = 1 it must hold the previous round's prices mapped
 * to this round's columns (INT64_MIN for new columns), and warm_col_dev
 * (int32 [n], device, or NULL) the previous round's column of each row in
 * this round's indices (-1 = none): previous pairs still tight under the
 * carried prices are kept and only the other rows are searched, instead of
 * the multilevel warm start.  Results are identical either way (optimal
 * total, canonical pairs); only the work changes.
 */
int mux_round_dev(mux_ctx_t* ctx, const mux_table_t* table,
                  const double* x_dev, const double* share_dev, int64_t n,
                  const double* y_dev, int64_t m, int qbits,
                  void* wq_dev, int64_t ldw, int32_t* col_of_row_dev,
                  int64_t* prices_dev, const int32_t* warm_col_dev, int warm,
                  int64_t* total_q, mux_stats_t* stats, void* stream);

/*
 * One scheduling round with the MLP plugin as the predictor, from HOST
 * feature arrays: on_host [n][4] and off_host [m][4] (gpu_utilization,
 * sm_activity, sm_occupancy, iter_time_separate), share_host [n].  H2D,
 * MLP scores of every pair quantised to rint(w * 2^qbits) (qbits <= 30, the
 * 1e-6 edge floor first), the exact matching with its tie
 * canonicalisation, D2H of col_of_row (-1 = unmatched).
 */
int mux_round_mlp(mux_ctx_t* ctx, const mux_mlp_t* mlp,
                  const double* on_host, const double* share_host, int64_t n,
                  const double* off_host, int64_t m, int qbits,
                  int32_t* col_of_row_host, int64_t* total_q,
                  mux_stats_t* stats, void* stream);

/*
 * Multi-GPU row-sharded scoring without a gather (one process per GPU,
 * sharded.py): the root exports a device buffer for the weight matrix
 * (allocated by the context, `bytes` long; handle_out receives the 64-byte
 * cudaIpcMemHandle), every other rank imports it (peer-mapped over NVLink,
 * one mapping per context) and passes `dev_ptr + its row offset` as the
 * out_dev of mux_score_table, so the scoring kernel's stores land in the
 * root's HBM directly.
 */
int mux_ipc_export(mux_ctx_t* ctx, int64_t bytes, void** dev_ptr, void* handle_out);
int mux_ipc_import(mux_ctx_t* ctx, const void* handle, void** dev_ptr);

#ifdef __cplusplus
}
#endif
#endif /* MUXFLOW_H */
