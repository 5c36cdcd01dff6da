/*
 * Oracle restatement of the reference Kuhn-Munkres solver -- TEST
 * INFRASTRUCTURE ONLY (never linked into the product library).
 *
 * Follows /root/reference/pkg/src/muxsim/matching.py:45-101
 * (`_solve_min_assignment`): shortest-augmenting-path Hungarian with exact
 * dual potentials u (rows) and v (columns).  Every per-element operation is
 * the same IEEE operation, in the same order, as the numpy statement it
 * restates:
 *     cur    = cost[i0] - u[i0] - v                 (matching.py:69)
 *     better = (~used) & (cur < minv)               (matching.py:70)
 *     j1     = argmin(minv with used -> inf)        (matching.py:73-75, first index)
 *     u[row_of_col[used]] += delta; v[used] -= delta (matching.py:77-78)
 *     u[i] += delta; minv[~used] -= delta            (matching.py:79-80)
 * so for float64 input the returned col_of_row / u / v are bit-identical to
 * the reference's (pinned by tests/test_oracle_golden.py).
 *
 * `hung_solve_i64` is the same algorithm on int64 costs: exact for the
 * integer-quantised weights used by the parity tests at sizes where float64
 * potentials could lose bits.
 */
#include <stdint.h>
#include <stdlib.h>
#include <math.h>

#define DEFINE_SOLVER(NAME, T, INF)                                            \
int NAME(const T* cost, int64_t n, int64_t* col_of_row, T* u, T* v) {          \
    if (n <= 0) return 0;                                                      \
    int64_t* row_of_col = (int64_t*)malloc(sizeof(int64_t) * n);               \
    T* minv = (T*)malloc(sizeof(T) * n);                                       \
    int64_t* way = (int64_t*)malloc(sizeof(int64_t) * n);                      \
    char* used = (char*)malloc(n);                                             \
    if (!row_of_col || !minv || !way || !used) {                               \
        free(row_of_col); free(minv); free(way); free(used); return 1;         \
    }                                                                          \
    for (int64_t j = 0; j < n; ++j) { u[j] = 0; v[j] = 0; row_of_col[j] = -1; }\
    for (int64_t i = 0; i < n; ++i) {                                          \
        for (int64_t j = 0; j < n; ++j) { minv[j] = INF; way[j] = -1; used[j] = 0; } \
        int64_t i0 = i, j_prev = -1, j1 = -1;                                  \
        int any_used = 0;                                                      \
        for (;;) {                                                             \
            const T* crow = cost + i0 * n;                                     \
            const T ui0 = u[i0];                                               \
            for (int64_t j = 0; j < n; ++j) {                                  \
                if (used[j]) continue;                                         \
                T cur = (crow[j] - ui0) - v[j];                                \
                if (cur < minv[j]) { minv[j] = cur; way[j] = j_prev; }         \
            }                                                                  \
            T delta = INF; j1 = -1;                                            \
            for (int64_t j = 0; j < n; ++j) {                                  \
                if (used[j]) continue;                                         \
                if (j1 < 0 || minv[j] < delta) { delta = minv[j]; j1 = j; }    \
            }                                                                  \
            if (any_used) {                                                    \
                for (int64_t j = 0; j < n; ++j)                                \
                    if (used[j]) { u[row_of_col[j]] += delta; v[j] -= delta; } \
            }                                                                  \
            u[i] += delta;                                                     \
            for (int64_t j = 0; j < n; ++j) if (!used[j]) minv[j] -= delta;    \
            used[j1] = 1; any_used = 1;                                        \
            if (row_of_col[j1] < 0) break;                                     \
            i0 = row_of_col[j1];                                               \
            j_prev = j1;                                                       \
        }                                                                      \
        int64_t j = j1;                                                        \
        for (;;) {                                                             \
            int64_t pj = way[j];                                               \
            if (pj < 0) { row_of_col[j] = i; break; }                          \
            row_of_col[j] = row_of_col[pj];                                    \
            j = pj;                                                            \
        }                                                                      \
    }                                                                          \
    for (int64_t j = 0; j < n; ++j) col_of_row[row_of_col[j]] = j;             \
    free(row_of_col); free(minv); free(way); free(used);                       \
    return 0;                                                                  \
}

DEFINE_SOLVER(hung_solve_f64, double, INFINITY)
DEFINE_SOLVER(hung_solve_i64, int64_t, INT64_MAX)
