// Host half of the tie canonicalisation (csrc/canon.cu): the reference's
// row-by-row repair loop (matching.py:173-199, _repair_path matching.py:104-145)
// over the sparse tight graph.  Plain C++ so tools/canon_host_bench.cpp can
// time it on dumped graphs (MUX_CANON_DUMP) without a GPU.
#pragma once
#include <cstdint>
#include <utility>
#include <vector>

namespace mux {
namespace canon_host {


struct TightGraph {
    int32_t N, M, n;
    const std::vector<int32_t>* ent;
    const std::vector<int32_t>* cnt;
    const std::vector<int64_t>* off;
    std::vector<int32_t> Z;       // columns tight to every padding row (N < M)
    std::vector<int32_t> Zpad;    // padding columns tight to rows with padrow_tight (N > M)
    std::vector<char> padrow_tight;
};

struct Canon {
    static constexpr uint32_t kLocked = 0xFFFFFFFFu;
    const TightGraph& G;
    std::vector<int32_t>& col;
    std::vector<int32_t> row_of_col;
    std::vector<uint32_t> stamp;      // column: epoch of the search that visited it, kLocked once locked
    std::vector<uint32_t> dead;       // row: dead-row epoch (see run())
    std::vector<int32_t> parent;
    std::vector<int32_t> queue;                          // BFS queue of rows (its prefix: the explored rows)
    std::vector<std::pair<int32_t, int32_t>> moves;      // the applied path
    uint32_t epoch = 0, dep = 0;
    long long searches = 0, visits = 0, fails = 0, pruned = 0;

    Canon(const TightGraph& g, std::vector<int32_t>& c)
        : G(g), col(c), row_of_col(g.n), stamp(g.n, 0), dead(g.n, 0), parent(g.n, -1), queue((size_t)g.n + 1) {
        for (int32_t i = 0; i < G.n; ++i) row_of_col[col[i]] = i;
    }
    bool seen(int32_t j) const { return stamp[j] >= epoch; }   // this search, or locked

    // matching.py:104-145: breadth-first search over tight edges for an
    // alternating path start_row -> ... -> target_col; applies it on success.
    bool repair(int32_t start_row, int32_t target_col, int32_t banned_row, int32_t banned_col) {
        ++searches;
        if (dead[start_row] == dep) { ++fails; ++pruned; return false; }
        ++epoch;
        stamp[banned_col] = epoch;
        // one FIFO queue: the same level-by-level order as a frontier / next-frontier
        // pair, and its prefix is the set of explored rows
        int32_t* q = queue.data();
        int32_t head = 0, tail = 0;
        q[tail++] = start_row;
        bool found = false, z_done = false, zp_done = false;
        const int32_t* ent = G.ent->data();
        const int64_t* off = G.off->data();
        const int32_t* cnt = G.cnt->data();
        auto visit = [&](int32_t r, int32_t j) -> bool {
            if (seen(j)) return false;
            ++visits;
            stamp[j] = epoch;
            parent[j] = r;
            if (j == target_col) return true;
            const int32_t r2 = row_of_col[j];
            if (r2 != banned_row && dead[r2] != dep) q[tail++] = r2;
            return false;
        };
        while (head < tail && !found) {
            const int32_t r = q[head++];
            if (r >= G.N) {                      // padding row: tight to Z
                if (!z_done) {
                    z_done = true;   // every later padding row finds Z visited
                    for (int32_t j : G.Z)
                        if (visit(r, j)) { found = true; break; }
                }
            } else {
                const int32_t* e = ent + off[r];
                const int32_t k = cnt[r];
                for (int32_t t = 0; t < k && !found; ++t)
                    if (visit(r, e[t] & 0x7fffffff)) found = true;
                if (!found && G.padrow_tight.size() && G.padrow_tight[r] && !zp_done) {
                    zp_done = true;
                    for (int32_t j : G.Zpad)
                        if (visit(r, j)) { found = true; break; }
                }
            }
        }
        if (!found) {
            ++fails;
            for (int32_t t = 0; t < tail; ++t) dead[q[t]] = dep;
            return false;
        }
        // reconstruct from the target back to start_row, then apply
        moves.clear();
        int32_t j = target_col;
        for (;;) {
            const int32_t r = parent[j];
            moves.emplace_back(r, j);
            if (r == start_row) break;
            j = col[r];
        }
        for (auto& m : moves) { row_of_col[m.second] = m.first; col[m.first] = m.second; }
        return true;
    }

    // matching.py:173-199.  Within one row's candidate loop every search has
    // the same target (the row's column), banned row and locked set; a row
    // explored by a failed search cannot reach the target (whatever column
    // the later search bans: a path through the earlier banned column leads
    // back into the failed search's tree), so later searches treat it as a
    // dead end and fail at once when they start on one.  Dead ends lie on no
    // path to the target, so the breadth-first path found -- the reference's
    // -- is unchanged.
    void run() {
        for (int32_t i = 0; i < G.N; ++i) {
            ++dep;
            int32_t j_cur = col[i];
            const int32_t* e = G.ent->data() + (*G.off)[i];
            const int32_t k = (*G.cnt)[i];
            bool emitted = false;
            if (j_cur < G.M)
                for (int32_t t = 0; t < k; ++t)
                    if ((e[t] & 0x7fffffff) == j_cur) { emitted = (e[t] >= 0); break; }
            for (int32_t t = 0; t < k; ++t) {
                if (e[t] < 0) continue;                 // zero weight
                const int32_t j = e[t];
                if (stamp[j] == kLocked) continue;
                if (emitted && j >= j_cur) break;
                if (!repair(row_of_col[j], j_cur, i, j)) continue;
                row_of_col[j] = i;
                col[i] = j;
                j_cur = j;
                break;
            }
            stamp[j_cur] = kLocked;
        }
    }
};

}  // namespace canon_host
}  // namespace mux
