// Times the canonicalisation host loop (csrc/canon_host.h) on a graph dumped
// by MUX_TUNING=1 MUX_CANON_DUMP=file and checks its output against the dump.
//   g++ -O3 -std=c++17 -I paper_2303_13803_b200/csrc tools/canon_host_bench.cpp -o /tmp/canon_bench
//   /tmp/canon_bench file [repeats]
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "canon_host.h"

using namespace mux::canon_host;

int main(int argc, char** argv) {
    if (argc < 2) { fprintf(stderr, "usage: %s dump [repeats]\n", argv[0]); return 2; }
    FILE* f = fopen(argv[1], "rb");
    if (!f) { perror(argv[1]); return 2; }
    int32_t h[7];
    if (fread(h, 4, 7, f) != 7) return 2;
    const int32_t N = h[0], M = h[1], n = h[2];
    std::vector<int32_t> col_in(n), rcnt(N), ent(h[3]), out(n);
    std::vector<int64_t> roff(N);
    TightGraph G;
    G.N = N; G.M = M; G.n = n;
    G.Z.resize(h[4]); G.Zpad.resize(h[5]); G.padrow_tight.resize(h[6]);
    bool ok = fread(col_in.data(), 4, n, f) == (size_t)n && fread(rcnt.data(), 4, N, f) == (size_t)N &&
              fread(roff.data(), 8, N, f) == (size_t)N && fread(ent.data(), 4, h[3], f) == (size_t)h[3] &&
              fread(G.Z.data(), 4, h[4], f) == (size_t)h[4] && fread(G.Zpad.data(), 4, h[5], f) == (size_t)h[5] &&
              fread(G.padrow_tight.data(), 1, h[6], f) == (size_t)h[6] && fread(out.data(), 4, n, f) == (size_t)n;
    fclose(f);
    if (!ok) { fprintf(stderr, "short dump\n"); return 2; }
    G.ent = &ent; G.cnt = &rcnt; G.off = &roff;
    const int reps = argc > 2 ? atoi(argv[2]) : 5;
    double best = 1e30;
    long long searches = 0, visits = 0, fails = 0, pruned = 0;
    bool same = true;
    for (int r = 0; r < reps; ++r) {
        std::vector<int32_t> col = col_in;
        const auto t0 = std::chrono::steady_clock::now();
        Canon K(G, col);
        K.run();
        const double ms = std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count();
        best = ms < best ? ms : best;
        searches = K.searches; visits = K.visits; fails = K.fails; pruned = K.pruned;
        same = same && col == out;
    }
    printf("N %d M %d n %d tight %d: %.3f ms (best of %d), %lld searches (%lld failed, %lld at once), %lld column visits, output %s\n",
           N, M, n, h[3], best, reps, searches, fails, pruned, visits, same ? "identical" : "DIFFERENT");
    return same ? 0 : 1;
}
