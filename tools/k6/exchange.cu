// K6 prototype measurement: the cost of exchanging one
// per-pop minimum between GPUs, the step a Dijkstra whose columns are split
// across GPUs would add to every pop.  Two (or more) GPUs run one
// persistent warp each; every step each GPU stores its key into every
// peer's mailbox over NVLink (st.release.sys through peer-mapped memory)
// and spins (ld.acquire.sys) until all peers' keys for that step arrived,
// then takes the minimum -- the exact dependency chain of a pop.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o exchange exchange.cu
//   ./exchange [gpus=2] [steps=200000]
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <chrono>
#include <thread>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t ck_ = (x); if (ck_ != cudaSuccess) { fprintf(stderr, "%s: %s\n", #x, cudaGetErrorString(ck_)); exit(1); } } while (0)

constexpr int kMaxG = 8;

// box[g] on GPU g: [2][kMaxG] slots (step parity x sender).  Double buffering
// by step parity: a sender can only reuse a parity slot (step s + 2) after it
// received every peer's step s + 1, which each peer sends only after reading
// the sender's step s -- no value is overwritten before it is read.
struct Boxes { unsigned long long* box[kMaxG]; };

__global__ void pingpong(Boxes B, int me, int G, int steps, unsigned long long* out) {
    if (threadIdx.x != 0) return;
    unsigned long long key = 0x1234567ull * (me + 1), acc = 0;
    for (int s = 1; s <= steps; ++s) {
        const unsigned long long v = ((unsigned long long)s << 40) | (key & 0xFFFFFFFFFFull);
        for (int g = 0; g < G; ++g) {
            if (g == me) continue;
            unsigned long long* dst = B.box[g] + (s & 1) * kMaxG + me;
            asm volatile("st.release.sys.global.u64 [%0], %1;" ::"l"(dst), "l"(v) : "memory");
        }
        unsigned long long mn = v;
        for (int g = 0; g < G; ++g) {
            if (g == me) continue;
            unsigned long long w;
            do {
                asm volatile("ld.acquire.sys.global.u64 %0, [%1];" : "=l"(w) : "l"(B.box[me] + (s & 1) * kMaxG + g) : "memory");
            } while ((w >> 40) != (unsigned long long)s);
            mn = w < mn ? w : mn;
        }
        key = (mn * 6364136223846793005ull + 1442695040888963407ull) >> 8;   // next pop depends on the minimum
        acc ^= mn;
    }
    *out = acc;
}

int main(int argc, char** argv) {
    const int G = argc > 1 ? atoi(argv[1]) : 2;
    const int steps = argc > 2 ? atoi(argv[2]) : 200000;
    int nd = 0;
    CK(cudaGetDeviceCount(&nd));
    if (nd < G) { printf("{\"error\": \"need %d GPUs, have %d\"}\n", G, nd); return 0; }
    Boxes B;
    std::vector<unsigned long long*> outs(G);
    for (int g = 0; g < G; ++g) {
        CK(cudaSetDevice(g));
        for (int h = 0; h < G; ++h) {
            if (h == g) continue;
            int can = 0;
            CK(cudaDeviceCanAccessPeer(&can, g, h));
            if (!can) { printf("{\"error\": \"no peer access %d->%d\"}\n", g, h); return 0; }
            cudaError_t e = cudaDeviceEnablePeerAccess(h, 0);
            if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) CK(e);
            cudaGetLastError();
        }
        CK(cudaMalloc(&B.box[g], sizeof(unsigned long long) * 2 * kMaxG));
        CK(cudaMemset(B.box[g], 0, sizeof(unsigned long long) * 2 * kMaxG));
        CK(cudaMalloc(&outs[g], 8));
    }
    for (int g = 0; g < G; ++g) { CK(cudaSetDevice(g)); CK(cudaDeviceSynchronize()); }
    // warm-up run, then the timed one (all GPUs launched back to back)
    double best = 1e30;
    for (int rep = 0; rep < 3; ++rep) {
        for (int g = 0; g < G; ++g) { CK(cudaSetDevice(g)); CK(cudaMemset(B.box[g], 0, sizeof(unsigned long long) * 2 * kMaxG)); CK(cudaDeviceSynchronize()); }
        const int n = rep == 0 ? 1000 : steps;
        auto t0 = std::chrono::steady_clock::now();
        for (int g = 0; g < G; ++g) { CK(cudaSetDevice(g)); pingpong<<<1, 32>>>(B, g, G, n, outs[g]); }
        for (int g = 0; g < G; ++g) { CK(cudaSetDevice(g)); CK(cudaDeviceSynchronize()); }
        const double us = std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count();
        if (rep > 0) best = std::min(best, us / n);
    }
    printf("{\"gpus\": %d, \"steps\": %d, \"us_per_exchange\": %.3f, \"note\": \"one dependent all-to-all minimum over NVLink per step (peer st.release.sys + ld.acquire.sys spin)\"}\n",
           G, steps, best);
    return 0;
}
