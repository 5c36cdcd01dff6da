// MLP speed-predictor plugin: every (online, offline) pair through
// in(9) -> 64 -> 64 -> 64 -> 1, layers 2 and 3 on the 5th-gen tensor cores.
//
// The reference has no MLP (its predictor is the table, predictor.py:85-118);
// the paper's is "four layers with hidden size 64x64".  The
// pair-feature build exploits that layer 1 is separable:
//   W1 [on; off; s] + b1 = P[u] + Q[v],  P = W1_on on_u + W1_s s_u + b1,  Q = W1_off off_v
// so per pair only relu(P[u] + Q[v]) is formed (CUDA cores, written straight
// into the UMMA shared-memory layout).  Per tile of 128 pairs (one online row
// u x 128 offline columns):
//   h1 (smem) --tcgen05.mma x9 (M128 N64 K16, W2 in smem)--> TMEM cols 0-63
//   epilogue 1: tcgen05.ld -> ReLU -> split -> tcgen05.st to TMEM cols 64-127
//   h2 (TMEM, the A operand) --tcgen05.mma x8 (W3 in smem)--> TMEM cols 0-63
//   epilogue 2: tcgen05.ld -> + b3 -> ReLU -> dot w4 + b4 -> clamp [0,1] -> store
// Software pipeline per CTA: tile t+1's h1 is built in shared memory (its
// inputs prefetched into registers one tile ahead) while tile t's layer-3
// MMAs run; tile t+1's layer 2 is issued once tile t's accumulator is read.
//
// Precision (the 1e-3 relative bar): operands are fp16 (kind::f16, fp32
// accumulation in TMEM).  The model's layer-2/3 weights and biases are fp16
// values (MlpPredictor stores them rounded), so B is exact; each activation
// is split as a = hi + lo with hi = fp16(a), lo = fp16(a - hi).  Layer 2 runs
// over K = [hi | lo | ones] against [W2; W2; b2] (9 K16 MMAs), layer 3 over
// K = [hi | lo] against [W3; W3] (8 MMAs, b3 added in fp32 in the epilogue):
// ~2^-22 relative per product instead of fp16's 2^-12 (measured ~1e-7
// absolute against the float64 oracle).
// One elected thread issues the MMAs and commits them to an mbarrier; three
// CTAs share an SM (128 TMEM columns each).
// Shared-memory operands use the K-major, no-swizzle canonical layout: 8-row x
// 16-byte core matrices, LBO = 128 B between K-adjacent cores, SBO = (K / 8)
// x 128 B between 8-row groups.  Layer 3's A operand in TMEM: row = lane,
// two consecutive k per 32-bit column (even k in the low half).
#include <cuda_fp16.h>

#include <cstring>
#include <string>

#include "common.cuh"



namespace mux {

constexpr int kH = 64;              // hidden width
constexpr int kKp = 144;            // GEMM K: 64 hi + 64 lo activation halves + a ones column (bias) padded to 16
constexpr int kKg = kKp / 8;        // 16-byte k-groups per operand row
constexpr int kSbo = kKg * 128;     // bytes between 8-row core groups (B operands)
constexpr int kSboA = kSbo + 16;    // A operand: +16 B per group rotates banks (conflict-free epilogue stores)
constexpr int kTile = 128;          // pairs per MMA tile (UMMA M)
constexpr int kMlpThreads = 128;    // 4 warps = the 4 TMEM lane quadrants
template <bool PF> struct MlpCfg { static constexpr int ctas = 3; };
constexpr uint32_t kTmemCols = 128; // columns 0-63: the accumulator of layers 2 and 3; 64-127: layer 3's A operand
constexpr int kK3 = 128;            // layer 3's GEMM K: hi | lo halves only (its bias is added in the epilogue)
constexpr int kSbo3 = (kK3 / 8) * 128;
constexpr int kSmemA = (((kTile / 8) * kSboA) + 1023) / 1024 * 1024;
constexpr int kSmemW = kH * kKp * 2;
constexpr int kSmemW3 = kH * kK3 * 2;
constexpr int kSmemDyn = kSmemA + kSmemW + kSmemW3;

struct MlpDev {
    const float* P;          // [n][64] per-row layer-1 partial (incl. b1)
    const float* Q;          // [m][64] per-column layer-1 partial
    const uint16_t* W2c;     // [64 x 144] fp16 bits, UMMA core layout: W2 | W2 | b2
    const uint16_t* W3c;     // [64 x 128] fp16 bits, UMMA core layout: W3 | W3 (b3 joins in the epilogue)
    const float* b3;
    const float* w4;
    float b4;
    int32_t n, m;
};

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// UMMA shared-memory descriptor, K-major, SWIZZLE_NONE (sm_100 version 1).
__device__ __forceinline__ uint64_t umma_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFFu);
    d |= (uint64_t)((lbo >> 4) & 0x3FFFu) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFFu) << 32;
    d |= (uint64_t)1 << 46;
    return d;
}

// kind::f16 instruction descriptor: fp16 x fp16 -> f32, K-major A and B.
__host__ __device__ constexpr uint32_t idesc_f16(int M, int N) {
    return (1u << 4) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
        :: "r"(tmem_d), "l"(da), "l"(db), "r"(idesc), "r"(acc) : "memory");
}
// A from TMEM (M rows on the lanes, K along the columns, two fp16 per column)
__device__ __forceinline__ void mma_f16_ta(uint32_t tmem_d, uint32_t tmem_a, uint64_t db, uint32_t idesc, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
        :: "r"(tmem_d), "r"(tmem_a), "l"(db), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void mma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];"
                 :: "r"(su32(bar)) : "memory");
}
__device__ __forceinline__ void tc_fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void tc_fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_async_smem() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void bar_init(uint64_t* bar) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" :: "r"(su32(bar)) : "memory");
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void bar_wait(uint64_t* bar, uint32_t parity) {
    asm volatile(
        "{\n.reg .pred p;\nW_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
        "@!p bra W_%=;\n}\n" :: "r"(su32(bar)), "r"(parity) : "memory");
}

// 16 consecutive fp32 columns of this warp's 32 TMEM lanes.
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int t = 0; t < 16; ++t) v[t] = __uint_as_float(r[t]);
}
__device__ __forceinline__ void tmem_wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory"); }

// 16 consecutive 32-bit columns of this warp's 32 TMEM lanes
__device__ __forceinline__ void tmem_st16(uint32_t taddr, const uint32_t (&r)[16]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x16.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16};"
        :: "r"(taddr), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(r[4]), "r"(r[5]), "r"(r[6]), "r"(r[7]),
           "r"(r[8]), "r"(r[9]), "r"(r[10]), "r"(r[11]), "r"(r[12]), "r"(r[13]), "r"(r[14]), "r"(r[15])
        : "memory");
}


// byte offset of core chunk (row r, k-group kg) in the A tile (K-major, kKp columns)
__device__ __forceinline__ uint32_t core_off(int r, int kg) {
    return (uint32_t)((r >> 3) * kSboA + kg * 128 + (r & 7) * 16);
}

// relu(a), relu(b) split into fp16 hi / lo halves: a = hi + lo to ~2^-22
__device__ __forceinline__ void relu_split_f16x2(float a, float b, uint32_t& hi, uint32_t& lo) {
    a = fmaxf(a, 0.f);
    b = fmaxf(b, 0.f);
    const __half2 h = __floats2half2_rn(a, b);
    const float2 hf = __half22float2(h);
    const __half2 l = __floats2half2_rn(a - hf.x, b - hf.y);
    hi = *reinterpret_cast<const uint32_t*>(&h);
    lo = *reinterpret_cast<const uint32_t*>(&l);
}

// PF = true: the next tile's P/Q rows are prefetched into registers under the
// current tile's MMAs (4 CTAs/SM); PF = false: each tile batch-loads its own
// inputs up front, trading the prefetch registers for a fifth CTA per SM.
template <int WT, bool PF>
__global__ void __launch_bounds__(kMlpThreads, MlpCfg<PF>::ctas)
mlp_pairs_kernel(MlpDev p, void* __restrict__ out, int64_t ldo, double qscale) {
    // dynamic shared memory: A tile (36 KB) + W2 / W3 operands (18 KB each)
    extern __shared__ __align__(1024) unsigned char dsm[];
    unsigned char* sA = dsm;
    unsigned char* sW2 = dsm + kSmemA;
    unsigned char* sW3 = sW2 + kSmemW;   // kSmemW3 bytes
    __shared__ __align__(16) float sw4[kH];
    __shared__ __align__(16) float sb3[kH];
    __shared__ uint64_t mbar;
    __shared__ uint32_t tmem_base;
    const int tid = threadIdx.x, warp = tid >> 5;

    for (int e = tid; e < kH * kKp / 8; e += kMlpThreads)
        reinterpret_cast<uint4*>(sW2)[e] = reinterpret_cast<const uint4*>(p.W2c)[e];
    for (int e = tid; e < kH * kK3 / 8; e += kMlpThreads)
        reinterpret_cast<uint4*>(sW3)[e] = reinterpret_cast<const uint4*>(p.W3c)[e];
    if (tid < kH) { sw4[tid] = p.w4[tid]; sb3[tid] = p.b3[tid]; }
    // constant bias k-groups of the A operand: column 128 = 1.0 (fp16), 129..143 = 0
    *reinterpret_cast<uint4*>(sA + core_off(tid, 16)) = make_uint4(0x3C00u, 0u, 0u, 0u);
    *reinterpret_cast<uint4*>(sA + core_off(tid, 17)) = make_uint4(0u, 0u, 0u, 0u);
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;"
                     :: "r"(su32(&tmem_base)), "r"(kTmemCols) : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 0) bar_init(&mbar);
    fence_async_smem();
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = tmem_base;
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    const uint32_t idesc = idesc_f16(kTile, kH);
    const uint32_t a_addr = su32(sA), w2_addr = su32(sW2), w3_addr = su32(sW3);
    uint32_t phase = 0;

    const int64_t tpr = (p.m + kTile - 1) / kTile;
    const int64_t ntiles = (int64_t)p.n * tpr;
    // Register prefetch of a tile's inputs: thread t owns chunks c = t + 128 j
    // (j < 8) of the 128 x 8 (row, k-group) chunk grid, all in k-group
    // (t >> 3) & 7, plus that k-group's 8 values of the tile's P row.
    float4 qa[8], qb[8];
    float4 pp0 = make_float4(0.f, 0.f, 0.f, 0.f), pp1 = pp0;
    const int kg_t = (tid >> 3) & 7;
    auto prefetch = [&](int64_t tile) {
        if (tile >= ntiles) return;
        const int32_t u = (int32_t)(tile / tpr);
        const int32_t v0 = (int32_t)(tile % tpr) * kTile;
        pp0 = __ldg(reinterpret_cast<const float4*>(p.P + (int64_t)u * kH + kg_t * 8));
        pp1 = __ldg(reinterpret_cast<const float4*>(p.P + (int64_t)u * kH + kg_t * 8) + 1);
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int c = tid + kMlpThreads * j;
            const int r = (c & 7) | ((c >> 6) << 3);
            const int v = v0 + r;
            if (v < p.m) {
                const float4* q = reinterpret_cast<const float4*>(p.Q + (int64_t)v * kH + kg_t * 8);
                qa[j] = __ldg(q);
                qb[j] = __ldg(q + 1);
            } else {
                qa[j] = make_float4(-1e30f, -1e30f, -1e30f, -1e30f);   // relu -> 0
                qb[j] = qa[j];
            }
        }
    };
    // h1 = relu(P[u] + Q[v]) -> fp16 hi (k-groups 0-7) / lo (8-15) halves in the UMMA layout
    auto build_h1 = [&]() {
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int c = tid + kMlpThreads * j;
            const int r = (c & 7) | ((c >> 6) << 3);
            const float4 q0 = qa[j], q1 = qb[j];
            uint4 hi, lo;
            relu_split_f16x2(pp0.x + q0.x, pp0.y + q0.y, hi.x, lo.x);
            relu_split_f16x2(pp0.z + q0.z, pp0.w + q0.w, hi.y, lo.y);
            relu_split_f16x2(pp1.x + q1.x, pp1.y + q1.y, hi.z, lo.z);
            relu_split_f16x2(pp1.z + q1.z, pp1.w + q1.w, hi.w, lo.w);
            *reinterpret_cast<uint4*>(sA + core_off(r, kg_t)) = hi;
            *reinterpret_cast<uint4*>(sA + core_off(r, kg_t + 8)) = lo;
        }
        fence_async_smem();
    };
    auto issue_layer2 = [&]() {
        if (tid == 0) {
            tc_fence_after();
#pragma unroll
            for (int ks = 0; ks < kKp / 16; ++ks)
                mma_f16(tmem, umma_desc(a_addr + ks * 256, 128, kSboA), umma_desc(w2_addr + ks * 256, 128, kSbo),
                        idesc, ks > 0);
            mma_commit(&mbar);
        }
    };
    // Software pipeline per CTA: tile t+1's h1 is built in shared memory while
    // tile t's layer-3 MMAs run (their A operand lives in TMEM), and its
    // layer-2 MMAs are issued as soon as tile t's accumulator is drained.
    int64_t tile = blockIdx.x;
    if (tile < ntiles) {
        prefetch(tile);
        build_h1();
        __syncthreads();
        issue_layer2();
        if (PF) prefetch(tile + gridDim.x);
    }
    for (; tile < ntiles; tile += gridDim.x) {
        const int32_t u = (int32_t)(tile / tpr);
        const int32_t v0 = (int32_t)(tile % tpr) * kTile;
        const int64_t next = tile + gridDim.x;
        bar_wait(&mbar, phase);
        phase ^= 1;
        tc_fence_after();
        // ---- epilogue 1: ReLU -> fp16 hi / lo -> layer 3's A operand in TMEM (own lane)
        const int row = tid;
#pragma unroll
        for (int half = 0; half < 2; ++half) {   // two TMEM loads in flight per wait
            float acc[2][16];
#pragma unroll
            for (int h = 0; h < 2; ++h) tmem_ld16(tmem + lane_base + (half * 2 + h) * 16, acc[h]);
            tmem_wait_ld();
            uint32_t w[16], wl[16];
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int t = 0; t < 8; ++t) relu_split_f16x2(acc[h][2 * t], acc[h][2 * t + 1], w[h * 8 + t], wl[h * 8 + t]);
            tmem_st16(tmem + lane_base + 64 + half * 16, w);        // k = 32 half .. : hi
            tmem_st16(tmem + lane_base + 96 + half * 16, wl);       // k = 64 + 32 half .. : lo
        }
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
        tc_fence_before();
        __syncthreads();
        // ---- layer 3 on the tensor cores, A from TMEM (columns 64-127: hi | lo)
        if (tid == 0) {
            tc_fence_after();
#pragma unroll
            for (int ks = 0; ks < kK3 / 16; ++ks)
                mma_f16_ta(tmem, tmem + 64 + ks * 8, umma_desc(w3_addr + ks * 256, 128, kSbo3), idesc, ks > 0);
            mma_commit(&mbar);
        }
        // ---- the next tile's h1 under the layer-3 MMAs (layer 2 of this tile is done with sA)
        if (next < ntiles) {
            if (!PF) prefetch(next);
            build_h1();
        }
        bar_wait(&mbar, phase);
        phase ^= 1;
        tc_fence_after();
        // ---- epilogue 2: ReLU(acc + b3), dot w4 + b4, clamp, store
        float o = p.b4;
#pragma unroll
        for (int half = 0; half < 2; ++half) {
            float acc[2][16];
#pragma unroll
            for (int h = 0; h < 2; ++h) tmem_ld16(tmem + lane_base + (half * 2 + h) * 16, acc[h]);
            tmem_wait_ld();
#pragma unroll
            for (int h = 0; h < 2; ++h)
#pragma unroll
                for (int t4 = 0; t4 < 4; ++t4) {
                    const float4 w4 = reinterpret_cast<const float4*>(sw4 + (half * 2 + h) * 16)[t4];
                    const float4 b3 = reinterpret_cast<const float4*>(sb3 + (half * 2 + h) * 16)[t4];
                    o = fmaf(fmaxf(acc[h][4 * t4 + 0] + b3.x, 0.f), w4.x, o);
                    o = fmaf(fmaxf(acc[h][4 * t4 + 1] + b3.y, 0.f), w4.y, o);
                    o = fmaf(fmaxf(acc[h][4 * t4 + 2] + b3.z, 0.f), w4.z, o);
                    o = fmaf(fmaxf(acc[h][4 * t4 + 3] + b3.w, 0.f), w4.w, o);
                }
        }
        o = fminf(1.f, fmaxf(0.f, o));
        const int v = v0 + row;
        if (v < p.m) {
            if (WT == MUX_W_F32) static_cast<float*>(out)[(int64_t)u * ldo + v] = o;
            else {
                const double w = o < 1e-6f ? 0.0 : (double)o;
                static_cast<int32_t*>(out)[(int64_t)u * ldo + v] = (int32_t)__double2ll_rn(w * qscale);
            }
        }
        tc_fence_before();
        __syncthreads();   // accumulator drained, next h1 complete
        if (next < ntiles) {
            issue_layer2();
            if (PF) prefetch(next + gridDim.x);
        }
    }
    __syncthreads();
    if (warp == 0) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" :: "r"(tmem), "r"(kTmemCols) : "memory");
    }
}

// layer-1 partials: P[u] = W1_on x_on + W1_s s + b1, Q[v] = W1_off x_off (fp32)
struct MlpL1 {
    float W1[kH * 9];
    float b1[kH];
    float shift[9];
    float scale[9];
};

__global__ void mlp_layer1_kernel(MlpL1 w, const double* __restrict__ on, const double* __restrict__ share,
                                  int32_t n, const double* __restrict__ off, int32_t m,
                                  float* __restrict__ P, float* __restrict__ Q) {
    const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
    const int64_t total = (int64_t)(n + m) * kH;
    if (t >= total) return;
    const int64_t row = t / kH;
    const int k = (int)(t % kH);
    if (row < n) {
        float acc = w.b1[k];
#pragma unroll
        for (int f = 0; f < 4; ++f) acc += w.W1[k * 9 + f] * (float)((on[row * 4 + f] - w.shift[f]) * w.scale[f]);
        acc += w.W1[k * 9 + 8] * (float)((share[row] - w.shift[8]) * w.scale[8]);
        P[row * kH + k] = acc;
    } else {
        const int64_t v = row - n;
        float acc = 0.f;
#pragma unroll
        for (int f = 0; f < 4; ++f)
            acc += w.W1[k * 9 + 4 + f] * (float)((off[v * 4 + f] - w.shift[4 + f]) * w.scale[4 + f]);
        Q[v * kH + k] = acc;
    }
}

}  // namespace mux

using namespace mux;

// W [64 out][64 in] row-major + bias -> UMMA K-major core layout of the
// [64 x 144] fp16 B operand: columns 0-63 and 64-127 = W (against the hi and
// lo activation halves), 128 = bias, 129-143 = 0; N = out.  The model's
// weights are fp16 values (MlpPredictor), so the conversion is exact.
static int to_core_layout(const float* W, const float* bias, uint16_t* dst) {
    for (int nn = 0; nn < kH; ++nn)
        for (int k = 0; k < kKp; ++k) {
            const float val = k < 2 * kH ? W[nn * kH + (k & (kH - 1))] : (k == 2 * kH ? bias[nn] : 0.f);
            const __half h = __float2half_rn(val);
            if (__half2float(h) != val) return MUX_EINVAL;   // not an fp16 value
            const size_t off = (size_t)(nn >> 3) * (kSbo / 2) + (size_t)(k >> 3) * 64 + (size_t)(nn & 7) * 8 + (k & 7);
            memcpy(&dst[off], &h, 2);
        }
    return MUX_OK;
}

// W [64 out][64 in] -> the [64 x 128] fp16 B operand [W | W] of layer 3 (its
// A operand carries no ones column; the bias is added in the epilogue)
static int to_core_layout3(const float* W, uint16_t* dst) {
    for (int nn = 0; nn < kH; ++nn)
        for (int k = 0; k < kK3; ++k) {
            const float val = W[nn * kH + (k & (kH - 1))];
            const __half h = __float2half_rn(val);
            if (__half2float(h) != val) return MUX_EINVAL;
            const size_t off = (size_t)(nn >> 3) * (kSbo3 / 2) + (size_t)(k >> 3) * 64 + (size_t)(nn & 7) * 8 + (k & 7);
            memcpy(&dst[off], &h, 2);
        }
    return MUX_OK;
}

int mux_score_mlp_impl(mux_ctx_t* ctx, const mux_mlp_t* w, const double* on, const double* share, int64_t n,
                       const double* off, int64_t m, int wtype, int qbits, void* out, int64_t ldo,
                       cudaStream_t st, int64_t* launches) {
    if (w->hidden != kH) { set_error("mux_score_mlp: hidden width must be 64"); return MUX_EINVAL; }
    // parameter block on device: W2c, W3c (fp16 core layout with the biases), w4
    const size_t o_w2 = 0, o_w3 = o_w2 + kH * kKp * 2, o_w4 = o_w3 + kH * kK3 * 2, o_b3 = o_w4 + kH * 4, o_end = o_b3 + kH * 4;
    std::string blob(o_end, '\0');
    if (to_core_layout(w->W2, w->b2, reinterpret_cast<uint16_t*>(&blob[o_w2])) != MUX_OK ||
        to_core_layout3(w->W3, reinterpret_cast<uint16_t*>(&blob[o_w3])) != MUX_OK) {
        set_error("mux_score_mlp: W2, b2, W3, b3 must be fp16 values");
        return MUX_EINVAL;
    }
    memcpy(&blob[o_w4], w->w4, kH * 4);
    for (int k = 0; k < kH; ++k) {   // b3 is an fp16 value too (the model's stored precision)
        const __half h = __float2half_rn(w->b3[k]);
        if (__half2float(h) != w->b3[k]) { set_error("mux_score_mlp: W2, b2, W3, b3 must be fp16 values"); return MUX_EINVAL; }
    }
    memcpy(&blob[o_b3], w->b3, kH * 4);
    const size_t pq_bytes = sizeof(float) * kH * (size_t)(n + m);
    MUX_TRY(ctx->mlp.ensure(o_end + 256 + pq_bytes));
    char* base = ctx->mlp.as<char>();
    MUX_CUDA_TRY(cudaMemcpyAsync(base, blob.data(), o_end, cudaMemcpyHostToDevice, st));
    float* P = reinterpret_cast<float*>(base + ((o_end + 255) / 256) * 256);
    float* Q = P + (size_t)kH * n;
    MlpL1 l1;
    memcpy(l1.W1, w->W1, sizeof(l1.W1));
    memcpy(l1.b1, w->b1, sizeof(l1.b1));
    memcpy(l1.shift, w->shift, sizeof(l1.shift));
    memcpy(l1.scale, w->scale, sizeof(l1.scale));
    const int64_t total = (n + m) * kH;
    if (total > 0) {
        mlp_layer1_kernel<<<(unsigned)((total + 255) / 256), 256, 0, st>>>(l1, on, share, (int32_t)n, off, (int32_t)m, P, Q);
        ++*launches;
    }
    MlpDev p;
    p.P = P; p.Q = Q;
    p.W2c = reinterpret_cast<const uint16_t*>(base + o_w2);
    p.W3c = reinterpret_cast<const uint16_t*>(base + o_w3);
    p.b3 = reinterpret_cast<const float*>(base + o_b3);
    p.w4 = reinterpret_cast<const float*>(base + o_w4);
    p.b4 = w->b4;
    p.n = (int32_t)n; p.m = (int32_t)m;
    const int64_t tiles = n * ((m + kTile - 1) / kTile);
    if (tiles > 0) {
        const bool pf = tuning().mlp_prefetch;
        MUX_CUDA_TRY(cudaFuncSetAttribute(mlp_pairs_kernel<MUX_W_F32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemDyn));
        MUX_CUDA_TRY(cudaFuncSetAttribute(mlp_pairs_kernel<MUX_W_I32, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemDyn));
        MUX_CUDA_TRY(cudaFuncSetAttribute(mlp_pairs_kernel<MUX_W_F32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemDyn));
        MUX_CUDA_TRY(cudaFuncSetAttribute(mlp_pairs_kernel<MUX_W_I32, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemDyn));
        const unsigned grid = (unsigned)std::min<int64_t>(tiles, (int64_t)ctx->num_sms * (pf ? MlpCfg<true>::ctas : MlpCfg<false>::ctas));
        const double qscale = ldexp(1.0, qbits);
        if (pf) {
            if (wtype == MUX_W_F32) mlp_pairs_kernel<MUX_W_F32, true><<<grid, kMlpThreads, kSmemDyn, st>>>(p, out, ldo, qscale);
            else mlp_pairs_kernel<MUX_W_I32, true><<<grid, kMlpThreads, kSmemDyn, st>>>(p, out, ldo, qscale);
        } else {
            if (wtype == MUX_W_F32) mlp_pairs_kernel<MUX_W_F32, false><<<grid, kMlpThreads, kSmemDyn, st>>>(p, out, ldo, qscale);
            else mlp_pairs_kernel<MUX_W_I32, false><<<grid, kMlpThreads, kSmemDyn, st>>>(p, out, ldo, qscale);
        }
        ++*launches;
    }
    MUX_CUDA_TRY(cudaGetLastError());
    return MUX_OK;
}
