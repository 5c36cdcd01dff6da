// Shared helpers for the muxflow CUDA library (sm_100a only).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <string>

#include "../../include/muxflow.h"

#if !defined(__CUDA_ARCH__) || (__CUDA_ARCH__ >= 1000)
#else
#error "muxflow targets sm_100a (B200) only"
#endif

namespace mux {

// thread-local last-error message (mux_last_error)
void set_error(const std::string& msg);

#define MUX_CUDA_TRY(expr)                                                     \
    do {                                                                       \
        cudaError_t _e = (expr);                                               \
        if (_e != cudaSuccess) {                                               \
            ::mux::set_error(std::string(#expr) + ": " + cudaGetErrorString(_e)); \
            return MUX_ECUDA;                                                  \
        }                                                                      \
    } while (0)

#define MUX_TRY(expr)                                                          \
    do {                                                                       \
        int _s = (expr);                                                       \
        if (_s != MUX_OK) return _s;                                           \
    } while (0)

constexpr int kWarp = 32;

// Device-side error flags (bit set by kernels, read back by the host).
enum : uint32_t {
    kErrQueryRange = 1u << 0,   // a coordinate outside [0, 1]
    kErrPriceBits = 1u << 1,    // auction price would overflow its packing
    kErrIterGuard = 1u << 2,    // auction round guard tripped
};

// Grow-only device buffer.
struct DevBuf {
    void* ptr = nullptr;
    size_t bytes = 0;
    int ensure(size_t need) {
        if (need <= bytes) return MUX_OK;
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
        size_t cap = need + need / 4 + 256;
        if (cudaMalloc(&ptr, cap) != cudaSuccess) {
            set_error("cudaMalloc failed for " + std::to_string(cap) + " bytes");
            return MUX_ENOMEM;
        }
        bytes = cap;
        return MUX_OK;
    }
    void release() {
        if (ptr) cudaFree(ptr);
        ptr = nullptr;
        bytes = 0;
    }
    template <class T> T* as() const { return static_cast<T*>(ptr); }
};

}  // namespace mux

// The opaque context (mux_ctx_t in the C ABI).
struct mux_ctx {
    int device = 0;
    int num_sms = 0;
    // scoring
    mux::DevBuf table;      // axes + values on device
    mux::DevBuf rowfeat;    // per-row interpolation features
    mux::DevBuf colfeat;    // per-column interpolation features
    mux::DevBuf flags;      // uint32 error flags + scratch scalars
    // round staging (mux_round)
    mux::DevBuf feat_in;    // x, share, y uploaded from host
    mux::DevBuf wq;         // quantised weights
    mux::DevBuf colout;     // int32 col_of_row on device
    // auction workspace
    mux::DevBuf auc;
    // multilevel shortest-path solver workspace (csrc/ssp.cu)
    mux::DevBuf ssp;
    // tie canonicalisation workspace (duals, tight-edge CSR)
    mux::DevBuf canon;
    // MLP plugin parameters + layer-1 partials
    mux::DevBuf mlp;
    size_t auc_n = 0;
    // pinned host staging
    void* pinned = nullptr;
    size_t pinned_bytes = 0;
};
