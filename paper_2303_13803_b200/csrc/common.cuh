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

// Every environment knob the library reads, parsed and range-checked in one
// place (tuning() in csrc/api.cu, re-read on each call).  Diagnostics are
// always honoured; everything that changes which kernels run or how is an
// experiment knob, honoured only under MUX_TUNING=1, so a stray variable in a
// production environment cannot change the solver.  An out-of-range value is
// an error (mux_last_error names it), not silently clamped.
struct Tuning {
    // diagnostics (always)
    bool verbose = false;        // MUX_VERBOSE: per-level solver log on stderr
    bool ssp_check = false;      // MUX_SSP_CHECK=1: dense dual certificate after every level
    bool ssp_time = false;       // MUX_SSP_TIME=1: per-pop cycle split of the long-path kernel
    // experiments (MUX_TUNING=1 only)
    bool force_auction = false;  // MUX_SOLVER=auction: epsilon-scaling auction for int32 too
    bool canon = true;           // MUX_CANON=0: skip the tie canonicalisation
    bool ssp_rect = true;        // MUX_SSP_RECT=0: rectangular rounds on the auction
    int ssp_f = 2;               // MUX_SSP_F [2, 16]: coarsening factor between levels
    int ssp_fx = 0;              // MUX_SSP_FX [110, 1600]: fractional coarsening factor x 100 (0 = MUX_SSP_F)
    int ssp_base = 48;           // MUX_SSP_BASE [8, 4096]: size of the coarsest level
    int ssp_steps = 24;          // MUX_SSP_STEPS [1, 100000]: pops before a warp search is deferred
    int ssp_deep = 4;            // MUX_SSP_DEEP [0, 1000]: dense re-scans before deferral
    int ssp_coarse_pops = 0;     // MUX_SSP_COARSE_POPS [0, 1e9]: long-search pop limit at coarse levels
    bool ssp_serial = false;     // MUX_SSP_SERIAL=1: one warp search at a time
    bool ssp_pf = false;         // MUX_SSP_PF=1: TMA prefetch of the runner-up's row slice in the long-path kernel
    int ssp_l2pf = 0;            // MUX_SSP_L2PF [0, 1]: L2 prefetch of every warp-minimum candidate's row slice
    bool ssp_ties = true;        // MUX_SSP_TIES=0: one pop per exchange step (no tie batching)
    bool ssp_cluster = true;     // MUX_SSP_CLUSTER=0: single-CTA / single-warp long paths
    bool ssp_sparsex = false;    // MUX_SSP_SPARSEX=1: single-warp sparse long paths
    int ssp_rslice = 1;          // MUX_SSP_RSLICE [0, 2]: 0 = large levels on the shared-memory sliced kernel, 2 = every cluster level on it
    int ssp_ct1 = 512;           // MUX_SSP_CT1 {512, 1024}: threads of the single-SM long-path kernel (512: levels <= 3072)
    int ssp_ct = 256;            // MUX_SSP_CT {128, 256, 512, 1024}: threads per CTA of the long-path kernel
    int ssp_taildef = 4;         // MUX_SSP_TAILDEF [0, 4096]: retried row lists up to this size go to the long-path kernel
    bool ssp_wide = true;        // MUX_SSP_WIDE=0: no 16-CTA clusters for the slice kernel (m > 16,384)
    bool ssp_cperm = true;       // MUX_SSP_CPERM=0: coarse levels store their columns in key order, not a stride order
    bool ssp_lwalk = true;       // MUX_SSP_LWALK=0: the slice kernel's path walk reads DSMEM / global per hop
    int ssp_rpf = 16;            // MUX_SSP_RPF [0, 64]: rank-neighbour L2 prefetch distance of the long-path kernel (0 = off)
    int ssp_rpf_mb = 64;         // MUX_SSP_RPF_MB [0, 65536]: levels whose matrix exceeds this many MiB use it
    int ssp_seq = 64;            // MUX_SSP_SEQ [0, 4096]: levels up to this size skip the parallel passes
    int ssp_dorder = 1;          // MUX_SSP_DORDER [0, 2]: long searches in defer order / ascending / descending row key
    const char* ssp_dump = nullptr;     // MUX_SSP_DUMP=dir: write each long-search batch's level state (analysis)
    const char* canon_dump = nullptr;   // MUX_CANON_DUMP=file: the canonicalisation host loop's inputs and output
    int ssp_one = 1300;          // MUX_SSP_ONE [0, 10240]: levels up to this size run long paths on one SM
    int auc_theta = 4;           // MUX_THETA [2, 64]: epsilon-scaling factor
    int auc_tail = -1;           // MUX_TAIL [-1, 2^20]: unassigned count that ends the Jacobi rounds (clamped to 16)
    int auc_k = 15;              // MUX_K [1, 15]: cached candidates per bidder
    bool auc_cg_sync = true;     // MUX_CG_SYNC=0: custom grid barrier
    int auc_async_tail = -1;     // MUX_ASYNC_TAIL [-1, 1]: concurrent tail chains (-1 = n >= 512)
    int auc_async_phases = 1 << 20;   // MUX_ASYNC_PHASES [0, 2^20]
    int auc_fresh = 1, auc_restage = 0, auc_order = 1;   // MUX_FRESH / MUX_RESTAGE / MUX_ORDER [0, 2]
    bool auc_no_smem = false;    // MUX_NO_SMEM=1: global-memory auction path
    bool mlp_prefetch = true;    // MUX_MLP_PREFETCH=0: each tile loads its inputs when it builds h1 (no register prefetch)
    bool error = false;          // an out-of-range value was given
};
// Current knob values; *err set to a message when a value is out of range.
const Tuning& tuning();

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
    mux::DevBuf canon_ent;  // tight-edge CSR entries when they outgrow the default buffer
    mux::DevBuf ipc_out;    // buffer exported to peer processes (mux_ipc_export)
    void* ipc_in = nullptr; // peer buffer mapped by mux_ipc_import
    // MLP plugin parameters + layer-1 partials
    mux::DevBuf mlp;
    size_t auc_n = 0;
    // pinned host staging
    void* pinned = nullptr;
    size_t pinned_bytes = 0;
};
