// internal.h -- shared host-side internals of libfhash.so (not part of the ABI).
#pragma once
#include <atomic>
#include <mutex>
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdint>
#include <cstdio>

#include "../../include/fhash.h"
#include "encode_params.h"

namespace fh {

// Thread-local last-error text (defined in fhash_api.cu).
extern thread_local char g_err[512];

inline fh_status fail(fh_status s, const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
    return s;
}

inline fh_status cuda_check(cudaError_t e, const char *what) {
    if (e != cudaSuccess) return fail(FH_E_CUDA, "%s: %s", what, cudaGetErrorString(e));
    return FH_OK;
}

inline bool aligned(const void *p, size_t a) { return (reinterpret_cast<uintptr_t>(p) % a) == 0; }
inline size_t dtype_size(fh_dtype d) { return d == FH_F32 ? 4 : 2; }

// Kernel launches issued by the library (fh_kernel_launches): incremented
// at every launch site of the method's kernels.
extern std::atomic<unsigned long long> g_launches;
inline void count_launch() { g_launches.fetch_add(1, std::memory_order_relaxed); }

// fhash_api.cu: backward launches and the gradient ranges they finalise.
int bwd_launch_count(fh_encoder e);
int bwd_launch_ranges(fh_encoder e, int launch, int64_t *ranges, int max);
fh_status encode_bwd_events(fh_encoder e, const float *coords, int64_t N, const float *dout, float *dtable,
                            fh_stream stream, cudaEvent_t *ev, int n_ev, bool overwrite = false,
                            bool level_major = false);

}  // namespace fh

struct fh_encoder_s {
    int kind = 0;  // 0: F-Hash Tesseract encoder; 1: MHE baseline (NEXT-3)
    int L = 0, F = 0;
    fh_dtype table_dtype = FH_F32;
    uint64_t cap = 0;
    fh_level_info info[FH_MAX_LEVELS];
    uint64_t entries = 0;
    fh::Params params;
    int *flag = nullptr;  // sticky domain flag (device), allocated by fh_build_levels (bind_device)
    int device = -1;
    // Level groups: consecutive levels whose table (fwd) or
    // fp32 grad (bwd) footprint fits an L2 budget run as one pass, so the
    // gathered / reduced region stays L2-resident.  g[i]..g[i+1] = group i.
    int n_gf = 0, gf[FH_MAX_LEVELS + 1] = {0};
    int n_gb = 0, gb[2 * FH_MAX_LEVELS + 2] = {0};  // bwd: pairs (begin, end) of non-small runs
    fh::SmallSet small{};                            // bwd: levels privatised in shared memory
    fh::SmallSet small_cta{};                        // ... launch with CTA copies (non-tiny levels)
    fh::SmallSet small_tiny[FH_MAX_LEVELS];          // ... one launch per tiny level (lane-private copies)
    int n_tiny = 0;
    struct SmallPlan { int threads = 0, smem = 0, copies = 1; int64_t cap = 0; };
    SmallPlan small_plan[FH_MAX_LEVELS + 1];         // launch shape of each few-cell launch (plan_small)
    bool small_warp_copies = true;                   // FH_SMALL_WARP=0: one CTA copy instead of per-warp copies
    bool rep[FH_MAX_LEVELS] = {false};               // backward: level reduced into replicated copies (own pass)
    bool inrep[FH_MAX_LEVELS] = {false};             // backward, F >= 4: contended level into in-pass replicated copies
    bool fuse_merge = true;                          // FH_FUSE_MERGE=0: every group's merge as its own launch
    double fwd_limit = 0.0, bwd_limit = 0.0;         // L2 budgets of one direct pass (bytes; 0 = one pass)
    int n_sm = 148;                                  // SMs of the device (set with the status word)
    int smem_optin = 0;                              // max dynamic shared memory per CTA (opt-in)
    bool infer_ready[4] = {false, false, false, false};   // fh_infer: kernels set up, per n_in/16 - 1
    // Shifted-pair scratch, one caller-owned slot per
    // stream (fh_encoder_attach_scratch): tsh = the table shifted by one
    // entry (forward), gsh = fp32 gradient scratch shifted by two floats
    // (backward; each range is zeroed right before the launch that uses it).
    struct Scratch {
        void *stream = nullptr;
        void *tsh = nullptr;
        size_t tsh_bytes = 0;
        float *gsh = nullptr;
        size_t gsh_bytes = 0;
    };
    static constexpr int kScratchSlots = 8;
    Scratch scratch[kScratchSlots];
    int pair_shift = 3;                              // FH_PAIR_SHIFT bits: 1 backward, 2 forward (default both)
    std::mutex mu;                                   // guards the scratch slots against host threads sharing the encoder
    bool shiftable[FH_MAX_LEVELS] = {false};         // backward: level uses the shifted gradient pairs
    bool bwd_split = true;                           // FH_BWD_SPLIT=0: no entry-range passes for big levels
};
