// fhash_api.cu -- host side of libfhash.so: the C ABI declared in
// include/fhash.h (level builder a1, launch logic, validation, errors).
#include <cuda_runtime.h>

#include <cstdarg>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <new>

#include "internal.h"
#include "encode_kernels.cuh"
#include "mhe_kernels.cuh"

namespace fh {
thread_local char g_err[512] = "";
std::atomic<unsigned long long> g_launches{0};
}
using fh::aligned;
using fh::cuda_check;
using fh::dtype_size;
using fh::fail;
using fh::g_err;

// Launch shape of the few-cell backward launches (bwd_small_kernel), fixed
// per encoder: part 0 = the CTA-copy levels, part p = tiny level p - 1
// (lane-private copies).  The kernel's dynamic shared-memory limit is raised
// once here, so the backward makes no attribute calls.
static fh_status plan_small(fh_encoder e) {
    const int optin = e->smem_optin > 0 ? e->smem_optin : 232448;
    int smem_max = 0;
    for (int part = 0; part <= e->n_tiny; part++) {
        const fh::SmallSet &S = part == 0 ? e->small_cta : e->small_tiny[part - 1];
        fh_encoder_s::SmallPlan &pl = e->small_plan[part];
        pl = fh_encoder_s::SmallPlan{};
        if (S.n == 0) continue;
        int threads = 256, smem = S.total * 4, copies = 1;
        int64_t cap;
        if (part == 0) {   // one copy per warp when 8 fit in 64 KB (fewer CAS retries between warps:
                           // Combustion's 728-entry level 161 -> 144 us), else one per CTA
            const bool pw = e->small_warp_copies && 8 * S.total * 4 <= 64 * 1024;
            copies = pw ? 8 : 1;
            smem = copies * S.total * 4;
            const int per_sm = 232448 / (smem + 2048);
            const int mx = pw ? 4 : 2;
            cap = (int64_t)e->n_sm * (per_sm < 1 ? 1 : per_sm > mx ? mx : per_sm);
        } else {           // lane-private copies: whole warps per CTA, as many CTAs per SM as fit
            const int w = (optin - 4096 - smem) / (S.ttotal * 4 * 32);
            threads = (w > 8 ? 8 : w < 1 ? 1 : w) * 32;
            smem += threads * S.ttotal * 4;
            const int per_sm = 232448 / (smem + 2048);   // the SM's shared memory, not the per-CTA opt-in
            cap = (int64_t)e->n_sm * (per_sm < 1 ? 1 : per_sm > 8 ? 8 : per_sm);
        }
        pl.threads = threads;
        pl.smem = smem;
        pl.copies = copies;
        pl.cap = cap;
        smem_max = smem > smem_max ? smem : smem_max;
    }
    if (!e->flag || smem_max == 0) return FH_OK;
    const void *k = e->F == 1 ? (const void *)fh::bwd_small_kernel<1> : e->F == 2 ? (const void *)fh::bwd_small_kernel<2>
                  : e->F == 4 ? (const void *)fh::bwd_small_kernel<4> : (const void *)fh::bwd_small_kernel<8>;
    return cuda_check(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max),
                      "cudaFuncSetAttribute(bwd_small)");
}

// Device binding of a new encoder (end of fh_build_levels / fh_build_mhe):
// the launch plan (level groups from the device's L2 size, the few-cell and
// replicated backward levels, the shifted-pair levels), the SM count and
// shared-memory limit, and the 16-byte status word -- the library's ONLY
// device allocation, made here once so that no encode call allocates or
// synchronises.  Without a CUDA device (host-only use: level queries,
// scratch sizing) the plan uses B200 defaults, no status word is made, and
// every device call returns FH_E_STATE.
static fh_status bind_device(fh_encoder e) {
    int ndev = 0, dev = -1;
    int l2 = 126 * 1048576;   // B200 L2 (cudaDevAttrL2CacheSize) when no device is present
    if (cudaGetDeviceCount(&ndev) == cudaSuccess && ndev > 0 && cudaGetDevice(&dev) == cudaSuccess) {
        fh_status s = cuda_check(cudaMalloc(&e->flag, 16), "cudaMalloc(status word)");
        if (s != FH_OK) return s;
        if ((s = cuda_check(cudaMemset(e->flag, 0, 16), "cudaMemset(status word)")) != FH_OK) {
            cudaFree(e->flag);
            e->flag = nullptr;
            return s;
        }
        e->device = dev;
        cudaDeviceGetAttribute(&l2, cudaDevAttrL2CacheSize, dev);
        cudaDeviceGetAttribute(&e->n_sm, cudaDevAttrMultiProcessorCount, dev);
        cudaDeviceGetAttribute(&e->smem_optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
    } else {
        cudaGetLastError();   // clear "no device"
    }
    auto budget = [&](const char *env, double frac) -> double {
        const char *v = getenv(env);
        if (v) return atof(v) * 1048576.0;  // MiB; 0 = one group
        return frac * (double)l2;
    };
    auto make_groups = [&](double limit, size_t bytes_per_entry, int *g, int &ng) {
        ng = 0;
        g[0] = 0;
        double acc = 0.0;
        for (int l = 0; l < e->L; l++) {
            const double b = (double)e->info[l].table_size * (double)bytes_per_entry;
            if (limit > 0.0 && l > g[ng] && acc + b > limit) {
                g[++ng] = l;
                acc = 0.0;
            }
            acc += b;
        }
        g[++ng] = e->L;
    };
    // Measured on B200 (cfg4, 305 MiB fp16 tables / 609 MiB grads): one pass
    // 6.06 / 19.95 ms fwd / bwd; groups of <= 0.55 L2: 2.98 / 6.34 ms.
    if (const char *v = getenv("FH_PAIR_SHIFT")) e->pair_shift = atoi(v);
    if (const char *v = getenv("FH_BWD_SPLIT")) e->bwd_split = atoi(v) != 0;
    if (const char *v = getenv("FH_FUSE_MERGE")) e->fuse_merge = atoi(v) != 0;
    if (const char *v = getenv("FH_SMALL_WARP")) e->small_warp_copies = atoi(v) != 0;
    e->fwd_limit = budget("FH_FWD_GROUP_MB", 0.55);
    // backward: 0.45 L2 (measured with the shifted gradient scratch, whose
    // grads + scratch double a level's footprint: cfg2 bwd 0.737 -> 0.711
    // ms, cfg3 0.248 -> 0.231 ms; cfg4's 64 MiB levels group alike)
    e->bwd_limit = budget("FH_BWD_GROUP_MB", 0.45);
    make_groups(e->fwd_limit, (size_t)e->F * dtype_size(e->table_dtype), e->gf, e->n_gf);
    // Backward: the coarse, contended levels (at most FH_SMALL_MAX_T = 2048
    // entries: the few-cell end of a fold schedule) are privatised in shared
    // memory (bwd_small_kernel: one copy per CTA, lane-private copies for the
    // tiniest), smallest first, within 96 KB; the others form contiguous runs
    // split by the L2 budget.  Measured on the Combustion fold-2 shape: its
    // 728-entry level is faster privatised, its 4900-entry level faster
    // through the L2 reductions (bwd 1.79 -> 1.28 ms moving it out); copies
    // per warp instead of per CTA were slower (1.80 ms: twice the shared
    // memory, one CTA per SM).
    {
        const double lim = e->bwd_limit;
        const char *sv = getenv("FH_SMALL_KB");
        const char *tv = getenv("FH_SMALL_MAX_T");
        const uint64_t max_t = tv ? (uint64_t)atoll(tv) : 2048;
        const int per_level_max = 1 << 30, total_max = sv ? atoi(sv) * 1024 : 96 * 1024;
        bool small[FH_MAX_LEVELS] = {false};
        int order[FH_MAX_LEVELS];
        for (int l = 0; l < e->L; l++) order[l] = l;
        for (int a = 0; a < e->L; a++)   // sort level ids by table size (tiny L: insertion sort)
            for (int b = a + 1; b < e->L; b++)
                if (e->info[order[b]].table_size < e->info[order[a]].table_size) {
                    const int t = order[a]; order[a] = order[b]; order[b] = t;
                }
        int used = 0;
        for (int a = 0; a < e->L && e->kind == 0; a++) {
            const int l = order[a];
            const uint64_t bytes = e->info[l].table_size * (uint64_t)e->F * 4;
            if (e->info[l].table_size > max_t || bytes > (uint64_t)per_level_max || used + (int)bytes > total_max) break;
            small[l] = true;
            used += (int)bytes;
        }
        e->small.n = 0;
        e->small.total = 0;
        e->small.ttotal = 0;
        const bool tiny_on = !getenv("FH_TINY") || atoi(getenv("FH_TINY")) != 0;
        for (int l = 0; l < e->L; l++)
            if (small[l]) {
                const int tf = (int)(e->info[l].table_size * (uint64_t)e->F);
                const int i = e->small.n;
                e->small.id[i] = l;
                e->small.soff[i] = e->small.total;
                e->small.toff[i] = -1;
                // tiny: lane-private accumulation (bwd_small_kernel, its own
                // launch sized so every lane's copy fits shared memory)
                if (tiny_on && tf <= fh::kMaxTinyLevel && e->small.ttotal + tf <= fh::kMaxTinyFloats) {
                    e->small.toff[i] = e->small.ttotal;
                    for (int q = 0; q < tf; q++) e->small.tmap[e->small.ttotal + q] = e->small.total + q;
                    e->small.ttotal += tf;
                }
                e->small.total += tf;
                e->small.n++;
            }
        // the launches: CTA copies (non-tiny levels), then one lane-private
        // launch per tiny level (each lane's copy is then only that level,
        // so more warps fit per SM: 2x2x2x2 -> ~55 warps, 7x4x2x2 -> ~8)
        e->small_cta = fh::SmallSet{};
        e->n_tiny = 0;
        for (int i = 0; i < e->small.n; i++) {
            const int l = e->small.id[i];
            const int tf = (int)(e->info[l].table_size * (uint64_t)e->F);
            if (e->small.toff[i] >= 0) e->small_tiny[e->n_tiny++] = fh::SmallSet{};
            fh::SmallSet &D = e->small.toff[i] >= 0 ? e->small_tiny[e->n_tiny - 1] : e->small_cta;
            D.id[D.n] = l;
            D.soff[D.n] = D.total;
            D.toff[D.n] = e->small.toff[i] >= 0 ? D.total : -1;
            if (e->small.toff[i] >= 0) {
                for (int q = 0; q < tf; q++) D.tmap[D.total + q] = D.total + q;
                D.ttotal += tf;
            }
            D.total += tf;
            D.n++;
        }
        // shifted gradient pairs for the levels whose grads
        // plus scratch stay within the L2 budget; a level beyond it runs in a
        // pass of its own from HBM, where the merge would cost more than the
        // reductions it saves (measured: Combustion fold-2 shape).
        for (int q = 0; q < e->L; q++) {
            const double g = (double)e->info[q].table_size * e->F * 4.0;
            e->shiftable[q] = (e->pair_shift & 1) && e->kind == 0 && e->F == 2 && (lim <= 0.0 || 2.0 * g <= lim);
        }
        // contended mid-size levels (not small, at most FH_REP_MAX_T entries):
        // a pass of their own into replicated gradient copies (see the
        // backward launch loop), F == 2 (the copies live in the shifted scratch;
        // F == 1 would need 4-entry alignment of the copies and the merge)
        // Measured: the Combustion fold-2 shape's 4900-entry level 223 ->
        // ~150 us replicated; cfg2's 8192-entry level slower in a pass of its
        // own than mixed with the other levels (bwd 0.713 -> 0.758 ms), so
        // strictly below 8192 entries by default.
        const char *rv = getenv("FH_REP_MAX_T");
        const uint64_t rep_max = rv ? (uint64_t)atoll(rv) : 8191;
        for (int q = 0; q < e->L; q++)
            e->rep[q] = e->kind == 0 && e->F == 2 && (e->pair_shift & 1) && !small[q] &&
                        e->info[q].table_size <= rep_max;
        // F >= 4: the contended coarse levels (at most FH_INREP_MAX_T
        // entries) reduce into in-pass replicated copies (RepSpec; the number
        // of copies is decided per call from the updates per entry).
        // Measured on cfg4 (2^22 samples; levels 0-2: 8192 / 21660 / 41262
        // entries, 8192 / 3098 / 1626 updates each, 8 / 4 / 2 copies): bwd
        // 5.37 -> 5.10 ms in the train step's form.
        const char *iv = getenv("FH_INREP_MAX_T");
        const uint64_t inrep_max = iv ? (uint64_t)atoll(iv) : (uint64_t)1 << 18;
        for (int q = 0; q < e->L; q++)
            e->inrep[q] = e->kind == 0 && e->F >= 4 && !small[q] && e->info[q].table_size <= inrep_max;
        e->n_gb = 0;
        int l = 0;
        while (l < e->L) {
            if (small[l]) { l++; continue; }
            const int b = l;
            double acc = 0.0;
            while (l < e->L && !small[l]) {
                const double sz = (double)e->info[l].table_size * e->F * 4.0 * (e->shiftable[l] ? 2.0 : 1.0);
                if (lim > 0.0 && l > b && acc + sz > lim) break;
                if (l > b && (e->rep[l] || e->rep[l - 1])) break;   // replicated levels run alone
                acc += sz;
                l++;
            }
            e->gb[2 * e->n_gb] = b;
            e->gb[2 * e->n_gb + 1] = l;
            e->n_gb++;
        }
    }
    return plan_small(e);
}

// ------------------------------------------------------- shifted-pair scratch
// The shifted-pair scratch is caller-owned: attached per
// stream with fh_encoder_attach_scratch.  A pass on a stream without one
// (or with one too small) runs without the shifted pairs -- same results,
// fewer aligned pair accesses.  Lookup only: never allocates.
static fh_encoder_s::Scratch *get_scratch(fh_encoder e, cudaStream_t s, size_t tsh_bytes, size_t gsh_bytes) {
    std::lock_guard<std::mutex> lock(e->mu);
    for (auto &sc : e->scratch)
        if (sc.stream == (void *)s && (sc.tsh || sc.gsh))
            return (tsh_bytes <= sc.tsh_bytes && gsh_bytes <= sc.gsh_bytes) ? &sc : nullptr;
    return nullptr;
}

// Encode calls need the device state bind_device made, on its device.
static fh_status device_ready(fh_encoder e) {
    if (!e->flag) return fail(FH_E_STATE, "encoder was built without a CUDA device");
    int dev = -1;
    if (cudaGetDevice(&dev) != cudaSuccess) return fail(FH_E_CUDA, "cudaGetDevice failed");
    if (dev != e->device) return fail(FH_E_STATE, "encoder bound to device %d used on device %d", e->device, dev);
    return FH_OK;
}

// ------------------------------------------------------------------ launches
static dim3 grid_for(int64_t N, int L) {
    const int64_t threads = N * (int64_t)L;
    return dim3((unsigned)((threads + 255) / 256));
}

// Split the levels with include[l] into direct-pass lists whose footprint
// (T_l * bytes_per_entry) fits `limit` bytes (0 = one list), in level order.
//
// align (levels per 32-byte sector of an output row, 1 = off): when every
// level is included, a cut that would end a group mid-sector is moved down
// to the last sector boundary inside the group if the levels it moves still
// fit the next group's budget, so a pass writes whole sectors of the
// [N][L*F] rows -- a group ending mid-sector leaves partially written
// sectors that the L2 must merge with DRAM on eviction.
static int split_lists(fh_encoder e, const bool *include, double bytes_per_entry, double limit, fh::LevelList *out,
                       const bool *doubled = nullptr, int align = 1) {
    bool all = true;
    for (int l = 0; l < e->L; l++) all &= include[l];
    if (!all) align = 1;
    double sz[FH_MAX_LEVELS];
    for (int l = 0; l < e->L; l++)
        sz[l] = (double)e->info[l].table_size * bytes_per_entry * (doubled && doubled[l] ? 2.0 : 1.0);
    int n = 0;
    double acc = 0.0;
    for (int l = 0; l < e->L; l++) {
        if (!include[l]) continue;
        if (n == 0) {
            out[n++].n = 0;
            acc = 0.0;
        } else if (limit > 0.0 && out[n - 1].n > 0 && acc + sz[l] > limit) {
            fh::LevelList &cur = out[n - 1];
            const int g0 = cur.id[0];
            const int a = l / align * align;   // last sector boundary at or before l
            double moved = sz[l];
            for (int m = a; m < l; m++) moved += sz[m];
            out[n].n = 0;
            acc = 0.0;
            if (align > 1 && a > g0 && a < l && moved <= limit) {
                for (int m = a; m < l; m++) out[n].id[out[n].n++] = m;
                cur.n -= l - a;
                acc = moved - sz[l];
            }
            n++;
        }
        out[n - 1].id[out[n - 1].n++] = l;
        acc += sz[l];
    }
    return n;
}

template <int F, typename T, typename O>
static void launch_fwd(fh_encoder e, const float *coords, int64_t N, const void *table, void *out,
                       cudaStream_t s) {
    constexpr int kEb = F * (int)sizeof(T);
    // The shifted copy of the table: slot j holds entry j+1,
    // so an x-pair at (i, i+1), i odd, is ONE aligned load.  Per level: only
    // where table + copy stay within the L2 budget (else the doubled
    // footprint misses to HBM; measured Combustion fold-2 shape 0.60 ->
    // 0.74 ms) and the pass gathers enough corners to pay for the copy.
    const T *tsh = nullptr;
    bool sh[FH_MAX_LEVELS] = {false};
    fh::Params prm = e->params;
    if ((kEb == 4 || kEb == 8 || kEb == 16) && (e->pair_shift & 2) && e->kind == 0 && N >= (1 << 15)) {
        bool any = false;
        for (int l = 0; l < e->L; l++) {
            const double t = (double)e->info[l].table_size;
            // table + copy within half the group budget (cfg4's 32 MiB
            // levels doubled to 64 MiB ran 2.94 -> 3.32 ms)
            sh[l] = (e->fwd_limit <= 0.0 || 4.0 * t * kEb <= e->fwd_limit) && 8.0 * (double)N >= t;
            any |= sh[l];
        }
        uint64_t end = 0;   // the copy only spans up to the last shifted level
        for (int l = 0; l < e->L; l++)
            if (sh[l] && e->info[l].offset + e->info[l].table_size > end) end = e->info[l].offset + e->info[l].table_size;
        fh_encoder_s::Scratch *sc = any ? get_scratch(e, s, (size_t)end * kEb, 0) : nullptr;
        if (sc) {
            // one copy per run of consecutive shifted levels: slot j = entry
            // j + 1 for the run's entries [b, en).  An odd pair (i, i + 1)
            // reads slots (i - 1, i), so a run starting at an odd b also
            // needs slot b - 1 (= entry b); slot b - 1 then lies in the
            // unshifted level before the run, which never reads tsh.
            for (int l = 0; l < e->L;) {
                if (!sh[l]) { l++; continue; }
                int r = l;
                while (r + 1 < e->L && sh[r + 1]) r++;
                const uint64_t b = e->info[l].offset, en = e->info[r].offset + e->info[r].table_size;
                const uint64_t s0 = b - (b & 1);
                if (en - s0 > 1)
                    cudaMemcpyAsync(reinterpret_cast<char *>(sc->tsh) + s0 * kEb,
                                    reinterpret_cast<const char *>(table) + (s0 + 1) * kEb, (en - s0 - 1) * kEb,
                                    cudaMemcpyDeviceToDevice, s);
                l = r + 1;
            }
            tsh = reinterpret_cast<const T *>(sc->tsh);
            for (int l = 0; l < e->L; l++) prm.lv[l].tshift = sh[l] ? 1u : 0u;
        } else {
            for (int l = 0; l < e->L; l++) sh[l] = false;
        }
    }
    const float4 *c4 = reinterpret_cast<const float4 *>(coords);
    bool include[FH_MAX_LEVELS];
    for (int l = 0; l < e->L; l++) include[l] = true;
    fh::LevelList lists[FH_MAX_LEVELS];
    // small batches (e.g. the renderer's ray batches) touch few entries: one
    // pass, fewer launches; large batches: L2-sized level groups
    const double limit = N < (1 << 15) ? 0.0 : e->fwd_limit;
    const int n = split_lists(e, include, (double)F * sizeof(T), limit, lists, sh,
                              (int)(32 / (F * sizeof(O))) > 1 ? (int)(32 / (F * sizeof(O))) : 1);
    for (int g = 0; g < n; g++)
        { dim3 gg = grid_for(N, lists[g].n);
          if (F >= 4) {   // grid-stride kernel: a capped grid (FH_FWD_GRID CTAs per SM, default 8)
              static const int cap = getenv("FH_FWD_GRID") ? atoi(getenv("FH_FWD_GRID")) : 8;
              if (cap > 0 && gg.x > (unsigned)(cap * e->n_sm)) gg.x = (unsigned)(cap * e->n_sm);
          }
          fh::fwd_kernel<F, T, O><<<gg, 256, 0, s>>>(
            prm, c4, N, reinterpret_cast<const T *>(table), tsh, reinterpret_cast<O *>(out), e->flag,
            lists[g]); fh::count_launch(); }
}

template <typename T, typename O>
static void dispatch_fwd_F(fh_encoder e, const float *coords, int64_t N, const void *table, void *out,
                           cudaStream_t s) {
    switch (e->F) {
        case 1: launch_fwd<1, T, O>(e, coords, N, table, out, s); break;
        case 2: launch_fwd<2, T, O>(e, coords, N, table, out, s); break;
        case 4: launch_fwd<4, T, O>(e, coords, N, table, out, s); break;
        default: launch_fwd<8, T, O>(e, coords, N, table, out, s); break;
    }
}

static fh_status check_common(fh_encoder e, const float *coords, int64_t N, const char *who) {
    if (!e) return fail(FH_E_ARG, "%s: NULL encoder", who);
    if (N < 0) return fail(FH_E_ARG, "%s: N = %lld < 0", who, (long long)N);
    if (N > 0 && !coords) return fail(FH_E_ARG, "%s: NULL coords", who);
    if (!aligned(coords, 16)) return fail(FH_E_ARG, "%s: coords not 16-byte aligned", who);
    if (N > (int64_t)1 << 40) return fail(FH_E_RANGE, "%s: N too large", who);
    return FH_OK;
}

extern "C" {

const char *fh_last_error(void) { return g_err; }
const char *fh_version(void) { return "fhash-b200 0.1 (sm_100a)"; }

fh_status fh_fold_schedule(const uint32_t S_xyz[3], uint32_t n_t, uint32_t fold, fh_level_res *out,
                           int *L_inout) {
    g_err[0] = 0;
    if (!S_xyz || !out || !L_inout) return fail(FH_E_ARG, "fh_fold_schedule: NULL pointer");
    if (fold < 2 || n_t < 2) return fail(FH_E_ARG, "fh_fold_schedule: fold and n_t must be >= 2");
    const uint32_t S[4] = {S_xyz[0], S_xyz[1], S_xyz[2], n_t};
    int Ls = 0;
    for (int a = 0; a < 4; a++) {
        if (S[a] < 2) return fail(FH_E_ARG, "fh_fold_schedule: S[%d] = %u < 2", a, S[a]);
        // Eq. 5: ceil(log_f S) as the least L >= 1 with f^L >= S (integer).
        int La = 1;
        for (uint64_t p = fold; p < S[a]; p *= fold) La++;
        Ls = La > Ls ? La : Ls;  // Eq. 6
    }
    if (Ls > *L_inout) {
        const int cap = *L_inout;
        *L_inout = Ls;
        return fail(FH_E_RANGE, "fh_fold_schedule: L_s = %d exceeds capacity %d", Ls, cap);
    }
    for (int a = 0; a < 4; a++) {
        uint32_t r = S[a];
        out[0].res[a] = r;  // Eq. 4
        for (int l = 1; l < Ls; l++) {
            r = (r > fold) ? (r + fold - 1) / fold : 2u;  // Eqs. 7-8
            out[l].res[a] = r;
        }
    }
    *L_inout = Ls;
    return FH_OK;
}

fh_status fh_build_levels(const fh_level_res *res, int L, int F, fh_dtype table_dtype, uint64_t cap,
                          fh_encoder *out) {
    return fh_build_levels_lin(res, L, F, table_dtype, cap, FH_LIN_EQ9, out);
}

fh_status fh_build_levels_lin(const fh_level_res *res, int L, int F, fh_dtype table_dtype, uint64_t cap,
                              int linearization, fh_encoder *out) {
    g_err[0] = 0;
    if (linearization != FH_LIN_EQ9 && linearization != FH_LIN_BRICK)
        return fail(FH_E_ARG, "fh_build_levels: linearization %d not FH_LIN_EQ9 or FH_LIN_BRICK", linearization);
    if (!res || !out) return fail(FH_E_ARG, "fh_build_levels: NULL pointer");
    *out = nullptr;
    if (L < 1 || L > FH_MAX_LEVELS) return fail(FH_E_ARG, "fh_build_levels: L = %d not in [1, %d]", L, FH_MAX_LEVELS);
    if (F != 1 && F != 2 && F != 4 && F != 8) return fail(FH_E_ARG, "fh_build_levels: F = %d not in {1,2,4,8}", F);
    if (table_dtype != FH_F32 && table_dtype != FH_F16)
        return fail(FH_E_ARG, "fh_build_levels: table dtype must be FH_F32 or FH_F16");
    if (cap & (cap - 1)) return fail(FH_E_ARG, "fh_build_levels: cap %llu is not a power of two", (unsigned long long)cap);
    if (cap > (1ull << 31)) return fail(FH_E_RANGE, "fh_build_levels: cap above 2^31");
    fh_encoder e = new (std::nothrow) fh_encoder_s();
    if (!e) return fail(FH_E_ARG, "fh_build_levels: out of host memory");
    e->L = L;
    e->F = F;
    e->table_dtype = table_dtype;
    e->cap = cap;
    uint64_t off = 0;
    e->params.L = L;
    e->params.F = F;
    for (int l = 0; l < L; l++) {
        uint64_t c = 1;
        for (int a = 0; a < 4; a++) {
            const uint32_t r = res[l].res[a];
            if (r < 2 || r > (1u << 24)) {
                delete e;
                return fail(FH_E_ARG, "fh_build_levels: level %d axis %d resolution %u not in [2, 2^24]", l, a, r);
            }
            c *= r;
        }
        fh_level_info &I = e->info[l];
        memcpy(I.res, res[l].res, sizeof(I.res));
        I.corners = c;
        I.hashed = (cap != 0 && c > cap) ? 1u : 0u;
        I.table_size = I.hashed ? cap : c;
        I.reserved = I.hashed ? 0u : (uint32_t)linearization;
        I.offset = off;
        off += I.table_size;
        if (off * (uint64_t)F >= (1ull << 32)) {
            delete e;
            return fail(FH_E_RANGE, "fh_build_levels: sum T_l * F >= 2^32 at level %d", l);
        }
        fh::Level &K = e->params.lv[l];
        memset(&K, 0, sizeof(K));
        for (int a = 0; a < 4; a++) {
            K.res[a] = I.res[a];
            K.scale[a] = (float)(I.res[a] - 1);
        }
        K.sy = I.res[0];
        K.sz = I.res[0] * I.res[1];
        K.st = I.hashed ? 0u : (uint32_t)((uint64_t)I.res[0] * I.res[1] * I.res[2]);
        if (I.hashed) K.sz = 0;  // unused on hashed levels (may overflow)
        K.hashed = I.hashed ? 1u : (linearization == FH_LIN_BRICK ? 2u : 0u);
        K.mask = I.hashed ? (uint32_t)(cap - 1) : 0u;
        K.offset = (uint32_t)I.offset;
    }
    e->entries = off;
    const fh_status st = bind_device(e);
    if (st != FH_OK) { delete e; return st; }
    *out = e;
    return FH_OK;
}

fh_status fh_level_info_get(fh_encoder e, int l, fh_level_info *out) {
    g_err[0] = 0;
    if (!e || !out) return fail(FH_E_ARG, "fh_level_info_get: NULL pointer");
    if (l < 0 || l >= e->L) return fail(FH_E_ARG, "fh_level_info_get: level %d out of range", l);
    *out = e->info[l];
    return FH_OK;
}

int fh_num_levels(fh_encoder e) { return e ? e->L : 0; }
int fh_feature_dim(fh_encoder e) { return e ? e->F : 0; }
uint64_t fh_table_entries(fh_encoder e) { return e ? e->entries : 0; }
uint64_t fh_param_count(fh_encoder e) { return e ? e->entries * (uint64_t)e->F : 0; }

void fh_encoder_destroy(fh_encoder e) {
    if (!e) return;
    if (e->flag) {
        int cur = -1;
        cudaGetDevice(&cur);
        if (cur != e->device) cudaSetDevice(e->device);
        cudaFree(e->flag);
        if (cur != e->device && cur >= 0) cudaSetDevice(cur);
    }
    delete e;
}

fh_status fh_build_mhe(const uint32_t *res, int L, int F, fh_dtype table_dtype, uint64_t T, uint32_t n_frames,
                       fh_encoder *out) {
    g_err[0] = 0;
    if (!res || !out) return fail(FH_E_ARG, "fh_build_mhe: NULL pointer");
    *out = nullptr;
    if (L < 1 || L > FH_MAX_LEVELS) return fail(FH_E_ARG, "fh_build_mhe: L = %d not in [1, %d]", L, FH_MAX_LEVELS);
    if (F != 1 && F != 2 && F != 4 && F != 8) return fail(FH_E_ARG, "fh_build_mhe: F not in {1,2,4,8}");
    if (table_dtype != FH_F32 && table_dtype != FH_F16) return fail(FH_E_ARG, "fh_build_mhe: bad table dtype");
    if (T < 2 || (T & (T - 1)) || T > (1ull << 31)) return fail(FH_E_ARG, "fh_build_mhe: T must be a power of two");
    if (n_frames < 1 || n_frames > (1u << 20)) return fail(FH_E_ARG, "fh_build_mhe: bad n_frames");
    fh_encoder e = new (std::nothrow) fh_encoder_s();
    if (!e) return fail(FH_E_ARG, "fh_build_mhe: out of host memory");
    e->kind = 1;
    e->L = L;
    e->F = F;
    e->table_dtype = table_dtype;
    e->cap = T;
    e->params.L = L;
    e->params.F = F;
    uint64_t off = 0;
    for (int l = 0; l < L; l++) {
        const uint32_t R = res[l];
        if (R < 2 || R > (1u << 20)) { delete e; return fail(FH_E_ARG, "fh_build_mhe: level %d R = %u", l, R); }
        const uint64_t cube = (uint64_t)R * R * R;
        fh_level_info &I = e->info[l];
        I.res[0] = I.res[1] = I.res[2] = R;
        I.res[3] = n_frames;
        I.corners = cube * n_frames;
        I.hashed = cube > T ? 1u : 0u;
        I.table_size = T * n_frames;   // fixed T per level and frame (bucket waste when cube < T)
        I.reserved = 0;
        I.offset = off;
        off += I.table_size;
        if (off * (uint64_t)F >= (1ull << 32)) { delete e; return fail(FH_E_RANGE, "fh_build_mhe: too many parameters"); }
        fh::Level &K = e->params.lv[l];
        memset(&K, 0, sizeof(K));
        for (int a = 0; a < 3; a++) { K.res[a] = R; K.scale[a] = (float)(R - 1); }
        K.res[3] = n_frames;
        K.scale[3] = (float)(n_frames > 1 ? n_frames - 1 : 0);
        K.sy = R;
        K.sz = I.hashed ? 0u : R * R;
        K.st = (uint32_t)T;
        K.hashed = I.hashed;
        K.mask = (uint32_t)(T - 1);
        K.offset = (uint32_t)I.offset;
    }
    e->entries = off;
    const fh_status st = bind_device(e);
    if (st != FH_OK) { delete e; return st; }
    *out = e;
    return FH_OK;
}

int fh_encoder_kind(fh_encoder e) { return e ? e->kind : -1; }

unsigned long long fh_kernel_launches(void) { return fh::g_launches.load(std::memory_order_relaxed); }

// Scratch bytes of one stream slot: tsh up to the end of the last level the
// forward may shift (table + copy within half the forward group budget),
// then gsh up to the end of the last shiftable backward level, or the 64
// replicated copies of a replicated level if larger.
// The shifted gradient scratch is placed at a fixed offset from dtable
// modulo kGshSlack (kGshRel; FH_GSH_REL overrides it): its reductions and
// dtable's run side by side over the same entries, and the cfg2 backward
// measured 0.730 ms with the scratch right after the forward's table copy
// in the caller's buffer, 0.693-0.705 ms over every offset from dtable
// tried with the placement (0, 4 KiB, 64 KiB, 1-24 MiB; best 2 MiB).
static constexpr size_t kGshSlack = (size_t)32 << 20;
static constexpr size_t kGshRel = (size_t)2 << 20;

// In-pass replicated copies (RepSpec): each copy the level's T F floats
// rounded up to 64 floats (256-byte aligned copies); at most kInRepMax
// copies and at most 2^20 entries over all copies of a level.
static constexpr int kInRepMax = 32;
static size_t inrep_stride(fh_encoder e, int l) {
    return ((size_t)e->info[l].table_size * e->F + 63) / 64 * 64;
}
static int inrep_rmax(fh_encoder e, int l) {
    const uint64_t r = ((uint64_t)1 << 20) / (e->info[l].table_size ? e->info[l].table_size : 1);
    return r >= (uint64_t)kInRepMax ? kInRepMax : r < 2 ? 2 : (int)r;
}

static size_t scratch_parts(fh_encoder e, size_t *tsh_bytes, size_t *gsh_bytes) {
    const size_t kEb = (size_t)e->F * dtype_size(e->table_dtype);
    uint64_t tend = 0, gend = 0;
    size_t g = 0;
    for (int l = 0; l < e->L; l++) {
        const fh_level_info &I = e->info[l];
        if ((kEb == 4 || kEb == 8 || kEb == 16) && (e->pair_shift & 2) &&
            (e->fwd_limit <= 0.0 || 4.0 * (double)I.table_size * kEb <= e->fwd_limit))
            tend = I.offset + I.table_size;
        if (e->shiftable[l]) gend = I.offset + I.table_size;
        if (e->rep[l]) {
            const size_t stride = (size_t)((I.table_size + 2) * e->F + 3) / 4 * 4;
            if (64 * stride * 4 > g) g = 64 * stride * 4;
        }
    }
    {   // in-pass replicated copies (F >= 4): up to inrep_rmax copies of every such level
        size_t ib = 0;
        for (int l = 0; l < e->L; l++)
            if (e->inrep[l]) ib += inrep_rmax(e, l) * inrep_stride(e, l) * 4;
        if (ib > g) g = ib;
    }
    if (gend > 0 && (size_t)gend * e->F * 4 + 64 > g) g = (size_t)gend * e->F * 4 + 64;
    if (g) g += kGshSlack;   // room to place the scratch at a chosen offset from dtable (place_gsh)
    const size_t ta = ((size_t)tend * kEb + 255) / 256 * 256;
    if (tsh_bytes) *tsh_bytes = ta;
    if (gsh_bytes) *gsh_bytes = g;
    return ta + g;
}

size_t fh_encoder_scratch_size(fh_encoder e) {
    if (!e || e->kind != 0) return 0;
    return scratch_parts(e, nullptr, nullptr);
}

fh_status fh_encoder_attach_scratch(fh_encoder e, fh_stream stream, void *ptr, size_t bytes) {
    g_err[0] = 0;
    if (!e) return fail(FH_E_ARG, "fh_encoder_attach_scratch: NULL encoder");
    if (e->kind != 0) return fail(FH_E_ARG, "fh_encoder_attach_scratch: MHE encoders use no scratch");
    size_t tb, gb;
    const size_t need = scratch_parts(e, &tb, &gb);
    if (ptr && (bytes < need || !aligned(ptr, 256)))
        return fail(FH_E_ARG, "fh_encoder_attach_scratch: need %zu bytes, 256-byte aligned", need);
    std::lock_guard<std::mutex> lock(e->mu);
    void *s = stream;
    fh_encoder_s::Scratch *slot = nullptr;
    for (auto &sc : e->scratch)
        if (sc.stream == s && (sc.tsh || sc.gsh)) { slot = &sc; break; }
    if (slot) {   // detach / replace: stream-ordered with earlier passes on this stream
        fh_status st = cuda_check(cudaStreamSynchronize(reinterpret_cast<cudaStream_t>(stream)), "attach_scratch sync");
        if (st != FH_OK) return st;
        *slot = fh_encoder_s::Scratch{};
    }
    if (!ptr || need == 0) return FH_OK;   // detached (or nothing to shift): passes run without the shifted pairs
    if (!slot)
        for (auto &sc : e->scratch)
            if (!sc.tsh && !sc.gsh) { slot = &sc; break; }
    if (!slot) return fail(FH_E_STATE, "fh_encoder_attach_scratch: all %d stream slots in use", fh_encoder_s::kScratchSlots);
    slot->stream = s;
    slot->tsh = tb ? ptr : nullptr;
    slot->tsh_bytes = tb;
    slot->gsh = gb ? reinterpret_cast<float *>(reinterpret_cast<char *>(ptr) + tb) : nullptr;
    slot->gsh_bytes = gb;
    if (!slot->tsh && !slot->gsh) *slot = fh_encoder_s::Scratch{};
    return FH_OK;
}

}  // extern "C"

template <typename T, typename O>
static void dispatch_mhe_fwd(fh_encoder e, const float *coords, int64_t N, const void *table, void *out,
                             cudaStream_t s) {
    for (int g = 0; g < e->n_gf; g++) {
        const int l0 = e->gf[g], lc = e->gf[g + 1] - e->gf[g];
        const float4 *c4 = reinterpret_cast<const float4 *>(coords);
        const T *tb = reinterpret_cast<const T *>(table);
        O *o = reinterpret_cast<O *>(out);
        switch (e->F) {
            case 1: { fh::mhe::fwd_kernel<1, T, O><<<grid_for(N, lc), 256, 0, s>>>(e->params, c4, N, tb, o, e->flag, l0, lc); fh::count_launch(); } break;
            case 2: { fh::mhe::fwd_kernel<2, T, O><<<grid_for(N, lc), 256, 0, s>>>(e->params, c4, N, tb, o, e->flag, l0, lc); fh::count_launch(); } break;
            case 4: { fh::mhe::fwd_kernel<4, T, O><<<grid_for(N, lc), 256, 0, s>>>(e->params, c4, N, tb, o, e->flag, l0, lc); fh::count_launch(); } break;
            default: { fh::mhe::fwd_kernel<8, T, O><<<grid_for(N, lc), 256, 0, s>>>(e->params, c4, N, tb, o, e->flag, l0, lc); fh::count_launch(); } break;
        }
    }
}

static fh_status encode_fwd_impl(fh_encoder e, const float *coords, int64_t N,
                                 const void *table, void *out, fh_dtype out_dtype, fh_stream stream) {
    g_err[0] = 0;
    fh_status st = check_common(e, coords, N, "fh_encode_fwd");
    if (st != FH_OK) return st;
    if (out_dtype != FH_F32 && out_dtype != FH_BF16)
        return fail(FH_E_ARG, "fh_encode_fwd: out dtype must be FH_F32 or FH_BF16");
    if (N == 0) return FH_OK;
    if (!table || !aligned(table, 32)) return fail(FH_E_ARG, "fh_encode_fwd: NULL or not 32-byte aligned table");
    const size_t ovec = (size_t)e->F * dtype_size(out_dtype);
    if (!out || !aligned(out, ovec > 16 ? 16 : ovec)) return fail(FH_E_ARG, "fh_encode_fwd: NULL/misaligned out");
    if ((st = device_ready(e)) != FH_OK) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (e->kind == 1) {
        if (e->table_dtype == FH_F32) {
            if (out_dtype == FH_F32) dispatch_mhe_fwd<float, float>(e, coords, N, table, out, s);
            else dispatch_mhe_fwd<float, __nv_bfloat16>(e, coords, N, table, out, s);
        } else {
            if (out_dtype == FH_F32) dispatch_mhe_fwd<__half, float>(e, coords, N, table, out, s);
            else dispatch_mhe_fwd<__half, __nv_bfloat16>(e, coords, N, table, out, s);
        }
        return cuda_check(cudaGetLastError(), "fh_encode_fwd (MHE) launch");
    }
    if (e->table_dtype == FH_F32) {
        if (out_dtype == FH_F32) dispatch_fwd_F<float, float>(e, coords, N, table, out, s);
        else dispatch_fwd_F<float, __nv_bfloat16>(e, coords, N, table, out, s);
    } else {
        if (out_dtype == FH_F32) dispatch_fwd_F<__half, float>(e, coords, N, table, out, s);
        else dispatch_fwd_F<__half, __nv_bfloat16>(e, coords, N, table, out, s);
    }
    return cuda_check(cudaGetLastError(), "fh_encode_fwd launch");
}

// ------------------------------------------------------------- backward
// One backward call's arguments, shared by the launch helpers below.
struct BwdCall {
    fh_encoder e;
    const float4 *c4;
    int64_t N;
    const float *dout;
    fh::DoutLayout dl;
    float *dtable;
    cudaStream_t s;
};

// bwd_kernel<F, RANGED> for the encoder's F (gsh only for F <= 2).
static void launch_bwd_kernel(const BwdCall &b, dim3 g, const fh::LevelList &ll, float *dt, float *gsh, bool ranged,
                              uint32_t lo = 0, uint32_t span = 0, uint32_t rep_n = 0, int64_t rep_stride = 0,
                              fh::MergeJob mj = fh::MergeJob{nullptr, 0, 0, 0},
                              const fh::RepSpec &rs = fh::RepSpec{0, {}, {}, {}, {}}) {
    const fh_encoder e = b.e;
    g.x += (unsigned)mj.ctas;   // the merge CTAs come first (blockIdx < mj.ctas)
#define FH_BWD(FF, RR, GG)                                                                                     \
    { fh::bwd_kernel<FF, RR><<<g, 256, 0, b.s>>>(e->params, b.c4, b.N, b.dout, b.dl, dt, GG, e->flag, ll, lo, span, \
                                                 rep_n, rep_stride, mj, rs); fh::count_launch(); }
    switch (e->F) {
        case 1: if (ranged) FH_BWD(1, true, gsh) else FH_BWD(1, false, gsh) break;
        case 2: if (ranged) FH_BWD(2, true, gsh) else FH_BWD(2, false, gsh) break;
        case 4: if (ranged) FH_BWD(4, true, nullptr) else FH_BWD(4, false, nullptr) break;
        default: if (ranged) FH_BWD(8, true, nullptr) else FH_BWD(8, false, nullptr) break;
    }
#undef FH_BWD
}

// The few-cell levels (bwd_small_kernel): one launch with CTA (or per-warp)
// copies for the non-tiny ones, one lane-private launch per tiny level.
static fh_status bwd_small_levels(const BwdCall &b) {
    const fh_encoder e = b.e;
    for (int part = 0; part <= e->n_tiny; part++) {
        const fh::SmallSet &S = part == 0 ? e->small_cta : e->small_tiny[part - 1];
        if (S.n == 0) continue;
        const fh_encoder_s::SmallPlan &pl = e->small_plan[part];
        fh::SmallSet Sx = S;
        Sx.copies = pl.copies;
        int64_t blocks = (b.N * S.n + pl.threads - 1) / pl.threads;
        if (blocks > pl.cap) blocks = pl.cap;
        const dim3 g((unsigned)blocks);
        switch (e->F) {
#define FH_SMALL(FF)                                                                                                 \
    { fh::bwd_small_kernel<FF><<<g, pl.threads, pl.smem, b.s>>>(e->params, Sx, b.c4, b.N, b.dout, b.dl, b.dtable, e->flag); \
      fh::count_launch(); }                                                                                          \
    break;
            case 1: FH_SMALL(1)
            case 2: FH_SMALL(2)
            case 4: FH_SMALL(4)
            default: FH_SMALL(8)
#undef FH_SMALL
        }
    }
    return FH_OK;
}

// The shifted gradient scratch of the calling stream:
// spans the shiftable levels and holds 64 replicated copies of any
// replicated level.  nullptr when no level needs it or no slot is free.
static float *bwd_scratch(fh_encoder e, cudaStream_t s, const float *dtable, size_t *bytes) {
    bool any = false;
    for (int l = 0; l < e->L; l++) any |= e->shiftable[l] || e->rep[l] || e->inrep[l];
    if (!any) return nullptr;
    uint64_t end = 0;
    size_t need = 64;
    for (int l = 0; l < e->L; l++) {
        if (e->shiftable[l] && e->info[l].offset + e->info[l].table_size > end)
            end = e->info[l].offset + e->info[l].table_size;
        if (e->rep[l]) {
            const size_t stride = (size_t)((e->info[l].table_size + 2) * e->F + 3) / 4 * 4;
            if (64 * stride * 4 > need) need = 64 * stride * 4;
        }
    }
    if ((size_t)end * e->F * 4 + 64 > need) need = (size_t)end * e->F * 4 + 64;
    {
        size_t ib = 0;
        for (int l = 0; l < e->L; l++)
            if (e->inrep[l]) ib += inrep_rmax(e, l) * inrep_stride(e, l) * 4;
        if (ib > need) need = ib;
    }
    fh_encoder_s::Scratch *sc = get_scratch(e, s, 0, need + kGshSlack);
    if (!sc) return nullptr;
    // place_gsh: (scratch - dtable) mod kGshSlack = the chosen offset
    static const size_t want = (getenv("FH_GSH_REL") ? (size_t)atoll(getenv("FH_GSH_REL")) : kGshRel) % kGshSlack;
    const uintptr_t base = reinterpret_cast<uintptr_t>(sc->gsh);
    const size_t rel = (size_t)(base - reinterpret_cast<uintptr_t>(dtable)) % kGshSlack;
    const size_t delta = ((want + kGshSlack - rel) % kGshSlack + 255) / 256 * 256 % kGshSlack;
    *bytes = sc->gsh_bytes - delta;
    return reinterpret_cast<float *>(base + delta);
}

// A contended mid-size level (e->rep) in a pass of its own into R
// replicated copies in the scratch (CTA b -> copy b % R), so same-address
// reductions spread over R addresses, then one summing kernel.  The copies
// start at the even entry at or below the level's offset, so the pairs keep
// their 16-byte alignment.  false: not applicable (the caller runs the
// level as a normal pass).
static bool bwd_replicated(const BwdCall &b, int l, dim3 g, const fh::LevelList &ll, float *scratch, size_t cap,
                           fh_status *st) {
    const fh_encoder e = b.e;
    const uint64_t T = e->info[l].table_size, off = e->info[l].offset, off_al = off & ~1ull;
    if (!scratch || (double)b.N * 16.0 < 4096.0 * (double)T) return false;
    const int64_t stride = (int64_t)((T + (off - off_al) + 1) * e->F + 3) / 4 * 4;   // floats
    int R = (int)(cap / ((size_t)stride * 4));
    if (R > 64) R = 64;
    if (R < 2) return false;
    if ((*st = cuda_check(cudaMemsetAsync(scratch, 0, (size_t)R * stride * 4, b.s), "zero replicas")) != FH_OK)
        return true;
    launch_bwd_kernel(b, g, ll, scratch - (int64_t)off_al * e->F, nullptr, false, 0, 0, (uint32_t)R, stride);
    const int64_t cnt = (int64_t)T * e->F;
    int64_t blocks = (cnt + 255) / 256;
    if (blocks > (int64_t)e->n_sm * 4) blocks = (int64_t)e->n_sm * 4;
    { fh::rep_reduce_kernel<<<(unsigned)blocks, 256, 0, b.s>>>(b.dtable + off * e->F, scratch + (off - off_al) * e->F,
                                                               R, stride, cnt); fh::count_launch(); }
    return true;
}

static fh_status encode_bwd_impl(fh_encoder e, const float *coords, int64_t N,
                                 const float *dout, float *dtable, fh_stream stream,
                                 cudaEvent_t *ev = nullptr, int n_ev = 0, bool zero = false,
                                 bool level_major = false) {
    g_err[0] = 0;
    fh_status st = check_common(e, coords, N, "fh_encode_bwd");
    if (st != FH_OK) return st;
    const size_t vec = (size_t)e->F * 4;
    if (!dtable || !aligned(dtable, vec > 16 ? 16 : vec)) return fail(FH_E_ARG, "fh_encode_bwd: NULL/misaligned dtable");
    if (level_major && e->kind == 1)
        return fail(FH_E_ARG, "fh_encode_bwd: level-major dout is not supported by the MHE encoder");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    // zero: dtable is overwritten -- zeroed range by range right before the
    // launch that reduces into it, so the zero lines are still in L2 when the
    // reductions arrive (no DRAM read of a zeroed gradient)
    auto zero_levels = [&](int l0, int l1) -> fh_status {
        const uint64_t a = e->info[l0].offset, b = e->info[l1 - 1].offset + e->info[l1 - 1].table_size;
        return cuda_check(cudaMemsetAsync(dtable + a * e->F, 0, (b - a) * e->F * 4, s), "fh_encode_bwd: zero dtable");
    };
    if (N == 0) return zero ? zero_levels(0, e->L) : FH_OK;
    if (!dout || !aligned(dout, vec > 16 ? 16 : vec)) return fail(FH_E_ARG, "fh_encode_bwd: NULL/misaligned dout");
    if ((st = device_ready(e)) != FH_OK) return st;
    const float4 *c4 = reinterpret_cast<const float4 *>(coords);
    const int64_t LF = (int64_t)e->L * e->F;
    const fh::DoutLayout dl = level_major ? fh::DoutLayout{e->F, N * e->F} : fh::DoutLayout{LF, e->F};
    const BwdCall b{e, c4, N, dout, dl, dtable, s};
    // launch 0 (when present): the few-cell levels in shared memory
    if (e->small.n > 0) {
        if (zero)
            for (int j = 0; j < e->small.n; j++)
                if ((st = zero_levels(e->small.id[j], e->small.id[j] + 1)) != FH_OK) return st;
        if ((st = bwd_small_levels(b)) != FH_OK) return st;
        if (ev && n_ev > 0) cudaEventRecord(ev[0], s);
    }
    const int ev0 = e->small.n > 0 ? 1 : 0;
    size_t scratch_bytes = 0;
    float *scratch = bwd_scratch(e, s, dtable, &scratch_bytes);
    auto record = [&](int k) {
        if (ev && ev0 + k < n_ev) cudaEventRecord(ev[ev0 + k], s);
    };
    // A group's merge of the shifted scratch is carried by the next group's
    // backward launch (its first CTAs, while that group's reductions run);
    // the group's event follows the launch that completes it.  A pending
    // merge before any other kind of launch, or at the end, runs on its own.
    struct Pending { bool on; float *gsh; int64_t m0, m1; int k; } pend{false, nullptr, 0, 0, 0};
    auto merge_blocks = [&](int64_t m0, int64_t m1) {
        int64_t blocks = ((m1 - m0 + 1) / 2 + 255) / 256;
        if (blocks > (int64_t)e->n_sm * 8) blocks = (int64_t)e->n_sm * 8;
        return blocks;
    };
    auto flush = [&]() {
        if (!pend.on) return;
        const int64_t blocks = merge_blocks(pend.m0, pend.m1);
        if (blocks > 0) { fh::merge_shift_kernel<<<(unsigned)blocks, 256, 0, s>>>(dtable, pend.gsh, pend.m0, pend.m1); fh::count_launch(); }
        record(pend.k);
        pend.on = false;
    };
    // then one launch group per run of levels (e->gb)
    for (int k = 0; k < e->n_gb; k++) {
        const int l0 = e->gb[2 * k], lc = e->gb[2 * k + 1] - e->gb[2 * k];
        const dim3 g = grid_for(N, lc);
        if (zero && (st = zero_levels(l0, l0 + lc)) != FH_OK) return st;
        if (e->kind == 1) {   // MHE baseline encoder
            flush();
            switch (e->F) {
                case 1: { fh::mhe::bwd_kernel<1><<<g, 256, 0, s>>>(e->params, c4, N, dout, dtable, e->flag, l0, lc); fh::count_launch(); } break;
                case 2: { fh::mhe::bwd_kernel<2><<<g, 256, 0, s>>>(e->params, c4, N, dout, dtable, e->flag, l0, lc); fh::count_launch(); } break;
                case 4: { fh::mhe::bwd_kernel<4><<<g, 256, 0, s>>>(e->params, c4, N, dout, dtable, e->flag, l0, lc); fh::count_launch(); } break;
                default: { fh::mhe::bwd_kernel<8><<<g, 256, 0, s>>>(e->params, c4, N, dout, dtable, e->flag, l0, lc); fh::count_launch(); } break;
            }
            record(k);
            continue;
        }
        fh::LevelList ll;
        ll.n = lc;
        bool shift = scratch != nullptr;
        for (int i = 0; i < lc; i++) {
            ll.id[i] = l0 + i;
            shift &= e->shiftable[l0 + i];
        }
        const uint64_t ge = e->info[l0 + lc - 1].offset + e->info[l0 + lc - 1].table_size - e->info[l0].offset;
        // the shifted pairs only for passes that reduce at least about as many
        // corners as the group has entries (else the merge costs more than it saves)
        float *gsh = shift && (double)N * lc * 2.0 >= (double)ge ? scratch : nullptr;
        if (lc == 1 && e->rep[l0]) {
            flush();   // the replicated copies live in the same scratch
            if (bwd_replicated(b, l0, g, ll, scratch, scratch_bytes, &st)) {
                if (st != FH_OK) return st;
                record(k);
                continue;
            }
        }
        // this group's range of the shifted scratch, zeroed right before use
        int64_t m0 = (int64_t)e->info[l0].offset * e->F - fh::kShiftFloats;
        const int64_t m1 =
            (int64_t)(e->info[l0 + lc - 1].offset + e->info[l0 + lc - 1].table_size) * e->F - fh::kShiftFloats;
        if (m0 < 0) m0 = 0;
        if (gsh && (st = cuda_check(cudaMemsetAsync(gsh + m0, 0, (size_t)(m1 - m0) * 4, s), "zero gsh")) != FH_OK)
            return st;
        // a single level whose gradients exceed the L2 budget: P passes over
        // entry ranges of it, each L2-resident.  Measured: Combustion fold-2
        // shape (F = 2, one 95 MB level) bwd 2.24 -> 2.14 ms; cfg4 (F = 4,
        // 64 MB levels) 6.05 -> 6.34 ms (the repeated index math and dout
        // reads cost more than the L2 hits gain at 16 B per corner), so F <= 2.
        const double gbytes = (double)e->info[l0].table_size * e->F * 4.0;
        if (lc == 1 && !gsh && e->F <= 2 && e->bwd_split && e->bwd_limit > 0.0 && gbytes > e->bwd_limit) {
            flush();
            const int P = (int)std::ceil(gbytes / e->bwd_limit);
            const uint64_t T = e->info[l0].table_size, off = e->info[l0].offset;
            for (int q = 0; q < P; q++) {
                const uint64_t a = off + T * q / P, c = off + T * (q + 1) / P;
                launch_bwd_kernel(b, g, ll, dtable, nullptr, true, (uint32_t)a, (uint32_t)(c - a));
            }
            record(k);
            continue;
        }
        // contended levels of this group into in-pass replicated copies
        // (F >= 4; for u updates per entry, R = u / FH_INREP_UPDATES (1024)
        // rounded up to a power of two, 2 <= R <= inrep_rmax; measured on
        // cfg4: 512 / 1024 / 2048 updates per copy 5.10 / 5.10 / 5.17 ms)
        fh::RepSpec rs{0, {}, {}, {}, {}};
        if (scratch && !gsh) {
            static const double per_copy = getenv("FH_INREP_UPDATES") ? atof(getenv("FH_INREP_UPDATES")) : 1024.0;
            size_t used = 0;
            for (int i = 0; i < lc && rs.n < fh::kMaxInRep; i++) {
                const int l = l0 + i;
                if (!e->inrep[l]) continue;
                const double u = (double)N * 16.0 / (double)e->info[l].table_size;
                int R = 1;
                while (R < kInRepMax && R * per_copy < u) R *= 2;
                if (R > inrep_rmax(e, l)) R = inrep_rmax(e, l);
                if (R < 2) continue;
                const size_t stride = inrep_stride(e, l);
                if ((used + R * stride) * 4 > scratch_bytes) break;
                float *copies = scratch + used;
                if ((st = cuda_check(cudaMemsetAsync(copies, 0, R * stride * 4, s), "zero replicas")) != FH_OK)
                    return st;
                rs.lvl[rs.n] = l;
                rs.R[rs.n] = R;
                rs.base[rs.n] = copies - (int64_t)e->info[l].offset * e->F;
                rs.stride[rs.n] = (int64_t)stride;
                rs.n++;
                used += R * stride;
            }
        }
        fh::MergeJob mj{nullptr, 0, 0, 0};
        if (pend.on && e->fuse_merge) {
            const int64_t blocks = merge_blocks(pend.m0, pend.m1);
            mj = fh::MergeJob{pend.gsh, pend.m0, pend.m1, (int)(blocks < 2 * e->n_sm ? blocks : 2 * e->n_sm)};
        } else {
            flush();
        }
        launch_bwd_kernel(b, g, ll, dtable, gsh, false, 0, 0, 0, 0, mj, rs);
        for (int q = 0; q < rs.n; q++) {   // dtable += the sum of the level's copies
            const int l = rs.lvl[q];
            const int64_t cnt = (int64_t)e->info[l].table_size * e->F;
            int64_t blocks = (cnt + 255) / 256;
            if (blocks > (int64_t)e->n_sm * 4) blocks = (int64_t)e->n_sm * 4;
            { fh::rep_reduce_kernel<<<(unsigned)blocks, 256, 0, s>>>(dtable + (int64_t)e->info[l].offset * e->F,
                                                                     rs.base[q] + (int64_t)e->info[l].offset * e->F,
                                                                     rs.R[q], rs.stride[q], cnt); fh::count_launch(); }
        }
        if (mj.ctas > 0) {
            record(pend.k);
            pend.on = false;
        }
        if (gsh) pend = Pending{true, gsh, m0, m1, k};
        else record(k);
    }
    flush();
    return cuda_check(cudaGetLastError(), "fh_encode_bwd launch");
}

namespace fh {
// Backward launches of fh_encode_bwd (natural order) and the table element
// ranges each one finalises -- for callers that overlap the gradient
// reduction with the rest of the backward (train_api.cu).
int bwd_launch_count(fh_encoder e) {
    if (!e) return -1;
    return (e->small.n > 0 ? 1 : 0) + e->n_gb;
}
int bwd_launch_ranges(fh_encoder e, int i, int64_t *r, int max) {
    const int cnt = bwd_launch_count(e);
    if (i < 0 || i >= cnt) return -1;
    const int64_t F = e->F;
    int k = 0;
    if (e->small.n > 0) {
        if (i == 0) {
            for (int j = 0; j < e->small.n; j++) {
                const fh_level_info &I = e->info[e->small.id[j]];
                if (k < max) { r[2 * k] = (int64_t)I.offset * F; r[2 * k + 1] = (int64_t)(I.offset + I.table_size) * F; }
                k++;
            }
            return k;
        }
        i -= 1;
    }
    const fh_level_info &a = e->info[e->gb[2 * i]], &b = e->info[e->gb[2 * i + 1] - 1];
    if (max > 0) { r[0] = (int64_t)a.offset * F; r[1] = (int64_t)(b.offset + b.table_size) * F; }
    return 1;
}
fh_status encode_bwd_events(fh_encoder e, const float *coords, int64_t N, const float *dout, float *dtable,
                            fh_stream stream, cudaEvent_t *ev, int n_ev, bool overwrite, bool level_major) {
    return encode_bwd_impl(e, coords, N, dout, dtable, stream, ev, n_ev, overwrite, level_major);
}
}  // namespace fh

extern "C" {

fh_status fh_encode_fwd(fh_encoder e, const float *coords, int64_t N, const void *table, void *out,
                        fh_dtype out_dtype, fh_stream stream) {
    return encode_fwd_impl(e, coords, N, table, out, out_dtype, stream);
}

fh_status fh_encode_bwd_ex(fh_encoder e, const float *coords, int64_t N, const float *dout, float *dtable,
                           unsigned flags, fh_stream stream) {
    if (flags & ~(unsigned)(FH_BWD_OVERWRITE | FH_BWD_DOUT_LEVEL_MAJOR))
        return fail(FH_E_ARG, "fh_encode_bwd_ex: unknown flags 0x%x", flags);
    return encode_bwd_impl(e, coords, N, dout, dtable, stream, nullptr, 0, (flags & FH_BWD_OVERWRITE) != 0,
                           (flags & FH_BWD_DOUT_LEVEL_MAJOR) != 0);
}

fh_status fh_encode_bwd(fh_encoder e, const float *coords, int64_t N, const float *dout, float *dtable,
                        fh_stream stream) {
    return encode_bwd_impl(e, coords, N, dout, dtable, stream);
}

fh_status fh_encode_indices(fh_encoder e, const float *coords, int64_t N, uint32_t *idx, float *w,
                            fh_stream stream) {
    g_err[0] = 0;
    fh_status st = check_common(e, coords, N, "fh_encode_indices");
    if (st != FH_OK) return st;
    if (N == 0) return FH_OK;
    if (!idx || !aligned(idx, 16) || !aligned(w, 16)) return fail(FH_E_ARG, "fh_encode_indices: NULL/misaligned output");
    if ((st = device_ready(e)) != FH_OK) return st;
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    if (e->kind == 1)
        { fh::mhe::indices_kernel<<<grid_for(N, e->L), 256, 0, s>>>(
            e->params, reinterpret_cast<const float4 *>(coords), N, idx, w, e->flag); fh::count_launch(); }
    else
        { fh::indices_kernel<<<grid_for(N, e->L), 256, 0, s>>>(e->params, reinterpret_cast<const float4 *>(coords),
                                                             N, idx, w, e->flag); fh::count_launch(); }
    return cuda_check(cudaGetLastError(), "fh_encode_indices launch");
}

fh_status fh_zero_grad(fh_encoder e, float *dtable, fh_stream stream) {
    g_err[0] = 0;
    if (!e || !dtable) return fail(FH_E_ARG, "fh_zero_grad: NULL pointer");
    return cuda_check(cudaMemsetAsync(dtable, 0, e->entries * e->F * 4, reinterpret_cast<cudaStream_t>(stream)),
                      "fh_zero_grad");
}

fh_status fh_encode_fwd_bwd(fh_encoder e, const float *coords, int64_t N, const void *table, void *out,
                            fh_dtype out_dtype, const float *dout, float *dtable, int zero_dtable,
                            fh_stream stream) {
    g_err[0] = 0;
    if (!e) return fail(FH_E_ARG, "fh_encode_fwd_bwd: NULL encoder");
    if (!dtable) return fail(FH_E_ARG, "fh_encode_fwd_bwd: NULL dtable");
    fh_status st;
    if ((st = fh_encode_fwd(e, coords, N, table, out, out_dtype, stream)) != FH_OK) return st;
    return fh_encode_bwd_ex(e, coords, N, dout, dtable, zero_dtable ? FH_BWD_OVERWRITE : 0, stream);
}

fh_status fh_encode_step_host(fh_encoder e, const float *coords_h, const float *dout_h, int64_t N,
                              const void *table_d, float *coords_d, float *dout_d, float *out_d,
                              float *dtable_d, float *out_h, float *dtable_h, fh_stream stream) {
    g_err[0] = 0;
    if (!e) return fail(FH_E_ARG, "fh_encode_step_host: NULL encoder");
    if (N < 0 || (N > 0 && (!coords_h || !dout_h || !coords_d || !dout_d || !out_d || !out_h)) || !dtable_d || !dtable_h)
        return fail(FH_E_ARG, "fh_encode_step_host: NULL pointer");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    const size_t LF = (size_t)e->L * e->F;
    fh_status st;
    if ((st = cuda_check(cudaMemcpyAsync(coords_d, coords_h, (size_t)N * 16, cudaMemcpyHostToDevice, s), "H2D coords")) != FH_OK) return st;
    if ((st = cuda_check(cudaMemcpyAsync(dout_d, dout_h, (size_t)N * LF * 4, cudaMemcpyHostToDevice, s), "H2D dout")) != FH_OK) return st;
    if ((st = fh_encode_fwd(e, coords_d, N, table_d, out_d, FH_F32, stream)) != FH_OK) return st;
    if ((st = fh_encode_bwd_ex(e, coords_d, N, dout_d, dtable_d, FH_BWD_OVERWRITE, stream)) != FH_OK) return st;
    if ((st = cuda_check(cudaMemcpyAsync(out_h, out_d, (size_t)N * LF * 4, cudaMemcpyDeviceToHost, s), "D2H out")) != FH_OK) return st;
    return cuda_check(cudaMemcpyAsync(dtable_h, dtable_d, e->entries * e->F * 4, cudaMemcpyDeviceToHost, s), "D2H dtable");
}

fh_status fh_status_sync(fh_encoder e, fh_stream stream) {
    g_err[0] = 0;
    if (!e) return fail(FH_E_ARG, "fh_status_sync: NULL encoder");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    fh_status st = cuda_check(cudaStreamSynchronize(s), "fh_status_sync");
    if (st != FH_OK || !e->flag) return st;
    int h = 0;
    if ((st = cuda_check(cudaMemcpy(&h, e->flag, sizeof(int), cudaMemcpyDeviceToHost), "read status word")) != FH_OK) return st;
    if (h) {
        if ((st = cuda_check(cudaMemset(e->flag, 0, sizeof(int)), "clear status word")) != FH_OK) return st;
        return fail(FH_E_DOMAIN, "out-of-domain or NaN coordinates were clamped to [0,1]");
    }
    return FH_OK;
}

}  // extern "C"

#include "stats.cuh"
