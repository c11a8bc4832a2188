// train_api.cu -- host side of the train step (include/fhash.h "train
// step" section): trainer object, launch sequence, Adam bookkeeping.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>

#include <dlfcn.h>

#include <cmath>
#include <cstring>
#include <new>
#include <vector>

#include "internal.h"
#include "mlp_kernels.cuh"
#include "infer_kernels.cuh"

using fh::aligned;
using fh::cuda_check;
using fh::fail;
using fh::g_err;

struct fh_trainer_s {
    fh_encoder enc = nullptr;
    int K0 = 0;
    fh_train_buffers b{};
    fh_adam adam{};
    int64_t max_batch = 0;
    int64_t step = 0;
    int n_sm = 148;
    // workspace carve-up
    __nv_bfloat16 *enc_out = nullptr;  // [max_batch][K0]
    float *dx = nullptr;               // [max_batch][K0], or [L][N][F] when dx_lm
    int dx_lm = 0;                     // F when dX is level-major (F >= 4; see make_mlp_maps), else 0
    int *flag = nullptr;               // bit 1: non-finite loss
    float *partial = nullptr;          // [2 n_sm][P] per-slot MLP gradient partials
    float *loss_scratch = nullptr;
    cudaEvent_t bwd_ev[FH_MAX_LEVELS + 1] = {};  // caller's events, recorded after each backward launch
    int n_bwd_ev = 0;
    bool flags_cleared = false;        // the workspace flags are zeroed on the first step's stream
    // fused data-parallel form (fh_trainer_set_comm)
    struct DP {
        void *comm = nullptr;
        int W = 1, rank = 0;
        cudaStream_t cs = nullptr;                 // communication stream
        cudaEvent_t ev[FH_MAX_LEVELS + 1] = {};    // after each backward launch
        cudaEvent_t ev_step = nullptr, ev_red = nullptr;
        struct Main { int launch; int64_t a, m; };
        std::vector<Main> mains;                   // reduce-scattered parts (overlap plan)
        std::vector<int64_t> tb, te;               // tails (replicated)
        float *shard = nullptr, *tail = nullptr;   // workspace views
        int64_t n_tail = 0;
    } dp;
};

namespace {

size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }

// The MLP kernel's per-slot gradient partials: 2 slots x (at most) one CTA
// per SM of the encoder's device.
size_t partial_bytes(fh_encoder enc, int K0) {
    return align_up((size_t)2 * enc->n_sm * ((fh::mlp::param_count(K0) + 3) / 4 * 4) * 4, 256);
}

template <int K0>
int mlp_smem() {
    using Lo = fh::mlp::Layout<K0>;
    // enough dynamic smem to keep ONE CTA per SM (the kernel owns all 512
    // TMEM columns of its SM)
    return (int)(Lo::SMEM > 120 * 1024 ? Lo::SMEM : 120 * 1024);
}

// Raise the MLP train kernel's dynamic shared-memory limit once (trainer
// creation), never on the step path.
fh_status set_mlp_attrs(int K0) {
    auto set = [](const void *k, int smem) {
        return cuda_check(cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, smem),
                          "cudaFuncSetAttribute(mlp)");
    };
    fh_status st = FH_OK;
    switch (K0) {
        case 16: st = set((const void *)fh::mlp::mlp_train_kernel<16>, mlp_smem<16>()); break;
        case 32: st = set((const void *)fh::mlp::mlp_train_kernel<32>, mlp_smem<32>()); break;
        case 48: st = set((const void *)fh::mlp::mlp_train_kernel<48>, mlp_smem<48>()); break;
        default: st = set((const void *)fh::mlp::mlp_train_kernel<64>, mlp_smem<64>()); break;
    }
    return st;
}

fh_status check_mlp(fh_encoder enc, const fh_mlp_desc *m) {
    if (!enc || !m) return fail(FH_E_ARG, "NULL encoder or MLP descriptor");
    if (m->n_hidden != 64 || m->n_hidden_layers != 2)
        return fail(FH_E_ARG, "MLP must be n_in -> 64 -> 64 -> 1 (n_hidden 64, 2 hidden layers)");
    if (m->n_in != enc->L * enc->F) return fail(FH_E_ARG, "MLP n_in %d != L*F = %d", m->n_in, enc->L * enc->F);
    if (m->n_in != 16 && m->n_in != 32 && m->n_in != 48 && m->n_in != 64)
        return fail(FH_E_ARG, "MLP n_in must be 16, 32, 48 or 64 (got %d)", m->n_in);
    return FH_OK;
}

// The MLP kernel's tensor maps for an N-sample launch (host-side encoding,
// no device work; the encode function comes from the driver through the
// runtime, no libcuda link):
//   x  [N][K0] bf16 as 4-D (8 elements, row % 8, 16-byte chunk, row / 8),
//      box (8, 8, K0 / 8, 16): a 128-row tile lands in the core-matrix
//      layout (SWIZZLE_NONE, SBO = K0 * 16); row groups past N read as zero;
//   dx [N][K0] fp32, box 128 rows x 16 columns, 64-byte swizzle (the
//      kernel's dX staging layout); rows past N are not written.
//      Level-major (tr->dx_lm = F >= 4): dX is [L][N][F], a 3-D map
//      (F, N, L), box (F, 128, 16 / F) = 8 KB, no swizzle -- the encode
//      backward's level passes then read contiguous 16-byte rows
//      (FH_BWD_DOUT_LEVEL_MAJOR; cfg4 bwd 6.11 -> 5.51 ms).
PFN_cuTensorMapEncodeTiled_v12000 tmap_encoder() {
    static PFN_cuTensorMapEncodeTiled_v12000 encode = nullptr;
    if (!encode) {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) == cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }
    return encode;
}

fh_status make_mlp_maps(fh_trainer tr, int64_t N, CUtensorMap *tm_x, CUtensorMap *tm_dx) {
    PFN_cuTensorMapEncodeTiled_v12000 encode = tmap_encoder();
    if (!encode) return fail(FH_E_CUDA, "cuTensorMapEncodeTiled not available from the driver");
    const cuuint64_t K0 = (cuuint64_t)tr->K0;
    {
        cuuint64_t dims[4] = {8, 8, K0 / 8, (cuuint64_t)((N + 7) / 8)};
        cuuint64_t strides[3] = {K0 * 2, 16, K0 * 16};
        cuuint32_t box[4] = {8, 8, (cuuint32_t)(K0 / 8), 16};
        cuuint32_t es[4] = {1, 1, 1, 1};
        const CUresult r = encode(tm_x, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 4, tr->enc_out, dims, strides, box, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(FH_E_CUDA, "cuTensorMapEncodeTiled(x) failed (%d)", (int)r);
    }
    if (tr->dx_lm) {
        const cuuint64_t F = (cuuint64_t)tr->dx_lm;
        cuuint64_t dims[3] = {F, (cuuint64_t)N, K0 / F};
        cuuint64_t strides[2] = {F * 4, (cuuint64_t)N * F * 4};
        cuuint32_t box[3] = {(cuuint32_t)F, 128, (cuuint32_t)(16 / F)};
        cuuint32_t es[3] = {1, 1, 1};
        const CUresult r = encode(tm_dx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, tr->dx, dims, strides, box, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(FH_E_CUDA, "cuTensorMapEncodeTiled(dx, level-major) failed (%d)", (int)r);
    } else {
        cuuint64_t dims[2] = {K0, (cuuint64_t)N};
        cuuint64_t strides[1] = {K0 * 4};
        cuuint32_t box[2] = {16, 128};
        cuuint32_t es[2] = {1, 1};
        const CUresult r = encode(tm_dx, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, tr->dx, dims, strides, box, es,
                                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B,
                                  CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r != CUDA_SUCCESS) return fail(FH_E_CUDA, "cuTensorMapEncodeTiled(dx) failed (%d)", (int)r);
    }
    return FH_OK;
}

template <int K0>
fh_status launch_mlp(fh_trainer tr, const float *target, int64_t N, int64_t N_global, float *loss,
                     cudaStream_t s) {
    const int smem = mlp_smem<K0>();
    CUtensorMap tm_x, tm_dx;
    fh_status st = make_mlp_maps(tr, N, &tm_x, &tm_dx);
    if (st != FH_OK) return st;
    fh::mlp::TrainArgs a;
    a.x = tr->enc_out;
    a.target = target;
    a.wsh = reinterpret_cast<const __nv_bfloat16 *>(tr->b.mlp_shadow);
    a.wmaster = tr->b.mlp_master;
    a.dx = tr->dx;
    a.grad = tr->b.mlp_grad;
    a.partial = tr->partial;
    a.P = (fh::mlp::param_count(K0) + 3) / 4 * 4;   // partial row stride (16-byte rows)
    a.loss = loss;
    a.flag = tr->flag;
    a.N = N;
    a.inv_n_global = (float)(1.0 / (double)N_global);
    a.dx_lm_log2 = tr->dx_lm == 8 ? 3 : tr->dx_lm == 4 ? 2 : 0;
    // level-major dX straight from registers, MMA5 overlapping that epilogue
    // (ncu, cfg4 2^22: 527 us per launch vs 585 through the staging tile and
    // 3-D TMA stores; FH_DX_STAGE=1 keeps the staged form, for A/B)
    static const bool stage = getenv("FH_DX_STAGE") != nullptr;
    a.dx_direct = stage ? 0 : 1;
    const int64_t tiles = (N + fh::mlp::TILE - 1) / fh::mlp::TILE;
    const int64_t pairs = (tiles + 1) / 2;  // two tile slots per CTA
    const int grid = (int)(pairs < tr->n_sm ? pairs : tr->n_sm);
    { fh::mlp::mlp_train_kernel<K0><<<grid, fh::mlp::TRAIN_THREADS, smem, s>>>(a, tm_x, tm_dx); fh::count_launch(); }
    const int rows = 2 * grid;
    const dim3 rg((unsigned)((a.P + 255) / 256), (unsigned)((rows + 15) / 16));
    { fh::mlp::mlp_grad_reduce_kernel<<<rg, 256, 0, s>>>(tr->b.mlp_grad, tr->partial, rows, a.P,
                                                          fh::mlp::param_count(K0)); fh::count_launch(); }
    return cuda_check(cudaGetLastError(), "mlp_train_kernel launch");
}

}  // namespace

extern "C" {

uint64_t fh_mlp_param_count(const fh_mlp_desc *m) {
    return m ? (uint64_t)fh::mlp::param_count(m->n_in) : 0;
}

size_t fh_train_workspace_size(fh_encoder enc, const fh_mlp_desc *m, int64_t max_batch) {
    if (!enc || !m || max_batch < 0) return 0;
    const size_t K0 = (size_t)m->n_in;
    // the encoder-output rows are sized to whole 8-row groups: the MLP
    // kernel's X tensor map reads the last group whole (rows past N zeroed)
    return align_up(align_up((size_t)max_batch, 8) * K0 * 2, 256) + align_up((size_t)max_batch * K0 * 4, 256) + 256 +
           partial_bytes(enc, m->n_in);
}

fh_status fh_trainer_create(fh_encoder enc, const fh_mlp_desc *m, const fh_train_buffers *b, const fh_adam *adam,
                            int64_t max_batch, fh_trainer *out) {
    g_err[0] = 0;
    if (!out || !b || !adam) return fail(FH_E_ARG, "fh_trainer_create: NULL pointer");
    *out = nullptr;
    fh_status st = check_mlp(enc, m);
    if (st != FH_OK) return st;
    if (max_batch < 1) return fail(FH_E_ARG, "fh_trainer_create: max_batch < 1");
    if (!enc->flag) return fail(FH_E_STATE, "fh_trainer_create: encoder was built without a CUDA device");
    const void *need16[] = {b->table_master, b->table_grad, b->table_m, b->table_v, b->mlp_master,
                            b->mlp_grad, b->mlp_m, b->mlp_v, b->mlp_shadow, b->workspace};
    for (const void *p : need16)
        if (!p || !aligned(p, 16)) return fail(FH_E_ARG, "fh_trainer_create: NULL or misaligned buffer");
    if (enc->table_dtype == FH_F16 && (!b->table_shadow || !aligned(b->table_shadow, 32)))
        return fail(FH_E_ARG, "fh_trainer_create: FH_F16 encoder needs a 32-byte aligned fp16 table_shadow");
    if (enc->table_dtype == FH_F32 && b->table_shadow)
        return fail(FH_E_ARG, "fh_trainer_create: FH_F32 encoder reads the master; pass table_shadow = NULL");
    if (enc->table_dtype == FH_F32 && !aligned(b->table_master, 32))
        return fail(FH_E_ARG, "fh_trainer_create: table_master must be 32-byte aligned");
    if (b->workspace_bytes < fh_train_workspace_size(enc, m, max_batch))
        return fail(FH_E_ARG, "fh_trainer_create: workspace too small");
    fh_trainer tr = new (std::nothrow) fh_trainer_s();
    if (!tr) return fail(FH_E_ARG, "fh_trainer_create: out of host memory");
    tr->enc = enc;
    tr->K0 = m->n_in;
    tr->b = *b;
    tr->adam = *adam;
    tr->max_batch = max_batch;
    tr->n_sm = enc->n_sm;
    // dL/d(enc) level-major for F >= 4 (FH_DX_ROW_MAJOR=1: the row-major form, for A/B)
    tr->dx_lm = (enc->F >= 4 && !getenv("FH_DX_ROW_MAJOR")) ? enc->F : 0;
    char *w = reinterpret_cast<char *>(b->workspace);
    tr->enc_out = reinterpret_cast<__nv_bfloat16 *>(w);
    w += align_up(align_up((size_t)max_batch, 8) * tr->K0 * 2, 256);
    tr->dx = reinterpret_cast<float *>(w);
    w += align_up((size_t)max_batch * tr->K0 * 4, 256);
    tr->flag = reinterpret_cast<int *>(w);
    tr->loss_scratch = reinterpret_cast<float *>(w + 16);
    tr->partial = reinterpret_cast<float *>(w + 256);
    // no device work here: the flags are cleared on the first step's stream
    if ((st = set_mlp_attrs(tr->K0)) != FH_OK) { delete tr; return st; }
    if (max_batch >= (int64_t)1 << 31) { delete tr; return fail(FH_E_ARG, "fh_trainer_create: max_batch >= 2^31"); }
    if (!tmap_encoder()) { delete tr; return fail(FH_E_CUDA, "cuTensorMapEncodeTiled not available from the driver"); }
    *out = tr;
    return FH_OK;
}

fh_status fh_train_fwd_bwd(fh_trainer tr, const float *coords, const float *target, int64_t N, int64_t N_global,
                           float *loss_dev, fh_stream stream) {
    g_err[0] = 0;
    if (!tr) return fail(FH_E_ARG, "fh_train_fwd_bwd: NULL trainer");
    if (N < 0 || N > tr->max_batch || N_global < N || N_global < 1)
        return fail(FH_E_ARG, "fh_train_fwd_bwd: need 0 <= N_local <= max_batch and N_global >= max(N_local, 1)");
    if (N > 0 && (!coords || !target)) return fail(FH_E_ARG, "fh_train_fwd_bwd: NULL coords/target");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    float *loss = loss_dev ? loss_dev : tr->loss_scratch;
    fh_status st;
    if (!tr->flags_cleared) {
        if ((st = cuda_check(cudaMemsetAsync(tr->flag, 0, 32, s), "clear trainer flags")) != FH_OK) return st;
        tr->flags_cleared = true;
    }
    st = cuda_check(cudaMemsetAsync(loss, 0, sizeof(float), s), "zero loss");
    if (st != FH_OK) return st;
    // the step's gradients OVERWRITE the grad buffers: the MLP kernel adds
    // into zeroed MLP grads; the encode backward zeroes each table level
    // group right before reducing into it (FH_BWD_OVERWRITE)
    st = cuda_check(cudaMemsetAsync(tr->b.mlp_grad, 0, (size_t)fh::mlp::param_count(tr->K0) * sizeof(float), s),
                    "zero mlp_grad");
    if (st != FH_OK) return st;
    if (N == 0) {   // no samples on this rank: zero gradients, and the caller's
                    // per-launch events still mark them final (DP overlap)
        st = cuda_check(cudaMemsetAsync(tr->b.table_grad, 0, (size_t)tr->enc->entries * tr->enc->F * sizeof(float), s),
                        "zero table_grad");
        if (st != FH_OK) return st;
        for (int i = 0; i < tr->n_bwd_ev; i++)
            if ((st = cuda_check(cudaEventRecord(tr->bwd_ev[i], s), "record bwd event")) != FH_OK) return st;
        return FH_OK;
    }
    const void *table = tr->b.table_shadow ? tr->b.table_shadow : tr->b.table_master;
    if ((st = fh_encode_fwd(tr->enc, coords, N, table, tr->enc_out, FH_BF16, stream)) != FH_OK) return st;
    switch (tr->K0) {
        case 16: st = launch_mlp<16>(tr, target, N, N_global, loss, s); break;
        case 32: st = launch_mlp<32>(tr, target, N, N_global, loss, s); break;
        case 48: st = launch_mlp<48>(tr, target, N, N_global, loss, s); break;
        default: st = launch_mlp<64>(tr, target, N, N_global, loss, s); break;
    }
    if (st != FH_OK) return st;
    return fh::encode_bwd_events(tr->enc, coords, N, tr->dx, tr->b.table_grad, stream, tr->bwd_ev, tr->n_bwd_ev,
                                 /*overwrite=*/true, /*level_major=*/tr->dx_lm != 0);
}

int fh_train_dx_layout(fh_trainer tr) { return tr ? tr->dx_lm : -1; }

int fh_train_bwd_launches(fh_trainer tr) { return tr ? fh::bwd_launch_count(tr->enc) : -1; }

fh_status fh_train_bwd_ranges(fh_trainer tr, int launch, int64_t *ranges, int max_ranges, int *n_ranges) {
    g_err[0] = 0;
    if (!tr || !ranges || !n_ranges || max_ranges < 0) return fail(FH_E_ARG, "fh_train_bwd_ranges: NULL argument");
    const int k = fh::bwd_launch_ranges(tr->enc, launch, ranges, max_ranges);
    if (k < 0) return fail(FH_E_ARG, "fh_train_bwd_ranges: launch %d out of range", launch);
    *n_ranges = k;
    if (k > max_ranges) return fail(FH_E_RANGE, "fh_train_bwd_ranges: %d ranges, capacity %d", k, max_ranges);
    return FH_OK;
}

fh_status fh_train_set_bwd_events(fh_trainer tr, void *const *events, int n) {
    g_err[0] = 0;
    if (!tr) return fail(FH_E_ARG, "fh_train_set_bwd_events: NULL trainer");
    const int cnt = fh::bwd_launch_count(tr->enc);
    if (n != 0 && n != cnt)
        return fail(FH_E_ARG, "fh_train_set_bwd_events: %d events for %d backward launches", n, cnt);
    if (n > 0 && !events) return fail(FH_E_ARG, "fh_train_set_bwd_events: NULL events");
    for (int i = 0; i < n; i++) tr->bwd_ev[i] = reinterpret_cast<cudaEvent_t>(events[i]);
    tr->n_bwd_ev = n;
    return FH_OK;
}

}  // extern "C"

// Adam over the table element ranges [begin_i, end_i) with gradients
// grad_i (indexed from begin_i), plus the whole MLP segment: ONE launch, one
// step of the bias-correction counter.
static fh_status apply_ranges_impl(fh_trainer tr, int n, const int64_t *begin, const int64_t *end,
                                   float *const *grad, cudaStream_t s) {
    using fh::mlp::AdamArgs;
    using fh::mlp::AdamSeg;
    if (n < 0 || n + 1 > fh::mlp::kMaxAdamSeg)
        return fail(FH_E_ARG, "Adam: %d table ranges (max %d)", n, fh::mlp::kMaxAdamSeg - 1);
    tr->step += 1;
    const double t = (double)tr->step;
    AdamArgs A;
    memset(&A, 0, sizeof(A));
    A.lr = tr->adam.lr;
    A.b1 = tr->adam.beta1;
    A.b2 = tr->adam.beta2;
    A.eps = tr->adam.eps;
    A.omb1 = (float)(1.0 - (double)tr->adam.beta1);
    A.omb2 = (float)(1.0 - (double)tr->adam.beta2);
    A.c1 = (float)(1.0 / (1.0 - std::pow((double)tr->adam.beta1, t)));
    A.c2 = (float)(1.0 / (1.0 - std::pow((double)tr->adam.beta2, t)));
    const int64_t cap = (int64_t)tr->n_sm * 16;
    int64_t total_n = 0;
    for (int i = 0; i < n; i++) total_n += end[i] - begin[i];
    int64_t blocks = 0;
    int k = 0;
    auto add = [&](AdamSeg g, int64_t want) {
        if (g.n <= 0) return;
        g.vec = (aligned(g.p, 16) && aligned(g.g, 16) && aligned(g.m, 16) && aligned(g.v, 16) &&
                 (g.kind == 0 || aligned(g.shadow, 8))) ? 1 : 0;
        if (want < 1) want = 1;
        A.seg[k] = g;
        A.block0[k] = blocks;
        blocks += want;
        k++;
    };
    for (int i = 0; i < n; i++) {
        AdamSeg T{};
        T.p = tr->b.table_master + begin[i];
        T.g = grad[i];
        T.m = tr->b.table_m + begin[i];
        T.v = tr->b.table_v + begin[i];
        T.shadow = tr->b.table_shadow ? reinterpret_cast<__half *>(tr->b.table_shadow) + begin[i] : nullptr;
        T.n = end[i] - begin[i];
        T.kind = tr->b.table_shadow ? 1 : 0;
        // blocks for ~4 float4 per thread, shared out of the cap in proportion to size
        int64_t want = (T.n / 4 + 256 * 4 - 1) / (256 * 4);
        if (total_n > 0 && want > cap * T.n / total_n + 1) want = cap * T.n / total_n + 1;
        add(T, want);
    }
    AdamSeg M{};
    M.p = tr->b.mlp_master;
    M.g = tr->b.mlp_grad;
    M.m = tr->b.mlp_m;
    M.v = tr->b.mlp_v;
    M.shadow = tr->b.mlp_shadow;
    M.n = fh::mlp::param_count(tr->K0);
    M.kind = 2;
    add(M, 4);
    A.nseg = k;
    A.block0[k] = blocks;
    { fh::mlp::adam_kernel<<<(unsigned)blocks, 256, 0, s>>>(A); fh::count_launch(); }
    return cuda_check(cudaGetLastError(), "adam_kernel launch");
}

// ------------------------------------------------------------ fused DP (NCCL)
// NCCL through the libnccl.so.2 torch already loaded (no link-time
// dependency; the C ABI of ncclUniqueId / enums is stable).
namespace nccl {
struct UniqueId { char internal[128]; };
typedef int (*GetUniqueId_t)(UniqueId *);
typedef int (*CommInitRank_t)(void **, int, UniqueId, int);
typedef int (*CommDestroy_t)(void *);
typedef int (*ReduceScatter_t)(const void *, void *, size_t, int, int, void *, cudaStream_t);
typedef int (*AllReduce_t)(const void *, void *, size_t, int, int, void *, cudaStream_t);
typedef int (*AllGather_t)(const void *, void *, size_t, int, void *, cudaStream_t);
typedef int (*Group_t)();
typedef const char *(*ErrStr_t)(int);
constexpr int kFloat16 = 6, kFloat32 = 7, kSum = 0;
struct Api {
    bool ok = false;
    GetUniqueId_t get_id; CommInitRank_t init; CommDestroy_t destroy;
    ReduceScatter_t reduce_scatter; AllReduce_t all_reduce; AllGather_t all_gather;
    Group_t group_start, group_end; ErrStr_t err;
};
static Api &api() {
    static Api a;
    static bool tried = false;
    if (tried) return a;
    tried = true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);
    if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.get_id = (GetUniqueId_t)dlsym(h, "ncclGetUniqueId");
    a.init = (CommInitRank_t)dlsym(h, "ncclCommInitRank");
    a.destroy = (CommDestroy_t)dlsym(h, "ncclCommDestroy");
    a.reduce_scatter = (ReduceScatter_t)dlsym(h, "ncclReduceScatter");
    a.all_reduce = (AllReduce_t)dlsym(h, "ncclAllReduce");
    a.all_gather = (AllGather_t)dlsym(h, "ncclAllGather");
    a.group_start = (Group_t)dlsym(h, "ncclGroupStart");
    a.group_end = (Group_t)dlsym(h, "ncclGroupEnd");
    a.err = (ErrStr_t)dlsym(h, "ncclGetErrorString");
    a.ok = a.get_id && a.init && a.destroy && a.reduce_scatter && a.all_reduce && a.all_gather && a.group_start &&
           a.group_end && a.err;
    return a;
}
static fh_status check(int r, const char *what) {
    if (r == 0) return FH_OK;
    return fail(FH_E_CUDA, "%s: NCCL error %d (%s)", what, r, api().err ? api().err(r) : "?");
}
}  // namespace nccl

// The partition of the table gradient (dp.overlap_plan): every range a
// backward launch finalises splits into a MAIN part [a, a + m) -- a = the
// range start rounded up to 4, m the largest multiple of 4 W that fits --
// reduce-scattered in W chunks of m / W (16-byte aligned for the vectorised
// Adam), and < 4 W + 4 TAIL elements all-reduced and updated on every rank.
static void dp_plan(fh_trainer tr, int W) {
    auto &d = tr->dp;
    d.mains.clear(); d.tb.clear(); d.te.clear();
    const int q = 4 * W;
    const int n = fh::bwd_launch_count(tr->enc);
    int64_t r[2 * 64];
    for (int li = 0; li < n; li++) {
        const int k = fh::bwd_launch_ranges(tr->enc, li, r, 64);
        for (int j = 0; j < k && j < 64; j++) {
            const int64_t b = r[2 * j], e = r[2 * j + 1];
            int64_t a = (b + 3) / 4 * 4;
            if (a > e) a = e;
            const int64_t m = (e - a) / q * q;
            if (a > b) { d.tb.push_back(b); d.te.push_back(a); }
            if (m > 0) d.mains.push_back({li, a, m});
            if (a + m < e) { d.tb.push_back(a + m); d.te.push_back(e); }
        }
    }
    d.n_tail = 0;
    for (size_t i = 0; i < d.tb.size(); i++) d.n_tail += d.te[i] - d.tb[i];
}

static size_t dp_bytes(fh_trainer tr, int W, size_t *shard_floats) {
    dp_plan(tr, W);
    size_t sf = 0;
    for (auto &m : tr->dp.mains) sf += (size_t)(m.m / W);
    if (shard_floats) *shard_floats = sf;
    const size_t P = (size_t)fh::mlp::param_count(tr->K0);
    return align_up(sf * 4, 256) + align_up(((size_t)tr->dp.n_tail + P) * 4, 256);
}

// One fused data-parallel step (fh_train_step with a communicator).
static fh_status dp_step(fh_trainer tr, const float *coords, const float *target, int64_t N, int64_t N_global,
                         float *loss_dev, fh_stream stream) {
    auto &d = tr->dp;
    auto &A = nccl::api();
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    fh_status st = fh_train_fwd_bwd(tr, coords, target, N, N_global, loss_dev, stream);
    if (st != FH_OK) return st;
    if ((st = cuda_check(cudaEventRecord(d.ev_step, s), "dp: record step")) != FH_OK) return st;
    float *g = tr->b.table_grad;
    const int W = d.W;
    // per backward launch: reduce-scatter its main parts once its gradients are final
    const int n_launch = fh::bwd_launch_count(tr->enc);
    size_t k = 0;
    float *sh = d.shard;
    for (int li = 0; li < n_launch; li++) {
        if ((st = cuda_check(cudaStreamWaitEvent(d.cs, d.ev[li], 0), "dp: wait bwd event")) != FH_OK) return st;
        if (k < d.mains.size() && d.mains[k].launch == li) {
            A.group_start();
            for (; k < d.mains.size() && d.mains[k].launch == li; k++) {
                const auto &m = d.mains[k];
                if ((st = nccl::check(A.reduce_scatter(g + m.a, sh, (size_t)(m.m / W), nccl::kFloat32, nccl::kSum,
                                                       d.comm, d.cs), "ncclReduceScatter")) != FH_OK) {
                    A.group_end();
                    return st;
                }
                sh += m.m / W;
            }
            if ((st = nccl::check(A.group_end(), "ncclGroupEnd")) != FH_OK) return st;
        }
    }
    // tails + MLP grads (the whole local step is done): all-reduce, MLP grads back
    if ((st = cuda_check(cudaStreamWaitEvent(d.cs, d.ev_step, 0), "dp: wait step")) != FH_OK) return st;
    float *t = d.tail;
    for (size_t i = 0; i < d.tb.size(); i++) {
        const int64_t n = d.te[i] - d.tb[i];
        if ((st = cuda_check(cudaMemcpyAsync(t, g + d.tb[i], (size_t)n * 4, cudaMemcpyDeviceToDevice, d.cs),
                             "dp: gather tails")) != FH_OK) return st;
        t += n;
    }
    const int64_t P = fh::mlp::param_count(tr->K0);
    if ((st = cuda_check(cudaMemcpyAsync(t, tr->b.mlp_grad, (size_t)P * 4, cudaMemcpyDeviceToDevice, d.cs),
                         "dp: mlp grads")) != FH_OK) return st;
    if ((st = nccl::check(A.all_reduce(d.tail, d.tail, (size_t)(d.n_tail + P), nccl::kFloat32, nccl::kSum, d.comm,
                                       d.cs), "ncclAllReduce")) != FH_OK) return st;
    if ((st = cuda_check(cudaMemcpyAsync(tr->b.mlp_grad, t, (size_t)P * 4, cudaMemcpyDeviceToDevice, d.cs),
                         "dp: mlp grads back")) != FH_OK) return st;
    if ((st = cuda_check(cudaEventRecord(d.ev_red, d.cs), "dp: record reduced")) != FH_OK) return st;
    if ((st = cuda_check(cudaStreamWaitEvent(s, d.ev_red, 0), "dp: wait reduced")) != FH_OK) return st;
    // ONE Adam over this rank's chunks + the tails (+ the MLP)
    std::vector<int64_t> b, e;
    std::vector<float *> gp;
    sh = d.shard;
    for (auto &m : d.mains) {
        const int64_t c = m.m / W;
        b.push_back(m.a + d.rank * c); e.push_back(m.a + (d.rank + 1) * c); gp.push_back(sh);
        sh += c;
    }
    t = d.tail;
    for (size_t i = 0; i < d.tb.size(); i++) {
        b.push_back(d.tb[i]); e.push_back(d.te[i]); gp.push_back(t);
        t += d.te[i] - d.tb[i];
    }
    if ((st = apply_ranges_impl(tr, (int)b.size(), b.data(), e.data(), gp.data(), s)) != FH_OK) return st;
    // all-gather the fp16 shadow chunks (in place) -- on the communication
    // stream too, so every NCCL call of the communicator is issued to ONE
    // stream in one order; the caller's stream waits for it
    if ((st = cuda_check(cudaEventRecord(d.ev_step, s), "dp: record adam")) != FH_OK) return st;
    if ((st = cuda_check(cudaStreamWaitEvent(d.cs, d.ev_step, 0), "dp: wait adam")) != FH_OK) return st;
    __half *shadow = reinterpret_cast<__half *>(tr->b.table_shadow);
    A.group_start();
    for (auto &m : d.mains) {
        const int64_t c = m.m / W;
        if ((st = nccl::check(A.all_gather(shadow + m.a + d.rank * c, shadow + m.a, (size_t)c, nccl::kFloat16, d.comm,
                                           d.cs), "ncclAllGather")) != FH_OK) {
            A.group_end();
            return st;
        }
    }
    if ((st = nccl::check(A.group_end(), "ncclGroupEnd")) != FH_OK) return st;
    if ((st = cuda_check(cudaEventRecord(d.ev_red, d.cs), "dp: record gathered")) != FH_OK) return st;
    return cuda_check(cudaStreamWaitEvent(s, d.ev_red, 0), "dp: wait gathered");
}

static fh_status apply_impl(fh_trainer tr, int64_t begin, int64_t end, float *tgrad, cudaStream_t s) {
    float *g[1] = {tgrad};
    return apply_ranges_impl(tr, end > begin ? 1 : 0, &begin, &end, g, s);
}

extern "C" {

fh_status fh_train_apply(fh_trainer tr, fh_stream stream) {
    g_err[0] = 0;
    if (!tr) return fail(FH_E_ARG, "fh_train_apply: NULL trainer");
    const int64_t n = (int64_t)(tr->enc->entries * (uint64_t)tr->enc->F);
    return apply_impl(tr, 0, n, tr->b.table_grad, reinterpret_cast<cudaStream_t>(stream));
}

fh_status fh_train_apply_ranges(fh_trainer tr, int n, const int64_t *begin, const int64_t *end,
                                const float *const *grad, fh_stream stream) {
    g_err[0] = 0;
    if (!tr) return fail(FH_E_ARG, "fh_train_apply_ranges: NULL trainer");
    if (n < 0 || n >= fh::mlp::kMaxAdamSeg || (n > 0 && (!begin || !end || !grad)))
        return fail(FH_E_ARG, "fh_train_apply_ranges: bad range list (n = %d, max %d)", n, fh::mlp::kMaxAdamSeg - 1);
    const int64_t nt = (int64_t)(tr->enc->entries * (uint64_t)tr->enc->F);
    for (int i = 0; i < n; i++) {
        if (begin[i] < 0 || end[i] < begin[i] || end[i] > nt)
            return fail(FH_E_ARG, "fh_train_apply_ranges: range %d [%lld, %lld) outside [0, %lld)", i,
                        (long long)begin[i], (long long)end[i], (long long)nt);
        if (end[i] > begin[i] && !grad[i]) return fail(FH_E_ARG, "fh_train_apply_ranges: NULL grad %d", i);
        for (int j = 0; j < i; j++)
            if (begin[i] < end[j] && begin[j] < end[i])
                return fail(FH_E_ARG, "fh_train_apply_ranges: ranges %d and %d overlap", j, i);
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    return apply_ranges_impl(tr, n, begin, end, const_cast<float *const *>(grad), s);
}

fh_status fh_train_apply_peers(fh_trainer tr, int W, const float *const *peer_table_grad,
                               void *const *peer_table_shadow, const float *const *peer_mlp_grad, int n,
                               const int64_t *begin, const int64_t *end, const int *broadcast, int with_mlp,
                               int new_step, fh_stream stream) {
    using fh::mlp::AdamArgs;
    using fh::mlp::AdamSeg;
    using fh::mlp::PeerArgs;
    g_err[0] = 0;
    if (!tr) return fail(FH_E_ARG, "fh_train_apply_peers: NULL trainer");
    if (W < 1 || W > fh::mlp::kMaxPeers) return fail(FH_E_ARG, "fh_train_apply_peers: W = %d not in [1, 8]", W);
    if (!tr->b.table_shadow) return fail(FH_E_STATE, "fh_train_apply_peers: needs an fp16 table shadow");
    if (n < 0 || n + (with_mlp ? 1 : 0) > fh::mlp::kMaxAdamSeg || (n > 0 && (!begin || !end || !broadcast)))
        return fail(FH_E_ARG, "fh_train_apply_peers: bad range list (n = %d)", n);
    if (!peer_table_grad || !peer_table_shadow || (with_mlp && !peer_mlp_grad))
        return fail(FH_E_ARG, "fh_train_apply_peers: NULL peer pointer table");
    for (int r = 0; r < W; r++)
        if (!peer_table_grad[r] || !peer_table_shadow[r] || (with_mlp && !peer_mlp_grad[r]))
            return fail(FH_E_ARG, "fh_train_apply_peers: NULL pointer for rank %d", r);
    const int64_t nt = (int64_t)(tr->enc->entries * (uint64_t)tr->enc->F);
    for (int i = 0; i < n; i++)
        if (begin[i] < 0 || end[i] < begin[i] || end[i] > nt)
            return fail(FH_E_ARG, "fh_train_apply_peers: range %d outside the table", i);
    if (new_step) tr->step += 1;
    if (tr->step < 1) return fail(FH_E_STATE, "fh_train_apply_peers: first call of a step must set new_step");
    const double t = (double)tr->step;
    AdamArgs A;
    PeerArgs P;
    memset(&A, 0, sizeof(A));
    memset(&P, 0, sizeof(P));
    A.lr = tr->adam.lr;
    A.b1 = tr->adam.beta1;
    A.b2 = tr->adam.beta2;
    A.eps = tr->adam.eps;
    A.omb1 = (float)(1.0 - (double)tr->adam.beta1);
    A.omb2 = (float)(1.0 - (double)tr->adam.beta2);
    A.c1 = (float)(1.0 / (1.0 - std::pow((double)tr->adam.beta1, t)));
    A.c2 = (float)(1.0 / (1.0 - std::pow((double)tr->adam.beta2, t)));
    P.W = W;
    for (int r = 0; r < W; r++) {
        P.pg[r] = peer_table_grad[r];
        P.psh[r] = reinterpret_cast<__half *>(peer_table_shadow[r]);
        P.pmg[r] = with_mlp ? peer_mlp_grad[r] : nullptr;
    }
    const int64_t cap = (int64_t)tr->n_sm * 16;
    int64_t blocks = 0;
    int k = 0;
    auto add = [&](AdamSeg g, int64_t off, int src, int bc) {
        if (g.n <= 0) return;
        int64_t want = (g.n + 256 * 4 - 1) / (256 * 4);
        if (want > cap) want = cap;
        if (want < 1) want = 1;
        A.seg[k] = g;
        P.off[k] = off;
        P.src[k] = src;
        P.bcast[k] = bc;
        A.block0[k] = blocks;
        blocks += want;
        k++;
    };
    for (int i = 0; i < n; i++) {
        AdamSeg T{};
        T.p = tr->b.table_master + begin[i];
        T.m = tr->b.table_m + begin[i];
        T.v = tr->b.table_v + begin[i];
        T.shadow = reinterpret_cast<__half *>(tr->b.table_shadow) + begin[i];
        T.n = end[i] - begin[i];
        T.kind = 1;
        add(T, begin[i], 0, broadcast[i] ? 1 : 0);
    }
    if (with_mlp) {
        AdamSeg M{};
        M.p = tr->b.mlp_master;
        M.m = tr->b.mlp_m;
        M.v = tr->b.mlp_v;
        M.shadow = tr->b.mlp_shadow;
        M.n = fh::mlp::param_count(tr->K0);
        M.kind = 2;
        add(M, 0, 1, 0);
    }
    if (k == 0) return FH_OK;
    A.nseg = k;
    A.block0[k] = blocks;
    { fh::mlp::adam_peers_kernel<<<(unsigned)blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(A, P); fh::count_launch(); }
    return cuda_check(cudaGetLastError(), "adam_peers_kernel launch");
}

fh_status fh_train_apply_multicast(fh_trainer tr, const float *mc_table_grad, void *mc_table_shadow,
                                   const float *mc_mlp_grad, int n, const int64_t *begin, const int64_t *end,
                                   const int *broadcast, int with_mlp, int new_step, fh_stream stream) {
    using fh::mlp::AdamArgs;
    using fh::mlp::AdamSeg;
    using fh::mlp::McArgs;
    g_err[0] = 0;
    if (!tr) return fail(FH_E_ARG, "fh_train_apply_multicast: NULL trainer");
    if (!tr->b.table_shadow) return fail(FH_E_STATE, "fh_train_apply_multicast: needs an fp16 table shadow");
    if (n < 0 || n + (with_mlp ? 1 : 0) > fh::mlp::kMaxAdamSeg || (n > 0 && (!begin || !end || !broadcast)))
        return fail(FH_E_ARG, "fh_train_apply_multicast: bad range list (n = %d)", n);
    if (!mc_table_grad || !mc_table_shadow || (with_mlp && !mc_mlp_grad))
        return fail(FH_E_ARG, "fh_train_apply_multicast: NULL multicast address");
    if (!aligned(mc_table_grad, 16) || !aligned(mc_table_shadow, 8) || (with_mlp && !aligned(mc_mlp_grad, 16)))
        return fail(FH_E_ARG, "fh_train_apply_multicast: misaligned multicast address");
    const int64_t nt = (int64_t)(tr->enc->entries * (uint64_t)tr->enc->F);
    for (int i = 0; i < n; i++)
        if (begin[i] < 0 || end[i] < begin[i] || end[i] > nt)
            return fail(FH_E_ARG, "fh_train_apply_multicast: range %d outside the table", i);
        else if (broadcast[i] && ((begin[i] | end[i]) & 1))
            return fail(FH_E_ARG, "fh_train_apply_multicast: broadcast range %d not in whole fp16 pairs", i);
    if (new_step) tr->step += 1;
    if (tr->step < 1) return fail(FH_E_STATE, "fh_train_apply_multicast: first call of a step must set new_step");
    const double t = (double)tr->step;
    AdamArgs A;
    McArgs M;
    memset(&A, 0, sizeof(A));
    memset(&M, 0, sizeof(M));
    A.lr = tr->adam.lr;
    A.b1 = tr->adam.beta1;
    A.b2 = tr->adam.beta2;
    A.eps = tr->adam.eps;
    A.omb1 = (float)(1.0 - (double)tr->adam.beta1);
    A.omb2 = (float)(1.0 - (double)tr->adam.beta2);
    A.c1 = (float)(1.0 / (1.0 - std::pow((double)tr->adam.beta1, t)));
    A.c2 = (float)(1.0 / (1.0 - std::pow((double)tr->adam.beta2, t)));
    M.g = mc_table_grad;
    M.sh = reinterpret_cast<__half *>(mc_table_shadow);
    M.mg = with_mlp ? mc_mlp_grad : nullptr;
    const int64_t cap = (int64_t)tr->n_sm * 16;
    int64_t blocks = 0;
    int k = 0;
    auto add = [&](AdamSeg g, int64_t off, int src, int bc) {
        if (g.n <= 0) return;
        int64_t want = (g.n + 256 * 4 - 1) / (256 * 4);
        if (want > cap) want = cap;
        if (want < 1) want = 1;
        A.seg[k] = g;
        M.off[k] = off;
        M.src[k] = src;
        M.bcast[k] = bc;
        A.block0[k] = blocks;
        blocks += want;
        k++;
    };
    for (int i = 0; i < n; i++) {
        AdamSeg T{};
        T.p = tr->b.table_master + begin[i];
        T.m = tr->b.table_m + begin[i];
        T.v = tr->b.table_v + begin[i];
        T.shadow = reinterpret_cast<__half *>(tr->b.table_shadow) + begin[i];
        T.n = end[i] - begin[i];
        T.kind = 1;
        T.vec = aligned(T.p, 16) && aligned(T.m, 16) && aligned(T.v, 16) && aligned(T.shadow, 8);
        add(T, begin[i], 0, broadcast[i] ? 1 : 0);
    }
    if (with_mlp) {
        AdamSeg Mg{};
        Mg.p = tr->b.mlp_master;
        Mg.m = tr->b.mlp_m;
        Mg.v = tr->b.mlp_v;
        Mg.shadow = tr->b.mlp_shadow;
        Mg.n = fh::mlp::param_count(tr->K0);
        Mg.kind = 2;
        Mg.vec = aligned(Mg.p, 16) && aligned(Mg.m, 16) && aligned(Mg.v, 16) && aligned(Mg.shadow, 8);
        add(Mg, 0, 1, 0);
    }
    if (k == 0) return FH_OK;
    A.nseg = k;
    A.block0[k] = blocks;
    { fh::mlp::adam_multicast_kernel<<<(unsigned)blocks, 256, 0, reinterpret_cast<cudaStream_t>(stream)>>>(A, M); fh::count_launch(); }
    return cuda_check(cudaGetLastError(), "adam_multicast_kernel launch");
}

fh_status fh_train_apply_sharded(fh_trainer tr, int64_t begin, int64_t end, const float *grad_shard,
                                 fh_stream stream) {
    g_err[0] = 0;
    if (!tr) return fail(FH_E_ARG, "fh_train_apply_sharded: NULL trainer");
    const int64_t n = (int64_t)(tr->enc->entries * (uint64_t)tr->enc->F);
    if (begin < 0 || end < begin || end > n || (begin % 4) != 0)
        return fail(FH_E_ARG, "fh_train_apply_sharded: need 0 <= begin <= end <= entries*F, begin %% 4 == 0");
    if (end > begin && (!grad_shard || !aligned(grad_shard, 16)))
        return fail(FH_E_ARG, "fh_train_apply_sharded: NULL or misaligned grad_shard");
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    return apply_impl(tr, begin, end, const_cast<float *>(grad_shard), s);
}

fh_status fh_train_step(fh_trainer tr, const float *coords, const float *target, int64_t N, int64_t N_global,
                        float *loss_dev, fh_stream stream) {
    if (tr && tr->dp.comm) return dp_step(tr, coords, target, N, N_global, loss_dev, stream);
    fh_status st = fh_train_fwd_bwd(tr, coords, target, N, N_global, loss_dev, stream);
    if (st != FH_OK) return st;
    return fh_train_apply(tr, stream);
}

fh_status fh_trainer_status(fh_trainer tr, fh_stream stream) {
    g_err[0] = 0;
    if (!tr) return fail(FH_E_ARG, "fh_trainer_status: NULL trainer");
    fh_status st = fh_status_sync(tr->enc, stream);
    if (st != FH_OK && st != FH_E_DOMAIN) return st;
    int h = 0;
    if (!tr->flags_cleared) return st == FH_E_DOMAIN ? fail(FH_E_DOMAIN, "out-of-domain coordinates") : FH_OK;
    fh_status st2 = cuda_check(cudaMemcpy(&h, tr->flag, sizeof(int), cudaMemcpyDeviceToHost), "read trainer flag");
    if (st2 != FH_OK) return st2;
    if (h & 2) {
        cudaMemset(tr->flag, 0, sizeof(int));
        return fail(FH_E_DIVERGED, "non-finite loss in the train step");
    }
    if (st == FH_E_DOMAIN) return fail(FH_E_DOMAIN, "out-of-domain or NaN coordinates were clamped to [0,1]");
    return FH_OK;
}

int64_t fh_trainer_step_count(fh_trainer tr) { return tr ? tr->step : -1; }

// Large batches over tables beyond the forward's L2 budget (the encode
// forward then runs as several L2-sized level groups, which one fused pass
// cannot: measured cfg5 shape 21.9 vs 12.6 ms at 2^24) take two launches:
// fh_encode_fwd into the workspace, then the kernel's MLP-only mode.
static bool infer_two_phase(fh_encoder enc, int64_t N) {
    const double table_bytes = (double)enc->entries * enc->F * fh::dtype_size(enc->table_dtype);
    return enc->fwd_limit > 0.0 && table_bytes > enc->fwd_limit && N >= (int64_t)enc->n_sm * fh::mlp::TILE * 8;
}

size_t fh_infer_workspace_size(fh_encoder enc, const fh_mlp_desc *m, int64_t max_batch) {
    if (!enc || !m || max_batch < 0 || !infer_two_phase(enc, max_batch)) return 0;   // fused: on chip
    return align_up((size_t)max_batch * (size_t)m->n_in * 2, 256);
}

}  // extern "C"

namespace {

// One fused inference launch (infer_kernels.cuh) for the encoder's F and
// table dtype and the MLP's K0.  The kernels' shared-memory limits are
// raised once per encoder (first call), never per call.
template <int F, typename T, int K0>
fh_status launch_infer(fh_encoder enc, const fh::infer::FusedArgs &a, cudaStream_t s) {
    using Lo = fh::infer::FusedLayout<K0>;
    constexpr int Gbig = fh::infer::Groups<F>::value;
    auto k1 = fh::infer::infer_fused_kernel<F, T, K0, 1>;      // short tiles: one gather group
    auto kG = fh::infer::infer_fused_kernel<F, T, K0, Gbig>;   // full tiles
    if (!enc->infer_ready[K0 / 16 - 1]) {
        fh_status st = cuda_check(cudaFuncSetAttribute(k1, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lo::SMEM),
                                  "cudaFuncSetAttribute(infer_fused)");
        if (st == FH_OK)
            st = cuda_check(cudaFuncSetAttribute(kG, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)Lo::SMEM),
                            "cudaFuncSetAttribute(infer_fused)");
        if (st != FH_OK) return st;
        enc->infer_ready[K0 / 16 - 1] = true;
    }
    // Tiles of R samples, one CTA per SM: the smallest power-of-two R in
    // [8, 128] that keeps every tile in one wave (each SM issues about one L2
    // request per cycle, so a small batch is spread over as many SMs as it
    // can use); large batches: R = 128 and every CTA loops over its tiles.
    // (R = 8 vs 16 vs 32 at 1024 samples: 8.25 / 8.88 / 10.3 us.)
    fh::infer::FusedArgs b = a;
    b.rows = fh::mlp::TILE;
    while (b.rows > 8 && (a.N + b.rows / 2 - 1) / (b.rows / 2) <= enc->n_sm) b.rows /= 2;
    const int64_t tiles = (a.N + b.rows - 1) / b.rows;
    const unsigned grid = (unsigned)(tiles < enc->n_sm ? tiles : enc->n_sm);
    if (b.rows < fh::mlp::TILE)
        k1<<<grid, fh::infer::Threads<1>::value, Lo::SMEM, s>>>(enc->params, b);
    else
        kG<<<grid, fh::infer::Threads<Gbig>::value, Lo::SMEM, s>>>(enc->params, b);
    fh::count_launch();
    return cuda_check(cudaGetLastError(), "infer_fused_kernel launch");
}

template <int F, typename T>
fh_status dispatch_infer_k0(fh_encoder enc, int K0, const fh::infer::FusedArgs &a, cudaStream_t s) {
    switch (K0) {
        case 16: return launch_infer<F, T, 16>(enc, a, s);
        case 32: return launch_infer<F, T, 32>(enc, a, s);
        case 48: return launch_infer<F, T, 48>(enc, a, s);
        default: return launch_infer<F, T, 64>(enc, a, s);
    }
}

template <typename T>
fh_status dispatch_infer(fh_encoder enc, int K0, const fh::infer::FusedArgs &a, cudaStream_t s) {
    switch (enc->F) {
        case 1: return dispatch_infer_k0<1, T>(enc, K0, a, s);
        case 2: return dispatch_infer_k0<2, T>(enc, K0, a, s);
        case 4: return dispatch_infer_k0<4, T>(enc, K0, a, s);
        default: return dispatch_infer_k0<8, T>(enc, K0, a, s);
    }
}

}  // namespace

extern "C" {

fh_status fh_infer(fh_encoder enc, const fh_mlp_desc *m, const void *table, const void *mlp_shadow,
                   const float *mlp_master, const float *coords, int64_t N, float *y, void *workspace,
                   size_t workspace_bytes, fh_stream stream) {
    g_err[0] = 0;
    fh_status st = check_mlp(enc, m);
    if (st != FH_OK) return st;
    if (enc->kind != 0) return fail(FH_E_ARG, "fh_infer: F-Hash encoders only");
    if (N < 0) return fail(FH_E_ARG, "fh_infer: N < 0");
    if (N == 0) return FH_OK;
    if (!coords || !aligned(coords, 16) || !table || !aligned(table, 32) || !mlp_shadow ||
        !aligned(mlp_shadow, 16) || !mlp_master || !y)
        return fail(FH_E_ARG, "fh_infer: NULL or misaligned pointer");
    if (!enc->flag) return fail(FH_E_STATE, "fh_infer: encoder was built without a CUDA device");
    fh::infer::FusedArgs a{reinterpret_cast<const float4 *>(coords), table,
                           reinterpret_cast<const __nv_bfloat16 *>(mlp_shadow), mlp_master, y, N, enc->flag,
                           fh::mlp::TILE, nullptr};
    if (infer_two_phase(enc, N)) {   // see fh_infer_workspace_size
        if (!workspace || !aligned(workspace, 16) || workspace_bytes < (size_t)N * m->n_in * 2)
            return fail(FH_E_ARG, "fh_infer: this batch needs fh_infer_workspace_size bytes of workspace");
        if ((st = fh_encode_fwd(enc, coords, N, table, workspace, FH_BF16, stream)) != FH_OK) return st;
        a.xin = reinterpret_cast<const __nv_bfloat16 *>(workspace);
    }
    cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
    return enc->table_dtype == FH_F32 ? dispatch_infer<float>(enc, m->n_in, a, s)
                                      : dispatch_infer<__half>(enc, m->n_in, a, s);
}

int64_t fh_arm_pace(int64_t n_rays, int64_t n_alive) {
    if (n_alive <= 0 || n_rays <= 0) return 0;
    int64_t p = n_rays / n_alive;
    if (p > 64) p = 64;
    return p < 1 ? 1 : p;
}

fh_status fh_nccl_unique_id(void *id128) {
    g_err[0] = 0;
    if (!id128) return fail(FH_E_ARG, "fh_nccl_unique_id: NULL id");
    auto &A = nccl::api();
    if (!A.ok) return fail(FH_E_STATE, "fh_nccl_unique_id: libnccl.so.2 not loadable");
    nccl::UniqueId id;
    fh_status st = nccl::check(A.get_id(&id), "ncclGetUniqueId");
    if (st == FH_OK) memcpy(id128, &id, sizeof(id));
    return st;
}

fh_status fh_nccl_comm_create(const void *id128, int nranks, int rank, void **comm) {
    g_err[0] = 0;
    if (!id128 || !comm) return fail(FH_E_ARG, "fh_nccl_comm_create: NULL pointer");
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(FH_E_ARG, "fh_nccl_comm_create: bad rank / nranks");
    auto &A = nccl::api();
    if (!A.ok) return fail(FH_E_STATE, "fh_nccl_comm_create: libnccl.so.2 not loadable");
    nccl::UniqueId id;
    memcpy(&id, id128, sizeof(id));
    *comm = nullptr;
    return nccl::check(A.init(comm, nranks, id, rank), "ncclCommInitRank");
}

fh_status fh_nccl_comm_destroy(void *comm) {
    g_err[0] = 0;
    if (!comm) return FH_OK;
    auto &A = nccl::api();
    if (!A.ok) return fail(FH_E_STATE, "fh_nccl_comm_destroy: libnccl.so.2 not loadable");
    return nccl::check(A.destroy(comm), "ncclCommDestroy");
}

size_t fh_trainer_dp_workspace_size(fh_trainer tr, int nranks) {
    if (!tr || nranks < 1) return 0;
    return dp_bytes(tr, nranks, nullptr);
}

fh_status fh_trainer_set_comm(fh_trainer tr, void *comm, int nranks, int rank, void *workspace, size_t bytes) {
    g_err[0] = 0;
    if (!tr) return fail(FH_E_ARG, "fh_trainer_set_comm: NULL trainer");
    auto &d = tr->dp;
    // detach (also before re-attaching): stream-ordered teardown of the old state
    if (d.cs) {
        cudaStreamSynchronize(d.cs);
        for (auto &e : d.ev) if (e) { cudaEventDestroy(e); e = nullptr; }
        if (d.ev_step) cudaEventDestroy(d.ev_step);
        if (d.ev_red) cudaEventDestroy(d.ev_red);
        cudaStreamDestroy(d.cs);
        tr->n_bwd_ev = 0;
    }
    tr->dp = fh_trainer_s::DP{};
    if (!comm) return FH_OK;
    if (nranks < 1 || rank < 0 || rank >= nranks) return fail(FH_E_ARG, "fh_trainer_set_comm: bad rank / nranks");
    if (!tr->b.table_shadow || tr->enc->table_dtype != FH_F16)
        return fail(FH_E_STATE, "fh_trainer_set_comm: the fused DP form needs an FH_F16 table (fp16 shadow)");
    size_t sf = 0;
    const size_t need = dp_bytes(tr, nranks, &sf);
    if (!workspace || bytes < need || !aligned(workspace, 256))
        return fail(FH_E_ARG, "fh_trainer_set_comm: need %zu bytes of 256-byte aligned workspace", need);
    if (d.mains.size() + d.tb.size() + 1 > (size_t)fh::mlp::kMaxAdamSeg)
        return fail(FH_E_RANGE, "fh_trainer_set_comm: %zu Adam ranges (max %d)", d.mains.size() + d.tb.size(),
                    fh::mlp::kMaxAdamSeg - 1);
    if (!nccl::api().ok) return fail(FH_E_STATE, "fh_trainer_set_comm: libnccl.so.2 not loadable");
    fh_status st = cuda_check(cudaStreamCreateWithFlags(&d.cs, cudaStreamNonBlocking), "dp: comm stream");
    if (st != FH_OK) return st;
    const int n = fh::bwd_launch_count(tr->enc);
    for (int i = 0; i < n && st == FH_OK; i++)
        st = cuda_check(cudaEventCreateWithFlags(&d.ev[i], cudaEventDisableTiming), "dp: events");
    if (st == FH_OK) st = cuda_check(cudaEventCreateWithFlags(&d.ev_step, cudaEventDisableTiming), "dp: events");
    if (st == FH_OK) st = cuda_check(cudaEventCreateWithFlags(&d.ev_red, cudaEventDisableTiming), "dp: events");
    if (st != FH_OK) return st;
    d.comm = comm;
    d.W = nranks;
    d.rank = rank;
    d.shard = reinterpret_cast<float *>(workspace);
    d.tail = reinterpret_cast<float *>(reinterpret_cast<char *>(workspace) + align_up(sf * 4, 256));
    for (int i = 0; i < n; i++) tr->bwd_ev[i] = d.ev[i];   // fh_train_fwd_bwd records them
    tr->n_bwd_ev = n;
    return FH_OK;
}

void fh_trainer_destroy(fh_trainer tr) {
    if (!tr) return;
    fh_trainer_set_comm(tr, nullptr, 1, 0, nullptr, 0);
    delete tr;
}

}  // extern "C"
