// f2c_dcp.cu -- host side of libf2c_dcp.so: the C ABI of include/f2c_dcp.h,
// argument validation, state-buffer layout, tensor maps, launch sequencing and the
// multi-rank protocol (slot-range sharding; NCCL over NVLink, or an emulated world
// on one device for testing).
#include <cuda.h>
#include <cuda_runtime.h>
#include <cudaTypedefs.h>
#include <dlfcn.h>
#include <stdarg.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <condition_variable>
#include <map>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include <nvtx3/nvToolsExt.h>  // header-only NVTX v3: ranges cost nothing without a tool attached

#include "../../include/f2c_dcp.h"
#include "dcp_main.cuh"
#include "kernels.cuh"
#include "dcp_pc4.cuh"

using namespace f2c;

// ============================================================================ errors
// NVTX range per phase of the hot path (enqueue, resolve, compaction, fused kernel, combine,
// each collective), visible in Nsight Systems / ncu --nvtx
struct NvtxRange {
    explicit NvtxRange(const char *name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

static thread_local std::string g_err;
static thread_local int g_launches = 0;

static int fail(int code, const char *fmt, ...) {
    char buf[512];
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(buf, sizeof buf, fmt, ap);
    va_end(ap);
    g_err = buf;
    return code;
}
#define CUDA_TRY(expr)                                                                       \
    do {                                                                                     \
        cudaError_t e_ = (expr);                                                             \
        if (e_ != cudaSuccess) return fail(F2C_ECUDA, "%s: %s", #expr, cudaGetErrorString(e_)); \
    } while (0)
#define LAUNCH_CHECK()                                                                       \
    do {                                                                                     \
        ++g_launches;                                                                        \
        cudaError_t e_ = cudaGetLastError();                                                 \
        if (e_ != cudaSuccess) return fail(F2C_ECUDA, "launch: %s", cudaGetErrorString(e_)); \
    } while (0)

// ============================================================================ NCCL (dlopen)
typedef struct { char internal[128]; } nccl_uid_t;
typedef void *nccl_comm_t;
enum { NCCL_INT8 = 0, NCCL_INT64 = 4, NCCL_FLOAT32 = 7, NCCL_FLOAT64 = 8 };
enum { NCCL_SUM = 0, NCCL_MAX = 2 };
struct NcclApi {
    int (*CommInitRank)(nccl_comm_t *, int, nccl_uid_t, int) = nullptr;
    int (*CommDestroy)(nccl_comm_t) = nullptr;
    int (*AllGather)(const void *, void *, size_t, int, nccl_comm_t, cudaStream_t) = nullptr;
    int (*AllReduce)(const void *, void *, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
    int (*ReduceScatter)(const void *, void *, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
    int (*GetUniqueId)(nccl_uid_t *) = nullptr;
    int (*GroupStart)() = nullptr;
    int (*GroupEnd)() = nullptr;
    int (*Send)(const void *, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
    int (*Recv)(void *, size_t, int, int, nccl_comm_t, cudaStream_t) = nullptr;
    const char *(*GetErrorString)(int) = nullptr;
    int (*CommGetAsyncError)(nccl_comm_t, int *) = nullptr;
    bool ok = false;
};
static NcclApi &nccl() {
    static NcclApi api;
    static bool tried = false;
    if (!tried) {
        tried = true;
        void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // the copy torch loaded
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (h) {
            api.CommInitRank = (decltype(api.CommInitRank))dlsym(h, "ncclCommInitRank");
            api.CommDestroy = (decltype(api.CommDestroy))dlsym(h, "ncclCommDestroy");
            api.AllGather = (decltype(api.AllGather))dlsym(h, "ncclAllGather");
            api.AllReduce = (decltype(api.AllReduce))dlsym(h, "ncclAllReduce");
            api.ReduceScatter = (decltype(api.ReduceScatter))dlsym(h, "ncclReduceScatter");
            api.GroupStart = (decltype(api.GroupStart))dlsym(h, "ncclGroupStart");
            api.GetUniqueId = (decltype(api.GetUniqueId))dlsym(h, "ncclGetUniqueId");
            api.GroupEnd = (decltype(api.GroupEnd))dlsym(h, "ncclGroupEnd");
            api.Send = (decltype(api.Send))dlsym(h, "ncclSend");
            api.Recv = (decltype(api.Recv))dlsym(h, "ncclRecv");
            api.GetErrorString = (decltype(api.GetErrorString))dlsym(h, "ncclGetErrorString");
            api.CommGetAsyncError = (decltype(api.CommGetAsyncError))dlsym(h, "ncclCommGetAsyncError");
            api.ok = api.CommInitRank && api.AllGather && api.AllReduce && api.ReduceScatter &&
                     api.GroupStart && api.GroupEnd && api.Send && api.Recv;
        }
    }
    return api;
}

// ============================================================================ layout
static inline size_t align_up(size_t v, size_t a) { return (v + a - 1) / a * a; }
static inline int64_t shard_lo(int64_t C, int W, int r) { return C * r / W; }

constexpr int G_MAX = 256;  // upper bound of the persistent grid (SM count)

// Test hook: F2C_FORCE_MULTI=1 routes a world-1 handle through the multi-rank protocol
// with a real 1-rank NCCL communicator (exercises the NCCL transport on one GPU).
static bool force_multi() {
    const char *v = getenv("F2C_FORCE_MULTI");
    return v && v[0] == '1';
}

struct Layout {
    size_t T, lab, sc, x_all, y_all, pair_all, blk_x, blk_y, inv_n, hslot, hkeys, hvals, tseq,
        comp_idx, pos_row, X_pos, row_ab, row_tgt, ttgt, seg_l, seg_mx, seg_O, rowloss, st_lse,
        st_cos, st_phi, st_ell, seg_arg, rs_buf, rs_all, dx_part, tseq_ext, dx32, tmax_glob, mu_fx, Traw, wslot,
        hgseq, row_hent, dup_cnt, dup_off, dup_list, ekeys, evals, ehslot, rseq, dst_seq, prog, ikeys, ivals, Tsh, total;
    int64_t C_loc, N, Mg, R_max, S_max;
    int H, He, HI;
};

static Layout make_layout(int64_t C, int d, int dtype, int W, int rank, int64_t n_loc, int64_t m_loc,
                          int K = 1) {
    Layout L{};
    const size_t es = dtype == F2C_BF16 ? 2 : 4;
    const int r = rank < 0 ? 0 : rank;
    L.C_loc = shard_lo(C, W, r + 1) - shard_lo(C, W, r);
    // emulated world: size for the largest shard
    if (rank < 0) L.C_loc = (C + W - 1) / W;
    L.N = n_loc * W;
    L.Mg = m_loc * W;
    // row groups of 64 (TP64), 128 (PC) or 256 (PC4); + 31 for the warp alignment of the NEXT-3
    // out-of-pool rows
    L.R_max = (L.N + 32 + 255) / 256 * 256;
    L.S_max = L.R_max / 64 + 2 * G_MAX + 1;  // units R*S <= 2G + R (tp_choose_S)
    int H = 64;
    while (H < 2 * L.N) H <<= 1;
    L.H = H;
    size_t o = 0;
    auto take = [&](size_t bytes, size_t al = 256) {
        o = align_up(o, al);
        size_t at = o;
        o += bytes;
        return at;
    };
    L.T = take(static_cast<size_t>(L.C_loc) * d * es, 1024);
    L.lab = take(static_cast<size_t>(L.C_loc) * 8);
    L.sc = take(sizeof(Scalars));
    const bool multi = W > 1 || (W == 1 && rank == 0 && force_multi());
    L.x_all = take(multi ? static_cast<size_t>(L.N) * d * es : 0);
    L.y_all = take(multi ? static_cast<size_t>(L.N) * 8 : 0);
    L.pair_all = take(multi ? static_cast<size_t>(L.N) * 4 : 0);
    L.blk_x = take(multi ? static_cast<size_t>(L.Mg) * K * d * es : 0);
    L.blk_y = take(multi ? static_cast<size_t>(L.Mg) * 8 : 0);
    L.inv_n = take(static_cast<size_t>(L.N) * 4);
    L.hslot = take(static_cast<size_t>(L.N) * 4);
    L.hkeys = take(static_cast<size_t>(H) * 8);
    L.hvals = take(static_cast<size_t>(H) * 8);
    L.tseq = take(static_cast<size_t>(L.N) * 8);
    L.comp_idx = take(static_cast<size_t>(L.N) * 4);
    L.pos_row = take(static_cast<size_t>(L.R_max) * 4);
    L.X_pos = take(static_cast<size_t>(L.R_max) * d * es, 1024);
    L.row_ab = take(static_cast<size_t>(L.R_max) * 8);
    L.row_tgt = take(static_cast<size_t>(L.R_max) * 4);
    L.ttgt = take(static_cast<size_t>(L.R_max) * 4);
    L.seg_l = take(static_cast<size_t>(L.S_max) * 128 * 4);
    L.seg_mx = take(static_cast<size_t>(L.S_max) * 128 * 4);
    L.seg_arg = take(static_cast<size_t>(L.S_max) * 128 * 4);
    L.seg_O = take(static_cast<size_t>(L.S_max) * 128 * d * 4);
    L.rowloss = take(static_cast<size_t>(L.N) * 8);
    L.st_lse = take(static_cast<size_t>(L.N) * 4);
    L.st_cos = take(static_cast<size_t>(L.N) * 4);
    L.st_phi = take(static_cast<size_t>(L.N) * 4);
    L.st_ell = take(static_cast<size_t>(L.N) * 4);
    // multi-rank exchange buffers: per global row 4 floats (C3), the packed (tseq, tmax)
    // MAX all-reduce buffer (C2), the linear dx share (C4) and its reduce-scatter output
    L.rs_buf = take(multi ? static_cast<size_t>(L.N) * 16 : 0);
    L.rs_all = take(multi ? static_cast<size_t>(W) * L.N * 16 : 0);
    L.dx_part = take(multi ? static_cast<size_t>(L.N) * d * 4 : 0);
    L.tseq_ext = take(multi ? static_cast<size_t>(L.N + 1) * 8 : 0);
    L.dx32 = take(multi ? static_cast<size_t>(n_loc) * d * 4 : 0);
    L.tmax_glob = take(64);
    L.mu_fx = take(static_cast<size_t>(d) * 8);  // this shard's pool sum mu, fixed point (k_mu_sum)
    // K >= 2: raw features [C_loc][K][d] (state) and 1/||T_bar_c|| (the T region holds T_bar)
    L.Traw = take(K > 1 ? static_cast<size_t>(L.C_loc) * K * d * es : 0, 1024);
    // (padded by one tile: the fused kernel's weight ring copies whole 128-slot tiles)
    L.wslot = take(K > 1 ? static_cast<size_t>(L.C_loc + 128) * 4 : 0);
    // NEXT-3 stale self-duplicate lists (f2c_dcp_set_dup_mode): per hash entry the target
    // write index, per compacted row its hash entry, per 128-slot tile a count / offset, and
    // at most one (slot, entry) pair per local slot
    const int64_t n_tiles = (L.C_loc + 127) / 128;
    L.hgseq = take(static_cast<size_t>(H) * 8);
    L.row_hent = take(static_cast<size_t>(L.R_max) * 4);
    L.dup_cnt = take(static_cast<size_t>(n_tiles) * 4);
    L.dup_off = take(static_cast<size_t>(n_tiles + 1) * 4);
    L.dup_list = take(static_cast<size_t>(L.C_loc) * 8);
    // NEXT-3 refresh-in-place enqueue: block-label hash, per block row the resident write
    // index (MAX all-reduce buffer for W > 1) and the planned destination (blk_seq)
    int He = 64;
    while (He < 2 * L.Mg) He <<= 1;
    L.He = He;
    L.ekeys = take(static_cast<size_t>(He) * 8);
    L.evals = take(static_cast<size_t>(He) * 8);
    L.ehslot = take(static_cast<size_t>(L.Mg) * 4);
    L.rseq = take(static_cast<size_t>(L.Mg) * 8);
    L.dst_seq = take(static_cast<size_t>(L.Mg) * 8);
    L.prog = take(static_cast<size_t>(L.S_max) * 8);  // fused kernel: per unit progress (range pacing)
    // the shard's label index (label -> newest seq, LabelIndex): >= 4 entries per slot, rebuilt by
    // the host before its keys (labels ever inserted since the last rebuild) pass half of it
    int HI = 1024;
    while (HI < 4 * L.C_loc) HI <<= 1;
    L.HI = HI;
    L.ikeys = take(static_cast<size_t>(HI) * 8);
    L.ivals = take(static_cast<size_t>(HI) * 8);
    // an fp32 pool's bf16 shadow (RNE of T, kept by the enqueue): the operand of the P x pool GEMM
    L.Tsh = take(dtype == F2C_F32 ? static_cast<size_t>(L.C_loc) * d * 2 : 0, 1024);
    L.total = align_up(o, 1024);
    return L;
}

// ============================================================================ loopback transport
// Test transport (F2C_LOOPBACK=1 at create, world > 1): the W ranks are W handles of ONE process on
// one device, each driven by its own host thread and stream, and every collective of the protocol is
// executed by device copies between the ranks' buffers, in the order NCCL requires (every rank issues
// the same sequence of collectives; point-to-point pieces match by (source, destination) order).  It
// runs the real multi-rank code path -- separate handles and state buffers, rank != 0 shards, the C5
// routing plan, the split of the reduce-scatter -- where a real communicator needs one GPU per rank.
// A batch (an NCCL group, or a single call): (1) every rank records `ready` on its stream and
// publishes its operations; barrier; (2) every rank enqueues, on its own stream, the copies and
// reductions that produce ITS outputs, after waiting on the producers' `ready`; records `done`;
// barrier; (3) every rank's stream waits on all `done` events (no rank overwrites a buffer another
// rank still reads); barrier.  Kernels never wait on each other: only streams do, through events.
struct LbOp {
    int kind;  // 0 all-gather (bytes per rank), 1 all-reduce MAX int64 (count), 2 reduce-scatter SUM fp32
               // (count per rank), 3 send (bytes, peer), 4 recv (bytes, peer)
    const void *send;
    void *recv;
    size_t n;
    int peer;
};
struct LbSlot {
    std::vector<LbOp> ops;
    cudaEvent_t ready = nullptr, done = nullptr;
};
struct LbGroup {
    int W = 0;
    std::mutex mu;
    std::condition_variable cv;
    int arrived = 0;
    long gen = 0;
    std::vector<LbSlot> slot;
    void barrier() {
        std::unique_lock<std::mutex> lk(mu);
        const long g = gen;
        if (++arrived == W) {
            arrived = 0;
            ++gen;
            cv.notify_all();
        } else {
            cv.wait(lk, [&] { return gen != g; });
        }
    }
};
static std::mutex g_lb_mu;
static std::map<std::string, std::shared_ptr<LbGroup>> g_lb_groups;

// ============================================================================ handle
struct Rank {
    int rank;
    int64_t lo, hi;
    Layout L;
    uint8_t *base;
    CUtensorMap tmT, tmX, tm3p, tm3q, tmO, tm4p;
    template <typename P>
    P *at(size_t off) const { return reinterpret_cast<P *>(base + off); }
    Scalars *sc() const { return at<Scalars>(L.sc); }
    LabelIndex ix() const { return LabelIndex{at<int64_t>(L.ikeys), at<long long>(L.ivals), L.HI}; }
    int64_t idx_keys_bound = 0;  // upper bound of the keys in the label index since its last rebuild
};

struct f2c_dcp {
    int64_t C;
    int d, dtype, W;
    int K = 1;  // features per slot (NEXT-1)
    // NEXT-3 L_cos variant (f2c_dcp_set_lcos): reduction, hinge, weight
    int phi_mode = 0, hinge = 0;
    float lam = 1.f;
    int excl_dup = 0;  // NEXT-3: exclude stale self-duplicates (f2c_dcp_set_dup_mode)
    int refresh = 0;   // NEXT-3: refresh-in-place enqueue (f2c_dcp_set_enqueue_mode)
    bool last_refresh = false;  // the last enqueue was a refresh (pairing checks use blk_seq)
    long long *n_app_host = nullptr;  // pinned: rows appended by the last refresh enqueue
    int *err_host = nullptr;          // mapped pinned {err, detail} per shard (Scalars::err_mirror)
    int neg_mode() const { return phi_mode == 2 ? 2 : (hinge ? 1 : 0); }
    bool emulated;
    int64_t n_local_max, m_local_max;
    int64_t E = 0, M_last = 0;
    int G = 148;
    std::vector<Rank> ranks;  // 1 (real rank) or W (emulated world)
    cudaStream_t last_stream = nullptr;
    nccl_comm_t comm = nullptr;
    std::shared_ptr<LbGroup> lb;   // loopback transport (tests), else null
    std::string lb_key;
    std::vector<LbOp> lb_ops;      // operations of the open batch
    int lb_grouping = 0;
    int64_t last_N = 0;
    bool multi = false;  // multi-rank protocol (world > 1, or the F2C_FORCE_MULTI test hook)
    // bench instrumentation
    bool prof = false;
    std::vector<cudaEvent_t> ev;
    size_t ev_used = 0;
    unsigned long long npos_base = 0;
    unsigned long long *dbg = nullptr;  // debug timestamps (f2c_dcp_debug_timestamps)
    bool use_tp64 = false;
    int pc4_mode = 0;               // 1: the 2-SM pair kernel where it applies (F2C_KERNEL=pc4)
    int G4 = 0;                     // co-resident 4-CTA clusters of dcp_pc4_kernel (its persistent grid / 4)
    unsigned int epoch = 0;         // fused-kernel launch tag (range pacing)
    int enq_occ = 8, enq_occ_k = 8; // resident k_enqueue / k_enqueue_k CTAs per SM (occupancy at create)
    int dbg_flags = 0;              // timing experiments (F2C_DBG_FLAGS)
    int dbg_cluster = 0;            // debug timestamps of this cluster (F2C_DBG_CLUSTER)
    ~f2c_dcp() {
        for (cudaEvent_t e : ev) cudaEventDestroy(e);
        if (lb) {
            LbSlot &sl = lb->slot[ranks[0].rank];
            if (sl.ready) cudaEventDestroy(sl.ready);
            if (sl.done) cudaEventDestroy(sl.done);
            std::lock_guard<std::mutex> g(g_lb_mu);
            if (lb.use_count() <= 2) g_lb_groups.erase(lb_key);  // (this handle and the registry)
        }
        if (n_app_host) cudaFreeHost(n_app_host);
        if (err_host) cudaFreeHost(err_host);
    }
};

// Which fused kernel a loss call runs (the combine must read the partials with the same row
// grouping): 1 = dcp_tp64_kernel (F2C_KERNEL=tp64), 2 = dcp_pc4_kernel (F2C_KERNEL=pc4: 2-SM
// pairs, 256-row groups; default variant, d % 256 == 0), 0 = dcp_pc_kernel (the default: it
// measured faster on every bench shape but one).
static int kernel_kind(const f2c_dcp *h, int64_t N) {
    (void)N;
    if (h->dtype == F2C_F32) return 0;  // (tf32 logits: dcp_pc_kernel only)
    const bool dflt = h->neg_mode() == 0 && !h->excl_dup;
    if (h->use_tp64 && dflt) return 1;
    if (dflt && h->K == 1 && h->d % 256 == 0 && h->G4 > 0 && h->pc4_mode > 0) return 2;
    return 0;
}

static int64_t occ_local(const f2c_dcp *h, const Rank &R) {
    const int64_t C_occ = h->E < h->C ? h->E : h->C;
    int64_t o = C_occ - R.lo;
    if (o > R.hi - R.lo) o = R.hi - R.lo;
    return o < 0 ? 0 : o;
}

static PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
    static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
    if (!fn) {
        void *p = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
                cudaSuccess &&
            q == cudaDriverEntryPointSuccess)
            fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
    }
    return fn;
}

static int make_tmap_bf16(CUtensorMap *m, void *ptr, int64_t rows, int d, int box_rows) {
    auto fn = encode_fn();
    if (!fn) return fail(F2C_ECUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(rows < 1 ? 1 : rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(d) * 2};
    cuuint32_t box[2] = {64, static_cast<cuuint32_t>(box_rows)};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, ptr, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(F2C_ECUDA, "cuTensorMapEncodeTiled failed (%d)", (int)r);
    return F2C_OK;
}

// The pool viewed as [d/64 chunks][rows][64] so that one box [64, 128, cps] lands in
// shared memory chunk-major: cps SW128 blocks of [128 slots x 64 d] (16 KB each).
static int make_tmap_pool3d(CUtensorMap *m, void *ptr, int64_t rows, int d, cuuint32_t cps,
                            cuuint32_t box_rows = 128) {
    auto fn = encode_fn();
    if (!fn) return fail(F2C_ECUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[3] = {64, static_cast<cuuint64_t>(rows < 1 ? 1 : rows), static_cast<cuuint64_t>(d / 64)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(d) * 2, 128};
    cuuint32_t box[3] = {64, box_rows, cps};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, ptr, dims, strides, box, es,
                    CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                    CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(F2C_ECUDA, "cuTensorMapEncodeTiled(3d) failed (%d)", (int)r);
    return F2C_OK;
}

// An fp32 pool viewed as [d/32 chunks][rows][32]: one box [32, 128, 2] lands two chunk-major SW128
// blocks of [128 slots x 32 fp32] (16 KB each) -- the tf32 producer stage (64 d columns)
static int make_tmap_pool3d_f32(CUtensorMap *m, void *ptr, int64_t rows, int d) {
    auto fn = encode_fn();
    if (!fn) return fail(F2C_ECUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[3] = {32, static_cast<cuuint64_t>(rows < 1 ? 1 : rows), static_cast<cuuint64_t>(d / 32)};
    cuuint64_t strides[2] = {static_cast<cuuint64_t>(d) * 4, 128};
    cuuint32_t box[3] = {32, 128, 2};
    cuuint32_t es[3] = {1, 1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, ptr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(F2C_ECUDA, "cuTensorMapEncodeTiled(3d f32) failed (%d)", (int)r);
    return F2C_OK;
}

// segment partials seg_O [rows][d] fp32 as a TMA-store target: box [16 fp32, 32 rows]
static int make_tmap_segO(CUtensorMap *m, void *ptr, int64_t rows, int d) {
    auto fn = encode_fn();
    if (!fn) return fail(F2C_ECUDA, "cuTensorMapEncodeTiled unavailable");
    cuuint64_t dims[2] = {static_cast<cuuint64_t>(d), static_cast<cuuint64_t>(rows)};
    cuuint64_t strides[1] = {static_cast<cuuint64_t>(d) * 4};
    cuuint32_t box[2] = {16, 32};
    cuuint32_t es[2] = {1, 1};
    CUresult r = fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, ptr, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                    CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return fail(F2C_ECUDA, "cuTensorMapEncodeTiled(seg_O) failed (%d)", (int)r);
    return F2C_OK;
}

static int check_device() {
    int dev = 0;
    CUDA_TRY(cudaGetDevice(&dev));
    cudaDeviceProp prop;
    CUDA_TRY(cudaGetDeviceProperties(&prop, dev));
    if (prop.major != 10)
        return fail(F2C_ECUDA, "device %d is sm_%d%d; this build needs sm_100 (B200)", dev,
                    prop.major, prop.minor);
    return F2C_OK;
}

static int latched(f2c_dcp *h, bool sync);

extern "C" {

const char *f2c_last_error(void) { return g_err.c_str(); }
int f2c_last_launch_count(void) { return g_launches; }

size_t f2c_dcp_state_bytes_k(int64_t C, int32_t K, int32_t d, int32_t dtype, int32_t world, int32_t rank,
                             int64_t n_local_max, int64_t m_local_max) {
    if (C < 1 || d < 128 || d % 128 || d > 512 || (dtype != F2C_BF16 && dtype != F2C_F32) ||
        world < 1 || rank < -1 || rank >= world || n_local_max < 1 || m_local_max < 1 ||
        C < world || K < 1 || K > 8 || (K > 1 && dtype != F2C_BF16))
        return 0;
    Layout L = make_layout(C, d, dtype, world, rank, n_local_max, m_local_max, K);
    return rank < 0 ? L.total * static_cast<size_t>(world) : L.total;
}

size_t f2c_dcp_state_bytes(int64_t C, int32_t d, int32_t dtype, int32_t world, int32_t rank,
                           int64_t n_local_max, int64_t m_local_max) {
    return f2c_dcp_state_bytes_k(C, 1, d, dtype, world, rank, n_local_max, m_local_max);
}

int f2c_dcp_create(int64_t C, int32_t d, int32_t dtype, int32_t world, int32_t rank,
                   const void *nccl_uid, void *state_buf, size_t state_bytes, int64_t n_local_max,
                   int64_t m_local_max, f2c_dcp **out) {
    return f2c_dcp_create_k(C, 1, d, dtype, world, rank, nccl_uid, state_buf, state_bytes, n_local_max,
                            m_local_max, out);
}

int f2c_dcp_create_k(int64_t C, int32_t K, int32_t d, int32_t dtype, int32_t world, int32_t rank,
                     const void *nccl_uid, void *state_buf, size_t state_bytes, int64_t n_local_max,
                     int64_t m_local_max, f2c_dcp **out) {
    g_launches = 0;
    if (!out) return fail(F2C_EINVAL, "out is NULL");
    *out = nullptr;
    if (C < 1 || n_local_max < 1 || m_local_max < 1)
        return fail(F2C_EINVAL, "C, n_local_max and m_local_max must be >= 1");
    if (dtype != F2C_BF16 && dtype != F2C_F32) return fail(F2C_EINVAL, "dtype must be 0 (bf16) or 1 (f32)");
    if (d < 128 || d % 128 || d > 512)
        return fail(F2C_EINVAL, "d = %d: must be a multiple of 128 and <= 512", d);
    if (world < 1 || rank < -1 || rank >= world) return fail(F2C_EINVAL, "bad world/rank");
    if (K < 1 || K > 8) return fail(F2C_EINVAL, "K = %d: must be in [1, 8]", K);
    if (K > 1 && dtype != F2C_BF16) return fail(F2C_EINVAL, "K > 1 requires bf16 features");
    if (C < world) return fail(F2C_EINVAL, "C < world");
    if (m_local_max * world > C) return fail(F2C_ECAPACITY, "world*m_local_max > C (S:276)");
    if (world > 1 && rank >= 0 && !nccl_uid) return fail(F2C_EINVAL, "nccl_uid required for world > 1");
    if ((world == 1 || rank < 0) && nccl_uid) return fail(F2C_EINVAL, "nccl_uid must be NULL");
    if (!state_buf || (reinterpret_cast<uintptr_t>(state_buf) & 255))
        return fail(F2C_EINVAL, "state_buf must be a 256-byte aligned device pointer");
    size_t need = f2c_dcp_state_bytes_k(C, K, d, dtype, world, rank, n_local_max, m_local_max);
    if (state_bytes < need) return fail(F2C_ESHAPE, "state_bytes %zu < required %zu", state_bytes, need);
    int rc = check_device();
    if (rc) return rc;

    f2c_dcp *h = new f2c_dcp();
    h->C = C; h->d = d; h->dtype = dtype; h->W = world; h->emulated = rank < 0; h->K = K;
    h->n_local_max = n_local_max; h->m_local_max = m_local_max;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&h->G, cudaDevAttrMultiProcessorCount, dev);
    if (h->G > G_MAX) h->G = G_MAX;
    if (const char *gc = getenv("F2C_CLUSTERS")) {  // timing experiments: fewer SMs
        const int n = atoi(gc);
        if (n >= 1 && 2 * n <= h->G) h->G = 2 * n;
    }
    {   // the fused kernel keeps each cluster's unit list in smem (PC_MAX_UNITS)
        const int64_t R_groups = (n_local_max * world + 32 + 127) / 128;  // (as L.R_max)
        if (2 + (R_groups + h->G / 2 - 1) / (h->G / 2) > PC_MAX_UNITS) {
            delete h;
            return fail(F2C_ECAPACITY, "world*n_local_max = %lld rows exceeds the fused kernel's schedule",
                        (long long)(n_local_max * world));
        }
    }
    const int nr = h->emulated ? world : 1;
    {   // latched device errors reach the host through mapped pinned words (no per-call copy)
        void *p = nullptr;
        if (cudaHostAlloc(&p, static_cast<size_t>(2 * nr) * sizeof(int), cudaHostAllocMapped) != cudaSuccess) {
            delete h;
            return fail(F2C_ECUDA, "cudaHostAlloc(error mirror) failed");
        }
        h->err_host = static_cast<int *>(p);
        memset(h->err_host, 0, static_cast<size_t>(2 * nr) * sizeof(int));
    }
    for (int i = 0; i < nr; ++i) {
        Rank R;
        R.rank = h->emulated ? i : rank;
        R.lo = shard_lo(C, world, R.rank);
        R.hi = shard_lo(C, world, R.rank + 1);
        R.L = make_layout(C, d, dtype, world, rank, n_local_max, m_local_max, K);
        R.base = static_cast<uint8_t *>(state_buf) + static_cast<size_t>(i) * R.L.total;
        if (cudaMemset(R.base, 0, R.L.total) != cudaSuccess) {
            delete h;
            return fail(F2C_ECUDA, "cudaMemset(state) failed");
        }
        {
            int *mirror = nullptr;
            if (cudaHostGetDevicePointer(reinterpret_cast<void **>(&mirror), h->err_host + 2 * i, 0) != cudaSuccess ||
                cudaMemcpy(&R.sc()->err_mirror, &mirror, sizeof mirror, cudaMemcpyHostToDevice) != cudaSuccess) {
                delete h;
                return fail(F2C_ECUDA, "error mirror setup failed");
            }
        }
        k_hash_clear<<<64, 256>>>(R.at<int64_t>(R.L.hkeys), R.at<unsigned long long>(R.L.hvals), R.L.H);
        k_idx_clear<<<256, 256>>>(R.ix());
        k_hash_clear<<<64, 256>>>(R.at<int64_t>(R.L.ekeys), R.at<unsigned long long>(R.L.evals), R.L.He);
        if (dtype == F2C_BF16) {
            if ((rc = make_tmap_bf16(&R.tmT, R.base + R.L.T, R.hi - R.lo, d, TP_TILE)) ||
                // producer: the logits GEMM reads the K raw rows of a slot ([C_loc][K d], NEXT-1)
                (rc = make_tmap_pool3d(&R.tm3p, R.base + (K > 1 ? R.L.Traw : R.L.T), R.hi - R.lo, K * d, 2)) ||
                (rc = make_tmap_pool3d(&R.tm3q, R.base + R.L.T, R.hi - R.lo, d, (d % 256 == 0) ? 4 : 2)) ||
                (rc = make_tmap_pool3d(&R.tm4p, R.base + R.L.T, R.hi - R.lo, d, 2, 64)) ||
                (rc = make_tmap_bf16(&R.tmX, R.base + R.L.X_pos, R.L.R_max, d, TP_R)) ||
                (rc = make_tmap_segO(&R.tmO, R.base + R.L.seg_O, R.L.S_max * 128, d))) {
                delete h;
                return rc;
            }
        } else if (d <= 256) {
            // fp32 pool: the producer reads the fp32 rows (tf32 logits), the consumer the bf16 shadow
            if ((rc = make_tmap_pool3d_f32(&R.tm3p, R.base + R.L.T, R.hi - R.lo, d)) ||
                (rc = make_tmap_pool3d(&R.tm3q, R.base + R.L.Tsh, R.hi - R.lo, d, (d % 256 == 0) ? 4 : 2)) ||
                (rc = make_tmap_segO(&R.tmO, R.base + R.L.seg_O, R.L.S_max * 128, d))) {
                delete h;
                return rc;
            }
        }
        h->ranks.push_back(R);
    }
    if (cudaDeviceSynchronize() != cudaSuccess) {
        delete h;
        return fail(F2C_ECUDA, "create: device sync failed: %s", cudaGetErrorString(cudaGetLastError()));
    }
    {
        const char *kv = getenv("F2C_KERNEL");
        h->use_tp64 = kv && strcmp(kv, "tp64") == 0 && K == 1;
        h->pc4_mode = !kv ? 0 : strcmp(kv, "pc4") == 0 ? 1 : strcmp(kv, "pc") == 0 ? -1 : 0;
        const char *fl = getenv("F2C_DBG_FLAGS");  // timing experiments only (results void)
        h->dbg_flags = fl ? atoi(fl) : 0;
        const char *fs = getenv("F2C_FORCE_S");    // timing experiments: force the range count S
        const int force_s = fs ? atoi(fs) : 0;
        cudaMemcpyToSymbol(g_force_S, &force_s, sizeof force_s);
    }
    if (cudaFuncSetAttribute(dcp_tp64_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             TP_SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(dcp_pc_kernel<false, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             PC_SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(dcp_pc_kernel<true, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             PC_SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(dcp_pc_kernel<false, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             PC_SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(dcp_pc_kernel<true, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             PC_SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(dcp_pc_kernel<false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             PC_SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(dcp_pc_kernel<true, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             PC_SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(dcp_pc_kernel<false, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             PC_SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(dcp_pc_kernel<true, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             PC_SMEM_BYTES) != cudaSuccess ||
        cudaFuncSetAttribute(dcp_pc4_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             P4_SMEM_BYTES) != cudaSuccess) {
        delete h;
        return fail(F2C_ECUDA, "cudaFuncSetAttribute(smem) failed");
    }
    {
        int occ = 0;
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_enqueue, 256, 0) == cudaSuccess && occ >= 1)
            h->enq_occ = occ;
        else
            cudaGetLastError();
        if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_enqueue_k, 256, 0) == cudaSuccess && occ >= 1)
            h->enq_occ_k = occ;
        else
            cudaGetLastError();
    }
    {   // dcp_pc_kernel's range pacing assumes every 2-CTA cluster of its persistent grid is
        // resident at once: size the grid by what the device can co-schedule (GPC floorsweeping,
        // MPS / green contexts can leave fewer than SMs / 2)
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 2;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(static_cast<unsigned>((h->G / 2) * 2));
        cfg.blockDim = dim3(PC_THREADS);
        cfg.dynamicSmemBytes = PC_SMEM_BYTES;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, dcp_pc_kernel<false, false, false>, &cfg) != cudaSuccess) {
            cudaGetLastError();
            ncl = 0;
        }
        if (ncl >= 1 && 2 * ncl < h->G) h->G = 2 * ncl;
        const int64_t R_groups = (n_local_max * world + 32 + 127) / 128;
        if (2 + (R_groups + h->G / 2 - 1) / (h->G / 2) > PC_MAX_UNITS) {
            delete h;
            return fail(F2C_ECAPACITY, "world*n_local_max = %lld rows exceeds the fused kernel's schedule on "
                        "%d co-resident clusters", (long long)(n_local_max * world), h->G / 2);
        }
        if (getenv("F2C_VERBOSE")) fprintf(stderr, "f2c: dcp_pc_kernel clusters %d (max active %d)\n", h->G / 2, ncl);
    }
    {   // 4-CTA clusters do not tile every GPC: the persistent grid is what fits at once
        cudaLaunchConfig_t cfg = {};
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = 4;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.gridDim = dim3(static_cast<unsigned>((h->G / 4) * 4));
        cfg.blockDim = dim3(P4_THREADS);
        cfg.dynamicSmemBytes = P4_SMEM_BYTES;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int ncl = 0;
        if (cudaOccupancyMaxActiveClusters(&ncl, dcp_pc4_kernel, &cfg) != cudaSuccess) {
            cudaGetLastError();
            ncl = 0;
        }
        h->G4 = ncl < h->G / 4 ? ncl : h->G / 4;
        const int64_t R4 = (n_local_max * world + 32 + 255) / 256;  // 256-row groups (as L.R_max)
        if (h->G4 > 0 && 2 + (R4 + h->G4 - 1) / h->G4 > PC_MAX_UNITS) h->G4 = 0;  // (unit list in smem)
        if (getenv("F2C_VERBOSE")) fprintf(stderr, "f2c: dcp_pc4_kernel clusters %d (of %d SMs)\n", h->G4, h->G);
    }
    h->multi = world > 1 || (rank == 0 && force_multi());
    const char *lbv = getenv("F2C_LOOPBACK");
    if (h->multi && !h->emulated && world > 1 && lbv && lbv[0] == '1') {
        // loopback test transport: join the in-process group named by the unique id's bytes
        h->lb_key.assign(static_cast<const char *>(nccl_uid), 128);
        std::lock_guard<std::mutex> g(g_lb_mu);
        auto &grp = g_lb_groups[h->lb_key];
        if (!grp) {
            grp = std::make_shared<LbGroup>();
            grp->W = world;
            grp->slot.resize(world);
        }
        if (grp->W != world) {
            delete h;
            return fail(F2C_EINVAL, "loopback group: world %d != %d", world, grp->W);
        }
        h->lb = grp;
        LbSlot &sl = grp->slot[rank];
        if (cudaEventCreateWithFlags(&sl.ready, cudaEventDisableTiming) != cudaSuccess ||
            cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming) != cudaSuccess) {
            delete h;
            return fail(F2C_ECUDA, "loopback events");
        }
    } else if (h->multi && !h->emulated) {
        NcclApi &api = nccl();
        if (!api.ok) {
            delete h;
            return fail(F2C_ENCCL, "libnccl.so.2 not loadable");
        }
        nccl_uid_t uid;
        if (nccl_uid) {
            memcpy(&uid, nccl_uid, sizeof uid);
        } else if (!api.GetUniqueId || api.GetUniqueId(&uid) != 0) {
            delete h;
            return fail(F2C_ENCCL, "ncclGetUniqueId failed");
        }
        int nr2 = api.CommInitRank(&h->comm, world, uid, rank);
        if (nr2 != 0) {
            delete h;
            return fail(F2C_ENCCL, "ncclCommInitRank: %s", api.GetErrorString ? api.GetErrorString(nr2) : "?");
        }
    }
    *out = h;
    return F2C_OK;
}

void f2c_dcp_destroy(f2c_dcp *h) {
    if (!h) return;
    if (h->comm && nccl().CommDestroy) nccl().CommDestroy(h->comm);
    delete h;
}

}  // extern "C"

// ============================================================================ comm helpers
// For world == 1 these are never called.  Emulated world: the ranks are the
// handle's Rank entries, collectives are device-to-device copies / reductions.
static int nccl_check(int r, const char *what) {
    if (r != 0)
        return fail(F2C_ENCCL, "%s: %s", what, nccl().GetErrorString ? nccl().GetErrorString(r) : "?");
    return F2C_OK;
}

// The protocol's collectives through NCCL or the loopback transport.  comm_group_start / _end
// bracket a batch (an NCCL group); outside a bracket every call is a batch of its own.
static unsigned grid_for(int64_t n);
static int lb_flush(f2c_dcp *h, cudaStream_t st, const char *what) {
    LbGroup &G = *h->lb;
    const int me = h->ranks[0].rank;
    LbSlot &mine = G.slot[me];
    mine.ops = h->lb_ops;
    h->lb_ops.clear();
    CUDA_TRY(cudaEventRecord(mine.ready, st));
    G.barrier();
    // phase 2: this rank's outputs
    std::vector<int> sent_seen(G.W, 0);  // per source: matched sends to me so far
    for (size_t k = 0; k < mine.ops.size(); ++k) {
        const LbOp &o = mine.ops[k];
        if (o.kind == 0) {
            for (int q = 0; q < G.W; ++q) {
                const LbOp &oq = G.slot[q].ops[k];
                if (oq.kind != 0 || oq.n != o.n) return fail(F2C_ENCCL, "%s: loopback all-gather mismatch", what);
                CUDA_TRY(cudaStreamWaitEvent(st, G.slot[q].ready, 0));
                CUDA_TRY(cudaMemcpyAsync(static_cast<uint8_t *>(o.recv) + q * o.n, oq.send, o.n, cudaMemcpyDeviceToDevice, st));
            }
        } else if (o.kind == 1) {
            // MAX into my buffer from every peer's (a peer's buffer read while it is being maxed itself
            // still holds values between its own and the global maximum: the result is the same)
            for (int q = 0; q < G.W; ++q) {
                if (q == me) continue;
                const LbOp &oq = G.slot[q].ops[k];
                if (oq.kind != 1 || oq.n != o.n) return fail(F2C_ENCCL, "%s: loopback all-reduce mismatch", what);
                CUDA_TRY(cudaStreamWaitEvent(st, G.slot[q].ready, 0));
                k_max_i64_into<<<grid_for(static_cast<int64_t>(o.n)), 256, 0, st>>>(
                    static_cast<int64_t *>(o.recv), static_cast<const int64_t *>(oq.send), static_cast<int64_t>(o.n));
                LAUNCH_CHECK();
            }
        } else if (o.kind == 2) {
            // my chunk: sum over ranks in rank order
            for (int q = 0; q < G.W; ++q) {
                const LbOp &oq = G.slot[q].ops[k];
                if (oq.kind != 2 || oq.n != o.n) return fail(F2C_ENCCL, "%s: loopback reduce-scatter mismatch", what);
                CUDA_TRY(cudaStreamWaitEvent(st, G.slot[q].ready, 0));
                const float *src = static_cast<const float *>(oq.send) + static_cast<size_t>(me) * o.n;
                if (q == 0) {
                    CUDA_TRY(cudaMemcpyAsync(o.recv, src, o.n * 4, cudaMemcpyDeviceToDevice, st));
                } else {
                    k_add_f32_into<<<grid_for(static_cast<int64_t>(o.n)), 256, 0, st>>>(static_cast<float *>(o.recv), src,
                                                                                      static_cast<int64_t>(o.n));
                    LAUNCH_CHECK();
                }
            }
        } else if (o.kind == 4) {
            // the n-th receive from q matches q's n-th send to me
            const int q = o.peer;
            int seen = 0;
            const LbOp *match = nullptr;
            for (const LbOp &oq : G.slot[q].ops)
                if (oq.kind == 3 && oq.peer == me && seen++ == sent_seen[q]) {
                    match = &oq;
                    break;
                }
            if (!match || match->n != o.n) return fail(F2C_ENCCL, "%s: loopback send/recv mismatch", what);
            ++sent_seen[q];
            CUDA_TRY(cudaStreamWaitEvent(st, G.slot[q].ready, 0));
            CUDA_TRY(cudaMemcpyAsync(o.recv, match->send, o.n, cudaMemcpyDeviceToDevice, st));
        }
    }
    CUDA_TRY(cudaEventRecord(mine.done, st));
    G.barrier();
    for (int q = 0; q < G.W; ++q)
        if (q != me) CUDA_TRY(cudaStreamWaitEvent(st, G.slot[q].done, 0));
    G.barrier();  // (nobody re-records its events before every peer has waited on them)
    return F2C_OK;
}
static void comm_group_start(f2c_dcp *h) {
    if (h->lb) ++h->lb_grouping;
    else nccl().GroupStart();
}
static int comm_group_end(f2c_dcp *h, cudaStream_t st, const char *what) {
    if (h->lb) return --h->lb_grouping == 0 ? lb_flush(h, st, what) : F2C_OK;
    return nccl_check(nccl().GroupEnd(), what);
}
static int lb_add(f2c_dcp *h, LbOp o, cudaStream_t st, const char *what) {
    h->lb_ops.push_back(o);
    return h->lb_grouping ? F2C_OK : lb_flush(h, st, what);
}
static int comm_allgather(f2c_dcp *h, const void *send, void *recv, size_t bytes, cudaStream_t st, const char *what) {
    if (h->lb) return lb_add(h, LbOp{0, send, recv, bytes, -1}, st, what);
    return nccl_check(nccl().AllGather(send, recv, bytes, NCCL_INT8, h->comm, st), what);
}
static int comm_allreduce_max_i64(f2c_dcp *h, int64_t *buf, size_t count, cudaStream_t st, const char *what) {
    if (h->lb) return lb_add(h, LbOp{1, buf, buf, count, -1}, st, what);
    return nccl_check(nccl().AllReduce(buf, buf, count, NCCL_INT64, NCCL_MAX, h->comm, st), what);
}
static int comm_reduce_scatter_f32(f2c_dcp *h, const float *send, float *recv, size_t count, cudaStream_t st,
                                   const char *what) {
    if (h->lb) return lb_add(h, LbOp{2, send, recv, count, -1}, st, what);
    return nccl_check(nccl().ReduceScatter(send, recv, count, NCCL_FLOAT32, NCCL_SUM, h->comm, st), what);
}
static int comm_send(f2c_dcp *h, const void *p, size_t bytes, int peer, cudaStream_t st, const char *what) {
    if (h->lb) return lb_add(h, LbOp{3, p, nullptr, bytes, peer}, st, what);
    return nccl_check(nccl().Send(p, bytes, NCCL_INT8, peer, h->comm, st), what);
}
static int comm_recv(f2c_dcp *h, void *p, size_t bytes, int peer, cudaStream_t st, const char *what) {
    if (h->lb) return lb_add(h, LbOp{4, nullptr, p, bytes, peer}, st, what);
    return nccl_check(nccl().Recv(p, bytes, NCCL_INT8, peer, h->comm, st), what);
}

// ============================================================================ label index
// Rebuild the shard's label index from its occupied slots (clear + one pass over the labels).
static int idx_rebuild(f2c_dcp *h, Rank &R, cudaStream_t st) {
    k_idx_clear<<<static_cast<unsigned>(R.L.HI / 256 < 4096 ? (R.L.HI + 255) / 256 : 4096), 256, 0, st>>>(R.ix());
    LAUNCH_CHECK();
    const int64_t occ = occ_local(h, R);
    if (occ > 0) {
        int64_t blocks = (occ + 255) / 256;
        if (blocks > h->G * 16) blocks = h->G * 16;
        k_idx_build<<<static_cast<unsigned>(blocks), 256, 0, st>>>(R.ix(), R.at<int64_t>(R.L.lab), occ, R.lo, h->C, h->E);
        LAUNCH_CHECK();
    }
    R.idx_keys_bound = occ;
    return F2C_OK;
}

// ============================================================================ C5 routing
static int shard_of(int64_t p, int64_t C, int W) {
    int q = static_cast<int>((p * W) / C);
    while (q + 1 < W && p >= shard_lo(C, W, q + 1)) ++q;
    while (q > 0 && p < shard_lo(C, W, q)) --q;
    return q;
}

extern "C" int64_t f2c_c5_plan(int64_t C, int32_t world, int64_t E, int64_t m_local, int64_t *pieces,
                               int64_t max_pieces) {
    if (C < 1 || world < 1 || C < world || E < 0 || m_local < 1 || m_local * world > C || !pieces) return -1;
    int64_t n = 0;
    for (int r = 0; r < world; ++r) {
        int64_t j = r * m_local;
        const int64_t end = j + m_local;
        while (j < end) {
            const int64_t p = (E + j) % C;
            const int q = shard_of(p, C, world);
            int64_t len = end - j;
            const int64_t to_shard_end = shard_lo(C, world, q + 1) - p;  // (the ring wraps at C = lo(W))
            if (len > to_shard_end) len = to_shard_end;
            if (n >= max_pieces) return -1;
            pieces[4 * n] = r;
            pieces[4 * n + 1] = q;
            pieces[4 * n + 2] = j;
            pieces[4 * n + 3] = len;
            ++n;
            j += len;
        }
    }
    return n;
}

// ============================================================================ enqueue
// NEXT-3 refresh-in-place (reading R7), part 1 on every shard: block-label hash, scan of the
// shard's labels -> rseq[j] = newest local write index of label y_j or -1
static int refresh_resolve(f2c_dcp *h, Rank &R, const int64_t *y, int64_t m_glob, cudaStream_t st) {
    const Layout &L = R.L;
    k_blk_insert<<<static_cast<unsigned>((m_glob + 255) / 256), 256, 0, st>>>(y, m_glob, R.at<int64_t>(L.ekeys), L.He,
                                                                             R.at<int>(L.ehslot), R.sc());
    LAUNCH_CHECK();
    // sigma_j = newest local write index of y_j, from the label index (one lookup per block row)
    k_idx_lookup<<<static_cast<unsigned>((m_glob + 255) / 256), 256, 0, st>>>(R.ix(), y, m_glob, R.at<int64_t>(L.rseq));
    LAUNCH_CHECK();
    return F2C_OK;
}

// part 2 (after the global MAX of rseq): destinations, identical on every shard
static int refresh_plan(f2c_dcp *h, Rank &R, int64_t m_glob, cudaStream_t st) {
    const Layout &L = R.L;
    k_refresh_plan<<<1, 1024, 0, st>>>(R.at<int64_t>(L.rseq), m_glob, h->E, h->C, R.at<int64_t>(L.dst_seq), R.sc(),
                                       R.at<int64_t>(L.ekeys), R.at<unsigned long long>(L.evals), L.He);
    LAUNCH_CHECK();
    return F2C_OK;
}

static int enqueue_rank(f2c_dcp *h, Rank &R, const uint8_t *g, const int64_t *y, int64_t m_glob,
                        cudaStream_t st) {
    int rc;
    if (R.idx_keys_bound + m_glob > R.L.HI / 2 && (rc = idx_rebuild(h, R, st))) return rc;
    R.idx_keys_bound += m_glob;  // (at most one new key per row that lands in this shard)
    // (timing experiment only, results void: F2C_DBG_FLAGS bit 1 << 20 skips the label index update)
    const LabelIndex ixe = (h->dbg_flags & (1 << 20)) ? LabelIndex{nullptr, nullptr, 0} : R.ix();
    if (h->K > 1) {
        int64_t blocks = (m_glob + 7) / 8;
        if (blocks > static_cast<int64_t>(h->G) * h->enq_occ_k) blocks = static_cast<int64_t>(h->G) * h->enq_occ_k;
        k_enqueue_k<<<static_cast<unsigned>(blocks), 256, 0, st>>>(
            reinterpret_cast<const __nv_bfloat16 *>(g), y, m_glob, h->K, h->d, h->E, h->C, R.lo, R.hi,
            R.at<__nv_bfloat16>(R.L.Traw), R.at<__nv_bfloat16>(R.L.T), R.at<float>(R.L.wslot),
            R.at<int64_t>(R.L.lab), R.sc(), h->refresh ? R.at<int64_t>(R.L.dst_seq) : nullptr,
            R.at<unsigned long long>(R.L.mu_fx), h->E < h->C ? h->E : h->C, ixe);
        LAUNCH_CHECK();
        return F2C_OK;
    }
    const int row_bytes = h->d * (h->dtype == F2C_BF16 ? 2 : 4);
    int64_t blocks = (m_glob + 7) / 8;                 // 8 rows (warps) per block per pass
    // one wave of resident CTAs (grid-stride over the rows): more CTAs only queue behind the first
    // wave and leave a tail
    if (blocks > static_cast<int64_t>(h->G) * h->enq_occ) blocks = static_cast<int64_t>(h->G) * h->enq_occ;
    k_enqueue<<<static_cast<unsigned>(blocks), 256, 0, st>>>(
        g, y, m_glob, h->E, h->C, R.lo, R.hi, row_bytes, h->dtype, R.base + R.L.T,
        R.at<int64_t>(R.L.lab), R.sc(), h->refresh ? R.at<int64_t>(R.L.dst_seq) : nullptr,
        R.at<unsigned long long>(R.L.mu_fx), ixe, h->dtype == F2C_F32 ? R.at<__nv_bfloat16>(R.L.Tsh) : nullptr);
    LAUNCH_CHECK();
    return F2C_OK;
}

extern "C" int f2c_dcp_enqueue(f2c_dcp *h, const void *g_feats, const int64_t *labels,
                               int64_t m_local, void *stream) {
    NvtxRange nv("f2c_dcp_enqueue (a1)");
    g_launches = 0;
    if (!h) return fail(F2C_EINVAL, "NULL handle");
    if (!g_feats || !labels) return fail(F2C_EINVAL, "NULL g_feats/labels");
    if (m_local < 1 || m_local > h->m_local_max)
        return fail(F2C_ESHAPE, "m_local %lld not in [1, %lld]", (long long)m_local, (long long)h->m_local_max);
    const int64_t m_glob = m_local * h->W;
    if (m_glob > h->C) return fail(F2C_ECAPACITY, "block of %lld rows > C (S:276)", (long long)m_glob);
    if (reinterpret_cast<uintptr_t>(g_feats) & 15) return fail(F2C_EINVAL, "g_feats must be 16-byte aligned");
    int rc = latched(h, false);
    if (rc) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    h->last_stream = st;
    const size_t es = h->dtype == F2C_BF16 ? 2 : 4;
    const uint8_t *gx = static_cast<const uint8_t *>(g_feats);
    const int64_t *gy = labels;
    if (h->multi && !h->emulated && !h->refresh) {
        // C5: route every block row to the rank that owns its slot (E + j) mod C: grouped
        // ncclSend / ncclRecv of the pieces of f2c_c5_plan into the owner's staging rows (the
        // enqueue kernel still needs each overwritten slot's old row and label, so the receive
        // cannot land in the pool itself); a rank's own rows are a device copy.  Each rank receives
        // exactly the rows it owns (the block's slots span one or two shards).
        NvtxRange nvc("f2c: C5 enqueue routed to the owners");
        Rank &R = h->ranks[0];
        const int me = R.rank;
        const size_t rb = static_cast<size_t>(h->K) * h->d * es;
        std::vector<int64_t> pc(4 * (2 * static_cast<size_t>(h->W) + 2));
        const int64_t np = f2c_c5_plan(h->C, h->W, h->E, m_local, pc.data(), static_cast<int64_t>(pc.size() / 4));
        if (np < 0) return fail(F2C_EINVAL, "C5 plan failed");
        uint8_t *bx = R.base + R.L.blk_x;
        int64_t *by = R.at<int64_t>(R.L.blk_y);
        const uint8_t *gsrc = static_cast<const uint8_t *>(g_feats);
        for (int64_t i = 0; i < np; ++i) {  // own rows: device copies
            const int64_t src = pc[4 * i], dst = pc[4 * i + 1], j = pc[4 * i + 2], len = pc[4 * i + 3];
            if (src != me || dst != me) continue;
            CUDA_TRY(cudaMemcpyAsync(bx + j * rb, gsrc + (j - me * m_local) * rb, len * rb, cudaMemcpyDeviceToDevice, st));
            CUDA_TRY(cudaMemcpyAsync(by + j, labels + (j - me * m_local), len * 8, cudaMemcpyDeviceToDevice, st));
        }
        comm_group_start(h);
        for (int64_t i = 0; i < np; ++i) {
            const int64_t src = pc[4 * i], dst = pc[4 * i + 1], j = pc[4 * i + 2], len = pc[4 * i + 3];
            if (src == dst) continue;
            if (src == me) {
                comm_send(h, gsrc + (j - me * m_local) * rb, len * rb, static_cast<int>(dst), st, "C5");
                comm_send(h, labels + (j - me * m_local), len * 8, static_cast<int>(dst), st, "C5");
            } else if (dst == me) {
                comm_recv(h, bx + j * rb, len * rb, static_cast<int>(src), st, "C5");
                comm_recv(h, by + j, len * 8, static_cast<int>(src), st, "C5");
            }
        }
        if ((rc = comm_group_end(h, st, "C5 send/recv"))) return rc;
        gx = bx;
        gy = by;
    } else if (h->multi && !h->emulated) {
        // refresh-in-place (NEXT-3, R7): destinations depend on residency over all shards, so
        // every rank receives the whole block (all-gather) and keeps the rows its plan assigns it
        Rank &R = h->ranks[0];
        comm_group_start(h);
        comm_allgather(h, g_feats, R.base + R.L.blk_x, m_local * h->K * h->d * es, st, "enqueue all-gather");
        comm_allgather(h, labels, R.base + R.L.blk_y, m_local * 8, st, "enqueue all-gather");
        if ((rc = comm_group_end(h, st, "enqueue all-gather"))) return rc;
        gx = R.base + R.L.blk_x;
        gy = R.at<int64_t>(R.L.blk_y);
    }
    // (emulated world: g_feats / labels already hold the rank-ordered global block)
    if (h->refresh) {
        // NEXT-3 refresh-in-place: residency over all shards (MAX of the newest write index),
        // then the same plan on every shard
        for (Rank &R : h->ranks)
            if ((rc = refresh_resolve(h, R, gy, m_glob, st))) return rc;
        if (h->emulated) {
            Rank &R0 = h->ranks[0];
            for (size_t q = 1; q < h->ranks.size(); ++q) {
                k_max_i64_into<<<static_cast<unsigned>((m_glob + 255) / 256), 256, 0, st>>>(
                    R0.at<int64_t>(R0.L.rseq), h->ranks[q].at<int64_t>(h->ranks[q].L.rseq), m_glob);
                LAUNCH_CHECK();
            }
            for (size_t q = 1; q < h->ranks.size(); ++q)
                CUDA_TRY(cudaMemcpyAsync(h->ranks[q].at<int64_t>(h->ranks[q].L.rseq), R0.at<int64_t>(R0.L.rseq),
                                         m_glob * 8, cudaMemcpyDeviceToDevice, st));
        } else if (h->multi) {
            Rank &R = h->ranks[0];
            if ((rc = comm_allreduce_max_i64(h, R.at<int64_t>(R.L.rseq), m_glob, st, "refresh all-reduce"))) return rc;
        }
        for (Rank &R : h->ranks)
            if ((rc = refresh_plan(h, R, m_glob, st))) return rc;
    }
    for (Rank &R : h->ranks)
        if ((rc = enqueue_rank(h, R, gx, gy, m_glob, st))) return rc;
    if (h->refresh) {
        // the number of appended rows is data-dependent: the host's E waits for it
        CUDA_TRY(cudaMemcpyAsync(h->n_app_host, &h->ranks[0].sc()->n_app, sizeof(long long), cudaMemcpyDeviceToHost, st));
        CUDA_TRY(cudaStreamSynchronize(st));
        h->E += *h->n_app_host;
    } else {
        h->E += m_glob;
    }
    h->last_refresh = h->refresh != 0;
    h->M_last = m_glob;
    return F2C_OK;
}

// ============================================================================ EMA
extern "C" int f2c_gnet_ema(const float *p, float *g, int64_t n, double momentum, void *stream) {
    NvtxRange nv("f2c_gnet_ema (a10)");
    g_launches = 0;
    if (n < 0) return fail(F2C_ESHAPE, "n < 0");
    if (!(momentum >= 0.0 && momentum <= 1.0)) return fail(F2C_EINVAL, "momentum must be in [0, 1]");
    if (n == 0) return F2C_OK;
    if (!p || !g) return fail(F2C_EINVAL, "NULL p/g");
    if ((reinterpret_cast<uintptr_t>(p) | reinterpret_cast<uintptr_t>(g)) & 15)
        return fail(F2C_EINVAL, "p and g must be 16-byte aligned");
    if ((p < g + n) && (g < p + n)) return fail(F2C_EINVAL, "p and g overlap");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const int64_t n4 = n / 4;
    if (n4 > 0) {
        const int64_t blocks = (n4 + EMA_THREADS * EMA_PER_THREAD - 1) / (EMA_THREADS * EMA_PER_THREAD);
        if (blocks > 0x7fffffffll) return fail(F2C_ESHAPE, "n too large");
        k_ema<<<static_cast<unsigned>(blocks), EMA_THREADS, 0, st>>>(reinterpret_cast<const float4 *>(p),
                                                             reinterpret_cast<float4 *>(g), n4,
                                                             momentum, 1.0 - momentum);
        LAUNCH_CHECK();
    }
    if (n4 * 4 < n) {
        k_ema_tail<<<1, 32, 0, st>>>(p, g, n4 * 4, n, momentum, 1.0 - momentum);
        LAUNCH_CHECK();
    }
    return F2C_OK;
}

// ============================================================================ loss
struct StepCtx {
    int64_t N;         // global batch rows
    float s, m;
    const uint8_t *x;  // global batch rows on this rank (W == 1: the input)
    const int64_t *y;
    const int32_t *pair;
    cudaStream_t st;
};


// a2 + a3: norms, batch-label hash (the stale-duplicate lists of NEXT-3 use it) and the local
// target resolve from the shard's label index: tseq = newest local seq of the row's label or -1
static int phase_resolve(f2c_dcp *h, Rank &R, const StepCtx &c) {
    NvtxRange nv("f2c: a2+a3 norms, label index lookup");
    const Layout &L = R.L;
    const unsigned rows_blocks = static_cast<unsigned>((c.N * 32 + 255) / 256);
    if (h->dtype == F2C_BF16)
        k_rownorm_insert<__nv_bfloat16><<<rows_blocks, 256, 0, c.st>>>(
            reinterpret_cast<const __nv_bfloat16 *>(c.x), c.y, c.N, h->d, R.at<float>(L.inv_n),
            R.at<int64_t>(L.hkeys), L.H, R.at<int>(L.hslot), R.sc(), R.ix(), R.at<int64_t>(L.tseq));
    else
        k_rownorm_insert<float><<<rows_blocks, 256, 0, c.st>>>(
            reinterpret_cast<const float *>(c.x), c.y, c.N, h->d, R.at<float>(L.inv_n),
            R.at<int64_t>(L.hkeys), L.H, R.at<int>(L.hslot), R.sc(), R.ix(), R.at<int64_t>(L.tseq));
    LAUNCH_CHECK();
    return F2C_OK;
}

// a3 split + compaction + gather
static int phase_compact(f2c_dcp *h, Rank &R, const StepCtx &c, const int *tmax_bits) {
    NvtxRange nv("f2c: a3 split + compaction + gather");
    const Layout &L = R.L;
    CompactArgs a;
    a.tseq = R.at<int64_t>(L.tseq);
    a.inv_n = R.at<float>(L.inv_n);
    a.pairing = c.pair;
    a.N = c.N; a.C = h->C; a.lo = R.lo; a.hi = R.hi; a.E = h->E; a.M_last = h->M_last;
    a.s = c.s;
    a.log2e_s = c.s * 1.4426950408889634f;
    a.a_scale = 1.0f / static_cast<float>(h->K);
    a.ref_scale = a.log2e_s * (1.0f + 1.0f / 1024.0f);
    a.R_max = static_cast<int>(L.R_max);
    a.comp_idx = R.at<int>(L.comp_idx);
    a.pos_row = R.at<int>(L.pos_row);
    a.row_ab = R.at<float2>(L.row_ab);
    a.row_tgt = R.at<int>(L.row_tgt);
    a.ttgt = R.at<float>(L.ttgt);
    a.sc = R.sc();
    a.tmax_bits = tmax_bits;
    a.neg_mode = h->neg_mode();
    a.blk_seq = h->last_refresh ? R.at<int64_t>(L.dst_seq) : nullptr;
    a.excl = h->excl_dup;
    a.hslot = R.at<int>(L.hslot);
    a.row_hent = R.at<int>(L.row_hent);
    a.hgseq = R.at<int64_t>(L.hgseq);
    {
        const int64_t occ_t = occ_local(h, R);
        // the fused kernel's range count S (dcp_pc_kernel; dcp_pc4_kernel with its 256-row groups)
        const int kind = kernel_kind(h, c.N);
        a.G_pc = kind == 0 ? h->G / 2 : kind == 2 ? h->G4 : 0;
        a.rg_pc = kind == 2 ? P4_RG : PC_R;
        a.seg_cap = static_cast<int>(L.S_max * 128 / a.rg_pc);
        a.n_tiles_pc = static_cast<int>((occ_t + PC_TILE - 1) / PC_TILE);
    }
    k_compact<<<static_cast<unsigned>((c.N + 1023) / 1024), 1024, 0, c.st>>>(a);
    LAUNCH_CHECK();
    const int64_t occ = occ_local(h, R);
    if (h->excl_dup && occ > 0) {  // NEXT-3: per-tile lists of the shard's stale self-duplicates
        const int n_tiles = static_cast<int>((occ + 127) / 128);
        int64_t blocks = (occ + 255) / 256;
        if (blocks > h->G * 16) blocks = h->G * 16;
        CUDA_TRY(cudaMemsetAsync(R.at<int>(L.dup_cnt), 0, static_cast<size_t>(n_tiles) * 4, c.st));
        k_dup_count<<<static_cast<unsigned>(blocks), 256, 0, c.st>>>(
            R.at<int64_t>(L.lab), occ, R.lo, h->C, h->E, R.at<int64_t>(L.hkeys), L.H, R.at<int64_t>(L.hgseq),
            R.at<int>(L.dup_cnt));
        LAUNCH_CHECK();
        k_dup_scan<<<1, 1024, 0, c.st>>>(R.at<int>(L.dup_cnt), R.at<int>(L.dup_off), n_tiles);
        LAUNCH_CHECK();
        k_dup_fill<<<static_cast<unsigned>(blocks), 256, 0, c.st>>>(
            R.at<int64_t>(L.lab), occ, R.lo, h->C, h->E, R.at<int64_t>(L.hkeys), L.H, R.at<int64_t>(L.hgseq),
            R.at<int>(L.dup_cnt), R.at<int>(L.dup_off), R.at<int2>(L.dup_list));
        LAUNCH_CHECK();
    }
    const int row_bytes = h->d * (h->dtype == F2C_BF16 ? 2 : 4);
    k_gather<<<static_cast<unsigned>(L.R_max / 8), 256, 0, c.st>>>(c.x, R.at<int>(L.pos_row), R.sc(), row_bytes,
                                                          R.base + L.X_pos, R.base + L.T, R.at<int>(L.row_tgt),
                                                          R.at<float2>(L.row_ab), static_cast<float>(h->K),
                                                          h->dtype == F2C_F32 ? 1 : 0);
    LAUNCH_CHECK();
    return F2C_OK;
}

static int phase_main(f2c_dcp *h, Rank &R, const StepCtx &c, int64_t occ_loc, const int *run_flag = nullptr) {
    NvtxRange nv("f2c: a4-a9 fused loss kernel");
    const Layout &L = R.L;
    TPParams p;
    p.d = h->d;
    p.n_slots = static_cast<int>(occ_loc);
    p.n_pos = &R.sc()->n_pos;
    p.row_ab = R.at<float2>(L.row_ab);
    p.row_tgt = R.at<int>(L.row_tgt);
    p.margin_l2 = c.s * c.m * 1.4426950408889634f;
    p.ttgt = R.at<float>(L.ttgt);
    p.seg_l = R.at<float>(L.seg_l);
    p.seg_mx = R.at<float>(L.seg_mx);
    p.seg_O = R.at<float>(L.seg_O);
    p.dbg = h->dbg;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (h->prof) {
        while (h->ev.size() < h->ev_used + 2) {
            cudaEvent_t e;
            CUDA_TRY(cudaEventCreate(&e));
            h->ev.push_back(e);
        }
        e0 = h->ev[h->ev_used];
        e1 = h->ev[h->ev_used + 1];
        h->ev_used += 2;
        CUDA_TRY(cudaEventRecord(e0, c.st));
    }
    const int kind = kernel_kind(h, c.N);
    if (kind == 1) {
        dcp_tp64_kernel<<<h->G, TP_THREADS, TP_SMEM_BYTES, c.st>>>(R.tmT, R.tmX, p);
    } else {
        PCParams q;
        q.d = p.d;
        q.n_slots = p.n_slots;
        q.n_pos = p.n_pos;
        q.n_rows = &R.sc()->n_rows;
        q.neg0 = &R.sc()->neg0;
        q.neg_mode = h->neg_mode();
        q.seg_arg = R.at<int>(L.seg_arg);
        q.row_ab = p.row_ab;
        q.row_tgt = p.row_tgt;
        q.X_pos = R.base + L.X_pos;
        q.wslot = h->K > 1 ? R.at<float>(L.wslot) : nullptr;
        q.kf = h->K;
        q.S_sched = &R.sc()->S_sched;
        q.margin_l2 = p.margin_l2;
        q.ttgt = p.ttgt;
        q.seg_l = p.seg_l;
        q.seg_mx = p.seg_mx;
        q.seg_O = p.seg_O;
        // short units (small pools): stage the O drain through smem + TMA stores, so the next
        // unit's GEMM 2 waits less; long units keep the direct drain and the smaller smem
        // footprint (measured: c1 +4-7 %, c2/c3 -1 % with staging)
        q.drain_tma = (p.n_slots + PC_TILE - 1) / PC_TILE <= 2048;
        const int smem = q.drain_tma ? PC_SMEM_BYTES : PC_SMEM_BYTES_NOSTG;
        q.excl = h->excl_dup;
        q.dup_off = R.at<int>(L.dup_off);
        q.dup_list = R.at<int2>(L.dup_list);
        q.row_hent = R.at<int>(L.row_hent);
        q.dbg = p.dbg;
        q.dbg_cluster = h->dbg_cluster;
        q.dbg_flags = h->dbg_flags;
        q.run_flag = run_flag;
        if (++h->epoch == 0) h->epoch = 1;
        q.epoch = h->epoch;
        q.prog = (h->dbg_flags & 262144) ? nullptr : R.at<unsigned long long>(L.prog);  // (262144: no pacing, A/B)
        if (kind == 2)
            dcp_pc4_kernel<<<h->G4 * 4, P4_THREADS, P4_SMEM_BYTES, c.st>>>(R.tm4p, R.tm3p, q);
        else {
            decltype(&dcp_pc_kernel<false, false, false>) kern;
            if (h->dtype == F2C_F32)
                kern = q.excl ? (q.neg_mode ? dcp_pc_kernel<true, true, true> : dcp_pc_kernel<true, false, true>)
                              : (q.neg_mode ? dcp_pc_kernel<false, true, true> : dcp_pc_kernel<false, false, true>);
            else
                kern = q.excl ? (q.neg_mode ? dcp_pc_kernel<true, true, false> : dcp_pc_kernel<true, false, false>)
                              : (q.neg_mode ? dcp_pc_kernel<false, true, false> : dcp_pc_kernel<false, false, false>);
            kern<<<(h->G / 2) * 2, PC_THREADS, smem, c.st>>>(R.tm3p, R.tm3q, R.tmO, q);
        }
    }
    LAUNCH_CHECK();
    if (e1) CUDA_TRY(cudaEventRecord(e1, c.st));
    return F2C_OK;
}


static CombineArgs combine_args(f2c_dcp *h, Rank &R, const StepCtx &c, int64_t occ, uint8_t *dx) {
    const Layout &L = R.L;
    CombineArgs a;
    a.x = c.x;
    a.inv_n = R.at<float>(L.inv_n);
    a.comp_idx = R.at<int>(L.comp_idx);
    a.row_ab = R.at<float2>(L.row_ab);
    a.row_tgt = R.at<int>(L.row_tgt);
    a.ttgt = R.at<float>(L.ttgt);
    a.seg_l = R.at<float>(L.seg_l);
    a.seg_mx = R.at<float>(L.seg_mx);
    a.seg_O = R.at<float>(L.seg_O);
    a.T = R.base + (h->dtype == F2C_F32 ? L.Tsh : L.T);  // (bf16: the GEMM-2 operand rows)
    a.Tc = R.base + (h->K > 1 ? L.Traw : L.T);            // (exact centers: fp32 rows, K raw rows, bf16 rows)
    a.Tc_kind = h->dtype == F2C_F32 ? 1 : (h->K > 1 ? 2 : 0);
    a.Kc = h->K;
    a.mu_fx = R.at<long long>(L.mu_fx);
    a.sc = R.sc();
    a.sc_w = R.sc();
    a.N = c.N;
    a.C_occ = h->E < h->C ? h->E : h->C;
    a.d = h->d;
    a.dtype = h->dtype;
    const int kind = kernel_kind(h, c.N);
    a.G = kind == 1 ? h->G : kind == 2 ? h->G4 : h->G / 2;
    a.rows_per_group = kind == 1 ? TP_R : kind == 2 ? P4_RG : PC_R;
    a.wide = kind == 0 || kind == 2 ? 1 : 0;  // (both take S from k_compact)
    a.n_tiles = static_cast<int>((occ + TP_TILE - 1) / TP_TILE);
    a.s = c.s;
    a.margin_l2 = c.s * c.m * 1.4426950408889634f;
    a.dx = dx;
    a.rowloss = R.at<double>(L.rowloss);
    a.st_lse = R.at<float>(L.st_lse);
    a.st_cos = R.at<float>(L.st_cos);
    a.st_phi = R.at<float>(L.st_phi);
    a.st_ell = R.at<float>(L.st_ell);
    a.neg_mode = h->neg_mode();
    a.phi_mean = h->phi_mode == 0;
    a.hinge = h->hinge;
    a.lam = h->lam;
    a.my_rank = R.rank < 0 ? 0 : R.rank;
    a.seg_arg = R.at<int>(L.seg_arg);
    a.wslot = h->K > 1 ? R.at<float>(L.wslot) : nullptr;
    a.hkeys = R.at<int64_t>(L.hkeys);
    a.hvals = R.at<unsigned long long>(L.hvals);
    a.H = L.H;
    return a;
}

// R1 fallback for large s (R1): rows whose largest non-target exponent fell far
// below their reference get it lowered to that maximum, and the fused kernel runs once more
// (its CTAs exit at once unless some row was refined).  Below s = 68 no row with |cos| <= 1 can
// get there, so the pass is not even launched.
static int phase_refine(f2c_dcp *h, Rank &R, const StepCtx &c, int64_t occ) {
    if (!(c.s > 68.f) || kernel_kind(h, c.N) == 1) return F2C_OK;
    NvtxRange nv("f2c: R1 refinement pass");
    CombineArgs a = combine_args(h, R, c, occ, nullptr);
    k_refine_ref<<<static_cast<unsigned>((c.N + 255) / 256), 256, 0, c.st>>>(a, R.at<float2>(R.L.row_ab));
    LAUNCH_CHECK();
    return phase_main(h, R, c, occ, &R.sc()->refine);
}

static unsigned grid_for(int64_t n) {
    int64_t b = (n + 255) / 256;
    if (b > 4096) b = 4096;
    return static_cast<unsigned>(b < 1 ? 1 : b);
}

// world > 1: slot-range sharding, SURVEY 8(e) / DESIGN.md section 7.
//   C1 all-gather x, labels, pairing | local resolve | C2 MAX all-reduce (target seq, norm
//   bound) | compaction + fused kernel on the local shard | local row partials | C3
//   all-gather of the partials | identical finalisation + linear dx share | C4
//   reduce-scatter of dx.  Emulated world: the same steps, collectives as device copies.
static int loss_multi(f2c_dcp *h, const uint8_t *x, const int64_t *labels, const int32_t *pairing,
                      int64_t n_local, float s, float m, float *loss, uint8_t *dx, cudaStream_t st) {
    const int W = h->W;
    const int64_t N = n_local * W;
    const size_t rb = static_cast<size_t>(h->d) * (h->dtype == F2C_BF16 ? 2 : 4);
    int rc;
    h->last_N = N;
    std::vector<StepCtx> ctx(h->ranks.size());
    // ---- C1
    if (h->emulated) {
        for (size_t q = 0; q < h->ranks.size(); ++q) ctx[q] = StepCtx{N, s, m, x, labels, pairing, st};
    } else {
        Rank &R = h->ranks[0];
        NvtxRange nvc("f2c: C1 all-gather x, labels, pairing");
        comm_group_start(h);
        comm_allgather(h, x, R.base + R.L.x_all, n_local * rb, st, "C1");
        comm_allgather(h, labels, R.base + R.L.y_all, n_local * 8, st, "C1");
        if (pairing) comm_allgather(h, pairing, R.base + R.L.pair_all, n_local * 4, st, "C1");
        if ((rc = comm_group_end(h, st, "C1 all-gather"))) return rc;
        ctx[0] = StepCtx{N, s, m, R.base + R.L.x_all, R.at<int64_t>(R.L.y_all),
                         pairing ? R.at<int32_t>(R.L.pair_all) : nullptr, st};
    }
    // ---- local resolve, then C2 (MAX of target write index and of the norm bound)
    for (size_t q = 0; q < h->ranks.size(); ++q) {
        Rank &R = h->ranks[q];
        if ((rc = phase_resolve(h, R, ctx[q]))) return rc;
        k_pack_tseq<<<grid_for(N + 1), 256, 0, st>>>(R.at<int64_t>(R.L.tseq), R.sc(), N, R.at<int64_t>(R.L.tseq_ext));
        LAUNCH_CHECK();
    }
    if (h->emulated) {
        Rank &R0 = h->ranks[0];
        for (size_t q = 1; q < h->ranks.size(); ++q) {
            k_max_i64_into<<<grid_for(N + 1), 256, 0, st>>>(R0.at<int64_t>(R0.L.tseq_ext),
                                                            h->ranks[q].at<int64_t>(h->ranks[q].L.tseq_ext), N + 1);
            LAUNCH_CHECK();
        }
        for (size_t q = 1; q < h->ranks.size(); ++q)
            CUDA_TRY(cudaMemcpyAsync(h->ranks[q].at<int64_t>(h->ranks[q].L.tseq_ext), R0.at<int64_t>(R0.L.tseq_ext),
                                     (N + 1) * 8, cudaMemcpyDeviceToDevice, st));
    } else {
        Rank &R = h->ranks[0];
        NvtxRange nvc("f2c: C2 MAX all-reduce");
        if ((rc = comm_allreduce_max_i64(h, R.at<int64_t>(R.L.tseq_ext), N + 1, st, "C2 all-reduce"))) return rc;
    }
    // ---- compaction, fused kernel on the local shard, local row partials
    for (size_t q = 0; q < h->ranks.size(); ++q) {
        Rank &R = h->ranks[q];
        k_unpack_tseq<<<grid_for(N + 1), 256, 0, st>>>(R.at<int64_t>(R.L.tseq_ext), N, R.at<int64_t>(R.L.tseq),
                                                       R.at<int>(R.L.tmax_glob));
        LAUNCH_CHECK();
        if ((rc = phase_compact(h, R, ctx[q], R.at<int>(R.L.tmax_glob)))) return rc;
        const int64_t occ = occ_local(h, R);
        if ((rc = phase_main(h, R, ctx[q], occ))) return rc;
        if ((rc = phase_refine(h, R, ctx[q], occ))) return rc;
        CombineArgs a = combine_args(h, R, ctx[q], occ, nullptr);
        k_local_rows<<<static_cast<unsigned>((N + CB_ROWS - 1) / CB_ROWS), 256, 0, st>>>(a, R.at<float4>(R.L.rs_buf));
        LAUNCH_CHECK();
    }
    // ---- C3: all-gather of the per-row partials
    if (h->emulated) {
        for (size_t q = 0; q < h->ranks.size(); ++q)
            for (size_t r = 0; r < h->ranks.size(); ++r)
                CUDA_TRY(cudaMemcpyAsync(h->ranks[q].at<float4>(h->ranks[q].L.rs_all) + r * N,
                                         h->ranks[r].at<float4>(h->ranks[r].L.rs_buf), N * 16,
                                         cudaMemcpyDeviceToDevice, st));
    } else {
        Rank &R = h->ranks[0];
        NvtxRange nvc("f2c: C3 all-gather row partials");
        if ((rc = comm_allgather(h, R.at<float4>(R.L.rs_buf), R.at<float4>(R.L.rs_all), N * 16, st, "C3 all-gather")))
            return rc;
    }
    // ---- finalisation (identical on every rank) + linear dx share, then C4
    for (size_t q = 0; q < h->ranks.size(); ++q) {
        Rank &R = h->ranks[q];
        CombineArgs a = combine_args(h, R, ctx[q], occ_local(h, R), nullptr);
        k_finalize_multi<<<static_cast<unsigned>((N + CB_ROWS - 1) / CB_ROWS), 256, 0, st>>>(
            a, R.at<float4>(R.L.rs_all), W, N, R.at<float>(R.L.dx_part), loss);
        LAUNCH_CHECK();
    }
    if (h->emulated) {
        Rank &R0 = h->ranks[0];
        for (size_t q = 1; q < h->ranks.size(); ++q) {
            k_add_f32_into<<<grid_for(N * h->d), 256, 0, st>>>(R0.at<float>(R0.L.dx_part),
                                                               h->ranks[q].at<float>(h->ranks[q].L.dx_part), N * h->d);
            LAUNCH_CHECK();
        }
        if (h->dtype == F2C_F32) {
            CUDA_TRY(cudaMemcpyAsync(dx, R0.at<float>(R0.L.dx_part), N * h->d * 4, cudaMemcpyDeviceToDevice, st));
        } else {
            k_cast_bf16<<<grid_for(N * h->d), 256, 0, st>>>(R0.at<float>(R0.L.dx_part),
                                                            reinterpret_cast<__nv_bfloat16 *>(dx), N * h->d);
            LAUNCH_CHECK();
        }
    } else {
        Rank &R = h->ranks[0];
        NvtxRange nvc("f2c: C4 reduce-scatter dx");
        float *rs_out = h->dtype == F2C_F32 ? static_cast<float *>(static_cast<void *>(dx)) : R.at<float>(R.L.dx32);
        if ((rc = comm_reduce_scatter_f32(h, R.at<float>(R.L.dx_part), rs_out, n_local * h->d, st, "C4 reduce-scatter")))
            return rc;
        if (h->dtype != F2C_F32) {
            k_cast_bf16<<<grid_for(n_local * h->d), 256, 0, st>>>(R.at<float>(R.L.dx32),
                                                                  reinterpret_cast<__nv_bfloat16 *>(dx), n_local * h->d);
            LAUNCH_CHECK();
        }
    }
    return F2C_OK;
}

extern "C" int f2c_dcp_loss_fwd_bwd(f2c_dcp *h, const void *x, const int64_t *labels,
                                    const int32_t *pairing, int64_t n_local, float s, float m,
                                    float *loss, void *dx, void *stream) {
    NvtxRange nv("f2c_dcp_loss_fwd_bwd (a2-a9)");
    g_launches = 0;
    if (!h) return fail(F2C_EINVAL, "NULL handle");
    if (!x || !labels || !loss || !dx) return fail(F2C_EINVAL, "NULL x/labels/loss/dx");
    if (n_local < 1 || n_local > h->n_local_max)
        return fail(F2C_ESHAPE, "n_local %lld not in [1, %lld]", (long long)n_local, (long long)h->n_local_max);
    if (!(s > 0.f) || !isfinite(s) || !isfinite(m)) return fail(F2C_EINVAL, "need s > 0 and finite m");
    if (x == dx) return fail(F2C_EINVAL, "dx must not alias x");
    if ((reinterpret_cast<uintptr_t>(x) | reinterpret_cast<uintptr_t>(dx)) & 15)
        return fail(F2C_EINVAL, "x and dx must be 16-byte aligned");
    if (h->dtype == F2C_F32 && h->d > 256)
        return fail(F2C_EINVAL, "fp32 pools: the loss path (tf32 logits, x_hat as fp32 in TMEM) needs d <= 256");
    int rc = latched(h, false);
    if (rc) return rc;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    h->last_stream = st;
    if (h->multi) return loss_multi(h, static_cast<const uint8_t *>(x), labels, pairing, n_local, s, m, loss,
                                     static_cast<uint8_t *>(dx), st);
    Rank &R = h->ranks[0];
    StepCtx c{n_local, s, m, static_cast<const uint8_t *>(x), labels, pairing, st};
    h->last_N = c.N;
    if ((rc = phase_resolve(h, R, c))) return rc;
    if ((rc = phase_compact(h, R, c, &R.sc()->tmax_bits))) return rc;
    const int64_t occ = occ_local(h, R);
    if ((rc = phase_main(h, R, c, occ))) return rc;
    if ((rc = phase_refine(h, R, c, occ))) return rc;
    CombineArgs a = combine_args(h, R, c, occ, static_cast<uint8_t *>(dx));
    k_combine<<<static_cast<unsigned>((c.N + CB_ROWS - 1) / CB_ROWS), 256, 0, st>>>(a, loss);
    LAUNCH_CHECK();
    return F2C_OK;
}

extern "C" int f2c_dcp_set_lcos(f2c_dcp *h, int32_t phi_mode, int32_t hinge, double lambda) {
    if (!h) return fail(F2C_EINVAL, "NULL handle");
    if (phi_mode < 0 || phi_mode > 2) return fail(F2C_EINVAL, "phi_mode %d not in {0 mean, 1 sum, 2 max}", phi_mode);
    if (hinge != 0 && hinge != 1) return fail(F2C_EINVAL, "hinge must be 0 or 1");
    if (!isfinite(lambda)) return fail(F2C_EINVAL, "lambda must be finite");
    h->phi_mode = phi_mode;
    h->hinge = hinge;
    h->lam = static_cast<float>(lambda);
    return F2C_OK;
}

extern "C" int f2c_dcp_set_enqueue_mode(f2c_dcp *h, int32_t refresh_in_place) {
    if (!h) return fail(F2C_EINVAL, "NULL handle");
    if (refresh_in_place != 0 && refresh_in_place != 1) return fail(F2C_EINVAL, "refresh_in_place must be 0 or 1");
    if (refresh_in_place && !h->n_app_host) {
        void *p = nullptr;
        CUDA_TRY(cudaMallocHost(&p, sizeof(long long)));
        h->n_app_host = static_cast<long long *>(p);
    }
    h->refresh = refresh_in_place;
    return F2C_OK;
}

extern "C" int f2c_dcp_set_dup_mode(f2c_dcp *h, int32_t exclude_stale) {
    if (!h) return fail(F2C_EINVAL, "NULL handle");
    if (exclude_stale != 0 && exclude_stale != 1) return fail(F2C_EINVAL, "exclude_stale must be 0 or 1");
    h->excl_dup = exclude_stale;
    return F2C_OK;
}

// ============================================================================ support
static const char *err_detail_text(int dd) {
    static const char *det[] = {"", "negative label", "zero-norm (or non-finite) feature row",
                                "pairing[i] does not name row i's target",
                                "non-finite loss", "softmax underflow (row max < 2^-100 of the reference)",
                                "duplicate label within a refresh-in-place enqueue block (S:277)"};
    return det[(dd >= 0 && dd <= 6) ? dd : 0];
}

// sync = false (every enqueue / loss call): read the mapped host mirror of each shard's error
// word (written by the kernel that latched it; no synchronisation, no copy), so a device error
// is reported by the first host call made after it became visible.  The error stays latched
// (every later call reports it) until f2c_dcp_check() clears it.
// sync = true (f2c_dcp_check, after a device synchronisation): read the device word itself,
// report it and clear it (device word and mirror).
static int latched(f2c_dcp *h, bool sync) {
    if (!sync) {
        if (!h->err_host) return F2C_OK;
        for (size_t i = 0; i < h->ranks.size(); ++i) {
            const volatile int *m = h->err_host + 2 * i;
            const int code = m[0];
            if (code != 0)
                return fail(code, "device error latched by an earlier call (rank %d): %s; "
                            "f2c_dcp_check() reports and clears it", h->ranks[i].rank, err_detail_text(m[1]));
        }
        return F2C_OK;
    }
    int worst = F2C_OK;
    for (size_t i = 0; i < h->ranks.size(); ++i) {
        Rank &R = h->ranks[i];
        Scalars s;
        if (cudaMemcpy(&s, R.sc(), sizeof s, cudaMemcpyDeviceToHost) != cudaSuccess)
            return fail(F2C_ECUDA, "reading the device error word failed");
        if (s.err) {
            fail(s.err, "device error (rank %d): %s", R.rank, err_detail_text(s.err_detail));
            worst = s.err;
            int zero[2] = {0, 0};
            cudaMemcpy(R.sc(), zero, sizeof zero, cudaMemcpyHostToDevice);
        }
        if (h->err_host) {
            h->err_host[2 * i] = 0;
            h->err_host[2 * i + 1] = 0;
        }
    }
    return worst;
}

extern "C" int f2c_dcp_check(f2c_dcp *h) {
    if (!h) return fail(F2C_EINVAL, "NULL handle");
    if (h->last_stream) CUDA_TRY(cudaStreamSynchronize(h->last_stream));
    CUDA_TRY(cudaDeviceSynchronize());
    if (h->comm && nccl().CommGetAsyncError) {  // failure detection of the collectives
        int async_err = 0;
        if (nccl().CommGetAsyncError(h->comm, &async_err) == 0 && async_err != 0)
            return fail(F2C_ENCCL, "NCCL asynchronous error: %s",
                        nccl().GetErrorString ? nccl().GetErrorString(async_err) : "?");
    }
    return latched(h, true);
}

extern "C" int f2c_dcp_get_state(f2c_dcp *h, void *feats_host, int64_t *labels_host,
                                 int64_t *enq_count_host) {
    if (!h) return fail(F2C_EINVAL, "NULL handle");
    CUDA_TRY(cudaDeviceSynchronize());
    const size_t rb = static_cast<size_t>(h->d) * h->K * (h->dtype == F2C_BF16 ? 2 : 4);
    int64_t row0 = 0;
    for (Rank &R : h->ranks) {
        const int64_t n = R.hi - R.lo;
        if (feats_host)
            CUDA_TRY(cudaMemcpy(static_cast<uint8_t *>(feats_host) + row0 * rb, R.base + (h->K > 1 ? R.L.Traw : R.L.T),
                                n * rb, cudaMemcpyDeviceToHost));
        if (labels_host) {
            CUDA_TRY(cudaMemcpy(labels_host + row0, R.at<int64_t>(R.L.lab), n * 8, cudaMemcpyDeviceToHost));
            const int64_t occ = occ_local(h, R);
            for (int64_t i = occ; i < n; ++i) labels_host[row0 + i] = -1;
        }
        row0 += n;
    }
    if (enq_count_host) *enq_count_host = h->E;
    return F2C_OK;
}

extern "C" int f2c_dcp_set_state(f2c_dcp *h, const void *feats_host, const int64_t *labels_host,
                                 int64_t enq_count) {
    if (!h) return fail(F2C_EINVAL, "NULL handle");
    if (!feats_host || !labels_host || enq_count < 0) return fail(F2C_EINVAL, "bad set_state arguments");
    const size_t rb = static_cast<size_t>(h->d) * h->K * (h->dtype == F2C_BF16 ? 2 : 4);
    const int64_t C_occ = enq_count < h->C ? enq_count : h->C;
    int64_t row0 = 0;
    for (Rank &R : h->ranks) {
        const int64_t n = R.hi - R.lo;
        for (int64_t i = 0; i < n; ++i) {
            const int64_t c = R.lo + i;
            const int64_t lb = labels_host[row0 + i];
            if (c < C_occ && lb < 0) return fail(F2C_EINVAL, "occupied slot %lld has a negative label", (long long)c);
            if (c >= C_occ && lb != -1) return fail(F2C_EINVAL, "slot %lld >= min(E, C) must be empty (-1)", (long long)c);
        }
        row0 += n;
    }
    CUDA_TRY(cudaDeviceSynchronize());
    row0 = 0;
    for (Rank &R : h->ranks) {
        const int64_t n = R.hi - R.lo;
        int64_t occ = C_occ - R.lo;
        if (occ > n) occ = n;
        if (occ < 0) occ = 0;
        uint8_t *dstT = R.base + (h->K > 1 ? R.L.Traw : R.L.T);
        CUDA_TRY(cudaMemset(dstT, 0, n * rb));
        if (h->K > 1) CUDA_TRY(cudaMemset(R.base + R.L.T, 0, n * static_cast<size_t>(h->d) * 2));
        if (occ > 0)
            CUDA_TRY(cudaMemcpy(dstT, static_cast<const uint8_t *>(feats_host) + row0 * rb,
                                occ * rb, cudaMemcpyHostToDevice));
        CUDA_TRY(cudaMemcpy(R.at<int64_t>(R.L.lab), labels_host + row0, n * 8, cudaMemcpyHostToDevice));
        int zero = 0;
        CUDA_TRY(cudaMemcpy(&R.sc()->tmax_bits, &zero, 4, cudaMemcpyHostToDevice));
        if (occ > 0 && h->K > 1) {
            CUDA_TRY(cudaMemset(R.at<float>(R.L.wslot), 0, static_cast<size_t>(n + 128) * 4));
            k_rebuild_k<<<static_cast<unsigned>((occ * 32 + 255) / 256), 256>>>(
                R.at<__nv_bfloat16>(R.L.Traw), occ, h->K, h->d, R.at<__nv_bfloat16>(R.L.T),
                R.at<float>(R.L.wslot), R.sc());
            CUDA_TRY(cudaGetLastError());
        } else if (occ > 0) {
            k_pool_norm_max<<<static_cast<unsigned>((occ * 32 + 255) / 256), 256>>>(
                R.base + R.L.T, occ, static_cast<int>(rb), h->dtype, R.sc());
            CUDA_TRY(cudaGetLastError());
        }
        if (h->dtype == F2C_F32) {  // the bf16 shadow of the restored fp32 rows (zeros beyond occ)
            CUDA_TRY(cudaMemset(R.base + R.L.Tsh, 0, n * static_cast<size_t>(h->d) * 2));
            if (occ > 0) {
                k_cast_bf16<<<grid_for(occ * h->d), 256>>>(R.at<float>(R.L.T), R.at<__nv_bfloat16>(R.L.Tsh), occ * h->d);
                CUDA_TRY(cudaGetLastError());
            }
        }
        // mu over the restored slots lo .. lo + occ - 1
        CUDA_TRY(cudaMemset(R.base + R.L.mu_fx, 0, static_cast<size_t>(h->d) * 8));
        if (occ > 0 && h->K > 1) {
            const int64_t blocks = (occ + 7) / 8 < 4 * static_cast<int64_t>(h->G) ? (occ + 7) / 8 : 4 * static_cast<int64_t>(h->G);
            k_mu_sum_k<<<static_cast<unsigned>(blocks), 256>>>(R.at<__nv_bfloat16>(R.L.Traw), R.at<float>(R.L.wslot),
                                                                occ, h->K, h->d, R.at<unsigned long long>(R.L.mu_fx));
            CUDA_TRY(cudaGetLastError());
        } else if (occ > 0) {
            const int64_t blocks = occ < 4 * static_cast<int64_t>(h->G) ? occ : 4 * static_cast<int64_t>(h->G);
            k_mu_sum<<<static_cast<unsigned>(blocks), 256>>>(
                R.base + R.L.T, h->dtype == F2C_BF16 ? 0 : 1, nullptr, h->d, occ, R.lo, h->C, R.lo, R.hi, nullptr, +1,
                R.at<unsigned long long>(R.L.mu_fx));
            CUDA_TRY(cudaGetLastError());
        }
        row0 += n;
    }
    CUDA_TRY(cudaDeviceSynchronize());
    h->E = enq_count;
    for (Rank &R : h->ranks) {
        int rc = idx_rebuild(h, R, nullptr);
        if (rc) return rc;
    }
    CUDA_TRY(cudaDeviceSynchronize());
    h->M_last = 0;            // (no block since the restore: pairing checks fail until the next enqueue)
    h->last_refresh = false;
    return F2C_OK;
}

extern "C" int f2c_dcp_fused_kernel(f2c_dcp *h, int64_t n_global, int32_t *kind, int32_t *ctas) {
    if (!h || !kind || !ctas) return fail(F2C_EINVAL, "NULL argument");
    const int k = kernel_kind(h, n_global);
    *kind = k;
    *ctas = k == 1 ? h->G : k == 2 ? h->G4 * 4 : (h->G / 2) * 2;
    return F2C_OK;
}

extern "C" int f2c_dcp_profile(f2c_dcp *h, int enable) {
    if (!h) return fail(F2C_EINVAL, "NULL handle");
    if (enable) {
        CUDA_TRY(cudaDeviceSynchronize());
        h->ev_used = 0;
        Scalars s;
        CUDA_TRY(cudaMemcpy(&s, h->ranks[0].sc(), sizeof s, cudaMemcpyDeviceToHost));
        h->npos_base = s.n_pos_sum;
    }
    h->prof = enable != 0;
    return F2C_OK;
}

extern "C" int f2c_dcp_profile_read(f2c_dcp *h, double *main_ms, int64_t *launches, int64_t *n_pos_sum) {
    if (!h) return fail(F2C_EINVAL, "NULL handle");
    CUDA_TRY(cudaDeviceSynchronize());
    double tot = 0.0;
    for (size_t i = 0; i + 1 < h->ev_used; i += 2) {
        float ms = 0.f;
        CUDA_TRY(cudaEventElapsedTime(&ms, h->ev[i], h->ev[i + 1]));
        tot += ms;
    }
    if (main_ms) *main_ms = tot;
    if (launches) *launches = static_cast<int64_t>(h->ev_used / 2);
    if (n_pos_sum) {
        Scalars s;
        CUDA_TRY(cudaMemcpy(&s, h->ranks[0].sc(), sizeof s, cudaMemcpyDeviceToHost));
        *n_pos_sum = static_cast<int64_t>(s.n_pos_sum - h->npos_base);
    }
    return F2C_OK;
}

// internal debugging aid (not in the public header): per-tile clock64 stamps of CTA 0
extern "C" int f2c_dcp_debug_timestamps(f2c_dcp *h, unsigned long long *dev_buf) {
    if (!h) return fail(F2C_EINVAL, "NULL handle");
    h->dbg = dev_buf;
    const char *fl = getenv("F2C_DBG_FLAGS");
    h->dbg_flags = fl ? atoi(fl) : 0;
    const char *cl = getenv("F2C_DBG_CLUSTER");
    h->dbg_cluster = cl ? atoi(cl) : 0;
    return F2C_OK;
}

extern "C" int f2c_dcp_row_stats(f2c_dcp *h, float *lse, int64_t *target_seq, float *cos_t,
                                 float *phi, float *ell, int64_t *counts) {
    if (!h) return fail(F2C_EINVAL, "NULL handle");
    CUDA_TRY(cudaDeviceSynchronize());
    Rank &R = h->ranks[0];
    const int64_t N = h->last_N;
    if (lse) CUDA_TRY(cudaMemcpy(lse, R.at<float>(R.L.st_lse), N * 4, cudaMemcpyDeviceToHost));
    if (target_seq) CUDA_TRY(cudaMemcpy(target_seq, R.at<int64_t>(R.L.tseq), N * 8, cudaMemcpyDeviceToHost));
    if (cos_t) CUDA_TRY(cudaMemcpy(cos_t, R.at<float>(R.L.st_cos), N * 4, cudaMemcpyDeviceToHost));
    if (phi) CUDA_TRY(cudaMemcpy(phi, R.at<float>(R.L.st_phi), N * 4, cudaMemcpyDeviceToHost));
    if (ell) CUDA_TRY(cudaMemcpy(ell, R.at<float>(R.L.st_ell), N * 4, cudaMemcpyDeviceToHost));
    if (counts) {
        Scalars s;
        CUDA_TRY(cudaMemcpy(&s, R.sc(), sizeof s, cudaMemcpyDeviceToHost));
        counts[0] = s.n_pos;
        counts[1] = s.n_neg;
        counts[2] = h->E < h->C ? h->E : h->C;
    }
    return F2C_OK;
}
