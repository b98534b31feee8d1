// dcp_pc4.cuh -- the fused DCP loss kernel with 2-SM tensor-core pairs (tcgen05 cta_group::2):
// a cluster of FOUR CTAs owns one group of 256 compacted rows and a range of pool tiles.
//
//   ranks 0, 1 = the producer pair, ranks 2, 3 = the consumer pair (the even rank of each pair
//   is its leader: it issues the pair's MMAs).  CTA 2h+p holds rows 128p .. 128p+127 of the group.
//   GEMM 1 (leader 0):  S[256 rows x 128 slots] = x_hat . T_tile^T, M = 256, K = d; A = x_hat
//     from each producer's TMEM (its 128 rows), B = the pool tile, each producer holding 64 of
//     its 128 slots (B is split by N).  Each producer's TMEM receives S for its own 128 rows.
//   softmax warps of each producer: exactly as in dcp_pc.cuh on their 128 rows; P (bf16) goes
//     to the consumer of the same half (rank 2 + p) by a DSMEM bulk copy.
//   GEMM 2 (leader 2):  O[256 rows x d] += P . T_tile, M = 256, N = 256 per d block, K = 128
//     slots; A = P (each consumer its 128 rows), B = the pool tile MN-major, each consumer
//     holding 128 of the block's 256 d columns.  Each consumer's TMEM holds O for its rows.
// Against the CTA-pair kernel (dcp_pc.cuh) every SM receives and reads HALF of each pool
// tile per 128 rows (the shared-memory traffic per tile and SM, the measured bound there),
// at the price of 256-row granularity.  Scope: the default variant (K = 1, L_cos mean / sum,
// no stale-duplicate exclusion), d a multiple of 256; the host falls back to dcp_pc_kernel
// otherwise.
//
// Barriers (same PC4Aux offsets in all four CTAs):
//   tfull[s]   leader 0: its arrive.expect_tx (both halves) + the complete_tx of both TMA loads
//              (the peer's load signals the leader's barrier: cp.async.bulk.tensor .cta_group::2)
//   tempty[s]  every producer: leader 0's multicast commit (mask 0b0011)
//   sfull[b]   every producer: multicast commit; sempty[b] leader 0: 16 softmax warps (8 remote)
//   xready     leader 0: 16 softmax warps; xfree: every producer, multicast commit
//   pready / pstage_free: per producer (softmax warps <-> the P mover)
//   pslot_free[b] every producer: leader 2's multicast commit (mask 0b0011) after GEMM 2 used slot b
//   pfull[b]   every consumer: complete_tx of its producer's P copy; the peer consumer relays
//              it to leader 2's pfull_peer[b]
//   qfull / qempty: as tfull / tempty for the consumer pair (mask 0b1100)
//   ofull      every consumer: leader 2's multicast commit at a unit's end; oempty: leader 2,
//              16 drain warps (8 remote)
#pragma once
#include "dcp_pc.cuh"

namespace f2c {

constexpr int P4_R = 128;                 // rows per CTA (TMEM lanes)
constexpr int P4_RG = 256;                // rows per cluster row group
constexpr int P4_TILE = 128;              // slots per tile
constexpr int P4_THREADS = 352;           // 11 warps
constexpr int P4P_NSTAGE = 6;             // producer ring: [2 chunks x 64 slots x 64 d] = 16 KB
constexpr int P4P_STAGE = 16384;
constexpr int P4Q_NSTAGE = 3;             // consumer ring: [2 chunks x 128 slots x 64 d] = 32 KB
constexpr int P4Q_STAGE = 32768;
constexpr int P4_PBYTES = P4_R * P4_TILE * 2;  // 32 KB
// P buffers: staging in the producer and slots in the consumer, three deep (the P path
// crosses three SMs per tile -- producer, consumer, peer relay -- and two-deep buffers
// measured as its bound)
constexpr int P4_NPS = 3;
constexpr int P4_NSLOT = 3;
constexpr int P4P_OFF_T = 0;
constexpr int P4P_OFF_PS = P4P_OFF_T + P4P_NSTAGE * P4P_STAGE;  // P staging
constexpr int P4Q_OFF_P = 0;                                    // P slots
constexpr int P4Q_OFF_T = P4Q_OFF_P + P4_NSLOT * P4_PBYTES;
constexpr int P4_OFF_AUX = 196608;
static_assert(P4P_OFF_PS + P4_NPS * P4_PBYTES <= P4_OFF_AUX, "producer smem");
static_assert(P4Q_OFF_T + P4Q_NSTAGE * P4Q_STAGE <= P4_OFF_AUX, "consumer smem");
constexpr int P4_SMEM_BYTES = P4_OFF_AUX + 4096 + 1024;

struct PC4Aux {
    uint64_t tfull[P4P_NSTAGE], tempty[P4P_NSTAGE];
    uint64_t sfull[2], sempty[2];
    uint64_t xready, xfree;
    uint64_t pready[P4_NPS], pstage_free[P4_NPS], pslot_free[P4_NSLOT];
    uint64_t qfull[P4Q_NSTAGE], qempty[P4Q_NSTAGE];
    uint64_t pfull[P4_NSLOT], pfull_peer[P4_NSLOT];
    uint64_t ofull, oempty;
    uint32_t tmem_base;
    uint32_t pad;
    float red_l[2][P4_R];
    float red_mx[2][P4_R];
    int4 units[PC_MAX_UNITS];
    int n_units;
};
static_assert(sizeof(PC4Aux) <= 4096, "PC4Aux must fit the aux region");

// ---- cta_group::2 issue helpers (one elected lane of the leader's issuing warp)
// GEMM 1 stage: 8 TS MMAs (2 chunks x 4 K steps of 16), then the multicast commit of `bar`
__device__ __forceinline__ void umma2_ts_stage8(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                                uint32_t acc0, uint32_t bar, uint16_t mask) {
    asm volatile(
        "{\n.reg .pred e, p, t;\n.reg .b32 r;\n"
        "elect.sync r|e, 0xffffffff;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "setp.eq.b32 t, 0, 0;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+8], %7, %3, t;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+16], %8, %3, t;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+24], %9, %3, t;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+32], %10, %3, t;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+40], %11, %3, t;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+48], %12, %3, t;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], [%1+56], %13, %3, t;\n"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%5], %6;\n}\n" ::"r"(
            d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc0), "r"(bar), "h"(mask), "l"(bdesc + 2), "l"(bdesc + 4),
        "l"(bdesc + 6), "l"(bdesc + 512), "l"(bdesc + 514), "l"(bdesc + 516), "l"(bdesc + 518)
        : "memory");
}
// GEMM 2 stage: 8 SS MMAs over the tile's 128 slots, then the multicast commit of `bar`
__device__ __forceinline__ void umma2_ss_stage8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                                uint32_t acc0, uint32_t bar, uint16_t mask) {
    asm volatile(
        "{\n.reg .pred e, p, t;\n.reg .b32 r;\n"
        "elect.sync r|e, 0xffffffff;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "setp.eq.b32 t, 0, 0;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %7, %8, %3, t;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %9, %10, %3, t;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %11, %12, %3, t;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %13, %14, %3, t;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %15, %16, %3, t;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %17, %18, %3, t;\n"
        "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %19, %20, %3, t;\n"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%5], %6;\n}\n" ::"r"(
            d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc0), "r"(bar), "h"(mask), "l"(adesc + 2), "l"(bdesc + 128),
        "l"(adesc + 4), "l"(bdesc + 256), "l"(adesc + 6), "l"(bdesc + 384), "l"(adesc + 1024), "l"(bdesc + 512),
        "l"(adesc + 1026), "l"(bdesc + 640), "l"(adesc + 1028), "l"(bdesc + 768), "l"(adesc + 1030),
        "l"(bdesc + 896)
        : "memory");
}
__device__ __forceinline__ void umma2_commit_mc_e(uint32_t bar, uint16_t mask) {
    asm volatile(
        "{\n.reg .pred e;\n.reg .b32 r;\nelect.sync r|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(
            bar),
        "h"(mask)
        : "memory");
}
// TMA load of this CTA's half stage, completing on the pair leader's barrier (cluster address)
__device__ __forceinline__ void tma2_load_3d(uint32_t dst, const CUtensorMap *m, uint32_t bar_cluster, int x, int y,
                                             int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(dst),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(bar_cluster), "r"(x), "r"(y), "r"(z)
        : "memory");
}
__device__ __forceinline__ void mbar_arrive_remote(uint32_t bar_cluster) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}
// Relaxed arrive on a (possibly remote) barrier, for hand-offs that order only tcgen05 traffic
// already completed by tcgen05.wait::ld / wait::st: a cluster-scope RELEASE arrive waits for the
// thread's earlier writes to become cluster-visible and measured ~1470 cycles per tile here.
__device__ __forceinline__ void mbar_arrive_remote_relaxed(uint32_t bar_cluster) {
    asm volatile("mbarrier.arrive.relaxed.cluster.shared::cluster.b64 _, [%0];" ::"r"(bar_cluster) : "memory");
}

__global__ void __cluster_dims__(4, 1, 1) __launch_bounds__(P4_THREADS, 1)
    dcp_pc4_kernel(const __grid_constant__ CUtensorMap tm4p, const __grid_constant__ CUtensorMap tm4q,
                   const PCParams p) {
    if (p.run_flag != nullptr && *p.run_flag == 0) return;  // (whole clusters exit together)
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~static_cast<uintptr_t>(1023));
    PC4Aux *aux = reinterpret_cast<PC4Aux *>(smem + P4_OFF_AUX);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t crank = cluster_ctarank();
    const uint32_t half = crank & 1;        // which 128 rows of the group / which operand half
    const bool is_leader = half == 0;
    const int d = p.d;
    const int nchunk = d >> 6;              // 64-wide d chunks
    const int nstg_p = nchunk / 2;          // producer stages per tile (2 chunks each)
    const int nstg_q = d / 256;             // consumer stages per tile (one 256-d block each)
    const int n_rows = *p.n_rows;
    const int n_rg = (n_rows + P4_RG - 1) / P4_RG;
    const int n_tiles = (p.n_slots + P4_TILE - 1) / P4_TILE;
    // debug hook: per-tile clocks of cluster dbg_cluster, dbg[16 jt + k] (each CTA its own SM clock)
    const bool dbgc = p.dbg && (blockIdx.x >> 2) == static_cast<unsigned>(p.dbg_cluster);
#define P4_STAMP(jt, k) do { if (dbgc && (jt) < 64) p.dbg[(jt) * 16 + (k)] = clock64(); } while (0)

    const long long t_start = clock64();
    unsigned long long g_start;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_start));
    if (threadIdx.x == 0) {
        for (int i = 0; i < P4P_NSTAGE; ++i) {
            mbar_init(&aux->tfull[i], 1);
            mbar_init(&aux->tempty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&aux->sfull[i], 1);
            mbar_init(&aux->sempty[i], 16);
        }
        for (int i = 0; i < P4_NPS; ++i) {
            mbar_init(&aux->pready[i], 8);
            mbar_init(&aux->pstage_free[i], 1);
        }
        for (int i = 0; i < P4_NSLOT; ++i) {
            mbar_init(&aux->pslot_free[i], 1);
            mbar_init(&aux->pfull[i], 1);
            mbar_init(&aux->pfull_peer[i], 1);
        }
        mbar_init(&aux->xready, 16);
        mbar_init(&aux->xfree, 1);
        for (int i = 0; i < P4Q_NSTAGE; ++i) {
            mbar_init(&aux->qfull[i], 1);
            mbar_init(&aux->qempty[i], 1);
        }
        mbar_init(&aux->ofull, 1);
        mbar_init(&aux->oempty, 16);
        if (crank >= 2 && !(p.dbg_flags & 128))  // arm the P slots before the producers can copy into them
            for (int i = 0; i < P4_NSLOT; ++i) mbar_arrive_expect_tx(&aux->pfull[i], P4_PBYTES);
        fence_mbar_init();
        TPSched ts;
        ts.init(blockIdx.x >> 2, gridDim.x >> 2, n_rg, n_tiles, *p.S_sched);  // (k_compact's multi-wave choice)
        int n = 0, a, b, c, s;
        while (n < PC_MAX_UNITS && ts.next(a, b, c, s)) aux->units[n++] = make_int4(a, b, c, s);
        aux->n_units = n;
    }
    if (warp == 9) {
        tma_prefetch_desc(&tm4p);
        tma_prefetch_desc(&tm4q);
        asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                         smem_u32(&aux->tmem_base))
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    const uint32_t tmem = aux->tmem_base;

    PCUnitIt sch{aux->units, aux->n_units, 0};
    int rg, t0, t1, seg;

    if (crank < 2) {
        // ================================================================= PRODUCER PAIR
        uint8_t *sT = smem + P4P_OFF_T;
        uint8_t *sPS = smem + P4P_OFF_PS;
        constexpr uint32_t X_COL = 0, S_COL = 256;
        if (warp == 8) {
            // -------- TMA: this CTA's 64 slots of each pool stage, on leader 0's barrier
            if (lane == 0) {
                uint32_t pc = 0;
                while (sch.next(rg, t0, t1, seg)) {
                    for (int t = t0; t < t1; ++t)
                        for (int g = 0; g < nstg_p; ++g, ++pc) {
                            const uint32_t st = pc % P4P_NSTAGE, ph = (pc / P4P_NSTAGE) & 1;
                            mbar_wait(&aux->tempty[st], ph ^ 1);
                            if (p.dbg_flags & 4) {  // timing experiment: no pool loads
                                if (is_leader) mbar_arrive(&aux->tfull[st]);
                                continue;
                            }
                            if (is_leader) mbar_arrive_expect_tx(&aux->tfull[st], 2 * P4P_STAGE);
                            tma2_load_3d(smem_u32(sT + st * P4P_STAGE), &tm4p, mapa_shared(smem_u32(&aux->tfull[st]), 0),
                                         0, t * P4_TILE + 64 * static_cast<int>(half), g * 2);
                        }
                }
            }
        } else if (warp == 9) {
            // -------- leader 0: GEMM 1 issue (M = 256, N = 128 slots, A = x_hat from TMEM)
            if (is_leader) {
                const uint32_t idesc = umma_idesc_bf16(256, P4_TILE, 0, 0);
                const uint64_t bdesc0 = umma_desc_sw128(smem_u32(sT), 16, 1024);
                uint32_t pc = 0, jt = 0, sg = 0;
                while (sch.next(rg, t0, t1, seg)) {
                    mbar_wait(&aux->xready, sg & 1);
                    tc_fence_after();
                    for (int t = t0; t < t1; ++t, ++jt) {
                        const uint32_t sb = jt & 1, sph = (jt >> 1) & 1;
                        const uint32_t dcol = tmem + S_COL + sb * P4_TILE;
                        if (lane == 0) P4_STAMP(jt, 0);
                        mbar_wait(&aux->sempty[sb], sph ^ 1);
                        tc_fence_after();
                        if (lane == 0) P4_STAMP(jt, 1);
                        for (int g = 0; g < nstg_p; ++g, ++pc) {
                            const uint32_t st = pc % P4P_NSTAGE, ph = (pc / P4P_NSTAGE) & 1;
                            mbar_wait(&aux->tfull[st], ph);
                            tc_fence_after();
                            const uint64_t bst = bdesc0 + static_cast<uint64_t>(st * (P4P_STAGE >> 4));
                            if (p.dbg_flags & 512)
                                umma2_commit_mc_e(smem_u32(&aux->tempty[st]), 0x3);
                            else
                                umma2_ts_stage8(dcol, tmem + X_COL + g * 64, bst, idesc, g != 0,
                                                smem_u32(&aux->tempty[st]), 0x3);
                        }
                        umma2_commit_mc_e(smem_u32(&aux->sfull[sb]), 0x3);
                        if (lane == 0) P4_STAMP(jt, 2);
                        if (t == t1 - 1) umma2_commit_mc_e(smem_u32(&aux->xfree), 0x3);
                    }
                    ++sg;
                }
            }
        } else if (warp == 10) {
            // -------- P mover: staging -> the consumer of this half (rank 2 + half)
            if (lane == 0) {
                uint32_t jt = 0;
                const uint32_t dst_rank = 2 + half;
                while (sch.next(rg, t0, t1, seg)) {
                    for (int t = t0; t < t1; ++t, ++jt) {
                        const uint32_t b = jt % P4_NPS, ph = (jt / P4_NPS) & 1;        // staging
                        const uint32_t sl = jt % P4_NSLOT, sph = (jt / P4_NSLOT) & 1;  // consumer slot
                        mbar_wait(&aux->pready[b], ph);
                        if (half == 0) P4_STAMP(jt, 5);
                        mbar_wait(&aux->pslot_free[sl], sph ^ 1);
                        if (half == 0) P4_STAMP(jt, 6);
                        const uint32_t dst = mapa_shared(smem_u32(smem + P4Q_OFF_P + sl * P4_PBYTES), dst_rank);
                        const uint32_t rbar = mapa_shared(smem_u32(&aux->pfull[sl]), dst_rank);
                        const uint32_t ck = P4_PBYTES / PC_P_CHUNKS;
                        if (p.dbg_flags & 128) mbar_arrive_remote(rbar);
                        else
                        for (int c = 0; c < PC_P_CHUNKS; ++c) {
                            asm volatile(
                                "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes"
                                " [%0], [%1], %2, [%3];" ::"r"(dst + c * ck),
                                "r"(smem_u32(sPS + b * P4_PBYTES) + c * ck), "r"(ck), "r"(rbar)
                                : "memory");
                            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                            asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");
                        }
                        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                        if (half == 0) P4_STAMP(jt, 7);
                        mbar_arrive(&aux->pstage_free[b]);
                    }
                }
                asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            }
        } else {
            // -------- softmax warps 0-7 (as dcp_pc_kernel, default variant): warp w -> rows
            // 32*(w%4)+lane of this CTA's half, slot half w/4 of each tile
            const int q = warp & 3, h = warp >> 2;
            const int r = q * 32 + lane;
            const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
            const uint32_t sempty_l = mapa_shared(smem_u32(&aux->sempty[0]), 0);
            const uint32_t xready_l = mapa_shared(smem_u32(&aux->xready), 0);
            uint32_t jt = 0, sg = 0;
            while (sch.next(rg, t0, t1, seg)) {
                const int row = rg * P4_RG + static_cast<int>(half) * P4_R + r;
                const float2 ab = p.row_ab[row];
                const int tg = p.row_tgt[row];
                mbar_wait(&aux->xfree, (sg & 1) ^ 1);
                tc_fence_after();
                {
                    const uint4 *src = reinterpret_cast<const uint4 *>(p.X_pos + static_cast<size_t>(row) * d * 2) +
                                       h * (d / 16);
                    const int ncol = d / 4;
                    for (int c0 = 0; c0 < ncol; c0 += 32) {
                        uint32_t w[32];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const uint4 v = src[c0 / 4 + u];
                            w[4 * u] = v.x; w[4 * u + 1] = v.y; w[4 * u + 2] = v.z; w[4 * u + 3] = v.w;
                        }
                        tmem_st32(tmem + lane_base + X_COL + h * ncol + c0, w);
                    }
                    tmem_wait_st();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_remote(xready_l);
                float lacc = 0.f, mx = -INFINITY;
                for (int t = t0; t < t1; ++t, ++jt) {
                    const uint32_t sb = jt & 1, sph = (jt >> 1) & 1;
                    mbar_wait(&aux->sfull[sb], sph);
                    tc_fence_after();
                    if (threadIdx.x == 0 && half == 0) P4_STAMP(jt, 3);
                    float e[64];
                    {
                        float v0[32], v1[32];
                        const uint32_t ta = tmem + lane_base + S_COL + sb * P4_TILE + h * 64;
                        tmem_ld32(ta, v0);
                        tmem_ld32(ta + 32, v1);
                        tmem_wait_ld();
                        if (threadIdx.x == 0 && half == 0) P4_STAMP(jt, 12);
#pragma unroll
                        for (int k = 0; k < 32; ++k) {
                            e[k] = v0[k];
                            e[32 + k] = v1[k];
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive_remote_relaxed(sempty_l + sb * 8);
                    if (threadIdx.x == 0 && half == 0) P4_STAMP(jt, 14);
                    if (p.dbg_flags & 64) {  // timing experiment: protocol only
                        const uint32_t b = jt % P4_NPS, ph = (jt / P4_NPS) & 1;
                        mbar_wait(&aux->pstage_free[b], ph ^ 1);
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&aux->pready[b]);
                        continue;
                    }
                    const int base = t * P4_TILE + h * 64;
                    const int nval = p.n_slots - base;
                    uint32_t w[32];
                    if (nval >= 64) {
#pragma unroll
                        for (int k = 0; k < 64; k += 2) ffma2_scalar(e[k], e[k + 1], ab.x, -ab.y);
                    } else {
#pragma unroll
                        for (int k = 0; k < 64; ++k) e[k] = k < nval ? fmaf(e[k], ab.x, -ab.y) : -INFINITY;
                    }
                    const bool hit = tg >= base && tg < base + 64;
                    if (__any_sync(__activemask(), hit)) {
                        if (hit) {
                            const int kt = tg - base;
#pragma unroll
                            for (int k = 0; k < 64; ++k)
                                if (k == kt) {
                                    p.ttgt[row] = e[k] - p.margin_l2;
                                    e[k] = -INFINITY;
                                }
                        }
                    }
                    float la[8] = {0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f, 0.f};
                    float ma[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                    for (int k = 0; k < 64; k += 2) {
                        const float p0 = ex2_approx(e[k]), p1 = ex2_approx(e[k + 1]);
                        const int c = (k >> 1) & 3;
                        fadd2_acc(la[2 * c], la[2 * c + 1], p0, p1);
                        fmax3_acc(ma[c], e[k], e[k + 1]);
                        w[k >> 1] = pack_bf16x2(p0, p1);
                    }
                    lacc += ((la[0] + la[1]) + (la[2] + la[3])) + ((la[4] + la[5]) + (la[6] + la[7]));
                    mx = fmaxf(mx, fmaxf(fmaxf(ma[0], ma[1]), fmaxf(ma[2], ma[3])));
                    // P -> staging, the consumer's K-major SW128 A layout (chunk h = slots 64h..)
                    const uint32_t b = jt % P4_NPS, ph = (jt / P4_NPS) & 1;
                    if (threadIdx.x == 0 && half == 0) P4_STAMP(jt, 13);
                    mbar_wait(&aux->pstage_free[b], ph ^ 1);
                    if (threadIdx.x == 0 && half == 0) P4_STAMP(jt, 15);
                    const uint32_t rowa = smem_u32(sPS + b * P4_PBYTES + h * 16384 + (r >> 3) * 1024 + (r & 7) * 128);
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        st_shared_v4(rowa + ((u ^ (r & 7)) << 4), w[4 * u], w[4 * u + 1], w[4 * u + 2], w[4 * u + 3]);
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&aux->pready[b]);
                    if (threadIdx.x == 0 && half == 0) P4_STAMP(jt, 4);
                }
                aux->red_l[h][r] = lacc;
                aux->red_mx[h][r] = mx;
                named_bar_sync(1, 256);
                if (h == 0) {
                    const size_t sr = static_cast<size_t>(seg) * P4_RG + half * P4_R + r;
                    p.seg_l[sr] = aux->red_l[0][r] + aux->red_l[1][r];
                    p.seg_mx[sr] = fmaxf(aux->red_mx[0][r], aux->red_mx[1][r]);
                }
                named_bar_sync(1, 256);
                ++sg;
            }
        }
    } else {
        // ================================================================= CONSUMER PAIR
        uint8_t *sP = smem + P4Q_OFF_P;
        uint8_t *sT = smem + P4Q_OFF_T;
        if (warp == 8) {
            // -------- TMA: this CTA's 128 d columns of each 256-d block, on leader 2's barrier
            if (lane == 0) {
                uint32_t qc = 0;
                while (sch.next(rg, t0, t1, seg)) {
                    for (int t = t0; t < t1; ++t)
                        for (int g = 0; g < nstg_q; ++g, ++qc) {
                            const uint32_t st = qc % P4Q_NSTAGE, ph = (qc / P4Q_NSTAGE) & 1;
                            mbar_wait(&aux->qempty[st], ph ^ 1);
                            if (p.dbg_flags & 8) {
                                if (is_leader) mbar_arrive(&aux->qfull[st]);
                                continue;
                            }
                            if (is_leader) mbar_arrive_expect_tx(&aux->qfull[st], 2 * P4Q_STAGE);
                            tma2_load_3d(smem_u32(sT + st * P4Q_STAGE), &tm4q, mapa_shared(smem_u32(&aux->qfull[st]), 2),
                                         0, t * P4_TILE, g * 4 + 2 * static_cast<int>(half));
                        }
                }
            }
        } else if (warp == 9) {
            if (is_leader) {
                // -------- leader 2: GEMM 2 issue (M = 256, N = 256 d, K = 128 slots)
                const uint32_t sPa = smem_u32(sP), sTa = smem_u32(sT);
                const uint32_t idesc = umma_idesc_bf16(256, 256, 0, 1);
                uint32_t qc = 0, jt = 0, sg = 0;
                while (sch.next(rg, t0, t1, seg)) {
                    for (int t = t0; t < t1; ++t, ++jt) {
                        const bool first = (t == t0);
                        const uint32_t b = jt % P4_NSLOT, ph = (jt / P4_NSLOT) & 1;
                        mbar_wait(&aux->pfull[b], ph);
                        if (lane == 0) P4_STAMP(jt, 8);
                        mbar_wait(&aux->pfull_peer[b], ph);
                        if (lane == 0) P4_STAMP(jt, 9);
                        if (lane == 0 && !(p.dbg_flags & 128)) mbar_arrive_expect_tx(&aux->pfull[b], P4_PBYTES);  // arm the next use
                        __syncwarp();
                        tc_fence_after();
                        if (first && sg > 0) {
                            mbar_wait(&aux->oempty, (sg - 1) & 1);
                            tc_fence_after();
                        }
                        for (int g = 0; g < nstg_q; ++g, ++qc) {
                            const uint32_t st = qc % P4Q_NSTAGE, qph = (qc / P4Q_NSTAGE) & 1;
                            mbar_wait(&aux->qfull[st], qph);
                            tc_fence_after();
                            if (p.dbg_flags & 256)
                                umma2_commit_mc_e(smem_u32(&aux->qempty[st]), 0xC);
                            else
                                umma2_ss_stage8(tmem + g * 256, umma_desc_sw128(sPa + b * P4_PBYTES, 16, 1024),
                                                umma_desc_sw128(sTa + st * P4Q_STAGE, 16384, 1024), idesc, !first,
                                                smem_u32(&aux->qempty[st]), 0xC);
                        }
                        umma2_commit_mc_e(smem_u32(&aux->pslot_free[b]), 0x3);  // both producers: slot b free
                        if (lane == 0) P4_STAMP(jt, 10);
                        if (t == t1 - 1) umma2_commit_mc_e(smem_u32(&aux->ofull), 0xC);
                    }
                    ++sg;
                }
            } else if (lane == 0) {
                // -------- peer consumer: relay its P arrivals to leader 2
                uint32_t jt = 0;
                const uint32_t peer_l = mapa_shared(smem_u32(&aux->pfull_peer[0]), 2);
                while (sch.next(rg, t0, t1, seg))
                    for (int t = t0; t < t1; ++t, ++jt) {
                        const uint32_t b = jt % P4_NSLOT, ph = (jt / P4_NSLOT) & 1;
                        mbar_wait(&aux->pfull[b], ph);
                        P4_STAMP(jt, 11);
                        if (!(p.dbg_flags & 128)) mbar_arrive_expect_tx(&aux->pfull[b], P4_PBYTES);  // arm the next use
                        mbar_arrive_remote(peer_l + b * 8);
                    }
            }
        } else if (warp < 8) {
            // -------- O drain at a unit's end: this CTA's 128 rows, eight warps
            const int q = warp & 3, hcol = warp >> 2;
            const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
            const int r = q * 32 + lane;
            const uint32_t oempty_l = mapa_shared(smem_u32(&aux->oempty), 2);
            uint32_t sg = 0;
            while (sch.next(rg, t0, t1, seg)) {
                mbar_wait(&aux->ofull, sg & 1);
                tc_fence_after();
                float4 *dst = reinterpret_cast<float4 *>(p.seg_O + (static_cast<size_t>(seg) * P4_RG + half * P4_R + r) * d);
                for (int c0 = hcol * (d / 2); c0 < (hcol + 1) * (d / 2); c0 += 32) {
                    float o[32];
                    tmem_ld32(tmem + lane_base + c0, o);
                    tmem_wait_ld();
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        dst[c0 / 4 + u] = make_float4(o[4 * u], o[4 * u + 1], o[4 * u + 2], o[4 * u + 3]);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive_remote(oempty_l);
                ++sg;
            }
        }
    }
#undef P4_STAMP
    tc_fence_before();
    __syncthreads();
    // debug hook: every cluster's span (cycles of its rank-0 CTA) and unit count
    if (p.dbg && crank == 0 && threadIdx.x == 0 && (blockIdx.x >> 2) < 32) {
        unsigned long long g_end;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(g_end));
        p.dbg[1024 + (blockIdx.x >> 2)] = clock64() - t_start;
        if ((blockIdx.x >> 2) < 8) {
            p.dbg[1056 + (blockIdx.x >> 2)] = g_end - g_start;
        }
    }
    cluster_sync_all();
    if (warp == 9) {
        tc_fence_after();
        asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
    }
}

}  // namespace f2c
