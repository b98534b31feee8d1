// dcp_pc.cuh -- the fused DCP loss kernel, producer/consumer CTA-pair version
// (hot-path steps a2, a4, a5, a7, a9).
//
// A cluster of two CTAs owns one group of 128 compacted rows and a range of pool tiles
// (128 slots each):
//   producer (cluster rank 0): x_hat rows live in TMEM as the UMMA A operand (bf16);
//     GEMM 1  S[r, c] = <x_r, T_c>        M = 128 rows, N = 128 slots, K = d
//     (A from TMEM, B = pool chunk from smem), double-buffered S in TMEM so the softmax
//     of tile j overlaps GEMM 1 of tile j+1.  Softmax warps (rows on TMEM lanes):
//     e = S*a_r - b_r, margin on the target column (recorded apart, excluded),
//     p = 2^e -> running l_r, max_r in registers; P (bf16) is written in the
//     consumer's A-operand layout and shipped to the consumer's smem by a DSMEM bulk
//     copy (cp.async.bulk shared::cta -> shared::cluster, complete_tx on the
//     consumer's mbarrier).
//   consumer (cluster rank 1): O[128 rows x d] fp32 occupies all 512 TMEM columns;
//     GEMM 2  O[r, :] += sum_c P[r, c] T[c, :]   M = 128, N = 256 (d block), K = slots
//     (A = P from smem, B = pool chunk MN-major from smem).  At a unit's end eight warps
//     drain O to the segment partial (through smem + TMA stores for short units).
// The N x C logit matrix only exists as one 128x128 tile at a time (TMEM, then smem).
// The softmax reference b_r (R1) is fixed per row before the pass, identical across
// slots, so partials of different clusters / tiles / ranks add without rescaling; rows that
// fall far below it (large s) are re-run by the refinement pass (run_flag).
// Variants: EXCL (stale self-duplicates masked per tile, NEXT-3), out-of-pool cosine rows for
// hinge / max (NEXT-3), with K >= 2 (NEXT-1) their weights w_c through an smem ring.
// A last row group of <= 64 rows runs as a 64-row tail unit (M = 64 MMAs: half the MMA work
// and energy of a padded group), and on long single-wave schedules the row groups of a tile
// range keep within PC_PACE_LAG tiles of each other (relaxed progress counters in global
// memory) so they share each pool tile through L2.
#pragma once
#include "dcp_main.cuh"
#include "sm100.cuh"

namespace f2c {

constexpr int PC_R = 128;                // rows per group (TMEM lanes)
constexpr int PC_TILE = 128;             // slots per tile (GEMM-1 N, GEMM-2 K)
constexpr int PC_THREADS = 352;          // 11 warps
constexpr int PC_P_NSTAGE = 4;           // producer pool ring: stages of [2 chunks x 128 slots x 64 d]
constexpr int PC_P_STAGE_BYTES = 32768;
constexpr int PC_Q_NSTAGE = 2;           // consumer pool ring: same stages (one d block each)
constexpr int PC_STAGE_BYTES = 65536;    // up to 4 chunks of 16 KB, one 3D TMA box
constexpr int PC_PBYTES = PC_R * PC_TILE * 2;  // one P tile, bf16 = 32 KB

// producer smem
constexpr int PCP_OFF_T = 0;                                         // 4 x 32 KB
constexpr int PCP_OFF_PS = PCP_OFF_T + PC_P_NSTAGE * PC_P_STAGE_BYTES;  // 2 x 32 KB P staging
constexpr int PCP_OFF_AUX = PCP_OFF_PS + 2 * PC_PBYTES;
// consumer smem
constexpr int PCQ_OFF_P = 0;                              // 2 x 32 KB P slots
constexpr int PCQ_OFF_T = PCQ_OFF_P + 2 * PC_PBYTES;      // 2 x 64 KB pool stages
constexpr int PCQ_OFF_AUX = PCQ_OFF_T + PC_Q_NSTAGE * PC_STAGE_BYTES;
constexpr int PC_OFF_AUX = PCP_OFF_AUX > PCQ_OFF_AUX ? PCP_OFF_AUX : PCQ_OFF_AUX;
// producer: the out-of-pool rows' weight ring (K >= 2), PC_WRING x 128 fp32 w_c; deep enough that the
// TMA warp (a tile or two ahead of the softmax warps) never waits on it
constexpr int PC_WRING = 8;
constexpr int PC_WBYTES = PC_TILE * 4;
constexpr int PC_OFF_WRING = PC_OFF_AUX + 4096;
// consumer: O-drain staging, one [32 rows x 16 fp32] TMA-store box per drain warp
constexpr int PC_OFF_OSTG = PC_OFF_WRING + PC_WRING * PC_WBYTES;
constexpr int PC_OSTG_BYTES = 8 * 2048;
constexpr int PC_SMEM_BYTES = PC_OFF_OSTG + PC_OSTG_BYTES + 1024;   // with the drain staging
constexpr int PC_SMEM_BYTES_NOSTG = PC_OFF_OSTG + 1024;            // without it

// the same struct (same offsets) in both CTAs, so multicast commits can target a
// barrier of the peer by its local offset
constexpr int PC_MAX_UNITS = 32;
constexpr int PC_PACE_LAG = 24;      // tiles a unit may run ahead of its range's slowest row group
constexpr int PC_PACE_EVERY = 8;     // progress published / checked every 8 tiles
constexpr int PC_PACE_SPINS = 8192;  // polls per unit (>= 256 ns each) before pacing is dropped for it
constexpr int PC_P_CHUNKS = 4;     // P transfer pieces (see the mover)
// (Measured and rejected: the softmax warps storing P straight into the consumer's smem with
// st.shared::cluster + fence.proxy.async.shared::cluster instead of staging + one bulk copy
// took 6300 cycles per tile against 2150.)  // host-checked: ceil(R*S/G) <= 32 for every R <= R_max/128

// the cluster's unit list, computed once per CTA (TPSched) and read by every role
struct PCUnitIt {
    const int4 *u;
    int n, i;
    __device__ bool next(int &rg, int &t0, int &t1, int &seg) {
        if (i >= n) return false;
        const int4 v = u[i++];
        rg = v.x;
        t0 = v.y;
        t1 = v.z;
        seg = v.w;
        return true;
    }
};

struct PCAux {
    // producer
    uint64_t tfull[PC_P_NSTAGE], tempty[PC_P_NSTAGE];
    uint64_t sfull[2], sempty[2];
    uint64_t xready, xfree;
    uint64_t pready[2], pstage_free[2];
    uint64_t pslot_free[2];            // arrived by the consumer's multicast commit
    uint64_t wfull[PC_WRING], wempty[PC_WRING];  // the out-of-pool rows' weight ring (K >= 2)
    // consumer
    uint64_t qfull[PC_Q_NSTAGE], qempty[PC_Q_NSTAGE];
    uint64_t pfull[2];                 // complete_tx by the producer's bulk copy
    uint64_t ofull, oempty;
    uint32_t tmem_base;
    uint32_t pad;
    float red_l[2][PC_R];
    float red_mx[2][PC_R];
    int red_arg[2][PC_R];
    int4 units[PC_MAX_UNITS];          // this cluster's (row group, t0, t1, segment) list
    int n_units;
    int single_wave;                   // every cluster runs at most one unit (range pacing)
    int range_len;                     // tiles per range (n_tiles / S, the same in every cluster)
};
static_assert(sizeof(PCAux) <= 4096, "PCAux must fit the aux region");

struct PCParams {
    int d;                 // feature dim (multiple of 128, <= 512)
    int n_slots;           // occupied slots of this shard
    const int *n_pos;      // device: in-pool rows
    const int *n_rows;     // device: rows to process (n_pos, or neg0 + N_neg with NEXT-3 neg rows)
    const int *neg0;       // device: first out-of-pool row (NEXT-3 hinge / max)
    int neg_mode;          // 0; 1 = hinge (p = [cos > 0] w_c, l = sum relu(cos)); 2 = max cos
    int *seg_arg;          // [S][128] local argmax slot (neg_mode 2)
    const float2 *row_ab;  // [R_max] (a_r, b_r)
    const int *row_tgt;    // [R_max] local target slot or -1
    const uint8_t *X_pos;  // [R_max, d] bf16 compacted rows
    const float *wslot;    // K >= 2: per-slot 1/||T_bar_c|| (fp32, padded by one tile; the NEXT-3
                           // out-of-pool rows' weight ring reads it); null for K = 1
    const int *S_sched;    // device: the range count S of this call's schedule (k_compact, pc_sched_cost)
    int kf;                // features per slot K: GEMM 1 contracts x_hat with the K raw rows of a slot
                           // (K d columns; 1/K is folded into a_r, so the logits use the exact mean)
    float margin_l2;       // s * m * log2(e)
    float *ttgt;           // [R_max]
    float *seg_l;          // [S][128]
    float *seg_mx;         // [S][128]
    float *seg_O;          // [S][128][d]
    // NEXT-3 "exclude stale self-duplicates" (excl != 0): per 128-slot tile t, entries
    // [dup_off[t], dup_off[t+1]) of dup_list = (local slot, label hash entry) of the stale
    // duplicates in that tile; a row skips the ones of its own hash entry row_hent[r]
    int excl;
    const int *dup_off;
    const int2 *dup_list;
    const int *row_hent;
    int drain_tma;         // O drain through smem staging + TMA stores (short units); else direct
                           // stores (launched without the staging smem)
    unsigned long long *dbg;
    int dbg_cluster;       // the cluster whose per-tile clocks the debug hook records
    const int *run_flag;   // refinement pass (R1 fallback): run only if *run_flag != 0
    // Range pacing (single-wave schedules with a 64-row tail unit, <= 8 row groups, ranges of
    // >= 512 tiles): every unit's producer publishes its progress through its tile range,
    // (epoch << 32) | tiles issued, with relaxed stores, and stays at most PC_PACE_LAG tiles ahead
    // of the slowest row group of the same range, so the range's row groups keep sharing each
    // pool tile through L2 (the faster tail unit drifted ahead and re-read part of the pool from
    // DRAM)
    unsigned long long *prog;  // [U] per unit (seg = range * n_rg + row group)
    unsigned int epoch;        // this launch's tag (never 0)
    int dbg_flags;         // timing experiments only: 1 = skip P smem writes, 128 = skip DSMEM copy,
                           // 4 / 8 = no producer / consumer pool loads, 16 = no softmax arithmetic,
                           // 16384 = every CTA loads only pool tiles 0-15 (L2-hot; same smem traffic),
                           // 64 = softmax warps idle (barrier protocol only), 256 = no GEMM-2 MMAs
};

__device__ __forceinline__ uint32_t cluster_ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cluster_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t cta) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(cta));
    return r;
}
// D[tmem] (+)= A[tmem] * B[smem]  (A operand from tensor memory)
__device__ __forceinline__ void umma_bf16_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                             uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
// Warp-wide issue helpers: the whole warp runs the issue loop (operands stay in
// uniform registers) and exactly one elected lane executes the instruction.
__device__ __forceinline__ void umma_ts_e(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p, e;\n.reg .b32 r;\nelect.sync r|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_ss_e(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n.reg .pred p, e;\n.reg .b32 r;\nelect.sync r|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}
__device__ __forceinline__ void umma_commit_e(uint64_t *bar) {
    asm volatile(
        "{\n.reg .pred e;\n.reg .b32 r;\nelect.sync r|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(bar))
        : "memory");
}

// One producer stage of GEMM 1 in a single elected issue: 8 TS MMAs (chunk c = i>>2 of the
// 32 KB stage, K step k = i&3) and the commit that releases the stage.  One asm block, one
// elect.sync: the operands go to uniform registers once per stage, not once per MMA.
__device__ __forceinline__ void umma_ts_stage8(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                               uint32_t acc0, uint64_t *bar) {
    asm volatile(
        "{\n.reg .pred e, p, t;\n.reg .b32 r;\n"
        "elect.sync r|e, 0xffffffff;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "setp.eq.b32 t, 0, 0;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1+8], %6, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1+16], %7, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1+24], %8, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1+32], %9, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1+40], %10, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1+48], %11, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1+56], %12, %3, t;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc0), "r"(smem_u32(bar)), "l"(bdesc + 2), "l"(bdesc + 4),
        "l"(bdesc + 6), "l"(bdesc + 1024), "l"(bdesc + 1026), "l"(bdesc + 1028), "l"(bdesc + 1030)
        : "memory");
}
// The same stage for an fp32 pool (kind::tf32, K = 8 per MMA: a 128-B chunk row is 32 fp32, so the
// A / B descriptor steps are those of bf16)
__device__ __forceinline__ void umma_ts_stage8_tf32(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc,
                                               uint32_t acc0, uint64_t *bar) {
    asm volatile(
        "{\n.reg .pred e, p, t;\n.reg .b32 r;\n"
        "elect.sync r|e, 0xffffffff;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "setp.eq.b32 t, 0, 0;\n"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+8], %6, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+16], %7, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+24], %8, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+32], %9, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+40], %10, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+48], %11, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1+56], %12, %3, t;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n}\n" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc0), "r"(smem_u32(bar)), "l"(bdesc + 2), "l"(bdesc + 4),
        "l"(bdesc + 6), "l"(bdesc + 1024), "l"(bdesc + 1026), "l"(bdesc + 1028), "l"(bdesc + 1030)
        : "memory");
}
// One consumer stage of GEMM 2: 8 SS MMAs over the tile's 128 slots (K steps of 16) and the
// commit that releases the pool stage.  a/b descriptors advance by +2 (32 B) / +128 (2 KB)
// per K step, plus +1024 (16 KB) for the A chunk after 4 steps.
__device__ __forceinline__ void umma_ss_stage8(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                               uint32_t acc0, uint64_t *bar) {
    asm volatile(
        "{\n.reg .pred e, p, t;\n.reg .b32 r;\n"
        "elect.sync r|e, 0xffffffff;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "setp.eq.b32 t, 0, 0;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %6, %7, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %8, %9, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %10, %11, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %12, %13, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %14, %15, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %16, %17, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %18, %19, %3, t;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%5];\n}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc0), "r"(smem_u32(bar)),
        "l"(adesc + 2), "l"(bdesc + 128), "l"(adesc + 4), "l"(bdesc + 256), "l"(adesc + 6), "l"(bdesc + 384),
        "l"(adesc + 1024), "l"(bdesc + 512), "l"(adesc + 1026), "l"(bdesc + 640), "l"(adesc + 1028),
        "l"(bdesc + 768), "l"(adesc + 1030), "l"(bdesc + 896)
        : "memory");
}
#include "gemm1_tile.inc"

__device__ __forceinline__ void umma_commit_mc_e(uint64_t *bar, uint16_t mask) {
    asm volatile(
        "{\n.reg .pred e;\n.reg .b32 r;\nelect.sync r|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;\n}\n" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
// arrive on the barrier at the same smem offset in every CTA of `mask`
__device__ __forceinline__ void umma_commit_mc(uint64_t *bar, uint16_t mask) {
    asm volatile(
        "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;" ::"r"(
            smem_u32(bar)),
        "h"(mask)
        : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile(
        "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
        "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
        "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
        "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
        "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
        "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),
        "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
        "r"(v[29]), "r"(v[30]), "r"(v[31])
        : "memory");
}
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *m, uint64_t *bar, int x, int y, int z) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
        : "memory");
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
          "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}
// TMA store of one 2D box from shared memory (bulk async-group)
__device__ __forceinline__ void tma_store_2d(const CUtensorMap *m, uint32_t src, int x, int y) {
    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
                     reinterpret_cast<uint64_t>(m)),
                 "r"(src), "r"(x), "r"(y)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
__device__ __forceinline__ void tmem_wait_st() {
    asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
}

// EXCL: the NEXT-3 "exclude stale self-duplicates" variant, a separate instantiation so the
// default softmax loop is compiled exactly as without it (measured: a runtime flag there cost
// 10 % at c3)
// NEG: the NEXT-3 hinge / max variants, whose out-of-pool rows run through the kernel as cosine rows
// (K >= 2: with their weights through an smem ring); the default instantiation carries none of it
// TF32: an fp32 pool (F2C_F32, d <= 256): GEMM 1 in kind::tf32 over the fp32 rows with x_hat as fp32 in
// TMEM (d columns); GEMM 2 and everything after it read the pool's bf16 shadow, unchanged
template <bool EXCL, bool NEG, bool TF32>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(PC_THREADS, 1)
    dcp_pc_kernel(const __grid_constant__ CUtensorMap tm3p, const __grid_constant__ CUtensorMap tm3q,
                  const __grid_constant__ CUtensorMap tmO, const PCParams p) {
    // the refinement pass exits before any barrier or TMEM allocation unless a row needs it
    // (every CTA reads the same flag, so whole clusters exit together)
    if (p.run_flag != nullptr && *p.run_flag == 0) return;
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~static_cast<uintptr_t>(1023));
    PCAux *aux = reinterpret_cast<PCAux *>(smem + PC_OFF_AUX);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const uint32_t crank = cluster_ctarank();
    const int d = p.d;
    const int nchunk = d >> 6;                  // 64-wide d chunks
    // producer stages: 2 chunks (32 KB) of the K d-wide raw rows of a tile (NEXT-1: GEMM 1 contracts
    // over K d, stage g pairs with x_hat stage g mod (d / 128)); consumer stages: one GEMM-2 d block
    // (2 or 4 chunks) of T_bar
    const int cps_p = 2, xstg = TF32 ? d / 64 : nchunk / 2, nstg_p = xstg * p.kf;
    const int cps = (d % 256 == 0) ? 4 : 2;
    const int nstg = nchunk / cps;
    const uint32_t stage_bytes = static_cast<uint32_t>(cps) * 16384;
    const int n_rows = *p.n_rows;
    const int neg0 = *p.neg0;
    const int n_rg = (n_rows + PC_R - 1) / PC_R;
    const int n_tiles = (p.n_slots + PC_TILE - 1) / PC_TILE;
    // 64-row tail unit: the last row group with at most 64 rows runs both GEMMs with M = 64
    // (cta_group::1 M = 64 keeps MMA row r on TMEM lane 32 (r / 16) + r % 16: lanes 0-15 of each
    // quadrant; profiles/r01c_umma2_probe.txt) -- half the MMA work and energy of a padded
    // 128-row unit.  Default variant only (the out-of-pool rows of hinge / max keep 128).
    // (dbg_flags 32768: off, for A/B runs)
    auto tail64 = [&](int g) {
        return p.neg_mode == 0 && g == n_rg - 1 && n_rows - g * PC_R <= 64 && !(p.dbg_flags & 32768);
    };
    if (p.dbg && threadIdx.x == 0 && (blockIdx.x >> 1) == static_cast<unsigned>(p.dbg_cluster)) {  // kernel-span clocks (debug hook)
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        p.dbg[1024 + (blockIdx.x & 1) * 4] = clock64();
        p.dbg[1025 + (blockIdx.x & 1) * 4] = gt;
    }

    // debug hook: prologue stamps [1040 + 8 * cta + k] of the recorded cluster
    const bool dbgc = p.dbg && (blockIdx.x >> 1) == static_cast<unsigned>(p.dbg_cluster);
#define PC_STAMP(k) do { if (dbgc) p.dbg[1040 + (blockIdx.x & 1) * 8 + (k)] = clock64(); } while (0)
    if (threadIdx.x == 0) PC_STAMP(0);
    if (threadIdx.x == 0) {
        for (int i = 0; i < PC_P_NSTAGE; ++i) {
            mbar_init(&aux->tfull[i], 1);
            mbar_init(&aux->tempty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&aux->sfull[i], 1);
            mbar_init(&aux->sempty[i], 8);
            mbar_init(&aux->pready[i], 8);
            mbar_init(&aux->pstage_free[i], 1);
            mbar_init(&aux->pslot_free[i], 1);
            mbar_init(&aux->pfull[i], 1);
        }
        mbar_init(&aux->xready, 8);
        mbar_init(&aux->xfree, 1);
        for (int i = 0; i < PC_Q_NSTAGE; ++i) {
            mbar_init(&aux->qfull[i], 1);
            mbar_init(&aux->qempty[i], 1);
        }
        mbar_init(&aux->ofull, 1);
        mbar_init(&aux->oempty, 8);
        for (int i = 0; i < PC_WRING; ++i) {
            mbar_init(&aux->wfull[i], 1);
            mbar_init(&aux->wempty[i], 8);  // every softmax warp of a weight unit
        }
        if (crank == 1 && !(p.dbg_flags & 128)) {  // arm both P slots before the producer can copy into them
            mbar_arrive_expect_tx(&aux->pfull[0], PC_PBYTES);
            mbar_arrive_expect_tx(&aux->pfull[1], PC_PBYTES);
        }
        fence_mbar_init();
        TPSched ts;
        ts.init(blockIdx.x >> 1, gridDim.x >> 1, n_rg, n_tiles, *p.S_sched);
        int n = 0, a, b, c, s;
        while (n < PC_MAX_UNITS && ts.next(a, b, c, s)) aux->units[n++] = make_int4(a, b, c, s);
        aux->n_units = n;
        aux->single_wave = ts.U <= ts.G;
        aux->range_len = n_tiles / ts.S;
        PC_STAMP(1);
    }
    if (warp == 9) {
        tma_prefetch_desc(&tm3p);
        tma_prefetch_desc(&tm3q);
        tma_prefetch_desc(&tmO);
        tmem_alloc(&aux->tmem_base, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    cluster_sync_all();
    tc_fence_after();
    if (threadIdx.x == 0) PC_STAMP(2);
    const uint32_t tmem = aux->tmem_base;

    PCUnitIt sch{aux->units, aux->n_units, 0};
    int rg, t0, t1, seg;

    if (crank == 0) {
        // ================================================================= PRODUCER
        uint8_t *sT = smem + PCP_OFF_T;
        uint8_t *sPS = smem + PCP_OFF_PS;
        constexpr uint32_t X_COL = 0, S_COL = 256;  // x_hat (A operand) | two S buffers
        if (warp == 8) {
            // -------- TMA: pool stages [cps chunks x 128 slots x 64 d] (3D box)
            if (lane == 0) {
                uint32_t pc = 0;
                uint32_t wc_n = 0;
                // (only where it pays: a 64-row tail unit -- the row group that drifts ahead --, few row
                // groups and long ranges; measured 1.5-8.5 % slower at c2 / c1 / c3r_8 otherwise)
                const bool pace = p.prog != nullptr && aux->single_wave && n_rg >= 2 && n_rg <= 8 &&
                                  tail64(n_rg - 1) && aux->range_len >= 512;
                while (sch.next(rg, t0, t1, seg)) {
                    int spins = 0;  // (per unit: a stalled peer costs at most PC_PACE_SPINS polls per unit)
                    const bool wmu = NEG && p.wslot != nullptr && p.neg_mode != 0 && rg * PC_R + PC_R - 1 >= neg0;
                    unsigned long long *pg0 = pace ? p.prog + (seg - rg) : nullptr;  // this range's row groups
                    for (int t = t0; t < t1; ++t) {
                        if (pace && ((t - t0) % PC_PACE_EVERY) == 0) {
                            const unsigned long long mine = (static_cast<unsigned long long>(p.epoch) << 32) |
                                                            static_cast<unsigned long long>(t - t0);
                            asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(pg0 + rg), "l"(mine) : "memory");
                            while (spins < PC_PACE_SPINS) {  // wait while > LAG tiles ahead of the slowest
                                long long slow = 1ll << 40;
                                for (int g = 0; g < n_rg; ++g) {
                                    unsigned long long v;
                                    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(pg0 + g) : "memory");
                                    const long long dn = (v >> 32) == p.epoch ? static_cast<long long>(v & 0xffffffffull) : 0;
                                    slow = dn < slow ? dn : slow;
                                }
                                if (slow + PC_PACE_LAG >= t - t0) break;
                                ++spins;
                                __nanosleep(256);
                            }
                        }
                        if (wmu) {  // the tile's fp32 weights w_c (512 B) -> weight ring
                            const uint32_t wb = wc_n % PC_WRING;
                            mbar_wait(&aux->wempty[wb], ((wc_n / PC_WRING) & 1) ^ 1);
                            mbar_arrive_expect_tx(&aux->wfull[wb], PC_WBYTES);
                            asm volatile(
                                "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], 512, [%2];" ::"r"(
                                    smem_u32(smem + PC_OFF_WRING + wb * PC_WBYTES)),
                                "l"(reinterpret_cast<uint64_t>(p.wslot + static_cast<size_t>(t) * PC_TILE)),
                                "r"(smem_u32(&aux->wfull[wb]))
                                : "memory");
                            ++wc_n;
                        }
                        for (int g = 0; g < nstg_p; ++g, ++pc) {
                            const uint32_t st = pc % PC_P_NSTAGE, ph = (pc / PC_P_NSTAGE) & 1;
                            mbar_wait(&aux->tempty[st], ph ^ 1);
                            if (p.dbg_flags & 4) {  // timing experiment: no pool loads
                                mbar_arrive(&aux->tfull[st]);
                                continue;
                            }
                            mbar_arrive_expect_tx(&aux->tfull[st], PC_P_STAGE_BYTES);
                            const int tl = (p.dbg_flags & 16384) ? (t & 15) : t;  // 16384: hot tiles (experiment)
                            tma_load_3d(sT + st * PC_P_STAGE_BYTES, &tm3p, &aux->tfull[st], 0, tl * PC_TILE, g * cps_p);
                        }
                    }
                    if (pace) {  // range done: never hold the others back
                        const unsigned long long fin = (static_cast<unsigned long long>(p.epoch) << 32) | 0xfffffffull;
                        asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(pg0 + rg), "l"(fin) : "memory");
                    }
                }
            }
        } else if (warp == 9) {
            // -------- UMMA issuer: GEMM 1 (A = x_hat from TMEM, B = pool chunk K-major)
            {  // whole warp; one elected lane issues
                // descriptors advance by immediates: the start-address field holds addr >> 4
                const uint64_t bdesc0 = umma_desc_sw128(smem_u32(sT), 16, 1024);
                uint32_t pc = 0, jt = 0, sg = 0;
                while (sch.next(rg, t0, t1, seg)) {
                    const uint32_t idesc = TF32 ? umma_idesc_tf32(tail64(rg) ? 64 : 128, PC_TILE, 0, 0)
                                                : umma_idesc_bf16(tail64(rg) ? 64 : 128, PC_TILE, 0, 0);
                    mbar_wait(&aux->xready, sg & 1);
                    if (lane == 0 && sg == 0) PC_STAMP(4);
                    tc_fence_after();
                    for (int t = t0; t < t1; ++t, ++jt) {
                        unsigned long long *dbg = (p.dbg && blockIdx.x == 2u * p.dbg_cluster && jt < 64 && lane == 0) ? p.dbg + jt * 16 : nullptr;
                        const uint32_t sb = jt & 1, sph = (jt >> 1) & 1;
                        const uint32_t dcol = tmem + S_COL + sb * PC_TILE;
                        if (!TF32 && nstg_p == 4 && p.kf == 1) {  // d = 512, K = 1: the whole tile in one elected issue
                            if (dbg) dbg[0] = clock64();
                            gemm1_tile_issue(dcol, tmem + X_COL, bdesc0, idesc, smem_u32(&aux->sempty[sb]), sph ^ 1,
                                             smem_u32(&aux->tfull[0]), smem_u32(&aux->tempty[0]), jt & 1,
                                             smem_u32(&aux->sfull[sb]));
                            pc += 4;
                        } else {
                        mbar_wait(&aux->sempty[sb], sph ^ 1);
                        tc_fence_after();
                        if (dbg) dbg[0] = clock64();
                        for (int g = 0; g < nstg_p; ++g, ++pc) {
                            const uint32_t st = pc % PC_P_NSTAGE, ph = (pc / PC_P_NSTAGE) & 1;
                            mbar_wait(&aux->tfull[st], ph);
                            tc_fence_after();
                            const uint64_t bst = bdesc0 + static_cast<uint64_t>(st * (PC_P_STAGE_BYTES >> 4));
                            if (TF32)
                                umma_ts_stage8_tf32(dcol, tmem + X_COL + (g % xstg) * 64, bst, idesc, g != 0, &aux->tempty[st]);
                            else
                                umma_ts_stage8(dcol, tmem + X_COL + (g % xstg) * 64, bst, idesc, g != 0, &aux->tempty[st]);
                        }
                        umma_commit_e(&aux->sfull[sb]);
                        }
                        if (dbg) dbg[1] = clock64();
                        if (t == t1 - 1) umma_commit_e(&aux->xfree);
                    }
                    ++sg;
                }
            }
        } else if (warp == 10) {
            // -------- P mover: staging buffer -> consumer's P slot (DSMEM bulk copy)
            if (lane == 0 && !(p.dbg_flags & 4096)) {
                uint32_t jt = 0;
                while (sch.next(rg, t0, t1, seg)) {
                    for (int t = t0; t < t1; ++t, ++jt) {
                        const uint32_t b = jt & 1, ph = (jt >> 1) & 1;
                        mbar_wait(&aux->pready[b], ph);
                        mbar_wait(&aux->pslot_free[b], ph ^ 1);
                        unsigned long long *dbg = (p.dbg && blockIdx.x == 2u * p.dbg_cluster && jt < 64) ? p.dbg + jt * 16 : nullptr;
                        if (dbg) dbg[4] = clock64();
                        const uint32_t dst = mapa_shared(smem_u32(smem + PCQ_OFF_P + b * PC_PBYTES), 1);
                        const uint32_t rbar = mapa_shared(smem_u32(&aux->pfull[b]), 1);
                        if (p.dbg_flags & 128) {  // timing experiment: no P transfer
                            asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
                        } else {
                            // in PC_P_CHUNKS pieces, at most two in flight:
                            // the SM's async-copy unit also serves the pool TMA loads, which would
                            // otherwise queue behind one long (DSMEM-rate) copy
                            const int nck = (p.dbg_flags & 8192) ? 1 : PC_P_CHUNKS;  // 8192: one piece (comparison)
                            const uint32_t ck = PC_PBYTES / nck;
                            for (int c = 0; c < nck; ++c) {
                                asm volatile(
                                    "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes"
                                    " [%0], [%1], %2, [%3];" ::"r"(dst + c * ck),
                                    "r"(smem_u32(sPS + b * PC_PBYTES) + c * ck), "r"(ck), "r"(rbar)
                                    : "memory");
                                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                                asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // two in flight
                            }
                            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                        }
                        if (dbg) dbg[5] = clock64();
                        mbar_arrive(&aux->pstage_free[b]);
                    }
                }
                asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
            }
        } else {
            // -------- softmax warps 0-7: warp w -> rows 32*(w%4)+lane, slot half w/4 (a 64-row
            // tail unit: rows 16*(w%4)+lane on lanes 0-15; lanes 16-31 idle)
            const int q = warp & 3, h = warp >> 2;
            const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
            {   // zero both S buffers once: TMEM lanes an M = 64 GEMM never writes must hold finite values
                uint32_t z[32];
#pragma unroll
                for (int k = 0; k < 32; ++k) z[k] = 0u;
                for (int c0 = 0; c0 < 2 * PC_TILE; c0 += 64) {
                    tmem_st32(tmem + lane_base + S_COL + c0 + h * 32, z);
                }
                tmem_wait_st();
            }
            uint32_t jt = 0, sg = 0, wc_n = 0;
            while (sch.next(rg, t0, t1, seg)) {
                const bool m64 = tail64(rg);
                const int r = m64 ? (lane < 16 ? q * 16 + lane : -1) : q * 32 + lane;
                const bool rv = r >= 0;
                const int row = rg * PC_R + (rv ? r : 0);
                const float2 ab = rv ? p.row_ab[row] : make_float2(0.f, INFINITY);
                const int tg = rv ? p.row_tgt[row] : -1;
                const int hent = EXCL && rv ? p.row_hent[row] : -1;
                // x_hat (this thread's row, d half h) -> TMEM A operand columns
                mbar_wait(&aux->xfree, (sg & 1) ^ 1);
                tc_fence_after();
                {
                    constexpr int ES = TF32 ? 4 : 2;
                    const uint4 *src = reinterpret_cast<const uint4 *>(p.X_pos + static_cast<size_t>(row) * d * ES) +
                                       h * (d * ES / 32);
                    const int ncol = d * ES / 8;  // 32-bit columns per half row (d/2 bf16 or fp32 elements)
                    for (int c0 = 0; c0 < ncol; c0 += 32) {
                        uint32_t w[32];
#pragma unroll
                        for (int u = 0; u < 8; ++u) {
                            const uint4 v = rv ? src[c0 / 4 + u] : make_uint4(0u, 0u, 0u, 0u);
                            w[4 * u] = v.x; w[4 * u + 1] = v.y; w[4 * u + 2] = v.z; w[4 * u + 3] = v.w;
                        }
                        tmem_st32(tmem + lane_base + X_COL + h * ncol + c0, w);
                    }
                    tmem_wait_st();
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&aux->xready);
                if (threadIdx.x == 0 && sg == 0) PC_STAMP(3);
                float lacc = 0.f, mx = -INFINITY;
                int barg = -1;
                // K >= 2: this unit's tiles bring their weights through the smem ring (it holds
                // out-of-pool rows of NEXT-3 hinge / max)
                const bool wmu = NEG && p.wslot != nullptr && p.neg_mode != 0 && rg * PC_R + PC_R - 1 >= neg0;
                // NEXT-3: out-of-pool rows compacted after the in-pool rows (a = 1/||x||, b = 0)
                // (the padding rows after n_rows take this path too: zero operands, discarded
                // results, and no divergence with the last out-of-pool rows of their warp)
                const bool negrow = NEG && p.neg_mode != 0 && row >= neg0;
                for (int t = t0; t < t1; ++t, ++jt) {
                    const uint32_t sb = jt & 1, sph = (jt >> 1) & 1;
                    mbar_wait(&aux->sfull[sb], sph);
                    tc_fence_after();
                    unsigned long long *dbg = (p.dbg && blockIdx.x == 2u * p.dbg_cluster && jt < 64 && threadIdx.x == 0) ? p.dbg + jt * 16 : nullptr;
                    if (dbg) dbg[2] = clock64();
                    if (p.dbg_flags & 64) {  // timing experiment: softmax warps only keep the protocol
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&aux->sempty[sb]);
                        if (wmu) {
                            mbar_wait(&aux->wfull[wc_n % PC_WRING], (wc_n / PC_WRING) & 1);
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&aux->wempty[wc_n % PC_WRING]);
                            ++wc_n;
                        }
                        const uint32_t b = jt & 1, ph = (jt >> 1) & 1;
                        if (!(p.dbg_flags & 4096)) {
                            mbar_wait(&aux->pstage_free[b], ph ^ 1);
                            __syncwarp();
                            if (lane == 0) mbar_arrive(&aux->pready[b]);
                        }
                        if (dbg) dbg[3] = clock64();
                        continue;
                    }
                    float e[64];
                    {
                        float v0[32], v1[32];
                        const uint32_t ta = tmem + lane_base + S_COL + sb * PC_TILE + h * 64;
                        tmem_ld32(ta, v0);
                        tmem_ld32(ta + 32, v1);
                        tmem_wait_ld();
#pragma unroll
                        for (int k = 0; k < 32; ++k) {
                            e[k] = v0[k];
                            e[32 + k] = v1[k];
                        }
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&aux->sempty[sb]);
                    if (wmu) mbar_wait(&aux->wfull[wc_n % PC_WRING], (wc_n / PC_WRING) & 1);  // weight ring
                    if (dbg) dbg[8] = clock64();
                    const int base = t * PC_TILE + h * 64;
                    const int nval = p.n_slots - base;  // valid slots in my 64-wide half
                    uint32_t w[32];
                    if (p.dbg_flags & 16) {  // timing experiment: no softmax arithmetic
#pragma unroll
                        for (int k = 0; k < 32; ++k) w[k] = __float_as_uint(e[2 * k]) & 0x3f803f80u;
                    } else if (!negrow) {
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
                        if constexpr (EXCL) {  // NEXT-3: drop this row's stale self-duplicates of tile t
                            const int o1 = p.dup_off[t + 1];
                            for (int o = p.dup_off[t]; o < o1; ++o) {
                                const int2 v = p.dup_list[o];
                                const int kt = v.x - base;
                                if (v.y == hent && kt >= 0 && kt < 64) {
#pragma unroll
                                    for (int k = 0; k < 64; ++k)
                                        if (k == kt) e[k] = -INFINITY;
                                }
                            }
                        }
                        // 2-wide packed sums (FADD2) and 3-input max (FMNMX3), 4 chains each for ILP
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
                    } else {
                        // cosine c = <x_hat, T_bar_c> w_c (w_c = 1 for K = 1; zero centers are
                        // no candidates for the max and contribute 0 to the hinge).
                        // Branch-free, four independent max chains (a per-element data-dependent
                        // branch here made these rows 5.8x slower than the softmax rows).
                        float pv[64];
                        if (!p.wslot) {
                            // K = 1: a_r = 1/||x|| > 0 scales every cosine of the row alike, so the
                            // hinge and the argmax work on the raw products e
#pragma unroll
                            for (int k = 0; k < 64; ++k) e[k] = k < nval ? e[k] : -INFINITY;
                            if (p.neg_mode == 1) {
                                float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                                for (int k = 0; k < 64; ++k) {
                                    s4[k & 3] += fmaxf(e[k], 0.f);
                                    pv[k] = e[k] > 0.f ? 1.f : 0.f;
                                }
                                lacc += ((s4[0] + s4[1]) + (s4[2] + s4[3])) * ab.x;
                            } else {
                                float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                                for (int k = 0; k < 64; k += 2) fmax3_acc(m4[(k >> 1) & 3], e[k], e[k + 1]);
                                const float m = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
                                int ka = -1;
#pragma unroll
                                for (int k = 63; k >= 0; --k) ka = e[k] == m ? k : ka;  // lowest slot on ties
                                const float c = m * ab.x;
                                if (ka >= 0 && c > mx) {  // strict: earlier tiles win ties
                                    mx = c;
                                    barg = base + ka;
                                }
#pragma unroll
                                for (int k = 0; k < 64; ++k) pv[k] = 0.f;
                            }
                        } else {
                        // K >= 2: the tile's fp32 weights w_c from the smem ring (the max cosine
                        // compares e_k w_k across slots, so w_c is not rounded)
                        float wv[64];
                        {
                            const float4 *src = reinterpret_cast<const float4 *>(smem + PC_OFF_WRING +
                                                                                 (wc_n % PC_WRING) * PC_WBYTES + h * 256);
#pragma unroll
                            for (int u = 0; u < 16; ++u) {
                                const float4 v = src[u];
                                const int k = 4 * u;
                                wv[k] = k < nval ? v.x : 0.f;
                                wv[k + 1] = k + 1 < nval ? v.y : 0.f;
                                wv[k + 2] = k + 2 < nval ? v.z : 0.f;
                                wv[k + 3] = k + 3 < nval ? v.w : 0.f;
                            }
                        }
                        // c_k / a_r = e_k w_k (a_r > 0 factored out as in the K = 1 path); zero
                        // centers (w = 0) are no candidates
#pragma unroll
                        for (int k = 0; k < 64; ++k) e[k] = wv[k] > 0.f ? e[k] * wv[k] : -INFINITY;
                        if (p.neg_mode == 1) {
                            float s4[4] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
                            for (int k = 0; k < 64; ++k) {
                                s4[k & 3] += fmaxf(e[k], 0.f);
                                pv[k] = e[k] > 0.f ? wv[k] : 0.f;
                            }
                            lacc += ((s4[0] + s4[1]) + (s4[2] + s4[3])) * ab.x;
                        } else {
                            float m4[4] = {-INFINITY, -INFINITY, -INFINITY, -INFINITY};
#pragma unroll
                            for (int k = 0; k < 64; k += 2) fmax3_acc(m4[(k >> 1) & 3], e[k], e[k + 1]);
                            const float m = fmaxf(fmaxf(m4[0], m4[1]), fmaxf(m4[2], m4[3]));
                            int ka = -1;
#pragma unroll
                            for (int k = 63; k >= 0; --k) ka = e[k] == m ? k : ka;  // lowest slot on ties
                            const float c = m * ab.x;
                            if (ka >= 0 && c > mx) {  // strict: earlier tiles win ties
                                mx = c;
                                barg = base + ka;
                            }
#pragma unroll
                            for (int k = 0; k < 64; ++k) pv[k] = 0.f;
                        }
                        }
#pragma unroll
                        for (int k = 0; k < 64; k += 2) w[k >> 1] = pack_bf16x2(pv[k], pv[k + 1]);
                    }
                    if (wmu) {  // this warp is done with the tile's weights
                        __syncwarp();
                        if (lane == 0) mbar_arrive(&aux->wempty[wc_n % PC_WRING]);
                        ++wc_n;
                    }
                    // P -> staging buffer in the consumer's K-major SW128 A layout:
                    // chunk h = slots [64h, 64h+64), row r: 128 B, 16-B unit u at u ^ (r & 7)
                    const uint32_t b = jt & 1, ph = (jt >> 1) & 1;
                    if (dbg) dbg[9] = clock64();
                    mbar_wait(&aux->pstage_free[b], ph ^ 1);
                    if (dbg) dbg[10] = clock64();
                    const uint32_t rowa = smem_u32(sPS + b * PC_PBYTES + h * 16384 + (r >> 3) * 1024 + (r & 7) * 128);
                    if (rv && !(p.dbg_flags & 1))
#pragma unroll
                    for (int u = 0; u < 8; ++u)
                        st_shared_v4(rowa + ((u ^ (r & 7)) << 4), w[4 * u], w[4 * u + 1], w[4 * u + 2],
                                     w[4 * u + 3]);
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&aux->pready[b]);
                    if (dbg) dbg[3] = clock64();
                }
                // segment end: l and max over both slot halves
                if (rv) {
                    aux->red_l[h][r] = lacc;
                    aux->red_mx[h][r] = mx;
                    aux->red_arg[h][r] = barg;
                }
                named_bar_sync(1, 256);
                if (h == 0 && rv) {
                    p.seg_l[static_cast<size_t>(seg) * PC_R + r] = aux->red_l[0][r] + aux->red_l[1][r];
                    const float m0 = aux->red_mx[0][r], m1 = aux->red_mx[1][r];
                    p.seg_mx[static_cast<size_t>(seg) * PC_R + r] = fmaxf(m0, m1);
                    if (negrow && p.neg_mode == 2) {  // first slot on ties
                        const int a0 = aux->red_arg[0][r], a1 = aux->red_arg[1][r];
                        const bool take1 = a1 >= 0 && (a0 < 0 || m1 > m0 || (m1 == m0 && a1 < a0));
                        p.seg_arg[static_cast<size_t>(seg) * PC_R + r] = take1 ? a1 : a0;
                    }
                }
                named_bar_sync(1, 256);
                ++sg;
            }
        }
    } else if (!(p.dbg_flags & 4096)) {  // (4096: timing experiment, producer alone)
        // ================================================================= CONSUMER
        uint8_t *sP = smem + PCQ_OFF_P;
        uint8_t *sT = smem + PCQ_OFF_T;
        if (warp == 8) {
            // -------- TMA: pool stages [cps chunks x 128 slots x 64 d] (3D box) = one d block
            if (lane == 0) {
                uint32_t qc = 0;
                while (sch.next(rg, t0, t1, seg)) {
                    for (int t = t0; t < t1; ++t)
                        for (int g = 0; g < nstg; ++g, ++qc) {
                            const uint32_t st = qc % PC_Q_NSTAGE, ph = (qc / PC_Q_NSTAGE) & 1;
                            mbar_wait(&aux->qempty[st], ph ^ 1);
                            if (p.dbg_flags & 8) {  // timing experiment: no pool loads
                                mbar_arrive(&aux->qfull[st]);
                                continue;
                            }
                            mbar_arrive_expect_tx(&aux->qfull[st], stage_bytes);
                            const int tl = (p.dbg_flags & 16384) ? (t & 15) : t;
                            tma_load_3d(sT + st * PC_STAGE_BYTES, &tm3q, &aux->qfull[st], 0, tl * PC_TILE, g * cps);
                        }
                }
            }
        } else if (warp == 9) {
            // -------- UMMA issuer: GEMM 2 (A = P K-major, B = pool MN-major, N = 256 d)
            {  // whole warp; one elected lane issues
                const uint32_t sPa = smem_u32(sP), sTa = smem_u32(sT);
                uint32_t qc = 0, jt = 0, sg = 0;
                while (sch.next(rg, t0, t1, seg)) {
                    const int mm = tail64(rg) ? 64 : 128;  // (M = 64 reads P rows 0-63 of each chunk)
                    const uint32_t idesc = cps == 4 ? umma_idesc_bf16(mm, 256, 0, 1) : umma_idesc_bf16(mm, 128, 0, 1);
                    for (int t = t0; t < t1; ++t, ++jt) {
                        const bool first = (t == t0);
                        const uint32_t b = jt & 1, ph = (jt >> 1) & 1;
                        mbar_wait(&aux->pfull[b], ph);
                        unsigned long long *dbg = (p.dbg && blockIdx.x == 2u * p.dbg_cluster + 1 && jt < 64 && lane == 0) ? p.dbg + jt * 16 : nullptr;
                        if (dbg) dbg[6] = clock64();
                        if (lane == 0 && !(p.dbg_flags & 128)) mbar_arrive_expect_tx(&aux->pfull[b], PC_PBYTES);  // arm the next use
                        __syncwarp();
                        tc_fence_after();
                        if (first && sg > 0) {
                            mbar_wait(&aux->oempty, (sg - 1) & 1);
                            tc_fence_after();
                        }
                        for (int g = 0; g < nstg; ++g, ++qc) {
                            const uint32_t st = qc % PC_Q_NSTAGE, qph = (qc / PC_Q_NSTAGE) & 1;
                            mbar_wait(&aux->qfull[st], qph);
                            tc_fence_after();
                            // 8 K steps of 16 slots: A = P (K-major, two 64-slot chunks), B = pool MN-major
                            if (p.dbg_flags & 256)  // timing / power experiment: no GEMM-2 MMAs
                                umma_commit_e(&aux->qempty[st]);
                            else
                                umma_ss_stage8(tmem + g * cps * 64, umma_desc_sw128(sPa + b * PC_PBYTES, 16, 1024),
                                               umma_desc_sw128(sTa + st * PC_STAGE_BYTES, 16384, 1024), idesc,
                                               !first, &aux->qempty[st]);
                        }
                        umma_commit_mc_e(&aux->pslot_free[b], 0x1);  // tell the producer slot b is free
                        if (dbg) dbg[7] = clock64();
                        if (t == t1 - 1) umma_commit_e(&aux->ofull);
                    }
                    ++sg;
                }
            }
        } else if (warp < 8) {
            // -------- O drain at segment end: warp w -> rows 32(w%4).. (its TMEM lane quadrant),
            // columns [w/4 * d/2, (w/4 + 1) * d/2): eight warps, so the next unit's GEMM 2 waits less
            const int q = warp & 3, hcol = warp >> 2;
            const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
            const int r = q * 32 + lane;
            uint32_t sg = 0;
            // staged through shared memory and written by TMA stores: each store is one
            // [32 rows x 16 fp32] box of seg_O (row-per-lane global stores scatter one row per
            // lane and took ~45K cycles per unit)
            const uint32_t stg = smem_u32(smem + PC_OFF_OSTG + warp * 2048);
            while (sch.next(rg, t0, t1, seg)) {
                mbar_wait(&aux->ofull, sg & 1);
                tc_fence_after();
                const bool m64 = tail64(rg);
                if (!p.drain_tma || m64) {  // long units: the drain is off the critical path
                    // (a 64-row tail unit: rows 16 q + lane on lanes 0-15 of quadrant q)
                    const int ro = m64 ? q * 16 + lane : r;
                    const bool st = !m64 || lane < 16;
                    float4 *dst = reinterpret_cast<float4 *>(p.seg_O + (static_cast<size_t>(seg) * PC_R + ro) * d);
                    for (int c0 = hcol * (d / 2); c0 < (hcol + 1) * (d / 2); c0 += 32) {
                        float o[32];
                        tmem_ld32(tmem + lane_base + c0, o);
                        tmem_wait_ld();
                        if (st)
#pragma unroll
                            for (int u = 0; u < 8; ++u)
                                dst[c0 / 4 + u] = make_float4(o[4 * u], o[4 * u + 1], o[4 * u + 2], o[4 * u + 3]);
                    }
                    tc_fence_before();
                    __syncwarp();
                    if (lane == 0) mbar_arrive(&aux->oempty);
                    ++sg;
                    continue;
                }
                const int row0 = seg * PC_R + q * 32;
                for (int c0 = hcol * (d / 2); c0 < (hcol + 1) * (d / 2); c0 += 16) {
                    float o[16];
                    tmem_ld16(tmem + lane_base + c0, o);
                    tmem_wait_ld();
                    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                    __syncwarp();
#pragma unroll
                    for (int u = 0; u < 4; ++u)
                        st_shared_v4(stg + lane * 64 + u * 16, __float_as_uint(o[4 * u]), __float_as_uint(o[4 * u + 1]),
                                     __float_as_uint(o[4 * u + 2]), __float_as_uint(o[4 * u + 3]));
                    fence_proxy_async_smem();
                    __syncwarp();
                    if (lane == 0) tma_store_2d(&tmO, stg, c0, row0);
                }
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&aux->oempty);
                if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
                __syncwarp();
                ++sg;
            }
        }
    }
    tc_fence_before();
    __syncthreads();
    if (p.dbg && threadIdx.x == 0 && (blockIdx.x >> 1) == static_cast<unsigned>(p.dbg_cluster)) {
        unsigned long long gt;
        asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt));
        p.dbg[1026 + (blockIdx.x & 1) * 4] = clock64();
        p.dbg[1027 + (blockIdx.x & 1) * 4] = gt;
    }
    cluster_sync_all();
    if (warp == 9) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

}  // namespace f2c
