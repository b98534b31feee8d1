// dcp_main.cuh -- the fused DCP loss kernel (steps a2, a4, a5, a7, a9 of the hot path).
//
// One pass over the occupied pool computes, for every in-pool ("compacted") row r
// of a 64-row group and every slot c of a tile of 128 slots:
//     S^T[c, r] = <T_c, x_r>                         (GEMM 1, Eq. 8 with K = 1)
//     e[c, r]   = S^T[c, r] * a_r - b_r               a_r = s*log2(e)/||x_r||, b_r = reference
//     p[c, r]   = 2^e                                 (target column: margin, recorded apart)
//     O^T[:, r] += T^T[:, c] * p[c, r]                (GEMM 2: the softmax-weighted pool sum)
// and accumulates l_r = sum_c p and max_c e, so that after the combine
//     dL/dx_hat_r = (s/N_pos) (O_r / l_r - (1 - p_t) T_t)          (Eq. 9 gradient, D12)
// The N x C logit matrix only ever exists as one 128x64 fp32 tile in TMEM.
//
// Layout ("transposed", d on TMEM lanes for O): for d = 512 a 128-row O tile would
// need all 512 TMEM columns, so rows live on the UMMA N dimension (64 per CTA) and
// both GEMMs use the pool tile as the A operand from the same shared-memory bytes:
// K-major for GEMM 1 (M = slots, K = d), MN-major for GEMM 2 (M = d, K = slots).
// The softmax reference b_r is an upper bound of every logit (s * max||T_c|| in
// log2 units), identical across slots, so partial sums from different CTAs,
// tiles and ranks add without rescaling.
//
// Warp roles (320 threads, one CTA per SM, persistent over a flattened
// (row group, tile) range): warps 0-7 softmax/epilogue, warp 8 TMA producer,
// warp 9 TMEM allocator + single-thread UMMA issuer.
#pragma once
#include "sm100.cuh"

namespace f2c {

constexpr int TP_R = 64;                // rows per group = UMMA N
constexpr int TP_TILE = 128;            // slots per tile = UMMA M of GEMM 1
constexpr int TP_CHUNK_BYTES = 16384;   // [128 slots x 64 d] bf16, one SW128 TMA box
constexpr int TP_PAIR_BYTES = 32768;    // two chunks = [128 slots x 128 d] = one GEMM-2 M block
constexpr int TP_NSTAGE = 4;            // pair stages in the pool ring (= one d=512 tile)
constexpr int TP_XCHUNK_BYTES = 8192;   // [64 rows x 64 d] bf16
constexpr int TP_THREADS = 320;
constexpr int TP_EPI_THREADS = 256;
constexpr int TP_S_COL = 0;             // TMEM columns of S^T (64)
constexpr int TP_O_COL = 256;           // TMEM columns of O^T (64 per 128-d block)

constexpr int TP_OFF_X = 0;                                  // 64 KB
constexpr int TP_OFF_T = 65536;                              // 128 KB
constexpr int TP_OFF_P = TP_OFF_T + TP_NSTAGE * TP_PAIR_BYTES;  // 16 KB
constexpr int TP_OFF_AUX = TP_OFF_P + 16384;                 // barriers + metadata
constexpr int TP_SMEM_BYTES = TP_OFF_AUX + 4096 + 1024;      // + alignment slack

struct TPParams {
    int d;                 // feature dim (multiple of 128, <= 512)
    int n_slots;           // occupied slots of this shard: tiles cover [0, n_slots)
    const int *n_pos;      // device: number of in-pool rows
    const float2 *row_ab;  // [R_max] (a_r, b_r) per compacted row (0,0 for padding)
    const int *row_tgt;    // [R_max] local slot of the row's target, -1 if not in this shard
    float margin_l2;       // s * m * log2(e)
    float *ttgt;           // [R_max] exponent of the margined target logit (owner writes)
    float *seg_l;          // [S][64]   sum of p over the segment's slots (target excluded)
    float *seg_mx;         // [S][64]   max exponent over the segment's slots (target excluded)
    float *seg_O;          // [S][64][d] sum_c p[c, r] T_c (target excluded)
    unsigned long long *dbg;  // optional per-tile timestamps of CTA 0 (null in production)
};

struct TPAux {
    uint64_t tfull[TP_NSTAGE];
    uint64_t tempty[TP_NSTAGE];
    uint64_t xfull, xempty, sfull, pfull, ofull, oempty;
    uint32_t tmem_base;
    uint32_t pad;
    float2 ab[TP_R];
    int tgt[TP_R];
    float red_l[4][TP_R];
    float red_mx[4][TP_R];
};

// Work schedule.  The occupied tiles are cut into S contiguous ranges; a unit is
// (range s, row group rg) with id u = s * R + rg (R = row groups).  CTA b runs units
// b, b + G, b + 2G, ...  Units that run concurrently share their range across all
// row groups, so every pool tile is read from HBM about once and served to the R
// row groups from L2.  S balances R*S units over G CTAs (waves) while keeping
// ranges long; the combine kernel recomputes the same S.  Unit id = segment id.
// timing experiments only (F2C_FORCE_S, set at create): force the number of ranges S
__constant__ int g_force_S;
__host__ __device__ inline int tp_choose_S(int R, int G, int n_tiles) {
    if (n_tiles <= 0 || R <= 0) return 1;
#ifdef __CUDA_ARCH__
#endif
    int s_lo = G / R;
    if (s_lo < 1) s_lo = 1;
    int s_hi = (2 * G) / R + 1;
    if (s_hi > n_tiles) s_hi = n_tiles;
#ifdef __CUDA_ARCH__
    // (the forced count stays within the candidates' bound: R S <= 2G + R, the partial buffer's size)
    if (g_force_S > 0) return g_force_S < s_hi ? g_force_S : s_hi;
#endif
    if (s_lo > s_hi) s_lo = s_hi;
    int best = s_lo;
    // (single precision: this runs in every CTA's prologue and in every combine row, and fp64
    // divisions there cost thousands of cycles)
    float best_eff = -1.f;
    const float work = static_cast<float>(n_tiles) * static_cast<float>(R) / static_cast<float>(G);
    for (int S = s_lo; S <= s_hi; ++S) {
        const int U = R * S;                 // (32-bit: R*S <= 2G + R)
        const int waves = (U + G - 1) / G;
        // time ~ waves * ceil(n_tiles / S); work ~ n_tiles * R / G per CTA
        const float t = static_cast<float>(waves) * static_cast<float>((n_tiles + S - 1) / S);
        // a second wave re-streams ranges whose row groups no longer run together (L2 reuse
        // is lost across waves): single-wave schedules get a 6 % credit
        const float eff = work / t * (waves == 1 ? 1.06f : 1.f);
        if (eff > best_eff + 0.01f) {
            best_eff = eff;
            best = S;
        }
    }
    return best;
}

// dcp_pc_kernel's schedule (round 2): S is chosen once per loss call, by k_compact as soon as the row
// count is known (one thread per candidate S, a block-wide argmin; sc->S_sched), and read by the fused
// kernel and the combine.  Candidates: R S <= 512 (the partial-buffer bound the layout always holds)
// and at most 30 units per cluster; cost t(S) = waves (ceil(n_tiles / S) + 8), the 8 tile-equivalents
// being the fixed per-unit cost (prologue, O drain); ties go to the smaller S.  Multi-wave schedules
// with fine ranges measured faster where one wave leaves clusters idle (c3, 5 row groups on 74
// clusters: S = 59 instead of 14, -3 to -5 %; c3r_8, 34 groups: S = 13 instead of 2, -2 to -6 %);
// c2 keeps its single wave (profiles/r02_ab_schedule_waves.txt).
__host__ __device__ inline int pc_s_hi(int R, int G, int n_tiles) {
    if (R <= 0 || n_tiles <= 0) return 1;
    int s_hi = 512 / R;
    if (30 * G / R < s_hi) s_hi = 30 * G / R;
    if (s_hi > n_tiles) s_hi = n_tiles;
    return s_hi < 1 ? 1 : s_hi;
}
__host__ __device__ inline float pc_sched_cost(int S, int R, int G, int n_tiles) {
    const int waves = (R * S + G - 1) / G;
    return static_cast<float>(waves) * (static_cast<float>((n_tiles + S - 1) / S) + 8.f);
}

// First tile of range s when n_tiles tiles are cut into S ranges: q or q + 1 tiles each (the
// first n_tiles % S ranges get one more).  32-bit arithmetic only: 64-bit divisions cost ~100
// instructions each, and this runs in every CTA's prologue and in every combine row.
__host__ __device__ inline int tp_range_begin(int s, int n_tiles, int S) {
    const int q = n_tiles / S, rem = n_tiles - q * S;
    return s * q + (s < rem ? s : rem);
}

struct TPSched {
    int R, S, n_tiles, G;
    int u, U;
    __device__ void init(int b, int G_, int R_, int nt, int S_fixed = 0) {
        R = R_;
        G = G_;
        n_tiles = nt;
        S = S_fixed > 0 ? S_fixed : tp_choose_S(R, G, nt);
        U = nt > 0 ? R * S : 0;
        u = b;
    }
    __device__ bool next(int &rg, int &t0, int &t1, int &seg) {
        while (u < U) {
            const int s = u / R;
            rg = u - s * R;
            seg = u;
            t0 = tp_range_begin(s, n_tiles, S);
            t1 = tp_range_begin(s + 1, n_tiles, S);
            u += G;
            if (t1 > t0) return true;
        }
        return false;
    }
};

// Sum (or max) 32 per-lane values across the warp so that lane L ends with the
// reduction of index L (31 shuffles, fixed order => deterministic).
template <bool MAX>
__device__ __forceinline__ float warp_transpose_reduce(float (&v)[32], int lane) {
#pragma unroll
    for (int s = 16; s >= 1; s >>= 1) {
        const bool upper = (lane & s) != 0;
#pragma unroll
        for (int i = 0; i < s; ++i) {
            float send = upper ? v[i] : v[i + s];
            float keep = upper ? v[i + s] : v[i];
            float recv = __shfl_xor_sync(0xffffffffu, send, s);
            v[i] = MAX ? fmaxf(keep, recv) : keep + recv;
        }
    }
    return v[0];
}

__global__ void __launch_bounds__(TP_THREADS, 1)
    dcp_tp64_kernel(const __grid_constant__ CUtensorMap tmT, const __grid_constant__ CUtensorMap tmX,
                    const TPParams p) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t *smem = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                                ~static_cast<uintptr_t>(1023));
    uint8_t *sX = smem + TP_OFF_X;
    uint8_t *sT = smem + TP_OFF_T;
    uint8_t *sP = smem + TP_OFF_P;
    TPAux *aux = reinterpret_cast<TPAux *>(smem + TP_OFF_AUX);

    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int d = p.d;
    const int npair = d >> 7;
    const int n_pos = *p.n_pos;
    const int n_rg = (n_pos + TP_R - 1) / TP_R;
    const int n_tiles = (p.n_slots + TP_TILE - 1) / TP_TILE;

    if (warp == 8 && lane == 0) {
        tma_prefetch_desc(&tmT);
        tma_prefetch_desc(&tmX);
        for (int i = 0; i < TP_NSTAGE; ++i) {
            mbar_init(&aux->tfull[i], 1);
            mbar_init(&aux->tempty[i], 1);
        }
        mbar_init(&aux->xfull, 1);
        mbar_init(&aux->xempty, 1);
        mbar_init(&aux->sfull, 1);
        mbar_init(&aux->pfull, 8);
        mbar_init(&aux->ofull, 1);
        mbar_init(&aux->oempty, 8);
        fence_mbar_init();
    }
    if (warp == 9) {
        tmem_alloc(&aux->tmem_base, 512);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = aux->tmem_base;

    TPSched sch;
    sch.init(blockIdx.x, gridDim.x, n_rg, n_tiles);
    int rg, t0, t1, seg;

    if (warp == 8) {
        // ------------------------------------------------------------ TMA producer
        if (lane == 0) {
            uint32_t pc = 0, sg = 0;
            while (sch.next(rg, t0, t1, seg)) {
                mbar_wait(&aux->xempty, (sg & 1) ^ 1);
                mbar_arrive_expect_tx(&aux->xfull, static_cast<uint32_t>(TP_R * d * 2));
                for (int c = 0; c < (d >> 6); ++c)
                    tma_load_2d(sX + c * TP_XCHUNK_BYTES, &tmX, &aux->xfull, c * 64, rg * TP_R);
                for (int t = t0; t < t1; ++t) {
                    const uint32_t jt_p = pc / npair;
                    for (int q = 0; q < npair; ++q, ++pc) {
                        if (p.dbg && blockIdx.x == 0 && jt_p < 64 && q == npair - 1) p.dbg[jt_p * 8 + 7] = clock64();
                        const uint32_t st = pc % TP_NSTAGE, ph = (pc / TP_NSTAGE) & 1;
                        mbar_wait(&aux->tempty[st], ph ^ 1);
                        mbar_arrive_expect_tx(&aux->tfull[st], TP_PAIR_BYTES);
                        uint8_t *dst = sT + st * TP_PAIR_BYTES;
                        tma_load_2d(dst, &tmT, &aux->tfull[st], (2 * q) * 64, t * TP_TILE);
                        tma_load_2d(dst + TP_CHUNK_BYTES, &tmT, &aux->tfull[st], (2 * q + 1) * 64,
                                    t * TP_TILE);
                    }
                }
                ++sg;
            }
        }
    } else if (warp == 9) {
        // ------------------------------------------------------------ UMMA issuer
        if (lane == 0) {
            constexpr uint32_t idesc1 = umma_idesc_bf16(128, TP_R, 0, 0);  // K-major A and B
            constexpr uint32_t idesc2 = umma_idesc_bf16(128, TP_R, 1, 1);  // MN-major A and B
            const uint32_t sTa = smem_u32(sT), sXa = smem_u32(sX), sPa = smem_u32(sP);
            uint32_t pc = 0, sg = 0, jt = 0;
            while (sch.next(rg, t0, t1, seg)) {
                mbar_wait(&aux->xfull, sg & 1);
                tc_fence_after();
                for (int t = t0; t < t1; ++t, ++jt) {
                    const bool first = (t == t0), last = (t == t1 - 1);
                    unsigned long long *dbg = (p.dbg && blockIdx.x == 0 && jt < 64) ? p.dbg + jt * 8 : nullptr;
                    if (dbg) dbg[0] = clock64();
                    // GEMM 1: S^T[slot, row] = sum_d T[slot, d] * x[row, d]
                    for (int q = 0; q < npair; ++q) {
                        const uint32_t pq = pc + q;
                        const uint32_t st = pq % TP_NSTAGE, ph = (pq / TP_NSTAGE) & 1;
                        mbar_wait(&aux->tfull[st], ph);
                        tc_fence_after();
#pragma unroll
                        for (int k = 0; k < 8; ++k) {
                            const uint32_t h = k >> 2, kk = k & 3;
                            const uint64_t a = umma_desc_sw128(
                                sTa + st * TP_PAIR_BYTES + h * TP_CHUNK_BYTES + kk * 32, 16, 1024);
                            const uint64_t b = umma_desc_sw128(
                                sXa + (2 * q + h) * TP_XCHUNK_BYTES + kk * 32, 16, 1024);
                            umma_bf16(tmem + TP_S_COL, a, b, idesc1, (q | k) != 0);
                        }
                    }
                    umma_commit(&aux->sfull);
                    if (last) umma_commit(&aux->xempty);
                    if (dbg) dbg[1] = clock64();
                    // wait for the softmax warps to publish P^T for this tile
                    mbar_wait(&aux->pfull, jt & 1);
                    tc_fence_after();
                    if (dbg) dbg[2] = clock64();
                    if (first && sg > 0) {
                        mbar_wait(&aux->oempty, (sg - 1) & 1);
                        tc_fence_after();
                    }
                    // GEMM 2: O^T[d, row] += sum_slot T[slot, d] * P^T[slot, row]
                    for (int q = 0; q < npair; ++q) {
                        const uint32_t st = (pc + q) % TP_NSTAGE;
#pragma unroll
                        for (int kk = 0; kk < 8; ++kk) {
                            const uint64_t a = umma_desc_sw128(
                                sTa + st * TP_PAIR_BYTES + kk * 2048, TP_CHUNK_BYTES, 1024);
                            const uint64_t b = umma_desc_sw128(sPa + kk * 2048, 8192, 1024);
                            umma_bf16(tmem + TP_O_COL + q * TP_R, a, b, idesc2,
                                      !(first && kk == 0));
                        }
                        umma_commit(&aux->tempty[st]);
                    }
                    pc += npair;
                    if (last) umma_commit(&aux->ofull);
                    if (dbg) dbg[3] = clock64();
                }
                ++sg;
            }
        }
    } else {
        // ------------------------------------------------------------ softmax / epilogue
        const int tid = threadIdx.x;  // 0..255
        const int qw = warp & 3;      // TMEM lane quarter -> slots qw*32 .. +31 of a tile
        const int hw = warp >> 2;     // row half -> rows hw*32 .. +31 of the group
        const uint32_t lane_base = static_cast<uint32_t>(qw * 32) << 16;
        const uint32_t sPa = smem_u32(sP);
        const int sr = qw * 32 + lane;  // slot row within the tile
        const uint32_t prow = sPa + (sr >> 3) * 1024 + (sr & 7) * 128;
        uint32_t sg = 0, jt = 0;
        while (sch.next(rg, t0, t1, seg)) {
            named_bar_sync(1, TP_EPI_THREADS);
            if (tid < TP_R) {
                aux->ab[tid] = p.row_ab[rg * TP_R + tid];
                aux->tgt[tid] = p.row_tgt[rg * TP_R + tid];
            }
            named_bar_sync(1, TP_EPI_THREADS);
            const int tg = aux->tgt[hw * 32 + lane];
            float lacc[32], mxacc[32];
#pragma unroll
            for (int k = 0; k < 32; ++k) {
                lacc[k] = 0.f;
                mxacc[k] = -INFINITY;
            }
            for (int t = t0; t < t1; ++t, ++jt) {
                unsigned long long *dbg = (p.dbg && blockIdx.x == 0 && jt < 64 && tid == 0) ? p.dbg + jt * 8 : nullptr;
                if (dbg) dbg[4] = clock64();
                mbar_wait(&aux->sfull, jt & 1);
                tc_fence_after();
                if (dbg) dbg[5] = clock64();
                float e[32];
                tmem_ld32(tmem + lane_base + TP_S_COL + hw * 32, e);
                tmem_wait_ld();
                const int slot = t * TP_TILE + sr;
                const bool valid = slot < p.n_slots;
#pragma unroll
                for (int k = 0; k < 32; ++k) {
                    const float2 ab = aux->ab[hw * 32 + k];
                    e[k] = valid ? fmaf(e[k], ab.x, -ab.y) : -INFINITY;
                }
                // rows whose target slot lies in this tile (rare): margin, record, exclude
                unsigned hit = __ballot_sync(0xffffffffu, tg >= t * TP_TILE && tg < (t + 1) * TP_TILE);
                while (hit) {
                    const int kh = __ffs(hit) - 1;
                    hit &= hit - 1;
                    const int tslot = __shfl_sync(0xffffffffu, tg, kh);
                    if (slot == tslot) {
#pragma unroll
                        for (int k = 0; k < 32; ++k)
                            if (k == kh) {
                                p.ttgt[rg * TP_R + hw * 32 + k] = e[k] - p.margin_l2;
                                e[k] = -INFINITY;
                            }
                    }
                }
                uint32_t pk[16];
#pragma unroll
                for (int k = 0; k < 32; k += 2) {
                    const float p0 = ex2_approx(e[k]), p1 = ex2_approx(e[k + 1]);
                    lacc[k] += p0;
                    lacc[k + 1] += p1;
                    mxacc[k] = fmaxf(mxacc[k], e[k]);
                    mxacc[k + 1] = fmaxf(mxacc[k + 1], e[k + 1]);
                    pk[k >> 1] = pack_bf16x2(p0, p1);
                }
#pragma unroll
                for (int u = 0; u < 4; ++u) {
                    const uint32_t unit = static_cast<uint32_t>(hw * 4 + u) ^ (sr & 7);
                    st_shared_v4(prow + unit * 16, pk[4 * u], pk[4 * u + 1], pk[4 * u + 2],
                                 pk[4 * u + 3]);
                }
                fence_proxy_async_smem();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&aux->pfull);
                if (dbg) dbg[6] = clock64();
            }
            // ---- segment end: reduce l and max over the 128 slot lanes
            const float lsum = warp_transpose_reduce<false>(lacc, lane);
            const float lmax = warp_transpose_reduce<true>(mxacc, lane);
            aux->red_l[qw][hw * 32 + lane] = lsum;
            aux->red_mx[qw][hw * 32 + lane] = lmax;
            named_bar_sync(1, TP_EPI_THREADS);
            if (tid < TP_R) {
                float ls = 0.f, mx = -INFINITY;
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    ls += aux->red_l[i][tid];
                    mx = fmaxf(mx, aux->red_mx[i][tid]);
                }
                p.seg_l[seg * TP_R + tid] = ls;
                p.seg_mx[seg * TP_R + tid] = mx;
            }
            // ---- O^T partial of this segment -> global
            mbar_wait(&aux->ofull, sg & 1);
            tc_fence_after();
            for (int q = 0; q < npair; ++q) {
                float o[32];
                tmem_ld32(tmem + lane_base + TP_O_COL + q * TP_R + hw * 32, o);
                tmem_wait_ld();
                const int dd = q * 128 + qw * 32 + lane;
                float *dst = p.seg_O + (static_cast<size_t>(seg) * TP_R + hw * 32) * d + dd;
#pragma unroll
                for (int k = 0; k < 32; ++k) dst[static_cast<size_t>(k) * d] = o[k];
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&aux->oempty);
            ++sg;
        }
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
        tc_fence_after();
        tmem_dealloc(tmem, 512);
    }
}

}  // namespace f2c
