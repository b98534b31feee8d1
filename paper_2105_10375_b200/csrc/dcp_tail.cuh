// dcp_tail.cuh -- the single-CTA tail role of dcp_pc_kernel (hot-path steps a4, a5, a7 for the
// last row group when it holds <= 32 rows, "tail role").
//
// A row group of a CTA pair streams every pool tile through both CTAs whatever its row count, so a
// last group of a few rows (c3 at W = 1: 23 of 535 in-pool rows) costs a full group's time.  Here
// one CTA runs both GEMMs for such a group over its own range of tiles, transposed so that the
// few rows are the N dimension and no TMEM is needed for them as an operand:
//   GEMM 1   S^T[c, r] = <T_c, x_r>        M = 128 slots, N = 32 rows, K = d
//            (A = the pool stage, K-major SW128 as loaded; B = the rows' x, K-major SW128 in smem)
//   softmax  lane = slot, column = row: e = S a_r - b_r with the row's fixed reference b_r (R1),
//            so the row sums need no running maximum: every thread keeps its slot's partial sums
//            per row and the 128 slots are reduced once, at the end of the range
//   GEMM 2   O^T[k, r] += sum_c T[c, k] P^T[c, r]   M = 128 (d block), N = 32 rows, K = 128 slots
//            (A = the same pool stage read MN-major; B = P^T, K-major SW128 in smem)
// The pool stage is read by both GEMMs before it is released, so the ring holds a tile plus one
// stage.  Results go to the same segment partials (l, max, O rows) as the pair kernel's units; the
// tail group's segments follow the main ones (seg = S (n_rg - 1) + range).
#pragma once
#include "dcp_main.cuh"
#include "sm100.cuh"

namespace f2c {

constexpr int TL_N = 32;                                   // rows of the tail group (GEMM N)
constexpr int TL_NSTAGE = 5;                               // pool ring: 32 KB stages [2 chunks x 128 slots x 64 d]
constexpr int TL_STAGE = 32768;
constexpr int TL_OFF_X = TL_NSTAGE * TL_STAGE;             // x rows: [d/64 chunks][32 rows x 128 B] SW128
constexpr int TL_OFF_P = TL_OFF_X + 8 * 4096;              // P^T: [2 buffers][2 chunks][32 rows x 128 B] SW128
constexpr int TL_OFF_AUX = TL_OFF_P + 2 * 8192;
constexpr uint32_t TL_S_COL = 0, TL_O_COL = 64;            // TMEM: S^T x 2 buffers (32 cols each), O^T blocks

struct TLAux {
    uint64_t tfull[TL_NSTAGE], tempty[TL_NSTAGE];
    uint64_t sfull[2], sempty[2], pfull[2], pempty[2];
    uint64_t xready, ofull;
    uint32_t tmem_base;
    uint32_t pad;
    float4 rows[TL_N];                                     // (a_r, b_r, target slot bits, 0)
    float red_l[4][TL_N];
    float red_mx[4][TL_N];
};

static_assert(TL_OFF_AUX + sizeof(TLAux) + 1024 <= PC_SMEM_BYTES, "the tail role must fit dcp_pc_kernel's launch footprint");

// GEMM 1 of one 32 KB stage: 8 SS MMAs (chunk c = i / 4, K step k = i % 4); A (pool) chunk +16 KB,
// B (x rows) chunk +4 KB, K step +32 B in both
__device__ __forceinline__ void tl_g1_stage(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
                                            uint32_t acc0) {
    asm volatile(
        "{\n.reg .pred e, p, t;\n.reg .b32 r;\n"
        "elect.sync r|e, 0xffffffff;\n"
        "setp.ne.b32 p, %4, 0;\n"
        "setp.eq.b32 t, 0, 0;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %5, %6, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %7, %8, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %9, %10, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %11, %12, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %13, %14, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %15, %16, %3, t;\n"
        "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %17, %18, %3, t;\n}\n" ::"r"(d_tmem),
        "l"(adesc), "l"(bdesc), "r"(idesc), "r"(acc0),
        "l"(adesc + 2), "l"(bdesc + 2), "l"(adesc + 4), "l"(bdesc + 4), "l"(adesc + 6), "l"(bdesc + 6),
        "l"(adesc + 1024), "l"(bdesc + 256), "l"(adesc + 1026), "l"(bdesc + 258), "l"(adesc + 1028),
        "l"(bdesc + 260), "l"(adesc + 1030), "l"(bdesc + 262)
        : "memory");
}
// GEMM 2 of one stage (one 128-wide d block): 8 SS MMAs over the tile's 128 slots, A (pool stage,
// MN-major) +2 KB per K step, B (P^T, K-major) +32 B per K step and +4 KB for the second 64-slot
// chunk; then the commit that releases the pool stage
__device__ __forceinline__ void tl_g2_stage(uint32_t d_tmem, uint64_t adesc, uint64_t bdesc, uint32_t idesc,
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
        "l"(adesc + 128), "l"(bdesc + 2), "l"(adesc + 256), "l"(bdesc + 4), "l"(adesc + 384), "l"(bdesc + 6),
        "l"(adesc + 512), "l"(bdesc + 256), "l"(adesc + 640), "l"(bdesc + 258), "l"(adesc + 768),
        "l"(bdesc + 260), "l"(adesc + 896), "l"(bdesc + 262)
        : "memory");
}
__device__ __forceinline__ void tl_commit(uint64_t *bar) {
    asm volatile(
        "{\n.reg .pred e;\n.reg .b32 r;\nelect.sync r|e, 0xffffffff;\n"
        "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n" ::"r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tl_st_shared_b16(uint32_t addr, uint16_t v) {
    asm volatile("st.shared.b16 [%0], %1;" ::"r"(addr), "h"(v) : "memory");
}

// The role.  tcta = this CTA's index among the 2 tail_G tail CTAs = its range of the tail group's
// tiles; seg0 = the tail group's first segment (S (n_rg - 1)).  P: the pair kernel's parameters.
template <typename PCP>
__device__ __forceinline__ void dcp_tail_role(const CUtensorMap &tm3p, const PCP &p, uint8_t *smem, int tcta,
                                              int n_tail, int seg0, int n_rows) {
    TLAux *aux = reinterpret_cast<TLAux *>(smem + TL_OFF_AUX);
    const int warp = threadIdx.x >> 5;
    const int lane = threadIdx.x & 31;
    const int d = p.d;
    const int nstg = d >> 7;                          // 32 KB stages (= 128-wide d blocks) per tile
    const int n_tiles = (p.n_slots + 127) / 128;
    const int t0 = tp_range_begin(tcta, n_tiles, n_tail), t1 = tp_range_begin(tcta + 1, n_tiles, n_tail);
    const int seg = seg0 + tcta;
    const int n_rg = (n_rows + 127) / 128;
    const int row0 = (n_rg - 1) * 128;
    const int nr = n_rows - row0;                     // 1 .. 32
    if (threadIdx.x == 0) {
        for (int i = 0; i < TL_NSTAGE; ++i) {
            mbar_init(&aux->tfull[i], 1);
            mbar_init(&aux->tempty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&aux->sfull[i], 1);
            mbar_init(&aux->sempty[i], 4);
            mbar_init(&aux->pfull[i], 4);
            mbar_init(&aux->pempty[i], 1);
        }
        mbar_init(&aux->xready, 4);
        mbar_init(&aux->ofull, 1);
        fence_mbar_init();
    }
    if (warp == 9) {
        tma_prefetch_desc(&tm3p);
        tmem_alloc(&aux->tmem_base, 256);
        tmem_relinquish();
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem = aux->tmem_base;
    const uint32_t sX = smem_u32(smem + TL_OFF_X), sP = smem_u32(smem + TL_OFF_P), sR = smem_u32(smem);

    if (t1 > t0) {
        if (warp == 8) {
            // -------- TMA: the range's pool tiles, stage by stage
            if (lane == 0) {
                uint32_t pc = 0;
                for (int t = t0; t < t1; ++t)
                    for (int g = 0; g < nstg; ++g, ++pc) {
                        const uint32_t st = pc % TL_NSTAGE, ph = (pc / TL_NSTAGE) & 1;
                        mbar_wait(&aux->tempty[st], ph ^ 1);
                        mbar_arrive_expect_tx(&aux->tfull[st], TL_STAGE);
                        tma_load_3d(smem + st * TL_STAGE, &tm3p, &aux->tfull[st], 0, t * 128, g * 2);
                    }
            }
        } else if (warp == 9) {
            // -------- UMMA issuer: GEMM 1 of tile j, then (once its P^T is written) GEMM 2 of tile j
            const uint32_t id1 = umma_idesc_bf16(128, TL_N, 0, 0), id2 = umma_idesc_bf16(128, TL_N, 1, 0);
            mbar_wait(&aux->xready, 0);
            tc_fence_after();
            uint32_t pc = 0;
            for (int t = t0, j = 0; t < t1; ++t, ++j) {
                const uint32_t sb = j & 1, ph = (j >> 1) & 1;
                mbar_wait(&aux->sempty[sb], ph ^ 1);
                tc_fence_after();
                for (int g = 0; g < nstg; ++g) {
                    const uint32_t st = (pc + g) % TL_NSTAGE, tph = ((pc + g) / TL_NSTAGE) & 1;
                    mbar_wait(&aux->tfull[st], tph);
                    tc_fence_after();
                    tl_g1_stage(tmem + TL_S_COL + sb * TL_N, umma_desc_sw128(sR + st * TL_STAGE, 16, 1024),
                                umma_desc_sw128(sX + g * 8192, 16, 1024), id1, g != 0);
                }
                tl_commit(&aux->sfull[sb]);
                mbar_wait(&aux->pfull[sb], ph);
                tc_fence_after();
                for (int g = 0; g < nstg; ++g, ++pc) {
                    const uint32_t st = pc % TL_NSTAGE;
                    tl_g2_stage(tmem + TL_O_COL + g * TL_N, umma_desc_sw128(sR + st * TL_STAGE, 16384, 1024),
                                umma_desc_sw128(sP + sb * 8192, 16, 1024), id2, j != 0, &aux->tempty[st]);
                }
                tl_commit(&aux->pempty[sb]);
            }
            tl_commit(&aux->ofull);
        } else if (warp < 4) {
            // -------- softmax warps: lane = slot 32 warp + lane of the tile
            const int q = warp;
            const uint32_t lane_base = static_cast<uint32_t>(q * 32) << 16;
            const int cl = q * 32 + lane;                 // slot within the tile
            if (lane < TL_N && q == 0) {
                const int r = lane, row = row0 + r;
                aux->rows[r] = r < nr ? make_float4(p.row_ab[row].x, p.row_ab[row].y, __int_as_float(p.row_tgt[row]), 0.f)
                                      : make_float4(0.f, INFINITY, __int_as_float(-1), 0.f);
            }
            // the rows' x (bf16) -> the GEMM-1 B operand, K-major SW128: chunk = 64 d, row r = 128 B
            {
                const int upr = d >> 3;                   // 16-B units per row
                for (int i = cl; i < TL_N * upr; i += 128) {
                    const int r = i / upr, u = i - r * upr;
                    uint4 v = make_uint4(0u, 0u, 0u, 0u);
                    if (r < nr) v = reinterpret_cast<const uint4 *>(p.X_pos + static_cast<size_t>(row0 + r) * d * 2)[u];
                    const int ch = u >> 3, uu = u & 7;
                    st_shared_v4(sX + ch * 4096 + (r >> 3) * 1024 + (r & 7) * 128 + ((uu ^ (r & 7)) << 4), v.x, v.y, v.z,
                                 v.w);
                }
                fence_proxy_async_smem();
                named_bar_sync(1, 128);
                if (lane == 0) mbar_arrive(&aux->xready);
            }
            float l[TL_N], mx[TL_N];
#pragma unroll
            for (int r = 0; r < TL_N; ++r) {
                l[r] = 0.f;
                mx[r] = -INFINITY;
            }
            const uint32_t pch = static_cast<uint32_t>(cl >> 6) * 4096, pu = static_cast<uint32_t>((cl & 63) >> 3),
                           pb2 = static_cast<uint32_t>(cl & 7) * 2;
            for (int t = t0, j = 0; t < t1; ++t, ++j) {
                const uint32_t sb = j & 1, ph = (j >> 1) & 1;
                mbar_wait(&aux->sfull[sb], ph);
                tc_fence_after();
                float s[TL_N];
                tmem_ld32(tmem + lane_base + TL_S_COL + sb * TL_N, s);
                tmem_wait_ld();
                tc_fence_before();
                __syncwarp();
                if (lane == 0) mbar_arrive(&aux->sempty[sb]);  // S^T buffer free for GEMM 1 of tile j + 2
                const int c = t * 128 + cl;
                const bool valid = c < p.n_slots;
                mbar_wait(&aux->pempty[sb], ph ^ 1);   // GEMM 2 of tile j - 2 has read this P^T buffer
                const uint32_t pbase = sP + sb * 8192 + pch;
#pragma unroll
                for (int r = 0; r < TL_N; ++r) {
                    const float4 rw = aux->rows[r];
                    const float e = fmaf(s[r], rw.x, -rw.y);
                    bool keep = valid && r < nr;
                    if (keep && c == __float_as_int(rw.z)) {  // the target column: recorded apart, excluded
                        p.ttgt[row0 + r] = e - p.margin_l2;
                        keep = false;
                    }
                    const float pv = keep ? ex2_approx(e) : 0.f;
                    if (keep) {
                        l[r] += pv;
                        mx[r] = fmaxf(mx[r], e);
                    }
                    const __nv_bfloat16 hb = __float2bfloat16_rn(pv);
                    tl_st_shared_b16(pbase + (r >> 3) * 1024 + (r & 7) * 128 + ((pu ^ (r & 7)) << 4) + pb2,
                                     *reinterpret_cast<const uint16_t *>(&hb));
                }
                fence_proxy_async_smem();
                __syncwarp();
                if (lane == 0) mbar_arrive(&aux->pfull[sb]);
            }
            // the range's partial sums over its slots, per row: lanes, then the 4 warps in order
            const float lr = warp_transpose_reduce<false>(l, lane);
            const float mr = warp_transpose_reduce<true>(mx, lane);
            aux->red_l[q][lane] = lr;
            aux->red_mx[q][lane] = mr;
            named_bar_sync(1, 128);
            if (q == 0 && lane < nr) {
                p.seg_l[static_cast<size_t>(seg) * 128 + lane] =
                    ((aux->red_l[0][lane] + aux->red_l[1][lane]) + aux->red_l[2][lane]) + aux->red_l[3][lane];
                p.seg_mx[static_cast<size_t>(seg) * 128 + lane] =
                    fmaxf(fmaxf(aux->red_mx[0][lane], aux->red_mx[1][lane]), fmaxf(aux->red_mx[2][lane], aux->red_mx[3][lane]));
            }
            // O^T -> the segment's O rows: warp q holds d = 128 g + 32 q + lane of every row
            mbar_wait(&aux->ofull, 0);
            tc_fence_after();
            for (int g = 0; g < nstg; ++g) {
                float o[TL_N];
                tmem_ld32(tmem + lane_base + TL_O_COL + g * TL_N, o);
                tmem_wait_ld();
#pragma unroll
                for (int r = 0; r < TL_N; ++r)
                    if (r < nr) p.seg_O[(static_cast<size_t>(seg) * 128 + r) * d + g * 128 + cl] = o[r];
            }
        }
    } else if (warp < 4) {
        // an empty range (more tail CTAs than tiles): zero partials, so the combine's sums are exact
        if (threadIdx.x < nr) {
            p.seg_l[static_cast<size_t>(seg) * 128 + threadIdx.x] = 0.f;
            p.seg_mx[static_cast<size_t>(seg) * 128 + threadIdx.x] = -INFINITY;
        }
        for (int i = threadIdx.x; i < nr * d; i += 128)
            p.seg_O[static_cast<size_t>(seg) * 128 * d + i] = 0.f;
    }
    tc_fence_before();
    __syncthreads();
    if (warp == 9) {
        tc_fence_after();
        tmem_dealloc(tmem, 256);
    }
}

}  // namespace f2c
