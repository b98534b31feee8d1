// issue_bench.cu -- what does the GEMM-1 issue loop of dcp_pc_kernel cost beyond the MMA
// floor?  One CTA per SM issues "tiles" of 32 TS-mode N=128 MMAs (A = TMEM, B = smem,
// 4 stages of 8 MMAs) with an increasing amount of the kernel's per-stage / per-tile
// synchronisation, and a "softmax" warp that waits for each tile's commit and releases
// the S buffer.  Reports cycles per MMA (floor 64).
#include <cstdio>
#include <cstdint>
#include "../paper_2105_10375_b200/csrc/sm100.cuh"
using namespace f2c;

__device__ __forceinline__ void umma_ts_e(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n.reg .pred p, e;\n.reg .b32 r;\nelect.sync r|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                 :: "r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void tmem_st32(uint32_t taddr, const uint32_t (&v)[32]) {
    asm volatile("tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], "
                 "{%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                 "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(taddr),
                 "r"(v[0]), "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7]),
                 "r"(v[8]), "r"(v[9]), "r"(v[10]), "r"(v[11]), "r"(v[12]), "r"(v[13]), "r"(v[14]),
                 "r"(v[15]), "r"(v[16]), "r"(v[17]), "r"(v[18]), "r"(v[19]), "r"(v[20]), "r"(v[21]),
                 "r"(v[22]), "r"(v[23]), "r"(v[24]), "r"(v[25]), "r"(v[26]), "r"(v[27]), "r"(v[28]),
                 "r"(v[29]), "r"(v[30]), "r"(v[31]) : "memory");
}
__device__ __forceinline__ void tmem_wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory"); }
__device__ __forceinline__ void commit_e(uint64_t *bar) {
    asm volatile("{\n.reg .pred e;\n.reg .b32 r;\nelect.sync r|e, 0xffffffff;\n"
                 "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}\n"
                 :: "r"(smem_u32(bar)) : "memory");
}

// V: bit 1 = per-stage commit, 2 = per-stage wait on a ready barrier (+fence), 4 = S double
// buffer with a softmax warp (sfull / sempty), 8 = stage ring released by the MMA commits
// and refilled by a "TMA" warp arriving (no data) -- the kernel's flags-68 harness.
__device__ volatile int g_done;
// SPIN: extra warps (4..) spin in try_wait on a barrier that completes only at the end
__device__ __forceinline__ void umma_ss_e(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n.reg .pred p, e;\n.reg .b32 r;\nelect.sync r|e, 0xffffffff;\nsetp.ne.b32 p, %4, 0;\n"
                 "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                 :: "r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
template <int V, int RND = 0, int SPIN = 0, int MIX = 0, int KL = 0, int DLY = 0>
__global__ void __launch_bounds__(384, 1) bench(unsigned long long *out, int tiles) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t tfull[4], tempty[4], sfull[2], sempty[2], ready, never;
    __shared__ uint32_t tbase;
    __shared__ volatile int done_s;
    if (threadIdx.x == 0) done_s = 0;
    uint8_t *s = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp == 0) { tmem_alloc(&tbase, 512); tmem_relinquish(); }
    if (threadIdx.x == 32) {
        for (int i = 0; i < 4; ++i) { mbar_init(&tfull[i], 1); mbar_init(&tempty[i], 1); }
        for (int i = 0; i < 2; ++i) { mbar_init(&sfull[i], 1); mbar_init(&sempty[i], KL ? 8 : 1); }
        mbar_init(&ready, 1);
        mbar_init(&never, 1);
        fence_mbar_init();
    }
    for (int i = threadIdx.x; i < 131072 / 4; i += 128) {
        uint32_t v = 0;
        if (RND) {  // random bf16 pairs in [-0.125, 0.125)
            uint32_t x = (i + 1) * 2654435761u ^ (blockIdx.x * 97u);
            x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
            const uint32_t lo = 0x3c00u | (x & 0x807fu), hi = 0x3c00u | ((x >> 16) & 0x807fu);
            v = lo | (hi << 16);
        }
        reinterpret_cast<uint32_t *>(s)[i] = v;
    }
    fence_proxy_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (RND && warp < 4) {  // random A operand in TMEM columns 0..255 (x_hat)
        for (int c0 = 0; c0 < 256; c0 += 32) {
            uint32_t w[32];
            for (int k = 0; k < 32; ++k) {
                uint32_t x = (threadIdx.x * 256 + c0 + k + 7) * 2246822519u;
                x ^= x >> 13; x *= 0x5bd1e995u; x ^= x >> 15;
                w[k] = (0x3c00u | (x & 0x807fu)) | ((0x3c00u | ((x >> 16) & 0x807fu)) << 16);
            }
            tmem_st32(tbase + ((uint32_t)(warp * 32) << 16) + c0, w);
        }
        tmem_wait_st();
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (threadIdx.x == 32) mbar_arrive(&ready);  // phase 0 completes: "stage ready" forever after
    __syncthreads();
    const uint32_t tm = tbase;
    constexpr uint32_t idesc = umma_idesc_bf16(128, 128, 0, 0);
    uint32_t crank;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(crank));
    const int W_ISS = KL ? 9 : 1, W_TMA = KL ? 8 : 3;
    if (MIX && (crank & 1) && warp == 1) {
        // the consumer's GEMM 2 shape: SS, N = 256, A = P K-major, B = pool MN-major, D = all 512 cols
        constexpr uint32_t id2 = umma_idesc_bf16(128, 256, 0, 1);
        const uint32_t sa = smem_u32(s), sbb = smem_u32(s + 65536);
        unsigned long long t0 = clock64();
        for (int t = 0; t < tiles; ++t)
            for (int hh = 0; hh < 2; ++hh)
#pragma unroll
                for (int ks = 0; ks < 8; ++ks)
                    umma_ss_e(tm + hh * 256, umma_desc_sw128(sa + (ks >> 2) * 16384 + (ks & 3) * 32, 16, 1024),
                              umma_desc_sw128(sbb + ks * 2048, 16384, 1024), id2, 1);
        commit_e(&sfull[0]);
        mbar_wait(&sfull[0], 0);
        __syncwarp();
        if (lane == 0) out[blockIdx.x] = clock64() - t0;
        if (lane == 0) mbar_arrive(&never);
    } else if (warp == W_ISS) {
        unsigned long long t0 = clock64();
        const uint64_t bdesc0 = umma_desc_sw128(smem_u32(s), 16, 1024);
        uint32_t pc = 0;
        for (int t = 0; t < tiles; ++t) {
            const uint32_t sb = (V & 4) ? (t & 1) : 0, sph = (t >> 1) & 1;
            if (V & 4) { mbar_wait(&sempty[sb], sph ^ 1); tc_fence_after(); }
            const uint32_t dcol = tm + 256 + sb * 128;
            for (int g = 0; g < 4; ++g, ++pc) {
                const uint32_t st = pc & 3, ph = (pc >> 2) & 1;
                if (V & 8) { mbar_wait(&tfull[st], ph); tc_fence_after(); }
                else if (V & 2) { mbar_wait(&ready, 0); tc_fence_after(); }
                const uint64_t bst = bdesc0 + static_cast<uint64_t>(st * (32768 >> 4));
                const uint32_t ast = tm + g * 64;
#pragma unroll
                for (int i = 0; i < 8; ++i)
                    umma_ts_e(dcol, ast + (i >> 2) * 32 + (i & 3) * 8,
                              bst + static_cast<uint64_t>(((i >> 2) * 16384 + (i & 3) * 32) >> 4), idesc,
                              (g | i) ? 1u : 0u);
                if (V & 1) commit_e(&tempty[st]);
                if (DLY) {  // issuer stall after each stage of 8 MMAs (512 cycles of MMA work)
                    const unsigned long long td = clock64();
                    while (clock64() - td < DLY) { }
                }
            }
            if (V & 4) commit_e(&sfull[sb]);
        }
        commit_e(&sfull[0]);
        if (!(V & 4)) mbar_wait(&sfull[0], 0);
        __syncwarp();
        if (lane == 0) out[blockIdx.x] = clock64() - t0;
        if (lane == 0) mbar_arrive(&never);
        if (lane == 0) done_s = 1;
    } else if (KL == 2 && warp < 8) {
        // busy softmax-like warps: FFMA + MUFU.EX2 chains with ILP until the issuer is done
        float a[16];
        for (int i = 0; i < 16; ++i) a[i] = threadIdx.x * 0.001f + i;
        int it = 0;
        while (!done_s) {
#pragma unroll
            for (int i = 0; i < 16; ++i) {
                a[i] = fmaf(a[i], 0.999f, -0.5f);
                a[i] = ex2_approx(a[i] * 0.01f) + a[i];
            }
            if ((++it & 255) == 0) __nanosleep(0);
        }
        float s = 0.f;
        for (int i = 0; i < 16; ++i) s += a[i];
        if (s == 1234.5f) out[0] = 0;
    } else if (KL && warp < 8) {
        for (int t = 0; t < tiles; ++t) {
            const uint32_t sb = t & 1, sph = (t >> 1) & 1;
            mbar_wait(&sfull[sb], sph);
            tc_fence_after();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sempty[sb]);
        }
    } else if (KL && warp == W_TMA) {
        if (lane == 0)
            for (int pc = 0; pc < tiles * 4; ++pc) {
                const uint32_t st = pc & 3, ph = (pc >> 2) & 1;
                mbar_wait(&tempty[st], ph ^ 1);
                mbar_arrive(&tfull[st]);
            }
    } else if (KL) {
    } else if (SPIN && warp >= 4) {
        mbar_wait(&never, 0);
    } else if (MIX && (crank & 1)) {
        if (SPIN && warp >= 4) mbar_wait(&never, 0);
    } else if (warp == 2 && (V & 4)) {
        // softmax: wait S, release it
        for (int t = 0; t < tiles; ++t) {
            const uint32_t sb = t & 1, sph = (t >> 1) & 1;
            mbar_wait(&sfull[sb], sph);
            tc_fence_after();
            __syncwarp();
            if (lane == 0) mbar_arrive(&sempty[sb]);
        }
    } else if (warp == 3 && (V & 8) && lane == 0) {
        // "TMA": refill each stage as soon as the MMAs released it (no data)
        for (int pc = 0; pc < tiles * 4; ++pc) {
            const uint32_t st = pc & 3, ph = (pc >> 2) & 1;
            mbar_wait(&tempty[st], ph ^ 1);
            mbar_arrive(&tfull[st]);
        }
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (warp == 0) tmem_dealloc(tm, 512);
}

template <int V, int RND = 0, int SPIN = 0, int CL = 1, int MIX = 0, int KL = 0, int DLY = 0>
void run(const char *name, int tiles = 2000, int reps = 1, int smem = 140000) {
    const int G = 148;
    unsigned long long *d;
    cudaMalloc(&d, G * 8);
    cudaFuncSetAttribute(bench<V, RND, SPIN, MIX, KL, DLY>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int nthr = (SPIN || KL) ? 352 : 128;
    cudaLaunchConfig_t lc = {};
    lc.gridDim = dim3(G);
    lc.blockDim = dim3(nthr);
    lc.dynamicSmemBytes = smem;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = CL;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    lc.attrs = at;
    lc.numAttrs = 1;
    cudaLaunchKernelEx(&lc, bench<V, RND, SPIN, MIX, KL, DLY>, d, 50);
    cudaError_t err = cudaDeviceSynchronize();
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    float ms = 0;
    for (int r = 0; r < reps; ++r) {
        cudaEventRecord(e0);
        cudaLaunchKernelEx(&lc, bench<V, RND, SPIN, MIX, KL, DLY>, d, tiles);
        cudaEventRecord(e1);
        err = cudaDeviceSynchronize();
        cudaEventElapsedTime(&ms, e0, e1);
    }
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    double cyc = 0, cyc1 = 0;
    for (int i = 0; i < G; i += (MIX ? 2 : 1)) cyc += h[i];
    cyc /= (MIX ? G / 2 : G);
    if (MIX) { for (int i = 1; i < G; i += 2) cyc1 += h[i]; cyc1 /= G / 2; }
    printf("%-44s err=%d cycles/MMA %.1f (floor 64)", name, (int)err, cyc / (tiles * 32.0));
    if (MIX) printf("   | odd CTAs SS N=256: %.1f cycles/MMA (floor 128)", cyc1 / (tiles * 16.0));
    printf("  [last of %d launches: %.2f ms, clock %.0f MHz, %.0f TFLOP/s]", reps, ms, cyc / (ms * 1e3),
           2.0 * 128 * 128 * 16 * 32.0 * tiles * (MIX ? G / 2 : G) / (ms * 1e-3) / 1e12);
    printf("\n");
    cudaFree(d);
}

int main() {
    run<11, 1>("V11 random (no S dbuf)");
    run<11, 1, 0, 1, 0, 2>("V11 + 8 busy ALU warps (kernel-like)");
    run<11, 1, 0, 1, 0, 2, 0>("V11 + 8 busy ALU warps, again");
    return 0;
}
