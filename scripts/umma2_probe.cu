// umma2_probe.cu -- semantics probe for 2-CTA tcgen05.mma (cta_group::2) before it is used in
// the fused kernel: TMEM allocation for the pair, operand split (A by rows,
// B by N), the D layout in each CTA's TMEM, and the multicast commit.  D = A * B^T, bf16 in,
// fp32 out, K = 64 (4 MMAs of K = 16), both operands K-major SW128 in shared memory.
// Modes: 1 = cta_group::1, M = 128 (reference); 2 = cta_group::2, M = 256; 3 = cta_group::2, M = 128.
// Every CTA dumps its whole 128-lane x 128-column TMEM accumulator; the host finds each
// expected D row in the dumps.  Waits are bounded: a timeout traps instead of hanging.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>
#include <vector>
#include <cstring>
#include <cuda_bf16.h>
#include "../paper_2105_10375_b200/csrc/sm100.cuh"
using namespace f2c;

__device__ __forceinline__ uint32_t ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ void wait_bounded(uint64_t *bar, uint32_t parity, int *err) {
    for (long long it = 0; it < 20000000; ++it) {
        uint32_t ok;
        asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
        if (ok) return;
    }
    atomicExch(err, 1);
    asm volatile("trap;");
}
// K-major SW128 tile [rows x 64] bf16: element (r, k) at r*128 + (((2k)/16) ^ (r%8))*16 + (2k)%16
__device__ __forceinline__ uint32_t sw128_off(int r, int k) {
    return r * 128 + ((((2 * k) >> 4) ^ (r & 7)) << 4) + ((2 * k) & 15);
}

__global__ void __cluster_dims__(2, 1, 1) probe(int mode, const __nv_bfloat16 *A, const __nv_bfloat16 *B,
                                                float *dump, int *err) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    uint8_t *s = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    uint8_t *sA = s, *sB = s + 16384;
    const uint32_t cr = ctarank();
    const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    // operand rows held by this CTA
    const bool g1 = mode == 1 || mode >= 7;            // cta_group::1 modes (each CTA on its own)
    const int arows = (mode >= 3 && mode != 6) ? 64 : 128;
    const int a0 = g1 ? 0 : cr * arows;                // global A row offset
    const int brows = g1 ? 128 : 64;
    const int b0 = g1 ? 0 : cr * 64;                   // global B (N) row offset
    for (int i = tid; i < arows * 64; i += blockDim.x) {
        const int r = i / 64, k = i % 64;
        *reinterpret_cast<__nv_bfloat16 *>(sA + sw128_off(r, k)) = A[(a0 + r) * 64 + k];
    }
    for (int i = tid; i < brows * 64; i += blockDim.x) {
        const int r = i / 64, k = i % 64;
        *reinterpret_cast<__nv_bfloat16 *>(sB + sw128_off(r, k)) = B[(b0 + r) * 64 + k];
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (tid == 0) {
        mbar_init(&bar, 1);
        fence_mbar_init();
    }
    if (warp == 0) {
        if (g1) {
            asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tbase)) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
        } else {
            asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(smem_u32(&tbase)) : "memory");
            asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
        }
    }
    tc_fence_before();
    __syncthreads();
    cl_sync();
    tc_fence_after();
    const uint32_t tmem = tbase;
    // zero this CTA's accumulator region first (so stale data cannot pass for a result)
    if (warp < 4) {
        uint32_t z[32];
        for (int i = 0; i < 32; ++i) z[i] = 0;
        for (int c0 = 0; c0 < 128; c0 += 32)
            asm volatile(
                "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
                "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0),
                "r"(z[0]), "r"(z[1]), "r"(z[2]), "r"(z[3]), "r"(z[4]), "r"(z[5]), "r"(z[6]), "r"(z[7]), "r"(z[8]), "r"(z[9]),
                "r"(z[10]), "r"(z[11]), "r"(z[12]), "r"(z[13]), "r"(z[14]), "r"(z[15]), "r"(z[16]), "r"(z[17]), "r"(z[18]),
                "r"(z[19]), "r"(z[20]), "r"(z[21]), "r"(z[22]), "r"(z[23]), "r"(z[24]), "r"(z[25]), "r"(z[26]), "r"(z[27]),
                "r"(z[28]), "r"(z[29]), "r"(z[30]), "r"(z[31])
                : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    cl_sync();
    tc_fence_after();
    const int M = (mode == 2 || mode == 6) ? 256 : mode >= 7 ? 64 : 128;
    const uint32_t idesc = umma_idesc_bf16(M, 128, 0, 0);
    const bool issuer = g1 || cr == 0;
    // modes 4/5: A (this CTA's 64 rows x 64 K, bf16 pairs per 32-bit column) into TMEM columns
    // [128, 160): mode 4 = rows on lanes 0-63 (lanes 64-127 zero); mode 5 = rows on lanes 0-63
    // for K 0-31 and on lanes 64-127 for K 32-63 (columns [128, 144))
    const uint32_t ACOL = 128;
    if (mode >= 4 && mode != 7 && warp < 4) {  // (mode 6: M = 256, rows 0-127 of this CTA on lanes 0-127)
        uint32_t w[32];
        const int lr = warp * 32 + lane;  // TMEM lane
        for (int j = 0; j < 32; ++j) {
            int row = -1, k0 = 0;
            if (mode == 4 && lr < 64) { row = lr; k0 = 2 * j; }
            if (mode == 6) { row = lr; k0 = 2 * j; }
            if (mode == 8 && lr < 64) { row = lr; k0 = 2 * j; }                              // M = 64: rows on lanes 0-63
            if (mode == 9 && (lr & 31) < 16) { row = (lr >> 5) * 16 + (lr & 15); k0 = 2 * j; }  // lanes 0-15 of each quadrant
            if (mode == 5 && j < 16) { row = lr & 63; k0 = (lr < 64 ? 0 : 32) + 2 * j; }
            uint32_t v = 0;
            if (row >= 0) {
                const __nv_bfloat16 lo = A[(a0 + row) * 64 + k0], hi = A[(a0 + row) * 64 + k0 + 1];
                v = static_cast<uint32_t>(__bfloat16_as_ushort(lo)) | (static_cast<uint32_t>(__bfloat16_as_ushort(hi)) << 16);
            }
            w[j] = v;
        }
        asm volatile(
            "tcgen05.st.sync.aligned.32x32b.x32.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,%16,"
            "%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31,%32};" ::"r"(tmem + (static_cast<uint32_t>(warp * 32) << 16) + ACOL),
            "r"(w[0]), "r"(w[1]), "r"(w[2]), "r"(w[3]), "r"(w[4]), "r"(w[5]), "r"(w[6]), "r"(w[7]), "r"(w[8]), "r"(w[9]),
            "r"(w[10]), "r"(w[11]), "r"(w[12]), "r"(w[13]), "r"(w[14]), "r"(w[15]), "r"(w[16]), "r"(w[17]), "r"(w[18]),
            "r"(w[19]), "r"(w[20]), "r"(w[21]), "r"(w[22]), "r"(w[23]), "r"(w[24]), "r"(w[25]), "r"(w[26]), "r"(w[27]),
            "r"(w[28]), "r"(w[29]), "r"(w[30]), "r"(w[31])
            : "memory");
        asm volatile("tcgen05.wait::st.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    cl_sync();
    tc_fence_after();
    if (warp == 1 && issuer && lane == 0) {
        for (int ks = 0; ks < 4; ++ks) {
            const uint64_t ad = umma_desc_sw128(smem_u32(sA) + ks * 32, 16, 1024);
            const uint64_t bd = umma_desc_sw128(smem_u32(sB) + ks * 32, 16, 1024);
            const uint32_t acc = ks > 0;
            if (mode == 7) {
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                             ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc) : "memory");
            } else if (mode >= 8) {
                const uint32_t acol = tmem + ACOL + ks * 8;
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                             ::"r"(tmem), "r"(acol), "l"(bd), "r"(idesc), "r"(acc) : "memory");
            } else if (mode >= 4) {
                // A from TMEM: K step ks = 16 bf16 = 8 columns (modes 4, 6) or 4 columns (mode 5)
                const uint32_t acol = tmem + ACOL + ks * (mode == 5 ? 4 : 8);
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                             ::"r"(tmem), "r"(acol), "l"(bd), "r"(idesc), "r"(acc) : "memory");
            } else if (mode == 1)
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                             ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc) : "memory");
            else
                asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}\n"
                             ::"r"(tmem), "l"(ad), "l"(bd), "r"(idesc), "r"(acc) : "memory");
        }
        if (g1)
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(smem_u32(&bar)) : "memory");
        else
            asm volatile("tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64 [%0], %1;"
                         ::"r"(smem_u32(&bar)), "h"(static_cast<uint16_t>(3)) : "memory");
    }
    wait_bounded(&bar, 0, err);
    tc_fence_after();
    if (warp < 4) {  // dump all 128 lanes x 128 columns of this CTA's accumulator
        for (int c0 = 0; c0 < 128; c0 += 32) {
            float v[32];
            tmem_ld32(tmem + (static_cast<uint32_t>(warp * 32) << 16) + c0, v);
            tmem_wait_ld();
            for (int i = 0; i < 32; ++i)
                dump[(static_cast<size_t>(blockIdx.x) * 128 + warp * 32 + lane) * 128 + c0 + i] = v[i];
        }
    }
    tc_fence_before();
    __syncthreads();
    cl_sync();
    if (warp == 0) {
        if (g1)
            asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
        else
            asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
    }
}

static float bf(float x) {  // round to bf16
    uint32_t u;
    memcpy(&u, &x, 4);
    u = (u + 0x7fff + ((u >> 16) & 1)) & 0xffff0000u;
    float r;
    memcpy(&r, &u, 4);
    return r;
}

int main() {
    const int MR = 256, NR = 128, K = 64;
    std::vector<float> A(MR * K), B(NR * K);
    std::vector<__nv_bfloat16> Ah(MR * K), Bh(NR * K);
    srand(7);
    for (int i = 0; i < MR * K; ++i) { A[i] = bf((rand() % 17 - 8) / 8.0f); Ah[i] = __float2bfloat16(A[i]); }
    for (int i = 0; i < NR * K; ++i) { B[i] = bf((rand() % 17 - 8) / 8.0f); Bh[i] = __float2bfloat16(B[i]); }
    std::vector<double> D(MR * NR);
    for (int r = 0; r < MR; ++r)
        for (int n = 0; n < NR; ++n) {
            double acc = 0;
            for (int k = 0; k < K; ++k) acc += (double)A[r * K + k] * B[n * K + k];
            D[r * NR + n] = acc;
        }
    __nv_bfloat16 *dA, *dB;
    float *dump;
    int *derr;
    cudaMalloc(&dA, MR * K * 2);
    cudaMalloc(&dB, NR * K * 2);
    cudaMalloc(&dump, 2 * 128 * 128 * 4);
    cudaMalloc(&derr, 4);
    cudaMemcpy(dA, Ah.data(), MR * K * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, Bh.data(), NR * K * 2, cudaMemcpyHostToDevice);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 40000);
    for (int mode = 1; mode <= 9; ++mode) {
        cudaMemset(dump, 0xff, 2 * 128 * 128 * 4);
        cudaMemset(derr, 0, 4);
        probe<<<2, 128, 40000>>>(mode, dA, dB, dump, derr);
        cudaError_t e = cudaDeviceSynchronize();
        int herr = 0;
        cudaMemcpy(&herr, derr, 4, cudaMemcpyDeviceToHost);
        std::vector<float> h(2 * 128 * 128);
        cudaMemcpy(h.data(), dump, h.size() * 4, cudaMemcpyDeviceToHost);
        printf("mode %d: launch/sync %s, timeout flag %d\n", mode, cudaGetErrorString(e), herr);
        if (e != cudaSuccess) return 1;
        // for every expected D row (M rows of this mode), find (cta, lane) whose 128 columns match it
        const int M = (mode == 2 || mode == 6) ? 256 : mode >= 7 ? 64 : 128;
        int found = 0, col_half_match = 0;
        for (int r = 0; r < M; ++r) {
            int where = -1;
            for (int cta = 0; cta < 2 && where < 0; ++cta)
                for (int ln = 0; ln < 128 && where < 0; ++ln) {
                    bool ok = true;
                    for (int n = 0; n < NR && ok; ++n) ok = fabs(h[(cta * 128 + ln) * 128 + n] - D[r * NR + n]) < 1e-3;
                    if (ok) where = cta * 128 + ln;
                }
            if (where >= 0) ++found;
            if (r < 4 || r == M / 2 || r == M / 2 + 1 || r == M - 1 || ((mode == 3 || mode >= 7) && r % 8 == 0))
                printf("  D row %3d -> %s cta %d lane %d\n", r, where >= 0 ? "found at" : "NOT FOUND", where >= 0 ? where / 128 : -1,
                       where >= 0 ? where % 128 : -1);
            (void)col_half_match;
        }
        printf("  rows found: %d of %d\n", found, M);
        if (mode >= 3 && mode != 6 && mode < 7) {  // partial matches: 64-column halves of D rows anywhere in the dumps
            int shown = 0;
            for (int cta = 0; cta < 2; ++cta)
                for (int ln = 0; ln < 128; ++ln)
                    for (int cs = 0; cs < 128; cs += 64) {
                        bool nz = false;
                        for (int n = 0; n < 64; ++n) nz |= h[(cta * 128 + ln) * 128 + cs + n] != 0.f;
                        if (!nz) continue;
                        int hit = -1, hh = -1;
                        for (int r = 0; r < 256 && hit < 0; ++r)
                            for (int half = 0; half < 2 && hit < 0; ++half) {
                                bool ok = true;
                                for (int n = 0; n < 64 && ok; ++n)
                                    ok = fabs(h[(cta * 128 + ln) * 128 + cs + n] - D[r * NR + half * 64 + n]) < 1e-3;
                                if (ok) { hit = r; hh = half; }
                            }
                        if (shown < 40 && (ln % 16 == 0 || ln % 16 == 15))
                            printf("  cta %d lane %3d cols %3d..: D row %d cols %d..\n", cta, ln, cs, hit, hh * 64), ++shown;
                    }
            int nzl[2] = {0, 0};
            for (int cta = 0; cta < 2; ++cta)
                for (int ln = 0; ln < 128; ++ln) {
                    bool nz = false;
                    for (int n = 0; n < 128; ++n) nz |= h[(cta * 128 + ln) * 128 + n] != 0.f;
                    nzl[cta] += nz;
                }
            printf("  non-zero lanes: cta0 %d, cta1 %d\n", nzl[0], nzl[1]);
        }
    }
    return 0;
}
