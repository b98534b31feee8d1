// umma_bench.cu -- microbenchmark of tcgen05.mma issue/execution cost per instruction
// for the operand shapes the DCP kernels can use (SS vs A-from-TMEM, N = 64/128/256,
// K-major vs MN-major).  One CTA per SM issues back-to-back MMAs on smem/TMEM
// operands (contents irrelevant), then reports cycles per instruction.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o umma_bench umma_bench.cu
#include <cstdio>
#include <cstdint>
#include "../paper_2105_10375_b200/csrc/sm100.cuh"
using namespace f2c;

__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a_tmem, uint64_t bdesc, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
                 "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                 :: "r"(d), "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(acc) : "memory");
}

__device__ volatile int g_stop;
template <int N, bool TS, int AMN, int BMN, int LDW = 0>
__global__ void __launch_bounds__(256, 1) bench(unsigned long long *out, int iters) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    uint8_t *s = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5;
    if (warp == 0) { tmem_alloc(&tbase, 512); tmem_relinquish(); }
    if (threadIdx.x == 32) { mbar_init(&bar, 1); fence_mbar_init(); }
    for (int i = threadIdx.x; i < 196608 / 4; i += 256) reinterpret_cast<uint32_t *>(s)[i] = 0;
    fence_proxy_async_smem();
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tm = tbase;
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = umma_idesc_bf16(128, N, AMN, BMN);
        const uint32_t sa = smem_u32(s), sb = smem_u32(s + 65536);
        unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it) {
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                uint64_t a = AMN ? umma_desc_sw128(sa + (k & 3) * 2048, 16384, 1024)
                                 : umma_desc_sw128(sa + (k & 3) * 32, 16, 1024);
                uint64_t b = BMN ? umma_desc_sw128(sb + (k & 3) * 2048, 16384, 1024)
                                 : umma_desc_sw128(sb + (k & 3) * 32, 16, 1024);
                if (TS) umma_ts(tm + 256, tm + ((k & 3) * 8), b, idesc, 1);
                else umma_bf16(tm + 256, a, b, idesc, 1);
            }
        }
        umma_commit(&bar);
        mbar_wait(&bar, 0);
        unsigned long long t1 = clock64();
        out[blockIdx.x] = t1 - t0;
        g_stop = 1;
    } else if (LDW && warp >= 4 && warp < 4 + LDW) {
        // concurrent TMEM readers: tcgen05.ld of 32 columns at the S region (cols 384..)
        float v[32];
        float acc = 0.f;
        for (int it = 0; it < iters * 4 && !g_stop; ++it) {
            tmem_ld32(tm + ((uint32_t)((warp & 3) * 32) << 16) + 384 + (it & 1) * 32, v);
            tmem_wait_ld();
            acc += v[it & 31];
        }
        if (acc == 12345.f) out[0] = 0;
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (warp == 0) tmem_dealloc(tm, 512);
}

template <int N, bool TS, int AMN, int BMN, int LDW = 0>
void run(const char *name) {
    const int G = 148, iters = 2048;
    unsigned long long *d;
    cudaMalloc(&d, G * 8);
    auto k = bench<N, TS, AMN, BMN, LDW>;
    int zero = 0; cudaMemcpyToSymbol(g_stop, &zero, sizeof(int));
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    k<<<G, 256, 200000>>>(d, 64);
    cudaDeviceSynchronize();
    cudaMemcpyToSymbol(g_stop, &zero, sizeof(int));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    cudaEventRecord(e0);
    k<<<G, 256, 200000>>>(d, iters);
    cudaEventRecord(e1);
    cudaError_t err = cudaDeviceSynchronize();
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    unsigned long long h[148];
    cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    double cyc = 0; for (int i = 0; i < G; ++i) cyc += h[i]; cyc /= G;
    const double ninst = iters * 8.0;
    const double flops = 2.0 * 128 * N * 16 * ninst * G;
    printf("%-28s err=%d cycles/instr %.1f  (floor %d)  TFLOP/s %.0f  eff-clock %.0f MHz\n", name, (int)err,
           cyc / ninst, 128 * N / 256, flops / (ms * 1e-3) / 1e12, cyc / (ms * 1e-3) / 1e6);
    cudaFree(d);
}


__device__ __forceinline__ uint32_t mapa_shared(uint32_t addr, uint32_t cta) {
    uint32_t r; asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(addr), "r"(cta)); return r;
}
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1) dsmem_bench(unsigned long long *out, int iters, int bytes) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[2], empty[2];
    uint32_t rank; asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
    uint8_t *s = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    if (threadIdx.x == 0) { for (int i = 0; i < 2; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); } fence_mbar_init(); }
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
    if (threadIdx.x == 0) {
        unsigned long long t0 = clock64();
        if (rank == 0) {
            for (int it = 0; it < iters; ++it) {
                int b = it & 1; uint32_t ph = (it >> 1) & 1;
                mbar_wait(&empty[b], ph ^ 1);   // remote-arrived by rank 1
                uint32_t dst = mapa_shared(smem_u32(s + b * 65536), 1);
                uint32_t rbar = mapa_shared(smem_u32(&full[b]), 1);
                asm volatile("cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             :: "r"(dst), "r"(smem_u32(s + 131072)), "r"(bytes), "r"(rbar) : "memory");
            }
            asm volatile("cp.async.bulk.commit_group; cp.async.bulk.wait_group 0;" ::: "memory");
        } else {
            for (int it = 0; it < iters; ++it) {
                int b = it & 1; uint32_t ph = (it >> 1) & 1;
                mbar_arrive_expect_tx(&full[b], bytes);
                mbar_wait(&full[b], ph);
                uint32_t rbar = mapa_shared(smem_u32(&empty[b]), 0);
                asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" :: "r"(rbar) : "memory");
            }
        }
        out[blockIdx.x] = clock64() - t0;
    }
    asm volatile("barrier.cluster.arrive.release.aligned; barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

int main() {
    run<128, true, 0, 0>("TS  N=128 B:K");
    run<128, true, 0, 0, 1>("TS  N=128 B:K +1 LDTM warp");
    run<128, true, 0, 0, 4>("TS  N=128 B:K +4 LDTM warps");
    run<128, false, 0, 0>("SS  N=128");
    run<128, false, 0, 0, 4>("SS  N=128 +4 LDTM warps");
    run<256, false, 0, 1>("SS  N=256 A:K B:MN");
    run<256, false, 0, 1, 4>("SS  N=256 +4 LDTM warps");
    return 0;
}
