// umma_tma_bench.cu -- MMA issue rate while a TMA stream writes shared memory concurrently.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "../paper_2105_10375_b200/csrc/sm100.cuh"
using namespace f2c;
__device__ __forceinline__ void umma_ts(uint32_t d, uint32_t a, uint64_t b, uint32_t idesc, uint32_t acc) {
    asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n}\n"
                 :: "r"(d), "r"(a), "l"(b), "r"(idesc), "r"(acc) : "memory");
}
__device__ __forceinline__ void tma3(void *dst, const CUtensorMap *m, uint64_t *bar, int x, int y, int z) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                 :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z) : "memory");
}
__device__ volatile int g_stop;
template <int N, bool TS>
__global__ void __launch_bounds__(128, 1) k(const __grid_constant__ CUtensorMap tm, int tma_on, int nbox, unsigned long long *out, int iters) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t bar, full[4], empty[4];
    __shared__ uint32_t tbase;
    uint8_t *s = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    const int warp = threadIdx.x >> 5;
    if (warp == 0) { tmem_alloc(&tbase, 512); tmem_relinquish(); }
    if (threadIdx.x == 32) { mbar_init(&bar, 1); for (int i = 0; i < 4; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); } fence_mbar_init(); }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    const uint32_t tm0 = tbase;
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = umma_idesc_bf16(128, N, 0, 0);
        const uint32_t sb = smem_u32(s);
        unsigned long long t0 = clock64();
        for (int it = 0; it < iters; ++it)
#pragma unroll
            for (int kk = 0; kk < 8; ++kk) {
                uint64_t b = umma_desc_sw128(sb + (kk & 3) * 32 + (kk >> 2) * 16384, 16, 1024);
                if (TS) umma_ts(tm0 + 256 + (it & 1) * 128, tm0 + kk * 8, b, idesc, 1);
                else umma_bf16(tm0 + 256 + (it & 1) * 128, umma_desc_sw128(sb + 32768 + (kk & 3) * 32, 16, 1024), b, idesc, 1);
            }
        umma_commit(&bar); mbar_wait(&bar, 0);
        out[blockIdx.x] = clock64() - t0;
        g_stop = 1;
    } else if (threadIdx.x == 32 && tma_on) {
        // stream 32 KB boxes into a separate 4-stage ring at smem offset 65536
        for (int pc = 0; !g_stop && pc < 1000000; ++pc) {
            int st = pc & 3; uint32_t ph = (pc >> 2) & 1;
            mbar_wait(&empty[st], ph ^ 1);
            mbar_arrive_expect_tx(&full[st], 32768);
            tma3(s + 65536 + st * 32768, &tm, &full[st], 0, (pc % nbox) * 128, 0);
        }
    } else if (threadIdx.x == 64 && tma_on) {
        for (int pc = 0; !g_stop && pc < 1000000; ++pc) {
            int st = pc & 3; uint32_t ph = (pc >> 2) & 1;
            mbar_wait(&full[st], ph);
            mbar_arrive(&empty[st]);
        }
    }
    tc_fence_before(); __syncthreads(); tc_fence_after();
    if (warp == 0) tmem_dealloc(tm0, 512);
}
template <int N, bool TS>
void run(const CUtensorMap &tm, int tma_on, const char *name) {
    unsigned long long *d; cudaMalloc(&d, 148 * 8);
    auto kk = k<N, TS>;
    cudaFuncSetAttribute(kk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200000);
    int z = 0; cudaMemcpyToSymbol(g_stop, &z, 4);
    const int iters = 4096;
    kk<<<148, 128, 200000>>>(tm, tma_on, 256, d, iters);
    cudaError_t e = cudaDeviceSynchronize();
    unsigned long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
    double c = 0; for (int i = 0; i < 148; ++i) c += h[i]; c /= 148;
    printf("%-36s err=%d cycles/MMA %.1f (floor %d)\n", name, (int)e, c / (iters * 8.0), N / 2);
    cudaFree(d);
}
int main() {
    PFN_cuTensorMapEncodeTiled_v12000 enc; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    void *buf; cudaMalloc(&buf, 65536LL * 1024); cudaMemset(buf, 0, 65536LL * 1024);
    CUtensorMap tm; cuuint64_t dims[3] = {64, 65536, 8}; cuuint64_t st[2] = {1024, 128};
    cuuint32_t box[3] = {64, 128, 2}; cuuint32_t es[3] = {1, 1, 1};
    enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    run<128, true>(tm, 0, "TS N=128 alt-D");
    run<128, true>(tm, 1, "TS N=128 alt-D + TMA stream");
    run<128, false>(tm, 0, "SS N=128 alt-D");
    run<128, false>(tm, 1, "SS N=128 alt-D + TMA stream");
    run<256, false>(tm, 0, "SS N=256");
    run<256, false>(tm, 1, "SS N=256 + TMA stream");
}
