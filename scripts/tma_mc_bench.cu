// tma_mc_bench.cu -- does sharing pool tiles between CTAs cut L2->SM (LTS) traffic?
// 148 CTAs stream 64 KB 3D TMA boxes ([64 d] x [128 slots] x [4 chunks]) of an L2-resident
// bf16 tensor into a smem ring and release them immediately.  Modes:
//   0 distinct : every CTA streams its own tiles (unique bytes = delivered bytes)
//   1 same     : every CTA streams the same tiles (no synchronisation between CTAs)
//   2 mc       : clusters of CS CTAs; rank 0 multicasts each box to the whole cluster
//   3 same-cl  : clusters of CS CTAs read their cluster's tiles with unicast loads
// Prints delivered bytes/s (sum over CTAs) and cycles per box.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "../paper_2105_10375_b200/csrc/sm100.cuh"
using namespace f2c;

__device__ __forceinline__ uint32_t ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t nctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t mapa(uint32_t a, uint32_t cta) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(a), "r"(cta));
    return r;
}
__device__ __forceinline__ void cl_sync() {
    asm volatile("barrier.cluster.arrive.release.aligned;\nbarrier.cluster.wait.acquire.aligned;" ::: "memory");
}
__device__ __forceinline__ void tma3(void *dst, const CUtensorMap *m, uint64_t *bar, int x, int y, int z) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                 :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z) : "memory");
}
__device__ __forceinline__ void tma3_mc(void *dst, const CUtensorMap *m, uint64_t *bar, int x, int y, int z, uint16_t mask) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes.multicast::cluster [%0], [%1, {%3, %4, %5}], [%2], %6;"
                 :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z), "h"(mask) : "memory");
}

constexpr int BOX = 65536;

__global__ void __launch_bounds__(64, 1) stream(const __grid_constant__ CUtensorMap tm, int mode, int NS, int boxes,
                                                int tiles_per_set, unsigned long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[8], empty[8];
    uint8_t *s = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    const uint32_t cr = ctarank(), cn = nctarank();
    const int cluster = blockIdx.x / cn;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], mode == 2 ? cn : 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    cl_sync();
    // tile set: distinct per CTA (0), shared by all (1), per cluster (2, 3)
    const int set = mode == 0 ? blockIdx.x : (mode == 1 ? 0 : cluster);
    unsigned long long t0 = clock64();
    if (threadIdx.x == 0) {
        if (mode != 2 || cr == 0) {
            for (int pc = 0; pc < boxes; ++pc) {
                const int st = pc % NS;
                const uint32_t ph = (pc / NS) & 1;
                mbar_wait(&empty[st], ph ^ 1);
                const int tile = set * tiles_per_set + (pc % tiles_per_set);
                if (mode == 2) {
                    tma3_mc(s + st * BOX, &tm, &full[st], 0, tile * 128, 0, static_cast<uint16_t>((1u << cn) - 1));
                } else {
                    mbar_arrive_expect_tx(&full[st], BOX);
                    tma3(s + st * BOX, &tm, &full[st], 0, tile * 128, 0);
                }
            }
        }
    } else if (threadIdx.x == 32) {
        if (mode == 2)
            for (int i = 0; i < NS; ++i) mbar_arrive_expect_tx(&full[i], BOX);
        for (int pc = 0; pc < boxes; ++pc) {
            const int st = pc % NS;
            const uint32_t ph = (pc / NS) & 1;
            mbar_wait(&full[st], ph);
            if (mode == 2) {
                if (pc + NS < boxes) mbar_arrive_expect_tx(&full[st], BOX);  // arm the next phase
                const uint32_t rb = mapa(smem_u32(&empty[st]), 0);
                asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rb) : "memory");
            } else {
                mbar_arrive(&empty[st]);
            }
        }
        out[blockIdx.x] = clock64() - t0;
    }
    __syncthreads();
    cl_sync();
}

int main() {
    PFN_cuTensorMapEncodeTiled_v12000 enc;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    const long long R = 148 * 4 * 128;  // 148 sets of 4 tiles: 38.8 MB, L2-resident
    void *buf;
    cudaMalloc(&buf, R * 1024);
    cudaMemset(buf, 0, R * 1024);
    unsigned long long *d;
    cudaMalloc(&d, 148 * 8);
    CUtensorMap t3;
    {
        cuuint64_t dims[3] = {64, (cuuint64_t)R, 8};
        cuuint64_t st[2] = {1024, 128};
        cuuint32_t box[3] = {64, 128, 4};
        cuuint32_t es[3] = {1, 1, 1};
        CUresult r = enc(&t3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                         CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
        if (r) printf("encode failed %d\n", (int)r);
    }
    const int NS = 3, boxes = 600;
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, NS * BOX + 2048);
    cudaFuncSetAttribute(stream, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
    struct Cfg { int mode, cs; const char *name; } cfgs[] = {
        {0, 1, "distinct     "}, {1, 1, "same (all)   "}, {3, 2, "same-cl  CS=2"}, {3, 4, "same-cl  CS=4"},
        {2, 2, "multicast CS=2"}, {2, 4, "multicast CS=4"}, {2, 8, "multicast CS=8"}};
    for (auto c : cfgs) {
        for (int rep = 0; rep < 2; ++rep) {
            cudaLaunchConfig_t lc = {};
            lc.gridDim = dim3(148 / c.cs * c.cs);
            lc.blockDim = dim3(64);
            lc.dynamicSmemBytes = NS * BOX + 2048;
            cudaLaunchAttribute at[1];
            at[0].id = cudaLaunchAttributeClusterDimension;
            at[0].val.clusterDim.x = c.cs;
            at[0].val.clusterDim.y = 1;
            at[0].val.clusterDim.z = 1;
            lc.attrs = at;
            lc.numAttrs = 1;
            cudaEvent_t e0, e1;
            cudaEventCreate(&e0);
            cudaEventCreate(&e1);
            cudaEventRecord(e0);
            cudaError_t le = cudaLaunchKernelEx(&lc, stream, t3, c.mode, NS, boxes, 4, d);
            cudaEventRecord(e1);
            cudaError_t err = cudaDeviceSynchronize();
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            const int nb = 148 / c.cs * c.cs;
            unsigned long long h[148];
            cudaMemcpy(h, d, nb * 8, cudaMemcpyDeviceToHost);
            double cyc = 0;
            for (int i = 0; i < nb; ++i) cyc += h[i];
            cyc /= nb;
            if (rep == 1)
                printf("%s launch=%d err=%d: %.0f cyc/box  %.1f B/cyc/SM delivered  %.2f TB/s delivered\n", c.name,
                       (int)le, (int)err, cyc / boxes, (double)boxes * BOX / cyc,
                       (double)boxes * BOX * nb / (ms * 1e-3) / 1e12);
        }
    }
    return 0;
}
