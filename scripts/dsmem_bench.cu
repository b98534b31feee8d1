// dsmem_bench.cu -- P hand-off bandwidth between the two CTAs of a cluster (the fused
// kernel moves a 32 KB bf16 P tile from the producer CTA to the consumer CTA every tile).
// Modes (producer CTA = rank 0, 256 threads; consumer = rank 1 waits and releases):
//   0 bulk  : threads write the tile to local smem (staging), one lane issues
//             cp.async.bulk.shared::cluster.shared::cta in 4 x 8 KB pieces (the kernel's way)
//   1 stasync: every thread stores its 128 B of the tile straight into the consumer's smem
//             with st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 (8 per thread)
// Double-buffered slots on both sides; prints cycles per 32 KB tile (producer side).
#include <cstdio>
#include <cstdint>
#include "../paper_2105_10375_b200/csrc/sm100.cuh"
using namespace f2c;

constexpr int TILE = 32768;
__device__ __forceinline__ uint32_t ctarank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
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
__device__ __forceinline__ void remote_arrive(uint32_t rbar) {
    asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(rbar) : "memory");
}

__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(256, 1) kern(int mode, int iters, unsigned long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[4], freeb[4];   // full: consumer side; freeb: producer side
    uint8_t *s = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    const uint32_t cr = ctarank();
    const int tid = threadIdx.x, lane = tid & 31;
    if (tid == 0) {
        for (int i = 0; i < 4; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&freeb[i], 1);
        }
        fence_mbar_init();
    }
    __syncthreads();
    cl_sync();
    unsigned long long t0 = clock64();
    if (cr == 1) {
        // consumer: slots at s + b*TILE; arm, wait, release
        if (tid == 0) {
            for (int b = 0; b < 4; ++b) mbar_arrive_expect_tx(&full[b], TILE);
            for (int it = 0; it < iters; ++it) {
                const int b = it & 3;
                mbar_wait(&full[b], (it >> 2) & 1);
                if (it + 4 < iters) mbar_arrive_expect_tx(&full[b], TILE);
                remote_arrive(mapa(smem_u32(&freeb[b]), 0));
            }
        }
    } else {
        uint8_t *stage = s + 4 * TILE;  // producer staging (mode 0)
        for (int it = 0; it < iters; ++it) {
            const int b = it & 3;
            mbar_wait(&freeb[b], ((it >> 2) & 1) ^ 1);  // consumer released slot b
            const uint32_t dst = mapa(smem_u32(s + b * TILE), 1);
            const uint32_t rbar = mapa(smem_u32(&full[b]), 1);
            if (mode == 0) {
                // write the tile locally (128 B per thread), then one bulk copy in 4 pieces
                const uint32_t la = smem_u32(stage + (b & 1) * TILE + tid * 128);
#pragma unroll
                for (int u = 0; u < 8; ++u) st_shared_v4(la + u * 16, it, u, tid, 0);
                fence_proxy_async_smem();
                __syncthreads();
                if (tid == 0) {
                    for (int c = 0; c < 4; ++c) {
                        asm volatile(
                            "cp.async.bulk.shared::cluster.shared::cta.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                                dst + c * 8192),
                            "r"(smem_u32(stage + (b & 1) * TILE) + c * 8192), "r"(8192), "r"(rbar)
                            : "memory");
                        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
                    }
                    asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory");  // (staging double-buffered)
                }
                __syncthreads();
            } else {
                // st.async: 8 x 16 B per thread straight into the consumer's slot
#pragma unroll
                for (int u = 0; u < 8; ++u) {
                    const uint32_t a = dst + tid * 128 + u * 16;
                    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.v4.b32 [%0], {%1, %2, %3, %4}, [%5];" ::"r"(a),
                                 "r"(it), "r"(u), "r"(tid), "r"(0), "r"(rbar)
                                 : "memory");
                }
            }
        }
    }
    if (tid == 0) out[blockIdx.x] = clock64() - t0;
    __syncthreads();
    cl_sync();
}

int main() {
    unsigned long long *d;
    cudaMalloc(&d, 148 * 8);
    const int smem = 6 * TILE + 2048;
    cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const int iters = 2000;
    const char *names[] = {"bulk copy (staging + 4 x 8 KB)", "st.async v4 from 256 threads"};
    for (int mode = 0; mode < 2; ++mode) {
        for (int grid : {2, 148}) {
            for (int rep = 0; rep < 2; ++rep) {
                kern<<<grid, 256, smem>>>(mode, iters, d);
                cudaError_t e = cudaDeviceSynchronize();
                unsigned long long h[148];
                cudaMemcpy(h, d, grid * 8, cudaMemcpyDeviceToHost);
                double cyc = 0;
                for (int i = 0; i < grid; i += 2) cyc += h[i];
                cyc /= (grid / 2);
                if (rep == 1)
                    printf("%-34s grid %3d err=%d: %.0f cycles per 32 KB tile = %.1f B/clk\n", names[mode], grid, (int)e,
                           cyc / iters, TILE / (cyc / iters));
            }
        }
    }
    return 0;
}
