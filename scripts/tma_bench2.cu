// tma_bench2.cu -- TMA latency/throughput with 2D 16 KB boxes vs 3D 64 KB boxes
// ([64 d] x [128 slots] x [4 chunks] -> chunk-major smem), all CTAs in lockstep on an
// L2-resident or HBM-resident [R x 512] bf16 tensor.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "../paper_2105_10375_b200/csrc/sm100.cuh"
using namespace f2c;

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *m, uint64_t *bar, int x, int y, int z) {
    asm volatile("cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5}], [%2];"
                 :: "r"(smem_u32(dst)), "l"(reinterpret_cast<uint64_t>(m)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z) : "memory");
}

__global__ void __launch_bounds__(64, 1) stream(const __grid_constant__ CUtensorMap tm, int dims3, int NS, int box_bytes,
                                                int boxes, int rows_total, unsigned long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[16], empty[16];
    uint8_t *s = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    if (threadIdx.x == 0) { for (int i = 0; i < NS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); } fence_mbar_init(); }
    __syncthreads();
    unsigned long long t0 = clock64();
    const int per_tile = dims3 ? 2 : 8;
    if (threadIdx.x == 0) {
        for (int pc = 0; pc < boxes; ++pc) {
            int st = pc % NS; uint32_t ph = (pc / NS) & 1;
            mbar_wait(&empty[st], ph ^ 1);
            mbar_arrive_expect_tx(&full[st], box_bytes);
            int tile = (pc / per_tile) % (rows_total / 128), c = pc % per_tile;
            if (dims3) tma_load_3d(s + st * box_bytes, &tm, &full[st], 0, tile * 128, c * 4);
            else tma_load_2d(s + st * box_bytes, &tm, &full[st], c * 64, tile * 128);
        }
    } else if (threadIdx.x == 32) {
        for (int pc = 0; pc < boxes; ++pc) {
            int st = pc % NS; uint32_t ph = (pc / NS) & 1;
            mbar_wait(&full[st], ph);
            mbar_arrive(&empty[st]);
        }
        out[blockIdx.x] = clock64() - t0;
    }
}

int main() {
    PFN_cuTensorMapEncodeTiled_v12000 enc; cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", (void **)&enc, cudaEnableDefault, &q);
    const long long R_big = 1 << 21;
    void *buf; cudaMalloc(&buf, R_big * 1024); cudaMemset(buf, 0, R_big * 1024);
    unsigned long long *d; cudaMalloc(&d, 148 * 8);
    cudaFuncSetAttribute(stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 230000);
    for (long long R : {(long long)65536, R_big}) {
        CUtensorMap t2, t3;
        { cuuint64_t dims[2] = {512, (cuuint64_t)R}; cuuint64_t st[1] = {1024}; cuuint32_t box[2] = {64, 128}; cuuint32_t es[2] = {1, 1};
          enc(&t2, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE); }
        { cuuint64_t dims[3] = {64, (cuuint64_t)R, 8}; cuuint64_t st[2] = {1024, 128}; cuuint32_t box[3] = {64, 128, 4}; cuuint32_t es[3] = {1, 1, 1};
          CUresult r = enc(&t3, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, buf, dims, st, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
          if (r) printf("3d encode failed %d\n", (int)r); }
        for (int dims3 : {0, 1}) {
            int bb = dims3 ? 65536 : 16384;
            for (int NS : {1, 2, 3, 4, 9, 13}) {
                if (NS * bb > 215000) continue;
                int boxes = dims3 ? 400 : 1600;
                stream<<<148, 64, NS * bb + 2048>>>(dims3 ? t3 : t2, dims3, NS, bb, 16, (int)R, d);
                cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
                cudaEventRecord(e0);
                stream<<<148, 64, NS * bb + 2048>>>(dims3 ? t3 : t2, dims3, NS, bb, boxes, (int)R, d);
                cudaEventRecord(e1);
                cudaError_t err = cudaDeviceSynchronize();
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                unsigned long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
                double cyc = 0; for (int i = 0; i < 148; ++i) cyc += h[i]; cyc /= 148;
                printf("%s %s NS=%2d err=%d: %.0f cyc/box  %.1f B/cyc/SM  total %.2f TB/s\n", R == R_big ? "HBM" : "L2 ",
                       dims3 ? "3D 64KB" : "2D 16KB", NS, (int)err, cyc / boxes, (double)boxes * bb / cyc,
                       (double)boxes * bb * 148 / (ms * 1e-3) / 1e12);
            }
        }
    }
}
