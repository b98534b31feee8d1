// tma_bench.cu -- TMA ingest rate per SM: one thread streams [rows x 64] bf16 SW128 boxes
// of a [R x 512] tensor into a ring of NS stages; another waits and frees them.
#include <cstdio>
#include <cstdint>
#include <cuda.h>
#include <cudaTypedefs.h>
#include "../paper_2105_10375_b200/csrc/sm100.cuh"
using namespace f2c;

__global__ void __launch_bounds__(64, 1) tma_stream(const __grid_constant__ CUtensorMap tm, int NS, int box_rows,
                                                    int tiles, int rows_total, int same_range,
                                                    unsigned long long *out) {
    extern __shared__ __align__(1024) uint8_t sm[];
    __shared__ uint64_t full[16], empty[16];
    uint8_t *s = reinterpret_cast<uint8_t *>((reinterpret_cast<uintptr_t>(sm) + 1023) & ~uintptr_t(1023));
    const int box_bytes = box_rows * 128;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i) { mbar_init(&full[i], 1); mbar_init(&empty[i], 1); }
        fence_mbar_init();
    }
    __syncthreads();
    // each CTA walks its own row range (or all CTAs the same range)
    const int chunks_per_tile = 8;  // 8 x 64 = 512 d
    const int tiles_total = rows_total / box_rows;
    const int start = same_range ? 0 : (int)((long long)blockIdx.x * tiles_total / gridDim.x);
    unsigned long long t0 = clock64();
    if (threadIdx.x == 0) {
        int pc = 0;
        for (int t = 0; t < tiles; ++t)
            for (int c = 0; c < chunks_per_tile; ++c, ++pc) {
                int st = pc % NS; uint32_t ph = (pc / NS) & 1;
                mbar_wait(&empty[st], ph ^ 1);
                mbar_arrive_expect_tx(&full[st], box_bytes);
                tma_load_2d(s + st * box_bytes, &tm, &full[st], c * 64, ((start + t) % tiles_total) * box_rows);
            }
    } else if (threadIdx.x == 32) {
        int pc = 0;
        for (int t = 0; t < tiles; ++t)
            for (int c = 0; c < chunks_per_tile; ++c, ++pc) {
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
    const long long R_big = 1 << 21;  // 2M rows x 512 bf16 = 2 GB
    void *buf; cudaMalloc(&buf, R_big * 1024);
    cudaMemset(buf, 0, R_big * 1024);
    unsigned long long *d; cudaMalloc(&d, 148 * 8);
    cudaFuncSetAttribute(tma_stream, cudaFuncAttributeMaxDynamicSharedMemorySize, 230000);
    for (int box_rows : {128, 32}) {
        for (long long R : {R_big, (long long)65536}) {  // HBM-resident vs L2-resident (64 MB)
            CUtensorMap tm;
            cuuint64_t dims[2] = {512, (cuuint64_t)R}; cuuint64_t strides[1] = {1024};
            cuuint32_t box[2] = {64, (cuuint32_t)box_rows}; cuuint32_t es[2] = {1, 1};
            enc(&tm, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, buf, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            for (int same : {0, 1})
            for (int NS : {4, 9, 14}) {
                const int box_bytes = box_rows * 128;
                if (NS * box_bytes > 220000) continue;
                const int tiles = (box_rows == 128 ? 400 : 1600);
                tma_stream<<<148, 64, NS * box_bytes + 2048>>>(tm, NS, box_rows, 8, (int)R, same, d);
                cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
                cudaEventRecord(e0);
                tma_stream<<<148, 64, NS * box_bytes + 2048>>>(tm, NS, box_rows, tiles, (int)R, same, d);
                cudaEventRecord(e1);
                cudaError_t err = cudaDeviceSynchronize();
                float ms; cudaEventElapsedTime(&ms, e0, e1);
                unsigned long long h[148]; cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
                double cyc = 0; for (int i = 0; i < 148; ++i) cyc += h[i]; cyc /= 148;
                double bytes = (double)tiles * 8 * box_bytes;
                printf("box %3dx64 src %s %s NS=%2d err=%d : %.1f B/cycle/SM, total %.2f TB/s\n", box_rows,
                       R == R_big ? "HBM(2GB)" : "L2(64MB)", same ? "same-range" : "own-range ", NS, (int)err,
                       bytes / cyc, bytes * 148 / (ms * 1e-3) / 1e12);
            }
        }
    }
    return 0;
}
