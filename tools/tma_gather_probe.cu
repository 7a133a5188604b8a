// Probe (design evidence for a TMA-staged gather): in-place HBM streaming of
// "gather items" made of many small 2-D TMA boxes (rows of 128 B, 8 or 16 rows per box) from
// scattered 16 KiB tiles, three-stage ring, one producer warp per stage (all lanes issue), no transform.
// Reports GB/s (read + write) per box shape.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -cudart shared -o tools/tma_gather_probe tools/tma_gather_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

constexpr int STAGES = 3;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void box_of(uint64_t j, int b, uint32_t tiles, int box_rows, int structured, int& tile,
                                       int& x0, int& c0) {
    if (structured) {  // C3-like: the items of a unit are its sub-blocks, taken by consecutive CTAs
        const int nsub = (32 / box_rows) * 4;
        const uint64_t unit = j / nsub;
        const int sub = (int)(j % nsub);
        tile = (int)((unit * 64 + (uint64_t)b * 977) % tiles);
        x0 = (sub / 4) * box_rows;
        c0 = (sub % 4) * 16;
    } else {
        const uint64_t h = (j * 0x9E3779B97F4A7C15ull + b * 0xBF58476D1CE4E5B9ull) >> 20;
        tile = (int)(h % tiles);
        x0 = (int)((h >> 32) % (32 / box_rows)) * box_rows;
        c0 = (int)((h >> 40) % 4) * 16;
    }
}

__global__ void __launch_bounds__(128, 1) gather_probe(const __grid_constant__ CUtensorMap tm, uint64_t n_items,
                                                        uint32_t tiles, int boxes_per_item, int box_rows,
                                                        uint32_t box_bytes, int structured) {
    extern __shared__ __align__(1024) unsigned char ring[];
    __shared__ __align__(8) uint64_t full[STAGES];
    const uint32_t stage_bytes = boxes_per_item * box_bytes;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (warp >= STAGES)
        return;
    // producer for stage `warp`: items j = blockIdx + (warp + k * STAGES) * gridDim
    const int s = warp;
    const uint32_t sb = smem_u32(ring) + s * stage_bytes;
    uint32_t parity = 0;
    bool have = false;
    uint64_t prev = 0;
    for (uint64_t j = blockIdx.x + (uint64_t)s * gridDim.x; j < n_items + (uint64_t)STAGES * gridDim.x;
         j += (uint64_t)STAGES * gridDim.x) {
        if (have) {  // store item prev back (same boxes), wait until the stage has been read out
            for (int b = lane; b < boxes_per_item; b += 32) {
                int tile, x0, c0;
                box_of(prev, b, tiles, box_rows, structured, tile, x0, c0);
                asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&tm),
                             "r"(c0), "r"(tile * 32 + x0), "r"(sb + b * box_bytes)
                             : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        if (j >= n_items)
            break;
        __syncwarp();
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                         "r"(stage_bytes));
        __syncwarp();
        for (int b = lane; b < boxes_per_item; b += 32) {
            int tile, x0, c0;
            box_of(j, b, tiles, box_rows, structured, tile, x0, c0);
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                    sb + b * box_bytes),
                "l"(&tm), "r"(c0), "r"(tile * 32 + x0), "r"(smem_u32(&full[s]))
                : "memory");
        }
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "W:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n}" ::"r"(smem_u32(&full[s])),
            "r"(parity));
        parity ^= 1;
        have = true;
        prev = j;
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const uint64_t tiles = 1u << 19;  // 512 Ki tiles x 16 KiB = 8 GiB
    double* d;
    if (cudaMalloc(&d, tiles * 16384) != cudaSuccess) {
        printf("alloc failed\n");
        return 1;
    }
    cudaMemset(d, 0, tiles * 16384);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int structured = 0; structured < 2; ++structured)
    for (int box_rows : {8, 16, 32}) {
        for (int swz = 1; swz < 2; ++swz) {
            CUtensorMap tm;
            cuuint64_t dims[2] = {64, tiles * 32};  // 64 doubles per tile row, all tile rows stacked
            cuuint64_t strides[1] = {64 * 8};
            cuuint32_t box[2] = {16, (cuuint32_t)box_rows}, estr[2] = {1, 1};
            CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box, estr,
                                                CU_TENSOR_MAP_INTERLEAVE_NONE,
                                                swz ? CU_TENSOR_MAP_SWIZZLE_128B : CU_TENSOR_MAP_SWIZZLE_NONE,
                                                CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            if (r != CUDA_SUCCESS) {
                printf("encode failed %d\n", (int)r);
                return 1;
            }
            const uint32_t box_bytes = 128 * box_rows;
            const int boxes = 65536 / box_bytes;  // 64 KiB items
            const uint32_t smem = STAGES * 65536;
            cudaFuncSetAttribute(gather_probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            const uint64_t items = (tiles * 16384ull) / 65536 * 2;  // two passes' worth of bytes
            gather_probe<<<sms, 128, smem>>>(tm, items / 4, tiles, boxes, box_rows, box_bytes, structured);
            cudaEventRecord(e0);
            gather_probe<<<sms, 128, smem>>>(tm, items, tiles, boxes, box_rows, box_bytes, structured);
            cudaEventRecord(e1);
            cudaError_t e = cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("%s: box %2d rows x 128 B (%5u B), %3d boxes/item, swizzle %s: %s  %.1f GB/s\n",
                   structured ? "unit sub-blocks" : "random tiles   ", box_rows, box_bytes, boxes, swz ? "128B" : "none",
                   cudaGetErrorString(e), 2.0 * items * 65536 / ms / 1e6);
        }
    }
    return 0;
}
