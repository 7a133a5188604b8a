// Probe (design evidence): in-place HBM streaming of k = 3 / two-grid-target gather
// items -- 16 scattered 16 KiB tiles x one 16 x 16 sub-block each (64 KiB) -- staged with
//   (A) 2-D boxes of 8 rows x 128 B (1 KiB, SWIZZLE_128B): 64 boxes per item (the engine today);
//   (B) 3-D boxes {128 B, 2 chunks, 8 rows} = 8 rows x 256 B contiguous (2 KiB, SWIZZLE_128B per
//       128-B chunk): 32 boxes per item;
//   (C) 3-D boxes of 16 rows x 256 B (4 KiB): 16 boxes per item;
//   (D) any of them behind a whole-tile L2 prefetch (cp.async.bulk.prefetch.L2, 16 KiB per tile) issued a few
//       grid strides ahead by the CTA that holds a unit's sub-block 0.
// Three-stage ring, one producer warp per stage, store back + reload (no transform).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -cudart shared -o tools/tma3d_probe tools/tma3d_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

constexpr int STAGES = 3;

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// box b of item j: tile, first row, first 256-B half (sub-block column 0 or 1 of the tile row)
__device__ __forceinline__ void box_of(uint64_t j, int b, uint32_t tiles, int rows, int wide, int& tile, int& x0,
                                       int& h) {
    const uint64_t unit = j / 4;  // 4 sub-blocks of 16 x 16 per 32 x 32 tile; 16 tiles per unit
    const int sub = (int)(j % 4);
    const int per_tile = wide ? 16 / rows : 2 * (16 / rows);  // boxes per tile and item
    const int t = b / per_tile, r = b % per_tile;
    tile = (int)((unit * 16 + (uint64_t)t * 977) % tiles);
    if (wide) {
        x0 = (sub / 2) * 16 + r * rows;
        h = sub % 2;  // 256-B half of the 512-B tile row
    } else {
        x0 = (sub / 2) * 16 + (r / 2) * rows;
        h = (sub % 2) * 2 + (r % 2);  // 128-B quarter
    }
}

__global__ void __launch_bounds__(128, 1) probe(const __grid_constant__ CUtensorMap tm, uint64_t n_items, uint32_t tiles,
                                                int boxes, int rows, uint32_t box_bytes, int wide, int pf,
                                                const unsigned char* base) {
    extern __shared__ __align__(1024) unsigned char ring[];
    __shared__ __align__(8) uint64_t full[STAGES];
    const uint32_t stage_bytes = boxes * box_bytes;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int s = 0; s < STAGES; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (warp >= STAGES)
        return;
    const int s = warp;
    const uint32_t sb = smem_u32(ring) + s * stage_bytes;
    uint32_t parity = 0;
    bool have = false;
    uint64_t prev = 0;
    for (uint64_t j = blockIdx.x + (uint64_t)s * gridDim.x; j < n_items + (uint64_t)STAGES * gridDim.x;
         j += (uint64_t)STAGES * gridDim.x) {
        if (have) {
            for (int b = lane; b < boxes; b += 32) {
                int tile, x0, h;
                box_of(prev, b, tiles, rows, wide, tile, x0, h);
                if (wide)
                    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(&tm),
                                 "r"(0), "r"(2 * h), "r"(tile * 32 + x0), "r"(sb + b * box_bytes)
                                 : "memory");
                else
                    asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];" ::"l"(&tm),
                                 "r"(16 * h), "r"(tile * 32 + x0), "r"(sb + b * box_bytes)
                                 : "memory");
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        }
        if (j >= n_items)
            break;
        __syncwarp();
        // (D) whole-tile L2 prefetch: the CTA that holds sub-block 0 of a unit asks L2 for the unit's 16
        // whole tiles pf grid strides ahead, so DRAM sees 16 KiB contiguous reads and the boxes hit L2
        if (pf && (j & 3) == 0 && lane < 16) {
            const uint64_t jp = j + (uint64_t)pf * gridDim.x;
            if (jp < n_items) {
                const uint64_t tile = ((jp / 4) * 16 + (uint64_t)lane * 977) % tiles;
                asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(base + tile * 16384), "r"(16384) : "memory");
            }
        }
        if (lane == 0)
            asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&full[s])),
                         "r"(stage_bytes));
        __syncwarp();
        for (int b = lane; b < boxes; b += 32) {
            int tile, x0, h;
            box_of(j, b, tiles, rows, wide, tile, x0, h);
            if (wide)
                asm volatile(
                    "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], [%5];" ::"r"(
                        sb + b * box_bytes),
                    "l"(&tm), "r"(0), "r"(2 * h), "r"(tile * 32 + x0), "r"(smem_u32(&full[s]))
                    : "memory");
            else
                asm volatile(
                    "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(
                        sb + b * box_bytes),
                    "l"(&tm), "r"(16 * h), "r"(tile * 32 + x0), "r"(smem_u32(&full[s]))
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
    const uint64_t tiles = 1u << 19;  // 8 GiB
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
    struct Cfg {
        int wide, rows, pf;
    } cfgs[] = {{0, 8, 0}, {0, 16, 0}, {1, 8, 0}, {1, 16, 0}, {0, 8, 1}, {0, 8, 2}, {0, 8, 4}, {0, 8, 8}, {1, 16, 2}, {1, 16, 4}};
    for (int rep = 0; rep < 2; ++rep)
        for (const Cfg& c : cfgs) {
            CUtensorMap tm;
            CUresult r;
            if (c.wide) {
                cuuint64_t dims[3] = {16, 4, tiles * 32};  // 16 doubles = 128 B, 4 chunks per row, rows
                cuuint64_t strides[2] = {128, 512};
                cuuint32_t box[3] = {16, 2, (cuuint32_t)c.rows}, estr[3] = {1, 1, 1};
                r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 3, d, dims, strides, box, estr,
                                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            } else {
                cuuint64_t dims[2] = {64, tiles * 32};
                cuuint64_t strides[1] = {512};
                cuuint32_t box[2] = {16, (cuuint32_t)c.rows}, estr[2] = {1, 1};
                r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box, estr,
                                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                           CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
            }
            if (r != CUDA_SUCCESS) {
                printf("encode failed %d\n", (int)r);
                return 1;
            }
            const uint32_t box_bytes = (c.wide ? 256 : 128) * c.rows;
            const int boxes = 65536 / box_bytes;
            const uint32_t smem = STAGES * 65536;
            cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
            const uint64_t items = (tiles * 16384ull) / 65536 * 2;
            probe<<<sms, 128, smem>>>(tm, items / 4, tiles, boxes, c.rows, box_bytes, c.wide, c.pf, (const unsigned char*)d);
            cudaEventRecord(e0);
            probe<<<sms, 128, smem>>>(tm, items, tiles, boxes, c.rows, box_bytes, c.wide, c.pf, (const unsigned char*)d);
            cudaEventRecord(e1);
            cudaError_t e = cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("%s box %2d rows x %3d B (%5u B), %2d boxes/item, L2 tile prefetch %d ahead: %s  %.1f GB/s\n",
                   c.wide ? "3-D" : "2-D", c.rows, c.wide ? 256 : 128, box_bytes, boxes, c.pf, cudaGetErrorString(e),
                   2.0 * items * 65536 / ms / 1e6);
        }
    return 0;
}
