// Probe (design evidence for the gather copy side): in-place streaming of 64 KiB
// gather items made of small 1-D bulk copies (cp.async.bulk, rows of `row_bytes` from scattered 16 KiB
// tiles, C3-like unit order) issued by many threads, vs 16-byte cp.async (LDGSTS) + st.global from
// the same threads.  Three stages, every copy thread works on every stage in turn.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -cudart shared -o tools/bulk_gather_probe tools/bulk_gather_probe.cu
#include <cuda_runtime.h>
#include <cstdint>
#include <cstdio>

constexpr int STAGES = 3;
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// piece p of item j: tile, element offset of the row start within the payload
__device__ __forceinline__ uint64_t piece(uint64_t j, int p, int row_elems, uint32_t tiles) {
    const int rows_per_tile = 4096 / 64 / row_elems * 0 + 8;  // 8 rows of each tile in an item
    const int t = p / rows_per_tile, r = p % rows_per_tile;
    const int nsub = 32 / 8 * (32 / row_elems);
    const uint64_t unit = j / nsub;
    const int sub = (int)(j % nsub);
    const uint64_t tile = (unit * 64 + (uint64_t)t * 977) % tiles;
    const int x0 = (sub / (32 / row_elems)) * 8, y0 = (sub % (32 / row_elems)) * row_elems;
    return tile * 1024 + (uint64_t)(x0 + r) * 32 + y0;
}

template <bool BULK>
__global__ void __launch_bounds__(512, 1) probe(double2* st, uint64_t n_items, uint32_t tiles, int row_elems) {
    extern __shared__ __align__(128) double2 ring[];
    __shared__ __align__(8) uint64_t full[STAGES];
    const int tid = threadIdx.x, NT = blockDim.x;
    const int pieces = 4096 / row_elems;  // 64 KiB item
    if (tid == 0)
        for (int s = 0; s < STAGES; ++s)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(NT));
    __syncthreads();
    const uint64_t nloc = blockIdx.x < n_items ? (n_items - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    auto item = [&](uint64_t i) { return blockIdx.x + i * gridDim.x; };
    auto load = [&](uint64_t i) {
        const int s = (int)(i % STAGES);
        double2* sb = ring + s * 4096;
        if (BULK) {
            if (tid == 0)
                asm volatile("mbarrier.expect_tx.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&full[s])), "r"(65536));
            __syncthreads();
            for (int p = tid; p < pieces; p += NT) {
                const double2* src = st + piece(item(i), p, row_elems, tiles);
                asm volatile(
                    "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                        smem_u32(sb + p * row_elems)),
                    "l"(src), "r"(row_elems * 16), "r"(smem_u32(&full[s]))
                    : "memory");
            }
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&full[s])) : "memory");
        } else {
            for (int e = tid; e < 4096; e += NT) {
                const int p = e / row_elems, c = e % row_elems;
                const double2* src = st + piece(item(i), p, row_elems, tiles) + c;
                asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(sb + e)), "l"(src) : "memory");
            }
            asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(smem_u32(&full[s])) : "memory");
        }
    };
    auto store = [&](uint64_t i) {
        const int s = (int)(i % STAGES);
        double2* sb = ring + s * 4096;
        if (BULK) {
            for (int p = tid; p < pieces; p += NT)
                asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                                 st + piece(item(i), p, row_elems, tiles)),
                             "r"(smem_u32(sb + p * row_elems)), "r"(row_elems * 16)
                             : "memory");
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        } else {
            for (int e = tid; e < 4096; e += NT) {
                const int p = e / row_elems, c = e % row_elems;
                st[piece(item(i), p, row_elems, tiles) + c] = sb[e];
            }
        }
        __syncthreads();
    };
    for (uint64_t i = 0; i < STAGES && i < nloc; ++i)
        load(i);
    for (uint64_t i = 0; i < nloc; ++i) {
        const int s = (int)(i % STAGES);
        asm volatile(
            "{\n\t.reg .pred p;\n"
            "W:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n}" ::"r"(smem_u32(&full[s])),
            "r"((uint32_t)((i / STAGES) & 1)));
        store(i);
        if (i + STAGES < nloc)
            load(i + STAGES);
    }
    asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

int main() {
    const uint64_t tiles = 1u << 19;  // 8 GiB
    double2* d;
    if (cudaMalloc(&d, tiles * 16384) != cudaSuccess)
        return 1;
    cudaMemset(d, 0, tiles * 16384);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const uint32_t smem = STAGES * 65536;
    cudaFuncSetAttribute(probe<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(probe<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    const uint64_t items = tiles * 16384ull / 65536 * 2;
    for (int row_elems : {8, 16, 32})
        for (int bulk = 0; bulk < 2; ++bulk) {
            auto k = bulk ? probe<true> : probe<false>;
            k<<<sms, 512, smem>>>(d, items / 4, tiles, row_elems);
            cudaEventRecord(e0);
            k<<<sms, 512, smem>>>(d, items, tiles, row_elems);
            cudaEventRecord(e1);
            cudaError_t e = cudaEventSynchronize(e1);
            float ms = 0;
            cudaEventElapsedTime(&ms, e0, e1);
            printf("rows of %3d B, %s: %s  %.1f GB/s\n", row_elems * 16,
                   bulk ? "cp.async.bulk per row (512 threads)" : "cp.async 16 B + st.global        ",
                   cudaGetErrorString(e), 2.0 * items * 65536 / ms / 1e6);
        }
    return 0;
}
