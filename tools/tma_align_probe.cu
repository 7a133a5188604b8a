// Probe: does a non-swizzled 2-D TMA load / store accept a shared-memory address that is only 16-byte
// aligned (not 128)?  Box = 16 rows x 16 complex (256-B rows, 4 KiB); destinations at 16-B skews.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -cudart shared -o tools/tma_align_probe tools/tma_align_probe.cu
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>
using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                              const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const __grid_constant__ CUtensorMap tin, const __grid_constant__ CUtensorMap tout, int skew) {
    extern __shared__ __align__(1024) double sm[];
    __shared__ __align__(8) uint64_t bar;
    const uint32_t dst = su32(sm) + 16u * skew;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(su32(&bar)));
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(su32(&bar)), "r"(4096u));
        asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                     ::"r"(dst), "l"(&tin), "r"(32), "r"(16), "r"(su32(&bar)) : "memory");
        asm volatile("{.reg .pred p; W: mbarrier.try_wait.parity.shared.b64 p, [%0], 0; @!p bra W;}" ::"r"(su32(&bar)));
        asm volatile("fence.proxy.async.shared::cta;");
        asm volatile("cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%1, %2}], [%3];"
                     ::"l"(&tout), "r"(0), "r"(0), "r"(dst) : "memory");
        asm volatile("cp.async.bulk.commit_group; cp.async.bulk.wait_group 0;" ::: "memory");
    }
}
int main() {
    void* fp = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fp, cudaEnableDefault, &q);
    auto enc = (EncodeFn)fp;
    const int rows = 64, cols = 64;  // doubles per row (32 complex)
    std::vector<double> h(rows * cols);
    for (int i = 0; i < rows * cols; ++i) h[i] = i;
    double *din, *dout;
    cudaMalloc(&din, h.size() * 8);
    cudaMalloc(&dout, 16 * 32 * 8);
    cudaMemcpy(din, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    CUtensorMap tin, tout;
    cuuint64_t d1[2] = {(cuuint64_t)cols, (cuuint64_t)rows}, s1[1] = {cols * 8};
    cuuint64_t d2[2] = {32, 16}, s2[1] = {32 * 8};
    cuuint32_t box[2] = {32, 16}, es[2] = {1, 1};
    int r1 = enc(&tin, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, din, d1, s1, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    int r2 = enc(&tout, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, dout, d2, s2, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                 CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode %d %d\n", r1, r2);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 8192);
    for (int skew = 0; skew < 8; ++skew) {
        cudaMemset(dout, 0, 16 * 32 * 8);
        k<<<1, 32, 8192>>>(tin, tout, skew);
        cudaError_t e = cudaDeviceSynchronize();
        std::vector<double> o(16 * 32);
        cudaMemcpy(o.data(), dout, o.size() * 8, cudaMemcpyDeviceToHost);
        int bad = 0;
        for (int r = 0; r < 16; ++r)
            for (int c = 0; c < 32; ++c)
                bad += o[r * 32 + c] != h[(16 + r) * cols + 32 + c];
        printf("skew %d x 16 B: %s, mismatches %d\n", skew, cudaGetErrorString(e), bad);
        if (e != cudaSuccess) return 1;
    }
    return 0;
}
