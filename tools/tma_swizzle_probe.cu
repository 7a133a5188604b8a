// Probe (design evidence for a TMA-staged gather): where does a SWIZZLE_128B TMA box
// land when its shared-memory base is 128-byte but not 1024-byte aligned?  Hypothesis A: the XOR uses
// absolute smem address bits (chunk' = chunk ^ ((addr >> 7) & 7)), so a base offset of phi * 128 B
// rotates the pattern; hypothesis B: the pattern is relative to the box (chunk' = chunk ^ row).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -cudart shared -o tools/tma_swizzle_probe tools/tma_swizzle_probe.cu -lcuda
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdint>
#include <vector>

__global__ void probe(const __grid_constant__ CUtensorMap tm, double* out, int tiles, int phase_mode) {
    extern __shared__ __align__(1024) unsigned char smem[];
    __shared__ __align__(8) uint64_t bar;
    const uint32_t sbase = (uint32_t)__cvta_generic_to_shared(smem);
    const uint32_t bar_a = (uint32_t)__cvta_generic_to_shared(&bar);
    const int bytes_per_tile = 2048;  // 1 KiB box + 1 KiB room for the phase offset
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(bar_a), "r"(1));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar_a), "r"(tiles * 1024));
        for (int t = 0; t < tiles; ++t) {
            const uint32_t phase = phase_mode ? (uint32_t)(t & 7) : 0u;
            const uint32_t dst = sbase + t * bytes_per_tile + phase * 128;
            int c0 = 0, c1 = t * 8;
            asm volatile(
                "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];" ::"r"(dst),
                "l"(&tm), "r"(c0), "r"(c1), "r"(bar_a)
                : "memory");
        }
    }
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "W:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n}" ::"r"(bar_a),
        "r"(0));
    const double* sd = reinterpret_cast<const double*>(smem);
    for (int i = threadIdx.x; i < tiles * bytes_per_tile / 8; i += blockDim.x)
        out[i] = sd[i];
}

int main() {
    const int tiles = 8, rows = 8 * tiles, cols = 16;  // 16 doubles = 128 B per row (8 complex)
    std::vector<double> h(rows * cols);
    for (int r = 0; r < rows; ++r)
        for (int c = 0; c < cols; ++c)
            h[r * cols + c] = r * 1000 + c;  // tile t = r / 8, row x = r % 8, 8-byte column c
    double *d, *out;
    cudaMalloc(&d, h.size() * 8);
    cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
    const int sbytes = tiles * 2048;
    cudaMalloc(&out, sbytes);
    CUtensorMap tm;
    cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
    cuuint64_t strides[1] = {(cuuint64_t)cols * 8};
    cuuint32_t box[2] = {16, 8}, estr[2] = {1, 1};
    CUresult r = cuTensorMapEncodeTiled(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, d, dims, strides, box, estr,
                                        CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                                        CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    printf("encode: %d\n", (int)r);
    cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, sbytes);
    for (int mode = 0; mode < 2; ++mode) {
        cudaMemset(out, 0xff, sbytes);
        probe<<<1, 128, sbytes>>>(tm, out, tiles, mode);
        cudaError_t e = cudaDeviceSynchronize();
        printf("mode %d (%s): %s\n", mode, mode ? "bases offset by (t & 7) * 128 B" : "1 KiB-aligned bases",
               cudaGetErrorString(e));
        if (e != cudaSuccess)
            return 1;
        std::vector<double> o(sbytes / 8);
        cudaMemcpy(o.data(), out, sbytes, cudaMemcpyDeviceToHost);
        int okA = 0, okB = 0, tot = 0;
        for (int t = 0; t < tiles; ++t) {
            const int phase = mode ? (t & 7) : 0;
            for (int x = 0; x < 8; ++x)
                for (int c = 0; c < 16; ++c) {
                    const double v = t * 8000 + x * 1000 + c;
                    const int chunk = c / 2, half = c % 2;
                    const uint32_t rowaddr = t * 2048 + phase * 128 + x * 128;
                    const int ca = chunk ^ ((rowaddr >> 7) & 7);  // absolute-address XOR
                    const int cb = chunk ^ x;                    // box-relative XOR
                    okA += o[(rowaddr + ca * 16) / 8 + half] == v;
                    okB += o[(rowaddr + cb * 16) / 8 + half] == v;
                    ++tot;
                }
        }
        printf("  absolute-address hypothesis %d/%d, box-relative hypothesis %d/%d\n", okA, tot, okB, tot);
    }
    return 0;
}
