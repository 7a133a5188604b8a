// FP64 throughput probe on B200 (design evidence for the k = 3 direct transform):
// DFMA (vector pipe) vs DMMA (mma.sync m8n8k4 f64 tensor path) vs both interleaved.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cudart shared -o tools/fp64_probe tools/fp64_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

constexpr int ITERS = 4096;

__global__ void dfma_kernel(double* out, double s) {
    double a[16];
#pragma unroll
    for (int i = 0; i < 16; ++i)
        a[i] = threadIdx.x * 1e-3 + i;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 16; ++i)
            a[i] = fma(a[i], s, 0.5);
    }
    double r = 0;
#pragma unroll
    for (int i = 0; i < 16; ++i)
        r += a[i];
    if (r == 12345.0)
        out[0] = r;
}

__device__ __forceinline__ void dmma(double (&d)[2], double a, double b) {
    asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                 : "+d"(d[0]), "+d"(d[1])
                 : "d"(a), "d"(b));
}

__global__ void dmma_kernel(double* out, double s) {
    double acc[8][2];
#pragma unroll
    for (int i = 0; i < 8; ++i)
        acc[i][0] = acc[i][1] = threadIdx.x * 1e-3 + i;
    const double a = s, b = 1.0 - s;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 8; ++i)
            dmma(acc[i], a, b);
    }
    double r = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
        r += acc[i][0] + acc[i][1];
    if (r == 12345.0)
        out[0] = r;
}

template <int CH>
__global__ void dmma_chains_kernel(double* out, double s) {
    double acc[CH][2];
#pragma unroll
    for (int i = 0; i < CH; ++i)
        acc[i][0] = acc[i][1] = threadIdx.x * 1e-3 + i;
    const double a = s, b = 1.0 - s;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i)
            dmma(acc[i], a, b);
    }
    double r = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i)
        r += acc[i][0] + acc[i][1];
    if (r == 12345.0)
        out[0] = r;
}

// distinct A/B operands per chain (as in the 3M transform: every DMMA reads its own registers)
template <int CH>
__global__ void dmma_distinct_kernel(double* out, double s) {
    double acc[CH][2], a[CH], b[CH];
#pragma unroll
    for (int i = 0; i < CH; ++i) {
        acc[i][0] = acc[i][1] = threadIdx.x * 1e-3 + i;
        a[i] = s + i * 1e-3;
        b[i] = 1.0 - s - i * 1e-3;
    }
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < CH; ++i) {
            dmma(acc[i], a[i], b[(i + it) % CH]);
            a[i] = acc[i][1];
        }
    }
    double r = 0;
#pragma unroll
    for (int i = 0; i < CH; ++i)
        r += acc[i][0] + acc[i][1];
    if (r == 12345.0)
        out[0] = r;
}

__global__ void mixed_kernel(double* out, double s) {
    double acc[4][2];
    double v[8];
#pragma unroll
    for (int i = 0; i < 4; ++i)
        acc[i][0] = acc[i][1] = threadIdx.x * 1e-3 + i;
#pragma unroll
    for (int i = 0; i < 8; ++i)
        v[i] = threadIdx.x * 1e-3 + i;
    const double a = s, b = 1.0 - s;
    for (int it = 0; it < ITERS; ++it) {
#pragma unroll
        for (int i = 0; i < 4; ++i)
            dmma(acc[i], a, b);
#pragma unroll
        for (int i = 0; i < 8; ++i)
            v[i] = fma(v[i], s, 0.5);
    }
    double r = 0;
#pragma unroll
    for (int i = 0; i < 4; ++i)
        r += acc[i][0] + acc[i][1];
#pragma unroll
    for (int i = 0; i < 8; ++i)
        r += v[i];
    if (r == 12345.0)
        out[0] = r;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    double* out;
    cudaMalloc(&out, 8);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    for (int threads : {256, 512, 1024}) {
        const int blocks = sms * (2048 / threads);
        float ms;
        // DFMA: 16 chains x ITERS per thread, 2 flop each
        dfma_kernel<<<blocks, threads>>>(out, 0.999);
        cudaEventRecord(e0);
        dfma_kernel<<<blocks, threads>>>(out, 0.999);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        cudaEventElapsedTime(&ms, e0, e1);
        const double fl_dfma = 2.0 * 16 * ITERS * (double)blocks * threads;
        // DMMA: m8n8k4 = 8*8*4 FMA per warp instruction, 8 per iteration
        dmma_kernel<<<blocks, threads>>>(out, 0.999);
        cudaEventRecord(e0);
        dmma_kernel<<<blocks, threads>>>(out, 0.999);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms2;
        cudaEventElapsedTime(&ms2, e0, e1);
        const double fl_dmma = 2.0 * 256 * 8 * ITERS * (double)blocks * threads / 32;
        mixed_kernel<<<blocks, threads>>>(out, 0.999);
        cudaEventRecord(e0);
        mixed_kernel<<<blocks, threads>>>(out, 0.999);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms3;
        cudaEventElapsedTime(&ms3, e0, e1);
        const double fl_mix = 2.0 * 256 * 4 * ITERS * (double)blocks * threads / 32 + 2.0 * 8 * ITERS * (double)blocks * threads;
        printf("threads=%d  DFMA %.2f TFLOP/s  DMMA %.2f TFLOP/s  mixed %.2f TFLOP/s (dmma part %.2f, dfma part %.2f)\n",
               threads, fl_dfma / ms / 1e9, fl_dmma / ms2 / 1e9, fl_mix / ms3 / 1e9,
               2.0 * 256 * 4 * ITERS * (double)blocks * threads / 32 / ms3 / 1e9,
               2.0 * 8 * ITERS * (double)blocks * threads / ms3 / 1e9);
    }
    // DMMA rate vs resident warps per SM and independent accumulator chains per warp
    for (int warps : {4, 8, 16, 32}) {
        auto run = [&](auto kern, int ch) {
            float ms;
            kern<<<sms, warps * 32>>>(out, 0.999);
            cudaEventRecord(e0);
            kern<<<sms, warps * 32>>>(out, 0.999);
            cudaEventRecord(e1);
            cudaEventSynchronize(e1);
            cudaEventElapsedTime(&ms, e0, e1);
            const double fl = 2.0 * 256 * ch * ITERS * (double)sms * warps;
            printf("  warps/SM=%d chains=%d: DMMA %.2f TFLOP/s\n", warps, ch, fl / ms / 1e9);
        };
        run(dmma_chains_kernel<1>, 1);
        run(dmma_chains_kernel<2>, 2);
        run(dmma_chains_kernel<4>, 4);
        run(dmma_chains_kernel<8>, 8);
        printf("  distinct operands:\n");
        run(dmma_distinct_kernel<2>, 2);
        run(dmma_distinct_kernel<6>, 6);
    }
    cudaError_t e = cudaGetLastError();
    printf("status: %s\n", cudaGetErrorString(e));
    return 0;
}
