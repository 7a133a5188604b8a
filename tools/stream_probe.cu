// stream_probe.cu -- micro-benchmark of in-place HBM streaming strategies on B200 (design probe
// for the conjugation kernels).  Each variant reads and rewrites
// every complex128 of a buffer once (x <- 0.5 x), like a transform that touches the whole state.
//   v1: plain LDG.128 / STG.128, grid-stride, UNR elements per thread in flight
//   v2: TMA bulk ring (1 CTA/SM, producer warp + consumer warps), chunk bytes / stages variable
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cudart shared -o stream_probe stream_probe.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>

#define CK(x)                                                                  \
    do {                                                                       \
        cudaError_t e = (x);                                                   \
        if (e != cudaSuccess) {                                                \
            printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e)); \
            exit(1);                                                           \
        }                                                                      \
    } while (0)

template <int UNR>
__global__ void __launch_bounds__(256) v1(double2* __restrict__ a, uint64_t n) {
    const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * UNR;
    for (uint64_t base = (uint64_t)blockIdx.x * blockDim.x * UNR + threadIdx.x; base < n; base += stride) {
        double2 v[UNR];
#pragma unroll
        for (int j = 0; j < UNR; ++j) {
            const uint64_t i = base + (uint64_t)j * blockDim.x;
            if (i < n)
                v[j] = a[i];
        }
#pragma unroll
        for (int j = 0; j < UNR; ++j) {
            const uint64_t i = base + (uint64_t)j * blockDim.x;
            if (i < n)
                a[i] = make_double2(0.5 * v[j].x, 0.5 * v[j].y);
        }
    }
}

__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}

// mode 0: producer waits for the store of item j-S to be read before loading item j (eager)
// mode 1: stores issued as soon as an item is done; loads refill lazily (wait_group.read S-1..)
template <int NCONS>
__global__ void __launch_bounds__(NCONS + 32, 1) v2(double2* __restrict__ a, uint64_t n, uint32_t chunk_elems,
                                                     uint32_t S, uint32_t pieces) {
    extern __shared__ __align__(128) double2 ring[];
    __shared__ __align__(8) uint64_t full[8], done[8];
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (uint32_t s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&done[s])), "r"(NCONS / 32));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint64_t nItems = n / chunk_elems;
    const uint64_t nlocal = blockIdx.x < nItems ? (nItems - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    const uint32_t bytes = chunk_elems * 16, pbytes = bytes / pieces;
    if (warp == NCONS / 32) {
        for (uint64_t j = 0; j < nlocal + S; ++j) {
            const uint32_t s = j % S;
            double2* sb = ring + (size_t)s * chunk_elems;
            if (j >= S) {
                const uint64_t jj = j - S;
                mwait(&done[s], (jj / S) & 1);
                double2* g = a + (blockIdx.x + jj * gridDim.x) * (uint64_t)chunk_elems;
                for (uint32_t p = lane; p < pieces; p += 32)
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"((char*)g + p * pbytes),
                                 "r"(su32(sb) + p * pbytes), "r"(pbytes) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            if (j < nlocal) {
                if (j >= S)
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                if (lane == 0)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(bytes) : "memory");
                __syncwarp();
                const double2* g = a + (blockIdx.x + j * gridDim.x) * (uint64_t)chunk_elems;
                for (uint32_t p = lane; p < pieces; p += 32)
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(sb) + p * pbytes),
                                 "l"((const char*)g + p * pbytes), "r"(pbytes), "r"(su32(&full[s])) : "memory");
            }
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        return;
    }
    for (uint64_t i = 0; i < nlocal; ++i) {
        const uint32_t s = i % S;
        double2* sb = ring + (size_t)s * chunk_elems;
        mwait(&full[s], (i / S) & 1);
        for (uint32_t e = tid; e < chunk_elems; e += NCONS) {
            double2 v = sb[e];
            sb[e] = make_double2(0.5 * v.x, 0.5 * v.y);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&done[s])) : "memory");
    }
}

// v3: 64 KiB items = 4 x 16 KiB chunks taken from `streams` separate address regions
template <int NCONS>
__global__ void __launch_bounds__(NCONS + 32, 1) v3(double2* __restrict__ a, uint64_t n, uint32_t S, uint32_t streams) {
    extern __shared__ __align__(128) double2 ring[];
    __shared__ __align__(8) uint64_t full[8], done[8];
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    const uint32_t chunk = 1024, per = 4 * chunk;  // elements
    if (tid == 0) {
        for (uint32_t s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&done[s])), "r"(NCONS / 32));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint64_t nItems = n / per;
    const uint64_t region = n / streams;            // elements per region
    const uint32_t cps = 4 / streams;               // chunks per stream per item
    auto addr = [&](uint64_t item, uint32_t c) -> double2* {
        const uint32_t r = c / cps, k = c % cps;
        return a + r * region + item * (uint64_t)cps * chunk + (uint64_t)k * chunk;
    };
    const uint64_t nlocal = blockIdx.x < nItems ? (nItems - blockIdx.x + gridDim.x - 1) / gridDim.x : 0;
    if (warp == NCONS / 32) {
        for (uint64_t j = 0; j < nlocal + S; ++j) {
            const uint32_t s = j % S;
            double2* sb = ring + (size_t)s * per;
            if (j >= S) {
                const uint64_t jj = j - S;
                mwait(&done[s], (jj / S) & 1);
                if (lane < 4)
                    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(addr(blockIdx.x + jj * gridDim.x, lane)),
                                 "r"(su32(sb) + lane * chunk * 16), "r"(chunk * 16) : "memory");
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            if (j < nlocal) {
                if (j >= S)
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                if (lane == 0)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(per * 16) : "memory");
                __syncwarp();
                if (lane < 4)
                    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(sb) + lane * chunk * 16),
                                 "l"(addr(blockIdx.x + j * gridDim.x, lane)), "r"(chunk * 16), "r"(su32(&full[s])) : "memory");
            }
        }
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        return;
    }
    for (uint64_t i = 0; i < nlocal; ++i) {
        const uint32_t s = i % S;
        double2* sb = ring + (size_t)s * per;
        mwait(&full[s], (i / S) & 1);
        for (uint32_t e = tid; e < per; e += NCONS) {
            double2 v = sb[e];
            sb[e] = make_double2(0.5 * v.x, 0.5 * v.y);
        }
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0)
            asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(&done[s])) : "memory");
    }
}

int main(int argc, char** argv) {
    const uint64_t bytes = (argc > 1 ? atoll(argv[1]) : 34376515584ull);
    const uint64_t n = bytes / 16;
    double2* a;
    CK(cudaMalloc(&a, n * 16));
    CK(cudaMemset(a, 0, n * 16));
    int sms;
    CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto report = [&](const char* name, auto&& launch) {
        launch();
        CK(cudaDeviceSynchronize());
        float best = 1e30f;
        for (int r = 0; r < 3; ++r) {
            cudaEventRecord(e0);
            launch();
            cudaEventRecord(e1);
            CK(cudaEventSynchronize(e1));
            float ms;
            cudaEventElapsedTime(&ms, e0, e1);
            if (ms < best)
                best = ms;
        }
        printf("%-48s %8.3f ms  %7.1f GB/s (r+w)\n", name, best, 2.0 * bytes / (best * 1e-3) / 1e9);
        fflush(stdout);
    };
    for (int mult : {4, 8, 16, 32}) {
        char nm[64];
        snprintf(nm, 64, "v1 LDG/STG unr=4 grid=%dxSM", mult);
        report(nm, [&] { v1<4><<<sms * mult, 256>>>(a, n); });
        snprintf(nm, 64, "v1 LDG/STG unr=8 grid=%dxSM", mult);
        report(nm, [&] { v1<8><<<sms * mult, 256>>>(a, n); });
    }
    struct Cfg {
        uint32_t chunk_kb, S, pieces;
    } cfgs[] = {{16, 4, 1}, {32, 4, 1}, {32, 6, 1}, {16, 8, 1}, {32, 4, 2}, {32, 4, 8}, {32, 4, 32}, {32, 4, 64},
                {48, 4, 1}, {64, 3, 1}, {8, 8, 1}};
    for (auto c : cfgs) {
        const uint32_t chunk = c.chunk_kb * 1024 / 16;
        const size_t smem = (size_t)c.S * chunk * 16;
        if (smem > 227 * 1024)
            continue;
        char nm[80];
        snprintf(nm, 80, "v2 TMA ring chunk=%uKB S=%u pieces=%u", c.chunk_kb, c.S, c.pieces);
        CK(cudaFuncSetAttribute(v2<256>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        report(nm, [&] { v2<256><<<sms, 288, smem>>>(a, n, chunk, c.S, c.pieces); });
    }
    for (uint32_t streams : {1u, 2u, 4u}) {
        const size_t smem = 3 * 4096 * 16;
        char nm[80];
        snprintf(nm, 80, "v3 64KB items of 4x16KB from %u stream(s), S=3", streams);
        CK(cudaFuncSetAttribute(v3<512>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        report(nm, [&] { v3<512><<<sms, 544, smem>>>(a, n, 3, streams); });
    }
    // two CTAs per SM
    for (auto c : {Cfg{16, 4, 1}, Cfg{32, 3, 1}, Cfg{24, 4, 1}}) {
        const uint32_t chunk = c.chunk_kb * 1024 / 16;
        const size_t smem = (size_t)c.S * chunk * 16;
        char nm[80];
        snprintf(nm, 80, "v2 TMA ring 2CTA/SM chunk=%uKB S=%u", c.chunk_kb, c.S);
        CK(cudaFuncSetAttribute(v2<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        report(nm, [&] { v2<128><<<sms * 2, 160, smem>>>(a, n, chunk, c.S, c.pieces); });
    }
    return 0;
}
