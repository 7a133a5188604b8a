// oop_probe.cu -- design probe: does an out-of-place pass (read buffer A, write buffer B) stream faster
// than the in-place pass (read and rewrite A) the conjugation kernels make?  Plain LDG.128 / STG.128,
// grid-stride, 4 elements per thread in flight; 2 x 16 GiB buffers (larger than L2 by far).
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -cudart shared -o tools/oop_probe tools/oop_probe.cu
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
__global__ void __launch_bounds__(256) pass(const double2* __restrict__ a, double2* __restrict__ b, uint64_t n) {
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
                b[i] = make_double2(0.5 * v[j].x, 0.5 * v[j].y);
        }
    }
}
// in place needs non-restrict pointers
template <int UNR>
__global__ void __launch_bounds__(256) pass_inplace(double2* a, uint64_t n) {
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


// Bulk-copy ring as in pipe_kernel (in place: 64 KiB items as 4 x 16 KiB bulk copies, 3 stages, one producer
// warp, 512 consumers), with optional L2 eviction-priority hints on the loads (HINT bit 0) and the
// stores (bit 1): createpolicy evict_first -- the state is streamed once per pass, nothing is reused.
__device__ __forceinline__ uint32_t su32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mwait(uint64_t* b, uint32_t ph) {
    asm volatile("{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W_%=;\n}\n" ::"r"(su32(b)), "r"(ph) : "memory");
}
template <int NCONS, int HINT>
__global__ void __launch_bounds__(NCONS + 32, 1) ringk(double2* __restrict__ a, uint64_t n) {
    extern __shared__ __align__(128) double2 ring[];
    __shared__ __align__(8) uint64_t full[8], done[8];
    constexpr uint32_t S = 3, chunk_elems = 4096, pieces = 4, bytes = chunk_elems * 16, pbytes = bytes / pieces;
    const uint32_t tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
    if (tid == 0) {
        for (uint32_t s = 0; s < S; ++s) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&full[s])), "r"(1));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(&done[s])), "r"(NCONS / 32));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    uint64_t pol_ef, pol_x;
    asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_ef));
    asm volatile("createpolicy.fractional.L2::evict_unchanged.b64 %0, 1.0;" : "=l"(pol_x));
    const uint64_t nItems = n / chunk_elems;
    const uint64_t per = (nItems + gridDim.x - 1) / gridDim.x;
    const uint64_t nlocal = (HINT & 16) ? (blockIdx.x * per < nItems ? (nItems - blockIdx.x * per < per ? nItems - blockIdx.x * per : per) : 0)
                                        : (blockIdx.x < nItems ? (nItems - blockIdx.x + gridDim.x - 1) / gridDim.x : 0);
    auto item_of = [&](uint64_t j) { return (HINT & 16) ? blockIdx.x * per + j : blockIdx.x + j * gridDim.x; };
    if (warp == NCONS / 32) {
        for (uint64_t j = 0; j < nlocal + S; ++j) {
            const uint32_t s = j % S;
            double2* sb = ring + (size_t)s * chunk_elems;
            if (j >= S) {
                const uint64_t jj = j - S;
                mwait(&done[s], (jj / S) & 1);
                double2* g = a + item_of(jj) * (uint64_t)chunk_elems;
                for (uint32_t p = lane; p < pieces; p += 32) {
                    if (HINT & 2)
                        asm volatile("cp.async.bulk.global.shared::cta.bulk_group.L2::cache_hint [%0], [%1], %2, %3;" ::"l"((char*)g + p * pbytes),
                                     "r"(su32(sb) + p * pbytes), "r"(pbytes), "l"((HINT & 8) ? pol_x : pol_ef) : "memory");
                    else
                        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"((char*)g + p * pbytes),
                                     "r"(su32(sb) + p * pbytes), "r"(pbytes) : "memory");
                }
                asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            if (j < nlocal) {
                if (j >= S)
                    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
                if (lane == 0)
                    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])), "r"(bytes) : "memory");
                __syncwarp();
                const double2* g = a + item_of(j) * (uint64_t)chunk_elems;
                for (uint32_t p = lane; p < pieces; p += 32) {
                    if (HINT & 1)
                        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(su32(sb) + p * pbytes),
                                     "l"((const char*)g + p * pbytes), "r"(pbytes), "r"(su32(&full[s])), "l"((HINT & 4) ? pol_x : pol_ef) : "memory");
                    else
                        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(su32(sb) + p * pbytes),
                                     "l"((const char*)g + p * pbytes), "r"(pbytes), "r"(su32(&full[s])) : "memory");
                }
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
template <int HINT>
static void run_ring(double2* a, uint64_t n, int sms, cudaEvent_t e0, cudaEvent_t e1, const char* name) {
    const size_t smem = 3 * 65536;
    CK(cudaFuncSetAttribute(ringk<512, HINT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    float best = 1e30f;
    for (int it = 0; it < 5; ++it) {
        CK(cudaEventRecord(e0));
        ringk<512, HINT><<<sms, 544, smem>>>(a, n);
        CK(cudaEventRecord(e1));
        CK(cudaEventSynchronize(e1));
        float ms;
        CK(cudaEventElapsedTime(&ms, e0, e1));
        if (it && ms < best)
            best = ms;
    }
    printf("bulk ring in place, %-34s %8.3f ms  %7.1f GB/s\n", name, best, 2.0 * n * sizeof(double2) / best / 1e6);
}

int main() {
    const uint64_t n = 1ull << 30;  // 16 GiB per buffer
    double2 *a, *b;
    CK(cudaMalloc(&a, n * sizeof(double2)));
    CK(cudaMalloc(&b, n * sizeof(double2)));
    CK(cudaMemset(a, 0, n * sizeof(double2)));
    CK(cudaMemset(b, 0, n * sizeof(double2)));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    for (int ctas = 4; ctas <= 8; ctas += 4)
        for (int rep = 0; rep < 2; ++rep)
            for (int mode = 0; mode < 3; ++mode) {
                float best = 1e30f;
                for (int it = 0; it < 6; ++it) {
                    CK(cudaEventRecord(e0));
                    if (mode == 0)
                        pass_inplace<4><<<sms * ctas, 256>>>(a, n);
                    else if (mode == 1)
                        pass<4><<<sms * ctas, 256>>>(a, b, n);
                    else
                        CK(cudaMemcpyAsync(b, a, n * sizeof(double2), cudaMemcpyDeviceToDevice));
                    CK(cudaEventRecord(e1));
                    CK(cudaEventSynchronize(e1));
                    float ms;
                    CK(cudaEventElapsedTime(&ms, e0, e1));
                    if (it && ms < best)
                        best = ms;
                }
                printf("ctas/SM %d  %-14s %8.3f ms  %7.1f GB/s\n", ctas,
                       mode == 0 ? "in place" : mode == 1 ? "out of place" : "cudaMemcpy D2D", best,
                       2.0 * n * sizeof(double2) / best / 1e6);
            }
    for (int rep = 0; rep < 2; ++rep) {
        run_ring<0>(a, n, sms, e0, e1, "no hints");
        run_ring<1>(a, n, sms, e0, e1, "loads evict_first");
        run_ring<2>(a, n, sms, e0, e1, "stores evict_first");
        run_ring<3>(a, n, sms, e0, e1, "loads + stores evict_first");
        run_ring<7>(a, n, sms, e0, e1, "loads evict_unchanged, stores evict_first");
        run_ring<16>(a, n, sms, e0, e1, "no hints, contiguous slab per CTA");
    }
    CK(cudaGetLastError());
    return 0;
}
