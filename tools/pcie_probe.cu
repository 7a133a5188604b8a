// Probe (design evidence for the end-to-end measurement): host <-> device copy rates
// from pinned memory on this box -- one direction alone, both directions at once, and each
// direction split over several streams (copy engines).
// nvcc -O2 -cudart shared -o tools/pcie_probe tools/pcie_probe.cu
#include <cuda_runtime.h>
#include <cstdio>
#include <vector>

int main() {
    const size_t bytes = 8ull << 30;  // 8 GiB each way
    void *h1, *h2, *d1, *d2;
    if (cudaHostAlloc(&h1, bytes, 0) || cudaHostAlloc(&h2, bytes, 0) || cudaMalloc(&d1, bytes) || cudaMalloc(&d2, bytes)) {
        printf("alloc failed\n");
        return 1;
    }
    cudaMemset(d1, 1, bytes);
    cudaMemset(d2, 2, bytes);
    std::vector<cudaStream_t> s(8);
    for (auto& x : s)
        cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    auto run = [&](bool up, bool down, int chunks) {
        cudaDeviceSynchronize();
        cudaEventRecord(e0, s[0]);
        for (int i = 0; i < 8; ++i)
            if (i)
                cudaStreamWaitEvent(s[i], e0, 0);
        const size_t c = bytes / chunks;
        for (int k = 0; k < chunks; ++k) {
            if (up)
                cudaMemcpyAsync((char*)d1 + k * c, (char*)h1 + k * c, c, cudaMemcpyHostToDevice, s[k % 4]);
            if (down)
                cudaMemcpyAsync((char*)h2 + k * c, (char*)d2 + k * c, c, cudaMemcpyDeviceToHost, s[4 + k % 4]);
        }
        for (int i = 1; i < 8; ++i) {
            cudaEvent_t ev;
            cudaEventCreate(&ev);
            cudaEventRecord(ev, s[i]);
            cudaStreamWaitEvent(s[0], ev, 0);
            cudaEventDestroy(ev);
        }
        cudaEventRecord(e1, s[0]);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        const double gb = (up + down) * bytes / 1e9;
        printf("%-5s %-5s chunks %d: %.1f GB/s total\n", up ? "H2D" : "", down ? "D2H" : "", chunks, gb / ms * 1e3);
    };
    for (int chunks : {1, 4}) {
        run(true, false, chunks);
        run(false, true, chunks);
        run(true, true, chunks);
    }
    return 0;
}
