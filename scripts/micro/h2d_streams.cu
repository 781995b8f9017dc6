// H2D bandwidth of page-locked 8 GiB in 256-row slabs (2D copies) issued on 1, 2 or 4
// streams (copy engines) at once: does a second engine add PCIe bandwidth?
#include <cstdio>
#include <cuda_runtime.h>
int main() {
    const size_t m = 2048, n = 1 << 18, esz = 16;  // 8 GiB
    void *h, *d;
    cudaHostAlloc(&h, m * n * esz, cudaHostAllocDefault);
    cudaMalloc(&d, m * n * esz);
    cudaStream_t s[4];
    for (auto& x : s) cudaStreamCreateWithFlags(&x, cudaStreamNonBlocking);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int rep = 0; rep < 2; ++rep)
    for (int ns : {1, 2, 4}) {
        cudaDeviceSynchronize();
        cudaEventRecord(e0, 0);
        for (int k = 0; k < ns; ++k) cudaStreamWaitEvent(s[k], e0, 0);
        const size_t rows = 256;
        int k = 0;
        for (size_t r0 = 0; r0 < m; r0 += rows, k = (k + 1) % ns)
            cudaMemcpy2DAsync((char*)d + r0 * esz, m * esz, (char*)h + r0 * esz, m * esz, rows * esz, n,
                              cudaMemcpyHostToDevice, s[k]);
        for (int j = 0; j < ns; ++j) { cudaEvent_t e; cudaEventCreate(&e); cudaEventRecord(e, s[j]); cudaStreamWaitEvent(0, e, 0); }
        cudaEventRecord(e1, 0);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"streams\": %d, \"GBps\": %.1f}\n", ns, m * n * esz / (ms * 1e6));
    }
    // one contiguous 1D copy for reference
    cudaEventRecord(e0, 0);
    cudaMemcpyAsync(d, h, m * n * esz, cudaMemcpyHostToDevice, 0);
    cudaEventRecord(e1, 0);
    cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    printf("{\"contiguous_1d\": true, \"GBps\": %.1f}\n", m * n * esz / (ms * 1e6));
    return 0;
}
