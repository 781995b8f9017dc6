// H2D bandwidth of cudaMemcpy2DAsync from page-locked memory vs row width (the
// row-slab upload of a column-major A: width = slab rows * 16 B, height = n).
#include <cstdio>
#include <cuda_runtime.h>
int main() {
    const size_t m = 2048, n = 1 << 18, esz = 16;  // 8 GiB
    void *h, *d;
    cudaHostAlloc(&h, m * n * esz, cudaHostAllocDefault);
    cudaMalloc(&d, m * n * esz);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (size_t rows : {2048, 1024, 512, 256, 128}) {
        cudaEventRecord(e0);
        for (size_t r0 = 0; r0 < m; r0 += rows)
            cudaMemcpy2DAsync((char*)d + r0 * esz, m * esz, (char*)h + r0 * esz, m * esz, rows * esz, n,
                              cudaMemcpyHostToDevice, 0);
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        printf("{\"slab_rows\": %zu, \"width_bytes\": %zu, \"GBps\": %.1f}\n", rows, rows * esz, m * n * esz / (ms * 1e6));
    }
    return 0;
}
