// Dev probe: kernel-driven PCIe bandwidth over mapped pinned host memory
// (coalesced 16-byte / 4-byte / 1-byte accesses), read and write, alone and both.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

template <typename T>
__global__ void k_copy(const T *__restrict__ src, T *__restrict__ dst, size_t n)
{
    for (size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x; i < n; i += (size_t)gridDim.x * blockDim.x)
        dst[i] = src[i];
}

int main()
{
    const size_t n = 3 << 20;
    uint8_t *h1, *h2, *d1, *d2;
    cudaHostAlloc(&h1, n, cudaHostAllocMapped); cudaHostAlloc(&h2, n, cudaHostAllocMapped);
    cudaMalloc(&d1, n); cudaMalloc(&d2, n);
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    auto run = [&](const char *name, auto f) {
        for (int i = 0; i < 5; i++) f();
        cudaEventRecord(a);
        for (int i = 0; i < 50; i++) f();
        cudaEventRecord(b); cudaEventSynchronize(b);
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("%-36s %7.1f us  %6.1f GB/s\n", name, ms * 1000 / 50, n / (ms / 50 * 1e-3) / 1e9);
    };
    for (int blocks : {148, 592, 2368}) {
        printf("blocks %d\n", blocks);
        run("read host 16B -> dev", [&] { k_copy<<<blocks, 256>>>((const uint4 *)h1, (uint4 *)d1, n / 16); });
        run("write dev -> host 16B", [&] { k_copy<<<blocks, 256>>>((const uint4 *)d1, (uint4 *)h2, n / 16); });
        run("read host 4B -> dev", [&] { k_copy<<<blocks, 256>>>((const uint32_t *)h1, (uint32_t *)d1, n / 4); });
        run("write dev -> host 4B", [&] { k_copy<<<blocks, 256>>>((const uint32_t *)d1, (uint32_t *)h2, n / 4); });
        run("read host 1B -> dev", [&] { k_copy<<<blocks, 256>>>(h1, d1, n); });
        run("host -> host 16B (both dirs)", [&] { k_copy<<<blocks, 256>>>((const uint4 *)h1, (uint4 *)h2, n / 16); });
    }
    run("cudaMemcpyAsync H2D", [&] { cudaMemcpyAsync(d1, h1, n, cudaMemcpyHostToDevice); });
    run("cudaMemcpyAsync D2H", [&] { cudaMemcpyAsync(h2, d1, n, cudaMemcpyDeviceToHost); });
    return 0;
}
