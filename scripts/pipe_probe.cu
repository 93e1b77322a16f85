// Dev probe: GPU-side timeline of the banded host pipeline (timing events).
// build: nvcc -O2 -std=c++17 -I include scripts/pipe_probe.cu -o scripts/pipe_probe -L paper_1009_0958_b200 -ldfg -Xlinker -rpath='$ORIGIN/../paper_1009_0958_b200'
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <vector>
#include <cuda_runtime.h>
#include "dirfilt_gpu.h"

int main(int argc, char **argv)
{
    const int H = argc > 1 ? atoi(argv[1]) : 1024, W = argc > 2 ? atoi(argv[2]) : 1024;
    const int nb = argc > 3 ? atoi(argv[3]) : 4;
    const size_t pitch = 3ull * W, n = pitch * H;
    uint8_t *hi, *ho, *di, *dout;
    cudaMallocHost(&hi, n); cudaMallocHost(&ho, n);
    cudaMalloc(&di, n); cudaMalloc(&dout, n);
    for (size_t i = 0; i < n; i++) hi[i] = (uint8_t)(i * 2654435761u >> 24);
    dfg_params p; memset(&p, 0, sizeof p);
    p.family = 3; p.strategy = 0; p.window = 3; p.border = 0; p.p = 2.0; p.lam = 2; p.threshold = 10.8;
    void *ws; cudaMalloc(&ws, 256); cudaMemset(ws, 0, 256);
    cudaStream_t sin, sout, sk[4];
    cudaStreamCreateWithFlags(&sin, cudaStreamNonBlocking); cudaStreamCreateWithFlags(&sout, cudaStreamNonBlocking);
    for (auto &s : sk) cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    std::vector<cudaEvent_t> e_h0(nb), e_h1(nb), e_k0(nb), e_k1(nb), e_d0(nb), e_d1(nb);
    auto mk = [](cudaEvent_t &e) { cudaEventCreate(&e); };
    for (int k = 0; k < nb; k++) { mk(e_h0[k]); mk(e_h1[k]); mk(e_k0[k]); mk(e_k1[k]); mk(e_d0[k]); mk(e_d1[k]); }
    cudaEvent_t t0; mk(t0);
    auto row0 = [&](int k) { return (int)((long long)k * H / nb); };
    for (int rep = 0; rep < 20; rep++) {
        cudaEventRecord(t0, sin);
        for (int s = 0; s < 4; s++) cudaStreamWaitEvent(sk[s], t0, 0);
        cudaStreamWaitEvent(sout, t0, 0);
        for (int k = 0; k < nb; k++) {
            const int r0 = row0(k), r1 = row0(k + 1);
            cudaEventRecord(e_h0[k], sin);
            cudaMemcpyAsync(di + r0 * pitch, hi + r0 * pitch, (r1 - r0) * pitch, cudaMemcpyHostToDevice, sin);
            cudaEventRecord(e_h1[k], sin);
        }
        for (int k = 0; k < nb; k++) {
            const int r0 = row0(k), r1 = row0(k + 1);
            const int need = k + 1 < nb ? k + 1 : k;
            cudaStream_t s = sk[k % 4];
            cudaStreamWaitEvent(s, e_h1[need], 0);
            cudaEventRecord(e_k0[k], s);
            dfg_filter_rows(di, H, W, 0, H, pitch, dout + r0 * pitch, r0, r1 - r0, pitch, &p, ws, 256, s);
            cudaEventRecord(e_k1[k], s);
            cudaStreamWaitEvent(sout, e_k1[k], 0);
            cudaEventRecord(e_d0[k], sout);
            cudaMemcpyAsync(ho + r0 * pitch, dout + r0 * pitch, (r1 - r0) * pitch, cudaMemcpyDeviceToHost, sout);
            cudaEventRecord(e_d1[k], sout);
        }
        cudaDeviceSynchronize();
    }
    auto ms = [&](cudaEvent_t e) { float v; cudaEventElapsedTime(&v, t0, e); return v * 1000.f; };
    printf("band   h2d[start,end]     kernel[start,end]   d2h[start,end]  (us from pipeline start)\n");
    for (int k = 0; k < nb; k++)
        printf("%4d  %7.1f %7.1f   %7.1f %7.1f   %7.1f %7.1f\n", k, ms(e_h0[k]), ms(e_h1[k]), ms(e_k0[k]), ms(e_k1[k]),
               ms(e_d0[k]), ms(e_d1[k]));
    return 0;
}
