// Dev probe: host-path (dfg_filter_host) time breakdown from C, no Python.
// build: nvcc -O2 -std=c++17 -I include scripts/host_probe.cu -o scripts/host_probe -L paper_1009_0958_b200 -ldfg -Xlinker -rpath='$ORIGIN/../paper_1009_0958_b200'
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>
#include "dirfilt_gpu.h"

static double now_us() { return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now().time_since_epoch()).count(); }

int main(int argc, char **argv)
{
    const int H = argc > 1 ? atoi(argv[1]) : 1024, W = argc > 2 ? atoi(argv[2]) : 1024;
    const size_t n = 3ull * H * W;
    uint8_t *hi, *ho, *di, *dout;
    cudaMallocHost(&hi, n); cudaMallocHost(&ho, n);
    cudaMalloc(&di, n); cudaMalloc(&dout, n);
    srand(1);
    for (size_t i = 0; i < n; i++) hi[i] = (uint8_t)(rand() & 255);
    dfg_params p; memset(&p, 0, sizeof p);
    p.family = 3; p.strategy = 0; p.window = 3; p.border = 0; p.p = 2.0; p.lam = 2; p.threshold = 10.8;  // ddf exact 3x3
    void *ws; size_t wsb = dfg_workspace_bytes((int64_t)H * W); cudaMalloc(&ws, wsb); cudaMemset(ws, 0, wsb);
    cudaStream_t st; cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    auto bench = [&](const char *name, auto f, int reps = 200) {
        for (int i = 0; i < 10; i++) f();
        cudaStreamSynchronize(st);
        double t = now_us();
        for (int i = 0; i < reps; i++) f();
        cudaStreamSynchronize(st);
        printf("%-40s %8.1f us\n", name, (now_us() - t) / reps);
    };
    bench("H2D 3B*px (sync each)", [&] { cudaMemcpyAsync(di, hi, n, cudaMemcpyHostToDevice, st); cudaStreamSynchronize(st); });
    bench("D2H 3B*px (sync each)", [&] { cudaMemcpyAsync(ho, dout, n, cudaMemcpyDeviceToHost, st); cudaStreamSynchronize(st); });
    cudaStream_t s2; cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking);
    bench("H2D || D2H on two streams", [&] {
        cudaMemcpyAsync(di, hi, n, cudaMemcpyHostToDevice, st);
        cudaMemcpyAsync(ho, dout, n, cudaMemcpyDeviceToHost, s2);
        cudaStreamSynchronize(s2); cudaStreamSynchronize(st); });
    bench("H2D 4 chunks", [&] {
        for (int k = 0; k < 4; k++) cudaMemcpyAsync(di + k * (n / 4), hi + k * (n / 4), n / 4, cudaMemcpyHostToDevice, st);
        cudaStreamSynchronize(st); });
    bench("dfg_filter (sync each)", [&] { dfg_filter(di, H, W, 3LL * W, dout, 3LL * W, &p, ws, wsb, st); cudaStreamSynchronize(st); });
    bench("dfg_filter (no sync, x200)", [&] { dfg_filter(di, H, W, 3LL * W, dout, 3LL * W, &p, ws, wsb, st); });
    bench("H2D+filter+D2H serial", [&] {
        cudaMemcpyAsync(di, hi, n, cudaMemcpyHostToDevice, st);
        dfg_filter(di, H, W, 3LL * W, dout, 3LL * W, &p, ws, wsb, st);
        cudaMemcpyAsync(ho, dout, n, cudaMemcpyDeviceToHost, st);
        cudaStreamSynchronize(st); });
    bench("dfg_filter_host", [&] { dfg_filter_host(hi, H, W, ho, &p, st); });
    double t0 = now_us();
    for (int i = 0; i < 1000; i++) { cudaEvent_t e; (void)e; cudaStreamQuery(st); }
    printf("%-40s %8.3f us\n", "cudaStreamQuery", (now_us() - t0) / 1000);
    return 0;
}
