// Micro-benchmark (development aid): single-thread latency of the float64
// building blocks of the re-decision kernel on the GPU.
#include <cstdio>
#include <cmath>
#include "../paper_1009_0958_b200/csrc/dfg_fixup.cu"

__global__ void k(double z, double *out, long long *cyc)
{
    double acc = z;
    long long t0 = clock64();
    for (int i = 0; i < 100; i++) acc = fma(acc, 1.0000001, 1e-9);
    long long t1 = clock64();
    double a = 0;
    for (int i = 0; i < 10; i++) a += acos(z + i * 1e-3 + acc * 1e-30);
    long long t2 = clock64();
    double c = 0;
    for (int i = 0; i < 10; i++) { double zz = z + i * 1e-3 + a * 1e-30; c += dfg::cr_acos_from(zz, acos(zz)); }
    long long t3 = clock64();
    double s = 0;
    for (int i = 0; i < 10; i++) s += sin(z + i + c * 1e-30);
    long long t4 = clock64();
    out[0] = acc + a + c + s;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3;
}

int main()
{
    double *o; long long *c;
    cudaMallocManaged(&o, 8); cudaMallocManaged(&c, 32);
    for (int rep = 0; rep < 2; rep++) {
        k<<<1, 1>>>(0.9, o, c); cudaDeviceSynchronize();
        printf("100 dependent DFMA: %lld cyc; acos: %lld cyc/call; cr_acos(z>=.5): %lld cyc/call; sin: %lld cyc/call\n",
               c[0], c[1] / 10, c[2] / 10, c[3] / 10);
        k<<<1, 1>>>(0.2, o, c); cudaDeviceSynchronize();
        printf("z=0.2: acos %lld, cr_acos %lld cyc/call\n", c[1] / 10, c[2] / 10);
    }
    return 0;
}
