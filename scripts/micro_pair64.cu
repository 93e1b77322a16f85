// Micro-benchmark (development aid): single-lane latency of the float64
// pieces of one exact-route pair (reference formula, -fmad=false).
#include <cstdio>
#include <cmath>
__global__ void k(const double *g, long long *cyc, double *out)
{
    double a0 = g[0], a1 = g[1], a2 = g[2], b0 = g[3], b1 = g[4], b2 = g[5], na = g[6], nb = g[7];
    long long t0 = clock64();
    const double dot = a0 * b0 + a1 * b1 + a2 * b2;
    long long t1 = clock64();
    const double sq = sqrt(na * nb + dot * 1e-300);
    long long t2 = clock64();
    double z = dot / sq;
    long long t3 = clock64();
    z = fmin(fmax(z, 0.0), 1.0);
    const double y = acos(z);
    long long t4 = clock64();
    const double d1 = a0 - b0, d2 = a1 - b1, d3 = a2 - b2;
    const double l = sqrt(d1 * d1 + d2 * d2 + d3 * d3 + y * 1e-300);
    long long t5 = clock64();
    out[0] = y + l;
    cyc[0] = t1 - t0; cyc[1] = t2 - t1; cyc[2] = t3 - t2; cyc[3] = t4 - t3; cyc[4] = t5 - t4;
}
int main()
{
    double h[8] = {120, 30, 200, 118, 33, 199, 120. * 120 + 30 * 30 + 200 * 200, 118. * 118 + 33 * 33 + 199 * 199};
    double *d, *o; long long *c;
    cudaMalloc(&d, sizeof h); cudaMemcpy(d, h, sizeof h, cudaMemcpyHostToDevice);
    cudaMallocManaged(&c, 64); cudaMallocManaged(&o, 8);
    for (int r = 0; r < 2; r++) { k<<<1, 1>>>(d, c, o); cudaDeviceSynchronize(); }
    printf("dot %lld, sqrt %lld, div %lld, clamp+acos %lld, L2 %lld cycles\n", c[0], c[1], c[2], c[3], c[4]);
    return 0;
}
