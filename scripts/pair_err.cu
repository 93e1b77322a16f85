// Dev harness: worst relative error of the FP32 exact-route pair angle
// (current atan2 form vs the half-angle form) against float64, over random,
// near-parallel and near-orthogonal integer vector pairs.
// build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -fmad=false
//        --expt-relaxed-constexpr -I include scripts/pair_err.cu -o scripts/pair_err
#include <cstdio>
#include <cstdint>
#include <cmath>
#include "../paper_1009_0958_b200/csrc/dfg_fast.cuh"

using namespace dfg;

__device__ uint32_t hash32(uint64_t x)
{
    x ^= x >> 33; x *= 0xff51afd7ed558ccdULL; x ^= x >> 33; x *= 0xc4ceb9fe1a85ec53ULL; x ^= x >> 33;
    return (uint32_t)x;
}

__device__ void gen(uint64_t i, int mode, float a[3], float b[3])
{
    uint32_t h = hash32(i * 7 + mode);
    for (int k = 0; k < 3; k++) { a[k] = (float)(hash32(i * 13 + k + 100 * mode) & 255); }
    if (a[0] + a[1] + a[2] == 0) a[0] = 1;
    if (mode == 0) {
        for (int k = 0; k < 3; k++) b[k] = (float)(hash32(i * 17 + k + 1000) & 255);
    } else if (mode == 1) {  // near-parallel: b ~ s * a + small noise
        float s = 0.05f + (h & 1023) / 1023.f * 5.f;
        for (int k = 0; k < 3; k++) {
            int n = (int)(hash32(i * 19 + k + 2000) % 5) - 2;
            int v = (int)rintf(a[k] * s) + n;
            b[k] = (float)min(255, max(0, v));
        }
    } else {  // near-orthogonal / sparse channels
        for (int k = 0; k < 3; k++) b[k] = (float)((hash32(i * 23 + k + 3000) & 7) == 0 ? (hash32(i + k) & 255) : (hash32(i * 29 + k) & 3));
        a[(h >> 3) % 3] = (float)(h & 3);
    }
    if (b[0] + b[1] + b[2] == 0) b[1] = 1;
    if (a[0] + a[1] + a[2] == 0) a[2] = 1;
}

__device__ void amax(float *p, float v) { atomicMax((int *)p, __float_as_int(v)); }

__global__ void k_err(uint64_t n, int mode, float *out)
{
    float w_old = 0.f, w_new = 0.f, z_old = 0.f, z_new = 0.f;
    for (uint64_t i = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; i < n; i += (uint64_t)gridDim.x * blockDim.x) {
        float a[3], b[3], a2[3], b2[3];
        gen(2 * i, mode, a, b);
        gen(2 * i + 1, mode, a2, b2);
        Pix p{a[0], a[1], a[2], __fsqrt_rn(a[0] * a[0] + a[1] * a[1] + a[2] * a[2])};
        // pair (p, b) and (p, b2): second lane uses p too
        Pair2 q{pk2(b[0], b2[0]), pk2(b[1], b2[1]), pk2(b[2], b2[2]),
                pk2(__fsqrt_rn(b[0] * b[0] + b[1] * b[1] + b[2] * b[2]),
                    __fsqrt_rn(b2[0] * b2[0] + b2[1] * b2[1] + b2[2] * b2[2]))};
        const P2 o = angle_exact2(p, q), h = angle_half2<false>(p, q);
        for (int l = 0; l < 2; l++) {
            const float *bb = l ? b2 : b;
            const double d = (double)a[0] * bb[0] + (double)a[1] * bb[1] + (double)a[2] * bb[2];
            const double c1 = (double)a[1] * bb[2] - (double)a[2] * bb[1];
            const double c2 = (double)a[2] * bb[0] - (double)a[0] * bb[2];
            const double c3 = (double)a[0] * bb[1] - (double)a[1] * bb[0];
            const double th = atan2(sqrt(c1 * c1 + c2 * c2 + c3 * c3), d);
            const float vo = l ? hi2(o) : lo2(o), vh = l ? hi2(h) : lo2(h);
            if (th == 0.0) {
                z_old = fmaxf(z_old, fabsf(vo));
                z_new = fmaxf(z_new, fabsf(vh));
            } else {
                w_old = fmaxf(w_old, (float)(fabs(vo - th) / th));
                w_new = fmaxf(w_new, (float)(fabs(vh - th) / th));
            }
        }
    }
    amax(out + 0, w_old); amax(out + 1, w_new); amax(out + 2, z_old); amax(out + 3, z_new);
}

int main()
{
    float *d;
    cudaMalloc(&d, 16 * sizeof(float));
    const uint64_t n = 1ull << 28;
    for (int mode = 0; mode < 3; mode++) {
        cudaMemset(d, 0, 16 * sizeof(float));
        k_err<<<148 * 8, 256>>>(n, mode, d);
        float h[4];
        cudaMemcpy(h, d, sizeof h, cudaMemcpyDeviceToHost);
        printf("mode %d  pairs %llu  max rel err: atan2-form %.3e (%.2f u)  half-angle %.3e (%.2f u)   theta=0: %.1e %.1e\n",
               mode, (unsigned long long)(2 * n), h[0], h[0] / 5.96e-8, h[1], h[1] / 5.96e-8, h[2], h[3]);
    }
    return 0;
}
