// dfg_metrics.cu -- the reference's effectiveness criteria (MAE, PSNR, NCD;
// reference metrics.py:64-109) as one device reduction over two uint8 images.
//
// MAE = mean |a - b| over 3MN components; PSNR = 10 log10(255^2 / MSE);
// NCD = 1000 * sum_px |Luv(b) - Luv(a)| / sum_px |Luv(a)|, sRGB -> linear ->
// XYZ (D65) -> CIE L*u*v* with the reference's constants (metrics.py:18-31).
// The sRGB linearisation of the 256 code values is tabulated on the host;
// sums are float64 (per-thread, warp, then atomic), so results agree with the
// reference's numpy reductions to ~1e-12 relative, not bitwise (summation
// order).
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/dirfilt_gpu.h"

namespace {

__constant__ double kLin[256];

struct MetricConsts {
    double m[9];
    double white_y, uprime_n, vprime_n, cbrt_eps;
};

__device__ __forceinline__ void luv(uint32_t r, uint32_t g, uint32_t b, const MetricConsts &k, double o[3])
{
    const double lr = kLin[r], lg = kLin[g], lb = kLin[b];
    const double x = lr * k.m[0] + lg * k.m[1] + lb * k.m[2];
    const double y = lr * k.m[3] + lg * k.m[4] + lb * k.m[5];
    const double z = lr * k.m[6] + lg * k.m[7] + lb * k.m[8];
    const double yr = y / k.white_y;
    const double L = yr > k.cbrt_eps ? 116.0 * cbrt(yr) - 16.0 : (29.0 / 3.0) * (29.0 / 3.0) * (29.0 / 3.0) * yr;
    const double den = x + 15.0 * y + 3.0 * z;
    const double up = den > 0.0 ? 4.0 * x / den : k.uprime_n;
    const double vp = den > 0.0 ? 9.0 * y / den : k.vprime_n;
    o[0] = L;
    o[1] = 13.0 * L * (up - k.uprime_n);
    o[2] = 13.0 * L * (vp - k.vprime_n);
}

__global__ void __launch_bounds__(256) dfg_metrics_kernel(const uint8_t *__restrict__ a, const uint8_t *__restrict__ b,
                                                          int H, int W, long long pa, long long pb, MetricConsts k,
                                                          double *acc)
{
    double s_abs = 0, s_sq = 0, s_err = 0, s_ref = 0;
    const long long npx = (long long)H * W;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < npx;
         i += (long long)gridDim.x * blockDim.x) {
        const int r = (int)(i / W), c = (int)(i - (long long)r * W);
        const uint8_t *x = a + r * pa + 3LL * c, *y = b + r * pb + 3LL * c;
        for (int ch = 0; ch < 3; ch++) {
            const double d = (double)y[ch] - (double)x[ch];
            s_abs += fabs(d);
            s_sq += d * d;
        }
        double lo[3], lt[3];
        luv(x[0], x[1], x[2], k, lo);
        luv(y[0], y[1], y[2], k, lt);
        const double e0 = lt[0] - lo[0], e1 = lt[1] - lo[1], e2 = lt[2] - lo[2];
        s_err += sqrt(e0 * e0 + e1 * e1 + e2 * e2);
        s_ref += sqrt(lo[0] * lo[0] + lo[1] * lo[1] + lo[2] * lo[2]);
    }
    for (int off = 16; off; off >>= 1) {
        s_abs += __shfl_xor_sync(0xffffffffu, s_abs, off);
        s_sq += __shfl_xor_sync(0xffffffffu, s_sq, off);
        s_err += __shfl_xor_sync(0xffffffffu, s_err, off);
        s_ref += __shfl_xor_sync(0xffffffffu, s_ref, off);
    }
    if ((threadIdx.x & 31) == 0) {
        atomicAdd(acc + 0, s_abs);
        atomicAdd(acc + 1, s_sq);
        atomicAdd(acc + 2, s_err);
        atomicAdd(acc + 3, s_ref);
    }
}

}  // namespace

extern "C" DFG_API int dfg_image_metrics(const uint8_t *d_ref, const uint8_t *d_test, int32_t H, int32_t W,
                                         int64_t ref_pitch, int64_t test_pitch, double *out3, void *d_scratch,
                                         void *stream)
{
    if (!d_ref || !d_test || !out3 || !d_scratch || H < 1 || W < 1 || ref_pitch < 3LL * W || test_pitch < 3LL * W)
        return DFG_E_ARG;
    static bool lut_ready = false;  // the table is the same for every device-visible context
    static int lut_dev = -1;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!lut_ready || lut_dev != dev) {
        double lin[256];
        for (int v = 0; v < 256; v++) {  // metrics.py:80-81
            const double cv = v / 255.0;
            lin[v] = cv <= 0.04045 ? cv / 12.92 : pow((cv + 0.055) / 1.055, 2.4);
        }
        if (cudaMemcpyToSymbol(kLin, lin, sizeof lin) != cudaSuccess) return DFG_E_CUDA;
        lut_ready = true;
        lut_dev = dev;
    }
    MetricConsts k;
    const double M[9] = {0.4124564, 0.3575761, 0.1804375, 0.2126729, 0.7151522,
                         0.0721750, 0.0193339, 0.1191920, 0.9503041};
    for (int i = 0; i < 9; i++) k.m[i] = M[i];
    const double wx = 0.95047, wy = 1.0, wz = 1.08883;
    const double dn = wx + 15.0 * wy + 3.0 * wz;
    k.white_y = wy;
    k.uprime_n = 4.0 * wx / dn;
    k.vprime_n = 9.0 * wy / dn;
    k.cbrt_eps = (6.0 / 29.0) * (6.0 / 29.0) * (6.0 / 29.0);
    cudaStream_t st = (cudaStream_t)stream;
    double *acc = (double *)d_scratch;
    if (cudaMemsetAsync(acc, 0, 4 * sizeof(double), st) != cudaSuccess) return DFG_E_CUDA;
    const long long npx = (long long)H * W;
    long long blocks = (npx + 255) / 256;
    if (blocks > 148 * 16) blocks = 148 * 16;
    dfg_metrics_kernel<<<(unsigned)blocks, 256, 0, st>>>(d_ref, d_test, H, W, ref_pitch, test_pitch, k, acc);
    double h[4];
    if (cudaMemcpyAsync(h, acc, sizeof h, cudaMemcpyDeviceToHost, st) != cudaSuccess) return DFG_E_CUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return DFG_E_CUDA;
    const double n3 = 3.0 * (double)npx;
    out3[0] = h[0] / n3;
    const double mse = h[1] / n3;
    out3[1] = mse == 0.0 ? INFINITY : 10.0 * log10(255.0 * 255.0 / mse);
    out3[2] = h[3] == 0.0 ? (h[2] == 0.0 ? 0.0 : INFINITY) : 1000.0 * (h[2] / h[3]);
    return DFG_OK;
}
