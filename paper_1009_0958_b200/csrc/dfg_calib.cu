// dfg_calib.cu -- the angle-vs-chromaticity calibration fit (reference
// calibration.py:83-125; paper Sec. 3, 10^8 pairs in "exact-replication
// mode") on the device.
//
// Samples: numpy's PCG64 stream as `sample_angle_chromaticity_pairs` draws it
// (calibration.py:92-101): va = uniform(0, 255, (pairs, 3)) consumes draws
// 0 .. 3*pairs-1, vb the next 3*pairs; uniform = 0 + 255 * next_double.
// Each thread jumps the LCG to its run of pairs (both streams) and
// regenerates the samples in every pass, so nothing is stored: pass 0 sums
// (B, A), pass 1 the central second moments about given means, pass 2 the
// residual sums about a given line.  Arithmetic is the reference's float64
// formula order (this unit is built with -fmad=false); per-block partial
// sums are reduced in a fixed order, so results are deterministic.
#include <cuda_runtime.h>
#include <math.h>
#include <stdint.h>

#include "../../include/dirfilt_gpu.h"

namespace {

struct u128 {
    uint64_t hi, lo;
};
__device__ __forceinline__ u128 mul128(u128 a, u128 b)
{
    u128 r;
    r.lo = a.lo * b.lo;
    r.hi = __umul64hi(a.lo, b.lo) + a.hi * b.lo + a.lo * b.hi;
    return r;
}
__device__ __forceinline__ u128 add128(u128 a, u128 b)
{
    u128 r;
    r.lo = a.lo + b.lo;
    r.hi = a.hi + b.hi + (r.lo < a.lo ? 1ull : 0ull);
    return r;
}
__device__ __constant__ u128 kMultC = {0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull};

__device__ u128 advance(u128 state, u128 inc, unsigned long long delta)
{
    u128 am = {0, 1}, ap = {0, 0}, cm = kMultC, cp = inc;
    while (delta) {
        if (delta & 1ull) {
            am = mul128(am, cm);
            ap = add128(mul128(ap, cm), cp);
        }
        cp = mul128(add128(cm, u128{0, 1}), cp);
        cm = mul128(cm, cm);
        delta >>= 1;
    }
    return add128(mul128(am, state), ap);
}
__device__ __forceinline__ double next_double(u128 &s, const u128 inc)
{
    s = add128(mul128(s, kMultC), inc);
    const uint64_t x = s.hi ^ s.lo;
    const unsigned rot = (unsigned)(s.hi >> 58);
    const uint64_t out = (x >> rot) | (x << ((64u - rot) & 63u));
    return (double)(out >> 11) * (1.0 / 9007199254740992.0);
}

constexpr int kRun = 64;      // pairs per thread run
constexpr int kThreads = 256;

// fixed-order block reduction -> one partial triple per block
__device__ void block_reduce3(double acc0, double acc1, double acc2, double *partials)
{
    __shared__ double red[3][kThreads];
    red[0][threadIdx.x] = acc0;
    red[1][threadIdx.x] = acc1;
    red[2][threadIdx.x] = acc2;
    __syncthreads();
    for (int w = kThreads / 2; w > 0; w >>= 1) {
        if ((int)threadIdx.x < w) {
            red[0][threadIdx.x] += red[0][threadIdx.x + w];
            red[1][threadIdx.x] += red[1][threadIdx.x + w];
            red[2][threadIdx.x] += red[2][threadIdx.x + w];
        }
        __syncthreads();
    }
    if (threadIdx.x == 0) {
        partials[3 * blockIdx.x + 0] = red[0][0];
        partials[3 * blockIdx.x + 1] = red[1][0];
        partials[3 * blockIdx.x + 2] = red[2][0];
    }
}

struct Sample {
    double b, a;
};

// calibration.py:102-113 for one pair
__device__ __forceinline__ Sample pair_sample(const double va[3], const double vb[3], double p)
{
    const double sa = (va[0] + va[1]) + va[2], sb = (vb[0] + vb[1]) + vb[2];
    double d[3];
    for (int k = 0; k < 3; k++) d[k] = fabs(va[k] / sa - vb[k] / sb);
    Sample r;
    if (p == 2.0) {
        r.b = sqrt((d[0] * d[0] + d[1] * d[1]) + d[2] * d[2]);
    } else {
        r.b = pow((pow(d[0], p) + pow(d[1], p)) + pow(d[2], p), 1.0 / p);
    }
    const double dot = (va[0] * vb[0] + va[1] * vb[1]) + va[2] * vb[2];
    const double na = (va[0] * va[0] + va[1] * va[1]) + va[2] * va[2];
    const double nb = (vb[0] * vb[0] + vb[1] * vb[1]) + vb[2] * vb[2];
    const double z = dot / sqrt(na * nb);
    r.a = acos(fmin(fmax(z, 0.0), 1.0));
    return r;
}

__global__ void __launch_bounds__(kThreads) dfg_calib_kernel(dfg_calib_params cp, int mode, double x0, double x1,
                                                             double *partials, double *d_b, double *d_a)
{
    const u128 s0 = {cp.state_hi, cp.state_lo}, inc = {cp.inc_hi, cp.inc_lo};
    const long long n = cp.pairs;
    const long long runs = (n + kRun - 1) / kRun;
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    for (long long run = blockIdx.x * (long long)kThreads + threadIdx.x; run < runs;
         run += (long long)gridDim.x * kThreads) {
        const long long i0 = run * kRun, i1 = i0 + kRun < n ? i0 + kRun : n;
        u128 sa = advance(s0, inc, 3ull * (unsigned long long)i0);
        u128 sb = advance(s0, inc, 3ull * (unsigned long long)(n + i0));
        for (long long i = i0; i < i1; i++) {
            double va[3], vb[3];
            for (int k = 0; k < 3; k++) va[k] = 0.0 + 255.0 * next_double(sa, inc);
            for (int k = 0; k < 3; k++) vb[k] = 0.0 + 255.0 * next_double(sb, inc);
            const Sample s = pair_sample(va, vb, cp.p);
            if (mode == 0) {
                acc0 += s.b;
                acc1 += s.a;
            } else if (mode == 1) {
                const double db = s.b - x0, da = s.a - x1;
                acc0 += db * db;
                acc1 += da * da;
                acc2 += db * da;
            } else if (mode == 2) {
                const double r = s.a - (x0 * s.b + x1);
                acc0 += r * r;
                acc1 += fabs(r);
            } else {
                d_b[i] = s.b;
                d_a[i] = s.a;
            }
        }
    }
    if (mode == 3) return;
    block_reduce3(acc0, acc1, acc2, partials);
}

// The same three reductions over stored samples (reference fit_line,
// calibration.py:47-80, on caller-provided (b, a) arrays).
__global__ void __launch_bounds__(kThreads) dfg_array_reduce_kernel(const double *__restrict__ b,
                                                                    const double *__restrict__ a, long long n,
                                                                    int mode, double x0, double x1,
                                                                    double *partials)
{
    double acc0 = 0.0, acc1 = 0.0, acc2 = 0.0;
    for (long long i = blockIdx.x * (long long)kThreads + threadIdx.x; i < n; i += (long long)gridDim.x * kThreads) {
        const double sb = b[i], sa = a[i];
        if (mode == 0) {
            acc0 += sb;
            acc1 += sa;
        } else if (mode == 1) {
            const double db = sb - x0, da = sa - x1;
            acc0 += db * db;
            acc1 += da * da;
            acc2 += db * da;
        } else {
            const double r = sa - (x0 * sb + x1);
            acc0 += r * r;
            acc1 += fabs(r);
        }
    }
    block_reduce3(acc0, acc1, acc2, partials);
}

constexpr int kBlocks = 148 * 8;

// per-block partial triples -> out3, summed in block order on the host
// (kBlocks x 3 doubles: a fixed-order, deterministic final reduction)
int sum_partials(const double *part, double *out3, cudaStream_t st)
{
    static thread_local double host[kBlocks * 3];
    if (cudaMemcpyAsync(host, part, sizeof host, cudaMemcpyDeviceToHost, st) != cudaSuccess) return DFG_E_CUDA;
    if (cudaStreamSynchronize(st) != cudaSuccess) return DFG_E_CUDA;
    double s[3] = {0.0, 0.0, 0.0};
    for (int b = 0; b < kBlocks; b++)
        for (int k = 0; k < 3; k++) s[k] += host[3 * b + k];
    out3[0] = s[0];
    out3[1] = s[1];
    out3[2] = s[2];
    return DFG_OK;
}

}  // namespace

extern "C" DFG_API size_t dfg_calib_scratch_bytes(void) { return (size_t)kBlocks * 3 * sizeof(double); }

extern "C" DFG_API int dfg_calib_reduce(const dfg_calib_params *cp, int32_t mode, double x0, double x1,
                                        double *out3, void *d_scratch, size_t scratch_bytes, void *stream)
{
    if (!cp || !out3 || !d_scratch || cp->pairs < 1 || mode < 0 || mode > 2 || !(cp->p >= 1.0) ||
        scratch_bytes < dfg_calib_scratch_bytes())
        return DFG_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    double *part = (double *)d_scratch;
    dfg_calib_kernel<<<kBlocks, kThreads, 0, st>>>(*cp, mode, x0, x1, part, nullptr, nullptr);
    if (cudaGetLastError() != cudaSuccess) return DFG_E_CUDA;
    return sum_partials(part, out3, st);
}

extern "C" DFG_API int dfg_moments_reduce(const double *d_b, const double *d_a, int64_t n, int32_t mode, double x0,
                                          double x1, double *out3, void *d_scratch, size_t scratch_bytes,
                                          void *stream)
{
    if (!d_b || !d_a || !out3 || !d_scratch || n < 1 || mode < 0 || mode > 2 ||
        scratch_bytes < dfg_calib_scratch_bytes())
        return DFG_E_ARG;
    cudaStream_t st = (cudaStream_t)stream;
    double *part = (double *)d_scratch;
    dfg_array_reduce_kernel<<<kBlocks, kThreads, 0, st>>>(d_b, d_a, n, mode, x0, x1, part);
    if (cudaGetLastError() != cudaSuccess) return DFG_E_CUDA;
    return sum_partials(part, out3, st);
}

extern "C" DFG_API int dfg_calib_samples(const dfg_calib_params *cp, double *d_b, double *d_a, void *stream)
{
    if (!cp || !d_b || !d_a || cp->pairs < 1 || !(cp->p >= 1.0)) return DFG_E_ARG;
    dfg_calib_kernel<<<kBlocks, kThreads, 0, (cudaStream_t)stream>>>(*cp, 3, 0.0, 0.0, nullptr, d_b, d_a);
    return cudaGetLastError() == cudaSuccess ? DFG_OK : DFG_E_CUDA;
}
