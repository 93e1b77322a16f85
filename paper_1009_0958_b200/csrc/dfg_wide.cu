// dfg_wide.cu -- window sides above 7 (any odd side up to kWideMaxSide).
//
// The reference accepts every odd window side >= 3 (filters.py:141-151,
// _engine.py:494-501).  Sides 3, 5 and 7 -- the ones the paper and the
// configs use -- run the FP32 decision kernels with their float64
// re-decision (dfg_fast.cuh, dfg_w3.cuh); larger windows are rare and are
// decided here directly in binary64 with the reference's operation order
// (the same arithmetic the re-decision stage uses, dfg_f64.cuh): one CTA per
// output pixel, one thread per window candidate i, which forms
//   agg[i] = self + sum_{j != i, ascending j} d(min(i, j), max(i, j))
// (_engine.py:232-314) evaluating its n - 1 pair distances itself (every pair
// is evaluated by both of its candidates: no pair table, so any n fits);
// warp 0 then selects (first strict minimum in window order, _engine.py:317-402;
// the ACWDDF switch, :451-487).  The exact route follows the re-decision's two
// passes: CUDA's acos first, and when a decision margin is below
// FParams::cr_margin the correctly rounded arccos.
#include "dfg_f64.cuh"
#include "dfg_internal.cuh"

namespace dfg {

namespace {

struct WideSel {
    int idx;
    bool close;
};

// value m of candidate i (m = 0: the family's own criterion; ACWDDF m = 1..3:
// the centre-weighted products for k = lam + m - 1)
__device__ inline double wide_value(const FParams &fp, int n, int m, double a, double l, double ad, double ld)
{
    switch (fp.family) {
    case FAM_VMF: return l;
    case FAM_BVDF: return a;
    case FAM_DDF: return a * l;
    case FAM_CWVMF: {
        const double w = (double)(n - 2 * fp.lam + 2 - 1);
        return l + w * ld;
    }
    case FAM_CWDDF: {
        const double w = (double)(n - 2 * fp.lam + 2 - 1);
        return (a + w * ad) * (l + w * ld);
    }
    default: {  // ACWDDF
        if (m == 0) return a * l;
        const double w = (double)(n - 2 * (fp.lam + m - 1) + 2 - 1);
        return (a + w * ad) * (l + w * ld);
    }
    }
}

// Warp 0: first strict minimum of value m over the n candidates (window
// order) and whether the relative gap to the best candidate of a different
// colour is below `margin` (select64m's rule).
__device__ inline WideSel wide_select(const FParams &fp, int n, int m, int lane, const E64 *e, const double *aA,
                                      const double *aL, const double *AD, const double *LD, double margin)
{
    const double INF = __longlong_as_double(0x7ff0000000000000LL);
    double bv = INF;
    int bi = 1 << 30;
    for (int i = lane; i < n; i += 32) {
        const double v = wide_value(fp, n, m, aA[i], aL[i], AD[i], LD[i]);
        if (v < bv) { bv = v; bi = i; }
    }
    for (int off = 16; off > 0; off >>= 1) {
        const double ov = __shfl_xor_sync(0xffffffffu, bv, off);
        const int oi = __shfl_xor_sync(0xffffffffu, bi, off);
        if (ov < bv || (ov == bv && oi < bi)) { bv = ov; bi = oi; }
    }
    double other = INF;
    for (int i = lane; i < n; i += 32) {
        const double v = wide_value(fp, n, m, aA[i], aL[i], AD[i], LD[i]);
        if (!same_col(e[i], e[bi]) && v > 0.0 && v < other) other = v;
    }
    for (int off = 16; off > 0; off >>= 1) other = fmin(other, __shfl_xor_sync(0xffffffffu, other, off));
    const double den = fmax(fabs(bv), fabs(other));
    WideSel r;
    r.idx = bi;
    r.close = !isinf(other) && (den == 0.0 || other - bv < margin * den);
    return r;
}

template <bool CR>
__device__ inline void wide_aggregates(const FParams &fp, int n, const E64 *e, double *aA, double *aL, double *AD,
                                       double *LD)
{
    const int dc = (n - 1) / 2;
    const bool needA = fp.family != FAM_VMF && fp.family != FAM_CWVMF;
    const bool needL = fp.family != FAM_BVDF && !CR;  // pass 2 changes the angular terms only
    const bool dup_rule = fp.family == FAM_CWDDF && fp.strategy == ST_MINIMAX;  // pair_tables, dfg_f64.cuh
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
        double a = fp.self_term, l = 0.0, ad = fp.self_term, ld = 0.0;
        for (int j = 0; j < n; j++) {
            if (j == i) continue;
            const E64 &x = e[j < i ? j : i], &y = e[j < i ? i : j];
            if (needA) {
                const double d = (dup_rule && same_col(x, y)) ? fp.cs[0] : pairA<CR>(x, y, fp);
                a += d;
                if (j == dc) ad = d;
            }
            if (needL) {
                const double d = mink64(x.raw, y.raw, fp.p);
                l += d;
                if (j == dc) ld = d;
            }
        }
        if (needA) { aA[i] = a; AD[i] = ad; }
        if (needL) { aL[i] = l; LD[i] = ld; }
    }
}

__device__ inline WideSel wide_decide(const FParams &fp, int n, int lane, const E64 *e, const double *aA,
                                      const double *aL, const double *AD, const double *LD)
{
    const int dc = (n - 1) / 2;
    const double cm = fp.cr_margin;
    if (fp.family != FAM_ACWDDF) return wide_select(fp, n, 0, lane, e, aA, aL, AD, LD, cm);
    // _engine.py:451-487
    const WideSel sd = wide_select(fp, n, 0, lane, e, aA, aL, AD, LD, cm);
    bool any = false;
    double sv = 0.0;
    for (int k = 0; k < 3; k++) {
        const WideSel s = wide_select(fp, n, 1 + k, lane, e, aA, aL, AD, LD, cm);
        any = any || s.close;
        double a = AD[s.idx];
        if (fp.strategy == ST_CHROMA) a = fp.slope * a + fp.intercept;
        sv += a * LD[s.idx];
    }
    const bool fires = sv > fp.threshold;
    if (fires) any = any || sd.close;
    const double den = fmax(fabs(sv), fabs(fp.threshold));
    any = any || den == 0.0 || fabs(sv - fp.threshold) < cm * den;
    WideSel r;
    r.idx = fires ? sd.idx : dc;
    r.close = any;
    return r;
}

__global__ void dfg_wide_kernel(const uint8_t *__restrict__ in, uint8_t *__restrict__ out, const __grid_constant__ KParams kp)
{
    extern __shared__ __align__(16) unsigned char smem[];
    const FParams &fp = kp.fp;
    const int s = fp.window, n = s * s, h = s / 2;
    E64 *e = reinterpret_cast<E64 *>(smem);
    double *aA = reinterpret_cast<double *>(e + n), *aL = aA + n, *AD = aL + n, *LD = AD + n;
    __shared__ int s_idx;
    __shared__ bool s_close;
    const long long per_frame = (long long)kp.out_rows * kp.W, total = per_frame * kp.n_frames;
    const int lane = threadIdx.x & 31;
    unsigned decided = 0;  // every pixel of this path is a float64 decision
    for (long long px = blockIdx.x; px < total; px += gridDim.x) {
        const int frame = (int)(px / per_frame);
        const long long rem = px - frame * per_frame;
        const int oy = (int)(rem / kp.W), ox = (int)(rem - (long long)oy * kp.W);
        const uint8_t *fin = in + (long long)frame * kp.in_fstride;
        for (int i = threadIdx.x; i < n; i += blockDim.x) {
            const int u = i / s, v = i - u * s;
            int gy = resolve_idx(kp.out_row0 + oy + u - h, kp.global_H, kp.border) - kp.in_row0;
            gy = min(max(gy, 0), kp.in_rows - 1);
            const int gx = resolve_idx(ox + v - h, kp.W, kp.border);
            const uint8_t *p = fin + (long long)gy * kp.in_pitch + 3 * gx;
            prep64(make_float4((float)p[0], (float)p[1], (float)p[2], 0.f), fp.strategy, e[i]);
        }
        __syncthreads();
        wide_aggregates<false>(fp, n, e, aA, aL, AD, LD);
        __syncthreads();
        if (threadIdx.x < 32) {
            const WideSel r = wide_decide(fp, n, lane, e, aA, aL, AD, LD);
            if (lane == 0) { s_idx = r.idx; s_close = r.close; }
        }
        __syncthreads();
        if (fp.strategy == ST_EXACT && fp.family != FAM_VMF && fp.family != FAM_CWVMF && s_close) {
            // pass 2: the correctly rounded arccos (dfg_f64.cuh)
            if (threadIdx.x == 0) atomicAdd(kp.flag_count + 1, 1u);
            wide_aggregates<true>(fp, n, e, aA, aL, AD, LD);
            __syncthreads();
            if (threadIdx.x < 32) {
                const WideSel r = wide_decide(fp, n, lane, e, aA, aL, AD, LD);
                if (lane == 0) s_idx = r.idx;
            }
            __syncthreads();
        }
        if (threadIdx.x == 0) {
            const E64 &w = e[s_idx];
            uint8_t *op = out + (long long)frame * kp.out_fstride + (long long)oy * kp.out_pitch + 3 * ox;
            op[0] = (uint8_t)w.raw[0];
            op[1] = (uint8_t)w.raw[1];
            op[2] = (uint8_t)w.raw[2];
        }
        __syncthreads();  // e / aggregates are reused by the next pixel
        decided++;
    }
    if (threadIdx.x == 0 && decided) atomicAdd(kp.flag_count, decided);
}

}  // namespace

cudaError_t launch_wide(cudaStream_t st, const uint8_t *in, uint8_t *out, const KParams &kp)
{
    const int n = kp.fp.window * kp.fp.window;
    const size_t smem = (size_t)n * (sizeof(E64) + 4 * sizeof(double));
    static bool attr_set[64] = {};
    int dev = 0;
    cudaGetDevice(&dev);
    if (!attr_set[dev & 63]) {
        cudaError_t e = cudaFuncSetAttribute(dfg_wide_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                             (int)((size_t)kWideMaxSide * kWideMaxSide * (sizeof(E64) + 4 * sizeof(double))));
        if (e != cudaSuccess) return e;
        attr_set[dev & 63] = true;
    }
    int threads = (n + 31) & ~31;
    if (threads > 512) threads = 512;
    const long long total = (long long)kp.out_rows * kp.W * kp.n_frames;
    const long long cap = (long long)sm_count(dev) * 64;  // persistent CTAs walking pixels
    const int grid = (int)(total < cap ? total : cap);
    dfg_wide_kernel<<<grid, threads, smem, st>>>(in, out, kp);
    return cudaGetLastError();
}

}  // namespace dfg
