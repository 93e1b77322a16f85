// dfg_f64.cuh -- float64 re-decision of the pixels the FP32 decision stage
// could not decide with certainty (decision margin inside its error budget).
//
// The n(n-1)/2 window pair distances are evaluated once, spread over the
// CTA's threads, into shared tables; then lane i (and i + 32) of one warp
// forms agg[i] = self + sum_{j != i, ascending j} d(min(i,j), max(i,j))
// in IEEE binary64 with the reference's exact operation order
// (_engine.py:46-164 planes and pair formulas, :232-314 aggregate order,
// :317-402 selection, :451-487 ACWDDF switch).  Every unit including this
// header is compiled with -fmad=false so no multiply-add is contracted:
// every product, sum, quotient and square root rounds exactly as numba's
// (fastmath=False); explicit fma() calls (double-double) are unaffected.
//
// The only non-IEEE-basic operation on the path is the exact route's acos
// (glibc libm in the reference).  Pass 1 uses CUDA's acos; when a decision
// margin of that pass is below FParams::cr_margin (1e-12 relative), pass 2
// recomputes with cr_acos_from(): a double-double Newton refinement that
// returns the correctly rounded arccos (verified against a 160-bit
// reference and against glibc on CPU: tests/test_abi.py).  glibc's acos is
// itself correctly rounded on all but ~0.1% of arguments, each off by one
// ulp; decisions that hinge on that last ulp are the documented residual
// near-ties ("Exactness").
#pragma once

#include <math.h>

#include "dfg_internal.cuh"

namespace dfg {

// ---------------- double-double helpers (host + device) --------------------
struct dd {
    double hi, lo;
};

__host__ __device__ static inline dd two_sum(double a, double b)
{
    double s = a + b;
    double bb = s - a;
    double e = (a - (s - bb)) + (b - bb);
    return {s, e};
}

__host__ __device__ static inline dd quick_two_sum(double a, double b)
{
    double s = a + b;
    return {s, b - (s - a)};
}

__host__ __device__ static inline dd two_prod(double a, double b)
{
    double p = a * b;
    return {p, fma(a, b, -p)};
}

__host__ __device__ static inline dd dd_add(dd a, dd b)
{
    dd s = two_sum(a.hi, b.hi);
    dd t = two_sum(a.lo, b.lo);
    s.lo += t.hi;
    s = quick_two_sum(s.hi, s.lo);
    s.lo += t.lo;
    return quick_two_sum(s.hi, s.lo);
}

__host__ __device__ static inline dd dd_mul(dd a, dd b)
{
    dd p = two_prod(a.hi, b.hi);
    p.lo += a.hi * b.lo + a.lo * b.hi;
    return quick_two_sum(p.hi, p.lo);
}

// (-1)^k / (2k+1)!  as double-double (exact rationals rounded, hi + lo)
#define DFG_SIN_TERMS 13
__host__ __device__ static inline dd sin_coef(int k)
{
    switch (k) {
    case 0: return {1.0, 0.0};
    case 1: return {-0.16666666666666666, -9.25185853854297e-18};
    case 2: return {0.008333333333333333, 1.1564823173178714e-19};
    case 3: return {-0.0001984126984126984, -1.7209558293420705e-22};
    case 4: return {2.7557319223985893e-06, -1.858393274046472e-22};
    case 5: return {-2.505210838544172e-08, 1.448814070935912e-24};
    case 6: return {1.6059043836821613e-10, 1.2585294588752098e-26};
    case 7: return {-7.647163731819816e-13, -7.03872877733453e-30};
    case 8: return {2.8114572543455206e-15, 1.6508842730861433e-31};
    case 9: return {-8.22063524662433e-18, -2.2141894119604265e-34};
    case 10: return {1.9572941063391263e-20, -1.3643503830087908e-36};
    case 11: return {-3.868170170630684e-23, 8.843177655482344e-40};
    default: return {6.446950284384474e-26, -1.9330404233703465e-42};
    }
}

// sin(x) for |x| <= pi/6 in double-double (Taylor, truncation < 1e-32)
__host__ __device__ static inline dd sin_dd(dd x)
{
    dd x2 = dd_mul(x, x);
    dd p = sin_coef(DFG_SIN_TERMS - 1);
    for (int k = DFG_SIN_TERMS - 2; k >= 0; k--) p = dd_add(dd_mul(p, x2), sin_coef(k));
    return dd_mul(p, x);
}

// Correctly rounded arccos on [0, 1] (up to a ~1e-16-ulp rounding window):
// one Newton step y = y0 + (cos y0 - z) / sin y0 from any starting value y0
// within a few ulps, the residual evaluated in double-double without
// cancellation: (1 - z) - 2 sin^2(y0/2) for z >= 1/2, sin(pi/2 - y0) - z else.
__host__ __device__ static inline double cr_acos_from(double z, double y0)
{
    if (z >= 1.0) return 0.0;
    const double PIO2_HI = 1.5707963267948966, PIO2_LO = 6.123233995736766e-17;
    dd r;
    if (z >= 0.5) {
        dd s = sin_dd({0.5 * y0, 0.0});
        dd s2 = dd_mul(s, s);
        r = dd_add({1.0 - z, 0.0}, {-2.0 * s2.hi, -2.0 * s2.lo});
    } else {
        dd x = dd_add(two_sum(PIO2_HI, -y0), {PIO2_LO, 0.0});
        r = dd_add(sin_dd(x), {-z, 0.0});
    }
    return y0 + (r.hi + r.lo) / sin(y0);
}

// ---------------- reference arithmetic in binary64 -------------------------
struct E64 {
    double raw[3];
    double g[3];
    double g4;
};

__device__ static inline void prep64(const float4 &rec, int strategy, E64 &e)
{
    const double r = rec.x, g = rec.y, b = rec.z;  // exact integers 0..255
    e.raw[0] = r; e.raw[1] = g; e.raw[2] = b;
    if (strategy == ST_CHROMA) {  // _engine.py:87-103
        const double s = r + g + b;
        if (s == 0.0) {
            const double third = 1.0 / 3.0;
            e.g[0] = e.g[1] = e.g[2] = third;
        } else {
            e.g[0] = r / s; e.g[1] = g / s; e.g[2] = b / s;
        }
        e.g4 = 0.0;
    } else {  // _engine.py:46-72
        double a1 = r, a2 = g, a3 = b;
        if (a1 == 0.0 && a2 == 0.0 && a3 == 0.0) a1 = a2 = a3 = 1.0;
        e.g[0] = a1; e.g[1] = a2; e.g[2] = a3;
        const double nsq = a1 * a1 + a2 * a2 + a3 * a3;
        e.g4 = (strategy == ST_MINIMAX) ? 1.0 / sqrt(nsq) : nsq;
    }
}

__device__ static inline double clamp01(double z)
{
    if (z < 0.0) z = 0.0;
    if (z > 1.0) z = 1.0;
    return z;
}

__device__ static inline double mink64(const double *x, const double *y, double p)
{
    const double d1 = x[0] - y[0], d2 = x[1] - y[1], d3 = x[2] - y[2];
    if (p == 2.0) return sqrt(d1 * d1 + d2 * d2 + d3 * d3);
    if (p == 1.0) return fabs(d1) + fabs(d2) + fabs(d3);
    return pow(pow(fabs(d1), p) + pow(fabs(d2), p) + pow(fabs(d3), p), 1.0 / p);
}

template <bool CR>
__device__ static inline double pairA(const E64 &a, const E64 &b, const FParams &fp)
{
    if (fp.strategy == ST_EXACT) {  // _engine.py:111-119
        const double dot = a.g[0] * b.g[0] + a.g[1] * b.g[1] + a.g[2] * b.g[2];
        const double z = clamp01(dot / sqrt(a.g4 * b.g4));
        const double y0 = acos(z);
        return CR ? cr_acos_from(z, y0) : y0;
    }
    if (fp.strategy == ST_MINIMAX) {  // _engine.py:134-147
        const double dot = a.g[0] * b.g[0] + a.g[1] * b.g[1] + a.g[2] * b.g[2];
        const double z = clamp01(dot * (a.g4 * b.g4));
        const double t = sqrt(1.0 - z);
        const double *c = fp.ca, *s = fp.cs;
        const double pa = c[0] + z * (c[1] + z * (c[2] + z * (c[3] + z * c[4])));
        const double ps = s[0] + t * (s[1] + t * (s[2] + t * (s[3] + t * s[4])));
        const double f = (z >= 0.5) ? 1.0 : 0.0;
        return f * ps + (1.0 - f) * pa;
    }
    return mink64(a.g, b.g, fp.p);  // chromaticity planes, _engine.py:264-281
}

struct Cand {
    double v;
    int i;
};

__device__ static inline bool same_col(const E64 &a, const E64 &b)
{
    return a.raw[0] == b.raw[0] && a.raw[1] == b.raw[1] && a.raw[2] == b.raw[2];
}

__device__ static inline double shfl_slot(const double v[2], int idx)
{
    const double a = __shfl_sync(0xffffffffu, v[0], idx & 31);
    const double b = __shfl_sync(0xffffffffu, v[1], idx & 31);
    return (idx >> 5) ? b : a;
}

// Pair table index of (i < j) in row-major upper-triangle order.
__device__ static inline int pair_index(int i, int j, int n) { return i * n - i * (i + 1) / 2 + (j - i - 1); }

// Evaluate every window pair once, spread over `nthreads` threads, into the
// shared tables dA / dL (binary64, reference formulas).  The caller
// synchronises before the tables are read.
template <bool CR>
__device__ static void pair_tables(const E64 *e, const FParams &fp, int t, int nthreads, double *dA, double *dL,
                                   bool needA, bool needL)
{
    const int n = fp.window * fp.window, P = n * (n - 1) / 2;
    for (int k = t; k < P; k += nthreads) {
        // invert k -> (i, j), i < j, row-major upper triangle
        int i = 0, rem = k;
        while (rem >= n - 1 - i) { rem -= n - 1 - i; i++; }
        const int j = i + 1 + rem;
        if (needA) {
            // the window-level forms the centre-weighted filters come from
            // (filters.py:296-337) special-case equal vectors under minimax:
            // fast_acos(1) = a0 exactly (distance.py:217-218)
            const bool cw_dup = (fp.family == FAM_CWDDF) && fp.strategy == ST_MINIMAX && same_col(e[i], e[j]);
            dA[k] = cw_dup ? fp.cs[0] : pairA<CR>(e[i], e[j], fp);
        }
        if (needL && !CR) dL[k] = mink64(e[i].raw, e[j].raw, fp.p);
    }
}

// Warp-sized variant for windows of N <= 2 x 32 pairs per lane (3x3: 36
// pairs): each lane evaluates its pairs k = lane and lane + 32 in one
// straight-line block (the second clamped to a valid pair, its store
// predicated), so the two float64 chains overlap instead of running one
// after the other -- the re-decision latency is what the row sweep waits on.
template <bool CR, int N>
__device__ static void pair_tables_warp(const E64 *e, const FParams &fp, int lane, double *dA, double *dL,
                                        bool needA, bool needL)
{
    constexpr int P = N * (N - 1) / 2;
    static_assert(P <= 64, "two pairs per lane at most");
    int ii[2], jj[2];
#pragma unroll
    for (int r = 0; r < 2; r++) {
        const int k = min(lane + 32 * r, P - 1);
        int i = 0, rem = k;
#pragma unroll
        for (int q = 0; q < N - 1; q++)
            if (rem >= N - 1 - i) { rem -= N - 1 - i; i++; }
        ii[r] = i;
        jj[r] = i + 1 + rem;
    }
    double va[2], vl[2];
#pragma unroll
    for (int r = 0; r < 2; r++) {
        const E64 &a = e[ii[r]], &b = e[jj[r]];
        if (needA) {
            const bool cw_dup = (fp.family == FAM_CWDDF) && fp.strategy == ST_MINIMAX && same_col(a, b);
            va[r] = cw_dup ? fp.cs[0] : pairA<CR>(a, b, fp);
        }
        if (needL && !CR) vl[r] = mink64(a.raw, b.raw, fp.p);
    }
#pragma unroll
    for (int r = 0; r < 2; r++) {
        const int k = lane + 32 * r;
        if (k < P) {
            if (needA) dA[k] = va[r];
            if (needL && !CR) dL[k] = vl[r];
        }
    }
}

// First strict minimum over the (up to 2 per lane) candidates of each of M
// value sets, and whether the relative gap to the best candidate of a
// different colour is below `margin` (no division: gap < margin  <=>
// other - v < margin * den).  The M butterflies run interleaved (ACWDDF's
// four selections cost one reduction's latency).
template <int N, int M>
__device__ static inline void select64m(const double (&v)[M][2], int lane, const E64 *e, double margin, Cand (&c)[M],
                                        bool (&close)[M])
{
    const double INF = __longlong_as_double(0x7ff0000000000000LL);
#pragma unroll
    for (int m = 0; m < M; m++) {
        c[m] = {INF, 1 << 20};
        if (lane < N) c[m] = {v[m][0], lane};
        if (lane + 32 < N && v[m][1] < c[m].v) c[m] = {v[m][1], lane + 32};
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
        for (int m = 0; m < M; m++) {
            const double ov = __shfl_xor_sync(0xffffffffu, c[m].v, off);
            const int oi = __shfl_xor_sync(0xffffffffu, c[m].i, off);
            if (ov < c[m].v || (ov == c[m].v && oi < c[m].i)) { c[m].v = ov; c[m].i = oi; }
        }
    }
    double other[M];
#pragma unroll
    for (int m = 0; m < M; m++) {
        other[m] = INF;
#pragma unroll
        for (int s = 0; s < (N + 31) / 32; s++) {
            const int i = lane + 32 * s;
            // exact zeros tie exactly with an exact-zero winner (first index
            // wins in the reference too): not competitors for the margin
            if (i < N && !same_col(e[i], e[c[m].i]) && v[m][s] > 0.0 && v[m][s] < other[m]) other[m] = v[m][s];
        }
    }
#pragma unroll
    for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
        for (int m = 0; m < M; m++) other[m] = fmin(other[m], __shfl_xor_sync(0xffffffffu, other[m], off));
    }
#pragma unroll
    for (int m = 0; m < M; m++) {
        const double den = fmax(fabs(c[m].v), fabs(other[m]));
        close[m] = !isinf(other[m]) && (den == 0.0 || other[m] - c[m].v < margin * den);
    }
}

// Decide one window of N pixels from the pair tables (one warp; lane i and
// i + 32 hold candidates i, i + 32): returns the chosen index and sets
// *close when the smallest relative decision margin (argmin gaps, ACWDDF
// threshold margin) is below fp.cr_margin -- the exact route's cue for the
// correctly rounded pass.  Family, strategy and window are compile-time, so
// the aggregate loops unroll with all table loads independent.
template <int N, int FAM, int ST>
__device__ static inline int decide64(const E64 *e, const FParams &fp, int lane, const double *dA, const double *dL,
                                      bool *close)
{
    constexpr int dc = (N - 1) / 2;
    constexpr bool needA = FAM != FAM_VMF && FAM != FAM_CWVMF;
    constexpr bool needL = FAM != FAM_BVDF;
    double aA[2] = {0, 0}, aL[2] = {0, 0}, AD[2] = {0, 0}, LD[2] = {0, 0};
#pragma unroll
    for (int sl = 0; sl < (N + 31) / 32; sl++) {
        const int i = lane + 32 * sl;
        if (i >= N) continue;
        // agg[i] = self + sum over j != i in ascending j (_engine.py:239-281);
        // pair (i, j), j > i: row i of the upper triangle; (j, i), j < i: row j
        const int row_i = i * N - i * (i + 1) / 2 - i - 1;
        double a = fp.self_term, l = 0.0, ad = fp.self_term, ld = 0.0;
#pragma unroll
        for (int j = 0; j < N; j++) {
            const int k = j < i ? j * N - j * (j + 1) / 2 + i - j - 1 : (j > i ? row_i + j : 0);
            if (needA) {
                const double d = dA[k];
                if (j != i) a += d;
                if (j == dc && i != dc) ad = d;
            }
            if (needL) {
                const double d = dL[k];
                if (j != i) l += d;
                if (j == dc && i != dc) ld = d;
            }
        }
        aA[sl] = a; aL[sl] = l; AD[sl] = ad; LD[sl] = ld;
    }
    const double cm = fp.cr_margin;
    if constexpr (FAM == FAM_VMF || FAM == FAM_BVDF || FAM == FAM_DDF || FAM == FAM_CWVMF || FAM == FAM_CWDDF) {
        double v[1][2];
        for (int sl = 0; sl < 2; sl++) {
            if constexpr (FAM == FAM_VMF) v[0][sl] = aL[sl];
            else if constexpr (FAM == FAM_BVDF) v[0][sl] = aA[sl];
            else if constexpr (FAM == FAM_DDF) v[0][sl] = aA[sl] * aL[sl];
            else {
                // filters.py:296-337: weight-1 = n - 2k + 1 on the centre column
                const double w = (double)(N - 2 * fp.lam + 2 - 1);
                v[0][sl] = FAM == FAM_CWVMF ? aL[sl] + w * LD[sl] : (aA[sl] + w * AD[sl]) * (aL[sl] + w * LD[sl]);
            }
        }
        Cand c[1];
        bool cl[1];
        select64m<N, 1>(v, lane, e, cm, c, cl);
        *close = cl[0];
        return c[0].i;
    } else {
        // ACWDDF (_engine.py:451-487): the DDF pick and the centre-weighted
        // picks for k = lam .. lam + 2, weights w_k = n - 2k + 2 - 1
        double v[4][2];
        for (int sl = 0; sl < 2; sl++) {
            v[0][sl] = aA[sl] * aL[sl];
#pragma unroll
            for (int k = 0; k < 3; k++) {
                const double w = (double)(N - 2 * (fp.lam + k) + 2 - 1);
                v[1 + k][sl] = (aA[sl] + w * AD[sl]) * (aL[sl] + w * LD[sl]);
            }
        }
        Cand c[4];
        bool cl[4];
        select64m<N, 4>(v, lane, e, cm, c, cl);
        bool any = cl[1] || cl[2] || cl[3];
        double sv = 0.0;
#pragma unroll
        for (int k = 0; k < 3; k++) {
            double a = shfl_slot(AD, c[1 + k].i);
            const double l = shfl_slot(LD, c[1 + k].i);
            if (ST == ST_CHROMA) a = fp.slope * a + fp.intercept;
            sv += a * l;
        }
        const bool fires = sv > fp.threshold;
        if (fires) any = any || cl[0];
        const double den = fmax(fabs(sv), fabs(fp.threshold));
        any = any || den == 0.0 || fabs(sv - fp.threshold) < cm * den;
        *close = any;
        return fires ? c[0].i : dc;
    }
}

}  // namespace dfg
