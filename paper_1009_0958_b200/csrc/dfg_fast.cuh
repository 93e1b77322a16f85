// dfg_fast.cuh -- FP32/SFU decision kernel for the sliding-window directional
// vector filters (BVDF, DDF, ACWDDF, and VMF), templated on the window side,
// the family, the angular strategy and the Minkowski order.
//
// Reference path replaced: _engine.py:232-487 (pair row loops, aggregates,
// selection, ACWDDF switch) driven by filters.apply_filter (filters.py:379-433).
//
// Design (one CTA = TILE_H x 32 output pixels, one thread per output pixel):
//   stage 0  the (TILE_H + 2h) x (32 + 2h) input region (border policy applied
//            by index resolution) is staged in shared memory once, each pixel
//            normalised once: gray-mapped integer vector (+ 1/|x| for minimax,
//            1/sum for chromaticity), raw vector, packed colour.
//   stage 1  for each row offset du (0..s-1) the CTA evaluates every pair
//            distance D_(du,dv)(p) = d(p, p + (du,dv)) of the region ONCE into
//            shared-memory planes (2s-1 planes; angular and Minkowski packed as
//            float2 for DDF/ACWDDF): each unique pixel pair is computed once and
//            reused by all (s-|du|)(s-|dv|) windows containing it, instead of
//            the reference's n(n-1)/2 evaluations per window.
//   stage 2  each thread adds the plane values of its window's pairs into its
//            n register-resident aggregates (fully unrolled, compile-time
//            indices), stashing the centre column for ACWDDF.
//   stage 3  first-strict-minimum selection in window order (+ the three
//            centre-weighted argmins and the switching sum for ACWDDF); the
//            selected input pixel is written.  A pixel whose decision margin
//            is within the FP32 error budget is appended to the re-decision
//            list for the float64 kernel (dfg_fixup.cu).
//
// Numerics: the angular distances are computed from the exact integer
// channels: dot and |a x b|^2 in FP32 (exact / one rounding), the exact angle
// as atan2(|a x b|, a.b) via one MUFU.RSQ + a minimax atan polynomial, the
// minimax route's sqrt(1 - z) as |a x b| / (|a||b| sqrt(1 + z)) -- no
// catastrophic cancellation near parallel vectors, which is where a naive
// acosf(dot * rsqrt * rsqrt) loses ~1% of decisions.
#pragma once

#include <type_traits>

#include "dfg_f64.cuh"
#include "dfg_internal.cuh"

namespace dfg {

constexpr float kHalfPi = 1.57079632679489662f;

__device__ __forceinline__ float rsqrt_approx(float x)
{
    float r;
    asm("rsqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

__device__ __forceinline__ float sqrt_approx(float x)
{
    float r;
    asm("sqrt.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
    return r;
}

// atan(m) for m in [0, 1]: m * P(m^2), minimax in relative error, |err| < 2.1e-7
// (fit by weighted least squares, FP32 Horner verified in the fit script).
__device__ __forceinline__ float atan01(float m)
{
    const float t = m * m;
    float p = -0.0046935188584029675f;
    p = fmaf(p, t, 0.0242534838616848f);
    p = fmaf(p, t, -0.05948825553059578f);
    p = fmaf(p, t, 0.09914451837539673f);
    p = fmaf(p, t, -0.14019551873207092f);
    p = fmaf(p, t, 0.19969739019870758f);
    p = fmaf(p, t, -0.33331993222236633f);
    p = fmaf(p, t, 0.9999998807907104f);
    return m * p;
}

struct Cross {
    float dot, cc;
};

// dot and |a x b|^2 of integer vectors (components <= 255): dot and every
// cross component are exact in FP32; cc carries one rounding per term.
__device__ __forceinline__ Cross cross_dot(const float4 &a, const float4 &b)
{
    Cross r;
    r.dot = fmaf(a.z, b.z, fmaf(a.y, b.y, a.x * b.x));
    const float c1 = fmaf(a.y, b.z, -(a.z * b.y));
    const float c2 = fmaf(a.z, b.x, -(a.x * b.z));
    const float c3 = fmaf(a.x, b.y, -(a.y * b.x));
    r.cc = fmaf(c3, c3, fmaf(c2, c2, c1 * c1));
    return r;
}

// Exact route: acos(a.b / |a||b|) = atan2(|a x b|, a.b), one MUFU.  The
// max(.., 1e-30) makes the parallel (cc = 0 -> 0) and orthogonal
// (dot = 0 -> pi/2) cases fall out of the same formula (m = 0).
__device__ __forceinline__ float angle_exact(const float4 &a, const float4 &b)
{
    const Cross x = cross_dot(a, b);
    const float dd = x.dot * x.dot;
    const float R = rsqrt_approx(fmaxf(x.cc * dd, 1e-30f));  // 1 / (|a x b| * a.b)
    const float m = fminf(x.cc, dd) * R;                     // min(tan, cot) in [0, 1]
    const float at = atan01(m);
    return (x.cc > dd) ? (kHalfPi - at) : at;
}

// Float64 replica of the reference's minimax pair (_engine.py:134-147), used
// only when z is within the FP32 uncertainty of the 0.5 branch seam.
__device__ __forceinline__ float minimax_seam64(const float4 a, const float4 b, const KParams &kp)
{
    const double a1 = a.x, a2 = a.y, a3 = a.z, b1 = b.x, b2 = b.y, b3 = b.z;
    const double na = __dadd_rn(__dadd_rn(__dmul_rn(a1, a1), __dmul_rn(a2, a2)), __dmul_rn(a3, a3));
    const double nb = __dadd_rn(__dadd_rn(__dmul_rn(b1, b1), __dmul_rn(b2, b2)), __dmul_rn(b3, b3));
    const double rna = __ddiv_rn(1.0, __dsqrt_rn(na));
    const double rnb = __ddiv_rn(1.0, __dsqrt_rn(nb));
    const double dot = __dadd_rn(__dadd_rn(__dmul_rn(a1, b1), __dmul_rn(a2, b2)), __dmul_rn(a3, b3));
    double z = __dmul_rn(dot, __dmul_rn(rna, rnb));
    z = fmin(fmax(z, 0.0), 1.0);
    const double t = __dsqrt_rn(__dadd_rn(1.0, -z));
    const double *c = kp.ca64, *s = kp.cs64;
    double pa = __dadd_rn(c[3], __dmul_rn(z, c[4]));
    pa = __dadd_rn(c[2], __dmul_rn(z, pa));
    pa = __dadd_rn(c[1], __dmul_rn(z, pa));
    pa = __dadd_rn(c[0], __dmul_rn(z, pa));
    double ps = __dadd_rn(s[3], __dmul_rn(t, s[4]));
    ps = __dadd_rn(s[2], __dmul_rn(t, ps));
    ps = __dadd_rn(s[1], __dmul_rn(t, ps));
    ps = __dadd_rn(s[0], __dmul_rn(t, ps));
    return (float)((z >= 0.5) ? ps : pa);
}

// Minimax route (paper method 1): a.w = 1/|a|.  Branch-free over the two
// polynomials like the reference (_engine.py:144-145).
__device__ __forceinline__ float angle_minimax(const float4 &a, const float4 &b, const KParams &kp)
{
    const Cross x = cross_dot(a, b);
    const float rnab = a.w * b.w;
    float z = x.dot * rnab;
    z = fminf(fmaxf(z, 0.f), 1.f);
    // sqrt(1 - z) = |a x b| / (|a||b| sqrt(1 + z))   (Lagrange identity)
    const float R = rsqrt_approx(fmaxf(x.cc * (1.f + z), 1e-30f));
    const float t = x.cc * R * rnab;  // cc = 0 (parallel) -> 0
    float pa = fmaf(kp.ca[4], z, kp.ca[3]);
    pa = fmaf(pa, z, kp.ca[2]);
    pa = fmaf(pa, z, kp.ca[1]);
    pa = fmaf(pa, z, kp.ca[0]);
    float ps = fmaf(kp.cs[4], t, kp.cs[3]);
    ps = fmaf(ps, t, kp.cs[2]);
    ps = fmaf(ps, t, kp.cs[1]);
    ps = fmaf(ps, t, kp.cs[0]);
    float d = (z >= 0.5f) ? ps : pa;
    if (fabsf(z - 0.5f) < 4e-6f) d = minimax_seam64(a, b, kp);
    return d;
}

// Minkowski distance of integer-valued 3-vectors (exact differences).
template <int PC>
__device__ __forceinline__ float minkowski(const float4 &a, const float4 &b, const KParams &kp)
{
    const float d1 = a.x - b.x, d2 = a.y - b.y, d3 = a.z - b.z;
    if (PC == PC_2) return sqrt_approx(fmaf(d3, d3, fmaf(d2, d2, d1 * d1)));
    if (PC == PC_1) return fabsf(d1) + fabsf(d2) + fabsf(d3);
    const float s = __powf(fabsf(d1), kp.p) + __powf(fabsf(d2), kp.p) + __powf(fabsf(d3), kp.p);
    return __powf(s, kp.invp);
}

// Chromaticity route (paper method 2): L_p between x/sum(x).  Integer
// numerators a_k*s_b - b_k*s_a are exact; a.w = 1/s_a; sa/sb = channel sums
// of the gray-mapped vectors (zero vector -> (1,1,1), chroma 1/3 each).
template <int PC>
__device__ __forceinline__ float chroma(const float4 &a, float sa, const float4 &b, float sb,
                                        const KParams &kp)
{
    const float n1 = fmaf(a.x, sb, -(b.x * sa));
    const float n2 = fmaf(a.y, sb, -(b.y * sa));
    const float n3 = fmaf(a.z, sb, -(b.z * sa));
    const float r = a.w * b.w;
    if (PC == PC_2) return sqrt_approx(fmaf(n3, n3, fmaf(n2, n2, n1 * n1))) * r;
    if (PC == PC_1) return (fabsf(n1) + fabsf(n2) + fabsf(n3)) * r;
    const float s = __powf(fabsf(n1) * r, kp.p) + __powf(fabsf(n2) * r, kp.p) + __powf(fabsf(n3) * r, kp.p);
    return __powf(s, kp.invp);
}

// Compile-time loop: f(std::integral_constant<int, I>) for I in [B, E).
template <int B, int E, typename F>
__device__ __forceinline__ void static_for(F &&f)
{
    if constexpr (B < E) {
        f(std::integral_constant<int, B>{});
        static_for<B + 1, E>(f);
    }
}

// Gray-mapped angular vector of a raw record (zero vector -> (1,1,1),
// _engine.py:60-63); aux (1/|g| or 1/sum(g)) is carried through.
__device__ __forceinline__ float4 gray(const float4 &r)
{
    const bool z = (r.x + r.y + r.z) == 0.f;
    return make_float4(z ? 1.f : r.x, z ? 1.f : r.y, z ? 1.f : r.z, r.w);
}

// Tile geometry: 32 columns x TR thread-rows; each thread owns OPT vertically
// adjacent output pixels (register blocking of the aggregation stage).
template <int S, int FAM, int OPT, int TR>
struct Cfg {
    static constexpr int H = S / 2, N = S * S, DC = (N - 1) / 2;
    static constexpr bool NEED_A = FAM != FAM_VMF;
    static constexpr bool NEED_L = FAM == FAM_VMF || FAM == FAM_DDF || FAM == FAM_ACWDDF;
    static constexpr bool BOTH = NEED_A && NEED_L;
    static constexpr int TW = 32, NT = TR * TW, TH = TR * OPT;
    static constexpr int RH = TH + 2 * H, RW = TW + 2 * H, RN = RH * RW;
    static constexpr int RN4 = (RN + 3) & ~3;
    static constexpr int NDV = 2 * S - 1;
    static constexpr int PADC = S - 1, RWS = RW + 2 * PADC;  // record rows padded for unclamped dv reads
    static constexpr int RECN = RH * RWS;
    using DT = typename std::conditional<BOTH, float2, float>::type;
    static constexpr size_t kSmem = (size_t)RECN * 16 + (size_t)RN4 * 4 + (size_t)NDV * RN * sizeof(DT);
};

__device__ __forceinline__ float dval_a(float v) { return v; }
__device__ __forceinline__ float dval_a(float2 v) { return v.x; }
__device__ __forceinline__ float dval_l(float v) { return v; }
__device__ __forceinline__ float dval_l(float2 v) { return v.y; }

// One-pass first-strict-minimum with "best competitor of a different colour"
// tracking.  Invariant: v2 = min over scanned candidates whose colour differs
// from the current winner's (the candidates that could change the output).
struct Sel {
    float v1, e1, v2, e2;
    int i1;
    uint32_t k1;
    float xa, xl;  // payload of the winner (ACWDDF centre distances)
    __device__ __forceinline__ void init(float v, float e, uint32_t k, float pa, float pl)
    {
        v1 = v; e1 = e; v2 = __int_as_float(0x7f800000); e2 = 0.f; i1 = 0; k1 = k; xa = pa; xl = pl;
    }
    __device__ __forceinline__ void add(float v, float e, int i, uint32_t k, float pa, float pl)
    {
        if (v < v1) {
            if (k != k1) { v2 = v1; e2 = e1; }
            v1 = v; e1 = e; i1 = i; k1 = k; xa = pa; xl = pl;
        } else if (k != k1 && v < v2) {
            v2 = v; e2 = e;
        }
    }
    // true when the FP32 order of winner and competitor is not certain
    __device__ __forceinline__ bool doubtful() const { return (v2 - v1) <= (e1 + e2); }
};

// Distance value(s) of one pair; p/q are raw records, pg/qg gray-mapped.
template <int FAM, int ST, int PC, typename DT>
__device__ __forceinline__ DT pair_value(const float4 &p, const float4 &pg, const float4 &q, const float4 &qg,
                                         const KParams &kp)
{
    constexpr bool NA = FAM != FAM_VMF;
    constexpr bool NL = FAM == FAM_VMF || FAM == FAM_DDF || FAM == FAM_ACWDDF;
    float da = 0.f, dl = 0.f;
    if (NA) {
        if (ST == ST_EXACT) da = angle_exact(pg, qg);
        else if (ST == ST_MINIMAX) da = angle_minimax(pg, qg, kp);
        else da = chroma<PC>(pg, pg.x + pg.y + pg.z, qg, qg.x + qg.y + qg.z, kp);
    }
    if (NL) dl = minkowski<PC>(p, q, kp);
    if constexpr (NA && NL) return make_float2(da, dl);
    else if constexpr (NA) return da;
    else return dl;
}

template <int S, int FAM, int ST, int PC, int OPT, int TR, int MINB>
__global__ void __launch_bounds__(TR * 32, MINB)
dfg_fast_kernel(const uint8_t *__restrict__ in, uint8_t *__restrict__ out, const KParams kp)
{
    using C = Cfg<S, FAM, OPT, TR>;
    using DT = typename C::DT;
    constexpr int H = C::H, N = C::N, DC = C::DC, RW = C::RW, RH = C::RH, RN = C::RN, NT = C::NT, TH = C::TH;
    constexpr bool ACW = FAM == FAM_ACWDDF;

    extern __shared__ __align__(16) unsigned char smem_raw[];
    float4 *sR = reinterpret_cast<float4 *>(smem_raw);           // raw channels + aux (padded rows)
    uint32_t *sK = reinterpret_cast<uint32_t *>(sR + C::RECN);   // packed colour
    DT *sD = reinterpret_cast<DT *>(sK + C::RN4);                // pair-distance planes
    constexpr int RWS = C::RWS, PADC = C::PADC;

    __shared__ unsigned s_nflag;          // this CTA's pixels needing float64 re-decision
    __shared__ uint16_t s_flag[TH * 32];  // (window top row << 5) | column
    __shared__ int s_b;
    __shared__ double s_m;

    const int tid = threadIdx.x;
    const int tx = tid & 31, ty = tid >> 5;
    const int tile_x0 = blockIdx.x * 32, tile_y0 = blockIdx.y * TH;
    const int frame = blockIdx.z;
    const uint8_t *fin = in + (long long)frame * kp.in_fstride;
    if (tid == 0) s_nflag = 0;

    // ---- stage 0: region staging + per-pixel normalisation ----------------
    for (int idx = tid; idx < RN; idx += NT) {
        const int ry = idx / RW, rx = idx - ry * RW;
        int gy = resolve_idx(kp.out_row0 + tile_y0 + ry - H, kp.global_H, kp.border) - kp.in_row0;
        gy = min(max(gy, 0), kp.in_rows - 1);
        const int gx = resolve_idx(tile_x0 + rx - H, kp.W, kp.border);
        const uint8_t *px = fin + (long long)gy * kp.in_pitch + gx * 3;
        const uint32_t r8 = px[0], g8 = px[1], b8 = px[2];
        const float4 raw = make_float4((float)r8, (float)g8, (float)b8, 0.f);
        const float4 g = gray(raw);
        float aux = 0.f;
        if (ST == ST_MINIMAX) aux = rsqrtf(fmaf(g.z, g.z, fmaf(g.y, g.y, g.x * g.x)));
        if (ST == ST_CHROMA) aux = __frcp_rn(g.x + g.y + g.z);
        sR[ry * RWS + PADC + rx] = make_float4(raw.x, raw.y, raw.z, aux);
        sK[idx] = r8 | (g8 << 8) | (b8 << 16);
    }
    for (int idx = tid; idx < RH * 2 * PADC; idx += NT) {  // pad columns (read, never used)
        const int ry = idx / (2 * PADC), c = idx - ry * 2 * PADC;
        sR[ry * RWS + (c < PADC ? c : RW + c)] = make_float4(1.f, 1.f, 1.f, 1.f);
    }

    float aA[OPT][C::NEED_A ? N : 1], aL[OPT][C::NEED_L ? N : 1];
    float AD[OPT][ACW ? N : 1], LD[OPT][ACW ? N : 1];
#pragma unroll
    for (int o = 0; o < OPT; o++) {
#pragma unroll
        for (int i = 0; i < N; i++) {
            if (C::NEED_A) aA[o][i] = kp.self_term;
            if (C::NEED_L) aL[o][i] = 0.f;
        }
        if (ACW) {
            AD[o][DC] = kp.self_term;
            LD[o][DC] = 0.f;
        }
    }
    __syncthreads();

    static_for<0, S>([&](auto du_c) {
        constexpr int du = decltype(du_c)::value;
        constexpr int dv0 = (du == 0) ? 1 : -(S - 1);
        constexpr int ndv = S - dv0;
        // ---- stage 1: pair distances of the region, each pair once --------
        // thread item = pixel p; p's record stays in registers across dv;
        // q reads are at constant offsets (padded rows, no clamping)
        constexpr int items = (RH - du) * RW;
        for (int it = tid; it < items; it += NT) {
            const int py = it / RW, px = it - py * RW;
            const float4 *prow = sR + py * RWS + PADC + px;
            const float4 pr = prow[0];
            const float4 pg = gray(pr);
            const float4 *qrow = prow + du * RWS + dv0;
#pragma unroll
            for (int k = 0; k < ndv; k++) {
                const float4 qr = qrow[k];
                sD[k * RN + it] = pair_value<FAM, ST, PC, DT>(pr, pg, qr, gray(qr), kp);
            }
        }
        __syncthreads();
        // ---- stage 2: window aggregation from the planes ------------------
        // rows r = 0 .. S-du-1+OPT-1 below the thread's first output row feed
        // output o's window row u = r - o.
        const DT *dbase = sD + (ty * OPT) * RW + tx;
        static_for<0, ndv>([&](auto k_c) {
            constexpr int k = decltype(k_c)::value;
            constexpr int dv = dv0 + k;
            constexpr int vlo = dv < 0 ? -dv : 0, vhi = dv > 0 ? S - dv : S;
#pragma unroll
            for (int r = 0; r < S - du + OPT - 1; r++) {
#pragma unroll
                for (int v = vlo; v < vhi; v++) {
                    const DT val = dbase[k * RN + r * RW + v];
#pragma unroll
                    for (int o = 0; o < OPT; o++) {
                        const int u = r - o;
                        if (u < 0 || u + du >= S) continue;
                        const int i = u * S + v, j = (u + du) * S + v + dv;
                        if (C::NEED_A) {
                            const float x = dval_a(val);
                            aA[o][i] += x;
                            aA[o][j] += x;
                            if (ACW) {
                                if (j == DC) AD[o][i] = x;
                                else if (i == DC) AD[o][j] = x;
                            }
                        }
                        if (C::NEED_L) {
                            const float x = dval_l(val);
                            aL[o][i] += x;
                            aL[o][j] += x;
                            if (ACW) {
                                if (j == DC) LD[o][i] = x;
                                else if (i == DC) LD[o][j] = x;
                            }
                        }
                    }
                }
            }
        });
        __syncthreads();
    });

    // ---- stage 3: selection ------------------------------------------------
    const float er = kp.er, ea = kp.ea;
    const int ox = tile_x0 + tx;
#pragma unroll
    for (int o = 0; o < OPT; o++) {
        const int ry0 = ty * OPT + o;  // window top row in region coordinates
        const int oy = tile_y0 + ry0;
        const bool valid = (oy < kp.out_rows) && (ox < kp.W);
        int b;
        bool doubt;
        if (ACW) {
            Sel sd, s0, s1, s2;
            const float w0 = kp.w[0], w1 = kp.w[1], w2 = kp.w[2];
#pragma unroll
            for (int i = 0; i < N; i++) {
                const uint32_t col = sK[(ry0 + i / S) * RW + tx + i % S];
                const float a = aA[o][i], l = aL[o][i];
                const float pd = a * l;
                const float a0 = fmaf(w0, AD[o][i], a), l0 = fmaf(w0, LD[o][i], l);
                const float a1 = fmaf(w1, AD[o][i], a), l1 = fmaf(w1, LD[o][i], l);
                const float a2 = fmaf(w2, AD[o][i], a), l2 = fmaf(w2, LD[o][i], l);
                const float p0 = a0 * l0, p1 = a1 * l1, p2 = a2 * l2;
                const float ed = 2.f * er * fabsf(pd) + 2.f * ea * l;
                const float e0 = 2.f * er * fabsf(p0) + 2.f * ea * l0;
                const float e1 = 2.f * er * fabsf(p1) + 2.f * ea * l1;
                const float e2 = 2.f * er * fabsf(p2) + 2.f * ea * l2;
                if (i == 0) {
                    sd.init(pd, ed, col, 0.f, 0.f);
                    s0.init(p0, e0, col, AD[o][i], LD[o][i]);
                    s1.init(p1, e1, col, AD[o][i], LD[o][i]);
                    s2.init(p2, e2, col, AD[o][i], LD[o][i]);
                } else {
                    sd.add(pd, ed, i, col, 0.f, 0.f);
                    s0.add(p0, e0, i, col, AD[o][i], LD[o][i]);
                    s1.add(p1, e1, i, col, AD[o][i], LD[o][i]);
                    s2.add(p2, e2, i, col, AD[o][i], LD[o][i]);
                }
            }
            float a = s0.xa;
            if (ST == ST_CHROMA) a = fmaf(kp.slope, a, kp.intercept);
            float sv = a * s0.xl;
            a = s1.xa;
            if (ST == ST_CHROMA) a = fmaf(kp.slope, a, kp.intercept);
            sv = fmaf(a, s1.xl, sv);
            a = s2.xa;
            if (ST == ST_CHROMA) a = fmaf(kp.slope, a, kp.intercept);
            sv = fmaf(a, s2.xl, sv);
            const float ld_sum = s0.xl + s1.xl + s2.xl;
            const float es = 4.f * er * fmaxf(fabsf(sv), kp.threshold) +
                             2.f * kp.ea_pair * (ST == ST_CHROMA ? kp.slope : 1.f) * ld_sum + 1e-6f;
            const bool fires = sv > kp.threshold;
            b = fires ? sd.i1 : DC;
            doubt = s0.doubtful() || s1.doubtful() || s2.doubtful() || fabsf(sv - kp.threshold) <= es ||
                    (fires && sd.doubtful());
        } else {
            Sel sl;
#pragma unroll
            for (int i = 0; i < N; i++) {
                const uint32_t col = sK[(ry0 + i / S) * RW + tx + i % S];
                float v, e;
                if (FAM == FAM_BVDF) {
                    v = aA[o][i];
                    e = er * fabsf(v) + ea;
                } else if (FAM == FAM_VMF) {
                    v = aL[o][i];
                    e = er * v;
                } else {
                    v = aA[o][i] * aL[o][i];
                    e = 2.f * er * fabsf(v) + 2.f * ea * aL[o][i];
                }
                if (i == 0) sl.init(v, e, col, 0.f, 0.f);
                else sl.add(v, e, i, col, 0.f, 0.f);
            }
            b = sl.i1;
            doubt = sl.doubtful();
        }

        if (kp.dbg != nullptr && valid) {
            float *d = kp.dbg + ((long long)frame * kp.out_rows * kp.W + (long long)oy * kp.W + ox) * (2 * N);
#pragma unroll
            for (int i = 0; i < N; i++) {
                d[i] = C::NEED_A ? aA[o][i] : 0.f;
                d[N + i] = C::NEED_L ? aL[o][i] : 0.f;
            }
        }

        if (valid) {
            const uint32_t col = sK[(ry0 + b / S) * RW + tx + b % S];
            uint8_t *op = out + (long long)frame * kp.out_fstride + (long long)oy * kp.out_pitch + ox * 3;
            op[0] = (uint8_t)(col & 0xff);
            op[1] = (uint8_t)((col >> 8) & 0xff);
            op[2] = (uint8_t)((col >> 16) & 0xff);
        }

        if (valid && doubt) {
            const unsigned slot = atomicAdd(&s_nflag, 1u);
            s_flag[slot] = (uint16_t)((ry0 << 5) | tx);
        }
    }

    // ---- stage 4: float64 re-decision of this CTA's doubtful pixels ---------
    // All threads of the CTA evaluate the window's pair table (the planes'
    // shared memory is free now), one warp aggregates and selects; the
    // work overlaps with other CTAs' FP32 stages on the same SM.
    __syncthreads();
    const unsigned nflag = s_nflag;
    if (nflag == 0) return;
    if (tid == 0) atomicAdd(kp.flag_count, nflag);
    constexpr int P = N * (N - 1) / 2;
    static_assert(N * sizeof(E64) + 2 * P * sizeof(double) <= C::NDV * C::RN * sizeof(DT),
                  "float64 scratch must fit in the plane buffer");
    E64 *e64 = reinterpret_cast<E64 *>(sD);
    double *dA = reinterpret_cast<double *>(e64 + N);
    double *dL = dA + P;
    const FParams &fp = kp.fp;
    for (unsigned f = 0; f < nflag; f++) {
        const int code = s_flag[f];
        const int ry0 = code >> 5, cx = code & 31;
        for (int i = tid; i < N; i += NT) prep64(sR[(ry0 + i / S) * RWS + PADC + cx + i % S], ST, e64[i]);
        __syncthreads();
        pair_tables<false>(e64, fp, tid, NT, dA, dL, C::NEED_A, C::NEED_L);
        __syncthreads();
        if (ty == 0) {
            double m;
            const int bb = decide64(e64, fp, tx, dA, dL, &m);
            if (tx == 0) { s_b = bb; s_m = m; }
        }
        __syncthreads();
        if (ST == ST_EXACT && C::NEED_A && s_m < fp.cr_margin) {
            // pass 2: correctly rounded arccos (dfg_f64.cuh)
            if (tid == 0) atomicAdd(kp.flag_count + 1, 1u);
            pair_tables<true>(e64, fp, tid, NT, dA, dL, C::NEED_A, C::NEED_L);
            __syncthreads();
            if (ty == 0) {
                double m;
                const int bb = decide64(e64, fp, tx, dA, dL, &m);
                if (tx == 0) s_b = bb;
            }
            __syncthreads();
        }
        if (tid == 0) {
            const int bb = s_b;
            const uint32_t col = sK[(ry0 + bb / S) * RW + cx + bb % S];
            uint8_t *op = out + (long long)frame * kp.out_fstride + (long long)(tile_y0 + ry0) * kp.out_pitch +
                          (tile_x0 + cx) * 3;
            op[0] = (uint8_t)(col & 0xff);
            op[1] = (uint8_t)((col >> 8) & 0xff);
            op[2] = (uint8_t)((col >> 16) & 0xff);
        }
        __syncthreads();
    }
}

// Per (window, family) launch shape: OPT outputs per thread (register
// blocking), TR thread-rows per CTA, MINB CTAs per SM.  Register-resident
// state per output is n (BVDF/VMF), 2n (DDF) or 4n (ACWDDF) floats.
template <int S, int FAM>
struct Shape {
    static constexpr int AGG = (FAM == FAM_ACWDDF ? 4 : (FAM == FAM_DDF ? 2 : 1)) * S * S;
    static constexpr int OPT = (S >= 5 && 2 * AGG + 32 <= 131) ? 2 : 1;
    static constexpr int NEED = OPT * AGG + 32;  // registers per thread, estimated
    static constexpr int TR = (NEED > 128 && NEED <= 131) ? 16 : 8;
    static constexpr int MINB = NEED <= 64 ? 4 : (NEED <= 128 ? 2 : 1);
};

template <int S, int FAM, int ST, int PC>
cudaError_t launch_fast(cudaStream_t st, const uint8_t *in, uint8_t *out, const KParams &kp)
{
    using SH = Shape<S, FAM>;
    using C = Cfg<S, FAM, SH::OPT, SH::TR>;
    auto kern = dfg_fast_kernel<S, FAM, ST, PC, SH::OPT, SH::TR, SH::MINB>;
    static unsigned long long configured = 0;  // per-device bit, idempotent
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(configured & (1ull << (dev & 63)))) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
        if (e != cudaSuccess) return e;
        configured |= 1ull << (dev & 63);
    }
    dim3 grid((kp.W + 31) / 32, (kp.out_rows + C::TH - 1) / C::TH, kp.n_frames);
    kern<<<grid, C::NT, C::kSmem, st>>>(in, out, kp);
    return cudaGetLastError();
}

}  // namespace dfg

// Family launcher bodies: dispatch strategy x Minkowski order, instantiating
// only the combinations a family can use.
#define DFG_P_SWITCH(S, FAM, ST)                                                    \
    switch (pcode) {                                                                \
    case dfg::PC_2: return dfg::launch_fast<S, FAM, ST, dfg::PC_2>(st, in, out, kp);  \
    case dfg::PC_1: return dfg::launch_fast<S, FAM, ST, dfg::PC_1>(st, in, out, kp);  \
    default: return dfg::launch_fast<S, FAM, ST, dfg::PC_GEN>(st, in, out, kp);       \
    }

#define DFG_DEFINE_LAUNCH_VMF(S)                                                    \
    cudaError_t dfg_launch_s##S##_vmf(int, int pcode, cudaStream_t st,              \
                                      const uint8_t *in, uint8_t *out,              \
                                      const dfg::KParams &kp)                       \
    {                                                                               \
        DFG_P_SWITCH(S, dfg::FAM_VMF, dfg::ST_EXACT)                                \
    }

#define DFG_DEFINE_LAUNCH_BVDF(S)                                                   \
    cudaError_t dfg_launch_s##S##_bvdf(int strategy, int pcode, cudaStream_t st,    \
                                       const uint8_t *in, uint8_t *out,             \
                                       const dfg::KParams &kp)                      \
    {                                                                               \
        if (strategy == dfg::ST_EXACT)                                              \
            return dfg::launch_fast<S, dfg::FAM_BVDF, dfg::ST_EXACT, dfg::PC_2>(st, in, out, kp); \
        if (strategy == dfg::ST_MINIMAX)                                            \
            return dfg::launch_fast<S, dfg::FAM_BVDF, dfg::ST_MINIMAX, dfg::PC_2>(st, in, out, kp); \
        DFG_P_SWITCH(S, dfg::FAM_BVDF, dfg::ST_CHROMA)                              \
    }

#define DFG_DEFINE_LAUNCH_PAIRED(S, FAM, FAMNAME)                                   \
    cudaError_t dfg_launch_s##S##_##FAMNAME(int strategy, int pcode, cudaStream_t st, \
                                            const uint8_t *in, uint8_t *out,        \
                                            const dfg::KParams &kp)                 \
    {                                                                               \
        if (strategy == dfg::ST_EXACT) { DFG_P_SWITCH(S, FAM, dfg::ST_EXACT) }      \
        if (strategy == dfg::ST_MINIMAX) { DFG_P_SWITCH(S, FAM, dfg::ST_MINIMAX) }  \
        DFG_P_SWITCH(S, FAM, dfg::ST_CHROMA)                                        \
    }
