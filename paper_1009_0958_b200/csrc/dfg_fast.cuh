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

#include <cuda.h>

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

// ---------------- packed f32x2 arithmetic (sm_100a FADD2/FMUL2/FFMA2) -------
// Two pairs are evaluated per instruction: lanes (lo, hi) = pairs (k, k+1).
struct P2 {
    unsigned long long v;
};
__device__ __forceinline__ P2 pk2(float lo, float hi)
{
    P2 r;
    asm("mov.b64 %0, {%1,%2};" : "=l"(r.v) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ P2 bc2(float x) { return pk2(x, x); }  // broadcast (FFMA2 .F32 operand)
__device__ __forceinline__ float lo2(P2 a)
{
    float l, h;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(l), "=f"(h) : "l"(a.v));
    return l;
}
__device__ __forceinline__ float hi2(P2 a)
{
    float l, h;
    asm("mov.b64 {%0,%1}, %2;" : "=f"(l), "=f"(h) : "l"(a.v));
    return h;
}
__device__ __forceinline__ P2 add2(P2 a, P2 b)
{
    P2 r;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
__device__ __forceinline__ P2 sub2(P2 a, P2 b)
{
    P2 r;
    asm("sub.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
__device__ __forceinline__ P2 mul2(P2 a, P2 b)
{
    P2 r;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r.v) : "l"(a.v), "l"(b.v));
    return r;
}
__device__ __forceinline__ P2 fma2(P2 a, P2 b, P2 c)
{
    P2 r;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r.v) : "l"(a.v), "l"(b.v), "l"(c.v));
    return r;
}

// Whole 16-byte shared-memory loads.  The compiler would otherwise split a
// record load into the two scalars it uses -- 4-byte accesses at a 16-byte
// lane stride, a 4-way bank conflict.
__device__ __forceinline__ float4 lds_f4(const float4 *p)
{
    float4 v;
    const unsigned a = (unsigned)__cvta_generic_to_shared(p);
    asm("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "r"(a));
    return v;
}
__device__ __forceinline__ ulonglong2 lds_u2(const void *p)
{
    ulonglong2 v;
    const unsigned a = (unsigned)__cvta_generic_to_shared(p);
    asm("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "r"(a));
    return v;
}

// Ordered variant: the plain helpers above are pure functions of their
// address to the compiler, which may hoist or merge them across barriers when
// the address is loop-invariant (the row sweep's compile-time ring slots);
// this one stays where it is written.
__device__ __forceinline__ ulonglong2 lds_u2_ordered(const void *p)
{
    ulonglong2 v;
    const unsigned a = (unsigned)__cvta_generic_to_shared(p);
    asm volatile("ld.shared.v2.u64 {%0, %1}, [%2];" : "=l"(v.x), "=l"(v.y) : "r"(a) : "memory");
    return v;
}

// Scalar pixel p (gray-mapped g, aux) against a packed pixel pair Q = (q, q+1).
struct Pix {
    float x, y, z, aux;
};
struct Pair2 {
    P2 x, y, z, aux;
};

// packed dot and |p x q|^2 (exact dot / cross components, as cross_dot)
__device__ __forceinline__ void cross_dot2(const Pix &p, const Pair2 &q, P2 &dot, P2 &cc)
{
    dot = fma2(bc2(p.z), q.z, fma2(bc2(p.y), q.y, mul2(bc2(p.x), q.x)));
    const P2 c1 = fma2(bc2(p.y), q.z, mul2(bc2(-p.z), q.y));
    const P2 c2 = fma2(bc2(p.z), q.x, mul2(bc2(-p.x), q.z));
    const P2 c3 = fma2(bc2(p.x), q.y, mul2(bc2(-p.y), q.x));
    cc = fma2(c3, c3, fma2(c2, c2, mul2(c1, c1)));
}

__device__ __forceinline__ P2 atan01_2(P2 m)
{
    const P2 t = mul2(m, m);
    P2 q = fma2(bc2(-0.0046935188584029675f), t, bc2(0.0242534838616848f));
    q = fma2(q, t, bc2(-0.05948825553059578f));
    q = fma2(q, t, bc2(0.09914451837539673f));
    q = fma2(q, t, bc2(-0.14019551873207092f));
    q = fma2(q, t, bc2(0.19969739019870758f));
    q = fma2(q, t, bc2(-0.33331993222236633f));
    q = fma2(q, t, bc2(0.9999998807907104f));
    return mul2(m, q);
}

// exact route, two pairs (angle_exact per lane)
__device__ __forceinline__ P2 angle_exact2(const Pix &p, const Pair2 &q)
{
    P2 dot, cc;
    cross_dot2(p, q, dot, cc);
    const P2 dd = mul2(dot, dot);
    const P2 P = mul2(cc, dd);
    const float c0 = lo2(cc), c1 = hi2(cc), d0 = lo2(dd), d1 = hi2(dd);
    const P2 m = mul2(pk2(fminf(c0, d0), fminf(c1, d1)),
                      pk2(rsqrt_approx(fmaxf(lo2(P), 1e-30f)), rsqrt_approx(fmaxf(hi2(P), 1e-30f))));
    const P2 at = atan01_2(m);
    const P2 alt = sub2(bc2(kHalfPi), at);
    return pk2(c0 > d0 ? lo2(alt) : lo2(at), c1 > d1 ? hi2(alt) : hi2(at));
}

// 2 atan(t) for t in [0, 1]: atan01's polynomial with every coefficient
// doubled (binary scaling: bit-identical to 2 * atan01(t)).
__device__ __forceinline__ P2 atan01x2_2(P2 m)
{
    const P2 t = mul2(m, m);
    P2 q = fma2(bc2(2.f * -0.0046935188584029675f), t, bc2(2.f * 0.0242534838616848f));
    q = fma2(q, t, bc2(2.f * -0.05948825553059578f));
    q = fma2(q, t, bc2(2.f * 0.09914451837539673f));
    q = fma2(q, t, bc2(2.f * -0.14019551873207092f));
    q = fma2(q, t, bc2(2.f * 0.19969739019870758f));
    q = fma2(q, t, bc2(2.f * -0.33331993222236633f));
    q = fma2(q, t, bc2(2.f * 0.9999998807907104f));
    return mul2(m, q);
}

// Exact route by the half-angle identity, two pairs: theta = 2 atan(t) with
// t = tan(theta / 2) = |a x b| / (|a||b| + a.b) in [0, 1] for non-negative
// vectors (theta <= pi/2), evaluated as t = cc * rsqrt(cc * den^2): one MUFU,
// no range reduction and no branch select.  aux = |x| (IEEE sqrt of the
// exact integer norm; the zero-pixel flag is its sign bit, cleared under ZC).
template <bool ZC>
__device__ __forceinline__ P2 angle_half2(const Pix &p, const Pair2 &q)
{
    P2 dot, cc;
    cross_dot2(p, q, dot, cc);
    float pa = p.aux;
    P2 qa = q.aux;
    if constexpr (ZC) {
        pa = fabsf(pa);
        qa = pk2(fabsf(lo2(qa)), fabsf(hi2(qa)));
    }
    const P2 den = fma2(bc2(pa), qa, dot);  // |a||b| + a.b, one rounding
    const P2 P = mul2(cc, mul2(den, den));
    // P is 0 (parallel: cc = 0) or >= 1 (cc and den^2 are >= 1 for nonzero
    // integer vectors), so P + 1e-30 is P exactly or 1e-30: max(P, 1e-30)
    // in one packed add
    const P2 Pt = add2(P, bc2(1e-30f));
    const P2 R = pk2(rsqrt_approx(lo2(Pt)), rsqrt_approx(hi2(Pt)));
    return atan01x2_2(mul2(cc, R));  // cc = 0 (parallel) -> exactly 0
}

// minimax route, two pairs (angle_minimax per lane, incl. the seam check)
__device__ __forceinline__ P2 angle_minimax2(const Pix &p, const Pair2 &q, const KParams &kp)
{
    P2 dot, cc;
    cross_dot2(p, q, dot, cc);
    const P2 rnab = mul2(bc2(p.aux), q.aux);
    const P2 zr = mul2(dot, rnab);
    const float z0 = fminf(lo2(zr), 1.f), z1 = fminf(hi2(zr), 1.f);  // dot >= 0: only the upper clamp bites
    const P2 z = pk2(z0, z1);
    const P2 u = mul2(cc, add2(z, bc2(1.f)));
    const P2 ut = add2(u, bc2(1e-30f));  // u = 0 or u >= cc >= 1: max(u, 1e-30) exactly (angle_half2)
    const P2 R = pk2(rsqrt_approx(lo2(ut)), rsqrt_approx(hi2(ut)));
    const P2 t = mul2(mul2(cc, R), rnab);
    P2 pa = fma2(bc2(kp.ca[4]), z, bc2(kp.ca[3]));
    pa = fma2(pa, z, bc2(kp.ca[2]));
    pa = fma2(pa, z, bc2(kp.ca[1]));
    pa = fma2(pa, z, bc2(kp.ca[0]));
    P2 ps = fma2(bc2(kp.cs[4]), t, bc2(kp.cs[3]));
    ps = fma2(ps, t, bc2(kp.cs[2]));
    ps = fma2(ps, t, bc2(kp.cs[1]));
    ps = fma2(ps, t, bc2(kp.cs[0]));
    float r0 = z0 >= 0.5f ? lo2(ps) : lo2(pa);
    float r1 = z1 >= 0.5f ? hi2(ps) : hi2(pa);
    if (fabsf(z0 - 0.5f) < 4e-6f || fabsf(z1 - 0.5f) < 4e-6f) {  // rare: decide the branch like the reference
        const float4 a = make_float4(p.x, p.y, p.z, p.aux);
        if (fabsf(z0 - 0.5f) < 4e-6f) r0 = minimax_seam64(a, make_float4(lo2(q.x), lo2(q.y), lo2(q.z), 0.f), kp);
        if (fabsf(z1 - 0.5f) < 4e-6f) r1 = minimax_seam64(a, make_float4(hi2(q.x), hi2(q.y), hi2(q.z), 0.f), kp);
    }
    return pk2(r0, r1);
}

// chromaticity route (p = 2), two pairs
__device__ __forceinline__ P2 chroma2_l2(const Pix &p, const Pair2 &q)
{
    const float sp = p.x + p.y + p.z;
    const P2 sq = add2(q.x, add2(q.y, q.z));
    const P2 n1 = fma2(bc2(p.x), sq, mul2(bc2(-sp), q.x));
    const P2 n2 = fma2(bc2(p.y), sq, mul2(bc2(-sp), q.y));
    const P2 n3 = fma2(bc2(p.z), sq, mul2(bc2(-sp), q.z));
    const P2 ss = fma2(n3, n3, fma2(n2, n2, mul2(n1, n1)));
    return mul2(pk2(sqrt_approx(lo2(ss)), sqrt_approx(hi2(ss))), mul2(bc2(p.aux), q.aux));
}

// Minkowski p = 2 on the gray-mapped values (exact for nonzero pixels; the
// caller repairs pairs touching a zero pixel)
__device__ __forceinline__ P2 l2_2(const Pix &p, const Pair2 &q)
{
    const P2 d1 = sub2(bc2(p.x), q.x), d2 = sub2(bc2(p.y), q.y), d3 = sub2(bc2(p.z), q.z);
    const P2 ss = fma2(d3, d3, fma2(d2, d2, mul2(d1, d1)));
    return pk2(sqrt_approx(lo2(ss)), sqrt_approx(hi2(ss)));
}

// Per-pixel aux word of the gray-mapped vector g and the zero-pixel flag it
// carries: exact route |g| (IEEE sqrt of the exact integer norm) with the
// flag in the sign bit -- set only when the Minkowski term needs it (FLAG),
// whose zero-check (ZC) pair path then takes |aux|; minimax 1/|g| and
// chromaticity 1/sum(g) with the flag in bit 0 (1 ulp of aux, inside the
// error budget).
template <int ST>
__device__ __forceinline__ uint32_t zbit()
{
    return ST == ST_EXACT ? 0x80000000u : 1u;
}
template <int ST, bool FLAG>
__device__ __forceinline__ float encode_aux(float gx, float gy, float gz, bool zero)
{
    const float n2 = fmaf(gz, gz, fmaf(gy, gy, gx * gx));  // exact integer
    if (ST == ST_EXACT) {
        const float a = __fsqrt_rn(n2);
        return (FLAG && zero) ? -a : a;
    }
    float aux = 0.f;
    if (ST == ST_MINIMAX) aux = rsqrtf(n2);
    if (ST == ST_CHROMA) aux = __frcp_rn(gx + gy + gz);
    return __uint_as_float((__float_as_uint(aux) & ~1u) | (zero ? 1u : 0u));
}
template <int ST>
__device__ __forceinline__ bool zflag(float aux)
{
    return (__float_as_uint(aux) & zbit<ST>()) != 0u;
}
template <int ST>
__device__ __forceinline__ float4 rawrec(float x, float y, float z, float aux)
{
    const bool zr = zflag<ST>(aux);
    return make_float4(zr ? 0.f : x, zr ? 0.f : y, zr ? 0.f : z, aux);
}

// Tile geometry: 32 columns x TR thread-rows; each thread owns OPT vertically
// adjacent output pixels (register blocking of the aggregation stage).
// Records: two arrays of 16-byte elements, element c of a padded row holding
// the pixel pair (c, c+1): A = {gx_c, gx_c+1, gy_c, gy_c+1}, B = {gz_c, gz_c+1,
// aux_c, aux_c+1}, so a pair of horizontally adjacent partners loads with two
// conflict-free LDS.128 straight into f32x2 operands.
template <int S, int FAM, int OPT, int TR>
struct Cfg {
    static constexpr int H = S / 2, N = S * S, DC = (N - 1) / 2;
    static constexpr bool NEED_A = FamT<FAM>::A;
    static constexpr bool NEED_L = FamT<FAM>::L;
    static constexpr bool BOTH = NEED_A && NEED_L;
    static constexpr bool CEN = FamT<FAM>::CEN;
    static constexpr int TW = 32, NT = TR * TW, TH = TR * OPT;
    static constexpr int RH = TH + 2 * H, RW = TW + 2 * H, RN = RH * RW;
    static constexpr int RN4 = (RN + 3) & ~3;
    static constexpr int NDV = 2 * S - 1;
    // padded record rows (unclamped dv reads); the pad is a multiple of 8
    // elements (128 B) so a warp straddling a row wrap keeps its bank mapping
    static constexpr int PADC = S, RWS = RW + ((2 * S + 1 + 7) & ~7);
    static constexpr int RECN = RH * RWS;
    using DT = typename std::conditional<BOTH, float2, float>::type;
    // Row offsets du are processed in groups of G (one barrier pair per
    // group): small windows evaluate all U planes at once.
    static constexpr int G = (S == 3) ? S : 1;
    __host__ __device__ static constexpr int ndv_of(int du) { return du == 0 ? S - 1 : 2 * S - 1; }
    __host__ __device__ static constexpr int plane_off(int du)
    {
        int o = 0;
        for (int d = (du / G) * G; d < du; d++) o += ndv_of(d);
        return o;
    }
    __host__ __device__ static constexpr int item_off(int du)
    {
        int o = 0;
        for (int d = (du / G) * G; d < du; d++) o += (RH - d) * RW;
        return o;
    }
    static constexpr int NPL = (G == S) ? plane_off(S - 1) + ndv_of(S - 1) : NDV;  // planes resident at once
    // 5x5 / 7x7: row-segment sums S_+du (double-buffered: the next row
    // offset's stage 1 writes one buffer while the outputs accumulate the
    // other) and S_-du, S values per pixel each
    static constexpr bool SEG = S >= 5;
    static constexpr int SEGN = SEG ? 3 * S : 0;
    // 5x5 / 7x7 records: pair elements split by the parity of their first
    // column (element e of a parity row holds columns c, c+1 with
    // c = 2 (e - PADE) + parity), so a thread owning the pixel pair
    // (2j, 2j+1) reads its partners -- all at even columns for du > 0, odd
    // for du = 0 -- as consecutive 16-byte elements across the warp; the row
    // pitch RWS2 = RW/2 + 8 keeps a warp's accesses bank-contiguous across
    // row wraps
    static constexpr int RW2 = RW / 2, PADE = H, RWS2 = RW2 + 8;
    // stage-1 items: horizontal pixel pairs (half the record loads) where
    // the register budget allows their live set (>= 168 per thread: the
    // 1-CTA-per-SM shapes); one pixel per item otherwise
    static constexpr bool ITEM2 = NT * 168 <= 65536;
    // elements per parity array.  One-pixel items read both parities in one
    // warp instruction (even lanes the even array, odd lanes the odd one):
    // the arrays then sit 64 bytes apart modulo 128 (RECN2 = 4 mod 8), so the
    // two lane groups of a 16-byte access use different banks
    static constexpr int RECN2 = ITEM2 ? RH * RWS2 : ((RH * RWS2 + 3) & ~7) + 4;
    static constexpr size_t kRecBytes = SEG ? (size_t)RECN2 * 64 : (size_t)RECN * 32;
    // TMA buffers (128-byte aligned): two raw uint8 regions (box of 144 bytes
    // x RH rows: a tile load must start at a 16-byte aligned column, so the
    // box starts up to 15 bytes left of the region) and the tile's output
    // colours (TH rows x 96 bytes)
    static constexpr int kRawPitch = 144, kRawBytes = RH * kRawPitch, kRawBuf = (kRawBytes + 127) & ~127;
    static_assert(3 * RW + 15 <= kRawPitch, "region row fits the TMA box");
    static constexpr size_t kBodyBytes =
        kRecBytes + (size_t)RN4 * 4 + (size_t)NPL * RN * sizeof(DT) + (size_t)SEGN * RN * sizeof(DT);
    static constexpr size_t kRawOff = (kBodyBytes + 127) & ~(size_t)127;
    static constexpr size_t kOutOff = kRawOff + 2 * (size_t)kRawBuf;
    static constexpr int kOutBuf = (TH * 96 + 127) & ~127;  // double-buffered (tile parity)
    static constexpr size_t kSmem = kOutOff + 2 * (size_t)kOutBuf + 128;  // + 128: runtime base alignment
};

// One-pass first-strict-minimum with "best competitor of a different colour"
// tracking.  Invariant: v2 = min over scanned candidates whose colour differs
// from the current winner's (the candidates that could change the output).
// The error bound of a candidate, er*|v| + ea*l (l = its Minkowski factor),
// is formed only for the two tracked candidates at the end.
struct Sel {
    float v1, l1, v2, l2;
    int i1;
    uint32_t k1;
    float xa, xl;  // payload of the winner (ACWDDF centre distances)
    __device__ __forceinline__ void init(float v, float l, uint32_t k, float pa, float pl)
    {
        v1 = v; l1 = l; v2 = __int_as_float(0x7f800000); l2 = 0.f; i1 = 0; k1 = k; xa = pa; xl = pl;
    }
    __device__ __forceinline__ void add(float v, float l, int i, uint32_t k, float pa, float pl)
    {
        if (v < v1) {
            if (k != k1) { v2 = v1; l2 = l1; }
            v1 = v; l1 = l; i1 = i; k1 = k; xa = pa; xl = pl;
        } else if (k != k1 && v < v2) {
            v2 = v; l2 = l;
        }
    }
    // true when the FP32 order of winner and competitor is not certain
    __device__ __forceinline__ bool doubtful(float er, float ea) const
    {
        // (no competitor: v2 = inf -> inf - inf = NaN -> false)
        return (v2 - v1) - er * fabsf(v2) <= er * fabsf(v1) + ea * (l1 + l2);
    }
};

// Window selection in two passes (cheaper than Sel's single pass):
//   1. first strict minimum v1 (window order, like the reference's argmin)
//      with its index, colour and optional payload;
//   2. the smallest value among candidates of a different colour.
// val(ic), col(ic), pa(ic), pl(ic) take std::integral_constant indices so the
// caller's register arrays stay compile-time indexed.
struct Pick {
    float v1, other, xa, xl;
    int i1;
    uint32_t k1;
    // FP32 order of winner and competitor not certain under the bound
    // er*|v| + ea*lmax per candidate (no competitor: inf - inf = NaN -> false)
    __device__ __forceinline__ bool doubtful(float er, float ea_lmax) const
    {
        return (other - v1) - er * fabsf(other) <= er * fabsf(v1) + 2.f * ea_lmax;
    }
};

// ZX: an FP32 value of exactly 0 is the reference's exact 0 (exact and
// chromaticity routes: a zero pair value means parallel vectors, which the
// reference also maps to exactly 0), so exact-zero competitors tie with an
// exact-zero winner exactly -- the first index wins in both -- and are not
// counted as competitors.  (A near-zero FP32 value the reference may round to
// 0 stays a competitor: the absolute bound flags it.)
// Tournament form of the window-order scan: each merge of two adjacent
// index ranges keeps the left (lower-index) winner unless the right one is
// strictly smaller, so the root is the first strict minimum -- the same
// result as the sequential scan (E:317-355) with log2(N) instead of N - 1
// dependent compare/select steps (same instruction count).
// Ranges of at most LEAF candidates are scanned sequentially (7x7 keeps the
// plain scan: a full tree's wider live set spills there, and four quarter
// scans merged by the tree measured no faster).
template <int LO, int HI, int LEAF, bool PAY, typename FV, typename FC, typename FA, typename FL>
__device__ __forceinline__ Pick pick_range(FV &val, FC &col, FA &pa, FL &pl)
{
    if constexpr (HI - LO <= LEAF) {
        Pick r;
        r.v1 = val(std::integral_constant<int, LO>{});
        r.i1 = LO;
        r.k1 = col(std::integral_constant<int, LO>{});
        if constexpr (PAY) {
            r.xa = pa(std::integral_constant<int, LO>{});
            r.xl = pl(std::integral_constant<int, LO>{});
        }
        static_for<LO + 1, HI>([&](auto ic) {
            constexpr int i = decltype(ic)::value;
            const float v = val(ic);
            const bool p = v < r.v1;
            r.v1 = p ? v : r.v1;
            r.i1 = p ? i : r.i1;
            r.k1 = p ? col(ic) : r.k1;
            if constexpr (PAY) {
                r.xa = p ? pa(ic) : r.xa;
                r.xl = p ? pl(ic) : r.xl;
            }
        });
        return r;
    } else {
        constexpr int MID = LO + (HI - LO + 1) / 2;
        Pick a = pick_range<LO, MID, LEAF, PAY>(val, col, pa, pl);
        const Pick b = pick_range<MID, HI, LEAF, PAY>(val, col, pa, pl);
        const bool p = b.v1 < a.v1;
        a.v1 = p ? b.v1 : a.v1;
        a.i1 = p ? b.i1 : a.i1;
        a.k1 = p ? b.k1 : a.k1;
        if constexpr (PAY) {
            a.xa = p ? b.xa : a.xa;
            a.xl = p ? b.xl : a.xl;
        }
        return a;
    }
}

// min (or max) over f(I), I in [LO, HI), as a balanced tree (exact: min and
// max do not round, so any order gives the same value)
template <int LO, int HI, bool MAX, int LEAF = 1, typename F>
__device__ __forceinline__ float tree_minmax(F &f)
{
    if constexpr (HI - LO <= LEAF) {
        float r = f(std::integral_constant<int, LO>{});
        static_for<LO + 1, HI>([&](auto ic) { r = MAX ? fmaxf(r, f(ic)) : fminf(r, f(ic)); });
        return r;
    } else {
        constexpr int MID = LO + (HI - LO + 1) / 2;
        const float a = tree_minmax<LO, MID, MAX, LEAF>(f), b = tree_minmax<MID, HI, MAX, LEAF>(f);
        return MAX ? fmaxf(a, b) : fminf(a, b);
    }
}

template <int N, bool PAY, bool ZX, typename FV, typename FC, typename FA, typename FL>
__device__ __forceinline__ Pick pick(FV val, FC col, FA pa, FL pl)
{
    constexpr int LEAF = N <= 25 ? 1 : N;
    Pick r = pick_range<0, N, LEAF, PAY>(val, col, pa, pl);
    const uint32_t k1 = r.k1;
    auto masked = [&](auto ic) {
        return (col(ic) != k1 && (!ZX || val(ic) > 0.f)) ? val(ic) : __int_as_float(0x7f800000);
    };
    r.other = tree_minmax<0, N, false, LEAF>(masked);
    return r;
}

// The reference's selection for one output (E:317-355, E:451-487) on the
// FP32 aggregates: A(ic)/L(ic) angular/Minkowski aggregates, AD/LD the
// ACWDDF centre column, col(ic) the candidate colours.  Returns the chosen
// window index and whether the decision is within the FP32 error budget.
template <int FAM, int ST, int N, int DC, typename FA, typename FL, typename FAD, typename FLD, typename FC>
__device__ __forceinline__ void select_window(const KParams &kp, FA A, FL L, FAD AD, FLD LD, FC col, uint32_t &kc,
                                              bool &doubt)
{
    const float er = kp.er, ea = kp.ea;
    constexpr bool ZX = ST != ST_MINIMAX;
    auto none = [](auto) { return 0.f; };
    if constexpr (FAM == FAM_ACWDDF) {
        const float w0 = kp.w[0], w1 = kp.w[1], w2 = kp.w[2];
        // largest Minkowski factor of any product (w0 >= w1 >= w2 >= 0)
        // (forming A + w AD and L + w LD as one packed FFMA2 measured no
        // faster on C3 and 2.7 % slower on C5b)
        auto lf = [&](auto ic) { return fmaf(w0, LD(ic), L(ic)); };
        const float lmax = fmaxf(tree_minmax<0, N, true, N <= 25 ? 1 : N>(lf), 0.f);
        const Pick sd = pick<N, false, ZX>([&](auto ic) { return A(ic) * L(ic); }, col, none, none);
        const Pick s0 = pick<N, true, ZX>([&](auto ic) { return fmaf(w0, AD(ic), A(ic)) * fmaf(w0, LD(ic), L(ic)); },
                                      col, AD, LD);
        const Pick s1 = pick<N, true, ZX>([&](auto ic) { return fmaf(w1, AD(ic), A(ic)) * fmaf(w1, LD(ic), L(ic)); },
                                      col, AD, LD);
        const Pick s2 = pick<N, true, ZX>([&](auto ic) { return fmaf(w2, AD(ic), A(ic)) * fmaf(w2, LD(ic), L(ic)); },
                                      col, AD, LD);
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
        kc = fires ? sd.k1 : col(std::integral_constant<int, DC>{});
        const float er2 = 2.f * er, eal = 2.f * ea * lmax;
        doubt = s0.doubtful(er2, eal) || s1.doubtful(er2, eal) || s2.doubtful(er2, eal) ||
                fabsf(sv - kp.threshold) <= es || (fires && sd.doubtful(er2, eal));
    } else if constexpr (FAM == FAM_CWDDF) {
        // filters.py:296-328: argmin (A + w AD)(L + w LD), w = n - 2k + 1
        const float w0 = kp.w[0];
        auto lf = [&](auto ic) { return fmaf(w0, LD(ic), L(ic)); };
        const float lmax = fmaxf(tree_minmax<0, N, true, N <= 25 ? 1 : N>(lf), 0.f);
        const Pick s = pick<N, false, ZX>([&](auto ic) { return fmaf(w0, AD(ic), A(ic)) * fmaf(w0, LD(ic), L(ic)); },
                                      col, none, none);
        kc = s.k1;
        doubt = s.doubtful(2.f * er, 2.f * ea * lmax);
    } else if constexpr (FAM == FAM_CWVMF) {
        // filters.py:331-337: argmin L + w LD
        const float w0 = kp.w[0];
        const Pick s = pick<N, false, ZX>([&](auto ic) { return fmaf(w0, LD(ic), L(ic)); }, col, none, none);
        kc = s.k1;
        doubt = s.doubtful(er, 0.f);
    } else if constexpr (FAM == FAM_DDF) {
        const float lmax = fmaxf(tree_minmax<0, N, true, N <= 25 ? 1 : N>(L), 0.f);
        const Pick s = pick<N, false, ZX>([&](auto ic) { return A(ic) * L(ic); }, col, none, none);
        kc = s.k1;
        doubt = s.doubtful(2.f * er, 2.f * ea * lmax);
    } else if constexpr (FAM == FAM_BVDF) {
        const Pick s = pick<N, false, ZX>(A, col, none, none);
        kc = s.k1;
        doubt = s.doubtful(er, ea);
    } else {
        const Pick s = pick<N, false, ZX>(L, col, none, none);
        kc = s.k1;
        doubt = s.doubtful(er, 0.f);
    }
}

// Two pairs (p, q) and (p, q+1): angular and/or Minkowski distances.
template <int FAM, int ST, int PC, bool ZC>
__device__ __forceinline__ void pair_values2(const Pix &p, const Pair2 &q, const KParams &kp, P2 &da, P2 &dl)
{
    constexpr bool NA = FamT<FAM>::A;
    constexpr bool NL = FamT<FAM>::L;
    if (NA) {
        if (ST == ST_EXACT) da = angle_half2<ZC>(p, q);
        else if (ST == ST_MINIMAX) da = angle_minimax2(p, q, kp);
        else if (PC == PC_2) da = chroma2_l2(p, q);
        else {
            const float4 a = make_float4(p.x, p.y, p.z, p.aux);
            da = pk2(chroma<PC>(a, p.x + p.y + p.z, make_float4(lo2(q.x), lo2(q.y), lo2(q.z), lo2(q.aux)),
                                lo2(q.x) + lo2(q.y) + lo2(q.z), kp),
                     chroma<PC>(a, p.x + p.y + p.z, make_float4(hi2(q.x), hi2(q.y), hi2(q.z), hi2(q.aux)),
                                hi2(q.x) + hi2(q.y) + hi2(q.z), kp));
        }
    }
    if (NL) {
        const bool anyz =
            ZC && ((__float_as_uint(p.aux) | __float_as_uint(lo2(q.aux)) | __float_as_uint(hi2(q.aux))) & zbit<ST>());
        if (PC == PC_2 && !anyz) {
            dl = l2_2(p, q);
        } else {  // zero pixels (raw 0 vs gray-mapped 1) or p != 2: per lane on raw values
            const float4 a = rawrec<ST>(p.x, p.y, p.z, p.aux);
            dl = pk2(minkowski<PC>(a, rawrec<ST>(lo2(q.x), lo2(q.y), lo2(q.z), lo2(q.aux)), kp),
                     minkowski<PC>(a, rawrec<ST>(hi2(q.x), hi2(q.y), hi2(q.z), hi2(q.aux)), kp));
        }
    }
}

__device__ __forceinline__ float dt_add(float a, float b) { return a + b; }
__device__ __forceinline__ float2 dt_add(float2 a, float2 b)
{
    const P2 r = add2(*reinterpret_cast<const P2 *>(&a), *reinterpret_cast<const P2 *>(&b));
    return *reinterpret_cast<const float2 *>(&r);
}
__device__ __forceinline__ float dt_zero(float) { return 0.f; }
__device__ __forceinline__ float2 dt_zero(float2) { return make_float2(0.f, 0.f); }

// Row-segment sums of one pixel: T[t], t = dv + S - 1, dv in [-(S-1), S-1]
// (distances to the pixels of one row at column offsets dv) ->
// Sg[v] = sum_{dv = -v}^{S-1-v} T = the distance sum to the S-wide segment of
// a window in which the pixel sits at column v.  Every window contains
// dv = 0, so Sg[v] = L[S-1-v] + R[2S-2-v] with suffix sums L of the left part
// and prefix sums R of the right part: additions only (no cancellation),
// 3S-4 adds for all S windows.
template <int S, typename DT>
__device__ __forceinline__ void seg_sums(const DT (&T)[2 * S - 1], DT (&Sg)[S])
{
    DT L[S - 1], R[S];
    L[S - 2] = T[S - 2];
#pragma unroll
    for (int t = S - 3; t >= 0; t--) L[t] = dt_add(T[t], L[t + 1]);
    R[0] = T[S - 1];
#pragma unroll
    for (int t = 1; t < S; t++) R[t] = dt_add(R[t - 1], T[S - 1 + t]);
    Sg[0] = R[S - 1];
#pragma unroll
    for (int v = 1; v < S; v++) Sg[v] = dt_add(L[S - 1 - v], R[S - 1 - v]);
}

// 5x5 / 7x7 aggregation by row segments.  For row offset du, stage 1
// evaluates the pair planes D_(du,dv)(p) and, from the same registers, the
// pixel's downward segment sums S_+du(p, v); after a barrier the upward sums
// S_-du(q, v) are read off the planes (the pairs whose upper pixel is in the
// row above); after a second barrier each output adds, for each window
// candidate (u, v), S_+du(q, v) if u + du < S and S_-du(q, v) if u >= du:
// agg(u, v) = sum_dy S_dy(q, v) covers every other window pixel exactly once.
// s^3 segment loads per output instead of n(n-1)/2 pair loads (343 vs 1176
// for 7x7), and the sums carry no cancellation.
//
// Schedule: a stage-1 item is a horizontal pixel PAIR (2j, 2j+1) against
// partner elements (q, q+1) at even columns: both pixels' pair values come
// from one element load (4 pairs per element, half the record traffic of
// one pixel per item), and their plane / segment values leave as one
// 16-byte store per plane.  Two barrier intervals per row offset: stage 1
// of du runs beside the outputs' accumulation of du - 1 (FP32-heavy item
// work next to shared-memory-heavy accumulation, which also fills the item
// loop's load imbalance; S_+du is double-buffered), then phase 2 of du.
// The row's own sums (du = 0) go to the S_- buffer; the centre-column
// stash is read in phase 2, before stage 1 of du + 1 overwrites the
// planes.  (Measured: pairing phase 2 with the S_+ half of the
// accumulation instead -- no double buffer -- ran 9 % slower on C5a: both
// halves of each pairing then contend for the same pipe.)
template <typename DT>
__device__ __forceinline__ void st_pair(DT *dst, DT a, DT b)  // dst 2-element aligned
{
    if constexpr (std::is_same<DT, float2>::value) {
        *reinterpret_cast<float4 *>(dst) = make_float4(a.x, a.y, b.x, b.y);
    } else {
        *reinterpret_cast<float2 *>(dst) = make_float2(a, b);
    }
}

template <int S, int FAM, int ST, int PC, int OPT, int TR, typename AG, typename CE, typename AA, typename AL>
__device__ __forceinline__ void seg_stages(const float4 *rec, typename Cfg<S, FAM, OPT, TR>::DT *sD, bool zchk,
                                           const KParams &kp, AG &ag, CE &cen, AA &aA, AL &aL, const int tid)
{
    using C = Cfg<S, FAM, OPT, TR>;
    using DT = typename C::DT;
    constexpr int H = C::H, DC = C::DC, RW = C::RW, RH = C::RH, RN = C::RN, NT = C::NT;
    constexpr int RW2 = C::RW2, RWS2 = C::RWS2, PADE = C::PADE, RECN2 = C::RECN2, NDV = C::NDV;
    constexpr bool CEN = C::CEN;
    constexpr bool BOTH = C::BOTH;
    DT *sP0 = sD + C::NPL * RN;  // S_+du [v][RN], even du
    DT *sP1 = sP0 + S * RN;      // S_+du [v][RN], odd du
    DT *sM = sP1 + S * RN;       // S_-du [v][RN] (du = 0: both sides in the row)
    const int tx = tid & 31, ty = tid >> 5;
    const float4 *recAe = rec, *recAo = rec + RECN2, *recBe = rec + 2 * RECN2, *recBo = rec + 3 * RECN2;

    auto to_dt = [](P2 da, P2 dl, bool hi) -> DT {
        if constexpr (BOTH) return hi ? make_float2(hi2(da), hi2(dl)) : make_float2(lo2(da), lo2(dl));
        else if constexpr (C::NEED_A) return hi ? hi2(da) : lo2(da);
        else return hi ? hi2(dl) : lo2(dl);
    };

    // ---- per-output accumulation of the segment sums of du: S_+du
    // (u + du < S) and S_-du (u >= du; du = 0: the row's both-sided sums);
    // one window row u per call ------------------------------------------
    auto accumulate_row = [&](auto du_c, auto u_c) {
        constexpr int du = decltype(du_c)::value, u = decltype(u_c)::value;
        const DT *sPd = (du & 1) ? sP1 : sP0;
        if constexpr (du == 0 || u + du < S || u >= du) {
#pragma unroll
            for (int o = 0; o < OPT; o++) {
                const int ry0 = ty * OPT + o;
#pragma unroll
                for (int v = 0; v < S; v++) {
                    const int i = u * S + v;
                    const int qi = (ry0 + u) * RW + tx + v;
                    DT add;
                    if constexpr (du == 0) add = sM[v * RN + qi];
                    else if constexpr (u + du < S && u >= du) add = dt_add(sPd[v * RN + qi], sM[v * RN + qi]);
                    else if constexpr (u + du < S) add = sPd[v * RN + qi];
                    else add = sM[v * RN + qi];
                    if constexpr (BOTH) {
                        ag[o][i] = add2(ag[o][i], *reinterpret_cast<const P2 *>(&add));
                    } else if constexpr (C::NEED_A) {
                        aA[o][i] += add;
                    } else {
                        aL[o][i] += add;
                    }
                }
            }
        }
    };
    auto accumulate = [&](auto du_c) { static_for<0, S>([&](auto u_c) { accumulate_row(du_c, u_c); }); };

    // ---- stage 1 of row offset du: planes (+ downward segment sums) --------
    auto stage1 = [&](auto du_c, auto zc_c) {
        constexpr int du = decltype(du_c)::value;
        constexpr bool ZC = decltype(zc_c)::value;
        constexpr int items = (RH - du) * RW2;
        // one item; `has` predicates its stores (a lane without an item of its
        // own evaluates a clamped one); chunk(c), c = 0 .. S-1, is called after
        // the c-th element evaluation (the interleaved accumulation below)
        auto item = [&](const int it2, const bool has, auto &&chunk) {
            const int py = it2 / RW2, j = it2 - py * RW2;
            const int it0 = py * RW + 2 * j;
            const int pe = py * RWS2 + PADE + j;  // the item's own element: pixels (2j, 2j+1)
            const ulonglong2 pa = lds_u2(recAe + pe), pb = lds_u2(recBe + pe);
            const Pix p0 = {lo2(P2{pa.x}), lo2(P2{pa.y}), lo2(P2{pb.x}), lo2(P2{pb.y})};
            const Pix p1 = {hi2(P2{pa.x}), hi2(P2{pa.y}), hi2(P2{pb.x}), hi2(P2{pb.y})};
            DT T0[NDV], T1[NDV];  // pair values of p0 / p1, t = offset - dv0 (fully unrolled)
            if constexpr (du > 0) {
                // partners at columns 2j + d, d = 2m - (S-1): p0 gets offsets
                // d, d+1 (t = 2m, 2m+1), p1 gets d-1, d (t = 2m-1, 2m).
                // Elements are visited right half first (m = H .. S-1:
                // the prefix sums R of the segment sums), then left half
                // descending (m = H-1 .. 0: the suffix sums L, each
                // completing one segment sum), so only R and a value or two
                // stay live -- the same operations and order as seg_sums.
                const int qe = (py + du) * RWS2 + PADE + j - H;
                DT R0[S], R1[S], L0, L1;
                auto eval = [&](auto m_c) {
                    constexpr int m = decltype(m_c)::value;
                    const ulonglong2 A2 = lds_u2(recAe + qe + m), B2 = lds_u2(recBe + qe + m);
                    const Pair2 q = {{A2.x}, {A2.y}, {B2.x}, {B2.y}};
                    P2 da0, dl0, da1, dl1;
                    pair_values2<FAM, ST, PC, ZC>(p0, q, kp, da0, dl0);
                    pair_values2<FAM, ST, PC, ZC>(p1, q, kp, da1, dl1);
                    T0[2 * m] = to_dt(da0, dl0, false);
                    if constexpr (m < S - 1) T0[2 * m + 1] = to_dt(da0, dl0, true);
                    if constexpr (m > 0) T1[2 * m - 1] = to_dt(da1, dl1, false);
                    T1[2 * m] = to_dt(da1, dl1, true);
                };
                static_for<H, S>([&](auto m_c) {  // right half, ascending t
                    constexpr int m = decltype(m_c)::value;
                    eval(m_c);
                    // t = 2m-1 (m > H) and t = 2m are complete for both pixels
                    if (has) {
                        if constexpr (m > H) st_pair(sD + (2 * m - 1) * RN + it0, T0[2 * m - 1], T1[2 * m - 1]);
                        st_pair(sD + (2 * m) * RN + it0, T0[2 * m], T1[2 * m]);
                    }
                    // prefix sums over t = S-1 .. : R[k] = sum of T[S-1 .. S-1+k]
                    static_for<0, S>([&](auto k_c) {
                        constexpr int k = decltype(k_c)::value, t = S - 1 + k;
                        if constexpr (t == 2 * m || t == 2 * m - 1) {
                            if constexpr (k == 0) {
                                R0[0] = T0[t];
                                R1[0] = T1[t];
                            } else {
                                R0[k] = dt_add(R0[k - 1], T0[t]);
                                R1[k] = dt_add(R1[k - 1], T1[t]);
                            }
                        }
                    });
                    chunk(std::integral_constant<int, m - H>{});
                });
                DT *sPd = (du & 1) ? sP1 : sP0;
                if (has) st_pair(sPd + it0, R0[S - 1], R1[S - 1]);  // v = 0: the whole right part
                static_for<0, H>([&](auto mm_c) {           // left half, descending t
                    constexpr int m = H - 1 - decltype(mm_c)::value;
                    eval(std::integral_constant<int, m>{});
                    // t = 2m+1 and t = 2m complete (t = 2m+1 = S-2 first)
                    static_for<0, 2>([&](auto w_c) {
                        constexpr int t = 2 * m + 1 - decltype(w_c)::value;
                        if (has) st_pair(sD + t * RN + it0, T0[t], T1[t]);
                        if constexpr (t == S - 2) {
                            L0 = T0[t];
                            L1 = T1[t];
                        } else {
                            L0 = dt_add(T0[t], L0);
                            L1 = dt_add(T1[t], L1);
                        }
                        // L = L[t]: segment sum of the window in which the
                        // pixel sits at column v = S-1-t
                        if (has) st_pair(sPd + (S - 1 - t) * RN + it0, dt_add(L0, R0[t]), dt_add(L1, R1[t]));
                    });
                    chunk(std::integral_constant<int, H + 1 + decltype(mm_c)::value>{});
                });
            } else {
                // same row, partners to the right: odd-column elements
                // (2j+1+2m, 2j+2+2m); p0 offsets 2m+1, 2m+2, p1 offsets 2m,
                // 2m+1 (plane k = offset - 1); each plane pair is stored as
                // soon as both values exist
                const int qe = py * RWS2 + PADE + j;
                static_for<0, H + 1>([&](auto m_c) {
                    constexpr int m = decltype(m_c)::value;
                    const ulonglong2 A2 = lds_u2(recAo + qe + m), B2 = lds_u2(recBo + qe + m);
                    const Pair2 q = {{A2.x}, {A2.y}, {B2.x}, {B2.y}};
                    P2 da0, dl0, da1, dl1;
                    if constexpr (m < H) {
                        pair_values2<FAM, ST, PC, ZC>(p0, q, kp, da0, dl0);
                        T0[2 * m] = to_dt(da0, dl0, false);
                        T0[2 * m + 1] = to_dt(da0, dl0, true);
                    }
                    pair_values2<FAM, ST, PC, ZC>(p1, q, kp, da1, dl1);
                    if constexpr (m > 0) {
                        T1[2 * m - 1] = to_dt(da1, dl1, false);
                        if (has) st_pair(sD + (2 * m - 1) * RN + it0, T0[2 * m - 1], T1[2 * m - 1]);
                    }
                    if constexpr (m < H) {
                        T1[2 * m] = to_dt(da1, dl1, true);
                        if (has) st_pair(sD + (2 * m) * RN + it0, T0[2 * m], T1[2 * m]);
                    }
                });
            }
        };
        for (int it2 = tid; it2 < items; it2 += NT) item(it2, true, [](auto) {});
    };
    // one-pixel items (register-tight shapes, Cfg::ITEM2 false): pixel p at
    // column c against the pair elements of c's parity, (q, q+1) at c - (S-1)
    // + 2m (du > 0) or c + 1 + 2m (du = 0, the other parity)
    auto stage1_px = [&](auto du_c, auto zc_c) {
        constexpr int du = decltype(du_c)::value;
        constexpr bool ZC = decltype(zc_c)::value;
        constexpr int items = (RH - du) * RW;
        constexpr int ndv = C::ndv_of(du);
        constexpr int NK2 = (ndv + 1) / 2;
        for (int it = tid; it < items; it += NT) {
            const int py = it / RW, c = it - py * RW;
            const int par = c & 1, e = (c >> 1) + PADE;
            const float4 *pA = par ? recAo : recAe, *pB = par ? recBo : recBe;
            const float4 a4 = lds_f4(pA + py * RWS2 + e), b4 = lds_f4(pB + py * RWS2 + e);
            const Pix p = {a4.x, a4.z, b4.x, b4.z};
            // partner elements: du > 0 same parity, from e - H; du = 0 the
            // other parity (element of column c + 1 = c + 1's own index)
            const float4 *qA = (du > 0) ? pA : (par ? recAe : recAo);
            const float4 *qB = (du > 0) ? pB : (par ? recBe : recBo);
            const int qe = (py + du) * RWS2 + ((du > 0) ? e - H : ((c + 1) >> 1) + PADE);
            DT T[NDV];
#pragma unroll
            for (int kk = 0; kk < NK2; kk++) {
                const ulonglong2 A2 = lds_u2(qA + qe + kk), B2 = lds_u2(qB + qe + kk);
                const Pair2 q = {{A2.x}, {A2.y}, {B2.x}, {B2.y}};
                P2 da, dl;
                pair_values2<FAM, ST, PC, ZC>(p, q, kp, da, dl);
                T[2 * kk] = to_dt(da, dl, false);
                sD[(2 * kk) * RN + it] = T[2 * kk];
                if (2 * kk + 1 < ndv) {
                    T[2 * kk + 1] = to_dt(da, dl, true);
                    sD[(2 * kk + 1) * RN + it] = T[2 * kk + 1];
                }
            }
            if constexpr (du > 0) {
                DT Sg[S];
                seg_sums<S>(T, Sg);
                DT *sPd = (du & 1) ? sP1 : sP0;
#pragma unroll
                for (int v = 0; v < S; v++) sPd[v * RN + it] = Sg[v];
            }
        }
    };
    auto run_stage1 = [&](auto du_c) {
        if constexpr (C::ITEM2) {
            if (zchk) stage1(du_c, std::true_type{});
            else stage1(du_c, std::false_type{});
        } else {
            if (zchk) stage1_px(du_c, std::true_type{});
            else stage1_px(du_c, std::false_type{});
        }
    };

    // ---- phase 2 of du: upward sums (du > 0) / both sides in the row (du = 0),
    // and the centre-column stash (read off the planes before stage 1 of
    // du + 1 overwrites them) --------------------------------------------
    auto phase2 = [&](auto du_c) {
        constexpr int du = decltype(du_c)::value;
        [[maybe_unused]] constexpr int dv0 = (du == 0) ? 1 : -(S - 1);
        constexpr int items = (RH - du) * RW;
        for (int it = tid; it < items; it += NT) {
            const int qi = it + du * RW;  // pixel q in rows du .. RH-1
            DT T[NDV];
            if constexpr (du == 0) {
#pragma unroll
                for (int t = 0; t < NDV; t++) {
                    const int dv = t - (S - 1);
                    if (dv > 0) T[t] = sD[(dv - 1) * RN + qi];
                    else if (dv < 0) T[t] = sD[(-dv - 1) * RN + qi + dv];
                    else T[t] = dt_zero(DT());
                }
            } else {
                // T_q(-du, dv) = D_(du, -dv)(q + (-du, dv)): plane 2S-2-t
#pragma unroll
                for (int t = 0; t < NDV; t++) {
                    const int dv = t - (S - 1);
                    T[t] = sD[(NDV - 1 - t) * RN + qi - du * RW + dv];
                }
            }
            // seg_sums' operations and order, each sum stored as it completes
            // (prefix sums R of the right part, then the suffix sums L of the
            // left part descending: Sg[v] = L[S-1-v] + R[S-1-v])
            DT R[S];
            R[0] = T[S - 1];
#pragma unroll
            for (int k = 1; k < S; k++) R[k] = dt_add(R[k - 1], T[S - 1 + k]);
            sM[qi] = R[S - 1];  // v = 0
            DT L = T[S - 2];
#pragma unroll
            for (int k = S - 2; k >= 0; k--) {
                if (k < S - 2) L = dt_add(T[k], L);
                sM[(S - 1 - k) * RN + qi] = dt_add(L, R[k]);
            }
        }
        if constexpr (CEN) {  // centre-column stash: the pair (i, centre) itself
#pragma unroll
            for (int o = 0; o < OPT; o++) {
                const int ry0 = ty * OPT + o;
#pragma unroll
                for (int i = 0; i < C::N; i++) {
                    const int u = i / S, v = i % S;
                    if (i < DC && H - u == du) {
                        cen[o][i] = sD[(H - v - dv0) * RN + (ry0 + u) * RW + tx + v];
                    } else if (i > DC && u - H == du) {
                        cen[o][i] = sD[(v - H - dv0) * RN + (ry0 + H) * RW + tx + H];
                    }
                }
            }
        }
    };

    run_stage1(std::integral_constant<int, 0>{});
    __syncthreads();
    phase2(std::integral_constant<int, 0>{});
    __syncthreads();
    static_for<1, S>([&](auto du_c) {
        constexpr int du = decltype(du_c)::value;
        // (interleaving this accumulation into the items, one window row per
        // element evaluation, measured 4 % slower on C5a; running the two
        // halves in opposite order on odd and even warps 63 % slower: two
        // instruction streams thrash the instruction cache)
        run_stage1(du_c);
        accumulate(std::integral_constant<int, du - 1>{});
        __syncthreads();
        phase2(du_c);
        __syncthreads();
    });
    accumulate(std::integral_constant<int, S - 1>{});
    __syncthreads();
}

// ---- TMA helpers (raw PTX; sm_90+ bulk tensor copies, mbarrier completion) --
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count)
{
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase)
{
    uint32_t done;
    do {
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}"
                     : "=r"(done)
                     : "r"(smem_u32(bar)), "r"(phase)
                     : "memory");
    } while (!done);
}
// one thread: region rows of a tile -> shared memory, completion on `bar`
__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, int c0, int c1, int c2, uint64_t *bar,
                                            uint32_t bytes)
{
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4}], "
        "[%5];" ::"r"(smem_u32(dst)),
        "l"(reinterpret_cast<uint64_t>(map)), "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(bar))
        : "memory");
}
__device__ __forceinline__ void tma_store_3d(const CUtensorMap *map, int c0, int c1, int c2, const void *src)
{
    asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%1, %2, %3}], [%4];" ::"l"(
                     reinterpret_cast<uint64_t>(map)),
                 "r"(c0), "r"(c1), "r"(c2), "r"(smem_u32(src))
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
// at most one bulk store group (the previous tile's) still reading its source
__device__ __forceinline__ void tma_store_wait_read1() { asm volatile("cp.async.bulk.wait_group.read 1;" ::: "memory"); }
__device__ __forceinline__ void tma_store_wait_all() { asm volatile("cp.async.bulk.wait_group 0;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }

// Persistent CTA kernel: each CTA walks tiles blockIdx.x, + gridDim.x, ...
// (x fastest, then tile rows, then frames).  Interior tiles of a
// TMA-eligible image (KParams::tma_in) receive their uint8 region by one
// bulk tensor copy issued while the CTA still works on the previous tile
// (double-buffered raw region, mbarrier completion); border tiles resolve
// the border policy with indexed loads.  The selected colours of a tile are
// assembled in shared memory (float64 re-decisions included) and leave as
// one bulk tensor store (KParams::tma_out; the tensor map clips partial
// tiles at the image edge), else as byte stores.
template <int S, int FAM, int ST, int PC, int OPT, int TR, int MINB>
__global__ void __launch_bounds__(TR * 32, MINB)
dfg_fast_kernel(const uint8_t *__restrict__ in, uint8_t *__restrict__ out, const __grid_constant__ KParams kp)
{
    using C = Cfg<S, FAM, OPT, TR>;
    using DT = typename C::DT;
    constexpr int H = C::H, N = C::N, DC = C::DC, RW = C::RW, RH = C::RH, RN = C::RN, NT = C::NT, TH = C::TH;
    constexpr int RWS = C::RWS, PADC = C::PADC;
    constexpr bool CEN = C::CEN;
    constexpr bool BOTH = C::BOTH;

    extern __shared__ __align__(128) unsigned char smem_raw[];
    float4 *sA = reinterpret_cast<float4 *>(smem_raw);       // {gx_c, gx_c+1, gy_c, gy_c+1}
    float4 *sB = sA + C::RECN;                                // {gz_c, gz_c+1, aux_c, aux_c+1}
    // (5x5 / 7x7: the same elements in the parity layout, Cfg::RWS2)
    uint32_t *sK = reinterpret_cast<uint32_t *>(smem_raw + C::kRecBytes);  // packed colour (unpadded region)
    DT *sD = reinterpret_cast<DT *>(sK + C::RN4);              // pair-distance planes (+ segment sums)
    // (the dynamic window's base is only guaranteed 16-byte aligned)
    uint8_t *abase = smem_raw + ((128u - (smem_u32(smem_raw) & 127u)) & 127u);
    uint8_t *sRaw = abase + C::kRawOff;  // [2][RH][kRawPitch] TMA region buffers
    uint8_t *sOut0 = abase + C::kOutOff;  // [2][TH][96] the tile's output colours (by tile parity)
    __shared__ unsigned s_nflag;          // this tile's pixels needing float64 re-decision
    __shared__ uint16_t s_flag[TH * 32];  // (window top row << 5) | column
    __shared__ int s_b;
    __shared__ bool s_close;
    __shared__ __align__(8) uint64_t s_bar[2];
    // per-tile state kept in shared memory rather than in registers live
    // across the tile loop (the unrolled stages need every register):
    // s_tile[parity] = {x0, y0, frame, inside} of the tile using raw buffer
    // `parity`; s_state bit 0 = this tile's parity, bits 1, 2 = mbarrier
    // phases of the two buffers
    __shared__ int s_tile[2][4];
    __shared__ uint32_t s_state;

    // (tile counts are recomputed from kp where needed: every register live
    // across the tile loop is taken from the unrolled stages' budget)
    auto n_tiles = [&]() { return ((kp.W + 31) / 32) * ((kp.out_rows + TH - 1) / TH) * kp.n_frames; };
    const float pad_aux = (ST == ST_MINIMAX) ? 0.57735026f : (ST == ST_CHROMA ? (1.f / 3.f) : 1.7320508f);
    const float4 neutral = make_float4(1.f, 1.f, 1.f, pad_aux);

    struct Tile {
        int x0, y0, frame, gy_top;
        bool inside;
    };
    // t / d for t < 2^24 by a float reciprocal and two correction steps
    // (a few instructions instead of an integer division per tile)
    auto divmod = [](int t, int d, int &q) {
        q = __float2int_rz(__int2float_rn(t) * __frcp_rn(__int2float_rn(d)));
        int r = t - q * d;
#pragma unroll
        for (int k = 0; k < 2; k++) {  // |error| <= 2 below 2^24
            if (r < 0) { q--; r += d; }
            if (r >= d) { q++; r -= d; }
        }
        return r;
    };
    auto tile_of = [&](int t) {
        const int tiles_x = (kp.W + 31) / 32, tiles_y = (kp.out_rows + TH - 1) / TH;
        Tile T;
        int r, f;
        T.x0 = divmod(t, tiles_x, r) * 32;
        T.y0 = divmod(r, tiles_y, f) * TH;
        T.frame = f;
        T.gy_top = kp.out_row0 + T.y0 - H;  // global row of region row 0
        T.inside = T.gy_top >= kp.in_row0 && T.gy_top + RH <= kp.in_row0 + kp.in_rows && T.gy_top >= 0 &&
                   T.gy_top + RH <= kp.global_H && T.x0 - H >= 0 && T.x0 - H + RW <= kp.W;
        return T;
    };
    auto issue_load = [&](const Tile &T, int buf) {  // one thread
        // (the box start column must be 16-byte aligned: the region starts
        // (3 (x0 - H)) & 15 bytes into the box)
        tma_load_3d(sRaw + buf * C::kRawBuf, &kp.tm_in, (3 * (T.x0 - H)) & ~15, T.gy_top - kp.in_row0, T.frame,
                    &s_bar[buf], C::kRawBytes);
    };
    auto publish = [&](const Tile &T, int par) {  // one thread
        s_tile[par][0] = T.x0;
        s_tile[par][1] = T.y0;
        s_tile[par][2] = T.frame;
        s_tile[par][3] = T.inside;
    };
    if constexpr (C::SEG) {
        // parity records: every element starts as the neutral gray pair (the pad
        // halves are never written again)
        for (int i = threadIdx.x; i < 2 * C::RECN2; i += NT) {
            sA[i] = make_float4(1.f, 1.f, 1.f, 1.f);
            sA[2 * C::RECN2 + i] = make_float4(1.f, 1.f, pad_aux, pad_aux);
        }
    }
    int t = blockIdx.x;
    if (threadIdx.x == 0) {
        mbar_init(&s_bar[0], 1);
        mbar_init(&s_bar[1], 1);
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        s_state = 0u;
        if (t < n_tiles()) {
            const Tile T0 = tile_of(t);
            publish(T0, 0);
            if (T0.inside && kp.tma_in) issue_load(T0, 0);
        }
    }
    __syncthreads();
#pragma unroll 1
    for (; t < n_tiles(); t += gridDim.x) {
        // the thread index re-read per tile (volatile): keeps the compiler
        // from hoisting every tid-derived shared-memory address of the
        // unrolled stages out of the tile loop (hundreds of live registers)
        int tid, tx, ty;
        asm volatile("mov.u32 %0, %%tid.x;" : "=r"(tid));
        __builtin_assume(tid >= 0 && tid < NT);  // (the range stays known)
        tx = tid & 31;
        ty = tid >> 5;
        const uint32_t par = s_state & 1u;
        Tile T;
        T.x0 = s_tile[par][0];
        T.y0 = s_tile[par][1];
        T.frame = s_tile[par][2];
        T.inside = s_tile[par][3] != 0;
        T.gy_top = kp.out_row0 + T.y0 - H;
        const int tile_x0 = T.x0, frame = T.frame;
        if (tid == 0) s_nflag = 0;

        // ---- stage 0: region staging + per-pixel normalisation ------------
        // Every region pixel is normalised once.  5x5 / 7x7: its four values
        // go straight into the two parity elements that contain it.  3x3: into
        // a temporary float4 record (in the plane buffer, free at this
        // point), from which a second pass assembles the pair elements
        // (c, c+1) with whole 16-byte stores.  Pad positions hold a neutral
        // gray pixel.
        float4 *tmp = reinterpret_cast<float4 *>(sD);
        static_assert((size_t)C::NPL * RN * sizeof(DT) >= (size_t)RN * sizeof(float4), "staging temp fits");
        const bool from_tma = kp.tma_in && T.inside;
        bool any_zero = false;
        auto norm = [&](int idx, int ry, int rx, uint32_t r8, uint32_t g8, uint32_t b8) {
            const bool zero = (r8 | g8 | b8) == 0;
            any_zero |= zero;
            const float gx = zero ? 1.f : (float)r8, gy = zero ? 1.f : (float)g8, gz = zero ? 1.f : (float)b8;
            const float aux = encode_aux<ST, C::NEED_L>(gx, gy, gz, zero);
            sK[idx] = r8 | (g8 << 8) | (b8 << 16);
            if constexpr (C::SEG) {
                // straight into the parity records: the pixel is the first half
                // of element (rx, rx+1) [parity rx & 1] and the second half of
                // element (rx-1, rx) [the other parity]; pad halves keep the
                // neutral pixel written once at kernel start
                float *a1 = reinterpret_cast<float *>(sA + (rx & 1) * C::RECN2 + ry * C::RWS2 + (rx >> 1) + C::PADE);
                float *a2 = reinterpret_cast<float *>(sA + ((rx + 1) & 1) * C::RECN2 + ry * C::RWS2 + ((rx + 1) >> 1) - 1 +
                                                      C::PADE);
                a1[0] = gx; a1[2] = gy; a1[8 * C::RECN2] = gz; a1[8 * C::RECN2 + 2] = aux;
                a2[1] = gx; a2[3] = gy; a2[8 * C::RECN2 + 1] = gz; a2[8 * C::RECN2 + 3] = aux;
            } else {
                tmp[idx] = make_float4(gx, gy, gz, aux);
            }
        };
        // the bulk store of two tiles ago (same parity) has read its sOut buffer
        if (tid == 0 && kp.tma_out) tma_store_wait_read1();
        if (from_tma) {  // the region from shared memory (its bulk copy was issued a tile ago)
            const uint32_t st = s_state;
            mbar_wait(&s_bar[par], (st >> (1 + par)) & 1u);
            const uint8_t *raw = sRaw + par * C::kRawBuf + ((3 * (tile_x0 - H)) & 15);
            for (int idx = tid; idx < RN; idx += NT) {
                const int ry = idx / RW, rx = idx - ry * RW;
                const uint8_t *px = raw + ry * C::kRawPitch + 3 * rx;
                norm(idx, ry, rx, px[0], px[1], px[2]);
            }
        } else {  // indexed loads, border policy by index resolution
            const uint8_t *fin = in + (long long)frame * kp.in_fstride;
            for (int idx = tid; idx < RN; idx += NT) {
                const int ry = idx / RW, rx = idx - ry * RW;
                int gyy, gxx;
                if (T.inside) {
                    gyy = T.gy_top + ry - kp.in_row0;
                    gxx = tile_x0 - H + rx;
                } else {
                    gyy = resolve_idx(T.gy_top + ry, kp.global_H, kp.border) - kp.in_row0;
                    gyy = min(max(gyy, 0), kp.in_rows - 1);
                    gxx = resolve_idx(tile_x0 + rx - H, kp.W, kp.border);
                }
                const uint8_t *px = fin + (long long)gyy * kp.in_pitch + gxx * 3;
                norm(idx, ry, rx, px[0], px[1], px[2]);
            }
        }
        // zero vectors (raw 0 vs gray-mapped 1) only matter to the Minkowski term
        const bool zany = __syncthreads_or(any_zero);  // also the pass-1 barrier
        const bool zchk = C::NEED_L && zany;
        // the next tile's region streams in while this one is computed (its
        // buffer was last read in the previous tile's pass 1)
        // (s_tile[par ^ 1] was last read by the previous tile's selection)
        if (tid == 0) {
            uint32_t st = s_state;
            if (from_tma) st ^= 2u << par;  // this buffer's phase completed
            if (t + (int)gridDim.x < n_tiles()) {
                const Tile Tn = tile_of(t + gridDim.x);
                publish(Tn, par ^ 1u);
                if (Tn.inside && kp.tma_in) issue_load(Tn, par ^ 1u);
            }
            s_state = st ^ 1u;  // read again only after the tile's last barrier
        }
        if constexpr (!C::SEG) {
            for (int idx = tid; idx < C::RECN; idx += NT) {
                const int ry = idx / RWS, c = idx - ry * RWS;
                const int r0 = c - PADC, r1 = r0 + 1;
                const float4 f = (r0 >= 0 && r0 < RW) ? tmp[ry * RW + r0] : neutral;
                const float4 s = (r1 >= 0 && r1 < RW) ? tmp[ry * RW + r1] : neutral;
                sA[idx] = make_float4(f.x, s.x, f.y, s.y);
                sB[idx] = make_float4(f.z, s.z, f.w, s.w);
            }
            __syncthreads();
        }

        // aggregates: BOTH -> packed (angular, Minkowski) pairs; else scalars
        P2 ag[OPT][BOTH ? N : 1];
        DT cen[OPT][CEN ? N : 1];  // centre column (angular, Minkowski) or (Minkowski)
        float aA[OPT][(C::NEED_A && !BOTH) ? N : 1], aL[OPT][(C::NEED_L && !BOTH) ? N : 1];
#pragma unroll
        for (int o = 0; o < OPT; o++) {
#pragma unroll
            for (int i = 0; i < N; i++) {
                if constexpr (BOTH) ag[o][i] = pk2(kp.self_term, 0.f);
                else if constexpr (C::NEED_A) aA[o][i] = kp.self_term;
                else aL[o][i] = 0.f;
            }
            if constexpr (CEN) {
                if constexpr (BOTH) cen[o][DC] = make_float2(kp.self_term, 0.f);
                else cen[o][DC] = dt_zero(DT());
            }
        }

        if constexpr (C::SEG) {
            seg_stages<S, FAM, ST, PC, OPT, TR>(sA, sD, zchk, kp, ag, cen, aA, aL, tid);
        } else
        static_for<0, S / C::G>([&](auto g_c) {
            constexpr int g0 = decltype(g_c)::value * C::G;
            constexpr int total = C::item_off(g0 + C::G - 1) + (RH - (g0 + C::G - 1)) * RW;
            // ---- stage 1: pair distances of the region, each pair once --------
            // thread item = pixel p (scalars in registers) for one row offset du;
            // partners q, q+1 per packed step at constant offsets in padded rows;
            // the items of the group's row offsets are flattened for balance
            auto stage1 = [&](auto zc_c) {
                constexpr bool ZC = decltype(zc_c)::value;
                for (int itg = tid; itg < total; itg += NT) {
                    static_for<g0, g0 + C::G>([&](auto du_c) {
                        constexpr int du = decltype(du_c)::value;
                        constexpr int dv0 = (du == 0) ? 1 : -(S - 1);
                        constexpr int ndv = C::ndv_of(du);
                        constexpr int NK2 = (ndv + 1) / 2;
                        constexpr int i0 = C::item_off(du), cnt = (RH - du) * RW;
                        constexpr int pl = C::plane_off(du);
                        if (C::G == 1 || (itg >= i0 && itg < i0 + cnt)) {
                            const int it = itg - i0;
                            const int py = it / RW, px = it - py * RW;
                            const int pidx = py * RWS + PADC + px;
                            const float4 a4 = lds_f4(sA + pidx), b4 = lds_f4(sB + pidx);
                            const Pix p = {a4.x, a4.z, b4.x, b4.z};
                            const ulonglong2 *qa = reinterpret_cast<const ulonglong2 *>(sA + pidx + du * RWS + dv0);
                            const ulonglong2 *qb = reinterpret_cast<const ulonglong2 *>(sB + pidx + du * RWS + dv0);
        #pragma unroll
                            for (int kk = 0; kk < NK2; kk++) {
                                const ulonglong2 A2 = lds_u2(qa + 2 * kk), B2 = lds_u2(qb + 2 * kk);
                                const Pair2 q = {{A2.x}, {A2.y}, {B2.x}, {B2.y}};
                                P2 da, dl;
                                pair_values2<FAM, ST, PC, ZC>(p, q, kp, da, dl);
                                const int k0 = pl + 2 * kk;
                                const bool second = 2 * kk + 1 < ndv;
                                if constexpr (BOTH) {
                                    sD[k0 * RN + it] = make_float2(lo2(da), lo2(dl));
                                    if (second) sD[(k0 + 1) * RN + it] = make_float2(hi2(da), hi2(dl));
                                } else if constexpr (C::NEED_A) {
                                    sD[k0 * RN + it] = lo2(da);
                                    if (second) sD[(k0 + 1) * RN + it] = hi2(da);
                                } else {
                                    sD[k0 * RN + it] = lo2(dl);
                                    if (second) sD[(k0 + 1) * RN + it] = hi2(dl);
                                }
                            }
                        }
                    });
                }
            };
            if (zchk) stage1(std::true_type{});
            else stage1(std::false_type{});
            __syncthreads();
            // ---- stage 2: window aggregation from the planes ------------------
            // rows r = 0 .. S-du-1+OPT-1 below the thread's first output row feed
            // output o's window row u = r - o.
            const DT *dbase = sD + (ty * OPT) * RW + tx;
            static_for<g0, g0 + C::G>([&](auto du_c) {
                constexpr int du = decltype(du_c)::value;
                constexpr int dv0 = (du == 0) ? 1 : -(S - 1);
                constexpr int ndv = C::ndv_of(du);
                constexpr int pl = C::plane_off(du);
                static_for<0, ndv>([&](auto k_c) {
                    constexpr int k = decltype(k_c)::value;
                    constexpr int dv = dv0 + k;
                    constexpr int vlo = dv < 0 ? -dv : 0, vhi = dv > 0 ? S - dv : S;
#pragma unroll
                    for (int r = 0; r < S - du + OPT - 1; r++) {
#pragma unroll
                        for (int v = vlo; v < vhi; v++) {
                            const DT val = dbase[(pl + k) * RN + r * RW + v];
#pragma unroll
                            for (int o = 0; o < OPT; o++) {
                                const int u = r - o;
                                if (u < 0 || u + du >= S) continue;
                                const int i = u * S + v, j = (u + du) * S + v + dv;
                                if constexpr (BOTH) {
                                    const P2 x = *reinterpret_cast<const P2 *>(&val);
                                    ag[o][i] = add2(ag[o][i], x);
                                    ag[o][j] = add2(ag[o][j], x);
                                } else if constexpr (C::NEED_A) {
                                    aA[o][i] += val;
                                    aA[o][j] += val;
                                } else {
                                    aL[o][i] += val;
                                    aL[o][j] += val;
                                }
                                if constexpr (CEN) {
                                    if (j == DC) cen[o][i] = val;
                                    else if (i == DC) cen[o][j] = val;
                                }
                            }
                        }
                    }
                });
            });
            __syncthreads();
        });


        // ---- stage 3: selection -> the tile's output colours in sOut --------
        // (tile coordinates re-read: not held live through the stages; the
        // next tile publishes into the other parity slot)
        const int tile_x0b = s_tile[par][0], tile_y0b = s_tile[par][1], frameb = s_tile[par][2];
        uint8_t *sOut = sOut0 + par * C::kOutBuf;
        const int ox = tile_x0b + tx;
#pragma unroll
        for (int o = 0; o < OPT; o++) {
            const int ry0 = ty * OPT + o;  // window top row in region coordinates
            const int oy = tile_y0b + ry0;
            const bool valid = (oy < kp.out_rows) && (ox < kp.W);
        uint32_t kc;
            bool doubt;
            {
                // window colours: up to 5x5 loaded once into registers for the
                // selection's passes (every pick reads each candidate's colour
                // twice); 7x7 reads them from shared memory (49 more registers
                // would spill the aggregates)
                constexpr bool WCR = N <= 25;
                uint32_t wc[WCR ? N : 1];
                if constexpr (WCR) {
#pragma unroll
                    for (int i = 0; i < N; i++) wc[i] = sK[(ry0 + i / S) * RW + tx + i % S];
                }
                auto col = [&](auto ic) {
                    constexpr int i = decltype(ic)::value;
                    if constexpr (WCR) return wc[i];
                    else return sK[(ry0 + i / S) * RW + tx + i % S];
                };
                if constexpr (BOTH) {
                    auto A = [&](auto ic) { return lo2(ag[o][decltype(ic)::value]); };
                    auto L = [&](auto ic) { return hi2(ag[o][decltype(ic)::value]); };
                    auto AD = [&](auto ic) { if constexpr (CEN) return cen[o][decltype(ic)::value].x; else return 0.f; };
                    auto LD = [&](auto ic) { if constexpr (CEN) return cen[o][decltype(ic)::value].y; else return 0.f; };
                    select_window<FAM, ST, N, DC>(kp, A, L, AD, LD, col, kc, doubt);
                } else if constexpr (C::NEED_A) {
                    auto V = [&](auto ic) { return aA[o][decltype(ic)::value]; };
                    auto Z = [](auto) { return 0.f; };
                    select_window<FAM, ST, N, DC>(kp, V, V, Z, Z, col, kc, doubt);
                } else {
                    auto V = [&](auto ic) { return aL[o][decltype(ic)::value]; };
                    auto Z = [](auto) { return 0.f; };
                    auto CD = [&](auto ic) { if constexpr (CEN) return cen[o][decltype(ic)::value]; else return 0.f; };
                    select_window<FAM, ST, N, DC>(kp, V, V, Z, CD, col, kc, doubt);
                }
            }

        if (kp.dbg != nullptr && valid) {
                float *d = kp.dbg + ((long long)frameb * kp.out_rows * kp.W + (long long)oy * kp.W + ox) * (2 * N);
#pragma unroll
                for (int i = 0; i < N; i++) {
                    if constexpr (BOTH) {
                        d[i] = lo2(ag[o][i]);
                        d[N + i] = hi2(ag[o][i]);
                    } else {
                        d[i] = C::NEED_A ? aA[o][i] : 0.f;
                        d[N + i] = C::NEED_L ? aL[o][i] : 0.f;
                    }
                }
            }

            {
                uint8_t *op = sOut + ry0 * 96 + 3 * tx;
                op[0] = (uint8_t)(kc & 0xff);
                op[1] = (uint8_t)((kc >> 8) & 0xff);
                op[2] = (uint8_t)((kc >> 16) & 0xff);
            }
            if (valid && doubt && !kp.diag_no_fixup) {
                const unsigned slot = atomicAdd(&s_nflag, 1u);
                s_flag[slot] = (uint16_t)((ry0 << 5) | tx);
            }
        }

        // ---- stage 4: float64 re-decision of this tile's doubtful pixels ----
        // All threads evaluate the window's pair table (the planes' shared
        // memory is free now), one warp aggregates and selects; the result
        // replaces the pixel's colour in sOut.
        __syncthreads();
        const unsigned nflag = s_nflag;
        if (nflag != 0) {
            if (tid == 0) atomicAdd(kp.flag_count, nflag);
            constexpr int P = N * (N - 1) / 2;
            static_assert(N * sizeof(E64) + 2 * P * sizeof(double) <= C::NPL * C::RN * sizeof(DT),
                          "float64 scratch must fit in the plane buffer");
            E64 *e64 = reinterpret_cast<E64 *>(sD);
            double *dA = reinterpret_cast<double *>(e64 + N);
            double *dL = dA + P;
            const FParams &fp = kp.fp;
            for (unsigned f = 0; f < nflag; f++) {
                const int code = s_flag[f];
                const int ry0 = code >> 5, cx = code & 31;
                for (int i = tid; i < N; i += NT) {
                    const uint32_t col = sK[(ry0 + i / S) * RW + cx + i % S];
                    prep64(make_float4((float)(col & 0xff), (float)((col >> 8) & 0xff), (float)((col >> 16) & 0xff),
                                       0.f),
                           ST, e64[i]);
                }
                __syncthreads();
                pair_tables<false>(e64, fp, tid, NT, dA, dL, C::NEED_A, C::NEED_L);
                __syncthreads();
                if (ty == 0) {
                    bool close;
                    const int bb = decide64<N, FAM, ST>(e64, fp, tx, dA, dL, &close);
                    if (tx == 0) { s_b = bb; s_close = close; }
                }
                __syncthreads();
                if (ST == ST_EXACT && C::NEED_A && s_close) {
                    // pass 2: correctly rounded arccos (dfg_f64.cuh)
                    if (tid == 0) atomicAdd(kp.flag_count + 1, 1u);
                    pair_tables<true>(e64, fp, tid, NT, dA, dL, C::NEED_A, C::NEED_L);
                    __syncthreads();
                    if (ty == 0) {
                        bool close;
                        const int bb = decide64<N, FAM, ST>(e64, fp, tx, dA, dL, &close);
                        if (tx == 0) s_b = bb;
                    }
                    __syncthreads();
                }
                if (tid == 0) {
                    const int bb = s_b;
                    const uint32_t col = sK[(ry0 + bb / S) * RW + cx + bb % S];
                    uint8_t *op = sOut + ry0 * 96 + 3 * cx;
                    op[0] = (uint8_t)(col & 0xff);
                    op[1] = (uint8_t)((col >> 8) & 0xff);
                    op[2] = (uint8_t)((col >> 16) & 0xff);
                }
                __syncthreads();
            }
        }

        // ---- the tile's colours -> global memory -----------------------------
        // (bulk store: issued after the tile's last barrier; it overlaps the
        // next tile and is waited for two tiles later)
        if (kp.tma_out) {
            fence_proxy_async();  // sOut writes visible to the bulk copy
        } else {
            __syncthreads();
            for (int b = tid; b < TH * 96; b += NT) {
                const int ry = b / 96, xb = b - ry * 96;
                if (tile_y0b + ry < kp.out_rows && tile_x0b * 3 + xb < 3 * kp.W)
                    out[(long long)frameb * kp.out_fstride + (long long)(tile_y0b + ry) * kp.out_pitch + 3 * tile_x0b + xb] =
                        sOut[b];
            }
        }
        __syncthreads();  // the next tile reuses every buffer
        if (kp.tma_out && tid == 0) tma_store_3d(&kp.tm_out, 3 * tile_x0b, tile_y0b, frameb, sOut);
    }
    if (threadIdx.x == 0 && kp.tma_out) tma_store_wait_all();
}

// Per (window, family) launch shape: OPT outputs per thread (register
// blocking), TR thread-rows per CTA, MINB CTAs per SM.  Register-resident
// state per output is n (BVDF/VMF), 2n (DDF, CWVMF) or 4n (ACWDDF, CWDDF) floats.
template <int FAM, int ST, int PC>
cudaError_t launch_w3(cudaStream_t st, const uint8_t *in, uint8_t *out, const KParams &kp);  // dfg_w3.cuh

template <int S, int FAM, int ST>
struct Shape {
    static constexpr int AGG =
        ((FamT<FAM>::A ? 1 : 0) + (FamT<FAM>::L ? 1 : 0)) * (FamT<FAM>::CEN ? 2 : 1) * S * S;
    static constexpr int OPT = (S >= 5 && 2 * AGG + 32 <= 131) ? 2 : 1;
    static constexpr int REG = OPT * AGG + 56;  // registers per thread, estimated (aggregates + working set)
    // The register file is split per SM sub-partition (16K registers each),
    // so the bound is warps per sub-partition, not per SM.
    static constexpr int WPS = 16384 / (REG * 32);
    static constexpr int TR0 = WPS >= 4 ? 8 : 4 * (WPS < 2 ? 2 : WPS);
    static constexpr int MINB0 = WPS >= 4 ? (WPS / 2 > 4 ? 4 : WPS / 2) : 1;
    // 5x5 / 7x7 minimax shapes that would run two CTAs per SM run one CTA
    // of twice the warps instead: a taller tile (less halo re-evaluation:
    // C4 DDF 432 -> 720 region pixels for 256 -> 512 outputs), the same
    // warps per SM, no register spills at 128 (measured: ddf:minimax 4.53 ->
    // 3.63 ms, bvdf:minimax 2.59 -> 2.30; the chromaticity route, lighter
    // per pair, keeps two CTAs with pixel-pair items: 1.35 vs 1.89 ms);
    // 3x3 BVDF/DDF/VMF: 2 CTAs of 16 warps at 64 registers
    static constexpr bool WIDE = S >= 5 && MINB0 >= 2 && ST == ST_MINIMAX;
    // (a 12-warp CTA with pixel-pair items measured 40-50 % slower for the
    // minimax shapes: bvdf 3.08 vs 2.21 ms, ddf 5.27 vs 3.56)
    static constexpr int TR = (S == 3 && !FamT<FAM>::CEN) ? 16 : (WIDE ? 2 * TR0 : TR0);
    static constexpr int MINB = (S == 3 && !FamT<FAM>::CEN) ? 2 : (WIDE ? MINB0 / 2 : MINB0);
};

template <int S, int FAM, int ST, int PC>
cudaError_t launch_fast(cudaStream_t st, const uint8_t *in, uint8_t *out, const KParams &kp)
{
    if constexpr (S == 3) {
        // 3x3: the warp-synchronous row-sweep kernel (dfg_w3.cuh) from C1's
        // 512^2 up (9 K strip-rows: 28 vs 35 us on the config image); for
        // very small inputs (< 8 K strip-rows, e.g. 256^2) the CTA kernel's
        // finer tiles win.  DFG_OPT_S3_SCHEDULE forces one (both are
        // parity-tested).
        const int force = options().s3_schedule;
        const long long strip_rows = (long long)((kp.W + 29) / 30) * kp.out_rows * kp.n_frames;
        const bool w3 = kp.in_pitch <= 0xffffffffLL &&
                        (force ? force == 1 : (kp.w3_rpc > 0 || strip_rows >= 8192));
        if (w3) return launch_w3<FAM, ST, PC>(st, in, out, kp);
    }
    using SH = Shape<S, FAM, ST>;
    using C = Cfg<S, FAM, SH::OPT, SH::TR>;
    auto kern = dfg_fast_kernel<S, FAM, ST, PC, SH::OPT, SH::TR, SH::MINB>;
    static int resident[64] = {};  // CTAs per SM, per device
    int dev = 0;
    cudaGetDevice(&dev);
    if (resident[dev & 63] == 0) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
        if (e != cudaSuccess) return e;
        int nb = 0;
        e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&nb, kern, C::NT, C::kSmem);
        if (e != cudaSuccess) return e;
        resident[dev & 63] = nb > 0 ? nb : 1;
    }
    KParams k2 = kp;
    // bulk tensor maps over the input / output rows (uint8, 3W bytes wide)
    const int box_in[3] = {C::kRawPitch, C::RH, 1}, box_out[3] = {96, C::TH, 1};
    k2.tma_in = (options().tma & 1) && encode_rows_map(&k2.tm_in, in, 3LL * kp.W, kp.in_rows, kp.n_frames, kp.in_pitch,
                                                 kp.in_fstride, box_in);
    k2.tma_out = (options().tma & 2) && encode_rows_map(&k2.tm_out, out, 3LL * kp.W, kp.out_rows, kp.n_frames,
                                                  kp.out_pitch, kp.out_fstride, box_out);
    // persistent CTAs: one wave, each walking tiles
    const long long tiles = (long long)((kp.W + 31) / 32) * ((kp.out_rows + C::TH - 1) / C::TH) * kp.n_frames;
    const long long slots = (long long)sm_count(dev) * resident[dev & 63];
    const int grid = (int)(tiles < slots || !options().persist ? tiles : slots);
    kern<<<grid, C::NT, C::kSmem, st>>>(in, out, k2);
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

#define DFG_DEFINE_LAUNCH_CWVMF(S)                                                  \
    cudaError_t dfg_launch_s##S##_cwvmf(int, int pcode, cudaStream_t st,            \
                                        const uint8_t *in, uint8_t *out,            \
                                        const dfg::KParams &kp)                     \
    {                                                                               \
        DFG_P_SWITCH(S, dfg::FAM_CWVMF, dfg::ST_EXACT)                              \
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

// DDF / ACWDDF / CWDDF: 3 strategies x 3 Minkowski orders.  One translation
// unit per Minkowski order (build time: the 7x7 kernels take ~30 s each):
// ..._PC defines that order's launcher, ..._DISPATCH (in the p = 2 unit) the
// family launcher over the three.
#define DFG_DEFINE_LAUNCH_PAIRED_PC(S, FAM, FAMNAME, PCNAME, PC)                    \
    cudaError_t dfg_launch_s##S##_##FAMNAME##_##PCNAME(int strategy, cudaStream_t st, \
                                                       const uint8_t *in, uint8_t *out, \
                                                       const dfg::KParams &kp)      \
    {                                                                               \
        if (strategy == dfg::ST_EXACT) return dfg::launch_fast<S, FAM, dfg::ST_EXACT, PC>(st, in, out, kp); \
        if (strategy == dfg::ST_MINIMAX) return dfg::launch_fast<S, FAM, dfg::ST_MINIMAX, PC>(st, in, out, kp); \
        return dfg::launch_fast<S, FAM, dfg::ST_CHROMA, PC>(st, in, out, kp);       \
    }

#define DFG_DEFINE_LAUNCH_PAIRED_DISPATCH(S, FAMNAME)                               \
    cudaError_t dfg_launch_s##S##_##FAMNAME##_p1(int, cudaStream_t, const uint8_t *, uint8_t *, const dfg::KParams &); \
    cudaError_t dfg_launch_s##S##_##FAMNAME##_pgen(int, cudaStream_t, const uint8_t *, uint8_t *, const dfg::KParams &); \
    cudaError_t dfg_launch_s##S##_##FAMNAME(int strategy, int pcode, cudaStream_t st, \
                                            const uint8_t *in, uint8_t *out,        \
                                            const dfg::KParams &kp)                 \
    {                                                                               \
        if (pcode == dfg::PC_2) return dfg_launch_s##S##_##FAMNAME##_p2(strategy, st, in, out, kp); \
        if (pcode == dfg::PC_1) return dfg_launch_s##S##_##FAMNAME##_p1(strategy, st, in, out, kp); \
        return dfg_launch_s##S##_##FAMNAME##_pgen(strategy, st, in, out, kp);       \
    }
