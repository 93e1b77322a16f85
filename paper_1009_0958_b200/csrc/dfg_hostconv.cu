// dfg_hostconv.cu -- host-side conversions of the float64 drop-in boundary
// (dfg_filter_host_f64): the reference's pixel array holds integers 0..255
// as float64 (image.py:65-75); the device path reads and writes uint8.
// Host code only.  AVX2 forms (runtime-dispatched) run ~5x the scalar loops,
// which were the float64 path's bottleneck (10 cycles per value).
#include <immintrin.h>
#include <stddef.h>
#include <stdint.h>

#include "../../include/dirfilt_gpu.h"

namespace dfg {

namespace {

unsigned f64_to_u8_scalar(const double *src, uint8_t *dst, size_t lo, size_t hi)
{
    unsigned b = 0;
    for (size_t i = lo; i < hi; i++) {
        const double v = src[i];
        const double c = (v >= 0.0 && v <= 255.0) ? v : -1.0;
        const int iv = (int)c;
        b |= (unsigned)((double)iv != c) | (unsigned)(iv < 0);
        dst[i] = (uint8_t)iv;
    }
    return b;
}

void u8_to_f64_scalar(const uint8_t *src, double *dst, size_t lo, size_t hi)
{
    for (size_t i = lo; i < hi; i++) dst[i] = (double)src[i];
}

#if defined(__x86_64__)
__attribute__((target("avx2"))) unsigned f64_to_u8_avx2(const double *src, uint8_t *dst, size_t lo, size_t hi)
{
    size_t i = lo;
    __m256d neq = _mm256_setzero_pd();   // lanes whose value is not its own truncation (incl. NaN)
    __m128i rng = _mm_setzero_si128();   // bits outside 0..255 (incl. the 0x80000000 of inf / huge values)
    const __m128i hi_bits = _mm_set1_epi32(~0xff);
    for (; i + 16 <= hi; i += 16) {
        __m128i q[4];
        for (int k = 0; k < 4; k++) {
            const __m256d v = _mm256_loadu_pd(src + i + 4 * k);
            const __m128i iv = _mm256_cvttpd_epi32(v);
            neq = _mm256_or_pd(neq, _mm256_cmp_pd(v, _mm256_cvtepi32_pd(iv), _CMP_NEQ_UQ));
            rng = _mm_or_si128(rng, _mm_and_si128(iv, hi_bits));
            q[k] = iv;
        }
        const __m128i w0 = _mm_packus_epi32(q[0], q[1]), w1 = _mm_packus_epi32(q[2], q[3]);
        _mm_storeu_si128(reinterpret_cast<__m128i *>(dst + i), _mm_packus_epi16(w0, w1));
    }
    unsigned b = (unsigned)(_mm256_movemask_pd(neq) != 0) | (unsigned)(!_mm_testz_si128(rng, rng));
    if (i < hi) b |= f64_to_u8_scalar(src, dst, i, hi);
    return b;
}

__attribute__((target("avx2"))) void u8_to_f64_avx2(const uint8_t *src, double *dst, size_t lo, size_t hi)
{
    size_t i = lo;
    while (i < hi && ((uintptr_t)(dst + i) & 31)) {  // to a 32-byte aligned destination
        dst[i] = (double)src[i];
        i++;
    }
    // streaming stores: the result is written once and not read back here
    for (; i + 16 <= hi; i += 16) {
        const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i *>(src + i));
        const __m256i a0 = _mm256_cvtepu8_epi32(b), a1 = _mm256_cvtepu8_epi32(_mm_srli_si128(b, 8));
        _mm256_stream_pd(dst + i, _mm256_cvtepi32_pd(_mm256_castsi256_si128(a0)));
        _mm256_stream_pd(dst + i + 4, _mm256_cvtepi32_pd(_mm256_extracti128_si256(a0, 1)));
        _mm256_stream_pd(dst + i + 8, _mm256_cvtepi32_pd(_mm256_castsi256_si128(a1)));
        _mm256_stream_pd(dst + i + 12, _mm256_cvtepi32_pd(_mm256_extracti128_si256(a1, 1)));
    }
    _mm_sfence();
    for (; i < hi; i++) dst[i] = (double)src[i];
}

bool have_avx2()
{
    static const bool v = __builtin_cpu_supports("avx2");
    return v;
}
#endif

}  // namespace

// Values [lo, hi) of a float64 pixel array -> uint8; nonzero when any value
// is not an integer in 0..255 (NaN and infinities included).
unsigned f64_to_u8(const double *src, uint8_t *dst, size_t lo, size_t hi)
{
#if defined(__x86_64__)
    if (have_avx2()) return f64_to_u8_avx2(src, dst, lo, hi);
#endif
    return f64_to_u8_scalar(src, dst, lo, hi);
}

void u8_to_f64(const uint8_t *src, double *dst, size_t lo, size_t hi)
{
#if defined(__x86_64__)
    if (have_avx2()) return u8_to_f64_avx2(src, dst, lo, hi);
#endif
    u8_to_f64_scalar(src, dst, lo, hi);
}

// scalar forms, for the tests that compare the two
unsigned f64_to_u8_reference(const double *src, uint8_t *dst, size_t lo, size_t hi) { return f64_to_u8_scalar(src, dst, lo, hi); }

}  // namespace dfg

extern "C" DFG_API int dfg_hostconv_selftest(const double *src, int64_t n, uint8_t *dst_fast, uint8_t *dst_ref, double *back)
{
    // returns bit 0: fast path flagged bad values, bit 1: scalar path did
    const unsigned a = dfg::f64_to_u8(src, dst_fast, 0, (size_t)n);
    const unsigned b = dfg::f64_to_u8_reference(src, dst_ref, 0, (size_t)n);
    dfg::u8_to_f64(dst_ref, back, 0, (size_t)n);
    return (int)((a ? 1u : 0u) | (b ? 2u : 0u));
}
