// dfg_noise.cu -- the reference's correlated impulsive noise simulator
// (paper Eq. 8; reference noise.py:85-116) on the device, bit-exact with its
// PCG64 stream.
//
// Stream contract (noise.py:13-19): every pixel, in row-major order,
// consumes five uniform doubles [event, branch, r1, r2, r3] from a numpy
// PCG64 generator; a double is (next_uint64 >> 11) * 2^-53 and next_uint64
// is the XSL-RR output of the 128-bit LCG state after one step.  A thread
// owns a run of consecutive pixels: it jumps the LCG to draw 5*i0 in
// O(log i0) 128-bit steps and then steps sequentially, so the whole image is
// generated in one launch with no host round trip.  The host passes the
// generator's initial (state, inc) -- numpy's SeedSequence seeding stays on
// the host, where the reference computes it too.
#include <cuda_runtime.h>
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

// PCG_DEFAULT_MULTIPLIER_128
__device__ __constant__ u128 kMult = {0x2360ED051FC65DA4ull, 0x4385DF649FCCF645ull};

// state after `delta` LCG steps (standard jump-ahead: A^d, C (A^d - 1)/(A - 1))
__device__ u128 advance(u128 state, u128 inc, unsigned long long delta)
{
    u128 acc_mult = {0, 1}, acc_plus = {0, 0}, cur_mult = kMult, cur_plus = inc;
    while (delta) {
        if (delta & 1ull) {
            acc_mult = mul128(acc_mult, cur_mult);
            acc_plus = add128(mul128(acc_plus, cur_mult), cur_plus);
        }
        cur_plus = mul128(add128(cur_mult, u128{0, 1}), cur_plus);
        cur_mult = mul128(cur_mult, cur_mult);
        delta >>= 1;
    }
    return add128(mul128(acc_mult, state), acc_plus);
}

__device__ __forceinline__ double next_double(u128 &s, const u128 inc)
{
    s = add128(mul128(s, kMult), inc);
    const uint64_t x = s.hi ^ s.lo;
    const unsigned rot = (unsigned)(s.hi >> 58);
    const uint64_t out = (x >> rot) | (x << ((64u - rot) & 63u));
    return (double)(out >> 11) * (1.0 / 9007199254740992.0);
}

constexpr int kRun = 16;  // pixels per thread

__global__ void __launch_bounds__(256) dfg_noise_kernel(const uint8_t *in, uint8_t *out,
                                                        int H, int W, long long in_pitch, long long out_pitch,
                                                        dfg_noise_params np)
{
    const long long npx = (long long)H * W;
    const long long i0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * kRun;
    if (i0 >= npx) return;
    const u128 inc = {np.inc_hi, np.inc_lo};
    u128 s = advance(u128{np.state_hi, np.state_lo}, inc, 5ull * (unsigned long long)i0);
    // branch thresholds exactly as the reference forms them (noise.py:103-105)
    const double c1 = np.phi1, c2 = np.phi1 + np.phi2, c3 = np.phi1 + np.phi2 + np.phi3;
    const long long i1 = i0 + kRun < npx ? i0 + kRun : npx;
    for (long long i = i0; i < i1; i++) {
        const double u_event = next_double(s, inc), u_branch = next_double(s, inc);
        double u[3];
        u[0] = next_double(s, inc);
        u[1] = next_double(s, inc);
        u[2] = next_double(s, inc);
        const int r = (int)(i / W), c = (int)(i - (long long)r * W);
        const uint8_t *p = in + r * in_pitch + 3LL * c;
        uint8_t *o = out + r * out_pitch + 3LL * c;
        uint8_t v[3] = {p[0], p[1], p[2]};
        if (u_event < np.phi) {
            uint8_t imp[3];
            for (int k = 0; k < 3; k++)  // noise.py:98-101 (saltpepper / uniform)
                imp[k] = np.impulse == 0 ? (u[k] < 0.5 ? 0 : 255) : (uint8_t)(int)floor(u[k] * 256.0);
            if (u_branch < c1) v[0] = imp[0];
            else if (u_branch < c2) v[1] = imp[1];
            else if (u_branch < c3) v[2] = imp[2];
            else { v[0] = imp[0]; v[1] = imp[1]; v[2] = imp[2]; }
        }
        o[0] = v[0];
        o[1] = v[1];
        o[2] = v[2];
    }
}

}  // namespace

extern "C" DFG_API int dfg_corrupt_image(const uint8_t *d_in, int32_t H, int32_t W, int64_t in_pitch,
                                         uint8_t *d_out, int64_t out_pitch, const dfg_noise_params *np,
                                         void *stream)
{
    if (!d_in || !d_out || !np || H < 1 || W < 1 || in_pitch < 3LL * W || out_pitch < 3LL * W) return DFG_E_ARG;
    if (!(np->phi >= 0.0 && np->phi <= 1.0) || np->phi1 < 0 || np->phi2 < 0 || np->phi3 < 0 ||
        np->phi1 + np->phi2 + np->phi3 > 1.0 + 1e-12 || (np->impulse != 0 && np->impulse != 1))
        return DFG_E_ARG;  // NoiseParams validation (noise.py:42-55)
    const long long npx = (long long)H * W;
    const long long threads = (npx + kRun - 1) / kRun;
    const unsigned blocks = (unsigned)((threads + 255) / 256);
    dfg_noise_kernel<<<blocks, 256, 0, (cudaStream_t)stream>>>(d_in, d_out, H, W, in_pitch, out_pitch, *np);
    return cudaGetLastError() == cudaSuccess ? DFG_OK : DFG_E_CUDA;
}
