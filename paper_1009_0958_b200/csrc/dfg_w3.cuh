// dfg_w3.cuh -- warp-synchronous 3x3 kernel (BVDF / DDF / ACWDDF / VMF).
//
// Same arithmetic, error budget and float64 re-decision as dfg_fast.cuh, with
// a schedule built for the small window: every warp owns a strip of 32 input
// columns (30 output columns, lanes 1..30) and sweeps DOWN a chunk of rows.
// Per row step each lane
//   1. stages its new pixel into a warp-private 3-row ring of records,
//   2. evaluates the 12 pairs whose LOWER pixel is that pixel
//      (E_d(q) = d(q - d, q) for the 12 canonical offsets d: 2 in its row,
//      5 in each of the two rows above) -- each unique pixel pair once --
//      with the packed f32x2 pair math, into a 3-row ring of pair values,
//   3. aggregates the 36 window pairs of the output pixel one row above
//      (its own and its two neighbours' ring entries) and selects.
// Only __syncwarp orders the ring; no CTA barrier, no halo-row recomputation
// (the reference's row loop, _engine.py:232-487, streams rows the same way).
#pragma once

#include "dfg_fast.cuh"

namespace dfg {

template <int FAM>
struct W3Cfg {
    static constexpr bool NEED_A = FamT<FAM>::A;
    static constexpr bool NEED_L = FamT<FAM>::L;
    static constexpr bool BOTH = NEED_A && NEED_L;
    using DT = typename std::conditional<BOTH, float2, float>::type;
    static constexpr int WARPS = 2;
    // ring row: element e = 2 + l holds the pixel pair (l, l+1); element 1 =
    // (pad, pixel 0) serves lane 1's same-row partner, element 0 is the pad
    // lane 0's (unused) same-row partner load touches
    static constexpr int EOFF = 2;
    static constexpr int LANES_E = 34;
    // per-warp shared layout (bytes)
    static constexpr int REC_BYTES = 3 * LANES_E * 32;         // 2 x float4 per element (A, B)
    static constexpr int COL_BYTES = 3 * 32 * 4;               // packed colours
    // pair-value ring: offsets k 0..6 (du 0, 1) for three rows, k 7..11 (du 2)
    // for the current row only -- the window of the output one row up reads
    // du <= 1 entries of the previous row and du = 0 entries two rows up
    static constexpr int E_BYTES = (3 * 7 + 5) * 32 * (int)sizeof(DT);
    static constexpr int F64_BYTES = 9 * (int)sizeof(E64) + 2 * 36 * 8 + 16;
    static constexpr int WARP_BYTES = (REC_BYTES + COL_BYTES + E_BYTES + F64_BYTES + 15) & ~15;
    static constexpr size_t kSmem = (size_t)WARPS * WARP_BYTES;
};

// canonical offset index k of (du, dv): du = 0 -> dv 1, 2 (k 0, 1);
// du = 1 -> dv -2..2 (k 2..6); du = 2 -> dv -2..2 (k 7..11)
__host__ __device__ constexpr int w3_k(int du, int dv) { return du == 0 ? dv - 1 : 2 + (du - 1) * 5 + (dv + 2); }

// resident blocks per SM: 8 (16 warps, 128 registers) -- the launch sizes
// its chunks for whole waves of 16 resident warps per SM (launch_w3);
// measured: 18 or 20 resident warps (96 registers) run 10-14% slower
template <int ST>
constexpr int w3_minb() { return 8; }

// Float64 re-decision of one window (whole warp): lane i < 9 holds the
// packed colour of window pixel i; returns the chosen window index.
template <int FAM, int ST>
__device__ __forceinline__ int w3_decide64(const KParams &kp, unsigned char *f64b, uint32_t cc)
{
    using C = W3Cfg<FAM>;
    constexpr int N = 9;
    const int lane = threadIdx.x & 31;
    E64 *e64 = reinterpret_cast<E64 *>(f64b);
    double *dA = reinterpret_cast<double *>(e64 + N);
    double *dL = dA + 36;
    if (lane < N)
        prep64(make_float4((float)(cc & 0xff), (float)((cc >> 8) & 0xff), (float)((cc >> 16) & 0xff), 0.f), ST,
               e64[lane]);
    __syncwarp();
    pair_tables_warp<false, N>(e64, kp.fp, lane, dA, dL, C::NEED_A, C::NEED_L);
    __syncwarp();
    bool close;
    int bb = decide64<N, FAM, ST>(e64, kp.fp, lane, dA, dL, &close);
    if (ST == ST_EXACT && C::NEED_A && close) {
        if (lane == 0) atomicAdd(kp.flag_count + 1, 1u);
        __syncwarp();
        pair_tables_warp<true, N>(e64, kp.fp, lane, dA, dL, C::NEED_A, C::NEED_L);
        __syncwarp();
        bb = decide64<N, FAM, ST>(e64, kp.fp, lane, dA, dL, &close);
    }
    __syncwarp();
    return bb;
}

// Inline re-decision of the doubtful pixels `mask` of one output row segment
// from the warp's ring (window row u of the output in ring slot sl[u]), right
// after the row step that found them.
template <int FAM, int ST>
__device__ __forceinline__ void w3_redecide(const KParams &kp, const uint32_t *rK, int sl0, int sl1, int sl2,
                                         unsigned char *f64b, unsigned mask, uint8_t *orow_px)
{
    const int lane = threadIdx.x & 31;
    if (lane == 0) atomicAdd(kp.flag_count, (unsigned)__popc(mask));
    while (mask) {
        const int fl = __ffs(mask) - 1;
        mask &= mask - 1;
        const int sr = lane < 3 ? sl2 : (lane < 6 ? sl1 : sl0);
        const uint32_t cc = lane < 9 ? rK[sr * 32 + fl - 1 + lane % 3] : 0u;
        const int bb = w3_decide64<FAM, ST>(kp, f64b, cc);
        const uint32_t kb = __shfl_sync(0xffffffffu, cc, bb);
        if (lane == 0) {
            uint8_t *op = orow_px + 3 * (fl - 1);
            op[0] = (uint8_t)(kb & 0xff);
            op[1] = (uint8_t)((kb >> 8) & 0xff);
            op[2] = (uint8_t)((kb >> 16) & 0xff);
        }
    }
}

// The ring slots of rows y, y-1, y-2 rotate at run time.  (Measured in round
// 2: unrolling the row loop by the ring period with compile-time slots --
// no rotation moves, no slot arithmetic -- triples the step's code and ran
// C2 45.7 -> 54.5 us, C5b 5.22 -> 7.53 ms: the instruction cache, not the
// ~45 moves, is what the step is short of.  That experiment also showed why
// the ring's record loads must be the ORDERED helper: with loop-invariant
// addresses the compiler hoisted the plain (pure) asm loads above the
// stores of the same step.)
//
// Aggregation by column sums (per window row t, for the lane's own pixel P_t
// of that row): V_t(dv) = sum over the three window rows of d(P_t, (row,
// col(P_t) + dv)), dv in -2..2; the aggregate of P_t in the window whose
// columns are col(P_t) + {0,1,2} / {-1,0,1} / {-2,-1,0} is the sum of three
// V's, and the outputs one lane right / here / one lane left receive those
// by shuffles: 14 additions per window row (42 per output) instead of 72.
// The values are the ring entries of the 36 window pairs' lower pixels, each
// loaded by the lane of P_t (the sums cover every other window pixel once,
// so the error budget's (n-1)-term summation bound holds unchanged).
template <int FAM, int ST, int PC, int MINB>
__global__ void __launch_bounds__(64, MINB)
dfg_w3_kernel(const uint8_t *__restrict__ in, uint8_t *__restrict__ out, const __grid_constant__ KParams kp, int n_strips,
              int n_chunks)
{
    using C = W3Cfg<FAM>;
    using DT = typename C::DT;
    constexpr bool CEN = FamT<FAM>::CEN;
    constexpr bool BOTH = C::BOTH;
    constexpr int N = 9, DC = 4;

    extern __shared__ __align__(16) unsigned char w3_smem[];
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int gw = blockIdx.x * C::WARPS + warp;  // global warp id within the frame
    if (gw >= n_strips * n_chunks) return;        // whole warp exits together
    const int strip = gw % n_strips, chunk = gw / n_strips;
    const int frame = blockIdx.z;
    const uint8_t *fin = in + (long long)frame * kp.in_fstride;

    unsigned char *wb = w3_smem + warp * C::WARP_BYTES;
    float4 *rA = reinterpret_cast<float4 *>(wb);                 // [3][LANES_E]
    float4 *rB = rA + 3 * C::LANES_E;
    uint32_t *rK = reinterpret_cast<uint32_t *>(wb + C::REC_BYTES);  // [3][32]
    DT *rE = reinterpret_cast<DT *>(wb + C::REC_BYTES + C::COL_BYTES);  // [3][7][32] + [5][32]
    DT *rE2 = rE + 3 * 7 * 32;
    unsigned char *f64b = wb + C::REC_BYTES + C::COL_BYTES + C::E_BYTES;

    const int col = strip * 30 - 1 + lane;  // input column of this lane
    const int colr = resolve_idx(col, kp.W, kp.border);
    // output rows [oy0, oy1) of the chunk (strip-local)
    const int oy0 = (int)((long long)chunk * kp.out_rows / n_chunks);
    const int oy1 = (int)((long long)(chunk + 1) * kp.out_rows / n_chunks);

    // pad element 0 of every ring row: neutral, never used
    if (lane < 3) {
        rA[lane * C::LANES_E] = make_float4(1.f, 1.f, 1.f, 1.f);
        rB[lane * C::LANES_E] = make_float4(1.f, 1.f, 1.f, 1.f);
    }

    bool zr0 = false, zr1 = false;  // zero vectors in the two previous staged rows
    // the pixel of the next row step is loaded one step ahead (its HBM
    // latency hides behind the current step's pair math)
    const uint8_t *cbase = fin + colr * 3;
    const unsigned pitch = (unsigned)kp.in_pitch;  // the host keeps rows < 4 GiB
    auto row_of = [&](int yy) {
        int gy = kp.out_row0 + yy;
        if ((unsigned)gy >= (unsigned)kp.global_H) gy = resolve_idx(gy, kp.global_H, kp.border);
        return min(max(gy - kp.in_row0, 0), kp.in_rows - 1);
    };
    // chunks whose rows oy0 - 1 .. oy1 need no border resolution (all but the
    // first and last chunk of a strip) advance the pixel pointer by one row
    // per step
    const int gy_lo = kp.out_row0 + oy0 - 1, gy_hi = kp.out_row0 + oy1;
    const bool interior = gy_lo >= 0 && gy_lo >= kp.in_row0 && gy_hi < kp.global_H && gy_hi < kp.in_row0 + kp.in_rows;
    const uint8_t *npx = cbase;
    auto load_px = [&](int yy, uint32_t &r, uint32_t &g, uint32_t &b) {
        if (interior && yy != oy0 - 1) npx += pitch;
        else npx = cbase + (size_t)((unsigned long long)(unsigned)row_of(yy) * pitch);
        r = npx[0];
        g = npx[1];
        b = npx[2];
    };
    uint32_t nr8 = 0, ng8 = 0, nb8 = 0;
    load_px(oy0 - 1, nr8, ng8, nb8);
    // this lane's pixels of the previous two row steps (the vertical pair's
    // partners for lane l-2); neutral until the warm-up steps fill them
    Pix pm1 = {1.f, 1.f, 1.f, 1.f}, pm2 = {1.f, 1.f, 1.f, 1.f};

    // row step y (strip-local input row, window of output row y - 1) in ring phase PH
    auto step = [&](const int S0, const int S1, const int S2, const int y) -> unsigned {
        __syncwarp();  // the previous step's readers are done with this slot
        // ---- 1. stage the new pixel ---------------------------------------
        const uint32_t r8 = nr8, g8 = ng8, b8 = nb8;
        if (y < oy1) load_px(y + 1, nr8, ng8, nb8);
        const uint32_t rgb = r8 | (g8 << 8) | (b8 << 16);
        const bool zero = rgb == 0u;
        // gray map: the zero vector -> (1, 1, 1) (its channels are 0, so OR-ing
        // the flag in maps exactly it); exact u8 -> float without I2F: 2^23 + v,
        // minus 2^23
        const uint32_t zf = zero ? 1u : 0u;
        Pix q;
        q.x = __uint_as_float(0x4B000000u | r8 | zf) - 8388608.f;
        q.y = __uint_as_float(0x4B000000u | g8 | zf) - 8388608.f;
        q.z = __uint_as_float(0x4B000000u | b8 | zf) - 8388608.f;
        q.aux = encode_aux<ST, C::NEED_L>(q.x, q.y, q.z, zero);
        {
            // element l = pixel pair (l, l+1): the right neighbour's record by
            // shuffle, two whole 16-byte stores (lane 31's second half: unused)
            const float sx = __shfl_down_sync(0xffffffffu, q.x, 1), sy = __shfl_down_sync(0xffffffffu, q.y, 1);
            const float sz = __shfl_down_sync(0xffffffffu, q.z, 1), sa = __shfl_down_sync(0xffffffffu, q.aux, 1);
            rA[S0 * C::LANES_E + C::EOFF + lane] = make_float4(q.x, sx, q.y, sy);
            rB[S0 * C::LANES_E + C::EOFF + lane] = make_float4(q.z, sz, q.aux, sa);
            if (lane == 0) {  // element 1 = (pad, pixel 0)
                rA[S0 * C::LANES_E + 1] = make_float4(1.f, q.x, 1.f, q.y);
                rB[S0 * C::LANES_E + 1] = make_float4(1.f, q.z, 1.f, q.aux);
            }
            rK[S0 * 32 + lane] = rgb;
        }
        const bool zr2 = __any_sync(0xffffffffu, zero);
        const bool zchk = C::NEED_L && (zr0 || zr1 || zr2);  // pairs reach two rows up
        zr0 = zr1;
        zr1 = zr2;
        __syncwarp();
        // ---- 2. pair values with lower pixel q ------------------------------
        // six packed evaluations for the 12 partners: row y: element
        // (l-2, l-1); rows y-1 and y-2: elements (l-2, l-1), (l, l+1); and
        // the vertical pair {(y-1, l+2), (y-2, l+2)}, shuffled in from lane
        // l+2's own previous two pixels (no shared-memory round trip)
        Pair2 pv;
        pv.x = pk2(__shfl_down_sync(0xffffffffu, pm1.x, 2), __shfl_down_sync(0xffffffffu, pm2.x, 2));
        pv.y = pk2(__shfl_down_sync(0xffffffffu, pm1.y, 2), __shfl_down_sync(0xffffffffu, pm2.y, 2));
        pv.z = pk2(__shfl_down_sync(0xffffffffu, pm1.z, 2), __shfl_down_sync(0xffffffffu, pm2.z, 2));
        pv.aux = pk2(__shfl_down_sync(0xffffffffu, pm1.aux, 2), __shfl_down_sync(0xffffffffu, pm2.aux, 2));
        // LV: 2 = every pair; 1 = the chunk's second warm-up row (the window
        // of its first output reaches one row up: du <= 1 and the vertical
        // pair's upper half); 0 = its first warm-up row (du = 0 only)
        auto eval = [&](auto zc_c, auto lv_c) {
            constexpr bool ZC = decltype(zc_c)::value;
            constexpr int LV = decltype(lv_c)::value;
            auto need = [](int t) { return LV == 2 || t == 0 || (LV == 1 && t != 3 && t != 4); };
            auto put = [&](int k, float a, float l) {
                DT v;
                if constexpr (BOTH) v = make_float2(a, l);
                else if constexpr (C::NEED_A) v = a;
                else v = l;
                if (k < 7) rE[(S0 * 7 + k) * 32 + lane] = v;
                else rE2[(k - 7) * 32 + lane] = v;
            };
            // all partner loads first, then the six independent packed pair
            // evaluations, then the stores: the pair math chains interleave
            const int rsl[5] = {S0, S1, S1, S2, S2};
            constexpr int els[5] = {0, 0, 2, 0, 2};  // + lane; lane 0's (l-2, l-1): pads, unused
            Pair2 pp[6];
#pragma unroll
            for (int t = 0; t < 5; t++) {
                if (!need(t)) continue;
                const ulonglong2 A2 = lds_u2_ordered(rA + rsl[t] * C::LANES_E + els[t] + lane);
                const ulonglong2 B2 = lds_u2_ordered(rB + rsl[t] * C::LANES_E + els[t] + lane);
                pp[t] = {{A2.x}, {A2.y}, {B2.x}, {B2.y}};
            }
            pp[5] = pv;
            P2 da[6], dl[6];
#pragma unroll
            for (int t = 0; t < 6; t++)
                if (need(t)) pair_values2<FAM, ST, PC, ZC>(q, pp[t], kp, da[t], dl[t]);
            // du = 0: partners (l-2, l-1) = dv 2, 1
            put(w3_k(0, 2), lo2(da[0]), lo2(dl[0]));
            put(w3_k(0, 1), hi2(da[0]), hi2(dl[0]));
#pragma unroll
            for (int du = 1; du <= 2; du++) {
                const int t = 1 + 2 * (du - 1);
                if (!need(t)) continue;
                put(w3_k(du, 2), lo2(da[t]), lo2(dl[t]));  // partners l-2, l-1 -> dv = 2, 1
                put(w3_k(du, 1), hi2(da[t]), hi2(dl[t]));
                put(w3_k(du, 0), lo2(da[t + 1]), lo2(dl[t + 1]));  // partners l, l+1 -> dv = 0, -1
                put(w3_k(du, -1), hi2(da[t + 1]), hi2(dl[t + 1]));
            }
            if (need(5)) {
                put(w3_k(1, -2), lo2(da[5]), lo2(dl[5]));  // vertical pair: partner l+2 in rows y-1, y-2
                if (LV == 2) put(w3_k(2, -2), hi2(da[5]), hi2(dl[5]));
            }
        };
        // warm-up rows take the zero-checking path (correct with or without
        // zero pixels) so only the full-row variant is instantiated twice
        if (y > oy0) {
            if (zchk) eval(std::true_type{}, std::integral_constant<int, 2>{});
            else eval(std::false_type{}, std::integral_constant<int, 2>{});
        } else if (y == oy0) {
            eval(std::integral_constant<bool, C::NEED_L>{}, std::integral_constant<int, 1>{});
        } else {
            eval(std::integral_constant<bool, C::NEED_L>{}, std::integral_constant<int, 0>{});
        }
        pm2 = pm1;
        pm1 = q;
        __syncwarp();
        // ---- 3. aggregate + select for output row y - 1 ---------------------
        const int oy = y - 1;
        if (oy < oy0) return 0u;  // warm-up rows (uniform across the warp)
        const bool valid = lane >= 1 && lane < 31 && oy < oy1 && col < kp.W;
        // ring entry of the pair {P, Q}, P = (window row t, this lane),
        // Q = (window row t2, lane + dv): stored at the lower pixel's lane
        const int SL[3] = {S2, S1, S0};  // window rows 0, 1, 2 = input rows y-2, y-1, y
        auto ring = [&](int slot, int k, int off) -> DT {
            return (k < 7) ? rE[(slot * 7 + k) * 32 + lane + off] : rE2[(k - 7) * 32 + lane + off];
        };
        auto pairv = [&](int t, int t2, int dv) -> DT {
            if (t2 > t || (t2 == t && dv > 0)) return ring(SL[t2], w3_k(t2 - t, dv), dv);  // Q lower
            return ring(SL[t], w3_k(t - t2, -dv), 0);                                      // P lower
        };
        using AG = typename std::conditional<BOTH, P2, float>::type;
        auto toag = [](DT v) -> AG {
            if constexpr (BOTH) return *reinterpret_cast<const P2 *>(&v);
            else return v;
        };
        auto agadd = [](AG a, AG b) -> AG {
            if constexpr (BOTH) return add2(a, b);
            else return a + b;
        };
        AG ag[N];
#pragma unroll
        for (int t = 0; t < 3; t++) {
            AG V[5];
#pragma unroll
            for (int dv = -2; dv <= 2; dv++) {
                AG acc{};
                bool first = true;
#pragma unroll
                for (int t2 = 0; t2 < 3; t2++) {
                    if (t2 == t && dv == 0) continue;  // the pixel itself: self term below
                    const AG x = toag(pairv(t, t2, dv));
                    acc = first ? x : agadd(acc, x);
                    first = false;
                }
                V[dv + 2] = acc;
            }
            if constexpr (ST == ST_MINIMAX && C::NEED_A) {  // the self term (angular only)
                if constexpr (BOTH) V[2] = add2(V[2], pk2(kp.self_term, 0.f));
                else V[2] += kp.self_term;
            }
            const AG a = agadd(V[2], V[3]);
            const AG aR = agadd(a, V[4]);                 // window columns +0..+2: output one lane right
            const AG aC = agadd(a, V[1]);                 // -1..+1: this lane's output
            const AG aL = agadd(agadd(V[0], V[1]), V[2]);  // -2..0: output one lane left
            if constexpr (BOTH) {
                ag[3 * t + 0].v = __shfl_up_sync(0xffffffffu, aR.v, 1);
                ag[3 * t + 2].v = __shfl_down_sync(0xffffffffu, aL.v, 1);
            } else {
                ag[3 * t + 0] = __shfl_up_sync(0xffffffffu, aR, 1);
                ag[3 * t + 2] = __shfl_down_sync(0xffffffffu, aL, 1);
            }
            ag[3 * t + 1] = aC;
        }
        DT cen[CEN ? N : 1];  // centre column d(i, centre): the centre is (window row 1, this lane)
        if constexpr (CEN) {
#pragma unroll
            for (int i = 0; i < N; i++) {
                const int u = i / 3, v = i % 3;
                if (i == DC) {
                    if constexpr (BOTH) cen[i] = make_float2(kp.self_term, 0.f);
                    else cen[i] = C::NEED_A ? kp.self_term : 0.f;
                } else if (u == 0) cen[i] = ring(S1, w3_k(1, 1 - v), 0);  // centre lower
                else if (u == 1) cen[i] = v == 0 ? ring(S1, w3_k(0, 1), 0) : ring(S1, w3_k(0, 1), 1);
                else cen[i] = ring(S0, w3_k(1, v - 1), v - 1);            // pixel i lower
            }
        }
        // colours of the window (rings hold input rows oy-1, oy, oy+1)
        const int lc = min(max(lane, 1), 30);  // clamp so lanes 0/31 read in-bounds (results unused)
        uint32_t wc[N];
#pragma unroll
        for (int i = 0; i < N; i++) wc[i] = rK[SL[i / 3] * 32 + lc - 1 + i % 3];
        uint32_t cb;
        bool doubt;
        {
            auto colf = [&](auto ic) { return wc[decltype(ic)::value]; };
            if constexpr (BOTH) {
                auto A = [&](auto ic) { return lo2(ag[decltype(ic)::value]); };
                auto L = [&](auto ic) { return hi2(ag[decltype(ic)::value]); };
                auto AD = [&](auto ic) { if constexpr (CEN) return cen[decltype(ic)::value].x; else return 0.f; };
                auto LD = [&](auto ic) { if constexpr (CEN) return cen[decltype(ic)::value].y; else return 0.f; };
                select_window<FAM, ST, N, DC>(kp, A, L, AD, LD, colf, cb, doubt);
            } else {
                auto V = [&](auto ic) { return ag[decltype(ic)::value]; };
                auto Z = [](auto) { return 0.f; };
                auto CD = [&](auto ic) { if constexpr (CEN) return cen[decltype(ic)::value]; else return 0.f; };
                select_window<FAM, ST, N, DC>(kp, V, V, Z, CD, colf, cb, doubt);
            }
        }
        uint8_t *orow = out + (long long)frame * kp.out_fstride + (long long)oy * kp.out_pitch;
        if (kp.dbg != nullptr && valid) {
            float *d = kp.dbg + ((long long)frame * kp.out_rows * kp.W + (long long)oy * kp.W + col) * (2 * N);
#pragma unroll
            for (int i = 0; i < N; i++) {
                if constexpr (BOTH) {
                    d[i] = lo2(ag[i]);
                    d[N + i] = hi2(ag[i]);
                } else {
                    d[i] = C::NEED_A ? ag[i] : 0.f;
                    d[N + i] = C::NEED_L ? ag[i] : 0.f;
                }
            }
        }
        // ---- 4. write; doubtful pixels are re-decided by the caller ---------
        if (valid) {
            uint8_t *op = orow + col * 3;
            op[0] = (uint8_t)(cb & 0xff);
            op[1] = (uint8_t)((cb >> 8) & 0xff);
            op[2] = (uint8_t)((cb >> 16) & 0xff);
        }
        return __ballot_sync(0xffffffffu, valid && doubt && !kp.diag_no_fixup);
    };
    int s0 = 0, s1 = 2, s2 = 1;  // ring slots of rows y, y-1, y-2 (rotated each step)
    for (int y = oy0 - 1; y <= oy1; y++) {
        const unsigned mask = step(s0, s1, s2, y);
        if (mask) {
            uint8_t *orow = out + (long long)frame * kp.out_fstride + (long long)(y - 1) * kp.out_pitch;
            w3_redecide<FAM, ST>(kp, rK, s0, s1, s2, f64b, mask, orow + strip * 30 * 3);
        }
        const int t = s2;
        s2 = s1;
        s1 = s0;
        s0 = t;
    }
}

template <int FAM, int ST, int PC>
cudaError_t launch_w3(cudaStream_t st, const uint8_t *in, uint8_t *out, const KParams &kp)
{
    using C = W3Cfg<FAM>;
    constexpr int minb = w3_minb<ST>();
    auto kern = dfg_w3_kernel<FAM, ST, PC, minb>;
    static unsigned long long configured = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(configured & (1ull << (dev & 63)))) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
        if (e != cudaSuccess) return e;
        configured |= 1ull << (dev & 63);
    }
    const Options &opt = options();
    const long long sms = sm_count(dev);
    const int n_strips = (kp.W + 29) / 30;
    // chunks per strip: fill whole waves of resident warps (wps per SM) with
    // equal row counts (chunk c covers rows [c R / n, (c+1) R / n)), at most
    // 64 rows per chunk; every chunk pays 2 warm-up row steps
    const long long cols = (long long)n_strips * kp.n_frames;  // independent strip columns
    const long long strip_rows = cols * kp.out_rows;
    // small single-wave frames (< 8 rows per chunk at 16 warps per SM): 12
    // warps per SM with longer chunks (C1 512^2: 22.6 -> 21.0 us; C2's 15-row
    // chunks stay at 16 warps: 12 measured 4.5 % slower there)
    long long wps = opt.w3_wps > 0 ? opt.w3_wps : 2 * minb;
    if (opt.w3_wps <= 0 && opt.w3_small_wps > 0 && strip_rows < 8LL * sms * wps) wps = opt.w3_small_wps;
    const long long slots = sms * wps;
    const long long waves = (strip_rows + slots * 64 - 1) / (slots * 64);
    long long n_chunks = (waves * slots) / cols;
    const int rpc_hint = opt.w3_rpc > 0 ? opt.w3_rpc : kp.w3_rpc;  // host pipeline bands: short chunks
    if (rpc_hint > 0) n_chunks = (kp.out_rows + rpc_hint - 1) / rpc_hint;
    n_chunks = n_chunks < 1 ? 1 : (n_chunks > kp.out_rows ? kp.out_rows : n_chunks);
    n_chunks = n_chunks < (kp.out_rows + 63) / 64 ? (kp.out_rows + 63) / 64 : n_chunks;
    const int warps = n_strips * (int)n_chunks;
    dim3 grid((warps + C::WARPS - 1) / C::WARPS, 1, kp.n_frames);
    kern<<<grid, C::WARPS * 32, C::kSmem, st>>>(in, out, kp, n_strips, (int)n_chunks);
    return cudaGetLastError();
}

}  // namespace dfg
