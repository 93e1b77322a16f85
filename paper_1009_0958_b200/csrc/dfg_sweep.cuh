// dfg_sweep.cuh -- row-sweeping CTA kernel for the 5x5 / 7x7 windows with
// PIXEL-OWNER aggregation (BVDF, DDF, VMF; all strategies).
//
// Reference path replaced: _engine.py:232-487 (pair row loops, aggregates,
// selection), as dfg_fast.cuh; same pair arithmetic (pair_values2), error
// budget, selection (select_window) and float64 re-decision (dfg_f64.cuh).
//
// Schedule.  A CTA owns a strip of RWP = 64 region columns (OW = 64 - 2h
// output columns) and sweeps DOWN a chunk of rows, one input row per step.
// The S most recent rows are live; each live row belongs to one group of
// WPR = 2 warps (ring slot = row mod S), one thread per pixel.  A thread
// keeps, in registers, its pixel's record and the pixel's n = S*S aggregates
// agg(p; u, v) -- one for every window that contains p, p sitting at window
// position (u, v) -- so segment sums are consumed where they are produced:
//   step t (new row r):
//   A  the group of the new row stages it (records ring, colours ring);
//   B  every group of age k = 0 .. S-1 (its row is r - k) evaluates the pair
//      distances between its own pixel and the new row's pixels (each unique
//      pair once: the new row is the lower partner), writes them to a plane
//      for the other side, forms its pixel's downward segment sums S_+k(p, v)
//      in registers and adds them to agg(p; u, v), u <= S-1-k;
//   C  group k reads the plane back transposed and forms the upward sums
//      S_-k(q, v) of the NEW row's pixels (exchange buffer); the new row's
//      group forms its own row's two-sided sums;
//   D  the new row's group adds S_-k(q, v), k = 1 .. S-1, to agg(q; u, v),
//      u >= k; every group now holds one COMPLETE window row of aggregates
//      (u = S-1-k: the window whose bottom row is r) and emits it;
//   E  a SELECTOR group (WPR more warps) gathers the n aggregates of each
//      output of row r - (S-1), selects, re-decides doubtful pixels in
//      float64 and writes the row -- while the owner groups already work on
//      step t + 1 (the emitted rows are handed over through a full / free
//      pair of named barriers; the retired row's group becomes the next
//      row's group at once).
// Barriers are named (bar.sync / bar.arrive with thread counts): the owner
// groups synchronise among themselves (records visible; upward sums
// visible), a group synchronises alone between B and C (its plane is read
// only by itself), and the selectors never stall the owners except through
// the one-row hand-over buffer.
// Against the tile kernel (dfg_fast.cuh): no vertical halo (every row's pairs
// are evaluated once), no segment-sum stores and loads (343 LDS.64 per
// output there; here 2n exchanged values per output), one horizontal halo of
// 2h columns per 64.
#pragma once

#include "dfg_fast.cuh"

namespace dfg {

template <int S, int FAM>
struct SwCfg {
    static constexpr int H = S / 2, N = S * S, NDV = 2 * S - 1, DC = (N - 1) / 2;
    static constexpr bool NEED_A = FamT<FAM>::A, NEED_L = FamT<FAM>::L, BOTH = NEED_A && NEED_L;
    using DT = typename std::conditional<BOTH, float2, float>::type;
    static constexpr int WPR = 2, RWP = 32 * WPR, OW = RWP - 2 * H;
    // S owner groups of WPR warps + one selector group of WPR warps
    static constexpr int NOWN = 32 * S * WPR, NT = NOWN + 32 * WPR;
    static constexpr int KS = S + 1;  // colour ring: a retired row stays one more step for the selectors
    // records: per ring slot, per column parity, ELEMS pair elements of 2 x 16 B
    // (A = {gx_c, gx_c+1, gy_c, gy_c+1}, B = {gz_c, gz_c+1, aux_c, aux_c+1});
    // element e of parity par holds columns 2 (e - PE) + par, + 1.  ELEMS * 16 B
    // = 64 mod 128, so the even and odd lanes of a warp (which read different
    // parity arrays) use different banks
    static constexpr int PE = 4, ELEMS = 44;
    static constexpr int REC_SLOT = 2 * ELEMS;            // float4 per array (A or B) per slot
    static constexpr int PADP = 8, PW = RWP + 2 * PADP;   // plane row: columns -8 .. 71
    static constexpr int NPL = (S - 1) * NDV + (S - 1);   // planes of k = 1 .. S-1, then same-row dv = 1 .. S-1
    static constexpr size_t kRec = (size_t)S * REC_SLOT * 2 * sizeof(float4);
    static constexpr size_t kPlanes = (size_t)NPL * PW * sizeof(DT);
    static constexpr size_t kXS = (size_t)(S - 1) * S * RWP * sizeof(DT);
    static constexpr size_t kE = (size_t)N * RWP * sizeof(DT);
    static constexpr size_t kK = (size_t)KS * RWP * sizeof(uint32_t);
    static constexpr size_t kF64 = (size_t)N * sizeof(E64) + (size_t)N * (N - 1) * sizeof(double);  // re-decision scratch
    static constexpr size_t kSmem = kRec + kPlanes + kXS + kE + kK + kF64 + 16;
    static_assert(ELEMS * 16 % 128 == 64, "parity arrays half a bank row apart");
    static_assert((RWP + S) / 2 + PE < ELEMS, "partner elements in range");
};

// named barriers
__device__ __forceinline__ void bar_sync(int id, int n) { asm volatile("bar.sync %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ void bar_arrive(int id, int n) { asm volatile("bar.arrive %0, %1;" ::"r"(id), "r"(n) : "memory"); }
__device__ __forceinline__ bool bar_or(int id, int n, bool pred)
{
    int r;
    asm volatile("{\n .reg .pred p, q;\n setp.ne.u32 q, %3, 0;\n barrier.red.or.pred p, %1, %2, q;\n selp.u32 %0, 1, 0, p;\n}"
                 : "=r"(r)
                 : "r"(id), "r"(n), "r"((unsigned)pred)
                 : "memory");
    return r != 0;
}
enum { SW_BAR_OWN = 1, SW_BAR_FULL = 2, SW_BAR_FREE = 3, SW_BAR_SEL = 4, SW_BAR_GRP = 5 };  // GRP + group index

template <int S, int FAM, int ST, int PC>
__global__ void __launch_bounds__(SwCfg<S, FAM>::NT, 1)
dfg_sweep_kernel(const uint8_t *__restrict__ in, uint8_t *__restrict__ out, const __grid_constant__ KParams kp, int n_strips,
                 int n_chunks)
{
    using C = SwCfg<S, FAM>;
    using DT = typename C::DT;
    constexpr int H = C::H, N = C::N, NDV = C::NDV, DC = C::DC, RWP = C::RWP, OW = C::OW, NT = C::NT, NOWN = C::NOWN;
    constexpr int PE = C::PE, ELEMS = C::ELEMS, PADP = C::PADP, PW = C::PW, KS = C::KS, GT = 32 * C::WPR;
    constexpr bool BOTH = C::BOTH;
    static_assert(SW_BAR_GRP + S <= 16, "named barriers");

    extern __shared__ __align__(16) unsigned char sw_smem[];
    float4 *recA = reinterpret_cast<float4 *>(sw_smem);  // [S][2][ELEMS]
    float4 *recB = recA + S * C::REC_SLOT;               // [S][2][ELEMS]
    DT *planes = reinterpret_cast<DT *>(sw_smem + C::kRec);              // [NPL][PW]
    DT *xS = reinterpret_cast<DT *>(sw_smem + C::kRec + C::kPlanes);     // [S-1][S][RWP]
    DT *eX = reinterpret_cast<DT *>(sw_smem + C::kRec + C::kPlanes + C::kXS);  // [N][RWP]
    uint32_t *rK = reinterpret_cast<uint32_t *>(sw_smem + C::kRec + C::kPlanes + C::kXS + C::kE);  // [KS][RWP]
    unsigned char *f64b = sw_smem + C::kRec + C::kPlanes + C::kXS + C::kE + C::kK;
    __shared__ unsigned s_nflag;
    __shared__ uint16_t s_flag[RWP];
    __shared__ int s_b;
    __shared__ bool s_close;

    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const int grp = warp / C::WPR, c = (warp % C::WPR) * 32 + lane;  // group (S = the selectors), region column
    const int strip = blockIdx.x % n_strips, chunk = blockIdx.x / n_strips, frame = blockIdx.y;
    const uint8_t *fin = in + (long long)frame * kp.in_fstride;
    uint8_t *fout = out + (long long)frame * kp.out_fstride;
    const int oy0 = (int)((long long)chunk * kp.out_rows / n_chunks);
    const int oy1 = (int)((long long)(chunk + 1) * kp.out_rows / n_chunks);
    const int x0 = strip * OW;                                   // first output column of the strip
    const int colr = resolve_idx(x0 - H + c, kp.W, kp.border);  // this thread's input column
    const float pad_aux = (ST == ST_MINIMAX) ? 0.57735026f : (ST == ST_CHROMA ? (1.f / 3.f) : 1.7320508f);

    // neutral records everywhere (pad elements keep them)
    for (int i = tid; i < S * C::REC_SLOT; i += NT) {
        recA[i] = make_float4(1.f, 1.f, 1.f, 1.f);
        recB[i] = make_float4(1.f, 1.f, pad_aux, pad_aux);
    }
    for (int i = tid; i < C::NPL * PW; i += NT) planes[i] = dt_zero(DT());
    if (tid == 0) s_nflag = 0u;

    using AG = typename std::conditional<BOTH, P2, float>::type;
    auto ag_init = [&]() -> AG {
        if constexpr (BOTH) return pk2(kp.self_term, 0.f);
        else if constexpr (C::NEED_A) return kp.self_term;
        else return 0.f;
    };
    auto ag_add = [](AG a, DT b) -> AG {
        if constexpr (BOTH) return add2(a, *reinterpret_cast<const P2 *>(&b));
        else return a + b;
    };
    AG ag[S][S];
#pragma unroll
    for (int u = 0; u < S; u++)
#pragma unroll
        for (int v = 0; v < S; v++) ag[u][v] = ag_init();

    auto row_of = [&](int ry) {  // strip-local input row of region row ry (global border policy)
        int gy = kp.out_row0 + oy0 - H + ry;
        if ((unsigned)gy >= (unsigned)kp.global_H) gy = resolve_idx(gy, kp.global_H, kp.border);
        return min(max(gy - kp.in_row0, 0), kp.in_rows - 1);
    };
    auto to_dt = [](P2 da, P2 dl, bool hi) -> DT {
        if constexpr (BOTH) return hi ? make_float2(hi2(da), hi2(dl)) : make_float2(lo2(da), lo2(dl));
        else if constexpr (C::NEED_A) return hi ? hi2(da) : lo2(da);
        else return hi ? hi2(dl) : lo2(dl);
    };
    __syncthreads();
    const int n_steps = (oy1 - oy0) + 2 * H;

    if (grp == S) {
        // =================== selectors ==========================================
        bar_arrive(SW_BAR_FREE, NT);  // the hand-over buffer starts free
        int sn = 0, ks = 0;           // ring slots of the new row: t mod S, t mod KS
        for (int t = 0; t < n_steps; t++, sn = (sn + 1 == S ? 0 : sn + 1), ks = (ks + 1 == KS ? 0 : ks + 1)) {
            bar_sync(SW_BAR_FULL, NT);  // step t's emitted rows are in eX
            if (t >= 2 * H) {
                const int oy = oy0 + t - 2 * H;
                const int xo = min(c, OW - 1);  // (lanes beyond the strip's outputs: clamped, unused)
                const bool valid = c < OW && x0 + c < kp.W;
#pragma unroll
                for (int u = 0; u < S; u++)
#pragma unroll
                    for (int v = 0; v < S; v++) {
                        const DT x = eX[(u * S + v) * RWP + xo + v];
                        if constexpr (BOTH) ag[u][v] = *reinterpret_cast<const P2 *>(&x);
                        else ag[u][v] = x;
                    }
                // colour ring slot of window row u: row t - (S-1) + u -> (ks + 2 + u) mod KS
                auto kslot = [&](int u) {
                    int sl = ks + 2 + u;
                    sl -= sl >= KS ? KS : 0;
                    return sl;
                };
                auto colf = [&](auto ic) {
                    constexpr int i = decltype(ic)::value, u = i / S, v = i % S;
                    return rK[kslot(u) * RWP + xo + v];
                };
                uint32_t kc;
                bool doubt;
                if constexpr (BOTH) {
                    auto A = [&](auto ic) { return lo2(ag[decltype(ic)::value / S][decltype(ic)::value % S]); };
                    auto L = [&](auto ic) { return hi2(ag[decltype(ic)::value / S][decltype(ic)::value % S]); };
                    auto Z = [](auto) { return 0.f; };
                    select_window<FAM, ST, N, DC>(kp, A, L, Z, Z, colf, kc, doubt);
                } else {
                    auto V = [&](auto ic) { return ag[decltype(ic)::value / S][decltype(ic)::value % S]; };
                    auto Z = [](auto) { return 0.f; };
                    select_window<FAM, ST, N, DC>(kp, V, V, Z, Z, colf, kc, doubt);
                }
                if (valid) {
                    uint8_t *op = fout + (long long)oy * kp.out_pitch + 3 * (x0 + c);
                    op[0] = (uint8_t)(kc & 0xff);
                    op[1] = (uint8_t)((kc >> 8) & 0xff);
                    op[2] = (uint8_t)((kc >> 16) & 0xff);
                    if (doubt && !kp.diag_no_fixup) s_flag[atomicAdd(&s_nflag, 1u)] = (uint16_t)c;
                }
                // float64 re-decision of this row's doubtful pixels (the selector group alone; rare)
                bar_sync(SW_BAR_SEL, GT);
                const unsigned nflag = s_nflag;
                if (nflag != 0u) {
                    const int st = tid - NOWN;  // 0 .. GT-1
                    if (st == 0) atomicAdd(kp.flag_count, nflag);
                    constexpr int P = N * (N - 1) / 2;
                    E64 *e64 = reinterpret_cast<E64 *>(f64b);
                    double *dA = reinterpret_cast<double *>(e64 + N);
                    double *dL = dA + P;
                    const FParams &fp = kp.fp;
                    for (unsigned f = 0; f < nflag; f++) {
                        const int cx = s_flag[f];
                        for (int i = st; i < N; i += GT) {
                            const uint32_t col = rK[kslot(i / S) * RWP + cx + i % S];
                            prep64(make_float4((float)(col & 0xff), (float)((col >> 8) & 0xff), (float)((col >> 16) & 0xff),
                                               0.f),
                                   ST, e64[i]);
                        }
                        bar_sync(SW_BAR_SEL, GT);
                        pair_tables<false>(e64, fp, st, GT, dA, dL, C::NEED_A, C::NEED_L);
                        bar_sync(SW_BAR_SEL, GT);
                        if (st < 32) {
                            bool close;
                            const int bb = decide64<N, FAM, ST>(e64, fp, lane, dA, dL, &close);
                            if (lane == 0) { s_b = bb; s_close = close; }
                        }
                        bar_sync(SW_BAR_SEL, GT);
                        if (ST == ST_EXACT && C::NEED_A && s_close) {
                            if (st == 0) atomicAdd(kp.flag_count + 1, 1u);
                            pair_tables<true>(e64, fp, st, GT, dA, dL, C::NEED_A, C::NEED_L);
                            bar_sync(SW_BAR_SEL, GT);
                            if (st < 32) {
                                bool close;
                                const int bb = decide64<N, FAM, ST>(e64, fp, lane, dA, dL, &close);
                                if (lane == 0) s_b = bb;
                            }
                            bar_sync(SW_BAR_SEL, GT);
                        }
                        if (st == 0) {
                            const int bb = s_b;
                            const uint32_t col = rK[kslot(bb / S) * RWP + cx + bb % S];
                            uint8_t *op = fout + (long long)oy * kp.out_pitch + 3 * (x0 + cx);
                            op[0] = (uint8_t)(col & 0xff);
                            op[1] = (uint8_t)((col >> 8) & 0xff);
                            op[2] = (uint8_t)((col >> 16) & 0xff);
                        }
                        bar_sync(SW_BAR_SEL, GT);
                    }
                    if (st == 0) s_nflag = 0u;
                    bar_sync(SW_BAR_SEL, GT);
                }
            }
            bar_arrive(SW_BAR_FREE, NT);  // eX and the retired row's colours may be overwritten
        }
        return;
    }

    // ======================= owner groups ========================================
    Pix own = {1.f, 1.f, 1.f, pad_aux};
    unsigned zhist = 0u;  // bit j: a zero vector in the row staged j steps ago
    // the next row's pixel of the group that stages it, loaded a step ahead
    uint32_t nrgb = 0u;
    if (grp == 0) {
        const uint8_t *px = fin + (long long)row_of(0) * kp.in_pitch + 3 * colr;
        nrgb = px[0] | (px[1] << 8) | (px[2] << 16);
    }
    int sn = 0, ks = 0;  // ring slots of the new row: t mod S (groups, records), t mod KS (colours)
    for (int t = 0; t < n_steps; t++, sn = (sn + 1 == S ? 0 : sn + 1), ks = (ks + 1 == KS ? 0 : ks + 1)) {
        const int k = sn - grp + (sn < grp ? S : 0);  // age of this group's row (0: the new row)
        // ---- A: the new row's group stages it --------------------------------
        bool zero = false;
        if (k == 0) {
            const uint32_t rgb = nrgb;
            zero = rgb == 0u;
            const float gx = zero ? 1.f : (float)(rgb & 0xff), gy = zero ? 1.f : (float)((rgb >> 8) & 0xff),
                        gz = zero ? 1.f : (float)((rgb >> 16) & 0xff);
            own = {gx, gy, gz, encode_aux<ST, C::NEED_L>(gx, gy, gz, zero)};
            // element (c, c+1) of parity c & 1: first half; element (c-1, c) of the other parity: second half
            float *a1 = reinterpret_cast<float *>(recA + sn * C::REC_SLOT + (c & 1) * ELEMS + (c >> 1) + PE);
            float *b1 = reinterpret_cast<float *>(recB + sn * C::REC_SLOT + (c & 1) * ELEMS + (c >> 1) + PE);
            a1[0] = own.x; a1[2] = own.y; b1[0] = own.z; b1[2] = own.aux;
            const int e2 = ((c + 1) >> 1) - 1 + PE;  // element of columns (c-1, c): parity (c-1) & 1 = (c+1) & 1
            float *a2 = reinterpret_cast<float *>(recA + sn * C::REC_SLOT + ((c + 1) & 1) * ELEMS + e2);
            float *b2 = reinterpret_cast<float *>(recB + sn * C::REC_SLOT + ((c + 1) & 1) * ELEMS + e2);
            a2[1] = own.x; a2[3] = own.y; b2[1] = own.z; b2[3] = own.aux;
            rK[ks * RWP + c] = rgb;
        }
        if (k == S - 1 && t + 1 < n_steps) {  // this group stages the next row: load its pixel now
            const uint8_t *px = fin + (long long)row_of(t + 1) * kp.in_pitch + 3 * colr;
            nrgb = px[0] | (px[1] << 8) | (px[2] << 16);
        }
        const bool zany = bar_or(SW_BAR_OWN, NOWN, zero);  // owners: records visible
        zhist = ((zhist << 1) | (zany ? 1u : 0u)) & ((1u << S) - 1u);
        const bool zchk = C::NEED_L && zhist != 0u;

        // ---- B: pairs (own pixel, new row), planes, downward sums --------------
        DT Sg[S];
        const int par = c & 1;
        auto stage1 = [&](auto zc_c) {
            constexpr bool ZC = decltype(zc_c)::value;
            if (k > 0) {
                // partners at columns c - (S-1) + 2m, + 1 (m = 0 .. S-1): parity of c
                const float4 *qa = recA + sn * C::REC_SLOT + par * ELEMS + (c >> 1) - H + PE;
                const float4 *qb = recB + sn * C::REC_SLOT + par * ELEMS + (c >> 1) - H + PE;
                DT T[NDV];
#pragma unroll
                for (int m = 0; m < S; m++) {
                    const ulonglong2 A2 = lds_u2_ordered(qa + m), B2 = lds_u2_ordered(qb + m);
                    const Pair2 q = {{A2.x}, {A2.y}, {B2.x}, {B2.y}};
                    P2 da, dl;
                    pair_values2<FAM, ST, PC, ZC>(own, q, kp, da, dl);
                    T[2 * m] = to_dt(da, dl, false);
                    if (2 * m + 1 < NDV) T[2 * m + 1] = to_dt(da, dl, true);
                }
                DT *pl = planes + (k - 1) * NDV * PW + c + PADP;
#pragma unroll
                for (int tt = 0; tt < NDV; tt++) pl[tt * PW] = T[tt];
                seg_sums<S>(T, Sg);
            } else {
                // same row, partners to the right: columns c + 1 + 2m, + 1 (m = 0 .. H-1): the other parity
                const int e = ((c + 1) >> 1) + PE;
                const float4 *qa = recA + sn * C::REC_SLOT + ((c + 1) & 1) * ELEMS + e;
                const float4 *qb = recB + sn * C::REC_SLOT + ((c + 1) & 1) * ELEMS + e;
                DT *pl = planes + (S - 1) * NDV * PW + c + PADP;
#pragma unroll
                for (int m = 0; m < H; m++) {
                    const ulonglong2 A2 = lds_u2_ordered(qa + m), B2 = lds_u2_ordered(qb + m);
                    const Pair2 q = {{A2.x}, {A2.y}, {B2.x}, {B2.y}};
                    P2 da, dl;
                    pair_values2<FAM, ST, PC, ZC>(own, q, kp, da, dl);
                    pl[(2 * m) * PW] = to_dt(da, dl, false);      // dv = 2m + 1
                    pl[(2 * m + 1) * PW] = to_dt(da, dl, true);   // dv = 2m + 2
                }
            }
        };
        if (zchk) stage1(std::true_type{});
        else stage1(std::false_type{});
        // agg(p; u, v) += S_+k(p, v) for u <= S-1-k (k is uniform per warp)
        static_for<1, S>([&](auto kk_c) {
            constexpr int kk = decltype(kk_c)::value;
            if (k == kk) {
#pragma unroll
                for (int u = 0; u + kk < S; u++)
#pragma unroll
                    for (int v = 0; v < S; v++) ag[u][v] = ag_add(ag[u][v], Sg[v]);
            }
        });
        bar_sync(SW_BAR_GRP + grp, GT);  // the group's plane is read back by the group alone

        // ---- C: upward sums of the new row's pixels (groups k >= 1); the new
        // row's own two-sided sums (group 0) ---------------------------------------
        {
            DT T[NDV];
            if (k > 0) {
                // T_q(t): the pair whose upper pixel is at column offset dv = t - (S-1)
                // from q: plane NDV-1-t of that pixel
                const DT *pl = planes + (k - 1) * NDV * PW + c + PADP;
#pragma unroll
                for (int tt = 0; tt < NDV; tt++) T[tt] = pl[(NDV - 1 - tt) * PW + tt - (S - 1)];
                seg_sums<S>(T, Sg);
                DT *xs = xS + (k - 1) * S * RWP + c;
#pragma unroll
                for (int v = 0; v < S; v++) xs[v * RWP] = Sg[v];
            } else {
                const DT *pl = planes + (S - 1) * NDV * PW + c + PADP;
#pragma unroll
                for (int tt = 0; tt < NDV; tt++) {
                    const int dv = tt - (S - 1);
                    if (dv > 0) T[tt] = pl[(dv - 1) * PW];
                    else if (dv < 0) T[tt] = pl[(-dv - 1) * PW + dv];
                    else T[tt] = dt_zero(DT());
                }
                seg_sums<S>(T, Sg);
#pragma unroll
                for (int u = 0; u < S; u++)
#pragma unroll
                    for (int v = 0; v < S; v++) ag[u][v] = ag_add(ag[u][v], Sg[v]);
            }
        }
        bar_sync(SW_BAR_OWN, NOWN);  // owners: the exchange buffer is visible

        // ---- D: the new row takes its upward sums; every group emits its
        // completed window row u = S-1-k -------------------------------------------
        if (k == 0) {
#pragma unroll
            for (int kk = 1; kk < S; kk++) {
#pragma unroll
                for (int v = 0; v < S; v++) {
                    const DT x = xS[((kk - 1) * S + v) * RWP + c];
#pragma unroll
                    for (int u = kk; u < S; u++) ag[u][v] = ag_add(ag[u][v], x);
                }
            }
        }
        bar_sync(SW_BAR_FREE, NT);  // the selectors are done with the previous row
        static_for<0, S>([&](auto kk_c) {
            constexpr int kk = decltype(kk_c)::value, u = S - 1 - kk;
            if (k == kk) {
#pragma unroll
                for (int v = 0; v < S; v++) {
                    if constexpr (BOTH) eX[(u * S + v) * RWP + c] = *reinterpret_cast<const float2 *>(&ag[u][v]);
                    else eX[(u * S + v) * RWP + c] = ag[u][v];
                }
            }
        });
        bar_arrive(SW_BAR_FULL, NT);
        if (k == S - 1) {
            // the group's pixel has left every window: fresh aggregates for its next row
#pragma unroll
            for (int u = 0; u < S; u++)
#pragma unroll
                for (int v = 0; v < S; v++) ag[u][v] = ag_init();
        }
    }
    bar_sync(SW_BAR_FREE, NT);  // (pairs the selectors' last arrive)
}

template <int S, int FAM, int ST, int PC>
cudaError_t launch_sweep(cudaStream_t st, const uint8_t *in, uint8_t *out, const KParams &kp)
{
    using C = SwCfg<S, FAM>;
    auto kern = dfg_sweep_kernel<S, FAM, ST, PC>;
    static unsigned long long configured = 0;
    int dev = 0;
    cudaGetDevice(&dev);
    if (!(configured & (1ull << (dev & 63)))) {
        cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)C::kSmem);
        if (e != cudaSuccess) return e;
        configured |= 1ull << (dev & 63);
    }
    const int n_strips = (kp.W + C::OW - 1) / C::OW;
    // chunks per strip: whole waves of one CTA per SM, chunks of >= 64 rows
    // where the frame allows (every chunk pays 2h warm-up steps)
    const long long sms = sm_count(dev);
    const long long cols = (long long)n_strips * kp.n_frames;
    long long n_chunks = (4 * sms + cols - 1) / cols;
    if (n_chunks > kp.out_rows / 64) n_chunks = kp.out_rows / 64;
    if (n_chunks < 1) n_chunks = 1;
    dim3 grid((unsigned)(n_strips * n_chunks), (unsigned)kp.n_frames, 1);
    kern<<<grid, C::NT, C::kSmem, st>>>(in, out, kp, n_strips, (int)n_chunks);
    return cudaGetLastError();
}

}  // namespace dfg
