// dfg_api.cu -- C ABI (include/dirfilt_gpu.h) over the directional filter
// kernels: validation (the reference's ValueError cases), parameter
// packing, the FP32 decision launch and the float64 re-decision launch.
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include <mutex>
#include <string>

#include "dfg_internal.cuh"

namespace {

thread_local std::string g_err;

int fail(int code, const char *msg)
{
    g_err = msg;
    return code;
}

int cuda_fail(cudaError_t e, const char *where)
{
    g_err = std::string(where) + ": " + cudaGetErrorString(e);
    return DFG_E_CUDA;
}

constexpr size_t kWsHeader = 256;

// Mirrors the reference's validation (filters.py:53-59, 110-123, 141-151,
// image.py:44-46): invalid -> DFG_E_ARG (ValueError); valid but outside
// this build -> DFG_E_UNSUP.
int validate(const dfg_params *p)
{
    if (!p) return fail(DFG_E_ARG, "null params");
    if (p->family < DFG_IDENTITY || p->family > DFG_ACWDDF) return fail(DFG_E_ARG, "unknown filter family");
    if (p->strategy < DFG_EXACT || p->strategy > DFG_CHROMA) return fail(DFG_E_ARG, "unknown strategy kind");
    if (p->border != DFG_REPLICATE && p->border != DFG_REFLECT) return fail(DFG_E_ARG, "unknown border mode");
    if (p->window < 3 || (p->window % 2) == 0) return fail(DFG_E_ARG, "window side must be odd and >= 3");
    if (!(p->p >= 1.0)) return fail(DFG_E_ARG, "Minkowski order must be >= 1");
    if (p->strategy == DFG_CHROMA && !(p->slope > 0.0)) return fail(DFG_E_ARG, "calibration slope must be positive");
    if (p->family == DFG_ACWDDF) {
        const int n = p->window * p->window, d = (n + 1) / 2;
        if (p->lam < 1) return fail(DFG_E_ARG, "lambda must be >= 1");
        if (p->lam + 2 > d) return fail(DFG_E_ARG, "lambda + 2 exceeds the number of smoothing levels");
        if (!(p->threshold >= 0.0)) return fail(DFG_E_ARG, "threshold must be nonnegative");
    }
    if (p->family != DFG_IDENTITY && p->window != 3 && p->window != 5 && p->window != 7)
        return fail(DFG_E_UNSUP, "this build supports window sides 3, 5 and 7");
    return DFG_OK;
}

// FP32 error budget of one aggregate: first-order
// worst-case bound of the per-pair relative error plus recursive summation of
// n - 1 nonnegative terms ((n-1) u, u = 2^-24), times a 1.25 safety factor;
// ea_pair covers the reference's own non-relative deviations (near-parallel
// acos rounding, the minimax duplicate-pair quirk of SURVEY A.6).
void error_budget(const dfg_params *p, dfg::KParams &kp)
{
    const int n = p->window * p->window;
    const bool gen_p = !(p->p == 2.0 || p->p == 1.0);
    float er_pair = 8e-7f, ea_pair = 1e-10f;
    if (p->strategy == DFG_MINIMAX) { er_pair = 1.2e-6f; ea_pair = 8e-8f; }
    if (p->strategy == DFG_CHROMA) { er_pair = 8e-7f; ea_pair = 1e-9f; }
    if (gen_p) er_pair += 4e-6f * (float)p->p;
    kp.er = 1.25f * (er_pair + (float)(n - 1) * 6e-8f);
    kp.ea_pair = 1.25f * ea_pair;
    kp.ea = 1.25f * (float)n * ea_pair;
}

void fill_params(const dfg_params *p, dfg::KParams &kp)
{
    dfg::FParams &fp = kp.fp;
    const int n = p->window * p->window;
    kp.border = p->border;
    kp.p = (float)p->p;
    kp.invp = (float)(1.0 / p->p);
    for (int k = 0; k < 5; k++) {
        kp.cs[k] = (float)p->asin_c[k];
        kp.ca[k] = (float)p->acos_c[k];
        kp.cs64[k] = p->asin_c[k];
        kp.ca64[k] = p->acos_c[k];
        fp.cs[k] = p->asin_c[k];
        fp.ca[k] = p->acos_c[k];
    }
    const double self_term = (p->strategy == DFG_MINIMAX) ? p->asin_c[0] : 0.0;
    kp.self_term = (float)self_term;
    kp.slope = (float)p->slope;
    kp.intercept = (float)p->intercept;
    kp.threshold = (float)p->threshold;
    for (int k = 0; k < 3; k++) kp.w[k] = (float)(n - 2 * (p->lam + k) + 2 - 1);
    error_budget(p, kp);
    fp.family = p->family;
    fp.strategy = p->strategy;
    fp.window = p->window;
    fp.p = p->p;
    fp.self_term = self_term;
    fp.lam = p->lam;
    fp.threshold = p->threshold;
    fp.slope = p->slope;
    fp.intercept = p->intercept;
    static const double cr_margin = [] {
        const char *e = getenv("DFG_CR_MARGIN");  // diagnostics only
        return e ? atof(e) : 1e-12;
    }();
    fp.cr_margin = cr_margin;
}

int pcode_of(double p) { return p == 2.0 ? dfg::PC_2 : (p == 1.0 ? dfg::PC_1 : dfg::PC_GEN); }

cudaError_t launch_fast(const dfg_params *p, cudaStream_t st, const uint8_t *in, uint8_t *out,
                        const dfg::KParams &kp)
{
    const int pc = pcode_of(p->p);
#define DFG_CASE(S)                                                                    \
    if (p->window == S) {                                                              \
        switch (p->family) {                                                           \
        case DFG_VMF: return dfg_launch_s##S##_vmf(p->strategy, pc, st, in, out, kp);  \
        case DFG_BVDF: return dfg_launch_s##S##_bvdf(p->strategy, pc, st, in, out, kp); \
        case DFG_DDF: return dfg_launch_s##S##_ddf(p->strategy, pc, st, in, out, kp);  \
        default: return dfg_launch_s##S##_acwddf(p->strategy, pc, st, in, out, kp);    \
        }                                                                              \
    }
    DFG_CASE(3)
    DFG_CASE(5)
    DFG_CASE(7)
#undef DFG_CASE
    return cudaErrorInvalidValue;
}

// Shared driver of dfg_filter / _rows / _batch.
int run(const uint8_t *d_in, int global_H, int W, int in_row0, int in_rows, long long in_pitch,
        long long in_fstride, uint8_t *d_out, int out_row0, int out_rows, long long out_pitch,
        long long out_fstride, int frames, const dfg_params *prm, void *ws, size_t ws_bytes,
        void *stream, float *dbg)
{
    int rc = validate(prm);
    if (rc) return rc;
    if (global_H < 1 || W < 1 || frames < 1) return fail(DFG_E_ARG, "image must contain at least one pixel");
    if (out_rows < 1 || out_row0 < 0 || out_row0 + out_rows > global_H) return fail(DFG_E_ARG, "bad output row range");
    if (in_rows < 1 || in_row0 < 0 || in_row0 + in_rows > global_H) return fail(DFG_E_ARG, "bad input row range");
    if (!d_in || !d_out) return fail(DFG_E_ARG, "null image pointer");
    if (in_pitch < 3LL * W || out_pitch < 3LL * W) return fail(DFG_E_ARG, "pitch smaller than 3 * W bytes");
    // every row the border policy resolves must be resident
    const int h = prm->window / 2;
    if (prm->family != DFG_IDENTITY) {
        for (int r = out_row0 - h; r < out_row0 + out_rows + h; r++) {
            const int g = dfg::resolve_idx(r, global_H, prm->border);
            if (g < in_row0 || g >= in_row0 + in_rows) return fail(DFG_E_ARG, "input rows do not cover the window halo");
        }
    }
    cudaStream_t st = (cudaStream_t)stream;
    if (prm->family == DFG_IDENTITY) {  // filters.py:394-395: a copy
        for (int f = 0; f < frames; f++) {
            cudaError_t e = cudaMemcpy2DAsync(d_out + f * out_fstride, out_pitch,
                                              d_in + f * in_fstride + (long long)(out_row0 - in_row0) * in_pitch,
                                              in_pitch, 3 * (size_t)W, out_rows, cudaMemcpyDeviceToDevice, st);
            if (e != cudaSuccess) return cuda_fail(e, "identity copy");
        }
        return DFG_OK;
    }
    const long long npx = (long long)out_rows * W * frames;
    if (npx > 0xffffffffLL) return fail(DFG_E_ARG, "more than 2^32 output pixels in one call");
    if (!ws || ws_bytes < dfg_workspace_bytes(npx)) return fail(DFG_E_WS, "workspace too small (dfg_workspace_bytes)");

    dfg::KParams kp;
    memset(&kp, 0, sizeof kp);
    kp.global_H = global_H;
    kp.W = W;
    kp.in_row0 = in_row0;
    kp.in_rows = in_rows;
    kp.out_row0 = out_row0;
    kp.out_rows = out_rows;
    kp.in_pitch = in_pitch;
    kp.out_pitch = out_pitch;
    kp.in_fstride = in_fstride;
    kp.out_fstride = out_fstride;
    kp.n_frames = frames;
    fill_params(prm, kp);
    kp.flag_count = (unsigned *)ws;
    kp.dbg = dbg;

    cudaError_t e = launch_fast(prm, st, d_in, d_out, kp);
    if (e != cudaSuccess) return cuda_fail(e, "fast kernel launch");
    return DFG_OK;
}

constexpr int kMaxBands = 8;

struct HostCache {
    uint8_t *d_in = nullptr, *d_out = nullptr;
    void *ws = nullptr;
    size_t px_cap = 0;
    int dev = -1;
    cudaStream_t s_in = nullptr, s_out = nullptr;  // copy streams (H2D / D2H engines)
    cudaEvent_t ev_start = nullptr, ev_done = nullptr, ev_in[kMaxBands] = {}, ev_k[kMaxBands] = {};
    void release()
    {
        if (d_in) cudaFree(d_in);
        if (d_out) cudaFree(d_out);
        if (ws) cudaFree(ws);
        d_in = d_out = nullptr;
        ws = nullptr;
        px_cap = 0;
    }
    ~HostCache() { release(); }
};
thread_local HostCache g_host;

}  // namespace

extern "C" {

int dfg_abi_version(void) { return DFG_ABI_VERSION; }

const char *dfg_last_error(void) { return g_err.c_str(); }

size_t dfg_workspace_bytes(int64_t n_pixels)
{
    if (n_pixels < 0) n_pixels = 0;
    (void)n_pixels;  // counters only: the float64 re-decision runs inside each CTA
    return kWsHeader;
}

int dfg_filter(const uint8_t *d_in, int32_t H, int32_t W, int64_t in_pitch, uint8_t *d_out,
               int64_t out_pitch, const dfg_params *prm, void *ws, size_t ws_bytes, void *stream)
{
    return run(d_in, H, W, 0, H, in_pitch, 0, d_out, 0, H, out_pitch, 0, 1, prm, ws, ws_bytes, stream, nullptr);
}

int dfg_filter_rows(const uint8_t *d_in, int32_t global_H, int32_t W, int32_t in_row0, int32_t in_rows,
                    int64_t in_pitch, uint8_t *d_out, int32_t out_row0, int32_t out_rows,
                    int64_t out_pitch, const dfg_params *prm, void *ws, size_t ws_bytes, void *stream)
{
    return run(d_in, global_H, W, in_row0, in_rows, in_pitch, 0, d_out, out_row0, out_rows, out_pitch, 0, 1,
               prm, ws, ws_bytes, stream, nullptr);
}

int dfg_filter_batch(const uint8_t *d_in, int32_t B, int32_t H, int32_t W, int64_t in_pitch,
                     int64_t in_frame_stride, uint8_t *d_out, int64_t out_pitch, int64_t out_frame_stride,
                     const dfg_params *prm, void *ws, size_t ws_bytes, void *stream)
{
    if (B > 65535) return fail(DFG_E_ARG, "at most 65535 frames per call");
    return run(d_in, H, W, 0, H, in_pitch, in_frame_stride, d_out, 0, H, out_pitch, out_frame_stride, B, prm,
               ws, ws_bytes, stream, nullptr);
}

int dfg_filter_host(const uint8_t *h_in, int32_t H, int32_t W, uint8_t *h_out, const dfg_params *prm,
                    void *stream)
{
    int rc = validate(prm);
    if (rc) return rc;
    if (H < 1 || W < 1) return fail(DFG_E_ARG, "image must contain at least one pixel");
    if (!h_in || !h_out) return fail(DFG_E_ARG, "null host pointer");
    int dev = 0;
    cudaGetDevice(&dev);
    HostCache &c = g_host;
    const size_t px = (size_t)H * W;
    cudaStream_t st = (cudaStream_t)stream;
    if (c.dev != dev || c.px_cap < px) {
        c.release();
        cudaError_t e = cudaMalloc(&c.d_in, 3 * px);
        if (e == cudaSuccess) e = cudaMalloc(&c.d_out, 3 * px);
        if (e == cudaSuccess) e = cudaMalloc(&c.ws, dfg_workspace_bytes((int64_t)px));
        if (e == cudaSuccess) e = cudaMemset(c.ws, 0, dfg_workspace_bytes((int64_t)px));
        if (e == cudaSuccess && c.dev != dev) {
            e = cudaStreamCreateWithFlags(&c.s_in, cudaStreamNonBlocking);
            if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c.s_out, cudaStreamNonBlocking);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.ev_start, cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.ev_done, cudaEventDisableTiming);
            for (int k = 0; k < kMaxBands && e == cudaSuccess; k++) {
                e = cudaEventCreateWithFlags(&c.ev_in[k], cudaEventDisableTiming);
                if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.ev_k[k], cudaEventDisableTiming);
            }
        }
        if (e != cudaSuccess) {
            c.release();
            return cuda_fail(e, "device staging allocation");
        }
        c.px_cap = px;
        c.dev = dev;
    }
    // Opt-in (DFG_HOST_ZEROCOPY=1) for pinned, device-mapped host buffers:
    // zero-copy -- the kernel reads its input and writes its output over
    // PCIe directly, one launch.  Measured slower than the banded copies
    // below for every config (byte-granular PCIe reads, halo re-reads), so
    // off by default.
    static const bool zc_env = [] {
        const char *e = getenv("DFG_HOST_ZEROCOPY");
        return e && e[0] == '1';
    }();
    if (zc_env) {
        cudaPointerAttributes ai, ao;
        if (cudaPointerGetAttributes(&ai, h_in) == cudaSuccess && cudaPointerGetAttributes(&ao, h_out) == cudaSuccess &&
            ai.type == cudaMemoryTypeHost && ao.type == cudaMemoryTypeHost && ai.devicePointer && ao.devicePointer) {
            rc = run((const uint8_t *)ai.devicePointer, H, W, 0, H, 3LL * W, 0, (uint8_t *)ao.devicePointer, 0, H,
                     3LL * W, 0, 1, prm, c.ws, dfg_workspace_bytes((int64_t)px), stream, nullptr);
            if (rc) return rc;
            cudaError_t e = cudaStreamSynchronize(st);
            if (e != cudaSuccess) return cuda_fail(e, "synchronize");
            return DFG_OK;
        }
        cudaGetLastError();  // pageable memory: clear the attribute query's error state
    }
    // Row-band pipeline: H2D of band k+1 (copy engine 1), the kernel of band
    // k (on `stream`) and D2H of band k-1 (copy engine 2) overlap.  Band k's
    // kernel waits for the input rows its windows reach (k+1's first rows).
    const int h = (prm->family == DFG_IDENTITY) ? 0 : prm->window / 2;
    static const int nb_env = [] {
        const char *s = getenv("DFG_HOST_BANDS");  // diagnostics only
        return s ? atoi(s) : 0;
    }();
    // each band costs ~25 us of API calls: bands only pay off when the
    // copies they hide are larger than that (>= ~0.5 M pixels per band)
    int nb = nb_env > 0 ? nb_env : (int)(px / (512 * 1024));
    if (nb > H / 64) nb = H / 64;
    nb = nb < 1 ? 1 : (nb > kMaxBands ? kMaxBands : nb);
    if (prm->border == DFG_REFLECT && H <= 4 * h) nb = 1;
    const long long pitch = 3LL * W;
    auto row0 = [&](int k) { return (int)((long long)k * H / nb); };
    cudaError_t e = cudaEventRecord(c.ev_start, st);  // buffers are free once prior work on `stream` is done
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c.s_in, c.ev_start, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c.s_out, c.ev_start, 0);
    for (int k = 0; k < nb && e == cudaSuccess; k++) {
        const int r0 = row0(k), r1 = row0(k + 1);
        e = cudaMemcpyAsync(c.d_in + r0 * pitch, h_in + r0 * pitch, (size_t)(r1 - r0) * pitch,
                            cudaMemcpyHostToDevice, c.s_in);
        if (e == cudaSuccess) e = cudaEventRecord(c.ev_in[k], c.s_in);
    }
    if (e != cudaSuccess) return cuda_fail(e, "H2D");
    for (int k = 0; k < nb; k++) {
        const int r0 = row0(k), r1 = row0(k + 1);
        int need = 0;  // last band whose rows the windows of band k reach
        while (need + 1 < nb && row0(need + 1) < r1 + h) need++;
        e = cudaStreamWaitEvent(st, c.ev_in[need], 0);
        if (e != cudaSuccess) return cuda_fail(e, "band dependency");
        rc = run(c.d_in, H, W, 0, H, pitch, 0, c.d_out + r0 * pitch, r0, r1 - r0, pitch, 0, 1, prm, c.ws,
                 dfg_workspace_bytes((int64_t)px), stream, nullptr);
        if (rc) return rc;
        e = cudaEventRecord(c.ev_k[k], st);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(c.s_out, c.ev_k[k], 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(h_out + r0 * pitch, c.d_out + r0 * pitch, (size_t)(r1 - r0) * pitch,
                                cudaMemcpyDeviceToHost, c.s_out);
        if (e != cudaSuccess) return cuda_fail(e, "D2H");
    }
    e = cudaEventRecord(c.ev_done, c.s_out);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, c.ev_done, 0);  // later work on `stream` sees the result
    if (e == cudaSuccess) e = cudaEventSynchronize(c.ev_done);
    if (e != cudaSuccess) return cuda_fail(e, "synchronize");
    return DFG_OK;
}

int dfg_fixup_count(const void *ws, void *stream, int64_t *count)
{
    if (!ws || !count) return fail(DFG_E_ARG, "null argument");
    unsigned v = 0;
    cudaError_t e = cudaMemcpyAsync(&v, ws, sizeof v, cudaMemcpyDeviceToHost, (cudaStream_t)stream);
    if (e == cudaSuccess) e = cudaStreamSynchronize((cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "fixup count read");
    *count = v;
    return DFG_OK;
}

int dfg_reset_counts(void *ws, void *stream)
{
    if (!ws) return fail(DFG_E_ARG, "null workspace");
    cudaError_t e = cudaMemsetAsync(ws, 0, 2 * sizeof(unsigned), (cudaStream_t)stream);
    if (e != cudaSuccess) return cuda_fail(e, "counter reset");
    return DFG_OK;
}

int dfg_debug_values(const uint8_t *d_in, int32_t H, int32_t W, int64_t in_pitch, float *d_vals,
                     const dfg_params *prm, void *stream)
{
    int rc = validate(prm);
    if (rc) return rc;
    if (prm->family == DFG_IDENTITY) return fail(DFG_E_ARG, "identity has no aggregates");
    if (!d_vals) return fail(DFG_E_ARG, "null output");
    const long long px = (long long)H * W;
    uint8_t *tmp_out = nullptr;
    void *ws = nullptr;
    cudaError_t e = cudaMalloc(&tmp_out, 3 * (size_t)px);
    if (e == cudaSuccess) e = cudaMalloc(&ws, dfg_workspace_bytes(px));
    if (e == cudaSuccess) e = cudaMemset(ws, 0, dfg_workspace_bytes(px));
    if (e != cudaSuccess) {
        if (tmp_out) cudaFree(tmp_out);
        return cuda_fail(e, "debug allocation");
    }
    rc = run(d_in, H, W, 0, H, in_pitch, 0, tmp_out, 0, H, 3LL * W, 0, 1, prm, ws, dfg_workspace_bytes(px),
             stream, d_vals);
    cudaStreamSynchronize((cudaStream_t)stream);
    cudaFree(tmp_out);
    cudaFree(ws);
    return rc;
}

}  // extern "C"
