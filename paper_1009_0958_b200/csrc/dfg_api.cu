// dfg_api.cu -- C ABI (include/dirfilt_gpu.h) over the directional filter
// kernels: validation (the reference's ValueError cases), parameter
// packing, the FP32 decision launch and the float64 re-decision launch.
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>
#if defined(__linux__)
#include <sys/mman.h>
#endif

#include <atomic>
#include <string>
#include <thread>
#include <vector>

#include "dfg_internal.cuh"

namespace dfg {

unsigned f64_to_u8(const double *src, uint8_t *dst, size_t lo, size_t hi);  // dfg_hostconv.cu
void u8_to_f64(const uint8_t *src, double *dst, size_t lo, size_t hi);

Options &options()
{
    static Options o;
    return o;
}

bool encode_rows_map(CUtensorMap *map, const void *base, long long row_bytes, int rows, int frames, long long pitch,
                     long long fstride, const int box[3])
{
    static PFN_cuTensorMapEncodeTiled_v12000 encode = [] {
        void *fn = nullptr;
        cudaDriverEntryPointQueryResult q;
        if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q) != cudaSuccess ||
            q != cudaDriverEntryPointSuccess) {
            cudaGetLastError();
            fn = nullptr;
        }
        return reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(fn);
    }();
    if (!encode || !base) return false;
    if (((uintptr_t)base & 15) || (pitch & 15) || (frames > 1 && (fstride & 15))) return false;
    if (row_bytes < 16 || rows < 1 || frames < 1 || pitch >= (1LL << 40) || fstride >= (1LL << 40)) return false;
    const cuuint64_t dims[3] = {(cuuint64_t)row_bytes, (cuuint64_t)rows, (cuuint64_t)frames};
    const cuuint64_t strides[2] = {(cuuint64_t)pitch, (cuuint64_t)(frames > 1 ? fstride : pitch * rows)};
    const cuuint32_t bx[3] = {(cuuint32_t)box[0], (cuuint32_t)box[1], (cuuint32_t)box[2]};
    const cuuint32_t es[3] = {1, 1, 1};
    return encode(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 3, const_cast<void *>(base), dims, strides, bx, es,
                  CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_128B,
                  CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

int sm_count(int dev)
{
    static int cache[64] = {};
    if (dev < 0 || dev >= 64) dev = 0;
    if (cache[dev] == 0) {
        int n = 0;
        if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0) {
            cudaGetLastError();
            n = 148;
        }
        cache[dev] = n;
    }
    return cache[dev];
}

}  // namespace dfg

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
    if (p->family < DFG_IDENTITY || p->family > DFG_CWDDF) return fail(DFG_E_ARG, "unknown filter family");
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
    if (p->family == DFG_CWVMF || p->family == DFG_CWDDF) {  // center_weight, filters.py:85-94
        const int n = p->window * p->window, d = (n + 1) / 2;
        if (p->lam < 1 || p->lam > d) return fail(DFG_E_ARG, "smoothing level k must be in [1, (n+1)/2]");
    }
    if (p->family != DFG_IDENTITY && p->window > dfg::kWideMaxSide)
        return fail(DFG_E_UNSUP, "this build supports odd window sides 3 .. 31");
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
    fp.cr_margin = dfg::options().cr_margin;
}

int pcode_of(double p) { return p == 2.0 ? dfg::PC_2 : (p == 1.0 ? dfg::PC_1 : dfg::PC_GEN); }

cudaError_t launch_fast(const dfg_params *p, cudaStream_t st, const uint8_t *in, uint8_t *out,
                        const dfg::KParams &kp)
{
    const int pc = pcode_of(p->p);
    if (p->window > 7) return dfg::launch_wide(st, in, out, kp);  // float64 direct (dfg_wide.cu)
#define DFG_CASE(S)                                                                    \
    if (p->window == S) {                                                              \
        switch (p->family) {                                                           \
        case DFG_VMF: return dfg_launch_s##S##_vmf(p->strategy, pc, st, in, out, kp);  \
        case DFG_BVDF: return dfg_launch_s##S##_bvdf(p->strategy, pc, st, in, out, kp); \
        case DFG_DDF: return dfg_launch_s##S##_ddf(p->strategy, pc, st, in, out, kp);  \
        case DFG_CWVMF: return dfg_launch_s##S##_cwvmf(p->strategy, pc, st, in, out, kp); \
        case DFG_CWDDF: return dfg_launch_s##S##_cwddf(p->strategy, pc, st, in, out, kp); \
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
        void *stream, float *dbg, int w3_rpc = 0)
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
    kp.diag_no_fixup = dfg::options().no_fixup;
    kp.w3_rpc = w3_rpc;

    cudaError_t e = launch_fast(prm, st, d_in, d_out, kp);
    if (e != cudaSuccess) return cuda_fail(e, "fast kernel launch");
    return DFG_OK;
}

constexpr int kMaxBands = 16;
constexpr int kGraphs = 4;
constexpr int kKStreams = 4;

// One captured host-path pipeline (pinned buffers): replayed with a single
// cudaGraphLaunch while the key matches.
struct GraphEntry {
    const uint8_t *h_in = nullptr;
    uint8_t *h_out = nullptr;
    int H = 0, W = 0, nb = 0;
    dfg_params prm{};
    cudaGraphExec_t exec = nullptr;
    unsigned long long used = 0;
};

struct HostCache {
    uint8_t *d_in = nullptr, *d_out = nullptr;
    void *ws = nullptr;
    size_t px_cap = 0;
    int dev = -1;
    cudaStream_t s_in = nullptr, s_out = nullptr, s_cap = nullptr;  // copy streams (H2D / D2H engines), capture
    cudaStream_t s_k[kKStreams] = {};                                // band kernels (overlapping)
    cudaEvent_t ev_start = nullptr, ev_done = nullptr, ev_in[kMaxBands] = {}, ev_k[kMaxBands] = {};
    cudaEvent_t ev_out[kMaxBands] = {};  // band k's D2H done (the float64 pipeline's output conversion waits on it)
    GraphEntry graphs[kGraphs];
    unsigned long long tick = 0;
    void drop_graphs()
    {
        for (GraphEntry &g : graphs) {
            if (g.exec) cudaGraphExecDestroy(g.exec);
            g = GraphEntry();
        }
    }
    void release()
    {
        drop_graphs();
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
    (void)n_pixels;  // diagnostic counters only (the size is kept in the ABI for growth)
    return kWsHeader;
}

int dfg_set_option(int32_t key, double value)
{
    dfg::Options &o = dfg::options();
    const int v = (int)value;
    switch (key) {
    case DFG_OPT_S3_SCHEDULE: o.s3_schedule = v; break;
    case DFG_OPT_NO_FIXUP: o.no_fixup = v; break;
    case DFG_OPT_HOST_BANDS: o.host_bands = v; break;
    case DFG_OPT_HOST_GRAPH: o.host_graph = v; break;
    case DFG_OPT_HOST_W3_RPC: o.host_w3_rpc = v; break;
    case DFG_OPT_FRAME_SLOTS: o.frame_slots = v; break;
    case DFG_OPT_W3_WPS: o.w3_wps = v; break;
    case DFG_OPT_W3_RPC: o.w3_rpc = v; break;
    case DFG_OPT_W3_SMALL_WPS: o.w3_small_wps = v; break;
    case DFG_OPT_CR_MARGIN: o.cr_margin = value; break;
    case DFG_OPT_TMA: o.tma = v; break;
    case DFG_OPT_PERSIST: o.persist = v; break;
    default: return fail(DFG_E_ARG, "unknown option key");
    }
    g_host.drop_graphs();  // captured pipelines bake the old settings in
    return DFG_OK;
}

double dfg_get_option(int32_t key)
{
    const dfg::Options &o = dfg::options();
    switch (key) {
    case DFG_OPT_S3_SCHEDULE: return o.s3_schedule;
    case DFG_OPT_NO_FIXUP: return o.no_fixup;
    case DFG_OPT_HOST_BANDS: return o.host_bands;
    case DFG_OPT_HOST_GRAPH: return o.host_graph;
    case DFG_OPT_HOST_W3_RPC: return o.host_w3_rpc;
    case DFG_OPT_FRAME_SLOTS: return o.frame_slots;
    case DFG_OPT_W3_WPS: return o.w3_wps;
    case DFG_OPT_W3_RPC: return o.w3_rpc;
    case DFG_OPT_W3_SMALL_WPS: return o.w3_small_wps;
    case DFG_OPT_CR_MARGIN: return o.cr_margin;
    case DFG_OPT_TMA: return o.tma;
    case DFG_OPT_PERSIST: return o.persist;
    default: return NAN;
    }
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

}  // extern "C"

namespace {

// Row-band pipeline: the H2D copies of all bands stream on one copy engine,
// the D2H copies on the other (PCIe is full duplex), and band k's kernel runs
// as soon as the input rows its windows reach (band k+1's first rows) have
// landed.  Band kernels go round-robin to kKStreams streams so they overlap
// each other as well as the copies; for 3x3 they use the warp row-sweep
// kernel with short chunks (low latency per band; the SMs are otherwise idle
// during the copies).  Fork and join are events on `st`, so the same sequence
// is also capturable into a CUDA graph.
int enqueue_bands(HostCache &c, const uint8_t *h_in, int H, int W, uint8_t *h_out, const dfg_params *prm,
                  cudaStream_t st, int nb, int w3_rpc)
{
    const int h = (prm->family == DFG_IDENTITY) ? 0 : prm->window / 2;
    const long long pitch = 3LL * W;
    const size_t px = (size_t)H * W;
    auto row0 = [&](int k) { return k >= nb ? H : (int)((long long)k * H / nb); };  // equal bands
    const int nks = nb < kKStreams ? nb : kKStreams;
    cudaError_t e = cudaEventRecord(c.ev_start, st);  // buffers are free once prior work on `st` is done
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c.s_in, c.ev_start, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c.s_out, c.ev_start, 0);
    for (int k = 0; k < nks && e == cudaSuccess; k++) e = cudaStreamWaitEvent(c.s_k[k], c.ev_start, 0);
    // band k's copy includes the h halo rows below it (rows the next band
    // copies again -- identical bytes), so its kernel depends on its own
    // copy only; the halo above arrived with the earlier bands
    for (int k = 0; k < nb && e == cudaSuccess; k++) {
        const int r0 = row0(k), r1 = row0(k + 1);
        const int c0 = k == 0 ? 0 : r0 + h, c1 = k + 1 == nb ? H : r1 + h;  // rows [c0, c1)
        if (c1 > c0)
            e = cudaMemcpyAsync(c.d_in + c0 * pitch, h_in + c0 * pitch, (size_t)(c1 - c0) * pitch,
                                cudaMemcpyHostToDevice, c.s_in);
        if (e == cudaSuccess) e = cudaEventRecord(c.ev_in[k], c.s_in);
    }
    if (e != cudaSuccess) return cuda_fail(e, "H2D");
    for (int k = 0; k < nb; k++) {
        const int r0 = row0(k), r1 = row0(k + 1);
        cudaStream_t sk = c.s_k[k % nks];
        e = cudaStreamWaitEvent(sk, c.ev_in[k], 0);
        if (e != cudaSuccess) return cuda_fail(e, "band dependency");
        int rc = run(c.d_in, H, W, 0, H, pitch, 0, c.d_out + r0 * pitch, r0, r1 - r0, pitch, 0, 1, prm, c.ws,
                     dfg_workspace_bytes((int64_t)px), sk, nullptr, nb > 1 ? w3_rpc : 0);
        if (rc) return rc;
        e = cudaEventRecord(c.ev_k[k], sk);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(c.s_out, c.ev_k[k], 0);
        if (e == cudaSuccess)
            e = cudaMemcpyAsync(h_out + r0 * pitch, c.d_out + r0 * pitch, (size_t)(r1 - r0) * pitch,
                                cudaMemcpyDeviceToHost, c.s_out);
        if (e != cudaSuccess) return cuda_fail(e, "D2H");
    }
    e = cudaEventRecord(c.ev_done, c.s_out);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, c.ev_done, 0);  // join: later work on `st` sees the result
    if (e != cudaSuccess) return cuda_fail(e, "join");
    return DFG_OK;
}

// Device staging, streams and events of the host paths (per thread; grows).
int ensure_host_cache(HostCache &c, size_t px)
{
    int dev = 0;
    cudaGetDevice(&dev);
    if (c.dev != dev || c.px_cap < px) {
        c.release();
        cudaError_t e = cudaMalloc(&c.d_in, 3 * px);
        if (e == cudaSuccess) e = cudaMalloc(&c.d_out, 3 * px);
        if (e == cudaSuccess) e = cudaMalloc(&c.ws, dfg_workspace_bytes((int64_t)px));
        if (e == cudaSuccess) e = cudaMemset(c.ws, 0, dfg_workspace_bytes((int64_t)px));
        if (e == cudaSuccess && c.dev != dev) {
            e = cudaStreamCreateWithFlags(&c.s_in, cudaStreamNonBlocking);
            if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c.s_out, cudaStreamNonBlocking);
            if (e == cudaSuccess) e = cudaStreamCreateWithFlags(&c.s_cap, cudaStreamNonBlocking);
            for (int k = 0; k < kKStreams && e == cudaSuccess; k++)
                e = cudaStreamCreateWithFlags(&c.s_k[k], cudaStreamNonBlocking);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.ev_start, cudaEventDisableTiming);
            if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.ev_done, cudaEventDisableTiming);
            for (int k = 0; k < kMaxBands && e == cudaSuccess; k++) {
                e = cudaEventCreateWithFlags(&c.ev_in[k], cudaEventDisableTiming);
                if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.ev_k[k], cudaEventDisableTiming);
                if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.ev_out[k], cudaEventDisableTiming);
            }
        }
        if (e != cudaSuccess) {
            c.release();
            return cuda_fail(e, "device staging allocation");
        }
        c.px_cap = px;
        c.dev = dev;
    }
    return DFG_OK;
}

bool is_pinned(const void *p)
{
    cudaPointerAttributes a;
    if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
        cudaGetLastError();  // clear the query's error state
        return false;
    }
    return a.type == cudaMemoryTypeHost;
}

}  // namespace

extern "C" {

int dfg_filter_host(const uint8_t *h_in, int32_t H, int32_t W, uint8_t *h_out, const dfg_params *prm,
                    void *stream)
{
    int rc = validate(prm);
    if (rc) return rc;
    if (H < 1 || W < 1) return fail(DFG_E_ARG, "image must contain at least one pixel");
    if (!h_in || !h_out) return fail(DFG_E_ARG, "null host pointer");
    HostCache &c = g_host;
    const size_t px = (size_t)H * W;
    cudaStream_t st = (cudaStream_t)stream;
    rc = ensure_host_cache(c, px);
    if (rc) return rc;
    const bool pinned = is_pinned(h_in) && is_pinned(h_out);
    const int h = (prm->family == DFG_IDENTITY) ? 0 : prm->window / 2;
    const dfg::Options &opt = dfg::options();
    const int nb_env = opt.host_bands;
    const bool use_graph = pinned && opt.host_graph != 0;
    // Eager issue costs ~25 us of API calls per band, so bands only pay off
    // above ~0.5 M pixels each; a replayed graph has no per-band host cost,
    // but every copy still costs the copy engine ~5 us: measured best at
    // 2-4 bands for 1024^2 (137-141 us vs 178 us unbanded), 4 for 4096^2.
    int nb = nb_env > 0 ? nb_env : (int)(px / (use_graph ? 256 * 1024 : 512 * 1024));
    if (nb_env <= 0 && nb > 8) nb = 8;
    if (nb > H / 64) nb = H / 64;
    nb = nb < 1 ? 1 : (nb > kMaxBands ? kMaxBands : nb);
    if (prm->border == DFG_REFLECT && H <= 4 * h) nb = 1;
    const int w3_rpc = opt.host_w3_rpc;
    cudaError_t e;
    if (use_graph) {
        GraphEntry *g = nullptr, *victim = &c.graphs[0];
        for (GraphEntry &x : c.graphs) {
            if (x.exec && x.h_in == h_in && x.h_out == h_out && x.H == H && x.W == W && x.nb == nb &&
                memcmp(&x.prm, prm, sizeof(dfg_params)) == 0) {
                g = &x;
                break;
            }
            if (!x.exec || x.used < victim->used) victim = &x;
        }
        if (!g) {
            // capture the pipeline once: the kernels' attributes are set
            // outside capture by an eager first call
            if (victim->exec) cudaGraphExecDestroy(victim->exec);
            *victim = GraphEntry();
            rc = enqueue_bands(c, h_in, H, W, h_out, prm, c.s_cap, nb, w3_rpc);
            if (rc) return rc;
            e = cudaStreamSynchronize(c.s_cap);
            if (e != cudaSuccess) return cuda_fail(e, "warm-up");
            cudaGraph_t graph = nullptr;
            e = cudaStreamBeginCapture(c.s_cap, cudaStreamCaptureModeThreadLocal);
            if (e != cudaSuccess) return cuda_fail(e, "begin capture");
            rc = enqueue_bands(c, h_in, H, W, h_out, prm, c.s_cap, nb, w3_rpc);
            e = cudaStreamEndCapture(c.s_cap, &graph);
            if (rc) {
                if (graph) cudaGraphDestroy(graph);
                return rc;
            }
            if (e != cudaSuccess) return cuda_fail(e, "end capture");
            e = cudaGraphInstantiate(&victim->exec, graph, 0);
            cudaGraphDestroy(graph);
            if (e != cudaSuccess) {
                victim->exec = nullptr;
                return cuda_fail(e, "graph instantiate");
            }
            victim->h_in = h_in;
            victim->h_out = h_out;
            victim->H = H;
            victim->W = W;
            victim->nb = nb;
            victim->prm = *prm;
            g = victim;
        }
        g->used = ++c.tick;
        e = cudaGraphLaunch(g->exec, st);
        if (e == cudaSuccess) e = cudaStreamSynchronize(st);
        if (e != cudaSuccess) return cuda_fail(e, "graph launch");
        return DFG_OK;
    }
    rc = enqueue_bands(c, h_in, H, W, h_out, prm, st, nb, w3_rpc);
    if (rc) return rc;
    e = cudaEventSynchronize(c.ev_done);
    if (e != cudaSuccess) return cuda_fail(e, "synchronize");
    return DFG_OK;
}

}  // extern "C"

namespace {

// Frame stream from host memory: frame_slots() device slots (default 4),
// each with its own input/output buffers, workspace and stream.  Frame f
// goes to slot f % S: H2D, kernel, D2H in that slot's stream, so frame f's
// H2D overlaps the kernels and D2H copies of the frames before it (PCIe is
// full duplex and the SMs are idle during the copies); a slot is reused only
// after its previous frame's D2H.  Measured (C2 frames, 3 MB each way):
// 2 slots 100 us per frame, 3 slots 86, 4 slots 72.5, 5 slots 73-83.
constexpr int kFrameSlots = 8;  // capacity; frame_slots() are used

struct FrameCache {
    uint8_t *d_in[kFrameSlots] = {}, *d_out[kFrameSlots] = {};
    void *ws[kFrameSlots] = {};
    cudaStream_t s[kFrameSlots] = {};
    cudaEvent_t ev_start = nullptr, ev_end[kFrameSlots] = {};
    size_t px_cap = 0;
    int dev = -1;
    void release()
    {
        for (int k = 0; k < kFrameSlots; k++) {
            if (d_in[k]) cudaFree(d_in[k]);
            if (d_out[k]) cudaFree(d_out[k]);
            if (ws[k]) cudaFree(ws[k]);
            d_in[k] = d_out[k] = nullptr;
            ws[k] = nullptr;
        }
        px_cap = 0;
    }
    ~FrameCache() { release(); }
};
thread_local FrameCache g_frames;

// slots in use (DFG_OPT_FRAME_SLOTS, 1..8); fixed by the first allocation
int frame_slots()
{
    const int v = dfg::options().frame_slots;
    return v < 1 ? 1 : (v > kFrameSlots ? kFrameSlots : v);
}

}  // namespace

extern "C" {

int dfg_filter_host_frames(const uint8_t *const *h_in, uint8_t *const *h_out, int32_t n_frames, int32_t H,
                           int32_t W, const dfg_params *prm, void *stream)
{
    int rc = validate(prm);
    if (rc) return rc;
    if (n_frames < 0) return fail(DFG_E_ARG, "negative frame count");
    if (H < 1 || W < 1) return fail(DFG_E_ARG, "image must contain at least one pixel");
    if (n_frames == 0) return DFG_OK;
    if (!h_in || !h_out) return fail(DFG_E_ARG, "null frame list");
    for (int f = 0; f < n_frames; f++)
        if (!h_in[f] || !h_out[f]) return fail(DFG_E_ARG, "null host frame pointer");
    int dev = 0;
    cudaGetDevice(&dev);
    FrameCache &c = g_frames;
    const size_t px = (size_t)H * W, nbytes = 3 * px;
    const size_t wsb = dfg_workspace_bytes((int64_t)px);
    cudaError_t e = cudaSuccess;
    if (c.dev != dev || c.px_cap < px) {
        c.release();
        for (int k = 0; k < frame_slots() && e == cudaSuccess; k++) {
            e = cudaMalloc(&c.d_in[k], nbytes);
            if (e == cudaSuccess) e = cudaMalloc(&c.d_out[k], nbytes);
            if (e == cudaSuccess) e = cudaMalloc(&c.ws[k], wsb);
            if (e == cudaSuccess) e = cudaMemset(c.ws[k], 0, wsb);
        }
        if (e == cudaSuccess && c.dev != dev) {
            e = cudaEventCreateWithFlags(&c.ev_start, cudaEventDisableTiming);
            for (int k = 0; k < kFrameSlots && e == cudaSuccess; k++) {
                e = cudaStreamCreateWithFlags(&c.s[k], cudaStreamNonBlocking);
                if (e == cudaSuccess) e = cudaEventCreateWithFlags(&c.ev_end[k], cudaEventDisableTiming);
            }
        }
        if (e != cudaSuccess) {
            c.release();
            return cuda_fail(e, "frame slot allocation");
        }
        c.px_cap = px;
        c.dev = dev;
    }
    cudaStream_t st = (cudaStream_t)stream;
    const int ns = frame_slots();
    // fork: the slots start after prior work on `st`
    e = cudaEventRecord(c.ev_start, st);
    for (int k = 0; k < ns && e == cudaSuccess; k++) e = cudaStreamWaitEvent(c.s[k], c.ev_start, 0);
    if (e != cudaSuccess) return cuda_fail(e, "fork");
    const long long pitch = 3LL * W;
    for (int f = 0; f < n_frames; f++) {
        const int k = f % ns;
        e = cudaMemcpyAsync(c.d_in[k], h_in[f], nbytes, cudaMemcpyHostToDevice, c.s[k]);
        if (e != cudaSuccess) return cuda_fail(e, "frame H2D");
        rc = run(c.d_in[k], H, W, 0, H, pitch, 0, c.d_out[k], 0, H, pitch, 0, 1, prm, c.ws[k], wsb, c.s[k], nullptr);
        if (rc) return rc;
        e = cudaMemcpyAsync(h_out[f], c.d_out[k], nbytes, cudaMemcpyDeviceToHost, c.s[k]);
        if (e != cudaSuccess) return cuda_fail(e, "frame D2H");
    }
    // join, then wait for the whole stream of frames
    for (int k = 0; k < ns && e == cudaSuccess; k++) {
        e = cudaEventRecord(c.ev_end[k], c.s[k]);
        if (e == cudaSuccess) e = cudaStreamWaitEvent(st, c.ev_end[k], 0);
    }
    if (e == cudaSuccess) e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) return cuda_fail(e, "frame stream synchronize");
    return DFG_OK;
}

}  // extern "C"

namespace {

// Run f(lo, hi) over [0, n) split into `threads` contiguous ranges.
template <typename F>
void parallel_ranges(size_t n, int threads, F &&f)
{
    if (threads <= 1 || n < (1u << 18)) {
        f((size_t)0, n);
        return;
    }
    std::vector<std::thread> pool;
    pool.reserve(threads - 1);
    const size_t step = (n + threads - 1) / threads;
    for (int t = 1; t < threads; t++) {
        const size_t lo = (size_t)t * step, hi = lo + step < n ? lo + step : n;
        if (lo < hi) pool.emplace_back([&f, lo, hi] { f(lo, hi); });
    }
    f((size_t)0, step < n ? step : n);
    for (std::thread &t : pool) t.join();
}

// Pinned uint8 staging of the float64 host path (per thread, grows).
struct F64Staging {
    uint8_t *in = nullptr, *out = nullptr;
    size_t cap = 0;
    void release()
    {
        if (in) cudaFreeHost(in);
        if (out) cudaFreeHost(out);
        in = out = nullptr;
        cap = 0;
    }
    ~F64Staging() { release(); }
};
thread_local F64Staging g_f64;

// float64 <-> uint8 conversions of the drop-in path: dfg_hostconv.cu
// Large frames: the conversions run band by band on `threads` host threads
// around the device pipeline, so the float64 -> uint8 pass of band k + 1
// overlaps band k's H2D / kernel / D2H, and the uint8 -> float64 pass of
// band k starts as soon as its D2H has landed (the sequential form -- convert
// everything, run the pipeline, convert everything back -- costs the sum of
// the three).  Bands, halo rows and stream roles are those of enqueue_bands.
// Nothing is written to h_out unless every input value passed the check.
int f64_pipeline(HostCache &c, F64Staging &g, const double *h_in, int H, int W, double *h_out, const dfg_params *prm,
                 int threads, cudaStream_t st, int nb)
{
    const int h = prm->window / 2;
    const long long pitch = 3LL * W;
    const size_t px = (size_t)H * W;
    auto row0 = [&](int k) { return k >= nb ? H : (int)((long long)k * H / nb); };
    const int nks = nb < kKStreams ? nb : kKStreams;
    int dev = 0;
    cudaGetDevice(&dev);
    cudaError_t e = cudaEventRecord(c.ev_start, st);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c.s_in, c.ev_start, 0);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(c.s_out, c.ev_start, 0);
    for (int k = 0; k < nks && e == cudaSuccess; k++) e = cudaStreamWaitEvent(c.s_k[k], c.ev_start, 0);
    if (e != cudaSuccess) return cuda_fail(e, "fork");

    const int T = threads < 1 ? 1 : threads;
    std::atomic<int> in_done[kMaxBands], state[kMaxBands];  // state: 0 pending, 1 enqueued, -1 abandoned
    for (int k = 0; k < kMaxBands; k++) {
        in_done[k].store(0);
        state[k].store(0);
    }
    std::atomic<unsigned> bad{0};
    int rc_enq = DFG_OK;          // thread 0 only
    cudaError_t e_enq = cudaSuccess;
    const char *where = "";
    const int w3_rpc = dfg::options().host_w3_rpc;

    auto enqueue_band = [&](int k) {  // thread 0: H2D, kernel, D2H of band k
        const int r0 = row0(k), r1 = row0(k + 1);
        const int c0 = k == 0 ? 0 : r0 + h, c1 = k + 1 == nb ? H : r1 + h;
        cudaStream_t sk = c.s_k[k % nks];
        if (c1 > c0)
            e_enq = cudaMemcpyAsync(c.d_in + c0 * pitch, g.in + c0 * pitch, (size_t)(c1 - c0) * pitch,
                                    cudaMemcpyHostToDevice, c.s_in);
        if (e_enq == cudaSuccess) e_enq = cudaEventRecord(c.ev_in[k], c.s_in);
        if (e_enq == cudaSuccess) e_enq = cudaStreamWaitEvent(sk, c.ev_in[k], 0);
        if (e_enq != cudaSuccess) { where = "H2D"; return; }
        rc_enq = run(c.d_in, H, W, 0, H, pitch, 0, c.d_out + r0 * pitch, r0, r1 - r0, pitch, 0, 1, prm, c.ws,
                     dfg_workspace_bytes((int64_t)px), sk, nullptr, w3_rpc);
        if (rc_enq) return;
        e_enq = cudaEventRecord(c.ev_k[k], sk);
        if (e_enq == cudaSuccess) e_enq = cudaStreamWaitEvent(c.s_out, c.ev_k[k], 0);
        if (e_enq == cudaSuccess)
            e_enq = cudaMemcpyAsync(g.out + r0 * pitch, c.d_out + r0 * pitch, (size_t)(r1 - r0) * pitch,
                                    cudaMemcpyDeviceToHost, c.s_out);
        if (e_enq == cudaSuccess) e_enq = cudaEventRecord(c.ev_out[k], c.s_out);
        if (e_enq != cudaSuccess) where = "D2H";
    };
    auto slice = [&](size_t lo, size_t hi, int t, size_t &a, size_t &b) {
        const size_t n = hi - lo, step = (n + T - 1) / T;
        a = lo + (size_t)t * step;
        b = a + step;
        if (a > hi) a = hi;
        if (b > hi) b = hi;
    };
    auto worker = [&](int t) {
        if (t != 0) cudaSetDevice(dev);
        // input bands: convert, then thread 0 enqueues the band's device work
        for (int k = 0; k < nb; k++) {
            const int r0 = row0(k), r1 = row0(k + 1);
            const int c0 = k == 0 ? 0 : r0 + h, c1 = k + 1 == nb ? H : r1 + h;
            size_t a, b;
            slice((size_t)c0 * pitch, (size_t)c1 * pitch, t, a, b);
            if (dfg::f64_to_u8(h_in, g.in, a, b)) bad.store(1u, std::memory_order_relaxed);
            in_done[k].fetch_add(1, std::memory_order_acq_rel);
            if (t == 0) {
                while (in_done[k].load(std::memory_order_acquire) < T) std::this_thread::yield();
                const bool ok = !bad.load() && rc_enq == DFG_OK && e_enq == cudaSuccess;
                if (ok) enqueue_band(k);
                state[k].store(ok && rc_enq == DFG_OK && e_enq == cudaSuccess ? 1 : -1, std::memory_order_release);
            }
        }
        // output bands: wait for the band's D2H, convert back.  (The last
        // input band is checked before any output is written: band nb - 1's
        // state is set only after every input value has been seen.)
        while (state[nb - 1].load(std::memory_order_acquire) == 0) std::this_thread::yield();
        if (state[nb - 1].load() < 0) return;
        for (int k = 0; k < nb; k++) {
            if (cudaEventSynchronize(c.ev_out[k]) != cudaSuccess) {
                bad.store(2u);
                return;
            }
            size_t a, b;
            slice((size_t)row0(k) * pitch, (size_t)row0(k + 1) * pitch, t, a, b);
            dfg::u8_to_f64(g.out, h_out, a, b);
        }
    };
    {
        std::vector<std::thread> pool;
        pool.reserve(T - 1);
        for (int t = 1; t < T; t++) pool.emplace_back(worker, t);
        worker(0);
        for (std::thread &th : pool) th.join();
    }
    // join: later work on `st` sees the result; drain whatever was enqueued
    e = cudaEventRecord(c.ev_done, c.s_out);
    if (e == cudaSuccess) e = cudaStreamWaitEvent(st, c.ev_done, 0);
    for (int k = 0; k < nks && e == cudaSuccess; k++) e = cudaStreamSynchronize(c.s_k[k]);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c.s_in);
    if (e == cudaSuccess) e = cudaStreamSynchronize(c.s_out);
    if (bad.load() == 1u) return fail(DFG_E_ARG, "pixel values must be integers in 0..255 on the GPU path");
    if (rc_enq) return rc_enq;
    if (e_enq != cudaSuccess) return cuda_fail(e_enq, where);
    if (e != cudaSuccess || bad.load() == 2u) return cuda_fail(e != cudaSuccess ? e : cudaGetLastError(), "float64 pipeline");
    return DFG_OK;
}

}  // namespace

extern "C" {

int dfg_filter_host_f64(const double *h_in, int32_t H, int32_t W, double *h_out, const dfg_params *prm,
                        int32_t threads, void *stream)
{
    int rc = validate(prm);
    if (rc) return rc;
    if (H < 1 || W < 1) return fail(DFG_E_ARG, "image must contain at least one pixel");
    if (!h_in || !h_out) return fail(DFG_E_ARG, "null host pointer");
    const size_t n = 3 * (size_t)H * W;
    if (threads <= 0) {
        const unsigned hc = std::thread::hardware_concurrency();
        threads = hc ? (int)hc : 1;
    }
    if (threads > 256) threads = 256;
    F64Staging &g = g_f64;
    if (g.cap < n) {
        g.release();
        cudaError_t e = cudaHostAlloc((void **)&g.in, n, cudaHostAllocDefault);
        if (e == cudaSuccess) e = cudaHostAlloc((void **)&g.out, n, cudaHostAllocDefault);
        if (e != cudaSuccess) {
            g.release();
            return cuda_fail(e, "pinned staging allocation");
        }
        g.cap = n;
    }
#if defined(__linux__)
    if (n * sizeof(double) >= (64u << 20)) {
        // a freshly allocated result array is first touched here: ask for huge
        // pages (2 MiB faults instead of 4 KiB ones; a hint, ignored if disabled)
        const uintptr_t a = ((uintptr_t)h_out + 4095) & ~(uintptr_t)4095;
        const uintptr_t b = ((uintptr_t)h_out + n * sizeof(double)) & ~(uintptr_t)4095;
        if (b > a) madvise((void *)a, b - a, MADV_HUGEPAGE);
    }
#endif
    // large frames: conversions pipelined around the device work, band by band
    const size_t px = (size_t)H * W;
    int nb = (int)(px / (1u << 20));
    if (nb > kMaxBands) nb = kMaxBands;
    if (nb > H / 64) nb = H / 64;
    const int h = prm->window / 2;
    if (prm->border == DFG_REFLECT && H <= 4 * h) nb = 1;
    if (dfg::options().host_bands > 0) nb = dfg::options().host_bands > kMaxBands ? kMaxBands : dfg::options().host_bands;
    if (prm->family != DFG_IDENTITY && nb >= 2 && nb <= H / (2 * h + 1)) {
        rc = ensure_host_cache(g_host, px);
        if (rc) return rc;
        return f64_pipeline(g_host, g, h_in, H, W, h_out, prm, threads, (cudaStream_t)stream, nb);
    }
    // float64 -> uint8 with the GPU path's one input restriction: integral
    // values in 0..255
    std::atomic<unsigned> bad{0};
    parallel_ranges(n, threads, [&](size_t lo, size_t hi) {
        if (dfg::f64_to_u8(h_in, g.in, lo, hi)) bad.store(1u, std::memory_order_relaxed);
    });
    if (bad.load()) return fail(DFG_E_ARG, "pixel values must be integers in 0..255 on the GPU path");
    rc = dfg_filter_host(g.in, H, W, g.out, prm, stream);
    if (rc) return rc;
    parallel_ranges(n, threads, [&](size_t lo, size_t hi) { dfg::u8_to_f64(g.out, h_out, lo, hi); });
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
