// dfg_internal.cuh -- shared device-side definitions for the directional
// filter kernels (fast FP32 decision kernel + float64 re-decision kernel).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "../../include/dirfilt_gpu.h"

namespace dfg {

enum { FAM_VMF = 1, FAM_BVDF = 2, FAM_DDF = 3, FAM_ACWDDF = 4, FAM_CWVMF = 5, FAM_CWDDF = 6 };

// What a family needs: angular aggregates (A), Minkowski aggregates (L), and
// the centre column d(i, centre) (CEN: ACWDDF, and the centre-weighted
// CWVMF / CWDDF of filters.py:296-337).
template <int FAM>
struct FamT {
    static constexpr bool A = FAM != FAM_VMF && FAM != FAM_CWVMF;
    static constexpr bool L = FAM != FAM_BVDF;
    static constexpr bool CEN = FAM == FAM_ACWDDF || FAM == FAM_CWVMF || FAM == FAM_CWDDF;
};
enum { ST_EXACT = 0, ST_MINIMAX = 1, ST_CHROMA = 2 };
enum { PC_2 = 0, PC_1 = 1, PC_GEN = 2 };  // Minkowski order: p == 2, p == 1, general

// Parameters of the float64 re-decision stage (reference constants in binary64).
struct FParams {
    int family, strategy, window;
    double p, self_term;
    double cs[5], ca[5];
    int lam;
    double threshold, slope, intercept;
    double cr_margin;  // relative decision margin below which pass 2 (CR acos) runs
};

// Kernel-side parameter block, passed by value (__grid_constant__: the
// tensor maps are read in place).
struct KParams {
    // bulk tensor maps of the input rows and the output rows ((3W bytes) x
    // rows x frames, uint8), valid when tma_in / tma_out (host-checked
    // alignment); the 5x5 / 7x7 / 3x3-CTA kernel uses them
    CUtensorMap tm_in, tm_out;
    int tma_in, tma_out;
    // geometry (rows are global image rows; see dfg_filter_rows)
    int global_H, W;
    int in_row0, in_rows;
    int out_row0, out_rows;
    long long in_pitch, out_pitch, in_fstride, out_fstride;
    int border;
    int n_frames;
    // FP32 copies of the spec constants
    float p, invp;
    float cs[5], ca[5];
    float self_term;
    float slope, intercept, threshold;
    float w[3];  // extra centre weights n - 2k + 1: ACWDDF k = lam..lam+2; CWVMF/CWDDF k = lam (w[0])
    // rigorous error budget of one FP32 aggregate against the reference's
    // float64 value: |agg32 - agg64| <= er * |agg| + ea   (angular term);
    // Minkowski aggregates carry er only.  ea_pair: one angular pair.
    float er, ea, ea_pair;
    // float64 constants (seam recompute in the minimax route)
    double cs64[5], ca64[5];
    // float64 re-decision stage
    FParams fp;
    unsigned *flag_count;  // [0] pixels re-decided in float64, [1] of those needing pass 2
    // diagnostics: 2n floats per pixel (angular aggregates, Minkowski aggregates)
    float *dbg;
    // 3x3 schedule hint: > 0 = the warp row-sweep kernel with this many rows
    // per chunk (host pipeline bands: short latency, overlapping launches)
    int w3_rpc;
    // diagnostics only (DFG_OPT_NO_FIXUP): skip the float64 re-decision, to
    // time its share -- results may then differ from the reference
    int diag_no_fixup;
};

// Process-wide schedule / diagnostic options (dfg_set_option, include/
// dirfilt_gpu.h): read by the host launch code, never from the environment.
struct Options {
    int s3_schedule = 0;    // DFG_OPT_S3_SCHEDULE: 0 auto, 1 warp row sweep, 2 CTA tiles
    int no_fixup = 0;       // DFG_OPT_NO_FIXUP (diagnostics: results may differ)
    int host_bands = 0;     // DFG_OPT_HOST_BANDS: 0 auto
    int host_graph = 1;     // DFG_OPT_HOST_GRAPH
    int host_w3_rpc = 8;    // DFG_OPT_HOST_W3_RPC: rows per chunk of the host pipeline's 3x3 band kernels
    int frame_slots = 4;    // DFG_OPT_FRAME_SLOTS: device slots of dfg_filter_host_frames (1..8)
    int w3_wps = 0;         // DFG_OPT_W3_WPS: resident warps per SM the 3x3 chunking targets (0 auto)
    int w3_rpc = 0;         // DFG_OPT_W3_RPC: rows per chunk of the 3x3 row sweep (0 auto)
    int w3_small_wps = 12;  // DFG_OPT_W3_SMALL_WPS: warps per SM for single-wave 3x3 frames
    double cr_margin = 1e-12;  // DFG_OPT_CR_MARGIN: relative margin that triggers the CR-acos pass
    int persist = 1;        // DFG_OPT_PERSIST: CTA kernels as one wave of persistent CTAs (0: one tile per CTA)
    int tma = 3;            // DFG_OPT_TMA: bulk tensor copies of the CTA kernels' tiles: 1 input, 2 output, 3 both
};
Options &options();
// Window sides above 7 run the float64 direct kernel (dfg_wide.cu), up to
// this side (its per-CTA tables are n * 88 bytes of shared memory)
constexpr int kWideMaxSide = 31;
cudaError_t launch_wide(cudaStream_t st, const uint8_t *in, uint8_t *out, const struct KParams &kp);
int sm_count(int dev);  // multiProcessorCount, cached per device
// A 3-D uint8 tensor map (row bytes x rows x frames) with the given box;
// false when the base / strides do not meet the bulk-copy alignment rules
// (16-byte base and strides) or the driver entry point is unavailable.
bool encode_rows_map(CUtensorMap *map, const void *base, long long row_bytes, int rows, int frames, long long pitch,
                     long long fstride, const int box[3]);

// Border policy resolution (image.py:158-176): replicate = clamp,
// reflect = numpy 'symmetric' (edge-inclusive mirror, periodic).
__host__ __device__ __forceinline__ int resolve_idx(int i, int size, int border)
{
    if (border == DFG_REPLICATE) return i < 0 ? 0 : (i >= size ? size - 1 : i);
    if (size == 1) return 0;
    int period = 2 * size;
    i %= period;
    if (i < 0) i += period;
    return i < size ? i : period - 1 - i;
}

}  // namespace dfg

// Launchers defined per instantiation unit (fast_s*.cu); return a cudaError_t.
#define DFG_DECLARE_LAUNCH(S, FAMNAME)                                                         \
    cudaError_t dfg_launch_s##S##_##FAMNAME(int strategy, int pcode, cudaStream_t st,           \
                                            const uint8_t *in, uint8_t *out,                   \
                                            const dfg::KParams &kp);

DFG_DECLARE_LAUNCH(3, vmf)
DFG_DECLARE_LAUNCH(3, bvdf)
DFG_DECLARE_LAUNCH(3, ddf)
DFG_DECLARE_LAUNCH(3, acwddf)
DFG_DECLARE_LAUNCH(5, vmf)
DFG_DECLARE_LAUNCH(5, bvdf)
DFG_DECLARE_LAUNCH(5, ddf)
DFG_DECLARE_LAUNCH(5, acwddf)
DFG_DECLARE_LAUNCH(7, vmf)
DFG_DECLARE_LAUNCH(7, bvdf)
DFG_DECLARE_LAUNCH(7, ddf)
DFG_DECLARE_LAUNCH(7, acwddf)
DFG_DECLARE_LAUNCH(3, cwvmf)
DFG_DECLARE_LAUNCH(3, cwddf)
DFG_DECLARE_LAUNCH(5, cwvmf)
DFG_DECLARE_LAUNCH(5, cwddf)
DFG_DECLARE_LAUNCH(7, cwvmf)
DFG_DECLARE_LAUNCH(7, cwddf)

