/*
 * dirfilt_gpu.h -- C ABI of the B200 (sm_100a) directional vector filter path.
 *
 * Drop-in boundary for the reference's whole-image driver:
 *
 *   reference                                     replaced by
 *   --------------------------------------------  -------------------------------
 *   filters.apply_filter            filters.py:379-433   dfg_filter / dfg_filter_host
 *   _engine.EnginePlanes (prep)     _engine.py:513-557   staging stage inside dfg_filter
 *   _engine.run_rows(.., r0, r1)    _engine.py:560-583   dfg_filter_rows (row band)
 *   apply_filter(workers=k) bands   filters.py:416-430   dfg_filter_rows per GPU strip
 *   (frame loop in bench/CLI)       bench.py:96-109      dfg_filter_batch
 *   noise.corrupt_image             noise.py:85-116      dfg_corrupt_image
 *   metrics.compare / mae/psnr/ncd  metrics.py:64-118    dfg_image_metrics
 *   calibration.fit_angular_...     calibration.py:83-125 dfg_calib_reduce/_samples
 *
 * The reference has no FFI of its own (pure Python + numba); these entry
 * points are what its filters.py would bind through ctypes -- INTEGRATION.md
 * shows that binding.  Plain C types only: device pointers, sizes, one POD
 * parameter struct, an opaque cudaStream_t passed as void*.
 *
 * Images are uint8 RGB, interleaved (H, W, 3), row pitch in bytes.  The
 * reference's float64 RasterImage holding integers 0..255 maps onto this
 * losslessly; non-integral or >255 pixels are rejected by the host shim.
 *
 * Results are the reference's selections: every output pixel is the input
 * pixel the reference's float64 engine selects for that window.  The fast
 * FP32 kernel decides every pixel whose decision margin exceeds its
 * rigorous error budget; the rest are re-decided by a float64 kernel that
 * repeats the reference's operation order ("Exactness").
 *
 * Every call returns 0 on success or a negative DFG_E* code; the message is
 * available from dfg_last_error() (thread-local).  Calls are stateless,
 * re-entrant per stream, and do not allocate (except dfg_filter_host, which
 * keeps a per-thread cached device staging buffer).
 */
#ifndef DIRFILT_GPU_H
#define DIRFILT_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define DFG_ABI_VERSION 1

#if defined(__GNUC__)
#define DFG_API __attribute__((visibility("default")))
#else
#define DFG_API
#endif

/* family: filters.py:34 FAMILIES */
#define DFG_IDENTITY 0
#define DFG_VMF 1
#define DFG_BVDF 2
#define DFG_DDF 3
#define DFG_ACWDDF 4
/* extensions: the reference's window-level centre-weighted
 * filters applied to every window -- cwvmf(w, k, p) filters.py:331-337 and
 * cwddf(w, k, p, strategy) filters.py:304-328; smoothing level k in `lam` */
#define DFG_CWVMF 5
#define DFG_CWDDF 6

/* strategy: filters.py:37-82 DirectionalStrategy.kind, _engine.py:25-28 */
#define DFG_EXACT 0
#define DFG_MINIMAX 1
#define DFG_CHROMA 2

/* border: image.py:32-55 BorderPolicy (replicate = np.pad edge, reflect = symmetric) */
#define DFG_REPLICATE 0
#define DFG_REFLECT 1

/* error codes */
#define DFG_OK 0
#define DFG_E_ARG (-1)     /* invalid argument (maps to the reference's ValueError) */
#define DFG_E_CUDA (-2)    /* CUDA runtime error */
#define DFG_E_UNSUP (-3)   /* valid spec outside this build (window side > 31) */
#define DFG_E_WS (-4)      /* workspace too small */

/* Mirrors FilterSpec (filters.py:126-151) + AcwddfParams (filters.py:97-123)
 * + the engine's padded coefficient tuples (_engine.py:504-510). */
typedef struct dfg_params {
    int32_t family;
    int32_t strategy;
    int32_t window;      /* odd side s >= 3; this build: up to 31 */
    int32_t border;
    double p;            /* Minkowski order: spec.p, or acwddf.p for ACWDDF (filters.py:398) */
    double asin_c[5];    /* ASIN polynomial a0..a4, zero-padded (minimax only) */
    double acos_c[5];    /* ACOS polynomial a0..a4, zero-padded (minimax only) */
    int32_t lam;         /* ACWDDF smoothing level lambda (>= 1, lambda + 2 <= (n+1)/2); CW*: k */
    int32_t reserved;
    double threshold;    /* ACWDDF switching threshold T */
    double slope;        /* chromaticity calibration (ACWDDF switching sum only) */
    double intercept;
} dfg_params;

DFG_API int dfg_abi_version(void);
DFG_API const char *dfg_last_error(void);

/* Device workspace of a filter call (n_pixels output pixels): the diagnostic
 * counters of dfg_fixup_count.  Zero it once after allocation; calls only
 * add to the counters, so calls on different streams may share it. */
DFG_API size_t dfg_workspace_bytes(int64_t n_pixels);

/* Whole image: d_in (H, W, 3) -> d_out (H, W, 3), both device memory. */
DFG_API int dfg_filter(const uint8_t *d_in, int32_t H, int32_t W, int64_t in_pitch,
               uint8_t *d_out, int64_t out_pitch, const dfg_params *prm,
               void *d_workspace, size_t workspace_bytes, void *stream);

/* Row band of an image of global_H rows (multi-GPU strips, reference
 * run_rows(r0, r1)).  d_in holds global rows [in_row0, in_row0 + in_rows);
 * it must include every row the border policy resolves for output rows
 * [out_row0, out_row0 + out_rows) (for replicate: a halo of s/2 rows
 * clipped to the image).  d_out receives exactly out_rows rows. */
DFG_API int dfg_filter_rows(const uint8_t *d_in, int32_t global_H, int32_t W,
                    int32_t in_row0, int32_t in_rows, int64_t in_pitch,
                    uint8_t *d_out, int32_t out_row0, int32_t out_rows, int64_t out_pitch,
                    const dfg_params *prm, void *d_workspace, size_t workspace_bytes,
                    void *stream);

/* B independent frames of (H, W, 3), frame strides in bytes. */
DFG_API int dfg_filter_batch(const uint8_t *d_in, int32_t B, int32_t H, int32_t W,
                     int64_t in_pitch, int64_t in_frame_stride,
                     uint8_t *d_out, int64_t out_pitch, int64_t out_frame_stride,
                     const dfg_params *prm, void *d_workspace, size_t workspace_bytes,
                     void *stream);

/* End to end from HOST memory (pinned or pageable), synchronised before
 * return: cached per-thread device buffers and a row-band pipeline -- H2D
 * and D2H copy streams, band kernels on four streams, each band's copy
 * carrying its halo rows; with pinned buffers the pipeline is captured once
 * and replayed as a CUDA graph (cache keyed on buffers, shape, params). */
DFG_API int dfg_filter_host(const uint8_t *h_in, int32_t H, int32_t W, uint8_t *h_out,
                    const dfg_params *prm, void *stream);

/* The reference's own boundary (RasterImage pixels: C-contiguous float64
 * (H, W, 3), image.py:65-75) end to end from HOST memory: the values are
 * validated and converted to uint8 on `threads` host threads (0: all cores)
 * into cached pinned staging buffers, filtered by the dfg_filter_host
 * pipeline, and written back to h_out as float64.  Values that are not
 * integers in 0..255 (incl. NaN/inf) return DFG_E_ARG -- the GPU path's one
 * restriction against the reference, which accepts any finite nonnegative
 * float64. */
DFG_API int dfg_filter_host_f64(const double *h_in, int32_t H, int32_t W, double *h_out,
                    const dfg_params *prm, int32_t threads, void *stream);

/* Test hook (CPU only): the float64 <-> uint8 conversions of
 * dfg_filter_host_f64 (csrc/dfg_hostconv.cu).  Converts src[0..n) with the
 * dispatched (AVX2) form into dst_fast and with the scalar form into dst_ref,
 * and dst_ref back to float64 into `back`.  Returns bit 0 / bit 1: the
 * dispatched / scalar form found a value that is not an integer in 0..255. */
DFG_API int dfg_hostconv_selftest(const double *src, int64_t n, uint8_t *dst_fast, uint8_t *dst_ref,
                    double *back);

/* A stream of n independent (H, W, 3) frames from HOST memory (one buffer
 * per frame, pinned for overlap), synchronised before return: the
 * reference's per-frame apply_filter loop (bench.py:96-109, cli filter over
 * several files) as one call.  Frames go round-robin to four cached device
 * slots, each with its own stream: frame f's H2D overlaps the kernels and
 * D2H copies of the frames before it.  Same outputs as n dfg_filter_host calls. */
DFG_API int dfg_filter_host_frames(const uint8_t *const *h_in, uint8_t *const *h_out,
                    int32_t n_frames, int32_t H, int32_t W,
                    const dfg_params *prm, void *stream);

/* Schedule / diagnostic options (process-wide; for tests and measurement
 * scripts -- the library reads no environment variables).  Defaults are the
 * production settings. */
#define DFG_OPT_S3_SCHEDULE 1   /* 3x3 schedule: 0 auto, 1 warp row sweep, 2 CTA tiles */
#define DFG_OPT_NO_FIXUP 2      /* 1: skip the float64 re-decision (timing only; results may differ) */
#define DFG_OPT_HOST_BANDS 3    /* dfg_filter_host row bands: 0 auto */
#define DFG_OPT_HOST_GRAPH 4    /* dfg_filter_host: replay pinned pipelines as CUDA graphs (default 1) */
#define DFG_OPT_HOST_W3_RPC 5   /* rows per chunk of the host pipeline's 3x3 band kernels (default 8) */
#define DFG_OPT_FRAME_SLOTS 6   /* dfg_filter_host_frames device slots, 1..8 (default 4) */
#define DFG_OPT_W3_WPS 7        /* 3x3 row sweep: resident warps per SM its chunking targets (0 auto) */
#define DFG_OPT_W3_RPC 8        /* 3x3 row sweep: rows per chunk (0 auto) */
#define DFG_OPT_W3_SMALL_WPS 9  /* 3x3 row sweep: warps per SM for single-wave frames (default 12) */
#define DFG_OPT_CR_MARGIN 10    /* relative margin below which the correctly rounded arccos pass runs */
#define DFG_OPT_PERSIST 12      /* CTA kernels as one wave of persistent CTAs (default 1; 0: one tile per CTA) */
#define DFG_OPT_TMA 11          /* CTA-kernel tiles by bulk tensor copies: bit 0 input, bit 1 output (default 3) */
DFG_API int dfg_set_option(int32_t key, double value);
DFG_API double dfg_get_option(int32_t key);

/* Pixels re-decided in float64 by the calls on this workspace since the last
 * dfg_reset_counts (synchronous read of the workspace counter; the filter
 * calls only add to it, so they need no reset launch of their own). */
DFG_API int dfg_fixup_count(const void *d_workspace, void *stream, int64_t *count);
DFG_API int dfg_reset_counts(void *d_workspace, void *stream);

/* Diagnostics: the FP32 selection value of every window candidate
 * (n floats per pixel, window order) as the fast kernel computes them, for
 * error-budget validation against the float64 oracle.  d_vals: H*W*n floats. */
DFG_API int dfg_debug_values(const uint8_t *d_in, int32_t H, int32_t W, int64_t in_pitch,
                     float *d_vals, const dfg_params *prm, void *stream);

/* Host-side double-double acos used by the float64 re-decision kernel, for
 * CPU verification against libm: starts from libm acos(z) moved by
 * perturb_ulps and refines. */
DFG_API double dfg_cr_acos_host(double z, int32_t perturb_ulps);

/* Correlated impulsive noise (paper Eq. 8) -- replaces corrupt_image
 * (reference noise.py:85-116).  The generator is numpy's PCG64 as seeded by
 * np.random.PCG64(seed): the caller passes its initial 128-bit state and
 * increment (bit_generator.state), and the device draws the same five
 * doubles per pixel in row-major order, so the output equals the
 * reference's bit for bit.  impulse: 0 = saltpepper, 1 = uniform. */
typedef struct dfg_noise_params {
    double phi, phi1, phi2, phi3;
    int32_t impulse;
    int32_t reserved;
    uint64_t state_hi, state_lo, inc_hi, inc_lo;
} dfg_noise_params;

DFG_API int dfg_corrupt_image(const uint8_t *d_in, int32_t H, int32_t W, int64_t in_pitch,
                      uint8_t *d_out, int64_t out_pitch, const dfg_noise_params *np,
                      void *stream);

/* Effectiveness criteria of reference metrics.py:64-109 (compare()):
 * out3 = {MAE, PSNR [dB] (inf when identical), NCD x 1000} of d_test
 * against d_ref, float64 sums on the device.  d_scratch: >= 32 bytes of
 * device memory.  Synchronises `stream` before returning. */
DFG_API int dfg_image_metrics(const uint8_t *d_ref, const uint8_t *d_test, int32_t H, int32_t W,
                      int64_t ref_pitch, int64_t test_pitch, double *out3, void *d_scratch,
                      void *stream);

/* Angle-vs-chromaticity calibration sampling (reference calibration.py:83-125):
 * `pairs` random RGB pairs drawn exactly as sample_angle_chromaticity_pairs
 * draws them from np.random.PCG64(seed) (state/inc as for dfg_noise_params),
 * B = chromaticity L_p distance, A = exact angle, float64.
 * dfg_calib_reduce: mode 0 -> out3 = {sum B, sum A, 0}; mode 1 -> central
 * second moments {sum (B-x0)^2, sum (A-x1)^2, sum (B-x0)(A-x1)}; mode 2 ->
 * residuals about A = x0*B + x1: {sum r^2, sum |r|, 0}.  Deterministic
 * (fixed-order reduction); synchronises `stream`.  d_scratch: device memory
 * of dfg_calib_scratch_bytes().  dfg_calib_samples writes the samples. */
typedef struct dfg_calib_params {
    int64_t pairs;
    double p;
    uint64_t state_hi, state_lo, inc_hi, inc_lo;
} dfg_calib_params;

DFG_API size_t dfg_calib_scratch_bytes(void);
DFG_API int dfg_calib_reduce(const dfg_calib_params *cp, int32_t mode, double x0, double x1, double *out3,
                     void *d_scratch, size_t scratch_bytes, void *stream);
DFG_API int dfg_calib_samples(const dfg_calib_params *cp, double *d_b, double *d_a, void *stream);
/* The same three reductions (modes 0-2) over n stored device samples
 * (d_b, d_a) -- reference fit_line, calibration.py:47-80. */
DFG_API int dfg_moments_reduce(const double *d_b, const double *d_a, int64_t n, int32_t mode, double x0, double x1,
                     double *out3, void *d_scratch, size_t scratch_bytes, void *stream);

#ifdef __cplusplus
}
#endif

#endif /* DIRFILT_GPU_H */
