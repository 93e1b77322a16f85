"""B200-native (sm_100a) directional vector filters -- BVDF, DDF, ACWDDF (+ VMF)
in the exact, minimax-polynomial and chromaticity forms of arXiv 1009.0958.

Drop-in for the reference package's filter path: ``apply_filter`` and the
spec/image types keep the reference's names, fields and errors
(reference ``pkg/src/dirfilt/__init__.py:6-47``, filter subset).  The work runs
in hand-written CUDA kernels in ``libdfg.so`` behind a C ABI
(``include/dirfilt_gpu.h``); there is no CPU fallback.
"""

from .filters import (
    apply_filter,
    filter_batch_device,
    filter_device,
    filter_host,
    filter_host_frames,
    filter_rows_device,
    fixup_counts,
    last_fixup_count,
)
from .calibration import LinearFit, fit_angular_chromaticity, fit_line, sample_angle_chromaticity_pairs
from .metrics import MetricsReport, compare, mae, metrics_device, ncd, psnr
from .noise import NoiseParams, corrupt_device, corrupt_image
from .image import REFLECT, REPLICATE, BorderPolicy, ColorVector, RasterImage, to_uint8
from .spec import (
    ACOS_COEFFICIENTS,
    ASIN_COEFFICIENTS,
    CALIBRATION_INTERCEPT,
    CALIBRATION_SLOPE,
    FAMILIES,
    CW_FAMILIES,
    AcwddfParams,
    CenterWeightedSpec,
    DirectionalStrategy,
    FastAcosTable,
    FilterSpec,
    MinimaxPoly,
    center_weight,
    parse_filter_spec,
)

__version__ = "0.1.0"

__all__ = [
    "ACOS_COEFFICIENTS", "ASIN_COEFFICIENTS", "AcwddfParams", "BorderPolicy",
    "CALIBRATION_INTERCEPT", "CALIBRATION_SLOPE", "ColorVector", "DirectionalStrategy",
    "FAMILIES", "FastAcosTable", "FilterSpec", "MinimaxPoly", "REFLECT", "REPLICATE",
    "RasterImage", "apply_filter", "center_weight", "filter_batch_device", "filter_device",
    "filter_host", "filter_host_frames", "filter_rows_device", "fixup_counts", "last_fixup_count", "parse_filter_spec", "to_uint8",
    "MetricsReport", "compare", "mae", "psnr", "ncd", "metrics_device",
    "NoiseParams", "corrupt_device", "corrupt_image",
    "LinearFit", "fit_angular_chromaticity", "fit_line", "sample_angle_chromaticity_pairs",
    "CW_FAMILIES", "CenterWeightedSpec",
]
