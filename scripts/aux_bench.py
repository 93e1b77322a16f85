"""Throughput of the 8(f) device kernels: on-device noise (dfg_corrupt_image)
and the MAE/PSNR/NCD reduction (dfg_image_metrics), at the C5a frame size.
Prints one JSON line per kernel (CUDA events, L2-cold inputs > 126 MB L2)."""
import json
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1009_0958_b200 import metrics, noise, synth  # noqa: E402

H = W = 8192
img = torch.from_numpy(synth.clean_image(H, W, 5)).cuda()
out = torch.empty_like(img)
p = noise.NoiseParams(phi=0.2, phi1=0.0, phi2=0.0, phi3=0.0, impulse="uniform", seed=5 + 10**6)
for _ in range(3):
    noise.corrupt_device(img, p, out=out)
torch.cuda.synchronize()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
n = 20
ev[0].record()
for _ in range(n):
    noise.corrupt_device(img, p, out=out)
ev[1].record()
torch.cuda.synchronize()
ms = ev[0].elapsed_time(ev[1]) / n
px = H * W
print(json.dumps({"kernel": "dfg_corrupt_image", "shape": [H, W], "ms": round(ms, 4),
                  "Mpx_s": round(px / ms / 1e3, 1), "GB_s": round(6 * px / ms / 1e6, 1),
                  "draws_per_s": round(5 * px / ms / 1e3, 1)}))
for _ in range(3):
    metrics.metrics_device(img, out)
torch.cuda.synchronize()
import time  # noqa: E402
t = time.perf_counter()
for _ in range(n):
    metrics.metrics_device(img, out)
ms = (time.perf_counter() - t) * 1e3 / n  # synchronous call (result read back)
print(json.dumps({"kernel": "dfg_image_metrics", "shape": [H, W], "ms": round(ms, 4),
                  "Mpx_s": round(px / ms / 1e3, 1), "GB_s": round(6 * px / ms / 1e6, 1)}))

# calibration fit at the paper's 10^8 pairs (three streamed passes)
from paper_1009_0958_b200 import calibration  # noqa: E402
import oracle  # noqa: E402

calibration.fit_angular_chromaticity(10**6, 0)
torch.cuda.synchronize()
t = time.perf_counter()
f = calibration.fit_angular_chromaticity(10**8, 0)
ms = (time.perf_counter() - t) * 1e3
print(json.dumps({"kernel": "dfg_calib (fit_angular_chromaticity)", "pairs": 10**8, "ms": round(ms, 2),
                  "Mpairs_s": round(1e8 / ms / 1e3, 1), "slope": f.slope, "intercept": f.intercept}))
t = time.perf_counter()
want = oracle.calib_fit(*oracle.calib_samples(10**7, 0))
cpu_ms = (time.perf_counter() - t) * 1e3
print(json.dumps({"cpu numpy reference restatement": "calib_samples + calib_fit", "pairs": 10**7,
                  "ms": round(cpu_ms, 1), "Mpairs_s": round(1e7 / cpu_ms / 1e3, 2)}))
