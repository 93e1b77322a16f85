import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
from paper_1009_0958_b200 import apply_filter, parse_filter_spec, synth, RasterImage
img = synth.noisy_image(8192, 8192, 5, ("correlated", 0.2))
ri = RasterImage(img.astype(np.float64))
s = parse_filter_spec("ddf:exact:window=7")
for i in range(3):
    t = time.perf_counter(); out = apply_filter(ri, s); print("call", (time.perf_counter() - t) * 1e3, "ms", file=sys.stderr)
