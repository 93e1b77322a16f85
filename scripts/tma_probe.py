"""Probe: one 5x5 filter on a 512x512 frame with the CTA kernel's bulk
tensor copies on / off (diagnostics for the TMA path)."""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle  # noqa: E402
from paper_1009_0958_b200 import _lib, filter_device, parse_filter_spec, synth  # noqa: E402

mode = int(sys.argv[1]) if len(sys.argv) > 1 else 1
img = synth.noisy_image(256, 512, 3, ("correlated", 0.2))
s = parse_filter_spec(sys.argv[2] if len(sys.argv) > 2 else "acwddf:exact:window=5")
with _lib.option("tma", mode):
    got = filter_device(torch.from_numpy(img).cuda(), s).cpu().numpy()
want = oracle.filter_image(img, s)
print("tma", mode, "mismatches", int((got != want).any(-1).sum()))
