import sys
import numpy as np, torch
sys.path.insert(0, ".")
import oracle
from paper_1009_0958_b200 import filter_device, parse_filter_spec, synth, _lib
img = synth.noisy_image(97, 61, 7, ("uncorrelated", 0.15))
for spec in ("ddf:exact",):
    sp = parse_filter_spec(spec)
    want = oracle.filter_image(img, sp)
    for rpc in (0, 97, 8):
        with _lib.option("s3_schedule", 1), _lib.option("w3_rpc", rpc):
            got = filter_device(torch.from_numpy(img).cuda(), sp).cpu().numpy()
        bad = (got != want).any(-1)
        print(spec, "rpc", rpc, int(bad.sum()), "per row:", bad.sum(1)[:40].tolist())
        print("   per col:", bad.sum(0).tolist())
