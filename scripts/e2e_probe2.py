"""Development probe: host-path pipeline timing vs band count."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_1009_0958_b200 import filter_host, parse_filter_spec, synth
img = synth.config_input("c2"); spec = parse_filter_spec("ddf:exact")
hin = torch.from_numpy(img).pin_memory(); hout = torch.empty_like(hin).pin_memory()
a, b = hin.numpy(), hout.numpy()
import numpy as np
pa, pb = img.copy(), np.empty_like(img)
for name, (x, y) in {"pinned": (a, b), "pageable": (pa, pb)}.items():
    for _ in range(3): filter_host(x, spec, out=y)
    t = time.perf_counter()
    for _ in range(50): filter_host(x, spec, out=y)
    print(name, f"{1e6 * (time.perf_counter() - t) / 50:.1f} us/call")
