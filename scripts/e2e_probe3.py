"""Development probe: filter_host from Python -- default vs side stream, call count."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_1009_0958_b200 import filter_host, parse_filter_spec, synth
img = synth.config_input("c2"); spec = parse_filter_spec("ddf:exact")
hin = torch.from_numpy(img).pin_memory(); hout = torch.empty_like(hin).pin_memory()
a, b = hin.numpy(), hout.numpy()
s = torch.cuda.Stream()
for name, st in (("default", None), ("side", s), ("default", None)):
    for n in (5, 30, 200):
        for _ in range(3): filter_host(a, spec, out=b, stream=st)
        t = time.perf_counter()
        for _ in range(n): filter_host(a, spec, out=b, stream=st)
        print(name, n, f"{1e6 * (time.perf_counter() - t) / n:.1f} us/call")
