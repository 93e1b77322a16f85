"""Development probe: where the host-path (e2e) time goes."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_1009_0958_b200 import filter_host, filter_device, parse_filter_spec, synth

img = synth.config_input("c2")
spec = parse_filter_spec("ddf:exact")
hin = torch.from_numpy(img).pin_memory(); hout = torch.empty_like(hin).pin_memory()
d = torch.empty_like(hin, device="cuda")
for _ in range(3):
    d.copy_(hin, non_blocking=True); hout.copy_(d, non_blocking=True)
torch.cuda.synchronize()
def timeit(f, n=50):
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(n): f()
    torch.cuda.synchronize(); return (time.perf_counter() - t) / n * 1e6
print("H2D 3MB us", timeit(lambda: d.copy_(hin, non_blocking=True)))
print("D2H 3MB us", timeit(lambda: hout.copy_(d, non_blocking=True)))
print("kernel us", timeit(lambda: filter_device(d, spec)))
a, b = hin.numpy(), hout.numpy()
for _ in range(3): filter_host(a, spec, out=b)
print("filter_host us", timeit(lambda: filter_host(a, spec, out=b)))
big = torch.empty(256 << 20, dtype=torch.uint8).pin_memory(); dbig = torch.empty_like(big, device="cuda")
print("H2D 256MB GB/s", (256 << 20) / timeit(lambda: dbig.copy_(big, non_blocking=True), 5) / 1e3)
print("D2H 256MB GB/s", (256 << 20) / timeit(lambda: big.copy_(dbig, non_blocking=True), 5) / 1e3)
