"""Development probe: which bench.py stage slows the host path afterwards."""
import sys, time
sys.path.insert(0, ".")
import torch
import bench
from paper_1009_0958_b200 import filter_host, filter_device, parse_filter_spec, synth

img = synth.config_input("c2"); spec = parse_filter_spec("ddf:exact")
hin = torch.from_numpy(img).pin_memory(); hout = torch.empty_like(hin).pin_memory()
a, b = hin.numpy(), hout.numpy()
def e2e(tag, n=50):
    for _ in range(3): filter_host(a, spec, out=b)
    t = time.perf_counter()
    for _ in range(n): filter_host(a, spec, out=b)
    print(f"{tag:30s} {1e6 * (time.perf_counter() - t) / n:.1f} us/call", flush=True)
e2e("fresh")
torch.cuda.set_device(0)
e2e("after set_device")
x = torch.from_numpy(img).cuda(); out = torch.empty_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
e2e("after allocs")
for k in range(30):
    flush.fill_(k); filter_device(x, spec, out=out)
torch.cuda.synchronize()
e2e("after device loop")
with bench.ClockSampler(0) as clk:
    for k in range(30):
        flush.fill_(k); filter_device(x, spec, out=out)
    torch.cuda.synchronize()
e2e("after clocksampler loop")
time.sleep(1.0)
e2e("1 s later")
with bench.ClockSampler(0) as clk:
    e2e("during clocksampler")
