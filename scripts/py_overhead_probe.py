"""Development probe: Python-side overhead of filter_device / filter_host."""
import cProfile, pstats, sys, time
sys.path.insert(0, ".")
import torch
from paper_1009_0958_b200 import filter_device, filter_host, parse_filter_spec, synth
from paper_1009_0958_b200 import filters as F

img = synth.config_input("c2"); spec = parse_filter_spec("ddf:exact")
d = torch.from_numpy(img).cuda(); out = torch.empty_like(d)
for _ in range(5): filter_device(d, spec, out=out)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(200): filter_device(d, spec, out=out)
t1 = time.perf_counter(); torch.cuda.synchronize(); t2 = time.perf_counter()
print(f"filter_device: {1e6*(t1-t)/200:.1f} us/call enqueue, {1e6*(t2-t)/200:.1f} us/call incl. sync")
pr = cProfile.Profile(); pr.enable()
for _ in range(200): filter_device(d, spec, out=out)
pr.disable(); torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("cumulative").print_stats(12)
