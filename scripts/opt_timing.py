"""Device time of one config's filter under library options (diagnostics).
usage: python scripts/opt_timing.py c5a "tma=0" "tma=3" ...  (prints ms per call, median of 15)"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

from paper_1009_0958_b200 import _lib, filter_batch_device, filter_device, parse_filter_spec, synth  # noqa: E402

cfg = sys.argv[1]
c = synth.CONFIGS[cfg]
spec = parse_filter_spec(c["spec"])
x = torch.from_numpy(synth.config_input(cfg)).cuda()
out = torch.empty_like(x)
flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
fn = filter_batch_device if x.dim() == 4 else filter_device
for combo in sys.argv[2:] or [""]:
    olds = []
    for kv in filter(None, combo.split(",")):
        k, v = kv.split("=")
        olds.append((k, _lib.set_option(k, float(v))))
    for _ in range(3):
        fn(x, spec, out=out)
    ts = []
    for _ in range(15):
        flush.fill_(1)
        torch.cuda._sleep(50000)
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        fn(x, spec, out=out)
        b.record()
        torch.cuda.synchronize()
        ts.append(a.elapsed_time(b))
    ts.sort()
    print(f"{cfg} [{combo}] {ts[len(ts) // 2]:.4f} ms (min {ts[0]:.4f})", flush=True)
    for k, v in reversed(olds):
        _lib.set_option(k, v)
