"""Device time of one filter step three ways: events around the direct call
(as bench.py), events around a CUDA-graph replay of the same call, and the
host time of the Python call alone (diagnostic for the bench timing)."""
import sys, time
sys.path.insert(0, ".")
import torch
from paper_1009_0958_b200 import synth, filters as F, _lib
from paper_1009_0958_b200.spec import parse_filter_spec

for config in sys.argv[1:] or ["c1", "c2"]:
    cfg = synth.CONFIGS[config]
    spec = parse_filter_spec(cfg["spec"])
    x = torch.from_numpy(synth.config_input(config)).cuda()
    if x.dim() == 4:
        x = x[0].contiguous()
    out = torch.empty_like(x)
    ws = torch.zeros(_lib.lib().dfg_workspace_bytes(x.shape[0] * x.shape[1]), dtype=torch.uint8, device="cuda")
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    step = lambda: F.filter_device(x, spec, out=out, ws=ws)
    for _ in range(10):
        step()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(200):
        step()
    torch.cuda.synchronize()
    host_us = (time.perf_counter() - t0) / 200 * 1e6
    def ev(fn, n=50):
        s = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
        e = [torch.cuda.Event(enable_timing=True) for _ in range(n)]
        for k in range(n):
            flush.fill_(k & 0xff)
            s[k].record(); fn(); e[k].record()
        torch.cuda.synchronize()
        ts = sorted(a.elapsed_time(b) * 1e3 for a, b in zip(s, e))
        return ts[len(ts) // 2], sum(ts) / len(ts)
    direct = ev(step)
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        step()
        with torch.cuda.graph(g, stream=st):
            step()
    torch.cuda.synchronize()
    graph = ev(g.replay)
    # back-to-back replays without flush (L2 warm; launch overhead amortised)
    s0 = torch.cuda.Event(enable_timing=True); e0 = torch.cuda.Event(enable_timing=True)
    s0.record()
    for _ in range(100):
        g.replay()
    e0.record(); torch.cuda.synchronize()
    b2b = s0.elapsed_time(e0) * 1e3 / 100
    print(f"{config}: host call {host_us:.1f} us; events direct median/mean {direct[0]:.1f}/{direct[1]:.1f} us; "
          f"graph {graph[0]:.1f}/{graph[1]:.1f} us; back-to-back graph {b2b:.1f} us", flush=True)
