"""Development probe: host-path (e2e) time per call vs the host CPUs / NUMA
node the pinned buffers live on.  Prints the GPU's PCIe-local CPU list and
times filter_host with the process bound to each NUMA node in turn."""
import os, sys, time
sys.path.insert(0, ".")
import numpy as np
import torch
from paper_1009_0958_b200 import filter_host, parse_filter_spec, synth

torch.cuda.set_device(0)
props = torch.cuda.get_device_properties(0)
bus = "%04x:%02x:%02x.0" % (getattr(props, "pci_domain_id", 0), props.pci_bus_id, props.pci_device_id)
base = "/sys/bus/pci/devices/" + bus
for f in ("numa_node", "local_cpulist", "current_link_speed", "current_link_width"):
    try:
        print(f, open(os.path.join(base, f)).read().strip())
    except OSError as e:
        print(f, "?", e)
nodes = sorted(int(d[4:]) for d in os.listdir("/sys/devices/system/node") if d.startswith("node") and d[4:].isdigit())
print("nodes", nodes, "cpus", os.cpu_count())


def cpus_of(node):
    s = open(f"/sys/devices/system/node/node{node}/cpulist").read().strip()
    out = set()
    for part in s.split(","):
        a, _, b = part.partition("-")
        out.update(range(int(a), int(b or a) + 1))
    return out


img = synth.config_input("c2")
spec = parse_filter_spec("ddf:exact")
for node in nodes + [None]:
    if node is not None:
        os.sched_setaffinity(0, cpus_of(node))
    else:
        os.sched_setaffinity(0, set(range(os.cpu_count())))
    hin = torch.from_numpy(img).pin_memory()
    hout = torch.empty_like(hin).pin_memory()
    a, b = hin.numpy(), hout.numpy()
    t = time.perf_counter()
    while time.perf_counter() - t < 0.5:
        filter_host(a, spec, out=b)
    for rep in range(3):
        ts = []
        for _ in range(100):
            t1 = time.perf_counter()
            filter_host(a, spec, out=b)
            ts.append((time.perf_counter() - t1) * 1e6)
        print(f"node {node}: min {min(ts):.1f} median {np.median(ts):.1f} mean {np.mean(ts):.1f} us/call", flush=True)
    del hin, hout
