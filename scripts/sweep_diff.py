import sys, time
import numpy as np, torch
sys.path.insert(0, ".")
import oracle
from paper_1009_0958_b200 import filter_device, parse_filter_spec, synth, _lib, last_fixup_count
specs = sys.argv[1:] or ["ddf:exact:window=7"]
for spec in specs:
    sp = parse_filter_spec(spec)
    for shape in ((40, 58), (97, 61), (150, 173), (33, 200)):
        for border in ("replicate", "reflect"):
            img = synth.noisy_image(*shape, 7, ("correlated", 0.2))
            img[5:9, 7:12] = 0
            want = oracle.filter_image(img, sp, border)
            last_fixup_count()
            with _lib.option("sweep", 1):
                got = filter_device(torch.from_numpy(img).cuda(), sp, border).cpu().numpy()
            bad = (got != want).any(-1)
            print(spec, shape, border, "mismatches", int(bad.sum()), "redecided", last_fixup_count(),
                  "rows", np.unique(np.nonzero(bad)[0])[:12], "cols", np.unique(np.nonzero(bad)[1])[:12])
    img = synth.noisy_image(2048, 2048, 5, ("correlated", 0.2))
    x = torch.from_numpy(img).cuda()
    for sw in (0, 1):
        with _lib.option("sweep", sw):
            o = filter_device(x, sp)
            torch.cuda.synchronize()
            t = time.perf_counter()
            for _ in range(5):
                o = filter_device(x, sp)
            torch.cuda.synchronize()
            print(spec, "2048^2 sweep" if sw else "2048^2 tile ", (time.perf_counter() - t) / 5 * 1e3, "ms")
        if sw == 0:
            ref = o.clone()
    print("sweep == tile kernel:", bool((o == ref).all()), int((o != ref).any(-1).sum()))
