"""Dev probe: fixup / pass-2 counts per C5b frame, single vs batch."""
import sys
sys.path.insert(0, ".")
import numpy as np, torch, oracle  # noqa: E401
from paper_1009_0958_b200 import filter_batch_device, filter_device, fixup_counts, parse_filter_spec, synth
frames = synth.config_input("c5b", frames=8)
s = parse_filter_spec("acwddf:exact")
for i in range(8):
    x = torch.from_numpy(frames[i]).cuda()
    fixup_counts(reset=True); filter_device(x, s); torch.cuda.synchronize()
    print("frame", i, fixup_counts(reset=True))
xb = torch.from_numpy(frames).cuda()
fixup_counts(reset=True); filter_batch_device(xb, s); torch.cuda.synchronize()
print("batch", fixup_counts(reset=True))
r = oracle.filter_image(frames[3], s, diag=True)
g = r["gap"]; print("oracle frame 3 gap<1e-12:", int((g < 1e-12).sum()), "gap==0:", int((g == 0).sum()),
                    "|tm|<1e-12:", int((np.abs(r["tmargin"]) < 1e-12).sum()))
