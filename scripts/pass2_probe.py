"""Dev probe: how often the correctly-rounded second pass triggers, per kernel / margin."""
import os, sys, subprocess
sys.path.insert(0, ".")
code = r'''
import sys; sys.path.insert(0, ".")
import numpy as np, torch, oracle
from paper_1009_0958_b200 import filter_device, fixup_counts, parse_filter_spec, synth
img = synth.config_input("c5b", frames=1)[0]
s = parse_filter_spec("acwddf:exact")
x = torch.from_numpy(img).cuda()
fixup_counts(reset=True); got = filter_device(x, s).cpu().numpy(); torch.cuda.synchronize()
c = fixup_counts(reset=True)
want = oracle.filter_image(img, s)
print(sys.argv[1], c, "mismatches", int((got != want).any(-1).sum()))
'''
for env in ({"DFG_S3_KERNEL": "w3"}, {"DFG_S3_KERNEL": "cta"}, {"DFG_S3_KERNEL": "w3", "DFG_CR_MARGIN": "0"},
            {"DFG_S3_KERNEL": "w3", "DFG_CR_MARGIN": "1e-300"}):
    e = dict(os.environ, **env)
    subprocess.run([sys.executable, "-c", code, str(env)], env=e)
