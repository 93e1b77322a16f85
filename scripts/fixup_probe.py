"""Float64 re-decision statistics of one filter call per config: pixels
re-decided, of those needing pass 2 (correctly rounded acos), and SM cycles
spent in the re-decision (DFG_DIAG_CYCLES=1, w3 kernel only)."""
import os, sys
os.environ["DFG_DIAG_CYCLES"] = "1"
sys.path.insert(0, ".")
import torch
from paper_1009_0958_b200 import synth, filters as F, _lib
from paper_1009_0958_b200.spec import parse_filter_spec

for config in sys.argv[1:] or ["c1", "c2", "c5b"]:
    cfg = synth.CONFIGS[config]
    spec = parse_filter_spec(cfg["spec"])
    x = torch.from_numpy(synth.config_input(config)).cuda()
    ws = torch.zeros(_lib.lib().dfg_workspace_bytes(x.numel() // 3), dtype=torch.uint8, device="cuda")
    for rep in range(2):
        ws[:64].zero_()
        if x.dim() == 4:
            F.filter_batch_device(x, spec, ws=ws)
        else:
            F.filter_device(x, spec, ws=ws)
        torch.cuda.synchronize()
    c32 = ws[:16].view(torch.int32).cpu().tolist()
    cyc = int(ws[16:24].view(torch.int64).item())
    n = max(c32[0], 1)
    print(f"{config}: re-decided px {c32[0]}, pass-2 {c32[1]}, cycles {cyc} ({cyc / n:.0f} per px)", flush=True)
