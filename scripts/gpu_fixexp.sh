for m in 1e-12 0; do
DFG_CR_MARGIN=$m python bench.py --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1 && DFG_CR_MARGIN=$m ncu --metrics gpu__time_duration.sum --clock-control none -c 30 --csv --log-file gpurun_out/launches_fix_$m.csv python bench.py --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1; echo $m=$?
done
python - <<'PY'
import ctypes, torch, sys
sys.path.insert(0,'.')
from paper_1009_0958_b200 import filter_device, parse_filter_spec, synth, _lib
from paper_1009_0958_b200 import filters as F
img = synth.config_input("c2"); x = torch.from_numpy(img).cuda()
for spec in ("ddf:exact","bvdf:exact","acwddf:exact:window=5"):
    filter_device(x, parse_filter_spec(spec)); torch.cuda.synchronize()
    ws = F.workspace(1); c = torch.empty(2, dtype=torch.int32); c.copy_(ws[:8].view(torch.int32))
    print(spec, "flagged", int(c[0]), "pass2", int(c[1]))
PY
