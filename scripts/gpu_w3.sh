# 3x3 iteration: parity + budget tests, benches, one full ncu capture of the w3 kernel
python -m pytest tests/test_gpu_parity.py tests/test_gpu_error_budget.py -m gpu -q -x -p no:cacheprovider -s > gpurun_out/gpu_parity.log 2>&1; echo parity=$?; grep -E "passed|failed|worst" gpurun_out/gpu_parity.log | tail -14
for c in c2 c1 c5b c4_ddf_minimax; do
  python bench.py --config $c --no-cpu --steps 30 > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; echo $c=$?
done
for w in 18; do DFG_W3_WPS=$w python bench.py --config c2 --no-cpu --steps 30 > gpurun_out/benchwps${w}_c2.json 2>/dev/null; done
python scripts/summarize.py
for f in gpurun_out/benchwps*_c2.json; do echo $f; python -c "import json;d=json.loads(open('$f').read().splitlines()[-1]);print(d['value'],d['ms_per_step'])"; done
CONFIG=c2 KREGEX=w3 TAG=${TAG:-w3} bash scripts/gpu_prof1.sh
