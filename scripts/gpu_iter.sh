# iteration: selected parity tests, benches of CONFIGS, optional ncu source capture of PROF config
python -m pytest ${TESTS:-tests/test_gpu_parity.py tests/test_gpu_error_budget.py} -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_iter_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_iter_tests.log
python scripts/timing_probe.py ${PROBE:-c2} > gpurun_out/timing_probe.log 2>&1; cat gpurun_out/timing_probe.log
for c in ${CONFIGS:-c2}; do
  python bench.py --config $c --no-cpu --steps 30 > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; echo $c=$?
  python -c "import json;d=json.loads(open('gpurun_out/bench_$c.json').read().splitlines()[-1]);print('$c', d['value'], d['ms_per_step'], d['roofline']['frac'], d['redecided_px_per_step'])"
done
for c in ${PROF}; do
python bench.py --config $c --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dfg_ -s 3 -c 1 -o gpurun_out/prof_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_$c.log 2>&1; echo prof_$c=$?
done
