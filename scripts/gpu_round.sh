# parity tests + bench lines for every config + launch list of the default bench
set -x
python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_tests.log
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
for c in c1 c3 c4_bvdf_minimax c4_bvdf_rgb c4_ddf_minimax c4_ddf_rgb c5b c5a; do
  python bench.py --config $c --steps 10 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c=$?
done
python bench.py --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none -c 40 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu_c2.log 2>&1; echo ncu=$?
