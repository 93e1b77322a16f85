python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/gpu_tests.log 2>&1; echo tests=$?; tail -3 gpurun_out/gpu_tests.log
for c in c2 c1 c5b; do
  python bench.py --config $c --no-cpu --steps 20 > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; echo $c=$?
  DFG_S3_CTA=1 python bench.py --config $c --no-cpu --steps 20 > gpurun_out/benchcta_$c.json 2>/dev/null
done
python bench.py --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,launch__registers_per_thread --clock-control none -c 20 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu_c2.log 2>&1; echo ncu=$?
