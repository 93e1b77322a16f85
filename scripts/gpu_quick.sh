# quick: c2 bench + launch list
python bench.py --no-cpu > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo bench=$?
python bench.py --config c1 --no-cpu > gpurun_out/bench_c1.json 2> gpurun_out/bench_c1.err
python bench.py --config c5b --no-cpu --steps 10 > gpurun_out/bench_c5b.json 2> gpurun_out/bench_c5b.err
python bench.py --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,launch__registers_per_thread --clock-control none -c 20 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu_c2.log 2>&1; echo ncu=$?
