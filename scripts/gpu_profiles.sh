# round profiles: launch list of the default bench command (PART=ll) or full captures of CONFIGS
if [ "${PART}" = "ll" ]; then
python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/plain.log 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,launch__registers_per_thread,launch__grid_size,launch__block_size,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu_ll.log 2>&1; echo ll=$?
fi
for c in ${CONFIGS}; do
python bench.py --config $c --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dfg_ -s 3 -c 1 -o gpurun_out/prof_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_$c.log 2>&1; echo $c=$?
done
