# timing probe + full ncu captures with source/SASS attribution for CONFIGS
python scripts/timing_probe.py c1 c2 c5b > gpurun_out/timing_probe.log 2>&1; echo probe=$?
for c in ${CONFIGS}; do
python bench.py --config $c --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dfg_ -s 3 -c 1 -o gpurun_out/prof_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_$c.log 2>&1; echo $c=$?
done
