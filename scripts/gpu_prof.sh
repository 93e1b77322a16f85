set -x
for c in ${CONFIGS:-c2 c5a}; do
python bench.py --config $c --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:dfg_fast_kernel -s 3 -c 1 -o gpurun_out/prof_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_$c.log 2>&1; echo $c=$?
done
