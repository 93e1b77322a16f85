# full ncu capture of one kernel: CONFIG, KREGEX
c=${CONFIG:-c2}; k=${KREGEX:-dfg_}
python bench.py --config $c --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:$k -s 3 -c 1 -o gpurun_out/prof_${TAG:-x}_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_$c.log 2>&1; echo prof=$?
