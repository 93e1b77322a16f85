# profiles only: launch list, full captures, on-box summary (see gpu_final.sh)
python bench.py --steps 5 --warmup 3 --no-cpu > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,launch__registers_per_thread,launch__grid_size,launch__block_size,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c2.csv python bench.py --steps 5 --warmup 3 --no-cpu > gpurun_out/ncu_ll.log 2>&1; echo ll=$?
for c in c1 c2 c3 c4_bvdf_minimax c4_bvdf_rgb c4_ddf_minimax c4_ddf_rgb c5a c5b; do
python bench.py --config $c --steps 1 --warmup 3 --no-cpu > /dev/null 2>&1 && \
ncu --set full --clock-control none --import-source on -k "regex:dfg_w3_kernel|dfg_fast_kernel" -s 3 -c 1 -f -o gpurun_out/prof_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu > gpurun_out/ncu_$c.log 2>&1; echo prof_$c=$?
done
# summaries on the box (ncu reports are ~20 MB each; gpurun returns <= 64 MiB)
python scripts/make_profile_summary.py r01 gpurun_out/launches_c2.csv gpurun_out/prof_*.ncu-rep > gpurun_out/summary.log 2>&1; echo summary=$?
cp profiles/r01_summary.md profiles/r01_traffic.json gpurun_out/
for c in c2 c3 c5a c5b; do ncu -i gpurun_out/prof_$c.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$c.csv 2>/dev/null; gzip -f gpurun_out/src_$c.csv; done
mkdir -p /tmp/reps && mv gpurun_out/prof_*.ncu-rep /tmp/reps/ && mv /tmp/reps/prof_c2.ncu-rep gpurun_out/
