# Round profiles (scripts/make_profile_summary.py TAG): the launch list of
# the default bench command (ncu --metrics gpu__time_duration.sum,...
# --clock-control none), then one ncu --set full capture per config of its
# filter kernel (the 4th launch: after bench.py's 3 warm-up steps), the
# summary + DRAM traffic table written on the box, SASS source pages of the
# main configs gzipped.  usage: bash scripts/gpu_profiles.sh r02
tag=${1:-r02}
python bench.py --steps 5 --warmup 3 --no-cpu --no-parity --no-table > /dev/null 2>&1 && \
ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,launch__registers_per_thread,launch__grid_size,launch__block_size,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none -c 400 --csv --log-file gpurun_out/launches_default.csv \
    python bench.py --steps 5 --warmup 3 --no-cpu --no-parity --no-table > gpurun_out/ncu_ll.log 2>&1; echo "ll=$?"
for c in c1 c2 c3 c4_bvdf_minimax c4_bvdf_rgb c4_ddf_minimax c4_ddf_rgb c5a c5b; do
  ncu --set full --clock-control none --import-source on -k "regex:dfg_w3_kernel|dfg_fast_kernel" -s 3 -c 1 -f \
      -o /tmp/prof_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu --no-parity --no-table \
      > gpurun_out/ncu_$c.log 2>&1; echo "prof_$c=$?"
done
python scripts/make_profile_summary.py $tag gpurun_out/launches_default.csv /tmp/prof_*.ncu-rep > gpurun_out/summary.log 2>&1; echo "summary=$?"
cp profiles/${tag}_summary.md profiles/${tag}_traffic.json gpurun_out/
for c in c2 c3 c5a c5b c4_ddf_minimax; do
  ncu -i /tmp/prof_$c.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$c.csv 2>/dev/null; gzip -f gpurun_out/src_$c.csv
  ncu -i /tmp/prof_$c.ncu-rep --page raw --csv > gpurun_out/raw_$c.csv 2>/dev/null
done
cp /tmp/prof_c5a.ncu-rep gpurun_out/ 2>/dev/null
