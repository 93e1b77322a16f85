# ncu --set full capture of the filter kernel of each given config (the 4th
# launch: after bench.py's 3 warm-up steps); raw metrics + SASS source page
# come back as CSV (the .ncu-rep stays on the box unless KEEP_REP=1)
# usage: bash scripts/gpu_prof.sh c5a c3 ...
for c in "$@"; do
  ncu --set full --clock-control none --import-source on -k "regex:dfg_w3_kernel|dfg_fast_kernel" -s 3 -c 1 -f \
      -o /tmp/prof_$c python bench.py --config $c --steps 1 --warmup 3 --no-cpu --no-parity --no-table \
      > gpurun_out/ncu_$c.log 2>&1; echo "ncu $c: $?" >> gpurun_out/ncu_status.log
  ncu -i /tmp/prof_$c.ncu-rep --page raw --csv > gpurun_out/raw_$c.csv 2>/dev/null
  ncu -i /tmp/prof_$c.ncu-rep --page source --csv --print-source sass > gpurun_out/src_$c.csv 2>/dev/null
  gzip -f gpurun_out/src_$c.csv
  if [ -n "$KEEP_REP" ]; then cp /tmp/prof_$c.ncu-rep gpurun_out/; fi
done
