# launch-cover / re-decision cost experiment for the small 3x3 configs
for c in c1 c2; do
  for v in "" "BENCH_NO_COVER=1" "DFG_DIAG_NO_FIXUP=1"; do
    echo -n "$c $v: "; env $v python bench.py --config $c --steps 50 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])"
  done
done
