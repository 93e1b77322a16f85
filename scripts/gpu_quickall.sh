# full GPU suite + one bench line per config (device value only)
python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/tq.log 2>&1; echo tests=$?; tail -2 gpurun_out/tq.log
for c in ${CONFIGS:-c1 c2 c3 c4_bvdf_minimax c4_bvdf_rgb c4_ddf_minimax c4_ddf_rgb c5b c5a}; do
  echo -n "$c: "; python bench.py --config $c --steps 20 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['frac'], d['redecided_px_per_step'], (d['e2e'] or {}).get('value'))"
done
