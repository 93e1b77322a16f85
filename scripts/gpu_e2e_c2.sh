# e2e frame-stream A/B over the slot count (DFG_FRAME_SLOTS), interleaved
for rep in 1 2; do for ns in 3 4 5 2; do
  echo -n "slots=$ns: "; DFG_FRAME_SLOTS=$ns python bench.py --config ${C:-c2} --steps 10 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['e2e']['value'], d['e2e']['ms_per_step'])"
done; done
