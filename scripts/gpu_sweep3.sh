# 3x3 minimum rows per chunk sweep (DFG_W3_MINRPC) on C1 / C2 / C5b, twice
for rep in 1 2; do
for c in c1 c2; do
  for v in "DFG_W3_MINRPC=0" "DFG_W3_MINRPC=4" "DFG_W3_MINRPC=5" "DFG_W3_MINRPC=6" "DFG_W3_MINRPC=7"; do
    echo -n "$c $v: "; env $v python bench.py --config $c --steps 50 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])"
  done
done
done
