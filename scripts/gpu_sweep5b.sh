# C5b chunk length sweep (ran with a temporary DFG_W3_MAXRPC build lifting the 64-row cap)
for rep in 1 2; do
  for v in "X=0" "DFG_W3_MAXRPC=2000 DFG_W3_RPC=90" "DFG_W3_MAXRPC=2000 DFG_W3_RPC=120" "DFG_W3_MAXRPC=2000 DFG_W3_RPC=180" "DFG_W3_MAXRPC=2000 DFG_W3_RPC=270"; do
    echo -n "c5b $v: "; env $v python bench.py --config c5b --steps 10 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])"
  done
done
