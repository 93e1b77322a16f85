# 3x3 small-frame warps per SM (DFG_W3_SMALL_WPS) on C1, interleaved repeats; C2 unaffected check
for rep in 1 2; do
  for v in "DFG_W3_SMALL_WPS=0" "DFG_W3_SMALL_WPS=8" "DFG_W3_SMALL_WPS=10" "DFG_W3_SMALL_WPS=12"; do
    echo -n "c1 $v: "; env $v python bench.py --config c1 --steps 40 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])"
  done
done
echo -n "c2: "; python bench.py --config c2 --steps 40 --no-cpu 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])"
python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "3x3 or golden or acceptance or config_size or extreme" > gpurun_out/tq.log 2>&1; echo tests=$?; tail -1 gpurun_out/tq.log
