for m in 8 9 10; do for c in c2 c5b c1; do
DFG_W3_MINB=$m python bench.py --config $c --no-cpu --steps 30 > gpurun_out/bm_${m}_$c.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/bm_${m}_$c.json').read().splitlines()[-1]);print('minb $m $c', d['value'], d['ms_per_step'], d['roofline']['frac'])"
done; done
