# share of the float64 re-decision: same benches with DFG_DIAG_NO_FIXUP=1
for c in c2 c5b c1 c3 c5a c4_ddf_minimax; do
for nf in 0 1; do
DFG_DIAG_NO_FIXUP=$nf python bench.py --config $c --no-cpu --steps 20 > gpurun_out/bnf_${nf}_$c.json 2>/dev/null
python -c "import json;d=json.loads(open('gpurun_out/bnf_${nf}_$c.json').read().splitlines()[-1]);print('nofix $nf $c', d['value'], d['ms_per_step'], d['roofline']['frac'], d['redecided_px_per_step'])"
done; done
