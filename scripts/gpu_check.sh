python -m pytest tests -m gpu -q -x -p no:cacheprovider 2>&1 | tail -3
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
for c in c2 c1 c5b c3 c5a c4_bvdf_minimax c4_bvdf_rgb c4_ddf_minimax c4_ddf_rgb; do python bench.py --config $c --no-cpu --steps 30 > gpurun_out/bench_$c.json 2>gpurun_out/bench_$c.err; echo $c=$?; done
python scripts/summarize.py
