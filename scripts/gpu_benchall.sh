# every config's bench line (default c2 with the CPU baseline, the rest --no-cpu)
python bench.py > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo c2=$?
for c in c1 c3 c4_bvdf_minimax c4_bvdf_rgb c4_ddf_minimax c4_ddf_rgb c5b c5a; do
  python bench.py --config $c --steps 20 --no-cpu > gpurun_out/bench_$c.json 2> gpurun_out/bench_$c.err; echo $c=$?
done
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref_c2.json 2> gpurun_out/bench_ref_c2.err; echo ref=$?
