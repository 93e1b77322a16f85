# one GPU session: the GPU test suite, then the default bench line
nvidia-smi --query-gpu=name,clocks.max.sm,memory.total --format=csv,noheader > gpurun_out/gpu.txt; nproc >> gpurun_out/gpu.txt
python -m pytest tests -q -m gpu -rf --durations=15 > gpurun_out/gputest.log 2>&1; echo "pytest=$?" >> gpurun_out/gputest.log
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo "bench=$?" >> gpurun_out/bench.err
