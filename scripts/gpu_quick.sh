# quick iteration: parity subset + device-only bench lines of the given configs
# usage: bash scripts/gpu_quick.sh "<pytest -k expr>" c5a c3 ...
export DFG_ALLOW_DEV_LIB=1  # quick iteration runs may carry a scripts/dev_unit.py build
k=$1; shift
python -m pytest tests -q -m gpu -x -k "$k" > gpurun_out/quick_test.log 2>&1; echo "pytest=$?" >> gpurun_out/quick_test.log
for c in "$@"; do
  python bench.py --config $c --no-table --no-cpu --no-parity --steps 20 > gpurun_out/quick_$c.json 2> gpurun_out/quick_$c.err
done
