set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest1.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest1.log
python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/bench1.log 2>&1; echo "bench rc=$?"
tail -c 3000 gpurun_out/bench1.log
