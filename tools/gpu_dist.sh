python -m pytest tests -m gpu -q -p no:cacheprovider -k "packed or pipelined or edge or row_blocks or host_streams" > gpurun_out/pytest_dist.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_dist.log
python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 1 > gpurun_out/bench_n1.log 2>&1; echo "bench rc=$?"; tail -c 1500 gpurun_out/bench_n1.log
