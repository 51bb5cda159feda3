#!/bin/bash
# quick check after an x2 / ik1 change: GPU tests, one bench line, ncu of x2 + ik1
python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; tail -3 gpurun_out/gpu_tests.log
python bench.py --no-cpu-baseline --e2e-steps 0 > gpurun_out/bench_q.jsonl 2> gpurun_out/bench_q.err; cat gpurun_out/bench_q.jsonl | python -c "import json,sys; d=json.loads(sys.stdin.readline()); print(d['ms_per_step'], d.get('split_ms'), d['roofline']['frac'])"
ncu --set full --clock-control none --import-source on -k regex:'x2_pairs|ik1_sym' -c 2 \
    -o gpurun_out/c4q python bench.py --no-cpu-baseline --steps 1 --warmup 1 --e2e-steps 0 \
    > gpurun_out/ncu_q.log 2>&1; tail -2 gpurun_out/ncu_q.log
