#!/bin/bash
# Round-end evidence on one B200 (run under gpurun): bench lines (C4, reference arm, C5),
# the ncu launch list of the default bench command, and one ncu --set full capture of the
# two C4 kernels.  Outputs in gpurun_out/; summaries are copied into profiles/ by hand.
set -x
python bench.py > gpurun_out/bench_default.jsonl 2> gpurun_out/bench_default.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_reference.jsonl 2> gpurun_out/bench_reference.err
python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/bench_c5.jsonl 2> gpurun_out/bench_c5.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv \
    python bench.py --steps 3 --warmup 3 --e2e-steps 1 --no-cpu-baseline > gpurun_out/ncu_launches.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'x2ws|ik1_sym' -c 2 \
    -o gpurun_out/c4full python bench.py --no-cpu-baseline --steps 1 --warmup 1 --e2e-steps 0 \
    > gpurun_out/ncu_full.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:'ystage_ws|band_seg_solve|gather_yts|st_phi_sym' -c 6 \
    -o gpurun_out/c5full python bench.py --workload c5 --steps 1 --warmup 0 > gpurun_out/ncu_c5.log 2>&1
