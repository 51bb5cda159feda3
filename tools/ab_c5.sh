#!/bin/bash
# A/B of library variants on the C5 bench (abtmp/lib_<name>.so)
for rep in 1 2; do for v in "$@"; do
  WQB200_LIB=$PWD/abtmp/lib_$v.so python bench.py --workload c5 --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.readline()); s=d.get('split_ms',{}); print('$v', round(d['ms_per_step'],2), {k: s[k] for k in ('wq_gather_fs','wq_add_st_phi','wq_band_solve_win') if k in s})"
done; done
