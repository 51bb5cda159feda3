#!/bin/bash
# A/B of library variants in abtmp/lib_<name>.so on the C4 bench (same box, interleaved)
for rep in 1 2; do for v in "$@"; do
  WQB200_LIB=$PWD/abtmp/lib_$v.so python bench.py --no-cpu-baseline --e2e-steps 0 --steps 30 2>/dev/null | \
    python -c "import json,sys; d=json.loads(sys.stdin.readline()); s=d['split_ms']; print('$v', round(d['ms_per_step'],3), round(s['ik1_sym'],3), round(s['x2_pairs'],3))"
done; done
