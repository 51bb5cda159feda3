# A/B of the x2 kernel versions (WQB200_X2) on the C4 bench split, then the parity tests
for v in 4 3; do
  WQB200_X2=$v python bench.py --steps 5 --warmup 3 --no-cpu-baseline --e2e-steps 0 > gpurun_out/ab_x2_$v.log 2>&1
  echo "x2 v$v rc=$?"; python - <<PY
import json
for ln in open("gpurun_out/ab_x2_$v.log"):
    if ln.startswith("{"):
        d = json.loads(ln); print("v$v", round(d["ms_per_step"], 3), d["split_ms"], round(d["roofline"]["frac"], 4))
PY
done
python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "parity or edge or scale" > gpurun_out/pytest_x2.log 2>&1; echo "pytest rc=$?"; tail -5 gpurun_out/pytest_x2.log
