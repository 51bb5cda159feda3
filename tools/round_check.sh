#!/bin/bash
# full GPU evidence pass (one B200): GPU tests, smoke, the default bench line, the C5 line,
# the reference arm; logs under gpurun_out/
python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/rc_pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/rc_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/rc_smoke.log 2>&1; echo "smoke rc=$?"; tail -3 gpurun_out/rc_smoke.log
python bench.py > gpurun_out/rc_bench.jsonl 2> gpurun_out/rc_bench.err; echo "bench rc=$?"; tail -c 2500 gpurun_out/rc_bench.jsonl
python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/rc_c5.jsonl 2> gpurun_out/rc_c5.err; echo "c5 rc=$?"; tail -c 1500 gpurun_out/rc_c5.jsonl
