python bench.py --workload c5 --steps 5 --warmup 3 > gpurun_out/b2_c5.jsonl 2> gpurun_out/b2_c5.err; echo "c5 rc=$?"; tail -c 3000 gpurun_out/b2_c5.jsonl
( time python bench.py --impl reference --steps 20 --warmup 5 ) > gpurun_out/b2_ref.jsonl 2> gpurun_out/b2_ref.err; echo "ref rc=$?"; tail -c 4000 gpurun_out/b2_ref.jsonl; tail -4 gpurun_out/b2_ref.err
