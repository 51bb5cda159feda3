# ncu --set full of one x2 launch (C4)
python tools/run_x2_once.py > gpurun_out/x2once.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'x2v4' -s 1 -c 1 \
    -o gpurun_out/x2prof -f python tools/run_x2_once.py > gpurun_out/ncu_x2.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu_x2.log
