python tools/c5_time.py > gpurun_out/c5once.log 2>&1 && \
ncu --set full --clock-control none --import-source on -k regex:'add_st_phi|gather_fs|ystage_mma_kernel' -c 4 \
    -o gpurun_out/c5prof -f python tools/c5_time.py > gpurun_out/ncu_c5.log 2>&1
echo "rc=$?"; tail -3 gpurun_out/ncu_c5.log
