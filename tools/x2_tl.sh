WQB200_X2=6 WQB200_LIB=tools/_build/libwqb200_tl.so python tools/x2_tl.py
for v in 6 4; do WQB200_X2=$v python tools/x2_time.py; done
WQB200_X2=6 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "matrix_parity or edge or config4 or packed or chunked or graph" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_q.log
