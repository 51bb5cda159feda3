python tools/x2_time.py
python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "matrix_parity or edge or config4 or packed or chunked or graph" > gpurun_out/pytest_q.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_q.log
