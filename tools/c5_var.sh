python tools/c5_time.py
python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "graded or general_path or per_pair or matrix_parity_full" > gpurun_out/pytest_st.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_st.log
