python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "end_node or segmented or graded" > gpurun_out/pytest_fix.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_fix.log
