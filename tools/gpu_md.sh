python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "multi_device or host_streams or packed or edge" > gpurun_out/pytest_md.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_md.log
