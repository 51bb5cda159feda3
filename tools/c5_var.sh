python tools/c5_time.py
python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "segmented or config5_full" > gpurun_out/pytest_seg.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_seg.log
