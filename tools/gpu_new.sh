python -m pytest tests -m gpu -q -p no:cacheprovider -k "nref2 or edge or components or rhs_parity or config5_full" > gpurun_out/pytest_new.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_new.log
