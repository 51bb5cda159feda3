python tools/c5_time.py /tmp/c5_seg.npy
SEG=0 python tools/c5_time.py /tmp/c5_win.npy
python -c "
import numpy as np; a=np.load("/tmp/c5_seg.npy"); b=np.load("/tmp/c5_win.npy"); print('seg vs win', np.abs(a-b).max()/np.abs(b).max())"
python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "segmented or graded or lattice or per_pair or general_path" > gpurun_out/pytest_c5.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_c5.log
