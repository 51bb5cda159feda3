"""Finer x2_pairs stage-0 timeline (temporary marks; tools only)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
exec(open(os.path.join(os.path.dirname(os.path.abspath(__file__)), 'x2_timeline.py')).read().split("d = np.diff")[0])
names = {2: "init sync", 3: "window issued", 5: "Bfr stored", 6: "window arrived",
         1: "phi0 start", 4: "phi1 start", 7: "end"}
for k in [2, 3, 5, 6, 1, 4, 7]:
    print(f"{names[k]:20s} {np.mean(t[:, k] - t[:, 0]):9.0f}  p10 {np.percentile(t[:, k] - t[:, 0], 10):9.0f}  p90 {np.percentile(t[:, k] - t[:, 0], 90):9.0f}")
