"""Top SASS lines of an ncu --set full capture by warp-stall samples, with the
dominant stall reasons (tools only).  Usage: ncu_lines.py report.ncu-rep [n] [kernel-substring]"""
import csv, io, subprocess, sys
rep = sys.argv[1]
n = int(sys.argv[2]) if len(sys.argv) > 2 else 30
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
S = h.index("Warp Stall Sampling (All Samples)")
reasons = [k for k in h if k.startswith("stall_") and "Not Issued" not in k]
data = []
for r in rows[2:]:
    if len(r) < len(h):
        continue
    try:
        v = int(r[S])
    except ValueError:
        continue
    rs = sorted(((int(r[h.index(k)] or 0), k[6:]) for k in reasons), reverse=True)[:3]
    data.append((v, r[0][-5:], r[1].strip(), rs))
tot = sum(d[0] for d in data) or 1
print("total samples", tot)
for v, a, src, rs in sorted(data, key=lambda x: -x[0])[:n]:
    print(f"{v:7d} {100 * v / tot:5.1f}% {a} {src[:70]:70s} " + " ".join(f"{k}:{c}" for c, k in rs if c))
