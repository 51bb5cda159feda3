"""Generate the B-bin table (default 16; argv[1]) of half_ln16 (wq_log.cuh): c_j near 1/mid_j (mid_j the
centre of mantissa bin j of [1, 2)) chosen so that 0.5*(-ln c_j) is within 2^-12 ulp
of a double (Tang's accurate-table trick): the table then needs one double for the
logarithm instead of a double-double pair.  Prints C++ initialisers."""
from decimal import Decimal, getcontext
import struct, math

getcontext().prec = 60

def ulp(x):
    return math.ulp(x)

rows = []
import sys
B = int(sys.argv[1]) if len(sys.argv) > 1 else 16
for j in range(B):
    mid = 1.0 + (j + 0.5) / B
    base = round((1.0 / mid) * 2 ** 24)
    best = None
    for t in range(0, 200000):
        for s in (1, -1):
            cand = (base + s * t) / 2 ** 24
            L = -(Decimal(cand).ln()) / 2  # 0.5 * (-ln c)
            h = float(L)
            res = abs(L - Decimal(h)) / Decimal(ulp(h)) if h != 0 else Decimal(0)
            if res < Decimal(2) ** -12:
                best = (cand, h, float(res))
                break
        if best:
            break
    c, h, res = best
    # |r| bound for m in bin j: m*c - 1
    lo_m, hi_m = 1 + j / B, 1 + (j + 1) / B
    rmax = max(abs(lo_m * c - 1), abs(hi_m * c - 1))
    rows.append((c, h, res, rmax))
    print(f"    {c!r}, {h!r},  // {j} resid {res:.1e} ulp |r| <= {rmax:.5f}")
print("max |r|", max(r[3] for r in rows))


def economised_series(a=0.0077945, n=4000):
    """Degree-4 q(r) of half_ln64t (kLn64C): Taylor to r^4 plus the r^5 term
    -r^5/14 Chebyshev-economised on |r| <= a; prints the coefficients and the
    largest absolute error of 0.5 ln(1+r) = r/2 - r^2 q(r) (mpmath, 40 digits)."""
    import mpmath as mp
    mp.mp.dps = 40
    a = mp.mpf(a)
    c = [mp.mpf(1) / 12, -mp.mpf(1) / 10 - 20 * a ** 2 / 224, mp.mpf(1) / 8,
         -mp.mpf(1) / 6 + 5 * a ** 4 / 224, mp.mpf(1) / 4]
    cd = [float(x) for x in c]
    worst = 0
    for i in range(-n, n + 1):
        r = a * i / n
        q = cd[0]
        for k in cd[1:]:
            q = r * q + k
        worst = max(worst, abs(mp.log(1 + r) / 2 - (r / 2 - r * r * q)))
    print("kLn64C series:", [repr(x) for x in cd], "max abs error", float(worst))


if len(sys.argv) > 2 and sys.argv[2] == "series":
    economised_series()
