"""Hot SASS of an `ncu --page source --csv --print-source sass` export:
instructions executed >= min_exec times, with their stall samples, in
address order (the critical path of a latency-bound loop reads top-down).
usage: python tools/sass_hot.py export.csv [min_exec] [min_samples]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = rows[1], rows[2:]
iS = hdr.index("Warp Stall Sampling (All Samples)")
iE = hdr.index("Instructions Executed")
min_exec = int(sys.argv[2]) if len(sys.argv) > 2 else 1000
min_s = int(sys.argv[3]) if len(sys.argv) > 3 else 0
tot = sum(int(r[iS] or 0) for r in data)
hot = [(i, r) for i, r in enumerate(data) if int(r[iE] or 0) >= min_exec]
print(f"total samples {tot}; {len(hot)} instructions executed >= {min_exec}x, "
      f"{sum(int(r[iS] or 0) for _, r in hot)} samples on them")
for i, r in hot:
    if int(r[iS] or 0) >= min_s:
        print(f"{i:5d} {int(r[iS] or 0):4d} {int(r[iE]):7d}  {r[1].strip()[:72]}")
