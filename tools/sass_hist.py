"""Opcode histogram (executed instructions, stall samples) of one kernel from
`ncu -i rep --page source --csv --print-source sass` output.  usage:
python tools/sass_hist.py src.csv [kernel_index] [top]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
kidx = int(sys.argv[2]) if len(sys.argv) > 2 else 0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 25
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
    elif r and r[0] == "Address":
        cur["hdr"] = r
    elif cur is not None and "hdr" in cur:
        cur["rows"].append(dict(zip(cur["hdr"], r)))
b = blocks[kidx]
data = b["rows"]
iv = lambda d, k: int(d.get(k) or 0)
ti = sum(iv(d, "Instructions Executed") for d in data)
ts = sum(iv(d, "Warp Stall Sampling (All Samples)") for d in data)
print(b["name"][:100], "inst", ti, "samples", ts)
ci, cs = Counter(), Counter()
for d in data:
    tok = d["Source"].strip().split()
    if not tok:
        continue
    op = tok[1] if tok[0].startswith("@") else tok[0]
    op = op.split(".")[0]
    ci[op] += iv(d, "Instructions Executed")
    cs[op] += iv(d, "Warp Stall Sampling (All Samples)")
for op, v in ci.most_common(top):
    print("%-10s inst %6.3f  samples %6.3f" % (op, v / ti, cs[op] / max(ts, 1)))
if "--lines" in sys.argv:
    for d in sorted(data, key=lambda d: -iv(d, "Warp Stall Sampling (All Samples)"))[:40]:
        print(d["Address"][-5:], iv(d, "Warp Stall Sampling (All Samples)"), iv(d, "Instructions Executed"), d["Source"].strip()[:90])
