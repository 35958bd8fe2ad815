"""Aggregate an ncu source-page (SASS) CSV: samples and stall reasons per opcode,
and the hottest instructions.   python tools/sass_stalls.py file.csv [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
hi = next(i for i, r in enumerate(rows[:10]) if "Source" in r)
hdr = rows[hi]
data = [r for r in rows[hi + 1:] if len(r) == len(hdr)]
S = hdr.index("Warp Stall Sampling (All Samples)")
stalls = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
ex = hdr.index("Instructions Executed")
by_op = collections.defaultdict(lambda: collections.Counter())
tot = collections.Counter()
for r in data:
    op = r[1].split()[0] if r[1].split() else "?"
    if op.startswith("@"):
        op = r[1].split()[1]
    op = op.split(".")[0]
    n = float(r[S] or 0)
    by_op[op]["samples"] += n
    by_op[op]["inst"] += float(r[ex] or 0)
    for i in stalls:
        v = float(r[i] or 0)
        by_op[op][hdr[i]] += v
        tot[hdr[i]] += v
allS = sum(v["samples"] for v in by_op.values())
print("total samples", allS)
print("stalls:", ", ".join(f"{k[6:]} {v / allS:.2f}" for k, v in tot.most_common(8)))
for op, c in sorted(by_op.items(), key=lambda kv: -kv[1]["samples"])[:12]:
    st = sorted(((v, k) for k, v in c.items() if k.startswith("stall_")), reverse=True)[:3]
    print(f"{op:10s} samples {c['samples'] / allS:5.2f} inst {c['inst']:.3g}  " +
          " ".join(f"{k[6:]}={v / allS:.2f}" for v, k in st))
print("--- hottest instructions")
for r in sorted(data, key=lambda r: -float(r[S] or 0))[:top]:
    st = sorted(((float(r[i] or 0), hdr[i][6:]) for i in stalls), reverse=True)[:2]
    print(f"{float(r[S] or 0) / allS:5.3f} {r[0]} {r[1][:60]:60s} {st}")
