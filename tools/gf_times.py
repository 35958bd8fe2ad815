"""Print the ncu launch-list durations of the kernels whose name matches argv[1]."""
import csv
import sys

rows = list(csv.reader(open(sys.argv[2] if len(sys.argv) > 2 else "gpurun_out/launches.csv")))
hdr, out = None, []
for r in rows:
    if "Kernel Name" in r and "ID" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if sys.argv[1] in d["Kernel Name"]:
            out.append(float(d["Metric Value"].replace(",", "")) / 1e3)
print(sys.argv[1], "us:", [round(v, 1) for v in out], "sum", round(sum(out), 1))
