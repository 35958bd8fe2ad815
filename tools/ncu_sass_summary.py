"""Summarise an ncu --page source --print-source=sass CSV: stall reasons, top instructions."""
import csv, sys
from collections import Counter
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[1]; idx = {h: i for i, h in enumerate(hdr)}
reasons = [h for h in hdr if h.startswith('stall_') and 'Not Issued' not in h]
tot = Counter(); inst = []
for r in rows[2:]:
    if len(r) < len(hdr) - 1: continue
    try:
        ex = float(r[idx['Instructions Executed']] or 0)
        samp = float(r[idx['Warp Stall Sampling (All Samples)']] or 0)
    except ValueError:
        continue
    for h in reasons:
        try: tot[h] += float(r[idx[h]] or 0)
        except ValueError: pass
    inst.append((samp, ex, r[idx['Address']][-5:], r[idx['Source']].strip()[:90]))
s = sum(tot.values())
print("stall reasons:", ", ".join(f"{k[6:]} {100*v/s:.1f}%" for k, v in tot.most_common(8)))
ts = sum(i[0] for i in inst)
for samp, ex, a, src in sorted(inst, reverse=True)[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{100*samp/ts:5.1f}%  {a}  {src}")
