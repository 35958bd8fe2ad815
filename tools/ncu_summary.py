"""Summarise an ncu launch list (+ optional --set full raw export) of one truncation
step per pipeline stage (library kernel tag).

    python tools/ncu_summary.py gpurun_out/launches.csv gpurun_out/tags.json [full_raw.csv] > summary.json

Writes per-tag: launches, ncu time (cold-cache, serialised), share of the step, and
from the full capture the DRAM bytes per launch (dram__bytes_read.sum +
dram__bytes_write.sum) and the DMMA pipe utilisation."""
import csv
import json
import sys


def kernels(path):
    rows = list(csv.reader(open(path)))
    hdr, out = None, {}
    for r in rows:
        if "Kernel Name" in r and "ID" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            out.setdefault(int(d["ID"]), {"name": d["Kernel Name"]})[d["Metric Name"]] = d["Metric Value"]
    return [out[k] for k in sorted(out)]


def num(v):
    try:
        return float(str(v).replace(",", ""))
    except ValueError:
        return float("nan")


OURS = ("ht::", "unnamed>::", "identity_kernel", "zero_kernel", "root_blocks_kernel", "kron_factor_kernel")
launches = [k for k in kernels(sys.argv[1]) if any(o in k["name"] for o in OURS)]
tags = json.load(open(sys.argv[2]))
if len(tags) != len(launches):
    sys.exit(f"tag log ({len(tags)}) and launch list ({len(launches)}) differ")
raw = None
if len(sys.argv) > 3:
    rows = list(csv.reader(open(sys.argv[3])))
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12}
    raw = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        for key in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            if key in d:
                d[key] = num(d[key]) * scale.get(units[hdr.index(key)], 1.0)
        raw.append(d)
    raw = [r for r in raw if any(o in r.get("Kernel Name", "") for o in OURS)]
step_us = sum(num(k["gpu__time_duration.sum"]) / 1e3 for k in launches)
# align the full-capture rows to the launch list by kernel name, in order
raw_for = [None] * len(launches)
if raw is not None:
    j = 0
    for i, k in enumerate(launches):
        base = k["name"].split("(")[0]
        if j < len(raw) and raw[j].get("Kernel Name", "").split("(")[0] == base:
            raw_for[i] = raw[j]
            j += 1
per = {}
for i, (k, (tag, flops, nbytes)) in enumerate(zip(launches, tags)):
    e = per.setdefault(tag, {"launches": 0, "ncu_us": 0.0, "flops": 0.0, "kernel": k["name"].split("(")[0]})
    e["launches"] += 1
    e["ncu_us"] += num(k["gpu__time_duration.sum"]) / 1e3
    e["flops"] += flops
    if raw_for[i] is not None:
        r = raw_for[i]
        e.setdefault("dram_bytes", 0.0)
        e["dram_bytes"] += num(r.get("dram__bytes_read.sum", 0)) + num(r.get("dram__bytes_write.sum", 0))
        e.setdefault("dmma_pct", []).append(num(r.get("sm__pipe_tensor_subpipe_dmma_cycles_active.avg.pct_of_peak_sustained_active", "nan")))
for tag, e in per.items():
    e["share_of_step"] = e["ncu_us"] / step_us
    e["tflops_ncu"] = e["flops"] / (e["ncu_us"] * 1e-6) / 1e12 if e["flops"] else None
    if "dram_bytes" in e:
        e["dram_bytes_per_launch"] = e["dram_bytes"] / e["launches"]
        v = [x for x in e.pop("dmma_pct") if x == x]
        e["dmma_pipe_pct_active_mean"] = sum(v) / len(v) if v else None
json.dump({"step_us_ncu": step_us, "launches": len(launches),
           "stages": dict(sorted(per.items(), key=lambda kv: -kv[1]["ncu_us"]))}, sys.stdout, indent=1)
