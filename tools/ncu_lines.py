"""Attribute ncu SASS-level warp samples to CUDA source lines.

    python tools/ncu_lines.py <sass.csv from ncu --page source --print-source sass> <source.cu> [kernel-index]

Line numbers come from `nvdisasm -g` of the in-tree library's cubin for <source.cu>."""
import csv
import os
import re
import subprocess
import sys
import tempfile

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sass_csv, src = sys.argv[1], sys.argv[2]
kidx = int(sys.argv[3]) if len(sys.argv) > 3 else 0
stem = os.path.splitext(os.path.basename(src))[0]
tmp = tempfile.mkdtemp()
subprocess.run(["cuobjdump", "-xelf", "all", os.path.join(ROOT, "paper_1708_03340_b200", "libht_b200.so")],
               cwd=tmp, capture_output=True)
cubin = os.path.join(tmp, f"{stem}.sm_100a.cubin")
dis = subprocess.run(["nvdisasm", "-g", "-c", cubin], capture_output=True, text=True).stdout
rows = list(csv.reader(open(sass_csv)))
blocks, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = {"name": r[1], "rows": []}
        blocks.append(cur)
        continue
    if r and r[0] == "Address":
        cur["hdr"] = r
        continue
    if cur is not None and r:
        cur["rows"].append(r)
b = blocks[kidx]
h = b["hdr"]
iN, iS = h.index("# Samples"), h.index("Source")
# split the disassembly per function; pick the one whose first opcodes match
funcs, name = {}, None
for l in dis.split("\n"):
    m = re.match(r"\s*\.text\.(\S+):", l)
    if m:
        name = m.group(1)
        funcs[name] = []
        continue
    if name:
        funcs[name].append(l)
want = re.sub(r"\(.*", "", b["name"]).split("::")[-1].split("<")[0]
cands = [f for f in funcs if want in f]
targs = re.findall(r"\(int\)(-?\d+)", b["name"].split("(ht::")[0]) or re.findall(r"<(.*)>", b["name"])
if targs and all(re.fullmatch(r"-?\d+", a) for a in targs):  # template instance: match the mangled args
    tag = "I" + "".join("Li%sE" % a.replace("-", "n") for a in targs) + "E"
    cands = [f for f in cands if tag in f] or cands
lines, curl = {}, None
for l in funcs[cands[0]]:
    m = re.search(r"line (\d+)", l)
    if m and "//##" in l:
        curl = int(m.group(1))
        continue
    m = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if m and curl is not None:
        lines[int(m.group(1), 16)] = curl
base = min(int(r[0], 16) for r in b["rows"])
stl = [(i, c) for i, c in enumerate(h) if c.startswith("stall_") and "Not Issued" not in c]
agg, tot, why = {}, 0, {}
for r in b["rows"]:
    n = int(r[iN] or 0)
    tot += n
    ln = lines.get(int(r[0], 16) - base, -1)
    agg[ln] = agg.get(ln, 0) + n
    w = why.setdefault(ln, {})
    for i, c in stl:
        w[c[6:]] = w.get(c[6:], 0) + float(r[i] or 0)
text = open(src).read().split("\n")
print(b["name"][:80], "samples", tot, "function", cands[0][:60])
for ln, n in sorted(agg.items(), key=lambda kv: -kv[1])[:30]:
    top = sorted(why.get(ln, {}).items(), key=lambda kv: -kv[1])[:3]
    ws = " ".join("%s:%d" % (k, v) for k, v in top if v > 0)
    print("%5.1f%%  %4d  %-70s %s" % (100 * n / max(tot, 1), ln,
                                      text[ln - 1].strip()[:70] if 0 < ln <= len(text) else "(inlined header)", ws))
