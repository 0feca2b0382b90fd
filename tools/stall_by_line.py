"""Stall samples of one ncu capture aggregated by CUDA source line.

ncu's source page prints per-SASS-instruction stall samples; nvdisasm -g maps
each SASS address of the same object to its (innermost inlined) source line.
usage: python tools/stall_by_line.py <report.ncu-rep> <object.o> <mangled kernel name> [top]
(the object must be the build that was profiled; compiled with -lineinfo)
"""
import collections
import csv
import io
import os
import re
import subprocess
import sys
import tempfile

rep, obj, kern = sys.argv[1], sys.argv[2], sys.argv[3]
top = int(sys.argv[4]) if len(sys.argv) > 4 else 30
with tempfile.TemporaryDirectory() as d:
    subprocess.run(["cuobjdump", "-xelf", "all", os.path.abspath(obj)], cwd=d, capture_output=True)
    cubin = [f for f in os.listdir(d) if f.endswith(".cubin")][0]
    dis = subprocess.run(["nvdisasm", "-g", "-c", os.path.join(d, cubin)], capture_output=True, text=True).stdout
lines = dis.split("\n")
start = next(i for i, l in enumerate(lines) if f".text.{kern}" in l and "section" in l)
end = next((i for i in range(start + 3, len(lines)) if lines[i].startswith("//-----") and ".text." in lines[i]),
           len(lines))
addr2line, cur = {}, None
for l in lines[start:end]:
    mm = re.match(r'\s*//## File "([^"]+)", line (\d+)', l)
    if mm:
        cur = (os.path.basename(mm.group(1)), int(mm.group(2)))
        continue
    ma = re.match(r"\s*/\*([0-9a-f]{4,})\*/", l)
    if ma and cur:
        addr2line[int(ma.group(1), 16)] = cur
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr, data = rows[1], rows[2:]
ia, iall, iex = hdr.index("Address"), hdr.index("Warp Stall Sampling (All Samples)"), hdr.index("Instructions Executed")
stall_cols = [i for i, h in enumerate(hdr) if h.startswith("stall_") and "Not Issued" not in h]
base = int(data[0][ia], 16)
agg = collections.defaultdict(lambda: [0, 0, collections.Counter()])
total = 0
for r in data:
    a = int(r[ia], 16) - base
    s = int(r[iall] or 0)
    total += s
    e = agg[addr2line.get(a, ("?", 0))]
    e[0] += s
    e[1] += int(r[iex] or 0)
    for i in stall_cols:
        if r[i] and r[i] != "0":
            e[2][hdr[i][6:]] += int(float(r[i]))
print(f"{total} stall samples over {len(data)} SASS instructions of {kern}")
print("source line          share   warp instr. executed   top stall reasons (samples)")
for (f, ln), (s, ex, c) in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{f + ':' + str(ln):<22} {100 * s / total:5.2f}%  {ex:>12}   " + ", ".join(f"{k} {v}" for k, v in c.most_common(3)))
