"""Digest of one ncu capture: key counters plus stall reasons and instruction mix by SASS opcode.

usage: python tools/ncu_digest.py <report.ncu-rep>   (needs ncu on PATH; reads the raw and source pages)
"""
import collections
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
d = dict(zip(rows[0], rows[2]))
units = dict(zip(rows[0], rows[1]))  # ncu's units row (e.g. "Mbyte", "usecond", "%"): printed with every value
print(f"kernel: {d.get('Kernel Name')}")
for k in ["gpu__time_duration.sum", "launch__registers_per_thread", "launch__block_size", "launch__grid_size",
          "dram__bytes_read.sum", "dram__bytes_write.sum", "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
          "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
          "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__warps_active.avg.per_cycle_active",
          "smsp__warps_eligible.avg.per_cycle_active", "l1tex__throughput.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts.avg.pct_of_peak_sustained_active",
          "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "lts__throughput.avg.pct_of_peak_sustained_elapsed"]:
    if k in d:
        u = units.get(k, "")
        print(f"  {k} = {d[k]}{' ' + u if u else ''}")
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(io.StringIO(src)))
hdr, data = rows[1], rows[2:]
ix = {h: i for i, h in enumerate(hdr)}
stalls = [h for h in hdr if h.startswith("stall_") and "Not Issued" not in h]
allst, tot, ex = collections.Counter(), collections.Counter(), collections.Counter()
n = 0
for r in data:
    if len(r) < len(hdr):
        continue
    op = r[ix["Source"]].strip().split()
    if not op:
        continue
    o = (op[1] if op[0].startswith("@") else op[0]).split(".")[0]
    s = int(r[ix["# Samples"]] or 0)
    n += s
    tot[o] += s
    ex[o] += int(r[ix["Instructions Executed"]] or 0)
    for st in stalls:
        allst[st] += int(r[ix[st]] or 0)
ne = sum(ex.values())
print(f"stall samples {n}: " + ", ".join(f"{k[6:]} {v / n * 100:.1f}%" for k, v in allst.most_common(10)))
print("opcodes (share of samples / of executed warp instructions): " +
      ", ".join(f"{o} {s / n * 100:.1f}/{ex[o] / ne * 100:.1f}%" for o, s in tot.most_common(14)))
