"""Instructions executed and stall samples per CUDA source line of the first kernel
in an ncu report (--import-source on, -lineinfo builds).

usage: ncu_lines.py REPORT [top]
"""
import collections
import csv
import subprocess
import sys

rep = sys.argv[1]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
fpath, cur, hdr = None, None, None
inst, samp, src = collections.Counter(), collections.Counter(), {}
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fpath = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None:
        continue
    if r[0]:
        cur = (fpath, int(r[0]))
        src[cur] = r[1]
    if len(r) > 7 and r[2]:
        try:
            inst[cur] += float(r[hdr.index("Instructions Executed")].replace(",", "") or 0)
            samp[cur] += float(r[hdr.index("Warp Stall Sampling (All Samples)")].replace(",", "") or 0)
        except ValueError:
            pass
tot = sum(inst.values()) or 1.0
ts = sum(samp.values()) or 1.0
for k, v in inst.most_common(top):
    print(f"{v / tot * 100:5.1f}% inst {samp[k] / ts * 100:5.1f}% stall  {k[0]}:{k[1]:<4d} {src.get(k, '').strip()[:88]}")
