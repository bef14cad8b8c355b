"""Per-CUDA-source-line instruction counts and stall samples of one kernel in an ncu
report (source page, cuda+sass view), sorted by samples.

usage: ncu_srclines.py REPORT [normaliser] [top] [kernel-regex | skip:N]
"""
import csv, subprocess, sys

rep = sys.argv[1]
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
top = int(sys.argv[3]) if len(sys.argv) > 3 else 60
cmd = ["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"]
if len(sys.argv) > 4:
    sel = sys.argv[4]
    cmd += (["--launch-skip", sel[5:], "--launch-count", "1"] if sel.startswith("skip:")
            else ["-k", "regex:" + sel, "-c", "1"])
out = subprocess.run(cmd, capture_output=True, text=True).stdout
fname, hdr, rows, func = None, None, [], None
for r in csv.reader(out.splitlines()):
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Function Name":
        if func is not None and r[1] != func:
            break
        func = r[1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or not r[0]:
        continue
    try:
        ie = int(r[hdr.index("Instructions Executed")])
        sm = int(r[hdr.index("# Samples")])
    except (ValueError, IndexError):
        continue
    if ie or sm:
        rows.append((sm, ie, f"{fname}:{r[0]}", r[1].strip()[:90]))
ts = sum(r[0] for r in rows) or 1
ti = sum(r[1] for r in rows) or 1
print(f"total instructions {ti} ({ti / norm:.1f} per unit), samples {ts}")
for sm, ie, loc, src in sorted(rows, reverse=True)[:top]:
    print(f"{sm / ts * 100:5.1f}% smp {ie / norm:7.1f} inst  {loc:24s} {src}")
