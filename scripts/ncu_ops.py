"""Dynamic SASS opcode histogram of the first kernel in an ncu report (source page, SASS rows).

usage: ncu_ops.py REPORT [normaliser]   -- counts are divided by the normaliser (e.g. warp-steps)
"""
import csv, collections, subprocess, sys

rep = sys.argv[1]
norm = float(sys.argv[2]) if len(sys.argv) > 2 else 1.0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"] + (["-k", sys.argv[3]] if len(sys.argv) > 3 else []),
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, fname = None, None
seen = set()
ops, samples = collections.Counter(), collections.Counter()
for r in rows:
    if not r:
        continue
    if r[0] == "Function Name":
        if fname and r[1] != fname:
            break
        fname = r[1]
        continue
    if r[0] in ("Address", "Line No"):
        hdr = r
        continue
    if hdr is None:
        continue
    ai = hdr.index("Address") if "Address" in hdr else None
    si = hdr.index("Source", ai + 1 if ai is not None else 0)
    addr = r[ai] if ai is not None else None
    if not addr or not addr.startswith("0x") or addr in seen:
        continue
    seen.add(addr)
    ie = r[hdr.index("Instructions Executed")]
    sm = r[hdr.index("# Samples")]
    op = r[si].split()[0] if r[si].split() else "?"
    if op.startswith("@"):
        op = r[si].split()[1]
    ops[op.split(".")[0]] += int(ie) if ie.isdigit() else 0
    samples[op.split(".")[0]] += int(sm) if sm.isdigit() else 0
tot = sum(ops.values())
ts = sum(samples.values()) or 1
print(f"total {tot} ({tot / norm:.1f} per unit), {len(seen)} SASS instructions")
for op, n in ops.most_common(40):
    print(f"  {op:10s} {n / norm:8.1f}  {n / tot * 100:5.1f}%  samples {samples[op] / ts * 100:5.1f}%")
