"""Summarise an ncu report: key throughput / stall metrics and the executed SASS mix."""
import csv, collections, subprocess, sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
KEYS = ["Kernel Name", "gpu__time_duration.sum", "launch__registers_per_thread", "launch__waves_per_multiprocessor",
        "sm__warps_active.avg.per_cycle_active", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed"]
for r in rows[2:]:
    for k in KEYS:
        if k in hdr:
            print(f"  {k} = {r[hdr.index(k)]} {units[hdr.index(k)]}")
    stalls = [(h.replace("smsp__average_warps_issue_stalled_", "").replace("_per_issue_active.ratio", ""), float(r[j]))
              for j, h in enumerate(hdr) if h.startswith("smsp__average_warps_issue_stalled_") and r[j] not in ("", "0")]
    print("  stalls/issue:", ", ".join(f"{n}={v:.2f}" for n, v in sorted(stalls, key=lambda x: -x[1])[:8]))
src = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(src.splitlines()))
for k, r in enumerate(rows):
    if r and r[0] == "Address":
        hdr = r
        data = rows[k + 1:]
        break
else:
    sys.exit(0)
ie, sc = hdr.index("Instructions Executed"), hdr.index("Source")
tot, ops = 0, collections.Counter()
for r in data:
    if len(r) <= ie or not r[ie].isdigit():
        continue
    n = int(r[ie])
    toks = r[sc].split()
    if not toks:
        continue
    op = toks[1] if toks[0].startswith("@") else toks[0]
    ops[op.split(".")[0]] += n
    tot += n
print(f"  executed warp-instructions: {tot}")
print("  mix:", ", ".join(f"{k} {v / tot * 100:.1f}%" for k, v in ops.most_common(22)))
