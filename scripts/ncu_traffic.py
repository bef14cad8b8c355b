"""Per-kernel DRAM traffic and utilisation from an `ncu --set full` report of a
bench.py run (one launch per kernel family).

usage: ncu_traffic.py REPORT OUT_JSON [OUT_TXT]
JSON: {"source": ..., "kernels": {name: [{dram_read_bytes, dram_write_bytes,
traffic_bytes, ncu_time, time_unit}, ...]}} (what bench.py reads for
roofline.traffic); TXT: a table with issue/occupancy/pipe figures.
"""
import csv
import json
import subprocess
import sys

rep, out_json = sys.argv[1], sys.argv[2]
out_txt = sys.argv[3] if len(sys.argv) > 3 else None
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units, data = rows[0], rows[1], rows[2:]


def get(r, name, scale_to=None):
    i = hdr.index(name)
    try:
        v = float(r[i].replace(",", ""))
    except ValueError:  # "no data" for a metric ncu could not collect on this kernel
        return float("nan")
    u = units[i]
    if scale_to == "bytes":
        v *= {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}.get(u, 1)
    if scale_to == "ms":
        v *= {"nsecond": 1e-6, "usecond": 1e-3, "msecond": 1.0, "second": 1e3}.get(u, 1)
    return v


kernels, lines = {}, []
cols = ["smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "sm__mem_tensor_cycles_active.avg.pct_of_peak_sustained_active"]
for r in data:
    name = r[hdr.index("Kernel Name")].split("(")[0].replace("void ", "").replace("ob::", "")
    rd, wr = get(r, "dram__bytes_read.sum", "bytes"), get(r, "dram__bytes_write.sum", "bytes")
    t = get(r, "gpu__time_duration.sum", "ms")
    kernels.setdefault(name, []).append(dict(dram_read_bytes=rd, dram_write_bytes=wr, traffic_bytes=rd + wr,
                                             ncu_time=t, time_unit="ms"))
    extra = "  ".join(f"{c.split('__')[1].split('.')[0]} {get(r, c):5.1f}%" for c in cols if c in hdr)
    lines.append(f"{name:28s} {t * 1e3:9.1f} us  read {rd / 1e6:8.1f} MB  write {wr / 1e6:8.1f} MB  "
                 f"{(rd + wr) / (t * 1e-3) / 1e12:5.2f} TB/s  {extra}")
with open(out_json, "w") as f:
    json.dump({"source": f"ncu --set full --clock-control none ({rep.split('/')[-1]}), bench.py --steps 1 "
                         "--warmup 3 (B=256 Vim-B W4A4), first quantized forward, block 0", "kernels": kernels}, f,
              indent=1)
text = "\n".join(lines)
print(text)
if out_txt:
    with open(out_txt, "w") as f:
        f.write(text + "\n")
