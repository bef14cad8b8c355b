"""Per-kernel summary of an `ncu --set full` capture of one forward (DRAM bytes, time,
issue / warp / pipe utilisation), and the scan kernel's (K3, the dominant kernel of
the bench forward) entry for bench.py's roofline (profiles/<round>/k3_ncu.json).

usage: ncu_k3_summary.py REPORT OUT_JSON OUT_TXT [source note]
"""
import csv, json, subprocess, sys

rep, out_json, out_txt = sys.argv[1:4]
note = sys.argv[4] if len(sys.argv) > 4 else rep
M = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
     "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
     "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
     "sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active",
     "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active",
     "sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active",
     "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active", "inst_executed",
     "launch__registers_per_thread"]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv", "--metrics", ",".join(M)], capture_output=True,
                     text=True).stdout
rows = list(csv.reader(raw.splitlines()))
hdr, units = rows[0], rows[1]
idx = {k: i for i, k in enumerate(hdr)}
kern = []
for r in rows[2:]:
    def g(k):
        try:
            return float(r[idx[k]].replace(",", ""))
        except (KeyError, ValueError):
            return None
    t_ms = g("gpu__time_duration.sum")
    tu = units[idx["gpu__time_duration.sum"]]
    t_ms = t_ms / 1e3 if tu == "us" else (t_ms / 1e6 if tu == "ns" else t_ms)
    scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    rd = g("dram__bytes_read.sum") * scale.get(units[idx["dram__bytes_read.sum"]], 1)
    wr = g("dram__bytes_write.sum") * scale.get(units[idx["dram__bytes_write.sum"]], 1)
    kern.append(dict(name=r[idx["Kernel Name"]], ms=t_ms, dram_read=rd, dram_write=wr,
                     issue_active_pct=g(M[3]), warps_active_pct=g(M[4]), fp64_pipe_pct=g(M[5]),
                     fma_pipe_pct=g(M[6]), xu_pipe_pct=g(M[7]), alu_pipe_pct=g(M[8]), tensor_pipe_pct=g(M[9]),
                     inst_executed=g(M[10]), registers=g(M[11])))
with open(out_txt, "w") as f:
    f.write(f"# {note}\n# ncu times are serialised / cold-cache (compare shares with bench.py, not absolutes)\n")
    f.write(f"{'kernel':48s} {'us':>8s} {'read MB':>9s} {'write MB':>9s} {'TB/s':>6s} {'issue%':>7s} {'warps%':>7s}"
            f" {'fp64%':>6s} {'fma%':>6s} {'xu%':>6s} {'alu%':>6s} {'tc%':>6s} {'regs':>5s}\n")
    for k in kern:
        tbs = (k["dram_read"] + k["dram_write"]) / (k["ms"] * 1e-3) / 1e12 if k["ms"] else 0
        f.write(f"{k['name'][:48]:48s} {k['ms'] * 1e3:8.1f} {k['dram_read'] / 1e6:9.1f} {k['dram_write'] / 1e6:9.1f}"
                f" {tbs:6.2f} {k['issue_active_pct'] or 0:7.1f} {k['warps_active_pct'] or 0:7.1f}"
                f" {k['fp64_pipe_pct'] or 0:6.1f} {k['fma_pipe_pct'] or 0:6.1f} {k['xu_pipe_pct'] or 0:6.1f}"
                f" {k['alu_pipe_pct'] or 0:6.1f} {k['tensor_pipe_pct'] or 0:6.1f} {k['registers'] or 0:5.0f}\n")
k3 = max((k for k in kern if "k3_scan" in k["name"]), key=lambda k: k["ms"])
summary = {"source": note, "kernel": k3["name"], "ncu_ms_per_launch": k3["ms"],
           "dram_bytes_per_launch": k3["dram_read"] + k3["dram_write"], "dram_read": k3["dram_read"],
           "dram_write": k3["dram_write"], "issue_active_pct": k3["issue_active_pct"],
           "warps_active_pct": k3["warps_active_pct"], "fp64_pipe_pct": k3["fp64_pipe_pct"],
           "fma_pipe_pct": k3["fma_pipe_pct"], "xu_pipe_pct": k3["xu_pipe_pct"], "alu_pipe_pct": k3["alu_pipe_pct"],
           "inst_executed": k3["inst_executed"], "registers": k3["registers"]}
with open(out_json, "w") as f:
    json.dump(summary, f, indent=1)
print(open(out_txt).read())
