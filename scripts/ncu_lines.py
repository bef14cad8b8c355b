"""Per-source-line executed instructions and stall samples of the first kernel in an ncu report."""
import csv, collections, subprocess, sys
rep = sys.argv[1]; top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
cur, hdr, line = None, None, None
agg, samp, src, nfun, fname = collections.Counter(), collections.Counter(), {}, 0, None
for r in rows:
    if not r: continue
    if r[0] == "Function Name":
        if nfun and r[1] != fname: break
        fname, nfun = r[1], 1
    if r[0] == "File Path": cur = r[1].split('/')[-1]; continue
    if r[0] == "Line No": hdr = r; continue
    if hdr is None or len(r) < 8: continue
    if r[0]: line = (cur, int(r[0])); src[line] = r[1][:95]
    ie, sm = hdr.index("Instructions Executed"), hdr.index("# Samples")
    if line and r[ie].isdigit():
        agg[line] += int(r[ie]); samp[line] += int(r[sm]) if r[sm].isdigit() else 0
ts = sum(samp.values()) or 1
ti = sum(agg.values()) or 1
for k in sorted(samp, key=lambda k: -samp[k])[:top]:
    print(f"samp {samp[k]/ts*100:5.1f}%  inst {agg[k]/ti*100:5.1f}%  {k[0]}:{k[1]:4d} {src[k]}")
