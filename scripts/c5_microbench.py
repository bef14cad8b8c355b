"""C5 quant-linear microbenchmark (SURVEY.md §8 configs, §8(d) K2 roofline).

Shapes M in {4096, 16384, 65536} x K, N in {192, 384, 768, 1536, 3072}; outlier
channel fraction f of K (the same channels for every token, as bench_gemm's
partial Fisher-Yates, gemm.cpp:272-291); inlier codes uniform in [-7, 7] (A4
values carried in int8), outlier codes in [-127, 127], scales U[0.005, 0.02].

Roofline per shape: ops = 2 M N (K + |O|); bytes = M K + N K + 8 M N (f64 output)
+ 9 M |O|; the hybrid epilogue adds (s_j w[r][ch_j]) xo_j per output and outlier
channel in f64 in the reference's order (gemm.cpp:208-216): 3 FP64 lane-ops
each. Bound time = max(ops / int8 peak, bytes / HBM peak, 3 M N |O| / FP64
lane-op peak), all three measured on the device. Prints one JSON line per shape
and a summary table; `frac` = bound time / measured time.

With PACKED=1 the activation operand is the nibble-packed A4 form (K1's codes4,
pack_int4's layout) through ouro_b200_quant_linear_packed, and the byte model
counts M K / 2 for it.

usage: [PACKED=1] c5_microbench.py [out.json]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2503_10959_b200 as ob

ctx = ob.Context(0)
i8_peak = ctx.measure_i8_peak()
f64_lane = ctx.measure_fp64_peak() / 2.0  # T lane-ops/s
with open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "MEASURED_PEAKS.json")) as f:
    hbm = json.load(f)["hbm_gbs"]
print(f"# measured int8 tensor peak {i8_peak:.0f} TOP/s, FP64 {f64_lane:.1f} T lane-ops/s, "
      f"HBM copy peak {hbm:.0f} GB/s", flush=True)
g = torch.Generator(device="cuda").manual_seed(0)
packed = os.environ.get("PACKED", "0") == "1"


def pack_int4(c):  # pack_int4's layout (gemm.cpp:60-73): low nibble = even column
    u = (c.to(torch.int16) & 0xF).to(torch.uint8)
    return (u[:, 0::2] | (u[:, 1::2] << 4)).contiguous()


rows = []
for M in (4096, 16384, 65536):
    for K in (192, 384, 768, 1536, 3072):
        codes = torch.randint(-7, 8, (M, K), dtype=torch.int8, device="cuda", generator=g)
        ocode = torch.randint(-127, 128, (M, K), dtype=torch.int8, device="cuda", generator=g)
        oscale = torch.rand(M, K, dtype=torch.float64, device="cuda", generator=g) * 0.015 + 0.005
        for N in (192, 384, 768, 1536, 3072):
            w = torch.randint(-7, 8, (N, K), dtype=torch.int8, device="cuda", generator=g)
            wt = w.t().contiguous()
            ws = torch.rand(N, dtype=torch.float64, device="cuda", generator=g) * 0.015 + 0.005
            out = torch.empty(M, N, dtype=torch.float64, device="cuda")
            for f in (0.0, 0.01, 0.05):
                n_o = int(round(f * K))
                chans = torch.randperm(K, device="cuda", generator=g)[:n_o].sort().values.cpu().numpy()
                words = np.zeros((K + 31) // 32, np.uint32)
                for ch in chans:
                    words[ch // 32] |= np.uint32(1) << np.uint32(ch % 32)
                cf = dict(codes4=pack_int4(codes)) if packed else dict(codes=codes)
                act = dict(**cf, s_row=torch.full((M,), 0.01, dtype=torch.float64, device="cuda"),
                           ocnt=torch.full((M,), n_o, dtype=torch.int32, device="cuda"),
                           omask=torch.from_numpy(np.tile(words.view(np.int32), (M, 1))).cuda(),
                           ocode=ocode, oscale=oscale)
                for _ in range(2):
                    ctx.quant_linear(act, w, wt, ws, out=out)
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                n = 5
                e0.record()
                for _ in range(n):
                    ctx.quant_linear(act, w, wt, ws, out=out)
                e1.record()
                torch.cuda.synchronize()
                us = e0.elapsed_time(e1) / n * 1e3
                ops = 2.0 * M * N * (K + n_o)
                byts = M * K * (0.5 if packed else 1.0) + N * K + 8.0 * M * N + 9.0 * M * n_o
                tops = ops / us / 1e6
                gbs = byts / us / 1e3
                t_b = {"tensor": ops / i8_peak / 1e6, "hbm": byts / hbm / 1e3,
                       "fp64": 3.0 * M * N * n_o / f64_lane / 1e6}  # us
                bound = max(t_b, key=t_b.get)
                r = dict(M=M, K=K, N=N, f=f, packed=packed, n_outlier_channels=n_o, us=us, tops=tops, gbs=gbs, bound=bound,
                         frac=t_b[bound] / us)
                rows.append(r)
                print(json.dumps(r), flush=True)
        del codes, ocode, oscale
summary = dict(i8_peak_tops=i8_peak, fp64_lane_tops=f64_lane, hbm_gbs=hbm, rows=rows)
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        json.dump(summary, f, indent=1)
print(f"{'M':>6} {'K':>5} {'N':>5} {'f':>5} {'us':>9} {'TOP/s':>7} {'GB/s':>6} {'bound':>6} {'frac':>5}")
for r in rows:
    print(f"{r['M']:6d} {r['K']:5d} {r['N']:5d} {r['f']:5.3f} {r['us']:9.1f} {r['tops']:7.1f} {r['gbs']:6.0f} "
          f"{r['bound']:>6} {r['frac']:5.2f}")
