#!/usr/bin/env python
"""Benchmark: W4A4 Vim-B quantized forward, images/s (BASELINE.json metric).

Workload (BASELINE.json configs[2], the metric's own config): Vim-Base toy
structure (E=768, N=16, 24 blocks, 224x224x3, patch 16, 196 tokens, 1000
classes, conv 4, row-forward + row-backward scans, D1 pre-norm residual),
W4A4 dynamic OuroMamba-Quant (outliers int8, n_refresh=10, rho=0.01,
D2 quantized linear inputs), batch 256 per GPU, synthetic N(0,1) f64 images,
random-init weights (make_toy_model, seed 1234). One step = one forward of the
batch on every rank (+ the NCCL logits all-gather when N > 1).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

N > 1 is launched by torchrun (one process per GPU). Rank 0 prints one JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIG = dict(workload="Vim-B W4A4 dynamic forward (OuroMamba-Quant), 224x224, batch 256/GPU",
              model="Vim-B toy structure E=768 N=16 24 blocks (D1 pre-norm residual, D2 quantized linear inputs)",
              global_batch=None, seq_len=196, image=224, patch=16, embed=768, state=16, blocks=24, classes=1000,
              quant="W4A4 dynamic, outliers int8, n_refresh=10, rho=0.01", parallelism=None,
              l2="inputs larger than L2 (308 MB of f64 images + ~3 GB of activations per step)")
METRIC = "W4A4 Vim-B images/sec"
UNIT = "images/s"
SEED = 1234


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--batch", type=int, default=256)
    ap.add_argument("--embed", type=int, default=768)
    ap.add_argument("--blocks", type=int, default=24)
    ap.add_argument("--abits", type=int, default=4)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--split-parts", type=int, default=None,
                    help="independent sub-batches on their own streams (engine default 2)")
    ap.add_argument("--feed-chunks", type=int, default=None,
                    help="H2D chunks of the e2e host feed (engine default 8)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "200"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for r in self.rows:
            try:
                sm.append(float(r[1]))
                mx = float(r[2])
                for n, v in zip(names, r[5:9]):
                    if v.strip().lower() == "active":
                        reasons.add(n)
            except (ValueError, IndexError):
                pass
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def cpu_baseline(model_dims, cal_export, images_np, abits, steps=1, warmup=0):
    """The reference's CPU implementation (oracle/_ref: the reference's own
    compiled primitives under the shared driver), all host threads, on a
    bounded sample: `threads` images through the first 2 of 24 blocks,
    extrapolated x12 to the 24-block forward. Returns (img/s, cores, sample)."""
    from oracle import oracle as O
    if not O.ref_available():
        return None
    chk = O.Checker(O.REF_SO)
    cores = os.cpu_count() or 1
    nblk = 2
    d = O.Dims(image=model_dims.image, channels=model_dims.channels, patch=model_dims.patch,
               embed=model_dims.embed, state=model_dims.state, blocks=nblk, classes=model_dims.classes,
               conv_width=model_dims.conv_width)
    m = chk.model(d, SEED)
    scan, lin = cal_export
    nd = 2
    spec = O.Spec(wbits=4, abits=abits, obits=8, n_refresh=10, rho=0.01, d1=True, d2=True)
    cal = O.Calibration(spec, scan=[O.TensorCal(t.theta, t.s_in, t.s_full, t.excluded) for t in scan[:nblk * nd * 3]],
                        lin=[O.TensorCal(t.theta, t.s_in, t.s_full, t.excluded) for t in lin[:nblk * (nd + 2)]])
    ch = m.calib_from(cal)
    n_img = min(cores, images_np.shape[0])
    imgs = np.ascontiguousarray(images_np[:n_img])
    for _ in range(warmup):
        m.forward(imgs, ch, 1, threads=cores)
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        m.forward(imgs, ch, 1, threads=cores)
        times.append(time.perf_counter() - t0)
    t = float(np.median(times))
    per_img_full = t * (model_dims.blocks / nblk) / n_img
    sample = (f"{n_img} images x {nblk} of {model_dims.blocks} blocks (x{model_dims.blocks // nblk} to the full "
              f"forward), W4A4 dynamic D1+D2, {cores} threads, median of {steps}")
    return 1.0 / per_img_full, cores, sample


def run_reference(args):
    rank, world, local = dist_env()
    if rank != 0:
        return 0
    import paper_2503_10959_b200 as ob  # noqa: F401  (only for Dims; no GPU work on this arm)
    from oracle import oracle as O
    if not O.ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref (reference build) missing"}))
        return 0
    dims = ob.Dims(embed=args.embed, blocks=args.blocks)
    chk = O.Checker(O.REF_SO)
    # calibration of the first 2 blocks on the CPU (FP forward with the recorder)
    d2 = O.Dims(image=dims.image, channels=dims.channels, patch=dims.patch, embed=dims.embed, state=dims.state,
                blocks=2, classes=dims.classes, conv_width=dims.conv_width)
    m = chk.model(d2, SEED)
    cores = os.cpu_count() or 1
    spec = O.Spec(wbits=4, abits=args.abits, obits=8, n_refresh=10, rho=0.01)
    cimgs = chk.normal(SEED + 7, 2 * dims.pix)
    cal = m.calibrate(cimgs, spec, threads=cores).export()
    imgs = chk.normal(SEED + 100, cores * dims.pix).reshape(cores, dims.image, dims.image, dims.channels)
    ips, cores, sample = cpu_baseline(dims, (cal.scan, cal.lin), imgs, args.abits, steps=args.steps,
                                      warmup=min(args.warmup, 1))
    cfg = dict(CONFIG, global_batch=args.batch * max(args.gpus, 1), parallelism=f"dp{max(args.gpus, 1)}")
    line = {"metric": METRIC, "value": ips, "unit": UNIT, "n_gpus": args.gpus, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": 1e3 * args.batch / ips, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "int8/f64", "data": "synthetic", "config": cfg,
            "impl": "reference",
            "cpu_baseline": {"value": ips, "unit": UNIT, "cores": cores, "kind": "reference", "sample": sample},
            "e2e": {"value": ips, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line))
    return 0


def run_ours(args):
    import torch
    import torch.distributed as dist
    import paper_2503_10959_b200 as ob

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    stream = torch.cuda.Stream()
    torch.cuda.set_stream(stream)
    ctx = ob.Context(local, stream=stream)
    dims = ob.Dims(embed=args.embed, blocks=args.blocks)
    B = args.batch
    model = ob.Model(ctx, dims, SEED)
    spec = ob.QuantSpec(wbits=4, abits=args.abits, obits=8, n_refresh=10, rho=0.01, d1=True, d2=True)
    gcal = torch.Generator(device="cuda").manual_seed(SEED + 7)
    cal_imgs = torch.randn(8, dims.image, dims.image, dims.channels, dtype=torch.float64, device="cuda",
                           generator=gcal)
    cal = model.calibrate(cal_imgs, spec, chunk=8)
    del cal_imgs
    gen = torch.Generator(device="cuda").manual_seed(SEED + 100 + rank)
    images = torch.randn(B, dims.image, dims.image, dims.channels, dtype=torch.float64, device="cuda", generator=gen)
    logits = torch.empty(B, dims.classes, dtype=torch.float64, device="cuda")
    gathered = [torch.empty_like(logits) for _ in range(world)] if world > 1 else None
    if args.split_parts is not None:
        model.set_option("split_parts", args.split_parts)
    if args.feed_chunks is not None:
        model.set_option("feed_chunks", args.feed_chunks)
    model.use_graphs(True)

    def step():
        model.forward(images, cal, ob.MODE_DYNAMIC, logits=logits)
        if world > 1:
            dist.all_gather(gathered, logits)

    for _ in range(max(args.warmup, 3)):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
    ms = e0.elapsed_time(e1)
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_per_step = ms / args.steps
    value = world * B * args.steps / (ms / 1e3)
    finite = bool(torch.isfinite(logits).all().item())

    # per-kernel device time of one forward (CUDA events around every launch)
    _, fam = model.forward_profile(images, cal, ob.MODE_DYNAMIC, logits=logits)
    launches_per_fwd = sum(n for _, n in fam.values())
    fp64_peak = ctx.measure_fp64_peak()

    # e2e: the C-ABI call with host buffers (H2D images + forward + D2H logits inside)
    # pinned host buffers (what a serving front end hands the library)
    host_imgs = torch.empty(images.shape, dtype=torch.float64, pin_memory=True)
    host_imgs.copy_(images)
    host_imgs = host_imgs.numpy()
    host_logits = torch.empty((B, dims.classes), dtype=torch.float64, pin_memory=True).numpy()
    for _ in range(max(args.warmup, 3)):  # graph capture of the host-feed path, pinned-page warm-up
        model.forward_host(host_imgs, cal, ob.MODE_DYNAMIC, logits=host_logits)
    n_e2e = max(1, args.steps)
    if world > 1:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(n_e2e):
        model.forward_host(host_imgs, cal, ob.MODE_DYNAMIC, logits=host_logits)
    e2e_s = (time.perf_counter() - t0) / n_e2e
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    e2e_val = world * B / e2e_s

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        try:
            cpu = cpu_baseline(dims, cal.export(), host_imgs, args.abits)
        except Exception as exc:  # reported, never fatal for the GPU number
            cpu = ("error", str(exc))

    if rank == 0:
        L, E, N = dims.tokens, dims.embed, dims.state
        scan_ms, scan_n = fam["k3_scan"]
        # Algorithmic work of one scan launch:
        # S*T*E*N state-element-steps per direction x 28 arithmetic lane-ops (discretize 2,
        # 3 quantizations x 7, update 2, output 2; the exp is not counted).
        # Peak: the measured f64 lane-op rate of this GPU (one DFMA = 1 op).
        ops_per_elem = 28.0
        elem = B * L * E * N * len(model.orders)  # one launch scans every direction
        # one scan op per block (its launches: the step-table prep + the scan kernel)
        achieved = elem * ops_per_elem / (scan_ms / dims.blocks * 1e-3) / 1e12
        peak_ops = fp64_peak / 2.0
        traffic = scan_traffic_bytes()
        cfg = dict(CONFIG, global_batch=B * world, parallelism=f"dp{world}")
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": max(args.warmup, 3), "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "weak", "vs_baseline": None, "dtype": "int8/f64", "data": "synthetic",
                "config": cfg,
                "e2e": {"value": e2e_val, "unit": UNIT, "h2d_bytes_per_step": int(host_imgs.nbytes),
                        "d2h_bytes_per_step": int(host_logits.nbytes)},
                "gpu_launches": int(launches_per_fwd * args.steps),
                "roofline": {"kernel": "k3_scan", "bound": "fp64", "achieved": achieved, "peak": peak_ops,
                             "unit": "Tops (f64 lane-ops/s)", "frac": achieved / peak_ops if peak_ops else None,
                             "traffic": traffic,
                             "traffic_unit": "bytes per launch (ncu dram read+write, profiles/r01/ncu_traffic_r01l.json)",
                             "peak_source": "measured in-process: DFMA probe (1 op per DFMA lane)",
                             "work": f"{ops_per_elem:.0f} f64 lane-ops x S*T*E*N*dirs state-element-steps per launch"},
                "kernels_ms_per_step": {k: v[0] for k, v in fam.items()},
                "kernels_launches_per_step": {k: v[1] for k, v in fam.items()},
                "clocks": clk.summary(), "logits_finite": finite}
        if cpu and cpu[0] != "error":
            line["cpu_baseline"] = {"value": cpu[0], "unit": UNIT, "cores": cpu[1], "kind": "reference",
                                    "sample": cpu[2]}
        elif cpu:
            line["cpu_baseline"] = {"error": cpu[1]}
        print(json.dumps(line))
    if world > 1:
        dist.destroy_process_group()
    return 0


def scan_traffic_bytes():
    """DRAM bytes (read + write) of one k3_scan_fast launch from the committed
    `ncu --set full` capture of this workload, or None."""
    path = os.path.join(os.path.dirname(os.path.abspath(__file__)), "profiles", "r01", "ncu_traffic_r01l.json")
    try:
        with open(path) as f:
            k = json.load(f)["kernels"]
        return [v for n, v in k.items() if n.startswith("k3_scan_fast")][0][0]["traffic_bytes"]
    except Exception:
        return None


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)
    return run_ours(args)


if __name__ == "__main__":
    sys.exit(main())
