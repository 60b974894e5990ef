#!/usr/bin/env python3
"""Benchmark: H-matrix (H1) compression time on B200 (BASELINE.json metric).

One step = one full ``compress()`` of the workload (all H1 levels + leaf
phase) with the operator and tree already resident (points in HBM, tree on
the host). Default workload: config 3 (N = 262144 starfish curve, on-the-fly
log kernel, quadtree leaf 128, k = 32, p = 10) -- the largest BASELINE config
whose factors fit one GPU; config 4's N = 2^20 is quoted on 8 GPUs.

  python bench.py [--gpus N --steps K --warmup W --config c3 --impl ours|reference]

Prints one JSON line (rank 0). Times: CUDA events on the device around the
synchronous compress call (max over ranks); L2 is flushed (512 MiB write)
before every timed step. ``e2e`` repeats the step through the public API with
host buffers: points H2D, tree build, compress, full factor export D2H.
``--impl reference`` times the reference's CPU path through the oracle
(oracle/cpu_model.py: the restated reference algorithm, per-color dense test
matrices through the black box) without loading the product library: config 1
in full, larger configs as a labelled extrapolation from measured samples
(see DESIGN.md "Measurement").
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

FP64_PEAK_TFLOPS = 37.1   # measured DMMA.8x8x4 peak on this pool's B200 (profiles/r01_fp64_peaks.txt)
FP64_PEAK_SOURCE = ("measured DMMA m8n8k4 peak, profiles/r02_fp64_peaks.txt (37.14 TF/s at 1965 MHz, clock record "
                    "included; MEASURED_PEAKS.json has no FP64 entry)")
METRIC = "H-matrix compression time (s)"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", default="c3")
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--n", type=int, default=0, help="override N (scaled workload)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--full-reference", action="store_true",
                    help="reference arm: compress the whole workload in the oracle (no extrapolation)")
    ap.add_argument("--clock-ms", type=int, default=200, help="nvidia-smi sampling period (0: off)")
    return ap.parse_args()


def dist_setup(args):
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if ws > 1:
        import torch
        import torch.distributed as dist
        if args.impl == "ours":
            torch.cuda.set_device(local)
            dist.init_process_group("nccl")
        else:
            dist.init_process_group("gloo")
    return ws, rank, local


def dist_max(x, ws, impl):
    if ws == 1:
        return x
    import torch
    import torch.distributed as dist
    dev = "cuda" if impl == "ours" else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def barrier(ws):
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()


class ClockSampler:
    """nvidia-smi clocks + throttle reasons during the timed region."""

    def __init__(self, gpu, period_ms=200):
        self.gpu = gpu
        self.period_ms = period_ms
        self.rows = []
        self.proc = None

    def __enter__(self):
        if self.period_ms <= 0:
            return self
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap,power.draw")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                 "-lms", str(self.period_ms)], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4) if r[2 + i].lower() == "active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def make_operator(hp, w, pts, device=0):
    if w.dense:
        # config 1: explicit dense A = log|x_i - x_j| (A_ii = 0) as the black box
        x = pts
        same = np.eye(len(x), dtype=bool)
        diff = x[:, None, :] - x[None, :, :]
        with np.errstate(divide="ignore"):
            a = np.log(np.sqrt(np.sum(diff * diff, axis=2)))
        a[same] = 0.0
        return hp.dense_operator(a, device)
    return hp.kernel_operator(w.kernel, pts, w.param, device)


# DRAM bytes (read + write) of one K2 launch from `ncu --set full` (config 3,
# level 7; profiles/r01_k2_int8_ncu.txt), per launch like `achieved`.
K2_NCU_TRAFFIC = 943549952 + 677325824
K2_NCU_SOURCE = "profiles/r02_k2_int8_ncu.txt: dram__bytes_read.sum + dram__bytes_write.sum of one level launch (config 3)"
INT8_PEAK_TOPS = 4500.0   # B200 dense INT8 tensor peak (datasheet; MEASURED_PEAKS.json has no INT8 entry)


def k2_roofline(report, w):
    """Dominant kernel K2 (black-box apply). achieved = useful FP64 flops of
    the rows read back (2 * rows * payload rows * 2r) / K2 device time,
    against the measured FP64 DMMA peak; the int8 path computes those flops
    exactly as 35 int8 digit-pair products per entry and column (padded to
    16), reported against the INT8 tensor peak in `int8`."""
    flops = sum(ph["apply_flops"] for ph in report["phases"] if ph["phase"] == "h1")
    ms = sum(ph["apply_ms"] for ph in report["phases"] if ph["phase"] == "h1")
    launches = sum(1 for ph in report["phases"] if ph["phase"] == "h1")
    ach = flops / (ms * 1e-3) / 1e12 if ms > 0 else 0.0
    r = w.rank + w.oversample
    np_pad = (r + 15) // 16 * 16
    int8_ops = flops / (4.0 * r) * 35 * 2 * (2 * np_pad)  # 35 digit pairs (a + b <= 7, 8 x 7 planes)
    int8_tops = int8_ops / (ms * 1e-3) / 1e12 if ms > 0 else 0.0
    int8_path = any(ph.get("apply_path") == "int8" for ph in report["phases"] if ph["phase"] == "h1")
    out = {"bound": "tensor", "achieved": round(ach, 3), "peak": FP64_PEAK_TFLOPS, "unit": "TFLOP/s",
           "frac": round(ach / FP64_PEAK_TFLOPS, 4), "traffic": K2_NCU_TRAFFIC, "traffic_source": K2_NCU_SOURCE,
           "kernel": ("sample_apply_i8_kernel (K2, FP64 apply emulated exactly on the int8 tensor cores)"
                      if int8_path else "sample_apply_kernel (K2, FP64 DMMA)"),
           "launches_per_step": launches, "avg_launch_ms": round(ms / max(launches, 1), 3),
           "flops_per_step": flops, "peak_source": FP64_PEAK_SOURCE,
           "achieved_meaning": "FP64-equivalent useful flops / K2 time (K2 event span on the apply stream; "
                               "the previous level's peel/QR/B kernels share the SMs during it)"}
    # the batched reconstruction kernels, same FP64 peak (spans on the main stream)
    others = {}
    for key, fk, tk, what in (("K3_peel", "peel_flops", "peel_ms", "peel_coeff_dmma + peel_apply (all phases)"),
                              ("K4_qr", "qr_flops", "qr_ms", "range finder (staged pivoted Cholesky-QR on DMMA, k_gqr.cu), nominal 2 m r^2 per U / V block"),
                              ("K5_bsolve", "bsolve_flops", "bsolve_ms",
                               "grams + two-kernel B solve (N1^-1 C N2^-1), the reference's flop formulas")):
        f = sum(ph.get(fk, 0.0) for ph in report["phases"])
        t = sum(ph[tk] for ph in report["phases"])
        if t > 0 and f > 0:
            a = f / (t * 1e-3) / 1e12
            others[key] = {"achieved": round(a, 3), "frac": round(a / FP64_PEAK_TFLOPS, 4), "unit": "TFLOP/s",
                           "ms_per_step": round(t, 2), "flops_per_step": f, "kernel": what}
    out["others"] = others
    if int8_path:
        out["int8"] = {"achieved_tops": round(int8_tops, 1), "peak_tops": INT8_PEAK_TOPS,
                       "frac": round(int8_tops / INT8_PEAK_TOPS, 4),
                       "ops_per_step": int8_ops,
                       "peak_source": "B200 datasheet dense INT8 (fallback: no INT8 entry in MEASURED_PEAKS.json)"}
    return out


def flush_l2(torch):
    buf = torch.empty(512 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
    buf.fill_(1.0)
    del buf


def reference_measure(w, steps, warmup, budget_s=10.0, full=False):
    """The reference's CPU path, timed through the oracle (oracle/cpu_model.py):
    never loads libhpeel_b200.so. Config 1 (and any N <= 8192) is compressed
    in full and measured per phase, on all host threads and on one; larger
    workloads are a labelled extrapolation: the black box's per-row cost is
    measured on a row subset of the full workload every step and multiplied
    by the exact column count of the oracle's own plans, and the peel / QR /
    B phases use per-flop rates calibrated on a measured compress of a scaled
    instance (N = 4096) times the full instance's reference flop counts."""
    import oracle as O
    from oracle import cpu_model as M
    threads = os.cpu_count() or 1
    pts = w.points(O)
    if pts.ndim == 1:
        pts = pts[:, None]
    vals, phases = [], None
    if full or w.dense or w.n <= 8192:
        for i in range(warmup + steps):
            total, times, _, _ = M.timed_compress(w, pts, threads)
            if i >= warmup:
                vals.append(total)
                phases = times
        extra = {"kind_of_value": "measured", "phases_s": {k: round(v, 4) for k, v in phases.items()}}
        sample = (f"full oracle compress of the whole workload (N = {w.n}), measured per step on {threads} threads")
        if w.dense or w.n <= 8192:
            one, one_times, _, _ = M.timed_compress(w, pts, 1)
            sample += f"; also measured once on 1 thread ({one:.2f} s)"
            extra["one_core"] = {"value": round(one, 4), "phases_s": {k: round(v, 4) for k, v in one_times.items()}}
        return float(np.median(vals)), threads, sample, extra
    from paper_2205_03406_b200 import configs as cfg
    ws = cfg.scaled(w.name, 4096)
    pts_s = ws.points(O)
    cal = M.calibrate(ws, pts_s, threads)
    tree = O.BoxTree(O.PointCloud(pts), w.leaf)
    adj = O.adjacency(tree)
    counts = M.workload_counts(tree, adj, w.rank, w.oversample)
    r = w.rank + w.oversample
    for i in range(warmup + steps):
        rate, rows = M.apply_rate(w, pts, r, budget_s if i >= warmup else budget_s / 4, threads)
        ph = M.extrapolate(counts, rate, cal)
        if i >= warmup:
            vals.append(ph["total"])
            phases = ph
    rate1, rows1 = M.apply_rate(w, pts, r, budget_s, 1)
    ph1 = M.extrapolate(counts, rate1, cal)
    sample = (f"EXTRAPOLATION (labelled): black-box apply measured each step on {rows} of {w.n} rows of one dense "
              f"test matrix ({threads} threads) x the exact {counts['h1_cols'] + counts['leaf_cols']} columns of the "
              f"oracle's plans; peel/QR/B per-flop rates from a measured oracle compress of the same config at "
              f"N = 4096 ({cal['total_s']:.1f} s), applied to the full instance's reference flop counts (ranks = k)")
    extra = {"kind_of_value": "extrapolated", "phases_s": {k: round(v, 2) for k, v in phases.items()},
             "calibration": {"n": cal["n"], "measured_s": round(cal["total_s"], 3),
                             "phases_s": {k: round(v, 4) for k, v in cal["times"].items()}},
             "columns": {"h1": counts["h1_cols"], "leaf": counts["leaf_cols"], "colors": counts["colors"]},
             "dense_equivalent_flops": M.dense_equivalent_flops(counts),
             "one_core": {"value": round(ph1["total"], 2), "apply_rows_sampled": rows1}}
    return float(np.median(vals)), threads, sample, extra


def run_reference(args, ws, rank):
    import paper_2205_03406_b200.configs as cfg
    if rank != 0:
        return
    w = cfg.CONFIGS[args.config] if not args.n else cfg.scaled(args.config, args.n)
    value, threads, sample, extra = reference_measure(w, args.steps, args.warmup, full=args.full_reference)
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": value * 1e3,
        "higher_is_better": False, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": {"workload": w.name, "n": w.n, "description": w.description},
        "cpu_baseline": {"value": value, "unit": "s", "cores": threads, "kind": "port", "sample": sample, **extra},
        "e2e": {"value": value, "unit": "s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_ours(args, ws, rank, local):
    import torch
    import paper_2205_03406_b200 as hp
    import paper_2205_03406_b200.configs as cfg
    w = cfg.CONFIGS[args.config] if not args.n else cfg.scaled(args.config, args.n)
    torch.cuda.set_device(local)
    pts = w.points()
    tree = hp.build_tree(pts, w.leaf)
    op = make_operator(hp, w, pts, local)
    kw = dict(rank=w.rank, oversample=w.oversample, seed=7)
    if ws > 1:
        # one process per GPU, owner-computes: each rank samples,
        # peels and factors the pairs of its boxes; crossing pairs' factors
        # move point-to-point over NCCL
        import torch.distributed as dist
        uid = [hp.Comm.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(uid, src=0)
        kw["comm"] = hp.Comm(uid[0], rank, ws, local)
    for _ in range(args.warmup):
        rep = hp.compress(op, tree, **kw)
        del rep
    torch.cuda.synchronize()
    times, walls = [], []
    launches0 = hp.launch_count()
    last = None
    with ClockSampler(local, args.clock_ms) as clk:
        for _ in range(args.steps):
            last = rep = None  # the previous representation is released outside the timed region
            flush_l2(torch)
            barrier(ws)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            w0 = time.perf_counter()
            e0.record()
            rep = hp.compress(op, tree, **kw)
            e1.record()
            w1 = time.perf_counter()
            torch.cuda.synchronize()
            times.append(e0.elapsed_time(e1) * 1e-3)
            walls.append((w1 - w0, rep.report["wall_s_total"]))
            last = rep
    launches = hp.launch_count() - launches0
    t_step = dist_max(float(np.mean(times)), ws, "ours")
    report = last.report
    roof = k2_roofline(report, w)
    # K2 timed alone: one more (untimed) compress with the levels serialized,
    # so no peel/QR/B kernel shares the SMs during the K2 events
    last = rep = None
    os.environ["HP_SERIAL_LEVELS"] = "1"
    try:
        rep = hp.compress(op, tree, **kw)
        torch.cuda.synchronize()
        solo = k2_roofline(rep.report, w)
    finally:
        del os.environ["HP_SERIAL_LEVELS"]
    roof["alone"] = {"achieved": solo["achieved"], "frac": solo["frac"], "avg_launch_ms": solo["avg_launch_ms"],
                     "compress_s": round(rep.report["wall_s_total"], 4),
                     "meaning": "one extra compress after the timed steps with HP_SERIAL_LEVELS=1 (levels not "
                                "overlapped): K2 events with no other kernel on the SMs"}
    if "int8" in solo:
        roof["alone"]["int8_frac"] = solo["int8"]["frac"]
    # the same for K3 / K4 / K5: in the timed (overlapped) steps their event
    # spans stretch while the next level's K2 holds the SMs
    for key, v in solo["others"].items():
        if key in roof["others"]:
            roof["others"][key]["alone"] = {"achieved": v["achieved"], "frac": v["frac"], "ms": v["ms_per_step"]}
    last = rep
    # e2e through the public API with host buffers
    e2e = None
    if not args.no_e2e:
        # the caller's result arrays: page-locked host memory, allocated once
        # outside the timed region (as the contract's pinned input buffers)
        nf, nd = hp.export_sizes(tree, w.rank, ws, rank)
        hf = hp.pinned_empty(nf)
        hd = hp.pinned_empty(max(nd, 1))
        host_pts_src = hp.pinned_empty(pts.size).reshape(pts.shape)
        host_pts_src[...] = pts
        etimes, parts = [], []
        n_e2e = max(1, min(args.steps, 3))
        for i in range(1 + n_e2e):  # one untimed warm-up pass (first use of the export path), then n_e2e timed
            barrier(ws)
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            # points from host memory -> tree (host) + operator (H2D) ->
            # compress with every level's factors and the dense blocks
            # streamed D2H into hf / hd as soon as they are final
            t_tree = hp.build_tree(host_pts_src, w.leaf)
            t1 = time.perf_counter()
            o2 = make_operator(hp, w, host_pts_src, local)
            t2 = time.perf_counter()
            r2 = hp.compress(o2, t_tree, **kw, export_to=(hf, hd))
            hp.device_synchronize()
            t3 = time.perf_counter()
            if i > 0:
                etimes.append(t3 - t0)
                parts.append((t1 - t0, t2 - t1, t3 - t2))
            del r2, o2
        d2h = (nf + nd) * 8
        e2e = {"value": dist_max(float(np.mean(etimes)), ws, "ours"), "unit": "s",
               "h2d_bytes_per_step": int(pts.size * 8), "d2h_bytes_per_step": int(d2h),
               "breakdown_s": {"tree_build": round(float(np.mean([p[0] for p in parts])), 4),
                               "operator_h2d": round(float(np.mean([p[1] for p in parts])), 4),
                               "compress_with_export": round(float(np.mean([p[2] for p in parts])), 4)},
               "steps": n_e2e, "warmup": 1,
               "includes": "points from pinned host memory: tree build, operator H2D, compress with every "
                           "factor and dense block streamed D2H into pinned host arrays as levels finish"}
    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        v, threads, sample, extra = reference_measure(w, 1, 0)
        cpu = {"value": v, "unit": "s", "cores": threads, "kind": "port", "sample": sample, **extra}
    if rank != 0:
        return
    phases = [{k: (round(v, 3) if isinstance(v, float) else v) for k, v in ph.items()
               if k in ("phase", "level", "colors", "apply_ms", "peel_ms", "qr_ms", "bsolve_ms", "wall_ms_total",
                        "host_wait_ms", "start_ms", "apply_path")}
              for ph in report["phases"]]
    line = {
        "metric": METRIC, "value": round(t_step, 4), "unit": "s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(t_step * 1e3, 2),
        "higher_is_better": False, "scaling": "strong", "vs_baseline": None,
        "dtype": "f64", "data": "synthetic",
        "config": {"workload": w.name, "n": w.n, "description": w.description, "rank": w.rank,
                   "oversample": w.oversample, "leaf": w.leaf, "parallelism": f"owner-computes x{ws}" if ws > 1 else "single",
                   "l2": "flushed (512 MiB write) before every timed step"},
        "roofline": roof, "e2e": e2e, "cpu_baseline": cpu, "gpu_launches": launches,
        "clocks": clk.summary(),
        "report": {"forward_cols": report["forward_cols"], "adjoint_cols": report["adjoint_cols"],
                   "max_sampling_colors": report["max_sampling_colors"], "net_flops": report["net_flops"],
                   "wall_s_net": round(report["wall_s_net"], 4), "setup_ms": round(report["setup_ms"], 1),
                   "phases": phases},
        "step_times_s": [round(t, 4) for t in times],
        "step_host_wall_s": [[round(a, 4), round(b, 4)] for a, b in walls],
        "storage_doubles": last.storage()["total"],
    }
    print(json.dumps(line), flush=True)


def main():
    args = parse()
    ws, rank, local = dist_setup(args)
    if args.impl == "reference":
        run_reference(args, ws, rank)
    else:
        run_ours(args, ws, rank, local)
    if ws > 1:
        import torch.distributed as dist
        dist.barrier()
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
