#!/usr/bin/env python3
"""Benchmark of the SRWCR value+gradient hot path (arXiv 1804.05061) on B200.

One step = one srwcr_eval: pass 1 + combine + pass 2 over the whole synthetic
workload (every row of SURVEY.md s8(a)), through the C ABI, inputs resident in HBM.

  python bench.py [--gpus N] [--steps K] [--warmup W] [--config C5] [--phi small]
  python bench.py --impl reference ...      (the fp64 CPU oracle as the reference arm)

N > 1 runs under torchrun (one process per GPU): the volume is split into z-slabs
(strong scaling); the library all-reduces the bin statistics and the gradient with
NCCL.  Rank 0 prints ONE JSON line.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "SRWCR value+gradient evals/sec and Gvoxel/s at 1/2/4/8 B200; % of HBM BW"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=10)
    ap.add_argument("--config", default="C5")
    ap.add_argument("--phi", default="small", choices=["zero", "small", "large"])
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-sample-slices", type=int, default=0, help="z-slices of the oracle sample (0 = auto)")
    ap.add_argument("--grad-exchange", default="allreduce", choices=["allreduce", "halo"],
                    help="N > 1: int64 all-reduce of the gradient (every rank gets it all) or the halo "
                         "exchange (each rank gets its owned node layers; srwcr_options.grad_exchange)")
    ap.add_argument("--no-paper-workloads", action="store_true",
                    help="skip the context timings of the paper's Table VIII workloads")
    return ap.parse_args()


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured"
    return 6650.0, "fallback"


def workload_desc(name, cfg):
    nx, ny, nz = cfg["dims"]
    delta = tuple(round(c / s, 4) for c, s in zip(cfg["control_mm"], cfg["spacing"]))
    return f"{name} {cfg['desc']}: {nx}x{ny}x{nz}, {cfg['cells']} spatial cells, {cfg['bins']} bins, control delta {delta} vox"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled DURING the timed region."""

    def __init__(self, gpu_index):
        self.gpu = gpu_index
        self.samples = []
        self.proc = None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.gpu), f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "100"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 6:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        mx = [float(s[1]) for s in self.samples if s[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[2 + i].lower().startswith("active")})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.samples)}


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


def oracle_sample(name, cfg, F, M, params, slices, nthreads=0):
    """Time the fp64 oracle (moment route: pass 1 + combine + pass 2) on z-slab [0, slices)
    of the same workload.  Returns (seconds, sample voxels, threads used)."""
    import oracle as O
    nx, ny, nz = cfg["dims"]
    L = cfg["bins"] - 1
    delta = tuple(c / s for c, s in zip(cfg["control_mm"], cfg["spacing"]))
    pb = O.Problem(dims=cfg["dims"], L=L, delta=delta, kcells=cfg["cells"], nthreads=nthreads)
    Fn, Mn = O.normalize(F, L), O.normalize(M, L)
    t0 = time.perf_counter()
    N, S, Q = O.moments(pb, Fn, Mn, params, 0, slices)
    D, al, be, ga, reg, Z = O.combine(pb, N, S, Q)
    O.grad_moments(pb, Fn, Mn, params, al, be, ga, Z, 0, slices)
    dt = time.perf_counter() - t0
    threads = nthreads if nthreads > 0 else (os.cpu_count() or 1)
    return dt, slices * nx * ny, threads


def auto_slices(cfg):
    # ~10-30 s of host work at ~0.5-1 us per voxel-eval per core
    nx, ny, nz = cfg["dims"]
    cores = os.cpu_count() or 1
    target = 15.0 * cores / 1.0e-6 / 2.0
    return int(max(2, min(nz, target // (nx * ny))))


def run_reference(args):
    import synth
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    cfg = synth.config(args.config)
    F, M = synth.make_pair(args.config, args.seed)
    nx, ny, nz = cfg["dims"]
    import oracle as O
    L = cfg["bins"] - 1
    pb = O.Problem(dims=cfg["dims"], L=L, delta=tuple(c / s for c, s in zip(cfg["control_mm"], cfg["spacing"])),
                   kcells=cfg["cells"])
    params = synth.make_params(pb.params_shape, args.phi, args.seed)
    slices = args.cpu_sample_slices or max(1, auto_slices(cfg) // max(1, args.steps + args.warmup) * 2)
    slices = min(slices, nz)
    for _ in range(args.warmup):
        oracle_sample(args.config, cfg, F, M, params, slices)
    times = []
    for _ in range(args.steps):
        dt, vox, threads = oracle_sample(args.config, cfg, F, M, params, slices)
        times.append(dt)
    T = sum(times)
    nvox = nx * ny * nz
    evals_per_s = args.steps * vox / (T * nvox)
    # a step is the bounded sample (so K steps fit the driver's run); ms_per_step is the time of
    # the work actually done, value the full-volume-equivalent rate of the same metric
    line = {
        "impl": "reference", "metric": METRIC, "value": evals_per_s, "unit": "evals/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": 1e3 * T / args.steps,
        "step_fraction_of_eval": vox / nvox, "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": workload_desc(args.config, cfg), "phi": args.phi, "seed": args.seed},
        "gvoxel_per_s": evals_per_s * nvox / 1e9,
        "cpu_baseline": {"value": evals_per_s, "unit": "evals/s", "cores": threads, "kind": "oracle",
                         "sample": f"z-slab [0,{slices}) of {nz} slices ({vox} voxels) per step, moment route "
                                   f"(pass 1 + combine + pass 2), scaled to the full volume"},
        "e2e": {"value": evals_per_s, "unit": "evals/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# Table VIII: one value+derivative iteration on DIR-Lab CT volumes at three
# sizes, delta = 5 voxels, L = 31 (32 bins), spatial bins = control nodes,
# GTX 1060.  Measured here on C3-shaped synthetic CT of the same sizes, same settings.
PAPER_TABLE_VIII = [((64, 64, 24), 21 + 4), ((128, 128, 49), 132 + 32), ((256, 256, 99), 851 + 238)]


def paper_workloads(device, steps=10):
    import torch
    import paper_1804_05061_b200 as S
    import synth
    out = []
    for dims, paper_ms in PAPER_TABLE_VIII:
        cfg = synth.config("C3", dims)
        F, M = synth.make_pair("C3", 1, dims)
        sp = cfg["spacing"]
        cells = tuple(max(1, int(n // 5)) for n in dims)
        g = S.Srwcr(torch.from_numpy(F).cuda(), torch.from_numpy(M).cuda(), sp, 32, cells, tuple(5.0 * x for x in sp),
                    device=device)
        p = torch.from_numpy(synth.make_params(g.params_shape, "small", 1)).cuda()
        gr = torch.empty_like(p)
        st = torch.cuda.ExternalStream(g.stream_handle())
        for _ in range(3):
            g.eval(p, grad=gr)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(steps):
            g.eval(p, grad=gr)
        e1.record(st)
        e1.synchronize()
        ms = e0.elapsed_time(e1) / steps
        out.append({"dims": list(dims), "bins": 32, "spatial_cells": list(cells), "ms_per_eval": ms,
                    "paper_gtx1060_ms": paper_ms, "speedup_vs_paper": paper_ms / ms})
        g.close()
    return out


def main():
    args = parse()
    if args.impl == "reference":
        return run_reference(args)

    import torch
    import paper_1804_05061_b200 as S
    import synth

    ws, rank, local = dist_env()
    if args.gpus > 1 and ws != args.gpus:
        print(f"--gpus {args.gpus} needs torchrun with {args.gpus} processes (WORLD_SIZE={ws})", file=sys.stderr)
        return 2
    torch.cuda.set_device(local)
    dist = None
    nccl_id = None
    if ws > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        obj = [torch.cuda.nccl.unique_id() if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        nccl_id = obj[0]

    cfg = synth.config(args.config)
    F, M = synth.make_pair(args.config, args.seed)
    nx, ny, nz = cfg["dims"]
    nvox = nx * ny * nz
    Ft = torch.from_numpy(F).cuda()
    Mt = torch.from_numpy(M).cuda()
    g = S.Srwcr(Ft, Mt, cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"], device=local,
                nranks=ws, rank=rank, nccl_id=nccl_id,
                grad_exchange=1 if (ws > 1 and args.grad_exchange == "halo") else 0)
    del Ft, Mt
    params_np = synth.make_params(g.params_shape, args.phi, args.seed)
    params = torch.from_numpy(params_np).cuda()
    grad = torch.empty_like(params)
    stream = torch.cuda.ExternalStream(g.stream_handle())

    # ---- device-resident timing
    g.set_timing(True)
    for _ in range(max(3, args.warmup)):
        g.eval(params, grad=grad)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    l0 = g.stats()["launches_total"]
    p1, p2, cb, pp = [], [], [], []
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        e0.record(stream)
        for _ in range(args.steps):
            D, _ = g.eval(params, grad=grad)
            st = g.stats()
            p1.append(st["ms_pass1"]); p2.append(st["ms_pass2"]); cb.append(st["ms_combine"]); pp.append(st["ms_prep"])
        e1.record(stream)
        e1.synchronize()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches = g.stats()["launches_total"] - l0
    ms = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    evals = 1e3 / ms_step

    # ---- the same step at the worst-gather Phi point (SURVEY 8(d) Phi_large), a short run
    phi_large = None
    if args.phi != "large":
        pl_np = synth.make_params(g.params_shape, "large", args.seed)
        pl = torch.from_numpy(pl_np).cuda()
        for _ in range(3):
            g.eval(pl, grad=grad)
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        nl = max(5, args.steps // 4)
        e0.record(stream)
        for _ in range(nl):
            g.eval(pl, grad=grad)
        e1.record(stream)
        e1.synchronize()
        msl = e0.elapsed_time(e1)
        if dist:
            t = torch.tensor([msl], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            msl = float(t.item())
        st = g.stats()
        phi_large = {"value": nl * 1e3 / msl, "unit": "evals/s", "ms_per_step": msl / nl, "steps": nl,
                     "exact_voxels": st["exact_voxels"]}
        del pl

    # ---- end to end through the public API with pinned HOST buffers (H2D params, D2H D + grad)
    g.set_timing(False)
    hp = torch.from_numpy(params_np.copy()).pin_memory()
    hg = torch.empty_like(hp).pin_memory()
    e_steps = max(10, args.steps // 3)
    for _ in range(3):
        g.eval(hp, grad=hg)
    if dist:
        dist.barrier()
    torch.cuda.synchronize()
    e0.record(stream)
    for _ in range(e_steps):
        g.eval(hp, grad=hg)
    e1.record(stream)
    e1.synchronize()
    ms_e2e = e0.elapsed_time(e1)
    if dist:
        t = torch.tensor([ms_e2e], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms_e2e = float(t.item())
    e2e = e_steps * 1e3 / ms_e2e

    if rank == 0:
        peak, peak_kind = peaks()
        G = int(np.prod(g.grid))
        # algorithmic bytes per launch: F + M once (8 B/voxel) of this rank's
        # slab, params read fp32 (12 B/node), pass 2 also writes the fp64 gradient (24 B/node)
        vox_rank = nvox / ws
        bytes_p1 = 8 * vox_rank + 12 * G
        bytes_p2 = 8 * vox_rank + 12 * G + 24 * G
        t1, t2 = statistics.mean(p1), statistics.mean(p2)
        fast = g.stats()["fast_path"] == 1
        n1, n2 = ("k_p1f", "k_p2f") if fast else ("k_pass1", "k_pass2")
        dom, tdom, bdom = (n1, t1, bytes_p1) if t1 >= t2 else (n2, t2, bytes_p2)
        achieved = bdom / (tdom * 1e-3) / 1e9
        traffic = None
        tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
        if os.path.exists(tp):
            try:
                traffic = json.load(open(tp)).get(args.config, {}).get(dom)
            except Exception:
                traffic = None
        cpu = None
        if not args.no_cpu_baseline and ws == 1:   # the oracle baseline: rank 0 at N = 1 only
            slices = args.cpu_sample_slices or auto_slices(cfg)
            dt, vox, threads = oracle_sample(args.config, cfg, F, M, params_np, slices)
            s1 = max(1, slices // 16)   # single-thread figure on a smaller slab
            dt1, vox1, _ = oracle_sample(args.config, cfg, F, M, params_np, s1, nthreads=1)
            try:
                aff = len(os.sched_getaffinity(0))
            except Exception:
                aff = None
            cpu = {"value": vox / (dt * nvox), "unit": "evals/s", "cores": threads, "kind": "oracle",
                   "cores_affinity": aff, "cpu_count": os.cpu_count(),
                   "single_thread": {"value": vox1 / (dt1 * nvox), "unit": "evals/s", "cores": 1,
                                     "sample": f"z-slab [0,{s1}) ({vox1} voxels) in {dt1:.1f} s"},
                   "sample": f"z-slab [0,{slices}) of {nz} slices ({vox} voxels), fp64 moment route "
                             f"(pass 1 + combine + pass 2) in {dt:.1f} s, scaled to the full volume"}
        line = {
            "metric": METRIC, "value": evals, "unit": "evals/s", "n_gpus": ws, "steps": args.steps,
            "warmup": max(3, args.warmup), "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f32", "data": "synthetic",
            "config": {"workload": workload_desc(args.config, cfg), "phi": args.phi, "seed": args.seed,
                       "parallelism": f"z-slab x{ws}" + (f" ({args.grad_exchange} gradient exchange)" if ws > 1 else ""), "l2": "inputs 671 MB > 126 MB L2 (no flush needed)"
                       if args.config in ("C4", "C5") else "inputs may be L2-resident (no flush)"},
            "gvoxel_per_s": evals * nvox / 1e9,
            "pass_ms": {"prep": statistics.mean(pp), "pass1": t1, "combine": statistics.mean(cb), "pass2": t2},
            "roofline": {"bound": "hbm", "kernel": dom, "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_kind": peak_kind,
                         "bytes_per_launch": bdom, "pass1_frac": bytes_p1 / (t1 * 1e-3) / 1e9 / peak,
                         "pass2_frac": bytes_p2 / (t2 * 1e-3) / 1e9 / peak},
            "cpu_baseline": cpu,
            "e2e": {"value": e2e, "unit": "evals/s", "h2d_bytes_per_step": int(params_np.nbytes),
                    "d2h_bytes_per_step": int(params_np.nbytes) + 8},
            "gpu_launches": int(launches),
            "decomposition": {k: g.stats()[k] for k in ("fast_path", "fast_items", "fast_warps", "fast_slots",
                                                        "warps_per_cta", "slot_capacity", "voxels_per_lane", "items",
                                                        "warps_per_cta2", "items2")},
            "phi_large": phi_large,
            "clocks": clk.summary(),
            "D": D,
            "paper_workloads": None if args.no_paper_workloads or ws > 1 else paper_workloads(local),
        }
        print(json.dumps(line), flush=True)
    g.close()
    if dist:
        dist.destroy_process_group()
    return 0


if __name__ == "__main__":
    sys.exit(main())
