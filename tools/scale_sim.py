"""Per-rank device time of the z-slab decomposition, measured on ONE GPU by running each
rank's kernels in turn (caller-driven exchange mode, exchange skipped: timing only).
max over ranks of (prep + pass 1 + combine + pass 2) estimates the N-GPU eval time
without the exchanges; the exchanges are then added from a stated MODEL (not measured:
every box here has one GPU): a collective costs LAT + bytes / BW, an all-reduce moving
2 (P - 1) / P of its buffer, the halo one neighbour transfer of the rank's boundary layers
(srwcr_plan_layers).  LAT = 10 us, BW = 700 GB/s (NVLink 5: 900 GB/s per direction)."""
import json, os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import synth
import paper_1804_05061_b200 as S

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
PS = [int(x) for x in sys.argv[2].split(",")] if len(sys.argv) > 2 else [1, 2, 4, 8]
cfg = synth.config(name)
F, M = synth.make_pair(name, 1, cfg["dims"])
Fd, Md = torch.from_numpy(F).cuda(), torch.from_numpy(M).cuda()
base = None
for P in PS:
    per = []
    halo_layers, g_stats_count = 0, 0
    for r in range(P):
        g = S.Srwcr(Fd, Md, cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"], nranks=P, rank=r)
        p = torch.from_numpy(synth.make_params(g.params_shape, "small", 1)).cuda()
        gr = torch.empty_like(p)
        g.set_timing(True)
        ts = []
        for i in range(12):
            g.eval_begin(p)
            g.eval_end(grad=gr)
            if i >= 2:
                ts.append(g.stats())
        med = {k: float(np.median([t[k] for t in ts])) for k in ("ms_prep", "ms_pass1", "ms_combine", "ms_pass2", "ms_total")}
        med["items"], med["items2"] = ts[-1]["items"], ts[-1]["items2"]
        med["fast_items"] = ts[-1]["fast_items"]
        per.append(med)
        t0, t1, o0, o1, r1 = g.grad_layers()
        halo_layers = max(halo_layers, max(0, t1 - o1))
        _, nst_ = g.stats_buffer()
        g_stats_count = nst_
        nparams = int(np.prod(g.params_shape))
        ndim, plane = g.params_shape[0], g.params_shape[2] * g.params_shape[3]
        g.close()
    worst = max(x["ms_total"] for x in per)
    base = base or worst
    LAT, BW = 0.010, 700e9 / 1e3   # ms, bytes per ms
    nst = 8 * g_stats_count   # int64 statistics
    ar = lambda b: 0.0 if P == 1 else LAT + b * 2 * (P - 1) / P / BW
    halo_b = 8 * halo_layers * plane * ndim
    ex_ar = ar(nst) + ar(8 * nparams)
    ex_halo = ar(nst) + (0.0 if P == 1 else LAT + halo_b / BW)
    print(json.dumps({"P": P, "fitems_mul": os.environ.get("SRWCR_FITEMS_MUL", "1"), "max_rank_ms": worst,
                      "max_p1": max(x["ms_pass1"] for x in per),
                      "max_p2": max(x["ms_pass2"] for x in per), "speedup_vs_1": base / worst,
                      "model_ms_allreduce": worst + ex_ar, "model_ms_halo": worst + ex_halo,
                      "model_speedup_allreduce": base / (worst + ex_ar), "model_speedup_halo": base / (worst + ex_halo),
                      "halo_bytes_per_rank": halo_b,
                      "ranks": [{k: round(v, 3) for k, v in x.items()} for x in per]}))
