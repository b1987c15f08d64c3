"""Per-rank device time of the z-slab decomposition, measured on ONE GPU by running each
rank's kernels in turn (caller-driven exchange mode, exchange skipped: timing only).
max over ranks of (prep + pass 1 + combine + pass 2) estimates the N-GPU eval time
without the two all-reduces (stats 2.7 MB, gradient 18 MB on C5)."""
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
        g.close()
    worst = max(x["ms_total"] for x in per)
    base = base or worst
    print(json.dumps({"P": P, "max_rank_ms": worst, "max_p1": max(x["ms_pass1"] for x in per),
                      "max_p2": max(x["ms_pass2"] for x in per), "speedup_vs_1": base / worst,
                      "ranks": [{k: round(v, 3) for k, v in x.items()} for x in per]}))
