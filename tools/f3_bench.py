"""Fine spatial lattice (F3, spatial bins = control cells) at a full config: eval time."""
import os, sys, time, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_1804_05061_b200 as S
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
bins = int(sys.argv[2]) if len(sys.argv) > 2 else 0
cfg = synth.config(name)
F, M = synth.make_pair(name, 1, cfg["dims"])
delta = [c / s for c, s in zip(cfg["control_mm"], cfg["spacing"])]
cells = tuple(int(n // d) for n, d in zip(cfg["dims"], delta))
nb = bins or cfg["bins"]
t = time.perf_counter()
g = S.Srwcr(torch.from_numpy(F).cuda(), torch.from_numpy(M).cuda(), cfg["spacing"], nb, cells, cfg["control_mm"])
tc = time.perf_counter() - t
p = torch.from_numpy(synth.make_params(g.params_shape, "small", 1)).cuda()
gr = torch.empty_like(p)
g.set_timing(True)
for _ in range(3): g.eval(p, grad=gr)
ts = []
for _ in range(10):
    g.eval(p, grad=gr); ts.append(g.stats())
med = lambda k: float(np.median([s[k] for s in ts]))
print(json.dumps({"cfg": name, "bins": nb, "cells": cells, "create_s": tc, "pass1": med("ms_pass1"), "pass2": med("ms_pass2"),
                  "combine": med("ms_combine"), "total": med("ms_total"), "items": ts[-1]["items"], "items2": ts[-1]["items2"],
                  "slots": ts[-1]["slot_capacity"], "W": ts[-1]["warps_per_cta"], "XV": ts[-1]["voxels_per_lane"]}))
