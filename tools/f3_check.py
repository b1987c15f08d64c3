"""Fine spatial lattice (spatial bins = control nodes) on a reduced
CT-like volume: GPU vs oracle, and the eval time against the coarse 8^3 lattice."""
import os, sys, time, json
_R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, _R); sys.path.insert(0, os.path.join(_R, 'tests'))
import numpy as np
import oracle as O, synth, paper_1804_05061_b200 as S
from gpu_common import rel, rel_l2
dims = (70, 66, 34)
cfg = synth.config("C3", dims)
F, M = synth.make_pair("C3", 1, dims)
L = cfg["bins"] - 1
delta = tuple(c / s for c, s in zip(cfg["control_mm"], cfg["spacing"]))
for cells in [cfg["cells"], tuple(int(n // d) for n, d in zip(dims, delta))]:
    pb = O.Problem(dims=dims, L=L, delta=delta, kcells=cells)
    g = S.Srwcr(F, M, cfg["spacing"], cfg["bins"], cells, cfg["control_mm"])
    p = synth.make_params(g.params_shape, "small", 1)
    D, gr = g.eval(p)
    t = time.perf_counter()
    for _ in range(10): g.eval(p)
    dt = (time.perf_counter() - t) / 10
    Fn, Mn = O.normalize(F, L), O.normalize(M, L)
    Do, go = O.eval_moments(pb, Fn, Mn, p)
    print(json.dumps({"cells": cells, "regions": pb.nregions, "relD": rel(D, Do), "relG": rel_l2(gr, go),
                      "ms_per_eval_wall": 1e3 * dt, "items": g.stats()["items"], "slots": g.stats()["slot_capacity"]}))
    g.close()
