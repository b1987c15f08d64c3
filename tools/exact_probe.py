"""Deferred exact-path voxels at L-BFGS iterates (C5): count per evaluation."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_1804_05061_b200 as S
cfg = synth.config("C5")
F, M = synth.make_pair("C5", 1, cfg["dims"])
g = S.Srwcr(torch.from_numpy(F).cuda(), torch.from_numpy(M).cuda(), cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"])
out = []
for it in (1, 2, 5, 10):
    x, rep = g.register(None, w_p=0.1, max_iter=it)
    g.set_timing(True)
    D, gr = g.eval(x)
    st = g.stats()
    g.set_timing(False)
    nz = float((x != 0).mean())
    out.append({"iters": it, "exact_voxels": st["exact_voxels"], "cap": st["exact_capacity"], "ms_pass2": st["ms_pass2"],
                "nonzero_param_frac": nz, "max_abs": float(np.abs(x).max())})
    print(json.dumps(out[-1]), flush=True)
