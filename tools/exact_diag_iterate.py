"""Save C5 (F, M) and an early L-BFGS iterate for tools/exact_diag.py (on the GPU box)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_1804_05061_b200 as S
cfg = synth.config("C5")
F, M = synth.make_pair("C5", 1, cfg["dims"])
np.savez("/tmp/srwcr_C5.npz", F=F, M=M)
g = S.Srwcr(torch.from_numpy(F).cuda(), torch.from_numpy(M).cuda(), cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"])
x, rep = g.register(None, w_p=0.1, max_iter=int(sys.argv[1]) if len(sys.argv) > 1 else 2)
np.save("/tmp/srwcr_C5_reg.npy", x)
g.eval(x); print("exact", g.stats()["exact_voxels"])
