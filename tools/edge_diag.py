"""Diagnose an edge-case parity failure of the fast passes: errors per Phi point, fast vs
round-1 passes, and where (node layer, component) the gradient error sits.
usage: python tools/edge_diag.py NX NY NZ CX CY CZ"""
import os, sys
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import oracle as O
import paper_1804_05061_b200 as S
import synth

nx, ny, nz, cx, cy, cz = (int(a) for a in sys.argv[1:7])
dims, cells = (nx, ny, nz), (cx, cy, cz)
cfg = synth.config("C5", dims)
F, M = synth.make_pair("C5", 2, dims)
L = 63
pb = O.Problem(dims=dims, L=L, delta=(5.0, 5.0, 5.0), kcells=cells)
Fn, Mn = O.normalize(F, L), O.normalize(M, L)
for phi in ("zero", "small", "large"):
    for nofast in ("0", "1"):
        if nofast == "1":
            os.environ["SRWCR_NOFAST"] = "1"
        else:
            os.environ.pop("SRWCR_NOFAST", None)
        g = S.Srwcr(F, M, (1.0, 1.0, 1.0), 64, cells, (5.0, 5.0, 5.0))
        params = synth.make_params(g.params_shape, phi, 2)
        st = g.stats()
        D, grad = g.eval(params)
        g.close()
        Do, go = O.eval_moments(pb, Fn, Mn, params)
        err = np.abs(grad - go)
        rg = np.linalg.norm(grad - go) / np.linalg.norm(go)
        print(f"phi {phi:5s} fast={st['fast_path']} XV={st['voxels_per_lane']} D rel {abs(D-Do)/abs(Do):.2e} grad relL2 {rg:.2e}")
        if rg > 1e-4:
            e = err.reshape(go.shape)
            for c in range(e.shape[0]):
                lay = e[c].max(axis=(1, 2))
                print("  comp", c, "max err per z-layer", np.round(lay / np.abs(go).max(), 4))
            idx = np.unravel_index(np.argmax(e), e.shape)
            print("  worst", idx, grad.reshape(go.shape)[idx], go[idx])
            ey = e.max(axis=(0, 1, 3)); ex = e.max(axis=(0, 1, 2))
            print("  per y", np.round(ey / np.abs(go).max(), 3)); print("  per x", np.round(ex / np.abs(go).max(), 3))
