"""Statistics of pass 1 (fast vs round-1 passes) against the oracle's moments: where a D
difference comes from.  Usage: python tools/stats_check.py [C5r] [phi]  (GPU box)."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np
import oracle as O
import paper_1804_05061_b200 as S
import synth

CASES = {"C3r": ("C3", (256, 66, 34)), "C4r": ("C4", (512, 34, 130)), "C5r": ("C5", (512, 66, 42))}
name = sys.argv[1] if len(sys.argv) > 1 else "C5r"
phi = sys.argv[2] if len(sys.argv) > 2 else "small"
base, dims = CASES[name]
cfg = synth.config(base, dims)
F, M = synth.make_pair(base, 1, cfg["dims"])
L = cfg["bins"] - 1
pb = O.Problem(dims=cfg["dims"], L=L, delta=tuple(c / s for c, s in zip(cfg["control_mm"], cfg["spacing"])),
               kcells=cfg["cells"])
params = synth.make_params(pb.params_shape, phi, 1)
N, Sx, Q = O.moments(pb, O.normalize(F, L), O.normalize(M, L), params)
R, B = Sx.shape
Qr = Q.sum(axis=1)
for fast in ([True] if os.environ.get("FAST_ONLY") else [True, False]):
    if fast: os.environ.pop("SRWCR_NOFAST", None)
    else: os.environ["SRWCR_NOFAST"] = "1"
    g = S.Srwcr(F, M, cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"])
    D, _ = g.eval(params, want_grad=False)
    d = g.debug_dump("SQ")
    Sg, Qg = d[:R * B].reshape(R, B), d[R * B:R * B + R]
    Ng = g.debug_dump("N").reshape(R, B)
    dS = np.abs(Sg - Sx)
    print(f"{name} {phi} fast={g.stats()['fast_path']}: D={D:.10f}  N max rel {np.abs(Ng - N).max() / np.abs(N).max():.2e}  "
          f"S maxabs {dS.max():.3e} (max|S| {np.abs(Sx).max():.3e}, sum|dS| {dS.sum():.3e})  "
          f"Q max rel {np.abs(Qg - Qr).max() / np.abs(Qr).max():.2e}  Q sum|dQ|/sum|Q| {np.abs(Qg - Qr).sum() / np.abs(Qr).sum():.2e}")
    i = np.unravel_index(np.argmax(dS), dS.shape)
    print(f"   worst S at r={i[0]} a={i[1]}: gpu {Sg[i]:.8f} oracle {Sx[i]:.8f} N {N[i]:.3f}")
    j = np.argmax(np.abs(Qg - Qr))
    print(f"   worst Q at r={j}: gpu {Qg[j]:.6f} oracle {Qr[j]:.6f}")
    # D from mixtures of GPU and oracle statistics (which statistic carries the D error)
    def Dof(Nx, Sx_, Qx):
        Qb = np.zeros((R, B)); Qb[:, 0] = Qx
        return O.combine(pb, Nx, Sx_, Qb)[0]
    Do_ = Dof(N, Sx, Qr)
    for lab, args in (("all gpu", (Ng, Sg, Qg)), ("gpu S", (N, Sg, Qr)), ("gpu Q", (N, Sx, Qg)), ("gpu N", (Ng, Sx, Qr))):
        print(f"   D rel err with {lab:8s}: {abs(Dof(*args) - Do_) / abs(Do_):.3e}")
    # where the signed S error sits: per bin (sum over regions) and its correlation with N
    dSs = Sg - Sx
    pb_ = np.abs(dSs.sum(axis=0))
    top = np.argsort(-pb_)[:5]
    print("   top |sum_r dS| bins:", ", ".join(f"a={a}:{dSs[:, a].sum():+.3e} (N {N[:, a].sum():.0f})" for a in top))
    print(f"   sum dS {dSs.sum():+.4e}  sum dS/N-weighted corr {np.corrcoef(dSs.ravel(), N.ravel())[0, 1]:+.3f}")
    g.close()
Do, _ = O.eval_moments(pb, O.normalize(F, L), O.normalize(M, L), params, want_grad=False)
print(f"oracle D={Do:.10f}")
