"""Round-2 fast passes vs the round-1 passes (SRWCR_NOFAST) and the fp64 oracle, with
per-pass device times.  Usage: python tools/fast_check.py [C5 C4 ...] (GPU box)."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np

import oracle as O
import paper_1804_05061_b200 as S
import synth

CASES = {
    "C2": None, "C3": None, "C4": None, "C5": None,
    "C3r": ("C3", (256, 66, 34)), "C4r": ("C4", (512, 34, 130)), "C5r": ("C5", (512, 66, 42)),
}


def run(name, phi="small", seed=1, oracle=False, reps=5):
    base, dims = CASES[name] if CASES[name] else (name, None)
    cfg = synth.config(base, dims)
    F, M = synth.make_pair(base, seed, cfg["dims"])
    out = {}
    for fast in (True, False):
        if fast:
            os.environ.pop("SRWCR_NOFAST", None)
        else:
            os.environ["SRWCR_NOFAST"] = "1"
        g = S.Srwcr(F, M, cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"])
        params = synth.make_params(g.params_shape, phi, seed)
        g.set_timing(True)
        D, grad = g.eval(params)
        D2, grad2 = g.eval(params)
        ts = []
        for _ in range(reps):
            g.eval(params)
            st = g.stats()
            ts.append((st["ms_prep"], st["ms_pass1"], st["ms_combine"], st["ms_pass2"], st["ms_total"]))
        st = g.stats()
        t = np.median(np.array(ts), axis=0)
        out[fast] = (D, grad, st)
        print(f"{name} {phi} fast={st['fast_path']} items={st['fast_items'] if fast else st['items']} W={st['fast_warps']}"
              f" S={st['fast_slots']} prep {t[0]:.3f} p1 {t[1]:.3f} comb {t[2]:.3f} p2 {t[3]:.3f} total {t[4]:.3f} ms;"
              f" repeat bitwise D={D == D2} grad={np.array_equal(grad, grad2)} exact={st['exact_voxels']}", flush=True)
        g.close()
    (Df, gf, _), (Ds, gs, _) = out[True], out[False]
    print(f"   fast vs round-1: D rel {abs(Df - Ds) / abs(Ds):.3e}  grad relL2 {np.linalg.norm(gf - gs) / np.linalg.norm(gs):.3e}")
    if oracle:
        L = cfg["bins"] - 1
        pb = O.Problem(dims=cfg["dims"], L=L, delta=tuple(c / s for c, s in zip(cfg["control_mm"], cfg["spacing"])),
                       kcells=cfg["cells"])
        t0 = time.time()
        Do, go = O.eval_moments(pb, O.normalize(F, L), O.normalize(M, L), params) if hasattr(O, "eval_moments") else \
            O.eval_literal(pb, O.normalize(F, L), O.normalize(M, L), params)
        print(f"   oracle ({time.time() - t0:.1f}s): fast D rel {abs(Df - Do) / abs(Do):.3e} grad relL2 "
              f"{np.linalg.norm(gf - go) / np.linalg.norm(go):.3e} max|dg|/max|g| {np.abs(gf - go).max() / np.abs(go).max():.3e};"
              f" round-1 D rel {abs(Ds - Do) / abs(Do):.3e} grad {np.linalg.norm(gs - go) / np.linalg.norm(go):.3e}", flush=True)


if __name__ == "__main__":
    names = sys.argv[1:] or ["C5r", "C4r", "C3r", "C2", "C5"]
    for nm in names:
        orc = nm.endswith("r") or nm == "C2"
        for phi in ("small", "zero", "large"):
            try:
                run(nm, phi, oracle=orc)
            except Exception as e:  # report and continue
                print(f"{nm} {phi}: ERROR {type(e).__name__}: {e}", flush=True)
