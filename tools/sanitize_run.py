"""Small end-to-end run of every kernel family for compute-sanitizer (memcheck, racecheck,
synccheck): both orientations, the round-1 passes (2-D, multi-cell), the fast passes (XV 1
and 2, split and fused pass 1), the exact-path fix, bending energy, two L-BFGS iterations
and the field utilities.  Sizes are tiny so the instrumented run finishes in minutes.
usage: compute-sanitizer --tool TOOL python tools/sanitize_run.py"""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1804_05061_b200 as S  # noqa: E402
import synth  # noqa: E402

CASES = [
    # (name, dims, cells, orientation, label)
    ("C1", (64, 64, 1), None, 0, "2-D, orientation 0"),
    ("C1", (64, 64, 1), None, 1, "2-D, orientation 1"),
    ("C2", (40, 36, 30), None, 0, "3-D multi-cell items, orientation 0"),
    ("C2", (40, 36, 30), None, 1, "3-D, orientation 1"),
    ("C3", (64, 20, 12), (2, 2, 2), 0, "fast passes XV 1"),
    ("C5", (128, 20, 12), (2, 2, 2), 0, "fast passes XV 2"),
]


def run(name, dims, cells, ori, label, split=None):
    cfg = synth.config(name, dims)
    F, M = synth.make_pair(name, 1, cfg["dims"])
    g = S.Srwcr(F, M, cfg["spacing"], cfg["bins"], cells or cfg["cells"], cfg["control_mm"], orientation=ori)
    st = g.stats()
    for kind in ("small", "large"):
        p = synth.make_params(g.params_shape, kind, 1)
        D, grad = g.eval(p)
        assert np.isfinite(D) and np.all(np.isfinite(grad))
    E, _ = g.bending(p)
    x, rep = g.register(None, max_iter=2)
    g.field(x)
    g.close()
    print(f"{label:40s} fast={st['fast_path']} D={D:.6f} C_p={E:.3e} register it={rep['iterations']}", flush=True)


for c in CASES:
    run(*c)
os.environ["SRWCR_SPLIT"] = "1"
run("C5", (128, 20, 12), (2, 2, 2), 0, "fast passes XV 2, split pass 1")
print("sanitize_run: ok")
