"""Run srwcr_register on a synthetic config and print the report (+ wall time)."""
import json
import sys
import time

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__import__("os").path.dirname(__import__("os").path.abspath(__file__))))
import synth  # noqa: E402
import paper_1804_05061_b200 as S  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 30
w_p = float(sys.argv[3]) if len(sys.argv) > 3 else 0.1
cfg = synth.config(name)
F, M = synth.make_pair(name, 1, cfg["dims"])
g = S.Srwcr(F, M, cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"])
g.eval(np.zeros(g.params_shape))
t = time.perf_counter()
x, rep = g.register(None, w_p=w_p, max_iter=iters, verbose=1)
dt = time.perf_counter() - t
rep.update(wall_s=dt, ms_per_eval=1e3 * dt / max(rep["evaluations"], 1), config=name,
           mean_abs_u=float(np.abs(x).mean()), max_abs_u=float(np.abs(x).max()))
print(json.dumps(rep))
