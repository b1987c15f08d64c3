import os
import sys, time, numpy as np
_R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, _R); sys.path.insert(0, os.path.join(_R, 'tests'))
import oracle as O
from gpu_common import problem, rel, rel_l2
for name in sys.argv[1:]:
    for kind in ("zero", "small", "large"):
        t = time.time()
        g, pb, Fn, Mn, params = problem(name, 1, params_kind=kind)
        t1 = time.time()
        D, grad = g.eval(params)
        t2 = time.time()
        Do, go = O.eval_moments(pb, Fn, Mn, params)
        t3 = time.time()
        print(f"{name} {kind}: D={D:.10f} Do={Do:.10f} relD={rel(D,Do):.2e} relG={rel_l2(grad,go):.2e} |g|={np.linalg.norm(go):.3e} create={t1-t:.1f}s gpu={t2-t1:.3f}s oracle={t3-t2:.1f}s", flush=True)
        g.close()
