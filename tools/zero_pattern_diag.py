"""Where the static counts N of the GPU and the oracle differ in their zero pattern."""
import os, sys
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT); sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np
import oracle as O
from gpu_common import problem
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
g, pb, Fn, Mn, params = problem(name, 1)
print("fast", g.stats()["fast_path"], "MC items", g.stats()["items"])
N, _, _ = O.moments(pb, Fn, Mn, params)
Ng = g.debug_dump("N").reshape(N.shape)
bad = np.argwhere((Ng != 0) != (N != 0))
print("mismatches", len(bad))
for r, a in bad[:20]:
    print(r, a, "gpu", Ng[r, a], "oracle", N[r, a])
print("max rel", np.abs(Ng - N).max() / N.max())
