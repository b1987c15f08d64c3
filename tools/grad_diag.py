"""Debug: where does the GPU-vs-oracle gradient error concentrate?"""
import os, sys, numpy as np
_R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, _R); sys.path.insert(0, os.path.join(_R, 'tests'))
import oracle as O
from gpu_common import problem, rel_l2
name, kind = sys.argv[1], sys.argv[2]
g, pb, Fn, Mn, params = problem(name, 1, params_kind=kind)
D, grad = g.eval(params)
Do, go = O.eval_moments(pb, Fn, Mn, params)
err = (grad - go).ravel()
o = np.argsort(-np.abs(err))
tot = np.linalg.norm(err)
print(f"{name} {kind}: rel L2 {rel_l2(grad, go):.3e}, |g| {np.linalg.norm(go):.3e}, |err| {tot:.3e}")
for k in (1, 10, 100, 1000):
    print(f"  top {k:5d} comps hold {np.linalg.norm(err[o[:k]])/tot:.3f} of the error norm")
for i in o[:8]:
    print("  ", np.unravel_index(i, grad.shape), f"gpu {grad.ravel()[i]:+.4e} oracle {go.ravel()[i]:+.4e}")
# the same with the oracle's own fp32-rounded params (isolates param rounding)
p32 = params.astype(np.float32).astype(np.float64)
Do2, go2 = O.eval_moments(pb, Fn, Mn, p32)
print(f"  oracle(params rounded to fp32) vs oracle: rel L2 {rel_l2(go2, go):.3e};  gpu vs that: {rel_l2(grad, go2):.3e}")
