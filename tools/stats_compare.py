"""Debug: compare the GPU's static counts N and unshifted moments S, Q (debug dumps)
with the oracle's moment tables, per region/bin, for one config."""
import os, sys, numpy as np
_R = os.path.dirname(os.path.dirname(os.path.abspath(__file__))); sys.path.insert(0, _R); sys.path.insert(0, os.path.join(_R, 'tests'))
import oracle as O
from gpu_common import problem, rel, rel_l2
name = sys.argv[1]; kind = sys.argv[2] if len(sys.argv) > 2 else "small"
g, pb, Fn, Mn, params = problem(name, 1, params_kind=kind)
D, grad = g.eval(params)
N, S, Q = O.moments(pb, Fn, Mn, params)
Do, al, be, ga, reg, Z = O.combine(pb, N, S, Q)
Ng = g.debug_dump("N").reshape(N.shape)
SQd = g.debug_dump("SQ")
SQg = [SQd[:N.size].reshape(N.shape), SQd[N.size:]]
regg = g.debug_dump("regions").reshape(-1, 6)
def rep(nm, a, b):
    d = np.abs(a - b); i = np.unravel_index(np.argmax(d), d.shape)
    print(f"{nm}: max abs err {d.max():.3e} at {i} (gpu {a[i]:.6e} oracle {b[i]:.6e}), rel to max {d.max()/max(np.abs(b).max(),1e-300):.2e}")
rep("N", Ng, N); rep("S", SQg[0], S); rep("Q_r", SQg[1], Q.sum(1))
rep("sigma2", regg[:,1], reg[:,1]); rep("1-CR", regg[:,3], reg[:,3])
print("retained gpu/oracle", int(regg[:,4].sum()), int(reg[:,4].sum()), "Z", regg[0,5], reg[0,5])
print(f"D gpu {D:.12f} oracle {Do:.12f} rel {rel(D,Do):.2e}")
