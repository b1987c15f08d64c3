"""Shared helpers of the GPU parity tests: build problems from the seeded generators,
run the CUDA path through the C ABI (paper_1804_05061_b200) and the oracle on the
same inputs.  The oracle only ever sees the synthetic inputs (never GPU outputs)."""
import numpy as np

import oracle as O
import synth
import paper_1804_05061_b200 as S

# reduced dims of the big configs: oracle in seconds, still many tiles + ragged tails
REDUCED = {
    "C1": (64, 64, 1),
    "C2": (128, 128, 128),
    "C3": (70, 66, 34),
    "C4": (130, 34, 258),
    "C5": (130, 126, 82),
}


def problem(name, seed=1, dims=None, params_kind="small", pseed=None, orientation=0, bins=None):
    """(gpu Srwcr, oracle Problem, Fn, Mn, params) for a config at the given dims."""
    cfg = synth.config(name, dims if dims is not None else REDUCED[name])
    F, M = synth.make_pair(name, seed, cfg["dims"])
    nb = bins if bins is not None else cfg["bins"]
    L = nb - 1
    delta = tuple(c / s for c, s in zip(cfg["control_mm"], cfg["spacing"]))
    pb = O.Problem(dims=cfg["dims"], L=L, delta=delta, kcells=cfg["cells"], orientation=orientation)
    g = S.Srwcr(F, M, cfg["spacing"], nb, cfg["cells"], cfg["control_mm"], orientation=orientation)
    assert g.params_shape == pb.params_shape, (g.params_shape, pb.params_shape)
    params = synth.make_params(pb.params_shape, params_kind, seed if pseed is None else pseed)
    Fn, Mn = O.normalize(F, L), O.normalize(M, L)
    return g, pb, Fn, Mn, params


def rel(a, b):
    return abs(a - b) / max(abs(b), 1e-300)


def rel_l2(a, b):
    return float(np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300))


G_COMP = 1e-3   # per-component gradient bound: max |g - g_o| <= 1e-3 max |g_o|


def comp(a, b):
    """max-norm gradient error relative to the oracle gradient's max (catches a localised
    error on boundary / halo nodes that a relative L2 can hide)."""
    a, b = np.asarray(a), np.asarray(b)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))
