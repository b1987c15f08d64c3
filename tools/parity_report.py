"""Measured parity of the CUDA path against the fp64 oracle (the numbers behind the
tests' pass/fail gates) -> one JSON document (profiles/r2_*_parity.json), with the kernel
variant each case ran and the dynamic bin-assignment mismatch counts."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tests"))
import numpy as np
import oracle as O
import synth
import paper_1804_05061_b200 as S
from gpu_common import REDUCED, problem, rel, rel_l2

out = []
def rec(tag, g, pb, Fn, Mn, params, literal=False):
    t = time.perf_counter()
    D, grad = g.eval(params)
    st = g.stats()
    # dynamic assignments: the moving bin n(m) = min(floor m, L-1) of the fp32
    # sample against the oracle's fp64 warp (the exact-path flag is undone first)
    mism = None
    try:
        mg = g.debug_dump("warped").reshape(pb.dims[2], pb.dims[1], pb.dims[0], 4)
        m_g = np.where(mg[..., 0] < 0, -1.0 - mg[..., 0], mg[..., 0])
        del mg
        m_o, _ = O.warp(pb, Mn, params)
        n_g = np.minimum(np.floor(m_g), pb.L - 1)
        n_o = np.minimum(np.floor(m_o), pb.L - 1)
        bad = n_g != n_o
        near = np.abs(m_o - np.round(m_o)) < 1e-4
        mism = {"bin_mismatches": int(bad.sum()), "voxels": int(bad.size),
                "mismatches_not_next_to_an_integer": int((bad & ~near).sum()),
                "max_abs_m_err": float(np.abs(m_g - m_o).max())}
    except Exception as ex:   # (2-D volumes etc.)
        mism = {"unavailable": str(ex)[:80]}
    g.close()
    Do, go = (O.eval_literal if literal else O.eval_moments)(pb, Fn, Mn, params)
    e = {"case": tag, "dims": list(pb.dims), "bins": pb.L + 1, "D": D, "D_oracle": Do, "D_rel": rel(D, Do),
         "grad_rel_l2": rel_l2(grad, go) if np.linalg.norm(go) > 0 else 0.0,
         "grad_max_err_over_max": float(np.abs(grad - go).max() / max(np.abs(go).max(), 1e-300)),
         "exact_voxels": st["exact_voxels"], "fast_path": st["fast_path"], "voxels_per_lane": st["voxels_per_lane"],
         "dynamic_bins": mism, "seconds": time.perf_counter() - t}
    out.append(e)
    print(json.dumps(e), flush=True)

for name in ["C1", "C2", "C3", "C4", "C5"]:
    for kind in ["zero", "small", "large"]:
        rec(f"{name} reduced {kind}", *problem(name, 1, params_kind=kind), literal=name == "C1")
for name in ["C1", "C3", "C4"]:
    rec(f"{name} reduced small orientation 1", *problem(name, 1, params_kind="small", orientation=1))
rec("C5 reduced small orientation 1 (64 bins)", *problem("C5", 1, params_kind="small", orientation=1, bins=64))
# the fast passes at the stand-in sizes of tests/test_gpu_fast.py (same kernel variant as full size)
FAST = {"C3": (256, 66, 34), "C4": (512, 34, 130), "C5": (512, 66, 42)}
for name, dims in FAST.items():
    for seed in (1, 2, 3):
        for kind in (["zero", "small", "large"] if seed == 1 else ["small"]):
            rec(f"{name} fast stand-in {dims} seed {seed} {kind}", *problem(name, seed, dims=dims, params_kind=kind))
for name in ("C3", "C4", "C5"):
    cfg = synth.config(name)
    for kind in ("zero", "small", "large"):
        rec(f"{name} FULL {kind}", *problem(name, 1, dims=cfg["dims"], params_kind=kind))
rec("C5 reduced small orientation 1 (128 bins)", *problem("C5", 1, params_kind="small", orientation=1, bins=128))
for dims in [(64, 64, 24), (128, 128, 49), (256, 256, 99)]:
    cfg = synth.config("C3", dims)
    F, M = synth.make_pair("C3", 1, dims)
    cells = tuple(max(1, int(n // 5)) for n in dims)
    g = S.Srwcr(F, M, cfg["spacing"], 32, cells, tuple(5.0 * x for x in cfg["spacing"]))
    pb = O.Problem(dims=dims, L=31, delta=(5.0, 5.0, 5.0), kcells=cells)
    params = synth.make_params(pb.params_shape, "small", 1)
    rec(f"Table VIII {dims} fine lattice", g, pb, O.normalize(F, 31), O.normalize(M, 31), params)
json.dump({"gates": {"D_rel": 1e-5, "grad_rel_l2": 1e-4}, "cases": out}, open(sys.argv[1] if len(sys.argv) > 1 else "parity.json", "w"), indent=1)
