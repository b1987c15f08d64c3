"""GPU parity at BASELINE.json's full sizes, in the configuration bench.py times.

bench.py's N=1 workload is C5 (512 x 512 x 320, 128 bins, 8^3 spatial cells) with the
"small" seed-1 parameters, on device tensors; its paper_workloads leg runs the Table
VIII shapes (fine spatial lattice at delta 5, 32 bins).  The oracle's moment
route finishes one full C5 evaluation in seconds on the host cores, so these compare the
WHOLE outputs (D and every gradient component), not samples, at the gates of
BASELINE.json: D relative error <= 1e-5, gradient relative L2 <= 1e-4.  The per-component
check adds a max-norm bound on the gradient error, scaled by the gradient's max.
"""
import numpy as np
import pytest

import oracle as O
import synth
from gpu_common import problem, rel, rel_l2, comp, G_COMP

pytestmark = pytest.mark.gpu

D_TOL = 1e-5
G_TOL = 1e-4


def _device_eval(g, params):
    """The call bench.py times: device params and gradient buffers."""
    torch = pytest.importorskip("torch")
    p = torch.from_numpy(params).cuda()
    gr = torch.empty_like(p)
    D, _ = g.eval(p, grad=gr)
    return D, gr.cpu().numpy()


@pytest.mark.parametrize("name,kind", [("C5", "zero"), ("C5", "small"), ("C5", "large"),
                                       ("C4", "zero"), ("C4", "small"), ("C4", "large")])
def test_full_size_config(name, kind):
    cfg = synth.config(name)
    g, pb, Fn, Mn, params = problem(name, 1, dims=cfg["dims"], params_kind=kind)
    assert pb.dims == cfg["dims"]
    D, grad = _device_eval(g, params)
    st = g.stats()
    g.close()
    Do, go = O.eval_moments(pb, Fn, Mn, params)
    assert rel(D, Do) <= D_TOL, (D, Do)
    assert rel_l2(grad, go) <= G_TOL, rel_l2(grad, go)
    assert comp(grad, go) <= G_COMP, comp(grad, go)
    # the decomposition bench.py reports is the one that ran
    assert st["items"] > 0 and st["items2"] > 0


@pytest.mark.parametrize("dims", [(64, 64, 24), (128, 128, 49), (256, 256, 99)])
def test_paper_table_viii_workloads(dims):
    """bench.py's paper_workloads: C3-shaped pairs at the Table VIII sizes, spatial bins =
    control cells (delta 5 voxels, reading c14 / row F3), 32 intensity bins."""
    import paper_1804_05061_b200 as S
    cfg = synth.config("C3", dims)
    F, M = synth.make_pair("C3", 1, dims)
    sp = cfg["spacing"]
    cells = tuple(max(1, int(n // 5)) for n in dims)
    g = S.Srwcr(F, M, sp, 32, cells, tuple(5.0 * x for x in sp))
    delta = (5.0, 5.0, 5.0)
    pb = O.Problem(dims=dims, L=31, delta=delta, kcells=cells)
    assert g.params_shape == pb.params_shape
    params = synth.make_params(pb.params_shape, "small", 1)
    D, grad = _device_eval(g, params)
    g.close()
    Do, go = O.eval_moments(pb, O.normalize(F, 31), O.normalize(M, 31), params)
    assert rel(D, Do) <= D_TOL, (D, Do)
    assert rel_l2(grad, go) <= G_TOL, rel_l2(grad, go)
    assert comp(grad, go) <= G_COMP, comp(grad, go)
