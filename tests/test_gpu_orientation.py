"""GPU parity of SURVEY 8(f) row F2 -- the moving image as the model image A (Eq 20-21,
App. II Eq 31; readings c4, c23) -- against the fp64 oracle, same gates as orientation 0:
D relative error <= 1e-5, gradient relative L2 <= 1e-4."""
import numpy as np
import pytest

import oracle as O
import synth
import paper_1804_05061_b200 as S
from gpu_common import problem, rel, rel_l2, comp, G_COMP

pytestmark = pytest.mark.gpu

D_TOL = 1e-5
G_TOL = 1e-4


@pytest.mark.parametrize("name,bins", [("C1", None), ("C2", None), ("C3", None), ("C4", None), ("C5", 64)])
@pytest.mark.parametrize("kind", ["zero", "small", "large"])
def test_orientation1_value_and_gradient(name, bins, kind):
    g, pb, Fn, Mn, params = problem(name, 1, params_kind=kind, orientation=1, bins=bins)
    D, grad = g.eval(params)
    if name == "C1":
        Do, go = O.eval_literal(pb, Fn, Mn, params)
    else:
        Do, go = O.eval_moments(pb, Fn, Mn, params)
    assert rel(D, Do) <= D_TOL, (D, Do)
    if np.linalg.norm(go) > 0:
        assert rel_l2(grad, go) <= G_TOL, rel_l2(grad, go)
        assert comp(grad, go) <= G_COMP, comp(grad, go)
    g.close()


def test_orientation1_swap_identity_at_zero_params():
    """At Phi = 0, orientation 1 on (F, M) equals orientation 0 on (M, F)."""
    cfg = synth.config("C3", (70, 66, 34))
    F, M = synth.make_pair("C3", 1, cfg["dims"])
    a = S.Srwcr(F, M, cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"], orientation=1)
    b = S.Srwcr(M, F, cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"], orientation=0)
    z = np.zeros(a.params_shape)
    Da, _ = a.eval(z, want_grad=False)
    Db, _ = b.eval(z, want_grad=False)
    assert rel(Da, Db) <= 2e-6, (Da, Db)
    a.close()
    b.close()


def test_orientation1_register_reduces_cost():
    g, pb, Fn, Mn, _ = problem("C3", 1, orientation=1)
    x, rep = g.register(None, max_iter=30)
    assert rep["final_cost"] < rep["initial_cost"] * (1 - 1e-3)
    g.close()


@pytest.mark.parametrize("bins", [65, 66, 80, 83, 100, 128])
def test_orientation1_bin_counts_near_the_limit(bins):
    """Orientation 1 keeps two slot groups per model bin in pass 1 (up to 254 slots: 8-word
    slot masks) and 3 (B + 2) gamma columns in pass 2 (16-bit column map): bin counts up to
    BASELINE's 128 against the oracle (C5-shaped pair, reduced).  Round 1 refused > 83 bins
    and was silently wrong above 65 (128-bit masks)."""
    g, pb, Fn, Mn, params = problem("C5", 1, params_kind="small", orientation=1, bins=bins)
    D, grad = g.eval(params)
    Do, go = O.eval_moments(pb, Fn, Mn, params)
    g.close()
    assert rel(D, Do) <= D_TOL, (D, Do)
    assert rel_l2(grad, go) <= G_TOL, rel_l2(grad, go)


def test_orientation1_model_bin_assignment_contract():
    """F2's bin-assignment contract (DESIGN c25): in orientation 1 the model bin of a voxel is
    n(m) = min(floor m, L-1) of the fp32 sample m (Eq 5 applied to A = M(T(x))); where fp64 m
    lies within fp32 rounding of an integer the voxel is decided by the fp64 exact path.  The
    dumped per-voxel m (pass 1) against the oracle's fp64 warp: bins differ only next to an
    integer, and only rarely."""
    g, pb, Fn, Mn, params = problem("C3", 1, params_kind="small", orientation=1)
    g.eval(params)
    mg = g.debug_dump("warped").reshape(pb.dims[2], pb.dims[1], pb.dims[0], 4)
    g.close()
    m_o, _ = O.warp(pb, Mn, params)
    L = pb.L
    m_g = np.where(mg[..., 0] < 0, -1.0 - mg[..., 0], mg[..., 0])
    n_g = np.minimum(np.floor(m_g), L - 1)
    n_o = np.minimum(np.floor(m_o), L - 1)
    mism = n_g != n_o
    near = np.abs(m_o - np.round(m_o)) < 1e-4
    assert not np.any(mism & ~near)
    assert int(mism.sum()) <= 1e-4 * m_o.size
    assert np.abs(m_g - m_o).max() < 1e-3
