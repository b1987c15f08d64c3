"""GPU checks of the multi-resolution registration utilities and of SURVEY 8(f) row F4
(the paper's S.III-A synthetic experiment, dataset-free): the dense FFD field
and the trilinear resampling against the fp64 oracle, the pyramid/composition identities,
and an end-to-end registration of a warped binary grid image that must recover the
ground-truth displacement (RMSE over the whole domain, as the paper measures it)."""
import numpy as np
import pytest
from scipy import ndimage

import oracle as O
import synth
import paper_1804_05061_b200 as S
from gpu_common import problem

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def test_field_matches_oracle_displacement():
    g, pb, Fn, Mn, params = problem("C3", 1, params_kind="large")
    u = g.field(params)                      # [3, Nz, Ny, Nx]
    rng = np.random.default_rng(0)
    nx, ny, nz = pb.dims
    for _ in range(200):
        x, y, z = int(rng.integers(nx)), int(rng.integers(ny)), int(rng.integers(nz))
        uo = O.displacement(pb, params, x, y, z)
        assert np.allclose(u[:, z, y, x], uo, atol=2e-5 * 15), (x, y, z, u[:, z, y, x], uo)
    g.close()


def test_resample_matches_oracle_sample():
    g, pb, Fn, Mn, params = problem("C3", 1, params_kind="large")
    u = g.field(params)
    g.close()
    Md = torch.from_numpy(Mn).cuda()
    out = S.resample(Md, torch.from_numpy(u).cuda()).cpu().numpy()
    rng = np.random.default_rng(1)
    nx, ny, nz = pb.dims
    for _ in range(200):
        x, y, z = int(rng.integers(nx)), int(rng.integers(ny)), int(rng.integers(nz))
        pos = np.array([x, y, z], dtype=np.float64) + u[:, z, y, x].astype(np.float64)
        m, _ = O.sample(pb, Mn, pos)
        assert abs(out[z, y, x] - m) <= 1e-4 * (1 + abs(m)), (x, y, z, out[z, y, x], m)


def test_pyramid_and_composition_identities():
    dev = "cuda"
    vol = torch.full((9, 10, 11), 3.5, device=dev)
    d = S.downsample2(vol)
    assert tuple(d.shape) == (5, 5, 6) and torch.allclose(d, torch.full_like(d, 3.5))
    c = torch.zeros((3, 5, 5, 6), device=dev)
    c[0] += 1.25
    c[2] -= 0.5
    f = S.upsample2_field(c, (9, 10, 11))
    assert torch.allclose(f[0], torch.full_like(f[0], 2.5)) and torch.allclose(f[2], torch.full_like(f[2], -1.0))
    U = torch.randn((3, 9, 10, 11), device=dev)
    zero = torch.zeros_like(U)
    # (the last voxel of an axis interpolates at t = 1: a + (b - a), exact to an ulp)
    assert torch.allclose(S.compose(U, zero), U, atol=1e-6)
    assert torch.allclose(S.compose(zero, U), U, atol=1e-6)
    # composing two constant shifts inside the volume adds them
    a = torch.zeros_like(U); a[0] += 1.0
    b = torch.zeros_like(U); b[1] += 2.0
    ab = S.compose(a, b)
    inner = ab[:, :, :7, :9]
    assert torch.allclose(inner[0], torch.ones_like(inner[0])) and torch.allclose(inner[1], torch.full_like(inner[1], 2.0))
    # resample by a zero field is the identity
    v = torch.rand((9, 10, 11), device=dev)
    assert torch.allclose(S.resample(v, zero), v, atol=1e-6)


def _grid_image(n):
    """S.III-A: a 3-D binary black-and-white grid image (period 16, thickness 2)."""
    z, y, x = np.meshgrid(*(np.arange(n),) * 3, indexing="ij")
    on = ((x % 16 < 2).astype(int) + (y % 16 < 2) + (z % 16 < 2)) >= 2
    return ndimage.gaussian_filter(on.astype(np.float32) * 100.0, 0.7).astype(np.float32)


def test_multires_recovers_synthetic_warp():
    """F4 at the paper's scale: 128^3 grid image; ground truth = a B-spline field
    with node amplitude <= 15 voxels (nodes every 16 voxels, seeded); fixed = the original
    warped by it, moving = the original ("O as M", M as B).  Three levels (shortened to
    60/60/40 iterations here) must cut the RMSE over the whole domain below 45 % of the
    initial one, and beat a single full-resolution level (large deformations need the
    coarse-to-fine strategy)."""
    n = 128
    Md = torch.from_numpy(_grid_image(n)).cuda()
    gt = S.Srwcr(Md, Md, (1.0, 1.0, 1.0), 32, (4, 4, 4), (16.0, 16.0, 16.0))
    phi = np.random.default_rng(7).uniform(-15.0, 15.0, size=gt.params_shape)
    Ut = torch.from_numpy(gt.field(phi)).cuda()
    gt.close()
    F = S.resample(Md, Ut)
    from paper_1804_05061_b200.multires import register_multires
    U, reps = register_multires(F, Md, (1.0, 1.0, 1.0), 32, (4, 4, 4), control_vox=5.0, levels=3,
                                iters=(60, 60, 40), w_p=0.1)
    rms = lambda V: float(torch.sqrt((V ** 2).sum(0).mean()))
    rmse0, rmse = rms(Ut), rms(U - Ut)
    assert len(reps) == 3 and all(r["final_cost"] <= r["initial_cost"] for r in reps)
    assert rmse < 0.45 * rmse0, (rmse0, rmse, reps)
    g = S.Srwcr(F, Md, (1.0, 1.0, 1.0), 32, (4, 4, 4), (5.0, 5.0, 5.0))
    x1, _ = g.register(None, w_p=0.1, max_iter=100)
    U1 = torch.from_numpy(g.field(x1)).cuda()
    g.close()
    assert rmse < rms(U1 - Ut), (rmse, rms(U1 - Ut))
