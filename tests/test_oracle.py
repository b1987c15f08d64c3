"""Pins of the fp64 CPU oracle (oracle/) against what the paper and mathematics fix.

Every test here is CPU-only.  Each pin is chosen so that a plausible mistake in the
oracle (a dropped term, a wrong sign or index, a transposed operand) fails one of
them: hand-evaluated values of Eq 5 / Eq 8 (tests/golden), closed forms, partitions
of unity, a textbook correlation-ratio example, brute force with an independent
(centered, symmetric) B-spline formulation, invariances, and central differences.
"""
import numpy as np
import pytest
from scipy import ndimage

import oracle as O
from conftest import golden


def _rows(name):
    out = []
    for line in open(golden(name)):
        line = line.strip()
        if line and not line.startswith("#"):
            out.append(line)
    return out


# ----------------------------------------------------------- Eq 5 Parzen window

def test_parzen_golden_values():
    for row in _rows("parzen_eq5.txt"):
        t, h, hp = map(float, row.split())
        assert O.parzen(t) == pytest.approx(h, abs=1e-15)
        assert O.parzen_deriv(t) == pytest.approx(hp, abs=1e-15)


def test_parzen_partition_of_unity_and_closed_form_moments():
    L = 31
    for v in np.concatenate([np.linspace(0, L, 997), np.arange(L + 1.0)]):
        h = np.array([O.parzen(a - v) for a in range(L + 1)])
        assert h.sum() == pytest.approx(1.0, abs=1e-13)
        n = min(int(np.floor(v)), L - 1)
        # g1 = sum_b b h(b - v) and g2 = sum_b b^2 h(b - v): closed forms at integers
        if v == np.floor(v):
            assert (np.arange(L + 1) * h).sum() == pytest.approx(v, abs=1e-12)
            assert (np.arange(L + 1) ** 2 * h).sum() == pytest.approx(v * v, abs=1e-10)
        assert h[n] + h[n + 1] == pytest.approx(1.0, abs=1e-13)   # only two active bins
    # max |g1(m) - m| = 0.1125 (attained at f = 0.25, 0.75)
    ms = np.linspace(3, 4, 4001)
    g1 = np.array([sum(b * O.parzen(b - m) for b in range(L + 1)) for m in ms])
    assert np.abs(g1 - ms).max() == pytest.approx(0.1125, abs=1e-9)


def test_parzen_derivative_matches_finite_differences():
    for t in np.linspace(-1.4, 1.4, 281):
        if min(abs(abs(t) - k) for k in (0.0, 1.0)) < 1e-3:
            continue
        h = 1e-6
        fd = (O.parzen(t + h) - O.parzen(t - h)) / (2 * h)
        assert O.parzen_deriv(t) == pytest.approx(fd, abs=1e-5)


# ---------------------------------------------------- Eq 8 / Eq 17 B-spline, FFD

def test_bspline_golden_and_partition():
    for row in _rows("bspline_eq8.txt"):
        vals = list(map(float, row.split()))
        assert np.allclose(O.beta(vals[0]), vals[1:], atol=1e-16, rtol=0)
    for t in np.linspace(0, 1, 101, endpoint=False):
        assert O.beta(t).sum() == pytest.approx(1.0, abs=1e-15)


def _B3(s):
    """Centered cubic B-spline kernel (the symmetric form, independent of Eq 8's pieces)."""
    a = abs(s)
    if a < 1:
        return 2.0 / 3.0 - a * a + 0.5 * a ** 3
    if a < 2:
        return (2 - a) ** 3 / 6.0
    return 0.0


def test_taps_match_centered_kernel():
    # node j sits at (j-1)*spacing; tap base floor(i/spacing); weights beta_l
    for spacing in (5.0, 3.7, 8.0, 1.6667):
        for i in range(0, 40):
            b, w = O.taps(i, spacing)
            for l in range(4):
                j = b + l
                assert w[l] == pytest.approx(_B3((i - (j - 1) * spacing) / spacing), abs=1e-14)
            # all other nodes carry zero weight
            for j in range(max(0, b - 3), b + 8):
                if not (b <= j <= b + 3):
                    assert _B3((i - (j - 1) * spacing) / spacing) == pytest.approx(0.0, abs=1e-14)


def test_grid_counts():
    pb = O.Problem(dims=(512, 512, 320), L=127, delta=(5, 5, 5), kcells=(8, 8, 8))
    G, K = pb.derived()
    assert G == (106, 106, 67) and K == (11, 11, 11)   # SURVEY 8(a) a3 node counts
    pb = O.Problem(dims=(64, 64, 1), L=31, delta=(8, 8, 8), kcells=(4, 4, 0))
    G, K = pb.derived()
    assert G == (11, 11, 1) and K == (7, 7, 4)


def test_ffd_identity_translation_linearity_and_jacobian():
    pb = O.Problem(dims=(20, 17, 13), L=15, delta=(4.0, 3.5, 5.0), kcells=(2, 2, 2))
    rng = np.random.default_rng(3)
    zero = np.zeros(pb.params_shape)
    const = np.zeros(pb.params_shape)
    const[0], const[1], const[2] = 1.25, -0.5, 2.0
    P1, P2 = rng.normal(size=pb.params_shape), rng.normal(size=pb.params_shape)
    for (x, y, z) in [(0, 0, 0), (19, 16, 12), (7, 3, 9), (4, 7, 5)]:
        assert np.all(O.displacement(pb, zero, x, y, z) == 0.0)                 # exact identity
        assert np.allclose(O.displacement(pb, const, x, y, z), [1.25, -0.5, 2.0], atol=1e-14)
        u = O.displacement(pb, 2 * P1 - 3 * P2, x, y, z)
        assert np.allclose(u, 2 * O.displacement(pb, P1, x, y, z) - 3 * O.displacement(pb, P2, x, y, z), atol=1e-12)
    # Jacobian at a node centre (Eq 17): (4/6)^3 = 8/27.  Voxel (8, 7, 10) sits on
    # node (3, 3, 3) for delta (4, 3.5, 5): node j at (j-1)*delta.
    unit = np.zeros(pb.params_shape)
    unit[1, 3, 3, 3] = 1.0
    assert O.displacement(pb, unit, 8, 7, 10)[1] == pytest.approx(8 / 27, abs=1e-15)
    # brute force with the centered kernel
    for (x, y, z) in [(5, 11, 2), (13, 0, 12)]:
        ref = np.zeros(3)
        for c in range(3):
            for gz in range(pb.params_shape[1]):
                for gy in range(pb.params_shape[2]):
                    for gx in range(pb.params_shape[3]):
                        w = _B3(x / 4.0 - (gx - 1)) * _B3(y / 3.5 - (gy - 1)) * _B3(z / 5.0 - (gz - 1))
                        ref[c] += w * P1[c, gz, gy, gx]
        assert np.allclose(O.displacement(pb, P1, x, y, z), ref, atol=1e-12)


# ------------------------------------------------------------ trilinear

def test_trilinear_exactness_gradient_and_clamp():
    pb = O.Problem(dims=(7, 6, 5), L=15, delta=(3, 3, 3), kcells=(1, 1, 1))
    zz, yy, xx = np.meshgrid(np.arange(5), np.arange(6), np.arange(7), indexing="ij")
    # trilinear function a + bx + cy + dz + e xy + f yz + g xz + h xyz is reproduced exactly
    M = (1.0 + 0.5 * xx - 0.25 * yy + 0.75 * zz + 0.125 * xx * yy - 0.0625 * yy * zz + 0.03125 * xx * zz
         + 0.015625 * xx * yy * zz).astype(np.float32)

    def fM(x, y, z):
        return 1 + 0.5 * x - 0.25 * y + 0.75 * z + 0.125 * x * y - 0.0625 * y * z + 0.03125 * x * z + 0.015625 * x * y * z

    def gM(x, y, z):
        return np.array([0.5 + 0.125 * y + 0.03125 * z + 0.015625 * y * z,
                         -0.25 + 0.125 * x - 0.0625 * z + 0.015625 * x * z,
                         0.75 - 0.0625 * y + 0.03125 * x + 0.015625 * x * y])

    rng = np.random.default_rng(5)
    for _ in range(50):
        p = rng.uniform([0, 0, 0], [6, 5, 4])
        m, g = O.sample(pb, M, p)
        assert m == pytest.approx(fM(*p), abs=1e-12)
        assert np.allclose(g, gM(*p), atol=1e-12)
    for (x, y, z) in [(0, 0, 0), (6, 5, 4), (3, 2, 1)]:
        assert O.sample(pb, M, (x, y, z))[0] == M[z, y, x]          # lattice points exact
    m, g = O.sample(pb, M, (-3.0, 2.0, 1.0))                          # clamped in x
    assert m == M[1, 2, 0] and g[0] == 0.0 and g[1] != 0.0
    m, g = O.sample(pb, M, (2.0, 9.0, 1.5))                           # clamped in y
    assert m == pytest.approx(fM(2, 5, 1.5), abs=1e-12) and g[1] == 0.0
    # against scipy's linear interpolation with edge clamping (a library routine)
    Mr = rng.random((5, 6, 7)).astype(np.float32)
    for _ in range(50):
        p = rng.uniform([-2, -2, -2], [8, 7, 6])
        ref = ndimage.map_coordinates(Mr.astype(np.float64), [[p[2]], [p[1]], [p[0]]], order=1, mode="nearest")[0]
        assert O.sample(pb, Mr, p)[0] == pytest.approx(ref, abs=1e-12)


def test_normalize_golden_and_range():
    for row in _rows("normalize_p53.txt"):
        L, vin, vout = row.split("|")
        out = O.normalize(np.array(vin.split(), dtype=np.float32), int(L))
        assert np.array_equal(out, np.array(vout.split(), dtype=np.float32))
    v = np.random.default_rng(2).normal(size=1000).astype(np.float32) * 300 - 40
    out = O.normalize(v, 63)
    assert out.min() == 0.0 and out.max() == 63.0 and out.dtype == np.float32


# --------------------------------------------------------- Eq 3 + Table I value

def _textbook_cr_D(A, B):
    """1 - Roche's correlation ratio Var(E[B|A])/Var(B), via numpy group-by."""
    A, B = A.ravel().astype(np.float64), B.ravel().astype(np.float64)
    var = B.var()
    within = sum((A == a).mean() * B[A == a].var() for a in np.unique(A))
    return within / var


def test_textbook_cr_golden():
    rows = dict((r.split()[0], r.split()[1:]) for r in _rows("cr_textbook.txt"))
    nx, ny, L = int(rows["nx"][0]), int(rows["ny"][0]), int(rows["L"][0])
    A = np.array(rows["A"], dtype=np.float32).reshape(1, ny, nx)
    B = np.array(rows["B"], dtype=np.float32).reshape(1, ny, nx)
    pb = O.Problem(dims=(nx, ny, 1), L=L, delta=(2, 2, 1), kcells=(0, 0, 0))
    zero = np.zeros(pb.params_shape)
    D_lit, _ = O.eval_literal(pb, A, B, zero, want_grad=False)
    D_mom, _ = O.eval_moments(pb, A, B, zero, want_grad=False)
    assert D_lit == pytest.approx(float(rows["D"][0]), abs=1e-15)
    assert D_mom == pytest.approx(float(rows["D"][0]), abs=1e-15)


@pytest.mark.parametrize("dims,L", [((12, 9, 7), 15), ((30, 20, 1), 31)])
def test_single_global_bin_is_textbook_cr(dims, L):
    rng = np.random.default_rng(11)
    sh = dims[::-1]
    A = rng.integers(0, L + 1, size=sh).astype(np.float32)
    B = np.clip(np.round(0.6 * A + rng.integers(-4, 5, size=sh)), 0, L).astype(np.float32)
    pb = O.Problem(dims=dims, L=L, delta=(3, 3, 3), kcells=(0, 0, 0))
    D, _ = O.eval_literal(pb, A, B, np.zeros(pb.params_shape), want_grad=False)
    assert D == pytest.approx(_textbook_cr_D(A, B), rel=1e-13)


def test_product_joint_gives_cr_zero_and_identity_gives_zero():
    # A depends on x only, B on y only: every a-group sees the same B distribution -> CR = 0
    nx, ny, L = 8, 6, 7
    xx, yy = np.meshgrid(np.arange(nx), np.arange(ny), indexing="xy")
    A = (xx % 2 * 3).astype(np.float32)[None]
    B = (yy % 3 * 2).astype(np.float32)[None]
    pb = O.Problem(dims=(nx, ny, 1), L=L, delta=(2, 2, 1), kcells=(0, 0, 0))
    D, _ = O.eval_literal(pb, A, B, np.zeros(pb.params_shape), want_grad=False)
    assert D == pytest.approx(1.0, abs=1e-14)
    # identical integer images: D = 0 and grad = 0 (functional dependence, reading c4)
    pb3 = O.Problem(dims=(9, 8, 7), L=15, delta=(3, 3, 3), kcells=(2, 2, 2))
    I = np.random.default_rng(4).integers(0, 16, size=(7, 8, 9)).astype(np.float32)
    for route in (O.eval_literal, O.eval_moments):
        D, g = route(pb3, I, I, np.zeros(pb3.params_shape))
        assert abs(D) < 1e-15 and np.abs(g).max() < 1e-15


def _brute_joint_hist(F, M, dims, L, delta, kcells, params):
    """Eq 3 by brute force with the centered kernel and scipy linear interpolation."""
    nx, ny, nz = dims
    K = [k + 3 if k > 0 else 4 for k in kcells]
    if nz == 1:
        K[2] = 4
    Delta = [dims[i] / kcells[i] if kcells[i] > 0 else None for i in range(3)]
    R = K[0] * K[1] * K[2]
    P = np.zeros((R, L + 1, L + 1))
    G = params.shape[1:][::-1]  # (Gx, Gy, Gz)
    for z in range(nz):
        for y in range(ny):
            for x in range(nx):
                pos = [x, y, z]
                u = np.zeros(3)
                for c in range(params.shape[0]):
                    for gz in range(G[2]):
                        wz = 1.0 if nz == 1 else _B3(z / delta[2] - (gz - 1))
                        for gy in range(G[1]):
                            for gx in range(G[0]):
                                w = _B3(x / delta[0] - (gx - 1)) * _B3(y / delta[1] - (gy - 1)) * wz
                                u[c] += w * params[c, gz, gy, gx]
                q = [pos[i] + u[i] for i in range(3)]
                coords = [[q[2]], [q[1]], [q[0]]] if nz > 1 else [[0.0], [q[1]], [q[0]]]
                m = ndimage.map_coordinates(M.astype(np.float64), coords, order=1, mode="nearest")[0]
                f = float(F[z, y, x])
                for r in range(R):
                    rx, ry, rz = r % K[0], (r // K[0]) % K[1], r // (K[0] * K[1])
                    w = 1.0
                    for ax, (ri, p) in enumerate(zip((rx, ry, rz), pos)):
                        if Delta[ax] is None or (ax == 2 and nz == 1):
                            w *= 1.0 if ri == 0 else 0.0
                        else:
                            w *= _B3(p / Delta[ax] - (ri - 1))
                    if w == 0.0:
                        continue
                    for a in range(L + 1):
                        ha = O.parzen(a - f)
                        if ha == 0.0:
                            continue
                        for b in range(L + 1):
                            P[r, a, b] += w * ha * O.parzen(b - m)
    return P


@pytest.mark.parametrize("dims,delta,kcells", [((6, 5, 4), (2.5, 2.0, 3.0), (2, 1, 2)),
                                               ((9, 7, 1), (3.0, 2.5, 1.0), (3, 2, 0))])
def test_joint_histogram_brute_force(dims, delta, kcells):
    L = 5
    rng = np.random.default_rng(7)
    sh = dims[::-1]
    F = rng.uniform(0, L, size=sh).astype(np.float32)
    M = rng.uniform(0, L, size=sh).astype(np.float32)
    pb = O.Problem(dims=dims, L=L, delta=delta, kcells=kcells)
    params = rng.uniform(-1.5, 1.5, size=pb.params_shape)
    P = O.joint_hist(pb, F, M, params)
    ref = _brute_joint_hist(F, M, dims, L, delta, kcells, params)
    assert np.abs(P - ref).max() < 1e-12
    # Z = sum of the PDF mass = number of voxels (partitions of unity)
    assert P.sum() == pytest.approx(np.prod(dims), rel=1e-13)


# ------------------------------------------------------ routes, bounds, invariance

def _rand_problem(seed, dims, L, delta, kcells):
    rng = np.random.default_rng(seed)
    sh = dims[::-1]
    base = np.linspace(0, 1, dims[0])[None, None, :] + np.linspace(0, 0.5, dims[1])[None, :, None]
    F = O.normalize((base + 0.3 * rng.random(sh)).astype(np.float32), L)
    M = O.normalize((np.sin(3 * base) + 0.3 * rng.random(sh)).astype(np.float32), L)
    pb = O.Problem(dims=dims, L=L, delta=delta, kcells=kcells)
    params = rng.uniform(-1.5, 1.5, size=pb.params_shape)
    return pb, F, M, params


CASES = [((16, 12, 10), 15, (4.0, 3.0, 2.5), (2, 2, 2)),
         ((23, 19, 1), 31, (5.0, 4.5, 1.0), (3, 2, 0)),
         ((14, 13, 11), 7, (3.3, 5.0, 4.0), (0, 3, 1)),
         ((20, 18, 9), 63, (5.0, 5.0, 2.0), (3, 3, 3))]


@pytest.mark.parametrize("dims,L,delta,kcells", CASES)
def test_literal_equals_moment_route(dims, L, delta, kcells):
    pb, F, M, params = _rand_problem(1, dims, L, delta, kcells)
    D1, g1 = O.eval_literal(pb, F, M, params)
    D2, g2 = O.eval_moments(pb, F, M, params)
    assert D1 == pytest.approx(D2, rel=1e-12)
    assert np.linalg.norm(g1 - g2) <= 1e-12 * np.linalg.norm(g1)


@pytest.mark.parametrize("dims,L,delta,kcells", CASES)
def test_cr_in_unit_interval_and_partitions(dims, L, delta, kcells):
    pb, F, M, params = _rand_problem(2, dims, L, delta, kcells)
    P = O.joint_hist(pb, F, M, params)
    D, reg, _ = O.value_table1(pb, P)
    ret = reg[:, 4] > 0
    assert ret.any()
    assert np.all(reg[ret, 3] >= -1e-12) and np.all(reg[ret, 3] <= 1 + 1e-12)   # 1-CR_r in [0,1]
    assert 0.0 <= D <= 1.0
    assert reg[:, 0].sum() == pytest.approx(1.0, abs=1e-12)                     # sum_r p(r) = 1
    assert P.sum() == pytest.approx(np.prod(dims), rel=1e-12)


def test_affine_invariance_of_moving_intensities():
    dims, L = (14, 12, 9), 31
    rng = np.random.default_rng(9)
    sh = dims[::-1]
    F = rng.integers(0, L + 1, size=sh).astype(np.float32)
    M = rng.integers(0, L + 1, size=sh).astype(np.float32)
    M[0, 0, 0], M[0, 0, 1] = 0.0, float(L)
    pb = O.Problem(dims=dims, L=L, delta=(4, 4, 3), kcells=(2, 2, 2))
    params = rng.uniform(-1, 1, size=pb.params_shape)
    D0, g0 = O.eval_literal(pb, F, O.normalize(M, L), params)
    for a, b in ((2.0, 3.0), (-2.0, 5.0), (0.5, -7.0)):
        Ma = O.normalize((a * M + b).astype(np.float32), L)     # exact in fp32 for these a, b
        D1, g1 = O.eval_literal(pb, F, Ma, params)
        assert D1 == pytest.approx(D0, rel=1e-13)
        assert np.linalg.norm(g1 - g0) <= 1e-11 * np.linalg.norm(g0)


# ----------------------------------------------------- gradient vs central diffs

@pytest.mark.parametrize("dims,L,delta,kcells", [((16, 14, 1), 15, (4.0, 3.5, 1.0), (2, 2, 0)),
                                                 ((10, 9, 8), 15, (3.5, 4.0, 3.0), (2, 2, 2)),
                                                 ((11, 8, 7), 31, (2.6, 3.0, 2.2), (1, 2, 0))])
def test_gradient_central_differences(dims, L, delta, kcells):
    pb, F, M, params = _rand_problem(3, dims, L, delta, kcells)
    D, g = O.eval_literal(pb, F, M, params)
    rng = np.random.default_rng(4)
    idx = list(np.ndindex(g.shape))
    sel = [idx[i] for i in rng.choice(len(idx), min(30, len(idx)), replace=False)]
    # add the components with the largest gradients so the check is not dominated by zeros
    sel += [np.unravel_index(i, g.shape) for i in np.argsort(-np.abs(g).ravel())[:10]]
    h = 1e-6
    num, ana = [], []
    for s in sel:
        pp, pm = params.copy(), params.copy()
        pp[s] += h
        pm[s] -= h
        num.append((O.eval_literal(pb, F, M, pp, False)[0] - O.eval_literal(pb, F, M, pm, False)[0]) / (2 * h))
        ana.append(g[s])
    num, ana = np.array(num), np.array(ana)
    assert np.linalg.norm(num - ana) <= 2e-5 * np.linalg.norm(num)


# ------------------------------------------------- slab decomposition (multi-GPU)

def test_slab_partials_sum_to_full():
    pb, F, M, params = _rand_problem(5, (12, 10, 11), 15, (3.0, 3.0, 2.5), (2, 2, 2))
    N, S, Q = O.moments(pb, F, M, params)
    cuts = [0, 3, 7, 11]
    parts = [O.moments(pb, F, M, params, a, b) for a, b in zip(cuts[:-1], cuts[1:])]
    for k, full in enumerate((N, S, Q)):
        assert np.allclose(sum(p[k] for p in parts), full, rtol=1e-13, atol=1e-12)
    D, al, be, ga, reg, Z = O.combine(pb, N, S, Q)
    g_full = O.grad_moments(pb, F, M, params, al, be, ga, Z)
    g_parts = sum(O.grad_moments(pb, F, M, params, al, be, ga, Z, a, b) for a, b in zip(cuts[:-1], cuts[1:]))
    assert np.linalg.norm(g_parts - g_full) <= 1e-13 * np.linalg.norm(g_full)


# ------------------------------------------------ bending energy C_p (F1, c19)

def _node_coords(pb):
    """Positions (voxels) of the control nodes: node j at (j - 1) * delta (reading c15)."""
    G = pb.derived()[0]
    xs = [(np.arange(G[a]) - 1.0) * pb.delta[a] for a in range(3)]
    if pb.dims[2] == 1:
        xs[2] = np.zeros(1)
    Z, Y, X = np.meshgrid(xs[2], xs[1], xs[0], indexing="ij")
    return X, Y, Z


@pytest.mark.parametrize("dims,delta", [((21, 17, 13), (4.0, 3.5, 5.0)), ((19, 23, 1), (3.0, 4.5, 1.0))])
def test_bending_zero_and_affine_fields_vanish(dims, delta):
    pb = O.Problem(dims=dims, L=15, delta=delta, kcells=(2, 2, 2 if dims[2] > 1 else 0))
    E, g = O.bending(pb, np.zeros(pb.params_shape))
    assert E == 0.0 and not g.any()
    # B-splines reproduce linear functions: an affine displacement has no curvature
    X, Y, Z = _node_coords(pb)
    rng = np.random.default_rng(3)
    phi = np.stack([rng.normal() * X + rng.normal() * Y + rng.normal() * Z + rng.normal()
                    for _ in range(pb.ndim)])
    E, _ = O.bending(pb, phi)
    assert abs(E) < 1e-20


@pytest.mark.parametrize("dims,delta", [((21, 17, 13), (4.0, 3.5, 5.0)), ((16, 16, 16), (2.5, 3.0, 4.0))])
def test_bending_closed_forms_3d(dims, delta):
    """Cubic B-splines reproduce quadratics with coefficients xi^2 - delta^2/3 (variance
    of the cubic B-spline kernel = delta^2/3) and products xi*eta exactly, so u = x^2
    gives u_xx = 2 everywhere (C_p = 4), u = x*y gives u_xy = 1 (C_p = 2, cross terms
    doubled), and terms on different components / second derivatives add."""
    pb = O.Problem(dims=dims, L=15, delta=delta, kcells=(2, 2, 2))
    X, Y, Z = _node_coords(pb)
    dx, dy, dz = pb.delta
    zero = np.zeros_like(X)
    cases = [
        ((X**2 - dx * dx / 3, zero, zero), 4.0),
        ((zero, Y**2 - dy * dy / 3, zero), 4.0),
        ((zero, zero, Z**2 - dz * dz / 3), 4.0),
        ((zero, X * Y, zero), 2.0),
        ((X * Z, zero, zero), 2.0),
        ((zero, zero, Y * Z), 2.0),
        ((zero, zero, Z**2 - dz * dz / 3 + X * Y), 6.0),
        ((0.5 * (X**2 - dx * dx / 3), 3 * Y * Z, zero), 1.0 + 18.0),
    ]
    for phi, want in cases:
        E, _ = O.bending(pb, np.stack(phi))
        assert E == pytest.approx(want, rel=1e-12), (want, E)


def test_bending_closed_forms_2d():
    pb = O.Problem(dims=(19, 23, 1), L=15, delta=(3.0, 4.5, 1.0), kcells=(2, 2, 0))
    X, Y, _ = _node_coords(pb)
    dx, dy = pb.delta[:2]
    E, _ = O.bending(pb, np.stack([X**2 - dx * dx / 3 + Y**2 - dy * dy / 3, np.zeros_like(X)]))
    assert E == pytest.approx(8.0, rel=1e-12)
    E, _ = O.bending(pb, np.stack([np.zeros_like(X), X * Y]))
    assert E == pytest.approx(2.0, rel=1e-12)


@pytest.mark.parametrize("dims,delta", [((13, 11, 9), (3.0, 2.5, 3.5)), ((14, 12, 1), (3.0, 4.0, 1.0))])
def test_bending_gradient_central_differences(dims, delta):
    pb = O.Problem(dims=dims, L=15, delta=delta, kcells=(1, 1, 1 if dims[2] > 1 else 0))
    rng = np.random.default_rng(5)
    phi = rng.normal(size=pb.params_shape)
    E, g = O.bending(pb, phi)
    assert E > 0
    flat = phi.reshape(-1)
    idx = rng.choice(flat.size, 40, replace=False)
    h = 1e-3
    for i in idx:   # C_p is quadratic: central differences are exact up to rounding
        p = flat.copy(); p[i] += h
        m = flat.copy(); m[i] -= h
        fd = (O.bending(pb, p.reshape(phi.shape), False)[0] - O.bending(pb, m.reshape(phi.shape), False)[0]) / (2 * h)
        assert g.reshape(-1)[i] == pytest.approx(fd, rel=1e-7, abs=1e-12)
    # quadratic form: phi . grad = 2 C_p
    assert float((phi * g).sum()) == pytest.approx(2 * E, rel=1e-12)


# ------------------------------------ orientation 1: moving image as model A (F2)

def _swap(pb, o):
    from dataclasses import replace
    return replace(pb, orientation=o)


@pytest.mark.parametrize("dims,L,delta,kcells", CASES)
def test_orientation1_at_identity_is_orientation0_with_images_swapped(dims, L, delta, kcells):
    """At Phi = 0 the warped moving image is M itself, so making M the model image A is
    the same as swapping the two images (Eq 3 with A and B exchanged)."""
    pb, F, M, _ = _rand_problem(6, dims, L, delta, kcells)
    zero = np.zeros(pb.params_shape)
    P1 = O.joint_hist(_swap(pb, 1), F, M, zero)
    P0 = O.joint_hist(_swap(pb, 0), M, F, zero)
    assert np.array_equal(P1, P0)
    for route in (O.eval_literal, O.eval_moments):
        D1, _ = route(_swap(pb, 1), F, M, zero, want_grad=False)
        D0, _ = route(_swap(pb, 0), M, F, zero, want_grad=False)
        assert D1 == pytest.approx(D0, rel=1e-13, abs=1e-15)
    # and the orientations differ in general (SRWCR is asymmetric)
    Da, _ = O.eval_moments(_swap(pb, 0), F, M, zero, want_grad=False)
    assert abs(Da - O.eval_moments(_swap(pb, 1), F, M, zero, want_grad=False)[0]) > 1e-6


@pytest.mark.parametrize("dims,L,delta,kcells", CASES)
def test_orientation1_literal_equals_moment_route(dims, L, delta, kcells):
    pb, F, M, params = _rand_problem(1, dims, L, delta, kcells)
    pb = _swap(pb, 1)
    D1, g1 = O.eval_literal(pb, F, M, params)
    D2, g2 = O.eval_moments(pb, F, M, params)
    assert D1 == pytest.approx(D2, rel=1e-12)
    assert 0.0 <= D1 <= 1.0
    assert np.linalg.norm(g1 - g2) <= 1e-11 * np.linalg.norm(g1)


@pytest.mark.parametrize("dims,L,delta,kcells", [((16, 14, 1), 15, (4.0, 3.5, 1.0), (2, 2, 0)),
                                                 ((10, 9, 8), 15, (3.5, 4.0, 3.0), (2, 2, 2)),
                                                 ((11, 8, 7), 31, (2.6, 3.0, 2.2), (1, 2, 0))])
def test_orientation1_gradient_central_differences(dims, L, delta, kcells):
    """Eq 31 (App. II) with reading c23 is the derivative of D: central differences."""
    pb, F, M, params = _rand_problem(3, dims, L, delta, kcells)
    pb = _swap(pb, 1)
    D, g = O.eval_literal(pb, F, M, params)
    rng = np.random.default_rng(4)
    idx = list(np.ndindex(g.shape))
    sel = [idx[i] for i in rng.choice(len(idx), min(30, len(idx)), replace=False)]
    sel += [np.unravel_index(i, g.shape) for i in np.argsort(-np.abs(g).ravel())[:10]]
    h = 1e-6
    num, ana = [], []
    for s in sel:
        pp, pm = params.copy(), params.copy()
        pp[s] += h
        pm[s] -= h
        num.append((O.eval_literal(pb, F, M, pp, False)[0] - O.eval_literal(pb, F, M, pm, False)[0]) / (2 * h))
        ana.append(g[s])
    num, ana = np.array(num), np.array(ana)
    assert np.linalg.norm(num - ana) <= 2e-5 * np.linalg.norm(num)


def test_orientation1_identical_images_and_slabs():
    pb3 = O.Problem(dims=(9, 8, 7), L=15, delta=(3, 3, 3), kcells=(2, 2, 2), orientation=1)
    I = np.random.default_rng(4).integers(0, 16, size=(7, 8, 9)).astype(np.float32)
    for route in (O.eval_literal, O.eval_moments):
        D, _ = route(pb3, I, I, np.zeros(pb3.params_shape), want_grad=False)
        assert abs(D) < 1e-15
    # slab partial statistics and gradients sum to the full ones (z-slab decomposition)
    pb, F, M, params = _rand_problem(5, (12, 10, 11), 15, (3.0, 3.0, 2.5), (2, 2, 2))
    pb = _swap(pb, 1)
    N, Sm, Q = O.moments(pb, F, M, params)
    cuts = [0, 4, 11]
    parts = [O.moments(pb, F, M, params, a, b) for a, b in zip(cuts[:-1], cuts[1:])]
    for k, full in enumerate((N, Sm, Q)):
        assert np.allclose(sum(p[k] for p in parts), full, rtol=1e-13, atol=1e-12)
    D, al, be, ga, reg, Z = O.combine(pb, N, Sm, Q)
    g_full = O.grad_moments_A(pb, F, M, params, N, ga, reg, Z)
    g_parts = sum(O.grad_moments_A(pb, F, M, params, N, ga, reg, Z, a, b) for a, b in zip(cuts[:-1], cuts[1:]))
    assert np.linalg.norm(g_parts - g_full) <= 1e-13 * np.linalg.norm(g_full)
    assert np.linalg.norm(g_full - O.eval_moments(pb, F, M, params)[1]) <= 1e-13 * np.linalg.norm(g_full)


# ------------------------------------------------------------ L-BFGS (F1, reading c20)

def test_lbfgs_quadratic_closed_form():
    """A strictly convex quadratic 1/2 x.Ax - b.x: the minimiser A^-1 b (closed form)."""
    from oracle.lbfgs import lbfgs
    rng = np.random.default_rng(7)
    Q = rng.standard_normal((12, 12))
    A = Q @ Q.T + 12 * np.eye(12)
    b = rng.standard_normal(12)
    x, rep, its = lbfgs(lambda x: (0.5 * x @ A @ x - b @ x, A @ x - b), np.zeros(12), max_iter=200,
                        epsilon=1e-8)
    assert rep["status_name"] == "converged"
    assert np.allclose(x, np.linalg.solve(A, b), rtol=0, atol=1e-8)


def test_lbfgs_rosenbrock_minimum():
    from oracle.lbfgs import lbfgs

    def rosen(x):
        f = (1 - x[0]) ** 2 + 100 * (x[1] - x[0] ** 2) ** 2
        g = np.array([-2 * (1 - x[0]) - 400 * x[0] * (x[1] - x[0] ** 2), 200 * (x[1] - x[0] ** 2)])
        return f, g
    x, rep, _ = lbfgs(rosen, np.array([-1.2, 1.0]), max_iter=500, epsilon=1e-9, stable_window=1000)
    assert np.allclose(x, [1.0, 1.0], atol=1e-6), (x, rep)


def test_lbfgs_first_step_and_wolfe_invariants():
    """First trial step 1/||g0|| along -g0; every accepted step satisfies the Armijo test
    and the regular Wolfe curvature test (c20) and is 1/||g0|| or 1 times 0.5^i 2.1^j."""
    from oracle.lbfgs import lbfgs
    rng = np.random.default_rng(3)
    A = np.diag(rng.uniform(1, 50, 8))

    calls = []

    def fun(x):
        calls.append(x.copy())
        return 0.25 * np.sum((A @ x) ** 2) ** 1.0 + np.sum(np.cos(x)), 0.5 * A @ (A @ x) - np.sin(x)
    x0 = rng.standard_normal(8)
    f0, g0 = fun(x0)
    calls.clear()
    _, rep, its = lbfgs(fun, x0, max_iter=15, stable_window=1000)
    assert np.allclose(calls[1], x0 - g0 / np.linalg.norm(g0), rtol=0, atol=1e-15)
    xprev, fprev, gprev = x0, f0, g0
    d = -g0
    for k, (xk, fk, st, _) in enumerate(its):
        s = xk - xprev
        dd = s / st
        fk2, gk = fun(xk)
        assert fk2 == fk
        assert fk <= fprev + 1e-4 * st * (gprev @ dd) + 1e-15
        assert gk @ dd >= 0.9 * (gprev @ dd) - 1e-15
        base = 1 / np.linalg.norm(g0) if k == 0 else 1.0
        ok = any(abs(st - base * 0.5 ** i * 2.1 ** j) <= 1e-12 * st for i in range(25) for j in range(25))
        assert ok, st
        xprev, fprev, gprev = xk, fk, gk


def test_lbfgs_one_dimensional_quadratic_second_step_is_newton():
    """1-D f = a x^2 / 2: after the first pair, H0 = y.s / y.y = 1/a makes the second
    direction the Newton step, accepted at step 1: x_2 = 0 (up to rounding)."""
    from oracle.lbfgs import lbfgs
    a = 3.7
    x, rep, its = lbfgs(lambda x: (0.5 * a * x @ x, a * x), np.array([2.0]), max_iter=2, stable_window=1000)
    assert len(its) == 2 and its[1][2] == 1.0
    assert abs(its[1][0][0]) < 1e-14


def test_lbfgs_stable_stop_and_line_search_failure():
    """A cost whose variation is far below 1e-5 of its size: the run stops 'stable' once
    stable_window costs (the start included) are within the tolerance.  A cost that is
    infeasible everywhere but the start: the line search fails."""
    from oracle.lbfgs import Infeasible, lbfgs
    x, rep, its = lbfgs(lambda x: (1e6 + np.sum(np.cos(x)), -np.sin(x)), np.array([3.0, 2.5, 2.0]),
                        stable_window=20)
    assert rep["status_name"] == "stable" and rep["iterations"] == 19

    def fun(x):
        if np.any(x != 1.0):
            raise Infeasible
        return 1.0, np.ones_like(x)
    x, rep, its = lbfgs(fun, np.ones(3), max_linesearch=7)
    assert rep["status_name"] == "line_search_failed" and rep["evaluations"] == 8 and np.all(x == 1.0)
