"""GPU parity: the sm_100a path (through the C ABI) against the fp64 oracle.

Gates (BASELINE.json north_star): D relative error <= 1e-5, gradient relative L2 error
<= 1e-4, static assignments bit-exact (normalised volumes, fixed-bin map a0, per-axis
tap bases of both lattices, nonzero pattern of N).
"""
import numpy as np
import pytest

import oracle as O
from gpu_common import REDUCED, problem, rel, rel_l2, comp, G_COMP

pytestmark = pytest.mark.gpu

D_TOL = 1e-5
G_TOL = 1e-4


def _oracle_eval(pb, Fn, Mn, params, literal=False):
    if literal:
        return O.eval_literal(pb, Fn, Mn, params)
    return O.eval_moments(pb, Fn, Mn, params)


@pytest.mark.parametrize("name", ["C1", "C2", "C3", "C4", "C5"])
@pytest.mark.parametrize("kind", ["zero", "small", "large"])
def test_value_and_gradient(name, kind):
    g, pb, Fn, Mn, params = problem(name, 1, params_kind=kind)
    D, grad = g.eval(params)
    Do, go = _oracle_eval(pb, Fn, Mn, params, literal=name in ("C1",))
    assert rel(D, Do) <= D_TOL, (D, Do)
    if np.linalg.norm(go) > 0:
        assert rel_l2(grad, go) <= G_TOL, rel_l2(grad, go)
        assert comp(grad, go) <= G_COMP, comp(grad, go)
    g.close()


@pytest.mark.parametrize("name", ["C1", "C2"])
@pytest.mark.parametrize("seed", [2, 3])
def test_more_seeds(name, seed):
    g, pb, Fn, Mn, params = problem(name, seed, params_kind="small")
    D, grad = g.eval(params)
    Do, go = O.eval_moments(pb, Fn, Mn, params)
    assert rel(D, Do) <= D_TOL
    assert rel_l2(grad, go) <= G_TOL
    assert comp(grad, go) <= G_COMP, comp(grad, go)
    g.close()


@pytest.mark.parametrize("name", ["C1", "C3", "C5"])
def test_static_assignments_bit_exact(name):
    g, pb, Fn, Mn, params = problem(name, 1)
    assert np.array_equal(g.debug_dump("fixed"), Fn.ravel())
    assert np.array_equal(g.debug_dump("moving"), Mn.ravel())
    a0 = np.minimum(np.floor(Fn.astype(np.float64)), pb.L - 1).astype(np.int16).ravel()
    assert np.array_equal(g.debug_dump("a0"), a0)
    # per-axis tap bases of the control and spatial lattices (Eq 17 / Eq 7)
    G, K = pb.derived()
    ct, st = g.debug_dump("ctrl_taps"), g.debug_dump("spat_taps")
    off = 0
    for ax, n in enumerate(pb.dims):
        for i in range(n):
            deg_c = ax == 2 and pb.dims[2] == 1
            deg_s = pb.kcells[ax] == 0 or deg_c
            bc, _ = O.taps(i, pb.delta[ax], deg_c)
            bs, _ = O.taps(i, 1.0 if deg_s else pb.dims[ax] / pb.kcells[ax], deg_s)
            assert ct[off + i] == bc and st[off + i] == bs
        off += n
    # static counts N: nonzero pattern exact, values to fp32-accumulation accuracy
    N, _, _ = O.moments(pb, Fn, Mn, params)
    Ng = g.debug_dump("N").reshape(N.shape)
    assert np.array_equal(Ng != 0, N != 0)
    assert np.abs(Ng - N).max() <= 1e-5 * N.max()
    g.close()


def test_identical_integer_images_optimum():
    rng = np.random.default_rng(5)
    I = rng.integers(0, 32, size=(24, 28, 30)).astype(np.float32)
    I[0, 0, 0], I[0, 0, 1] = 0, 31
    import paper_1804_05061_b200 as S
    g = S.Srwcr(I, I, (1, 1, 1), 32, (2, 2, 2), (5, 5, 5))
    D, grad = g.eval(np.zeros(g.params_shape))
    assert abs(D) < 1e-6
    assert np.abs(grad).max() < 1e-6
    g.close()


def test_single_global_bin_is_textbook_cr():
    rng = np.random.default_rng(6)
    A = rng.integers(0, 16, size=(20, 24, 26)).astype(np.float32)
    B = np.clip(np.round(0.6 * A + rng.integers(-3, 4, size=A.shape)), 0, 15).astype(np.float32)
    A[0, 0, :2] = (0, 15)
    B[0, 0, :2] = (0, 15)
    import paper_1804_05061_b200 as S
    g = S.Srwcr(A, B, (1, 1, 1), 16, (0, 0, 0), (5, 5, 5), inputs_normalized=True)
    D, _ = g.eval(np.zeros(g.params_shape))
    a, b = A.ravel().astype(np.float64), B.ravel().astype(np.float64)
    within = sum((a == k).mean() * b[a == k].var() for k in np.unique(a))
    # integer-valued images make the fixed-point rounding of the line tables coherent
    # (every voxel of a (bin, value) pair rounds alike): held to the D gate, not tighter
    assert rel(D, within / b.var()) <= D_TOL
    g.close()


def test_host_and_device_pointers_agree():
    torch = pytest.importorskip("torch")
    g, pb, Fn, Mn, params = problem("C1", 1)
    D1, g1 = g.eval(params)
    pt = torch.from_numpy(params).cuda()
    gt = torch.empty_like(pt)
    D2, _ = g.eval(pt, grad=gt)
    # fp32 shared-memory atomics (column/cell tables) make the summation
    # order -- not the arithmetic -- differ between evaluations: fp32-rounding-sized noise
    assert rel(D2, D1) <= 2e-7
    assert rel_l2(gt.cpu().numpy(), g1) <= 1e-5
    g.close()


def _cudart():
    import ctypes
    import glob
    for cand in ["libcudart.so", *glob.glob("/usr/local/cuda/lib64/libcudart.so*")]:
        try:
            return ctypes.CDLL(cand)
        except OSError:
            continue
    raise RuntimeError("libcudart not found")


@pytest.mark.parametrize("P", [2, 3])
def test_slab_decomposition_on_one_gpu(P):
    """The z-slab path of nranks = P with the exchange done by the caller (sum of rank
    partials) equals the single-GPU result: same kernels, different summation order."""
    import ctypes
    import synth
    import paper_1804_05061_b200 as S
    name = "C3"
    cfg = synth.config(name, REDUCED[name])
    F, M = synth.make_pair(name, 1, cfg["dims"])
    g1 = S.Srwcr(F, M, cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"])
    params = synth.make_params(g1.params_shape, "small", 1)
    D1, grad1 = g1.eval(params)
    ranks = [S.Srwcr(F, M, cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"], nranks=P, rank=k)
             for k in range(P)]
    for r in ranks:
        r.eval_begin(params)
    rt = _cudart()
    bufs = []
    for r in ranks:
        p, n = r.stats_buffer()
        h = np.empty(n, np.float64)
        assert rt.cudaMemcpy(h.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(p), ctypes.c_size_t(8 * n), 4) == 0
        bufs.append(h)
    tot = np.sum(bufs, axis=0)
    for r in ranks:
        p, n = r.stats_buffer()
        assert rt.cudaMemcpy(ctypes.c_void_p(p), tot.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(8 * n), 4) == 0
    outs = [r.eval_end() for r in ranks]
    for D, _ in outs:
        assert rel(D, D1) <= 2e-7   # fp32 atomic summation order (see above)
    gsum = np.sum([gk for _, gk in outs], axis=0)
    assert rel_l2(gsum, grad1) <= 1e-5
    for r in ranks + [g1]:
        r.close()


def test_exact_path_voxels_and_scan_fallback(monkeypatch):
    """Voxels whose per-voxel derivative is discontinuous within fp32 rounding are
    deferred by pass 2 to the fp64 k_exact_fix kernel; with the list capacity forced to
    1 the kernel falls back to scanning the slab's flags.  Both must agree with each
    other and with the oracle."""
    g, pb, Fn, Mn, params = problem("C5", 1, params_kind="large")
    D1, g1 = g.eval(params)
    st = g.stats()
    assert st["exact_voxels"] > 1, st
    g.close()
    monkeypatch.setenv("SRWCR_XCAP", "1")
    g2, *_ = problem("C5", 1, params_kind="large")
    assert g2.stats()["exact_capacity"] == 1
    D2, g2r = g2.eval(params)
    assert g2.stats()["exact_voxels"] > 1
    g2.close()
    assert rel(D2, D1) <= 2e-7
    assert rel_l2(g2r, g1) <= 1e-5
    Do, go = O.eval_moments(pb, Fn, Mn, params)
    assert rel_l2(g2r, go) <= G_TOL
    assert comp(g2r, go) <= G_COMP, comp(g2r, go)


def test_nccl_exchange_path_single_rank():
    """The library-driven exchange (ncclCommInitRank from a caller-broadcast unique id,
    ncclAllReduce of the statistics and of the gradient on the library stream) with one
    rank: the NCCL plumbing of the z-slab decomposition runs on the GPU box and leaves the
    result unchanged (a sum over one rank)."""
    torch = pytest.importorskip("torch")
    import synth
    import paper_1804_05061_b200 as S
    name = "C3"
    cfg = synth.config(name, REDUCED[name])
    F, M = synth.make_pair(name, 1, cfg["dims"])
    g1 = S.Srwcr(F, M, cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"])
    params = synth.make_params(g1.params_shape, "small", 1)
    D1, grad1 = g1.eval(params)
    uid = torch.cuda.nccl.unique_id()
    g2 = S.Srwcr(F, M, cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"], nranks=1, rank=0, nccl_id=uid)
    D2, grad2 = g2.eval(params)
    x, rep = g2.register(params, max_iter=3)
    assert rep["iterations"] >= 1
    assert rel(D2, D1) <= 2e-7
    assert rel_l2(grad2, grad1) <= 1e-5
    g1.close()
    g2.close()


@pytest.mark.parametrize("orientation", [0, 1])
def test_fine_spatial_lattice(orientation):
    """SURVEY 8(f) row F3, the paper's own regime: one spatial cell per control
    cell (here 14 x 13 x 17 cells, 5440 regions) -- the same kernels, work items of one
    control cell each."""
    import synth
    import paper_1804_05061_b200 as S
    dims = REDUCED["C3"]
    cfg = synth.config("C3", dims)
    F, M = synth.make_pair("C3", 1, dims)
    L = cfg["bins"] - 1
    delta = tuple(c / s for c, s in zip(cfg["control_mm"], cfg["spacing"]))
    cells = tuple(int(n // d) for n, d in zip(dims, delta))
    pb = O.Problem(dims=dims, L=L, delta=delta, kcells=cells, orientation=orientation)
    g = S.Srwcr(F, M, cfg["spacing"], cfg["bins"], cells, cfg["control_mm"], orientation=orientation)
    params = synth.make_params(g.params_shape, "small", 2)
    D, grad = g.eval(params)
    Do, go = O.eval_moments(pb, O.normalize(F, L), O.normalize(M, L), params)
    assert pb.nregions == 5440
    assert rel(D, Do) <= D_TOL
    assert rel_l2(grad, go) <= G_TOL
    assert comp(grad, go) <= G_COMP, comp(grad, go)
    g.close()


EDGE = [((2, 2, 1), 3, (1.5, 1.5, 1.0), (0, 0, 0)),        # smallest legal volume (2-D)
        ((5, 3, 2), 7, (1.5, 1.25, 1.5), (1, 1, 1)),        # two slices, one cell
        ((33, 17, 1), 15, (4.0, 3.0, 1.0), (3, 2, 0)),      # 2-D, ragged cells
        ((37, 29, 23), 31, (3.3, 2.9, 4.1), (5, 0, 3)),     # one degenerate spatial axis
        ((70, 9, 40), 63, (5.0, 2.0, 6.0), (7, 1, 2))]      # flat rows (9), wide x


@pytest.mark.parametrize("orientation", [0, 1])
@pytest.mark.parametrize("dims,L,delta,kcells", EDGE)
def test_edge_geometries(dims, L, delta, kcells, orientation):
    """Degenerate and ragged geometries (tiny volumes, 2-D, degenerate spatial axes,
    non-integer control spacings) in both orientations against the oracle."""
    import paper_1804_05061_b200 as S
    rng = np.random.default_rng(sum(dims) + orientation)
    sh = dims[::-1]
    F = rng.uniform(0, 1000, size=sh).astype(np.float32)
    M = (0.5 * F + rng.uniform(0, 300, size=sh)).astype(np.float32)
    sp = (1.0, 1.0, 1.0)
    g = S.Srwcr(F, M, sp, L + 1, kcells, delta, orientation=orientation)
    pb = O.Problem(dims=dims, L=L, delta=delta, kcells=kcells, orientation=orientation)
    assert g.params_shape == pb.params_shape
    params = rng.uniform(-1.0, 1.0, size=pb.params_shape)
    D, grad = g.eval(params)
    Do, go = O.eval_literal(pb, O.normalize(F, L), O.normalize(M, L), params)
    assert rel(D, Do) <= D_TOL, (D, Do)
    if np.linalg.norm(go) > 1e-12:
        assert rel_l2(grad, go) <= G_TOL, rel_l2(grad, go)
        assert comp(grad, go) <= G_COMP, comp(grad, go)
    g.close()


def test_graph_replay_matches_eager_launches():
    """options.use_graph: srwcr_eval with device buffers replays a captured CUDA graph
    (re-captured when a pointer changes); it must give the eager launches' result, follow
    new parameter values written into the same buffer, and count its kernels."""
    torch = pytest.importorskip("torch")
    import synth
    import paper_1804_05061_b200 as S
    name = "C3"
    cfg = synth.config(name, REDUCED[name])
    F, M = synth.make_pair(name, 1, cfg["dims"])
    ge = S.Srwcr(F, M, cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"], use_graph=False)
    gg = S.Srwcr(F, M, cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"], use_graph=True)
    p1 = synth.make_params(ge.params_shape, "small", 1)
    p2 = synth.make_params(ge.params_shape, "large", 2)
    pt = torch.from_numpy(p1).cuda()
    gt = torch.empty_like(pt)
    n0 = gg.stats()["launches_total"]
    for p in (p1, p2, p1):
        pt.copy_(torch.from_numpy(p))
        Dg, _ = gg.eval(pt, grad=gt)
        De, ge_grad = ge.eval(p)
        assert rel(Dg, De) <= 2e-7
        assert rel_l2(gt.cpu().numpy(), ge_grad) <= 1e-5
    st = gg.stats()
    assert st["launches_total"] - n0 == 3 * st["launches_per_eval"]
    gt2 = torch.empty_like(pt)   # new gradient buffer: re-capture
    Dg2, _ = gg.eval(pt, grad=gt2)
    assert rel(Dg2, Dg) <= 2e-7 and rel_l2(gt2.cpu().numpy(), gt.cpu().numpy()) <= 1e-5
    gg.set_timing(True)          # per-pass event records captured into the graph
    gg.eval(pt, grad=gt2)
    gg.eval(pt, grad=gt2)
    st = gg.stats()
    assert st["ms_pass1"] > 0 and st["ms_pass2"] > 0 and st["ms_total"] >= st["ms_pass1"] + st["ms_pass2"]
    ge.close()
    gg.close()


@pytest.mark.parametrize("xcap,orientation", [(None, 0), ("1", 0), (None, 1)])
def test_pipelined_host_buffers_match_device_path(monkeypatch, xcap, orientation):
    """Host params / host gradient on one rank: the params upload overlaps pass 1 and the
    final gradient layers go back while pass 2's last items run (here with 4-item
    "waves" so that a reduced volume is split; xcap=1 forces the list overflow, whose
    final scan re-copies the whole gradient).  Same result as the device-buffer path and
    the oracle."""
    torch = pytest.importorskip("torch")
    monkeypatch.setenv("SRWCR_PIPE_WAVE", "4")
    if xcap:
        monkeypatch.setenv("SRWCR_XCAP", xcap)
    g, pb, Fn, Mn, params = problem("C5", 1, params_kind="large", orientation=orientation,
                                    bins=64 if orientation else None)
    st = g.stats()
    assert st["pipe_items1"] > 0 and st["pipe_items2"] > 0, st
    hp = torch.from_numpy(params.copy()).pin_memory()
    hg = torch.empty_like(hp).pin_memory()
    D1, _ = g.eval(hp, grad=hg)
    pt = hp.cuda()
    gt = torch.empty_like(pt)
    D2, _ = g.eval(pt, grad=gt)
    D3, g3 = g.eval(params)            # pageable host buffers: the same pipelined path
    g.close()
    assert rel(D1, D2) <= 2e-7 and rel(D3, D2) <= 2e-7
    assert rel_l2(hg.numpy(), gt.cpu().numpy()) <= 1e-5
    assert rel_l2(g3, gt.cpu().numpy()) <= 1e-5
    Do, go = O.eval_moments(pb, Fn, Mn, params)
    assert rel(D1, Do) <= D_TOL
    assert rel_l2(hg.numpy(), go) <= G_TOL
    assert comp(hg.numpy(), go) <= G_COMP, comp(hg.numpy(), go)


def test_debug_dump_statistics_match_oracle_moments():
    """SRWCR_DUMP_SQ re-runs the last combine with its S output on: the unshifted binned
    first moments S[r][a] and the binless Q[r] of the last pass 1 equal the oracle's
    moments (Eq 3 in moment form) to fp32-accumulation accuracy."""
    g, pb, Fn, Mn, params = problem("C3", 1, params_kind="small")
    D, _ = g.eval(params)
    N, Sx, Q = O.moments(pb, Fn, Mn, params)
    d = g.debug_dump("SQ")
    R, B = Sx.shape
    Sg, Qg = d[:R * B].reshape(R, B), d[R * B:R * B + R]
    assert np.abs(Sg - Sx).max() <= 2e-5 * np.abs(Sx).max()
    Qr = Q.sum(axis=1)          # the GPU keeps the binless per-region second moment
    assert np.abs(Qg - Qr).max() <= 2e-5 * np.abs(Qr).max()
    D2, _ = g.eval(params)     # the dump left the evaluation state as it was
    assert rel(D2, D) <= 2e-7
    g.close()


def test_timing_on_every_path():
    """srwcr_set_timing: per-pass CUDA events on the host-buffer path, the device-buffer
    (graph) path and inside srwcr_register."""
    torch = pytest.importorskip("torch")
    g, pb, Fn, Mn, params = problem("C3", 1, params_kind="small")
    g.set_timing(True)
    D1, _ = g.eval(params)
    st = g.stats()
    assert st["ms_pass1"] > 0 and st["ms_pass2"] > 0
    pt = torch.from_numpy(params).cuda()
    D2, _ = g.eval(pt, grad=torch.empty_like(pt))
    assert g.stats()["ms_pass1"] > 0 and rel(D2, D1) <= 2e-7
    x, rep = g.register(None, max_iter=2)
    assert rep["iterations"] >= 1
    g.close()
