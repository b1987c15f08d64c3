"""GPU parity of the round-2 fast passes (srwcr_fast.cuh) against the fp64 oracle.

The fast passes evaluate every 3-D, moving-as-B configuration whose spatial x-cells are at
least 32 voxels wide (the benchmarked C5 and C3/C4 at their BASELINE sizes).  The reduced
stand-ins here keep the x-cell width -- and so the kernel variant (XV, interior/general
items) -- of the full-size run, and shrink y and z so that the oracle finishes in seconds.
Gates (BASELINE north_star): D relative error <= 1e-5, gradient relative L2 <= 1e-4, and
per component max |g - g_o| <= 1e-3 max |g_o|.
"""
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

D_TOL, G_TOL, G_COMP = 1e-5, 1e-4, 1e-3

# same x-cell width as the full-size config (C3: 32 -> XV 1; C4, C5: 64 -> XV 2)
FAST_DIMS = {"C2": None, "C3": (256, 66, 34), "C4": (512, 34, 130), "C5": (512, 66, 42)}


def _case(name, seed, phi, dims=None):
    import oracle as O
    import paper_1804_05061_b200 as S
    import synth
    cfg = synth.config(name, dims if dims is not None else FAST_DIMS[name])
    F, M = synth.make_pair(name, seed, cfg["dims"])
    L = cfg["bins"] - 1
    pb = O.Problem(dims=cfg["dims"], L=L, delta=tuple(c / s for c, s in zip(cfg["control_mm"], cfg["spacing"])),
                   kcells=cfg["cells"])
    g = S.Srwcr(F, M, cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"])
    params = synth.make_params(g.params_shape, phi, seed)
    return g, pb, O.normalize(F, L), O.normalize(M, L), params


def _check(D, grad, Do, go):
    rd = abs(D - Do) / abs(Do)
    rg = float(np.linalg.norm(grad - go) / np.linalg.norm(go))
    rc = float(np.abs(grad - go).max() / np.abs(go).max())
    assert rd <= D_TOL, rd
    assert rg <= G_TOL, rg
    assert rc <= G_COMP, rc
    return rd, rg, rc


@pytest.mark.parametrize("name", ["C2", "C3", "C4", "C5"])
@pytest.mark.parametrize("phi", ["zero", "small", "large"])
def test_fast_path_parity(name, phi):
    import oracle as O
    g, pb, Fn, Mn, params = _case(name, 1, phi)
    st = g.stats()
    assert st["fast_path"] == 1, "the configuration must run the fast passes"
    D, grad = g.eval(params)
    g.close()
    Do, go = O.eval_moments(pb, Fn, Mn, params)
    _check(D, grad, Do, go)


@pytest.mark.parametrize("name", ["C3", "C4", "C5"])
@pytest.mark.parametrize("seed", [2, 3])
def test_fast_path_parity_seeds(name, seed):
    import oracle as O
    g, pb, Fn, Mn, params = _case(name, seed, "small")
    D, grad = g.eval(params)
    g.close()
    Do, go = O.eval_moments(pb, Fn, Mn, params)
    _check(D, grad, Do, go)


def test_fast_path_is_deterministic():
    """int32 line tables, fixed-order cell folds and int64 global sums: two evaluations of
    the same inputs are bitwise identical (value and gradient), host and device buffers."""
    torch = pytest.importorskip("torch")
    g, pb, Fn, Mn, params = _case("C5", 1, "small")
    D1, g1 = g.eval(params)
    D2, g2 = g.eval(params)
    pt = torch.from_numpy(params).cuda()
    gt = torch.empty_like(pt)
    D3, _ = g.eval(pt, grad=gt)
    D4, _ = g.eval(pt, grad=gt)
    g.close()
    assert D1 == D2 == D3 == D4
    assert np.array_equal(g1, g2)
    assert np.array_equal(g1, gt.cpu().numpy())


def test_fast_path_agrees_with_round1_passes(monkeypatch):
    """The fast passes and the round-1 passes (SRWCR_NOFAST=1) evaluate the same method:
    both within the gates of each other."""
    g, pb, Fn, Mn, params = _case("C3", 1, "small")
    D1, g1 = g.eval(params)
    g.close()
    monkeypatch.setenv("SRWCR_NOFAST", "1")
    g2, *_ = _case("C3", 1, "small")
    assert g2.stats()["fast_path"] == 0
    D2, gr2 = g2.eval(params)
    g2.close()
    assert abs(D1 - D2) / abs(D2) <= D_TOL
    assert np.linalg.norm(g1 - gr2) / np.linalg.norm(gr2) <= G_TOL


def test_fast_path_c3_full_size():
    """C3 at its BASELINE size (256x256x128, 64 bins, delta (5,5,2)): the kernel variant the
    bench-like full-size run uses (XV 1, 32-voxel x-cells), all three Phi points."""
    import oracle as O
    for phi in ("zero", "small", "large"):
        g, pb, Fn, Mn, params = _case("C3", 1, phi, dims=(256, 256, 128))
        assert g.stats()["fast_path"] == 1
        D, grad = g.eval(params)
        g.close()
        Do, go = O.eval_moments(pb, Fn, Mn, params)
        _check(D, grad, Do, go)


def test_dynamic_bin_mismatch_report():
    """the dynamic moving bin n(m) = min(floor m, L-1) (Eq 5) decided in fp32 on
    the GPU vs fp64 in the oracle.  Mismatches can only occur where fp64 m lies within
    fp32 rounding of an integer; the count is reported (profiles/) and must be tiny."""
    import oracle as O
    g, pb, Fn, Mn, params = _case("C5", 1, "small")
    g.eval(params)
    mg = g.debug_dump("warped").reshape(pb.dims[2], pb.dims[1], pb.dims[0], 4)
    g.close()
    m_o, grad_o = O.warp(pb, Mn, params)
    L = pb.L
    m_g = np.abs(mg[..., 0])
    m_g = np.where(mg[..., 0] < 0, -1.0 - mg[..., 0], mg[..., 0])   # the exact-path flag (cleared after the fix)
    n_g = np.minimum(np.floor(m_g), L - 1)
    n_o = np.minimum(np.floor(m_o), L - 1)
    mism = int((n_g != n_o).sum())
    near = np.abs(m_o - np.round(m_o)) < 1e-4
    assert mism <= int(near.sum())                 # only next to an integer
    assert np.abs(m_g - m_o).max() < 1e-3           # fp32 sample of fp64 quality
    assert mism <= 1e-4 * m_o.size


@pytest.mark.parametrize("grad_exchange", [0, 1])
def test_fast_path_nccl_single_rank_graph(grad_exchange):
    """The library-driven z-slab exchange (int64 ncclAllReduce of the statistics and of the
    gradient -- or, grad_exchange = 1, the grouped ncclSend/Recv halo exchange and
    k_halo_finish -- captured into the per-rank CUDA graph with the kernels) on one rank:
    bitwise the result of the context without a communicator (both compute the same
    deterministic static counts), and bitwise reproducible across graph replays."""
    torch = pytest.importorskip("torch")
    import paper_1804_05061_b200 as S
    import synth
    g1, pb, Fn, Mn, params = _case("C5", 1, "small")
    pt = torch.from_numpy(params).cuda()
    gt1 = torch.empty_like(pt)
    D1, _ = g1.eval(pt, grad=gt1)
    cfg = synth.config("C5", FAST_DIMS["C5"])
    F, M = synth.make_pair("C5", 1, cfg["dims"])
    g2 = S.Srwcr(F, M, cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"], nranks=1, rank=0,
                 nccl_id=torch.cuda.nccl.unique_id(), grad_exchange=grad_exchange)
    assert g2.stats()["fast_path"] == 1
    gz = g2.params_shape[1]
    assert g2.grad_layers() == (0, gz, 0, gz, 0)
    if grad_exchange:
        with pytest.raises(S.SrwcrError):   # the in-library L-BFGS is replicated: it needs the all-reduce
            g2.register(None, max_iter=1)
    gt2 = torch.empty_like(pt)
    D2, _ = g2.eval(pt, grad=gt2)      # captured
    g2c = gt2.clone()
    D3, _ = g2.eval(pt, grad=gt2)      # replayed
    D4, g4 = g2.eval(params)           # host buffers with a communicator (not pipelined, not a graph)
    g1.close()
    g2.close()
    assert D3 == D2 and torch.equal(g2c, gt2)
    assert D2 == D1 and torch.equal(gt2, gt1)
    assert D4 == D1 and np.array_equal(g4, gt1.cpu().numpy())


@pytest.mark.parametrize("name", ["C3", "C5"])
def test_split_pass1_bitwise_equals_fused(name, monkeypatch):
    """Pass 1 split into its sample half (k_p1w: FFD, gathers, trilinear, exact flags -> MG
    and m) and its moment half (k_p1f MODE 2: m -> line tables) runs the same per-voxel
    arithmetic as the fused kernel: bitwise-equal statistics, D and gradient (one context;
    SRWCR_SPLIT, set at create to allocate the split's m array, is re-read at each launch)."""
    monkeypatch.setenv("SRWCR_SPLIT", "0")
    g, pb, Fn, Mn, params = _case(name, 1, "small")
    res = []
    for split in ("0", "1", "0"):
        monkeypatch.setenv("SRWCR_SPLIT", split)
        D, grad = g.eval(params)
        res.append((D, grad, g.debug_dump("SQ"), g.debug_dump("warped")))
    g.close()
    for r in res[1:]:
        assert r[0] == res[0][0]
        for k in (1, 2, 3):
            assert np.array_equal(r[k], res[0][k])


def test_checked_build_small_cases():
    """The library built with -DSRWCR_CHECK (device-side bounds checks of every shared-memory
    table index of the fast passes; a failed check traps) runs tools/sanitize_run.py: both
    orientations, round-1 and fast passes (XV 1 and 2, fused and split pass 1), bending,
    L-BFGS and field utilities.  (compute-sanitizer is closed on the GPU pool.)"""
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    lib = os.path.join(root, "build_variants", "libsrwcr_check.so")
    src = os.path.join(root, "paper_1804_05061_b200", "csrc", "srwcr.cu")
    if not os.path.exists(lib) or os.path.getmtime(lib) < max(
            os.path.getmtime(os.path.join(os.path.dirname(src), f)) for f in os.listdir(os.path.dirname(src))):
        os.makedirs(os.path.dirname(lib), exist_ok=True)
        import paper_1804_05061_b200 as S
        subprocess.check_call([os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc"), *S.NVCC_FLAGS, "-DSRWCR_CHECK",
                               "-o", lib, src, "-ldl"])
    env = dict(os.environ, SRWCR_LIB=lib)
    out = subprocess.run([sys.executable, os.path.join(root, "tools", "sanitize_run.py")], env=env,
                         capture_output=True, text=True, timeout=900)
    assert out.returncode == 0, out.stdout[-2000:] + out.stderr[-2000:]
    assert "sanitize_run: ok" in out.stdout


def test_contexts_are_bitwise_identical():
    """Two contexts created from the same inputs compute bitwise the same static counts N,
    moment shifts, statistics, D and gradient (the create-time reductions are fixed-order
    fp64 per box with int64 sums across boxes)."""
    res = []
    for _ in range(2):
        g, pb, Fn, Mn, params = _case("C5", 1, "small")
        D, grad = g.eval(params)
        res.append((D, grad, g.debug_dump("N"), g.debug_dump("SQ")))
        g.close()
    assert res[0][0] == res[1][0]
    for k in (1, 2, 3):
        assert np.array_equal(res[0][k], res[1][k])


def _custom(F, M, cells, control_vox, bins, phi, seed=1):
    import oracle as O
    import paper_1804_05061_b200 as S
    import synth
    dims = (F.shape[2], F.shape[1], F.shape[0])
    L = bins - 1
    pb = O.Problem(dims=dims, L=L, delta=tuple(float(c) for c in control_vox), kcells=cells)
    g = S.Srwcr(F, M, (1.0, 1.0, 1.0), bins, cells, tuple(float(c) for c in control_vox))
    params = synth.make_params(g.params_shape, phi, seed)
    return g, pb, O.normalize(F, L), O.normalize(M, L), params


@pytest.mark.parametrize("phi", ["small", "large"])
def test_fast_path_noisy_fixed_image_many_bins_per_line(phi):
    """Uniform-noise F with 128 bins: every 64-voxel line touches ~50 fixed bins, so the line
    fold runs its > 32-slot path and items carry ~128 slots; M a smooth ramp plus noise."""
    import oracle as O
    rng = np.random.default_rng(11)
    nz, ny, nx = 24, 20, 128
    F = rng.uniform(0, 1000, size=(nz, ny, nx)).astype(np.float32)
    z, y, x = np.meshgrid(np.arange(nz), np.arange(ny), np.arange(nx), indexing="ij")
    M = (3.0 * x + 2.0 * y + rng.normal(0, 20, size=x.shape)).astype(np.float32)
    g, pb, Fn, Mn, params = _custom(F, M, (2, 1, 1), (5, 5, 5), 128, phi)
    st = g.stats()
    assert st["fast_path"] == 1 and st["fast_slots"] > 34
    D, grad = g.eval(params)
    g.close()
    Do, go = O.eval_moments(pb, Fn, Mn, params)
    _check(D, grad, Do, go)


@pytest.mark.parametrize("dims,cells", [((100, 22, 9), (2, 2, 1)), ((70, 17, 31), (2, 1, 3)), ((96, 40, 5), (3, 2, 1))])
def test_fast_path_ragged_cells_and_thin_z(dims, cells):
    """Ragged x-cells (50, 35, 32 voxels: padding lanes in every line), odd y / z extents and
    a z-extent below the 4 control taps: the fast passes against the oracle at Phi large
    (samples leave the volume: the clamp variant)."""
    import oracle as O
    import synth
    cfg = synth.config("C5", dims)
    F, M = synth.make_pair("C5", 2, cfg["dims"])
    g, pb, Fn, Mn, params = _custom(F, M, cells, (5, 5, 5), 64, "large", seed=2)
    assert g.stats()["fast_path"] == 1
    D, grad = g.eval(params)
    g.close()
    Do, go = O.eval_moments(pb, Fn, Mn, params)
    _check(D, grad, Do, go)


@pytest.mark.parametrize("P", [2, 3])
def test_fast_path_slabs_on_one_gpu(P):
    """The fast passes under a z-slab decomposition whose boundaries cut spatial cells
    (42 slices, 8 z-cells, P = 2 or 3): each rank runs the single-GPU items restricted to its
    slab (items cut at the boundary), the caller sums the rank partials.  The int64 partials
    add exactly; items cut in z fold their fp32 column tables over fewer slices, so D and
    the gradient agree with one rank to fp32 rounding, and all stay within the oracle gates."""
    import ctypes
    import oracle as O
    import paper_1804_05061_b200 as S
    import synth
    from test_gpu_parity import _cudart
    g1, pb, Fn, Mn, params = _case("C5", 1, "small")
    D1, grad1 = g1.eval(params)
    cfg = synth.config("C5", FAST_DIMS["C5"])
    F, M = synth.make_pair("C5", 1, cfg["dims"])
    ranks = [S.Srwcr(F, M, cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"], nranks=P, rank=k)
             for k in range(P)]
    assert all(r.stats()["fast_path"] == 1 for r in ranks)
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
    Ds = {D for D, _ in outs}
    assert len(Ds) == 1   # every rank combines the same statistics
    D = outs[0][0]
    gsum = np.sum([gk for _, gk in outs], axis=0)
    for r in ranks + [g1]:
        r.close()
    assert abs(D - D1) / abs(D1) <= 1e-7
    assert np.linalg.norm(gsum - grad1) / np.linalg.norm(grad1) <= 1e-5
    Do, go = O.eval_moments(pb, Fn, Mn, params)
    _check(D, gsum, Do, go)


@pytest.mark.parametrize("phi,conc", [("small", "1"), ("large", "1"), ("small", "0")])
def test_pipelined_host_evaluation_bitwise(phi, conc, monkeypatch):
    """Host params / gradient buffers: the parts-pipelined evaluation (params uploaded in parts
    overlapped with pass 1 -- the parts concurrent on their own streams, or in one stream with
    SRWCR_PIPE_CONC=0 -- gradient layers converted and copied back while later pass-2 parts
    run; parts forced small with SRWCR_PIPE_WAVE / SRWCR_PIPE_Q) runs the same kernels on item
    ranges, with integer sums: bitwise the device-buffer evaluation."""
    torch = pytest.importorskip("torch")
    monkeypatch.setenv("SRWCR_PIPE_WAVE", "16")
    monkeypatch.setenv("SRWCR_PIPE_CONC", conc)
    monkeypatch.setenv("SRWCR_PIPE_Q", "8")
    monkeypatch.setenv("SRWCR_PIPE_Q2", "8")
    g, pb, Fn, Mn, params = _case("C5", 1, phi)
    st = g.stats()
    assert st["fast_path"] == 1
    D1, g1 = g.eval(params)                      # pageable host buffers: pipelined
    pt = torch.from_numpy(params).cuda()
    gt = torch.empty_like(pt)
    D2, _ = g.eval(pt, grad=gt)                  # device buffers: one launch per kernel (graph)
    D3, g3 = g.eval(params)
    hp = torch.from_numpy(params.copy()).pin_memory()
    hg = torch.empty_like(hp).pin_memory()
    D4, _ = g.eval(hp, grad=hg)                  # pinned host buffers: the pipelined parts as a graph
    g4 = hg.numpy().copy()
    D5, _ = g.eval(hp, grad=hg)                  # replayed
    g.close()
    assert D1 == D2 == D3 == D4 == D5
    assert np.array_equal(g1, gt.cpu().numpy()) and np.array_equal(g1, g3)
    assert np.array_equal(g1, g4) and np.array_equal(g1, hg.numpy())


def test_pipelined_concurrent_parts_list_overflow(monkeypatch):
    """The concurrent pass-2 parts give each part its own exact-path list; with the capacity
    forced to 1 (0 per part) every part with a deferred voxel overflows, the host sees it
    and redoes the evaluation without parts (the slab scan fixes the voxels): bitwise the
    device-buffer evaluation, which overflows and scans too."""
    torch = pytest.importorskip("torch")
    monkeypatch.setenv("SRWCR_PIPE_WAVE", "16")
    monkeypatch.setenv("SRWCR_PIPE_Q", "8")
    monkeypatch.setenv("SRWCR_PIPE_Q2", "8")
    monkeypatch.setenv("SRWCR_XCAP", "1")
    g, pb, Fn, Mn, params = _case("C5", 1, "large")
    assert g.stats()["exact_capacity"] == 1
    hp = torch.from_numpy(params.copy()).pin_memory()
    hg = torch.empty_like(hp).pin_memory()
    D1, _ = g.eval(hp, grad=hg)
    assert g.stats()["exact_voxels"] > 1
    pt = hp.cuda()
    gt = torch.empty_like(pt)
    D2, _ = g.eval(pt, grad=gt)
    g.close()
    assert D1 == D2 and np.array_equal(hg.numpy(), gt.cpu().numpy())
    _check(D1, hg.numpy(), *__import__("oracle").eval_moments(pb, Fn, Mn, params))


def test_value_only_evaluation():
    """srwcr_eval with grad = NULL (the L-BFGS line-search trials) runs pass 1 and the combine
    only: the same D, bitwise, as the value + gradient evaluation, on host and device buffers
    (pipelined and graph paths)."""
    torch = pytest.importorskip("torch")
    g, pb, Fn, Mn, params = _case("C5", 1, "small")
    D1, grad = g.eval(params)
    D2, none = g.eval(params, want_grad=False)
    pt = torch.from_numpy(params).cuda()
    D3, _ = g.eval(pt, want_grad=False)
    gt = torch.empty_like(pt)
    D4, _ = g.eval(pt, grad=gt)
    g.close()
    assert none is None
    assert D1 == D2 == D3 == D4
    assert np.array_equal(grad, gt.cpu().numpy())
