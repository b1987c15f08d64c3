"""CPU-only checks of the product library and of the multi-rank host logic.

* libsrwcr.so builds for sm_100a, loads without a GPU, and exports every function
  declared in include/srwcr.h (no compute call is made here).
* srwcr_plan_slab (host-only) partitions the slices.
* The ALGEBRA of the z-slab decomposition used by nranks > 1 -- rank-partial bin
  statistics summed across ranks, then a rank-partial gradient summed across ranks --
  reproduces the single-process result: 2 gloo processes each running the ORACLE on its
  slab (no library context here).  The library's own nranks = 2 path runs as 2 processes
  on one GPU in tests/test_gpu_multirank.py (caller-driven exchange over gloo) and its
  slab kernels in tests/test_gpu_parity.py::test_slab_decomposition_on_one_gpu.
"""
import ctypes
import os
import re
import socket

import numpy as np
import pytest

import paper_1804_05061_b200 as S

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def lib():
    S.build()
    return S.lib()


def _declared_functions():
    src = open(os.path.join(ROOT, "include", "srwcr.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(srwcr_[a-z_0-9]+)\s*\(", src)))


def test_header_symbols_are_exported(lib):
    names = _declared_functions()
    assert len(names) >= 15
    so = ctypes.CDLL(S._LIB)
    for n in names:
        assert hasattr(so, n), f"{n} declared in include/srwcr.h but not exported"
    # the binding lists the same set
    assert set(S.EXPORTS) == set(names)


def test_library_is_sm100a():
    import subprocess
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", S.build()], capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_default_options_and_argument_errors(lib):
    opt = S._Options()
    assert lib.srwcr_default_options(ctypes.byref(opt)) == S.OK
    assert opt.struct_size == ctypes.sizeof(S._Options)
    assert (opt.nranks, opt.rank, opt.moment_shift, opt.use_graph) == (1, 0, 1, 1)
    assert opt.eps_mass == 1e-12 and opt.eps_sigma == 1e-6
    ctx = ctypes.c_void_p()
    dims = (ctypes.c_int64 * 3)(8, 8, 8)
    sp = (ctypes.c_double * 3)(1, 1, 1)
    sb = (ctypes.c_int32 * 3)(1, 1, 1)
    cs = (ctypes.c_double * 3)(4, 4, 4)
    # NULL fixed image -> EINVAL with a message naming it (no CUDA call is reached)
    st = lib.srwcr_create(ctypes.byref(ctx), None, None, dims, sp, 32, sb, cs, None)
    assert st == S.EINVAL
    assert b"fixed" in lib.srwcr_last_error(ctx)
    lib.srwcr_destroy(ctx)
    buf = np.zeros(512, np.float32)
    p = buf.ctypes.data_as(ctypes.c_void_p)
    for bad_bins in (1, 129):
        ctx = ctypes.c_void_p()
        assert lib.srwcr_create(ctypes.byref(ctx), p, p, dims, sp, bad_bins, sb, cs, None) == S.EINVAL
        assert b"intensity_bins" in lib.srwcr_last_error(ctx)
        lib.srwcr_destroy(ctx)
    # orientation must be 0 or 1
    opt.orientation = 2
    ctx = ctypes.c_void_p()
    assert lib.srwcr_create(ctypes.byref(ctx), p, p, dims, sp, 32, sb, cs, ctypes.byref(opt)) == S.EINVAL
    lib.srwcr_destroy(ctx)
    # the passes use 32-bit voxel offsets: >= 2^31 voxels is refused before any allocation
    big = (ctypes.c_int64 * 3)(2048, 2048, 512)
    ctx = ctypes.c_void_p()
    assert lib.srwcr_create(ctypes.byref(ctx), p, p, big, sp, 32, sb, cs, None) == S.EINVAL
    assert b"volume too large" in lib.srwcr_last_error(ctx)
    lib.srwcr_destroy(ctx)


@pytest.mark.parametrize("nz,P", [(320, 8), (128, 3), (7, 4), (1, 1), (5, 5)])
def test_plan_slab_partition(lib, nz, P):
    cover = []
    sizes = []
    for r in range(P):
        z0, z1 = S.plan_slab(nz, P, r)
        assert 0 <= z0 <= z1 <= nz
        cover.extend(range(z0, z1))
        sizes.append(z1 - z0)
    assert cover == list(range(nz))
    assert max(sizes) - min(sizes) <= 1
    with pytest.raises(S.SrwcrError):
        S.plan_slab(nz, P, P)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _rank_main(rank, world, port, q):
    import torch
    import torch.distributed as dist

    import oracle as O
    import synth

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.config("C3", (40, 36, 30))
        F, M = synth.make_pair("C3", 1, cfg["dims"])
        L = cfg["bins"] - 1
        pb = O.Problem(dims=cfg["dims"], L=L, delta=tuple(c / s for c, s in zip(cfg["control_mm"], cfg["spacing"])),
                       kcells=cfg["cells"], nthreads=1)
        Fn, Mn = O.normalize(F, L), O.normalize(M, L)
        params = synth.make_params(pb.params_shape, "small", 1)
        # the nccl unique id is broadcast from rank 0 exactly as bench.py does
        obj = [bytes(range(128)) if rank == 0 else None]
        dist.broadcast_object_list(obj, src=0)
        assert obj[0] == bytes(range(128))
        z0, z1 = S.plan_slab(cfg["dims"][2], world, rank)
        N, Sm, Q = (torch.from_numpy(t) for t in O.moments(pb, Fn, Mn, params, z0, z1))
        for t in (N, Sm, Q):
            dist.all_reduce(t)
        D, al, be, ga, reg, Z = O.combine(pb, N.numpy(), Sm.numpy(), Q.numpy())
        g = torch.from_numpy(O.grad_moments(pb, Fn, Mn, params, al, be, ga, Z, z0, z1))
        dist.all_reduce(g)
        if rank == 0:
            D1, g1 = O.eval_moments(pb, Fn, Mn, params)
            q.put((D, D1, float(np.linalg.norm(g.numpy() - g1) / np.linalg.norm(g1))))
    finally:
        dist.destroy_process_group()


def test_oracle_zslab_algebra_gloo_two_ranks():
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_rank_main, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    D, D1, gerr = q.get(timeout=10)
    assert abs(D - D1) <= 1e-12 * abs(D1)
    assert gerr <= 1e-12


def _halo_rank_main(rank, world, port, q):
    """The halo gradient exchange on the oracle's slab partials: the
    library's host-only layer plan decides what rank k sends to k + 1; after the exchange
    each rank keeps its owned layers, and the rank gradients must partition the full one."""
    import torch
    import torch.distributed as dist

    import oracle as O
    import synth

    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = synth.config("C3", (40, 36, 30))
        F, M = synth.make_pair("C3", 1, cfg["dims"])
        L = cfg["bins"] - 1
        delta = tuple(c / s for c, s in zip(cfg["control_mm"], cfg["spacing"]))
        pb = O.Problem(dims=cfg["dims"], L=L, delta=delta, kcells=cfg["cells"], nthreads=1)
        Fn, Mn = O.normalize(F, L), O.normalize(M, L)
        params = synth.make_params(pb.params_shape, "small", 1)
        nz, gz = cfg["dims"][2], pb.params_shape[1]
        cbz = [O.taps(z, delta[2])[0] for z in range(nz)]
        t0, t1, o0, o1, r1 = S.plan_layers(nz, world, rank, cbz, gz)
        z0, z1 = S.plan_slab(nz, world, rank)
        N, Sm, Q = (torch.from_numpy(t) for t in O.moments(pb, Fn, Mn, params, z0, z1))
        for t in (N, Sm, Q):
            dist.all_reduce(t)
        D, al, be, ga, reg, Z = O.combine(pb, N.numpy(), Sm.numpy(), Q.numpy())
        g = torch.from_numpy(O.grad_moments(pb, Fn, Mn, params, al, be, ga, Z, z0, z1))   # [ndim, Gz, Gy, Gx]
        # the partial is zero outside the touched layers (Eq 17 taps of slices z0 .. z1-1)
        assert not g[:, :t0].any() and not g[:, t1:].any()
        reqs = []
        if rank + 1 < world and t1 > o1:
            reqs.append(dist.isend(g[:, o1:t1].contiguous(), rank + 1))
        if rank > 0 and r1 > o0:
            buf = torch.empty_like(g[:, o0:r1])
            dist.recv(buf, rank - 1)
            g[:, o0:r1] += buf
        for r in reqs:
            r.wait()
        g[:, :o0] = 0
        g[:, o1:] = 0
        owned = torch.zeros(gz, dtype=torch.int64)
        owned[o0:o1] = 1
        dist.all_reduce(owned)
        gsum = g.clone()
        dist.all_reduce(gsum)
        if rank == 0:
            D1, g1 = O.eval_moments(pb, Fn, Mn, params)
            q.put((owned.tolist(), float(np.linalg.norm(gsum.numpy() - g1) / np.linalg.norm(g1))))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3])
def test_halo_gradient_exchange_plan_gloo(world):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_halo_rank_main, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=300)
        assert p.exitcode == 0
    owned, gerr = q.get(timeout=10)
    assert all(o == 1 for o in owned)   # the owned ranges partition the node layers
    assert gerr <= 1e-12


def test_plan_layers_properties():
    """Host-only layer plan: touched ranges follow the Eq 17 taps of the slab's slices, the
    owned ranges partition [0, Gz), and slabs thinner than the taps are refused."""
    import oracle as O
    nz, d = 96, 6.0
    cbz = [O.taps(z, d)[0] for z in range(nz)]
    gz = max(cbz) + 4
    for P in (1, 2, 3, 4):
        plans = [S.plan_layers(nz, P, k, cbz, gz) for k in range(P)]
        assert plans[0][2] == 0 and plans[-1][3] == gz
        for k, (t0, t1, o0, o1, r1) in enumerate(plans):
            z0, z1 = S.plan_slab(nz, P, k)
            assert (t0, t1) == (cbz[z0], min(cbz[z1 - 1] + 4, gz))
            assert o0 <= o1 and o0 <= r1 <= o1
            if k > 0:
                assert o0 == plans[k - 1][3] and r1 == max(o0, plans[k - 1][1])
    assert S.plan_layers(nz, 1, 0, cbz, gz) == (0, gz, 0, gz, 0)
    with pytest.raises(S.SrwcrError):
        S.plan_layers(nz, 5, 0, cbz, gz)    # 19-slice slabs: rank 0 reaches rank 2's layers
    with pytest.raises(S.SrwcrError):
        S.plan_layers(nz, 2, 0, cbz[::-1], gz)   # bases must not decrease
    with pytest.raises(S.SrwcrError):
        S.plan_layers(nz, 2, 2, cbz, gz)


def test_buffer_marshalling_rejects_wrong_params_and_outputs():
    """The binding hands raw pointers to the C ABI, which reads / writes nparams doubles:
    wrong dtypes or sizes, and non-contiguous outputs, must be refused before the call."""
    import numpy as np
    import pytest
    from paper_1804_05061_b200 import _ptr
    ok = np.zeros(12)
    assert _ptr(ok, 12, "params")[0] is not None
    with pytest.raises(ValueError):
        _ptr(np.zeros(12, dtype=np.float32), 12, "params")
    with pytest.raises(ValueError):
        _ptr(np.zeros(11), 12, "params")
    with pytest.raises(ValueError):
        _ptr(np.zeros((4, 6))[:, ::2], 12, "grad", out=True)
    p, keep = _ptr(np.zeros((4, 6))[:, ::2], 12, "params")   # inputs are copied contiguous
    assert keep.flags["C_CONTIGUOUS"]
    torch = pytest.importorskip("torch")
    with pytest.raises(ValueError):
        _ptr(torch.zeros(12, dtype=torch.float32), 12, "params")
    with pytest.raises(ValueError):
        _ptr(torch.zeros(4, 6, dtype=torch.float64)[:, ::2], 12, "grad", out=True)


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    """No CPU fallback: with the CUDA library absent the product path raises instead of
    computing anything (the oracle is test infrastructure, never a fallback)."""
    monkeypatch.setattr(S, "_lib", None)
    monkeypatch.setattr(S, "_LIB", str(tmp_path / "libsrwcr.so"))
    with pytest.raises(RuntimeError, match="missing"):
        S.lib()
    f = np.zeros((4, 8, 8), np.float32)
    with pytest.raises(RuntimeError, match="missing"):
        S.Srwcr(f, f, (1.0, 1.0, 1.0), 8, (1, 1, 1), (4.0, 4.0, 4.0))
