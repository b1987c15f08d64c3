"""The z-slab decomposition run by the LIBRARY in two processes: each process
is one rank (srwcr_options.nranks = 2, rank = k) on the one GPU of the box, the caller-driven
exchange (srwcr_eval_begin -> statistics sum over gloo -> srwcr_eval_end -> gradient sum
over gloo) replaces NCCL (nothing here makes one rank's kernels wait on the other's: the
exchange happens on the host between the library calls).

With slab boundaries on spatial z-cells, each rank runs exactly the work items of the
single-GPU decomposition that lie in its slab, the statistics are int64 fixed-point sums
(exact in fp64 after the conversion, so the caller's fp64 sum is exact too), and every
context computes bitwise the same static counts N, Z and moment shifts (k_static_N): D of
the two-rank run equals the single-rank D bitwise.  The gradient partials are converted to
fp64 before this caller-driven sum (the NCCL path sums the int64 partials instead), so the
gradient agrees to fp64 rounding.
"""
import os
import socket
import tempfile

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

# C5-shaped, 8 spatial z-cells of 6 slices: the 2-rank split (24 / 24) falls on a cell boundary
DIMS = (512, 34, 48)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_main(rank, world, port, out_dir, halo=False):
    import torch
    import torch.distributed as dist

    import paper_1804_05061_b200 as S
    import synth
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = synth.config("C5", DIMS)
    F, M = synth.make_pair("C5", 1, cfg["dims"])
    g = S.Srwcr(F, M, cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"], nranks=world, rank=rank)
    params = synth.make_params(g.params_shape, "small", 1)
    g.eval_begin(params)
    p, n = g.stats_buffer()
    h = torch.from_numpy(_d2h(p, n))
    dist.all_reduce(h, op=dist.ReduceOp.SUM)
    _h2d(p, h.numpy())
    D, grad = g.eval_end()
    gt = torch.from_numpy(np.ascontiguousarray(grad)).reshape(g.params_shape)
    if halo:
        # the halo exchange by the library's layer plan: the partial is
        # zero outside the touched layers; rank k sends [o1, t1) to k + 1 and adds rank
        # k - 1's [o0, r1); each rank then holds the gradient on its owned layers only
        t0, t1, o0, o1, r1 = g.grad_layers()
        cbz = g.debug_dump("ctrl_taps")[DIMS[0] + DIMS[1]:]   # the z part (Nx + Ny + Nz values)
        assert (t0, t1, o0, o1, r1) == S.plan_layers(DIMS[2], world, rank, cbz, g.params_shape[1])
        assert not gt[:, :t0].any() and not gt[:, t1:].any()
        if rank + 1 < world and t1 > o1:
            dist.send(gt[:, o1:t1].contiguous(), rank + 1)
        if rank > 0 and r1 > o0:
            buf = torch.empty_like(gt[:, o0:r1])
            dist.recv(buf, rank - 1)
            gt[:, o0:r1] += buf
        gt[:, :o0] = 0
        gt[:, o1:] = 0
        np.save(os.path.join(out_dir, f"own{rank}.npy"), np.array([o0, o1]))
    dist.all_reduce(gt, op=dist.ReduceOp.SUM)
    if rank == 0:
        np.save(os.path.join(out_dir, "grad.npy"), gt.numpy())
        np.save(os.path.join(out_dir, "D.npy"), np.array([D]))
    g.close()
    dist.destroy_process_group()


def _cudart():
    import ctypes
    import glob
    for cand in ["libcudart.so", *glob.glob("/usr/local/cuda/lib64/libcudart.so*")]:
        try:
            return ctypes.CDLL(cand)
        except OSError:
            continue
    raise RuntimeError("libcudart not found")


def _d2h(p, n):
    import ctypes
    h = np.empty(n, np.float64)
    assert _cudart().cudaMemcpy(h.ctypes.data_as(ctypes.c_void_p), ctypes.c_void_p(p), ctypes.c_size_t(8 * n), 2) == 0
    return h


def _h2d(p, h):
    import ctypes
    h = np.ascontiguousarray(h)
    assert _cudart().cudaMemcpy(ctypes.c_void_p(p), h.ctypes.data_as(ctypes.c_void_p), ctypes.c_size_t(h.nbytes), 1) == 0
    # a pageable H2D cudaMemcpy may return before its DMA has landed: complete it (the library's
    # srwcr_eval_end waits for the device too)
    assert _cudart().cudaDeviceSynchronize() == 0


@pytest.mark.parametrize("halo", [False, True])
def test_two_rank_library_gloo_exchange(halo):
    import torch.multiprocessing as mp

    import oracle as O
    import paper_1804_05061_b200 as S
    import synth
    cfg = synth.config("C5", DIMS)
    F, M = synth.make_pair("C5", 1, cfg["dims"])
    g1 = S.Srwcr(F, M, cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"])
    assert g1.stats()["fast_path"] == 1
    params = synth.make_params(g1.params_shape, "small", 1)
    D1, grad1 = g1.eval(params)
    g1.close()
    with tempfile.TemporaryDirectory() as td:
        mp.start_processes(_rank_main, args=(2, _free_port(), td, halo), nprocs=2, join=True, start_method="spawn")
        D2 = float(np.load(os.path.join(td, "D.npy"))[0])
        grad2 = np.load(os.path.join(td, "grad.npy")).reshape(grad1.shape)
        if halo:   # the owned ranges partition the node layers
            own = [np.load(os.path.join(td, f"own{r}.npy")) for r in range(2)]
            assert own[0][0] == 0 and own[0][1] == own[1][0] and own[1][1] == grad1.shape[1]
    assert D2 == D1, (D2, D1)
    assert np.linalg.norm(grad2 - grad1) / np.linalg.norm(grad1) <= 1e-14
    L = cfg["bins"] - 1
    pb = O.Problem(dims=cfg["dims"], L=L, delta=tuple(c / s for c, s in zip(cfg["control_mm"], cfg["spacing"])),
                   kcells=cfg["cells"])
    Do, go = O.eval_moments(pb, O.normalize(F, L), O.normalize(M, L), params)
    assert abs(D2 - Do) / abs(Do) <= 1e-5
    assert np.linalg.norm(grad2 - go) / np.linalg.norm(go) <= 1e-4
