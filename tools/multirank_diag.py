"""Diagnose the two-process caller-driven z-slab run: each rank's statistics partial (after
srwcr_eval_begin) compared with the same rank's partial computed alone in the parent, and
the combined D.  usage: python tools/multirank_diag.py"""
import os, sys, tempfile
sys.path.insert(0, os.getcwd())
sys.path.insert(0, os.path.join(os.getcwd(), "tests"))
import numpy as np
import torch
import torch.multiprocessing as mp
import test_gpu_multirank as T
import paper_1804_05061_b200 as S
import synth


def stats_of(rank, world):
    cfg = synth.config("C5", T.DIMS)
    F, M = synth.make_pair("C5", 1, cfg["dims"])
    g = S.Srwcr(F, M, cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"], nranks=world, rank=rank)
    params = synth.make_params(g.params_shape, "small", 1)
    out = [g.debug_dump("N").copy()]
    for _ in range(2):
        g.eval_begin(params)
        p, n = g.stats_buffer()
        out.append(T._d2h(p, n).copy())
        g.eval_end()
    g.close()
    return out


def rank_main(rank, world, port, td):
    import torch.distributed as dist
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    hs = stats_of(rank, world)
    np.save(os.path.join(td, f"n{rank}.npy"), hs[0])
    np.save(os.path.join(td, f"h{rank}.npy"), np.stack(hs[1:]))
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    ref = [stats_of(r, 2) for r in range(2)]
    for rep in range(4):
        with tempfile.TemporaryDirectory() as td:
            mp.start_processes(rank_main, args=(2, T._free_port(), td), nprocs=2, join=True, start_method="spawn")
            for r in range(2):
                h = np.load(os.path.join(td, f"h{r}.npy"))
                nn = np.load(os.path.join(td, f"n{r}.npy"))
                nb = int((nn != ref[r][0]).sum())
                bad = [int((h[k] != ref[r][k + 1]).sum()) for k in (0, 1)]
                mx = float(np.abs(h[0] - ref[r][1]).max())
                i = np.nonzero(h[0] != ref[r][1])[0][:3]
                print("rep", rep, "rank", r, "N mismatches", nb, "stats mismatches", bad, "max |diff|", mx,
                      "first", i.tolist(), h[0][i].tolist(), ref[r][1][i].tolist(), flush=True)
