"""SURVEY 8(d) measurement matrix: every config C1-C5 at the three Phi points (zero,
small U(-2,2), large smooth <= 15 voxels) and seeds 1-3, full sizes, device-resident
params, median of >= 200 evaluations after 20 warm-ups (CUDA events on the library
stream).  -> JSON (profiles/r1_perf_matrix.json)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synth
import paper_1804_05061_b200 as S

out = []
for name in ["C1", "C2", "C3", "C4", "C5"]:
    cfg = synth.config(name)
    nvox = int(np.prod(cfg["dims"]))
    for seed in (1, 2, 3):
        F, M = synth.make_pair(name, seed, cfg["dims"])
        g = S.Srwcr(torch.from_numpy(F).cuda(), torch.from_numpy(M).cuda(), cfg["spacing"], cfg["bins"], cfg["cells"],
                    cfg["control_mm"])
        st = torch.cuda.ExternalStream(g.stream_handle())
        for kind in ("zero", "small", "large"):
            p = torch.from_numpy(synth.make_params(g.params_shape, kind, seed)).cuda()
            gr = torch.empty_like(p)
            for _ in range(20):
                g.eval(p, grad=gr)
            ts = []
            for _ in range(200):
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record(st)
                D, _ = g.eval(p, grad=gr)
                e1.record(st)
                e1.synchronize()
                ts.append(e0.elapsed_time(e1))
            ms = float(np.median(ts))
            rec = {"config": name, "seed": seed, "phi": kind, "dims": list(cfg["dims"]), "ms_median": ms,
                   "ms_p10": float(np.percentile(ts, 10)), "ms_p90": float(np.percentile(ts, 90)),
                   "evals_per_s": 1e3 / ms, "gvoxel_per_s": nvox / ms / 1e6, "D": D,
                   "exact_voxels": g.stats()["exact_voxels"]}
            out.append(rec)
            print(json.dumps(rec), flush=True)
        g.close()
json.dump({"method": "median of 200 srwcr_eval calls after 20 warm-ups, CUDA events on the library stream, "
                     "device-resident params and gradient, full-size synthetic inputs (synth/)", "rows": out},
          open(sys.argv[1] if len(sys.argv) > 1 else "perf_matrix.json", "w"), indent=1)
