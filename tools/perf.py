"""Quick perf harness: C5 (or another config) at full size, device-resident params,
per-pass CUDA-event times of the library.  Inputs are generated once and cached in
/tmp for the duration of one gpurun call.  Usage: python tools/perf.py [config] [steps]"""
import os, sys, time, json
import numpy as np
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth
import paper_1804_05061_b200 as S

name = sys.argv[1] if len(sys.argv) > 1 else "C5"
steps = int(sys.argv[2]) if len(sys.argv) > 2 else 50
phi = sys.argv[3] if len(sys.argv) > 3 else "small"
ori = int(sys.argv[4]) if len(sys.argv) > 4 else 0
bins_override = int(sys.argv[5]) if len(sys.argv) > 5 else None
cache = f"/tmp/srwcr_{name}.npz"
if os.path.exists(cache):
    d = np.load(cache); F, M = d["F"], d["M"]
else:
    F, M = synth.make_pair(name, 1); np.savez(cache, F=F, M=M)
cfg = synth.config(name)
g = S.Srwcr(torch.from_numpy(F).cuda(), torch.from_numpy(M).cuda(), cfg["spacing"], bins_override or cfg["bins"],
            cfg["cells"], cfg["control_mm"], orientation=ori)
if phi == "reg":   # an L-BFGS iterate (large, irregular displacements)
    x, _ = g.register(None, max_iter=20)
    np.save(f"/tmp/srwcr_{name}_reg.npy", x)
    p = torch.from_numpy(x).cuda()
elif phi == "regload":
    p = torch.from_numpy(np.load(f"/tmp/srwcr_{name}_reg.npy")).cuda()
else:
    p = torch.from_numpy(synth.make_params(g.params_shape, phi, 1)).cuda()
gr = torch.empty_like(p)
g.set_timing(True)
def ev():
    try:
        return g.eval(p, grad=gr)[0]
    except S.SrwcrError as e:   # ablation experiments may zero the statistics
        return float("nan")
for _ in range(3): ev()
t1 = []; t2 = []; tt = []
for _ in range(steps):
    D = ev(); s = g.stats(); t1.append(s["ms_pass1"]); t2.append(s["ms_pass2"]); tt.append(s["ms_total"])
s = g.stats()
env = {k: v for k, v in os.environ.items() if k.startswith("SRWCR_")}
print(json.dumps({"cfg": name, "phi": phi, "ori": ori, "env": env, "pass1": float(np.median(t1)), "pass2": float(np.median(t2)),
                  "total": float(np.median(tt)), "D": D, "W": s["warps_per_cta"], "S": s["slot_capacity"], "XV": s["voxels_per_lane"], "items": s["items"]}))
