"""CUPTI timeline (torch.profiler) of srwcr_register iterations on C5: kernel / copy time
by name and the idle gaps."""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import synth, paper_1804_05061_b200 as S
cfg = synth.config("C5")
F, M = synth.make_pair("C5", 1, cfg["dims"])
g = S.Srwcr(torch.from_numpy(F).cuda(), torch.from_numpy(M).cuda(), cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"])
g.register(None, w_p=0.1, max_iter=3)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    x, rep = g.register(None, w_p=0.1, max_iter=10)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
from collections import defaultdict
agg = defaultdict(lambda: [0, 0.0])
for e in ev:
    a = agg[e.name[:60]]; a[0] += 1; a[1] += e.device_time_total if hasattr(e, "device_time_total") else e.cuda_time_total
tot = sum(v[1] for v in agg.values())
print(json.dumps({"report": {k: rep[k] for k in ("iterations", "evaluations", "gradient_evaluations")},
                  "kernels_us": {k: [v[0], round(v[1], 1)] for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]},
                  "total_device_us": tot}, indent=1))
prof.export_chrome_trace(sys.argv[1])
