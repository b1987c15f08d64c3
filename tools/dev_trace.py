"""CUPTI timeline (torch.profiler) of device-buffer evaluations (the graph path): kernel
durations and the gaps between consecutive kernels.  usage: python tools/dev_trace.py [config]"""
import os, sys, json
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import synth, paper_1804_05061_b200 as S
name = sys.argv[1] if len(sys.argv) > 1 else "C5"
cfg = synth.config(name)
F, M = synth.make_pair(name, 1, cfg["dims"])
g = S.Srwcr(torch.from_numpy(F).cuda(), torch.from_numpy(M).cuda(), cfg["spacing"], cfg["bins"], cfg["cells"], cfg["control_mm"])
p = torch.from_numpy(synth.make_params(g.params_shape, "small", 1)).cuda()
gr = torch.empty_like(p)
for _ in range(3): g.eval(p, grad=gr)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    for _ in range(3): g.eval(p, grad=gr)
    torch.cuda.synchronize()
ev = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
ev.sort(key=lambda e: e.time_range.start)
prev = None
for e in ev[-40:]:
    s, d = e.time_range.start, e.time_range.end - e.time_range.start
    gap = s - prev if prev is not None else 0
    print(f"{e.name[:50]:50s} dur {d:8.1f} us  gap {gap:6.1f} us")
    prev = e.time_range.end
